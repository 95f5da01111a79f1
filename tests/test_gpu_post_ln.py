"""N4: the post-LN layer of the original encoder (reading A-16) through the C ABI against the fp64
oracle's ``layer_forward_post`` / ``layer_backward_post`` (pinned in test_oracle_model.py against torch
autograd and central differences).  Same bars as the pre-LN path: fp32 1e-5, bf16 2e-2, counters exact
and equal to the pre-LN ones (the flag changes the layer, not the schedule)."""
import numpy as np
import pytest

import synth
from gpu_util import TENSOR_TOL, assert_per_tensor, oracle_run, per_layer_rel, rel
from oracle import counters as oc

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2106_02679_b200 import LGA_BF16, LGA_FP32, LGA_LAYERED, LGA_STANDARD, Config, Trainer  # noqa: E402
from paper_2106_02679_b200._abi import LGA_FLAG_NO_GRAPH, LGA_FLAG_NO_RECOMPUTE, LGA_FLAG_POST_LN  # noqa: E402


def _run(sh, precision=LGA_FP32, schedule=LGA_LAYERED, chunk=0, causal=0, steps=1, flags=0):
    init = synth.init_params(sh, style="parity")
    cfg = Config(layers=sh.layers, d_model=sh.d, heads=sh.heads, seq_len=sh.seq, micro_batch=sh.micro_batch,
                 n_micro=sh.n_micro, precision=precision, schedule=schedule, chunk=chunk, causal=causal, lr=1e-3,
                 retain_grads=1, flags=flags | LGA_FLAG_POST_LN)
    tr = Trainer(cfg, rank=0, world=1, device=0, init_params=init)
    batches = [synth.batch(sh, step=k) for k in range(steps)]
    losses = [tr.step(torch.from_numpy(X[0]).cuda(), torch.from_numpy(T[0]).cuda()) for X, T in batches]
    out = dict(params=tr.params(), grads=tr.grads(), losses=losses, stats=tr.comm_stats()[0])
    tr.close()
    ref = oracle_run(sh, init, batches, causal=causal, post_ln=True)
    if precision == LGA_BF16:   # reference of the per-tensor checks: gradients at the bf16 weight copy
        out["mp_params"], _, out["mp_grads"] = oracle_run(sh, init, batches, causal=causal, post_ln=True,
                                                          param_round="bf16")
    return out, ref, init


def _check(sh, out, ref, init, tol, elem, no_recompute=False):
    rp, rl, rg = ref
    assert max(per_layer_rel(out["grads"], rg, sh.layers)) < tol, per_layer_rel(out["grads"], rg, sh.layers)
    assert rel(out["params"], rp) < tol
    mg, mp = out.get("mp_grads", rg), out.get("mp_params", rp)   # bf16: against the 16-bit-weight oracle
    assert_per_tensor(out["grads"], mg, sh.d, sh.layers, TENSOR_TOL["fp32" if tol <= 1e-5 else "bf16"])
    assert_per_tensor(out["params"], mp, sh.d, sh.layers, TENSOR_TOL["fp32" if tol <= 1e-5 else "bf16"], grads=False,
                      init=init)
    # the update itself (AdamW at t = 1 is lr sign(g) where |g| >> eps: elements with a rounding-level gradient
    # flip sign, so the update's relative error is set by how many gradients sit near 0, not by the arithmetic)
    assert rel(out["params"] - init, rp - init) < (1e-4 if tol <= 1e-5 else 1e-1)
    np.testing.assert_allclose(out["losses"], rl, rtol=max(tol, 1e-6))
    c = oc.comm_counters(oc.StepShape(layers=sh.layers, d=sh.d, seq=sh.seq, micro_batch=sh.micro_batch,
                                      n_micro=sh.n_micro), param_bytes=elem, grad_bytes=elem, no_recompute=no_recompute)
    for k, v in c.items():
        assert out["stats"][k] == v, k


C1 = synth.Shape(layers=2, d=64, heads=4, seq=32, micro_batch=2, n_micro=4)


@pytest.mark.parametrize("causal", [0, 1])
@pytest.mark.parametrize("chunk", [0, 2])
def test_fp32_post_ln_layered_parity(causal, chunk):
    out, ref, init = _run(C1, chunk=chunk, causal=causal, steps=2)
    _check(C1, out, ref, init, 1e-5, 4)


def test_fp32_post_ln_standard_and_no_recompute():
    for kw in (dict(schedule=LGA_STANDARD), dict(flags=LGA_FLAG_NO_RECOMPUTE)):
        out, ref, init = _run(C1, **kw)
        _check(C1, out, ref, init, 1e-5, 4, no_recompute="flags" in kw)


def test_fp32_post_ln_ragged():
    sh = synth.Shape(layers=2, d=48, heads=3, seq=37, micro_batch=1, n_micro=3)
    out, ref, init = _run(sh)
    _check(sh, out, ref, init, 1e-5, 4)


@pytest.mark.parametrize("heads", [4, 2], ids=["dh64", "dh128"])
def test_bf16_post_ln_parity(heads):
    sh = synth.Shape(layers=2, d=256, heads=heads, seq=128, micro_batch=2, n_micro=4)
    out, ref, init = _run(sh, precision=LGA_BF16, steps=2)
    _check(sh, out, ref, init, 2e-2, 2)


def test_bf16_post_ln_x32_layer():
    """One X_32 layer (d = 1024, 16 heads, s = 512, bidirectional): the shape bench.py --post-ln times."""
    sh = synth.Shape(layers=1, d=1024, heads=16, seq=512, micro_batch=1, n_micro=2)
    out, ref, init = _run(sh, precision=LGA_BF16)
    _check(sh, out, ref, init, 2e-2, 2)


def test_bf16_post_ln_graph_replay_is_bitwise_eager():
    sh = synth.Shape(layers=2, d=256, heads=4, seq=128, micro_batch=2, n_micro=2)
    res = []
    for flags in (0, LGA_FLAG_NO_GRAPH):
        init = synth.init_params(sh, style="parity")
        cfg = Config(layers=sh.layers, d_model=sh.d, heads=sh.heads, seq_len=sh.seq, micro_batch=sh.micro_batch,
                     n_micro=sh.n_micro, precision=LGA_BF16, causal=0, lr=1e-3, retain_grads=1,
                     flags=flags | LGA_FLAG_POST_LN)
        tr = Trainer(cfg, rank=0, world=1, device=0, init_params=init)
        X, T = synth.batch(sh, step=0)
        x, t = torch.from_numpy(X[0]).cuda(), torch.from_numpy(T[0]).cuda()
        losses = [tr.step(x, t) for _ in range(3)]
        res.append((losses, tr.params()))
        tr.close()
    assert res[0][0] == res[1][0]
    np.testing.assert_array_equal(res[0][1], res[1][1])
