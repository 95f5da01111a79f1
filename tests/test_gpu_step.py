"""Parity of the CUDA step (through the C ABI) with the fp64 oracle, single GPU.

Gradients and updated parameters within relative Frobenius 1e-5 (fp32 mode) / 2e-2 (bf16 mode)
(BASELINE.json north star) globally, per layer, and PER TENSOR of every layer (the key bias, whose
exact gradient is 0 by pin P4, is held absolutely against the query bias gradient); counters exact
(SURVEY.md 8(c) O8)."""
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


def _run(sh, precision=LGA_FP32, schedule=LGA_LAYERED, chunk=0, causal=1, steps=1, lr=1e-3, wd=0.0, style="parity",
         flags=0):
    init = synth.init_params(sh, style=style)
    cfg = Config(layers=sh.layers, d_model=sh.d, heads=sh.heads, seq_len=sh.seq, micro_batch=sh.micro_batch,
                 n_micro=sh.n_micro, precision=precision, schedule=schedule, chunk=chunk, causal=causal, lr=lr,
                 weight_decay=wd, retain_grads=1, flags=flags)
    tr = Trainer(cfg, rank=0, world=1, device=0, init_params=init)
    batches = [synth.batch(sh, step=k) for k in range(steps)]
    losses = []
    for X, T in batches:
        xt = torch.from_numpy(X[0]).cuda()
        tt = torch.from_numpy(T[0]).cuda()
        losses.append(tr.step(xt, tt))
    out = dict(params=tr.params(), grads=tr.grads(), losses=losses, stats=tr.comm_stats()[0], stages=tr.layer_stage(),
               timing=tr.timing())
    tr.close()
    ref_params, ref_losses, ref_grads = oracle_run(sh, init, batches, causal=causal, lr=lr, wd=wd)
    if precision == LGA_BF16:   # reference of the per-tensor checks: gradients at the bf16 weight copy
        out["mp_params"], _, out["mp_grads"] = oracle_run(sh, init, batches, causal=causal, lr=lr, wd=wd,
                                                          param_round="bf16")
    return out, (ref_params, ref_losses, ref_grads, init)


C1 = synth.Shape(layers=2, d=64, heads=4, seq=32, micro_batch=2, n_micro=4)


@pytest.mark.parametrize("chunk", [0, 1, 2])
def test_fp32_c1_layered_parity(chunk):
    out, (rp, rl, rg, init) = _run(C1, chunk=chunk)
    assert rel(out["grads"], rg) < 1e-5, per_layer_rel(out["grads"], rg, C1.layers)
    assert_per_tensor(out["grads"], rg, C1.d, C1.layers, TENSOR_TOL["fp32"])
    assert_per_tensor(out["params"], rp, C1.d, C1.layers, TENSOR_TOL["fp32"], grads=False, init=init)
    assert max(per_layer_rel(out["grads"], rg, C1.layers)) < 1e-5
    assert rel(out["params"], rp) < 1e-5
    # the update itself, not just the parameters
    assert rel(out["params"] - init, rp - init) < 1e-4
    assert abs(out["losses"][0] - rl[0]) < 1e-6 * abs(rl[0])
    c = oc.comm_counters(oc.StepShape(layers=2, d=64, seq=32, micro_batch=2, n_micro=4), param_bytes=4, grad_bytes=4)
    for k, v in c.items():
        assert out["stats"][k] == v, k
    assert out["stages"] == [0, 0]


def test_fp32_standard_schedule_parity():
    out, (rp, rl, rg, _) = _run(C1, schedule=LGA_STANDARD)
    assert rel(out["grads"], rg) < 1e-5
    assert rel(out["params"], rp) < 1e-5


def test_fp32_multi_step_weight_decay_noncausal():
    sh = synth.Shape(layers=2, d=48, heads=3, seq=37, micro_batch=1, n_micro=3)   # ragged tiles, d_h = 16
    out, (rp, rl, rg, _) = _run(sh, causal=0, steps=3, wd=0.1)
    assert rel(out["grads"], rg) < 1e-5
    assert rel(out["params"], rp) < 1e-5
    np.testing.assert_allclose(out["losses"], rl, rtol=1e-5)


def test_fp32_deterministic():
    a, _ = _run(C1, chunk=2)
    b, _ = _run(C1, chunk=2)
    assert np.array_equal(a["grads"], b["grads"]) and np.array_equal(a["params"], b["params"])


BF = [synth.Shape(layers=2, d=256, heads=4, seq=128, micro_batch=2, n_micro=4),     # d_h = 64
      synth.Shape(layers=3, d=256, heads=2, seq=200, micro_batch=1, n_micro=4)]     # d_h = 128, ragged seq


@pytest.mark.parametrize("sh", BF, ids=["dh64", "dh128"])
@pytest.mark.parametrize("chunk", [0, 1])
def test_bf16_layered_parity(sh, chunk):
    """bf16 operands / fp32 accumulation: 2e-2 relative Frobenius (BASELINE.json north star)."""
    out, (rp, rl, rg, init) = _run(sh, precision=LGA_BF16, chunk=chunk)
    per = per_layer_rel(out["grads"], rg, sh.layers)
    assert rel(out["grads"], rg) < 2e-2 and max(per) < 2e-2, per
    assert rel(out["params"], rp) < 2e-2
    assert_per_tensor(out["grads"], out["mp_grads"], sh.d, sh.layers, TENSOR_TOL["bf16"])
    assert_per_tensor(out["params"], out["mp_params"], sh.d, sh.layers, TENSOR_TOL["bf16"], grads=False, init=init)
    assert abs(out["losses"][0] - rl[0]) < 1e-2 * abs(rl[0])


# ---------------------------------------------------------------- full-size launch configurations
# The bench configs' per-layer shapes exactly (d, heads, s, b; chunk = N so one launch covers all
# micro-batches, as bench.py times it) with L and N small enough for the fp64 oracle (seconds).
FULL = [synth.Shape(layers=2, d=2048, heads=16, seq=2048, micro_batch=1, n_micro=2),     # 1.3B layer (C3)
        synth.Shape(layers=1, d=768, heads=12, seq=1024, micro_batch=4, n_micro=2),       # GPT-2-small layer (C2)
        synth.Shape(layers=1, d=4096, heads=32, seq=2048, micro_batch=1, n_micro=2),      # ~10B layer (C4)
        # C3 layer with 4 micro-batches in one launch: M = 8192 rows, so every GEMM of the layer takes the
        # n-fastest raster the bench's M = 32768 launches take (as many m-blocks as n-blocks or more)
        synth.Shape(layers=1, d=2048, heads=16, seq=2048, micro_batch=1, n_micro=4)]


@pytest.mark.parametrize("sh", FULL, ids=["c3_layer", "c2_layer", "c4_layer", "c3_layer_n4"])
def test_bf16_full_width_parity(sh):
    out, (rp, rl, rg, init) = _run(sh, precision=LGA_BF16, style="train")
    per = per_layer_rel(out["grads"], rg, sh.layers)
    assert max(per) < 2e-2 and rel(out["grads"], rg) < 2e-2, per
    # the update itself: AdamW at t = 1 is lr sign(g) where |g| >> eps, so elements whose gradient is at the
    # rounding level flip sign and the update is ill-conditioned; the parameters are the quantity the bar binds
    assert rel(out["params"] - init, rp - init) < 1e-1
    assert rel(out["params"], rp) < 2e-2
    assert abs(out["losses"][0] - rl[0]) < 1e-3 * abs(rl[0])
    assert_per_tensor(out["grads"], out["mp_grads"], sh.d, sh.layers, TENSOR_TOL["bf16"])
    assert_per_tensor(out["params"], out["mp_params"], sh.d, sh.layers, TENSOR_TOL["bf16"], grads=False, init=init)


@pytest.mark.parametrize("d,heads,seq", [(1024, 8, 96), (2048, 16, 80), (4096, 32, 64)], ids=["d1024", "d2048", "d4096"])
def test_fp32_wide_parity_per_tensor(d, heads, seq):
    """fp32 mode at the configs' widths: the fused LayerNorm backward (d = 1024, 2048: 4 / 8 columns per lane),
    the warp-per-row LayerNorm kernels up to 32 column groups (d = 4096) and the wide bias column sums are
    held to 1e-5 per tensor -- the bf16 tolerance alone cannot see a wrong LayerNorm gamma / beta gradient."""
    sh = synth.Shape(layers=1, d=d, heads=heads, seq=seq, micro_batch=1, n_micro=2)
    out, (rp, rl, rg, init) = _run(sh)
    assert_per_tensor(out["grads"], rg, sh.d, sh.layers, TENSOR_TOL["fp32"])
    assert_per_tensor(out["params"], rp, sh.d, sh.layers, TENSOR_TOL["fp32"], grads=False, init=init)
    assert abs(out["losses"][0] - rl[0]) < 1e-6 * abs(rl[0])


def test_bf16_single_position_degenerate():
    """s = 1: softmax over one key is exactly 1, so dL/dW_Q, dL/dW_K, dL/db_Q, dL/db_K vanish (pin P3);
    on the GPU they are rounding-level only, while the value-path gradients match the oracle."""
    sh = synth.Shape(layers=1, d=128, heads=2, seq=1, micro_batch=8, n_micro=2)
    out, (rp, rl, rg, _) = _run(sh, precision=LGA_BF16)
    from oracle import model as om
    g = om.unpack(out["grads"].astype(np.float64), sh.d)
    r = om.unpack(rg, sh.d)
    d = sh.d
    qk = np.abs(g["Wqkv"][:, :2 * d]).max()
    assert qk < 1e-3 * np.abs(r["Wqkv"][:, 2 * d:]).max()
    assert rel(g["Wqkv"][:, 2 * d:], r["Wqkv"][:, 2 * d:]) < 2e-2
    assert rel(out["grads"], rg) < 2e-2


def test_fp32_single_microbatch_and_wide_batch():
    for sh in (synth.Shape(layers=1, d=64, heads=2, seq=16, micro_batch=1, n_micro=1),
               synth.Shape(layers=1, d=32, heads=1, seq=8, micro_batch=9, n_micro=2)):
        out, (rp, rl, rg, _) = _run(sh)
        assert rel(out["grads"], rg) < 1e-5 and rel(out["params"], rp) < 1e-5


def test_bf16_layered_equals_standard_on_gpu():
    """Property at any size: the two schedules compute the same gradient."""
    sh = synth.Shape(layers=2, d=256, heads=2, seq=256, micro_batch=1, n_micro=4)
    a, _ = _run(sh, precision=LGA_BF16, schedule=LGA_LAYERED)
    b, _ = _run(sh, precision=LGA_BF16, schedule=LGA_STANDARD)
    assert rel(a["grads"], b["grads"]) < 1e-2
    # and the step counters differ exactly as the closed forms say (D = 1: no collectives)
    assert a["stats"]["fwd_units"] == b["stats"]["fwd_units"] == 8


NO_RECOMPUTE, KEEP_PARAMS = 0x10, 0x8


@pytest.mark.parametrize("chunk", [0, 2])
def test_fp32_no_recompute_parity(chunk):
    """N2c: intermediates kept per layer for all micro-batches, no forward recompute -- same result,
    recompute_units = 0."""
    out, (rp, rl, rg, init) = _run(C1, chunk=chunk, steps=2, flags=NO_RECOMPUTE)
    assert rel(out["grads"], rg) < 1e-5 and rel(out["params"], rp) < 1e-5
    assert out["stats"]["recompute_units"] == 0 and out["stats"]["bwd_units"] == C1.n_micro * C1.layers


def test_bf16_no_recompute_parity_and_flags_without_dp():
    sh = synth.Shape(layers=2, d=256, heads=2, seq=128, micro_batch=1, n_micro=4)
    out, (rp, rl, rg, _) = _run(sh, precision=LGA_BF16, flags=NO_RECOMPUTE | KEEP_PARAMS)
    assert rel(out["grads"], rg) < 2e-2 and rel(out["params"], rp) < 2e-2
    assert_per_tensor(out["grads"], out["mp_grads"], sh.d, sh.layers, TENSOR_TOL["bf16"])
    assert out["stats"]["ag_calls"] == 0 and out["stats"]["recompute_units"] == 0


def test_variant_flags_rejected_with_standard():
    from paper_2106_02679_b200._abi import LgaError
    with pytest.raises(LgaError):
        _run(C1, schedule=LGA_STANDARD, flags=NO_RECOMPUTE)


def _steps(sh, flags, precision, n, swap_x_at=None, alternate=False):
    init = synth.init_params(sh, style="parity")
    cfg = Config(layers=sh.layers, d_model=sh.d, heads=sh.heads, seq_len=sh.seq, micro_batch=sh.micro_batch,
                 n_micro=sh.n_micro, precision=precision, lr=1e-3, retain_grads=1, flags=flags)
    tr = Trainer(cfg, rank=0, world=1, device=0, init_params=init)
    X, T = synth.batch(sh, step=0)
    xs = [torch.from_numpy(X[0]).cuda(), torch.from_numpy(X[0]).cuda()]
    t = torch.from_numpy(T[0]).cuda()
    losses = []
    for k in range(n):
        x = xs[1] if (swap_x_at is not None and k >= swap_x_at) else xs[0]
        if alternate:
            x = xs[k % 2]
        losses.append(tr.step(x, t))
    out = dict(params=tr.params(), losses=losses, stats=tr.comm_stats()[0], timing=tr.timing())
    tr.close()
    return out


def test_graph_cache_for_double_buffered_inputs():
    """A loader alternating two input buffers: two captures (steps 2 and 3), then replays; same bits as eager."""
    sh = synth.Shape(layers=2, d=256, heads=2, seq=128, micro_batch=1, n_micro=4)
    eager = _steps(sh, 0x2, LGA_BF16, 6, alternate=True)
    graph = _steps(sh, 0, LGA_BF16, 6, alternate=True)
    assert np.array_equal(eager["params"], graph["params"]) and eager["losses"] == graph["losses"]
    assert graph["timing"]["graph_captures"] == 2 and eager["timing"]["graph_captures"] == 0


@pytest.mark.parametrize("precision", [LGA_FP32, LGA_BF16])
def test_cuda_graph_replay_is_bitwise_eager(precision):
    """The step graph (captured at the 2nd call, re-captured when the input pointer changes) replays
    exactly the eager step: same parameters bit for bit, same losses and counters."""
    sh = C1 if precision == LGA_FP32 else synth.Shape(layers=2, d=256, heads=2, seq=128, micro_batch=1, n_micro=4)
    eager = _steps(sh, 0x2, precision, 4)
    graph = _steps(sh, 0, precision, 4, swap_x_at=3)
    assert np.array_equal(eager["params"], graph["params"])
    assert eager["losses"] == graph["losses"]
    assert eager["stats"] == graph["stats"]
    assert graph["timing"]["kernel_launches"] == eager["timing"]["kernel_launches"] > 0


def test_bf16_d1024_parity():
    """d = 1024 (d_h = 128): the fused LayerNorm backward with 4 columns per lane, ragged row groups."""
    sh = synth.Shape(layers=2, d=1024, heads=8, seq=130, micro_batch=1, n_micro=2)
    out, (rp, rl, rg, _) = _run(sh, precision=LGA_BF16)
    assert rel(out["grads"], rg) < 2e-2 and rel(out["params"], rp) < 2e-2
    assert_per_tensor(out["grads"], out["mp_grads"], sh.d, sh.layers, TENSOR_TOL["bf16"])


@pytest.mark.parametrize("precision", [LGA_FP32, LGA_BF16])
def test_step_host_equals_step(precision):
    """lga_step_host (x copied per micro-batch, layer 0 launched per micro-batch as each copy lands, target
    copied on the side) computes exactly what lga_step computes from device inputs."""
    sh = C1 if precision == LGA_FP32 else synth.Shape(layers=2, d=256, heads=2, seq=128, micro_batch=1, n_micro=4)
    init = synth.init_params(sh, style="parity")
    outs = []
    for host in (False, True):
        cfg = Config(layers=sh.layers, d_model=sh.d, heads=sh.heads, seq_len=sh.seq, micro_batch=sh.micro_batch,
                     n_micro=sh.n_micro, precision=precision, lr=1e-3, retain_grads=1)
        tr = Trainer(cfg, rank=0, world=1, device=0, init_params=init)
        losses = []
        for k in range(2):
            X, T = synth.batch(sh, step=k)
            if host:
                losses.append(tr.step_host(np.ascontiguousarray(X[0]), np.ascontiguousarray(T[0])))
            else:
                losses.append(tr.step(torch.from_numpy(X[0]).cuda(), torch.from_numpy(T[0]).cuda()))
        outs.append((tr.params(), losses, tr.comm_stats()[0]))
        tr.close()
    assert np.array_equal(outs[0][0], outs[1][0])
    assert outs[0][1] == outs[1][1] and outs[0][2] == outs[1][2]


@pytest.mark.parametrize("precision", [LGA_FP32, LGA_BF16])
def test_checkpoint_resume_is_bitwise(precision):
    """lga_save_state after step 2, a fresh handle, lga_load_state, step 3: the same parameters and loss bit for bit
    as three uninterrupted steps (the AdamW step t travels with the state; flag epochs stay per handle); a state
    of another configuration is refused."""
    sh = C1 if precision == LGA_FP32 else synth.Shape(layers=2, d=256, heads=2, seq=128, micro_batch=1, n_micro=4)
    init = synth.init_params(sh, style="parity")
    cfg = Config(layers=sh.layers, d_model=sh.d, heads=sh.heads, seq_len=sh.seq, micro_batch=sh.micro_batch,
                 n_micro=sh.n_micro, precision=precision, lr=1e-3, weight_decay=0.1, retain_grads=1)
    batches = [synth.batch(sh, step=k) for k in range(3)]
    dev = [(torch.from_numpy(X[0]).cuda(), torch.from_numpy(T[0]).cuda()) for X, T in batches]
    a = Trainer(cfg, rank=0, world=1, device=0, init_params=init)
    la = [a.step(x, t) for x, t in dev]
    pa = a.params()
    a.close()
    b = Trainer(cfg, rank=0, world=1, device=0, init_params=init)
    lb = [b.step(x, t) for x, t in dev[:2]]
    state = b.save_state()
    b.close()
    other = synth.init_params(sh, seed=99, style="parity")   # the loaded state must win over the init
    c = Trainer(cfg, rank=0, world=1, device=0, init_params=other)
    c.load_state(state)
    lb.append(c.step(*dev[2]))
    pc = c.params()
    c.close()
    assert lb == la and np.array_equal(pa, pc)
    from paper_2106_02679_b200._abi import LgaError
    cfg2 = Config(**{**cfg.__dict__, "layers": sh.layers * 2})
    d2 = Trainer(cfg2, rank=0, world=1, device=0, init_params=np.concatenate([init, init]))
    with pytest.raises(LgaError):
        d2.load_state(state)
    d2.close()
