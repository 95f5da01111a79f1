"""Multi-rank parity and exact counters (one process per rank, torchrun): ZeRO-partitioned data
parallelism (D = 2, 4) and the modular pipeline (P = 2, D x P = 4), against the fp64 oracle.

With fewer GPUs than ranks, the ranks share the visible GPUs (rank r on device r mod #GPUs): every data
path except the NCCL baseline runs over CUDA IPC peer memory, which works between processes on one GPU
(the ranks' kernels then run time-sliced), so a one-GPU box runs these tests too.  Only the NCCL
baseline (LGA_FLAG_NCCL_DP: NCCL refuses two ranks on one device) needs one GPU per rank."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import synth
from gpu_util import TENSOR_TOL, assert_per_tensor, oracle_run, per_layer_rel, rel
from oracle import counters as oc

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]
torch = pytest.importorskip("torch")
NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0
HERE = os.path.dirname(os.path.abspath(__file__))
_port = [29611]


def _launch(tmp_path, sh, precision=0, schedule=0, chunk=0, steps=1, flags=0, env=None, resume_at=0):
    world = sh.dp * sh.pp
    if NGPU < 1:
        pytest.skip("needs a GPU")
    if NGPU < world and (flags & NCCL_DP):
        pytest.skip(f"the NCCL baseline needs {world} GPUs (one per rank), have {NGPU}")
    _port[0] += 1
    shape = json.dumps(dict(layers=sh.layers, d=sh.d, heads=sh.heads, seq=sh.seq, micro_batch=sh.micro_batch,
                            n_micro=sh.n_micro, dp=sh.dp, pp=sh.pp))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={_port[0]}", os.path.join(HERE, "dist_worker.py"),
           "--out", str(tmp_path), "--shape", shape, "--precision", str(precision), "--schedule", str(schedule),
           "--chunk", str(chunk), "--steps", str(steps), "--flags", str(flags), "--resume-at", str(resume_at)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env={**os.environ, **(env or {})})
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return [dict(np.load(os.path.join(tmp_path, f"rank{k}.npz"))) for k in range(world)]


# LGA_FLAG_* variant bits (include/lga.h) -> oracle.counters keyword arguments
KEEP, NORECOMP, UNPART, CONTIG, NCCL_DP, POST_LN = 0x8, 0x10, 0x20, 0x40, 0x80, 0x100


def _variant(flags):
    return dict(keep_params=bool(flags & KEEP), no_recompute=bool(flags & NORECOMP),
                unpartitioned=bool(flags & UNPART), pipeline="contiguous" if flags & CONTIG else "modular")


def _check(outs, sh, tol, steps=1, schedule="layered", elem=4, flags=0):
    batches = [synth.batch(sh, step=k) for k in range(steps)]
    init = synth.init_params(sh, style="parity")
    rp, rl, rg = oracle_run(sh, init, batches, lr=1e-3, post_ln=bool(flags & POST_LN))
    mp, mg = rp, rg   # bf16: the per-tensor checks use gradients at the 16-bit weight copy
    if elem == 2:
        mp, _, mg = oracle_run(sh, init, batches, lr=1e-3, post_ln=bool(flags & POST_LN), param_round="bf16")
    pl = sh.d * sh.d * 12 + 13 * sh.d
    for o in outs:
        stage = int(o["stage"])
        var = _variant(flags)
        layers = oc.local_layers(stage, sh.layers, sh.pp, var["pipeline"])
        sel = np.concatenate([np.arange(i * pl, (i + 1) * pl) for i in layers])
        g, p = o["grads"], o["params"]
        assert rel(g, rg[sel]) < tol, (stage, per_layer_rel(g, rg[sel], len(layers)))
        assert rel(p, rp[sel]) < tol
        assert_per_tensor(g, mg[sel], sh.d, len(layers), TENSOR_TOL["fp32" if tol <= 1e-5 else "bf16"])
        assert_per_tensor(p, mp[sel], sh.d, len(layers), TENSOR_TOL["fp32" if tol <= 1e-5 else "bf16"], grads=False,
                          init=init[sel])
        np.testing.assert_allclose(o["losses"], rl, rtol=max(tol, 1e-6))
        assert list(o["stages"]) == [oc.stage_of_layer(i, sh.pp, sh.layers, var["pipeline"]) for i in range(sh.layers)]
        last = json.loads(str(o["last"]))
        ref = oc.comm_counters(oc.StepShape(layers=sh.layers, d=sh.d, seq=sh.seq, micro_batch=sh.micro_batch,
                                            n_micro=sh.n_micro, dp=sh.dp, pp=sh.pp),
                               stage=stage, schedule=schedule, param_bytes=elem, grad_bytes=elem, **var)
        for k, v in ref.items():
            assert last[k] == v, (k, last[k], v, stage)


@pytest.mark.parametrize("dp", [2, 4])
def test_dp_fp32_layered(tmp_path, dp):
    sh = synth.Shape(layers=4, d=64, heads=4, seq=32, micro_batch=2, n_micro=4, dp=dp)
    _check(_launch(tmp_path, sh), sh, 1e-5)


def test_dp2_fp32_standard(tmp_path):
    sh = synth.Shape(layers=2, d=64, heads=4, seq=32, micro_batch=2, n_micro=3, dp=2)
    _check(_launch(tmp_path, sh, schedule=1), sh, 1e-5, schedule="standard")


def test_dp2_fp32_two_steps_chunked(tmp_path):
    sh = synth.Shape(layers=2, d=64, heads=4, seq=32, micro_batch=2, n_micro=4, dp=2)
    _check(_launch(tmp_path, sh, chunk=2, steps=2), sh, 1e-5, steps=2)


def test_pp2_fp32_modular_pipeline(tmp_path):
    sh = synth.Shape(layers=4, d=64, heads=4, seq=32, micro_batch=2, n_micro=4, dp=1, pp=2)
    _check(_launch(tmp_path, sh), sh, 1e-5)


def test_pp2_dp2_fp32(tmp_path):
    sh = synth.Shape(layers=4, d=64, heads=4, seq=32, micro_batch=2, n_micro=4, dp=2, pp=2)
    _check(_launch(tmp_path, sh), sh, 1e-5)


def test_dp2_bf16(tmp_path):
    sh = synth.Shape(layers=2, d=256, heads=2, seq=128, micro_batch=1, n_micro=4, dp=2)
    _check(_launch(tmp_path, sh, precision=1), sh, 2e-2, elem=2)


def test_pp4_fp32_modular_pipeline(tmp_path):
    """P = 4: the ring has four distinct edges (stage 3 -> 0 wraps)."""
    sh = synth.Shape(layers=8, d=64, heads=4, seq=32, micro_batch=2, n_micro=4, dp=1, pp=4)
    _check(_launch(tmp_path, sh), sh, 1e-5)


def test_pp4_bf16_modular_pipeline(tmp_path):
    sh = synth.Shape(layers=4, d=256, heads=2, seq=128, micro_batch=1, n_micro=4, dp=1, pp=4)
    _check(_launch(tmp_path, sh, precision=1), sh, 2e-2, elem=2)


# ---- variants: N2a keep params, N2b unpartitioned, N2c no recompute, N3 contiguous pipeline
@pytest.mark.parametrize("flags", [KEEP, UNPART, NORECOMP, KEEP | NORECOMP])
def test_dp2_fp32_variants(tmp_path, flags):
    sh = synth.Shape(layers=4, d=64, heads=4, seq=32, micro_batch=2, n_micro=4, dp=2)
    _check(_launch(tmp_path, sh, chunk=2, steps=2, flags=flags), sh, 1e-5, steps=2, flags=flags)


@pytest.mark.parametrize("flags", [KEEP | NORECOMP, UNPART])
def test_dp2_bf16_variants(tmp_path, flags):
    sh = synth.Shape(layers=2, d=256, heads=2, seq=128, micro_batch=1, n_micro=4, dp=2)
    _check(_launch(tmp_path, sh, precision=1, flags=flags), sh, 2e-2, elem=2, flags=flags)


def test_pp2_fp32_contiguous_pipeline(tmp_path):
    sh = synth.Shape(layers=4, d=64, heads=4, seq=32, micro_batch=2, n_micro=4, dp=1, pp=2)
    _check(_launch(tmp_path, sh, flags=CONTIG), sh, 1e-5, flags=CONTIG)


def test_pp2_dp2_fp32_contiguous_unpartitioned(tmp_path):
    sh = synth.Shape(layers=4, d=64, heads=4, seq=32, micro_batch=2, n_micro=4, dp=2, pp=2)
    f = CONTIG | UNPART | NORECOMP
    _check(_launch(tmp_path, sh, flags=f), sh, 1e-5, flags=f)


def test_pp4_bf16_contiguous_pipeline(tmp_path):
    sh = synth.Shape(layers=8, d=256, heads=2, seq=128, micro_batch=1, n_micro=4, dp=1, pp=4)
    _check(_launch(tmp_path, sh, precision=1, flags=CONTIG), sh, 2e-2, elem=2, flags=CONTIG)


# ---- N1: the default data-parallel path is NVLink peer memory (copy-engine all-gathers, reduce-scatter fused
# into AdamW); LGA_FLAG_NCCL_DP keeps NCCL as the A/B baseline -- both must meet the same bar
@pytest.mark.parametrize("flags", [NCCL_DP, NCCL_DP | KEEP])
def test_dp2_fp32_nccl_baseline(tmp_path, flags):
    sh = synth.Shape(layers=4, d=64, heads=4, seq=32, micro_batch=2, n_micro=4, dp=2)
    _check(_launch(tmp_path, sh, chunk=2, steps=2, flags=flags), sh, 1e-5, steps=2, flags=flags)


def test_dp4_bf16_peer_memory_three_steps(tmp_path):
    """Peer-memory DP over 3 steps (graph replay from step 2): flags and epochs across steps."""
    sh = synth.Shape(layers=4, d=256, heads=2, seq=128, micro_batch=1, n_micro=4, dp=4)
    _check(_launch(tmp_path, sh, precision=1, steps=3), sh, 2e-2, steps=3, elem=2)


@pytest.mark.parametrize("flags,R", [(0, 2), (KEEP, 1)])
def test_dp2_peer_memory_path_is_the_one_that_runs(tmp_path, flags, R):
    """The default D > 1 LAYERED path really is peer memory: per step it launches exactly 4 more kernels per
    layer (two flag waits and two signals around the fused reduce-scatter + AdamW) and 2 more per
    all-gather (flag wait + read signal; the copies are copy-engine memcpys) than the NCCL baseline."""
    sh = synth.Shape(layers=4, d=64, heads=4, seq=32, micro_batch=2, n_micro=4, dp=2)
    (tmp_path / "peer").mkdir()
    (tmp_path / "nccl").mkdir()
    peer = _launch(tmp_path / "peer", sh, flags=flags)
    nccl = _launch(tmp_path / "nccl", sh, flags=flags | NCCL_DP)
    lloc = sh.layers
    for a, b in zip(peer, nccl):
        ka = json.loads(str(a["timing"]))["kernel_launches"]
        kb = json.loads(str(b["timing"]))["kernel_launches"]
        assert ka - kb == 4 * lloc + 2 * R * lloc, (ka, kb)
        np.testing.assert_allclose(a["params"], b["params"], rtol=1e-6, atol=1e-8)


def test_dp2_peer_kernels_counted_against_one_replica(tmp_path):
    """Runs on one GPU too: a D = 2 rank launches exactly the peer-memory kernels more than a D = 1 run of the
    same shape -- per layer two flag waits and two signals around the fused reduce-scatter + AdamW, a flag wait
    and a read signal per all-gather (R = 2 gathers per layer per step), plus the peer loss all-reduce."""
    sh2 = synth.Shape(layers=4, d=64, heads=4, seq=32, micro_batch=2, n_micro=4, dp=2)
    sh1 = synth.Shape(layers=4, d=64, heads=4, seq=32, micro_batch=2, n_micro=4, dp=1)
    (tmp_path / "d2").mkdir()
    (tmp_path / "d1").mkdir()
    two = _launch(tmp_path / "d2", sh2)
    one = _launch(tmp_path / "d1", sh1)
    k1 = json.loads(str(one[0]["timing"]))["kernel_launches"]
    for o in two:
        k2 = json.loads(str(o["timing"]))["kernel_launches"]
        assert k2 - k1 == (4 + 2 * 2) * sh2.layers + 1, (k2, k1)
    _check(two, sh2, 1e-5)


@pytest.mark.parametrize("shape,prec,flags", [(dict(dp=2), 1, 0), (dict(pp=2), 0, 0), (dict(dp=2), 0, UNPART),
                                               (dict(dp=2, pp=2), 0, 0)], ids=["dp2_bf16", "pp2", "dp2_unpart", "pp2_dp2"])
def test_guarded_arenas_multi_rank(tmp_path, shape, prec, flags):
    """The peer-memory paths write into other ranks' arenas (staging reads, flags, loss slots, pipeline
    transfers): with LGA_ARENA_GUARD=1 no canary of any rank's arena changes over 3 steps, and parity holds."""
    if prec == 1:
        sh = synth.Shape(layers=2, d=256, heads=2, seq=128, micro_batch=1, n_micro=4, **shape)
    else:
        sh = synth.Shape(layers=4, d=64, heads=4, seq=32, micro_batch=2, n_micro=4, **shape)
    outs = _launch(tmp_path, sh, precision=prec, steps=3, flags=flags, env={"LGA_ARENA_GUARD": "1"})
    assert [int(o["guard"]) for o in outs] == [0] * len(outs)
    _check(outs, sh, 2e-2 if prec else 1e-5, steps=3, elem=2 if prec else 4, flags=flags)


@pytest.mark.parametrize("shape,prec", [(dict(dp=2), 1), (dict(dp=2, pp=2), 0)], ids=["dp2_bf16", "pp2_dp2"])
def test_checkpoint_resume_multi_rank(tmp_path, shape, prec):
    """Every rank saves its shard after step 2 and a fresh world of handles resumes (new IPC mappings, flag epochs
    from 0, the AdamW step from the state): the 3-step result matches the oracle with exact counters."""
    if prec == 1:
        sh = synth.Shape(layers=2, d=256, heads=2, seq=128, micro_batch=1, n_micro=4, **shape)
    else:
        sh = synth.Shape(layers=4, d=64, heads=4, seq=32, micro_batch=2, n_micro=4, **shape)
    outs = _launch(tmp_path, sh, precision=prec, steps=3, resume_at=2)
    _check(outs, sh, 2e-2 if prec else 1e-5, steps=3, elem=2 if prec else 4)


# ---- N4: post-LN layer (reading A-16) under peer-memory DP and the modular pipeline
def test_dp2_bf16_post_ln(tmp_path):
    sh = synth.Shape(layers=2, d=256, heads=2, seq=128, micro_batch=1, n_micro=4, dp=2)
    _check(_launch(tmp_path, sh, precision=1, steps=2, flags=POST_LN), sh, 2e-2, steps=2, elem=2, flags=POST_LN)


def test_pp2_dp2_fp32_post_ln(tmp_path):
    sh = synth.Shape(layers=4, d=64, heads=4, seq=32, micro_batch=2, n_micro=4, dp=2, pp=2)
    _check(_launch(tmp_path, sh, flags=POST_LN), sh, 1e-5, flags=POST_LN)
