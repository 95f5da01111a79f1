"""World-size-2 / 4 gloo tests on CPU (no GPU).  These are ORACLE-CONSISTENCY tests of the decompositions the
library implements, played in Python with the fp64 oracle as the compute: they do not call liblga.  The
library's own host logic is checked on CPU by test_abi_cpu.py::test_rank_plan_matches_closed_forms (lga_plan:
the rank grid, local layers and pipeline flag targets lga_init uses), and its multi-rank data paths by the
-m gpu tests of test_gpu_dist.py (which also run with all ranks sharing one GPU).

* the data-parallel decomposition the library implements -- per-replica micro-batch ownership (A-10),
  unscaled sums reduced over replicas with one 1/(D N) scale (A-3), shards of the 64 D-padded layer vector
  updated independently by AdamW and gathered back -- reproduces the single-process oracle step exactly
  (P5: D ranks x N == 1 rank x D N);
* the modular pipeline's host protocol (A11) -- layer i on stage i mod P, layer-major forward with
  x_{i+1}[m] sent around the ring, loss on the last layer's stage, backward with recompute and dX_i[m] sent
  back -- reproduces the single-process oracle gradient and loss, and each stage's send / receive count equals
  the closed-form p2p counter (P10);
* bench.py's reference arm under torchrun: rank 0 alone runs the oracle and prints one JSON line, every
  rank exits 0."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import synth
from gpu_util import oracle_run, rel

torch = pytest.importorskip("torch")
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
_port = [29811]


def _torchrun(args, nproc=2, timeout=300):
    _port[0] += 1
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={_port[0]}"] + args
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="", OMP_NUM_THREADS="1")
    return subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT, env=env)


def test_gloo_data_parallel_decomposition(tmp_path):
    sh = synth.Shape(layers=2, d=32, heads=2, seq=8, micro_batch=2, n_micro=2, dp=2)
    shape = json.dumps(dict(layers=sh.layers, d=sh.d, heads=sh.heads, seq=sh.seq, micro_batch=sh.micro_batch,
                            n_micro=sh.n_micro, dp=sh.dp))
    r = _torchrun([os.path.join(HERE, "dist_cpu_worker.py"), "--out", str(tmp_path), "--shape", shape])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    outs = [dict(np.load(os.path.join(tmp_path, f"rank{k}.npz"))) for k in range(2)]
    init = synth.init_params(sh, style="parity")
    rp, rl, rg = oracle_run(sh, init, [synth.batch(sh, step=0)], lr=1e-3)
    for o in outs:
        assert rel(o["grads"], rg) < 1e-12
        assert rel(o["params"], rp) < 1e-12
    assert outs[0]["shard"][1] == outs[1]["shard"][1] and outs[1]["shard"][0] == outs[0]["shard"][1]


@pytest.mark.parametrize("pp,dp", [(2, 1), (2, 2)])
def test_gloo_modular_pipeline_decomposition(tmp_path, pp, dp):
    from oracle import counters as oc
    from oracle import model as om
    from oracle import schedule as osch
    sh = synth.Shape(layers=4, d=32, heads=2, seq=8, micro_batch=2, n_micro=3, pp=pp, dp=dp)
    shape = json.dumps(dict(layers=sh.layers, d=sh.d, heads=sh.heads, seq=sh.seq, micro_batch=sh.micro_batch,
                            n_micro=sh.n_micro, pp=sh.pp, dp=sh.dp))
    r = _torchrun([os.path.join(HERE, "pipe_cpu_worker.py"), "--out", str(tmp_path), "--shape", shape],
                  nproc=pp * dp)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    outs = [dict(np.load(os.path.join(tmp_path, f"rank{k}.npz"))) for k in range(pp * dp)]
    init = synth.init_params(sh, style="parity")
    params = [p.astype(np.float64) for p in synth.split_layers(init, sh.layers)]
    X, T = synth.batch(sh, step=0)
    ref_loss, ref_g = osch.grads_standard(params, X, T, om.LayerCfg(d=sh.d, heads=sh.heads, causal=True))
    for k, o in enumerate(outs):
        assert rel(o["grads"], np.concatenate(ref_g)) < 1e-12
        assert abs(float(o["loss"][0]) - ref_loss) < 1e-12 * abs(ref_loss)
        c = oc.comm_counters(oc.StepShape(layers=sh.layers, d=sh.d, seq=sh.seq, micro_batch=sh.micro_batch,
                                          n_micro=sh.n_micro, pp=sh.pp), stage=k % pp)
        assert int(o["sends"]) == c["p2p_send_calls"] and int(o["recvs"]) == c["p2p_recv_calls"]
    # 2 N (L - 1) crossings per replica per step (P10)
    assert sum(int(o["sends"]) for o in outs) == dp * 2 * sh.n_micro * (sh.layers - 1)


def test_reference_arm_under_torchrun_rank0_only():
    r = _torchrun(["bench.py", "--impl", "reference", "--gpus", "2", "--workload", "tiny", "--steps", "1",
                   "--warmup", "0"])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "oracle"
