"""One rank of the CPU (gloo) data-parallel decomposition test, launched by tests/test_dist_cpu.py through
torchrun.  It plays the host-side protocol of the library's partitioned data parallelism with the fp64 oracle
as the compute (TEST INFRASTRUCTURE): replica r sums the gradients of ITS micro-batches (reading A-10: replica
r owns micro-batches rN..rN+N-1; A-3: unscaled sums), every layer is padded to a multiple of 64 D and
reduced over the replicas, rank r keeps shard r (A-10) scaled by 1/(D N) (A-3), updates it with AdamW
(O7), and the shards are all-gathered back.  Writes <out>/rank<r>.npz."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from oracle import counters as oc  # noqa: E402
from oracle import model as om  # noqa: E402
from oracle import schedule as osch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--shape", required=True)
    a = ap.parse_args()
    import torch
    import torch.distributed as dist
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo")
    sh = synth.Shape(**json.loads(a.shape))
    assert sh.dp == world
    X, T = synth.batch(sh, step=0)
    init = synth.init_params(sh, style="parity")
    cfg = om.LayerCfg(d=sh.d, heads=sh.heads, causal=True)
    params = [p.astype(np.float64) for p in synth.split_layers(init, sh.layers)]
    # this replica's micro-batches only; grads_standard returns the mean over them -> x N = the sum
    _, g = osch.grads_standard(params, X[rank:rank + 1], T[rank:rank + 1], cfg)
    pl, pad = om.layer_param_count(sh.d), oc.padded_layer_params(sh.d, world)
    S = pad // world
    padded = np.zeros((sh.layers, pad))
    padded[:, :pl] = np.stack(g) * sh.n_micro
    t = torch.from_numpy(padded)
    dist.all_reduce(t)                                            # sum over the D replicas
    shard_g = t.numpy()[:, rank * S:(rank + 1) * S] / (world * sh.n_micro)
    master = np.zeros((sh.layers, pad))
    master[:, :pl] = np.stack(params)
    opt = osch.AdamW(lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.0)
    mine = np.stack([opt.update(master[l, rank * S:(rank + 1) * S], shard_g[l],
                                opt.init_state(master[l, rank * S:(rank + 1) * S])) for l in range(sh.layers)])
    parts = [torch.zeros(mine.shape, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(parts, torch.from_numpy(np.ascontiguousarray(mine)))
    full = np.concatenate([p.numpy() for p in parts], axis=1)[:, :pl].reshape(-1)
    grads = np.concatenate([t.numpy()[:, :pl] / (world * sh.n_micro)], axis=0).reshape(-1)
    np.savez(os.path.join(a.out, f"rank{rank}.npz"), params=full, grads=grads, shard=np.array([rank * S, S]))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
