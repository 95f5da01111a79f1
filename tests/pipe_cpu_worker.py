"""One rank (stage = rank mod P of replica = rank div P, the rank grid of include/lga.h) of the CPU (gloo)
modular-pipeline ORACLE-CONSISTENCY test, launched by tests/test_dist_cpu.py through torchrun (it does not
call liblga; lga_plan is checked against the same closed forms in test_abi_cpu.py).  It plays the
protocol of the library's modular pipeline with the fp64 oracle as the compute (TEST
INFRASTRUCTURE): layer i lives on stage i mod P (reading A-11); the layered schedule runs every
layer over all N micro-batches before the next; after the forward of (layer i, micro-batch m) the
owner sends x_{i+1}[m] to stage (i+1) mod P of its replica, the stage of layer L-1 computes the loss, and
in backward the owner of layer i recomputes it from its checkpoint and sends dX_i[m] to stage
(i-1) mod P.  Each stage accumulates only its own layers' gradients; replica r takes micro-batches
r N ... r N + N - 1 (reading A-10) and gradients are summed over replicas with one 1/(D N) scale (A-3).
Writes <out>/rank<r>.npz with the assembled gradient vector, the loss and this rank's send/recv counts."""
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
    assert sh.pp * sh.dp == world
    L, N, P, D = sh.layers, sh.n_micro, sh.pp, sh.dp
    me, replica = rank % P, rank // P                  # rank grid of include/lga.h: stage = rank mod P
    X, T = synth.batch(sh, step=0)
    init = synth.init_params(sh, style="parity")
    cfg = om.LayerCfg(d=sh.d, heads=sh.heads, causal=True)
    params = [p.astype(np.float64) for p in synth.split_layers(init, L)]
    stage = lambda i: oc.stage_of_layer(i, P)
    peer = lambda st: replica * P + st                 # the same replica's rank of stage st
    msg_shape = (sh.micro_batch, sh.seq, sh.d)
    sends = recvs = 0

    def send(t, dst):
        nonlocal sends
        dist.send(torch.from_numpy(np.ascontiguousarray(t)), peer(dst))
        sends += 1

    def recv(src):
        nonlocal recvs
        buf = torch.zeros(msg_shape, dtype=torch.float64)
        dist.recv(buf, peer(src))
        recvs += 1
        return buf.numpy()

    # forward, layer-major; ckpt[i][m] = input of layer i (kept only where layer i lives)
    ckpt = {0: [np.asarray(X[replica, m], dtype=np.float64) for m in range(N)]} if stage(0) == me else {}
    out_L = None
    for i in range(L):
        if stage(i) == me:
            ys = [om.layer_forward(ckpt[i][m], params[i], cfg)[0] for m in range(N)]
            if i == L - 1:
                out_L = ys
            elif stage(i + 1) == me:
                ckpt[i + 1] = ys
            else:
                for y in ys:
                    send(y, stage(i + 1))
        elif i < L - 1 and stage(i + 1) == me:
            ckpt[i + 1] = [recv(stage(i)) for _ in range(N)]
    # loss + seed gradient on the stage of layer L-1 (reading A-2)
    loss = 0.0
    dY = {}
    if stage(L - 1) == me:
        seeds = [om.mse_loss(out_L[m], np.asarray(T[replica, m], dtype=np.float64)) for m in range(N)]
        loss = sum(s[0] for s in seeds) / N
        dY[L - 1] = [s[1] for s in seeds]
    # backward, layer-major with recompute; one gradient buffer per local layer
    pl = om.layer_param_count(sh.d)
    grads = np.zeros((L, pl))
    for i in reversed(range(L)):
        if stage(i) == me:
            dxs = []
            for m in range(N):
                _, cache = om.layer_forward(ckpt[i][m], params[i], cfg)       # recompute
                dx, g = om.layer_backward(dY[i][m], cache, params[i], cfg)
                grads[i] += g
                dxs.append(dx)
            if i > 0:
                if stage(i - 1) == me:
                    dY[i - 1] = dxs
                else:
                    for dx in dxs:
                        send(dx, stage(i - 1))
        elif i > 0 and stage(i - 1) == me:
            dY[i - 1] = [recv(stage(i)) for _ in range(N)]
    g = torch.from_numpy(grads / (D * N))
    dist.all_reduce(g)     # sum over replicas; assembles the full vector (each layer lives on one stage)
    lt = torch.tensor([loss], dtype=torch.float64)
    dist.all_reduce(lt)
    lt /= D
    np.savez(os.path.join(a.out, f"rank{rank}.npz"), grads=g.numpy().reshape(-1), loss=lt.numpy(),
             sends=np.array(sends), recvs=np.array(recvs))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
