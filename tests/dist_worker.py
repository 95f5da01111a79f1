"""One rank of a multi-GPU parity run (launched by tests/test_gpu_dist.py through torchrun).

Writes its lga_grads / lga_params / counters / stage map to <out>/rank<r>.npz."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--shape", required=True)       # json of synth.Shape fields
    ap.add_argument("--precision", type=int, default=0)
    ap.add_argument("--schedule", type=int, default=0)
    ap.add_argument("--chunk", type=int, default=0)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--lr", type=float, default=1e-3)
    ap.add_argument("--flags", type=int, default=0)   # LGA_FLAG_* variants
    ap.add_argument("--resume-at", type=int, default=0)   # save the state after this many steps, resume in a new handle
    a = ap.parse_args()
    import torch
    import torch.distributed as dist
    from paper_2106_02679_b200 import Config, Trainer
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    local = local % torch.cuda.device_count()   # fewer GPUs than ranks: ranks share devices (peer memory over IPC)
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    sh = synth.Shape(**json.loads(a.shape))
    init = synth.init_params(sh, style="parity")
    cfg = Config(layers=sh.layers, d_model=sh.d, heads=sh.heads, seq_len=sh.seq, micro_batch=sh.micro_batch,
                 n_micro=sh.n_micro, dp=sh.dp, pp=sh.pp, precision=a.precision, schedule=a.schedule, chunk=a.chunk,
                 lr=a.lr, retain_grads=1, flags=a.flags)
    tr = Trainer(cfg, rank=rank, world=world, device=local, init_params=init)
    losses = []
    for k in range(a.steps):
        if a.resume_at and k == a.resume_at:   # checkpoint / resume: a fresh handle continues from the saved state
            state = tr.save_state()
            tr.close()
            tr = Trainer(cfg, rank=rank, world=world, device=local, init_params=init)
            tr.load_state(state)
        X, T = synth.batch(sh, step=k)
        r = tr.replica
        x = torch.from_numpy(X[r]).cuda()
        t = torch.from_numpy(T[r]).cuda()
        losses.append(tr.step(x, t))
    last, tot = tr.comm_stats()
    guard = -1
    if os.environ.get("LGA_ARENA_GUARD") == "1":
        import ctypes as C
        from paper_2106_02679_b200 import _abi
        f = _abi.lib().lgatest_arena_guard_check
        f.restype, f.argtypes = C.c_int64, [C.c_void_p]
        guard = int(f(tr._h))
    out = dict(grads=tr.grads(), params=tr.params(), losses=np.array(losses), stage=tr.stage, replica=tr.replica,
               guard=guard,
               stages=np.array(tr.layer_stage()), timing=json.dumps(tr.timing()), last=json.dumps(last),
               total=json.dumps(tot))
    np.savez(os.path.join(a.out, f"rank{rank}.npz"), **out)
    tr.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
