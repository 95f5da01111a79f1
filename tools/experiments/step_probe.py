"""Run a few LGA steps of an arbitrary config (hang / speed probing).
   torchrun ... tools/step_probe.py L d heads s b N dp pp [chunk]"""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2106_02679_b200 import Config, Trainer
L, d, H, s, b, N, dp, pp = [int(v) for v in sys.argv[1:9]]
chunk = int(sys.argv[9]) if len(sys.argv) > 9 else 0
world = int(os.environ.get("WORLD_SIZE", "1")); rank = int(os.environ.get("RANK", "0")); local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
if world > 1:
    import torch.distributed as dist
    dist.init_process_group("gloo")
cfg = Config(layers=L, d_model=d, heads=H, seq_len=s, micro_batch=b, n_micro=N, dp=dp, pp=pp, chunk=chunk)
tr = Trainer(cfg, rank=rank, world=world, device=local)
x = torch.randn(N, b, s, d, device="cuda"); t = torch.randn(N, b, s, d, device="cuda")
for k in range(3):
    t0 = time.time(); loss = tr.step(x, t); print(f"rank {rank} step {k} loss {loss:.5f} {time.time()-t0:.3f}s", flush=True)
tr.close()
