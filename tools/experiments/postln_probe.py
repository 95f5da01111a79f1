"""Probe: per-tensor gradient error of the bf16 post-LN step after 1 and 2 steps (ln weights at ~2 %)."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import synth
from gpu_util import oracle_run, per_tensor_rel, _split
from paper_2106_02679_b200 import LGA_BF16, LGA_FP32, Config, Trainer
from paper_2106_02679_b200._abi import LGA_FLAG_POST_LN

def run(sh, steps, prec, post=True, causal=0):
    init = synth.init_params(sh, style="parity")
    cfg = Config(layers=sh.layers, d_model=sh.d, heads=sh.heads, seq_len=sh.seq, micro_batch=sh.micro_batch,
                 n_micro=sh.n_micro, precision=prec, causal=causal, lr=1e-3, retain_grads=1,
                 flags=LGA_FLAG_POST_LN if post else 0)
    tr = Trainer(cfg, rank=0, world=1, device=0, init_params=init)
    batches = [synth.batch(sh, step=k) for k in range(steps)]
    for X, T in batches:
        tr.step(torch.from_numpy(X[0]).cuda(), torch.from_numpy(T[0]).cuda())
    g, p = tr.grads(), tr.params(); tr.close()
    rp, rl, rg = oracle_run(sh, init, batches, causal=causal, lr=1e-3, post_ln=post)
    return g, rg, p, rp

sh = synth.Shape(layers=2, d=256, heads=4, seq=128, micro_batch=2, n_micro=4)
for post in (True, False):
    for steps in (1, 2, 3):
        for prec in (LGA_BF16,):
            g, rg, p, rp = run(sh, steps, prec, post)
            r = per_tensor_rel(g, rg, sh.d, sh.layers)
            print(f"post={post} steps={steps} prec={prec}:", {k: f"{v:.4f}" for k, v in r[0].items() if k in ("ln1_w", "ln2_w", "ln1_b", "ln2_b", "Wq", "W1", "bk_abs")})
            pl = g.size // sh.layers
            for name in ("ln1_w", "ln2_w"):
                a, b = _split(g[:pl], sh.d)[name], _split(rg[:pl], sh.d)[name]
                alpha = float(a @ b / (b @ b))
                print(f"   {name}: alpha={alpha:.5f} resid={np.linalg.norm(a - alpha * b) / np.linalg.norm(b):.4f} |r|={np.linalg.norm(b):.3e} rel_max_elem={np.max(np.abs(a-b))/np.max(np.abs(b)):.4f}")
