"""Print the measured parity (relative Frobenius error vs the fp64 oracle) of the CUDA step for the
configs the tests cover; output goes to profiles/parity_<round>.txt.  Needs a GPU."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import synth  # noqa: E402
from gpu_util import max_per_tensor, oracle_run, per_layer_rel, per_tensor_rel, rel  # noqa: E402
from paper_2106_02679_b200 import LGA_BF16, LGA_FP32, Config, Trainer  # noqa: E402

CASES = [
    ("C1 tiny fp32 (L2 d64 h4 s32 b2 N4)", synth.Shape(2, 64, 4, 32, 2, 4), LGA_FP32, "parity"),
    ("fp32 ragged (L2 d48 h3 s37 b1 N3)", synth.Shape(2, 48, 3, 37, 1, 3), LGA_FP32, "parity"),
    ("bf16 d256 h4 s128 b2 N4", synth.Shape(2, 256, 4, 128, 2, 4), LGA_BF16, "parity"),
    ("bf16 d256 h2 (dh128) s200 b1 N4", synth.Shape(3, 256, 2, 200, 1, 4), LGA_BF16, "parity"),
    ("bf16 C2 layer (L1 d768 h12 s1024 b4 N2)", synth.Shape(1, 768, 12, 1024, 4, 2), LGA_BF16, "train"),
    ("bf16 C3 layer (L2 d2048 h16 s2048 b1 N2)", synth.Shape(2, 2048, 16, 2048, 1, 2), LGA_BF16, "train"),
    ("bf16 C4 layer (L1 d4096 h32 s2048 b1 N2)", synth.Shape(1, 4096, 32, 2048, 1, 2), LGA_BF16, "train"),
    ("fp32 d1024 h8 s96 b1 N2 (L1)", synth.Shape(1, 1024, 8, 96, 1, 2), LGA_FP32, "parity"),
    ("fp32 d2048 h16 s80 b1 N2 (L1)", synth.Shape(1, 2048, 16, 80, 1, 2), LGA_FP32, "parity"),
    ("fp32 d4096 h32 s64 b1 N2 (L1)", synth.Shape(1, 4096, 32, 64, 1, 2), LGA_FP32, "parity"),
    ("bf16 d256 h4 s128 b2 N4 parity-init", synth.Shape(2, 256, 4, 128, 2, 4), LGA_BF16, "parity"),
    ("bf16 d1024 h8 s256 b1 N2 parity-init", synth.Shape(1, 1024, 8, 256, 1, 2), LGA_BF16, "parity"),
    ("bf16 d2048 h16 s512 b1 N2 parity-init", synth.Shape(1, 2048, 16, 512, 1, 2), LGA_BF16, "parity"),
]


def main():
    lines = ["# parity of the CUDA LGA step vs the fp64 oracle (relative Frobenius error), one AdamW step lr=1e-3",
             "# bar: fp32 mode 1e-5, bf16 mode 2e-2 (BASELINE.json north star), global / per layer; per tensor:",
             "# fp32 1e-4, bf16 2e-2 against the oracle at the 16-bit weight copy (tests/gpu_util.py TENSOR_TOL)",
             "# 'update' = params - init (ill-conditioned: AdamW t=1 is lr*sign(g) where |g| >> eps); the 'train'-init",
             "# rows' zero-initialised tensors (biases, LN beta) have param == update, so the tests leave them out",
             f"{'config':48s} {'grads':>9s} {'max/layer':>9s} {'params':>9s} {'update':>9s} {'loss':>9s}"]
    for name, sh, prec, style in CASES:
        init = synth.init_params(sh, style=style)
        cfg = Config(layers=sh.layers, d_model=sh.d, heads=sh.heads, seq_len=sh.seq, micro_batch=sh.micro_batch,
                     n_micro=sh.n_micro, precision=prec, lr=1e-3, retain_grads=1)
        tr = Trainer(cfg, rank=0, world=1, device=0, init_params=init)
        X, T = synth.batch(sh, step=0)
        loss = tr.step(torch.from_numpy(X[0]).cuda(), torch.from_numpy(T[0]).cuda())
        g, p = tr.grads(), tr.params()
        tr.close()
        rp, rl, rg = oracle_run(sh, init, [(X, T)], lr=1e-3)
        lines.append(f"{name:48s} {rel(g, rg):9.2e} {max(per_layer_rel(g, rg, sh.layers)):9.2e} {rel(p, rp):9.2e} "
                     f"{rel(p - init, rp - init):9.2e} {abs(loss - rl[0]) / abs(rl[0]):9.2e}")
        mt = max_per_tensor(per_tensor_rel(g, rg, sh.d, sh.layers))
        if prec == LGA_BF16:
            mpp, _, mpg = oracle_run(sh, init, [(X, T)], lr=1e-3, param_round="bf16")
            mm = max_per_tensor(per_tensor_rel(g, mpg, sh.d, sh.layers))
            lines.append("    per-tensor grad max vs the 16-bit-weight oracle (P:50): "
                         + " ".join(f"{k}={v:.1e}" for k, v in mm.items()))
        mp = max_per_tensor(per_tensor_rel(p - init, rp - init, sh.d, sh.layers, grads=False))
        mq = max_per_tensor(per_tensor_rel(p, rp, sh.d, sh.layers, grads=False))
        lines.append("    per-tensor grad max: " + " ".join(f"{k}={v:.1e}" for k, v in mt.items()))
        lines.append("    per-tensor param max: " + " ".join(f"{k}={v:.1e}" for k, v in mq.items()))
        lines.append("    per-tensor update max: " + " ".join(f"{k}={v:.1e}" for k, v in mp.items()))
        print("\n".join(lines[-(5 if prec == LGA_BF16 else 4):]), flush=True)
    out = os.path.join(ROOT, "profiles", f"parity_{sys.argv[1] if len(sys.argv) > 1 else 'r1'}.txt")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
