"""Sanitizer driver: a few LGA steps through the C ABI on small shapes, for
    compute-sanitizer --tool {memcheck,synccheck,racecheck,initcheck} python tools/sanitize_step.py [fp32|bf16|all]
fp32: C1 (L2 d64 h4 s32 b2 N4, SIMT kernels), chunked and not, eager and graph-replayed.
bf16: L2 d256 (d_h 64 and 128) s128/200 b1-2 N4 -- the tcgen05 GEMMs (single-CTA and CTA-pair tiles), tcgen05
attention forward / backward, the fused epilogues, LayerNorm kernels, AdamW -- eager and graph-replayed."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2106_02679_b200 import LGA_BF16, LGA_FP32, Config, Trainer  # noqa: E402
from paper_2106_02679_b200._abi import LGA_FLAG_NO_GRAPH  # noqa: E402


def run(sh, precision, chunk=0, flags=0, steps=3):
    init = synth.init_params(sh, style="parity")
    cfg = Config(layers=sh.layers, d_model=sh.d, heads=sh.heads, seq_len=sh.seq, micro_batch=sh.micro_batch,
                 n_micro=sh.n_micro, precision=precision, chunk=chunk, lr=1e-3, retain_grads=1, flags=flags)
    tr = Trainer(cfg, rank=0, world=1, device=0, init_params=init)
    X, T = synth.batch(sh, step=0)
    x, t = torch.from_numpy(X[0]).cuda(), torch.from_numpy(T[0]).cuda()
    losses = [tr.step(x, t) for _ in range(steps)]
    g = tr.grads()
    tr.close()
    assert np.all(np.isfinite(g)) and all(np.isfinite(losses))
    print(f"ok {sh} prec={precision} chunk={chunk} flags={flags:#x} losses={[round(l, 6) for l in losses]}", flush=True)


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    if which in ("fp32", "all"):
        c1 = synth.Shape(layers=2, d=64, heads=4, seq=32, micro_batch=2, n_micro=4)
        run(c1, LGA_FP32)
        run(c1, LGA_FP32, chunk=2, flags=LGA_FLAG_NO_GRAPH, steps=2)
    if which in ("bf16", "all"):
        run(synth.Shape(layers=2, d=256, heads=4, seq=128, micro_batch=2, n_micro=4), LGA_BF16)
        run(synth.Shape(layers=2, d=256, heads=2, seq=200, micro_batch=1, n_micro=4), LGA_BF16, chunk=2,
            flags=LGA_FLAG_NO_GRAPH, steps=2)


if __name__ == "__main__":
    main()
