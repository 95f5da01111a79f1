"""Helpers for the GPU parity tests: run the CUDA path through the C ABI and the fp64 oracle on
the same seeded inputs (synth), compare with relative Frobenius error (reading A-15)."""
from __future__ import annotations

import numpy as np

import synth
from oracle import model as om
from oracle import schedule as osch


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / nb) if nb > 0 else float(np.linalg.norm(a - b))


def oracle_run(sh: synth.Shape, init: np.ndarray, batches, causal=True, lr=1e-3, wd=0.0, schedule="standard",
               post_ln=False):
    cfg = om.LayerCfg(d=sh.d, heads=sh.heads, causal=bool(causal), post_ln=bool(post_ln))
    params = [p.astype(np.float64) for p in synth.split_layers(init, sh.layers)]
    opt = osch.AdamW(lr=lr, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=wd)
    new, losses, grads = osch.train_steps(params, batches, cfg, opt, schedule)
    return np.concatenate(new), losses, np.concatenate(grads)


def per_layer_rel(a, b, layers):
    pl = a.size // layers
    return [rel(a[l * pl:(l + 1) * pl], b[l * pl:(l + 1) * pl]) for l in range(layers)]
