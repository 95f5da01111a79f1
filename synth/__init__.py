"""Seeded synthetic inputs shared by the oracle side and the GPU side.

This module holds NONE of the method's arithmetic: it only draws random numbers
(NumPy PCG64) in the shapes of the paper's workload, so that ``oracle/`` and the
CUDA path can be fed bit-identical fp32 inputs.  Recipe:

* activations x and targets T: i.i.d. N(0, 1) fp32, shape [D][N][b][s][d]
  (stand-ins for embedded tokens; the embedding and LM head are excluded);
* parameters, canonical flat layout per layer (see ``layout``):
  - ``style="train"``: weights N(0, 0.02^2), W_o and W_2 N(0, (0.02/sqrt(2L))^2),
    biases 0, LayerNorm gain 1, shift 0 (GPT-2 practice);
  - ``style="parity"``: as "train" but gains 1 + 0.1 N(0,1) and shifts/biases
    0.02 N(0,1), so every gradient path is non-trivial and a transposed operand
    shows up in the parity tests.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

DEFAULT_PARAM_SEED = 1234
DEFAULT_DATA_SEED = 5678


@dataclass(frozen=True)
class Shape:
    layers: int
    d: int
    heads: int
    seq: int
    micro_batch: int
    n_micro: int
    dp: int = 1
    pp: int = 1
    ffn_mult: int = 4


def layout(d: int, ffn_mult: int = 4):
    """Names, offsets and shapes of one layer's canonical flat parameter vector
    (pure bookkeeping; both sides state this layout independently and a test checks
    that they agree)."""
    f = ffn_mult * d
    spec = [("ln1_w", (d,)), ("ln1_b", (d,)), ("Wqkv", (d, 3 * d)), ("bqkv", (3 * d,)),
            ("Wo", (d, d)), ("bo", (d,)), ("ln2_w", (d,)), ("ln2_b", (d,)),
            ("W1", (d, f)), ("b1", (f,)), ("W2", (f, d)), ("b2", (d,))]
    out, off = [], 0
    for name, shape in spec:
        n = int(np.prod(shape))
        out.append((name, off, shape))
        off += n
    return out, off


def init_params(sh: Shape, seed: int = DEFAULT_PARAM_SEED, style: str = "parity") -> np.ndarray:
    """All layers' parameters, fp32, concatenated canonical layout, length L * P_l."""
    rng = np.random.Generator(np.random.PCG64(seed))
    spec, pl = layout(sh.d, sh.ffn_mult)
    out = np.empty(sh.layers * pl, dtype=np.float32)
    std = 0.02
    std_res = 0.02 / np.sqrt(2.0 * sh.layers)
    for l in range(sh.layers):
        base = l * pl
        for name, off, shape in spec:
            n = int(np.prod(shape))
            if name in ("Wqkv", "W1"):
                v = rng.standard_normal(n) * std
            elif name in ("Wo", "W2"):
                v = rng.standard_normal(n) * std_res
            elif name in ("ln1_w", "ln2_w"):
                v = np.ones(n) if style == "train" else 1.0 + 0.1 * rng.standard_normal(n)
            else:  # biases and LayerNorm shifts
                v = np.zeros(n) if style == "train" else 0.02 * rng.standard_normal(n)
            out[base + off: base + off + n] = v.astype(np.float32)
    return out


def batch(sh: Shape, step: int = 0, seed: int = DEFAULT_DATA_SEED):
    """(X, T) for one step, fp32 [D][N][b][s][d] each; replica r uses X[r]."""
    rng = np.random.Generator(np.random.PCG64(seed + step))
    shape = (sh.dp, sh.n_micro, sh.micro_batch, sh.seq, sh.d)
    X = rng.standard_normal(shape, dtype=np.float32)
    T = rng.standard_normal(shape, dtype=np.float32)
    return X, T


def split_layers(flat: np.ndarray, layers: int):
    """Split the concatenated vector into per-layer views."""
    pl = flat.size // layers
    return [flat[l * pl:(l + 1) * pl] for l in range(layers)]
