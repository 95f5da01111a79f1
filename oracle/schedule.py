"""Gradient-accumulation schedules and AdamW in fp64.  TEST INFRASTRUCTURE ONLY.

The objective of one step (readings A-2, A-3):

    L(theta) = 1/(D N) * sum_{r<D, m<N} l(f_theta(X[r, m]), T[r, m])

with l the per-micro-batch MSE of ``model.mse_loss``.  Three schedules compute
its gradient; the paper's claim is that they are the same computation reordered:

* ``grads_standard`` -- standard gradient accumulation: "processing multiple
  micro-batches sequentially between weight updates"; each micro-batch
  runs the whole stack forward then backward (Fig. 1 top).  This is the
  reference value.
* ``grads_layered`` -- layered gradient accumulation: "we split the input into
  micro-batches exactly as in standard gradient accumulation, but we process
  all the micro-batches for a given layer before proceeding to the next one.
  We take such layers as the intervals between activation checkpoints"
  (P:104).  Forward keeps only each layer's output (the checkpoint);
  backward recomputes the layer from its checkpoint and accumulates all
  micro-batches' gradients of that layer into one buffer before moving on.
* ``grads_fullbatch`` -- no accumulation: one pass over all D*N*b sequences.

AdamW follows torch.optim.AdamW (reading A-4): "The Adam optimizer is assumed".

Mixed precision ("the bulk of the computation is done in half-precision, while the weights
are stored and updated in single-precision"; bfloat16 named there): ``train_steps(...,
param_round="bf16")`` evaluates each step's gradient at the 16-bit copy of the weights,
round-to-nearest-even of the stored weights (reading A-9), and applies it to the stored weights.
This is the gradient the mixed-precision method defines; the default (None) is the plain
definition at the stored weights.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .model import LayerCfg, layer_backward, layer_forward, mse_loss


def round_bf16(a) -> np.ndarray:
    """Round-to-nearest-even of float32(a) to bfloat16, returned as float64 (reading A-9): keep the top 16
    bits of the fp32 pattern after adding 0x7FFF plus the lowest kept bit (ties to even)."""
    u = np.ascontiguousarray(np.asarray(a, dtype=np.float32)).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def _as64(a):
    return np.asarray(a, dtype=np.float64)


def loss(params, X, T, cfg: LayerCfg) -> float:
    """L(theta) by its definition: forward only, mean over the D*N micro-batch losses."""
    D, N = X.shape[0], X.shape[1]
    tot = 0.0
    for r in range(D):
        for m in range(N):
            x = _as64(X[r, m])
            for p in params:
                x, _ = layer_forward(x, p, cfg)
            tot += mse_loss(x, _as64(T[r, m]))[0]
    return tot / (D * N)


def grads_standard(params, X, T, cfg: LayerCfg):
    """Micro-batch-major accumulation.  params: list of L flat fp64 layer vectors;
    X, T: [D, N, b, s, d].  Returns (loss, grads) with grads a list of L flat vectors
    of dL/dtheta for the global mean loss."""
    D, N = X.shape[0], X.shape[1]
    L = len(params)
    acc = [np.zeros_like(p) for p in params]
    loss = 0.0
    for r in range(D):
        for m in range(N):
            x = _as64(X[r, m])
            caches = []
            for l in range(L):                       # full forward of micro-batch (r, m)
                x, c = layer_forward(x, params[l], cfg)
                caches.append(c)
            lm, dy = mse_loss(x, _as64(T[r, m]))
            loss += lm
            for l in reversed(range(L)):             # full backward of micro-batch (r, m)
                dy, g = layer_backward(dy, caches[l], params[l], cfg)
                acc[l] += g
    scale = 1.0 / (D * N)
    return loss * scale, [a * scale for a in acc]


def grads_layered(params, X, T, cfg: LayerCfg):
    """Layer-major accumulation with checkpoints at layer outputs and recompute."""
    D, N = X.shape[0], X.shape[1]
    L = len(params)
    # forward: layer by layer over all micro-batches, keep only the checkpoints
    ckpt = [[[None] * N for _ in range(D)] for _ in range(L + 1)]
    for r in range(D):
        for m in range(N):
            ckpt[0][r][m] = _as64(X[r, m])
    for l in range(L):
        for r in range(D):
            for m in range(N):
                ckpt[l + 1][r][m], _ = layer_forward(ckpt[l][r][m], params[l], cfg)
    loss = 0.0
    dY = [[None] * N for _ in range(D)]
    for r in range(D):
        for m in range(N):
            lm, dY[r][m] = mse_loss(ckpt[L][r][m], _as64(T[r, m]))
            loss += lm
    # backward: layer by layer, recompute from checkpoint, one gradient buffer per layer
    grads = [None] * L
    for l in reversed(range(L)):
        buf = np.zeros_like(params[l])
        for r in range(D):
            for m in range(N):
                _, cache = layer_forward(ckpt[l][r][m], params[l], cfg)      # recompute
                dY[r][m], g = layer_backward(dY[r][m], cache, params[l], cfg)
                buf += g
        grads[l] = buf
    scale = 1.0 / (D * N)
    return loss * scale, [g * scale for g in grads]


def grads_fullbatch(params, X, T, cfg: LayerCfg):
    """One pass over all D*N*b sequences.  The mean over all elements equals the mean of the
    per-micro-batch means because all micro-batches have the same size."""
    D, N, b, s, d = X.shape
    x = _as64(X).reshape(D * N * b, s, d)
    caches = []
    for l in range(len(params)):
        x, c = layer_forward(x, params[l], cfg)
        caches.append(c)
    loss, dy = mse_loss(x, _as64(T).reshape(D * N * b, s, d))
    grads = [None] * len(params)
    for l in reversed(range(len(params))):
        dy, grads[l] = layer_backward(dy, caches[l], params[l], cfg)
    return loss, grads


@dataclass
class AdamW:
    """torch.optim.AdamW semantics, step counter t from 1 (reading A-4, O7):
        theta <- theta (1 - lr wd)
        m <- b1 m + (1-b1) g ;  v <- b2 v + (1-b2) g^2
        theta <- theta - lr (m / (1-b1^t)) / (sqrt(v / (1-b2^t)) + eps)
    """
    lr: float = 1e-4
    beta1: float = 0.9
    beta2: float = 0.95
    eps: float = 1e-8
    weight_decay: float = 0.0

    def init_state(self, theta):
        return dict(m=np.zeros_like(theta), v=np.zeros_like(theta), t=0)

    def update(self, theta, g, state):
        state["t"] += 1
        t = state["t"]
        theta = theta * (1.0 - self.lr * self.weight_decay)
        state["m"] = self.beta1 * state["m"] + (1.0 - self.beta1) * g
        state["v"] = self.beta2 * state["v"] + (1.0 - self.beta2) * g * g
        mhat = state["m"] / (1.0 - self.beta1 ** t)
        vhat = state["v"] / (1.0 - self.beta2 ** t)
        return theta - self.lr * mhat / (np.sqrt(vhat) + self.eps)


SCHEDULES = {"standard": grads_standard, "layered": grads_layered, "fullbatch": grads_fullbatch}


def train_steps(params, batches, cfg: LayerCfg, opt: AdamW, schedule="standard", param_round=None):
    """Run len(batches) optimizer steps.  batches: list of (X, T).  Returns
    (params, losses, last_grads).  Parameters are fp64 copies; the caller passes the fp32
    initial values the GPU side received (O1).  param_round="bf16": each gradient is taken at
    round_bf16 of the stored weights (mixed precision; module docstring)."""
    params = [_as64(p).copy() for p in params]
    states = [opt.init_state(p) for p in params]
    losses, grads = [], None
    fn = SCHEDULES[schedule]
    for X, T in batches:
        at = params if param_round is None else [round_bf16(p) for p in params]
        loss, grads = fn(at, X, T, cfg)
        losses.append(loss)
        params = [opt.update(p, g, s) for p, g, s in zip(params, grads, states)]
    return params, losses, grads
