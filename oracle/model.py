"""One transformer layer in fp64 NumPy: forward, backward, MSE loss.  TEST INFRASTRUCTURE ONLY.

Paper: "A transformer encoder consists of d_l identical layers, each composed of
a multi-head attention module followed by a non-linearity ... d_a attention
heads of size d_h, for a layer width d_m = d_a x d_h, while the latter consists
of a two-layer dense feedforward network with intermediate size d_I = n_I x d_m"
(P:152); n_I = 4.  The exact per-layer parameter count
p_l = (4+2n_I) d_m^2 + 13 d_m fixes the biases and the two LayerNorms
("12x^5+13x^3").

Readings where the paper is silent (A-1, A-2): pre-LN (GPT-2 style),
causal mask by default (``causal=False`` gives the paper's encoder), exact-erf
GELU, no dropout, LayerNorm with biased variance and eps = 1e-5, softmax scale
1/sqrt(d_h), loss = 1/2 mean over b*s*d of (y - T)^2 on the stack output.

Canonical flat parameter layout of one layer (row = input feature, y = x W):
    ln1.w[d], ln1.b[d], Wqkv[d][3d], bqkv[3d], Wo[d][d], bo[d],
    ln2.w[d], ln2.b[d], W1[d][4d], b1[4d], W2[4d][d], b2[d]
Wqkv columns are [Q | K | V]; head h owns columns h*d_h ... (h+1)*d_h-1 of each.

The layer (per sequence x in R^{s x d}) -- O3 of SURVEY.md section 8(c):
    a  = LN(x; g1, b1)
    qkv = a Wqkv + bqkv ;  S_h = q_h k_h^T / sqrt(d_h) (+ causal mask) ;  P_h = softmax(S_h)
    o  = concat_h P_h v_h
    h1 = x + o Wo + bo
    c  = LN(h1; g2, b2)
    u  = c W1 + b1 ;  g = u Phi(u)
    y  = h1 + g W2 + b2

Post-LN option (``LayerCfg.post_ln``, reading A-16): the original transformer encoder that P:150
follows ("following the original approach [Vaswani et al.]") normalises after each residual add,
with the same parameters:
    h1 = LN(x + Attn(x) Wo + bo; g1, b1) ;  y = LN(h1 + GELU(h1 W1 + b1) W2 + b2; g2, b2)
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

LN_EPS = 1e-5


def layer_param_count(d: int, ffn_mult: int = 4) -> int:
    """p_l = (4 + 2 n_I) d^2 + 13 d."""
    return (4 + 2 * ffn_mult) * d * d + 13 * d


def param_count(d: int, layers: int, ffn_mult: int = 4) -> int:
    """p = d_l * p_l."""
    return layers * layer_param_count(d, ffn_mult)


def layer_offsets(d: int, ffn_mult: int = 4) -> dict[str, tuple[int, tuple[int, ...]]]:
    """Offsets and shapes of each tensor in the canonical flat layout (module docstring)."""
    f = ffn_mult * d
    spec = [
        ("ln1_w", (d,)), ("ln1_b", (d,)),
        ("Wqkv", (d, 3 * d)), ("bqkv", (3 * d,)),
        ("Wo", (d, d)), ("bo", (d,)),
        ("ln2_w", (d,)), ("ln2_b", (d,)),
        ("W1", (d, f)), ("b1", (f,)),
        ("W2", (f, d)), ("b2", (d,)),
    ]
    out, off = {}, 0
    for name, shape in spec:
        out[name] = (off, shape)
        off += int(np.prod(shape))
    assert off == layer_param_count(d, ffn_mult)
    return out


def unpack(flat: np.ndarray, d: int, ffn_mult: int = 4) -> dict[str, np.ndarray]:
    """Views of one layer's flat parameter vector, by name."""
    return {k: flat[o:o + int(np.prod(s))].reshape(s) for k, (o, s) in layer_offsets(d, ffn_mult).items()}


@dataclass(frozen=True)
class LayerCfg:
    d: int
    heads: int
    causal: bool = True
    ffn_mult: int = 4
    ln_eps: float = LN_EPS
    post_ln: bool = False   # reading A-16: the "original approach" places LN after each residual add

    @property
    def dh(self) -> int:
        return self.d // self.heads


# ----------------------------------------------------------------------------- pieces

def layernorm_fwd(x, w, b, eps):
    """Row-wise LayerNorm with biased variance (reading A-1)."""
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + eps)
    xhat = (x - mu) * rstd
    return xhat * w + b, (xhat, rstd)


def layernorm_bwd(dout, w, cache):
    """dx = rstd * (dxhat - mean(dxhat) - xhat * mean(dxhat * xhat)), dxhat = dout * w  (O5)."""
    xhat, rstd = cache
    dxhat = dout * w
    dx = rstd * (dxhat - dxhat.mean(axis=-1, keepdims=True)
                 - xhat * (dxhat * xhat).mean(axis=-1, keepdims=True))
    dw = (dout * xhat).reshape(-1, w.shape[0]).sum(axis=0)
    db = dout.reshape(-1, w.shape[0]).sum(axis=0)
    return dx, dw, db


try:  # library primitive for erf (a step the definition names, not a reformulation)
    from scipy.special import erf as _erf
except ImportError:  # pragma: no cover
    _erf = np.vectorize(math.erf, otypes=[np.float64])


def gelu(u):
    """Exact GELU, g = u * Phi(u), Phi the standard normal CDF (reading A-1)."""
    return u * 0.5 * (1.0 + _erf(u / math.sqrt(2.0)))


def gelu_grad(u):
    """GELU'(u) = Phi(u) + u * phi(u)  (O5)."""
    phi = np.exp(-0.5 * u * u) / math.sqrt(2.0 * math.pi)
    Phi = 0.5 * (1.0 + _erf(u / math.sqrt(2.0)))
    return Phi + u * phi


def attention_fwd(q, k, v, causal):
    """Per head: P = softmax(q k^T / sqrt(d_h) + mask), o = P v.  q,k,v: [b, heads, s, d_h]."""
    dh = q.shape[-1]
    S = q @ np.swapaxes(k, -1, -2) / math.sqrt(dh)
    if causal:
        s = q.shape[-2]
        S = np.where(np.tril(np.ones((s, s), dtype=bool)), S, -np.inf)
    S = S - S.max(axis=-1, keepdims=True)
    P = np.exp(S)
    P = P / P.sum(axis=-1, keepdims=True)
    return P @ v, P


def attention_bwd(do, q, k, v, P):
    """dS = P (dP - rowsum(dP P)); dq = dS k / sqrt(d_h); dk = dS^T q / sqrt(d_h); dv = P^T do  (O5)."""
    dh = q.shape[-1]
    dv = np.swapaxes(P, -1, -2) @ do
    dP = do @ np.swapaxes(v, -1, -2)
    dS = P * (dP - (dP * P).sum(axis=-1, keepdims=True))
    dq = dS @ k / math.sqrt(dh)
    dk = np.swapaxes(dS, -1, -2) @ q / math.sqrt(dh)
    return dq, dk, dv


def _split_heads(t, heads):
    b, s, d = t.shape
    return t.reshape(b, s, heads, d // heads).transpose(0, 2, 1, 3)


def _merge_heads(t):
    b, h, s, dh = t.shape
    return t.transpose(0, 2, 1, 3).reshape(b, s, h * dh)


# ----------------------------------------------------------------------------- layer

def layer_forward(x: np.ndarray, flat: np.ndarray, cfg: LayerCfg):
    """Forward of one layer on x: [b, s, d] (fp64).  Returns (y, cache)."""
    if cfg.post_ln:
        return layer_forward_post(x, flat, cfg)
    p = unpack(flat, cfg.d, cfg.ffn_mult)
    d = cfg.d
    a, ln1c = layernorm_fwd(x, p["ln1_w"], p["ln1_b"], cfg.ln_eps)
    qkv = a @ p["Wqkv"] + p["bqkv"]
    q = _split_heads(qkv[..., 0:d], cfg.heads)
    k = _split_heads(qkv[..., d:2 * d], cfg.heads)
    v = _split_heads(qkv[..., 2 * d:3 * d], cfg.heads)
    oh, P = attention_fwd(q, k, v, cfg.causal)
    o = _merge_heads(oh)
    h1 = x + o @ p["Wo"] + p["bo"]
    c, ln2c = layernorm_fwd(h1, p["ln2_w"], p["ln2_b"], cfg.ln_eps)
    u = c @ p["W1"] + p["b1"]
    g = gelu(u)
    y = h1 + g @ p["W2"] + p["b2"]
    cache = dict(x=x, a=a, ln1c=ln1c, q=q, k=k, v=v, P=P, o=o, h1=h1, c=c, ln2c=ln2c, u=u, g=g)
    return y, cache


def layer_backward(dy: np.ndarray, cache: dict, flat: np.ndarray, cfg: LayerCfg):
    """Reverse mode through ``layer_forward``.  Returns (dx, dflat) with dflat in canonical layout."""
    if cfg.post_ln:
        return layer_backward_post(dy, cache, flat, cfg)
    p = unpack(flat, cfg.d, cfg.ffn_mult)
    d = cfg.d
    grads = np.zeros_like(flat)
    gv = unpack(grads, cfg.d, cfg.ffn_mult)

    def flat2(t):
        return t.reshape(-1, t.shape[-1])

    # y = h1 + g W2 + b2
    gv["W2"][...] = flat2(cache["g"]).T @ flat2(dy)
    gv["b2"][...] = flat2(dy).sum(axis=0)
    dg = dy @ p["W2"].T
    du = dg * gelu_grad(cache["u"])
    # u = c W1 + b1
    gv["W1"][...] = flat2(cache["c"]).T @ flat2(du)
    gv["b1"][...] = flat2(du).sum(axis=0)
    dc = du @ p["W1"].T
    # c = LN(h1)
    dh1, gv["ln2_w"][...], gv["ln2_b"][...] = layernorm_bwd(dc, p["ln2_w"], cache["ln2c"])
    dh1 = dh1 + dy
    # h1 = x + o Wo + bo
    gv["Wo"][...] = flat2(cache["o"]).T @ flat2(dh1)
    gv["bo"][...] = flat2(dh1).sum(axis=0)
    do = dh1 @ p["Wo"].T
    dq, dk, dv = attention_bwd(_split_heads(do, cfg.heads), cache["q"], cache["k"], cache["v"], cache["P"])
    dqkv = np.concatenate([_merge_heads(dq), _merge_heads(dk), _merge_heads(dv)], axis=-1)
    # qkv = a Wqkv + bqkv
    gv["Wqkv"][...] = flat2(cache["a"]).T @ flat2(dqkv)
    gv["bqkv"][...] = flat2(dqkv).sum(axis=0)
    da = dqkv @ p["Wqkv"].T
    dx, gv["ln1_w"][...], gv["ln1_b"][...] = layernorm_bwd(da, p["ln1_w"], cache["ln1c"])
    dx = dx + dh1
    return dx, grads


def _attn_block(a, p, cfg):
    d = cfg.d
    qkv = a @ p["Wqkv"] + p["bqkv"]
    q = _split_heads(qkv[..., 0:d], cfg.heads)
    k = _split_heads(qkv[..., d:2 * d], cfg.heads)
    v = _split_heads(qkv[..., 2 * d:3 * d], cfg.heads)
    oh, P = attention_fwd(q, k, v, cfg.causal)
    return q, k, v, P, _merge_heads(oh)


def layer_forward_post(x: np.ndarray, flat: np.ndarray, cfg: LayerCfg):
    """Post-LN layer of the original transformer encoder (reading A-16), same parameters:
    h1 = LN1(x + Attn(x) Wo + bo),  y = LN2(h1 + GELU(h1 W1 + b1) W2 + b2)."""
    p = unpack(flat, cfg.d, cfg.ffn_mult)
    q, k, v, P, o = _attn_block(x, p, cfg)
    s1 = x + o @ p["Wo"] + p["bo"]
    h1, ln1c = layernorm_fwd(s1, p["ln1_w"], p["ln1_b"], cfg.ln_eps)
    u = h1 @ p["W1"] + p["b1"]
    g = gelu(u)
    s2 = h1 + g @ p["W2"] + p["b2"]
    y, ln2c = layernorm_fwd(s2, p["ln2_w"], p["ln2_b"], cfg.ln_eps)
    cache = dict(x=x, q=q, k=k, v=v, P=P, o=o, ln1c=ln1c, h1=h1, u=u, g=g, ln2c=ln2c)
    return y, cache


def layer_backward_post(dy: np.ndarray, cache: dict, flat: np.ndarray, cfg: LayerCfg):
    """Reverse mode through ``layer_forward_post``."""
    p = unpack(flat, cfg.d, cfg.ffn_mult)
    grads = np.zeros_like(flat)
    gv = unpack(grads, cfg.d, cfg.ffn_mult)

    def flat2(t):
        return t.reshape(-1, t.shape[-1])

    # y = LN2(s2)
    ds2, gv["ln2_w"][...], gv["ln2_b"][...] = layernorm_bwd(dy, p["ln2_w"], cache["ln2c"])
    # s2 = h1 + g W2 + b2
    gv["W2"][...] = flat2(cache["g"]).T @ flat2(ds2)
    gv["b2"][...] = flat2(ds2).sum(axis=0)
    du = (ds2 @ p["W2"].T) * gelu_grad(cache["u"])
    # u = h1 W1 + b1
    gv["W1"][...] = flat2(cache["h1"]).T @ flat2(du)
    gv["b1"][...] = flat2(du).sum(axis=0)
    dh1 = du @ p["W1"].T + ds2
    # h1 = LN1(s1)
    ds1, gv["ln1_w"][...], gv["ln1_b"][...] = layernorm_bwd(dh1, p["ln1_w"], cache["ln1c"])
    # s1 = x + o Wo + bo
    gv["Wo"][...] = flat2(cache["o"]).T @ flat2(ds1)
    gv["bo"][...] = flat2(ds1).sum(axis=0)
    do = ds1 @ p["Wo"].T
    dq, dk, dv = attention_bwd(_split_heads(do, cfg.heads), cache["q"], cache["k"], cache["v"], cache["P"])
    dqkv = np.concatenate([_merge_heads(dq), _merge_heads(dk), _merge_heads(dv)], axis=-1)
    # qkv = x Wqkv + bqkv
    gv["Wqkv"][...] = flat2(cache["x"]).T @ flat2(dqkv)
    gv["bqkv"][...] = flat2(dqkv).sum(axis=0)
    dx = dqkv @ p["Wqkv"].T + ds1
    return dx, grads


def mse_loss(y: np.ndarray, T: np.ndarray):
    """l = 1/2 mean over b*s*d of (y - T)^2 and its seed gradient dY = (y - T)/(b s d)  (reading A-2)."""
    diff = y - T
    return 0.5 * float(np.mean(diff * diff)), diff / diff.size


def stack_forward(x, params: list[np.ndarray], cfg: LayerCfg):
    """Forward through all layers, keeping per-layer caches (no checkpointing)."""
    caches = []
    for flat in params:
        x, c = layer_forward(x, flat, cfg)
        caches.append(c)
    return x, caches


def stack_backward(dy, caches, params, cfg: LayerCfg):
    grads = [None] * len(params)
    for l in reversed(range(len(params))):
        dy, grads[l] = layer_backward(dy, caches[l], params[l], cfg)
    return dy, grads
