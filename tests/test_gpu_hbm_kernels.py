"""Single HBM-bound kernels of the step (LayerNorm forward / backward with the dgamma / dbeta column
partials, bias column sums, sharded AdamW, the reduce-scatter fused into AdamW, the peer-slice
reduction) against the fp64 oracle's formulas, ELEMENT BY ELEMENT, through the test hooks
(include/lga_testing.h).  Row counts are ragged and the widths cover every kernel variant the step
dispatches: the block kernel (d % 128 != 0), the warp-per-row kernels (d = 128 k up to 4096) and the
fused LayerNorm backward (d = 1024, 2048).

Tolerances: fp32 outputs |a - b| <= 1e-5 (|b| + scale); a bf16 output is the round-to-nearest of the
fp32 value, so it is held to 2^-8 relative (one bf16 ulp) on top of that."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle import model as om  # noqa: E402
from oracle import schedule as osch  # noqa: E402
from paper_2106_02679_b200 import _abi  # noqa: E402

L = _abi.lib()
VP, I, I64, F = C.c_void_p, C.c_int, C.c_int64, C.c_float
L.lgatest_ln_fwd.argtypes = [VP, VP, VP, I, VP, I, VP, I, I, F, VP]
L.lgatest_ln_bwd.argtypes = [VP, VP, VP, VP, I, VP, VP, VP, I, VP, VP, VP, VP, VP, I, I, VP]
L.lgatest_ln_bwd_partial_floats.restype = I64
L.lgatest_ln_bwd_partial_floats.argtypes = [I, I]
L.lgatest_colsum.argtypes = [VP, I, I64, I, I, VP, VP, I, VP, VP]
L.lgatest_colsum_partial_floats.restype = I64
L.lgatest_colsum_partial_floats.argtypes = [I, I]
L.lgatest_adamw.argtypes = [VP, I, F, VP, VP, VP, VP, I, VP, I64, F, F, F, F, F, VP, VP]
L.lgatest_adamw_rs.argtypes = [VP, I64, I, I, F, VP, VP, VP, VP, I, VP, I64, F, F, F, F, F, VP, VP]
L.lgatest_peer_reduce.argtypes = [VP, I64, I, I, VP, I, VP, I64, VP]
for f in ("lgatest_ln_fwd", "lgatest_ln_bwd", "lgatest_colsum", "lgatest_adamw", "lgatest_adamw_rs", "lgatest_peer_reduce"):
    getattr(L, f).restype = I


def P(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def DT(t):
    return 0 if t.dtype == torch.float32 else 1


def S():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def f64(t):
    return t.detach().double().cpu().numpy()


def close(a, b, rtol=1e-5, scale=None, bf16=False):
    """element-wise |a - b| <= rtol (|b| + scale) (+ one bf16 ulp of |b| for a bf16 output)"""
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    scale = np.sqrt(np.mean(b * b)) if scale is None else scale
    bound = rtol * (np.abs(b) + scale) + (2.0 ** -8) * np.abs(b) * bf16
    bad = np.abs(a - b) > bound
    assert not bad.any(), (int(bad.sum()), float(np.max(np.abs(a - b) / (np.abs(b) + scale))))


WIDTHS = [64, 192, 256, 768, 1024, 2048, 4096]   # block kernel, warp kernels, fused backward (1024, 2048)


def _ln_inputs(rows, d, pdt, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(rows, d, device="cuda", generator=g) * 1.7 + torch.randn(rows, 1, device="cuda", generator=g)
    gamma = (1 + 0.1 * torch.randn(d, device="cuda", generator=g)).to(pdt)
    beta = (0.05 * torch.randn(d, device="cuda", generator=g)).to(pdt)
    return g, x, gamma, beta


@pytest.mark.parametrize("d", WIDTHS)
@pytest.mark.parametrize("bf", [False, True])
def test_layernorm_fwd(d, bf):
    rows = 333
    pdt = torch.bfloat16 if bf else torch.float32
    _, x, gamma, beta = _ln_inputs(rows, d, pdt, d)
    y = torch.empty(rows, d, device="cuda", dtype=pdt)
    stats = torch.empty(rows, 2, device="cuda")
    assert L.lgatest_ln_fwd(P(x), P(gamma), P(beta), DT(gamma), P(y), DT(y), P(stats), rows, d, 1e-5, S()) == 0
    torch.cuda.synchronize()
    ref, (xhat, rstd) = om.layernorm_fwd(f64(x), f64(gamma), f64(beta), 1e-5)
    close(f64(y), ref, bf16=bf)
    close(f64(stats[:, 0]), f64(x).mean(axis=1), scale=np.abs(f64(x)).mean())
    close(f64(stats[:, 1]), rstd[:, 0])


@pytest.mark.parametrize("d", WIDTHS)
@pytest.mark.parametrize("bf,resid,extra", [(False, True, False), (True, True, True), (False, False, True),
                                            (True, True, False)])
def test_layernorm_bwd_and_gamma_beta_grads(d, bf, resid, extra):
    """LayerNorm backward: dx (+ resid), dgamma, dbeta and, with `extra`, the column sums of resid and dx that the
    step takes as bias gradients (pre-LN LN2: db2 = sum dY, db_o = sum dh1)."""
    rows = 333 if d != 2048 else 1000   # several row groups of the fused kernel, ragged tail
    pdt = torch.bfloat16 if bf else torch.float32
    g, x, gamma, beta = _ln_inputs(rows, d, pdt, 7 * d + 1)
    y = torch.empty(rows, d, device="cuda", dtype=pdt)
    stats = torch.empty(rows, 2, device="cuda")
    assert L.lgatest_ln_fwd(P(x), P(gamma), P(beta), DT(gamma), P(y), DT(y), P(stats), rows, d, 1e-5, S()) == 0
    dout = torch.randn(rows, d, device="cuda", generator=g)
    res = torch.randn(rows, d, device="cuda", generator=g) if resid else None
    dx = torch.full((rows, d), float("nan"), device="cuda")
    dxe = torch.empty(rows, d, device="cuda", dtype=pdt)
    dgam = torch.full((d,), float("nan"), device="cuda")
    dbet = torch.full((d,), float("nan"), device="cuda")
    sres = torch.full((d,), float("nan"), device="cuda") if extra else None
    sdx = torch.full((d,), float("nan"), device="cuda") if extra else None
    part = torch.empty(2 * int(L.lgatest_ln_bwd_partial_floats(rows, d)), device="cuda")
    assert L.lgatest_ln_bwd(P(dout), P(x), P(stats), P(gamma), DT(gamma), P(res), P(dx), P(dxe), DT(dxe), P(dgam),
                            P(dbet), P(sres), P(sdx), P(part), rows, d, S()) == 0
    torch.cuda.synchronize()
    _, cache = om.layernorm_fwd(f64(x), f64(gamma), f64(beta), 1e-5)
    rdx, rdg, rdb = om.layernorm_bwd(f64(dout), f64(gamma), cache)
    if resid:
        rdx = rdx + f64(res)
    close(f64(dx), rdx)
    close(f64(dxe), rdx, bf16=bf)
    # column sums over `rows` terms: fp32 accumulation error grows like sqrt(rows) ulps
    close(f64(dgam), rdg, rtol=2e-5)
    close(f64(dbet), rdb, rtol=2e-5)
    if extra:
        close(f64(sres), f64(res).sum(0) if resid else np.zeros(d), rtol=2e-5, scale=1.0 if not resid else None)
        close(f64(sdx), rdx.sum(0), rtol=2e-5)


@pytest.mark.parametrize("n,ldx", [(64, 64), (768, 2304), (3 * 1024, 3 * 1024), (8192, 8192), (100, 132)])
@pytest.mark.parametrize("xbf,acc,obf", [(False, False, False), (True, True, False), (True, False, True)])
def test_bias_column_sums(n, ldx, xbf, acc, obf):
    rows = 1000
    g = torch.Generator(device="cuda").manual_seed(n + ldx)
    X = torch.randn(rows, ldx, device="cuda", generator=g).to(torch.bfloat16 if xbf else torch.float32)
    acc_in = torch.randn(n, device="cuda", generator=g) if acc else None
    out = torch.empty(n, device="cuda", dtype=torch.bfloat16 if obf else torch.float32)
    part = torch.empty(int(L.lgatest_colsum_partial_floats(rows, n)), device="cuda")
    assert L.lgatest_colsum(P(X), DT(X), ldx, rows, n, P(acc_in), P(out), DT(out), P(part), S()) == 0
    torch.cuda.synchronize()
    ref = f64(X)[:, :n].sum(axis=0) + (f64(acc_in) if acc else 0.0)
    close(f64(out), ref, rtol=2e-5, bf16=obf)


def _adam_state(n, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    master = 0.02 * torch.randn(n, device="cuda", generator=g)
    return g, master, torch.zeros(n, device="cuda"), torch.zeros(n, device="cuda")


HP = dict(lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1)


@pytest.mark.parametrize("gbf,pbf", [(False, False), (True, True), (False, True)])
def test_adamw_three_steps(gbf, pbf):
    """AdamW (torch semantics, t = 1, 2, 3, decoupled weight decay) against oracle.schedule.AdamW in fp64:
    master / m / v / the kept gradient element by element, the 16-bit parameter copy within one ulp."""
    n = 100_003   # ragged: the float4 body plus a scalar tail
    g, master, m, v = _adam_state(n, 11)
    opt = osch.AdamW(**HP)
    theta = f64(master)
    st = opt.init_state(theta)
    pout = torch.empty(n, device="cuda", dtype=torch.bfloat16 if pbf else torch.float32)
    keep = torch.empty(n, device="cuda")
    gscale = 1.0 / 8
    for t in range(1, 4):
        gin = (torch.randn(n, device="cuda", generator=g) * 10.0 ** (-t)).to(torch.bfloat16 if gbf else torch.float32)
        tstep = torch.tensor([t], device="cuda", dtype=torch.int64)
        assert L.lgatest_adamw(P(gin), DT(gin), gscale, P(master), P(m), P(v), P(pout), DT(pout), P(keep), n, HP["lr"],
                               HP["beta1"], HP["beta2"], HP["eps"], HP["weight_decay"], P(tstep), S()) == 0
        torch.cuda.synchronize()
        gg = f64(gin) * gscale
        theta = opt.update(theta, gg, st)
        close(f64(keep), gg)
        close(f64(m), st["m"])
        close(f64(v), st["v"], rtol=3e-5)
        close(f64(master), theta, scale=HP["lr"])
        close(f64(pout), theta, scale=HP["lr"], bf16=pbf)


@pytest.mark.parametrize("D,gbf", [(2, True), (3, False), (8, True)])
def test_adamw_fused_reduce_scatter(D, gbf):
    """The reduce-scatter fused into AdamW: this rank's shard gradient = sum over the D replicas' staging slices
    in fixed rank order (here D buffers of one process stand in for the peers' IPC-mapped staging)."""
    n, goff = 65_536 + 64, 4096
    g, master, m, v = _adam_state(n, 12 + D)
    dt = torch.bfloat16 if gbf else torch.float32
    bufs = [torch.randn(goff + n + 128, device="cuda", generator=g).to(dt) for _ in range(D)]
    gbase = torch.tensor([b.data_ptr() for b in bufs], device="cuda", dtype=torch.int64)
    pout = torch.empty(n, device="cuda", dtype=torch.bfloat16)
    keep = torch.empty(n, device="cuda")
    tstep = torch.tensor([1], device="cuda", dtype=torch.int64)
    gscale = 1.0 / (D * 4)
    opt = osch.AdamW(**HP)
    theta0 = f64(master)
    assert L.lgatest_adamw_rs(P(gbase), goff, D, 1 if gbf else 0, gscale, P(master), P(m), P(v), P(pout), 1, P(keep), n,
                              HP["lr"], HP["beta1"], HP["beta2"], HP["eps"], HP["weight_decay"], P(tstep), S()) == 0
    torch.cuda.synchronize()
    gsum = sum(f64(b)[goff:goff + n] for b in bufs) * gscale
    theta = opt.update(theta0, gsum, opt.init_state(theta0))
    close(f64(keep), gsum)
    close(f64(master), theta, scale=HP["lr"])
    close(f64(pout), theta, scale=HP["lr"], bf16=True)


@pytest.mark.parametrize("D,gbf", [(2, True), (4, False)])
def test_peer_reduce(D, gbf):
    n, goff = 40_960, 1024
    g = torch.Generator(device="cuda").manual_seed(40 + D)
    dt = torch.bfloat16 if gbf else torch.float32
    bufs = [torch.randn(goff + n, device="cuda", generator=g).to(dt) for _ in range(D)]
    gbase = torch.tensor([b.data_ptr() for b in bufs], device="cuda", dtype=torch.int64)
    ref = sum(f64(b)[goff:goff + n] for b in bufs)
    # unpartitioned all-reduce, phase 1: the staging dtype output
    out = torch.empty(n, device="cuda", dtype=dt)
    assert L.lgatest_peer_reduce(P(gbase), goff, D, 1 if gbf else 0, None, 0, P(out), n, S()) == 0
    # STANDARD: fp32 accumulation over micro-batches (first, then += )
    acc = torch.full((n,), float("nan"), device="cuda")
    assert L.lgatest_peer_reduce(P(gbase), goff, D, 1 if gbf else 0, P(acc), 1, None, n, S()) == 0
    assert L.lgatest_peer_reduce(P(gbase), goff, D, 1 if gbf else 0, P(acc), 0, None, n, S()) == 0
    torch.cuda.synchronize()
    close(f64(out), ref, bf16=gbf)
    close(f64(acc), 2 * ref)
