"""Per-kernel micro-benchmarks through the test hooks (include/lga_testing.h), CUDA-event timed.

    python tools/kbench.py [attn] [gemm] [--dh 128 --seq 2048 --nseq 16 --heads 16]

Prints one line per kernel: shape, ms per launch, achieved TFLOP/s (algorithmic flops).
Development tool; bench.py is the measurement of record.
"""
import argparse
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2106_02679_b200 import _abi  # noqa: E402

L = _abi.lib()
L.lgatest_gemm.restype = C.c_int
L.lgatest_gemm.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.c_int64,
                           C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                           C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.c_void_p]
L.lgatest_attn_fwd.restype = C.c_int
L.lgatest_attn_fwd.argtypes = [C.c_int] * 6 + [C.c_void_p] * 3 + [C.c_void_p]
L.lgatest_attn_bwd.restype = C.c_int
L.lgatest_attn_bwd.argtypes = [C.c_int] * 6 + [C.c_void_p] * 8 + [C.c_void_p]


def P(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def timeit(fn, iters=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def attn(args):
    nseq, s, H, dh = args.nseq, args.seq, args.heads, args.dh
    d = H * dh
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    qkv = torch.randn(nseq * s, 3 * d, device="cuda").bfloat16()
    o = torch.empty(nseq * s, d, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(nseq, H, s, device="cuda")
    dO = torch.randn(nseq * s, d, device="cuda").bfloat16()
    dsum = torch.empty(nseq, H, s, device="cuda")
    dqkv = torch.empty_like(qkv)
    flops = 4.0 * dh * (s * (s + 1) / 2) * H * nseq
    for path, name in ((1, "fwd tcgen05"),):
        ms = timeit(lambda: L.lgatest_attn_fwd(path, nseq, s, H, dh, 1, P(qkv), P(o), P(lse), st))
        print(f"attn {name:14s} nseq={nseq} s={s} H={H} dh={dh}: {ms:.3f} ms  {flops / ms / 1e9:.1f} TFLOP/s")
    L.lgatest_attn_fwd(1, nseq, s, H, dh, 1, P(qkv), P(o), P(lse), st)
    s128 = (s + 127) // 128 * 128
    ds = torch.empty(nseq * H * s128 * s128, device="cuda", dtype=torch.bfloat16)
    # the step passes the qkv-bias column partials (one row per (sequence, key tile, lane quadrant))
    cs = torch.empty(nseq * (s128 // 128) * 4 * 3 * d, device="cuda")
    for name, ws, csum in (("bwd 5-mm", ds, cs), ("bwd 5-mm nocs", ds, None), ("bwd 7-mm", None, cs)):
        ms = timeit(lambda: L.lgatest_attn_bwd(1, nseq, s, H, dh, 1, P(qkv), P(o), P(lse), P(dO), P(dsum), P(dqkv),
                                               P(csum), P(ws), st))
        print(f"attn {name:14s} nseq={nseq} s={s} H={H} dh={dh}: {ms:.3f} ms  {2 * flops / ms / 1e9:.1f} TFLOP/s (algorithmic 2x fwd)")


def gemm(args):
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    T, d = args.tokens, args.d
    f = 4 * d
    cases = [
        ("qkv fwd   ", T, 3 * d, d, True, False, 1, "bias_bf16"),
        ("oproj fwd ", T, d, d, True, False, 0, "bias_res_f32"),
        ("ffn1 fwd  ", T, f, d, True, False, 1, "gelu"),
        ("ffn2 fwd  ", T, d, f, True, False, 0, "bias_res_f32"),
        ("ffn2 dgrad", T, f, d, True, True, 1, "gelu_bwd"),
        ("ffn1 dgrad", T, d, f, True, True, 0, "f32"),
        ("w1 wgrad  ", d, f, T, False, False, 0, "acc"),
        ("wqkv wgrad", d, 3 * d, T, False, False, 0, "acc"),
        ("wo wgrad  ", d, d, T, False, False, 0, "acc"),
    ]
    for name, M, N, K, ak, bk, outbf, kind in cases:
        A = torch.randn((M, K) if ak else (K, M), device="cuda").bfloat16()
        B = torch.randn((N, K) if bk else (K, N), device="cuda").bfloat16()
        out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16 if outbf else torch.float32)
        bias = torch.randn(N, device="cuda").bfloat16() if kind in ("bias_bf16", "bias_res_f32", "gelu") else None
        res = torch.randn(M, N, device="cuda") if kind == "bias_res_f32" else None
        acc = torch.randn(M, N, device="cuda") if kind == "acc" else None
        aux = torch.randn(M, N, device="cuda").bfloat16() if kind in ("gelu", "gelu_bwd") else None
        ek = 1 if kind == "gelu" else (2 if kind == "gelu_bwd" else 0)
        dt = lambda t: 0 if t is None or t.dtype == torch.float32 else 1
        fn = lambda: L.lgatest_gemm(1, M, N, K, P(A), A.shape[1], int(ak), P(B), B.shape[1], int(bk), ek, P(bias), dt(bias),
                                    P(res), P(acc), P(aux), dt(aux), P(out), N, dt(out), None, st)
        assert fn() == 0
        ms = timeit(fn)
        print(f"gemm {name} M={M} N={N} K={K} {kind:12s}: {ms:.3f} ms  {2.0 * M * N * K / ms / 1e9:.1f} TFLOP/s")


def ln(args):
    """LayerNorm forward / fused backward (with the 4 column sums) at the step's shape: DRAM GB/s."""
    T, d = args.tokens, args.d
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    VP, I = C.c_void_p, C.c_int
    L.lgatest_ln_fwd.argtypes = [VP, VP, VP, I, VP, I, VP, I, I, C.c_float, VP]
    L.lgatest_ln_bwd.argtypes = [VP, VP, VP, VP, I, VP, VP, VP, I, VP, VP, VP, VP, VP, I, I, VP]
    L.lgatest_ln_bwd_partial_floats.restype = C.c_int64
    x = torch.randn(T, d, device="cuda")
    g = torch.ones(d, device="cuda").bfloat16()
    b = torch.zeros(d, device="cuda").bfloat16()
    y = torch.empty(T, d, device="cuda", dtype=torch.bfloat16)
    stats = torch.empty(T, 2, device="cuda")
    fwd = lambda: L.lgatest_ln_fwd(P(x), P(g), P(b), 1, P(y), 1, P(stats), T, d, 1e-5, st)
    ms = timeit(fwd)
    print(f"ln fwd      T={T} d={d}: {ms:.3f} ms  {T * d * (4 + 2) / ms / 1e6:.0f} GB/s")
    dout, res = torch.randn(T, d, device="cuda"), torch.randn(T, d, device="cuda")
    dx = torch.empty(T, d, device="cuda")
    dxe = torch.empty(T, d, device="cuda", dtype=torch.bfloat16)
    v = [torch.empty(d, device="cuda") for _ in range(4)]
    part = torch.empty(2 * int(L.lgatest_ln_bwd_partial_floats(T, d)), device="cuda")
    bwd = lambda: L.lgatest_ln_bwd(P(dout), P(x), P(stats), P(g), 1, P(res), P(dx), P(dxe), 1, P(v[0]), P(v[1]), P(v[2]),
                                   P(v[3]), P(part), T, d, st)
    ms = timeit(bwd)
    print(f"ln bwd+sums T={T} d={d}: {ms:.3f} ms  {T * d * (3 * 4 + 4 + 2) / ms / 1e6:.0f} GB/s")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("what", nargs="*", default=["attn", "gemm"])
    ap.add_argument("--dh", type=int, default=128)
    ap.add_argument("--seq", type=int, default=2048)
    ap.add_argument("--nseq", type=int, default=16)
    ap.add_argument("--heads", type=int, default=16)
    ap.add_argument("--tokens", type=int, default=32768)
    ap.add_argument("--d", type=int, default=2048)
    a = ap.parse_args()
    if "attn" in a.what:
        attn(a)
    if "gemm" in a.what:
        gemm(a)
    if "ln" in a.what:
        ln(a)
