"""Per-iteration pipeline timeline of the persistent dK/dV kernel from an LGA_DKV_TRACE build (development tool).
CTA 0: global iterations g (64 queries x 128 keys each), SM cycles relative to the first S^T issue."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tools.kbench as kb  # noqa: E402

L = kb.L
P = kb.P
nseq, s, H, dh = 16, 2048, 16, 128
d = H * dh
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
qkv = torch.randn(nseq * s, 3 * d, device="cuda").bfloat16()
o = torch.empty(nseq * s, d, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(nseq, H, s, device="cuda")
dO = torch.randn(nseq * s, d, device="cuda").bfloat16()
dsum = torch.empty(nseq, H, s, device="cuda")
dqkv = torch.empty_like(qkv)
s128 = (s + 127) // 128 * 128
ds = torch.empty(nseq * H * s128 * s128, device="cuda", dtype=torch.bfloat16)
cs = torch.empty(nseq * (s128 // 128) * 4 * 3 * d, device="cuda")
L.lgatest_attn_fwd(1, nseq, s, H, dh, 1, P(qkv), P(o), P(lse), st)
for _ in range(3):
    L.lgatest_attn_bwd(1, nseq, s, H, dh, 1, P(qkv), P(o), P(lse), P(dO), P(dsum), P(dqkv), P(cs), P(ds), st)
torch.cuda.synchronize()
it = np.zeros((96, 8), dtype=np.int64)
items = np.zeros((32, 4), dtype=np.int64)
L.lgatest_dkv_trace.argtypes = [C.c_void_p, C.c_void_p]
assert L.lgatest_dkv_trace(it.ctypes.data, items.ctypes.data) == 0
t0 = it[0, 0]
print(" g   S^T    dP^T  | EW: S seen  P arrive | dV      dK     | EW dur  P->dV  S->seen  iter(S^T)")
prev = None
for g in range(64):
    r = it[g] - t0
    itv = r[0] - prev if prev is not None else 0
    prev = r[0]
    print(f"{g:2d} {r[0]:7d} {r[1]:7d} | {r[2]:9d} {r[3]:9d} | {r[4]:7d} {r[5]:7d} | {r[3] - r[2]:6d} {r[4] - r[3]:6d} {r[2] - r[1]:7d} {itv:6d}")
print("\nitems (CTA 0): drain start / end, MMA item start")
for i in range(8):
    r = items[i] - t0
    print(i, r[0], r[1], r[2], "drain", r[1] - r[0])
