"""Per-iteration pipeline timeline of the dK/dV kernel from an LGA_BWD_TRACE build (development tool).

    LGA_EXTRA_DEFINES=LGA_BWD_TRACE python -m paper_2106_02679_b200.build --force
    python tools/bwd_trace.py [kt ...]

Columns (SM cycles relative to the CTA start): p_full seen by the MMA issuer, g_done(i) seen, q_full(i)
seen (issue of S(i)), element-wise leader of the group: S(i) seen / P(i) arrive.
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tools.kbench as kb  # noqa: E402

L = kb.L
nseq, s, H, dh = 16, 2048, 16, 128
d = H * dh
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
qkv = torch.randn(nseq * s, 3 * d, device="cuda").bfloat16()
o = torch.empty(nseq * s, d, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(nseq, H, s, device="cuda")
dO = torch.randn(nseq * s, d, device="cuda").bfloat16()
dsum = torch.empty(nseq, H, s, device="cuda")
dqkv = torch.empty_like(qkv)
P = kb.P
L.lgatest_attn_fwd(1, nseq, s, H, dh, 1, P(qkv), P(o), P(lse), st)
for _ in range(3):
    L.lgatest_attn_bwd(1, nseq, s, H, dh, 1, P(qkv), P(o), P(lse), P(dO), P(dsum), P(dqkv), st)
torch.cuda.synchronize()
buf = np.zeros((16, 40, 8), dtype=np.int64)
L.lgatest_bwd_trace.argtypes = [C.c_void_p]
assert L.lgatest_bwd_trace(buf.ctypes.data) == 0
kts = [int(x) for x in sys.argv[1:]] or [0, 8, 15]
for kt in kts:
    t = buf[kt]
    t0 = t[39, 0]
    nq = 32 - 2 * kt
    print(f"kt={kt} nq={nq}: K/V landed {t[39, 1] - t0}, end {t[39, 2] - t0} cycles "
          f"({(t[39, 2] - t[39, 1]) / nq:.0f} per iteration after K/V)")
    print("   i   q_full(S)  S seen(EW)  P arrive    p_full(MMA)  g_done     | EW dur  P->MMA  iter")
    prev = None
    for i in range(nq):
        r = t[i] - t0
        ew = r[5] - r[4]
        lat = r[0] - r[5]
        it = (r[0] - prev) if prev is not None else 0
        prev = r[0]
        print(f"  {i:2d} {r[3]:10d} {r[4]:10d} {r[5]:10d} {r[0]:12d} {r[2] if r[2] > 0 else 0:10d} | {ew:6d} {lat:6d} {it:6d}")

# dQ kernel: CTA 0 of (sequence 0, head 0) -- the heaviest query tile (16 key tiles)
if hasattr(L, "lgatest_dq_trace"):
    qb = np.zeros((40, 8), dtype=np.int64)
    L.lgatest_dq_trace.argtypes = [C.c_void_p]
    assert L.lgatest_dq_trace(qb.ctypes.data) == 0
    t0 = qb[0, 0]
    print("dQ: j  K seen  S issue  |  EW: S seen  S loaded  P arrive(w4)  P arrive(w19) | p_full(MMA)  | EW dur  iter")
    prev = None
    for j in range(16):
        r = qb[j] - t0
        it = r[1] - prev if prev is not None else 0
        prev = r[1]
        print(f"  {j:2d} {r[0]:8d} {r[1]:8d} | {r[3]:8d} {r[4]:8d} {r[5]:8d} {r[6]:8d} | {r[2]:8d} | {r[5] - r[3]:6d} {it:5d}")
