"""Per-tile pipeline timeline of the attention forward from an LGA_FWD_TRACE build (development tool).
CTA 0's first work item (the heaviest query tile).  SM cycles relative to S(0) issue."""
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
for _ in range(3):
    L.lgatest_attn_fwd(1, nseq, s, H, dh, 1, kb.P(qkv), kb.P(o), kb.P(lse), st)
torch.cuda.synchronize()
buf = np.zeros((40, 8), dtype=np.int64)
L.lgatest_fwd_trace.argtypes = [C.c_void_p]
assert L.lgatest_fwd_trace(buf.ctypes.data) == 0
t0 = buf[0, 0]
print(" j   S issue  p_full0  p_full1 | sm: S seen  exps done  o_done ok  P0 arrive  P1 arrive | exp dur  iter")
prev = None
for j in range(16):
    r = buf[j] - t0
    it = r[0] - prev if prev is not None else 0
    prev = r[0]
    print(f"{j:2d} {r[0]:9d} {r[1]:8d} {r[2]:8d} | {r[3]:10d} {r[4]:10d} {r[5]:10d} {r[6]:10d} {r[7]:10d} | {r[4] - r[3]:7d} {it:5d}")

# per item of CTA 0 (MMA start, last PV issued, epilogue start / end) and the CTAs' start / end spread
items = np.zeros((64, 4), dtype=np.int64)
cta = np.zeros((256, 2), dtype=np.int64)
L.lgatest_fwd_trace_items.argtypes = [C.c_void_p, C.c_void_p]
assert L.lgatest_fwd_trace_items(items.ctypes.data, cta.ctypes.data) == 0
n_items = (s // 128) * H * nseq
per = [len(range(i, n_items, 148)) for i in range(1)][0]
nqt = s // 128
print("\nCTA 0 items: it  qt  tiles  mma_start  last_pv  epi_start  epi_end | span  cycles/tile  gap_to_next")
G = 16
for it in range(min(per, 64)):
    t = it * 148
    chunk, w = t // (G * nqt), t % (G * nqt)
    np_ = min(G, H * nseq - chunk * G)
    qt = nqt - 1 - w // np_
    r = items[it] - items[0, 0]
    nxt = items[it + 1, 0] - items[0, 0] if it + 1 < per else r[3]
    span = r[3] - r[0]
    print(f"  {it:3d} {qt:3d} {qt + 1:6d} {r[0]:10d} {r[1]:8d} {r[2]:9d} {r[3]:8d} | {span:6d} {span / (qt + 1):9.0f} {nxt - r[0]:9d}")
g = cta[:148]
t0 = g[:, 0].min()
st, en = (g[:, 0] - t0) / 1e3, (g[:, 1] - t0) / 1e3
print(f"\nCTA start spread {st.max():.1f} us; end min/median/max {en.min():.1f} / {np.median(en):.1f} / {en.max():.1f} us")

# item boundaries of CTA 0: when the MMA warp starts / ends waiting for the epilogue's o_free before the next
# item's first PV, and when the epilogue saw the item's PVs done / released the accumulators
if hasattr(L, "lgatest_fwd_trace_items2"):
    it2 = np.zeros((64, 4), dtype=np.int64)
    L.lgatest_fwd_trace_items2.argtypes = [C.c_void_p]
    assert L.lgatest_fwd_trace_items2(it2.ctypes.data) == 0
    print("\nit  o_free wait (MMA, next item)   epi: PV done  o_free arrive | MMA wait  epi PV->free")
    for it in range(1, min(per, 64)):
        a = it2[it] - items[0, 0]
        e = it2[it - 1] - items[0, 0]
        print(f"{it:3d} {a[0]:10d} {a[1]:10d} | {e[2]:10d} {e[3]:10d} | {a[1] - a[0]:8d} {e[3] - e[2]:8d}")
