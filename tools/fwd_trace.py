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
