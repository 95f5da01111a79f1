"""Run the tcgen05 attention forward at one shape (argv: nseq s heads dh) and check finiteness (dev tool)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tools.kbench as kb  # noqa: E402

nseq, s, H, dh = (int(x) for x in sys.argv[1:5])
d = H * dh
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
qkv = torch.randn(nseq * s, 3 * d, device="cuda").bfloat16()
o = torch.empty(nseq * s, d, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(nseq, H, s, device="cuda")
rc = kb.L.lgatest_attn_fwd(1, nseq, s, H, dh, 1, kb.P(qkv), kb.P(o), kb.P(lse), st)
torch.cuda.synchronize()
print(f"nseq={nseq} s={s} H={H} dh={dh}: rc={rc} finite={bool(torch.isfinite(o.float()).all())} items={(s // 128) * H * nseq}")
