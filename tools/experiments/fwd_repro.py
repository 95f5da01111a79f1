"""Attention-forward launch check through the test hook: return code and device error per shape (development)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import tools.kbench as kb  # noqa: E402

L = kb.L
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for (nseq, s, H, dh) in [(1, 128, 1, 64), (1, 128, 1, 128), (2, 200, 3, 64), (2, 256, 2, 128), (16, 2048, 16, 128)]:
    d = H * dh
    qkv = torch.randn(nseq * s, 3 * d, device="cuda").bfloat16()
    o = torch.zeros(nseq * s, d, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(nseq, H, s, device="cuda")
    rc = L.lgatest_attn_fwd(1, nseq, s, H, dh, 1, kb.P(qkv), kb.P(o), kb.P(lse), st)
    try:
        torch.cuda.synchronize()
        err = "ok"
    except Exception as e:  # noqa: BLE001
        print(nseq, s, H, dh, "rc", rc, "device error:", str(e).split("\n")[0])
        sys.exit(1)
    q, k, v = qkv.float().view(nseq, s, 3, H, dh).unbind(2)
    ref = torch.nn.functional.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2), v.transpose(1, 2),
                                                           is_causal=True).transpose(1, 2).reshape(nseq * s, d)
    print(nseq, s, H, dh, "rc", rc, err, "max err", (o.float() - ref).abs().max().item())
