"""Forward attention error vs SDPA (fp32 and fp64 references) and run-to-run determinism, per shape."""
import math
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import test_gpu_kernels as T  # noqa: E402


def one(path, dh, s, causal, mag, nseq, H, reps=4):
    d = H * dh
    g = torch.Generator(device="cuda").manual_seed(3)
    qkv = (torch.randn(nseq * s, 3 * d, device="cuda", generator=g)
           * torch.linspace(0.3, mag, nseq * s, device="cuda")[:, None]).to(torch.bfloat16)
    outs = []
    for _ in range(reps):
        o = torch.empty(nseq * s, d, device="cuda", dtype=torch.bfloat16)
        lse = torch.empty(nseq, H, s, device="cuda")
        assert T.L.lgatest_attn_fwd(path, nseq, s, H, dh, causal, T.P(qkv), T.P(o), T.P(lse), T.stream()) == 0
        torch.cuda.synchronize()
        outs.append(o.clone())
    same = all(torch.equal(outs[0], x) for x in outs[1:])
    x = qkv.double().view(nseq, s, 3, H, dh).permute(2, 0, 3, 1, 4)
    q, k, v = x[0], x[1], x[2]
    S = q @ k.transpose(-1, -2) / math.sqrt(dh)
    if causal:
        S = S.masked_fill(torch.triu(torch.ones(s, s, device="cuda", dtype=torch.bool), 1), float("-inf"))
    ref = (torch.softmax(S, -1) @ v).permute(0, 2, 1, 3).reshape(nseq * s, d)
    e = [float((x.double() - ref).norm() / ref.norm()) for x in outs]
    rb = ref.to(torch.bfloat16).double()
    floor = float((rb - ref).norm() / ref.norm())
    # backward determinism on the same inputs
    o, lse = outs[0], torch.empty(nseq, H, s, device="cuda")
    assert T.L.lgatest_attn_fwd(path, nseq, s, H, dh, causal, T.P(qkv), T.P(o), T.P(lse), T.stream()) == 0
    dO = torch.randn(nseq * s, d, device="cuda", generator=g).to(torch.bfloat16)
    grads = []
    for _ in range(reps):
        dsum = torch.empty(nseq, H, s, device="cuda")
        dqkv = torch.full((nseq * s, 3 * d), float("nan"), device="cuda", dtype=torch.bfloat16)
        assert T.L.lgatest_attn_bwd(path, nseq, s, H, dh, causal, T.P(qkv), T.P(o), T.P(lse), T.P(dO), T.P(dsum),
                                    T.P(dqkv), T.stream()) == 0
        torch.cuda.synchronize()
        grads.append(dqkv.clone())
    bsame = all(torch.equal(grads[0], x) for x in grads[1:])
    print(f"path{path} dh{dh} s{s} c{causal} mag{mag} nseq{nseq} H{H}: relerr {min(e):.5f}..{max(e):.5f} "
          f"deterministic={same} bf16-rounding floor {floor:.5f} bwd deterministic={bsame}", flush=True)


for cfg in [(1, 128, 512, 1, 1, 16, 16), (1, 128, 512, 1, 1, 2, 3), (1, 64, 512, 1, 6, 16, 16),
            (1, 128, 384, 0, 1, 16, 16), (1, 128, 512, 0, 1, 2, 3), (1, 64, 1024, 1, 1, 2, 3),
            (2, 128, 512, 1, 1, 16, 16), (1, 128, 2048, 1, 1, 4, 16), (1, 64, 512, 0, 1, 16, 16)]:
    one(*cfg)
