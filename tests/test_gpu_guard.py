"""Own memory checker in place of compute-sanitizer (refused by the GPU pool, profiles/r2_sanitizer_unavailable.txt):
with LGA_ARENA_GUARD=1 every arena buffer is followed by a 4 KB canary; after several steps (eager and
graph-replayed) of each configuration no canary byte may have changed -- no kernel of the step writes past the
end of any buffer it was given (GEMM epilogues incl. split-K partials, attention, LayerNorm and the fused bias
partials, AdamW, loss, flags).  The results must still match the oracle (the guard only moves buffers)."""
import ctypes as C
import os

import numpy as np
import pytest

import synth
from gpu_util import oracle_run, rel

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2106_02679_b200 import LGA_BF16, LGA_FP32, LGA_STANDARD, Config, Trainer, _abi  # noqa: E402

L = _abi.lib()
L.lgatest_arena_guard_check.restype = C.c_int64
L.lgatest_arena_guard_check.argtypes = [C.c_void_p]
L.lgatest_arena_guard_poke.restype = C.c_int
L.lgatest_arena_guard_poke.argtypes = [C.c_void_p]

CASES = [
    ("fp32 C1", synth.Shape(2, 64, 4, 32, 2, 4), LGA_FP32, 0, 0, 1e-5),
    ("fp32 ragged chunked", synth.Shape(2, 48, 3, 37, 1, 4), LGA_FP32, 2, 0, 1e-5),
    ("bf16 dh64", synth.Shape(2, 256, 4, 128, 2, 4), LGA_BF16, 0, 0, 2e-2),
    ("bf16 dh128 chunk 1", synth.Shape(2, 256, 2, 200, 1, 4), LGA_BF16, 1, 0, 2e-2),
    ("bf16 post-LN no-recompute", synth.Shape(2, 256, 4, 128, 1, 4), LGA_BF16, 0, 0x110, 2e-2),
    ("bf16 d768 split-K", synth.Shape(1, 768, 12, 256, 1, 4), LGA_BF16, 0, 0, 2e-2),
    ("bf16 standard", synth.Shape(2, 256, 4, 128, 1, 4), LGA_BF16, 0, -1, 2e-2),
]


@pytest.mark.parametrize("name,sh,prec,chunk,flags,tol", CASES, ids=[c[0] for c in CASES])
def test_no_write_past_any_arena_buffer(name, sh, prec, chunk, flags, tol, monkeypatch):
    monkeypatch.setenv("LGA_ARENA_GUARD", "1")
    schedule = LGA_STANDARD if flags == -1 else 0
    flags = max(flags, 0)
    init = synth.init_params(sh, style="parity")
    cfg = Config(layers=sh.layers, d_model=sh.d, heads=sh.heads, seq_len=sh.seq, micro_batch=sh.micro_batch,
                 n_micro=sh.n_micro, precision=prec, chunk=chunk, schedule=schedule, lr=1e-3, retain_grads=1,
                 flags=flags)
    tr = Trainer(cfg, rank=0, world=1, device=0, init_params=init)
    X, T = synth.batch(sh, step=0)
    x, t = torch.from_numpy(X[0]).cuda(), torch.from_numpy(T[0]).cuda()
    for _ in range(3):   # eager, capture, replay
        tr.step(x, t)
    bad = L.lgatest_arena_guard_check(tr._h)
    g = tr.grads()
    tr.close()
    assert bad == 0, f"{bad} canary bytes overwritten"
    _, _, rg = oracle_run(sh, init, [(X, T)] * 3, lr=1e-3, post_ln=bool(flags & 0x100))
    assert rel(g, rg) < tol


def test_guard_check_sees_a_one_byte_overrun(monkeypatch):
    """Negative control: one byte written past the end of the last buffer is reported; without the env var the
    handle is not in guard mode."""
    sh = synth.Shape(1, 64, 4, 32, 1, 2)
    cfg = Config(layers=1, d_model=64, heads=4, seq_len=32, micro_batch=1, n_micro=2, precision=LGA_FP32)
    plain = Trainer(cfg, rank=0, world=1, device=0, init_params=synth.init_params(sh))
    assert L.lgatest_arena_guard_check(plain._h) == -1
    plain.close()
    monkeypatch.setenv("LGA_ARENA_GUARD", "1")
    tr = Trainer(cfg, rank=0, world=1, device=0, init_params=synth.init_params(sh))
    X, T = synth.batch(sh, step=0)
    tr.step(torch.from_numpy(X[0]).cuda(), torch.from_numpy(T[0]).cuda())
    assert L.lgatest_arena_guard_check(tr._h) == 0
    assert L.lgatest_arena_guard_poke(tr._h) == 0
    assert L.lgatest_arena_guard_check(tr._h) == 1
    tr.close()
