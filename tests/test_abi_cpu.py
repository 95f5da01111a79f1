"""CPU-only checks of the boundary: liblga.so loads, exports every symbol include/lga.h
declares, and its host-only entry points behave (no GPU compute is called here)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "lga.h")).read()
    return sorted(set(re.findall(r"^(?:const )?[a-z_0-9]+\*? *\*?(lga_[a-z_]+)\(", txt, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2106_02679_b200 import _abi
    L = _abi.lib()
    declared = _header_symbols()
    assert "lga_init" in declared and "lga_step" in declared and "lga_grads" in declared and "lga_comm_bytes" in declared
    for name in declared:
        assert hasattr(L, name), name
    assert sorted(_abi.EXPORTED) == declared


def test_struct_layout_matches_header():
    from paper_2106_02679_b200 import _abi
    # lga_config: 1 uint32 + 13 int32 + 6 float + 1 int32 + 1 uint32 = 22 * 4 bytes
    assert C.sizeof(_abi.lga_config) == 22 * 4
    assert C.sizeof(_abi.lga_comm_stats) == 14 * 8   # ABI v2: + allreduce_bytes
    assert C.sizeof(_abi.lga_timing) == 8 * 4 + 3 * 4 + 4 + 3 * 8 + 8 + 8   # padding; ABI v3: + graph_captures
    # and against the C compiler's view of include/lga.h: every binding struct, size and field offsets
    import os
    import subprocess
    import tempfile
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    structs = {"lga_config": _abi.lga_config, "lga_comm_stats": _abi.lga_comm_stats, "lga_timing": _abi.lga_timing,
               "lga_rank_plan": _abi.lga_rank_plan}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "lga.h"', "int main(void) {"]
    for name, cls in structs.items():
        lines.append(f'printf("{name} %zu\\n", sizeof({name}));')
        for f, _ in cls._fields_:
            lines.append(f'printf("{name}.{f} %zu\\n", offsetof({name}, {f}));')
    lines.append("return 0; }")
    with tempfile.TemporaryDirectory() as td:
        src, exe = os.path.join(td, "s.c"), os.path.join(td, "s")
        open(src, "w").write("\n".join(lines))
        subprocess.run(["gcc", "-I", os.path.join(root, "include"), src, "-o", exe], check=True)
        out = dict(l.split() for l in subprocess.run([exe], capture_output=True, text=True).stdout.splitlines())
    for name, cls in structs.items():
        assert int(out[name]) == C.sizeof(cls), name
        for f, _ in cls._fields_:
            assert int(out[f"{name}.{f}"]) == getattr(cls, f).offset, (name, f)


def test_param_count_host_only():
    from paper_2106_02679_b200 import Config
    assert Config(layers=2, d_model=4, heads=1, seq_len=32, micro_batch=1, n_micro=1).param_count() == (244, 488)
    assert Config(layers=24, d_model=2048, heads=16, seq_len=2048, micro_batch=1, n_micro=16).param_count()[1] \
        == 1_208_598_528


def test_invalid_configs_rejected_without_side_effects():
    from paper_2106_02679_b200 import Config, _abi
    L = _abi.lib()
    cases = [
        (dict(d_model=65, heads=4), 1),                       # d % heads
        (dict(layers=3, pp=2, dp=1), 1),                      # L % P
        (dict(ffn_mult=3), 2),                                # n_I must be 4
        (dict(precision=1, d_model=96, heads=3), 2),          # bf16 head size 32 unsupported
        (dict(schedule=1, pp=2, layers=4, n_micro=4), 1),     # STANDARD needs P = 1
        (dict(chunk=3), 1),                                   # N % chunk
    ]
    for kw, status in cases:
        base = dict(layers=2, d_model=64, heads=4, seq_len=32, micro_batch=2, n_micro=4, precision=0)
        base.update(kw)
        cfg = Config(**base)
        h = C.c_void_p()
        world = cfg.dp * cfg.pp
        nid = C.create_string_buffer(128) if world > 1 else None
        st = L.lga_init(C.byref(cfg.to_c()), 0, world, 0, _abi.ALLGATHER_FN(), None, nid, None, None, 0, C.byref(h))
        assert st == status, (kw, st, L.lga_last_error())
        assert not h.value
    # world mismatch
    cfg = Config(layers=2, d_model=64, heads=4, seq_len=32, micro_batch=2, n_micro=4, dp=2, precision=0)
    h = C.c_void_p()
    assert L.lga_init(C.byref(cfg.to_c()), 0, 3, 0, _abi.ALLGATHER_FN(), None, C.create_string_buffer(128), None, None,
                      0, C.byref(h)) == 1
    assert b"world" in L.lga_last_error()
    # world > 1 without any bootstrap (no allgather callback, no NCCL id)
    assert L.lga_init(C.byref(cfg.to_c()), 0, 2, 0, _abi.ALLGATHER_FN(), None, None, None, None, 0, C.byref(h)) == 1
    assert b"bootstrap" in L.lga_last_error()
    assert not h.value
    # the NCCL baseline needs an NCCL id
    cfg = Config(layers=2, d_model=64, heads=4, seq_len=32, micro_batch=2, n_micro=4, dp=2, precision=0,
                 flags=_abi.LGA_FLAG_NCCL_DP)
    cb = _abi.ALLGATHER_FN(lambda ctx, a, b, n: 0)
    assert L.lga_init(C.byref(cfg.to_c()), 0, 2, 0, cb, None, None, None, None, 0, C.byref(h)) == 1
    assert b"nccl_id" in L.lga_last_error()
    assert not h.value


def test_status_strings():
    from paper_2106_02679_b200 import _abi
    L = _abi.lib()
    for k, v in _abi.STATUS.items():
        assert L.lga_status_string(k).decode() == v


@pytest.mark.parametrize("L,P,D,N,contig", [(4, 2, 1, 4, False), (8, 4, 1, 4, False), (4, 2, 2, 4, False),
                                            (48, 4, 2, 32, False), (8, 4, 1, 8, True), (4, 2, 2, 4, True),
                                            (24, 1, 8, 16, False)])
def test_rank_plan_matches_closed_forms(L, P, D, N, contig):
    """lga_plan (no GPU): the library's host-side rank plan -- the same function lga_init uses for the pipeline
    flag epochs -- against oracle.counters: stage = rank mod P, the stage's local layers (modular i mod P,
    P:127; contiguous blocks), per-step transfers = the closed-form p2p call counts, shard size."""
    from oracle import counters as oc
    from paper_2106_02679_b200 import Config, _abi
    flags = _abi.LGA_FLAG_CONTIGUOUS_PP if contig else 0
    cfg = Config(layers=L, d_model=64, heads=4, seq_len=32, micro_batch=2, n_micro=N, dp=D, pp=P, precision=0,
                 flags=flags)
    pipeline = "contiguous" if contig else "modular"
    for rank in range(D * P):
        p = cfg.plan(rank)
        assert p["stage"] == rank % P and p["replica"] == rank // P
        mine = oc.local_layers(p["stage"], L, P, pipeline)
        assert [p["first_layer"] + k * p["layer_stride"] for k in range(p["local_layers"])] == mine
        ref = oc.comm_counters(oc.StepShape(layers=L, d=64, seq=32, micro_batch=2, n_micro=N, dp=D, pp=P),
                               stage=p["stage"], pipeline=pipeline)
        assert p["p2p_send_fwd"] + p["p2p_send_bwd"] == ref["p2p_send_calls"]
        assert p["p2p_recv_fwd"] + p["p2p_recv_bwd"] == ref["p2p_recv_calls"]
        assert p["p2p_send_fwd"] == p["p2p_recv_bwd"] and p["p2p_recv_fwd"] == p["p2p_send_bwd"]
        assert p["layer_elems_padded"] == oc.padded_layer_params(64, D)
        assert p["shard_elems"] == p["layer_elems_padded"] // D
        want = N if P == 1 else max(c for c in range(1, N // P + 1) if N % c == 0 and c * 2 * 32 <= 8192)
        assert p["chunk"] == want
