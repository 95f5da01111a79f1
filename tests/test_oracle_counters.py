"""Pins for oracle.counters against the paper's closed forms (P:67, P:118, P:127, P:138,
P:565) and printed examples (tests/golden/bubble_examples.txt)."""
import os

import pytest

from oracle import counters as oc
from oracle import model as om

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _shape(**kw):
    base = dict(layers=24, d=2048, seq=2048, micro_batch=1, n_micro=16, dp=8, pp=1)
    base.update(kw)
    return oc.StepShape(**base)


@pytest.mark.parametrize("D", [2, 4, 8])
def test_layered_volume_is_three_halves_of_nonpartitioned(D):
    """in+out bytes = 2 (ag + rs) = 3/2 * 8 (D-1) p / D when no padding is needed."""
    sh = _shape(dp=D)
    p = om.param_count(sh.d, sh.layers)
    assert oc.padded_layer_params(sh.d, D) == om.layer_param_count(sh.d)   # C3 needs no padding
    c = oc.comm_counters(sh)
    assert 2 * (c["ag_bytes"] + c["rs_bytes"]) == oc.paper_dp_bytes_partitioned_layered(D, p, D)


def test_c3_counters_exact():
    c = oc.comm_counters(_shape())
    assert (c["ag_calls"], c["rs_calls"]) == (48, 24)
    assert c["ag_bytes"] == 4_230_094_848 and c["rs_bytes"] == 2_115_047_424
    assert c["fwd_units"] == c["bwd_units"] == c["recompute_units"] == 384


@pytest.mark.parametrize("N", [1, 2, 7, 16, 64])
def test_layered_independent_of_n_and_standard_is_n_times(N):
    """P:583 / P:118 (layered: same as without accumulation) and P:576 (standard: x n_mu)."""
    lay = oc.comm_counters(_shape(n_micro=N, dp=4), schedule="layered")
    ref = oc.comm_counters(_shape(n_micro=1, dp=4), schedule="layered")
    std = oc.comm_counters(_shape(n_micro=N, dp=4), schedule="standard")
    for k in ("ag_calls", "rs_calls", "ag_bytes", "rs_bytes"):
        assert lay[k] == ref[k]
        assert std[k] == N * lay[k]
    p = om.param_count(2048, 24)
    assert 2 * (std["ag_bytes"] + std["rs_bytes"]) == oc.paper_dp_bytes_partitioned_standard(4, p, 4, N)


def test_no_comm_without_data_parallelism():
    c = oc.comm_counters(oc.StepShape(layers=2, d=64, seq=32, micro_batch=2, n_micro=4))
    assert c["ag_calls"] == c["rs_calls"] == c["ag_bytes"] == c["rs_bytes"] == 0
    assert c["fwd_units"] == 8


def test_padding_counted_tiny_dist():
    """L=4, d=64, fp32: P_l = 49,984 padded to a multiple of 64 D."""
    for D, ag, rs in [(2, 800_768, 400_384), (4, 1_204_224, 602_112), (8, 1_404_928, 702_464)]:
        c = oc.comm_counters(oc.StepShape(layers=4, d=64, seq=32, micro_batch=2, n_micro=4, dp=D),
                             param_bytes=4, grad_bytes=4)
        assert (c["ag_calls"], c["rs_calls"], c["ag_bytes"], c["rs_bytes"]) == (8, 4, ag, rs)


def test_stage_map_is_modular():
    """"the first instance gets the layers 1, n_l+1, etc., the second gets the layers 2, n_l+2"."""
    assert [oc.stage_of_layer(i, 4) for i in range(8)] == [0, 1, 2, 3, 0, 1, 2, 3]
    assert oc.local_layers(1, 8, 4) == [1, 5]


def test_pipeline_p2p_counts():
    """Each micro-batch crosses every layer boundary once forward and once backward:
    summed over stages, 2 N (L-1) crossings of b*s*d activations."""
    sh = _shape(layers=48, d=4096, n_micro=32, dp=2, pp=4)
    per = [oc.comm_counters(sh, stage=s) for s in range(4)]
    assert [c["p2p_send_calls"] for c in per] == [736, 768, 768, 736]
    assert sum(c["p2p_send_calls"] for c in per) == 2 * 32 * 47
    assert per[0]["p2p_send_bytes"] == 736 * 2048 * 4096 * 4
    # the paper's per-crossing in+out volume at 2 B/element is 4 b d_s d_m
    assert oc.paper_pipeline_bytes_per_crossing(1, 2048, 4096, 2) == 4 * 2048 * 4096
    assert per[0]["ag_calls"] == 24 and per[0]["ag_bytes"] == 4_833_116_160


def test_bubble_examples():
    for line in open(os.path.join(GOLDEN, "bubble_examples.txt")):
        if not line.strip() or line.startswith("#"):
            continue
        kind, pp, nmu, dl, expect, tol, _src = line.split()
        pp, nmu, dl, expect, tol = int(pp), int(nmu), int(dl), float(expect), float(tol)
        got = oc.bubble_contiguous(pp, nmu) if kind == "contiguous" else oc.bubble_modular(pp, nmu, dl)
        assert abs(got - expect) <= tol, (line, got)


def test_forward_flops_are_two_per_token_per_weight():
    """"two floating point operations for each input token and parameter": the GEMM part
    of the forward count is 2 (p_l - biases - LN) per token; attention is counted by brute force."""
    d, s = 64, 32
    gemm_params = 12 * d * d
    f_nomask = oc.flops_per_token_forward(d, s, causal=False)
    assert f_nomask - 4 * d * s == 2 * gemm_params
    # causal: token i attends to i+1 keys; QK^T and PV each cost 2 d flops per (query, key) pair
    pairs = sum(i + 1 for i in range(s))
    assert oc.flops_per_token_forward(d, s, causal=True) == 2 * gemm_params + 4 * d * pairs / s
    assert oc.flops_per_token_hw(2, d, s) == 4 / 3 * oc.flops_per_token_model(2, d, s)


# ---- variants ------------------------------------------------------------

@pytest.mark.parametrize("D", [2, 4, 8])
def test_keep_params_and_unpartitioned_move_the_nonpartitioned_volume(D):
    """Keeping the forward gather (1 AG + 1 RS) or dropping the partition (1 all-reduce = scatter-
    reduce + all-gather) moves exactly 8 (D-1) p / D in+out, the non-partitioned volume of P:565 --
    i.e. the partition's +50% is exactly the second all-gather."""
    sh = _shape(dp=D)
    p = om.param_count(sh.d, sh.layers)
    keep = oc.comm_counters(sh, keep_params=True)
    assert 2 * (keep["ag_bytes"] + keep["rs_bytes"]) == oc.paper_dp_bytes_nonpartitioned(D, p, D)
    assert (keep["ag_calls"], keep["rs_calls"]) == (24, 24)
    unp = oc.comm_counters(sh, unpartitioned=True)
    assert unp["ag_calls"] == unp["rs_calls"] == 0
    assert unp["allreduce_calls"] == 1 + 24
    assert 2 * unp["allreduce_bytes"] == oc.paper_dp_bytes_nonpartitioned(D, p, D)
    full = oc.comm_counters(sh)
    assert 2 * (full["ag_bytes"] + full["rs_bytes"]) == 1.5 * 2 * (keep["ag_bytes"] + keep["rs_bytes"])


def test_no_recompute_units():
    c = oc.comm_counters(_shape(), no_recompute=True)
    assert c["recompute_units"] == 0 and c["fwd_units"] == c["bwd_units"] == 384
    assert c["ag_bytes"] == oc.comm_counters(_shape())["ag_bytes"]   # communication unchanged


def test_variants_without_data_parallelism_move_nothing():
    for kw in (dict(keep_params=True), dict(unpartitioned=True)):
        c = oc.comm_counters(_shape(dp=1), **kw)
        assert c["ag_bytes"] == c["rs_bytes"] == c["allreduce_bytes"] == 0 and c["allreduce_calls"] == 1


def test_contiguous_stage_map_and_crossings():
    """Contiguous blocks of L/P layers: activations cross stages only at the P-1 block
    boundaries, 2 N (P-1) crossings per step in total (vs 2 N (L-1) for the modular map)."""
    assert [oc.stage_of_layer(i, 4, 8, "contiguous") for i in range(8)] == [0, 0, 1, 1, 2, 2, 3, 3]
    assert oc.local_layers(1, 8, 4, "contiguous") == [2, 3]
    sh = _shape(layers=48, d=4096, n_micro=32, dp=2, pp=4)
    per = [oc.comm_counters(sh, stage=s, pipeline="contiguous") for s in range(4)]
    assert [c["p2p_send_calls"] for c in per] == [32, 64, 64, 32]
    assert sum(c["p2p_send_calls"] for c in per) == 2 * 32 * (4 - 1)
    assert [c["p2p_recv_calls"] for c in per] == [32, 64, 64, 32]
    modular = sum(c["p2p_send_calls"] for c in (oc.comm_counters(sh, stage=s) for s in range(4)))
    assert modular == 2 * 32 * 47
