"""Closed-form per-step counters, stage map, bubble and flop counts.  TEST INFRASTRUCTURE ONLY.

Definitions (readings A-5, A-7, A-10, A-11):

* Parameters are restored (all-gathered) in the forward AND the backward pass and
  gradients reduce-scattered once: "Each parameter is used in both the forward and
  backward pass, so should be restored at least twice"; the partition adds
  "an extra all-gather in the forward pass" and "increases the network
  communication by 50%".
* With layered accumulation these happen once per layer per step, independent of
  N: "the network usage remains the same"; "requires the same bandwidth as
  without gradient accumulation".  Standard accumulation with a partition
  repeats them per micro-batch: "the network operations need to be done for each
  micro-batch, resulting in 3/2 n_mu times the network bandwidth".
* Modular pipeline: layer i on stage i mod P ("the first instance gets the layers
  1, n_l+1, etc.", P:127, 0-indexed here); activations cross a stage boundary after
  every layer in forward and their gradients in backward.
* Bubble: (n_l - 1)/n_mu for a contiguous pipeline, divided by d_l/n_l for the
  modular one.
* Variants: keeping the forward's gathered parameters until the
  backward removes the second all-gather; without a partition there is no all-gather and
  the gradient is all-reduced ("the gradient reduction (scatter-reduce + all-gather)",
  P:565) -- both then move exactly the non-partitioned volume 8 (n_b - 1) p / n_gpu of
  P:565; no recompute drops the recompute units; the contiguous pipeline ("the first
  instance gets the first n_l layers" layout of P:71, the standard one) crosses stages only
  at the P - 1 block boundaries.

Byte counts are per rank per step: all-gather counts the bytes a rank RECEIVES,
reduce-scatter the bytes it SENDS (ring algorithms send and receive the same
amount); p2p counts bytes sent (and, symmetrically, received).
"""

from __future__ import annotations

from dataclasses import dataclass

from .model import layer_param_count


def padded_layer_params(d: int, dp: int, ffn_mult: int = 4) -> int:
    """P_l_pad = ceil(P_l / (64 D)) * 64 D: each layer's flat vector is padded at its end so
    that it splits into D equal, 64-element-aligned shards (reading A-10)."""
    q = 64 * dp
    pl = layer_param_count(d, ffn_mult)
    return (pl + q - 1) // q * q


@dataclass(frozen=True)
class StepShape:
    layers: int
    d: int
    seq: int
    micro_batch: int
    n_micro: int
    dp: int = 1
    pp: int = 1
    ffn_mult: int = 4


def stage_of_layer(i: int, pp: int, layers: int | None = None, pipeline: str = "modular") -> int:
    """Pipeline map, 0-indexed: modular, layer i on stage i mod P; contiguous, layer i on
    stage i // (L/P)  (blocks of L/P consecutive layers, the standard layout of P:71)."""
    if pipeline == "contiguous":
        return i // (layers // pp)
    return i % pp


def local_layers(stage: int, layers: int, pp: int, pipeline: str = "modular") -> list[int]:
    return [i for i in range(layers) if stage_of_layer(i, pp, layers, pipeline) == stage]


def comm_counters(sh: StepShape, stage: int = 0, schedule: str = "layered",
                  param_bytes: int = 2, grad_bytes: int = 2, act_bytes: int = 4,
                  keep_params: bool = False, unpartitioned: bool = False, no_recompute: bool = False,
                  pipeline: str = "modular") -> dict:
    """O8: exact integer counters for one step on one rank of the given pipeline stage."""
    L_loc = sh.layers // sh.pp
    P_pad = padded_layer_params(sh.d, sh.dp, sh.ffn_mult)
    S_l = P_pad // sh.dp
    k = 1 if schedule == "layered" else sh.n_micro
    out = dict(ag_calls=0, rs_calls=0, ag_bytes=0, rs_bytes=0,
               p2p_send_calls=0, p2p_recv_calls=0, p2p_send_bytes=0, p2p_recv_bytes=0,
               allreduce_calls=1, allreduce_bytes=0,
               fwd_units=sh.n_micro * L_loc, bwd_units=sh.n_micro * L_loc,
               recompute_units=0 if no_recompute else sh.n_micro * L_loc)
    if sh.dp > 1 and unpartitioned:
        # one ring all-reduce of the padded layer gradient per layer per step: a rank sends
        # 2 (D-1)/D of it (scatter-reduce + all-gather)
        out["allreduce_calls"] += L_loc * k
        out["allreduce_bytes"] = L_loc * k * 2 * (sh.dp - 1) * S_l * grad_bytes
    elif sh.dp > 1:
        out["ag_calls"] = (1 if keep_params else 2) * L_loc * k
        out["rs_calls"] = L_loc * k
        out["ag_bytes"] = out["ag_calls"] * (sh.dp - 1) * S_l * param_bytes
        out["rs_bytes"] = out["rs_calls"] * (sh.dp - 1) * S_l * grad_bytes
    if sh.pp > 1:
        st = lambda i: stage_of_layer(i, sh.pp, sh.layers, pipeline)
        mine = local_layers(stage, sh.layers, sh.pp, pipeline)
        crossings = (sum(1 for i in mine if i < sh.layers - 1 and st(i + 1) != stage)
                     + sum(1 for i in mine if i > 0 and st(i - 1) != stage))
        calls = sh.n_micro * crossings
        msg = sh.micro_batch * sh.seq * sh.d * act_bytes
        out.update(p2p_send_calls=calls, p2p_recv_calls=calls,
                   p2p_send_bytes=calls * msg, p2p_recv_bytes=calls * msg)
    return out


# --- the paper's own closed forms, used as pins for comm_counters -------------------------

def paper_dp_bytes_nonpartitioned(dp: int, p: int, n_gpu: int) -> float:
    """Gradient reduction (scatter-reduce + all-gather), in+out bytes per device: 8 (n_b - 1) p / n_gpu."""
    return 8.0 * (dp - 1) * p / n_gpu


def paper_dp_bytes_partitioned_layered(dp: int, p: int, n_gpu: int) -> float:
    """Partition adds 50%; with LGA the usage is independent of n_mu."""
    return 1.5 * paper_dp_bytes_nonpartitioned(dp, p, n_gpu)


def paper_dp_bytes_partitioned_standard(dp: int, p: int, n_gpu: int, n_micro: int) -> float:
    """3/2 n_mu times the non-partitioned volume."""
    return 1.5 * n_micro * paper_dp_bytes_nonpartitioned(dp, p, n_gpu)


def paper_pipeline_bytes_per_crossing(micro_batch: int, seq: int, d: int, act_bytes: int = 2) -> float:
    """In+out bytes of one stage crossing of an instance's batch: 4 b d_s d_m at 2 B/element."""
    return 2.0 * act_bytes * micro_batch * seq * d


def bubble_contiguous(pp: int, n_micro: int) -> float:
    """(n_l - 1)/n_mu."""
    return (pp - 1) / n_micro


def bubble_modular(pp: int, n_micro: int, layers: int) -> float:
    """(n_l - 1)/n_mu divided by d_l/n_l."""
    return bubble_contiguous(pp, n_micro) / (layers / pp)


# --- flop counts -------------------------------------------------------

def flops_per_token_forward(d: int, seq: int, ffn_mult: int = 4, causal: bool = True) -> float:
    """One layer's forward flops per token: 2*(4 + 2 n_I) d^2 for the weight GEMMs (the paper's
    2 b d_s p) plus the attention matmuls QK^T and PV, which the paper neglects:
    2*2*d*(s+1)/2 per token averaged over the causal triangle, 2*2*d*s without the mask."""
    gemm = 2.0 * (4 + 2 * ffn_mult) * d * d
    attn = 2.0 * d * (seq + 1) if causal else 4.0 * d * seq
    return gemm + attn


def flops_per_token_model(layers: int, d: int, seq: int, **kw) -> float:
    """forward + backward = 3x forward  (backward = 2x forward)."""
    return 3.0 * layers * flops_per_token_forward(d, seq, **kw)


def flops_per_token_hw(layers: int, d: int, seq: int, **kw) -> float:
    """+ activation recomputation = 4x forward, the paper's 8 b d_s p per batch."""
    return 4.0 * layers * flops_per_token_forward(d, seq, **kw)
