"""ctypes binding of include/lga.h -- argument marshalling only.

Every step of the training path runs inside liblga.so (hand-written sm_100a kernels); this
module only loads the library, mirrors its structs and turns non-zero lga_status codes into
``LgaError``.  There is no fallback: if the library is missing this raises at import of the
binding's first use.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liblga.so")

ABI_VERSION = 3
NCCL_ID_BYTES = 128

LGA_FP32, LGA_BF16 = 0, 1
LGA_LAYERED, LGA_STANDARD = 0, 1
LGA_FLAG_NO_COMM = 0x1
LGA_FLAG_NO_GRAPH = 0x2         # every step eager (default: CUDA graph from the second lga_step)
LGA_FLAG_PROFILE = 0x4
LGA_FLAG_KEEP_PARAMS = 0x8       # N2a: 1 all-gather per layer per step
LGA_FLAG_NO_RECOMPUTE = 0x10     # N2c: keep intermediates, no forward recompute
LGA_FLAG_UNPARTITIONED = 0x20    # N2b: full state per replica, one all-reduce per layer
LGA_FLAG_CONTIGUOUS_PP = 0x40    # N3: layer i on stage i // (L/P)
LGA_FLAG_NCCL_DP = 0x80          # N1 baseline: NCCL all-gather / reduce-scatter instead of peer memory
LGA_FLAG_POST_LN = 0x100         # N4: post-LN layer (original encoder; reading A-16)

STATUS = {0: "LGA_OK", 1: "LGA_ERR_INVALID_ARG", 2: "LGA_ERR_UNSUPPORTED", 3: "LGA_ERR_OUT_OF_MEMORY",
          4: "LGA_ERR_CUDA", 5: "LGA_ERR_NCCL", 6: "LGA_ERR_SIZE_MISMATCH", 7: "LGA_ERR_BAD_STATE"}


class LgaError(RuntimeError):
    def __init__(self, status: int, detail: str):
        self.status = status
        super().__init__(f"{STATUS.get(status, status)}: {detail}")


class lga_config(C.Structure):
    _fields_ = [("abi_version", C.c_uint32), ("layers", C.c_int32), ("d_model", C.c_int32), ("heads", C.c_int32),
                ("seq_len", C.c_int32), ("micro_batch", C.c_int32), ("n_micro", C.c_int32), ("dp", C.c_int32),
                ("pp", C.c_int32), ("ffn_mult", C.c_int32), ("precision", C.c_int32), ("schedule", C.c_int32),
                ("causal", C.c_int32), ("chunk", C.c_int32), ("lr", C.c_float), ("beta1", C.c_float),
                ("beta2", C.c_float), ("adam_eps", C.c_float), ("weight_decay", C.c_float), ("ln_eps", C.c_float),
                ("retain_grads", C.c_int32), ("flags", C.c_uint32)]


class lga_comm_stats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "steps", "ag_calls", "rs_calls", "p2p_send_calls", "p2p_recv_calls", "allreduce_calls",
        "ag_bytes", "rs_bytes", "p2p_send_bytes", "p2p_recv_bytes", "fwd_units", "bwd_units", "recompute_units",
        "allreduce_bytes")]

    def as_dict(self):
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


class lga_timing(C.Structure):
    _fields_ = ([(n, C.c_float) for n in ("step_ms", "comm_wait_ms", "p2p_wait_ms", "fwd_ms", "bwd_ms",
                                          "gemm_ms", "attn_ms", "adam_ms")]
                + [(n, C.c_uint32) for n in ("gemm_launches", "attn_launches", "adam_launches")]
                + [(n, C.c_double) for n in ("gemm_flop", "attn_flop", "adam_bytes")]
                + [("kernel_launches", C.c_uint64), ("graph_captures", C.c_uint64)])

    def as_dict(self):
        return {n: float(getattr(self, n)) for n, _ in self._fields_}


# int32_t (*lga_allgather_fn)(void* ctx, const void* send, void* recv, uint64_t bytes)  (include/lga.h)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64)

class lga_rank_plan(C.Structure):
    _fields_ = ([(n, C.c_int32) for n in ("stage", "replica", "local_layers", "chunk", "first_layer", "layer_stride")]
                + [(n, C.c_uint64) for n in ("p2p_send_fwd", "p2p_recv_fwd", "p2p_send_bwd", "p2p_recv_bwd",
                                             "shard_elems", "layer_elems_padded")])

    def as_dict(self):
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


_lib = None


def lib():
    """Load liblga.so (built in-tree by ``python -m paper_2106_02679_b200.build``)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2106_02679_b200.build` "
                          "(there is no CPU or PyTorch fallback)")
    L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    H = C.c_void_p
    sigs = {
        "lga_abi_version": (C.c_uint32, []),
        "lga_status_string": (C.c_char_p, [C.c_int]),
        "lga_last_error": (C.c_char_p, []),
        "lga_param_count": (C.c_int, [C.POINTER(lga_config), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
        "lga_nccl_unique_id": (C.c_int, [C.c_char_p]),
        "lga_plan": (C.c_int, [C.POINTER(lga_config), C.c_int32, C.c_int32, C.POINTER(lga_rank_plan)]),
        "lga_init": (C.c_int, [C.POINTER(lga_config), C.c_int32, C.c_int32, C.c_int32, ALLGATHER_FN, C.c_void_p,
                               C.c_char_p, C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(H)]),
        "lga_step": (C.c_int, [H, C.c_void_p, C.c_void_p, C.POINTER(C.c_double)]),
        "lga_step_host": (C.c_int, [H, C.c_void_p, C.c_void_p, C.POINTER(C.c_double)]),
        "lga_grads": (C.c_int, [H, C.c_void_p, C.c_uint64, C.c_int32]),
        "lga_params": (C.c_int, [H, C.c_void_p, C.c_uint64, C.c_int32]),
        "lga_comm_bytes": (C.c_int, [H, C.POINTER(lga_comm_stats), C.POINTER(lga_comm_stats)]),
        "lga_layer_stage": (C.c_int, [H, C.POINTER(C.c_int32), C.c_int32]),
        "lga_state_bytes": (C.c_int, [H, C.POINTER(C.c_uint64)]),
        "lga_save_state": (C.c_int, [H, C.c_void_p, C.c_uint64]),
        "lga_load_state": (C.c_int, [H, C.c_void_p, C.c_uint64]),
        "lga_timing_last": (C.c_int, [H, C.POINTER(lga_timing)]),
        "lga_destroy": (None, [H]),
    }
    for name, (res, args) in sigs.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    if L.lga_abi_version() != ABI_VERSION:
        raise ImportError(f"liblga.so ABI {L.lga_abi_version()} != binding {ABI_VERSION}")
    _lib = L
    return L


def check(status: int):
    if status != 0:
        raise LgaError(status, lib().lga_last_error().decode(errors="replace"))


EXPORTED = ["lga_abi_version", "lga_status_string", "lga_last_error", "lga_param_count", "lga_plan", "lga_nccl_unique_id",
            "lga_init", "lga_step", "lga_step_host", "lga_grads", "lga_params", "lga_comm_bytes", "lga_layer_stage",
            "lga_state_bytes", "lga_save_state", "lga_load_state",
            "lga_timing_last", "lga_destroy"]
