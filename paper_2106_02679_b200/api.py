"""Config + Trainer: thin wrappers over the C ABI (include/lga.h).  Argument marshalling only."""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, fields

import numpy as np

from . import _abi
from ._abi import check, lib


@dataclass
class Config:
    """Mirrors ``lga_config`` (include/lga.h); names follow the paper's notation."""
    layers: int
    d_model: int
    heads: int
    seq_len: int
    micro_batch: int
    n_micro: int
    dp: int = 1
    pp: int = 1
    ffn_mult: int = 4
    precision: int = _abi.LGA_BF16
    schedule: int = _abi.LGA_LAYERED
    causal: int = 1
    chunk: int = 0
    lr: float = 1e-4
    beta1: float = 0.9
    beta2: float = 0.95
    adam_eps: float = 1e-8
    weight_decay: float = 0.0
    ln_eps: float = 1e-5
    retain_grads: int = 0
    flags: int = 0

    def to_c(self) -> _abi.lga_config:
        c = _abi.lga_config()
        c.abi_version = _abi.ABI_VERSION
        for f in fields(self):
            setattr(c, f.name, getattr(self, f.name))
        return c

    @property
    def tokens_per_replica(self) -> int:
        return self.n_micro * self.micro_batch * self.seq_len

    def plan(self, rank: int = 0):
        """lga_plan: this configuration's host-side plan of `rank` (no GPU needed)."""
        out = _abi.lga_rank_plan()
        check(lib().lga_plan(C.byref(self.to_c()), rank, self.dp * self.pp, C.byref(out)))
        return out.as_dict()

    def param_count(self):
        pl, tot = C.c_uint64(), C.c_uint64()
        check(lib().lga_param_count(C.byref(self.to_c()), C.byref(pl), C.byref(tot)))
        return int(pl.value), int(tot.value)


def _ptr(t):
    """Raw device pointer of a torch tensor (or None)."""
    if t is None:
        return None
    return C.c_void_p(t.data_ptr())


def torch_allgather(group=None):
    """An ``lga_allgather_fn`` over torch.distributed (any backend; bytes travel as a Python object): the
    bootstrap exchange of lga_init (include/lga.h).  Returns the ctypes callback; keep it alive during the call."""
    import torch.distributed as dist

    def fn(ctx, send, recv, nbytes):
        try:
            mine = C.string_at(send, nbytes)
            out = [None] * dist.get_world_size(group)
            dist.all_gather_object(out, mine, group=group)
            blob = b"".join(out)
            if len(blob) != nbytes * len(out):
                return 1
            C.memmove(recv, blob, len(blob))
            return 0
        except Exception:   # a Python exception must not cross the C ABI
            return 1

    return _abi.ALLGATHER_FN(fn)


class Trainer:
    """One rank of the LGA step.  For world > 1, torch.distributed must be initialised (any backend): it
    carries only the bootstrap exchange of lga_init (IPC handles), on a gloo group; every data path runs
    inside liblga.so over CUDA IPC peer memory.  The NCCL baseline (LGA_FLAG_NCCL_DP) also broadcasts an
    NCCL unique id.  Several ranks may share one GPU (device = LOCAL_RANK modulo the visible devices)."""

    def __init__(self, cfg: Config, rank: int | None = None, world: int | None = None, device: int | None = None,
                 init_params: np.ndarray | None = None, seed: int = 1234, stream=None):
        import torch
        self.cfg = cfg
        if world is None:
            world = int(os.environ.get("WORLD_SIZE", "1"))
        if rank is None:
            rank = int(os.environ.get("RANK", "0"))
        if device is None:
            device = int(os.environ.get("LOCAL_RANK", str(rank))) % max(1, torch.cuda.device_count())
        self.rank, self.world, self.device = rank, world, device
        torch.cuda.set_device(device)
        nid = None
        cb = _abi.ALLGATHER_FN()   # NULL
        if world > 1:
            import torch.distributed as dist
            group = None if dist.get_backend() == "gloo" else dist.new_group(backend="gloo")
            cb = torch_allgather(group)
            if cfg.dp > 1 and (cfg.flags & _abi.LGA_FLAG_NCCL_DP):
                buf = C.create_string_buffer(_abi.NCCL_ID_BYTES)
                if rank == 0:
                    check(lib().lga_nccl_unique_id(buf))
                obj = [bytes(buf.raw) if rank == 0 else None]
                dist.broadcast_object_list(obj, src=0, group=group)
                nid = C.create_string_buffer(obj[0], _abi.NCCL_ID_BYTES)
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.stream = stream
        ip = None
        if init_params is not None:
            self._init_params = np.ascontiguousarray(init_params, dtype=np.float32)
            pl, tot = cfg.param_count()
            if self._init_params.size != tot:
                raise ValueError(f"init_params has {self._init_params.size} floats, expected {tot}")
            ip = self._init_params.ctypes.data_as(C.c_void_p)
        h = C.c_void_p()
        check(lib().lga_init(C.byref(cfg.to_c()), rank, world, device, cb, None, nid, C.c_void_p(stream.cuda_stream),
                             ip, C.c_uint64(seed), C.byref(h)))
        self._h = h
        self.stage = rank % cfg.pp
        self.replica = rank // cfg.pp

    # ---------------------------------------------------------------- step
    def step(self, x, target, sync: bool = True):
        """x, target: torch CUDA fp32 contiguous [N][b][s][d] (this replica's micro-batches)."""
        loss = C.c_double()
        check(lib().lga_step(self._h, _ptr(x), _ptr(target), C.byref(loss) if sync else None))
        return float(loss.value) if sync else None

    def step_host(self, x: np.ndarray | None, target: np.ndarray | None, sync: bool = True):
        """Host fp32 inputs; copied to the device inside the library call (end-to-end path)."""
        loss = C.c_double()
        xp = None if x is None else x.ctypes.data_as(C.c_void_p)
        tp = None if target is None else target.ctypes.data_as(C.c_void_p)
        check(lib().lga_step_host(self._h, xp, tp, C.byref(loss) if sync else None))
        return float(loss.value) if sync else None

    # ---------------------------------------------------------------- queries
    def _local_count(self):
        pl, _ = self.cfg.param_count()
        return (self.cfg.layers // self.cfg.pp) * pl

    def grads(self) -> np.ndarray:
        out = np.empty(self._local_count(), dtype=np.float32)
        check(lib().lga_grads(self._h, out.ctypes.data_as(C.c_void_p), out.size, 0))
        return out

    def params(self) -> np.ndarray:
        out = np.empty(self._local_count(), dtype=np.float32)
        check(lib().lga_params(self._h, out.ctypes.data_as(C.c_void_p), out.size, 0))
        return out

    def grads_device(self):
        """lga_grads into a CUDA fp32 tensor (no host round trip; full-size models)."""
        import torch
        out = torch.empty(self._local_count(), dtype=torch.float32, device="cuda")
        check(lib().lga_grads(self._h, C.c_void_p(out.data_ptr()), out.numel(), 1))
        return out

    def params_device(self):
        import torch
        out = torch.empty(self._local_count(), dtype=torch.float32, device="cuda")
        check(lib().lga_params(self._h, C.c_void_p(out.data_ptr()), out.numel(), 1))
        return out

    def save_state(self) -> bytes:
        """lga_save_state: this rank's training state (header + fp32 master / m / v shard) as bytes."""
        n = C.c_uint64()
        check(lib().lga_state_bytes(self._h, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        check(lib().lga_save_state(self._h, buf, n.value))
        return buf.raw

    def load_state(self, state: bytes):
        """lga_load_state: resume from save_state's bytes (same configuration and rank)."""
        buf = C.create_string_buffer(state, len(state))
        check(lib().lga_load_state(self._h, buf, len(state)))

    def comm_stats(self):
        last, tot = _abi.lga_comm_stats(), _abi.lga_comm_stats()
        check(lib().lga_comm_bytes(self._h, C.byref(last), C.byref(tot)))
        return last.as_dict(), tot.as_dict()

    def layer_stage(self):
        arr = (C.c_int32 * self.cfg.layers)()
        check(lib().lga_layer_stage(self._h, arr, self.cfg.layers))
        return list(arr)

    def timing(self):
        t = _abi.lga_timing()
        check(lib().lga_timing_last(self._h, C.byref(t)))
        return t.as_dict()

    def close(self):
        if getattr(self, "_h", None):
            lib().lga_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
