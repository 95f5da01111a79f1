#!/usr/bin/env python
"""bench.py -- tokens/s of the B200-native layered-gradient-accumulation (LGA) training step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload 1.3b|gpt2s|10b|tiny] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...          (N > 1, one process per GPU)

One step = one full pass of the hot path over one batch: layer-major
forward over all N micro-batches with the all-gather of the next layer overlapped, MSE loss,
layer-major recompute + backward with in-place fp32 gradient accumulation, reduce-scatter and
sharded AdamW overlapped with the next layer's backward.  Default workload: the 1.3B config
(BASELINE.json configs[2]: L=24, d=2048, s=2048, b=1, N=16 per replica) with D = N GPUs (weak
scaling; the metric's targets -- >=7x over 1 GPU, exposed comm < 10%, GEMM tensor pipe >= 60% --
are stated at this config).  Inputs are synthetic (N(0,1) activations and targets, generated once
on the device and reused), parameters random-init ("train" recipe), state partitioned.

Prints ONE JSON line on rank 0.  `value` is device-timed (CUDA events on the caller stream around
K steps, barrier + synchronize on both sides, max over ranks).  `e2e` is the same metric through
lga_step_host with pinned host inputs copied in every step and the loss read back every step.
`roofline` is for the dominant kernel family (the tcgen05 GEMM), from per-launch CUDA events
recorded by the library on its compute stream during the timed steps (LGA_FLAG_PROFILE).
`cpu_baseline` times the fp64 oracle (oracle/, the one place bench.py runs it) on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "training tokens/s per box at 1/2/4/8 B200; exposed comm ms/step"

WORKLOADS = {
    # name: (description, per-replica shape, pipeline degree)
    "1.3b": ("1.3B L=24 d=2048 16 heads s=2048, b=1 x N=16 per replica, ZeRO-partitioned, layered GA",
             dict(layers=24, d_model=2048, heads=16, seq_len=2048, micro_batch=1, n_micro=16), 1),
    "gpt2s": ("GPT-2-small-shaped L=12 d=768 12 heads s=1024, b=4 x N=8 per replica",
              dict(layers=12, d_model=768, heads=12, seq_len=1024, micro_batch=4, n_micro=8), 1),
    "10b": ("~10B L=48 d=4096 32 heads s=2048, b=1 x N=32, modular pipeline P=4 x data-parallel D",
            dict(layers=48, d_model=4096, heads=32, seq_len=2048, micro_batch=1, n_micro=32), 4),
    # N4: the paper's own encoder family X_[x] (d_a = x/2 heads, d_h = 2x, d_l = x, d_s = 16x, d_m = x^2;
    # P:444-452), bidirectional attention; pre-LN as everywhere (reading A-1)
    "x32": ("X_32 encoder L=32 d=1024 16 heads s=512 non-causal, b=8 x N=8 per replica",
            dict(layers=32, d_model=1024, heads=16, seq_len=512, micro_batch=8, n_micro=8, causal=0), 1),
    "tiny": ("tiny L=2 d=64 4 heads s=32, b=2 x N=4 (fp32)",
             dict(layers=2, d_model=64, heads=4, seq_len=32, micro_batch=2, n_micro=4), 1),
}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured (MEASURED_PEAKS.json)"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, \
        "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device=0):
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")
        # the physical GPU this rank drives (nvidia-smi lists every GPU of the box)
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        self.index = vis.split(",")[device].strip() if vis else str(device)

    def start(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", self.index, f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append(dict(sm=float(parts[1]), smax=float(parts[2]), power=float(parts[3]),
                                 hw=parts[5], hwt=parts[6], swt=parts[7], swp=parts[8]))
            except ValueError:
                continue
        if not rows:
            return None
        load = [r for r in rows if r["power"] > 250.0] or rows
        reasons = set()
        for r in rows:
            for k, name in (("hw", "hw_slowdown"), ("hwt", "hw_thermal_slowdown"), ("swt", "sw_thermal_slowdown"),
                            ("swp", "sw_power_cap")):
                if r[k].lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(r["sm"] for r in load), "sm_max_mhz": max(r["smax"] for r in rows),
                "samples": len(rows), "samples_under_load": len(load), "reasons": sorted(reasons)}


class NvlinkCounters:
    """NVLink payload byte counters of this rank's GPU (NVML field values, all links summed), read around the
    timed region: the transfers the peer-memory data path really put on NVLink, per step."""
    TX, RX = 138, 139   # NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX / _RX (KiB, cumulative)

    def __init__(self, device=0):
        self.ok = False
        try:
            import pynvml as nv
            nv.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[device]) if vis else device
            self.nv, self.h = nv, nv.nvmlDeviceGetHandleByIndex(idx)
            self.ok = self.read() is not None
        except Exception:
            self.ok = False

    def read(self):
        try:
            nv = self.nv
            vals = nv.nvmlDeviceGetFieldValues(self.h, [(self.TX, 0xFFFFFFFF), (self.RX, 0xFFFFFFFF)])
            out = []
            for v in vals:
                if v.nvmlReturn != 0:
                    return None
                out.append(int(v.value.ullVal) * 1024)
            return out
        except Exception:
            return None


# ----------------------------------------------------------------------------- oracle (CPU) arm
POST_LN = [False]   # --post-ln: the oracle sample runs the same layer variant as the timed path


def oracle_sample_seconds(shape: dict, repeats: int = 1):
    """Time the fp64 oracle, as it stands, on one layer x one micro-batch forward + backward of the
    workload's shape (the bounded sample); returns (seconds per sample, threads used)."""
    import numpy as np

    import synth
    from oracle import model as om
    sh = synth.Shape(layers=1, d=shape["d_model"], heads=shape["heads"], seq=shape["seq_len"],
                     micro_batch=shape["micro_batch"], n_micro=1)
    flat = synth.init_params(sh, style="train").astype(np.float64)
    X, T = synth.batch(sh, step=0)
    cfg = om.LayerCfg(d=sh.d, heads=sh.heads, causal=bool(shape.get("causal", 1)), post_ln=POST_LN[0])
    try:
        from threadpoolctl import threadpool_info
        threads = max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        threads = len(os.sched_getaffinity(0))
    best = None
    for _ in range(repeats):
        t0 = time.perf_counter()
        y, cache = om.layer_forward(X[0, 0].astype(np.float64), flat, cfg)
        _, dy = om.mse_loss(y, T[0, 0].astype(np.float64))
        om.layer_backward(dy, cache, flat, cfg)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return best, threads


def cpu_baseline(shape: dict, repeats: int = 1):
    sec, threads = oracle_sample_seconds(shape, repeats)
    tokens = shape["micro_batch"] * shape["seq_len"]
    # one micro-batch through all L layers takes L samples; tokens/s of the oracle on this host
    value = tokens / (sec * shape["layers"])
    return {"value": value, "unit": "tokens/s", "cores": threads, "kind": "oracle",
            "sample": f"oracle.model fp64 forward+backward of 1 layer x 1 micro-batch "
                      f"(b*s={tokens} tokens, d={shape['d_model']}), best of {repeats}, "
                      f"{sec:.2f} s, extrapolated x {shape['layers']} layers"}


def run_reference(args, shape, desc, world, rank):
    if rank != 0:
        return 0
    secs = []
    threads = 1
    for _ in range(args.warmup):
        oracle_sample_seconds(shape, 1)
    for _ in range(args.steps):
        s, threads = oracle_sample_seconds(shape, 1)
        secs.append(s)
    ms = statistics.mean(secs) * 1000.0
    tokens = shape["micro_batch"] * shape["seq_len"]
    value = tokens / (statistics.mean(secs) * shape["layers"])
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc, "per_step_sample": "1 layer x 1 micro-batch, extrapolated to the model"},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "oracle",
                             "sample": "oracle.model fp64 fwd+bwd of 1 layer x 1 micro-batch per step, x L layers"},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="1.3b", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--schedule", default="layered", choices=["layered", "standard"])
    ap.add_argument("--chunk", type=int, default=0)
    ap.add_argument("--n-micro", type=int, default=0, help="override N (micro-batch count sweep, config 5)")
    ap.add_argument("--no-comm", action="store_true", help="A/B: skip collectives (exposed-comm measurement)")
    ap.add_argument("--keep-params", action="store_true", help="N2a: keep forward gathers (1 AG per layer per step)")
    ap.add_argument("--unpartitioned", action="store_true", help="N2b: no ZeRO partition, all-reduce per layer")
    ap.add_argument("--no-recompute", action="store_true", help="N2c: keep intermediates, no forward recompute")
    ap.add_argument("--pipeline", default="modular", choices=["modular", "contiguous"], help="N3: stage map")
    ap.add_argument("--nccl-dp", action="store_true", help="N1 baseline: NCCL all-gather / reduce-scatter")
    ap.add_argument("--post-ln", action="store_true", help="N4: post-LN layer (original encoder, reading A-16)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ab", action="store_true", help="skip the no-comm A/B run (second exposed-comm measure)")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    POST_LN[0] = args.post_ln

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    desc, shape, pp = WORKLOADS[args.workload]
    shape = dict(shape)
    if args.n_micro:
        shape["n_micro"] = args.n_micro
    if args.impl == "reference":
        return run_reference(args, shape, desc, world, rank)

    import torch
    from paper_2106_02679_b200 import LGA_BF16, LGA_FP32, LGA_LAYERED, LGA_STANDARD, Config, Trainer, _abi

    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    ngpu = max(1, torch.cuda.device_count())
    shared = world > ngpu            # more ranks than GPUs: ranks share devices (peer memory over CUDA IPC)
    local = local % ngpu
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        # NCCL refuses two ranks on one device: gloo for the harness's own barriers when ranks share GPUs
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    if world % pp:
        raise SystemExit(f"workload {args.workload} needs a multiple of {pp} GPUs")
    dp = world // pp
    precision = LGA_FP32 if args.workload == "tiny" else LGA_BF16
    flags = _abi.LGA_FLAG_PROFILE | (_abi.LGA_FLAG_NO_COMM if args.no_comm else 0)
    variant = [n for n, on in (("keep_params", args.keep_params), ("unpartitioned", args.unpartitioned),
                               ("no_recompute", args.no_recompute), ("contiguous_pp", args.pipeline == "contiguous"),
                               ("nccl_dp", args.nccl_dp), ("post_ln", args.post_ln)) if on]
    flags |= ((_abi.LGA_FLAG_KEEP_PARAMS if args.keep_params else 0) | (_abi.LGA_FLAG_UNPARTITIONED if args.unpartitioned else 0)
              | (_abi.LGA_FLAG_NO_RECOMPUTE if args.no_recompute else 0)
              | (_abi.LGA_FLAG_CONTIGUOUS_PP if args.pipeline == "contiguous" else 0)
              | (_abi.LGA_FLAG_NCCL_DP if args.nccl_dp else 0) | (_abi.LGA_FLAG_POST_LN if args.post_ln else 0))
    cfg = Config(dp=dp, pp=pp, precision=precision, chunk=args.chunk,
                 schedule=LGA_LAYERED if args.schedule == "layered" else LGA_STANDARD, flags=flags, **shape)
    tr = Trainer(cfg, rank=rank, world=world, device=local, init_params=None, seed=1234)
    stream = tr.stream
    # synthetic inputs, generated once on the device and reused (data loading is not on the path)
    N, b, s, d = shape["n_micro"], shape["micro_batch"], shape["seq_len"], shape["d_model"]
    gen = torch.Generator(device="cuda").manual_seed(5678 + tr.replica)
    x = torch.randn((N, b, s, d), device="cuda", generator=gen, dtype=torch.float32)
    tgt = torch.randn((N, b, s, d), device="cuda", generator=gen, dtype=torch.float32)
    in_bytes = x.numel() * 4

    def barrier():
        if dist is not None:
            dist.barrier()

    def all_ranks(v: float) -> list:
        if dist is None:
            return [v]
        dev = "cpu" if shared else "cuda"
        out = [torch.zeros(1, device=dev, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(out, torch.tensor([v], device=dev, dtype=torch.float64))
        return [float(t.item()) for t in out]

    def max_over_ranks(v: float) -> float:
        if dist is None:
            return v
        t = torch.tensor([v], device="cpu" if shared else "cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            tr.step(x, tgt, sync=False)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        clocks = ClockSampler(local) if rank == 0 else None
        if clocks:
            clocks.start()
        nvl = NvlinkCounters(local) if world > 1 else None
        nvl0 = nvl.read() if nvl and nvl.ok else None
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        step_ms = []   # per-step device time (library events on the caller stream), for median / p90
        prof = dict(gemm_ms=0.0, gemm_flop=0.0, gemm_launches=0, attn_ms=0.0, attn_flop=0.0, adam_ms=0.0,
                    adam_bytes=0.0, comm_wait_ms=0.0, p2p_wait_ms=0.0, launches=0)
        e0.record(stream)
        for _ in range(args.steps):
            tr.step(x, tgt, sync=False)
            t = tr.timing()      # waits for this step's completion event; reads its launch events
            for k in ("gemm_ms", "gemm_flop", "gemm_launches", "attn_ms", "attn_flop", "adam_ms", "adam_bytes",
                      "comm_wait_ms", "p2p_wait_ms"):
                prof[k] += t[k]
            prof["launches"] += int(t["kernel_launches"])
            step_ms.append(float(t["step_ms"]))
        e1.record(stream)
        torch.cuda.synchronize()
        nvl1 = nvl.read() if nvl0 is not None else None
        barrier()
        torch.cuda.synchronize()
        clk = clocks.stop() if clocks else None
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    stall_ranks = all_ranks(prof["comm_wait_ms"] / args.steps)
    p2p_ranks = all_ranks(prof["p2p_wait_ms"] / args.steps)
    stats_last, _ = tr.comm_stats()
    nvlink = None
    if nvl1 is not None:
        nvlink = {"tx_bytes_per_step": (nvl1[0] - nvl0[0]) / args.steps, "rx_bytes_per_step": (nvl1[1] - nvl0[1]) / args.steps,
                  "counted_bytes_per_step": stats_last["ag_bytes"] + stats_last["rs_bytes"] + stats_last["p2p_send_bytes"]
                  + stats_last["allreduce_bytes"],
                  "source": "NVML NVLink data throughput counters (rank 0's GPU, all links), timed region"}
    tokens_per_step = dp * N * b * s
    value = tokens_per_step / (ms / 1000.0)

    # ---- end to end through the public API: pinned host inputs copied in, loss read back, every step
    e2e = None
    if not args.no_e2e:
        xh = x.cpu().pin_memory()
        th = tgt.cpu().pin_memory()
        import ctypes as C
        xp = C.c_void_p(xh.data_ptr()) if tr.stage == 0 else None
        tp = C.c_void_p(th.data_ptr()) if (shape["layers"] - 1) % pp == tr.stage else None
        loss = C.c_double()
        with torch.cuda.stream(stream):
            for _ in range(2):
                _abi.check(_abi.lib().lga_step_host(tr._h, xp, tp, C.byref(loss)))
            torch.cuda.synchronize()
            barrier()
            f0 = torch.cuda.Event(enable_timing=True)
            f1 = torch.cuda.Event(enable_timing=True)
            f0.record(stream)
            for _ in range(args.steps):
                _abi.check(_abi.lib().lga_step_host(tr._h, xp, tp, C.byref(loss)))
            f1.record(stream)
            torch.cuda.synchronize()
            barrier()
        e2e_ms = max_over_ranks(f0.elapsed_time(f1) / args.steps)
        h2d = (in_bytes if xp is not None else 0) + (in_bytes if tp is not None else 0)
        e2e = {"value": tokens_per_step / (e2e_ms / 1000.0), "unit": "tokens/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 8, "loss": loss.value}

    # ---- second exposed-comm measure: the same step with every transfer skipped after the
    # first (LGA_FLAG_NO_COMM), on the same GPUs right after; exposed = T(step) - T(step without comm)
    ab = None
    if world > 1 and not args.no_comm and not args.no_ab:
        tr.close()
        cfg_ab = Config(dp=dp, pp=pp, precision=precision, chunk=args.chunk,
                        schedule=LGA_LAYERED if args.schedule == "layered" else LGA_STANDARD,
                        flags=(flags | _abi.LGA_FLAG_NO_COMM) & ~_abi.LGA_FLAG_PROFILE, **shape)
        tr_ab = Trainer(cfg_ab, rank=rank, world=world, device=local, init_params=None, seed=1234)
        with torch.cuda.stream(tr_ab.stream):
            for _ in range(args.warmup):
                tr_ab.step(x, tgt, sync=False)
            torch.cuda.synchronize()
            barrier()
            a0 = torch.cuda.Event(enable_timing=True)
            a1 = torch.cuda.Event(enable_timing=True)
            a0.record(tr_ab.stream)
            for _ in range(args.steps):
                tr_ab.step(x, tgt, sync=False)
            a1.record(tr_ab.stream)
            torch.cuda.synchronize()
            barrier()
        ab_ms = max_over_ranks(a0.elapsed_time(a1) / args.steps)
        tr_ab.close()
        tr = None
        ab = {"no_comm_ms_per_step": ab_ms, "exposed_comm_ms_per_step": ms - ab_ms,
              "frac_of_step": (ms - ab_ms) / ms}

    peaks, peak_src = measured_peaks()
    gemm_tflops = prof["gemm_flop"] / (prof["gemm_ms"] / 1000.0) / 1e12 if prof["gemm_ms"] > 0 else 0.0
    peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
    # measured DRAM bytes per GEMM launch from the committed launch list of this workload's step
    # (tools/gemm_traffic.py -> profiles/gemm_traffic.json), beside the algorithmic (compulsory) bytes
    traffic, traffic_info = None, None
    tp_path = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    if os.path.exists(tp_path):
        try:
            traffic_info = json.load(open(tp_path)).get(args.workload)
            traffic = traffic_info["traffic_bytes_per_launch"] if isinstance(traffic_info, dict) else None
        except Exception:
            traffic, traffic_info = None, None
    roofline = {"bound": "tensor", "kernel": "gemm_tc_kernel (tcgen05 bf16, all GEMM launches of the step)",
                "achieved": gemm_tflops, "peak": peak, "unit": "TFLOP/s",
                "frac": gemm_tflops / peak if peak else None, "traffic": traffic,
                "traffic_detail": traffic_info,
                "peak_source": peak_src + " bf16_tflops_sustained (kernel timed inside a long step)",
                "launches": prof["gemm_launches"],
                "flop_per_launch": prof["gemm_flop"] / max(1, prof["gemm_launches"]),
                "avg_launch_ms": prof["gemm_ms"] / max(1, prof["gemm_launches"]),
                "share_of_step": prof["gemm_ms"] / (ms * args.steps) if ms > 0 else None}
    others = {"attention": {"achieved_tflops": prof["attn_flop"] / (prof["attn_ms"] / 1e3) / 1e12 if prof["attn_ms"] else 0,
                            "share_of_step": prof["attn_ms"] / (ms * args.steps)},
              "adamw": {"achieved_gbs": prof["adam_bytes"] / (prof["adam_ms"] / 1e3) / 1e9 if prof["adam_ms"] else 0,
                        "peak_gbs": peaks.get("hbm_gbs"), "share_of_step": prof["adam_ms"] / (ms * args.steps)}}
    if rank != 0:
        if tr is not None:
            tr.close()
        if dist is not None:
            dist.destroy_process_group()
        return 0
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(shape, repeats=1)
    from oracle import counters as oc
    fpt = oc.flops_per_token_model(shape["layers"], d, s)
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": min(world, ngpu), "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16" if precision == LGA_BF16 else "f32", "data": "synthetic",
        "config": {"workload": desc, "layers": shape["layers"], "d_model": d, "heads": shape["heads"], "seq_len": s,
                   "micro_batch": b, "n_micro": N, "dp": dp, "pp": pp, "global_batch": dp * N * b,
                   "tokens_per_step": tokens_per_step, "schedule": args.schedule,
                   "chunk": cfg.chunk or ("N" if pp == 1 else cfg.plan(rank)["chunk"]), "parallelism": f"dp{dp}" + (f"xpp{pp}" if pp > 1 else ""),
                   "l2": f"inputs larger than L2 (x and target {in_bytes / 1e6:.0f} MB each per replica, reused)",
                   "no_comm": bool(args.no_comm), "ranks": world,
                   "ranks_share_gpus": bool(shared), "variant": variant or "paper default (partitioned, recompute, modular); DP over NVLink peer memory"},
        "step_ms_median": statistics.median(step_ms) if step_ms else None,
        "step_ms_p90": sorted(step_ms)[min(len(step_ms) - 1, int(0.9 * len(step_ms)))] if step_ms else None,
        "exposed_comm_ms_per_step": prof["comm_wait_ms"] / args.steps,
        "exposed_comm_ab": ab,
        "nvlink": nvlink,
        "p2p_wait_ms_per_step": prof["p2p_wait_ms"] / args.steps,
        # per rank (rank order): a pipeline stage on a faster GPU also waits for the slowest stage; the minimum
        # over ranks is the bubble the schedule itself leaves
        "exposed_comm_ms_per_step_ranks": stall_ranks,
        "p2p_wait_ms_per_step_ranks": p2p_ranks,
        "model_tflops_per_gpu": value * fpt / world / 1e12,
        "mfu_vs_measured_peak": value * fpt / world / 1e12 / peaks.get("bf16_tflops", 1620.5),
        "roofline": roofline,
        "kernels": others,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": prof["launches"],
        "gpu_launches_per_step": prof["launches"] / args.steps,
        "comm_last_step_rank0": stats_last,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    if tr is not None:
        tr.close()
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
