"""NVLink evidence for the fused peer-memory data path, one process driving two GPUs.

GPU 0 plays the rank that runs the reduce-scatter fused into AdamW (adamw_rs_kernel) for one C3 layer shard
at D = 2: its own staging slice is local, the other replica's is on GPU 1 and is read over NVLink (peer access
enabled both ways, as the IPC mapping does between two processes).  The all-gather's copy-engine pull of the
peer shard is timed the same way.  Run plain for CUDA-event times, and under
    ncu -k regex:adamw_rs --metrics nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
for the kernel's NVLink bytes (expected RX = one bf16 slice = 2 S bytes, S = plpad / 2)."""
import ctypes as C
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2106_02679_b200 import _abi  # noqa: E402

L = _abi.lib()
VP, I, I64, F = C.c_void_p, C.c_int, C.c_int64, C.c_float
L.lgatest_adamw_rs.argtypes = [VP, I64, I, I, F, VP, VP, VP, VP, I, VP, I64, F, F, F, F, F, VP, VP]
L.lgatest_adamw_rs.restype = I
import nvidia.cuda_runtime as _cr  # noqa: E402  the libcudart torch itself loads

RT = C.CDLL(os.path.join(_cr.__path__[0], "lib", "libcudart.so.12"))


def P(t):
    return C.c_void_p(t.data_ptr())


def main():
    d = 2048
    pl = 12 * d * d + 13 * d
    q = 64 * 2
    S = (pl + q - 1) // q * q // 2          # C3 shard per layer at D = 2
    torch.cuda.set_device(0)
    for a, b in ((0, 1), (1, 0)):           # peer access (what cudaIpcMemLazyEnablePeerAccess does)
        torch.cuda.set_device(a)
        torch.empty(1, device=f"cuda:{a}")   # context up
        r = RT.cudaDeviceEnablePeerAccess(b, 0)
        assert r in (0, 704), r              # 704 = already enabled
    torch.cuda.set_device(0)
    g = torch.Generator(device="cuda:0").manual_seed(0)
    local = torch.randn(S, device="cuda:0", generator=g).bfloat16()
    remote = torch.randn(S, device="cuda:0", generator=g).bfloat16().to("cuda:1")
    gbase = torch.tensor([local.data_ptr(), remote.data_ptr()], device="cuda:0", dtype=torch.int64)
    master = torch.randn(S, device="cuda:0", generator=g) * 0.02
    m = torch.zeros(S, device="cuda:0")
    v = torch.zeros(S, device="cuda:0")
    pout = torch.empty(S, device="cuda:0", dtype=torch.bfloat16)
    tstep = torch.ones(1, device="cuda:0", dtype=torch.int64)
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def rs_adam():
        assert L.lgatest_adamw_rs(P(gbase), 0, 2, 1, 1.0 / 32, P(master), P(m), P(v), P(pout), 1, None, S, 1e-4, 0.9,
                                  0.95, 1e-8, 0.0, P(tstep), st) == 0

    slot = torch.empty(S, device="cuda:0", dtype=torch.bfloat16)
    res = {"S_elements": S, "expected_nvlink_rx_bytes_adamw_rs": 2 * S, "expected_gather_bytes": 2 * S}
    for name, fn in (("adamw_rs", rs_adam), ("gather_copy", lambda: slot.copy_(remote, non_blocking=True))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 20
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        res[name + "_ms"] = ms
        if name == "adamw_rs":
            algo = S * (2 * 2 + 24 + 2)   # D bf16 grads + master/m/v read+write + bf16 param
            res["adamw_rs_algorithmic_GBps"] = algo / ms / 1e6
            res["adamw_rs_nvlink_GBps"] = 2 * S / ms / 1e6
        else:
            res["gather_copy_nvlink_GBps"] = 2 * S / ms / 1e6
    print(json.dumps(res))


if __name__ == "__main__":
    main()
