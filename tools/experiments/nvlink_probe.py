"""Which NVML NVLink counters move when 1 GiB crosses GPU0 -> GPU1?"""
import subprocess
import pynvml as nv
import torch
nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(0)
cands = {"XMIT_BYTES(202)": 202, "RCV_BYTES(204)": 204, "TP_DATA_TX(138)": 138, "TP_DATA_RX(139)": 139,
         "TP_RAW_TX(140)": 140, "TP_RAW_RX(141)": 141}
def read():
    out = {}
    for name, fid in cands.items():
        for scope in (0xFFFFFFFF, 0):
            try:
                v = nv.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
                out[f"{name}/s{scope:x}"] = (v.nvmlReturn, int(v.value.ullVal))
            except Exception as e:
                out[f"{name}/s{scope:x}"] = ("exc", str(e)[:40])
    return out
a = read()
x = torch.ones(256 * 1024 * 1024, device="cuda:0")  # 1 GiB
y = torch.empty_like(x, device="cuda:1")
for _ in range(4):
    y.copy_(x)
torch.cuda.synchronize()
b = read()
for k in a:
    print(k, a[k], b[k], (b[k][1] - a[k][1]) if isinstance(a[k][1], int) and isinstance(b[k][1], int) else None)
print(subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", "0"], capture_output=True, text=True).stdout[:1500])
