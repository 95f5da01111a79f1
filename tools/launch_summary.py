"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel: share, launches, ns.

    python tools/launch_summary.py gpurun_out/launches_r1_final.csv [--last N] [header lines...]

--last N: only the last N launches of the list (one step: bench.py prints gpu_launches_per_step).
"""
import csv
import re
import sys
from collections import defaultdict

args = sys.argv[2:]
last = None
if args[:1] == ["--last"]:
    last, args = int(args[1]), args[2:]
rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
hdr = rows[0]
ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
iid = hdr.index("ID")
ids = sorted({int(r[iid]) for r in rows[1:] if len(r) > iv})
keep = set(ids[-last:]) if last else set(ids)
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows[1:]:
    if len(r) <= iv or r[im] != "gpu__time_duration.sum" or int(r[iid]) not in keep:
        continue
    name = re.sub(r"\(.*", "", r[ik]).replace("lga::", "")
    tot[name] += float(r[iv].replace(",", ""))
    cnt[name] += 1
s = sum(tot.values())
for line in args:
    print("#", line)
print(f"# {sum(cnt.values())} launches; unit ns\n")
print(f"  share launches         sum_ns  kernel")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{100 * tot[k] / s:6.1f}% {cnt[k]:8d} {tot[k]:14.0f}  {k}")
g = sum(v for k, v in tot.items() if "gemm" in k)
a = sum(v for k, v in tot.items() if "fat" in k)
print(f"\n# GEMM family share {100 * g / s:.1f}%, attention {100 * a / s:.1f}%")
