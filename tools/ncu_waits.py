"""Summarise an ncu source page (SASS) for one kernel: total stall samples, the hottest instructions, and
every mbarrier try-wait with its retry count (the retry loop's executed-instruction count) -- which
barrier each warp role actually waits on.  Development tool.

    python tools/ncu_waits.py report.ncu-rep kernel_regex [top]
"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
i_s, i_e = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
data = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break
    if len(r) > 5:
        data.append(r)
v = lambda r: int(r[i_s] or 0)
print("kernel:", rows[0][1][:90], " total samples:", sum(v(r) for r in data))
for i in sorted(sorted(range(len(data)), key=lambda i: -v(data[i]))[:top]):
    print(f"{i:5d} {v(data[i]):7d}  {data[i][1][:100]}")
print("--- try-waits: line, retries(executed), samples on the following branch, instruction")
for i, r in enumerate(data):
    if "TRYWAIT" in r[1]:
        print(f"{i:5d} {r[i_e]:>10s} {v(data[i + 1]):6d}  {r[1].strip()[:90]}")
