"""One line per profiled launch of an ncu --set full report: duration, DRAM traffic, pipe utilisation.

    python tools/ncu_summary.py report.ncu-rep [header ...]
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "sm__cycles_elapsed.avg.per_second"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
for line in sys.argv[2:]:
    print("#", line)
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    parts = [f"{k}={r[hdr.index(k)]} {units[hdr.index(k)]}".strip() for k in KEYS if k in hdr]
    print(f"{name[:60]}; grid={r[hdr.index('Grid Size')]}; " + "; ".join(parts))
