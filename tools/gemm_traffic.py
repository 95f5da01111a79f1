"""GEMM DRAM traffic of one step from a committed ncu launch list (--metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum, every launch of one step), against the algorithmic (compulsory) bytes
of the same GEMMs computed from the layer's shapes; writes the per-launch means bench.py reports as
roofline.traffic (profiles/gemm_traffic.json, keyed by workload).

    python tools/gemm_traffic.py <launches.csv> <workload> <launches_per_step>
"""
import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = {"1.3b": dict(L=24, d=2048, T=16 * 2048, D=1), "gpt2s": dict(L=12, d=768, T=8 * 4 * 1024, D=1)}


def algorithmic_bytes(L, d, T, D, recompute=True):
    """Compulsory bytes of every GEMM of one step (pre-LN layer, bf16 operands, fp32 residual stream; the last
    chunk's weight-gradient epilogue writes the fp32 (D = 1) or bf16 staging, D > 1)."""
    b, f4, f = 2, 4, 4 * d
    g_out = 4 if D == 1 else 2
    fwd = [T * d * b + d * 3 * d * b + T * 3 * d * b,                      # QKV (+ bias)
           T * d * b + d * d * b + T * d * f4 + T * d * f4,                # O-proj (+ residual, fp32 out)
           T * d * b + d * f * b + T * f * b * (1 if recompute else 2),    # FFN1 (+ GELU: g out; u only if kept)
           T * f * b + f * d * b + T * d * f4 + T * d * f4]                # FFN2 (+ residual, fp32 out)
    # the recompute's FFN1 writes u (read by the GELU backward) and g
    rec = fwd[:2] + [T * d * b + d * f * b + 2 * T * f * b] if recompute else []
    bwd = [T * f * b + T * d * b + f * d * g_out,                         # FFN2 wgrad
           T * d * b + f * d * b + T * f * b + T * f * b,                  # FFN2 dgrad (+ GELU' reads u, writes dU)
           T * d * b + T * f * b + d * f * g_out,                          # FFN1 wgrad
           T * f * b + d * f * b + T * d * f4,                             # FFN1 dgrad -> dC fp32
           T * d * b + T * d * b + d * d * g_out,                          # O wgrad
           T * d * b + d * d * b + T * d * b,                              # O dgrad -> dO bf16
           T * d * b + T * 3 * d * b + d * 3 * d * g_out,                  # QKV wgrad
           T * 3 * d * b + 3 * d * d * b + T * d * f4]                     # QKV dgrad -> dA fp32
    per_layer = fwd + rec + bwd
    return L * sum(per_layer), L * len(per_layer)


def main():
    path, workload, per_step = sys.argv[1], sys.argv[2], int(sys.argv[3])
    rows = list(csv.reader(l for l in open(path) if l.startswith('"')))
    h = rows[0]
    ik, iv, im, iid = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name"), h.index("ID")
    by = {}
    for r in rows[1:]:
        d = by.setdefault(int(r[iid]), {"k": r[ik]})
        d[r[im]] = float(r[iv].replace(",", ""))
    ids = sorted(by)[-per_step:]
    gem = [by[i] for i in ids if "gemm_tc" in by[i]["k"]]
    meas = sum(g.get("dram__bytes_read.sum", 0) + g.get("dram__bytes_write.sum", 0) for g in gem)
    alg, n_alg = algorithmic_bytes(**SHAPES[workload])
    out_path = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    data = json.load(open(out_path)) if os.path.exists(out_path) else {}
    data = {k: v for k, v in data.items() if isinstance(v, dict)}
    data[workload] = {"traffic_bytes_per_launch": meas / len(gem), "algorithmic_bytes_per_launch": alg / n_alg,
                      "ratio": (meas / len(gem)) / (alg / n_alg), "gemm_launches": len(gem),
                      "gemm_launches_model": n_alg, "source": os.path.relpath(path, ROOT)}
    json.dump(data, open(out_path, "w"), indent=1)
    print(json.dumps(data[workload]))


if __name__ == "__main__":
    main()
