#!/usr/bin/env python3
"""Join an ncu launch list of decode steps (gpu__time_duration + dram bytes per launch) with the
event-timed step profile (algorithmic bytes per family) into profiles/ncu_traffic.json, which
bench.py reads for roofline.traffic.

  ncu_traffic.py <launches.csv> <step_prof.json> <steps> [out.json]
"""
import csv
import json
import sys
from collections import defaultdict

FAMILY = [("gemm_sk_kernel", "gemm"), ("attn_decode_kernel", "attention"),
          ("attn_prefill", "attention"), ("attn_combine_kernel", "attention"),
          ("rms_stats_kernel", "rms"), ("gather_rows_kernel", "gather"),
          ("scatter_rows_kernel", "scatter")]


def family(name):
    for key, fam in FAMILY:
        if key in name:
            return fam
    return name


def main():
    path, prof_path, steps = sys.argv[1], sys.argv[2], int(sys.argv[3])
    out = sys.argv[4] if len(sys.argv) > 4 else None
    lines = open(path).read().splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
    rows, names = defaultdict(dict), {}
    for r in csv.DictReader(lines[start:]):
        if not r.get("ID", "").isdigit():
            continue
        i = int(r["ID"])
        names[i] = r["Kernel Name"]
        try:
            rows[i][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
        except ValueError:
            pass
    agg = defaultdict(lambda: {"kernels": 0, "ns": 0.0, "dram": 0.0})
    for i, m in rows.items():
        a = agg[family(names[i])]
        a["kernels"] += 1
        a["ns"] += m.get("gpu__time_duration.sum", 0.0)
        a["dram"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    prof = json.load(open(prof_path))["families"]
    total_ns = sum(a["ns"] for a in agg.values())
    res = {}
    for fam, a in agg.items():
        p = prof.get(fam, {})
        launches = p.get("launches", 0) * steps  # exec_batch launches (attention: + combine)
        per = launches or a["kernels"]
        res[fam] = {"dram_bytes_per_launch": round(a["dram"] / per),
                    "algorithmic_bytes_per_launch": round(p["bytes"] / p["launches"]) if p else None,
                    "kernels": a["kernels"], "launches": launches,
                    "ncu_us_per_launch": round(a["ns"] / per / 1e3, 2),
                    "ncu_share": round(a["ns"] / total_ns, 4),
                    "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over "
                              f"{steps} C2 decode step(s) (NVTX range 'step'), {a['kernels']} "
                              f"kernels; cold per-launch serialised replay"}
    txt = json.dumps(res, indent=1)
    print(txt)
    if out:
        with open(out, "w") as f:
            f.write(txt + "\n")


if __name__ == "__main__":
    main()
