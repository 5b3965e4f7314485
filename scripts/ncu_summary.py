#!/usr/bin/env python3
"""Summarise an ncu --csv launch list: per-kernel-name launch count, total/mean device time,
share of the step, DRAM bytes per launch. Usage: ncu_summary.py launches.csv [steps]"""
import csv
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    rows = defaultdict(dict)
    names = {}
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    for r in csv.DictReader(lines[start:]):
        if not r.get("ID", "").isdigit():
            continue
        i = int(r["ID"])
        names[i] = (r["Kernel Name"].split("(")[0], r["Grid Size"], r["Block Size"])
        try:
            rows[i][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
        except ValueError:
            pass
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    total = 0.0
    for i, m in rows.items():
        t = m.get("gpu__time_duration.sum", 0.0)
        b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        k = names[i][0]
        agg[k][0] += 1
        agg[k][1] += t
        agg[k][2] += b
        total += t
    print(f"launches={len(rows)} total_device_time={total/1e6:.3f} ms ({total/1e6/steps:.3f} ms/step over {steps} steps)")
    print(f"{'kernel':40s} {'n':>6s} {'total_ms':>9s} {'share':>6s} {'mean_us':>8s} {'MB/launch':>10s} {'GB/s':>7s}")
    for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:40]:40s} {n:6d} {t/1e6:9.3f} {t/total:6.1%} {t/n/1e3:8.2f} {b/n/1e6:10.2f} {b/t if t else 0:7.0f}")


if __name__ == "__main__":
    main()
