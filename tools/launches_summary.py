"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into a
markdown table of kernels: launches, average duration, share of the total.

usage: python tools/launches_summary.py <launches.csv> <out.md> [title]"""

import csv
import sys
from collections import defaultdict


def main():
    src, dst = sys.argv[1], sys.argv[2]
    title = sys.argv[3] if len(sys.argv) > 3 else "ncu launch list"
    lines = open(src).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for row in csv.DictReader(lines[start:]):
        if row.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(row["Metric Value"].replace(",", ""))
        unit = row.get("Metric Unit", "ns")
        v = v * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1e-3)
        k = row["Kernel Name"][:90]
        tot[k] += v
        cnt[k] += 1
    total = sum(tot.values()) or 1.0
    out = [f"{title} (cold-cache, serialised: compare shares)", "",
           "| kernel | launches | avg us | share |", "|---|---|---|---|"]
    for k in sorted(tot, key=lambda k: -tot[k]):
        out.append(f"| {k} | {cnt[k]} | {tot[k] / cnt[k]:.2f} | {100 * tot[k] / total:.1f}% |")
    open(dst, "w").write("\n".join(out) + "\n")
    print("\n".join(out[:12]))


if __name__ == "__main__":
    main()
