"""Per-kernel warp-stall summary from `ncu --page source --csv --print-source sass`:
stall reasons aggregated over the kernel and the top stalled SASS lines."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
kernels, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        kernels.append(cur)
        continue
    if r and r[0] == "Address":
        cur["hdr"] = r
        continue
    if cur is not None and r:
        cur["rows"].append(r)
for k in kernels:
    h, rs = k["hdr"], k["rows"]
    si = h.index("Warp Stall Sampling (All Samples)")
    cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    tot = sum(int(r[si] or 0) for r in rs)
    agg = {c: sum(int(r[h.index(c)] or 0) for r in rs) for c in cols}
    print(f"### {k['name'][:140]}\n\nsamples {tot}; ", ", ".join(
        f"{c[6:]} {100 * v / max(tot, 1):.0f}%" for v, c in sorted(((v, c) for c, v in agg.items() if v), reverse=True)[:8]))
    print("\n| samples | SASS | main stall |\n|---|---|---|")
    for r in sorted(rs, key=lambda r: -int(r[si] or 0))[:12]:
        st = max(cols, key=lambda c: int(r[h.index(c)] or 0))
        print(f"| {r[si]} | `{r[1].strip()[:70]}` | {st[6:]} |")
    print()
