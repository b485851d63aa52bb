"""Summarise an ncu --set full capture (.ncu-rep) into profiles/.

usage: python tools/ncu_summary.py <report.ncu-rep> <out-prefix> [--traffic]

Writes <out-prefix>.json (per-kernel key metrics) and <out-prefix>.md (a
table); with --traffic also updates profiles/ncu_traffic.json, which
bench.py reads for the roofline "traffic" field (dram read + write bytes per
launch of the kernel)."""

import csv
import io
import json
import re
import subprocess
import sys
from pathlib import Path

KEYS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio": "stall_long_sb",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio": "stall_barrier",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "smsp__inst_executed.sum": "warp_inst",
    "smsp__sass_inst_executed_op_local_ld.sum": "local_ld",
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "ns": 1, "usecond": 1e3,
              "us": 1e3, "msecond": 1e6, "ms": 1e6}


def main():
    rep, prefix = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(head, r))
        u = dict(zip(head, units))
        name = d.get("Kernel Name", "")
        short = re.sub(r"\(.*", "", name)
        k = {"kernel": short, "id": d.get("ID")}
        for key, alias in KEYS.items():
            if key in d and d[key] not in ("", "n/a"):
                v = float(d[key].replace(",", ""))
                v *= UNIT_SCALE.get(u.get(key, ""), 1)
                k[alias] = v
        if "dram_read" in k:
            k["dram_bytes"] = k["dram_read"] + k.get("dram_write", 0.0)
        if "duration_ns" in k and "dram_bytes" in k:
            k["dram_gbs"] = k["dram_bytes"] / k["duration_ns"]
        out.append(k)
    Path(prefix + ".json").write_text(json.dumps(out, indent=1))
    cols = ["kernel", "duration_ns", "dram_bytes", "dram_gbs", "regs", "grid", "warps_active_pct",
            "issue_active_pct", "stall_long_sb", "l2_hit_pct", "local_ld"]
    lines = ["| " + " | ".join(cols) + " |", "|" + "---|" * len(cols)]
    for k in out:
        cells = []
        for c in cols:
            v = k.get(c, "")
            cells.append(f"{v:.4g}" if isinstance(v, float) else str(v))
        lines.append("| " + " | ".join(cells) + " |")
    Path(prefix + ".md").write_text("\n".join(lines) + "\n")
    print("\n".join(lines))
    if "--traffic" in sys.argv:
        tp = Path(__file__).resolve().parents[1] / "profiles" / "ncu_traffic.json"
        cur = json.loads(tp.read_text()) if tp.exists() else {}
        for k in out:
            m = re.match(r"(?:void )?(k_\w+)<.*?(Op\w+)", k["kernel"])
            if m and "dram_bytes" in k:
                cur[f"{m.group(1)}<{m.group(2)}>"] = k["dram_bytes"]
        tp.write_text(json.dumps(cur, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
