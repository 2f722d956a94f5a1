"""Summarise an `ncu --set full` report into profiles/ (markdown + JSON).

    python tools/ncu_summary.py gpurun_out/X.ncu-rep profiles/r01_ncu_full

writes <out>.md (one row per profiled launch) and <out>.json (per kernel:
duration, DRAM bytes read+write per launch -- the `traffic` bench.py reports
-- and the issue / occupancy counters the compositing kernels are bound by).
"""

import csv
import io
import json
import subprocess
import sys
from pathlib import Path

METRICS = {
    "gpu__time_duration.sum": "us",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_pct",
    "smsp__inst_executed.sum": "inst",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__cycles_active.avg": "cyc_avg",
    "sm__cycles_active.max": "cyc_max",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
}


def _num(s):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return None


def main():
    rep, out = Path(sys.argv[1]), Path(sys.argv[2])
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], check=True,
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, data = rows[0], rows[1], rows[2:]
    col = {m: head.index(m) for m in METRICS if m in head}
    kcol = head.index("Kernel Name")
    recs = []
    for r in data:
        rec = {"kernel": r[kcol].split("(")[0].replace("void ", "").split("<")[0]}
        for m, c in col.items():
            v = _num(r[c])
            if m == "gpu__time_duration.sum" and v is not None:
                v *= {"ns": 1e-3, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(units[c].strip(), 1.0)
            if m.startswith("dram__bytes") and v is not None:
                unit = units[c].strip()
                v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            rec[METRICS[m]] = v
        rb, wb = rec.get("dram_read") or 0, rec.get("dram_write") or 0
        rec["traffic_bytes"] = rb + wb
        rec["dram_gbs"] = (rb + wb) / (rec["us"] * 1e-6) / 1e9 if rec.get("us") else None
        recs.append(rec)
    by_kernel = {}
    for rec in recs:
        by_kernel.setdefault(rec["kernel"], rec)
    out.with_suffix(".json").write_text(json.dumps({"report": rep.name, "kernels": by_kernel}, indent=1))
    cols = ["kernel", "us", "traffic_bytes", "dram_gbs", "sm_pct", "issue_pct", "fma_pipe_pct", "warps_pct",
            "regs", "grid", "block", "inst", "cyc_avg", "cyc_max"]
    lines = [f"# ncu --set full summary ({rep.name})", "",
             "Times are ncu's (serialised launch, cache flushed, its own clock control); "
             "use them for shares and counters, not as bench numbers.", "",
             "| " + " | ".join(cols) + " |", "|" + "---|" * len(cols)]
    for rec in recs:
        cells = []
        for c in cols:
            v = rec.get(c)
            cells.append(f"{v:.4g}" if isinstance(v, float) else str(v))
        lines.append("| " + " | ".join(cells) + " |")
    out.with_suffix(".md").write_text("\n".join(lines) + "\n")
    print(out.with_suffix(".md"))


if __name__ == "__main__":
    main()
