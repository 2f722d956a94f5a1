"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python tools/launch_summary.py gpurun_out/launches.csv profiles/r01_launches

writes <out>.csv (the raw per-launch list, our kernels only) and <out>.md
(per kernel: launches, total / mean us, share of the listed time).  ncu
serialises launches and flushes caches, so shares -- not absolute times --
are what to compare with bench.py's in-graph stage timing.
"""

import csv
import sys
from collections import OrderedDict
from pathlib import Path


def main():
    src, out = Path(sys.argv[1]), Path(sys.argv[2])
    rows = [r for r in csv.reader(src.open()) if len(r) > 10]
    head = rows[0]
    ki, vi, ui = head.index("Kernel Name"), head.index("Metric Value"), head.index("Metric Unit")
    recs = []
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("void ", "")
        v = float(r[vi].replace(",", ""))
        v = v / 1e3 if r[ui].strip() == "ns" else (v * 1e3 if r[ui].strip() == "ms" else v)
        recs.append((name, v))
    with out.with_suffix(".csv").open("w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["launch", "kernel", "us"])
        for i, (n, v) in enumerate(recs):
            w.writerow([i, n, f"{v:.3f}"])
    agg = OrderedDict()
    for n, v in recs:
        a = agg.setdefault(n, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    lines = [f"# ncu launch list summary ({src.name}, {len(recs)} launches)", "",
             "| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
    for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| {n} | {c} | {t:.1f} | {t / c:.2f} | {100 * t / tot:.1f}% |")
    out.with_suffix(".md").write_text("\n".join(lines) + "\n")
    print(out.with_suffix(".md"))


if __name__ == "__main__":
    main()
