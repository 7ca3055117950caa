#!/usr/bin/env python
"""Summarise ncu evidence into profiles/ (tracked).

    python tools/summarize_ncu.py launches <launches.csv> <out.md>
    python tools/summarize_ncu.py full <report.ncu-rep> <out.md> [--algo-bytes B] [--pair-evals P]

``launches``: the per-launch gpu__time_duration list of one bench command
(cold-cache, serialised: compare SHARES, not absolutes).
``full``: the headline metrics of one ``ncu --set full`` capture (pipe
utilisation, issue, occupancy, stall reasons, DRAM traffic).
"""
from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from collections import defaultdict


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("void ", "")
        agg[name].append(float(r[vi].replace(",", "")))
    total = sum(sum(v) for v in agg.values())
    lines = [f"# ncu launch list: `{path}`", "",
             "gpu__time_duration.sum per launch (ncu, --clock-control none; cold-cache and "
             "serialised, so compare shares, not absolutes)", "",
             "| kernel | launches | mean us | total us | share |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / 1e3:.1f} | "
                     f"{sum(v) / total:.4f} |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


WANT = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__waves_per_multiprocessor",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
]


def full(path, out, algo_bytes=None, pair_evals=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines = [f"# ncu --set full: `{path}`", ""]
    summary = []
    for r in rows[2:]:
        rec = dict(zip(hdr, r))
        name = rec.get("Kernel Name", "?").split("(")[0].replace("void ", "")
        lines += [f"## `{name}`", "", "| metric | value | unit |", "|---|---|---|"]
        vals = {}
        for k in WANT:
            if k in rec:
                lines.append(f"| {k} | {rec[k]} | {units[hdr.index(k)]} |")
                vals[k] = rec[k]
        try:
            rd = float(rec["dram__bytes_read.sum"].replace(",", ""))
            wr = float(rec["dram__bytes_write.sum"].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd *= scale.get(units[hdr.index("dram__bytes_read.sum")], 1)
            wr *= scale.get(units[hdr.index("dram__bytes_write.sum")], 1)
            vals["dram_traffic_bytes"] = rd + wr
            lines.append(f"| dram traffic (read+write) | {rd + wr:.4g} | byte |")
            if algo_bytes:
                lines.append(f"| algorithmic bytes (12 B/unit) | {algo_bytes:.4g} | byte |")
        except (KeyError, ValueError):
            pass
        lines.append("")
        summary.append({"kernel": name, **vals})
    open(out, "w").write("\n".join(lines) + "\n")
    json.dump(summary, open(out.rsplit(".", 1)[0] + ".json", "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        kw = {}
        if "--algo-bytes" in sys.argv:
            kw["algo_bytes"] = float(sys.argv[sys.argv.index("--algo-bytes") + 1])
        full(sys.argv[2], sys.argv[3], **kw)
