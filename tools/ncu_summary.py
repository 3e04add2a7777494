#!/usr/bin/env python
"""Summarise an ncu launch list (CSV of gpu__time_duration.sum) and/or an
ncu --set full report into markdown for profiles/.

    python tools/ncu_summary.py --launches gpurun_out/launches.csv [--report x.ncu-rep]
"""

import argparse
import collections
import csv
import io
import subprocess


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    starts = [i for i, d in enumerate(data) if "k_init_paths" in d["Kernel Name"]]
    last = data[starts[-1]:] if starts else data
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    agg = collections.OrderedDict()
    for d in last:
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        v = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1e-6)
        a = agg.setdefault(name, [0.0, 0])
        a[0] += v
        a[1] += 1
    tot = sum(v for v, _ in agg.values())
    out = [f"Last pass of `{path}`: {len(last)} launches, {tot:.3f} ms of kernel time "
           "(ncu-serialised, cold caches: compare shares, not absolutes).", "",
           "| kernel | launches | ms | share |", "|---|---|---|---|"]
    for k, (v, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
        out.append(f"| `{k}` | {c} | {v:.3f} | {100 * v / tot:.1f}% |")
    return "\n".join(out)


WANT = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__average_thread_inst_executed_pred_on_per_inst_executed_realtime.ratio",
        "smsp__warps_issue_stalled_long_scoreboard_per_warp_active.pct",
        "smsp__warps_issue_stalled_math_pipe_throttle_per_warp_active.pct",
        "smsp__warps_issue_stalled_wait_per_warp_active.pct",
        "smsp__warps_issue_stalled_short_scoreboard_per_warp_active.pct",
        "smsp__warps_issue_stalled_barrier_per_warp_active.pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum"]


def report(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    out = [f"`{path}` (ncu --set full --clock-control none):", "", "| metric | value |",
           "|---|---|"]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        out.append(f"| kernel | `{d.get('Kernel Name', '')[:80]}` |")
        for k in WANT:
            if k in d:
                out.append(f"| {k} | {d[k]} {u.get(k, '')} |")
    return "\n".join(out)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--report")
    a = ap.parse_args()
    if a.launches:
        print(launches(a.launches))
        print()
    if a.report:
        print(report(a.report))
