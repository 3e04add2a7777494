#!/usr/bin/env python
"""Key metrics of `ncu --page raw --csv` exports (one kernel per file) as a
markdown table: python tools/ncu_raw_summary.py tag=file.csv ..."""
import csv
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__registers_per_thread", "registers"),
    ("launch__block_size", "block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu pipe %"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads / inst"),
    ("smsp__inst_executed.sum", "warp inst"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    # warps stalled per issued instruction (ncu 2025 names; older releases
    # report smsp__average_warp_latency_issue_stalled_*.ratio instead)
] + [(f"smsp__average_warps_issue_stalled_{k}_per_issue_active.ratio", f"stall {lab} / issue")
     for k, lab in (("long_scoreboard", "long_sb"), ("short_scoreboard", "short_sb"),
                    ("wait", "wait"), ("math_pipe_throttle", "math"),
                    ("not_selected", "not_selected"), ("barrier", "barrier"),
                    ("mio_throttle", "mio"), ("lg_throttle", "lg"),
                    ("dispatch_stall", "dispatch"), ("branch_resolving", "branch"))]


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    names, units, vals = rows[hdr], rows[hdr + 1], rows[hdr + 2]
    d = {n: (v, u) for n, u, v in zip(names, units, vals)}
    return d


def main():
    specs = [a.split("=", 1) for a in sys.argv[1:]]
    data = {t: load(p) for t, p in specs}
    tags = [t for t, _ in specs]
    print("| metric | " + " | ".join(tags) + " |")
    print("|---|" + "---|" * len(tags))
    first = data[tags[0]]
    kn = first.get("Kernel Name", ("?", ""))[0]
    for key, label in [("Kernel Name", "kernel")] + METRICS:
        cells = []
        for t in tags:
            v, u = data[t].get(key, None) or data[t].get(
                key.replace("average_warps_issue_stalled_", "average_warp_latency_issue_stalled_")
                   .replace("_per_issue_active", ""), ("-", ""))
            if "_stalled_" in key:
                u = ""
            if key == "Kernel Name":
                v = v.split("(")[0].replace("void wfpg::", "")
                u = ""
            cells.append(f"{v} {u}".strip())
        print(f"| {label} | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main()
