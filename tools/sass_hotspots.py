#!/usr/bin/env python
"""Per-source-line instruction / stall hotspots of one kernel in an ncu report.

ncu's CSV source page lists SASS with per-instruction counters but (for our
reports) no CUDA-line mapping; nvdisasm -gi on the cubin gives the mapping.
This joins the two by instruction order.

    python tools/sass_hotspots.py REPORT.ncu-rep "k_fields<(int)128>" fields 'k_fieldsILi128'
"""

import csv
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(REPO, "paper_2405_06997_b200", "csrc")


def ncu_rows(report, kernel):
    txt = subprocess.run(["ncu", "-i", report, "--page", "source", "--csv", "--print-source",
                          "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name" and kernel in r[1]]
    if not starts:
        raise SystemExit(f"kernel {kernel!r} not in report")
    s = starts[0]
    e = next((i for i in range(s + 1, len(rows)) if rows[i] and rows[i][0] == "Kernel Name"),
             len(rows))
    return rows[s + 1], rows[s + 2:e]


def sass_lines(cubin_stem, func_sub):
    tmp = tempfile.mkdtemp()
    lib = os.path.join(REPO, "paper_2405_06997_b200", "libwfpg_b200.so")
    subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, capture_output=True)
    cub = [f for f in os.listdir(tmp) if f.startswith(cubin_stem) and f.endswith(".cubin")][0]
    txt = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(tmp, cub)], capture_output=True,
                         text=True).stdout
    parts = re.split(r"\n\s*\.text\.(\S+):", txt)
    body = next(parts[i + 1] for i in range(1, len(parts), 2) if func_sub in parts[i])
    cur, out, fresh = None, [], True
    for ln in body.splitlines():
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            if fresh:  # the first annotation after an instruction is the innermost
                cur = (m.group(1).split("/")[-1], int(m.group(2)))
                fresh = False
            continue
        m2 = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m2:
            out.append((cur, m2.group(2)))
            fresh = True
    return out


def main(report, kernel, cubin_stem, func_sub, top=40):
    h, data = ncu_rows(report, kernel)
    ie = h.index("Instructions Executed")
    ws = h.index("Warp Stall Sampling (All Samples)")
    sass = sass_lines(cubin_stem, func_sub)

    def op(s):
        return s.split()[0] if s.split() else ""

    a = [op(x[1]) for x in data]
    b = [op(s[1]) for s in sass]
    best = max(((sum(1 for i in range(0, len(b), 5) if 0 <= i + o < len(a) and a[i + o] == b[i]),
                 o) for o in range(-64, 65)))
    off = best[1]
    agg = defaultdict(lambda: [0.0, 0.0])
    tot = sum(float(x[ie] or 0) for x in data)
    st = sum(float(x[ws] or 0) for x in data)
    for i, (loc, _) in enumerate(sass):
        j = i + off
        if loc and 0 <= j < len(data):
            agg[loc][0] += float(data[j][ie] or 0)
            agg[loc][1] += float(data[j][ws] or 0)
    src = {}
    for f in os.listdir(CSRC):
        if f.endswith((".cu", ".cuh")):
            src[f] = open(os.path.join(CSRC, f)).read().splitlines()
    print(f"alignment {best[0]}/{len(b) // 5} at offset {off}; total inst {tot:.3e}")
    for (f, ln), (v, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        code = src[f][ln - 1].strip()[:72] if f in src and ln <= len(src[f]) else ""
        print(f"{100 * v / tot:5.1f}% inst {100 * s / st:5.1f}% stall  {f}:{ln:<4d} {code}")


if __name__ == "__main__":
    main(*sys.argv[1:5], top=int(sys.argv[5]) if len(sys.argv) > 5 else 40)
