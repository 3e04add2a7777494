#!/usr/bin/env python
"""Warp-stall reasons and stall samples / executed instructions of the
field kernel grouped by source region, from an `ncu --set full
--import-source on` report (used for profiles/round1_ncu_fields128_c2.md).

    python tools/ncu_regions.py gpurun_out/x.ncu-rep
"""

import collections
import csv
import io
import re
import subprocess
import sys

CSRC = "paper_2405_06997_b200/csrc/"


def _page(rep, what):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", what],
                         capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def _line_of(path, pattern):
    for k, ln in enumerate(open(CSRC + path), 1):
        if re.search(pattern, ln):
            return k
    raise ValueError(pattern)


def regions():
    """(file, first line, last line, region) from the current sources."""
    f = "fields.cu"
    g = "geometry.cuh"
    c = "common.cuh"
    return [
        (f, _line_of(f, r"void blur_rows\("), _line_of(f, r"^#ifdef WFPG_FIELD_PHASES") - 1,
         "blur (fold-aware separable, numpy tap order)"),
        (f, _line_of(f, r"3\. epsilon floor"), 10 ** 6,
         "epsilon floor, row sums, marginal, prefix sums, table stores"),
        (f, _line_of(f, r"auto setup = "), _line_of(f, r"int64_t b = blockIdx.x;"),
         "per-bin setup (uv tables, triangle records)"),
        (f, 0, 10 ** 6, "trace loop control, tile / bin scheduling, barriers"),
        (g, 0, _line_of(g, r"double warp_sum_d") - 1, "per-bin setup (uv tables, triangle records)"),
        (g, 0, _line_of(g, r"while \(m\) \{") - 1, "warp tile cone bound + triangle cull"),
        (g, 0, 10 ** 6, "candidate Moeller-Trumbore tests"),
        ("svo_query.cuh", 0, 10 ** 6, "SVO query at the hit (quantise, level, descent, side mean)"),
        (c, _line_of(c, r"^struct SvoView"), 10 ** 6,
         "SVO query at the hit (quantise, level, descent, side mean)"),
        (c, 0, 10 ** 6, "octahedral cell map (one division, polynomial sin/cos)"),
        ("shade.cuh", 0, 10 ** 6, "epsilon floor, row sums, marginal, prefix sums, table stores"),
    ]


def main(rep):
    rows = _page(rep, "sass")
    hdr = rows[1]
    idx = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    tot = collections.Counter()
    for r in rows[2:]:
        for i in idx:
            try:
                tot[hdr[i]] += int(r[i])
            except (ValueError, IndexError):
                pass
    s = sum(tot.values())
    print("Warp-state samples (all samples, `--page source`), top reasons:\n")
    print("| reason | share |\n|---|---|")
    for k, v in tot.most_common(9):
        print(f"| {k} | {100 * v / s:.1f}% |")
    table = regions()
    per, ins = collections.Counter(), collections.Counter()
    f = None
    for r in _page(rep, "cuda,sass"):
        if r and r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if len(r) < 8 or r[0] in ("Line No", "Function Name", ""):
            continue
        try:
            line, sm, ii = int(r[0]), int(r[4]), int(r[7])
        except ValueError:
            continue
        name = "intrinsics (atomics, shuffles)"
        for fn, lo, hi, reg in table:
            if fn == f and lo <= line <= hi:
                name = reg
                break
        per[name] += sm
        ins[name] += ii
    ts, ti = sum(per.values()), sum(ins.values())
    print("\nStall samples and executed warp instructions grouped by source region "
          "(`--page source --print-source cuda,sass`):\n")
    print("| region | samples | instructions |\n|---|---|---|")
    for k, v in per.most_common():
        print(f"| {k} | {100 * v / ts:.1f}% | {100 * ins[k] / ti:.1f}% |")


if __name__ == "__main__":
    main(sys.argv[1])
