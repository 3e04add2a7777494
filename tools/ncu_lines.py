#!/usr/bin/env python
"""Top source lines by warp-stall samples / executed instructions from an
`ncu --page source --csv --print-source cuda,sass` export.
    python tools/ncu_lines.py export.csv [top]"""
import collections
import csv
import sys


def main(path, top=40):
    per, ins, text = collections.Counter(), collections.Counter(), {}
    f = None
    for r in csv.reader(open(path)):
        if r and r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if len(r) < 8 or not r[0].isdigit():
            continue
        key = (f, int(r[0]))
        try:
            per[key] += int(r[4])
            ins[key] += int(r[7])
        except ValueError:
            continue
        text[key] = r[1].strip()[:90]
    ts, ti = sum(per.values()), sum(ins.values())
    print("| file:line | samples | instructions | source |\n|---|---|---|---|")
    for k, v in per.most_common(top):
        print(f"| {k[0]}:{k[1]} | {100 * v / ts:.1f}% | {100 * ins[k] / ti:.1f}% | `{text[k]}` |")
    byfile = collections.Counter()
    for k, v in per.items():
        byfile[k[0]] += v
    print("\nby file:", {k: f"{100 * v / ts:.1f}%" for k, v in byfile.most_common()})


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
