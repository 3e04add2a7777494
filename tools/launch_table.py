#!/usr/bin/env python
"""Per-kernel totals from an `ncu --metrics gpu__time_duration.sum[,dram__bytes_*] --csv`
launch list (optionally only launches [first, last) by ID).
    python tools/launch_table.py launches.csv [first last]"""
import collections
import csv
import sys


def main(path, first=None, last=None):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[h]
    ix = {k: i for i, k in enumerate(hdr)}
    per = collections.OrderedDict()
    for r in rows[h + 1:]:
        if len(r) < len(hdr):
            continue
        i = int(r[ix["ID"]])
        if first is not None and not (first <= i < last):
            continue
        d = per.setdefault(i, {"name": r[ix["Kernel Name"]]})
        unit = r[ix["Metric Unit"]]
        v = float(r[ix["Metric Value"]].replace(",", ""))
        scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0,
                 "ms": 1.0, "second": 1e3, "byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3,
                 "Gbyte": 1.0}.get(unit.strip(), 1.0)
        d[r[ix["Metric Name"]]] = v * scale
    agg = collections.OrderedDict()
    for d in per.values():
        name = d["name"].split("(")[0].replace("void ", "")
        a = agg.setdefault(name, [0, 0.0, 0.0, 0.0])
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0.0)
        a[2] += d.get("dram__bytes_read.sum", 0.0)
        a[3] += d.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    print(f"{len(per)} launches, {tot:.3f} ms\n\n| kernel | launches | ms | share | DRAM R GB | DRAM W GB |\n|---|---|---|---|---|---|")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {a[0]} | {a[1]:.3f} | {100 * a[1] / tot:.1f}% | {a[2]:.2f} | {a[3]:.2f} |")


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0], *(int(x) for x in a[1:3])) if len(a) >= 3 else main(a[0])
