#!/usr/bin/env python
"""Write profiles/round2.md from the round-2 measurement files copied from
gpurun_out/round/ (tools/round_measure.sh) into profiles/round2_*."""

import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(REPO, "profiles")


def J(name):
    path = os.path.join(P, f"round2_bench_{name}.json")
    lines = [ln for ln in open(path) if ln.startswith("{")]
    return json.loads(lines[-1])


def launches(name, rows=None):
    out = subprocess.run([sys.executable, os.path.join(REPO, "tools", "ncu_summary.py"),
                          "--launches", os.path.join("profiles", name)], cwd=REPO,
                         capture_output=True, text=True, check=True).stdout.strip()
    return "\n".join(out.splitlines()[:rows]) if rows else out


def main():
    c2, c3, k4, pr, ts, rf = (J(n) for n in ("c2", "c3", "4k", "prod", "tess", "reference_c2"))
    M = lambda d: d["value"] / 1e6  # noqa: E731
    r = c2["roofline"]
    cb = c2["cpu_baseline"]
    e2e_ratio = c2["e2e"]["value"] / rf["value"]
    ncu = subprocess.run([sys.executable, os.path.join(REPO, "tools", "ncu_raw_summary.py"),
                          "f128=" + os.path.join(P, "round2_ncu_f128_raw.csv")],
                         capture_output=True, text=True).stdout
    shade = subprocess.run([sys.executable, os.path.join(REPO, "tools", "ncu_raw_summary.py"),
                            "shade=" + os.path.join(P, "round2_ncu_shade_raw.csv")],
                           capture_output=True, text=True).stdout
    import csv as _csv
    _rows = list(_csv.reader(open(os.path.join(P, "round2_ncu_shade_raw.csv"))))
    _h = next(i for i, r in enumerate(_rows) if r and r[0] == "ID")
    _d, _u = dict(zip(_rows[_h], _rows[_h + 2])), dict(zip(_rows[_h], _rows[_h + 1]))
    _sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    shade_r = float(_d["dram__bytes_read.sum"].replace(",", "")) * _sc[_u["dram__bytes_read.sum"]] / 2073600
    shade_w = float(_d["dram__bytes_write.sum"].replace(",", "")) * _sc[_u["dram__bytes_write.sum"]] / 2073600
    lines = subprocess.run([sys.executable, os.path.join(REPO, "tools", "ncu_lines.py"),
                            os.path.join(P, "round2_ncu_f128_source.csv"), "25"],
                           capture_output=True, text=True).stdout
    body = f"""# Round 2 profiles (1x B200)

All numbers: `tools/round_measure.sh` on one B200 (files `profiles/round2_*`).

## Bench lines

* **C2** (`python bench.py`, round2_bench_c2.json): Cornell 1920x1080, SVO R=1024 (depth 10), D=G=4, N0=128, plain guiding — **{M(c2):.1f} M path samples/s** ({c2['ms_per_step']:.2f} ms per guided pass: CUDA-graph replays, two runners on two streams with pass i+1's start overlapping pass i's end); e2e through `wavefront.FramePipeline` (every frame in pinned host memory) **{c2['e2e']['value'] / 1e6:.1f} M/s**.  Depth-1 field kernel {r['launch_ms']:.2f} ms = {r['gcones_per_s']:.1f} G cones/s, {r['achieved'] / 1e3:.2f} TB/s algorithmic (78 B/cone) = **{r['frac']:.3f}** of the measured {r['peak']:.1f} GB/s; fields are {100 * r['field_share_of_step']:.0f}% of the step.  SM clock {c2['clocks']['sm_mhz']:.0f} MHz, reasons {c2['clocks']['reasons']}.
* **Reference arm** (`python bench.py --impl reference`, round2_bench_reference_c2.json): the CPU oracle renders every warm-up and timed step as a FULL guided pass ({rf['cpu_baseline']['cores']} host threads, no CUDA, no product library mapped): **{rf['value'] / 1e6:.3f} M path samples/s** ({rf['ms_per_step'] / 1e3:.2f} s per pass) → e2e ratio **{e2e_ratio:.0f}x**.  The b200 arm's `cpu_baseline` (one full oracle pass continuing the device run's SVO state): {cb['value'] / 1e6:.3f} M/s.
* **C3** (`--scene c3`, round2_bench_c3.json): occluded-light two-room interior, SVO R=2048 — **{M(c3):.1f} M/s** ({c3['ms_per_step']:.2f} ms), e2e {c3['e2e']['value'] / 1e6:.1f} M/s.
* **Product guiding** (`--product`): **{M(pr):.1f} M/s** ({pr['ms_per_step']:.2f} ms), {100 * (1 - pr['value'] / c2['value']):.0f}% below plain (round 1: 19%).
* **4K on one GPU** (`--width 3840 --height 2160`): {M(k4):.1f} M/s ({k4['ms_per_step']:.1f} ms per pass).
* **BVH paths** (`--scene tess`, 2,304 triangles): {M(ts):.1f} M/s ({ts['ms_per_step']:.1f} ms); field tracer {ts["roofline"]["gcones_per_s"]:.1f} G cones/s (warp-cooperative packet walk, shared-memory stacks).

## Dominant kernel: `k_fields<128, plain>` (depth-1 fields), ncu --set full

{ncu}
Top source lines by warp-stall samples (`tools/ncu_lines.py`):

{lines}
## `k_shade<brute, plain>` (first guided depth-1 launch), ncu --set full

{shade}
Per live path at depth 1 (2.07 M paths): {shade_r:.0f} B read + {shade_w:.0f} B written from DRAM against SURVEY §8(d)'s 172 B algorithmic — the rest is the guide-table probes of the samplers (1.26 GB of depth-1 tables, far beyond L2; ~10 dependent probes per guided path).  Round 1: 747 MB read / 219 MB written for the same launch; the depth-major path records (full-sector record stores) removed most of the difference.

## C5 microbenchmark

`profiles/round2_c5.md` (SVO build + cone trace, 1 M – 64 M points, depth 8 – 12).

## Launch list (C2)

`ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e` (round2_launches_c2.csv; C3 round2_launches_c3.csv).  ncu serialises kernels with cold caches: compare shares, not absolutes.

{launches("round2_launches_c2.csv")}

C3 (top rows):

{launches("round2_launches_c3.csv", 14)}
"""
    extra = os.path.join(P, "round2_notes.md")
    if os.path.exists(extra):
        body += "\n" + open(extra).read()
    open(os.path.join(P, "round2.md"), "w").write(body)
    t = json.load(open(os.path.join(P, "traffic.json")))
    raw = subprocess.run([sys.executable, "-c", f"""
import csv
rows=list(csv.reader(open({os.path.join(P, 'round2_ncu_f128_raw.csv')!r})))
h=next(i for i,r in enumerate(rows) if r and r[0]=='ID')
d=dict(zip(rows[h],rows[h+2])); u=dict(zip(rows[h],rows[h+1]))
def b(k):
    v=float(d[k].replace(',','')); s={{'byte':1,'Kbyte':1e3,'Mbyte':1e6,'Gbyte':1e9}}[u[k]]
    return int(v*s)
print(b('dram__bytes_read.sum'), b('dram__bytes_write.sum'))
"""], capture_output=True, text=True).stdout.split()
    if len(raw) == 2:
        key = "c2:1920x1080:R1024:D4:N128"
        t[key].update({"dram_read_bytes": int(raw[0]), "dram_write_bytes": int(raw[1]),
                       "report": "profiles/round2.md (round2_ncu_f128_raw.csv)"})
        json.dump(t, open(os.path.join(P, "traffic.json"), "w"), indent=1)
    print("wrote profiles/round2.md")


if __name__ == "__main__":
    main()
