#!/usr/bin/env python
"""Rewrite the table of profiles/round2_c5.md from profiles/round2_c5.jsonl
(tools/bench_c5.py output), with round 1's build times beside it; the text
around the table is kept."""
import json
import os

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(REPO, "profiles")


def rows(name):
    return [json.loads(ln) for ln in open(os.path.join(P, name)) if ln.startswith("{")]


def main():
    r1 = {(d["n_points"], d["svo_depth"]): d["build_ms"] for d in rows("round1_c5.jsonl")}
    out = ["| N | depth | nodes | build ms (round 1) | build ms | Mpts/s | build frac | cone ms | "
           "G cones/s | cone frac | SVO bit-exact | cones within 1e-9 |",
           "|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for d in rows("round2_c5.jsonl"):
        n, dep = d["n_points"], d["svo_depth"]
        o = d.get("oracle") or {}
        old = r1.get((n, dep))
        out.append(
            f"| {n >> 20}M | {dep} | {d['svo_nodes']:,} | {old:.2f} | {d['build_ms']:.2f} | "
            f"{d['build_mpts_per_s']:.0f} | {d['build_roofline']['frac']:.3f} | {d['cone_ms']:.2f} | "
            f"{d['gcones_per_s']:.2f} | {d['cone_roofline']['frac']:.3f} | "
            f"{o.get('svo_bitexact', '-')} | {o.get('cones_within_1e-9', '-')} |"
            if old is not None else "")
    path = os.path.join(P, "round2_c5.md")
    lines = open(path).read().split("\n")
    i = next(k for k, ln in enumerate(lines) if ln.startswith("| N | depth"))
    j = i
    while j < len(lines) and lines[j].startswith("|"):
        j += 1
    lines[i:j] = [ln for ln in out if ln]
    open(path, "w").write("\n".join(lines))
    print("wrote", path)


if __name__ == "__main__":
    main()
