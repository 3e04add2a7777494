#!/usr/bin/env python
"""Full-size parity (BASELINE configs[1] / C2, or C3): one PT-first pass and
one guided pass at 1920x1080 on the device and on the CPU oracle (test
infrastructure: the checker only), from the same SVO state.  Reports the
Alg. 2 bin counts per depth, the identical-path fraction (same emitter
depth, every record within 1e-5 x diagonal), the radiance agreement on
identical paths, the SVO deposit weights after PT-first (bitwise) and the
frame means.

    python tools/parity_full.py [--scene c2|c3] [--out profiles/x.jsonl]
"""

import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

SCENES = {"c2": ("cornell.scene", 1024), "c3": ("c3_two_rooms.scene", 2048)}


def identical(st_pos, st_emit, o_pos, o_emit, diag):
    same = st_emit == o_emit
    return same & (np.abs(st_pos - o_pos).max(axis=(1, 2)) <= 1e-5 * diag)


def rel(a, b):
    return (np.abs(a - b) / np.maximum(np.abs(b), 1e-12)).max(axis=1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scene", default="c2", choices=list(SCENES))
    ap.add_argument("--width", type=int, default=1920)
    ap.add_argument("--height", type=int, default=1080)
    ap.add_argument("--product", action="store_true", help="product guiding in the guided pass")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    from oracle import render as OR
    from paper_2405_06997_b200 import scene as S, svo, wavefront

    fname, res = SCENES[a.scene]
    sc = S.load_scene(os.path.join(REPO, "scenes", fname))
    cam = sc.camera
    sc.camera = S.Camera(cam.position, cam.target, cam.up, cam.vfov_deg, a.width, a.height)
    depth = res.bit_length() - 1
    base = dict(max_depth=4, field_res=128, l_min=min(5, depth - 1), c_ray=512, seed=0)
    t0 = time.perf_counter()
    tree = svo.build_from_scene(sc, res, seed=0)
    osc = OR.Scene(sc)
    osvo = OR.Svo.from_scene(sc, res, 0)
    t_build = time.perf_counter() - t0
    out = {"bench": "parity_full", "scene": a.scene, "product": a.product,
           "image": [a.width, a.height],
           "svo_resolution": res, "oracle_build_s": t_build}
    for tag, sample, g in (("pt_first", 0, 0), ("guided", 1, 4)):
        kw = dict(base, guided_depths=g, product=bool(a.product and g))
        cfg = wavefront.GuidingConfig(**kw)
        frame, st = wavefront.render_pass(sc, tree, cfg, [sample])
        state = wavefront._RUNNERS[next(iter(wavefront._RUNNERS))].state
        t0 = time.perf_counter()
        ostats = {}
        oframe, ost = OR.render_pass(osc, osvo, dict(kw), sample, ostats)
        t_oracle = time.perf_counter() - t0
        ident = identical(state.rec_pos, state.emit_depth, ost["rec_pos"], ost["emit_depth"],
                          sc.diagonal)
        r = rel(state.radiance, ost["radiance"])[ident]
        row = {"device_bins_per_depth": [int(x) for x in st.bins_per_depth],
               "oracle_bins_per_depth": [int(x) for x in ostats.get("bins", [])],
               "identical_paths": float(ident.mean()),
               "radiance_within_1e-4_on_identical": float(np.mean(r <= 1e-4)),
               "frame_mean_device": float(frame.mean()), "frame_mean_oracle": float(oframe.mean()),
               "oracle_pass_s": t_oracle}
        if g == 0:
            row["svo_weight_a_bitwise"] = bool(np.array_equal(tree.weight_a, osvo.weight_a))
            row["svo_weight_b_bitwise"] = bool(np.array_equal(tree.weight_b, osvo.weight_b))
            row["svo_sum_a_max_rel"] = float(np.max(np.abs(tree.sum_a - osvo.sum_a) /
                                                    np.maximum(np.abs(osvo.sum_a), 1e-300)))
        out[tag] = row
        # continue from the oracle's exitance state so the guided pass starts
        # from identical SVO contents
        for k in ("sum_a", "sum_b", "weight_a", "weight_b"):
            setattr(tree, k, getattr(osvo, k))
        tree.propagate_up()
        print(tag, json.dumps(row), flush=True)
    line = json.dumps(out)
    print(line)
    if a.out:
        with open(a.out, "a") as fh:
            fh.write(line + "\n")


if __name__ == "__main__":
    main()
