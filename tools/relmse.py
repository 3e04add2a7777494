#!/usr/bin/env python
"""Equal-spp and equal-time relMSE of guided vs unguided rendering on the
B200 (BASELINE metric "relMSE at equal time").

1. Reference: --ref-spp samples of unguided path tracing (independent seed).
2. Guided (pt-first, Eq. 7 "pt-first" heuristic, the CLI's default) and
   unguided PT, each accumulated on the device through cli.render's loop;
   at every power-of-two spp the running image is resolved and compared with
   the reference (relMSE = mean((x - r)^2 / (r^2 + 1e-2)), plus the
   tone-mapped MSE of accumulation.mse).  Device time (CUDA events, resolves
   excluded) is accumulated per curve; the guided time includes its SVO
   build.
3. Equal time: PT keeps rendering until it has used the guided run's total
   time; the relMSE of both at that time is the headline pair.

Prints one JSON line per scene (and appends it to --out).

    python tools/relmse.py --scene c2 --spp 64 --ref-spp 16384
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


def curve(scene, svo, conf, max_spp, checkpoints, ref, time_budget_ms=None, extra_ms=0.0):
    """Accumulate passes; returns [(spp, device ms, relMSE, mse)] at checkpoints
    (and at the time budget when given)."""
    import torch

    from paper_2405_06997_b200 import accumulation as A, cli, wavefront

    cam = scene.camera
    guided = conf.guided_depths if conf.mode != "pt" else 0
    pt_first = conf.heuristic == "pt-first" and conf.mode != "pt"
    runners = {}

    def runner(g):
        if g not in runners:
            c = cli._pass_cfg(conf, g)
            if svo is not None:
                c.l_min = conf.effective_lmin(svo.depth)
            runners[g] = wavefront.PassRunner(scene, svo, c, 1)
        return runners[g]

    buf = A.AccumulationBuffer(cam.height, cam.width, conf.heuristic)
    out = []
    ms = extra_ms
    cur = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(cur)
    i = 0
    while True:
        i += 1
        g = 0 if (pt_first and i == 1) else guided
        r = runner(g)
        r.launch(i - 1, want_stats=False)
        buf.add_sample(r.frame, i)
        at_cp = i in checkpoints
        over = time_budget_ms is not None and i % 8 == 0
        if at_cp or over or i == max_spp:
            e1.record(cur)
            torch.cuda.synchronize()
            ms += e0.elapsed_time(e1)
            if at_cp or i == max_spp or (time_budget_ms is not None and ms >= time_budget_ms):
                if ref is None:
                    out.append((i, ms, None, None))
                else:
                    f = buf.resolve()
                    out.append((i, ms, A.rel_mse(f, ref), A.mse(f, ref)))
            if i >= max_spp or (time_budget_ms is not None and ms >= time_budget_ms):
                break
            e0.record(cur)
    return out, buf


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scene", default="c2", choices=list(SCENES))
    ap.add_argument("--width", type=int, default=1920)
    ap.add_argument("--height", type=int, default=1080)
    ap.add_argument("--svo-res", type=int, default=None)
    ap.add_argument("--depth", type=int, default=5)
    ap.add_argument("--spp", type=int, default=64)
    ap.add_argument("--ref-spp", type=int, default=16384)
    ap.add_argument("--mode", default="wfpg", choices=["wfpg", "wfpg-product"])
    ap.add_argument("--out", default=None)
    ap.add_argument("--save-ref", default=None, help="write the reference frame (PFM)")
    args = ap.parse_args()

    import torch

    from paper_2405_06997_b200 import cli, imageio, scene as S, svo as svo_mod

    name, res = SCENES[args.scene]
    res = args.svo_res or res
    sc = S.load_scene(os.path.join(REPO, "scenes", name))
    cam = sc.camera
    sc.camera = S.Camera(cam.position, cam.target, cam.up, cam.vfov_deg, args.width, args.height)
    path = os.path.join(REPO, "scenes", name)
    t0 = time.perf_counter()
    # reference: unguided, independent seed, only the final image
    ref_conf = cli.RunConfig(path, mode="pt", spp=args.ref_spp, depth=args.depth, seed=1_000_003)
    ref_pts, ref_buf = curve(sc, None, ref_conf, args.ref_spp, set(), None)
    ref_ms = ref_pts[-1][1]
    ref = ref_buf.resolve()
    del ref_buf
    if args.save_ref:
        imageio.write_pfm(args.save_ref, ref)
    cps = {1 << k for k in range(0, 20)}
    # guided (SVO build timed with events and charged to the guided curve)
    g_conf = cli.RunConfig(path, mode=args.mode, spp=args.spp, depth=args.depth, svo_res=res,
                           seed=7)
    cur = torch.cuda.current_stream()
    b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    b0.record(cur)
    tree = svo_mod.build_from_scene(sc, res, seed=g_conf.seed)
    b1.record(cur)
    torch.cuda.synchronize()
    build_ms = b0.elapsed_time(b1)
    g_pts, _ = curve(sc, tree, g_conf, args.spp, cps, ref, extra_ms=build_ms)
    g_ms = g_pts[-1][1]
    # unguided at equal spp, continuing to equal time
    p_conf = cli.RunConfig(path, mode="pt", spp=1 << 30, depth=args.depth, seed=7)
    p_pts, _ = curve(sc, None, p_conf, 1 << 30, cps, ref, time_budget_ms=g_ms)
    eq_spp = [p for p in p_pts if p[0] == args.spp]
    line = {
        "bench": "relmse", "scene": args.scene, "image": [args.width, args.height],
        "svo_res": res, "max_depth": args.depth, "mode": args.mode,
        "reference": {"spp": args.ref_spp, "device_ms": ref_ms, "seed": 1_000_003},
        "svo_build_ms": build_ms,
        "guided": [{"spp": s, "ms": m, "rel_mse": r, "mse": e} for s, m, r, e in g_pts],
        "pt": [{"spp": s, "ms": m, "rel_mse": r, "mse": e} for s, m, r, e in p_pts],
        "equal_spp": {"spp": args.spp, "guided_rel_mse": g_pts[-1][2],
                      "pt_rel_mse": eq_spp[0][2] if eq_spp else None},
        "equal_time": {"ms": g_ms, "guided_rel_mse": g_pts[-1][2], "pt_spp": p_pts[-1][0],
                       "pt_rel_mse": p_pts[-1][2]},
        "wall_s": time.perf_counter() - t0,
    }
    print(json.dumps(line), flush=True)
    if args.out:
        with open(args.out, "a") as fh:
            fh.write(json.dumps(line) + "\n")


if __name__ == "__main__":
    main()
