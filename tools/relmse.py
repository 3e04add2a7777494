#!/usr/bin/env python
"""Equal-spp and equal-time relMSE of guided vs unguided rendering on the
B200 (BASELINE metric "relMSE at equal time").

1. Reference: --ref-spp samples of unguided path tracing (independent seed).
2. Costs: steady-state device time of one guided pass and one unguided pass
   (CUDA-graph replay, CUDA events, after eager + capture warm-up) and of the
   SVO build.
3. Guided (pt-first, Eq. 7 "pt-first" heuristic, the CLI's default) and
   unguided PT, each accumulated on the device; at every power-of-two spp
   the running image is compared with the reference (relMSE = mean((x - r)^2
   / (r^2 + 1e-2)), plus the tone-mapped MSE of accumulation.mse).
4. Equal time: PT renders as many samples as cost the guided run's time
   (build + spp x guided pass); the relMSE of both is the headline pair.

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

SCENES = {"c2": ("cornell.scene", 1024), "c3": ("c3_two_rooms.scene", 2048),
          "enclosed": ("cornell_enclosed.scene", 256)}


def _runners(scene, svo, conf, k=1):
    """Pass i (1-based) -> its PassRunner; every pass renders k samples per
    pixel (render_pass with a k-entry sample list: one set of fields per k
    samples, wavefront.py:198-215)."""
    from paper_2405_06997_b200 import cli, wavefront

    guided = conf.guided_depths if conf.mode != "pt" else 0
    pt_first = conf.heuristic == "pt-first" and conf.mode != "pt"
    runners = {}

    def runner(g):
        if g not in runners:
            c = cli._pass_cfg(conf, g)
            if svo is not None:
                c.l_min = conf.effective_lmin(svo.depth)
            runners[g] = wavefront.PassRunner(scene, svo, c, k, skip_unguided_bins=True)
        return runners[g]

    return lambda i: runner(0 if (pt_first and i == 1) else guided)


def pass_ms(scene, svo, conf, reps=10, k=1):
    """Steady-state device time of one pass (graph replay), CUDA events."""
    import torch

    get = _runners(scene, svo, conf, k)
    r = get(2)  # a guided pass (or the PT pass in pt mode)
    for j in range(3):  # eager, capture, replay
        r.launch((j + 2) * k, want_stats=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for j in range(reps):
        r.launch((j + 5) * k, want_stats=False)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def curve(scene, svo, conf, max_spp, checkpoints, ref, k=1):
    """Accumulate passes of k samples up to max_spp samples; [(spp, relMSE,
    mse)] at the checkpoints and at max_spp (the accumulated frame when ref
    is None)."""
    from paper_2405_06997_b200 import accumulation as A

    cam = scene.camera
    get = _runners(scene, svo, conf, k)
    buf = A.AccumulationBuffer(cam.height, cam.width, conf.heuristic)
    out = []
    for i in range(1, max_spp // k + 1):
        r = get(i)
        r.launch((i - 1) * k, want_stats=False)
        buf.add_sample(r.frame, i)
        spp = i * k
        if ref is not None and (spp in checkpoints or i == max_spp // k):
            f = buf.resolve()
            out.append((spp, A.rel_mse(f, ref), A.mse(f, ref)))
    return out, buf


def _bins_per_depth(scene, svo, conf, k):
    """Bins per depth of one more guided pass on a copy-free probe (stats)."""
    get = _runners(scene, svo, conf, k)
    r = get(2)
    r.launch(10_000 * k, want_stats=True)
    return r, r.pass_stats().bins_per_depth


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
    ap.add_argument("--save-ref", default=None, help="write the reference frame (.npy)")
    ap.add_argument("--ref-file", default=None,
                    help="reuse a reference frame written by --save-ref (same scene/size/depth)")
    ap.add_argument("--guided-depths", type=int, default=4)
    ap.add_argument("--seed", type=int, default=7, help="seed of the guided and PT runs")
    ap.add_argument("--field-res", type=int, default=128)
    ap.add_argument("--skip-pt", action="store_true", help="guided curve only")
    ap.add_argument("--lmin", type=int, default=5)
    ap.add_argument("--c-ray", type=int, default=512)
    ap.add_argument("--spp-per-pass", type=int, default=1,
                    help="samples per guided pass (one set of fields per pass)")
    args = ap.parse_args()

    import torch

    from paper_2405_06997_b200 import cli, scene as S, svo as svo_mod

    name, res = SCENES[args.scene]
    res = args.svo_res or res
    sc = S.load_scene(os.path.join(REPO, "scenes", name))
    cam = sc.camera
    sc.camera = S.Camera(cam.position, cam.target, cam.up, cam.vfov_deg, args.width, args.height)
    path = os.path.join(REPO, "scenes", name)
    t0 = time.perf_counter()
    # reference: unguided, independent seed, only the final image
    if args.ref_file and os.path.exists(args.ref_file):
        ref = np.load(args.ref_file)
    else:
        ref_conf = cli.RunConfig(path, mode="pt", spp=args.ref_spp, depth=args.depth,
                                 seed=1_000_003)
        _, ref_buf = curve(sc, None, ref_conf, args.ref_spp, set(), None)
        ref = ref_buf.resolve()
        del ref_buf
        if args.save_ref:
            np.save(args.save_ref, ref)
    cps = {1 << k for k in range(0, 20)}
    g_conf = cli.RunConfig(path, mode=args.mode, spp=args.spp, depth=args.depth, svo_res=res,
                           seed=args.seed, guided_depths=min(args.guided_depths, args.depth),
                           field_res=args.field_res, lmin=args.lmin, cray=args.c_ray)
    kpp = args.spp_per_pass
    p_conf = cli.RunConfig(path, mode="pt", spp=1 << 30, depth=args.depth, seed=args.seed)
    # steady-state costs: SVO build, guided pass (on a scratch SVO), PT pass
    cur = torch.cuda.current_stream()
    b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    svo_mod.build_from_scene(sc, res, seed=g_conf.seed)  # warm-up
    b0.record(cur)
    scratch = svo_mod.build_from_scene(sc, res, seed=g_conf.seed)
    b1.record(cur)
    torch.cuda.synchronize()
    build_ms = b0.elapsed_time(b1)
    g_ms = pass_ms(sc, scratch, g_conf, k=kpp) / kpp  # per sample
    p_ms = pass_ms(sc, None, p_conf)
    del scratch
    # quality: guided to spp; unguided to the spp that costs the same time
    tree = svo_mod.build_from_scene(sc, res, seed=g_conf.seed)
    g_pts, _ = curve(sc, tree, g_conf, args.spp, cps, ref, k=kpp)
    _, bins = _bins_per_depth(sc, tree, g_conf, kpp)
    budget = build_ms + args.spp * g_ms
    pt_spp = max(args.spp, int(budget / p_ms))
    p_pts = [(0, float("nan"), float("nan"))] if args.skip_pt else \
        curve(sc, None, p_conf, pt_spp, cps | {args.spp}, ref)[0]
    eq_spp = [p for p in p_pts if p[0] == args.spp]
    line = {
        "bench": "relmse", "scene": args.scene, "image": [args.width, args.height],
        "svo_res": res, "max_depth": args.depth, "mode": args.mode,
        "guided_depths": g_conf.guided_depths, "field_res": g_conf.field_res,
        "l_min": g_conf.effective_lmin(tree.depth), "c_ray": g_conf.cray,
        "spp_per_pass": kpp, "bins_per_depth": bins,
        "reference": {"spp": args.ref_spp, "seed": 1_000_003, "kind": "unguided PT"},
        "svo_build_ms": build_ms, "guided_pass_ms": g_ms, "pt_pass_ms": p_ms,
        "guided": [{"spp": s_, "ms": build_ms + s_ * g_ms, "rel_mse": r, "mse": e}
                   for s_, r, e in g_pts],
        "pt": [{"spp": s_, "ms": s_ * p_ms, "rel_mse": r, "mse": e} for s_, r, e in p_pts],
        "equal_spp": {"spp": args.spp, "guided_rel_mse": g_pts[-1][1],
                      "pt_rel_mse": eq_spp[0][1] if eq_spp else None},
        "equal_time": {"ms": budget, "guided_rel_mse": g_pts[-1][1], "pt_spp": p_pts[-1][0],
                       "pt_rel_mse": p_pts[-1][1]},
        "timing": "steady-state device pass times (CUDA-graph replay, CUDA events); "
                  "curves rendered separately, so image resolves cost nothing",
        "wall_s": time.perf_counter() - t0,
    }
    print(json.dumps(line), flush=True)
    if args.out:
        with open(args.out, "a") as fh:
            fh.write(json.dumps(line) + "\n")


if __name__ == "__main__":
    main()
