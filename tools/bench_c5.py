#!/usr/bin/env python
"""SVO build + cone-trace microbenchmark on synthetic path
vertices — N in {1M, 4M, 16M, 64M} points uniform by area on the Cornell
triangles, quantised at R = 2^d, d in {8..12}.

Points: counter RNG (seed 0, stream = point index), triangle through the
area CDF with u1 rescaled for the square-root barycentric warp (scene.py:
257-263 of the reference), normal = the triangle normal.  Build = quantise ->
Morton -> radix sort -> unique -> levels -> dual normals
(svo.build_from_points).  Cones: M = N, origin = point + ray_eps * normal,
direction uniform on the sphere from counters 2,3 of the point's stream,
omega = 4 pi / 128^2, against a non-trivial exitance state (leaf sums from
the same RNG, propagated).

Per (N, d) one JSON line: device build ms (CUDA events around the whole
build incl. its host sync for the level sizes), cone-trace ms and G cones/s,
both against the HBM roofline with SURVEY §8(d)'s algorithmic bytes (build:
48 B per input vertex + 41 B per node; cone: 5 d + 28 B); plus, at
N <= --check-n, parity against the CPU oracle (bit-exact SVO arrays; cones
within 1e-9 on a subsample) and the oracle's own build / cone-trace time on
the host cores.

    python tools/bench_c5.py [--n 1M,4M,16M,64M] [--depths 8,9,10,11,12]
"""

import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def parse_n(s):
    out = []
    for t in s.split(","):
        t = t.strip().upper()
        out.append(int(float(t[:-1]) * (1 << 20)) if t.endswith("M") else int(t))
    return out


def synth_points(sc, n, seed=0, chunk=1 << 22):
    """Host fp64 points (n,3), triangle ids (n,), cone dirs (n,3)."""
    from paper_2405_06997_b200 import core

    area = 0.5 * np.linalg.norm(np.cross(sc.e1, sc.e2), axis=1)
    cdf = np.cumsum(area) / area.sum()
    pts = np.empty((n, 3))
    tri = np.empty(n, dtype=np.int32)
    dirs = np.empty((n, 3))
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        key = core.stream_key(np.uint64(seed), np.arange(s, e, dtype=np.uint64))
        u1, u2 = core.u01_at(key, np.uint64(0)), core.u01_at(key, np.uint64(1))
        k = np.minimum(np.searchsorted(cdf, u1, side="right"), len(cdf) - 1)
        lo = np.where(k > 0, cdf[k - 1], 0.0)
        span = cdf[k] - lo
        b1 = np.where(span > 0, (u1 - lo) / np.where(span > 0, span, 1.0), 0.0)
        b1 = np.clip(b1, 0.0, 1.0 - 1e-12)
        su = np.sqrt(b1)
        a = 1.0 - su
        b = u2 * su
        pts[s:e] = (sc.v0[k] * (1.0 - a - b)[:, None] + sc.v1[k] * a[:, None]
                    + sc.v2[k] * b[:, None])
        tri[s:e] = k
        z = 1.0 - 2.0 * core.u01_at(key, np.uint64(2))
        phi = 2.0 * np.pi * core.u01_at(key, np.uint64(3))
        r = np.sqrt(np.maximum(0.0, 1.0 - z * z))
        dirs[s:e] = np.stack([r * np.cos(phi), r * np.sin(phi), z], axis=1)
    return pts, tri, dirs


def peak_gbs():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except (OSError, ValueError, KeyError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def exitance_state(tree, seed=0):
    """Leaf sums/weights from the counter RNG, propagated on the device."""
    from paper_2405_06997_b200 import _dev, _lib, core

    lo, hi = int(tree.level_off[tree.depth]), int(tree.level_off[tree.depth + 1])
    m = hi - lo
    key = core.stream_key(np.uint64(seed + 1), np.arange(m, dtype=np.uint64))
    for side, c0 in (("a", 0), ("b", 3)):
        s = np.zeros((tree.node_count, 3))
        w = np.zeros(tree.node_count)
        s[lo:hi] = np.stack([core.u01_at(key, np.uint64(c0 + j)) for j in range(3)], axis=1)
        w[lo:hi] = (core.u01_at(key, np.uint64(7 + c0)) < 0.7).astype(np.float64)
        tree.dev("sum_" + side).copy_(_dev.upload(s * w[:, None]))
        tree.dev("weight_" + side).copy_(_dev.upload(w))
    s = tree.abi()
    _lib.call("wfpg_svo_propagate", _lib.C.byref(s), _dev.stream())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", default="1M,4M,16M,64M")
    ap.add_argument("--depths", default="8,9,10,11,12")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--check-n", type=int, default=1 << 20,
                    help="oracle parity + CPU timing for N up to this")
    ap.add_argument("--cone-sample", type=int, default=1 << 16)
    ap.add_argument("--out", default=None, help="also append the lines to this file")
    args = ap.parse_args()

    import torch

    from paper_2405_06997_b200 import _dev, _lib, scene as S, svo

    sc = S.load_scene(os.path.join(REPO, "scenes", "cornell.scene"))
    cube_lo, side = svo.scene_cube(sc)
    omega = 4.0 * np.pi / 128 ** 2
    peak, peak_kind = peak_gbs()
    st = _dev.stream()
    lines = []
    for n in parse_n(args.n):
        t0 = time.perf_counter()
        pts, tri, dirs = synth_points(sc, n)
        gen_s = time.perf_counter() - t0
        d_pts = _dev.upload(pts)
        d_nrm = _dev.upload(sc.normals[tri])
        d_org = _dev.upload(pts + sc.ray_eps * sc.normals[tri])
        d_dir = _dev.upload(dirs)
        d_out = _dev.empty((n, 3), np.float64)
        for depth in [int(x) for x in args.depths.split(",")]:
            res = 1 << depth
            times = []
            for _ in range(args.reps + 1):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(torch.cuda.current_stream())
                tree = svo.build_from_points(d_pts, d_nrm, cube_lo, side, res, seed=0)
                e1.record(torch.cuda.current_stream())
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1))
            build_ms = float(np.median(times[1:]))
            nodes = tree.node_count
            exitance_state(tree)
            s = tree.abi()
            scab = sc.abi()
            ct = []
            for _ in range(args.reps + 1):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(torch.cuda.current_stream())
                _lib.call("wfpg_trace_cones", _lib.C.byref(scab), _lib.C.byref(s),
                          _lib.ptr(d_org), 3, _lib.ptr(d_dir), n, omega, _lib.ptr(d_out), st)
                e1.record(torch.cuda.current_stream())
                torch.cuda.synchronize()
                ct.append(e0.elapsed_time(e1))
            cone_ms = float(np.median(ct[1:]))
            b_bytes = 48 * n + 41 * nodes
            c_bytes = (5 * depth + 28) * n
            line = {"bench": "c5", "n_points": n, "svo_depth": depth, "svo_nodes": nodes,
                    "leaves": int(tree.level_off[depth + 1] - tree.level_off[depth]),
                    "build_ms": build_ms, "build_mpts_per_s": n / build_ms / 1e3,
                    "build_roofline": {"bound": "hbm", "achieved": b_bytes / build_ms / 1e6,
                                       "peak": peak, "unit": "GB/s",
                                       "frac": b_bytes / build_ms / 1e6 / peak,
                                       "bytes": b_bytes},
                    "cone_ms": cone_ms, "gcones_per_s": n / cone_ms / 1e6,
                    "cone_roofline": {"bound": "hbm", "achieved": c_bytes / cone_ms / 1e6,
                                      "peak": peak, "unit": "GB/s",
                                      "frac": c_bytes / cone_ms / 1e6 / peak, "bytes": c_bytes},
                    "peak_kind": peak_kind, "host_point_gen_s": gen_s}
            if n <= args.check_n:
                line.update(oracle_check(sc, tree, pts, tri, dirs, d_out, omega, depth,
                                         args.cone_sample))
            print(json.dumps(line), flush=True)
            lines.append(line)
            del tree
            torch.cuda.empty_cache()
        del d_pts, d_nrm, d_org, d_dir, d_out
        torch.cuda.empty_cache()
    if args.out:
        with open(args.out, "a") as fh:
            for ln in lines:
                fh.write(json.dumps(ln) + "\n")


def oracle_check(sc, tree, pts, tri, dirs, d_out, omega, depth, m):
    """Bit-exact SVO arrays and cone radiance vs the CPU oracle (test
    infrastructure, the checker only), plus the oracle's host timings."""
    from oracle import oracle as O
    from oracle import render as OR
    from paper_2405_06997_b200 import svo as _svo

    res = 1 << depth
    cube_lo, side = _svo.scene_cube(sc)
    scale = res / side
    q = ((pts - cube_lo) * scale)
    coords = np.clip(np.trunc(q), 0, res - 1).astype(np.int64)
    t0 = time.perf_counter()
    b = O.build_octree(coords, sc.normals[tri], res, 0)
    cpu_build = time.perf_counter() - t0
    same = all(np.array_equal(np.asarray(b[k]).astype(np.int64),
                              np.asarray(getattr(tree, k)).astype(np.int64))
               for k in ("level_off", "child_base", "child_mask", "parent"))
    same &= np.array_equal(b["codes"], tree.codes)
    same &= np.array_equal(np.asarray(b["normal"]).view(np.uint64), tree.normal.view(np.uint64))
    osvo = OR.Svo(b, cube_lo, side, res)
    for k in ("sum_a", "sum_b", "weight_a", "weight_b"):
        setattr(osvo, k, np.ascontiguousarray(getattr(tree, k)))
    osvo.propagate()
    rng = np.random.default_rng(0)
    idx = np.sort(rng.choice(len(pts), size=min(m, len(pts)), replace=False))
    org = pts[idx] + sc.ray_eps * sc.normals[tri[idx]]
    osc = OR.Scene(sc)
    t0 = time.perf_counter()
    ref = OR.trace_cones(osc, osvo, org, dirs[idx], omega)
    cpu_cone = time.perf_counter() - t0
    got = d_out.cpu().numpy()[idx]
    close = np.all(np.isclose(got, ref, rtol=1e-9, atol=1e-300), axis=1)
    return {"oracle": {"svo_bitexact": bool(same), "cones_within_1e-9": float(close.mean()),
                       "cone_sample": int(len(idx)),
                       "cpu_build_s": cpu_build, "cpu_build_mpts_per_s": len(pts) / cpu_build / 1e6,
                       "cpu_gcones_per_s": len(idx) / cpu_cone / 1e9,
                       "cpu_cores": os.cpu_count(), "kind": "port"}}


if __name__ == "__main__":
    main()
