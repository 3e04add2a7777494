#!/usr/bin/env python
"""Field-kernel phase shares (cycles of each CTA's thread 0 between the phase
marks of k_fields, summed over bins) for guided C2 passes, from a library
built with -DWFPG_FIELD_PHASES:
    tools/field_phases.py --build /tmp/phases.so   (cross-compiles the variant)
    WFPG_LIB=/tmp/phases.so python tools/field_phases.py [--scene c2|c3]"""
import argparse
import ctypes
import os
import shutil
import subprocess
import sys
import tempfile

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
PHASES = ["bin start barrier", "cone trace (+ next setup)", "blur", "floor + value stores",
          "row / block sums, marginal + prefix sums", "marginal / prefix-sum stores"]


def build(out):
    tmp = tempfile.mkdtemp()
    src = os.path.join(tmp, "paper_2405_06997_b200", "csrc")
    shutil.copytree(os.path.join(REPO, "paper_2405_06997_b200", "csrc"), src,
                    ignore=shutil.ignore_patterns("build"))
    os.makedirs(os.path.join(tmp, "include"), exist_ok=True)
    shutil.copy(os.path.join(REPO, "include", "wfpg_b200.h"), os.path.join(tmp, "include"))
    flags = ("-O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a "
             "-Xcompiler -fPIC,-O3 --expt-relaxed-constexpr -DWFPG_FIELD_PHASES")
    subprocess.run(["make", "-s", "-j16", "-C", src,
                    f"OUT={os.path.abspath(out)}", f"NVFLAGS={flags}"], check=True)
    print("built", out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--build", default=None)
    ap.add_argument("--scene", default="c2")
    ap.add_argument("--passes", type=int, default=3)
    a = ap.parse_args()
    if a.build:
        build(a.build)
        return
    import numpy as np
    from paper_2405_06997_b200 import _lib, scene as S, svo, wavefront
    name = {"c2": "cornell.scene", "c3": "c3_two_rooms.scene"}[a.scene]
    sc = S.load_scene(os.path.join(REPO, "scenes", name))
    cam = sc.camera
    sc.camera = S.Camera(cam.position, cam.target, cam.up, cam.vfov_deg, 1920, 1080)
    tree = svo.build_from_scene(sc, 1024 if a.scene == "c2" else 2048, seed=0)
    cfg0 = wavefront.GuidingConfig(max_depth=4, guided_depths=0, field_res=128, l_min=5,
                                   c_ray=512, seed=0)
    wavefront.render_pass(sc, tree, cfg0, [0])
    cfg = wavefront.GuidingConfig(max_depth=4, guided_depths=4, field_res=128, l_min=5,
                                  c_ray=512, seed=0)
    fn = _lib.load().wfpg_field_phases
    buf = (ctypes.c_ulonglong * 40)()
    wavefront.render_pass(sc, tree, cfg, [1])
    fn(buf, 1)
    for s in range(a.passes):
        wavefront.render_pass(sc, tree, cfg, [2 + s])
    fn(buf, 0)
    v = np.array(list(buf), dtype=np.float64).reshape(5, 8)[:, :6]
    sizes = [8, 16, 32, 64, 128]
    print("| phase | " + " | ".join(f"N={n}" for n in sizes) + " |\n|---|" + "---|" * 5)
    for k, name in enumerate(PHASES):
        print(f"| {name} | " + " | ".join(
            f"{100 * v[r, k] / max(v[r].sum(), 1):.1f}%" for r in range(5)) + " |")
    print("| total Mcycles (thread 0 of every CTA) | " + " | ".join(
        f"{v[r].sum() / 1e6:.1f}" for r in range(5)) + " |")


if __name__ == "__main__":
    main()
