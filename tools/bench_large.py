#!/usr/bin/env python
"""Large-scene run: the Cornell box with every triangle
split into 4^levels (levels 7: 589,824 triangles), generated under /tmp, so
the scene takes the device-built linear BVH; a PT-first pass, then guided
1080p passes (CUDA events over 5 graph replays).

    python tools/bench_large.py [--levels 7]
"""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--levels", type=int, default=7)
    ap.add_argument("--passes", type=int, default=5)
    a = ap.parse_args()
    import torch

    from paper_2405_06997_b200 import scene as S, scenegen, svo, wavefront

    path = scenegen.write_tessellated_cornell(f"/tmp/wfpg_large_{a.levels}", levels=a.levels)
    sc = S.load_scene(path)
    cam = sc.camera
    sc.camera = S.Camera(cam.position, cam.target, cam.up, cam.vfov_deg, 1920, 1080)
    torch.cuda.init()
    torch.zeros(1, device="cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sc.abi()
    torch.cuda.synchronize()
    upload_bvh_s = time.perf_counter() - t0
    tree = svo.build_from_scene(sc, 1024, seed=0)
    kw = dict(max_depth=4, field_res=128, l_min=5, c_ray=512, seed=0)
    pt = wavefront.PassRunner(sc, tree, wavefront.GuidingConfig(guided_depths=0, **kw))
    gr = wavefront.PassRunner(sc, tree, wavefront.GuidingConfig(guided_depths=4, **kw))
    pt.launch(0)
    for s in range(1, 4):
        gr.launch(s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in range(4, 4 + a.passes):
        gr.launch(s)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.passes
    print(json.dumps({"bench": "large_scene", "triangles": sc.triangle_count,
                      "device_bvh": sc.device_bvh, "upload_and_bvh_s": upload_bvh_s,
                      "guided_pass_ms": ms, "path_samples_per_s": 1920 * 1080 / ms * 1e3}))


if __name__ == "__main__":
    main()
