#!/usr/bin/env python
"""Break down the end-to-end render_pass cost (launch+sync, frame download)."""
import os
import sys
import time

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2405_06997_b200 import scene as S, svo, wavefront  # noqa: E402

sc = S.load_scene(os.path.join(REPO, "scenes", "cornell.scene"))
c = sc.camera
sc.camera = S.Camera(c.position, c.target, c.up, c.vfov_deg, 1920, 1080)
tree = svo.build_from_scene(sc, 1024)
pt = wavefront.GuidingConfig(l_min=5, max_depth=4, guided_depths=0)
g = wavefront.GuidingConfig(l_min=5, max_depth=4, guided_depths=4)
wavefront.render_pass(sc, tree, pt, [0])
wavefront.render_pass(sc, tree, g, [1])
r = wavefront._RUNNERS[next(iter(wavefront._RUNNERS))]
K = 10


def timeit(label, fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(K):
        fn(k)
    torch.cuda.synchronize()
    print(f"{label:40s} {1e3 * (time.perf_counter() - t0) / K:8.3f} ms")


timeit("launch (no stats)", lambda k: r.launch(2 + k, want_stats=False))
timeit("launch + stats sync", lambda k: r.launch(2 + k, want_stats=True))
timeit("frame .cpu().numpy()", lambda k: r.frame.cpu().numpy())
pin = torch.empty(r.frame.shape, dtype=r.frame.dtype, pin_memory=True)
timeit("pinned copy_ + sync", lambda k: (pin.copy_(r.frame, non_blocking=True),
                                          torch.cuda.current_stream().synchronize()))
timeit("pinned copy + numpy copy", lambda k: (pin.copy_(r.frame, non_blocking=True),
                                               torch.cuda.current_stream().synchronize(),
                                               pin.numpy().copy()))
timeit("render_pass (public API)", lambda k: wavefront.render_pass(sc, tree, g, [20 + k]))
