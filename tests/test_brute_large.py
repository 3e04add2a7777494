"""A brute-force scene near the 512-triangle limit (kMaxBruteTris): the
Cornell box with its white mesh midpoint-subdivided twice (30 x 16 + 6 = 486
triangles).  Every per-block triangle table then exceeds the 48 KB default
shared-memory window somewhere — the camera-ray records (144 B each, 70 KB),
the field kernel's records next to its N=128 field (about 200 KB) — so the
launches must opt in to the larger window.  A PT-first, a plain-guided and a
product-guided pass on the device against the CPU oracle on its own build,
path for path."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _write_scene(out_dir, src_dir):
    from paper_2405_06997_b200 import scenegen as G

    levels = {"white": 2, "red": 0, "green": 0, "light": 0}
    for mesh, lv in levels.items():
        tris = [t for tri in G._read_obj(os.path.join(src_dir, f"cornell_{mesh}.obj"))
                for t in G._subdivide(tri, lv)]
        G._write_obj(os.path.join(out_dir, f"big_{mesh}.obj"), tris)
    src = open(os.path.join(src_dir, "cornell.scene")).read()
    for mesh in levels:
        src = src.replace(f"cornell_{mesh}.obj", f"big_{mesh}.obj")
    path = os.path.join(out_dir, "big.scene")
    open(path, "w").write(src)
    return path


def test_brute_scene_at_the_triangle_limit(tmp_path, scene_path):
    from oracle import render as OR
    from paper_2405_06997_b200 import scene as S, svo, wavefront

    path = _write_scene(str(tmp_path), os.path.dirname(scene_path("cornell.scene")))
    sc = S.load_scene(path)
    assert sc.triangle_count == 486
    assert sc.abi().brute == 1  # still the shared-memory brute-force path
    cam = sc.camera
    sc.camera = S.Camera(cam.position, cam.target, cam.up, cam.vfov_deg, 64, 48)
    tree = svo.build_from_scene(sc, 128, seed=0)
    osvo = OR.Svo.from_scene(sc, 128, 0)
    assert np.array_equal(tree.normal.view(np.uint64), osvo.normal.view(np.uint64))
    osc = OR.Scene(sc)
    base = dict(max_depth=4, field_res=128, l_min=3, c_ray=64, seed=5)
    for sample, g, product in ((0, 0, False), (1, 4, False), (2, 4, True)):
        kw = dict(base, guided_depths=g, product=product)
        frame, st = wavefront.render_pass(sc, tree, wavefront.GuidingConfig(**kw), [sample])
        state = wavefront._RUNNERS[next(iter(wavefront._RUNNERS))].state
        ostats = {}
        oframe, ost = OR.render_pass(osc, osvo, dict(kw), sample, ostats)
        assert list(st.bins_per_depth) == ostats["bins"]
        same = state.emit_depth == ost["emit_depth"]
        same &= np.abs(state.rec_pos - ost["rec_pos"]).max(axis=(1, 2)) <= 1e-5 * sc.diagonal
        assert same.mean() >= 0.995, (sample, same.mean())
        rel = (np.abs(state.radiance - ost["radiance"]) /
               np.maximum(np.abs(ost["radiance"]), 1e-12)).max(axis=1)[same]
        assert np.mean(rel <= 1e-4) >= 0.99
        for k in ("sum_a", "sum_b", "weight_a", "weight_b"):
            setattr(tree, k, getattr(osvo, k))
        tree.propagate_up()
