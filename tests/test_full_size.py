"""Parity at the headline size (BASELINE configs[1] / C2: Cornell 1920x1080,
SVO R=1024, D=4, N0=128): a PT-first pass and a guided pass on the device
against the CPU oracle (pinned to the reference's goldens), path for path.
The oracle works on the device-built SVO structure (bit-exact with the
oracle's own build, tests/test_svo_build.py) to skip its 30 s build."""


import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_c2_1080p_paths_match_oracle(scene_path):
    from oracle import render as OR
    from paper_2405_06997_b200 import scene as S, svo, wavefront

    sc = S.load_scene(scene_path("cornell.scene"))
    cam = sc.camera
    sc.camera = S.Camera(cam.position, cam.target, cam.up, cam.vfov_deg, 1920, 1080)
    tree = svo.build_from_scene(sc, 1024, seed=0)
    built = {"level_off": np.asarray(tree.level_off, dtype=np.int64),
             "parent": np.asarray(tree.parent, dtype=np.int64),
             "child_base": np.asarray(tree.child_base, dtype=np.int64),
             "child_mask": np.asarray(tree.child_mask, dtype=np.uint8),
             "normal": np.asarray(tree.normal, dtype=np.float64)}
    lo, side = svo.scene_cube(sc)
    osvo = OR.Svo(built, lo, side, 1024)
    osc = OR.Scene(sc)
    base = dict(max_depth=4, field_res=128, l_min=5, c_ray=512, seed=0)
    for sample, g in ((0, 0), (1, 4)):
        kw = dict(base, guided_depths=g)
        frame, st = wavefront.render_pass(sc, tree, wavefront.GuidingConfig(**kw), [sample])
        state = wavefront._RUNNERS[next(iter(wavefront._RUNNERS))].state
        ostats = {}
        oframe, ost = OR.render_pass(osc, osvo, dict(kw), sample, ostats)
        assert list(st.bins_per_depth)[0] == ostats["bins"][0]
        assert np.abs(np.subtract(st.bins_per_depth, ostats["bins"])).max() <= 2
        same = state.emit_depth == ost["emit_depth"]
        same &= np.abs(state.rec_pos - ost["rec_pos"]).max(axis=(1, 2)) <= 1e-5 * sc.diagonal
        assert same.mean() >= 0.999, (sample, same.mean())
        rel = (np.abs(state.radiance - ost["radiance"]) /
               np.maximum(np.abs(ost["radiance"]), 1e-12)).max(axis=1)[same]
        assert np.mean(rel <= 1e-4) >= 0.999
        np.testing.assert_allclose(frame.mean(), oframe.mean(), rtol=1e-6)
        if g == 0:
            assert np.array_equal(tree.weight_a, osvo.weight_a)
            assert np.array_equal(tree.weight_b, osvo.weight_b)
        for k in ("sum_a", "sum_b", "weight_a", "weight_b"):
            setattr(tree, k, getattr(osvo, k))
        tree.propagate_up()
