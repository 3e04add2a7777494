"""Edge cases of the device pass against the CPU oracle (which is pinned to
the reference): images that miss the scene entirely, a single pixel, odd
sizes that leave partial warps and tiles, the smallest field resolution,
deeper paths, Russian roulette, and product guiding with few bins."""

import numpy as np
import pytest

from oracle import render as OR

pytestmark = pytest.mark.gpu


def _scene(scene_path, w, h, look=None):
    from paper_2405_06997_b200 import scene as S

    sc = S.load_scene(scene_path("cornell.scene"))
    cam = sc.camera
    target = cam.target if look is None else look
    sc.camera = S.Camera(cam.position, target, cam.up, cam.vfov_deg, w, h)
    return sc


def _compare(sc, res, passes, min_identical=0.98):
    """Run the same pass sequence on the device and the oracle; compare bins
    of the first depth, per-path records and the SVO weights after PT."""
    from paper_2405_06997_b200 import svo, wavefront

    tree = svo.build_from_scene(sc, res, seed=0)
    osc = OR.Scene(sc)
    osvo = OR.Svo.from_scene(sc, res, 0)
    for sample, kw in passes:
        cfg = wavefront.GuidingConfig(**kw)
        frame, st = wavefront.render_pass(sc, tree, cfg, [sample])
        stats = {}
        _, ost = OR.render_pass(osc, osvo, dict(kw), sample, stats)
        assert list(st.bins_per_depth)[:1] == stats.get("bins", [])[:1]
        state = wavefront._RUNNERS[next(iter(wavefront._RUNNERS))].state
        same = state.emit_depth == ost["emit_depth"]
        same &= np.abs(state.rec_pos - ost["rec_pos"]).max(axis=(1, 2)) <= 1e-5 * sc.diagonal
        assert same.mean() >= min_identical, (sample, kw, same.mean())
        if kw.get("guided_depths", 0) == 0:
            assert np.array_equal(tree.weight_a, osvo.weight_a)
        # continue both from the oracle's state so one divergence cannot cascade
        for k in ("sum_a", "sum_b", "weight_a", "weight_b"):
            setattr(tree, k, getattr(osvo, k))
        tree.propagate_up()
    return frame


def test_all_rays_miss(scene_path):
    from paper_2405_06997_b200 import svo, wavefront

    sc = _scene(scene_path, 24, 16, look=[278.0, 273.0, -2000.0])  # facing away
    tree = svo.build_from_scene(sc, 32, seed=0)
    for g in (0, 3):
        cfg = wavefront.GuidingConfig(max_depth=3, guided_depths=g, field_res=16, l_min=2,
                                      c_ray=8, seed=1)
        frame, st = wavefront.render_pass(sc, tree, cfg, [g])
        assert not frame.any()
        assert list(st.bins_per_depth) == [0] and list(st.rays_per_depth) == [0]
        assert st.live_per_depth == [24 * 16]


@pytest.mark.parametrize("w,h", [(1, 1), (33, 17), (7, 45)])
def test_odd_image_sizes(scene_path, w, h):
    sc = _scene(scene_path, w, h)
    base = dict(max_depth=4, field_res=16, l_min=2, c_ray=4, seed=3)
    _compare(sc, 32, [(0, dict(base, guided_depths=0)), (1, dict(base, guided_depths=4))],
             min_identical=0.97 if w * h > 1 else 1.0)


def test_smallest_fields_deep_paths_and_rr(scene_path):
    sc = _scene(scene_path, 20, 20)
    base = dict(max_depth=7, field_res=16, l_min=2, c_ray=8, seed=9)  # N = 8 from depth 2
    _compare(sc, 32, [(0, dict(base, guided_depths=0)),
                      (1, dict(base, guided_depths=7)),
                      (2, dict(base, guided_depths=3, russian_roulette=True, rr_depth=2))])


def test_product_guiding_few_bins(scene_path):
    sc = _scene(scene_path, 16, 12)
    base = dict(max_depth=3, field_res=16, l_min=1, c_ray=1000, seed=4)
    _compare(sc, 16, [(0, dict(base, guided_depths=0)),
                      (1, dict(base, guided_depths=3, product=True))])


def test_any_sample_list(scene_path):
    """render_pass accepts any sample list (wavefront.py:198-215): a PT pass
    over samples [3, 1] is the sample-major mean of the single-sample passes
    3 and 1, bit for bit; a consecutive list needs no table and a reversed
    one differs from it."""
    from paper_2405_06997_b200 import svo, wavefront

    sc = _scene(scene_path, 24, 16)
    tree = svo.build_from_scene(sc, 32, seed=0)
    cfg = wavefront.GuidingConfig(max_depth=4, guided_depths=0, field_res=16, l_min=2,
                                  c_ray=8, seed=3)
    f31, st = wavefront.render_pass(sc, tree, cfg, [3, 1])
    f3, _ = wavefront.render_pass(sc, tree, cfg, [3])
    f1, _ = wavefront.render_pass(sc, tree, cfg, [1])
    np.testing.assert_array_equal(f31, (f3 + f1) / 2.0)
    f13, _ = wavefront.render_pass(sc, tree, cfg, [1, 3])
    np.testing.assert_array_equal(f13, (f1 + f3) / 2.0)
    f57, _ = wavefront.render_pass(sc, tree, cfg, [5, 7])
    f5, _ = wavefront.render_pass(sc, tree, cfg, [5])
    f7, _ = wavefront.render_pass(sc, tree, cfg, [7])
    np.testing.assert_array_equal(f57, (f5 + f7) / 2.0)
    assert st.live_per_depth[0] == 2 * 24 * 16
