"""The drop-in at the reference's own seam: the UNMODIFIED reference package
(baseline/_ref, installed from /root/reference/pkg by pip)
renders with ``wfpg.backend.set_backend(paper_2405_06997_b200.backend_cuda)``
(backend.py:25-28) — its render_pass, partition, field generation and
exitance update run unchanged, every kernel call lands in libwfpg_b200.so —
and its paths must be those of its own compiled backend.  Skipped when the
reference is not installed."""

import os

import numpy as np
import pytest

from conftest import REPO

REF = os.path.join(REPO, "baseline", "_ref")


@pytest.fixture(scope="module")
def wfpg():
    if not os.path.isdir(os.path.join(REF, "wfpg")):
        pytest.skip("reference not installed in baseline/_ref")
    import sys

    sys.path.insert(0, REF)
    try:
        import wfpg as w
        from wfpg import backend  # noqa: F401
    except ImportError as e:  # pragma: no cover
        pytest.skip(f"reference not importable: {e}")
    return w


def _capture(wfpg, sc, tree, cfg, sample):
    from wfpg import wavefront

    cap = {}
    orig = wavefront.update_exitance

    def upd(state, svo):
        cap.update({k: getattr(state, k).copy() for k in ("radiance", "rec_pos", "emit_depth")})
        return orig(state, svo)

    wavefront.update_exitance = upd
    try:
        frame, stats = wavefront.render_pass(sc, tree, cfg, [sample])
    finally:
        wavefront.update_exitance = orig
    return frame, stats, cap


@pytest.mark.gpu
@pytest.mark.parametrize("product", [False, True])
def test_reference_render_pass_on_the_cuda_backend(wfpg, scene_path, product):
    from wfpg import backend, scene, svo, wavefront

    from paper_2405_06997_b200 import backend_cuda

    sc = scene.load_scene(scene_path("cornell.scene"))
    c = sc.camera
    sc.camera = scene.Camera(c.position, c.target, c.up, c.vfov_deg, 32, 32)
    base = dict(max_depth=4, field_res=32, l_min=3, c_ray=16, seed=7)
    runs = {}
    orig = backend.get()
    assert orig.NAME == "compiled"
    for name, mod in (("compiled", orig), ("cuda", backend_cuda)):
        backend.set_backend(mod)
        try:
            tree = svo.build_from_scene(sc, 64, seed=0)  # the reference's own numpy build
            _, st0, c0 = _capture(wfpg, sc, tree, wavefront.GuidingConfig(guided_depths=0, **base),
                                  0)
            _, st1, c1 = _capture(wfpg, sc, tree, wavefront.GuidingConfig(
                guided_depths=4, product=product, **base), 1)
            runs[name] = (st0, c0, st1, c1, tree.weight_a.copy(), tree.mean_a.copy())
        finally:
            backend.set_backend(orig)
    a, b = runs["compiled"], runs["cuda"]
    assert backend_cuda.NAME == "cuda-sm100a" and backend_cuda.COMPILED
    # PT-first: identical paths and bins; guided: the reference's bins
    assert a[0].bins_per_depth == b[0].bins_per_depth
    assert a[0].material_groups == b[0].material_groups
    diag = sc.diagonal
    for k in (1, 3):
        ca, cb = a[k], b[k]
        same = (ca["emit_depth"] == cb["emit_depth"]) & (
            np.abs(ca["rec_pos"] - cb["rec_pos"]).max(axis=(1, 2)) <= 1e-5 * diag)
        assert same.mean() >= (1.0 if k == 1 else 0.98), (k, same.mean())
        rel = (np.abs(ca["radiance"] - cb["radiance"])
               / np.maximum(np.abs(ca["radiance"]), 1e-12)).max(axis=1)
        assert np.mean(rel[same] <= 1e-4) >= 0.99, k
    assert a[2].bins_per_depth == b[2].bins_per_depth
    # the PT-first deposits land in the same leaves
    assert np.array_equal(a[4] > 0, b[4] > 0)


@pytest.mark.gpu
def test_reference_objects_through_every_entry_point(wfpg, scene_path):
    """Each of the eight backend functions on the reference's numpy objects
    equals the reference's compiled backend (ids exact, floats to 1e-9)."""
    from wfpg import _kernelshim as K, scene, svo

    from paper_2405_06997_b200 import backend_cuda as B

    sc = scene.load_scene(scene_path("cornell.scene"))
    tree = svo.build_from_scene(sc, 64, seed=0)
    rng = np.random.default_rng(3)
    m = 2048
    lo, hi = sc.bbox_lo, sc.bbox_hi
    org = lo + (hi - lo) * (0.05 + 0.9 * rng.random((m, 3)))
    d = rng.standard_normal((m, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    t1, i1 = K.intersect_rays(sc, org, d, sc.ray_eps)
    t2, i2 = B.intersect_rays(sc, org, d, sc.ray_eps)
    assert np.array_equal(i1, i2)
    np.testing.assert_allclose(t2[i2 >= 0], t1[i1 >= 0], rtol=1e-12)
    tm = np.where(np.isfinite(t1), 0.5 * t1, 10.0)
    assert np.array_equal(K.occluded_rays(sc, org, d, sc.ray_eps, tm),
                          B.occluded_rays(sc, org, d, sc.ray_eps, tm))
    for x, y in zip(K.descend_tracked(tree, org), B.descend_tracked(tree, org)):
        assert np.array_equal(x, y)
    assert np.array_equal(K.descend_leaves(tree, org), B.descend_leaves(tree, org))
    tree.mean_a[:] = rng.random(tree.mean_a.shape)
    tree.mean_b[:] = rng.random(tree.mean_b.shape)
    for omega in (4 * np.pi / 32 ** 2, 4 * np.pi / 128 ** 2):
        ra = K.trace_cones_multi(tree, sc, org, d, omega)
        rb = B.trace_cones_multi(tree, sc, org, d, omega)
        assert np.mean(np.all(np.abs(ra - rb) <= 1e-9 * np.abs(ra) + 1e-12, axis=1)) >= 0.995
    keys = rng.integers(0, 2 ** 63, 500, dtype=np.uint64)
    pix = rng.integers(0, sc.camera.width * sc.camera.height, 500)
    oa, da = K.camera_rays(sc.camera, keys, pix)
    ob, db = B.camera_rays(sc.camera, keys, pix)
    assert np.array_equal(oa, ob)
    np.testing.assert_allclose(db, da, rtol=0, atol=1e-15)
