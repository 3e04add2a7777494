"""Properties of the host-side reference API (core / scene helpers) that the
reference's own suite (pkg/tests/test_core.py, test_scene.py) pins, restated
here as property tests against this package: octahedral map, Morton codes,
fold-aware blur (vs a dense-matrix oracle), counter RNG, scene loading
errors, camera, BSDF / NEE helpers; and, on the GPU, intersection and
occlusion against a numpy brute-force oracle.
"""

import math

import numpy as np
import pytest

from paper_2405_06997_b200 import core, scene as S


# -- octahedral map ------------------------------------------------------------
def test_octa_round_trip_and_poles():
    rng = np.random.default_rng(1)
    d = rng.standard_normal((20000, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    u, v = core.octa_dir_to_uv(d)
    back = core.octa_uv_to_dir(u, v)
    ang = np.arccos(np.clip(np.sum(back * d, axis=1), -1.0, 1.0))
    assert ang.max() < 1e-6
    np.testing.assert_allclose(core.octa_uv_to_dir(0.5, 0.5), [0.0, 0.0, 1.0], atol=1e-15)
    for uv in ((0.0, 0.0), (1.0 - 1e-12, 1.0 - 1e-12)):
        assert core.octa_uv_to_dir(*uv)[2] < -0.999999


def test_octa_cells_equal_area_and_distinct():
    n = 8
    rng = np.random.default_rng(2)
    d = rng.standard_normal((400000, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    u, v = core.octa_dir_to_uv(d)
    cell = np.minimum((v * n).astype(int), n - 1) * n + np.minimum((u * n).astype(int), n - 1)
    frac = np.bincount(cell, minlength=n * n) / len(d)
    np.testing.assert_allclose(frac, 1.0 / (n * n), rtol=0.06)  # equal solid angle 4pi/n^2
    c = (np.arange(n) + 0.5) / n
    gu, gv = np.meshgrid(c, c)
    centres = core.octa_uv_to_dir(gu, gv).reshape(-1, 3)
    assert len(np.unique(np.round(centres, 12), axis=0)) == n * n


# -- Morton ----------------------------------------------------------------------
def test_morton_properties():
    assert core.morton_encode(0, 0, 0) == 0
    assert core.morton_encode(1, 0, 0) == 1 and core.morton_encode(0, 1, 0) == 2
    assert core.morton_encode(0, 0, 1) == 4
    top = (1 << 21) - 1
    assert core.morton_encode(top, top, top) == (1 << 63) - 1
    rng = np.random.default_rng(3)
    x, y, z = (rng.integers(0, 1 << 21, 5000) for _ in range(3))
    c = core.morton_encode(x, y, z)
    dx, dy, dz = core.morton_decode(c)
    assert np.array_equal(dx, x) and np.array_equal(dy, y) and np.array_equal(dz, z)
    # monotone in each coordinate with the others fixed
    assert np.all(np.diff(core.morton_encode(np.arange(100), 7, 9).astype(np.int64)) > 0)
    with pytest.raises(ValueError):
        core.morton_encode(1 << 21, 0, 0)
    with pytest.raises(ValueError):
        core.morton_encode(-1, 0, 0)


# -- blur ------------------------------------------------------------------------
def _fold_matrix(n, sigma):
    """Dense (n*n, n*n) operator of the fold-aware separable blur."""
    taps, r = core._blur_kernel(sigma)
    idx, flip = core._fold_lut(n, r)

    def one_axis():
        # M[(row, out_col), (src_row, src_col)] for a blur along columns
        m = np.zeros((n, n, n, n))
        for j in range(n):
            for i in range(n):
                for k, w in enumerate(taps):
                    c, f = idx[i + k], flip[i + k]
                    m[j, i, n - 1 - j if f else j, c] += w
        return m.reshape(n * n, n * n)

    h = one_axis()
    t = np.zeros((n * n, n * n))  # transpose permutation
    for j in range(n):
        for i in range(n):
            t[i * n + j, j * n + i] = 1.0
    return t @ h @ t @ h


@pytest.mark.parametrize("n,sigma", [(8, 1.0), (16, 2.5)])
def test_blur_matches_dense_oracle(n, sigma):
    rng = np.random.default_rng(n)
    g = rng.random((n, n))
    ref = (_fold_matrix(n, sigma) @ g.reshape(-1)).reshape(n, n)
    np.testing.assert_allclose(core.gaussian_blur(g, sigma), ref, rtol=1e-12, atol=1e-14)
    imp = np.zeros((n, n))
    imp[0, 1] = 1.0  # boundary impulse: its mass folds back onto the grid
    np.testing.assert_allclose(core.gaussian_blur(imp, sigma).sum(), 1.0, rtol=1e-12)


def test_blur_constant_linear_batched():
    g = np.full((16, 16), 3.25)
    np.testing.assert_allclose(core.gaussian_blur(g, 1.0), g, rtol=1e-14)
    rng = np.random.default_rng(5)
    a, b = rng.random((2, 16, 16))
    np.testing.assert_allclose(core.gaussian_blur(2 * a + b, 1.0),
                               2 * core.gaussian_blur(a, 1.0) + core.gaussian_blur(b, 1.0),
                               rtol=1e-12)
    batch = rng.random((3, 16, 16))
    out = core.gaussian_blur(batch, 1.5)
    for k in range(3):
        assert np.array_equal(out[k], core.gaussian_blur(batch[k], 1.5))
    with pytest.raises(ValueError):
        core.gaussian_blur(g, 0.0)


# -- RNG --------------------------------------------------------------------------
def test_counter_rng_properties():
    a, b = core.RngStream(9, 4), core.RngStream(9, 4)
    xs = [a.next() for _ in range(5)]
    assert xs == [b.next() for _ in range(5)]
    c = core.RngStream(9, 4, counter=2)
    assert c.next() == xs[2]
    u = core.RngStream(1, 2).next_n(100000)
    assert u.min() >= 0.0 and u.max() < 1.0
    srt = np.sort(u)
    ks = np.max(np.abs(srt - (np.arange(1, len(u) + 1) / len(u))))
    assert ks < 1.63 / math.sqrt(len(u))  # KS 1 % level
    v = core.RngStream(1, 3).next_n(100000)
    assert abs(np.corrcoef(u, v)[0, 1]) < 0.02
    w = core.RngStream(0, 0, counter=(1 << 64) - 1)
    w.next()
    assert w.counter == 0


# -- scene loading ----------------------------------------------------------------
def _write(tmp_path, body, obj=True):
    if obj:
        (tmp_path / "t.obj").write_text("v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 3\n")
    p = tmp_path / "s.scene"
    p.write_text(body)
    return str(p)


GOOD = ("wfpg-scene v1\ncamera 0 0 -1  0 0 0  0 1 0  40 8 8\n"
        "material w lambert 0.5 0.5 0.5\nmaterial l emitter 1 1 1\nmesh t.obj w\nmesh t.obj l\n")


def test_scene_loader_errors(tmp_path, scene_path):
    sc = S.load_scene(_write(tmp_path, GOOD))
    assert sc.triangle_count == 2
    bad = {
        "unknown material": GOOD.replace("lambert", "velvet"),
        "missing mesh": GOOD.replace("mesh t.obj w", "mesh none.obj w"),
        "header": GOOD.replace("wfpg-scene v1\n", ""),
        "emitter": GOOD.replace("mesh t.obj l\n", ""),
    }
    for name, body in bad.items():
        with pytest.raises(S.SceneError):
            S.load_scene(_write(tmp_path, body))
    (tmp_path / "nan.obj").write_text("v 0 0 nan\nv 1 0 0\nv 0 1 0\nf 1 2 3\n")
    with pytest.raises(S.SceneError):
        S.load_scene(_write(tmp_path, GOOD.replace("mesh t.obj w", "mesh nan.obj w"), obj=False))
    assert S.load_scene(scene_path("cornell.scene")).triangle_count == 36


# -- camera -----------------------------------------------------------------------
def test_camera_corner_symmetry_and_fov(scene_path):
    cam = S.load_scene(scene_path("cornell.scene")).camera
    w, h = cam.width, cam.height
    d = cam.ray_directions(np.array([0, w - 1, 0, w - 1]), np.array([0, 0, h - 1, h - 1]),
                           0.5, 0.5)
    f = cam.forward
    cosines = d @ f
    np.testing.assert_allclose(cosines, cosines[0], rtol=1e-12)
    half = math.radians(cam.vfov_deg) / 2
    # even width: pixel w/2 with zero sub-pixel offset is the centre column;
    # the top edge of row 0 lies at half the vertical field of view
    top = cam.ray_directions(np.array([w // 2]), np.array([0]), 0.0, 0.0)[0]
    assert w % 2 == 0 and abs(math.acos(float(top @ f)) - half) < 1e-12


# -- BSDF / NEE helpers -------------------------------------------------------------
def test_lambert_sampling_and_pdf():
    n = np.array([0.0, 0.0, 1.0])
    rng = np.random.default_rng(6)
    u1, u2 = rng.random(200000), rng.random(200000)
    wi = S.sample_cosine(n, u1, u2)
    np.testing.assert_allclose(np.linalg.norm(wi, axis=1), 1.0, rtol=1e-12)
    cos = wi @ n
    assert cos.min() >= 0.0
    hist, _ = np.histogram(cos ** 2, bins=10, range=(0, 1))  # cos^2 ~ U(0,1)
    np.testing.assert_allclose(hist / len(cos), 0.1, atol=0.005)
    m = S.Material("w", S.LAMBERT, [0.5, 0.5, 0.5])
    w0, pdf, f, delta = S.sample_bsdf(m, n, n, 0.3, 0.7)
    assert not delta and pdf == pytest.approx(S.pdf_bsdf(m, n, w0, n), rel=1e-14)
    np.testing.assert_allclose(f, 0.5 / np.pi)
    assert S.pdf_bsdf(m, n, -n, n) == 0.0


def test_mirror_is_exact_reflection():
    n = np.array([0.0, 1.0, 0.0])
    wo = np.array([0.6, 0.8, 0.0])
    m = S.Material("m", S.MIRROR, [1, 1, 1])
    wi, pdf, f, delta = S.sample_bsdf(m, wo, n, 0.1, 0.2)
    np.testing.assert_allclose(wi, [-0.6, 0.8, 0.0], atol=1e-15)
    assert delta and pdf == 0.0


def test_nee_pdf_conversion(scene_path):
    sc = S.load_scene(scene_path("cornell.scene"))
    p = np.array([278.0, 10.0, 279.0])
    d, dist, pdf, rad, _ = S.sample_nee(sc, p, 0.37, 0.61)
    lp, ln, _, _ = S.sample_emitter_points(sc, 0.37, 0.61)
    cos_l = float(ln[0] @ -d)
    assert pdf == pytest.approx(dist * dist / (sc.emitter_area * cos_l), rel=1e-12)
    assert S.pdf_nee(sc, p, lp[0], ln[0]) == pytest.approx(pdf, rel=1e-12)
    assert np.all(rad > 0)


# -- device intersection vs a numpy brute-force oracle --------------------------------
def _brute(sc, o, d, tmin):
    e1, e2, v0 = sc.e1, sc.e2, sc.v0
    p = np.cross(d[:, None, :], e2[None])
    det = np.einsum("tk,ntk->nt", e1, p)
    tv = o[:, None, :] - v0[None]
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / det
        u = np.einsum("ntk,ntk->nt", tv, p) * inv
        q = np.cross(tv, e1[None])
        v = np.einsum("nk,ntk->nt", d, q) * inv
        t = np.einsum("tk,ntk->nt", e2, q) * inv
    ok = (np.abs(det) > 1e-300) & (u >= 0) & (v >= 0) & (u + v <= 1) & (t > tmin)
    t = np.where(ok, t, np.inf)
    return t.min(axis=1), np.where(np.isfinite(t.min(axis=1)), t.argmin(axis=1), -1)


@pytest.mark.gpu
def test_device_intersection_matches_brute_force(scene_path):
    sc = S.load_scene(scene_path("cornell.scene"))
    rng = np.random.default_rng(7)
    o = sc.bbox_lo + (sc.bbox_hi - sc.bbox_lo) * rng.random((5000, 3))
    d = rng.standard_normal((5000, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    t, tri = sc.intersect_batch(o, d)
    bt, btri = _brute(sc, o, d, sc.ray_eps)
    assert np.mean(tri == btri) > 0.9995
    same = (tri == btri) & (tri >= 0)
    np.testing.assert_allclose(t[same], bt[same], rtol=1e-9)
    assert np.all(np.isinf(t[tri < 0]))
    # occlusion consistent with the nearest hit
    hit = tri >= 0
    occ_before = sc.occluded_batch(o[hit], d[hit], 0.999 * t[hit])
    occ_after = sc.occluded_batch(o[hit], d[hit], 1.001 * t[hit])
    assert not occ_before.any() and occ_after.all()
    assert S.intersect(sc, [278.0, 273.0, 200.0], [0.0, 0.0, 1.0]).triangle_id >= 0


def test_bvh_native_build_equals_restatement(scene_path):
    """The C++ host BVH build (csrc/bvh_host.cu) reproduces the numpy
    restatement of the reference's build array for array."""
    from paper_2405_06997_b200 import bvh, scene as S

    rng = np.random.default_rng(3)
    v0 = rng.random((3000, 3)) * 50.0
    cases = [(v0, v0 + rng.random((3000, 3)), v0 + rng.random((3000, 3)))]
    flat = v0.copy()
    flat[:, 2] = 0.0
    cases.append((flat, flat + [1.0, 0.0, 0.0], flat + [0.0, 1.0, 0.0]))  # zero extent in z
    for f in ("cornell.scene", "cornell_tess.scene", "c3_two_rooms.scene"):
        sc = S.load_scene(scene_path(f))
        cases.append((sc.v0, sc.v1, sc.v2))
    for a, b, c in cases:
        x, y = bvh.build(a, b, c), bvh.build_py(a, b, c)
        for k in ("lo", "hi", "left", "right", "count", "order"):
            assert np.array_equal(getattr(x, k), getattr(y, k)), k
