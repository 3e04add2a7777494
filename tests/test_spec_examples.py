"""Known-answer examples of the reference specification for the
hot path, checked against this package (GPU) and the CPU oracle:

* voxelize: an axis-aligned unit quad at R=4 touches exactly 16 voxels;
* build_distribution: the 2x2 field [1,3;2,2] -> marginal CDF [0.5, 1.0],
  first-row conditional [0.25, 1.0]; a uniform field -> pdf 1/(4 pi);
  sample_guided returns exactly pdf_guided of its direction;
* Eq. 5: a 2-vertex path with T ratio 0.125/0.5 and L_e = 8 deposits 2.0;
  re-running update_exitance doubles every weight, leaves every mean;
* Alg. 2: all rays in one leaf with count >= c_ray -> one bin at leaf level;
  counts below c_ray everywhere -> every bin at level l_min;
* render_pass with guiding disabled is bitwise plain path tracing;
* Eq. 7: DiscardFirst {10,2,4} -> 3, Constant -> 16/3, Linear with equal
  frames -> the frame, OneTwo {a,b} -> (a+2b)/3; tonemap 0 -> 0, 1 -> 0.5.
"""

import numpy as np
import pytest

from paper_2405_06997_b200 import core, guiding, scene as S


def _quad_scene(w=8, h=8):
    """Unit quad (2 triangles) at z = 0.5 plus a small emitter at z = 1."""
    v0 = np.array([[0, 0, 0.5], [0, 0, 0.5], [0.4, 0.4, 1.0]], dtype=float)
    v1 = np.array([[1, 0, 0.5], [1, 1, 0.5], [0.6, 0.4, 1.0]], dtype=float)
    v2 = np.array([[1, 1, 0.5], [0, 1, 0.5], [0.5, 0.6, 1.0]], dtype=float)
    mats = [S.Material("white", 0, [0.7, 0.7, 0.7]), S.Material("light", 2, [5, 5, 5])]
    cam = S.Camera([0.5, 0.5, -2.0], [0.5, 0.5, 0.5], [0, 1, 0], 40.0, w, h)
    return S.Scene(v0, v1, v2, np.array([0, 0, 1], dtype=np.int32), mats, cam)


def test_quad_voxelizes_to_16_voxels_oracle():
    from oracle import oracle as O

    sc = _quad_scene()
    lo, side = O.scene_cube(sc.bbox_lo, sc.bbox_hi)
    coords, tris = O.voxelize(sc.v0, sc.v1, sc.v2, lo, side, 4)
    quad = coords[tris < 2]
    assert len(np.unique(quad, axis=0)) == 16
    assert set(np.unique(quad[:, 2])) == {1}


def test_two_by_two_field_tables():
    fld = guiding.RadianceField(np.array([[1.0, 3.0], [2.0, 2.0]]), np.zeros(3))
    d = guiding.build_distribution(fld)
    np.testing.assert_array_equal(d.marginal_cdf, [0.5, 1.0])
    np.testing.assert_array_equal(d.conditional_cdf[0], [0.25, 1.0])
    uni = guiding.build_distribution(guiding.RadianceField(np.full((8, 8), 0.3), np.zeros(3)))
    np.testing.assert_allclose(uni.pdf_table, 1.0 / (4.0 * np.pi), rtol=1e-15)


def test_sample_guided_pdf_consistency():
    rng = np.random.default_rng(4)
    fld = guiding.RadianceField(np.maximum(rng.random((16, 16)) ** 3, 1e-2), np.zeros(3))
    d = guiding.build_distribution(fld)
    for u1, u2 in rng.random((200, 2)):
        w, pdf = guiding.sample_guided(d, u1, u2)
        assert pdf > 0.0
        assert pdf == guiding.pdf_guided(d, w)
        np.testing.assert_allclose(np.linalg.norm(w), 1.0, rtol=1e-12)


def test_eq7_and_tonemap_examples_host():
    from paper_2405_06997_b200 import accumulation as A

    assert A.tonemap_reinhard(np.array([0.0]))[0] == 0.0
    assert A.tonemap_reinhard(np.array([1.0]))[0] == 0.5
    h = A.HEURISTICS
    assert [h["discard-first"](i) for i in (1, 2, 3)] == [0.0, 1.0, 1.0]
    assert [h["one-two"](i) for i in (1, 2)] == [1.0, 2.0]


@pytest.mark.gpu
def test_eq7_examples_device():
    from paper_2405_06997_b200 import accumulation as A

    def run(heur, frames):
        buf = A.AccumulationBuffer(1, 1, heur)
        for i, v in enumerate(frames, start=1):
            buf.add_sample(np.full((1, 1, 3), float(v)), i)
        return buf.resolve()[0, 0, 0]

    assert run("discard-first", [10, 2, 4]) == 3.0
    assert run("constant", [10, 2, 4]) == pytest.approx(16.0 / 3.0, rel=1e-15)
    assert run("linear", [0.7] * 6) == pytest.approx(0.7, rel=1e-15)
    assert run("one-two", [1.0, 4.0]) == pytest.approx(3.0, rel=1e-15)
    with pytest.raises(ValueError):
        run("discard-first", [5.0])


@pytest.mark.gpu
def test_quad_voxelizes_to_16_voxels_device():
    from paper_2405_06997_b200 import svo

    frags = svo.voxelize(_quad_scene(), 4)
    quad = frags.coords[frags.tris < 2]
    assert len(np.unique(quad, axis=0)) == 16


@pytest.mark.gpu
def test_eq5_deposit_and_running_mean():
    """2-vertex path: T(p1) = 0.5, T(p2) = 0.125 at the emitter, L_e = 8 ->
    the vertex-1 deposit is (0.125 / 0.5) * 8 = 2.0; re-running the update
    doubles the weights and keeps the means."""
    from paper_2405_06997_b200 import svo, wavefront

    sc = _quad_scene()
    tree = svo.build_from_scene(sc, 16, seed=0)
    st = wavefront.PathState(1, 3, sc.camera.position)
    rp = np.zeros((1, 4, 3))
    rp[0, 0] = [0.5, 0.5, 2.0]      # previous vertex above: the nudge stays in the quad's voxel
    rp[0, 1] = [0.5, 0.5, 0.5]      # on the quad
    rp[0, 2] = [0.5, 0.45, 1.0]     # on the emitter
    rt = np.zeros((1, 4, 3))
    rt[0, 1] = 0.5
    rt[0, 2] = 0.125
    st.set("rec_pos", rp)
    st.set("rec_T", rt)
    st.dev["emit_le"].fill_(8.0)
    st.dev["emit_depth"].fill_(2)
    dirty = wavefront.update_exitance(st, tree)
    assert wavefront.update_exitance.last_deposits == 1
    sums = tree.sum_a + tree.sum_b
    w = tree.weight_a + tree.weight_b
    k = int(np.flatnonzero(w)[0])
    # the reference's return value: the dirty leaf ids (wavefront.py:266-269)
    assert dirty.dtype == np.int64 and list(dirty) == [k]
    tree.propagate_up(dirty)
    np.testing.assert_array_equal(sums[k], [2.0, 2.0, 2.0])
    means = (tree.mean_a.copy(), tree.mean_b.copy())
    wa, wb = tree.weight_a.copy(), tree.weight_b.copy()
    wavefront.update_exitance(st, tree)
    np.testing.assert_array_equal(tree.weight_a, 2 * wa)
    np.testing.assert_array_equal(tree.weight_b, 2 * wb)
    np.testing.assert_array_equal(tree.mean_a, means[0])
    np.testing.assert_array_equal(tree.mean_b, means[1])


@pytest.mark.gpu
def test_partition_threshold_examples():
    from paper_2405_06997_b200 import svo, wavefront

    sc = _quad_scene()
    tree = svo.build_from_scene(sc, 64, seed=0)
    d = tree.depth
    # all rays in one leaf, count >= c_ray: one bin at leaf level
    pos = np.tile([[0.3, 0.3, 0.5]], (40, 1))
    bins = wavefront.partition_spatial(tree, pos, np.arange(40), l_min=2, c_ray=16)
    assert len(bins) == 1 and bins[0].level == d and len(bins[0].members) == 40
    # spread below c_ray everywhere: every bin at level l_min
    rng = np.random.default_rng(0)
    pos = np.c_[rng.random((200, 2)), np.full(200, 0.5)]
    bins = wavefront.partition_spatial(tree, pos, np.arange(200), l_min=2, c_ray=10 ** 6)
    assert all(b.level == 2 for b in bins)
    assert sum(len(b.members) for b in bins) == 200


@pytest.mark.gpu
def test_guiding_disabled_is_plain_path_tracing(scene_path):
    from paper_2405_06997_b200 import svo, wavefront

    sc = S.load_scene(scene_path("cornell.scene"))
    tree = svo.build_from_scene(sc, 64, seed=0)
    cfg = wavefront.GuidingConfig(max_depth=4, guided_depths=0, l_min=3, c_ray=16, seed=11)
    with_svo, _ = wavefront.render_pass(sc, tree, cfg, [3])
    plain, _ = wavefront.render_pass(sc, None, cfg, [3])
    assert np.array_equal(with_svo.view(np.uint64), plain.view(np.uint64))
