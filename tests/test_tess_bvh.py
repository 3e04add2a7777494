"""BVH paths: the Cornell box with every triangle
midpoint-subdivided 3x (2,304 triangles, above the 512-triangle brute-force
limit), so nearest-hit, shadow and field queries all traverse the BVH —
which is the reference's own BVH, rebuilt identically on the host.  Golden
vectors from the real reference (tests/golden/make_golden.py tess)."""

import hashlib
import os

import numpy as np
import pytest

from oracle import oracle as O
from oracle import render as OR


def _digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


@pytest.fixture(scope="module")
def G(golden):
    return golden("tess_golden.npz")


def _cfg(G):
    return dict(zip([str(k) for k in G["cfg_keys"]], [int(v) for v in G["cfg_vals"]]))


def _scene(scene_path, c):
    from paper_2405_06997_b200 import scene as S

    sc = S.load_scene(scene_path("cornell_tess.scene"))
    cam = sc.camera
    sc.camera = S.Camera(cam.position, cam.target, cam.up, cam.vfov_deg, c["W"], c["H"])
    return sc


def _identical(G, tag, rec_pos, emit_depth, diag):
    same = emit_depth == G[f"{tag}_emit_depth"]
    return same & (np.abs(rec_pos - G[f"{tag}_rec_pos"]).max(axis=(1, 2)) <= 1e-5 * diag)


def test_generator_and_oracle(G, tmp_path, scene_path):
    from paper_2405_06997_b200 import scenegen

    scenegen.write_tessellated_cornell(str(tmp_path))
    for f in os.listdir(tmp_path):
        assert open(tmp_path / f).read() == open(scene_path(f)).read(), f
    c = _cfg(G)
    sc0 = _scene(scene_path, c)
    assert sc0.triangle_count == 2304
    lo, side = O.scene_cube(sc0.bbox_lo, sc0.bbox_hi)
    f = str(G["svo_digests"][0]).split(",")
    coords, tris = O.voxelize(sc0.v0, sc0.v1, sc0.v2, lo, side, int(f[0]))
    b = O.build_octree(coords, sc0.normals[tris], int(f[0]), int(f[1]))
    assert [str(len(coords)), str(int(b["level_off"][-1])), _digest(b["codes"]),
            _digest(b["normal"])] == [f[2], f[3], f[5], f[9]]
    # the oracle's BVH traversal reproduces the reference's hits
    sc = OR.Scene(sc0)
    assert sc.c.brute == 0
    t, tri = OR.intersect(sc, G["isect_o"], G["isect_d"])
    assert np.array_equal(tri, G["isect_tri"])
    # and its PT-first pass the reference's paths
    svo = OR.Svo.from_scene(sc0, c["R"], c["svo_seed"])
    stats = {}
    cfg = dict(max_depth=c["max_depth"], guided_depths=0, field_res=c["field_res"],
               l_min=c["l_min"], c_ray=c["c_ray"], seed=c["seed"])
    _, st = OR.render_pass(sc, svo, cfg, 0, stats)
    assert stats["bins"] == list(G["p0_bins_per_depth"])
    assert _identical(G, "p0", st["rec_pos"], st["emit_depth"], sc0.diagonal).mean() == 1.0


@pytest.mark.gpu
def test_device_bvh_paths(G, scene_path):
    from paper_2405_06997_b200 import svo, wavefront

    c = _cfg(G)
    sc = _scene(scene_path, c)
    assert sc.abi().brute == 0
    for row in G["svo_digests"]:
        f = str(row).split(",")
        tree = svo.build_from_scene(sc, int(f[0]), seed=int(f[1]))
        assert [str(tree.node_count), _digest(tree.codes), _digest(tree.normal)] == \
            [f[3], f[5], f[9]]
    t, tri = sc.intersect_batch(G["isect_o"], G["isect_d"])
    assert np.mean(tri == G["isect_tri"]) >= 0.9995
    ok = (tri == G["isect_tri"]) & (tri >= 0)
    np.testing.assert_allclose(t[ok], G["isect_t"][ok], rtol=1e-12)
    tree = svo.build_from_scene(sc, c["R"], seed=c["svo_seed"])
    for tag, sample, g, floor in (("p0", 0, 0, 0.999), ("p1", 1, c["max_depth"], 0.98)):
        cfg = wavefront.GuidingConfig(max_depth=c["max_depth"], guided_depths=g,
                                      field_res=c["field_res"], l_min=c["l_min"],
                                      c_ray=c["c_ray"], seed=c["seed"])
        if tag == "p1":
            for k in ("sum_a", "sum_b", "weight_a", "weight_b"):
                setattr(tree, k, G["p0_svo_" + k])
            tree.propagate_up()
        frame, stats = wavefront.render_pass(sc, tree, cfg, [sample])
        st = wavefront._RUNNERS[next(iter(wavefront._RUNNERS))].state
        assert list(stats.bins_per_depth)[:1] == list(G[f"{tag}_bins_per_depth"])[:1]
        same = _identical(G, tag, st.rec_pos, st.emit_depth, sc.diagonal)
        assert same.mean() >= floor, (tag, same.mean())
        if tag == "p0":
            assert np.array_equal(tree.weight_a, G["p0_svo_weight_a"])


@pytest.mark.gpu
@pytest.mark.parametrize("n", [16, 128])
def test_device_bvh_fields_match_oracle(G, scene_path, n):
    """Field generation over the BVH (the warp-cooperative packet walk of the
    field tracer, geometry.cuh warp_bvh_nearest) against the oracle's per-ray
    BVH traversal (_kernels.pyx:398-445 restated) on the same SVO state:
    guiding.py:231-251 with the reference's tolerance bar."""
    from paper_2405_06997_b200 import guiding, svo

    c = _cfg(G)
    sc = _scene(scene_path, c)
    tree = svo.build_from_scene(sc, c["R"], seed=c["svo_seed"])
    for k in ("sum_a", "sum_b", "weight_a", "weight_b"):
        setattr(tree, k, G["p0_svo_" + k])
    tree.propagate_up()
    osvo = OR.Svo.from_scene(sc, c["R"], c["svo_seed"])
    osvo.mean_a = np.ascontiguousarray(tree.mean_a)
    osvo.mean_b = np.ascontiguousarray(tree.mean_b)
    # origins: surface points seen by the reference's test rays (on walls,
    # inside the box), jitters from a fixed stream
    hit = G["isect_tri"] >= 0
    o = G["isect_o"][hit] + G["isect_t"][hit, None] * G["isect_d"][hit]
    o = o[:: max(1, len(o) // 24)][:24]
    jit = np.random.default_rng(7).random((len(o), 2))
    got = guiding.generate_fields_batch(tree, sc, o, n, jit, blur_sigma=1.0)
    ref = OR.fields(OR.Scene(sc), osvo, o, jit, n)
    rel = np.abs(got - ref) / np.maximum(np.abs(ref), 1e-300)
    assert np.mean(rel < 1e-9) >= 0.99, np.mean(rel < 1e-9)
    np.testing.assert_allclose(got.sum(axis=(1, 2)), ref.sum(axis=(1, 2)), rtol=1e-3)
