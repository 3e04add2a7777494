"""Pin the CPU oracle (oracle/) to the reference's golden vectors.

CPU only: these run in the no-GPU suite.  The oracle is the checker of the
GPU tests at sizes the golden fixtures do not cover, so it must first match
what the real reference produced (tests/golden/make_golden.py).
"""

import hashlib

import numpy as np
import pytest

from oracle import oracle as O
from oracle import render as OR


def _digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def _scene(scene_path, name="cornell.scene", w=None, h=None):
    from paper_2405_06997_b200 import scene as S

    sc = S.load_scene(scene_path(name))
    if w is not None:
        c = sc.camera
        sc.camera = S.Camera(c.position, c.target, c.up, c.vfov_deg, w, h)
    return sc


def test_rng_and_morton_known_answers():
    assert int(O.morton_encode(2, 3, 1)) == 30
    assert int(O.morton_encode(1, 1, 1)) == 7
    k = O.stream_key(0, 4)
    from paper_2405_06997_b200 import core

    assert k == int(core.stream_key(np.uint64(0), np.uint64(4)))
    assert O.u01(k, 3) == float(core.u01_at(np.uint64(k), np.uint64(3)))


@pytest.mark.parametrize("tag,scene,res,seed", [("c64s1", "cornell.scene", 64, 1),
                                                ("e32s3", "cornell_enclosed.scene", 32, 3)])
def test_oracle_svo_build_bitwise(golden, scene_path, tag, scene, res, seed):
    g = golden("svo_golden.npz")
    sc = _scene(scene_path, scene)
    lo, side = O.scene_cube(sc.bbox_lo, sc.bbox_hi)
    coords, tris = O.voxelize(sc.v0, sc.v1, sc.v2, lo, side, res)
    assert np.array_equal(coords, g[f"{tag}_frag_coords"])
    assert np.array_equal(tris, g[f"{tag}_frag_tris"])
    b = O.build_octree(coords, sc.normals[tris], res, seed)
    for k in ("level_off", "codes", "child_base", "child_mask", "parent", "sorted_codes",
              "sort_perm"):
        assert np.array_equal(b[k], g[f"{tag}_{k}"]), k
    assert np.array_equal(b["normal"].view(np.uint64), g[f"{tag}_normal"].view(np.uint64))


def test_oracle_svo_build_digest_c1_enclosed_r128(golden, scene_path):
    g = golden("svo_golden.npz")
    row = [str(r).split(",") for r in g["digests"] if str(r).startswith("cornell_enclosed.scene,128")]
    f = row[0]
    sc = _scene(scene_path, "cornell_enclosed.scene")
    lo, side = O.scene_cube(sc.bbox_lo, sc.bbox_hi)
    coords, tris = O.voxelize(sc.v0, sc.v1, sc.v2, lo, side, 128)
    b = O.build_octree(coords, sc.normals[tris], 128, 3)
    assert [_digest(b["codes"]), _digest(b["normal"])] == [f[10], f[14]]


@pytest.fixture(scope="module")
def rsetup(golden, scene_path):
    R = golden("render_golden.npz")
    c = dict(zip([str(k) for k in R["cfg_keys"]], [int(v) for v in R["cfg_vals"]]))
    sc0 = _scene(scene_path, "cornell.scene", c["W"], c["H"])
    return R, c, sc0, OR.Scene(sc0), OR.Svo.from_scene(sc0, c["R"], c["svo_seed"])


def _load(svo, R, prefix):
    for k in ("sum_a", "sum_b", "weight_a", "weight_b"):
        setattr(svo, k, R[f"{prefix}_svo_{k}"].copy())
    svo.propagate()


def test_oracle_propagate_intersect_cones_partition(rsetup):
    R, c, sc0, sc, svo = rsetup
    _load(svo, R, "p0")
    assert np.array_equal(svo.mean_a.view(np.uint64), R["p0_svo_mean_a"].view(np.uint64))
    t, tri = OR.intersect(sc, R["cone_origins"], R["cone_dirs"])
    assert np.array_equal(tri, R["isect_tri"])
    for res in (32, 128):
        got = OR.trace_cones(sc, svo, R["cone_origins"], R["cone_dirs"],
                             float(R[f"cone_{res}_omega"]))
        assert np.all(np.isclose(got, R[f"cone_{res}_rgb"], rtol=1e-9, atol=1e-300))
    for d in range(1, 5):
        nodes, mem = OR.partition(svo, R[f"p0_d{d}_positions"], c["l_min"], c["c_ray"])
        assert np.array_equal(nodes, R[f"p0_d{d}_bin_nodes"])
        pidx = R[f"p0_d{d}_path_idx"]
        assert np.array_equal(np.concatenate([pidx[m] for m in mem]), R[f"p0_d{d}_bin_members"])


def test_oracle_fields_and_tables(golden, scene_path):
    F = golden("fields_golden.npz")
    sc0 = _scene(scene_path)
    sc = OR.Scene(sc0)
    svo = OR.Svo.from_scene(sc0, 64, 0)
    for k in ("sum_a", "sum_b", "weight_a", "weight_b"):
        setattr(svo, k, F["svo_" + k].copy())
    svo.propagate()
    for n in (8, 16, 32, 64, 128):
        got = OR.fields(sc, svo, F["origins"], F["jitters"], n)
        assert np.all(np.abs(got - F[f"vals_{n}"]) <= 1e-9 * np.abs(F[f"vals_{n}"])), n
        tb = OR.tables(F[f"vals_{n}"], 2)
        for k in ("marg", "cond", "pdftab", "block_sums", "blk_marg", "blk_cond"):
            assert np.array_equal(tb[k].view(np.uint64), F[f"tab_{n}_{k}"].view(np.uint64)), k


def _identical(R, tag, st, diag):
    same = st["emit_depth"] == R[f"{tag}_emit_depth"]
    same &= np.abs(st["rec_pos"] - R[f"{tag}_rec_pos"]).max(axis=(1, 2)) <= 1e-5 * diag
    rel = (np.abs(st["radiance"] - R[f"{tag}_radiance"])
           / np.maximum(np.abs(R[f"{tag}_radiance"]), 1e-12)).max(axis=1)
    return same, rel


@pytest.mark.parametrize("tag,guided,product,sample", [("p0", False, False, 0),
                                                       ("p1", True, False, 1),
                                                       ("p1x", True, True, 1)])
def test_oracle_render_pass(rsetup, tag, guided, product, sample):
    R, c, sc0, sc, svo = rsetup
    if tag == "p0":
        for k in ("sum_a", "sum_b", "weight_a", "weight_b"):
            setattr(svo, k, np.zeros_like(R["p0_svo_" + k]))
        svo.propagate()
    else:
        _load(svo, R, "p0")
    cfg = dict(max_depth=c["max_depth"], guided_depths=c["max_depth"] if guided else 0,
               field_res=c["field_res"], l_min=c["l_min"], c_ray=c["c_ray"], seed=c["seed"],
               product=product)
    stats = {}
    _, st = OR.render_pass(sc, svo, cfg, sample, stats)
    assert stats["bins"] == list(R[f"{tag}_bins_per_depth"])
    assert stats["rays"] == list(R[f"{tag}_rays_per_depth"])
    same, rel = _identical(R, tag, st, sc0.diagonal)
    assert same.mean() == 1.0
    assert np.all(rel[same] <= 1e-4)
    np.testing.assert_allclose(svo.sum_a, R[f"{tag}_svo_sum_a"], rtol=1e-9, atol=1e-12)
    assert np.array_equal(svo.weight_a, R[f"{tag}_svo_weight_a"])


def test_oracle_c2_svo_equals_the_reference_build(golden, scene_path):
    """The oracle's R=1024 build (C2's SVO, ~1 min here) against the
    reference's own build digests (make_golden.py gen_r1024)."""
    import hashlib

    G = golden("r1024_golden.npz")
    sc0 = _scene(scene_path)
    svo = OR.Svo.from_scene(sc0, 1024, 0)
    dig = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]  # noqa: E731
    assert np.array_equal(svo.level_off, G["level_off"])
    for k, dt in (("codes", np.uint64), ("child_base", np.int64), ("child_mask", np.uint8),
                  ("parent", np.int64)):
        assert dig(np.asarray(svo.d[k]).astype(dt)) == str(G[k]), k
    assert dig(svo.normal) == str(G["normal"])
