"""Item 1 — SVO builder parity: device build vs the reference's golden arrays
(bit-exact integer arrays and normals) and vs the CPU oracle on random
fragment sets."""

import hashlib

import numpy as np
import pytest

from conftest import SCENES  # noqa: F401


def _digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


@pytest.mark.gpu
@pytest.mark.parametrize("tag,scene,res,seed", [("c64s1", "cornell.scene", 64, 1),
                                                ("e32s3", "cornell_enclosed.scene", 32, 3)])
def test_build_from_scene_matches_reference(golden, scene_path, tag, scene, res, seed):
    from paper_2405_06997_b200 import scene as S, svo

    g = golden("svo_golden.npz")
    sc = S.load_scene(scene_path(scene))
    frags = svo.voxelize(sc, res)
    assert np.array_equal(frags.coords, g[f"{tag}_frag_coords"])
    assert np.array_equal(frags.tris, g[f"{tag}_frag_tris"])
    tree = svo.build_from_scene(sc, res, seed=seed)
    codes, perm = svo.sorted_fragments(tree)
    assert np.array_equal(codes, g[f"{tag}_sorted_codes"])
    assert np.array_equal(perm, g[f"{tag}_sort_perm"])
    assert np.array_equal(tree.level_off, g[f"{tag}_level_off"])
    assert np.array_equal(tree.codes, g[f"{tag}_codes"])
    assert np.array_equal(tree.child_base, g[f"{tag}_child_base"])
    assert np.array_equal(tree.child_mask, g[f"{tag}_child_mask"])
    assert np.array_equal(tree.parent, g[f"{tag}_parent"])
    # normals bit-exact (signed zeros included)
    assert np.array_equal(tree.normal.view(np.uint64), g[f"{tag}_normal"].view(np.uint64))


@pytest.mark.gpu
def test_build_digests_c1_size(golden, scene_path):
    """SVO depth 8 (C1) and the enclosed variant: sha256 digests of every array."""
    from paper_2405_06997_b200 import scene as S, svo

    g = golden("svo_golden.npz")
    for row in g["digests"]:
        f = str(row).split(",")
        sc = S.load_scene(scene_path(f[0]))
        res, seed = int(f[1]), int(f[2])
        frags = svo.voxelize(sc, res)
        tree = svo.build_from_scene(sc, res, seed=seed)
        codes, perm = svo.sorted_fragments(tree)
        got = [str(len(frags)), str(tree.node_count), _digest(frags.coords), _digest(frags.tris),
               _digest(codes), _digest(perm), _digest(tree.level_off), _digest(tree.codes),
               _digest(tree.child_base), _digest(tree.child_mask), _digest(tree.parent),
               _digest(tree.normal)]
        assert got == f[3:], (f[0], res, seed)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_build_random_fragments_vs_oracle(seed):
    """Random fragment clouds (clustered so leaves and parents need k-means)."""
    from oracle import oracle as O
    from paper_2405_06997_b200 import svo

    rng = np.random.default_rng(seed)
    res = [16, 64, 256][seed]
    n = [500, 20000, 200000][seed]
    centers = rng.integers(0, res, size=(max(4, n // 50), 3))
    coords = np.clip(centers[rng.integers(0, len(centers), n)] + rng.integers(-2, 3, (n, 3)),
                     0, res - 1).astype(np.int64)
    normals = rng.standard_normal((n, 3))
    normals /= np.linalg.norm(normals, axis=1, keepdims=True)
    # some exactly repeated normals (copy shortcuts) and exact opposites
    normals[::7] = normals[0]
    normals[::11] = -normals[0]
    frags = svo.VoxelFragments(coords, normals, np.arange(n))
    tree = svo.build_octree(frags, np.zeros(3), 1.0, res, seed=seed + 5)
    ref = O.build_octree(coords, normals, res, seed=seed + 5)
    for k in ("level_off", "codes", "child_base", "child_mask", "parent"):
        assert np.array_equal(getattr(tree, k), ref[k]), k
    assert np.array_equal(tree.normal.view(np.uint64), ref["normal"].view(np.uint64))


@pytest.mark.gpu
def test_single_fragment_chain_and_full_mask():
    """SPEC.md:197 known answers: one fragment -> depth+1 chain; 8 siblings -> 0xFF."""
    from paper_2405_06997_b200 import svo

    one = svo.VoxelFragments(np.array([[3, 5, 7]]), np.array([[0.0, 0.0, 1.0]]), np.array([0]))
    t = svo.build_octree(one, np.zeros(3), 1.0, 16)
    assert t.node_count == 5 and list(t.parent) == [-1, 0, 1, 2, 3]
    eight = np.array([[x, y, z] for z in (0, 1) for y in (0, 1) for x in (0, 1)])
    t8 = svo.build_octree(svo.VoxelFragments(eight, np.tile([0.0, 1.0, 0.0], (8, 1)),
                                             np.arange(8)), np.zeros(3), 1.0, 2)
    assert int(t8.child_mask[0]) == 0xFF and t8.leaf_count == 8


@pytest.mark.gpu
def test_empty_fragments_rejected():
    from paper_2405_06997_b200 import svo

    with pytest.raises(ValueError):
        svo.build_octree(svo.VoxelFragments(np.zeros((0, 3), dtype=np.int64), np.zeros((0, 3)),
                                            np.zeros(0, dtype=np.int64)), np.zeros(3), 1.0, 16)


@pytest.mark.gpu
def test_dump_format_matches_reference(tmp_path, scene_path):
    """WFPGSVO1 (svo.py:344-397): a device build dumps to the same bytes as the
    reference's dump of the same build; the reference's dump of an exitance
    state loads back and re-dumps byte for byte."""
    import os

    from conftest import GOLDEN
    from paper_2405_06997_b200 import scene as S, svo

    sc = S.load_scene(scene_path("cornell.scene"))
    tree = svo.build_from_scene(sc, 16, seed=0)
    out = tmp_path / "fresh.wfpgsvo"
    tree.dump(str(out))
    ref_fresh = open(os.path.join(GOLDEN, "svo_cornell_r16_fresh.wfpgsvo"), "rb").read()
    assert out.read_bytes() == ref_fresh
    ref_pt = os.path.join(GOLDEN, "svo_cornell_r16_pt.wfpgsvo")
    loaded = svo.SvoCache.load_dump(ref_pt)
    assert loaded.node_count == tree.node_count and loaded.weight_a.sum() > 0
    again = tmp_path / "again.wfpgsvo"
    loaded.dump(str(again))
    assert again.read_bytes() == open(ref_pt, "rb").read()
    # the loaded tree answers queries like the built one (descents, cones)
    pts = sc.bbox_lo + (sc.bbox_hi - sc.bbox_lo) * np.random.default_rng(1).random((500, 3))
    assert np.array_equal(loaded.descend_batch(pts), tree.descend_batch(pts))
    with pytest.raises(ValueError):
        bad = tmp_path / "bad.wfpgsvo"
        bad.write_bytes(b"NOTASVO!" + ref_fresh[8:])
        svo.SvoCache.load_dump(str(bad))
