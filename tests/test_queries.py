"""Direct parity of helpers the render loop uses implicitly, against the
reference's own outputs (tests/golden/queries_golden.npz, make_golden.py
gen_queries): descend_tracked's (node, present, deepest) triple
(_kernelshim.py:60-71 -> _kernels.pyx:591-658), SvoCache.ancestor_chain
(svo.py:326-340), PassStats.material_groups
(wavefront.py:88-95,250-253), and the atomic splat variant of
accumulate_batch (svo.py:254-263) against the deterministic one."""

import numpy as np
import pytest


def _dense(groups, shape):
    out = np.zeros(shape, dtype=np.int64)
    for d, g in enumerate(groups):
        for m, k in g.items():
            out[d, m] = k
    return out


def test_oracle_descend_matches_reference(golden, scene_path):
    """CPU: the oracle's descent (the checker the render tests rely on)."""
    from oracle import render as OR
    from paper_2405_06997_b200 import scene as S

    Q = golden("queries_golden.npz")
    sc = S.load_scene(scene_path("cornell.scene"))
    svo = OR.Svo.from_scene(sc, 64, 0)
    node, present = svo.descend(Q["desc_points"])
    assert np.array_equal(present, Q["desc_present"])
    assert np.array_equal(node, Q["desc_node"])


def test_oracle_ancestor_chain_matches_reference(golden, scene_path):
    """CPU: a Morton-prefix walk over the oracle's arrays gives the
    reference's chains (root first, stops at the first absent octant)."""
    from oracle import render as OR
    from paper_2405_06997_b200 import scene as S

    Q = golden("queries_golden.npz")
    sc = S.load_scene(scene_path("cornell.scene"))
    svo = OR.Svo.from_scene(sc, 64, 0)
    flat = Q["chain_flat"]
    off = np.concatenate([[0], np.cumsum(Q["chain_len"])])
    for k, (x, y, z) in enumerate(Q["chain_coords"]):
        node, chain = 0, [0]
        for level in range(1, svo.depth + 1):
            sh = svo.depth - level
            o = ((x >> sh) & 1) | (((y >> sh) & 1) << 1) | (((z >> sh) & 1) << 2)
            m = int(svo.child_mask[node])
            if not (m >> o) & 1:
                break
            node = int(svo.child_base[node]) + bin(m & ((1 << o) - 1)).count("1")
            chain.append(node)
        assert chain == list(flat[off[k]:off[k + 1]]), k


@pytest.mark.gpu
def test_descend_tracked_matches_reference(golden, scene_path):
    from paper_2405_06997_b200 import backend_cuda, scene as S, svo

    Q = golden("queries_golden.npz")
    sc = S.load_scene(scene_path("cornell.scene"))
    tree = svo.build_from_scene(sc, 64, seed=0)
    node, present, deepest = backend_cuda.descend_tracked(tree, Q["desc_points"])
    assert np.array_equal(present, Q["desc_present"])
    assert np.array_equal(node, Q["desc_node"])
    assert np.array_equal(deepest, Q["desc_deepest"])
    leaves = backend_cuda.descend_leaves(tree, Q["desc_points"])
    assert np.array_equal(leaves, np.where(Q["desc_present"], Q["desc_node"], -1))


@pytest.mark.gpu
def test_ancestor_chain_matches_reference(golden, scene_path):
    from paper_2405_06997_b200 import scene as S, svo

    Q = golden("queries_golden.npz")
    sc = S.load_scene(scene_path("cornell.scene"))
    tree = svo.build_from_scene(sc, 64, seed=0)
    flat = Q["chain_flat"]
    off = np.concatenate([[0], np.cumsum(Q["chain_len"])])
    for k, cc in enumerate(Q["chain_coords"]):
        assert tree.ancestor_chain(cc) == list(flat[off[k]:off[k + 1]]), k
    # SPEC.md:227 known answer: the root is always the chain's first node
    assert tree.ancestor_chain((0, 0, 0))[0] == 0
    with pytest.raises(ValueError):
        tree.ancestor_chain((-1, 0, 0))


@pytest.mark.gpu
def test_material_groups_match_reference(golden, scene_path):
    from paper_2405_06997_b200 import scene as S, svo, wavefront

    Q = golden("queries_golden.npz")
    R = golden("render_golden.npz")
    c = dict(zip([str(k) for k in R["cfg_keys"]], [int(v) for v in R["cfg_vals"]]))
    base = dict(max_depth=c["max_depth"], field_res=c["field_res"], l_min=c["l_min"],
                c_ray=c["c_ray"], seed=c["seed"])
    sc = S.load_scene(scene_path("cornell.scene"))
    cam = sc.camera
    sc.camera = S.Camera(cam.position, cam.target, cam.up, cam.vfov_deg, c["W"], c["H"])
    tree = svo.build_from_scene(sc, c["R"], seed=c["svo_seed"])
    for tag, g, sample in (("p0", 0, 0), ("p1", c["max_depth"], 1)):
        _, st = wavefront.render_pass(sc, tree, wavefront.GuidingConfig(guided_depths=g, **base),
                                      [sample])
        want = Q[tag + "_mat_groups"]
        assert np.array_equal(_dense(st.material_groups, want.shape), want), tag
    sc.camera = S.Camera(cam.position, cam.target, cam.up, cam.vfov_deg, 48, 40)
    tree2 = svo.build_from_scene(sc, 64, seed=0)
    _, st = wavefront.render_pass(sc, tree2, wavefront.GuidingConfig(guided_depths=0, **base),
                                  [0])
    want = Q["w48_mat_groups"]
    assert np.array_equal(_dense(st.material_groups, want.shape), want)


@pytest.mark.gpu
def test_atomic_splat_matches_ordered_splat(golden, scene_path):
    """accumulate_batch with fp64 atomics (the north star's 'atomic splat',
    wfpg_svo_accumulate deterministic=0) vs the np.add.at-ordered splat:
    weights are counts (bitwise), sums agree to fp reassociation."""
    from paper_2405_06997_b200 import scene as S, svo

    sc = S.load_scene(scene_path("cornell.scene"))
    a = svo.build_from_scene(sc, 64, seed=0)
    b = svo.build_from_scene(sc, 64, seed=0)
    lo, hi = a.level_off[a.depth], a.level_off[a.depth + 1]
    rng = np.random.default_rng(5)
    m = 200_000  # heavy contention: ~8 deposits per leaf
    leaf = rng.integers(lo, hi, m)
    dirs = rng.standard_normal((m, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    rad = rng.random((m, 3)) * 10.0
    a.accumulate_batch(leaf, dirs, rad, deterministic=True)
    b.accumulate_batch(leaf, dirs, rad, deterministic=False)
    for k in ("weight_a", "weight_b"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
    for k in ("sum_a", "sum_b"):
        np.testing.assert_allclose(getattr(b, k), getattr(a, k), rtol=1e-12, atol=1e-12)
    a.propagate_up()
    b.propagate_up()
    np.testing.assert_allclose(b.mean_a, a.mean_a, rtol=1e-11, atol=1e-12)
