"""Parity of the device render path against golden vectors from the real
reference (tests/golden/render_golden.npz, fields_golden.npz).

Bit-exact where the reference arithmetic is reproducible (binning, exitance
splat/propagation, CDF tables from given values); tolerance where the
reference's compiled kernels contract FMAs or use libm transcendentals
(intersection t, cone hits, shading) — see oracle/NUMERICS.md.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def R(golden):
    return golden("render_golden.npz")


@pytest.fixture(scope="module")
def F(golden):
    return golden("fields_golden.npz")


def _cfg(R):
    return dict(zip([str(k) for k in R["cfg_keys"]], [int(v) for v in R["cfg_vals"]]))


@pytest.fixture(scope="module")
def setup(R, scene_path):
    from paper_2405_06997_b200 import scene as S, svo

    c = _cfg(R)
    sc = S.load_scene(scene_path("cornell.scene"))
    cam = sc.camera
    sc.camera = S.Camera(cam.position, cam.target, cam.up, cam.vfov_deg, c["W"], c["H"])
    tree = svo.build_from_scene(sc, c["R"], seed=c["svo_seed"])
    return sc, tree, c


def _set_svo_state(tree, R, prefix):
    for k in ("sum_a", "sum_b", "weight_a", "weight_b"):
        setattr(tree, k, R[f"{prefix}_svo_{k}"])
    tree.propagate_up()


def test_intersect_and_occlusion(R, setup):
    sc, _, _ = setup
    t, tri = sc.intersect_batch(R["cone_origins"], R["cone_dirs"])
    assert np.array_equal(tri, R["isect_tri"])
    hit = tri >= 0
    assert np.all(np.isinf(t[~hit]))
    np.testing.assert_allclose(t[hit], R["isect_t"][hit], rtol=1e-12)
    tmax = 0.5 * np.where(np.isfinite(R["isect_t"]), R["isect_t"], 1e3)
    occ = sc.occluded_batch(R["cone_origins"], R["cone_dirs"], tmax)
    assert np.array_equal(occ, R["occ_half"])


def test_propagate_matches_reference_bitwise(R, setup):
    _, tree, _ = setup
    _set_svo_state(tree, R, "p0")
    assert np.array_equal(tree.mean_a.view(np.uint64), R["p0_svo_mean_a"].view(np.uint64))
    assert np.array_equal(tree.mean_b.view(np.uint64), R["p0_svo_mean_b"].view(np.uint64))


@pytest.mark.parametrize("res", [32, 128])
def test_cone_trace(R, setup, res):
    from paper_2405_06997_b200 import backend_cuda

    sc, tree, _ = setup
    _set_svo_state(tree, R, "p0")
    ref = R[f"cone_{res}_rgb"]
    got = backend_cuda.trace_cones_multi(tree, sc, R["cone_origins"], R["cone_dirs"],
                                         float(R[f"cone_{res}_omega"]))
    close = np.all(np.isclose(got, ref, rtol=1e-9, atol=1e-300), axis=1)
    # ulp-level hit-point differences may move a cone across a voxel face
    assert close.mean() >= 0.995, close.mean()


def test_partition_spatial_bitwise(R, setup):
    from paper_2405_06997_b200 import wavefront

    _, tree, c = setup
    for d in range(1, 5):
        if f"p0_d{d}_positions" not in R:
            continue
        pidx = R[f"p0_d{d}_path_idx"]
        pos = R[f"p0_d{d}_positions"]
        bins = wavefront.partition_spatial(tree, pos, pidx, c["l_min"], c["c_ray"])
        assert np.array_equal([b.node for b in bins], R[f"p0_d{d}_bin_nodes"])
        sizes = R[f"p0_d{d}_bin_sizes"]
        assert np.array_equal([len(b.members) for b in bins], sizes)
        if len(bins):
            assert np.array_equal(np.concatenate([b.members for b in bins]),
                                  R[f"p0_d{d}_bin_members"])
    # counters are cleared again
    assert not np.any(tree.counter)


def test_guide_tables_bitwise_from_values(F):
    from paper_2405_06997_b200 import guiding

    for n in (8, 16, 32, 64, 128):
        vals = F[f"vals_{n}"]
        t = guiding.GuideTables(2, n, len(vals))
        t.fill_batch(vals)
        for k in ("marg", "cond", "pdftab", "block_sums", "blk_marg", "blk_cond"):
            a, b = getattr(t, k), F[f"tab_{n}_{k}"]
            assert a.shape == b.shape, (n, k)
            assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), (n, k)


@pytest.fixture(scope="module")
def field_setup(F, scene_path):
    from paper_2405_06997_b200 import scene as S, svo

    sc = S.load_scene(scene_path("cornell.scene"))
    tree = svo.build_from_scene(sc, 64, seed=0)
    for k in ("sum_a", "sum_b", "weight_a", "weight_b"):
        setattr(tree, k, F["svo_" + k])
    tree.propagate_up()
    return sc, tree


@pytest.mark.parametrize("n", [8, 16, 32, 64, 128])
def test_fields_match_reference(F, field_setup, n):
    from paper_2405_06997_b200 import guiding

    sc, tree = field_setup
    got = guiding.generate_fields_batch(tree, sc, F["origins"], n, F["jitters"], blur_sigma=1.0)
    ref = F[f"vals_{n}"]
    assert got.shape == ref.shape
    rel = np.abs(got - ref) / np.maximum(np.abs(ref), 1e-300)
    assert np.mean(rel < 1e-9) >= 0.99, np.mean(rel < 1e-9)
    np.testing.assert_allclose(got.sum(axis=(1, 2)), ref.sum(axis=(1, 2)), rtol=1e-3)


def test_fields_blur_variants(F, field_setup):
    from paper_2405_06997_b200 import guiding

    sc, tree = field_setup
    for sigma, key in ((2.5, "vals_16_s25"), (0.0, "vals_16_s0")):
        got = guiding.generate_fields_batch(tree, sc, F["origins"], 16, F["jitters"],
                                            blur_sigma=sigma)
        rel = np.abs(got - F[key]) / np.maximum(np.abs(F[key]), 1e-300)
        assert np.mean(rel < 1e-9) >= 0.99


def _identical(R, tag, state, diag, tol=1e-5):
    same_depth = state.emit_depth == R[f"{tag}_emit_depth"]
    dpos = np.abs(state.rec_pos - R[f"{tag}_rec_pos"]).max(axis=(1, 2))
    return same_depth & (dpos <= tol * diag)


def _rel(a, b):
    den = np.maximum(np.abs(b), 1e-12)
    return (np.abs(a - b) / den).max(axis=1)


def test_pt_first_pass(R, setup):
    """Sample 0, PT-first (no guiding): per-path records, radiance, SVO deposits."""
    from paper_2405_06997_b200 import wavefront

    sc, tree, c = setup
    for k in ("sum_a", "sum_b", "weight_a", "weight_b"):
        setattr(tree, k, np.zeros_like(R["p0_svo_" + k]))
    tree.propagate_up()
    cfg = wavefront.GuidingConfig(max_depth=c["max_depth"], guided_depths=0,
                                  field_res=c["field_res"], l_min=c["l_min"], c_ray=c["c_ray"],
                                  seed=c["seed"])
    frame, stats = wavefront.render_pass(sc, tree, cfg, [0])
    assert list(stats.bins_per_depth) == list(R["p0_bins_per_depth"])
    assert list(stats.rays_per_depth) == list(R["p0_rays_per_depth"])
    r = wavefront._RUNNERS[next(iter(wavefront._RUNNERS))]
    st = r.state
    ident = _identical(R, "p0", st, sc.diagonal)
    assert ident.mean() >= 0.999, ident.mean()
    rel = _rel(st.radiance, R["p0_radiance"])[ident]
    assert np.mean(rel <= 1e-4) >= 0.995
    np.testing.assert_allclose(frame.sum(), R["p0_frame"].sum(), rtol=1e-6)
    # exitance deposits land in the same leaves with the same weights
    assert np.array_equal(tree.weight_a, R["p0_svo_weight_a"])
    assert np.array_equal(tree.weight_b, R["p0_svo_weight_b"])
    np.testing.assert_allclose(tree.sum_a, R["p0_svo_sum_a"], rtol=1e-9, atol=1e-12)
    # the pass refreshes only the deposited subtrees; a full recompute agrees bitwise
    ma, mb = tree.mean_a, tree.mean_b
    tree.propagate_up()
    assert np.array_equal(ma.view(np.uint64), tree.mean_a.view(np.uint64))
    assert np.array_equal(mb.view(np.uint64), tree.mean_b.view(np.uint64))


@pytest.mark.parametrize("tag,product", [("p1", False), ("p1x", True)])
def test_guided_pass(R, setup, tag, product):
    """Sample 1 guided from the reference's PT-first SVO state."""
    from paper_2405_06997_b200 import wavefront

    sc, tree, c = setup
    _set_svo_state(tree, R, "p0")
    cfg = wavefront.GuidingConfig(max_depth=c["max_depth"], guided_depths=c["max_depth"],
                                  field_res=c["field_res"], l_min=c["l_min"], c_ray=c["c_ray"],
                                  seed=c["seed"], product=product)
    frame, stats = wavefront.render_pass(sc, tree, cfg, [1])
    ref_bins = list(R[f"{tag}_bins_per_depth"])
    assert list(stats.bins_per_depth)[:1] == ref_bins[:1]
    r = wavefront._RUNNERS[next(iter(wavefront._RUNNERS))]
    st = r.state
    ident = _identical(R, tag, st, sc.diagonal)
    assert ident.mean() >= 0.98, ident.mean()
    rel = _rel(st.radiance, R[f"{tag}_radiance"])[ident]
    assert np.mean(rel <= 1e-4) >= 0.99
    np.testing.assert_allclose(frame.mean(), R[f"{tag}_frame"].mean(), rtol=0.05)


def test_graph_replay_matches_eager(R, setup):
    """Passes replayed from a captured CUDA graph are bitwise identical to
    eagerly enqueued passes (same SVO learning sequence)."""
    from paper_2405_06997_b200 import wavefront

    sc, tree, c = setup
    cfg = wavefront.GuidingConfig(max_depth=c["max_depth"], guided_depths=c["max_depth"],
                                  field_res=c["field_res"], l_min=c["l_min"], c_ray=c["c_ray"],
                                  seed=c["seed"])
    results = []
    for graph in (False, True):
        _set_svo_state(tree, R, "p0")
        r = wavefront.PassRunner(sc, tree, cfg, use_graph=graph)
        frames = []
        for sample in range(1, 6):  # eager, capture, then three replays
            r.launch(sample)
            frames.append(r.frame.cpu().numpy().copy())
        results.append((frames, tree.mean_a, tree.sum_b))
    (fe, ma_e, sb_e), (fg, ma_g, sb_g) = results
    for a, b in zip(fe, fg):
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    assert np.array_equal(ma_e.view(np.uint64), ma_g.view(np.uint64))
    assert np.array_equal(sb_e.view(np.uint64), sb_g.view(np.uint64))


def test_frame_pipeline_matches_render_pass(R, setup):
    """FramePipeline (two alternating runners, overlapped frame copies) gives
    the same frames and the same SVO learning sequence as render_pass."""
    from paper_2405_06997_b200 import wavefront

    sc, tree, c = setup
    cfg = wavefront.GuidingConfig(max_depth=c["max_depth"], guided_depths=c["max_depth"],
                                  field_res=c["field_res"], l_min=c["l_min"], c_ray=c["c_ray"],
                                  seed=c["seed"])
    _set_svo_state(tree, R, "p0")
    ref = [wavefront.render_pass(sc, tree, cfg, [s])[0].copy() for s in range(1, 6)]
    ref_mean = tree.mean_a
    _set_svo_state(tree, R, "p0")
    pipe = wavefront.FramePipeline(sc, tree, cfg, want_stats=True)
    got = [(s, f.copy(), st) for s, f, st in pipe.run(range(1, 6))]
    assert [s for s, _, _ in got] == [1, 2, 3, 4, 5]
    for (_, f, st), r in zip(got, ref):
        assert np.array_equal(f.view(np.uint64), r.view(np.uint64))
        assert st.bins_per_depth
    assert np.array_equal(tree.mean_a.view(np.uint64), ref_mean.view(np.uint64))


@pytest.mark.gpu
@pytest.mark.parametrize("res,l_min,c_ray", [(256, 5, 512), (256, 3, 16), (1024, 5, 512)])
def test_partition_matches_oracle_at_scale(scene_path, res, l_min, c_ray):
    """Alg. 2 on the device (incl. the dense top-index start when l_min is
    deep enough) against the CPU oracle, 200k hit points on the Cornell walls."""
    from oracle import render as OR
    from paper_2405_06997_b200 import scene as S, svo, wavefront

    sc0 = S.load_scene(scene_path("cornell.scene"))
    tree = svo.build_from_scene(sc0, res, seed=0)
    osc = OR.Scene(sc0)
    built = {k: getattr(tree, k) for k in ("level_off", "codes", "child_base", "child_mask",
                                           "parent", "normal")}
    osvo = OR.Svo(built, tree.cube_lo, tree.cube_size, tree.resolution)
    rng = np.random.default_rng(res + l_min)
    o = np.tile(sc0.camera.position, (200000, 1))
    d = rng.standard_normal((200000, 3))
    d[:, 2] = np.abs(d[:, 2]) + 0.5
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    t, tri = OR.intersect(osc, o, d)
    pos = (o + t[:, None] * d)[tri >= 0]
    nodes, members = OR.partition(osvo, pos, l_min, c_ray)
    bins = wavefront.partition_spatial(tree, pos, np.arange(len(pos)), l_min, c_ray)
    assert [b.node for b in bins] == list(nodes)
    assert all(np.array_equal(b.members, m) for b, m in zip(bins, members))


@pytest.mark.gpu
@pytest.mark.parametrize("product", [False, True])
def test_pass_pipeline_equals_sequential_passes(golden, scene_path, product):
    """wavefront.PassPipeline (two runners on two streams, pass i+1's start
    overlapping pass i's end, CUDA graphs captured and replayed) renders
    exactly what sequential render_pass calls render: frames and SVO arrays
    bit for bit (the overlap events keep every SVO access in pass order)."""
    import torch

    from paper_2405_06997_b200 import scene as S, svo, wavefront

    sc = S.load_scene(scene_path("cornell.scene"))
    cam = sc.camera
    sc.camera = S.Camera(cam.position, cam.target, cam.up, cam.vfov_deg, 96, 64)
    base = dict(max_depth=4, field_res=32, l_min=3, c_ray=16, seed=3, product=product)
    pt = wavefront.GuidingConfig(guided_depths=0, **base)
    g = wavefront.GuidingConfig(guided_depths=4, **base)
    seq = svo.build_from_scene(sc, 64, seed=0)
    wavefront.render_pass(sc, seq, pt, [0])
    want = [wavefront.render_pass(sc, seq, g, [s])[0].copy() for s in range(1, 9)]
    par = svo.build_from_scene(sc, 64, seed=0)
    wavefront.render_pass(sc, par, pt, [0])
    pipe = wavefront.PassPipeline(sc, par, g)
    got = []
    for s in range(1, 9):
        _, r = pipe.launch(s)
        with torch.cuda.stream(pipe.streams[(s - 1) % 2]):
            got.append(r.frame.clone())
    pipe.join()
    torch.cuda.synchronize()
    for s in range(8):
        np.testing.assert_array_equal(got[s].cpu().numpy().reshape(want[s].shape), want[s])
    for k in ("sum_a", "sum_b", "weight_a", "weight_b", "mean_a", "mean_b"):
        assert np.array_equal(getattr(par, k).view(np.uint64), getattr(seq, k).view(np.uint64)), k
