"""Command line, Eq. 7 accumulation, image files and collect_bin_image
 against the reference's own outputs
(tests/golden/cli_golden.npz, made by make_golden.py cli)."""

import json
import os

import numpy as np
import pytest

from paper_2405_06997_b200 import cli, imageio


@pytest.fixture(scope="module")
def G(golden):
    return golden("cli_golden.npz")


def test_run_config_validation_and_json():
    c = cli.RunConfig("x.scene")
    assert (c.mode, c.spp, c.depth, c.guided_depths, c.field_res, c.lmin, c.cray, c.svo_res,
            c.heuristic) == ("wfpg", 8, 5, 4, 128, 5, 512, 256, "pt-first")
    assert cli.RunConfig.from_json(c.to_json()) == c
    assert cli.RunConfig("x.scene", "pt", 3).spp == 3  # positional order of the reference
    bad = [dict(mode="bdpt"), dict(spp=0), dict(depth=0), dict(guided_depths=6),
           dict(svo_res=100), dict(field_res=48), dict(heuristic="nope"), dict(cray=0)]
    msgs = ["mode must be one of", "spp must be >= 1", "depth must be >= 1",
            "guided-depths must be within [0, depth]", "svo-res must be a power of two",
            "field-res must be one of 16, 32, 64, 128", "unknown heuristic 'nope'",
            "cray must be >= 1"]
    for kw, msg in zip(bad, msgs):
        with pytest.raises(ValueError, match=msg.replace("[", r"\[").replace("]", r"\]")):
            cli.RunConfig("x.scene", **kw)
    assert cli.RunConfig("x.scene", svo_res=2048).svo_res == 2048  # B200 superset
    assert c.effective_lmin(4) == 3 and c.effective_lmin(10) == 5


def test_config_json_matches_reference(G):
    for tag in ("pt", "wfpg", "prod"):
        ref = json.loads(str(G[f"cli_{tag}_config"]))
        mine = cli.RunConfig.from_json(json.dumps(ref))
        assert json.loads(mine.to_json()) == ref


def test_argument_parsing():
    c = cli.config_from_args(["--scene", "s.scene", "--mode", "pt", "--spp", "4", "--depth", "3",
                              "--guided-depths", "9", "--dump-field", "3,4", "--rr"])
    assert (c.mode, c.spp, c.depth, c.guided_depths, c.dump_field, c.rr) == \
        ("pt", 4, 3, 3, (3, 4), True)
    with pytest.raises(ValueError, match="--dump-field expects X,Y"):
        cli.config_from_args(["--scene", "s", "--dump-field", "3"])
    assert cli.main(["--scene", "s", "--spp", "0"]) == 2
    assert cli.main(["--scene", "/nonexistent.scene"]) == 1


def test_bin_false_color():
    img = np.array([[-1, 7], [7, 123456789]])
    rgb = cli._bin_false_color(img)
    assert np.all(rgb[0, 0] == 0.0)
    assert np.array_equal(rgb[0, 1], rgb[1, 0])
    assert np.all((rgb[0, 1] >= 0.15) & (rgb[0, 1] <= 1.0))
    assert not np.array_equal(rgb[0, 1], rgb[1, 1])


def test_image_files_roundtrip(tmp_path):
    rng = np.random.default_rng(0)
    f = rng.random((5, 7, 3)) * 4
    imageio.write_pfm(tmp_path / "a.pfm", f)
    raw = (tmp_path / "a.pfm").read_bytes()
    assert raw.startswith(b"PF\n7 5\n-1.0\n") and len(raw) == 12 + 5 * 7 * 3 * 4
    # bottom row first, little-endian float32
    first = np.frombuffer(raw[12:24], dtype="<f4")
    assert np.array_equal(first, f[-1, 0].astype(np.float32))
    back = imageio.read_pfm(tmp_path / "a.pfm")
    assert np.array_equal(back, f.astype(np.float32).astype(np.float64))
    imageio.write_png(tmp_path / "a.png", f)
    from PIL import Image

    px = np.asarray(Image.open(tmp_path / "a.png"))
    assert np.array_equal(px, np.clip(f / (1 + f) * 255 + 0.5, 0, 255).astype(np.uint8))


def test_metrics():
    from paper_2405_06997_b200 import accumulation as A

    a = np.full((2, 2, 3), 1.0)
    b = np.full((2, 2, 3), 3.0)
    assert A.mse(a, b) == pytest.approx((0.5 - 0.75) ** 2)
    assert A.mean_abs_diff(a, b) == pytest.approx(0.25)
    assert A.rel_mse(a, b) == pytest.approx(4.0 / 9.01)
    assert [A.HEURISTICS[h](i) for h in ("linear", "quadratic", "one-two", "discard-first")
            for i in (1, 3, 9)] == [1, 3, 5, 1, 9, 25, 1, 2, 2, 0, 1, 1]
    with pytest.raises(ValueError):
        A.mse(a, np.zeros((1, 2, 3)))


# ---------------------------------------------------------------------------
@pytest.mark.gpu
def test_accumulation_buffer_bitwise():
    from paper_2405_06997_b200 import _dev, accumulation as A

    rng = np.random.default_rng(3)
    frames = [rng.random((4, 5, 3)) for _ in range(6)]
    buf = A.AccumulationBuffer(4, 5, "linear")
    ws, w = np.zeros((4, 5, 3)), 0.0
    for i, f in enumerate(frames, start=1):
        (buf.add_sample(f, i) if i % 2 else buf.add_sample(_dev.upload(f), i))
        hw = 1.0 * A.HEURISTICS["linear"](i)
        ws += hw * f
        w += hw
    assert np.array_equal(buf.resolve().view(np.uint64), (ws / w).view(np.uint64))
    bad = frames[0].copy()
    bad[1, 1, 1] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        buf.add_sample(bad)
    # the rejected frame left the running sums untouched (the reference raises
    # before touching weighted_sum)
    assert np.array_equal(buf.resolve().view(np.uint64), (ws / w).view(np.uint64))


@pytest.mark.gpu
def test_collect_bin_image_matches_reference(G, golden, scene_path):
    from paper_2405_06997_b200 import scene as S, svo, wavefront

    R = golden("render_golden.npz")
    c = dict(zip([str(k) for k in R["cfg_keys"]], [int(v) for v in R["cfg_vals"]]))
    sc = S.load_scene(scene_path("cornell.scene"))
    cam = sc.camera
    sc.camera = S.Camera(cam.position, cam.target, cam.up, cam.vfov_deg, c["W"], c["H"])
    tree = svo.build_from_scene(sc, c["R"], seed=c["svo_seed"])
    cfg = wavefront.GuidingConfig(max_depth=c["max_depth"], guided_depths=0,
                                  field_res=c["field_res"], l_min=c["l_min"], c_ray=c["c_ray"],
                                  seed=c["seed"])
    for tag, samples in (("bins1", [0]), ("bins2", [0, 1])):
        frame, st, img = wavefront.render_pass(sc, tree, cfg, samples, collect_bin_image=True)
        assert list(st.bins_per_depth) == list(G[tag + "_bins_per_depth"])
        assert np.array_equal(img, G[tag + "_image"]), tag
        np.testing.assert_allclose(frame, G[tag + "_frame"], rtol=1e-6, atol=1e-9)


@pytest.mark.gpu
@pytest.mark.parametrize("tag,kw", [
    ("pt", dict(mode="pt", spp=2)),
    ("wfpg", dict(mode="wfpg", spp=3, depth=4, svo_res=64, field_res=32, lmin=3, cray=16,
                  seed=5)),
    ("prod", dict(mode="wfpg-product", spp=2, depth=3, guided_depths=3, svo_res=32,
                  field_res=16, lmin=2, cray=8, seed=1, heuristic="linear"))])
def test_cli_run_matches_reference(G, scene_path, tmp_path, tag, kw):
    conf = cli.RunConfig(scene_path("cornell.scene"), out=str(tmp_path / f"{tag}.pfm"), **kw)
    logs = []
    status, frame = cli.run(conf, log=logs.append)
    assert status == 0
    ref = G[f"cli_{tag}_frame"]
    assert frame.shape == ref.shape
    for ext in (".pfm", ".png"):
        assert os.path.exists(tmp_path / f"{tag}{ext}")
    assert np.array_equal(imageio.read_pfm(tmp_path / f"{tag}.pfm"),
                          frame.astype(np.float32).astype(np.float64))
    rel = np.abs(frame - ref) / np.maximum(np.abs(ref), 1e-12)
    if tag == "pt":  # unguided: every pixel is the same paths
        assert np.mean(rel <= 1e-4) >= 0.995
    else:  # guided: SVO learning between passes amplifies ulp differences
        np.testing.assert_allclose(frame.mean(), ref.mean(), rtol=0.05)
        got = [ln for ln in logs if ln.startswith("sample ")]
        want = [str(x) for x in G[f"cli_{tag}_log"]]
        assert len(got) == len(want)
        # the first pass (and its bins) is identical
        assert got[0] == want[0]


@pytest.mark.gpu
def test_two_sample_guided_pass_matches_reference(G, golden, scene_path):
    """render_pass over consecutive samples [1, 2] with guiding: bins pool both
    samples' paths and bin streams use the first index (wavefront.py:249)."""
    from paper_2405_06997_b200 import scene as S, svo, wavefront

    R = golden("render_golden.npz")
    c = dict(zip([str(k) for k in R["cfg_keys"]], [int(v) for v in R["cfg_vals"]]))
    sc = S.load_scene(scene_path("cornell.scene"))
    cam = sc.camera
    sc.camera = S.Camera(cam.position, cam.target, cam.up, cam.vfov_deg, c["W"], c["H"])
    tree = svo.build_from_scene(sc, c["R"], seed=c["svo_seed"])
    for k in ("sum_a", "sum_b", "weight_a", "weight_b"):
        setattr(tree, k, G["multi_pre_" + k])
    tree.propagate_up()
    cfg = wavefront.GuidingConfig(max_depth=c["max_depth"], guided_depths=c["max_depth"],
                                  field_res=c["field_res"], l_min=c["l_min"], c_ray=c["c_ray"],
                                  seed=c["seed"])
    frame, st = wavefront.render_pass(sc, tree, cfg, [1, 2])
    assert list(st.bins_per_depth)[:1] == list(G["multi_bins_per_depth"])[:1]
    state = wavefront._RUNNERS[next(iter(wavefront._RUNNERS))].state
    assert state.n == 2 * c["W"] * c["H"]
    same = state.emit_depth == G["multi_emit_depth"]
    same &= np.abs(state.rec_pos - G["multi_rec_pos"]).max(axis=(1, 2)) <= 1e-5 * sc.diagonal
    assert same.mean() >= 0.98, same.mean()
    np.testing.assert_allclose(frame.mean(), G["multi_frame"].mean(), rtol=0.05)
