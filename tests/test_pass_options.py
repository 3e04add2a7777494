"""Pass options that must not change what a pass computes: skipping the
Alg. 2 binning of non-guided depths (wfpg_pass_config.skip_unguided_bins;
the reference bins every depth only to report PassStats, wavefront.py:
240-256) leaves the frame and the learned SVO bit-identical."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("guided", [0, 1, 2])
def test_skip_unguided_bins_same_frames_and_svo(golden, scene_path, guided):
    from paper_2405_06997_b200 import scene as S, svo, wavefront

    R = golden("render_golden.npz")
    c = dict(zip([str(k) for k in R["cfg_keys"]], [int(v) for v in R["cfg_vals"]]))
    sc = S.load_scene(scene_path("cornell.scene"))
    cam = sc.camera
    sc.camera = S.Camera(cam.position, cam.target, cam.up, cam.vfov_deg, c["W"], c["H"])
    cfg = wavefront.GuidingConfig(max_depth=c["max_depth"], guided_depths=guided,
                                  field_res=c["field_res"], l_min=c["l_min"], c_ray=c["c_ray"],
                                  seed=c["seed"])
    out = []
    for skip in (False, True):
        tree = svo.build_from_scene(sc, c["R"], seed=c["svo_seed"])
        r = wavefront.PassRunner(sc, tree, cfg, skip_unguided_bins=skip)
        frames = []
        for s in range(3):  # the SVO learns between passes
            r.launch(s, want_stats=True)
            frames.append(r.frame.cpu().numpy().copy())
        stats = r.pass_stats()
        out.append((frames, tree.mean_a.copy(), tree.mean_b.copy(), stats))
    (fa, ma, mba, sa), (fb, mb, mbb, sb) = out
    for x, y in zip(fa, fb):
        assert np.array_equal(x.view(np.uint64), y.view(np.uint64))
    assert np.array_equal(ma.view(np.uint64), mb.view(np.uint64))
    assert np.array_equal(mba.view(np.uint64), mbb.view(np.uint64))
    # the guided depths' bins are reported either way; the others only without skipping
    g = guided
    assert list(sa.bins_per_depth)[:g] == list(sb.bins_per_depth)[:g]
    assert all(b > 0 for b in list(sa.bins_per_depth)[g:])
    assert all(b == 0 for b in list(sb.bins_per_depth)[g:])
