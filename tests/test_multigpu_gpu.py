"""Multi-GPU data path on ONE GPU without collectives (the ranks are run one
after the other in one process; nothing waits on another kernel): pixel
bands with deposit export + rank-ordered splat reproduce the single-GPU pass
and SVO update bit for bit (PT pass: binning cannot change the paths)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 3])
def test_banded_pass_with_deposit_exchange_equals_one_gpu(golden, scene_path, world):
    import torch

    from paper_2405_06997_b200 import multigpu, scene as S, svo, wavefront

    R = golden("render_golden.npz")
    c = dict(zip([str(k) for k in R["cfg_keys"]], [int(v) for v in R["cfg_vals"]]))
    sc = S.load_scene(scene_path("cornell.scene"))
    cam = sc.camera
    sc.camera = S.Camera(cam.position, cam.target, cam.up, cam.vfov_deg, c["W"], c["H"])
    cfg = wavefront.GuidingConfig(max_depth=c["max_depth"], guided_depths=0,
                                  field_res=c["field_res"], l_min=c["l_min"], c_ray=c["c_ray"],
                                  seed=c["seed"])
    one = svo.build_from_scene(sc, c["R"], seed=c["svo_seed"])
    frame1, st1 = wavefront.render_pass(sc, one, cfg, [0])
    multi = svo.build_from_scene(sc, c["R"], seed=c["svo_seed"])
    ex = multigpu.DepositExchange(multi)
    lists, frames = [], []
    for r in range(world):
        off, npx = multigpu.band(c["W"] * c["H"], r, world)
        run = wavefront.PassRunner(sc, multi, cfg, pixel_offset=off, n_pixels=npx,
                                   deposit_sink=ex, use_graph=False)
        run.launch(0)
        frames.append(run.frame.cpu().numpy().copy())
        lists.append(tuple(t.clone() for t in ex.local()))
    # SVO untouched by the exporting passes
    assert not np.any(multi.weight_a) and not np.any(multi.weight_b)
    leaf, dirs, rad = (torch.cat([l[k] for l in lists]) for k in range(3))
    n = ex.apply(leaf, dirs, rad)
    assert n == st1.deposits
    np.testing.assert_array_equal(np.concatenate(frames).reshape(frame1.shape), frame1)
    for k in ("sum_a", "sum_b", "weight_a", "weight_b", "mean_a", "mean_b"):
        a, b = getattr(multi, k), getattr(one, k)
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), k
