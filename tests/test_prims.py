"""Device primitives the hot path is built on: the stable LSD radix sort
(csrc/prims.cu: chunked 9-bit-digit passes) against numpy's stable argsort,
and the two path-record layouts of the exitance update (wfpg_paths.
rec_depth_major) against each other."""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,bits", [(1, 8), (2, 1), (1000, 8), (5000, 9), (4097, 17),
                                    (70_000, 24), (300_000, 27), (1_000_003, 33),
                                    (1_300_000, 36), (9000, 63), (9000, 64)])
def test_sort_pairs_u64_matches_stable_argsort(n, bits):
    from paper_2405_06997_b200 import _dev, _lib

    rng = np.random.default_rng(n + bits)
    hi = (1 << bits) - 1 if bits < 64 else np.iinfo(np.uint64).max
    # clustered keys (few distinct high digits, many equal keys) and random low bits
    keys = rng.integers(0, max(2, hi // 3), size=n, dtype=np.uint64, endpoint=False)
    keys[::7] = keys[0]
    if bits < 64:
        keys &= np.uint64(hi)
    vals = np.arange(n, dtype=np.uint32)
    dk, dv = _dev.upload(keys.view(np.int64)), _dev.upload(vals.view(np.int32))
    ws = _dev.workspace(_lib.load().wfpg_sort_workspace_bytes(n))
    _lib.call("wfpg_sort_pairs_u64", _lib.ptr(dk), _lib.ptr(dv), n, None, bits, _lib.ptr(ws),
              ws.numel(), _dev.stream())
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(_dev.download(dk).view(np.uint64), keys[order])
    assert np.array_equal(_dev.download(dv).view(np.uint32), vals[order])


def test_sort_pairs_device_count():
    """Only the first *n_dev items are sorted; the rest stay untouched."""
    from paper_2405_06997_b200 import _dev, _lib

    n_max, n = 50_000, 31_337
    rng = np.random.default_rng(5)
    keys = rng.integers(0, 1 << 30, size=n_max, dtype=np.uint64)
    vals = np.arange(n_max, dtype=np.uint32)
    dk, dv = _dev.upload(keys.view(np.int64)), _dev.upload(vals.view(np.int32))
    cnt = _dev.upload(np.array([n], dtype=np.int32))
    ws = _dev.workspace(_lib.load().wfpg_sort_workspace_bytes(n_max))
    _lib.call("wfpg_sort_pairs_u64", _lib.ptr(dk), _lib.ptr(dv), n_max, _lib.ptr(cnt), 30,
              _lib.ptr(ws), ws.numel(), _dev.stream())
    order = np.argsort(keys[:n], kind="stable")
    got_k, got_v = _dev.download(dk).view(np.uint64), _dev.download(dv).view(np.uint32)
    assert np.array_equal(got_k[:n], keys[:n][order])
    assert np.array_equal(got_v[:n], vals[:n][order])
    assert np.array_equal(got_k[n:], keys[n:]) and np.array_equal(got_v[n:], vals[n:])


def test_exitance_update_record_layouts_agree(golden, scene_path):
    """The same records in the reference's (P, D+1, 3) layout and in the
    device-major (D+1, P, 3) layout give bit-identical SVO updates."""
    from paper_2405_06997_b200 import _dev, _lib, scene as S, svo, wavefront

    R = golden("render_golden.npz")
    c = dict(zip([str(k) for k in R["cfg_keys"]], [int(v) for v in R["cfg_vals"]]))
    sc = S.load_scene(scene_path("cornell.scene"))
    cam = sc.camera
    sc.camera = S.Camera(cam.position, cam.target, cam.up, cam.vfov_deg, c["W"], c["H"])
    cfg = wavefront.GuidingConfig(max_depth=c["max_depth"], guided_depths=0,
                                  field_res=c["field_res"], l_min=c["l_min"], c_ray=c["c_ray"],
                                  seed=c["seed"])
    trees = [svo.build_from_scene(sc, c["R"], seed=c["svo_seed"]) for _ in range(2)]
    wavefront.render_pass(sc, trees[0], cfg, [0])
    st = wavefront._RUNNERS[next(iter(wavefront._RUNNERS))].state
    rec_pos, rec_T = st.rec_pos, st.rec_T  # (P, D+1, 3), masked by n_rec
    # path-major copy through the C ABI (rec_depth_major = 0)
    p = st.abi()
    keep = {"rec_pos": _dev.upload(np.ascontiguousarray(rec_pos)),
            "rec_T": _dev.upload(np.ascontiguousarray(rec_T))}
    p.rec_pos, p.rec_T = keep["rec_pos"].data_ptr(), keep["rec_T"].data_ptr()
    p.rec_depth_major, p.n_rec = 0, None
    ws = _dev.workspace(_lib.load().wfpg_update_exitance_workspace_bytes(st.n, st.max_depth))
    s1 = trees[1].abi()
    _lib.call("wfpg_update_exitance", C.byref(s1), C.byref(p), 1, None, _lib.ptr(ws),
              ws.numel(), _dev.stream())
    for k in ("sum_a", "sum_b", "weight_a", "weight_b", "mean_a", "mean_b"):
        a, b = getattr(trees[0], k), getattr(trees[1], k)
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), k
    assert trees[0].weight_a.sum() + trees[0].weight_b.sum() > 0
