"""The reference's backend API (backend.py / _kernelshim.py) on the B200.

``NAME``, ``COMPILED`` and the eight kernel entry points with the signatures
and return contracts of wfpg._kernelshim (numpy in, numpy out), each one
C-ABI call into libwfpg_b200.so.  The module is installable INTO THE
REFERENCE with ``wfpg.backend.set_backend(paper_2405_06997_b200.backend_cuda)``
(backend.py:25-28): every entry point accepts the reference's own objects —
its numpy ``Scene`` / ``Camera`` / ``SvoCache`` / ``PathState`` /
``GuideTables`` — as well as this package's device-resident ones.

Reference objects are adapted on first use and cached per object (weakly):
the scene arrays (bit-for-bit, including the fp64 normals and the host BVH)
and the SVO structure are uploaded once; the SVO's mutable means are
re-uploaded by the calls that read them (the reference refreshes them on the
host between passes); ``shade_depth`` uploads the PathState, shades on the
device and writes every mutated array back into the caller's numpy arrays
in place, as the compiled kernel does.  This package's own render path never
goes through these numpy wrappers: render_pass keeps every array on the
device.
"""

import ctypes as C
import weakref

import numpy as np

from . import _dev, _lib
from . import scene as _S
from . import svo as _V

NAME = "cuda-sm100a"
COMPILED = True

_SCENES = weakref.WeakKeyDictionary()
_SVOS = weakref.WeakKeyDictionary()


def _f64(a, cols=3):
    return _dev.upload(np.ascontiguousarray(np.atleast_2d(a), dtype=np.float64).reshape(-1, cols))


# ---------------------------------------------------------------------------
# adapters for the reference's objects
# ---------------------------------------------------------------------------
def _scene(scene):
    """This package's Scene for `scene` (itself, or the cached adapter of a
    reference Scene: same arrays bit for bit, same host BVH)."""
    if isinstance(scene, _S.Scene):
        return scene
    ad = _SCENES.get(scene)
    if ad is None or ad._src_v0 is not scene.v0:
        ad = _S.Scene.from_arrays(scene)
        ad._src_v0 = scene.v0
        _SCENES[scene] = ad
    return ad


def _svo(svo, means=False):
    """This package's SvoCache for `svo`; for a reference SvoCache the cached
    device copy of its structure, with mean_a / mean_b re-uploaded when the
    caller reads them (means=True)."""
    if isinstance(svo, _V.SvoCache):
        return svo
    ad = _SVOS.get(svo)
    if ad is None or ad._src_codes is not svo.codes:
        ad = _V.SvoCache.from_arrays(svo)
        ad._src_codes = svo.codes
        _SVOS[svo] = ad
    elif means:
        ad.mean_a = svo.mean_a
        ad.mean_b = svo.mean_b
    return ad


def _camera_abi(camera):
    if hasattr(camera, "as_abi"):
        return camera.as_abi()
    c = _lib.Camera()
    c.position[:] = np.asarray(camera.position, dtype=np.float64).tolist()
    c.forward[:] = np.asarray(camera.forward, dtype=np.float64).tolist()
    c.right[:] = np.asarray(camera.right, dtype=np.float64).tolist()
    c.up[:] = np.asarray(camera.up_ortho, dtype=np.float64).tolist()
    c.tan_half = float(camera.tan_half)
    c.width, c.height = int(camera.width), int(camera.height)
    return c


# ---------------------------------------------------------------------------
# the eight entry points (_kernelshim.py:33-151)
# ---------------------------------------------------------------------------
def intersect_rays(scene, origins, dirs, t_min):
    """Nearest hits (t, tri); misses t = inf, tri = -1 (_kernelshim.py:33-44)."""
    sc = _scene(scene)
    o, d = _f64(origins), _f64(dirs)
    n = o.shape[0]
    t = _dev.empty((max(n, 1),), np.float64)
    tri = _dev.empty((max(n, 1),), np.int32)
    _lib.call("wfpg_intersect", C.byref(sc.abi()), _lib.ptr(o), _lib.ptr(d), n, float(t_min),
              _lib.ptr(t), _lib.ptr(tri), _dev.stream())
    return _dev.download(t)[:n], _dev.download(tri)[:n].astype(np.int64)


def occluded_rays(scene, origins, dirs, t_min, t_max):
    """Any hit in (t_min, t_max) per ray (_kernelshim.py:47-57)."""
    sc = _scene(scene)
    o, d = _f64(origins), _f64(dirs)
    n = o.shape[0]
    tm = _dev.upload(np.ascontiguousarray(np.broadcast_to(np.asarray(t_max, dtype=np.float64),
                                                          (n,))))
    out = _dev.empty((max(n, 1),), np.uint8)
    _lib.call("wfpg_occluded", C.byref(sc.abi()), _lib.ptr(o), _lib.ptr(d), n, float(t_min),
              _lib.ptr(tm), _lib.ptr(out), _dev.stream())
    return _dev.download(out)[:n].astype(bool)


def descend_tracked(svo, positions):
    """(node, present, deepest) per position (_kernelshim.py:60-71)."""
    return _svo(svo).descend_tracked(positions)


def descend_leaves(svo, positions):
    node, present, _ = descend_tracked(svo, positions)
    return np.where(present, node, -1)


def trace_cones_multi(svo, scene, origins, dirs, omega):
    """Cone queries (_kernelshim.py:79-93): origins broadcast against dirs."""
    sv = _svo(svo, means=True)
    sc = _scene(scene)
    d = _f64(dirs)
    n = d.shape[0]
    o = _f64(origins)
    stride = 3 if o.shape[0] == n and n > 1 else 0
    if stride == 0:
        o = o[:1]
    out = _dev.empty((max(n, 1), 3), np.float64)
    _lib.call("wfpg_trace_cones", C.byref(sc.abi()), C.byref(sv.abi()), _lib.ptr(o), stride,
              _lib.ptr(d), n, float(omega), _lib.ptr(out), _dev.stream())
    return _dev.download(out)[:n]


def trace_cones(svo, scene, origin, dirs, omega):
    return trace_cones_multi(svo, scene, np.asarray(origin, dtype=np.float64)[None, :], dirs,
                             omega)


def camera_rays(camera, keys, pixels):
    """Pinhole rays (_kernelshim.py:101-110)."""
    keys = _dev.upload(np.ascontiguousarray(keys, dtype=np.uint64))
    pix = _dev.upload(np.ascontiguousarray(pixels, dtype=np.int64))
    n = keys.shape[0]
    o = _dev.empty((max(n, 1), 3), np.float64)
    d = _dev.empty((max(n, 1), 3), np.float64)
    cam = _camera_abi(camera)
    _lib.call("wfpg_camera_rays", C.byref(cam), _lib.ptr(keys), _lib.ptr(pix), n, _lib.ptr(o),
              _lib.ptr(d), _dev.stream())
    return _dev.download(o)[:n], _dev.download(d)[:n]


# PathState arrays shade_depth reads / writes (wavefront.py:53-71)
_STATE_IO = ("ray_o", "ray_d", "beta", "radiance", "key", "ctr", "alive", "prev_pdf", "rec_pos",
             "rec_T", "emit_le", "emit_depth")
_STATE_DT = {"key": np.uint64, "ctr": np.uint64, "alive": np.uint8, "emit_depth": np.int32}


def _guide_abi(guide):
    """wfpg_guide for this package's GuideTables or the reference's
    (floored values uploaded; row sums, marginal, totals and product block
    sums by wfpg_guide_fill, bitwise fill_batch's, guiding.py:293-309)."""
    if hasattr(guide, "abi"):
        return guide.abi(), None
    vals = np.asarray(guide.vals, dtype=np.float64)
    b, n = vals.shape[0], int(guide.n)
    keep = {"vals": _dev.upload(vals.reshape(max(b, 1), n, n) if b else np.zeros((1, n, n))),
            "row_sum": _dev.zeros((max(b, 1), n), np.float64),
            "marg": _dev.zeros((max(b, 1), n), np.float64),
            "total": _dev.zeros((max(b, 1),), np.float64),
            "upper": _dev.upload(np.ascontiguousarray(guide.upper_dirs, dtype=np.float64))}
    g = _lib.Guide()
    g.mode, g.n, g.capacity, g.eps = int(guide.mode), n, max(b, 1), float(guide.epsilon)
    g.vals, g.row_sum = keep["vals"].data_ptr(), keep["row_sum"].data_ptr()
    g.marg, g.total = keep["marg"].data_ptr(), keep["total"].data_ptr()
    if g.mode == 2:
        keep["block_sums"] = _dev.zeros((max(b, 1), 8, 8), np.float64)
        keep["block_rows"] = _dev.zeros((max(b, 1), 8, 8, max(1, n // 8)), np.float64)
        g.block_sums = keep["block_sums"].data_ptr()
        g.block_rows = keep["block_rows"].data_ptr()
    g.upper_dirs = keep["upper"].data_ptr()
    if b:
        _lib.call("wfpg_guide_fill", C.byref(g), b, _dev.stream())
    return g, keep


def shade_depth(state, scene, depth, hit_t, hit_tri, guide, bin_slot, rr_enabled=False,
                rr_depth=3):
    """One bounce for every live path (_kernelshim.py:113-151), mutating the
    PathState in place: a device PathState (this package's) directly, a
    reference numpy PathState through an upload / write-back round trip."""
    sc = _scene(scene)
    t = _dev.torch()
    host = not hasattr(state, "dev")
    if host:
        n = int(state.n)
        dev = {k: _dev.upload(np.ascontiguousarray(getattr(state, k), dtype=_STATE_DT.get(
            k, np.float64))) for k in _STATE_IO}
        p = _lib.Paths()
        p.n, p.max_depth = n, int(state.rec_pos.shape[1]) - 1
        for k in _STATE_IO:
            setattr(p, k, dev[k].data_ptr())
        p.n_rec = None  # every record slot is written and read as is
        alive = dev["alive"]
    else:
        p = state.abi()
        alive = state.dev["alive"]
    active = t.nonzero(alive).reshape(-1).to(t.int32)
    n_act = int(active.numel())
    if n_act == 0:
        return
    ht = _dev.upload(np.asarray(hit_t, dtype=np.float64))
    htri = _dev.upload(np.asarray(hit_tri), np.int32)
    g, keep = _guide_abi(guide) if guide is not None else (None, None)
    slots = (_dev.upload(np.asarray(bin_slot), np.int32)
             if (guide is not None and bin_slot is not None) else None)
    _lib.call("wfpg_shade_depth", C.byref(sc.abi()), C.byref(p), int(depth),
              _lib.ptr(active), n_act, None, _lib.ptr(ht), _lib.ptr(htri),
              C.byref(g) if g is not None else None, _lib.ptr(slots),
              1 if rr_enabled else 0, int(rr_depth), _dev.stream())
    del keep
    if host:
        for k in _STATE_IO:
            if k == "key":
                continue  # read only
            out = _dev.download(dev[k])
            dst = getattr(state, k)
            np.copyto(dst, out.astype(bool) if dst.dtype == bool else out.astype(dst.dtype))
