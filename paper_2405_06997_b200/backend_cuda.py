"""The reference's backend API (backend.py / _kernelshim.py) on the B200.

``NAME``, ``COMPILED`` and the eight kernel entry points with the signatures
of wfpg._kernelshim (numpy in, numpy out), each implemented by one C-ABI call
into libwfpg_b200.so.  A reference user can install this module with
``wfpg.backend.set_backend(paper_2405_06997_b200.backend_cuda)`` when their
scene / svo objects are this package's.  The render path
itself never goes through these numpy wrappers: render_pass keeps every
array on the device.
"""

import ctypes as C

import numpy as np

from . import _dev, _lib

NAME = "cuda-sm100a"
COMPILED = True


def _f64(a, cols=3):
    return _dev.upload(np.ascontiguousarray(np.atleast_2d(a), dtype=np.float64).reshape(-1, cols))


def intersect_rays(scene, origins, dirs, t_min):
    """Nearest hits (t, tri); misses t = inf, tri = -1 (_kernelshim.py:33-44)."""
    o, d = _f64(origins), _f64(dirs)
    n = o.shape[0]
    t = _dev.empty((max(n, 1),), np.float64)
    tri = _dev.empty((max(n, 1),), np.int32)
    _lib.call("wfpg_intersect", C.byref(scene.abi()), _lib.ptr(o), _lib.ptr(d), n, float(t_min),
              _lib.ptr(t), _lib.ptr(tri), _dev.stream())
    return _dev.download(t)[:n], _dev.download(tri)[:n].astype(np.int64)


def occluded_rays(scene, origins, dirs, t_min, t_max):
    """Any hit in (t_min, t_max) per ray (_kernelshim.py:47-57)."""
    o, d = _f64(origins), _f64(dirs)
    n = o.shape[0]
    tm = _dev.upload(np.ascontiguousarray(np.broadcast_to(np.asarray(t_max, dtype=np.float64),
                                                          (n,))))
    out = _dev.empty((max(n, 1),), np.uint8)
    _lib.call("wfpg_occluded", C.byref(scene.abi()), _lib.ptr(o), _lib.ptr(d), n, float(t_min),
              _lib.ptr(tm), _lib.ptr(out), _dev.stream())
    return _dev.download(out)[:n].astype(bool)


def descend_tracked(svo, positions):
    return svo.descend_tracked(positions)


def descend_leaves(svo, positions):
    node, present, _ = svo.descend_tracked(positions)
    return np.where(present, node, -1)


def trace_cones_multi(svo, scene, origins, dirs, omega):
    d = _f64(dirs)
    n = d.shape[0]
    o = _f64(origins)
    stride = 3 if o.shape[0] == n and n > 1 else 0
    if stride == 0:
        o = o[:1]
    out = _dev.empty((max(n, 1), 3), np.float64)
    _lib.call("wfpg_trace_cones", C.byref(scene.abi()), C.byref(svo.abi()), _lib.ptr(o), stride,
              _lib.ptr(d), n, float(omega), _lib.ptr(out), _dev.stream())
    return _dev.download(out)[:n]


def trace_cones(svo, scene, origin, dirs, omega):
    return trace_cones_multi(svo, scene, np.asarray(origin, dtype=np.float64)[None, :], dirs,
                             omega)


def camera_rays(camera, keys, pixels):
    keys = _dev.upload(np.ascontiguousarray(keys, dtype=np.uint64))
    pix = _dev.upload(np.ascontiguousarray(pixels, dtype=np.int64))
    n = keys.shape[0]
    o = _dev.empty((max(n, 1), 3), np.float64)
    d = _dev.empty((max(n, 1), 3), np.float64)
    cam = camera.as_abi()
    _lib.call("wfpg_camera_rays", C.byref(cam), _lib.ptr(keys), _lib.ptr(pix), n, _lib.ptr(o),
              _lib.ptr(d), _dev.stream())
    return _dev.download(o)[:n], _dev.download(d)[:n]


def shade_depth(state, scene, depth, hit_t, hit_tri, guide, bin_slot, rr_enabled=False,
                rr_depth=3):
    """One bounce for every live path of a device PathState (_kernelshim.py:113-151).

    ``state`` is a wavefront.PathState (device resident); ``guide`` a
    guiding.GuideTables or None; ``bin_slot`` per-path slots or None."""
    alive = state.dev["alive"]
    active = _dev.torch().nonzero(alive).reshape(-1).to(_dev.torch().int32)
    n_act = int(active.numel())
    if n_act == 0:
        return
    ht = _dev.upload(np.asarray(hit_t, dtype=np.float64))
    htri = _dev.upload(np.asarray(hit_tri), np.int32)
    g = guide.abi() if guide is not None else None
    slots = _dev.upload(np.asarray(bin_slot), np.int32) if (guide is not None and
                                                           bin_slot is not None) else None
    _lib.call("wfpg_shade_depth", C.byref(scene.abi()), C.byref(state.abi()), int(depth),
              _lib.ptr(active), n_act, None, _lib.ptr(ht), _lib.ptr(htri),
              C.byref(g) if g is not None else None, _lib.ptr(slots),
              1 if rr_enabled else 0, int(rr_depth), _dev.stream())
