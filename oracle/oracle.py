"""CPU oracle for the B200 hot path — TEST INFRASTRUCTURE, not product code.

Restates the reference algorithm (numpy for integer bookkeeping, the C file
wfpg_oracle.c for fp64 arithmetic in the reference's exact operation order).
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module.  Each function cites the reference file:line it follows
(paths relative to /root/reference/pkg/src/wfpg/).

Parity pinned: tests/test_oracle.py checks every function here against the
golden fixtures in tests/golden/, which the real reference produced.
"""

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libwfpg_oracle.so")

_lib = None


def build():
    """Compile the C restatement (gcc, explicit FMAs only)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = C.CDLL(LIB)
        vp, i64, u64, dbl, i32 = C.c_void_p, C.c_int64, C.c_uint64, C.c_double, C.c_int
        L.ov_voxelize.restype = i64
        L.ov_voxelize.argtypes = [i32, vp, vp, vp, vp, dbl, i32, vp, vp, i64]
        L.ov_cluster_normals.restype = None
        L.ov_cluster_normals.argtypes = [vp, i32, u64, vp]
        L.ov_svo_normals.restype = None
        L.ov_svo_normals.argtypes = [i32, vp, vp, vp, vp, vp, vp, u64, vp]
        L.ov_stream_key.restype = u64
        L.ov_stream_key.argtypes = [u64, u64]
        L.ov_u01.restype = dbl
        L.ov_u01.argtypes = [u64, u64]
        _extra_sigs(L)
        _lib = L
    return _lib


def _extra_sigs(L):
    """Signatures of the render-path functions (filled in as they are added)."""
    for name, res, args in _RENDER_SIGS:
        f = getattr(L, name, None)
        if f is not None:
            f.restype = res
            f.argtypes = args


_RENDER_SIGS = []


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------------------
# core (core.py:88-138, 204-228)
# ---------------------------------------------------------------------------
def _spread(v):
    v = v.astype(np.uint64) & np.uint64(0x1FFFFF)
    for sh, m in ((32, 0x1F00000000FFFF), (16, 0x1F0000FF0000FF), (8, 0x100F00F00F00F00F),
                  (4, 0x10C30C30C30C30C3), (2, 0x1249249249249249)):
        v = (v | (v << np.uint64(sh))) & np.uint64(m)
    return v


def morton_encode(x, y, z):
    x, y, z = (np.asarray(a, dtype=np.int64) for a in (x, y, z))
    return _spread(x) | (_spread(y) << np.uint64(1)) | (_spread(z) << np.uint64(2))


def stream_key(seed, stream):
    return int(lib().ov_stream_key(int(seed) & (2**64 - 1), int(stream) & (2**64 - 1)))


def u01(key, counter):
    return float(lib().ov_u01(int(key) & (2**64 - 1), int(counter) & (2**64 - 1)))


def _mix64_np(x):
    x = x.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        x ^= x >> np.uint64(30)
        x *= np.uint64(0xBF58476D1CE4E5B9)
        x ^= x >> np.uint64(27)
        x *= np.uint64(0x94D049BB133111EB)
        x ^= x >> np.uint64(31)
    return x


def stream_keys(seed, streams):
    """Vectorised stream_key (core.py:213-219) over a uint64 array."""
    s = _mix64_np(np.array([int(seed) & (2**64 - 1)], dtype=np.uint64))
    with np.errstate(over="ignore"):
        m = _mix64_np(np.asarray(streams, dtype=np.uint64)) * np.uint64(0x9E3779B97F4A7C15)
    return _mix64_np(s ^ m)


# ---------------------------------------------------------------------------
# SVO build (svo.py:39-46, 94-136, 416-500)
# ---------------------------------------------------------------------------
def scene_cube(bbox_lo, bbox_hi, pad=1e-4):
    center = 0.5 * (bbox_lo + bbox_hi)
    side = float((bbox_hi - bbox_lo).max()) * (1.0 + pad)
    return center - 0.5 * side, side


def voxelize(v0, v1, v2, cube_lo, side, r):
    v0, v1, v2 = (np.ascontiguousarray(a, dtype=np.float64) for a in (v0, v1, v2))
    lo = np.ascontiguousarray(cube_lo, dtype=np.float64)
    T = len(v0)
    n = lib().ov_voxelize(T, _p(v0), _p(v1), _p(v2), _p(lo), side, r, None, None, 0)
    coords = np.zeros((max(n, 1), 3), dtype=np.int64)
    tris = np.zeros(max(n, 1), dtype=np.int64)
    lib().ov_voxelize(T, _p(v0), _p(v1), _p(v2), _p(lo), side, r, _p(coords), _p(tris), n)
    return coords[:n], tris[:n]


def build_octree(coords, frag_normals, resolution, seed=0):
    """Returns a dict with level_off, codes, child_base, child_mask, parent,
    normal, plus sorted_codes / sort_perm / leaf_start."""
    depth = int(resolution).bit_length() - 1
    codes = morton_encode(coords[:, 0], coords[:, 1], coords[:, 2])
    perm = np.argsort(codes, kind="stable")
    sc = codes[perm]
    first = np.ones(len(sc), dtype=bool)
    first[1:] = sc[1:] != sc[:-1]
    leaf_start = np.append(np.nonzero(first)[0], len(sc)).astype(np.int64)
    levels = [sc[first]]
    for _ in range(depth):
        up = levels[-1] >> np.uint64(3)
        keep = np.ones(len(up), dtype=bool)
        keep[1:] = up[1:] != up[:-1]
        levels.append(up[keep])
    levels.reverse()
    level_off = np.concatenate([[0], np.cumsum([len(c) for c in levels])]).astype(np.int64)
    n = int(level_off[-1])
    child_base = np.full(n, -1, dtype=np.int64)
    child_mask = np.zeros(n, dtype=np.uint8)
    parent = np.full(n, -1, dtype=np.int64)
    for lv in range(depth):
        po, co = level_off[lv], level_off[lv + 1]
        kids = levels[lv + 1]
        owner = np.searchsorted(levels[lv], kids >> np.uint64(3))
        parent[co:co + len(kids)] = po + owner
        starts = np.ones(len(kids), dtype=bool)
        starts[1:] = owner[1:] != owner[:-1]
        child_base[po + owner[starts]] = co + np.nonzero(starts)[0]
        bits = (np.uint8(1) << (kids & np.uint64(7)).astype(np.uint8)).astype(np.uint8)
        np.bitwise_or.at(child_mask, po + owner, bits)
    all_codes = np.concatenate(levels)
    normal = np.zeros((n, 3))
    fn = np.ascontiguousarray(frag_normals[perm], dtype=np.float64)
    lib().ov_svo_normals(depth, _p(level_off), _p(all_codes), _p(child_base), _p(child_mask),
                         _p(fn), _p(leaf_start), int(seed) & (2**64 - 1), _p(normal))
    return {"level_off": level_off, "codes": all_codes, "child_base": child_base,
            "child_mask": child_mask, "parent": parent, "normal": normal,
            "sorted_codes": sc, "sort_perm": perm.astype(np.int64), "leaf_start": leaf_start}
