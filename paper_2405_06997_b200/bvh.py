"""Host-side binned-SAH BVH, flattened for the device traversal kernels.

Built on first use by the C++ port in libwfpg_b200.so (csrc/bvh_host.cu) with
the reference's decisions (bvh.py:33-119; ``build_py`` is the numpy
restatement it is checked against), then uploaded; traversal runs in the
CUDA kernels (geometry.cuh).  The build
makes the same split decisions as the reference so that the device traversal
visits the same boxes: 16 centroid bins on the widest centroid axis, at most
4 triangles per leaf, surface-area cost with strict improvement, stable
left/right partition, median fallback, and depth-first node numbering with
both children allocated before descending into the left one.
"""

import numpy as np

MAX_LEAF_TRIS = 4
N_BINS = 16


class Bvh:
    """Flattened two-child BVH: for inner nodes ``left``/``right`` are child
    node ids and ``count`` is 0; for leaves ``left`` indexes ``order`` and
    ``count`` is the triangle count."""

    def __init__(self, lo, hi, left, right, count, order):
        self.lo = lo
        self.hi = hi
        self.left = left
        self.right = right
        self.count = count
        self.order = order

    @property
    def node_count(self):
        return len(self.count)


def _area(lo, hi):
    ex, ey, ez = np.maximum(hi - lo, 0.0)
    return 2.0 * (ex * ey + ey * ez + ez * ex)


def _choose_split(tri_lo, tri_hi, cen, ids):
    """Returns (sorted ids for the node range, left count) or None for a median split."""
    clo = cen[ids].min(axis=0)
    chi = cen[ids].max(axis=0)
    axis = int(np.argmax(chi - clo))
    extent = chi[axis] - clo[axis]
    if extent <= 0.0:
        return None
    scale = N_BINS / extent
    b = np.minimum((cen[ids, axis] - clo[axis]) * scale, N_BINS - 1).astype(np.int64)
    blo = np.full((N_BINS, 3), np.inf)
    bhi = np.full((N_BINS, 3), -np.inf)
    cnt = np.zeros(N_BINS, dtype=np.int64)
    for k in range(N_BINS):
        hit = b == k
        if hit.any():
            blo[k] = tri_lo[ids[hit]].min(axis=0)
            bhi[k] = tri_hi[ids[hit]].max(axis=0)
            cnt[k] = hit.sum()
    best, split = np.inf, -1
    for s in range(1, N_BINS):
        nl, nr = cnt[:s].sum(), cnt[s:].sum()
        if nl == 0 or nr == 0:
            continue
        cost = (_area(blo[:s].min(axis=0), bhi[:s].max(axis=0)) * nl
                + _area(blo[s:].min(axis=0), bhi[s:].max(axis=0)) * nr)
        if cost < best:
            best, split = cost, s
    if split < 0:
        return None
    go_left = b < split
    return np.concatenate([ids[go_left], ids[~go_left]]), int(go_left.sum())


def build(v0, v1, v2):
    """The reference's BVH (see the module doc), built by the C++ port in
    libwfpg_b200.so (csrc/bvh_host.cu); bitwise the arrays of build_py."""
    import ctypes as C

    from . import _lib

    v0, v1, v2 = (np.ascontiguousarray(a, dtype=np.float64) for a in (v0, v1, v2))
    n = len(v0)
    cap = max(2 * n - 1, 1)
    lo, hi = np.empty((cap, 3)), np.empty((cap, 3))
    left, right, count = (np.empty(cap, dtype=np.int32) for _ in range(3))
    order = np.empty(n, dtype=np.int32)
    nn = C.c_int64(0)
    p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    _lib.call("wfpg_bvh_build_host", p(v0), p(v1), p(v2), n, p(lo), p(hi), p(left), p(right),
              p(count), p(order), C.byref(nn))
    k = nn.value
    return Bvh(lo[:k].copy(), hi[:k].copy(), left[:k].astype(np.int64),
               right[:k].astype(np.int64), count[:k].astype(np.int64), order.astype(np.int64))


def build_py(v0, v1, v2):
    """numpy restatement of the reference's build (kept as the checker of
    the C++ port, tests/test_host_api.py)."""
    n = len(v0)
    tri_lo = np.minimum(np.minimum(v0, v1), v2)
    tri_hi = np.maximum(np.maximum(v0, v1), v2)
    cen = (tri_lo + tri_hi) * 0.5
    order = np.arange(n, dtype=np.int64)

    lo, hi, left, right, count = [None], [None], [-1], [-1], [0]
    todo = [(0, 0, n)]
    while todo:
        node, start, end = todo.pop()
        ids = order[start:end]
        lo[node] = tri_lo[ids].min(axis=0)
        hi[node] = tri_hi[ids].max(axis=0)
        m = end - start
        if m <= MAX_LEAF_TRIS:
            left[node] = start
            count[node] = m
            continue
        mid = start + m // 2
        choice = _choose_split(tri_lo, tri_hi, cen, ids)
        if choice is not None:
            perm, n_left = choice
            order[start:end] = perm
            if 0 < n_left < m:
                mid = start + n_left
        kids = []
        for _ in range(2):
            lo.append(None)
            hi.append(None)
            left.append(-1)
            right.append(-1)
            count.append(0)
            kids.append(len(count) - 1)
        left[node], right[node] = kids
        # LIFO: the left child is processed first, like the reference recursion
        todo.append((kids[1], mid, end))
        todo.append((kids[0], start, mid))
    return Bvh(np.asarray(lo, dtype=np.float64), np.asarray(hi, dtype=np.float64),
               np.asarray(left, dtype=np.int64), np.asarray(right, dtype=np.int64),
               np.asarray(count, dtype=np.int64), order)
