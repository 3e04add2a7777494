"""CPU oracle of the guided render pass — TEST INFRASTRUCTURE.

numpy bookkeeping + the C kernels of render_oracle.c, restating the
reference's render path: wavefront.render_pass (wavefront.py:198-277),
partition_spatial (:98-157), _build_guide_tables (:170-195),
GuideTables.fill_batch (guiding.py:293-309), update_exitance (:286-332),
SvoCache.accumulate_batch / propagate_up (svo.py:254-313).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
use it.  It is pinned to the reference by tests/test_oracle.py against
tests/golden/render_golden.npz.
"""

import ctypes as C
import os
import time

import numpy as np

from . import oracle as O

vp, i32, i64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_double


class OvScene(C.Structure):
    _fields_ = [("n_tris", C.c_int), ("v0", vp), ("e1", vp), ("e2", vp), ("normals", vp),
                ("tri_mat", vp), ("mat_kind", vp), ("mat_rgb", vp), ("n_emit", C.c_int),
                ("em_cdf", vp), ("em_tris", vp), ("em_area", dbl), ("ray_eps", dbl),
                ("blo", vp), ("bhi", vp), ("bleft", vp), ("bright", vp), ("bcount", vp),
                ("border", vp), ("brute", C.c_int)]


class OvSvo(C.Structure):
    _fields_ = [("depth", C.c_int), ("resolution", C.c_int), ("lo", dbl * 3), ("size", dbl),
                ("child_base", vp), ("child_mask", vp), ("parent", vp), ("normal", vp),
                ("mean_a", vp), ("mean_b", vp)]


class OvGuide(C.Structure):
    _fields_ = [("mode", C.c_int), ("n", C.c_int), ("m", C.c_int), ("eps", dbl),
                ("marg", vp), ("cond", vp), ("pdftab", vp), ("vals", vp), ("block_sums", vp),
                ("blk_marg", vp), ("blk_cond", vp), ("upper_dirs", vp)]


class OvPaths(C.Structure):
    _fields_ = [("ray_o", vp), ("ray_d", vp), ("beta", vp), ("radiance", vp), ("key", vp),
                ("ctr", vp), ("alive", vp), ("prev_pdf", vp), ("rec_pos", vp), ("rec_T", vp),
                ("emit_le", vp), ("emit_depth", vp), ("rec_depths", C.c_int)]


P = C.POINTER
O._RENDER_SIGS.extend([
    ("ov_intersect", None, [P(OvScene), vp, vp, i64, dbl, vp, vp]),
    ("ov_descend", None, [P(OvSvo), vp, i64, vp, vp]),
    ("ov_trace_cones", None, [P(OvScene), P(OvSvo), vp, C.c_int, vp, i64, dbl, vp]),
    ("ov_fields", None, [P(OvScene), P(OvSvo), vp, vp, i64, C.c_int, vp, C.c_int, dbl, vp]),
    ("ov_camera", None, [vp, vp, i64, C.c_int, C.c_int, vp, vp, vp, vp, dbl, vp, vp]),
    ("ov_shade", None, [P(OvScene), P(OvGuide), P(OvPaths), C.c_int, vp, i64, vp, vp, vp,
                        C.c_int, C.c_int]),
])


def _p(a):
    return None if a is None else a.ctypes.data_as(vp)


def lib():
    L = O.lib()
    O._extra_sigs(L)
    return L


# ---------------------------------------------------------------------------
# data
# ---------------------------------------------------------------------------
def _oracle_bvh(sc):
    """The scene's BVH without touching the product library: a BVH the caller
    already built, else the numpy restatement of bvh.py:33-119 (bvh.build_py,
    pure numpy; the oracle's any-hit queries traverse it)."""
    built = sc.__dict__.get("_bvh")
    if built is not None:
        return built
    from paper_2405_06997_b200 import bvh as _bvh  # numpy module, no native code

    return _bvh.build_py(np.asarray(sc.v0), np.asarray(sc.v1), np.asarray(sc.v2))


class Scene:
    """Host arrays of a scene (any object with the reference Scene attributes)."""

    def __init__(self, sc):
        c = lambda a, dt: np.ascontiguousarray(a, dtype=dt)  # noqa: E731
        self.src = sc
        self.v0, self.e1, self.e2 = c(sc.v0, np.float64), c(sc.e1, np.float64), c(sc.e2, np.float64)
        self.normals = c(sc.normals, np.float64)
        self.mat_ids = c(sc.mat_ids, np.int32)
        self.mat_kind = c(sc.mat_kind, np.int32)
        self.mat_rgb = c(sc.mat_rgb, np.float64)
        self.em_cdf = c(sc.emitter_cdf, np.float64)
        self.em_tris = c(sc.emitter_tris, np.int64)
        b = _oracle_bvh(sc)
        self.blo, self.bhi = c(b.lo, np.float64), c(b.hi, np.float64)
        self.bl, self.br = c(b.left, np.int64), c(b.right, np.int64)
        self.bc, self.bo = c(b.count, np.int64), c(b.order, np.int64)
        s = OvScene()
        s.n_tris = len(self.v0)
        s.v0, s.e1, s.e2, s.normals = _p(self.v0), _p(self.e1), _p(self.e2), _p(self.normals)
        s.tri_mat, s.mat_kind, s.mat_rgb = _p(self.mat_ids), _p(self.mat_kind), _p(self.mat_rgb)
        s.n_emit, s.em_cdf, s.em_tris = len(self.em_cdf), _p(self.em_cdf), _p(self.em_tris)
        s.em_area, s.ray_eps = float(sc.emitter_area), float(sc.ray_eps)
        s.blo, s.bhi, s.bleft, s.bright = _p(self.blo), _p(self.bhi), _p(self.bl), _p(self.br)
        s.bcount, s.border = _p(self.bc), _p(self.bo)
        s.brute = 1 if len(self.v0) <= 512 else 0
        self.c = s
        self.camera = sc.camera
        self.ray_eps = float(sc.ray_eps)


class Svo:
    """Oracle SVO: structure from oracle.build_octree + accumulators."""

    def __init__(self, built, cube_lo, size, resolution):
        self.d = built
        self.depth = int(resolution).bit_length() - 1
        self.resolution = int(resolution)
        self.cube_lo = np.asarray(cube_lo, dtype=np.float64)
        self.cube_size = float(size)
        self.level_off = built["level_off"]
        n = int(self.level_off[-1])
        self.parent = built["parent"]
        self.child_base = built["child_base"]
        self.child_mask = built["child_mask"]
        self.normal = np.ascontiguousarray(built["normal"])
        self.sum_a, self.sum_b = np.zeros((n, 3)), np.zeros((n, 3))
        self.weight_a, self.weight_b = np.zeros(n), np.zeros(n)
        self.mean_a, self.mean_b = np.zeros((n, 3)), np.zeros((n, 3))

    @classmethod
    def from_scene(cls, sc, resolution, seed=0):
        lo, side = O.scene_cube(sc.bbox_lo, sc.bbox_hi)
        coords, tris = O.voxelize(sc.v0, sc.v1, sc.v2, lo, side, resolution)
        return cls(O.build_octree(coords, sc.normals[tris], resolution, seed), lo, side,
                   resolution)

    def c(self):
        s = OvSvo()
        s.depth, s.resolution = self.depth, self.resolution
        s.lo[:] = self.cube_lo.tolist()
        s.size = self.cube_size
        s.child_base, s.child_mask, s.parent = (_p(self.child_base), _p(self.child_mask),
                                                _p(self.parent))
        s.normal, s.mean_a, s.mean_b = _p(self.normal), _p(self.mean_a), _p(self.mean_b)
        return s

    def descend(self, pts):
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        n = len(pts)
        node = np.zeros(n, dtype=np.int64)
        pres = np.zeros(n, dtype=np.uint8)
        lib().ov_descend(C.byref(self.c()), _p(pts), n, _p(node), _p(pres))
        return node, pres.astype(bool)

    def level_of(self, nodes):
        return np.searchsorted(self.level_off, nodes, side="right") - 1

    # svo.py:254-263: side a iff einsum(dir, normal) >= 0; np.add.at in order
    def accumulate(self, leaf, dirs, rad):
        nn = self.normal[leaf]
        dot = (dirs[:, 0] * nn[:, 0] + dirs[:, 2] * nn[:, 2]) + dirs[:, 1] * nn[:, 1]
        a = dot >= 0.0
        np.add.at(self.sum_a, leaf[a], rad[a])
        np.add.at(self.weight_a, leaf[a], 1.0)
        np.add.at(self.sum_b, leaf[~a], rad[~a])
        np.add.at(self.weight_b, leaf[~a], 1.0)

    # svo.py:265-313 as a full bottom-up recompute
    def propagate(self):
        d = self.depth
        lo, hi = self.level_off[d], self.level_off[d + 1]
        for s, w, m in ((self.sum_a, self.weight_a, self.mean_a),
                        (self.sum_b, self.weight_b, self.mean_b)):
            ww = w[lo:hi]
            m[lo:hi] = np.where((ww > 0)[:, None], s[lo:hi] / np.where(ww > 0, ww, 1.0)[:, None],
                                0.0)
        for lv in range(d - 1, -1, -1):
            nodes = np.arange(self.level_off[lv], self.level_off[lv + 1])
            cnt = np.array([bin(int(x)).count("1") for x in self.child_mask[nodes]])
            kid = np.repeat(self.child_base[nodes], cnt) + (
                np.arange(cnt.sum()) - np.repeat(np.cumsum(cnt) - cnt, cnt))
            own = np.repeat(np.arange(len(nodes)), cnt)
            cn, pn = self.normal[kid], self.normal[nodes][own]
            al = ((cn[:, 0] * pn[:, 0] + cn[:, 2] * pn[:, 2]) + cn[:, 1] * pn[:, 1]) >= 0.0
            ca = np.where(al[:, None], self.mean_a[kid], self.mean_b[kid])
            cb = np.where(al[:, None], self.mean_b[kid], self.mean_a[kid])
            acc_a, acc_b = np.zeros((len(nodes), 3)), np.zeros((len(nodes), 3))
            np.add.at(acc_a, own, ca)
            np.add.at(acc_b, own, cb)
            self.mean_a[nodes] = acc_a / cnt[:, None]
            self.mean_b[nodes] = acc_b / cnt[:, None]


# ---------------------------------------------------------------------------
# kernels
# ---------------------------------------------------------------------------
def intersect(sc, o, d, tmin=None):
    o = np.ascontiguousarray(o, dtype=np.float64).reshape(-1, 3)
    d = np.ascontiguousarray(d, dtype=np.float64).reshape(-1, 3)
    n = len(o)
    t = np.zeros(n)
    tri = np.zeros(n, dtype=np.int64)
    lib().ov_intersect(C.byref(sc.c), _p(o), _p(d), n, sc.ray_eps if tmin is None else tmin,
                       _p(t), _p(tri))
    return t, tri


def trace_cones(sc, svo, origins, dirs, omega):
    d = np.ascontiguousarray(dirs, dtype=np.float64).reshape(-1, 3)
    o = np.ascontiguousarray(origins, dtype=np.float64).reshape(-1, 3)
    stride = 3 if len(o) == len(d) else 0
    out = np.zeros((len(d), 3))
    lib().ov_trace_cones(C.byref(sc.c), C.byref(svo.c()), _p(o), stride, _p(d), len(d),
                         float(omega), _p(out))
    return out


def blur_taps(sigma):
    radius = max(1, int(np.ceil(3.0 * sigma)))
    k = np.exp(-0.5 * (np.arange(-radius, radius + 1) / sigma) ** 2)
    return k / k.sum(), radius


def fields(sc, svo, origins, jitters, n, blur_sigma=1.0, eps=1e-2):
    origins = np.ascontiguousarray(origins, dtype=np.float64).reshape(-1, 3)
    jitters = np.ascontiguousarray(jitters, dtype=np.float64).reshape(-1, 2)
    b = len(origins)
    out = np.zeros((b, n, n))
    if blur_sigma > 0:
        w, r = blur_taps(blur_sigma)
    else:
        w, r = np.zeros(1), 0
    w = np.ascontiguousarray(w)
    lib().ov_fields(C.byref(sc.c), C.byref(svo.c()), _p(origins), _p(jitters), b, n, _p(w), r,
                    eps, _p(out))
    return out


def _tables_chunk(values, mode):
    b, n, _ = values.shape
    rows = values.sum(axis=2)
    tot = rows.sum(axis=1)
    t = {"marg": np.cumsum(rows, axis=1) / tot[:, None],
         "cond": np.cumsum(values, axis=2) / rows[:, :, None],
         "pdftab": values * (n * n / (4.0 * np.pi)) / tot[:, None, None],
         "vals": values}
    m = n // 8
    if mode == 2:
        blocks = values.reshape(b, 8, m, 8, m).transpose(0, 1, 3, 2, 4)
        sums = blocks.sum(axis=(3, 4))
        brow = blocks.sum(axis=4)
        t["block_sums"] = sums
        t["blk_marg"] = np.cumsum(brow, axis=3) / sums[..., None]
        t["blk_cond"] = np.cumsum(blocks, axis=4) / brow[..., None]
    return t


def tables(values, mode):
    """guiding.py:293-309 restated (per-bin arithmetic, so chunks of bins are
    evaluated on a thread pool with identical results)."""
    b = values.shape[0]
    nt = min(_threads(), max(1, b // 64))
    if nt <= 1:
        t = _tables_chunk(values, mode)
    else:
        from concurrent.futures import ThreadPoolExecutor

        cuts = np.linspace(0, b, nt + 1).astype(int)
        with ThreadPoolExecutor(nt) as ex:
            parts = list(ex.map(lambda k: _tables_chunk(values[cuts[k]:cuts[k + 1]], mode),
                                range(nt)))
        t = {k: np.concatenate([p[k] for p in parts]) for k in parts[0]}
    return {k: np.ascontiguousarray(v) for k, v in t.items()}


def _upper_dirs():
    uc = (np.arange(8) + 0.5) / 8
    gu, gv = np.meshgrid(uc, uc, indexing="xy")
    a, b = 2.0 * gu - 1.0, 2.0 * gv - 1.0
    ap, bp = np.abs(a), np.abs(b)
    sd = 1.0 - (ap + bp)
    r = 1.0 - np.abs(sd)
    phi = np.where(r == 0.0, 1.0, (bp - ap) / np.where(r == 0.0, 1.0, r) + 1.0) * (np.pi / 4.0)
    z = np.copysign(1.0 - r * r, sd)
    rho = r * np.sqrt(np.maximum(2.0 - r * r, 0.0))
    out = np.stack([np.copysign(np.cos(phi), a) * rho, np.copysign(np.sin(phi), b) * rho, z], -1)
    out /= np.linalg.norm(out, axis=-1, keepdims=True)
    return np.ascontiguousarray(out)


UPPER_DIRS = _upper_dirs()


# ---------------------------------------------------------------------------
# the pass
# ---------------------------------------------------------------------------
def partition(svo, pos, l_min, c_ray):
    """Alg. 2 restated: per-path ancestor counts above l_min, ascent, stable sort."""
    node, _ = svo.descend(pos)
    lev = svo.level_of(node)
    counter = np.zeros(int(svo.level_off[-1]), dtype=np.int64)
    cur, cl = node.copy(), lev.copy()
    for lv in range(svo.depth, l_min, -1):
        sel = cl == lv
        np.add.at(counter, cur[sel], 1)
        cur[sel] = svo.parent[cur[sel]]
        cl[sel] -= 1
    b, bl = node.copy(), lev.copy()
    while True:
        step = (bl > l_min) & (counter[b] < c_ray)
        if not step.any():
            break
        b[step] = svo.parent[b[step]]
        bl[step] -= 1
    order = np.argsort(b, kind="stable")
    nodes, starts = np.unique(b[order], return_index=True)
    ends = np.append(starts[1:], len(order))
    return nodes, [order[s:e] for s, e in zip(starts, ends)]


def _paths_struct(st):
    p = OvPaths()
    for k in ("ray_o", "ray_d", "beta", "radiance", "key", "ctr", "alive", "prev_pdf", "rec_pos",
              "rec_T", "emit_le", "emit_depth"):
        setattr(p, k, _p(st[k]))
    p.rec_depths = st["rec_pos"].shape[1]
    return p


def render_pass(sc, svo, cfg, sample, stats=None):
    """One pass (1 spp) with the reference's semantics; returns (frame, state)."""
    cam = sc.camera
    w, h = cam.width, cam.height
    n = w * h
    D = cfg["max_depth"]
    st = {"ray_o": np.zeros((n, 3)), "ray_d": np.zeros((n, 3)), "beta": np.ones((n, 3)),
          "radiance": np.zeros((n, 3)), "key": np.zeros(n, dtype=np.uint64),
          "ctr": np.full(n, 2, dtype=np.uint64), "alive": np.ones(n, dtype=np.uint8),
          "prev_pdf": np.full(n, -1.0), "rec_pos": np.zeros((n, D + 1, 3)),
          "rec_T": np.zeros((n, D + 1, 3)), "emit_le": np.zeros((n, 3)),
          "emit_depth": np.zeros(n, dtype=np.int32)}
    st["rec_pos"][:, 0] = cam.position
    pix = np.arange(n, dtype=np.int64)
    st["key"] = O.stream_keys(cfg["seed"], (np.uint64(sample * n) + np.arange(n, dtype=np.uint64))
                              * np.uint64(4))
    lib().ov_camera(_p(st["key"]), _p(pix), n, w, h, _p(np.ascontiguousarray(cam.position)),
                    _p(np.ascontiguousarray(cam.forward)), _p(np.ascontiguousarray(cam.right)),
                    _p(np.ascontiguousarray(cam.up_ortho)), cam.tan_half, _p(st["ray_o"]),
                    _p(st["ray_d"]))
    ps = _paths_struct(st)
    hit_t = np.zeros(n)
    hit_tri = np.zeros(n, dtype=np.int64)
    for depth in range(1, D + 1):
        act = np.nonzero(st["alive"])[0].astype(np.int64)
        if len(act) == 0:
            break
        t, tri = intersect(sc, st["ray_o"][act], st["ray_d"][act])
        hit_t[act], hit_tri[act] = t, tri
        g = OvGuide()
        g.mode = 0
        slots = np.full(n, -1, dtype=np.int32)
        keep = []
        if svo is not None:
            ok = tri >= 0
            kinds = np.full(len(act), -1)
            kinds[ok] = sc.mat_kind[sc.mat_ids[tri[ok]]]
            lam = act[kinds == 0]
            pos = st["ray_o"][lam] + hit_t[lam][:, None] * st["ray_d"][lam]
            nodes, members = partition(svo, pos, cfg["l_min"], cfg["c_ray"]) if len(lam) else ([], [])
            if stats is not None:
                stats.setdefault("bins", []).append(len(nodes))
                stats.setdefault("rays", []).append(len(lam))
            if depth <= cfg["guided_depths"] and len(nodes):
                nf = max(8, cfg["field_res"] >> (depth - 1))
                keys = [O.stream_key(cfg["seed"], (((sample * 64 + depth) << 32) + int(nd)) * 4 + 1)
                        for nd in nodes]
                origins = np.array([pos[m[min(int(O.u01(k, 0) * len(m)), len(m) - 1)]]
                                    for k, m in zip(keys, members)])
                jit = np.array([[O.u01(k, 1), O.u01(k, 2)] if cfg.get("jitter", True)
                                else [0.5, 0.5] for k in keys])
                for slot, m in enumerate(members):
                    slots[lam[m]] = slot
                mode = 2 if cfg.get("product") else 1
                tb = tables(fields(sc, svo, origins, jit, nf), mode)
                keep = [tb]
                g.mode, g.n, g.m, g.eps = mode, nf, nf // 8, 1e-2
                for k in ("marg", "cond", "pdftab", "vals", "block_sums", "blk_marg", "blk_cond"):
                    setattr(g, k, _p(tb.get(k)))
                g.upper_dirs = _p(UPPER_DIRS)
        lib().ov_shade(C.byref(sc.c), C.byref(g), C.byref(ps), depth, _p(act), len(act),
                       _p(hit_t), _p(hit_tri), _p(slots), int(bool(cfg.get("russian_roulette", False))),
                       int(cfg.get("rr_depth", 3)))
        del keep
    if svo is not None:
        update_exitance(st, svo)
    return st["radiance"].reshape(h, w, 3).copy(), st


def update_exitance(st, svo):
    """wavefront.py:286-332 restated."""
    ed, le = st["emit_depth"].astype(np.int64), st["emit_le"]
    paths = np.nonzero((ed >= 2) & (le.sum(axis=1) > 0.0))[0]
    cnt = ed[paths] - 1
    pk = np.repeat(paths, cnt)
    kk = np.arange(cnt.sum()) - np.repeat(np.cumsum(cnt) - cnt, cnt) + 1
    if len(pk):
        ok = np.all(st["rec_T"][pk, kk] > 0.0, axis=1)
        pk, kk = pk[ok], kk[ok]
    if not len(pk):
        svo.propagate()
        return 0
    tk = st["rec_T"][pk, kk]
    tn = st["rec_T"][pk, ed[pk]]
    rad = (tn / tk) * le[pk]
    pos, prev = st["rec_pos"][pk, kk], st["rec_pos"][pk, kk - 1]
    out = prev - pos
    out /= np.sqrt((out[:, 0] * out[:, 0] + out[:, 1] * out[:, 1]) + out[:, 2] * out[:, 2])[:, None]
    q = pos + out * ((svo.cube_size / svo.resolution) * 1e-3)
    tiny = svo.cube_size * 1e-12
    q = np.clip(q, svo.cube_lo + tiny, svo.cube_lo + svo.cube_size - tiny)
    leaf, pres = svo.descend(q)
    good = pres
    svo.accumulate(leaf[good], out[good], rad[good])
    svo.propagate()
    return int(good.sum())


# ---------------------------------------------------------------------------
# CPU baseline for bench.py
# ---------------------------------------------------------------------------
def _cfg_dict(cfg):
    g = (lambda k, d=None: getattr(cfg, k, d)) if not isinstance(cfg, dict) else cfg.get
    return dict(max_depth=g("max_depth"), guided_depths=g("guided_depths"),
                field_res=g("field_res"), l_min=g("l_min"), c_ray=g("c_ray"), seed=g("seed", 0),
                product=bool(g("product", False)), jitter=bool(g("jitter", True)))


def _threads():
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


class CpuWorkload:
    """The bench workload entirely on the host, with the reference's pass
    sequence: oracle SVO build (svo.build_from_scene), a PT-first pass
    (sample 0, guided_depths 0, SVO updated), then every call of ``run_pass``
    renders the next guided sample in full (wavefront.render_pass,
    wavefront.py:198-277, with its exitance update) — nothing extrapolated."""

    def __init__(self, scene, resolution, cfg, seed=0, svo=None):
        self.sc = Scene(scene)
        self.cfg = _cfg_dict(cfg)
        t0 = time.perf_counter()
        self.svo = svo if svo is not None else Svo.from_scene(scene, resolution, seed)
        self.build_s = time.perf_counter() - t0
        self.pt_s = 0.0
        self.next_sample = 1
        if svo is None:
            t0 = time.perf_counter()
            render_pass(self.sc, self.svo, dict(self.cfg, guided_depths=0), 0, {})
            self.pt_s = time.perf_counter() - t0

    @classmethod
    def from_device(cls, scene, tree, cfg, next_sample):
        """Continue a device run on the host: the device SVO's structure and
        exitance state (bit-exact with the oracle's, tests/test_full_size.py)."""
        built = {k: np.ascontiguousarray(getattr(tree, k)) for k in (
            "level_off", "codes", "child_base", "child_mask", "parent", "normal")}
        svo = Svo(built, tree.cube_lo, tree.cube_size, tree.resolution)
        for k in ("sum_a", "sum_b", "weight_a", "weight_b", "mean_a", "mean_b"):
            setattr(svo, k, np.ascontiguousarray(getattr(tree, k)))
        w = cls(scene, tree.resolution, cfg, svo=svo)
        w.next_sample = int(next_sample)
        return w

    def run_pass(self):
        """Render the next guided sample; returns (seconds, stats)."""
        stats = {}
        t0 = time.perf_counter()
        render_pass(self.sc, self.svo, self.cfg, self.next_sample, stats)
        dt = time.perf_counter() - t0
        self.next_sample += 1
        return dt, stats

    def describe(self):
        return (f"oracle SVO build {self.build_s:.1f} s, PT-first pass {self.pt_s:.1f} s")


def time_guided_passes(workload, n_paths, passes=1):
    """cpu_baseline object: ``passes`` full guided oracle passes, timed."""
    secs, bins = [], None
    for _ in range(passes):
        dt, st = workload.run_pass()
        secs.append(dt)
        bins = st.get("bins")
    tot = sum(secs)
    return {"value": n_paths * len(secs) / tot if tot > 0 else None, "unit": "path samples/s",
            "cores": _threads(), "kind": "port",
            "sample": f"{len(secs)} full guided pass(es) of the same workload by the CPU oracle "
                      f"(oracle/: C + OpenMP field generation on all host threads, numpy "
                      f"bookkeeping), samples {workload.next_sample - len(secs)}.."
                      f"{workload.next_sample - 1}, {tot:.1f} s; bins per depth {bins}",
            "pass_seconds": secs}
