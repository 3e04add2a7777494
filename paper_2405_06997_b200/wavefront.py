"""Wavefront render loop — the whole pass runs on the device.

Drop-in for wavefront.py of the reference (wavefront.py:1-332): same
GuidingConfig, PassStats, SpatialBin, partition_spatial, bin_stream_id,
render_pass, render_sample and update_exitance.  ``render_pass`` enqueues one
device pass (csrc/render.cu): camera rays, then per depth compaction,
intersection, Alg. 2 binning, per-bin field + table generation and shading,
then the Eq. 5 exitance update and the bottom-up SVO refresh.  Path state
lives in HBM (``PathState`` holds torch tensors; numpy views on access).
"""

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _dev, _lib, core, guiding

PATH_STREAM_SPACE = 4
BIN_STREAM_TAG = 1


@dataclass
class GuidingConfig:
    """Guiding knobs (wavefront.py:21-50); defaults mirror the reference."""

    l_min: int = 5
    c_ray: int = 512
    field_res: int = 128
    guided_depths: int = 4
    max_depth: int = 5
    product: bool = False
    jitter: bool = True
    blur_sigma: float = 1.0
    epsilon: float = guiding.EPSILON_FLOOR
    russian_roulette: bool = False
    rr_depth: int = 3
    seed: int = 0

    def validate(self, svo_depth=None):
        if self.field_res not in (16, 32, 64, 128):
            raise ValueError("field_res must be one of 16, 32, 64, 128")
        if self.c_ray < 1:
            raise ValueError("c_ray must be >= 1")
        if self.guided_depths > self.max_depth:
            raise ValueError("guided_depths cannot exceed max_depth")
        if svo_depth is not None and self.l_min >= svo_depth:
            raise ValueError("l_min must be below the SVO depth")

    def field_res_at(self, depth):
        return max(8, self.field_res >> (depth - 1))


_STATE = {
    # name: (dtype, trailing shape builder)
    "ray_o": (np.float64, lambda d: (3,)), "ray_d": (np.float64, lambda d: (3,)),
    "beta": (np.float64, lambda d: (3,)), "radiance": (np.float64, lambda d: (3,)),
    "key": (np.uint64, lambda d: ()), "ctr": (np.uint64, lambda d: ()),
    "alive": (np.uint8, lambda d: ()), "prev_pdf": (np.float64, lambda d: ()),
    # records: (D+1, P, 3) on the device (depth-major: one depth's records of
    # consecutive paths are contiguous); read back as the reference's (P, D+1, 3)
    "rec_pos": (np.float64, lambda d: (d + 1, 3)), "rec_T": (np.float64, lambda d: (d + 1, 3)),
    "emit_le": (np.float64, lambda d: (3,)), "emit_depth": (np.int32, lambda d: ()),
    # deepest record slot written this pass: slots above it are stale on the
    # device (the pass does not re-zero them) and read back as zeros
    "n_rec": (np.uint8, lambda d: ()),
}


_RECORDS = ("rec_pos", "rec_T")


class PathState:
    """SoA wavefront state in HBM (wavefront.py:53-71).  Attribute access
    returns numpy copies; ``dev[name]`` is the device tensor."""

    def __init__(self, n_paths, max_depth, camera_pos):
        self.n = int(n_paths)
        self.max_depth = int(max_depth)
        self.dev = {}
        for name, (dt, shp) in _STATE.items():
            if name in _RECORDS:
                self.dev[name] = _dev.zeros((self.max_depth + 1, self.n, 3), dt)
                continue
            self.dev[name] = _dev.zeros((self.n,) + shp(self.max_depth), dt)
        self.dev["beta"].fill_(1.0)
        self.dev["alive"].fill_(1)
        self.dev["prev_pdf"].fill_(-1.0)
        cp = np.asarray(camera_pos, dtype=np.float64)
        self.dev["rec_pos"][0, :] = _dev.upload(cp)
        self.pixel = np.arange(self.n, dtype=np.int64)

    def abi(self):
        p = _lib.Paths()
        p.n = self.n
        p.max_depth = self.max_depth
        for name in _STATE:
            setattr(p, name, self.dev[name].data_ptr())
        p.rec_depth_major = 1
        return p

    def set(self, name, host):
        """Upload a host array in the reference's layout ((P, D+1, 3) for the
        records)."""
        a = np.asarray(host, dtype=_STATE[name][0])
        t = _dev.upload(np.ascontiguousarray(a.transpose(1, 0, 2)) if name in _RECORDS else a)
        self.dev[name].copy_(t.reshape(self.dev[name].shape))

    def __getattr__(self, name):
        if name in _STATE and "dev" in self.__dict__:
            a = _dev.download(self.dev[name])
            if name in _RECORDS:
                a = np.ascontiguousarray(a.transpose(1, 0, 2))
                n_rec = _dev.download(self.dev["n_rec"]).astype(np.int64)
                a[np.arange(a.shape[1])[None, :] > n_rec[:, None]] = 0.0
            return a.astype(bool) if name == "alive" else a
        raise AttributeError(name)


@dataclass
class SpatialBin:
    node: int
    level: int
    members: np.ndarray


@dataclass
class PassStats:
    bins_per_depth: list = field(default_factory=list)
    rays_per_depth: list = field(default_factory=list)
    material_groups: list = field(default_factory=list)
    live_per_depth: list = field(default_factory=list)
    deposits: int = 0


def partition_material(mat_ids, path_idx):
    """Stable grouping of live paths by material id (stats only)."""
    order = np.argsort(mat_ids, kind="stable")
    srt = mat_ids[order]
    return {int(m): path_idx[order[np.searchsorted(srt, m, "left"):np.searchsorted(srt, m, "right")]]
            for m in np.unique(mat_ids)}


def partition_spatial(svo, positions, path_idx, l_min, c_ray):
    """Alg. 2 positional binning (wavefront.py:98-157) on the device; returns
    SpatialBin records ordered by node id with members in path order."""
    if l_min >= svo.depth:
        raise ValueError("l_min must be below the SVO depth")
    path_idx = np.asarray(path_idx)
    n = len(path_idx)
    if n == 0:
        return []
    pos = _dev.upload(np.asarray(positions, dtype=np.float64).reshape(n, 3))
    pidx = _dev.upload(path_idx, np.int32)
    cap = n
    node = _dev.empty((cap,), np.int32)
    start = _dev.empty((cap,), np.int32)
    count = _dev.empty((cap,), np.int32)
    members = _dev.empty((n,), np.int32)
    nb = _dev.zeros((1,), np.int32)
    ws = _dev.workspace(_lib.load().wfpg_partition_workspace_bytes(n, svo.node_count))
    _lib.call("wfpg_partition_spatial", C.byref(svo.abi()), _lib.ptr(pos), _lib.ptr(pidx), n,
              None, int(l_min), int(c_ray), _lib.ptr(node), _lib.ptr(start), _lib.ptr(count),
              _lib.ptr(members), _lib.ptr(nb), cap, _lib.ptr(ws), ws.numel(), _dev.stream())
    k = int(_dev.download(nb)[0])
    node_h = _dev.download(node[:k]).astype(np.int64)
    start_h = _dev.download(start[:k])
    count_h = _dev.download(count[:k])
    mem_h = _dev.download(members).astype(np.int64)
    levels = np.searchsorted(svo.level_off, node_h, side="right") - 1
    return [SpatialBin(int(node_h[b]), int(levels[b]), mem_h[start_h[b]:start_h[b] + count_h[b]])
            for b in range(k)]


def bin_stream_id(sample_index, depth, node_id):
    sid = ((sample_index * 64 + depth) << 32) + node_id
    return sid * PATH_STREAM_SPACE + BIN_STREAM_TAG


def bin_stream(cfg_seed, sample_index, depth, node_id):
    return core.RngStream(cfg_seed, bin_stream_id(sample_index, depth, node_id))


def _release_graph(ptr):
    try:
        _lib.load().wfpg_graph_release(_lib.C.c_void_p(ptr))
    except Exception:  # interpreter shutdown
        pass


class PassRunner:
    """Owns the device buffers of repeated passes with one configuration
    (path state, frame, workspace) so that steady-state rendering allocates
    nothing.  ``render_pass`` uses a cached runner per (scene, svo, cfg)."""

    def __init__(self, scene, svo, cfg, n_samples=1, deterministic=True, pixel_offset=0,
                 n_pixels=None, leaf_acc=None, use_graph=True, collect_bin_image=False,
                 comm=None, wire_capacity=0, skip_unguided_bins=False):
        cam = scene.camera
        self.scene = scene
        self.svo = svo
        self.cfg = cfg
        self.n_samples = int(n_samples)
        self.n_pix = int(n_pixels) if n_pixels else cam.width * cam.height
        self.P = self.n_pix * self.n_samples
        self.cam = cam.as_abi()
        self.state = PathState(self.P, cfg.max_depth, cam.position)
        self.frame = _dev.zeros((self.n_pix, 3), np.float64)
        self.pc = _lib.PassConfig()
        pc = self.pc
        pc.l_min, pc.c_ray, pc.field_res = int(cfg.l_min), int(cfg.c_ray), int(cfg.field_res)
        pc.guided_depths, pc.max_depth = int(cfg.guided_depths), int(cfg.max_depth)
        pc.product, pc.jitter = int(bool(cfg.product)), int(bool(cfg.jitter))
        pc.blur_sigma, pc.epsilon = float(cfg.blur_sigma), float(cfg.epsilon)
        pc.russian_roulette, pc.rr_depth = int(bool(cfg.russian_roulette)), int(cfg.rr_depth)
        pc.seed = int(cfg.seed) & 0xFFFFFFFFFFFFFFFF
        pc.n_samples = self.n_samples
        pc.deterministic = 1 if deterministic else 0
        radius, taps = guiding.blur_params(cfg.blur_sigma)
        pc.blur_radius = radius
        for i, w in enumerate(taps[:2 * radius + 1] if radius else []):
            pc.blur_w[i] = float(w)
        pc.upper_dirs = guiding.upper_dirs_device().data_ptr() if cfg.product else None
        pc.pixel_offset = int(pixel_offset)
        pc.n_pixels = self.n_pix
        self.leaf_acc = leaf_acc
        pc.leaf_acc = leaf_acc.data_ptr() if leaf_acc is not None else None
        pc.use_graph = 1 if use_graph else 0  # replay the pass as a CUDA graph
        # the bins of non-guided depths only feed PassStats: callers that do
        # not read those stats may skip their Alg. 2 passes (same frames / SVO)
        pc.skip_unguided_bins = 1 if skip_unguided_bins else 0
        # depth-1 bin node per pixel (wavefront.py:221,254-256)
        self.bin_image = _dev.empty((self.n_pix,), np.int32) if collect_bin_image else None
        pc.bin_image = self.bin_image.data_ptr() if collect_bin_image else None
        # multi-GPU (multigpu.Communicator): global binning of the guided
        # depths and the in-pass deposit exchange; this runner renders the
        # band [pixel_offset, pixel_offset + n_pixels) of rank comm.rank
        self.comm = comm
        pc.comm = comm.ptr if comm is not None else None
        pc.dep_wire_capacity = int(wire_capacity)
        self.svo_abi = svo.abi() if svo is not None else None
        self.ws = None
        self._fit_workspace()
        self.stats = _lib.PassStats()

    def _fit_workspace(self):
        """(Re)size the pass workspace for the current configuration; a new
        workspace drops the old one's captured graph."""
        import weakref

        nbytes = _lib.load().wfpg_render_workspace_bytes(
            C.byref(self.scene.abi()), C.byref(self.svo_abi) if self.svo is not None else None,
            C.byref(self.cam), C.byref(self.pc))
        if self.ws is not None and self.ws.numel() >= nbytes:
            return
        if self.ws is not None:
            self._ws_finalizer()
        self.ws = _dev.workspace(nbytes)
        # drop this workspace's captured graph when the runner goes away
        self._ws_finalizer = weakref.finalize(self, _release_graph, self.ws.data_ptr())

    def set_ownership(self, bins_per_depth, margin=1.05, slack=64, first_depth=2):
        """Multi-GPU bin ownership for the guided depths >= first_depth
        (wfpg_pass_config.own_bins): each rank generates 1/W of the bins and
        the values are all-gathered.  bins_per_depth: the global bin counts of
        a previous pass (PassStats.bins_per_depth, identical on every rank);
        the estimate E = margin * bins + slack, and a pass whose bins exceed
        W * ceil(E / W) falls back to the exact needed-bin policy."""
        for d in range(32):
            self.pc.own_bins[d] = 0
        if self.comm is None:
            return
        for d, b in enumerate(bins_per_depth, start=1):
            if first_depth <= d <= min(31, int(self.cfg.guided_depths)):
                self.pc.own_bins[d] = int(b * margin) + int(slack)
        self._fit_workspace()

    def launch(self, sample_index, want_stats=True, sample_list=None):
        """Enqueue one pass; with want_stats the call synchronises and fills self.stats.
        sample_list: the pass's sample indices when they are not sample_index,
        sample_index + 1, ... (any list, as the reference accepts)."""
        self.pc.sample_index = int(sample_index)
        if sample_list is not None:
            lst = np.asarray(sample_list, dtype=np.int64).reshape(-1)
            if len(lst) != self.n_samples or lst[0] != sample_index:
                raise ValueError("sample_list must hold n_samples entries starting at sample_index")
            if getattr(self, "_samples_dev", None) is None:
                self._samples_dev = _dev.empty((self.n_samples,), np.int64)
            self._samples_dev.copy_(_dev.upload(lst), non_blocking=False)
            self.pc.sample_list = self._samples_dev.data_ptr()
        else:
            self.pc.sample_list = None
        _lib.call("wfpg_render_pass", C.byref(self.scene.abi()),
                  C.byref(self.svo_abi) if self.svo is not None else None, C.byref(self.cam),
                  C.byref(self.pc), C.byref(self.state.abi()), _lib.ptr(self.frame),
                  C.byref(self.stats) if want_stats else None, _lib.ptr(self.ws),
                  self.ws.numel(), _dev.stream())

    def pass_stats(self):
        s = self.stats
        st = PassStats()
        for d in range(s.depths_run):
            st.live_per_depth.append(int(s.live_per_depth[d]))
            if self.svo is not None:
                st.bins_per_depth.append(int(s.bins_per_depth[d]))
                st.rays_per_depth.append(int(s.rays_per_depth[d]))
                groups = {m: int(s.mat_groups[d][m]) for m in range(64) if s.mat_groups[d][m]}
                st.material_groups.append(groups)
        st.deposits = int(s.deposits)
        return st


_RUNNERS = {}


def _camera_key(cam):
    return (tuple(cam.position.tolist()), tuple(cam.target.tolist()), tuple(cam.up.tolist()),
            cam.vfov_deg, cam.width, cam.height)


def _runner(scene, svo, cfg, n_samples, collect_bin_image=False):
    # the camera is part of the key: the reference reads scene.camera on every
    # pass, so a reassigned camera must not replay the old view
    key = (id(scene), id(svo), tuple(sorted(vars(cfg).items())), n_samples,
           bool(collect_bin_image), _camera_key(scene.camera))
    r = _RUNNERS.get(key)
    if r is None or r.scene is not scene or r.svo is not svo:
        _RUNNERS.clear()  # one live configuration at a time keeps HBM bounded
        r = PassRunner(scene, svo, cfg, n_samples, collect_bin_image=collect_bin_image)
        _RUNNERS[key] = r
    return r


def pinned_frame(scene):
    """A page-locked (H, W, 3) float64 host array for render_pass(out=...):
    the frame then arrives by one DMA instead of a pageable copy."""
    t = _dev.torch()
    cam = scene.camera
    return t.empty((cam.height, cam.width, 3), dtype=t.float64, pin_memory=True).numpy()


def render_pass(scene, svo, cfg, sample_indices, collect_bin_image=False, out=None):
    """One wavefront pass over every pixel for each sample index (any list;
    bins use the first index's streams); returns (frame (H,W,3), PassStats).  ``out`` (optional, e.g.
    from pinned_frame) receives the frame instead of a fresh array."""
    samples = np.asarray(sample_indices, dtype=np.int64).reshape(-1)
    if len(samples) == 0:
        raise ValueError("render_pass needs at least one sample index")
    if svo is not None:
        cfg.validate(svo.depth)
    collect = bool(collect_bin_image) and svo is not None
    r = _runner(scene, svo, cfg, len(samples), collect)
    # any sample list (wavefront.py:207-215): consecutive lists need no table
    consecutive = bool(np.all(np.diff(samples) == 1))
    r.launch(int(samples[0]), sample_list=None if consecutive else samples)
    cam = scene.camera
    if out is not None:
        t = _dev.torch()
        dst = t.from_numpy(out).view(-1, 3)
        dst.copy_(r.frame, non_blocking=dst.is_pinned())
        t.cuda.current_stream().synchronize()
        frame = out
    else:
        frame = _dev.download(r.frame).reshape(cam.height, cam.width, 3)
    if collect_bin_image:
        if collect:
            img = _dev.download(r.bin_image).astype(np.int64).reshape(cam.height, cam.width)
        else:
            img = np.full((cam.height, cam.width), -1, dtype=np.int64)
        return frame, r.pass_stats(), img
    return frame, r.pass_stats()


class _Event:
    """A native cudaEvent_t (wfpg_event_create) for the overlap chain."""

    def __init__(self):
        self.h = C.c_void_p()
        _lib.call("wfpg_event_create", C.byref(self.h))

    def __del__(self):  # pragma: no cover - interpreter shutdown
        try:
            _lib.load().wfpg_event_destroy(self.h)
        except Exception:
            pass


class PassPipeline:
    """Consecutive passes of one configuration on two streams that overlap
    where the reference's pass order allows (wfpg_pass_config ev_*): pass
    i+1's ray generation, depth-1 intersection and binning run while pass i
    finishes its last depth and its exitance update; every SVO access (the
    Alg. 2 counters, the exitance read by the fields and written by the
    update) still happens in pass order, so the results equal calling
    render_pass once per sample, bit for bit.  Two PassRunners alternate
    (two path states, frames and workspaces); ``launch(sample)`` returns the
    runner of that pass; ``join()`` makes the caller's stream wait for all
    of them."""

    def __init__(self, scene, svo, cfg, runners=None):
        t = _dev.torch()
        if svo is not None:
            cfg.validate(svo.depth)
        self.runners = runners or [PassRunner(scene, svo, cfg) for _ in range(2)]
        self.streams = [t.cuda.Stream() for _ in self.runners]
        self.rec_counters = [_Event() for _ in self.runners]
        self.rec_svo = [_Event() for _ in self.runners]
        self.done = [t.cuda.Event() for _ in self.runners]
        n = len(self.runners)
        for k, r in enumerate(self.runners):
            prev = (k - 1) % n
            r.pc.ev_wait_counters = self.rec_counters[prev].h.value
            r.pc.ev_wait_svo = self.rec_svo[prev].h.value
            r.pc.ev_rec_counters = self.rec_counters[k].h.value
            r.pc.ev_rec_svo = self.rec_svo[k].h.value
        self.k = 0
        self._forked = False

    def _fork(self):
        t = _dev.torch()
        cur = t.cuda.current_stream()
        for s in self.streams:
            s.wait_stream(cur)
        self._forked = True

    def launch(self, sample, want_stats=False, before=None):
        """Enqueue the next pass; `before` (optional) is a torch event the
        pass's stream waits for first (e.g. its frame's previous copy)."""
        t = _dev.torch()
        if not self._forked:
            self._fork()
        slot = self.k % len(self.runners)
        self.k += 1
        r = self.runners[slot]
        with t.cuda.stream(self.streams[slot]):
            if before is not None:
                self.streams[slot].wait_event(before)
            r.launch(int(sample), want_stats=want_stats)
            self.done[slot].record(self.streams[slot])
        return slot, r

    def join(self):
        t = _dev.torch()
        cur = t.cuda.current_stream()
        for s in self.streams:
            cur.wait_stream(s)
        self._forked = False


class FramePipeline:
    """Consecutive single-sample passes whose frames arrive in page-locked host
    memory: the passes run as a PassPipeline (pass i+1's start overlapping
    pass i's end on a second stream), the device-to-host copy of pass i runs
    on a copy stream overlapped with pass i+1, and a runner only writes its
    frame again once that frame's previous copy has finished.  The SVO
    learning sequence is exactly that of calling render_pass once per
    sample.  ``run(samples)`` yields (sample_index, frame, stats) with the
    frame an (H, W, 3) view of a pinned buffer that stays valid until the
    iterator advances twice more; stats are collected only if want_stats.
    """

    def __init__(self, scene, svo, cfg, want_stats=False):
        t = _dev.torch()
        self.scene, self.svo, self.cfg = scene, svo, cfg
        self.want_stats = want_stats
        self.pipe = PassPipeline(scene, svo, cfg)
        self.runners = self.pipe.runners
        self.host = [pinned_frame(scene) for _ in range(2)]
        self.copy_stream = t.cuda.Stream()
        self.copy_done = [t.cuda.Event() for _ in range(2)]
        self.copied = [False, False]

    def _submit(self, k, sample):
        t = _dev.torch()
        slot = k % 2
        before = self.copy_done[slot] if self.copied[slot] else None
        slot, r = self.pipe.launch(int(sample), want_stats=self.want_stats, before=before)
        self.copy_stream.wait_event(self.pipe.done[slot])
        with t.cuda.stream(self.copy_stream):
            dst = t.from_numpy(self.host[slot]).view(-1, 3)
            dst.copy_(r.frame, non_blocking=True)
        self.copy_done[slot].record(self.copy_stream)
        self.copied[slot] = True
        return slot

    def _deliver(self, slot, sample):
        self.copy_done[slot].synchronize()
        stats = self.runners[slot].pass_stats() if self.want_stats else None
        return int(sample), self.host[slot], stats

    def run(self, sample_indices):
        pending = None
        for k, s in enumerate(sample_indices):
            slot = self._submit(k, s)
            if pending is not None:
                yield self._deliver(*pending)
            pending = (slot, s)
        if pending is not None:
            yield self._deliver(*pending)
        self.pipe.join()


def render_sample(scene, svo, cfg, sample_index):
    frame, _ = render_pass(scene, svo, cfg, [sample_index])
    return frame


def update_exitance(state, svo, deterministic=True):
    """Eq. 5 back-propagation of emitter radiance into the SVO leaves
    (wavefront.py:286-332).  Returns the dirty leaf ids (sorted int64, the
    reference's return value, which its caller hands to svo.propagate_up);
    the device refresh of the touched subtrees has already run, so that
    call is a no-op refresh here.  ``update_exitance.last_deposits`` holds
    the deposit count."""
    lo, hi = int(svo.level_off[svo.depth]), int(svo.level_off[svo.depth + 1])
    t = _dev.torch()
    before = t.stack([svo.dev("weight_a")[lo:hi], svo.dev("weight_b")[lo:hi]]).clone()
    n_dep = _dev.zeros((1,), np.int32)
    ws = _dev.workspace(_lib.load().wfpg_update_exitance_workspace_bytes(state.n, state.max_depth))
    _lib.call("wfpg_update_exitance", C.byref(svo.abi()), C.byref(state.abi()),
              1 if deterministic else 0, _lib.ptr(n_dep), _lib.ptr(ws), ws.numel(),
              _dev.stream())
    after = t.stack([svo.dev("weight_a")[lo:hi], svo.dev("weight_b")[lo:hi]])
    # every deposit adds 1 to its leaf's side weight, so the touched leaves are
    # exactly those whose weights changed
    dirty = t.nonzero((after != before).any(dim=0)).reshape(-1) + lo
    update_exitance.last_deposits = int(_dev.download(n_dep)[0])
    return _dev.download(dirty).astype(np.int64)


update_exitance.last_deposits = 0
