"""Multi-GPU image tiling with an exitance exchange.

One process per GPU.  Rank r renders the pixel band
[r * n_pix / world, (r + 1) * n_pix / world) of the global image; paths use
global pixel indices for their RNG streams, so a path draws exactly what it
draws on one GPU.  The SVO structure is built identically on every rank.
After each pass every rank has splatted its own Eq. 5 deposits into a zeroed
per-leaf buffer (4 planes: sum_a, sum_b, weight_a, weight_b); the buffers are
summed with one NCCL all-reduce and added into every rank's leaf
accumulators, followed by the same bottom-up refresh on every rank, so all
ranks hold the same exitance cache for the next pass (ExitanceAllReduce:
432 MB per pass at depth 10).

DepositExchange is the sparse alternative the survey recommends and the one
bench.py uses: each rank exports its pass's deposit list (leaf, direction,
radiance; ~0.03 deposits per path, a few MB at 1080p) instead of splatting
it, the lists are all-gathered (counts first, then one padded
all_gather_into_tensor), concatenated in rank order — which is global path
order, because bands are contiguous pixel ranges — and splatted
deterministically + refreshed on every rank.  The SVO update is then bitwise
the 1-GPU update of the same paths.  Binning (Alg. 2) is
per rank: bins depend on the rank's own paths, so multi-GPU images agree with
the 1-GPU image statistically, not per pixel.
"""

import ctypes as C

import numpy as np

from . import _dev, _lib


def band(n_pix, rank, world):
    """(pixel_offset, n_pixels) of a rank's contiguous band."""
    lo = n_pix * rank // world
    hi = n_pix * (rank + 1) // world
    return lo, hi - lo


class ExitanceAllReduce:
    def __init__(self, svo, group=None):
        self.svo = svo
        self.group = group
        self.n_leaves = svo.leaf_count
        self.acc = _dev.zeros((8 * self.n_leaves,), np.float64)

    @staticmethod
    def reduce(acc, group=None):
        import torch.distributed as dist

        dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=group)
        return acc

    def apply(self):
        _lib.call("wfpg_svo_apply_leaf_acc", C.byref(self.svo.abi()), _lib.ptr(self.acc),
                  _dev.stream())

    def reduce_and_apply(self, runner=None):
        self.reduce(self.acc, self.group)
        self.apply()


class DepositExchange:
    """Sparse per-pass exitance exchange (see module doc).  Pass it to
    PassRunner(deposit_sink=...); call exchange(runner) after each pass."""

    PACK = 7  # leaf (as float64, exact below 2^53), dir xyz, rad xyz

    def __init__(self, svo, group=None):
        self.svo = svo
        self.group = group
        self.capacity = 0
        self.dirty = _dev.zeros((max(svo.node_count, 1),), np.uint8)
        self._ws = None

    def bind(self, pc, capacity):
        """Allocate the export buffers (capacity deposits) and point the pass
        configuration at them."""
        if capacity > self.capacity:
            self.capacity = int(capacity)
            self.leaf = _dev.empty((self.capacity,), np.int32)
            self.dir = _dev.empty((self.capacity, 3), np.float64)
            self.rad = _dev.empty((self.capacity, 3), np.float64)
            self.count = _dev.zeros((1,), np.int32)
        pc.dep_leaf, pc.dep_dir = self.leaf.data_ptr(), self.dir.data_ptr()
        pc.dep_rad, pc.dep_count = self.rad.data_ptr(), self.count.data_ptr()
        pc.dep_capacity = self.capacity

    def local(self):
        n = int(_dev.download(self.count)[0])
        return self.leaf[:n], self.dir[:n], self.rad[:n]

    @classmethod
    def gather(cls, leaf, dirs, rad, group=None):
        """All-gather variable-length deposit lists; returns the concatenation
        in rank order as (leaf int32 (n,), dir (n,3), rad (n,3)) tensors on the
        input's device.  Works for any backend (gloo on CPU in the tests)."""
        import torch
        import torch.distributed as dist

        world = dist.get_world_size(group)
        home = leaf.device
        if dist.get_backend(group) == "gloo" and home.type != "cpu":
            # gloo collectives on host copies (1-GPU functional runs)
            out = cls.gather(leaf.cpu(), dirs.cpu(), rad.cpu(), group)
            return tuple(t.to(home) for t in out)
        n = torch.tensor([leaf.shape[0]], dtype=torch.int64, device=leaf.device)
        counts = [torch.zeros_like(n) for _ in range(world)]
        dist.all_gather(counts, n, group=group)
        counts = [int(c.item()) for c in counts]
        cap = max(max(counts), 1)
        pack = torch.zeros((cap, cls.PACK), dtype=torch.float64, device=leaf.device)
        k = leaf.shape[0]
        if k:
            pack[:k, 0] = leaf.to(torch.float64)
            pack[:k, 1:4] = dirs
            pack[:k, 4:7] = rad
        everyone = torch.empty((world * cap, cls.PACK), dtype=torch.float64, device=leaf.device)
        dist.all_gather_into_tensor(everyone, pack, group=group)
        rows = torch.cat([everyone[r * cap:r * cap + c] for r, c in enumerate(counts)])
        return (rows[:, 0].to(torch.int32).contiguous(), rows[:, 1:4].contiguous(),
                rows[:, 4:7].contiguous())

    def apply(self, leaf, dirs, rad):
        """Deterministic splat of the gathered deposits + dirty refresh."""
        n = int(leaf.shape[0])
        s = self.svo.abi()
        if n:
            need = _lib.load().wfpg_accumulate_workspace_bytes(n)
            if self._ws is None or self._ws.numel() < need:
                self._ws = _dev.workspace(need)
            _lib.call("wfpg_svo_accumulate", C.byref(s), _lib.ptr(leaf), _lib.ptr(dirs),
                      _lib.ptr(rad), n, None, 1, _lib.ptr(self._ws), self._ws.numel(),
                      _dev.stream())
        _lib.call("wfpg_svo_refresh_leaves", C.byref(s), _lib.ptr(leaf) if n else None, n,
                  _lib.ptr(self.dirty), _dev.stream())
        return n

    def exchange(self, runner=None):
        leaf, dirs, rad = self.local()
        if self.group is not None or _dist_ready():
            leaf, dirs, rad = self.gather(leaf, dirs, rad, self.group)
        return self.apply(leaf, dirs, rad)

    reduce_and_apply = exchange


def _dist_ready():
    try:
        import torch.distributed as dist

        return dist.is_available() and dist.is_initialized()
    except ImportError:  # pragma: no cover
        return False


def leaf_acc_planes(acc, n_leaves):
    """Split a flat accumulator into (sum_a (L,3), sum_b (L,3), weight_a, weight_b)."""
    a = np.asarray(acc)
    L = n_leaves
    return (a[:3 * L].reshape(L, 3), a[3 * L:6 * L].reshape(L, 3), a[6 * L:7 * L], a[7 * L:8 * L])
