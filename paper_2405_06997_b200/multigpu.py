"""Multi-GPU image tiling with an exitance all-reduce.

One process per GPU.  Rank r renders the pixel band
[r * n_pix / world, (r + 1) * n_pix / world) of the global image; paths use
global pixel indices for their RNG streams, so a path draws exactly what it
draws on one GPU.  The SVO structure is built identically on every rank.
After each pass every rank has splatted its own Eq. 5 deposits into a zeroed
per-leaf buffer (4 planes: sum_a, sum_b, weight_a, weight_b); the buffers are
summed with one NCCL all-reduce and added into every rank's leaf
accumulators, followed by the same bottom-up refresh on every rank, so all
ranks hold the same exitance cache for the next pass.  Binning (Alg. 2) is
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


def leaf_acc_planes(acc, n_leaves):
    """Split a flat accumulator into (sum_a (L,3), sum_b (L,3), weight_a, weight_b)."""
    a = np.asarray(acc)
    L = n_leaves
    return (a[:3 * L].reshape(L, 3), a[3 * L:6 * L].reshape(L, 3), a[6 * L:7 * L], a[7 * L:8 * L])
