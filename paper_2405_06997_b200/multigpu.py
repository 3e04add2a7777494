"""Multi-GPU image tiling: one process per GPU, pixel bands,
and the exchange steps of the render pass behind one communicator.

Rank r renders the pixel band [r * n_pix / world, (r + 1) * n_pix / world)
of the image; paths use global pixel indices for their RNG streams, so a path
draws exactly what it draws on one GPU.  The SVO structure is built
identically on every rank.  A pass given a communicator
(``PassRunner(comm=...)``, include/wfpg_b200.h ``wfpg_pass_config.comm``) is
the 1-GPU pass restricted to the band, path for path:

* guided depths bin GLOBALLY: every rank all-gathers the Alg. 2 start nodes
  of all ranks' lambert hits (one int32 per path), runs the same partition
  and takes each bin's origin from the rank owning that path (an all-reduce
  of bit patterns; wavefront.py:98-195).  At depth 1 a rank generates the
  fields of only the bins its own paths belong to (they split with the
  image); at deeper depths, after ``PassRunner.set_ownership``, rank r
  generates a contiguous 1/W of the bins and the floored values of all bins
  are all-gathered, the other tables derived locally (bitwise the owners');
* after the last depth every rank's Eq. 5 deposits are all-gathered and
  splatted in global path order (wavefront.py:286-332), so every rank's SVO
  equals the 1-GPU SVO bit for bit.

With NCCL the collectives are enqueued by the native library on the pass
stream and captured into the pass's CUDA graph: no torch op, host copy or
host synchronisation per pass (one event wait on the previous pass, which
decides whether its deposit wire overflowed).  ``Communicator.host`` runs the
same steps through a Python exchange callback — over torch.distributed (gloo
on host copies) or between threads of one process (``ThreadGroup``, used by
the single-GPU tests to run W ranks' passes side by side).

``ExitanceAllReduce`` is the dense alternative the north star names (one
all-reduce of the 8 per-leaf accumulator planes per pass, then a full
bottom-up refresh); it is exact up to fp summation order.
"""

import ctypes as C
import threading

import numpy as np

from . import _dev, _lib


def band(n_pix, rank, world):
    """(pixel_offset, n_pixels) of a rank's contiguous band."""
    lo = n_pix * rank // world
    hi = n_pix * (rank + 1) // world
    return lo, hi - lo


_DTYPES = {0: ("int32", 4), 1: ("int64", 8), 2: ("float64", 8)}  # u64 travels as int64 bits


class Communicator:
    """Owner of a native wfpg_comm (see the module doc)."""

    def __init__(self, handle, world, rank, kind, keep=None):
        self.handle = handle
        self.world = int(world)
        self.rank = int(rank)
        self.kind = kind
        self._keep = keep  # the ctypes callback must outlive the communicator

    @property
    def ptr(self):
        return self.handle.value

    @classmethod
    def nccl(cls, group=None):
        """NCCL communicator over the torch.distributed group (the unique id
        travels over the group; the collectives themselves are the library's)."""
        import torch.distributed as dist

        lib = _lib.load()
        if not lib.wfpg_comm_nccl_available():
            raise _lib.WfpgError("libnccl.so.2 is not loadable")
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        uid = (C.c_uint8 * 128)()
        if rank == 0:
            _lib.call("wfpg_comm_nccl_unique_id", uid)
        box = [bytes(uid) if rank == 0 else None]
        dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group else 0,
                                   group=group)
        uid = (C.c_uint8 * 128).from_buffer_copy(box[0])
        h = C.c_void_p()
        _lib.call("wfpg_comm_init_nccl", world, rank, uid, C.byref(h))
        return cls(h, world, rank, "nccl")

    @classmethod
    def host(cls, world, rank, exchange):
        """Host-exchange communicator; exchange(op, send_tensor) -> recv_tensor
        performs the collective on torch tensors (op 0 all-gather, 1 all-reduce
        sum) and is called with the pass stream synchronised."""
        t = _dev.torch()

        def fn(user, op, send, recv, count, dtype, stream):
            try:
                name, size = _DTYPES[int(dtype)]
                n = int(count)
                dev = t.device("cuda", t.cuda.current_device())
                src = t.empty((n,), dtype=getattr(t, name), device=dev)
                _lib.call("wfpg_memcpy", C.c_void_p(src.data_ptr()), C.c_void_p(send),
                          n * size, C.c_void_p(stream))
                out = exchange(int(op), src)
                out = out.to(dev).contiguous()
                want = n * (self_world if int(op) == 0 else 1)
                if out.numel() != want:
                    return 3
                _lib.call("wfpg_memcpy", C.c_void_p(recv), C.c_void_p(out.data_ptr()),
                          want * size, C.c_void_p(stream))
                return 0
            except Exception as e:  # reported through the library's status
                import sys

                print(f"wfpg host exchange failed: {e!r}", file=sys.stderr)
                return 2

        self_world = int(world)
        cb = _lib.EXCHANGE_FN(fn)
        h = C.c_void_p()
        _lib.call("wfpg_comm_init_host", int(world), int(rank), cb, None, C.byref(h))
        return cls(h, world, rank, "host", keep=cb)

    @classmethod
    def torch_distributed(cls, group=None):
        """Host exchange over torch.distributed (gloo: host copies)."""
        import torch.distributed as dist

        world, rank = dist.get_world_size(group), dist.get_rank(group)
        return cls.host(world, rank, lambda op, x: dist_exchange(op, x, group))

    def settle(self):
        """Finish the deposit exchange of the last pass (wfpg_comm_settle)."""
        _lib.call("wfpg_comm_settle", self.handle)

    def close(self):
        if self.handle is not None and self.handle.value:
            _lib.call("wfpg_comm_destroy", self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter shutdown
        try:
            self.close()
        except Exception:
            pass


def dist_exchange(op, x, group=None):
    """One collective of the host-exchange protocol over torch.distributed:
    op 0 all-gather (rank order), op 1 all-reduce sum.  gloo collectives run
    on host copies."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    home = x.device
    if dist.get_backend(group) == "gloo" and home.type != "cpu":
        x = x.cpu()
    if op == 0:
        out = x.new_empty((world * x.numel(),))
        dist.all_gather_into_tensor(out, x.contiguous(), group=group)
    else:
        out = x.clone()
        dist.all_reduce(out, op=dist.ReduceOp.SUM, group=group)
    return out.to(home)


class ThreadGroup:
    """In-process exchange between W threads (each thread one rank, each with
    its own CUDA stream): the host-side barrier synchronises the ranks, the
    kernels never wait on each other.  For single-GPU tests of the banded
    multi-rank pass."""

    def __init__(self, world):
        self.world = int(world)
        self.slots = [None] * self.world
        self.barrier = threading.Barrier(self.world)

    def exchange(self, rank, op, x):
        import torch as t

        self.slots[rank] = x
        self.barrier.wait()
        if op == 0:
            out = t.cat([s.to(x.device) for s in self.slots])
        else:
            out = self.slots[0].clone()
            for s in self.slots[1:]:
                out += s.to(x.device)
        self.barrier.wait()  # every rank has read the slots
        return out

    def communicator(self, rank):
        return Communicator.host(self.world, rank, lambda op, x: self.exchange(rank, op, x))


class ExitanceAllReduce:
    """Dense per-leaf exitance all-reduce (the north star's formulation):
    render with PassRunner(leaf_acc=acc.acc), then reduce_and_apply()."""

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
