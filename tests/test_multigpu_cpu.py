"""Multi-GPU host logic on CPU (gloo, world size 2): pixel bands, global RNG
streams, and the leaf-exitance all-reduce that keeps every rank's SVO equal."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2405_06997_b200 import core, multigpu


def test_bands_cover_the_image_once():
    for n_pix in (1, 7, 64 * 64, 1920 * 1080 * 4):
        for world in (1, 2, 3, 4, 8):
            spans = [multigpu.band(n_pix, r, world) for r in range(world)]
            assert spans[0][0] == 0
            assert sum(n for _, n in spans) == n_pix
            for (o1, n1), (o2, _) in zip(spans, spans[1:]):
                assert o1 + n1 == o2


def test_band_paths_use_global_rng_streams():
    """wavefront.py:214: key = stream_key(seed, (sample * n_pix + pixel) * 4) with the
    global pixel index, so a path's draws do not depend on the rank layout."""
    n_pix, seed, sample = 97 * 13, 5, 3
    full = core.stream_key(np.uint64(seed),
                           ((sample * n_pix + np.arange(n_pix)) * 4).astype(np.uint64))
    for world in (2, 4):
        keys = []
        for r in range(world):
            off, n = multigpu.band(n_pix, r, world)
            pix = off + np.arange(n)
            keys.append(core.stream_key(np.uint64(seed),
                                        ((sample * n_pix + pix) * 4).astype(np.uint64)))
        assert np.array_equal(np.concatenate(keys), full)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_leaves, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(100 + rank)
    acc = torch.from_numpy(rng.random(8 * n_leaves))
    multigpu.ExitanceAllReduce.reduce(acc)
    out[rank] = acc.numpy().copy()
    dist.destroy_process_group()


def test_leaf_accumulator_allreduce_gloo():
    world, n_leaves = 2, 1000
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, n_leaves, out), nprocs=world, join=True)
        res = [out[r] for r in range(world)]
    expect = sum(np.random.default_rng(100 + r).random(8 * n_leaves) for r in range(world))
    for r in range(world):
        np.testing.assert_allclose(res[r], expect, rtol=1e-15)
    # every rank ends with the same accumulator -> identical SVO state
    assert np.array_equal(res[0], res[1])
    sa, sb, wa, wb = multigpu.leaf_acc_planes(res[0], n_leaves)
    assert sa.shape == (n_leaves, 3) and wb.shape == (n_leaves,)


@pytest.mark.parametrize("world", [2])
def test_summed_deposits_equal_single_rank_deposits(world):
    """Splitting a deposit list across ranks and summing per-leaf accumulators
    gives the same weights as one rank splatting all deposits (sums equal up to
    fp reassociation), which is what makes the per-pass all-reduce exact."""
    rng = np.random.default_rng(3)
    n_leaves, m = 50, 2000
    leaf = rng.integers(0, n_leaves, m)
    rad = rng.random((m, 3))
    side = rng.random(m) < 0.5
    full = np.zeros((n_leaves, 3))
    wfull = np.zeros(n_leaves)
    np.add.at(full, leaf[side], rad[side])
    np.add.at(wfull, leaf[side], 1.0)
    parts = np.array_split(np.arange(m), world)
    acc = np.zeros((n_leaves, 3))
    wacc = np.zeros(n_leaves)
    for p in parts:
        s = side[p]
        np.add.at(acc, leaf[p][s], rad[p][s])
        np.add.at(wacc, leaf[p][s], 1.0)
    assert np.array_equal(wacc, wfull)
    np.testing.assert_allclose(acc, full, rtol=1e-13)


def _gather_worker(rank, world, port, sizes, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(200 + rank)
    n = sizes[rank]
    leaf = torch.from_numpy(rng.integers(-1, 1000, n).astype(np.int32))
    dirs = torch.from_numpy(rng.random((n, 3)))
    rad = torch.from_numpy(rng.random((n, 3)))
    g = multigpu.DepositExchange.gather(leaf, dirs, rad)
    out[rank] = tuple(t.numpy().copy() for t in g)
    dist.destroy_process_group()


@pytest.mark.parametrize("sizes", [(5, 3), (0, 4), (7, 0), (0, 0)])
def test_deposit_gather_is_rank_ordered_concatenation(sizes):
    """DepositExchange.gather returns every rank's list in rank order (= global
    path order for contiguous bands), bit-exact, whatever the lengths."""
    world = len(sizes)
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_gather_worker, args=(world, port, sizes, out), nprocs=world, join=True)
        res = [out[r] for r in range(world)]
    exp = []
    for r, n in enumerate(sizes):
        rng = np.random.default_rng(200 + r)
        exp.append((rng.integers(-1, 1000, n).astype(np.int32), rng.random((n, 3)),
                    rng.random((n, 3))))
    for k in range(3):
        want = np.concatenate([e[k] for e in exp])
        for r in range(world):
            assert np.array_equal(res[r][k], want)
    assert res[0][0].dtype == np.int32


def test_rank_ordered_deposits_reproduce_the_single_rank_splat():
    """np.add.at over the rank-ordered concatenation IS the single-rank splat
    (same order, same arithmetic) — bitwise, unlike summed partial sums."""
    rng = np.random.default_rng(9)
    n_leaves, m = 40, 3000
    leaf = rng.integers(0, n_leaves, m)
    rad = rng.random((m, 3)) * 1e3
    full = np.zeros((n_leaves, 3))
    np.add.at(full, leaf, rad)
    parts = np.array_split(np.arange(m), 3)
    cat = np.concatenate(parts)
    acc = np.zeros((n_leaves, 3))
    np.add.at(acc, leaf[cat], rad[cat])
    assert np.array_equal(acc.view(np.uint64), full.view(np.uint64))
