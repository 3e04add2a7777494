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


def _exchange_worker(rank, world, port, n, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(200 + rank)
    res = {}
    for name, dt in (("i32", np.int32), ("i64", np.int64), ("f64", np.float64)):
        x = torch.from_numpy((rng.random(n) * 1e6).astype(dt))
        res["gather_" + name] = multigpu.dist_exchange(0, x).numpy().copy()
        res["sum_" + name] = multigpu.dist_exchange(1, x).numpy().copy()
    out[rank] = res
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 5), (3, 1), (2, 0)])
def test_host_exchange_protocol_over_gloo(world, n):
    """The host-exchange protocol of a wfpg_comm over torch.distributed: op 0
    is the rank-ordered concatenation (global path order for contiguous
    bands), op 1 the element-wise sum, bit-exact for every wire dtype."""
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_exchange_worker, args=(world, port, n, out), nprocs=world, join=True)
        res = [out[r] for r in range(world)]
    for name, dt in (("i32", np.int32), ("i64", np.int64), ("f64", np.float64)):
        xs = [(np.random.default_rng(200 + r).random(n) * 1e6).astype(dt) for r in range(world)]
        # the generator is consumed in dtype order: regenerate the same way
        xs = []
        for r in range(world):
            rng = np.random.default_rng(200 + r)
            for nm, d in (("i32", np.int32), ("i64", np.int64), ("f64", np.float64)):
                v = (rng.random(n) * 1e6).astype(d)
                if nm == name:
                    xs.append(v)
        cat = np.concatenate(xs)
        tot = xs[0].copy()
        for v in xs[1:]:
            tot = tot + v
        for r in range(world):
            assert np.array_equal(res[r]["gather_" + name], cat)
            assert res[r]["gather_" + name].dtype == dt
            assert np.array_equal(res[r]["sum_" + name], tot)


def test_thread_group_exchange_on_host_tensors():
    """ThreadGroup (the single-GPU multi-rank tests' exchange): every rank
    thread gets the rank-ordered concatenation / the sum."""
    import threading

    world = 3
    g = multigpu.ThreadGroup(world)
    got = [None] * world

    def rank_main(r):
        x = torch.arange(4, dtype=torch.int64) + 10 * r
        got[r] = (g.exchange(r, 0, x).clone(), g.exchange(r, 1, x).clone())

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    cat = torch.cat([torch.arange(4) + 10 * r for r in range(world)])
    tot = sum(torch.arange(4) + 10 * r for r in range(world))
    for r in range(world):
        assert torch.equal(got[r][0], cat) and torch.equal(got[r][1], tot)


def test_bit_pattern_sum_is_an_exact_copy():
    """Bin origins travel as u64 bit patterns summed over ranks with exactly
    one non-zero contributor: the sum reproduces every double bit for bit
    (signed zeros, subnormals, NaN payloads included)."""
    vals = np.array([-0.0, 0.0, 5e-324, -1.5, np.inf, np.nan, 1e308], dtype=np.float64)
    bits = vals.view(np.int64)
    for owner in range(3):
        parts = [bits if r == owner else np.zeros_like(bits) for r in range(3)]
        tot = parts[0] + parts[1] + parts[2]
        assert np.array_equal(tot, bits)


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
