"""Multi-GPU row-block path, host logic on CPU (gloo, world_size 2).

The CUDA shard kernels cannot run here; the exchange logic (equal padded
row blocks, in-place all-gather into the next x buffer, buffer swap) is
exercised with the C oracle as the per-rank local SpMV, and the iterate is
compared bit for bit with the oracle's full-matrix iteration (row sums are
computed in the same order on a shard as on the whole matrix).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.oracle import random_crs
from paper_2407_00019_b200 import dist as D


def test_partition_range_matches_reference_kats(kat):
    for c in kat["partition_range"]:
        if c.get("error"):
            with pytest.raises(ValueError):
                D.partition_range(c["len"], c["lanes"])
        else:
            assert D.partition_range(c["len"], c["lanes"]) == (c["istart"], c["iend"])


def test_block_ranges_cover_rows_once():
    for n in (1, 7, 64, 1000, 1 << 20):
        for world in (1, 2, 3, 4, 8):
            covered = []
            for r in range(world):
                a, b = D.block_range(n, world, r)
                assert 0 <= b - a <= D.block_rows(n, world)
                covered.extend(range(a, b))
            assert covered == list(range(n))


def test_shard_arrays_reassemble_the_matrix():
    rng = np.random.default_rng(3)
    n, rp, ci, v = random_crs(rng, 50, 600)
    rp0, ci0 = rp - 1, ci - 1
    for world in (1, 2, 3, 5):
        parts_c, parts_v, lens = [], [], []
        for r in range(world):
            r0, lrp, lci, lv = D.shard_arrays(rp0, ci0, v, n, world, r)
            assert r0 == D.block_range(n, world, r)[0]
            assert lrp[0] == 0 and lrp.shape[0] == D.block_rows(n, world) + 1
            parts_c.append(lci)
            parts_v.append(lv)
            lens.extend(np.diff(lrp)[: D.block_range(n, world, r)[1] - r0])
        np.testing.assert_array_equal(np.concatenate(parts_c), ci0)
        np.testing.assert_array_equal(np.concatenate(parts_v), v)
        np.testing.assert_array_equal(np.array(lens), np.diff(rp0))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, rp0, ci0, v, x0, steps, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Port
    port_lib = Port()
    r0, lrp, lci, lv = D.shard_arrays(rp0, ci0, v, n, world, rank)
    rows = D.block_rows(n, world)

    def local_apply(x_full, y_slot):
        xx = x_full[:n].numpy()
        y = port_lib.spmv_crs(rows, lrp + 1, lci + 1, lv, xx) if lci.size else np.zeros(rows)
        y_slot.copy_(torch.from_numpy(y))

    it = D.DistSpMV(n, world, rank, local_apply, "cpu")
    it.set_x(x0)
    for _ in range(steps):
        it.step()
    q.put((rank, it.x.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_dist_iteration_gloo(world):
    rng = np.random.default_rng(11)
    n, rp, ci, v = random_crs(rng, 300, 3000)
    rp0, ci0 = rp - 1, ci - 1
    x0 = rng.uniform(-1, 1, n)
    steps = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, rp0, ci0, v, x0, steps, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle.oracle import Port
    port_lib = Port()
    want = x0.copy()
    for _ in range(steps):
        want = port_lib.spmv_crs(n, rp, ci, v, want)
    for r in range(world):
        assert results[r].tobytes() == want.tobytes(), r


def _push_worker(rank, world, port, n, rp0, ci0, v, x0, steps, q):
    """The push exchange's semantics with gloo standing in for NVLink stores:
    masks from the gathered needed-column sets, each source's rows delivered
    only where its mask says; own rows must follow the full iteration."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Port
    port_lib = Port()
    r0, lrp, lci, lv = D.shard_arrays(rp0, ci0, v, n, world, rank)
    chunk = D.block_rows(n, world)
    npad = chunk * world
    need = D.needed_columns(torch.from_numpy(lci.astype(np.int32)), npad).to(torch.uint8)
    allneed = [torch.empty(npad, dtype=torch.uint8) for _ in range(world)]
    dist.all_gather(allneed, need)
    allneed = torch.stack(allneed).bool()
    masks_local = D.push_mask(allneed, rank, chunk)
    masks = [torch.empty(chunk, dtype=torch.uint8) for _ in range(world)]
    dist.all_gather(masks, masks_local)
    x = torch.zeros(npad, dtype=torch.float64)
    x[:n] = torch.from_numpy(x0)
    for _ in range(steps):
        xx = x[:n].numpy()
        y = (port_lib.spmv_crs(chunk, lrp + 1, lci + 1, lv, xx) if lci.size
             else np.zeros(chunk))
        ys = [torch.empty(chunk, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(ys, torch.from_numpy(y))
        x_next = torch.full((npad,), float("nan"), dtype=torch.float64)  # stale = poison
        D.apply_pushes(ys, masks, rank, chunk, x_next)
        x = x_next
    q.put((rank, x[r0: r0 + chunk].numpy().copy(), masks_local.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,kind", [(2, "banded"), (3, "random")])
def test_push_exchange_semantics_gloo(world, kind):
    rng = np.random.default_rng(5 + world)
    n = 400
    if kind == "banded":
        rows = [np.arange(max(0, i - 4), min(n, i + 5)) for i in range(n)]
    else:
        rows = [np.sort(rng.choice(n, size=10, replace=False)) for _ in range(n)]
    ci0 = np.concatenate(rows).astype(np.int64)
    rp0 = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    v = rng.standard_normal(ci0.shape[0])
    x0 = rng.uniform(-1, 1, n)
    steps = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_push_worker,
                         args=(r, world, port, n, rp0, ci0, v, x0, steps, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = {}
    for _ in range(world):
        r, xr, m = q.get(timeout=120)
        results[r] = (xr, m)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle.oracle import Port
    port_lib = Port()
    want = x0.copy()
    for _ in range(steps):
        want = port_lib.spmv_crs(n, rp0 + 1, ci0 + 1, v, want)
    chunk = D.block_rows(n, world)
    for r in range(world):
        a, b = D.block_range(n, world, r)
        assert results[r][0][: b - a].tobytes() == want[a:b].tobytes(), r
    if kind == "banded":
        # only the 4-row halos cross between neighbouring ranks
        m0 = results[0][1].astype(np.int32)
        assert ((m0 >> 1) & 1).sum() == 4
        assert (m0 & 1).all()


def test_interior_range_banded_and_random():
    """Interior rows (every column in the rank's own block) of a banded shard
    are the middle run; a scattered shard has none."""
    n, world, half = 300, 3, 4
    rows = [np.arange(max(0, i - half), min(n, i + half + 1)) for i in range(n)]
    ci = np.concatenate(rows).astype(np.int64)
    rp = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    chunk = D.block_rows(n, world)
    for rank in range(world):
        r0, lrp, lci, lv = D.shard_arrays(rp, ci, np.ones(ci.shape[0]), n, world, rank)
        rows_here = D.block_range(n, world, rank)[1] - r0
        ia, ib = D.interior_range(lrp, lci, r0, rows_here, chunk)
        want_a = 0 if rank == 0 else half
        want_b = rows_here if rank == world - 1 else rows_here - half
        assert (ia, ib) == (want_a, want_b), (rank, ia, ib)
    rng = np.random.default_rng(1)
    rows = [np.sort(rng.choice(n, size=12, replace=False)) for _ in range(n)]
    ci = np.concatenate(rows).astype(np.int64)
    rp = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    r0, lrp, lci, lv = D.shard_arrays(rp, ci, np.ones(ci.shape[0]), n, world, 1)
    ia, ib = D.interior_range(lrp, lci, r0, chunk, chunk)
    assert ib - ia <= 2
