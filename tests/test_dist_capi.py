"""Multi-GPU path behind the C ABI (spmvtk_dist_*, spmvtk_partition_rows,
spmvtk_gen_baseline_shard*): the host logic on CPU -- entry-balanced row
blocks, shard-only generation, and (gloo, world 2/3) the iterate's exchange
with variable-size blocks in rank order -- and one rank over NCCL on the GPU.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2407_00019_b200 import spmvtk as sp


def _partition_rows_ref(rp, world):
    """Restatement of gen::partition_rows: begin[k] = first row whose start
    reaches k*nnz/world."""
    n, nnz = rp.shape[0] - 1, rp[-1] - rp[0]
    begin = [0]
    for k in range(1, world):
        target = rp[0] + nnz * k // world
        begin.append(max(begin[-1], int(np.searchsorted(rp[: n + 1], target, side="left"))))
    begin.append(n)
    return np.array(begin)


def test_partition_rows_balances_entries():
    rng = np.random.default_rng(5)
    for n in (1, 2, 33, 1000, 50000):
        lens = np.minimum(n, np.round(rng.lognormal(1.5, 1.3, size=n)).astype(np.int64))
        rp = np.concatenate([[0], np.cumsum(lens)])
        for world in (1, 2, 3, 4, 8):
            b = sp.partition_rows(rp, world)
            np.testing.assert_array_equal(b, _partition_rows_ref(rp, world))
            assert b[0] == 0 and b[-1] == n and np.all(np.diff(b) >= 0)
            # every block holds its share of entries up to one row
            ent = rp[b[1:]] - rp[b[:-1]]
            assert np.all(np.abs(ent - rp[-1] / world) <= lens.max(initial=0) + 1)
    with pytest.raises(sp.SpmvtkError):
        sp.partition_rows(np.array([0, 1, 2]), 0)


@pytest.mark.parametrize("config,param,dparam", [(1, 16, 0.0), (2, 5000, 0.0), (3, 9, 0.0),
                                                 (4, 20000, 0.0), (5, 8192, 1.0)])
def test_shards_tile_the_generated_matrix(config, param, dparam):
    """spmvtk_gen_baseline_shard_host: every rank generates only its rows,
    and the rank-ordered shards are the full matrix, byte for byte."""
    full = sp.HostCrs(config, param, dparam, 9)
    rp, ci, v = full.arrays(0)
    for world in (1, 2, 3, 4):
        begin = sp.partition_rows(rp, world)
        cols, vals, lens = [], [], []
        for r in range(world):
            h = sp.gen_baseline_shard_host(config, param, dparam, 9, r, world)
            assert h.row_offset == begin[r] and h.n == begin[r + 1] - begin[r]
            assert h.ncols == full.n
            lrp, lci, lv = h.arrays(0)
            assert lrp[0] == 0
            cols.append(lci)
            vals.append(lv)
            lens.extend(np.diff(lrp))
            h.free()
        np.testing.assert_array_equal(np.concatenate(cols), ci)
        assert np.concatenate(vals).tobytes() == v.tobytes()
        np.testing.assert_array_equal(np.array(lens, np.int64), np.diff(rp))
    full.free()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, config, param, steps, q):
    """One rank: its shard from the shard-only generator, its rows of
    x_{t+1} from the oracle's sequential CRS product, then the blocks
    exchanged in rank order with per-rank counts (what the grouped
    ncclBroadcast of spmvtk_dist_spmv_iterate does)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Port
    port_lib = Port()
    h = sp.gen_baseline_shard_host(config, param, 0.0, 9, rank, world)
    lrp, lci, lv = h.arrays(1)
    n, r0, rows = h.ncols, h.row_offset, h.n
    begin = [None] * world
    dist.all_gather_object(begin, (r0, rows))
    x = sp.gen_vector(n, 4)
    for _ in range(steps):
        nxt = np.empty(n)
        mine = port_lib.spmv_crs(rows, lrp, lci, lv, x) if rows else np.zeros(0)
        for src in range(world):
            b0, cnt = begin[src]
            buf = torch.from_numpy(mine.copy() if src == rank else np.empty(cnt))
            if cnt:
                dist.broadcast(buf, src=src)
            nxt[b0:b0 + cnt] = buf.numpy()
        x = nxt
    q.put((rank, x))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,config,param", [(2, 4, 20000), (3, 2, 3000)])
def test_dist_iterate_exchange_gloo(world, config, param):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    steps = 3
    procs = [ctx.Process(target=_worker, args=(r, world, port, config, param, steps, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle.oracle import Port
    port_lib = Port()
    full = sp.HostCrs(config, param, 0.0, 9)
    rp, ci, v = full.arrays(1)
    want = sp.gen_vector(full.n, 4)
    for _ in range(steps):
        want = port_lib.spmv_crs(full.n, rp, ci, v, want)
    for r in range(world):
        assert results[r].tobytes() == want.tobytes(), r


@pytest.mark.gpu
def test_dist_capi_single_rank_nccl(gpu, port):
    """spmvtk_dist_* on one GPU (a one-rank NCCL communicator): shard-only
    generation, distribute() from host arrays, and the iterate against the
    port's sequential iteration."""
    torch.cuda.set_device(0)
    sp.set_stream(torch.cuda.current_stream().cuda_stream)
    d = sp.Dist(0, 1, sp.Dist.unique_id())
    try:
        for config, param in ((2, 20000), (4, 40000), (3, 12)):
            shard = d.shard(config, param, 0.0, 9)
            desc = shard.describe()
            full = sp.HostCrs(config, param, 0.0, 9)
            rp, ci, v = full.arrays(1)
            assert desc.n == full.n and desc.ncols == full.n and desc.row_offset == 0
            x0 = sp.gen_vector(full.n, 4)
            want = x0.copy()
            for _ in range(3):
                want = port.spmv_crs(full.n, rp, ci, v, want)
            for h, k in ((shard, sp.Kernel.CRS), (shard.convert(sp.Format.ELL), sp.Kernel.ELL_INNER),
                         (d.distribute(full.n, rp, ci, v, index_base=1), sp.Kernel.CRS)):
                x = torch.from_numpy(x0).cuda()
                sec = d.iterate(h, k, x.data_ptr(), 3)
                got = x.cpu().numpy()
                err = np.max(np.abs(got - want)) / np.max(np.abs(want))
                assert err <= 1e-12 and sec > 0, (config, k, err)
                if h is not shard:
                    h.free()
            # the exchange folded into the SpMV: same iterate (CRS and ELL)
            for h, k in ((shard, sp.Kernel.CRS), (shard.convert(sp.Format.ELL), sp.Kernel.ELL_INNER)):
                for sparse in (True, False):
                    pu = d.push(h, k, sparse=sparse)
                    x = torch.from_numpy(x0).cuda()
                    sec = pu.iterate(x.data_ptr(), 3)
                    got = x.cpu().numpy()
                    err = np.max(np.abs(got - want)) / np.max(np.abs(want))
                    assert err <= 1e-12 and sec > 0, (config, k, sparse, err)
                    x = torch.from_numpy(x0).cuda()  # a second run on the same buffers
                    pu.iterate(x.data_ptr(), 3)
                    assert np.max(np.abs(x.cpu().numpy() - want)) / np.max(np.abs(want)) <= 1e-12
                    pu.free()
                if h is not shard:
                    h.free()
            shard.free()
            full.free()
    finally:
        d.free()
