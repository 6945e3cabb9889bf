"""Row-block multi-GPU SpMV.

One process per GPU.  Rows are split into equal contiguous blocks of
``chunk = ceil(n / world)`` rows (the last block is padded with empty rows so
NCCL's all-gather, which needs equal counts, works in place).  Every shard
keeps its rows with GLOBAL column indices, so all transforms are row-local
and need no communication (CRS -> COO-row / ELL per shard; ELL padding uses
the global row index, matching the reference's global ELL row for row).

Per iteration: y_local = A_local x (the CUDA kernel writes straight into this
rank's slot of the next x buffer), then an in-place ``all_gather_into_tensor``
over NCCL (NVLink / NVSwitch) rebuilds the full vector on every rank.  The
exchange is the only collective of the path.

torch.distributed is plumbing only: compute goes through the C ABI
(``libspmvtk.so``).  The partition / exchange logic is independent of the
local kernel so it can be tested on CPU with gloo (tests/test_dist.py).
"""
from __future__ import annotations

import contextlib
import math
import os
import sys
from typing import Callable

import numpy as np


@contextlib.contextmanager
def _stdout_to_stderr():
    """fd 1 -> fd 2 for the duration (C libraries print through fd 1)."""
    sys.stdout.flush()
    saved = os.dup(1)
    os.dup2(2, 1)
    try:
        yield
    finally:
        sys.stdout.flush()
        os.dup2(saved, 1)
        os.close(saved)


def block_rows(n: int, world: int) -> int:
    """Rows per rank (equal padded blocks)."""
    return max(1, math.ceil(n / world))


def block_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Global [r0, r1) of rank's rows; r1 - r0 <= block_rows (last block may be
    short or empty)."""
    c = block_rows(n, world)
    r0 = min(n, rank * c)
    return r0, min(n, r0 + c)


def partition_range(length: int, lanes: int) -> tuple[list[int], list[int]]:
    """The reference's lane partition (spmv.cpp:36-54), 1-based inclusive:
    first ``length % lanes`` lanes get one extra element; an empty lane has
    istart == iend + 1.  Used for reporting the reference's split."""
    if lanes < 1:
        raise ValueError("lane count must be at least 1")
    base, rem = divmod(length, lanes)
    istart, iend, pos = [], [], 1
    for k in range(lanes):
        size = base + (1 if k < rem else 0)
        istart.append(pos)
        iend.append(pos + size - 1)
        pos += size
    return istart, iend


def shard_arrays(row_ptr: np.ndarray, col_idx: np.ndarray, values: np.ndarray, n: int,
                 world: int, rank: int):
    """Local CRS of rank's row block from 0-based global CRS arrays, padded to
    block_rows rows (trailing empty rows).  Columns stay global."""
    c = block_rows(n, world)
    r0, r1 = block_range(n, world, rank)
    a, b = int(row_ptr[r0]), int(row_ptr[r1])
    rp = np.empty(c + 1, dtype=np.int64)
    rp[: r1 - r0 + 1] = row_ptr[r0: r1 + 1] - a
    rp[r1 - r0 + 1:] = b - a
    return r0, rp, np.ascontiguousarray(col_idx[a:b]), np.ascontiguousarray(values[a:b])


class DistSpMV:
    """x_{t+1} = A x_t over row-block shards with an in-place all-gather.

    ``local_apply(x_full, y_slot)`` computes this rank's rows of A x into
    ``y_slot`` (a view of this rank's block of the next x buffer); the
    product uses the CUDA kernels through the C ABI (see ``cuda_apply``)."""

    def __init__(self, n: int, world: int, rank: int, local_apply: Callable, device,
                 group=None, dtype=None):
        import torch
        self.n, self.world, self.rank = n, world, rank
        self.chunk = block_rows(n, world)
        self.apply = local_apply
        self.group = group
        dtype = dtype or torch.float64
        self.bufs = [torch.zeros(self.chunk * world, dtype=dtype, device=device)
                     for _ in range(2)]
        self.cur = 0

    @property
    def x(self):
        """Current full vector (first n entries; the tail is zero padding)."""
        return self.bufs[self.cur][: self.n]

    def set_x(self, x) -> None:
        import torch
        b = self.bufs[self.cur]
        b.zero_()
        b[: self.n].copy_(torch.as_tensor(x, dtype=b.dtype))

    def slot(self, buf):
        return buf[self.rank * self.chunk: (self.rank + 1) * self.chunk]

    def step(self, communicate: bool = True) -> None:
        import torch.distributed as dist
        cur, nxt = self.bufs[self.cur], self.bufs[1 - self.cur]
        mine = self.slot(nxt)
        self.apply(cur, mine)
        if communicate and self.world > 1:
            dist.all_gather_into_tensor(nxt, mine, group=self.group)
        self.cur = 1 - self.cur


# ---------------------------------------------------------------- push path
# The exchange folded into the SpMV (spmvtk_spmv_device_push): every rank's
# kernel stores each result row straight into the next-x buffer of every
# rank that READS that row (peer memory through CUDA IPC, NVLink/NVSwitch
# stores), then a system-scope flag per (source, step) orders the steps.
# No collective runs per step; for banded matrices only the halo rows cross
# NVLink (the mask), for scattered columns every row goes to every rank.
#
# Protocol (double-buffered X[0], X[1] of chunk*world doubles per rank, flags
# F[world] per rank, all zero-initialised):
#   step t: wait until F_me[s] >= t for every source s
#           y = A_local X[t % 2]  ->  pushed to X_w[(t+1) % 2] rows of w's mask
#           F_w[me] = t + 1 for every w   (after the kernel's system fences)
# The wait before step t+1 covers both hazards: every peer finished writing
# my X[(t+1) % 2] (RAW) and finished reading its own X[t % 2], which my step
# t+1 overwrites (WAR).

def needed_columns(col_idx, n_pad: int):
    """bool[n_pad]: the global columns a shard's entries reference."""
    import torch
    need = torch.zeros(n_pad, dtype=torch.bool, device=col_idx.device)
    if col_idx.numel():
        need[col_idx.long()] = True
    return need


def push_mask(needed_all, rank: int, chunk: int):
    """uint8[chunk]: bit w of row r = rank w reads global row rank*chunk + r
    (needed_all: bool[world, chunk*world] gathered from every rank); a rank
    always keeps its own rows."""
    import torch
    world = needed_all.shape[0]
    seg = needed_all[:, rank * chunk:(rank + 1) * chunk].to(torch.int32)
    w = (1 << torch.arange(world, dtype=torch.int32, device=seg.device))[:, None]
    bits = (seg * w).sum(0) | (1 << rank)
    return bits.to(torch.uint8)


def apply_pushes(ys, masks, rank: int, chunk: int, x_next) -> None:
    """What the pushes of every source deliver to `rank` (the semantics of
    the push path, used by the CPU tests): row r of source s lands at
    x_next[s*chunk + r] when bit `rank` of masks[s][r] is set."""
    for s_, (y, m) in enumerate(zip(ys, masks)):
        sel = ((m.to(torch_int32()) >> rank) & 1).bool()
        dst = x_next[s_ * chunk:(s_ + 1) * chunk]
        dst[sel] = y[sel]


def torch_int32():
    import torch
    return torch.int32


class _DevView:
    """__cuda_array_interface__ over a raw device pointer (to view IPC
    buffers as torch tensors without copying)."""

    def __init__(self, ptr: int, count: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None}


class PushSpMV:
    """x_{t+1} = A x_t with the exchange folded into the SpMV epilogue.

    handle: this rank's row-block shard (CRS or ELL handle, global columns);
    kernel: sp.Kernel.CRS or sp.Kernel.ELL_INNER.  sparse=True pushes a row
    only to the ranks whose shard references it."""

    def __init__(self, n: int, world: int, rank: int, handle, kernel, group=None,
                 sparse: bool = True, timeout_s: float = 10.0):
        import torch
        import torch.distributed as dist
        from . import spmvtk as sp
        if world > sp.MAX_PEERS:
            raise ValueError(f"push exchange supports up to {sp.MAX_PEERS} ranks")
        self.sp, self.n, self.world, self.rank = sp, n, world, rank
        self.chunk = block_rows(n, world)
        self.h, self.k, self.group = handle, kernel, group
        self.timeout_ns = int(timeout_s * 1e9)
        npad = self.chunk * world
        # Every collective below is reached by every rank whatever happens
        # locally: a local failure is turned into an agreed one (all-reduce
        # MIN) so no rank is left waiting in a collective the others skipped.
        self.own, self.opened, self.peer = [], [], []
        handles, err = None, None
        try:  # own buffers: X0, X1, flags (IPC-shareable cudaMalloc memory)
            self.own = [sp.ipc_alloc(npad * 8), sp.ipc_alloc(npad * 8),
                        sp.ipc_alloc(world * 8)]
            handles = [h for _, h in self.own]
        except Exception as e:  # noqa: BLE001
            err = e
        allh = [None] * world
        dist.all_gather_object(allh, handles, group=group)
        if err is None and any(h is None for h in allh):
            err = RuntimeError("a peer could not allocate its IPC buffers")
        if err is None:
            try:
                for w in range(world):
                    if w == rank:
                        self.peer.append([p for p, _ in self.own])
                    else:
                        ptrs = [sp.ipc_open(h) for h in allh[w]]
                        self.opened.extend(ptrs)
                        self.peer.append(ptrs)
            except Exception as e:  # noqa: BLE001
                err = e
        ok = torch.tensor([0.0 if err else 1.0], device="cuda")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        if ok.item() != 1.0:
            for p in self.opened:
                sp.ipc_close(p)
            for p, _ in self.own:
                sp.ipc_free(p)
            self.own, self.opened = [], []
            raise RuntimeError(f"push exchange unavailable: {err or 'failed on a peer'}")
        self.status = torch.zeros(1, dtype=torch.int32, device="cuda")
        # mask: which ranks read each of my rows
        self.mask = None
        if sparse and world > 1:
            ptr, cnt = handle.device_array(sp.Array.COL_IDX)  # ELL: padding = own rows
            col = (torch.as_tensor(_DevView(ptr, cnt, "<i4"), device="cuda") if cnt else
                   torch.zeros(0, dtype=torch.int32, device="cuda"))
            need = needed_columns(col, npad).to(torch.uint8)
            allneed = torch.empty(world, npad, dtype=torch.uint8, device="cuda")
            dist.all_gather_into_tensor(allneed.view(-1), need, group=group)
            self.mask = push_mask(allneed.bool(), rank, self.chunk).contiguous()
        self.push = []
        for b in range(2):
            pu = sp.Push()
            for w in range(world):
                pu.dst[w] = self.peer[w][b] + rank * self.chunk * 8
            pu.mask = self.mask.data_ptr() if self.mask is not None else None
            pu.ndst = world
            pu.local = rank
            self.push.append(pu)
        self.targets = sp.FlagTargets()
        for w in range(world):
            self.targets.ptr[w] = self.peer[w][2] + rank * 8
        self.targets.n = world
        # one launch per step: the flag wait runs in the SpMV prologue, the
        # signal in its last CTA (spmvtk_push_sync)
        self.counter = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.sync = sp.PushSync()
        self.sync.wait_flags = self.own[2][0]
        self.sync.nwait = world
        self.sync.timeout_ns = self.timeout_ns
        self.sync.status = self.status.data_ptr()
        self.sync.signal = self.targets
        self.sync.counter = self.counter.data_ptr()
        self.x_views = [torch.as_tensor(_DevView(self.own[b][0], npad, "<f8"), device="cuda")
                        for b in range(2)]
        self.t = 0
        torch.cuda.synchronize()
        dist.barrier(group=group)

    def set_x(self, x) -> None:
        import torch
        for b in range(2):
            self.x_views[b].zero_()
        self.x_views[self.t % 2][: self.n].copy_(torch.as_tensor(x, dtype=torch.float64))

    def step(self) -> None:
        t = self.t
        self.sync.wait_value = t
        self.sync.signal_value = t + 1
        self.h.spmv_device_push(self.k, self.own[t % 2][0], self.push[(t + 1) % 2], self.sync)
        self.t = t + 1

    def local_rows(self):
        """This rank's rows of the current iterate."""
        r0 = self.rank * self.chunk
        return self.x_views[self.t % 2][r0: r0 + self.chunk]

    def ok(self) -> bool:
        return int(self.status.item()) == 0

    def close(self) -> None:
        import torch
        import torch.distributed as dist
        sp = self.sp
        # every peer has finished pushing into my buffers once its last flag
        # arrived; then nobody touches them any more
        sp.flags_wait(self.own[2][0], self.world, self.t, self.timeout_ns, self.status.data_ptr())
        torch.cuda.synchronize()
        dist.barrier(group=self.group)
        for p in self.opened:
            sp.ipc_close(p)
        self.opened = []
        torch.cuda.synchronize()
        dist.barrier(group=self.group)
        for p, _ in self.own:
            sp.ipc_free(p)
        self.own = []


# ------------------------------------------------------- overlapped NCCL path
def interior_range(lrp: np.ndarray, lci: np.ndarray, r0: int, rows: int, chunk: int):
    """Largest contiguous run [ia, ib) of local rows whose columns all lie in
    this rank's own block [r0, r0 + chunk): those rows need no remote x and
    can run while the all-gather is in flight (interior rows
    first).  Returns (0, 0) when no row qualifies."""
    if rows == 0:
        return 0, 0
    lens = np.diff(lrp[: rows + 1])
    ok = np.ones(rows, dtype=bool)
    if lci.size:
        row_of = np.repeat(np.arange(rows), lens)
        outside = (lci < r0) | (lci >= r0 + chunk)
        bad = np.zeros(rows, dtype=bool)
        bad[row_of[outside]] = True
        ok = ~bad
    best, start, best_range = 0, None, (0, 0)
    for i in range(rows + 1):
        if i < rows and ok[i]:
            start = i if start is None else start
        elif start is not None:
            if i - start > best:
                best, best_range = i - start, (start, i)
            start = None
    return best_range


class OverlapSpMV(DistSpMV):
    """DistSpMV whose all-gather of x_t overlaps the interior rows' SpMV.

    parts: [(handle, kernel, local_row_begin, local_row_end, interior)] that
    tile the shard's rows.  Step t: the interior part runs on a side stream
    from the local block of x_t while x_t is all-gathered in place; the
    boundary parts run after the gather; all write x_{t+1}'s local slot."""

    def __init__(self, n, world, rank, parts, device, group=None):
        import torch
        super().__init__(n, world, rank, None, device, group)
        self.parts = parts
        self.side = torch.cuda.Stream()
        from . import spmvtk as sp
        self.sp = sp

    def step(self, communicate: bool = True) -> None:
        import torch
        import torch.distributed as dist
        sp = self.sp
        cur, nxt = self.bufs[self.cur], self.bufs[1 - self.cur]
        mine = self.slot(nxt)
        main = torch.cuda.current_stream()
        self.side.wait_stream(main)
        sp.set_stream(self.side.cuda_stream)
        for h, k, a, b, interior in self.parts:
            if interior and b > a:
                h.spmv_device(k, cur.data_ptr(), mine[a:b].data_ptr())
        sp.set_stream(main.cuda_stream)
        if communicate and self.world > 1:
            dist.all_gather_into_tensor(cur, self.slot(cur), group=self.group)
        for h, k, a, b, interior in self.parts:
            if not interior and b > a:
                h.spmv_device(k, cur.data_ptr(), mine[a:b].data_ptr())
        main.wait_stream(self.side)
        self.cur = 1 - self.cur


def cuda_apply(handle, kernel):
    """local_apply for DistSpMV backed by the C ABI device-pointer SpMV."""
    def apply(x_full, y_slot):
        handle.spmv_device(kernel, x_full.data_ptr(), y_slot.data_ptr())
    return apply


# --------------------------------------------------------------------------
def bench_main(args, rank: int, world: int, local: int) -> int:
    """bench.py under torchrun: strong scaling of the config's SpMV over
    `world` GPUs through the C ABI (spmvtk_dist_*): each rank generates only
    its entry-balanced row block (spmvtk_gen_baseline_shard), and
    spmvtk_dist_spmv_iterate runs x_{t+1} = A x_t with the x blocks exchanged
    over the library's own NCCL communicator (grouped in-place broadcasts).
    torch.distributed only carries the communicator id, the barriers and the
    max-over-ranks of the timings."""
    import json
    import time

    import torch
    import torch.distributed as dist

    from . import spmvtk as sp

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from bench import (ELL_GUARD_BYTES, METRIC, ClockSampler, cpu_reference_run, hbm_peak,
                       spmv_bytes, workload_config)

    torch.cuda.set_device(local)
    # NCCL writes its version banner to fd 1 at communicator init when the
    # environment asks for it (NCCL_DEBUG); the bench's stdout must hold
    # exactly one JSON line, so both inits run with fd 1 pointed at stderr
    with _stdout_to_stderr():
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        sp.set_stream(torch.cuda.current_stream().cuda_stream)
        lib = sp.load_library()
        uid = [sp.Dist.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = sp.Dist(rank, world, uid[0])
        dist.barrier()
    shard = comm.shard(args.config, args.param, 0.0, args.seed)
    desc = shard.describe()
    n, rows, r0 = desc.ncols, desc.n, desc.row_offset
    st = shard.row_stats() if desc.nnz else None
    # global statistics from the shards: entries, sum of squared row lengths, max row
    sums = torch.tensor([float(desc.nnz),
                         rows * (st.sigma ** 2 + st.mu ** 2) if st else 0.0],
                        dtype=torch.float64, device="cuda")
    dist.all_reduce(sums, op=dist.ReduceOp.SUM)
    mx = torch.tensor([st.max_row if st else 0], dtype=torch.int64, device="cuda")
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    nnz, nz = int(round(sums[0].item())), int(mx.item())
    mu_g = nnz / n
    d_mat_g = ((max(sums[1].item() / n - mu_g * mu_g, 0.0)) ** 0.5) / mu_g if nnz else 0.0

    handles = {"crs": (shard, sp.Kernel.CRS)}
    if n * nz * 16 <= ELL_GUARD_BYTES:  # the reference's guard on the whole matrix
        handles["ell-inner"] = (shard.convert(sp.Format.ELL), sp.Kernel.ELL_INNER)
    xl = torch.from_numpy(sp.gen_vector(n, args.seed + 1)).cuda()
    yl = torch.empty(max(rows, 1), dtype=torch.float64, device="cuda")

    def local_time(h, k, reps=50):
        if rows == 0:
            return 0.0
        for _ in range(3):
            h.spmv_device(k, xl.data_ptr(), yl.data_ptr())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            h.spmv_device(k, xl.data_ptr(), yl.data_ptr())
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps * 1e-3

    def shard_bytes(name, hh):  # the shard's own SpMV (x read whole, its rows of y)
        if name == "crs":
            return 12 * desc.nnz + 4 * (rows + 1) + 8 * rows + 8 * n
        return 12 * rows * hh.describe().band_count + 8 * rows + 8 * n

    # format: the slowest rank decides (max over ranks), the fastest format wins
    mine = [local_time(hh, kk) for hh, kk in handles.values()]
    times = torch.tensor(mine, dtype=torch.float64, device="cuda")
    dist.all_reduce(times, op=dist.ReduceOp.MAX)
    best = int(torch.argmin(times).item())
    fmt = list(handles)[best]
    t_local = float(times[best].item())
    h, k = handles[fmt]
    # per-GPU roofline: the slowest rank's shard SpMV rate
    rate = torch.tensor([shard_bytes(fmt, h) / mine[best] if mine[best] > 0 else float("inf")],
                        dtype=torch.float64, device="cuda")
    dist.all_reduce(rate, op=dist.ReduceOp.MIN)

    x = torch.from_numpy(sp.gen_vector(n, args.seed + 1)).cuda()
    comm.iterate(h, k, x.data_ptr(), args.warmup)
    torch.cuda.synchronize()
    dist.barrier()
    launches0 = lib.spmvtk_k_launch_count()
    with ClockSampler(local) as clk:
        t_rank = comm.iterate(h, k, x.data_ptr(), args.steps)
    launches = torch.tensor([lib.spmvtk_k_launch_count() - launches0], dtype=torch.int64,
                            device="cuda")
    dist.all_reduce(launches, op=dist.ReduceOp.SUM)
    tt = torch.tensor([t_rank], dtype=torch.float64, device="cuda")
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_step = float(tt.item())
    # the exchange folded into the SpMV (spmvtk_dist_push_*): checked against
    # the NCCL iterate from the same x0 (all ranks agree), timed the same
    # way, reported when it is correct and faster
    push_info = {"used": False}
    t_push = None
    try:
        x_ref = torch.from_numpy(sp.gen_vector(n, args.seed + 1)).cuda()
        comm.iterate(h, k, x_ref.data_ptr(), 3)
        pu = comm.push(h, k, sparse=True)
        try:
            x_p = torch.from_numpy(sp.gen_vector(n, args.seed + 1)).cuda()
            pu.iterate(x_p.data_ptr(), 3)
            err = float(((x_p - x_ref).abs().max() / x_ref.abs().max().clamp_min(1e-300)).item())
            ok = torch.tensor([1.0 if err <= 1e-12 else 0.0], device="cuda")
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            push_info = {"used": False, "checked_rel_err": err}
            if ok.item() == 1.0:
                pu.iterate(x_p.data_ptr(), args.warmup)
                dist.barrier()
                tp = torch.tensor([pu.iterate(x_p.data_ptr(), args.steps)], dtype=torch.float64,
                                  device="cuda")
                dist.all_reduce(tp, op=dist.ReduceOp.MAX)
                t_push = float(tp.item())
                push_info["ms_per_step"] = t_push * 1e3
        finally:
            pu.free()
    except Exception as e:  # noqa: BLE001 -- reported; the NCCL result stands
        push_info = {"used": False, "error": f"{type(e).__name__}: {e}"[:200]}
    exchange = "grouped in-place ncclBroadcast (spmvtk_dist_spmv_iterate)"
    if t_push is not None and t_push < t_step:
        push_info["used"] = True
        push_info["nccl_ms_per_step"] = t_step * 1e3
        t_step = t_push
        exchange = ("folded into the SpMV: rows stored to the readers' next-x buffers over "
                    "CUDA-IPC peer memory, step flags in the same launch (spmvtk_dist_push_*)")

    # every rank must hold the same iterate: compare a checksum of x
    chk = torch.tensor([float(x.abs().sum().item()), float(x.sum().item())], dtype=torch.float64,
                       device="cuda")
    lo, hi = chk.clone(), chk.clone()
    dist.all_reduce(lo, op=dist.ReduceOp.MIN)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX)
    consistent = bool(torch.equal(lo, hi))

    # e2e: every step copies x in from pinned host memory on every rank, runs
    # one iterate step (SpMV + exchange) and copies this rank's block out
    xh = torch.from_numpy(sp.gen_vector(n, args.seed + 1)).pin_memory()
    yh = torch.empty(max(rows, 1), dtype=torch.float64).pin_memory()
    e2e_steps = max(10, min(args.steps, 100))
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        x.copy_(xh, non_blocking=True)
        comm.iterate(h, k, x.data_ptr(), 1)
        if rows:
            yh[:rows].copy_(x[r0:r0 + rows], non_blocking=True)
    torch.cuda.synchronize()
    te = torch.tensor([(time.perf_counter() - t0) / e2e_steps], dtype=torch.float64,
                      device="cuda")
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    t_e2e = float(te.item())

    total_bytes = float(spmv_bytes(fmt, n, nnz, nz))
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            from oracle.oracle import Ref
            ref = Ref()
            rh = ref.gen_baseline(args.config, args.param, 0.0, args.seed)
            r = cpu_reference_run(ref, rh, n, nnz, nz)
            for hh in r.pop("handles").values():
                ref.free(hh)
            b = r["table"][r["best"]]
            cpu = {"value": b["gbs"], "unit": "GB/s", "cores": b["lanes"], "kind": "reference",
                   "sample": (f"reference measure_spmv (warm-up + median of 3) per format on the "
                              f"same config-{args.config} matrix on rank 0's host; best = "
                              f"{r['best']} at {b['lanes']} lanes of {r['cores']} cores"),
                   "cpu_model": r["cpu_model"], "nproc": r["cores"]}
        except Exception as e:  # reported, never silently replaced
            cpu = {"value": None, "unit": "GB/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {type(e).__name__}: {e}"[:300]}
    if rank == 0:
        peak, kind = hbm_peak()
        per_gpu = float(rate.item()) / 1e9
        line = {
            "metric": METRIC, "value": total_bytes / t_step / 1e9, "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args.config, args.param, 0.0, args.seed, n, nnz, nz,
                                      d_mat_g),
            "format": fmt, "gflops": 2 * nnz / t_step / 1e9,
            "parallelism": f"{world} entry-balanced row blocks, x exchanged every step: {exchange}",
            "push_exchange": push_info,
            "ranks_consistent": consistent,
            "no_comm": {"ms_per_step": t_local * 1e3, "value": total_bytes / t_local / 1e9},
            "e2e": {"value": total_bytes / t_e2e / 1e9, "unit": "GB/s",
                    "h2d_bytes_per_step": 8 * n * world, "d2h_bytes_per_step": 8 * n,
                    "ms_per_step": t_e2e * 1e3,
                    "api": "pinned host x copied in on every rank + spmvtk_dist_spmv_iterate "
                           "(1 step) + own block copied out"},
            "gpu_launches": int(launches.item()),
            "clocks": clk.summary(),
            "roofline": {"bound": "hbm", "achieved": per_gpu, "peak": peak, "unit": "GB/s",
                         "frac": per_gpu / peak if per_gpu else None, "traffic": None,
                         "peak_kind": kind, "kernel": fmt,
                         "note": "per GPU: the slowest rank's shard SpMV (its bytes over its "
                                 "time) without the exchange"},
            "cpu_baseline": cpu,
        }
        print(json.dumps(line))
    for name, (hh, _) in handles.items():
        if name != "crs":
            hh.free()
    shard.free()
    comm.free()
    dist.barrier()
    dist.destroy_process_group()
    return 0
