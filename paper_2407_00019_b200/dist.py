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

import math
from typing import Callable

import numpy as np


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


def cuda_apply(handle, kernel):
    """local_apply for DistSpMV backed by the C ABI device-pointer SpMV."""
    def apply(x_full, y_slot):
        handle.spmv_device(kernel, x_full.data_ptr(), y_slot.data_ptr())
    return apply


# --------------------------------------------------------------------------
def bench_main(args, rank: int, world: int, local: int) -> int:
    """bench.py under torchrun: strong scaling of the config's SpMV over
    `world` GPUs (matrix fixed, rows split), x all-gathered every step."""
    import json
    import os
    import time

    import torch
    import torch.distributed as dist

    from . import spmvtk as sp

    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    sp.set_stream(torch.cuda.current_stream().cuda_stream)
    host = sp.HostCrs(args.config, args.param, 0.0, args.seed)
    n, nnz = host.n, host.nnz
    rp, ci, v = host.arrays(index_base=0)
    r0, lrp, lci, lv = shard_arrays(rp, ci, v, n, world, rank)
    del rp, ci, v
    host.free()
    shard = sp.Matrix.from_crs_block(block_rows(n, world), n, r0, lrp, lci, lv)
    del lrp, lci, lv
    st = shard.row_stats() if shard.describe().nnz else None
    local_max = st.max_row if st else 0
    t = torch.tensor([local_max], dtype=torch.int64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    nz_global = int(t.item())

    handles = {"crs": (shard, sp.Kernel.CRS),
               "ell-inner": (shard.convert(sp.Format.ELL), sp.Kernel.ELL_INNER)}

    def bytes_of(fmt):
        d = shard.describe()
        rows, entries = d.n, d.nnz
        if fmt == "crs":
            return 12 * entries + 4 * (rows + 1) + 8 * n + 8 * rows
        return 12 * rows * handles["ell-inner"][0].describe().band_count + 8 * n + 8 * rows

    x = torch.from_numpy(sp.gen_vector(n, args.seed + 1)).cuda()
    y = torch.empty(block_rows(n, world), dtype=torch.float64, device="cuda")

    def local_time(fmt, reps=50):
        h, k = handles[fmt]
        for _ in range(3):
            h.spmv_device(k, x.data_ptr(), y.data_ptr())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            h.spmv_device(k, x.data_ptr(), y.data_ptr())
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps * 1e-3

    # format choice: slowest rank decides (max over ranks), best format wins
    times = torch.tensor([local_time(f) for f in handles], dtype=torch.float64, device="cuda")
    dist.all_reduce(times, op=dist.ReduceOp.MAX)
    fmt = list(handles)[int(torch.argmin(times).item())]
    h, k = handles[fmt]
    it = DistSpMV(n, world, rank, cuda_apply(h, k), "cuda")
    it.set_x(sp.gen_vector(n, args.seed + 1))

    def timed(steps, communicate):
        for _ in range(args.warmup):
            it.step(communicate)
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            it.step(communicate)
        e1.record()
        torch.cuda.synchronize()
        dist.barrier()
        tt = torch.tensor([e0.elapsed_time(e1) * 1e-3 / steps], dtype=torch.float64,
                          device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from bench import ClockSampler, hbm_peak
    with ClockSampler(local) as clk:
        t_step = timed(args.steps, True)
    t_local = timed(max(20, args.steps // 4), False)
    b = torch.tensor([bytes_of(fmt)], dtype=torch.float64, device="cuda")
    dist.all_reduce(b, op=dist.ReduceOp.SUM)
    total_bytes = float(b.item())

    # e2e: the C ABI call with pinned host x (ncols) and y (local rows)
    xh = torch.from_numpy(sp.gen_vector(n, args.seed + 1)).pin_memory()
    yh = torch.empty(block_rows(n, world), dtype=torch.float64).pin_memory()
    for _ in range(3):
        h.spmv(xh.numpy(), k, 1, out=yh.numpy())
    dist.barrier()
    t0 = time.perf_counter()
    e2e_steps = max(10, min(args.steps, 100))
    for _ in range(e2e_steps):
        h.spmv(xh.numpy(), k, 1, out=yh.numpy())
    te = torch.tensor([(time.perf_counter() - t0) / e2e_steps], dtype=torch.float64,
                      device="cuda")
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    t_e2e = float(te.item())

    if rank == 0:
        line = {
            "metric": ("SpMV GB/s & GFLOP/s per format; CRS→ELL/COO transform time in "
                       "CRS-SpMV units"),
            "value": total_bytes / t_step / 1e9, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"baseline config {args.config}", "n": n, "nnz": nnz,
                       "format": fmt, "band_count_global": nz_global,
                       "parallelism": f"row-block x{world}, NCCL all_gather of x per step",
                       "gflops": 2 * nnz / t_step / 1e9},
            "no_comm": {"ms_per_step": t_local * 1e3,
                        "value": total_bytes / t_local / 1e9},
            "e2e": {"value": total_bytes / t_e2e / 1e9, "unit": "GB/s",
                    "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * block_rows(n, world),
                    "api": "spmvtk_spmv per rank (pinned host x / y block)"},
            "gpu_launches": args.steps * (1 if fmt != "ell-outer" else 2),
            "clocks": clk.summary(),
        }
        peak, kind = hbm_peak()
        per_gpu = total_bytes / world / t_local / 1e9
        line["roofline"] = {"bound": "hbm", "achieved": per_gpu, "peak": peak, "unit": "GB/s",
                            "frac": per_gpu / peak, "traffic": None, "peak_kind": kind,
                            "kernel": fmt, "note": "per GPU, SpMV shard without the exchange"}
        print(json.dumps(line))
    dist.barrier()
    dist.destroy_process_group()
    return 0
