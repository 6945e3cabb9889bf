"""The multi-GPU push exchange (SpMV epilogue stores rows into the ranks'
next-x buffers + step flags), emulated on ONE GPU.

B200_PROFILING.md: ranks whose kernels wait on one another must not run as
separate launches on one GPU.  Here the W "ranks" run their steps in order on
one stream, so every flag wait is already satisfied when it executes (each
source signalled step t+1 earlier in the stream); the data movement -- the
push kernels' fan-out into W buffers through the per-row masks, the buffer
double-buffering and the flag protocol -- is exactly the multi-GPU one.  The
iterate is compared with the C port's full-matrix iteration (1e-12).
"""
import numpy as np
import pytest

from oracle.oracle import max_rel_error

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _banded(rng, n, half):
    rows = [np.arange(max(0, i - half), min(n, i + half + 1)) for i in range(n)]
    ci = np.concatenate(rows)
    rp = np.concatenate([[0], np.cumsum([len(r) for r in rows])])
    return rp, ci, rng.standard_normal(ci.shape[0])


def _random(rng, n, per_row):
    rows = [np.sort(rng.choice(n, size=per_row, replace=False)) for _ in range(n)]
    ci = np.concatenate(rows)
    rp = np.concatenate([[0], np.cumsum([len(r) for r in rows])])
    return rp, ci, rng.standard_normal(ci.shape[0])


@pytest.mark.parametrize("world,kind,fmt,sparse,fused", [
    (1, "banded", "crs", True, False), (2, "banded", "crs", True, False),
    (3, "banded", "ell", True, False), (3, "random", "crs", True, False),
    (4, "random", "ell", False, False), (2, "banded", "crs", False, False),
    (1, "banded", "crs", True, True), (3, "banded", "ell", True, True),
    (4, "random", "crs", True, True), (2, "longrows", "crs", True, True)])
def test_push_iteration_emulated(gpu, port, world, kind, fmt, sparse, fused):
    import torch
    from paper_2407_00019_b200 import dist as D
    sp = gpu
    sp.set_stream(torch.cuda.current_stream().cuda_stream)
    rng = np.random.default_rng(world * 7 + len(kind))
    n = 3001
    if kind == "longrows":  # rows past the vector kernel's limit: long-row pass signals
        rp, ci, v = _random(rng, n, 3)
        lens = np.diff(rp)
        lens[[7, 2500]] = [3000, 2900]
        rows = [np.sort(rng.choice(n, size=int(ln), replace=False)) for ln in lens]
        ci = np.concatenate(rows)
        rp = np.concatenate([[0], np.cumsum(lens)])
        v = rng.standard_normal(ci.shape[0])
    else:
        rp, ci, v = _banded(rng, n, 9) if kind == "banded" else _random(rng, n, 12)
    x0 = rng.uniform(-1, 1, n)
    steps = 4
    chunk = D.block_rows(n, world)
    npad = chunk * world
    kernel = sp.Kernel.CRS if fmt == "crs" else sp.Kernel.ELL_INNER
    shards, X, F = [], [], []
    for r in range(world):
        r0, lrp, lci, lv = D.shard_arrays(rp, ci, v, n, world, r)
        h = sp.Matrix.from_crs_block(chunk, n, r0, lrp, lci, lv)
        if fmt == "ell":
            h = h.convert(sp.Format.ELL)
        shards.append(h)
        X.append([torch.zeros(npad, dtype=torch.float64, device="cuda") for _ in range(2)])
        F.append(torch.zeros(world, dtype=torch.int64, device="cuda"))
        X[r][0][:n] = torch.from_numpy(x0)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    masks = [None] * world
    if sparse and world > 1:
        need = []
        for h in shards:
            ptr, cnt = h.device_array(sp.Array.COL_IDX)
            col = torch.as_tensor(D._DevView(ptr, cnt, "<i4"), device="cuda")
            need.append(D.needed_columns(col, npad))
        allneed = torch.stack(need)
        masks = [D.push_mask(allneed, r, chunk).contiguous() for r in range(world)]
    pushes, targets = [], []
    for r in range(world):
        per_buf = []
        for b in range(2):
            pu = sp.Push()
            for w in range(world):
                pu.dst[w] = X[w][b].data_ptr() + r * chunk * 8
            pu.mask = masks[r].data_ptr() if masks[r] is not None else None
            pu.ndst = world
            pu.local = r
            per_buf.append(pu)
        pushes.append(per_buf)
        tg = sp.FlagTargets()
        for w in range(world):
            tg.ptr[w] = F[w].data_ptr() + r * 8
        tg.n = world
        targets.append(tg)
    counters = [torch.zeros(1, dtype=torch.int32, device="cuda") for _ in range(world)]
    for t in range(steps):
        for r in range(world):
            if fused:  # wait in the SpMV prologue, signal from its last CTA
                sy = sp.PushSync()
                sy.wait_flags = F[r].data_ptr()
                sy.nwait = world
                sy.wait_value = t
                sy.timeout_ns = 2_000_000_000
                sy.status = status.data_ptr()
                sy.signal = targets[r]
                sy.signal_value = t + 1
                sy.counter = counters[r].data_ptr()
                shards[r].spmv_device_push(kernel, X[r][t % 2].data_ptr(),
                                           pushes[r][(t + 1) % 2], sy)
                continue
            sp.flags_wait(F[r].data_ptr(), world, t, 2_000_000_000, status.data_ptr())
            shards[r].spmv_device_push(kernel, X[r][t % 2].data_ptr(), pushes[r][(t + 1) % 2])
            sp.flags_signal(targets[r], t + 1)
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    assert all(int(f.min().item()) == steps for f in F)
    assert all(int(c.item()) == 0 for c in counters)
    want = x0.copy()
    for _ in range(steps):
        want = port.spmv_crs(n, rp + 1, ci + 1, v, want)
    got = np.concatenate([X[r][steps % 2][r * chunk: (r + 1) * chunk].cpu().numpy()
                          for r in range(world)])[:n]
    assert max_rel_error(got, want) <= TOL
    if masks[0] is not None and kind == "banded":
        # a banded shard only needs its neighbours' halo rows
        m0 = masks[0].cpu().numpy()
        assert ((m0 >> 1) & 1).sum() <= 9 and ((m0 >> 2) & 1).sum() == 0


def test_flags_wait_times_out_without_hanging(gpu):
    """A wait whose flag never arrives returns after the timeout and marks
    the status word; a second wait then fails fast."""
    import time

    import torch
    sp = gpu
    sp.set_stream(torch.cuda.current_stream().cuda_stream)
    flags = torch.zeros(2, dtype=torch.int64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    t0 = time.perf_counter()
    sp.flags_wait(flags.data_ptr(), 2, 1, 50_000_000, status.data_ptr())  # 50 ms
    torch.cuda.synchronize()
    assert int(status.item()) == 1
    assert time.perf_counter() - t0 < 5.0
    t1 = time.perf_counter()
    sp.flags_wait(flags.data_ptr(), 2, 5, 10_000_000_000, status.data_ptr())
    torch.cuda.synchronize()
    assert time.perf_counter() - t1 < 1.0


def test_ipc_buffers_roundtrip(gpu):
    """IPC allocation (zeroed) and the push entry point's argument checks."""
    import torch
    from paper_2407_00019_b200 import dist as D
    sp = gpu
    ptr, handle = sp.ipc_alloc(4096)
    assert len(handle) == sp.IPC_HANDLE_BYTES
    view = torch.as_tensor(D._DevView(ptr, 512, "<f8"), device="cuda")
    assert float(view.abs().sum().item()) == 0.0
    view.fill_(2.0)
    torch.cuda.synchronize()
    assert float(view.sum().item()) == 1024.0
    sp.ipc_free(ptr)
    m = sp.Matrix.gen_banded(100, 1)
    bad = sp.Push()
    bad.ndst = 0
    x = torch.zeros(100, dtype=torch.float64, device="cuda")
    with pytest.raises(sp.SpmvtkError):
        m.spmv_device_push(sp.Kernel.CRS, x.data_ptr(), bad)
    bad = sp.Push()
    bad.dst[0] = x.data_ptr()
    bad.ndst = 1
    bad.local = 1  # must index a destination
    with pytest.raises(sp.SpmvtkError):
        m.spmv_device_push(sp.Kernel.CRS, x.data_ptr(), bad)
    ok = sp.Push()
    ok.dst[0] = x.data_ptr()
    ok.ndst = 1
    with pytest.raises(sp.SpmvtkError):
        m.spmv_device_push(sp.Kernel.COO_ROW_OUTER, x.data_ptr(), ok)


def test_overlap_step_matches_plain_iteration(gpu, port):
    """OverlapSpMV (interior rows on a side stream, boundary rows after the
    exchange) iterates exactly like the plain product: one rank, the rows
    split into head / interior / tail parts of CRS and ELL handles."""
    import torch
    from paper_2407_00019_b200 import dist as D
    sp = gpu
    sp.set_stream(torch.cuda.current_stream().cuda_stream)
    rng = np.random.default_rng(5)
    n = 5000
    rp, ci, v = _banded(rng, n, 6)
    x0 = rng.uniform(-1, 1, n)
    for fmt in ("crs", "ell"):
        parts = []
        kern = sp.Kernel.CRS if fmt == "crs" else sp.Kernel.ELL_INNER
        for a, b, inner in ((0, 700, False), (700, 4300, True), (4300, n, False)):
            prp = (rp[a:b + 1] - rp[a]).astype(np.int64)
            h = sp.Matrix.from_crs_block(b - a, n, a, prp, ci[rp[a]:rp[b]], v[rp[a]:rp[b]])
            if fmt == "ell":
                h = h.convert(sp.Format.ELL)
            parts.append((h, kern, a, b, inner))
        it = D.OverlapSpMV(n, 1, 0, parts, "cuda")
        it.set_x(x0)
        for _ in range(3):
            it.step(True)
        torch.cuda.synchronize()
        want = x0.copy()
        for _ in range(3):
            want = port.spmv_crs(n, rp + 1, ci + 1, v, want)
        assert max_rel_error(it.x.cpu().numpy(), want) <= TOL, fmt
