"""Benchmark of the hot path on BASELINE.json's workload.

Metric (BASELINE.json): "SpMV GB/s & GFLOP/s per format; CRS->ELL/COO
transform time in CRS-SpMV units".  Workload: config 2 (random rows, n=2^20,
row lengths U{8..24}, columns uniform in [0,n), values N(0,1), seeded
synthetic data -- the paper's SuiteSparse set is not available).

A step = one SpMV y = A x in the best format for the matrix (every format is
measured; the per-format table, the transform times in CRS-SpMV units and
the AT decision are reported beside the headline).  `value` = algorithmic
bytes of one SpMV (GPU layout) x steps / device time, inputs
resident in HBM (the matrix, 222 MB, is larger than the 126 MB L2, so no
flush is needed between steps).  `e2e` = the same metric through the C ABI
with pinned HOST x / y, every step's copy-in and copy-out inside the timed
region: the streaming spmvtk_pipeline_* calls (products overlap each
other's copies), and under e2e.sync the reference's synchronous
spmvtk_spmv().

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("SpMV GB/s & GFLOP/s per format; CRS→ELL/COO transform time in "
          "CRS-SpMV units")
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback


def ncu_traffic(config: int, kernel: str):
    """DRAM read+write bytes per launch of `kernel` on this config, from the
    committed ncu launch list (profiles/traffic_*.json), or None."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "traffic_r*.json")), reverse=True):
        try:
            with open(path) as f:
                v = json.load(f).get(f"config{config}", {}).get(kernel)
            if v:
                return float(v)
        except Exception:
            continue
    return None


def hbm_peak():
    try:
        with open(PEAKS_FILE) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


# the reference's ELL memory guard as its own bench uses it (SURVEY.md 8d:
# config 4's ELL, ~206 GB in the GPU layout, is refused, not attempted)
ELL_GUARD_BYTES = 48 << 30


def spmv_bytes(fmt: str, n: int, nnz: int, nz: int = 0) -> int:
    """Compulsory bytes of one SpMV in the GPU layout (fp64 values, int32
    indices; x read once, y written once).  SURVEY.md §8(d)."""
    if fmt == "crs":
        return 12 * nnz + 4 * (n + 1) + 16 * n
    if fmt in ("coo-row", "coo-col"):
        return 16 * nnz + 16 * n
    if fmt in ("ell-inner", "ell-outer", "ell-row"):
        return 12 * n * nz + 16 * n  # padding included (north_star)
    raise ValueError(fmt)


def transform_bytes(to: str, n: int, nnz: int, nz: int = 0) -> int:
    if to == "coo-row":
        return 28 * nnz + 4 * n
    if to == "ccs":
        return 28 * nnz + 12 * n
    if to == "coo-col":  # Phase I + column expansion (no CCS copy)
        return 32 * nnz + 16 * n
    if to in ("ell", "ell-row"):
        return 12 * nnz + 4 * (n + 1) + 12 * n * nz + 4 * n
    raise ValueError(to)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int = 0):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            time.sleep(0.15)
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.06)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


# --------------------------------------------------------------------------
def l2_resident_graph(sp, torch, seed, peak, iters=1000):
    """Config 1 SpMVs captured into one CUDA graph of `iters` launches
    (x -> y -> x ping-pong), replayed and timed with events: per-SpMV time
    of an L2-resident matrix without the launch overhead."""
    m = sp.HostCrs(1, 256, 0.0, seed).upload()
    d = m.describe()
    nz = m.row_stats().max_row
    ell = m.convert(sp.Format.ELL)
    out = {"label": "L2-resident", "n": d.n, "nnz": d.nnz, "iters_per_graph": iters}
    for name, h, k in (("crs", m, sp.Kernel.CRS), ("ell-inner", ell, sp.Kernel.ELL_INNER)):
        a = torch.from_numpy(sp.gen_vector(d.n, seed + 1)).cuda()
        b = torch.empty_like(a)
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            sp.set_stream(stream.cuda_stream)
            for _ in range(3):  # warm-up (caches row statistics, loads modules)
                h.spmv_device(k, a.data_ptr(), b.data_ptr())
            stream.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                for i in range(iters):
                    src, dst = (a, b) if i % 2 == 0 else (b, a)
                    h.spmv_device(k, src.data_ptr(), dst.data_ptr())
            g.replay()
            stream.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(5):
                g.replay()
            e1.record(stream)
            stream.synchronize()
        sp.set_stream(torch.cuda.current_stream().cuda_stream)
        t = e0.elapsed_time(e1) * 1e-3 / (5 * iters)
        by = spmv_bytes(name, d.n, d.nnz, nz)
        out[name] = {"us": t * 1e6, "gbs": by / t / 1e9, "gflops": 2 * d.nnz / t / 1e9,
                     "frac_of_hbm_peak": by / t / 1e9 / peak}
        del g
    ell.free()
    m.free()
    return out


def gather_peak(sp, torch, n_pow2=1 << 20, iters=256):
    """Measured random-gather rate (8-byte loads, L2-resident x of n_pow2
    doubles, nothing else in flight): the denominator of the gather roofline."""
    lib = sp.load_library()
    x = torch.zeros(n_pow2, dtype=torch.float64, device="cuda")
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    rc = lib.spmvtk_k_gather_probe(x.data_ptr(), n_pow2, iters, out.data_ptr(), stream)
    if rc:
        raise RuntimeError(f"gather probe failed ({rc})")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        lib.spmvtk_k_gather_probe(x.data_ptr(), n_pow2, iters, out.data_ptr(), stream)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) * 1e-3 / 10
    return 1024 * 148 * iters / t


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_reference_run(host, n, nnz, nz, per_call_repeats=3):
    """The reference's own CPU path (oracle/_ref, compiled from the reference
    sources) on this host's cores, on the same matrix."""
    from oracle.oracle import Ref
    ref = Ref()
    cores = os.cpu_count() or 1
    rp, ci, v = host.arrays(index_base=1)
    h = ref.matrix(n, rp, ci, v)
    del rp, ci, v
    res = {}
    # transforms: one cold conversion each (autotune.cpp:122-128, :197-214)
    t_ell, ell = ref.measure_transformation(h, 4, 0)
    t_coo, coo = ref.measure_transformation(h, 2, 0)
    # SpMV: warm-up + median of repeats (autotune.cpp:95-120); CRS is
    # sequential in the reference (autotune.cpp:186), the others use lanes
    t_crs = ref.measure_spmv(h, 0, 1, per_call_repeats)
    res["crs"] = (t_crs, 1)
    res["ell-inner"] = (ref.measure_spmv(ell, 3, cores, per_call_repeats), cores)
    res["ell-outer"] = (ref.measure_spmv(ell, 4, cores, per_call_repeats), cores)
    res["coo-row"] = (ref.measure_spmv(coo, 1, cores, per_call_repeats), cores)
    # the lane-parallel kernels also at one lane
    one = {"ell-inner@1": ref.measure_spmv(ell, 3, 1, per_call_repeats),
           "ell-outer@1": ref.measure_spmv(ell, 4, 1, per_call_repeats),
           "coo-row@1": ref.measure_spmv(coo, 1, 1, per_call_repeats)}
    table = {}
    for k, (t, lanes) in res.items():
        b = spmv_bytes(k, n, nnz, nz)
        table[k] = {"gbs": b / t / 1e9, "gflops": 2 * nnz / t / 1e9, "ms": t * 1e3, "lanes": lanes}
    best = max(table, key=lambda k: table[k]["gbs"])
    for k, t in one.items():
        b = spmv_bytes(k.split("@")[0], n, nnz, nz)
        table[k] = {"gbs": b / t / 1e9, "gflops": 2 * nnz / t / 1e9, "ms": t * 1e3, "lanes": 1}
    out = {"table": table, "best": best, "cores": cores, "cpu_model": cpu_model(),
           "transforms": {"ell": {"ms": t_ell * 1e3, "tt": t_ell / t_crs},
                          "coo-row": {"ms": t_coo * 1e3, "tt": t_coo / t_crs}},
           "handles": (ref, h, ell, coo)}
    return out


def impl_reference(args):
    rank, world, _ = dist_env()
    if world > 1 and rank != 0:
        return 0
    from paper_2407_00019_b200 import spmvtk as sp
    # host-side generation only: this arm never touches the GPU
    host = sp.HostCrs(args.config, args.param, 0.0, args.seed)
    n, nnz = host.n, host.nnz
    rp, _, _ = host.arrays(index_base=0)
    nz = int(np.max(np.diff(rp))) if n else 0
    del rp
    r = cpu_reference_run(host, n, nnz, nz)
    ref, h, ell, coo = r.pop("handles")
    best = r["best"]
    kern = {"crs": 0, "coo-row": 1, "ell-inner": 3, "ell-outer": 4}[best]
    handle = {"crs": h, "coo-row": coo, "ell-inner": ell, "ell-outer": ell}[best]
    lanes = r["table"][best]["lanes"]
    x = np.ones(n)
    tw = time.perf_counter()
    for _ in range(args.warmup):
        ref.spmv(handle, kern, x, lanes)
    t_one = (time.perf_counter() - tw) / max(1, args.warmup)
    # bounded sample: at most ~60 s of CPU work whatever K is
    steps = int(max(3, min(args.steps, 60.0 / max(t_one, 1e-9))))
    t0 = time.perf_counter()
    for _ in range(steps):
        ref.spmv(handle, kern, x, lanes)
    dt = (time.perf_counter() - t0) / steps
    args.steps_requested, args.steps = args.steps, steps
    b = spmv_bytes(best, n, nnz, nz)
    value = b / dt / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "steps_requested": args.steps_requested,
        "warmup": args.warmup,
        "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"baseline config {args.config}", "n": n, "nnz": nnz,
                   "best_format": best,
                   "bounded_sample": "steps capped at ~60 s of CPU work"},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": lanes, "kind": "reference",
                         "sample": f"{args.steps} SpMVs ({best}, {lanes} lanes) of the full "
                                   f"config-{args.config} matrix; oracle/_ref = reference "
                                   "compiled from its sources; std::thread lanes, no OpenMP",
                         "cpu_model": r.get("cpu_model"), "nproc": r.get("cores")},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "formats": r["table"], "transforms": r["transforms"],
    }
    print(json.dumps(line))
    return 0


# --------------------------------------------------------------------------
def impl_ours(args):
    import torch

    from paper_2407_00019_b200 import spmvtk as sp

    rank, world, local = dist_env()
    if world > 1 or args.force_dist:
        from paper_2407_00019_b200 import dist
        return dist.bench_main(args, rank, world, local)

    torch.cuda.set_device(0)
    stream = torch.cuda.current_stream()
    sp.set_stream(stream.cuda_stream)
    peak, peak_kind = hbm_peak()

    host = sp.HostCrs(args.config, args.param, 0.0, args.seed)
    m = host.upload()
    d = m.describe()
    n, nnz = d.n, d.nnz
    st = m.row_stats()
    nz = st.max_row

    # ---- transforms.  t_trans = one conversion timed as the reference's
    # measure_transformation (autotune.cpp:122-128): wall clock inside the
    # library around the conversion with the device synchronised on both
    # sides (spmvtk_matrix_convert_timed), allocation -- from the
    # stream-ordered pool, grown once up front -- and the band-count
    # reduction's host round trip included (median of 3 conversions); kernel =
    # median device time of the transform's kernels alone with outputs
    # preallocated.
    sp.reserve_device_memory(8 << 30)
    # process warm-up (first-call costs of the ctypes bindings and the
    # conversion paths) on a small unrelated matrix, never on the one timed
    warm = sp.HostCrs(1, 256, 0.0, args.seed).upload()
    for fmt in (sp.Format.COO_ROW, sp.Format.CCS, sp.Format.COO_COL, sp.Format.ELL,
                sp.Format.ELL_ROWMAJOR):
        warm.convert(fmt).free()
    warm.free()
    torch.cuda.synchronize()
    handles = {"crs": m}
    transforms = {}
    for name, fmt in (("coo-row", sp.Format.COO_ROW), ("ccs", sp.Format.CCS),
                      ("coo-col", sp.Format.COO_COL), ("ell", sp.Format.ELL),
                      ("ell-row", sp.Format.ELL_ROWMAJOR)):
        torch.cuda.synchronize()
        try:
            # median of 3 such conversions (each recomputes everything:
            # nothing of a conversion is cached on the handle), for a stable
            # single-conversion time
            samples = []
            for rep in range(3):
                h, t_one = m.convert_timed(
                    fmt, max_bytes=ELL_GUARD_BYTES if name.startswith("ell") else 0)
                samples.append(t_one)
                if rep < 2:
                    h.free()
            t_trans = sorted(samples)[1]
        except sp.SpmvtkError as e:  # the reference's guard (config 4's ELL)
            if e.status != sp.Status.ERR_MEMORY_LIMIT:
                raise
            transforms[name] = {"refused": e.message}
            continue
        k = m.transform_kernel_seconds(fmt, 5)
        transforms[name] = {"t_trans_ms": t_trans * 1e3, "kernel_ms": k * 1e3,
                            "gbs_kernel": transform_bytes(name, n, nnz, nz) / k / 1e9,
                            "bytes": transform_bytes(name, n, nnz, nz)}
        handles[name] = h

    x = torch.from_numpy(sp.gen_vector(n, args.seed + 1)).cuda()
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    kernels = {name: (handles[h], k) for name, h, k in (
        ("crs", "crs", sp.Kernel.CRS), ("coo-row", "coo-row", sp.Kernel.COO_ROW_OUTER),
        ("coo-col", "coo-col", sp.Kernel.COO_COL_OUTER), ("ell-inner", "ell", sp.Kernel.ELL_INNER),
        ("ell-outer", "ell", sp.Kernel.ELL_OUTER), ("ell-row", "ell-row", sp.Kernel.ELL_ROWMAJOR))
        if h in handles}

    def run(name, count):
        h, k = kernels[name]
        for _ in range(count):
            h.spmv_device(k, x.data_ptr(), y.data_ptr())

    def timed(name, count):
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        ev0.record()
        run(name, count)
        ev1.record()
        torch.cuda.synchronize()
        return ev0.elapsed_time(ev1) * 1e-3 / count

    table = {}
    per_fmt_steps = max(20, min(args.steps, 500))
    for name in kernels:
        run(name, max(3, args.warmup))
        t = timed(name, per_fmt_steps)
        b = spmv_bytes(name, n, nnz, nz)
        table[name] = {"gbs": b / t / 1e9, "gflops": 2 * nnz / t / 1e9, "ms": t * 1e3,
                       "bytes": b, "frac": b / t / 1e9 / peak}
    t_crs = table["crs"]["ms"] * 1e-3
    for name, tr in transforms.items():
        if "refused" in tr:
            continue
        tr["tt"] = tr["t_trans_ms"] * 1e-3 / t_crs       # in CRS-SpMV units
        tr["tt_kernel"] = tr["kernel_ms"] * 1e-3 / t_crs
    # AT model on GPU timings, ELL-inner variant (Eq. 1-3 as implemented);
    # a guarded ELL is an excluded record, as in the reference's profile
    if "ell-inner" in table:
        t_ell = table["ell-inner"]["ms"] * 1e-3
        t_trans = transforms["ell"]["t_trans_ms"] * 1e-3
        sp_, tt_, r_ = sp.compute_metrics(t_crs, t_ell, t_trans)
    else:
        sp_ = tt_ = r_ = None

    best = max(table, key=lambda k: table[k]["gbs"])
    launches_per_step = 1 if best != "ell-outer" else 2

    # ---- headline: K steps of the best format, device time, inputs in HBM
    run(best, args.warmup)
    with ClockSampler(0) as clk:
        t_step = timed(best, args.steps)
    bytes_step = spmv_bytes(best, n, nnz, nz)
    value = bytes_step / t_step / 1e9
    # second roofline: the x gathers.  Random columns make every x load an
    # L2 sector fetch; their rate, not HBM bandwidth, bounds config 2
    # (DESIGN.md §3).  Gathers per step = nnz (padding slots read the own
    # row's x, coalesced); peak = the measured random-gather rate.
    try:
        gpk = gather_peak(sp, torch)
        gather_roofline = {"bound": "l2-gather", "achieved": nnz / t_step / 1e9,
                           "peak": gpk / 1e9, "unit": "Ggathers/s",
                           "frac": (nnz / t_step) / gpk,
                           "peak_kind": "measured live (spmvtk_k_gather_probe)"}
    except Exception as e:  # noqa: BLE001 -- reported, not fatal
        gather_roofline = {"error": f"{type(e).__name__}: {e}"[:200]}

    # ---- e2e: through spmvtk_spmv() with pinned host buffers
    xh = torch.from_numpy(sp.gen_vector(n, args.seed + 1)).pin_memory()
    yh = torch.empty(n, dtype=torch.float64).pin_memory()
    xn, yn = xh.numpy(), yh.numpy()
    h, k = kernels[best]
    e2e_steps = max(10, min(args.steps, 200))
    for _ in range(3):
        h.spmv(xn, k, 1, out=yn)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        h.spmv(xn, k, 1, out=yn)
    t_e2e_sync = (time.perf_counter() - t0) / e2e_steps
    h.spmv_device(k, x.data_ptr(), y.data_ptr())
    torch.cuda.synchronize()
    assert np.allclose(yn, y.cpu().numpy(), rtol=1e-12, atol=0), "e2e result mismatch"
    # streaming: spmvtk_pipeline_submit keeps products in flight, so one
    # product's copy-in, another's SpMV and a third's copy-out overlap (PCIe
    # is full duplex); every step still copies its own x in and its y out
    xs = [xh, torch.from_numpy(sp.gen_vector(n, args.seed + 2)).pin_memory()]
    ys = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(2)]
    pipe = sp.Pipeline(h, k)
    for i in range(4):
        pipe.submit(xs[i % 2].numpy(), ys[i % 2].numpy())
    pipe.wait()
    t0 = time.perf_counter()
    for i in range(e2e_steps):
        pipe.submit(xs[i % 2].numpy(), ys[i % 2].numpy())
    pipe.wait()
    t_e2e = (time.perf_counter() - t0) / e2e_steps
    for i in range(2):
        xd = xs[i].cuda()
        h.spmv_device(k, xd.data_ptr(), y.data_ptr())
        torch.cuda.synchronize()
        assert np.array_equal(ys[i].numpy(), y.cpu().numpy()), "streaming e2e mismatch"
    pipe.free()

    # ---- the same kernels on config 3 (27-point stencil: x gathers are local,
    # so SpMV meets the HBM roofline there; config 2's random columns make
    # every kernel L2-sector-bound)
    also = {}
    if not args.no_also and args.config != 3:
        m3 = sp.HostCrs(3, 128, 0.0, args.seed).upload()
        d3 = m3.describe()
        nz3 = m3.row_stats().max_row
        x3 = torch.from_numpy(sp.gen_vector(d3.n, args.seed + 1)).cuda()
        y3 = torch.empty(d3.n, dtype=torch.float64, device="cuda")
        e3 = m3.convert(sp.Format.ELL)
        c3 = m3.convert(sp.Format.COO_ROW)
        tab3 = {}
        for name, h3, k3 in (("crs", m3, sp.Kernel.CRS), ("ell-inner", e3, sp.Kernel.ELL_INNER),
                             ("coo-row", c3, sp.Kernel.COO_ROW_OUTER)):
            for _ in range(5):
                h3.spmv_device(k3, x3.data_ptr(), y3.data_ptr())
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(200):
                h3.spmv_device(k3, x3.data_ptr(), y3.data_ptr())
            e1.record()
            torch.cuda.synchronize()
            t3 = e0.elapsed_time(e1) / 200 * 1e-3
            b3 = spmv_bytes(name, d3.n, d3.nnz, nz3)
            tab3[name] = {"gbs": b3 / t3 / 1e9, "gflops": 2 * d3.nnz / t3 / 1e9,
                          "us": t3 * 1e6, "frac": b3 / t3 / 1e9 / peak}
        also["config3"] = {"n": d3.n, "nnz": d3.nnz, "formats": tab3,
                           "ell_transform_kernel_ms":
                               m3.transform_kernel_seconds(sp.Format.ELL, 3) * 1e3}
        for h3 in (e3, c3, m3):
            h3.free()
        # config 1 (5 MB, L2-resident, launch-bound): SURVEY.md §8d asks for a
        # CUDA graph of >= 1000 SpMVs so launch overhead does not dominate
        try:
            also["config1_graph"] = l2_resident_graph(sp, torch, args.seed, peak)
        except Exception as e:  # reported, not fatal for the headline
            also["config1_graph"] = {"error": f"{type(e).__name__}: {e}"[:200]}

    # ---- CPU baseline: the reference itself on this host (bounded sample)
    cpu = None
    if not args.no_cpu_baseline:
        try:
            r = cpu_reference_run(host, n, nnz, nz)
            r.pop("handles")
            b = r["table"][r["best"]]
            cpu = {"value": b["gbs"], "unit": "GB/s", "cores": b["lanes"], "kind": "reference",
                   "sample": (f"reference measure_spmv (warm-up + median of 3) per format on the "
                              f"same config-{args.config} matrix; best = {r['best']} at "
                              f"{b['lanes']} lanes of {r['cores']} cores; std::thread lanes "
                              "(the reference has no OpenMP)"),
                   "formats": r["table"], "transforms": r["transforms"],
                   "cpu_model": r["cpu_model"], "nproc": r["cores"]}
        except Exception as e:  # reported, never silently replaced
            cpu = {"value": None, "unit": "GB/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"baseline config {args.config} (random rows U{{8..24}}, "
                               f"n={n})" if args.config == 2 else f"baseline config {args.config}",
                   "n": n, "nnz": nnz, "max_row": nz, "d_mat": st.d_mat, "format": best,
                   "gflops": 2 * nnz / t_step / 1e9,
                   "l2": "inputs larger than L2 (no flush)"},
        "roofline": {"bound": "hbm", "achieved": value, "peak": peak, "unit": "GB/s",
                     "frac": value / peak, "traffic": ncu_traffic(args.config, best),
                     "peak_kind": peak_kind,
                     "kernel": best, "bytes_per_launch": bytes_step},
        "roofline_gather": gather_roofline,
        "e2e": {"value": bytes_step / t_e2e / 1e9, "unit": "GB/s", "h2d_bytes_per_step": 8 * n,
                "d2h_bytes_per_step": 8 * n, "ms_per_step": t_e2e * 1e3,
                "api": "spmvtk_pipeline_submit/wait (C ABI streaming host SpMV, pinned "
                       "host x/y, copies of one product overlap other products)",
                "sync": {"value": bytes_step / t_e2e_sync / 1e9, "ms_per_step": t_e2e_sync * 1e3,
                         "api": "spmvtk_spmv (the reference's synchronous call)"}},
        "gpu_launches": args.steps * launches_per_step,
        "clocks": clk.summary(),
        "formats": table, "transforms": transforms,
        "at": {"variant": "ell-inner", "sp": sp_, "tt": tt_, "r": r_},
        "also": also,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--param", type=int, default=None)
    ap.add_argument("--seed", type=int, default=2407)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-also", action="store_true", help="skip the config-3 side table")
    ap.add_argument("--force-dist", action="store_true",
                    help="use the row-block/NCCL path even on one rank (testing)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.param is None:
        args.param = {1: 256, 2: 1 << 20, 3: 128, 4: 1 << 22, 5: 1 << 21}[args.config]
    if args.impl == "reference":
        return impl_reference(args)
    return impl_ours(args)


if __name__ == "__main__":
    sys.exit(main())
