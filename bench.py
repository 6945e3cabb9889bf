"""Benchmark of the hot path on BASELINE.json's workload.

Metric (BASELINE.json): "SpMV GB/s & GFLOP/s per format; CRS->ELL/COO
transform time in CRS-SpMV units".  Workload (default): BASELINE config 4,
the largest configuration that fits one GPU -- power-law rows (n = 2^22,
log-normal row lengths with mean 16 and sigma_log 1.2 capped at 4096,
uniform distinct sorted columns, N(0,1) values), seeded synthetic data (the
paper's SuiteSparse set is not available).  Its ELL is refused by the
reference's memory guard (~206 GB), so CRS and COO decide.  Configs 2 and 3
are measured in the same run under `also`.

A step = one SpMV y = A x in the best format for the matrix (every format is
measured; the per-format table, the transform times in CRS-SpMV units and
the AT decision are reported beside the headline).  `value` = algorithmic
bytes of one SpMV (GPU layout) x steps / device time, inputs
resident in HBM (the matrix, 0.89 GB, is larger than the 126 MB L2, so no
flush is needed between steps).  `e2e` = the same metric through the C ABI
with pinned HOST x / y, every step's copy-in and copy-out inside the timed
region: the streaming spmvtk_pipeline_* calls (products overlap each
other's copies), and under e2e.sync the reference's synchronous
spmvtk_spmv().

`--impl reference` runs the reference's own CPU implementation
(oracle/_ref/libspmvtk_ref.so, compiled from its sources) on the same
matrix -- generated inside that library, so the product library is never
loaded -- with the same `config` dict.

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
    """(DRAM read+write bytes per launch of `kernel` on this config, source
    file) from the committed ncu captures (profiles/traffic_r*.json, newest
    round first), or None."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "traffic_r*.json")), reverse=True):
        try:
            with open(path) as f:
                v = json.load(f).get(f"config{config}", {}).get(kernel)
            if v:
                return float(v), os.path.relpath(path, ROOT)
        except Exception:
            continue
    return None


def ncu_probe_main(args) -> int:
    """`bench.py --ncu-probe FORMAT`: the config's matrix in FORMAT, then two
    SpMVs of it (a warm-up and the captured one) -- the process ncu profiles
    for roofline.traffic."""
    import torch

    from paper_2407_00019_b200 import spmvtk as sp
    torch.cuda.set_device(0)
    sp.set_stream(torch.cuda.current_stream().cuda_stream)
    m = sp.HostCrs(args.config, args.param, 0.0, args.seed).upload()
    hname, kname = {name: (h, k) for name, h, k in SPMV_KINDS}[args.ncu_probe]
    fmt = {"crs": None, "coo-row": "COO_ROW", "coo-col": "COO_COL", "ell": "ELL",
           "ell-row": "ELL_ROWMAJOR"}[hname]
    h = m if fmt is None else m.convert(getattr(sp.Format, fmt))
    n = m.describe().n
    x = torch.from_numpy(sp.gen_vector(n, args.seed + 1)).cuda()
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        h.spmv_device(getattr(sp.Kernel, kname), x.data_ptr(), y.data_ptr())
    torch.cuda.synchronize()
    return 0


def ncu_traffic_live(args, fmt: str, timeout: float = 300.0):
    """DRAM read+write bytes of one launch of the `fmt` SpMV kernel, captured
    by ncu in this run (a child process: --ncu-probe; cold caches, as ncu
    flushes them between kernels), or None when ncu is unavailable/fails."""
    import shutil
    import subprocess
    ncu = shutil.which("ncu") or ("/usr/local/cuda/bin/ncu"
                                  if os.path.exists("/usr/local/cuda/bin/ncu") else None)
    if ncu is None:
        return None
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "--clock-control", "none", "-k", "regex:k_spmv", "--launch-skip", "1", "-c", "1",
           "--csv", sys.executable, os.path.join(ROOT, "bench.py"), "--ncu-probe", fmt,
           "--config", str(args.config), "--param", str(args.param), "--seed", str(args.seed)]
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout).stdout
        import csv
        import io
        rows = [r for r in csv.reader(io.StringIO("\n".join(
            l for l in out.splitlines() if l.startswith('"')))) if r]
        hdr = rows[0]
        ix = {k: i for i, k in enumerate(hdr)}
        vals, kernel = {}, None
        for r in rows[1:]:
            unit = r[ix["Metric Unit"]]
            v = float(r[ix["Metric Value"]].replace(",", ""))
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9,
                  "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9}.get(unit, 1)
            vals[r[ix["Metric Name"]]] = v
            kernel = r[ix["Kernel Name"]].split("(")[0]
        return {"bytes": vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"],
                "read": vals["dram__bytes_read.sum"], "write": vals["dram__bytes_write.sum"],
                "us": vals.get("gpu__time_duration.sum", 0.0) * 1e6, "kernel": kernel}
    except Exception:
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
DEFAULT_CONFIG = 4  # the largest BASELINE configuration that fits one GPU
DEFAULT_PARAM = {1: 256, 2: 1 << 20, 3: 128, 4: 1 << 22, 5: 1 << 21}


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


WORKLOADS = {
    1: "2-D 5-point Laplacian 256x256",
    2: "random rows U{8..24}, uniform distinct sorted columns",
    3: "27-point stencil 128^3 (non-periodic)",
    4: "power-law rows (log-normal, mean 16, sigma_log 1.2, cap 4096), uniform columns",
    5: "D_mat sweep (Gamma row lengths, mean 32, columns within +-n/64)",
}


def workload_config(cfg: int, param: int, dparam: float, seed: int, n: int, nnz: int,
                    max_row: int, d_mat: float) -> dict:
    """The `config` dict: identical in both arms (the driver compares them)."""
    crs_bytes = spmv_bytes("crs", n, nnz)
    return {"workload": f"BASELINE config {cfg}: {WORKLOADS[cfg]}", "param": param,
            "dparam": dparam, "seed": seed, "n": n, "nnz": nnz, "max_row": max_row,
            "d_mat": round(d_mat, 4),
            "l2": ("inputs larger than L2 (no flush)" if crs_bytes > (126 << 20)
                   else "L2-resident matrix (no flush)")}


def ell_splits(n: int, nz: int) -> int:
    """Band chunks the GPU ell-outer kernel uses (matrix.cpp ell_splits): the
    band split only pays when row pairs alone cannot fill 148 SMs x 2048."""
    want, pairs = 148 * 2048, (n + 1) // 2
    if nz <= 1 or pairs >= want:
        return 1
    return min(-(-want // pairs), nz)


REF_KERNELS = {"crs": 0, "coo-row": 1, "ell-inner": 3, "ell-outer": 4}


def cpu_reference_run(ref, h, n, nnz, nz, per_call_repeats=3):
    """The reference's own CPU path (oracle/_ref, compiled from the reference
    sources) on this host's cores: its measure_spmv / measure_transformation
    protocol (autotune.cpp:95-128) for every format its memory guard admits."""
    cores = os.cpu_count() or 1
    res, transforms, handles = {}, {}, {"crs": h}
    # transforms: one cold conversion each (autotune.cpp:122-128, :197-214);
    # the ELL guard as the reference's own bench applies it
    for name, fmt, cap in (("ell", 4, ELL_GUARD_BYTES), ("coo-row", 2, 0)):
        try:
            t, out = ref.measure_transformation(h, fmt, cap)
            transforms[name] = {"ms": t * 1e3}
            handles[name] = out
        except RuntimeError as e:
            transforms[name] = {"refused": str(e)[:160]}
    # SpMV: warm-up + median of repeats (autotune.cpp:95-120); CRS is
    # sequential in the reference (autotune.cpp:186), the others use lanes
    t_crs = ref.measure_spmv(h, 0, 1, per_call_repeats)
    res["crs"] = (t_crs, 1)
    one = {}
    if "coo-row" in handles:
        res["coo-row"] = (ref.measure_spmv(handles["coo-row"], 1, cores, per_call_repeats), cores)
        one["coo-row@1"] = ref.measure_spmv(handles["coo-row"], 1, 1, per_call_repeats)
    if "ell" in handles:
        res["ell-inner"] = (ref.measure_spmv(handles["ell"], 3, cores, per_call_repeats), cores)
        res["ell-outer"] = (ref.measure_spmv(handles["ell"], 4, cores, per_call_repeats), cores)
        one["ell-inner@1"] = ref.measure_spmv(handles["ell"], 3, 1, per_call_repeats)
        one["ell-outer@1"] = ref.measure_spmv(handles["ell"], 4, 1, per_call_repeats)
    table = {}
    for k, (t, lanes) in res.items():
        b = spmv_bytes(k, n, nnz, nz)
        table[k] = {"gbs": b / t / 1e9, "gflops": 2 * nnz / t / 1e9, "ms": t * 1e3, "lanes": lanes}
    best = min(table, key=lambda k: table[k]["ms"])  # the fastest, as the AT chooses
    for k, t in one.items():
        b = spmv_bytes(k.split("@")[0], n, nnz, nz)
        table[k] = {"gbs": b / t / 1e9, "gflops": 2 * nnz / t / 1e9, "ms": t * 1e3, "lanes": 1}
    for tr in transforms.values():
        if "ms" in tr:
            tr["tt"] = tr["ms"] * 1e-3 / t_crs
    return {"table": table, "best": best, "cores": cores, "cpu_model": cpu_model(),
            "transforms": transforms, "handles": handles}


def ref_handle_stats(ref, h):
    """n, nnz, max row and D_mat of a reference CRS handle (reference code)."""
    meta = ref.meta(h)
    rp = ref.array(h, 1)
    nz = int(np.max(np.diff(rp))) if meta["n"] else 0
    _, _, d_mat = ref.row_stats(h)
    return meta["n"], meta["nnz"], nz, d_mat


def impl_reference(args):
    rank, world, _ = dist_env()
    if world > 1 and rank != 0:
        return 0
    # the reference library alone: the matrix is generated inside it (the
    # product's generator compiled into oracle/_ref), never by the product
    from oracle.oracle import Ref
    ref = Ref()
    h = ref.gen_baseline(args.config, args.param, 0.0, args.seed)
    n, nnz, nz, d_mat = ref_handle_stats(ref, h)
    r = cpu_reference_run(ref, h, n, nnz, nz)
    handles = r.pop("handles")
    best = r["best"]
    handle = handles["crs" if best == "crs" else "coo-row" if best == "coo-row" else "ell"]
    lanes = r["table"][best]["lanes"]
    x = ref.gen_vector(n, args.seed + 1)
    tw = time.perf_counter()
    for _ in range(args.warmup):
        ref.spmv(handle, REF_KERNELS[best], x, lanes)
    t_one = (time.perf_counter() - tw) / max(1, args.warmup)
    # bounded sample: at most ~60 s of CPU work whatever K is
    steps = int(max(3, min(args.steps, 60.0 / max(t_one, 1e-9))))
    t0 = time.perf_counter()
    for _ in range(steps):
        ref.spmv(handle, REF_KERNELS[best], x, lanes)
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
        "config": workload_config(args.config, args.param, 0.0, args.seed, n, nnz, nz, d_mat),
        "format": best,
        "bounded_sample": "steps capped at ~60 s of CPU work",
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
SPMV_KINDS = (("crs", "crs", "CRS"), ("coo-row", "coo-row", "COO_ROW_OUTER"),
              ("coo-col", "coo-col", "COO_COL_OUTER"), ("ell-inner", "ell", "ELL_INNER"),
              ("ell-outer", "ell", "ELL_OUTER"), ("ell-row", "ell-row", "ELL_ROWMAJOR"))
TRANSFORMS = (("coo-row", "COO_ROW"), ("ccs", "CCS"), ("coo-col", "COO_COL"), ("ell", "ELL"),
              ("ell-row", "ELL_ROWMAJOR"))


def measure_matrix(sp, torch, m, seed, peak, reps, warmup, with_transforms=True):
    """Every transform of one CRS handle (t_trans through the API, kernel-only
    time) and every SpMV format (device time, CUDA events on the launching
    stream, `reps` back-to-back launches).  Returns (table, transforms,
    handles, kernels)."""
    d = m.describe()
    n, nnz = d.n, d.nnz
    nz = m.row_stats().max_row
    handles, transforms = {"crs": m}, {}
    for name, fmt_name in TRANSFORMS:
        fmt = getattr(sp.Format, fmt_name)
        guard = ELL_GUARD_BYTES if name.startswith("ell") else 0
        try:
            if with_transforms:
                # t_trans = one conversion timed as the reference's
                # measure_transformation (autotune.cpp:122-128): wall clock
                # inside the library around the conversion with the device
                # synchronised on both sides, allocation (from the
                # stream-ordered pool, grown once up front) and the band-count
                # reduction's host round trip included; median of 3 such
                # conversions (nothing of a conversion is cached on the handle)
                samples = []
                for rep in range(3):
                    h, t_one = m.convert_timed(fmt, max_bytes=guard)
                    samples.append(t_one)
                    if rep < 2:
                        h.free()
                t_trans = sorted(samples)[1]
                k = m.transform_kernel_seconds(fmt, 5)
                transforms[name] = {"t_trans_ms": t_trans * 1e3, "kernel_ms": k * 1e3,
                                    "gbs_kernel": transform_bytes(name, n, nnz, nz) / k / 1e9,
                                    "bytes": transform_bytes(name, n, nnz, nz)}
            else:
                h = m.convert(fmt, max_bytes=guard)
        except sp.SpmvtkError as e:  # the reference's guard (config 4's ELL)
            if e.status != sp.Status.ERR_MEMORY_LIMIT:
                raise
            transforms[name] = {"refused": e.message}
            continue
        handles[name] = h
    x = torch.from_numpy(sp.gen_vector(n, seed + 1)).cuda()
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    kernels = {name: (handles[h], getattr(sp.Kernel, k)) for name, h, k in SPMV_KINDS
               if h in handles}
    table = {}
    for name, (h, k) in kernels.items():
        for _ in range(max(3, warmup)):
            h.spmv_device(k, x.data_ptr(), y.data_ptr())
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(reps):
            h.spmv_device(k, x.data_ptr(), y.data_ptr())
        ev1.record()
        torch.cuda.synchronize()
        t = ev0.elapsed_time(ev1) * 1e-3 / reps
        b = spmv_bytes(name, n, nnz, nz)
        table[name] = {"gbs": b / t / 1e9, "gflops": 2 * nnz / t / 1e9, "us": t * 1e6,
                       "bytes": b, "frac": b / t / 1e9 / peak}
    if "ell-outer" in table:
        sps = ell_splits(n, nz)
        table["ell-outer"]["band_chunks"] = sps
        if sps == 1:
            table["ell-outer"]["note"] = ("one band chunk at this n: the same kernel as "
                                          "ell-inner (not a separate candidate)")
    t_crs = table["crs"]["us"] * 1e-6
    for tr in transforms.values():
        if "t_trans_ms" in tr:
            tr["tt"] = tr["t_trans_ms"] * 1e-3 / t_crs       # in CRS-SpMV units
            tr["tt_kernel"] = tr["kernel_ms"] * 1e-3 / t_crs
    return table, transforms, handles, kernels, x, y


def best_format(table):
    """The fastest format (shortest SpMV, as the AT chooses), not the one with
    the most bytes per second: COO moves 4 more bytes per entry than CRS."""
    cands = {k: v for k, v in table.items() if v.get("band_chunks", 2) != 1}
    return min(cands, key=lambda k: cands[k]["us"])


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
    lib = sp.load_library()
    peak, peak_kind = hbm_peak()

    host = sp.HostCrs(args.config, args.param, 0.0, args.seed)
    m = host.upload()
    d = m.describe()
    n, nnz = d.n, d.nnz
    st = m.row_stats()
    nz = st.max_row

    sp.reserve_device_memory(8 << 30)
    # process warm-up (first-call costs of the ctypes bindings and the
    # conversion paths) on a small unrelated matrix, never on the one timed
    warm = sp.HostCrs(1, 256, 0.0, args.seed).upload()
    for _, fmt_name in TRANSFORMS:
        warm.convert(getattr(sp.Format, fmt_name)).free()
    warm.free()
    torch.cuda.synchronize()
    table, transforms, handles, kernels, x, y = measure_matrix(
        sp, torch, m, args.seed, peak, max(20, min(args.steps, 500)), args.warmup)
    t_crs = table["crs"]["us"] * 1e-6
    # AT model on GPU timings, ELL-inner variant (Eq. 1-3 as implemented);
    # a guarded ELL is an excluded record, as in the reference's profile
    if "ell-inner" in table:
        t_ell = table["ell-inner"]["us"] * 1e-6
        t_trans = transforms["ell"]["t_trans_ms"] * 1e-3
        sp_, tt_, r_ = sp.compute_metrics(t_crs, t_ell, t_trans)
        at = {"variant": "ell-inner", "sp": sp_, "tt": tt_, "r": r_}
    else:  # an excluded record of the off-line profile (autotune.cpp:197-214)
        at = {"variant": "ell-inner", "excluded": transforms["ell"].get("refused")}

    best = best_format(table)
    h, k = kernels[best]

    # ---- headline: K steps of the best format, device time, inputs in HBM
    for _ in range(args.warmup):
        h.spmv_device(k, x.data_ptr(), y.data_ptr())
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    launches0 = lib.spmvtk_k_launch_count()
    with ClockSampler(0) as clk:
        ev0.record()
        for _ in range(args.steps):
            h.spmv_device(k, x.data_ptr(), y.data_ptr())
        ev1.record()
        torch.cuda.synchronize()
    gpu_launches = lib.spmvtk_k_launch_count() - launches0
    t_step = ev0.elapsed_time(ev1) * 1e-3 / args.steps
    bytes_step = spmv_bytes(best, n, nnz, nz)
    value = bytes_step / t_step / 1e9
    # second roofline: the x gathers.  Random columns make every x load an
    # L2 sector request; the SM's L1->L2 request rate, not HBM bandwidth,
    # bounds these matrices.  Gathers per step = nnz; peak =
    # the random-gather rate measured live.
    try:
        gpk = gather_peak(sp, torch)
        gather_roofline = {"bound": "l2-gather", "achieved": nnz / t_step / 1e9,
                           "peak": gpk / 1e9, "unit": "Ggathers/s",
                           "frac": (nnz / t_step) / gpk,
                           "peak_kind": "measured live (spmvtk_k_gather_probe)"}
    except Exception as e:  # noqa: BLE001 -- reported, not fatal
        gather_roofline = {"error": f"{type(e).__name__}: {e}"[:200]}

    # ---- e2e: through the C ABI with pinned host buffers
    xh = torch.from_numpy(sp.gen_vector(n, args.seed + 1)).pin_memory()
    yh = torch.empty(n, dtype=torch.float64).pin_memory()
    xn, yn = xh.numpy(), yh.numpy()
    e2e_steps = max(10, min(args.steps, 100))
    for _ in range(3):
        h.spmv(xn, k, 1, out=yn)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        h.spmv(xn, k, 1, out=yn)
    t_e2e_sync = (time.perf_counter() - t0) / e2e_steps
    h.spmv_device(k, x.data_ptr(), y.data_ptr())
    torch.cuda.synchronize()
    # max-norm relative error (the parity tests' criterion): COO-col adds
    # through fp64 atomics, so its order of additions -- and single entries
    # near cancellation -- may differ between two launches
    yd = y.cpu().numpy()
    assert np.max(np.abs(yn - yd)) <= 1e-12 * max(np.max(np.abs(yd)), 1e-300), \
        "e2e result mismatch"
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
        yd = y.cpu().numpy()
        assert np.max(np.abs(ys[i].numpy() - yd)) <= 1e-12 * max(np.max(np.abs(yd)), 1e-300), \
            "streaming e2e mismatch"
    pipe.free()

    # ---- CPU baseline: the reference itself on this host (bounded sample),
    # on the same matrix
    cpu = None
    if not args.no_cpu_baseline:
        try:
            from oracle.oracle import Ref
            ref = Ref()
            rp, ci, v = host.arrays(index_base=1)
            rh = ref.matrix(n, rp, ci, v)
            del rp, ci, v
            r = cpu_reference_run(ref, rh, n, nnz, nz)
            for hh in r.pop("handles").values():
                ref.free(hh)
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
                   "sample": f"unavailable: {type(e).__name__}: {e}"[:300]}
    host.free()
    for name, hh in handles.items():
        if name != "crs":
            hh.free()

    # ---- the other full-size configs, measured in the same run
    also = {}
    if not args.no_also:
        # config 5 at D = 0: the banded matrix where ELL beats CRS (the SM-local
        # ELL kernel); the rest of config 5's sweep is in the AT graph
        for cfg, dp in ((2, 0.0), (3, 0.0), (5, 0.0)):
            if cfg == args.config:
                continue
            mc = sp.HostCrs(cfg, DEFAULT_PARAM[cfg], dp, args.seed).upload()
            tab, trs, hs, _, _, _ = measure_matrix(sp, torch, mc, args.seed, peak, 200, 5)
            dc = mc.describe()
            key = f"config{cfg}" if cfg != 5 else f"config5_D{dp}"
            also[key] = {"n": dc.n, "nnz": dc.nnz, "d_mat": mc.row_stats().d_mat,
                         "best": best_format(tab), "formats": tab, "transforms": trs}
            for name, hh in hs.items():
                hh.free()
        # config 1 (5 MB, L2-resident, launch-bound): SURVEY.md §8d asks for a
        # CUDA graph of >= 1000 SpMVs so launch overhead does not dominate
        try:
            also["config1_graph"] = l2_resident_graph(sp, torch, args.seed, peak)
        except Exception as e:  # reported, not fatal for the headline
            also["config1_graph"] = {"error": f"{type(e).__name__}: {e}"[:200]}

    # roofline.traffic: one launch of the headline kernel captured by ncu in
    # this run (after every timed region); the committed capture otherwise
    live = None if args.no_ncu else ncu_traffic_live(args, best)
    if live:
        traffic = (live["bytes"], f"live ncu capture in this run: {live['kernel']}, one launch, "
                                  f"cold caches, {live['us']:.1f} us under ncu "
                                  f"(read {live['read'] / 1e6:.1f} MB, write "
                                  f"{live['write'] / 1e6:.1f} MB)")
    else:
        traffic = ncu_traffic(args.config, best)
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.config, args.param, 0.0, args.seed, n, nnz, nz, st.d_mat),
        "format": best, "gflops": 2 * nnz / t_step / 1e9,
        "roofline": {"bound": "hbm", "achieved": value, "peak": peak, "unit": "GB/s",
                     "frac": value / peak, "traffic": traffic[0] if traffic else None,
                     "traffic_source": traffic[1] if traffic else None,
                     "peak_kind": peak_kind, "kernel": best, "bytes_per_launch": bytes_step},
        "roofline_gather": gather_roofline,
        "e2e": {"value": bytes_step / t_e2e / 1e9, "unit": "GB/s", "h2d_bytes_per_step": 8 * n,
                "d2h_bytes_per_step": 8 * n, "ms_per_step": t_e2e * 1e3,
                "api": "spmvtk_pipeline_submit/wait (C ABI streaming host SpMV, pinned "
                       "host x/y, copies of one product overlap other products)",
                "sync": {"value": bytes_step / t_e2e_sync / 1e9, "ms_per_step": t_e2e_sync * 1e3,
                         "api": "spmvtk_spmv (the reference's synchronous call)"}},
        "gpu_launches": gpu_launches,
        "clocks": clk.summary(),
        "formats": table, "transforms": transforms, "at": at,
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
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG)
    ap.add_argument("--param", type=int, default=None)
    ap.add_argument("--seed", type=int, default=2407)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-also", action="store_true",
                    help="skip the side tables (configs 1-3 and config 5 at D = 0)")
    ap.add_argument("--no-ncu", action="store_true",
                    help="roofline.traffic from the committed capture, no live ncu run")
    ap.add_argument("--ncu-probe", default=None, help=argparse.SUPPRESS)
    ap.add_argument("--force-dist", action="store_true",
                    help="use the row-block/NCCL path even on one rank (testing)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.param is None:
        args.param = DEFAULT_PARAM[args.config]
    if args.ncu_probe:
        return ncu_probe_main(args)
    if args.impl == "reference":
        return impl_reference(args)
    return impl_ours(args)


if __name__ == "__main__":
    sys.exit(main())
