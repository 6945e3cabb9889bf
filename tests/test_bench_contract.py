"""bench.py's reference arm runs on the host only, so its JSON contract is
checked here on CPU (config 1, a few steps): the driver parses this line."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libspmvtk_ref.so")):
        pytest.skip("oracle/_ref not built")
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "1",
                          "--steps", "3", "--warmup", "1"], cwd=ROOT, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    # the lane-parallel reference kernels are reported at one lane too
    assert {"ell-inner@1", "coo-row@1", "crs"} <= set(line["formats"])


def test_reference_arm_loads_only_the_reference_library():
    """The reference arm must not map the product library (the driver voids
    the ratio otherwise): its matrix is generated inside oracle/_ref."""
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libspmvtk_ref.so")):
        pytest.skip("oracle/_ref not built")
    code = ("import sys; sys.argv=['bench.py','--impl','reference','--config','2','--param',"
            "'4096','--steps','3','--warmup','1']\n"
            "import bench; bench.main()\n"
            "maps=open('/proc/self/maps').read()\n"
            "print('MAPPED', sorted({l.split()[-1] for l in maps.splitlines() "
            "if 'spmvtk' in l}))\n")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    mapped = [ln for ln in out.stdout.splitlines() if ln.startswith("MAPPED")][0]
    assert "libspmvtk_ref.so" in mapped and "paper_2407_00019_b200" not in mapped, mapped


def test_both_arms_share_the_config_dict():
    """workload_config() is the one source of the `config` dict in both arms."""
    sys.path.insert(0, ROOT)
    import bench
    a = bench.workload_config(4, 1 << 22, 0.0, 2407, 4194304, 67171957, 4096, 1.80181234)
    b = bench.workload_config(4, 1 << 22, 0.0, 2407, 4194304, 67171957, 4096, 1.80179999)
    assert a == b and a["workload"].startswith("BASELINE config 4")


@pytest.mark.gpu
def test_gpu_arm_json_line():
    """Our arm on the GPU (default config 4, few steps): every key the driver
    and the judge read, with sane values (the driver re-runs the full default)."""
    out = subprocess.run([sys.executable, "bench.py", "--steps", "30", "--warmup", "3",
                          "--no-also"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert key in line, key
    assert line["n_gpus"] == 1 and line["steps"] == 30 and line["warmup"] == 3
    assert line["value"] > 0 and line["unit"] == "GB/s" and line["higher_is_better"] is True
    assert line["config"]["workload"].startswith("BASELINE config 4")
    rf = line["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(rf)
    assert 0 < rf["frac"] < 2 and abs(rf["achieved"] / rf["peak"] - rf["frac"]) < 1e-9
    cb = line["cpu_baseline"]
    assert {"value", "unit", "cores", "kind", "sample"} <= set(cb) and cb["value"] > 0
    e2e = line["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert line["gpu_launches"] >= line["steps"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(line["clocks"])
    # the transforms table carries TT for every format the guard admits
    assert all("tt" in v for v in line["transforms"].values() if "refused" not in v)
