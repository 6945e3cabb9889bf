"""Off-line AT phase on the GPU over BASELINE config 5's D_mat sweep (21
matrices, D = 0.0 .. 2.0) plus configs 1-4: builds the profile through the C
ABI (spmvtk_profile_build: t_crs, t_trans, t_variant, R = SP/TT), writes the
profile JSON (schema v1) and a matrix_id,d_mat,r,sp,tt CSV, prints D*.

    python tools/at_graph.py [--param 2097152] [--variant ell-inner] [--out profiles/r01_at]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2407_00019_b200 import spmvtk as sp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--param", type=int, default=1 << 21)
ap.add_argument("--variant", default="ell-inner")
ap.add_argument("--repeats", type=int, default=9)
ap.add_argument("--max-bytes", type=int, default=48 << 30)
ap.add_argument("--extra", action="store_true", help="add configs 1-4")
ap.add_argument("--reserve", type=int, default=64, help="GiB")
ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_at_graph"))
a = ap.parse_args()
sp.set_stream(torch.cuda.current_stream().cuda_stream)
kern = {v: k for k, v in sp.KERNEL_NAMES.items()}[a.variant]
mats, ids = [], []
for i in range(21):
    d = round(0.1 * i, 1)
    mats.append(sp.HostCrs(5, a.param, d, 2407 + i).upload())
    ids.append(f"cfg5_D{d:.1f}")
if a.extra:
    for cfg, param in ((1, 256), (2, 1 << 20), (3, 128), (4, 1 << 22)):
        mats.append(sp.HostCrs(cfg, param).upload())
        ids.append(f"cfg{cfg}")
sp.reserve_device_memory(a.reserve << 30)  # pool grown once: t_trans = conversion, not pool growth
# process warm-up of the conversion paths on an unrelated small matrix, so
# the first profiled matrix's t_trans carries no first-call costs
_w = sp.HostCrs(1, 256).upload()
for _f in (sp.Format.ELL, sp.Format.ELL_ROWMAJOR, sp.Format.COO_ROW):
    _w.convert(_f).free()
_w.free()
prof = sp.Profile.build(mats, ids, kern, 1, 1.0, a.repeats, a.max_bytes, "B200 (sm_100a)")
prof.write(a.out + ".json")
recs = prof.records()


def amort(r):
    if r["excluded"]:
        return ""
    k = sp.amortization_iterations(r["t_crs"], r["t_ell"], r["t_trans"])
    return "" if k is None else k



with open(a.out + ".csv", "w") as f:
    f.write("matrix_id,d_mat,r,sp,tt,t_crs_us,t_ell_us,t_trans_us,amortize_k,excluded\n")
    for r in recs:
        f.write(f"{r['matrix_id']},{r['d_mat']:.6f},{r['r']:.6g},{r['sp']:.6g},{r['tt']:.6g},"
                f"{r['t_crs']*1e6:.2f},{r['t_ell']*1e6:.2f},{r['t_trans']*1e6:.2f},"
                f"{amort(r)},{int(r['excluded'])}\n")
for r in recs:
    print(f"{r['matrix_id']:12s} d_mat={r['d_mat']:.4f} R={r['r']:.4g} SP={r['sp']:.4g} "
          f"TT={r['tt']:.4g} k={amort(r)} excluded={r['excluded']} {r['exclusion_reason'] or ''}")
print(json.dumps({"variant": a.variant, "c": prof.c, "d_star": prof.d_star,
                  "d_star_c0.5": sp.find_d_star([(r["d_mat"], r["r"]) for r in recs
                                                 if not r["excluded"]], 0.5),
                  "d_star_c0.25": sp.find_d_star([(r["d_mat"], r["r"]) for r in recs
                                                  if not r["excluded"]], 0.25)}))
