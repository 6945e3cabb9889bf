"""Off-line AT phase on k GPUs (torchrun, one rank per GPU): every matrix of
BASELINE config 5's D_mat sweep (plus configs 1-3 with --extra) is cut into
the entry-balanced row blocks the multi-GPU SpMV uses, each rank generating
only its own block (spmvtk_gen_baseline_shard_host); each
rank times its shard with spmvtk_bench (t_crs, t_ell, t_trans -- the
reference's protocol), the job's time is the max over ranks, and
R = SP / TT and D* follow from those (autotune.cpp:36-44, :130-158).  D_mat
is the global matrix's.  On one GPU this reproduces tools/at_graph.py.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/at_graph_dist.py \\
        [--param 2097152] [--extra] [--out profiles/r01_at_graph_dist]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2407_00019_b200 import spmvtk as sp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--param", type=int, default=1 << 21)
ap.add_argument("--repeats", type=int, default=9)
ap.add_argument("--max-bytes", type=int, default=48 << 30)
ap.add_argument("--extra", action="store_true", help="add configs 1-3")
ap.add_argument("--reserve", type=int, default=64, help="GiB of pool grown up front")
ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_at_graph_dist"))
a = ap.parse_args()
rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
sp.set_stream(torch.cuda.current_stream().cuda_stream)
sp.reserve_device_memory(a.reserve << 30)  # t_trans = conversion, not pool growth
w = sp.HostCrs(1, 256).upload()  # first-call costs out of the first record
for f in (sp.Format.ELL, sp.Format.COO_ROW):
    w.convert(f).free()
w.free()

work = [(f"cfg5_D{0.1 * i:.1f}", 5, a.param, round(0.1 * i, 1), 2407 + i) for i in range(21)]
if a.extra:
    work += [(f"cfg{c}", c, p, 0.0, 2407) for c, p in ((1, 256), (2, 1 << 20), (3, 128))]
records = []
for mid, cfg, param, dp, seed in work:
    # t = [t_crs, t_ell, t_trans, excluded, failed, rows, entries, sum of squared lengths]
    t = torch.zeros(8, dtype=torch.float64, device="cuda")
    err = ""
    try:
        host = sp.gen_baseline_shard_host(cfg, param, dp, seed, rank, world)
        lrp, _, _ = host.arrays(index_base=0)
        lens = np.diff(lrp).astype(np.float64)
        t[5:8] = torch.tensor([host.n, lens.sum(), (lens * lens).sum()], dtype=torch.float64)
        n = host.ncols
        shard = host.upload()
        host.free()
        try:
            b = sp.bench(shard, sp.Kernel.ELL_INNER, 1, a.repeats, a.max_bytes)
            t[:3] = torch.tensor([b["t_crs"], b["t_ell"], b["t_trans"]], dtype=torch.float64)
        except sp.SpmvtkError as e:  # the memory guard: excluded on every rank
            if e.status != sp.Status.ERR_MEMORY_LIMIT:
                raise
            t[3] = 1.0
        finally:
            shard.free()
    except Exception as e:  # noqa: BLE001 -- agreed below, never a lone raise
        t[4] = 1.0
        err = f"{type(e).__name__}: {e}"
    mx = t[:5].clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    sums = t[5:].clone()
    dist.all_reduce(sums, op=dist.ReduceOp.SUM)
    if mx[4].item():  # some rank failed: every rank stops here together
        raise SystemExit(f"rank {rank}: {mid} failed on a rank ({err or 'another rank'})")
    t = torch.cat([mx[:4], sums])
    rows_g, ent_g, sq_g = (float(u) for u in sums.tolist())
    mu = ent_g / rows_g
    d_mat = (max(sq_g / rows_g - mu * mu, 0.0) ** 0.5) / mu
    t_crs, t_ell, t_trans, excl = (float(u) for u in t[:4].tolist())
    rec = {"matrix_id": mid, "d_mat": d_mat, "excluded": bool(excl)}
    if not excl:
        spd, tt, r = sp.compute_metrics(t_crs, t_ell, t_trans)
        rec.update(t_crs=t_crs, t_ell=t_ell, t_trans=t_trans, sp=spd, tt=tt, r=r)
    records.append(rec)
    if rank == 0:
        print(f"{mid:12s} d_mat={d_mat:.4f} " + ("excluded" if excl else
              f"R={rec['r']:.4g} SP={rec['sp']:.4g} TT={rec['tt']:.4g} "
              f"t_crs={t_crs * 1e6:.1f}us t_ell={t_ell * 1e6:.1f}us "
              f"t_trans={t_trans * 1e6:.1f}us"), flush=True)
if rank == 0:
    pairs = [(r["d_mat"], r["r"]) for r in records if not r["excluded"]]
    with open(f"{a.out}{world}.csv", "w") as f:
        f.write("matrix_id,d_mat,r,sp,tt,t_crs_us,t_ell_us,t_trans_us,excluded\n")
        for r in records:
            if r["excluded"]:
                f.write(f"{r['matrix_id']},{r['d_mat']:.6f},,,,,,,1\n")
            else:
                f.write(f"{r['matrix_id']},{r['d_mat']:.6f},{r['r']:.6g},{r['sp']:.6g},"
                        f"{r['tt']:.6g},{r['t_crs'] * 1e6:.2f},{r['t_ell'] * 1e6:.2f},"
                        f"{r['t_trans'] * 1e6:.2f},0\n")
    print(json.dumps({"gpus": world, "variant": "ell-inner",
                      "d_star": sp.find_d_star(pairs, 1.0),
                      "d_star_c0.5": sp.find_d_star(pairs, 0.5)}), flush=True)
dist.barrier()
dist.destroy_process_group()
