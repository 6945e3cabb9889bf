"""Lists the hottest SASS instructions (warp-stall samples) of one kernel in
an ncu report: sass_hot.py rep kernel_regex [top]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--kernel-name", f"regex:{kern}", "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
ix = {k: i for i, k in enumerate(h)}
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
body = [r for r in rows[hi + 1:] if len(r) == len(h) and r[0] != "Address"]
tot = sum(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in body)
body.sort(key=lambda r: -float(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
for r in body[:top]:
    smp = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    st = sorted(((float(r[ix[k]] or 0), k[6:]) for k in stalls), reverse=True)[:2]
    print(f"{r[0]:>6} {100*smp/tot:5.1f}%  {r[1][:60]:60s} " +
          " ".join(f"{k}={v:.0f}" for v, k in st if v))
