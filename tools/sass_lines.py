"""Aggregates an ncu report's per-instruction warp-stall samples of one kernel
by CUDA source line, using the line table of the kernel's cubin.

    python tools/sass_lines.py rep.ncu-rep KERNEL_SUBSTR build/obj.o [top] [skip]

KERNEL_SUBSTR selects the kernel both in the report (regex) and among the
cubin's mangled names (substring, e.g. k_bkt_sortILi512); "REGEX::SUBSTR"
gives the two separately (e.g. k_bkt_scatter::13k_bkt_scatterP with skip 1
for the second matching launch).  Needs the object
compiled with -lineinfo (the Makefile does)."""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, kern, obj = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
skip = sys.argv[5] if len(sys.argv) > 5 else "0"  # matching launches to skip
kregex, kern = kern.split("::", 1) if "::" in kern else (re.sub(r"ILi\d+E?.*", "", kern), kern)

# ncu: instructions in address order with samples
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--kernel-name", "regex:" + kregex,
                      "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
ix = {k: i for i, k in enumerate(h)}
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
body, seen = [], set()
for r in rows[hi + 1:]:
    if len(r) != len(h) or r[0] == "Address" or r[0] in seen:
        continue
    seen.add(r[0])
    body.append(r)
base = min(int(r[0], 16) for r in body)

# cubin line table
with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=td,
                   capture_output=True)
    cubins = [os.path.join(td, f) for f in os.listdir(td) if f.endswith(".cubin")]
    sass = subprocess.run(["nvdisasm", "-g", "-c", cubins[0]], capture_output=True,
                          text=True).stdout
line_of, cur_fn, cur_line = {}, None, None
for ln in sass.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", ln) or re.match(r"^(_Z\S+):$", ln.strip())
    if ln.startswith(".text.") and ln.endswith(":"):
        cur_fn = ln[6:-1]
        continue
    m = re.search(r'## File "([^"]+)", line (\d+)', ln)
    if m:
        cur_line = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and cur_fn and kern in cur_fn:
        line_of[int(m.group(1), 16)] = cur_line

agg = collections.defaultdict(lambda: collections.Counter())
tot = 0.0
for r in body:
    off = int(r[0], 16) - base
    key = line_of.get(off, ("?", 0))
    smp = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    tot += smp
    agg[key]["samples"] += smp
    agg[key]["inst"] += float(r[ix["Instructions Executed"]] or 0)
    for k in stalls:
        agg[key][k[6:]] += float(r[ix[k]] or 0)
src = {}
for key in agg:
    if key[0] != "?":
        for d in ("paper_2407_00019_b200/csrc", "include/spmvtk"):
            p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), d, key[0])
            if os.path.exists(p):
                src[key[0]] = open(p).read().splitlines()
for key, c in sorted(agg.items(), key=lambda kv: -kv[1]["samples"])[:top]:
    text = src.get(key[0], [])
    code = text[key[1] - 1].strip()[:58] if 0 < key[1] <= len(text) else ""
    st = sorted(((v, k) for k, v in c.items() if k not in ("samples", "inst")), reverse=True)[:2]
    print(f"{key[0][:18]:18s}:{key[1]:<5d} {100 * c['samples'] / tot:5.1f}%  inst={c['inst']:9.0f}  "
          f"{code:58s} " + " ".join(f"{k}={100 * v / max(c['samples'], 1):.0f}%" for v, k in st if v))
