"""One CRS->CCS (or COO-col) conversion of a BASELINE config after a warm-up,
for ncu launch lists: python tools/ccs_one.py CONFIG [coo] [D]
(CCS_KNOBS="name=value,..." sets spmvtk_k_tune knobs first)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_00019_b200 import spmvtk as sp  # noqa: E402

PARAM = {1: 256, 2: 1 << 20, 3: 128, 4: 1 << 22, 5: 1 << 21}
cfg = int(sys.argv[1])
fmt = sp.Format.COO_COL if len(sys.argv) > 2 and sys.argv[2] == "coo" else sp.Format.CCS
for kv in filter(None, os.environ.get("CCS_KNOBS", "").split(",")):
    k, v = kv.split("=")
    sp.load_library().spmvtk_k_tune(k.encode(), int(v))
dp = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0
m = sp.HostCrs(cfg, PARAM[cfg], dp).upload()
m.convert(fmt).free()  # warm-up (pool, module load)
sp.synchronize()
m.convert(fmt).free()
sp.synchronize()
