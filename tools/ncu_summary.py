"""Summarises ncu --set full reports (.ncu-rep) into a markdown table:
duration, DRAM bytes/throughput, L1/L2 throughput, occupancy, registers and
the dominant warp stall reasons.  Usage: ncu_summary.py rep [rep ...]"""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Achieved Occupancy", "Registers Per Thread", "L2 Hit Rate",
        "Compute (SM) Throughput"]


def rows(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True,
                         text=True).stdout
    return list(csv.reader(io.StringIO(out)))


for rep in sys.argv[1:]:
    print(f"### {rep.split('/')[-1]}\n")
    det = rows(rep, "details")
    h = det[0]
    ix = {k: i for i, k in enumerate(h)}
    per = {}
    for r in det[1:]:
        key = (r[ix["ID"]], r[ix["Kernel Name"]].split("(")[0].replace("<unnamed>::", ""))
        if r[ix["Metric Name"]] in WANT:
            per.setdefault(key, {})[r[ix["Metric Name"]]] = f"{r[ix['Metric Value']]} {r[ix['Metric Unit']]}"
    raw = rows(rep, "raw")
    rh = raw[0]
    stalls = {}
    dram = {}
    for r in raw[2:]:
        key = (r[rh.index("ID")], r[rh.index("Kernel Name")].split("(")[0].replace("<unnamed>::", ""))
        items = []
        for i, k in enumerate(rh):
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    items.append((float(r[i]), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in items) or 1
        stalls[key] = ", ".join(f"{n} {v / tot:.0%}" for v, n in sorted(items, reverse=True)[:3])
        try:
            dram[key] = (float(r[rh.index("dram__bytes_read.sum")]) +
                         float(r[rh.index("dram__bytes_write.sum")]))
            unit = raw[1][rh.index("dram__bytes_read.sum")]
            dram[key] = f"{dram[key]:.1f} {unit}"
        except (ValueError, IndexError):
            dram[key] = "?"
    print("| ID | kernel | " + " | ".join(WANT) + " | DRAM read+write | top stalls |")
    print("|---" * (len(WANT) + 4) + "|")
    for key, d in per.items():
        print(f"| {key[0]} | {key[1]} | " + " | ".join(d.get(w, "") for w in WANT) +
              f" | {dram.get(key, '')} | {stalls.get(key, '')} |")
    print()
