"""Warp-stall samples per CUDA source line of one kernel in an ncu report
(needs -lineinfo builds and --import-source on).

    python tools/ncu_lines.py report.ncu-rep <kernel-regex> [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass", "-k", f"regex:{kern}"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(r for r in rows if r and r[0] == "Line No")
    i_samp = hdr.index("Warp Stall Sampling (All Samples)")
    i_inst = hdr.index("Instructions Executed")
    per, src, tot = {}, {}, 0
    for r in rows:
        if len(r) <= i_samp or not r[0].isdigit() or r[2] != "-":
            continue
        ln = int(r[0])
        s = int(r[i_samp] or 0)
        per[ln] = per.get(ln, 0) + s
        src[ln] = (r[1].strip(), int(r[i_inst] or 0))
        tot += s
    print(f"total samples {tot}")
    for ln, s in sorted(per.items(), key=lambda x: -x[1])[:top]:
        print(f"{ln:5d} {100 * s / max(tot, 1):5.1f}%  inst={src[ln][1]:>10}  {src[ln][0][:90]}")


if __name__ == "__main__":
    main()
