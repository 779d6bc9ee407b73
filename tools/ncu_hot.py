#!/usr/bin/env python3
"""Top SASS lines by warp-stall samples from an ncu report's source page:
  python tools/ncu_hot.py gpurun_out/prof_conv_r01.ncu-rep [N]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    lines = txt.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    h = rows[0]
    ia, isrc, iall = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    data = [(float(r[iall] or 0), r[ia], r[isrc]) for r in rows[1:] if len(r) > iall]
    tot = sum(d[0] for d in data) or 1
    for s, a, src in sorted(data, reverse=True)[:n]:
        print(f"{100 * s / tot:5.1f}%  {a}  {src[:110]}")


if __name__ == "__main__":
    main()
