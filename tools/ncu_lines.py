#!/usr/bin/env python
"""Warp-stall samples and executed instructions per CUDA source line of one ncu report.

    python tools/ncu_lines.py REPORT.ncu-rep [top] [launch index]
"""
import csv
import io
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--launch-skip", skip, "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[h]
iS, iI = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
src = open(os.path.join(ROOT, "paper_2510_11331_b200/csrc/sdedge.cu")).read().splitlines()
agg = []
for r in rows[h + 1:]:
    if r and r[0].isdigit():
        try:
            agg.append((int(r[0]), int(r[iS]), int(r[iI])))
        except ValueError:
            pass
tS, tI = sum(a[1] for a in agg), sum(a[2] for a in agg)
print(f"samples {tS}  warp instructions {tI}")
for ln, s, i in sorted(agg, key=lambda a: -a[1])[:top]:
    print(f"{ln:5d} {100 * s / tS:5.1f}% {100 * i / tI:5.1f}%  {src[ln - 1].strip()[:100]}")
