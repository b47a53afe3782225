#!/usr/bin/env python
"""Registers / spills per kernel instantiation from `nvcc -Xptxas -v` (checked before spending GPU time).

    python tools/ptxas_report.py [-D NAME=VALUE ...]
"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_11331_b200 import _build as b  # noqa: E402

defs = [a for a in sys.argv[1:]]
cmd = [b.nvcc(), *b.NVCC_FLAGS, "-Xptxas", "-v", *defs, "-I", os.path.join(ROOT, "include"), "-o", "/tmp/_ptxas.so",
       b.SRC]
err = subprocess.run(cmd, capture_output=True, text=True).stderr
cur = None
for line in err.splitlines():
    m = re.search(r"Compiling entry function '(\w+)'", line)
    if m:
        name = re.search(r"\d+([a-z_]+_kernel)", m.group(1)).group(1)
        targs = re.search(r"_kernelI(\w*?)EEv", m.group(1))
        args = re.findall(r"^([df])|Li(\d+)E", targs.group(1)) if targs else []
        cur = name + "<" + ",".join(a or b for a, b in args) + ">"
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        sp = f"spill st {m.group(1)} ld {m.group(2)}"
    m2 = re.search(r"Used (\d+) registers", line)
    if m2 and cur:
        print(f"{cur:40s} regs {m2.group(1):>4s}  {sp}")
        cur = None
