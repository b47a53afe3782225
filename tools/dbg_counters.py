#!/usr/bin/env python
"""Event counters of the tiled DP on C4 samples, from a development build with -DSDEDGE_DBG=1:

    nvcc ... -DSDEDGE_DBG=1 -o /tmp/libsdedge_dbg.so paper_2510_11331_b200/csrc/sdedge.cu
    SDEDGE_LIB=/tmp/libsdedge_dbg.so python tools/dbg_counters.py 68M-7B 1.1B-7B

Prints per-scenario averages of the counters the DBG_ADD sites in sdedge.cu increment.
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import scengen  # noqa: E402
import paper_2510_11331_b200 as sd  # noqa: E402
from tests.parity import gpu_solve  # noqa: E402

NAMES = ["spec_needs_merge", "no_phaseA_winner", "intile_wins", "serial_builds", "pred_segments_at_serial"]


def main(pairs, n=20000):
    f = sd.lib().sdedge_debug_counters
    f.argtypes = [C.c_void_p]
    buf = (C.c_ulonglong * 16)()
    for pair in pairs:
        pd, sc, _ = scengen.config("C4", 0, n, pair=pair)
        gpu_solve(pd, sc, trace=False)
        f(buf)                                   # clear (first call includes warm-up)
        gpu_solve(pd, sc, trace=False)
        f(buf)
        print(pair, {nm: round(buf[i] / n, 2) for i, nm in enumerate(NAMES)})


if __name__ == "__main__":
    main(sys.argv[1:] or ["68M-7B"])
