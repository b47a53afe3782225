#!/usr/bin/env python
"""Run the same seeded scenarios through the library in $SDEDGE_LIB (or the
default build) and dump the outputs, so two builds can be compared bit for bit
(e.g. the exact-pruning build against SDEDGE_PRUNE=0).

    python tools/compare_libs.py dump OUT.npz [config ...]
    python tools/compare_libs.py diff A.npz B.npz
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def dump(path, cfgs):
    import scengen
    from tests.parity import gpu_solve
    res = {}
    for cfg in cfgs:
        name, n, pair = cfg.split(":")
        pd, sc, _ = scengen.config(name, 0, int(n), pair=pair or None)
        for prec in (0, 1):
            out = gpu_solve(pd, sc, precision=prec)
            for k, v in out.items():
                if v is not None:
                    res[f"{cfg}/{prec}/{k}"] = v
    np.savez(path, **res)


def diff(a, b):
    A, B = np.load(a), np.load(b)
    bad = [k for k in A.files if not np.array_equal(A[k], B[k], equal_nan=True)]
    print(f"{len(A.files)} arrays compared, {len(bad)} differ", bad[:10])
    return 1 if bad else 0


if __name__ == "__main__":
    if sys.argv[1] == "dump":
        dump(sys.argv[2], sys.argv[3:] or ["C4:20000:68M-7B", "C4:20000:1.1B-7B", "C3:50000:", "C5256:500:",
                                           "C2:3:"])
    else:
        sys.exit(diff(sys.argv[2], sys.argv[3]))
