#!/usr/bin/env python
"""Write the oracle's results on the large-config parity samples to
tests/data/oracle_<name>.npz (test infrastructure).

Calls ONLY oracle/ (the plain C solver) and scengen/ (the seeded inputs): no
value in these files comes from the CUDA path.  The GPU parity tests
(tests/test_gpu_parity.py) solve the full launches on the device and compare
the sampled scenarios with these stored oracle results, so the round-end GPU
box does not spend ~10 core-hours re-running the oracle.  Each file carries a
SHA-256 of the sampled inputs; tests/test_fixtures.py (-m "not gpu") checks
that fingerprint against scengen and re-solves a few stored scenarios with the
oracle, so a stale file fails loudly.

    python tools/make_oracle_fixtures.py [name ...]   (default: all)
"""
from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import scengen  # noqa: E402

OUT = os.path.join(ROOT, "tests", "data")

# name -> (config, pair, scenario indices): SURVEY 8(d) "Oracle timing beside the GPU"
# (C4: s = 0 mod 500, 2000 scenarios) and VERDICT r01 (C5 at the full gamma range).
FIXTURES = {
    "c4_68M-7B": ("C4", "68M-7B", np.arange(0, 1_000_000, 500)),
    "c4_1.1B-7B": ("C4", "1.1B-7B", np.arange(0, 1_000_000, 2000)),
    "c5_256": ("C5256", "68M-7B", np.array([0, 1, 2])),
    "c5_512": ("C5512", "68M-7B", np.array([0, 1])),
    "c5_1024": ("C51024", "68M-7B", np.array([0, 1])),
}


def sample(cfg, pair, idx):
    """The sampled scenarios of a config (scengen only)."""
    pd, _, _ = scengen.config(cfg, 0, 1, pair=pair)
    parts = [scengen.config(cfg, int(s), int(s) + 1, pair=pair)[1] for s in idx]
    sc = {k: (np.concatenate([q[k] for q in parts]) if parts[0][k] is not None else None) for k in parts[0]}
    return pd, sc


def fingerprint(sc) -> str:
    h = hashlib.sha256()
    for k in ("I", "p", "g", "alpha"):
        h.update(np.ascontiguousarray(sc[k]).tobytes())
    return h.hexdigest()


def make(name):
    cfg, pair, idx = FIXTURES[name]
    pd, sc = sample(cfg, pair, idx)
    t0 = time.time()
    r = oracle.solve_batch(pd, sc, nthreads=os.cpu_count())
    dt = time.time() - t0
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, f"oracle_{name}.npz"), idx=idx, sha=np.array(fingerprint(sc)),
                        config=np.array(cfg), pair=np.array(pair),
                        **{k: v for k, v in r.items() if k != "nthreads"})
    print(f"{name}: {len(idx)} scenarios in {dt:.0f} s on {r['nthreads']} threads; "
          f"exempt(1e-9) {int(np.sum(np.minimum(r['min_row_gap'], r['gamma_gap']) < 1e-9))}, "
          f"min gap {np.min(r['min_row_gap']):.3e}", flush=True)


if __name__ == "__main__":
    oracle.build()
    for nm in (sys.argv[1:] or list(FIXTURES)):
        make(nm)
