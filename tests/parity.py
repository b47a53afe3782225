"""Shared parity helpers for the GPU tests, smoke() and bench.py.

Compares the CUDA path's outputs with the oracle's on the same seeded inputs,
with the tolerances of BASELINE.json's north_star (SURVEY.md 8(c) "T"):
  fp64: T, T_com, T_inf within 1e-12 relative; gamma*, M, batch_end, order
        bit-identical; w within 1e-12 -- unless the oracle's best-vs-second
        gap (any row of any gamma, or between gammas) is < 1e-9, in which case
        the scenario is "exempt" and must instead be self-consistent: the
        oracle's literal eq:time evaluation of the GPU's own plan equals the
        GPU's T_inf within 1e-12.
  fp32: 1e-5 relative; schedule identity only where the gap >= 1e-5.
"""
from __future__ import annotations

import numpy as np

TOL = {0: dict(rel=1e-12, gap=1e-9), 1: dict(rel=1e-5, gap=1e-5)}


def to_numpy(out: dict) -> dict:
    r = {}
    for k, v in out.items():
        if v is None:
            r[k] = None
        elif hasattr(v, "cpu"):
            r[k] = v.cpu().numpy()
        else:
            r[k] = np.asarray(v)
    return r


def compare(pd: dict, sc: dict, gpu: dict, orc: dict, precision: int = 0, orc_mod=None,
            idx=None) -> dict:
    """Element-by-element comparison; returns counts and raises AssertionError
    listing the first failures."""
    tol = TOL[precision]
    n = len(orc["status"])
    idx = np.arange(n) if idx is None else np.asarray(idx)
    fails, exempt, exact = [], 0, 0
    worst = 0.0
    for a, s in enumerate(idx):
        st_o, st_g = int(orc["status"][a]), int(gpu["status"][s])
        if st_o != st_g:
            fails.append(f"s={s}: status gpu {st_g} != oracle {st_o}")
            continue
        if not np.array_equal(gpu["order"][s], orc["order"][a]):
            fails.append(f"s={s}: order differs")
        if st_o != 0:
            if gpu["gamma"][s] != -1 or gpu["M"][s] != 0 or np.any(gpu["batch_end"][s] != 0):
                fails.append(f"s={s}: failed scenario outputs not cleared")
            lo, lg = orc["lat"][a], gpu["lat"][s]
            for q in range(3):
                if not (np.isnan(lo[q]) and np.isnan(lg[q])) and not (lo[q] == lg[q]) and not (
                        np.isfinite(lo[q]) and abs(lg[q] - lo[q]) <= tol["rel"] * abs(lo[q])):
                    fails.append(f"s={s}: status {st_o} latency[{q}] gpu {lg[q]} oracle {lo[q]}")
            continue
        lo, lg = orc["lat"][a], gpu["lat"][s]
        r = np.abs(lg - lo) / np.abs(lo)
        gap = min(orc["min_row_gap"][a], orc["gamma_gap"][a])
        same_sched = (gpu["gamma"][s] == orc["gamma"][a] and gpu["M"][s] == orc["M"][a]
                      and np.array_equal(gpu["batch_end"][s], orc["batch_end"][a]))
        if gap < tol["gap"]:
            exempt += 1
            if orc_mod is not None and precision == 0:
                K = pd["K"]
                Is = sc["I"][s][gpu["order"][s]]
                co = None if sc.get("coeffs") is None else sc["coeffs"][s]
                ends = list(gpu["batch_end"][s][: gpu["M"][s]])
                ev = orc_mod.eval_plan_nopipe if pd.get("batching_policy", 0) == 1 else orc_mod.eval_plan
                v = ev(dict(pd, K=K), Is, float(sc["alpha"][s]), int(gpu["gamma"][s]), ends, coeffs=co)
                if abs(v - lg[2]) > 1e-12 * abs(v) or lg[2] > lo[2] * (1 + 1e-6):
                    fails.append(f"s={s}: exempt scenario not self-consistent ({v} vs {lg[2]})")
            continue
        worst = max(worst, float(r.max()))
        if r.max() > tol["rel"]:
            fails.append(f"s={s}: latency rel err {r.max():.3e} (gpu {lg}, oracle {lo})")
        if not same_sched:
            fails.append(f"s={s}: schedule differs: gpu gamma {gpu['gamma'][s]} M {gpu['M'][s]} "
                         f"vs oracle gamma {orc['gamma'][a]} M {orc['M'][a]} (gap {gap:.2e})")
        if gpu.get("w") is not None and orc.get("w") is not None:
            rw = np.abs(gpu["w"][s] - orc["w"][a]) / np.abs(orc["w"][a])
            if rw.max() > max(tol["rel"], 1e-12):
                fails.append(f"s={s}: w rel err {rw.max():.3e}")
        exact += 1
    res = dict(n=len(idx), exact=exact, exempt=exempt, failures=len(fails), worst_rel=worst)
    if fails:
        raise AssertionError(f"{len(fails)} parity failures, e.g.:\n  " + "\n  ".join(fails[:12]) +
                             f"\n{res}")
    return res


def gpu_solve(pd: dict, sc: dict, device="cuda:0", precision=0, algo=0, idx=None):
    """Run the CUDA path on a scengen dict; returns numpy outputs."""
    import torch
    import paper_2510_11331_b200 as sd
    sel = (lambda a: a) if idx is None else (lambda a: a[idx])
    I = torch.from_numpy(np.ascontiguousarray(sel(sc["I"]))).to(device)
    p = torch.from_numpy(np.ascontiguousarray(sel(sc["p"]))).to(device)
    g = torch.from_numpy(np.ascontiguousarray(sel(sc["g"]))).to(device)
    al = torch.from_numpy(np.ascontiguousarray(sel(sc["alpha"]))).to(device)
    co = None if sc.get("coeffs") is None else torch.from_numpy(np.ascontiguousarray(sel(sc["coeffs"]))).to(device)
    out = sd.solve(pd, I, p, g, al, co, precision=precision, algo=algo)
    torch.cuda.synchronize()
    return to_numpy(out)
