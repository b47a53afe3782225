"""Shared parity helpers for the GPU tests, smoke() and bench.py.

Compares the CUDA path's outputs with the oracle's on the same seeded inputs,
with the tolerances of BASELINE.json's north_star made concrete in SURVEY.md
8(c) "T":
  * every status-0 scenario: T_com within `rel` of the oracle's (it does not
    depend on the DP);
  * gamma*, M and batch_end identical to the oracle's -> T and T_inf within
    `rel` (and w within max(rel, 1e-12));
  * a different schedule is allowed only where the oracle's best-vs-second gap
    (any row of any gamma, or between gammas) is below `gap`, and then only if
    the near-tie branching replay reproduces it: the oracle re-runs Algorithm 1
    at the GPU's gamma with every row forced to the GPU's own choice (its
    exported S vector, `trace`), and at every row the forced candidate must be
    within `gap` of that row's best candidate (a branch Algorithm 1 can take at
    a near tie), the forced chain's T_inf must equal the GPU's
    within `rel`, and it must be within `gap` of the oracle's best T_inf over
    gamma.
Tolerances: fp64 rel 1e-12, gap 1e-9; fp32 rel 1e-5, gap 1e-5.
Counts (exact / exempt-but-identical / replayed) are returned and collected
for the session summary (tests/conftest.py).
"""
from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor
import os

import numpy as np

TOL = {0: dict(rel=1e-12, gap=1e-9), 1: dict(rel=1e-5, gap=1e-5)}
STATS: list = []          # (label, result dict) of every compare() in this session
HERE = os.path.dirname(os.path.abspath(__file__))


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


def replay(orc_mod, pd, Is, alpha, gamma_g, trace, T_inf_g, T_inf_best, tol, coeffs=None):
    """Near-tie branching replay of one GPU schedule (see module doc).
    Returns None if it reproduces, else the reason."""
    t, S, gap, rb, rt, _ = orc_mod.dp_trace(pd, Is, alpha, int(gamma_g), force=trace, coeffs=coeffs)
    if not np.isfinite(t):
        return f"forced chain infeasible ({t})"
    dev = np.where(rb > 0, (rt - rb) / np.where(rb > 0, rb, 1.0), np.where(rt == rb, 0.0, np.inf))
    bad = np.nonzero(dev > tol["gap"])[0]
    if len(bad):
        r = int(bad[0])
        return f"row {r + 1}: GPU took j={trace[r]} at {dev[r]:.3e} above the best (gap threshold {tol['gap']})"
    if abs(t - T_inf_g) > tol["rel"] * abs(t):
        return f"forced-chain T_inf {t!r} vs GPU {T_inf_g!r}"
    if t > T_inf_best * (1 + tol["gap"]):
        return f"gamma {gamma_g}: T_inf {t!r} not within the gap of the best {T_inf_best!r}"
    return None


def compare(pd: dict, sc: dict, gpu: dict, orc: dict, precision: int = 0, orc_mod=None,
            idx=None, label: str = "") -> dict:
    """Element-by-element comparison of the sampled scenarios `idx` (GPU
    indices; orc holds the oracle's results for exactly those, in order).
    Returns counts; raises AssertionError listing the first failures."""
    tol = TOL[precision]
    n = len(orc["status"])
    idx = np.arange(n) if idx is None else np.asarray(idx)
    pol = pd.get("batching_policy", 0)
    fails, exact, exempt_same, replayed, worst = [], 0, 0, 0, 0.0
    todo = []
    for a, s in enumerate(idx):
        st_o, st_g = int(orc["status"][a]), int(gpu["status"][s])
        if st_o != st_g:
            fails.append(f"s={s}: status gpu {st_g} != oracle {st_o}")
            continue
        if not np.array_equal(gpu["order"][s], orc["order"][a]):
            fails.append(f"s={s}: order differs")
        lo, lg = orc["lat"][a], gpu["lat"][s]
        if st_o != 0:
            if gpu["gamma"][s] != -1 or gpu["M"][s] != 0 or np.any(gpu["batch_end"][s] != 0):
                fails.append(f"s={s}: failed scenario outputs not cleared")
            for q in range(3):
                if not (np.isnan(lo[q]) and np.isnan(lg[q])) and not (lo[q] == lg[q]) and not (
                        np.isfinite(lo[q]) and abs(lg[q] - lo[q]) <= tol["rel"] * abs(lo[q])):
                    fails.append(f"s={s}: status {st_o} latency[{q}] gpu {lg[q]} oracle {lo[q]}")
            continue
        if abs(lg[1] - lo[1]) > tol["rel"] * abs(lo[1]):
            fails.append(f"s={s}: T_com gpu {lg[1]!r} oracle {lo[1]!r}")
        if gpu.get("w") is not None and orc.get("w") is not None:
            rw = np.abs(gpu["w"][s] - orc["w"][a]) / np.abs(orc["w"][a])
            if rw.max() > max(tol["rel"], 1e-12):
                fails.append(f"s={s}: w rel err {rw.max():.3e}")
        gap = min(orc["min_row_gap"][a], orc["gamma_gap"][a])
        same = (gpu["gamma"][s] == orc["gamma"][a] and gpu["M"][s] == orc["M"][a]
                and np.array_equal(gpu["batch_end"][s], orc["batch_end"][a]))
        if pol == 6:                      # per-batch gamma: every batch's gamma is part of the schedule
            same = same and np.array_equal(gpu["batch_gamma"][s], orc["batch_gamma"][a])
        if same:
            with np.errstate(divide="ignore", invalid="ignore"):
                r = np.where(lg == lo, 0.0, np.abs(lg - lo) / np.abs(lo))
            worst = max(worst, float(r.max()))
            if r.max() > tol["rel"]:
                fails.append(f"s={s}: latency rel err {r.max():.3e} (gpu {lg}, oracle {lo})")
            if gap < tol["gap"]:
                exempt_same += 1
            else:
                exact += 1
            continue
        if gap >= tol["gap"]:
            fails.append(f"s={s}: schedule differs: gpu gamma {gpu['gamma'][s]} M {gpu['M'][s]} "
                         f"vs oracle gamma {orc['gamma'][a]} M {orc['M'][a]} (gap {gap:.2e})")
            continue
        if orc_mod is None:
            fails.append(f"s={s}: schedule differs at a near tie (gap {gap:.2e}) and no oracle to replay")
            continue
        K = pd["K"]
        Is = sc["I"][s][gpu["order"][s]]
        co = None if sc.get("coeffs") is None else sc["coeffs"][s]
        ends = [int(x) for x in gpu["batch_end"][s][: gpu["M"][s]]]
        if pol == 0:
            tr = gpu.get("trace")
            if tr is None:
                fails.append(f"s={s}: schedule differs at a near tie (gap {gap:.2e}); no GPU trace to replay")
                continue
            if orc_mod.backtrack(tr[s]) != ends:
                fails.append(f"s={s}: GPU trace does not backtrack to its batch_end")
                continue
            todo.append((s, dict(pd, K=K), Is, float(sc["alpha"][s]), int(gpu["gamma"][s]),
                         np.array(tr[s]), float(lg[2]), float(lo[2]), co))
        elif pol == 1:
            # SD w/o pipeline: the additive DP is exact, so a differing plan must cost the same
            v = orc_mod.eval_plan_nopipe(dict(pd, K=K), Is, float(sc["alpha"][s]), int(gpu["gamma"][s]), ends,
                                         coeffs=co)
            if abs(v - lg[2]) > tol["rel"] * abs(v) or abs(lg[2] - lo[2]) > tol["gap"] * lo[2]:
                fails.append(f"s={s}: no-pipeline near tie not reproduced ({v} vs {lg[2]} vs {lo[2]})")
            else:
                replayed += 1
        else:
            fails.append(f"s={s}: fixed-plan policy {pol} schedule differs")
    if todo:
        with ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as ex:
            res = list(ex.map(lambda t: replay(orc_mod, *t[1:8], tol, coeffs=t[8]), todo))
        for t, why in zip(todo, res):
            if why is None:
                replayed += 1
            else:
                fails.append(f"s={t[0]}: near-tie replay failed: {why}")
    res = dict(n=len(idx), exact=exact, exempt_same=exempt_same, replayed=replayed, failures=len(fails),
               worst_rel=worst, precision=precision)
    STATS.append((label or f"K={pd['K']} prec={precision} pol={pol}", res))
    if fails:
        raise AssertionError(f"{len(fails)} parity failures, e.g.:\n  " + "\n  ".join(fails[:12]) +
                             f"\n{res}")
    return res


def gpu_solve(pd: dict, sc: dict, device="cuda:0", precision=0, algo=0, idx=None, trace=True):
    """Run the CUDA path on a scengen dict; returns numpy outputs (with the
    row-choice trace of gamma* unless trace=False)."""
    import torch
    import paper_2510_11331_b200 as sd
    sel = (lambda a: a) if idx is None else (lambda a: a[idx])
    I = torch.from_numpy(np.ascontiguousarray(sel(sc["I"]))).to(device)
    p = torch.from_numpy(np.ascontiguousarray(sel(sc["p"]))).to(device)
    g = torch.from_numpy(np.ascontiguousarray(sel(sc["g"]))).to(device)
    al = torch.from_numpy(np.ascontiguousarray(sel(sc["alpha"]))).to(device)
    co = None if sc.get("coeffs") is None else torch.from_numpy(np.ascontiguousarray(sel(sc["coeffs"]))).to(device)
    out = sd.solve(pd, I, p, g, al, co, precision=precision, algo=algo, trace=trace)
    torch.cuda.synchronize()
    return to_numpy(out)


def load_fixture(name: str, check_inputs: bool = True):
    """Stored oracle results of a large-config sample (tools/make_oracle_fixtures.py,
    which calls only oracle/).  Returns (params, sampled scenarios, idx, oracle
    results); the inputs are regenerated by scengen and their fingerprint checked."""
    import hashlib
    import scengen
    z = np.load(os.path.join(HERE, "data", f"oracle_{name}.npz"))
    idx = z["idx"]
    cfg, pair = str(z["config"]), str(z["pair"])
    pd, _, _ = scengen.config(cfg, 0, 1, pair=pair)
    parts = [scengen.config(cfg, int(s), int(s) + 1, pair=pair)[1] for s in idx]
    sc = {k: (np.concatenate([q[k] for q in parts]) if parts[0][k] is not None else None) for k in parts[0]}
    if check_inputs:
        h = hashlib.sha256()
        for k in ("I", "p", "g", "alpha"):
            h.update(np.ascontiguousarray(sc[k]).tobytes())
        assert h.hexdigest() == str(z["sha"]), f"fixture {name} is stale: scengen inputs changed"
    orc = {k: z[k] for k in ("status", "gamma", "M", "lat", "order", "batch_end", "w", "min_row_gap",
                             "gamma_gap", "W")}
    return pd, sc, idx, orc
