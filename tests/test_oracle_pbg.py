"""Pins for the per-batch speculation-length extension of the oracle
(not in the paper: one global l, P:555, P:757-767;
SPEC.md:540) -- -m "not gpu".

orc_eval_plan_pbg is pinned against the two-machine flow-shop closed form over
each step's ACTIVE batches (eq:time + eq:latency_infer_batch) and
reduces to orc_eval_plan when every batch has the same gamma; orc_dp_pbg
reduces to Algorithm 1 (orc_dp) when gamma_min = gamma_max, is exact at K = 1,
never beats the brute force over (partition x per-batch gamma), returns the
eq:time value of its own plan, and breaks exact ties to the largest j, then the
smallest gamma (reading NB1)."""
import itertools

import numpy as np

import scengen
from tests.test_oracle_pins import _instances, rel


def _flowshop(orc, pd, Is, a, ends, gammas, co=None):
    """T_inf = sum_n max over active m of (sum_{m' <= m} T^d + sum_{m' >= m} T^v) (the
    makespan of a two-machine flow shop in the given order), active = n_m >= n."""
    Ls = [orc.expected_tokens(a, g) for g in gammas]
    ns = [orc.decode_steps(pd["O_max"], L) for L in Ls]
    tot = 0.0
    for n in range(1, max(ns) + 1):
        act, st = [], 1
        for m, e in enumerate(ends):
            b, I = e - st + 1, int(Is[e - 1])
            if ns[m] >= n:
                act.append((orc.draft_time(pd, b, I, gammas[m], Ls[m], n, co),
                            orc.verify_time(pd, b, I, gammas[m], Ls[m], n, co)))
            st = e + 1
        tot += max(sum(d for d, _ in act[:m + 1]) + sum(v for _, v in act[m:]) for m in range(len(act)))
    return tot


def test_eval_plan_pbg_flowshop_and_reduction(orc):
    rng = np.random.default_rng(31)
    for K in (1, 3, 6):
        for pd, co, Is, a in _instances(rng, 6, K):
            for _ in range(3):
                cuts = sorted(rng.choice(np.arange(1, K), size=int(rng.integers(0, K)), replace=False)) if K > 1 else []
                ends = [int(c) for c in cuts] + [K]
                gms = [int(x) for x in rng.integers(0, 9, len(ends))]
                v = orc.eval_plan_pbg(pd, Is, a, ends, gms, coeffs=co)
                if not np.isfinite(v):
                    continue
                assert rel(v, _flowshop(orc, pd, Is, a, ends, gms, co)) < 1e-12
                g = gms[0]
                assert orc.eval_plan_pbg(pd, Is, a, ends, [g] * len(ends), coeffs=co) == \
                    orc.eval_plan(pd, Is, a, g, ends, coeffs=co)


def test_dp_pbg_single_gamma_is_algorithm1(orc):
    rng = np.random.default_rng(32)
    for K in (1, 4, 9):
        for pd, co, Is, a in _instances(rng, 5, K):
            for g in (0, 2, 7):
                p1 = dict(pd, gamma_min=g, gamma_max=g)
                t, S, Gm, gap, W = orc.dp_pbg(p1, Is, a, coeffs=co)
                t0, S0, gap0, W0 = orc.dp(p1, Is, a, g, coeffs=co)
                assert list(S) == list(S0) and W == W0
                if np.isfinite(t0):
                    assert rel(t, t0) < 1e-12 and np.all(Gm == g)
                else:
                    assert np.isinf(t)


def test_dp_pbg_vs_brute_force(orc):
    rng = np.random.default_rng(33)
    n_eq = n_tot = 0
    for K in (1, 2, 3, 4):
        for pd, co, Is, a in _instances(rng, 6, K):
            pd = dict(pd, gamma_min=1, gamma_max=3)
            t, S, Gm, gap, W = orc.dp_pbg(pd, Is, a, coeffs=co)
            plan = orc.backtrack(S)
            gms = [int(Gm[e - 1]) for e in plan]
            if np.isfinite(t):
                assert rel(orc.eval_plan_pbg(pd, Is, a, plan, gms, coeffs=co), t) < 1e-12   # self-consistent
            bf = np.inf
            for mask in range(1 << (K - 1)):
                ends = [q + 1 for q in range(K - 1) if mask >> q & 1] + [K]
                for gg in itertools.product((1, 2, 3), repeat=len(ends)):
                    bf = min(bf, orc.eval_plan_pbg(pd, Is, a, ends, list(gg), coeffs=co))
            if np.isinf(bf):
                assert np.isinf(t)
                continue
            assert t >= bf * (1 - 1e-12)
            if K == 1:
                assert rel(t, bf) < 1e-12
            n_tot += 1
            n_eq += rel(t, bf) < 1e-12
    assert n_eq > 0 and n_tot > 0


def test_dp_pbg_tie_rule(orc):
    pd = scengen.params("68M-7B", K=4, O_max=8, gamma_min=1, gamma_max=3, c1_draft=0.0, c1_verify=0.0,
                        c2_draft=0.0, c2_verify=0.0)
    t, S, Gm, gap, W = orc.dp_pbg(pd, [10, 20, 30, 40], 0.5)
    assert t == 0.0 and list(S) == [1, 2, 3, 4] and list(Gm) == [1, 1, 1, 1]


def test_solve_per_batch_policy(orc):
    pd = dict(scengen.params("1.1B-7B", K=6, gamma_min=1, gamma_max=4, O_max=256), batching_policy=6)
    sc = scengen.generate(61, 6, 0, 4)
    for s in range(4):
        r = orc.solve(pd, sc["I"][s], sc["p"][s], sc["g"][s], float(sc["alpha"][s]))
        Is = np.sort(sc["I"][s])
        ends = [int(x) for x in r["batch_end"][: r["M"]]]
        gms = [int(x) for x in r["batch_gamma"][: r["M"]]]
        assert r["status"] == 0 and r["gamma"] == gms[-1] and np.all(r["batch_gamma"][r["M"]:] == 0)
        assert rel(orc.eval_plan_pbg(pd, Is, float(sc["alpha"][s]), ends, gms), r["T_inf"]) < 1e-12
        assert r["T"] == r["T_com"] + r["T_inf"]
