"""Pins for the CPU oracle (-m "not gpu").

Each test checks the oracle against something other than itself: printed or
independently-derived example values (tests/golden/, cited), closed forms,
invariants, brute force on tiny inputs, or Monte-Carlo.  A plausible mistake
in the oracle (dropped term, wrong index/sign, transposed operand, wrong tie
rule) fails at least one of these.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import scengen

GOLD = os.path.join(os.path.dirname(__file__), "golden")
M68, M11, M7, M13 = (scengen.MODELS[k] for k in ("68M", "1.1B", "7B", "13B"))


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def rel(a, b):
    return abs(a - b) / abs(b)


# ------------------------------------------------------------- eq:ol, eq:step_n
def test_expected_tokens_pins(orc):
    ex = gold("spec_examples.json")
    e = ex["expected_tokens_0.8_7"]
    exact = Fraction(e["num"], e["den"])
    # exact rational value 325089/78125; fp64 evaluation within 2 ulp
    assert abs(orc.expected_tokens(0.8, 7) - float(exact)) <= 2 * math.ulp(float(exact))
    assert float(Fraction(1) - Fraction(4, 5) ** 8) / float(Fraction(1, 5)) == pytest.approx(
        orc.expected_tokens(0.8, 7), rel=1e-15)
    assert orc.expected_tokens(0.5, 1) == 1.5
    assert orc.expected_tokens(0.37, 0) == 1.0  # gamma = 0: only the bonus token (AD)
    rng = np.random.default_rng(1)
    for _ in range(200):
        a = rng.uniform(0.01, 0.99)
        g = int(rng.integers(1, 20))
        L, L0 = orc.expected_tokens(a, g), orc.expected_tokens(a, g - 1)
        assert abs((L - L0) - a ** g) <= 1e-12  # telescoping identity
        assert 1.0 < L <= g + 1 + 1e-12


def test_expected_tokens_monte_carlo(orc):
    """eq:ol is the mean of (accepted prefix length + bonus token) of gamma
    i.i.d. Bernoulli(alpha) acceptances (SPEC acceptance #1)."""
    rng = np.random.default_rng(7)
    for a in (0.5, 0.8):
        for g in (1, 4, 7):
            acc = rng.random((400_000, g)) < a
            prefix = np.where(acc.all(1), g, np.argmin(acc, axis=1))
            mc = (prefix + 1).mean()
            assert rel(mc, orc.expected_tokens(a, g)) < 0.01


def test_decode_steps(orc):
    assert orc.decode_steps(2048, orc.expected_tokens(0.8, 7)) == 493
    assert orc.decode_steps(4, 2.0) == 2
    assert orc.decode_steps(1, 3.7) == 1
    assert orc.decode_steps(2048, 1.0) == 2048  # gamma = 0
    rng = np.random.default_rng(2)
    for _ in range(500):
        a = rng.uniform(0.05, 0.95)
        g = int(rng.integers(0, 17))
        O = int(rng.integers(1, 4096))
        L = orc.expected_tokens(a, g)
        N = orc.decode_steps(O, L)
        assert N * L >= O and (N - 1) * L < O


# ------------------------------------------------------------- memory / FLOPs
def test_memory_pins(orc):
    ex = gold("spec_examples.json")
    assert orc.param_memory(*M68) == ex["param_memory_68M"]["value"] == 2 * (8 * 768**2 + 4 * 768 * 3072)
    assert orc.param_memory(*M11) == ex["param_memory_1.1B"]["value"]
    assert orc.kv_memory_per_task(2, 768, 512, 2048) == ex["kv_per_task_68M_I512_O2048"]["value"]


def test_flops_pins(orc):
    ex = gold("spec_examples.json")
    assert orc.flops_draft(M68, 128, 3.0, 1, 1) == ex["forward_flops_68M_new128_kv0"]["value"]
    assert orc.flops_draft(M68, 128, 3.0, 2, 1) == ex["draft_68M_I128_i2_n1"]["value"]
    e = ex["draft_68M_I128_L4.1611392_i1_n2"]
    assert rel(orc.flops_draft(M68, 128, 4.1611392, 1, 2), e["value"]) < e["rel"]
    assert orc.flops_verify(M7, 128, 4, 3.0, 1) == ex["verify_7B_I128_l4_n1"]["value"]
    e = ex["verify_7B_I128_l4_L3.3616_n2"]
    assert rel(orc.flops_verify(M7, 128, 4, 3.3616, 2), e["value"]) < e["rel"]
    # decode pass i+1 costs exactly one more KV slot than pass i (SPEC cost_model invariant)
    J, h1, _ = M68
    assert orc.flops_draft(M68, 300, 2.5, 3, 5) - orc.flops_draft(M68, 300, 2.5, 2, 5) == 4 * J * h1
    # gamma = 0 verify at n >= 2 is a single-token AD decode with kv = I + n - 2
    J, h1, h2 = M7
    for n in (2, 3, 50):
        kv = 100 + (n - 1) * 1.0 - 1
        assert orc.flops_verify(M7, 100, 0, 1.0, n) == 4.0 * J * h1 * (2 * h1 + kv + 1 + h2)


def test_runtime_pins(orc):
    ex = gold("spec_examples.json")
    e = ex["runtime_4_1.337890701312e12"]
    assert rel(orc.runtime(2.08e-14, 1.28e-2, 1.337890701312e12, 4), e["value"]) < e["rel"]
    e = ex["runtime_1_1e12"]
    assert rel(orc.runtime(2.08e-14, 1.28e-2, 1e12, 1), e["value"]) < e["rel"]
    pd = scengen.params("68M-7B", K=1)
    e = ex["draft_68M_b1_I128_l2_n1"]
    assert rel(orc.draft_time(pd, 1, 128, 2, 3.0, 1), e["value"]) < e["rel"]


def closed_forms(pd, b, I, gamma, L, co=None):
    """stage times summed over passes in closed form
    (a different expression from the oracle's pass-by-pass loop)."""
    Jd, hd, h2d = pd["draft"]
    Jv, hv, h2v = pd["verify"]
    c1d, c2d, c1v, c2v = co if co is not None else (pd["c1_draft"], pd["c2_draft"], pd["c1_verify"], pd["c2_verify"])
    cd, cv = c1d * b * 4 * Jd * hd, c1v * b * 4 * Jv * hv
    g = gamma
    if g == 0:
        Td1, Ad, Bd = 0.0, 0.0, 0.0
    else:
        Td1 = cd * (I * (2 * hd + I + h2d) + (g - 1) * (2 * hd + h2d + I) + g * (g - 1) / 2) + g * c2d
        Ad = cd * (g * (2 * hd + h2d + I) + g * (g - 1) / 2) + g * c2d
        Bd = cd * g * L
    Tv1 = cv * (I + g) * (2 * hv + I + g + h2v) + c2v
    Av = cv * (1 + g) * (2 * hv + h2v + I + g) + c2v
    Bv = cv * (1 + g) * L
    return Td1, Ad, Bd, Tv1, Av, Bv


@pytest.mark.parametrize("pair", ["68M-7B", "1.1B-7B", "1.1B-13B"])
def test_stage_times_vs_closed_form(orc, pair):
    pd = scengen.params(pair, K=1)
    rng = np.random.default_rng(3)
    for _ in range(60):
        g = int(rng.integers(0, 17))
        a = rng.uniform(0.5, 0.9)
        L = orc.expected_tokens(a, g)
        b = int(rng.integers(1, 64))
        I = int(rng.integers(1, 513))
        Td1, Ad, Bd, Tv1, Av, Bv = closed_forms(pd, b, I, g, L)
        for n in (1, 2, 3, 17, 600):
            td = orc.draft_time(pd, b, I, g, L, n)
            tv = orc.verify_time(pd, b, I, g, L, n)
            etd = Td1 if n == 1 else Ad + Bd * (n - 1)
            etv = Tv1 if n == 1 else Av + Bv * (n - 1)
            assert td == pytest.approx(etd, rel=1e-13, abs=1e-300)
            assert tv == pytest.approx(etv, rel=1e-13)


# ------------------------------------------------------------- bandwidth (P1)
def test_bandwidth_spec_example(orc):
    ex = gold("spec_examples.json")["alloc_two_tasks"]
    pd = scengen.params("1.1B-7B", K=2, noise_w=1.0)  # lambda = 16(2048+4096) = 98304
    # log2(1 + p g / sigma^2) = 10 and 5  <=>  p g = 1023 and 31
    t, w = orc.bandwidth(pd, [100, 300], [1.0, 1.0], [1023.0, 31.0])
    assert np.allclose(w, ex["w"], rtol=1e-14)
    assert rel(t, ex["t_com"]) < 1e-14
    # lambda I / (w B s) with w = 1, s = 25
    assert rel(98304 * 512 / (1.0 * 20e6 * 25), 0.100663296) < 1e-14


def test_bandwidth_optimality(orc):
    """Equal finish, sum w = 1, and min-max optimality against random feasible
    allocations and against an independent bisection on t."""
    rng = np.random.default_rng(4)
    pd = scengen.params("68M-7B", K=16)
    lam, B, s2 = 16 * (768 + 4096), pd["bandwidth_hz"], pd["noise_w"]
    for _ in range(30):
        sc = scengen.generate(int(rng.integers(1 << 30)), 16, 0, 1)
        I, p, g = sc["I"][0], sc["p"][0], sc["g"][0]
        t, w = orc.bandwidth(pd, I, p, g)
        s = np.log2(1 + p * g / s2)
        Tk = lam * I / (w * B * s)  # eq:ul_latency_k
        assert abs(w.sum() - 1) < 1e-12
        assert np.all(np.abs(Tk - t) / t < 1e-12)
        for _ in range(50):
            u = rng.random(16)
            u /= u.sum() * rng.uniform(1.0, 1.5)
            assert np.max(lam * I / (u * B * s)) >= t * (1 - 1e-12)
        lo, hi = 0.0, 1e6  # smallest t with sum_k lam I_k / (t B s_k) <= 1
        for _ in range(200):
            mid = 0.5 * (lo + hi)
            if np.sum(lam * I / (mid * B * s)) <= 1:
                hi = mid
            else:
                lo = mid
        assert rel(hi, t) < 1e-12


def test_bandwidth_remark1_and_invariances(orc):
    pd = scengen.params("68M-7B", K=4)
    I = [200, 200, 200, 200]
    t, w = orc.bandwidth(pd, I, [0.2] * 4, [1e-10, 1e-9, 1e-8, 1e-7])
    assert np.all(np.diff(w) < 0)  # Remark 1
    I2 = [17, 300, 5, 511]
    g2 = [3e-9, 1e-8, 2e-10, 7e-9]
    t1, w1 = orc.bandwidth(pd, I2, [0.2] * 4, g2)
    t3, w3 = orc.bandwidth(pd, [3 * x for x in I2], [0.2] * 4, g2)
    assert rel(t3, 3 * t1) < 1e-14 and np.allclose(w1, w3, rtol=1e-14)  # scale invariance
    t4, w4 = orc.bandwidth(dict(pd, bandwidth_hz=40e6), I2, [0.2] * 4, g2)
    assert rel(t4, t1 / 2) < 1e-14 and np.allclose(w1, w4, rtol=1e-14)  # w* independent of B_w


# ------------------------------------------------------------- pipeline recursion
def test_eval_plan_recursion_vs_flowshop_and_des(orc):
    """eq:time against (a) the two-machine flow-shop closed form
    T_n = max_m (sum_{m'<=m} Td_m' + sum_{m'>=m} Tv_m') and (b) an event
    simulation of two unit-capacity stages (SPEC pipeline_sched)."""
    ex = gold("spec_examples.json")["schedule_step"]

    def des(td, tv):
        free_d = free_v = 0.0
        fin = []
        for a, b in zip(td, tv):
            end_d = free_d + a
            free_d = end_d
            start_v = max(end_d, free_v)
            free_v = start_v + b
            fin.append(free_v)
        return fin

    assert des(ex["draft"], ex["verify"]) == ex["C"]
    rng = np.random.default_rng(5)
    pd = scengen.params("1.1B-7B", K=6, O_max=40)
    for _ in range(20):
        Is = np.sort(rng.integers(1, 513, 6)).astype(np.int32)
        cuts = sorted(rng.choice(np.arange(1, 6), size=int(rng.integers(0, 5)), replace=False).tolist())
        ends = cuts + [6]
        g = int(rng.integers(1, 9))
        a = rng.uniform(0.5, 0.9)
        L = orc.expected_tokens(a, g)
        N = orc.decode_steps(40, L)
        tot_fs = tot_des = 0.0
        for n in range(1, N + 1):
            td, tv, st = [], [], 1
            for e in ends:
                td.append(orc.draft_time(pd, e - st + 1, int(Is[e - 1]), g, L, n))
                tv.append(orc.verify_time(pd, e - st + 1, int(Is[e - 1]), g, L, n))
                st = e + 1
            M = len(ends)
            tot_fs += max(sum(td[: m + 1]) + sum(tv[m:]) for m in range(M))
            tot_des += des(td, tv)[-1]
        v = orc.eval_plan(pd, Is, a, g, ends)
        assert rel(v, tot_fs) < 1e-12 and rel(v, tot_des) < 1e-12


# ------------------------------------------------------------- Algorithm 1
def test_dp_k1_closed_form(orc):
    """K = 1: T_inf = [Td1 + Tv1] + (N-1)(Ad + Av) + (Bd + Bv)(N-1)N/2 (P7)."""
    rng = np.random.default_rng(6)
    for pair in ("68M-7B", "1.1B-13B"):
        pd = scengen.params(pair, K=1)
        for _ in range(20):
            I = int(rng.integers(1, 513))
            g = int(rng.integers(0, 17))
            a = rng.uniform(0.5, 0.9)
            L = orc.expected_tokens(a, g)
            N = orc.decode_steps(2048, L)
            Td1, Ad, Bd, Tv1, Av, Bv = closed_forms(pd, 1, I, g, L)
            exp = Td1 + Tv1 + (N - 1) * (Ad + Av) + (Bd + Bv) * (N - 1) * N / 2
            t, S, gap, W = orc.dp(pd, [I], a, g)
            assert rel(t, exp) < 1e-12 and list(S) == [1] and W == N


def _instances(rng, n, K):
    for _ in range(n):
        pair = ["68M-7B", "1.1B-7B", "1.1B-13B"][int(rng.integers(3))]
        scale = [0.25, 1.0, 4.0][int(rng.integers(3))]
        O = int(rng.choice([64, 256, 2048]))
        pd = scengen.params(pair, K=K, O_max=O)
        co = [pd["c1_draft"] * scale, pd["c2_draft"] * scale, pd["c1_verify"], pd["c2_verify"]]
        Is = np.sort(rng.integers(1, 513, K)).astype(np.int32)
        yield pd, co, Is, float(rng.uniform(0.5, 0.9))


def test_dp_vs_brute_force(orc):
    """P8: DP >= BF always; DP == BF for K <= 2, gamma = 0, or the
    verify-dominated regime; DP value == eval_plan of its own plan (P6)."""
    rng = np.random.default_rng(8)
    n_eq = n_gt = n_vd = 0
    for K in (1, 2, 3, 5, 7):
        for pd, co, Is, a in _instances(rng, 12, K):
            for g in (0, 1, 3, 8):
                t, S, gap, W = orc.dp(pd, Is, a, g, coeffs=co)
                plan = orc.backtrack(S)
                assert rel(orc.eval_plan(pd, Is, a, g, plan, coeffs=co), t) < 1e-12
                bf, bg, bplan = orc.brute_force(pd, Is, a, g, g, coeffs=co)
                assert t >= bf * (1 - 1e-12)
                L = orc.expected_tokens(a, g)
                N = orc.decode_steps(pd["O_max"], L)
                # verify-dominated: max draft stage <= min verify stage over all batches, all n
                tdmax = max(orc.draft_time(pd, b, int(Is[i - 1]), g, L, n, co)
                            for i in range(1, K + 1) for b in range(1, i + 1) for n in (1, 2, N))
                tvmin = min(orc.verify_time(pd, b, int(Is[i - 1]), g, L, n, co)
                            for i in range(1, K + 1) for b in range(1, i + 1) for n in (1, 2, N))
                vd = tdmax <= tvmin
                n_vd += vd
                if K <= 2 or g == 0 or vd:
                    assert rel(t, bf) < 1e-12, (K, g, vd)
                if rel(t, bf) < 1e-12:
                    n_eq += 1
                else:
                    n_gt += 1
    assert n_eq > 0 and n_vd > 0


def test_dp_trace_forced_chains(orc):
    """Near-tie branching replay (SURVEY 8(c) "T"): orc_dp_trace with a force
    vector.  Pinned against (i) the free DP (force = its own S gives the same
    chain, row_taken == row_best everywhere), (ii) the literal eq:time
    evaluation of the backtracked plan of ANY forced chain (P6: the taken chain
    is that plan's pipeline state), (iii) brute force: the minimum over forced
    chains whose plan is each contiguous partition equals the exhaustive optimum,
    and row_best <= row_taken at every row."""
    rng = np.random.default_rng(21)
    for K in (1, 3, 5, 6):
        for pd, co, Is, a in _instances(rng, 6, K):
            for g in (1, 4):
                t0, S0, gap0, W0 = orc.dp(pd, Is, a, g, coeffs=co)
                t1, S1, gap1, rb1, rt1, W1 = orc.dp_trace(pd, Is, a, g, force=S0, coeffs=co)
                assert t1 == t0 and list(S1) == list(S0) and W1 == W0
                assert np.array_equal(rb1, rt1) and np.array_equal(gap0, gap1)
                best_forced = np.inf
                for mask in range(1 << (K - 1)):
                    plan = [t + 1 for t in range(K - 1) if mask >> t & 1] + [K]
                    f = np.zeros(K, np.int32)
                    st = 1
                    for e in plan:
                        f[e - 1] = st
                        st = e + 1
                    # rows off the plan take a random memory-feasible j: they do not enter the plan's state
                    for r in range(1, K + 1):
                        if f[r - 1] == 0:
                            j = int(rng.integers(1, r + 1))
                            fits = np.isfinite(orc.eval_plan(dict(pd, K=r - j + 1), Is[j - 1:r], a, g, [r - j + 1],
                                                             coeffs=co))
                            f[r - 1] = j if fits else 0
                    ev = orc.eval_plan(pd, Is, a, g, plan, coeffs=co)
                    t, S, gap, rb, rt, W = orc.dp_trace(pd, Is, a, g, force=f, coeffs=co)
                    assert np.isnan(t) == (not np.isfinite(ev))   # NaN exactly when a forced batch overflows
                    if np.isfinite(ev):
                        assert orc.backtrack(S) == plan
                        assert rel(t, ev) < 1e-12
                        ok = np.isfinite(rt)
                        assert np.all(rb[ok] <= rt[ok])
                        best_forced = min(best_forced, t)
                bf, _, _ = orc.brute_force(pd, Is, a, g, g, coeffs=co)
                if np.isfinite(bf):
                    assert rel(best_forced, bf) < 1e-12


def test_dp_counterexample_regression(orc):
    """Algorithm 1 returns the suboptimal {1}{2}{3}."""
    gd = gold("survey_B1_counterexample.json")
    pd = scengen.params(gd["pair"], K=3, O_max=gd["O_max"], c1_draft=gd["c1_draft"], c2_draft=gd["c2_draft"])
    t, S, gap, W = orc.dp(pd, gd["Is"], gd["alpha"], gd["gamma"])
    assert orc.backtrack(S) == gd["dp_plan"] and rel(t, gd["dp_T_inf"]) < 1e-12
    bf, bg, plan = orc.brute_force(pd, gd["Is"], gd["alpha"], gd["gamma"], gd["gamma"])
    assert list(map(int, plan)) == gd["bf_plan"] and rel(bf, gd["bf_T_inf"]) < 1e-12
    for k, v in gd["other_plans"].items():
        assert rel(orc.eval_plan(pd, gd["Is"], gd["alpha"], gd["gamma"], [int(x) for x in k.split(",")]), v) < 1e-12
    s = gd["second"]
    pd = scengen.params(s["pair"], K=4, O_max=s["O_max"])
    t, S, _, _ = orc.dp(pd, s["Is"], s["alpha"], s["gamma"])
    bf, _, _ = orc.brute_force(pd, s["Is"], s["alpha"], s["gamma"], s["gamma"])
    assert abs((t - bf) / bf - s["dp_over_bf_rel"]) < 5e-6


def test_dp_tie_rule_largest_j(orc):
    """Alg. 1 line 21 ('>=') -> the largest j wins an exact tie.  With every
    coefficient zero all candidates cost exactly 0, so every row ties."""
    pd = scengen.params("68M-7B", K=4, O_max=8, c1_draft=0.0, c1_verify=0.0, c2_draft=0.0,
                        c2_verify=0.0)
    t, S, gap, W = orc.dp(pd, [10, 20, 30, 40], 0.5, 1)
    assert t == 0.0 and list(S) == [1, 2, 3, 4]
    assert list(gap[1:]) == [0.0, 0.0, 0.0] and math.isinf(gap[0])
    # a strict improvement is still taken: cheaper verify intercept favours one batch
    pd = scengen.params("68M-7B", K=4, O_max=8, c1_draft=0.0, c1_verify=0.0, c2_draft=0.0,
                        c2_verify=1.0)
    t, S, gap, W = orc.dp(pd, [10, 20, 30, 40], 0.5, 1)
    assert list(S) == [1, 1, 1, 1] and t == 6.0  # N = ceil(8 / 1.5) steps x c2v


def test_gamma0_is_autoregressive(orc):
    """P9: gamma = 0 reduces to AD on the verify node: independent of the
    draft model, equal to brute force, and equal to the hand composition
    sum_n sum_m (c1v b_m F_AD(n) + c2v) with sequential batches."""
    rng = np.random.default_rng(9)
    for _ in range(10):
        K = int(rng.integers(1, 6))
        Is = np.sort(rng.integers(1, 513, K)).astype(np.int32)
        a = rng.uniform(0.5, 0.9)
        vals = []
        for pair in ("68M-7B", "1.1B-7B"):
            pd = scengen.params(pair, K=K, O_max=48)
            t, S, _, _ = orc.dp(pd, Is, a, 0)
            vals.append(t)
            plan = orc.backtrack(S)
            Jv, hv, h2v = pd["verify"]
            hand, st = 0.0, 1
            for e in plan:
                b, I = e - st + 1, int(Is[e - 1])
                for n in range(1, 49):
                    F = 4 * Jv * hv * I * (2 * hv + I + h2v) if n == 1 else 4 * Jv * hv * (2 * hv + I + n - 2 + 1 + h2v)
                    hand += pd["c1_verify"] * F * b + pd["c2_verify"]
                st = e + 1
            assert rel(t, hand) < 1e-12
            assert rel(t, orc.brute_force(pd, Is, a, 0, 0)[0]) < 1e-12
        assert rel(vals[0], vals[1]) < 1e-15


def test_memory_window(orc):
    """b_max(1.1B, Gamma_s = 16e9, O_max = 2048) = 38 / 34 / 30 at I = 1 / 256 / 512
    (P:336-353 + cons. (b)); plans never contain an over-capacity batch."""
    pd = scengen.params("1.1B-7B", K=45)
    for I, bmax in ((1, 38), (256, 34), (512, 30)):
        Is = np.full(45, I, np.int32)
        assert np.isfinite(orc.eval_plan(pd, Is, 0.8, 1, [bmax, 45]))
        assert np.isinf(orc.eval_plan(pd, Is, 0.8, 1, [bmax + 1, 45]))
        t, S, _, _ = orc.dp(pd, Is, 0.8, 1)
        plan = orc.backtrack(S)
        sizes = np.diff([0] + plan)
        assert sizes.max() <= bmax
    r = orc.solve(dict(pd, mem_capacity_bytes=1_000_000_000), [10] * 45, [0.2] * 45, [1e-8] * 45, 0.8)
    assert r["status"] == 1 and math.isinf(r["T"]) and r["gamma"] == -1 and r["M"] == 0


def test_work_count(orc):
    """O(K^2 N) per gamma: with no memory window, W = sum_g N_g K(K+1)/2."""
    pd = scengen.params("68M-7B", K=9, gamma_min=1, gamma_max=3, O_max=300)
    sc = scengen.generate(11, 9, 0, 1)
    r = orc.solve(pd, sc["I"][0], sc["p"][0], sc["g"][0], float(sc["alpha"][0]))
    a = float(sc["alpha"][0])
    assert r["W"] == sum(orc.decode_steps(300, orc.expected_tokens(a, g)) for g in (1, 2, 3)) * 45


# ------------------------------------------------------------- full solver
def test_golden_B3(orc):
    gd = gold("survey_B3_golden_K4.json")
    for pair, v in gd["pairs"].items():
        pd = scengen.params(pair, K=4, gamma_min=0, gamma_max=4)
        r = orc.solve(pd, gd["I"], [gd["p"]] * 4, gd["g"], gd["alpha"])
        assert r["status"] == 0 and r["gamma"] == v["gamma"]
        assert rel(r["T"], v["T"]) < 1e-12 and rel(r["T_com"], v["T_com"]) < 1e-12
        assert np.allclose(r["tinf_gamma"], v["T_inf"], rtol=1e-12, atol=0)
        assert np.allclose(r["w"], gd["w"], rtol=1e-11)
        if "N" in v:
            assert [orc.decode_steps(2048, orc.expected_tokens(0.8, g)) for g in range(5)] == v["N"]
        if "batch_end" in v:
            assert list(r["batch_end"][: r["M"]]) == v["batch_end"]
        assert list(r["order"]) == [1, 3, 2, 0]


def test_solver_joint_brute_force(orc):
    """Joint (gamma, partition) brute force: T_inf(solver) >= BF, equality when
    every per-gamma DP is exact (SPEC solver example, corrected per P8)."""
    rng = np.random.default_rng(10)
    for pd, co, Is, a in _instances(rng, 15, 5):
        pd = dict(pd, gamma_min=0, gamma_max=4)
        r = orc.solve(pd, Is, [0.2] * 5, [1e-8] * 5, a, coeffs=co)
        bf, bg, plan = orc.brute_force(pd, Is, a, 0, 4, coeffs=co)
        assert r["T_inf"] >= bf * (1 - 1e-12)
        exact = all(rel(orc.dp(pd, Is, a, g, coeffs=co)[0],
                        orc.brute_force(pd, Is, a, g, g, coeffs=co)[0]) < 1e-12 for g in range(5))
        if exact:
            assert rel(r["T_inf"], bf) < 1e-12
        # gamma* is the smallest argmin over gamma (reading A7)
        tg = r["tinf_gamma"]
        assert r["gamma"] == int(np.argmin(tg)) and tg[r["gamma"]] == r["T_inf"]


def test_permutation_and_decoupling(orc):
    """P10/P11: shuffling tasks changes only order and w; T_inf, gamma*, M and
    batch_end are independent of B_w, p, g; T strictly decreases in B_w."""
    rng = np.random.default_rng(12)
    pd = scengen.params("68M-7B", K=12, gamma_min=1, gamma_max=4, O_max=256)
    sc = scengen.generate(12, 12, 0, 1)
    I, p, g, a = sc["I"][0], sc["p"][0], sc["g"][0], float(sc["alpha"][0])
    r0 = orc.solve(pd, I, p, g, a)
    perm = rng.permutation(12)
    r1 = orc.solve(pd, I[perm], p[perm], g[perm], a)
    for k in ("T", "T_inf", "T_com"):
        assert rel(r1[k], r0[k]) < 1e-12
    assert r1["gamma"] == r0["gamma"] and r1["M"] == r0["M"]
    assert np.array_equal(r1["batch_end"], r0["batch_end"])
    assert np.allclose(r1["w"], r0["w"][perm], rtol=1e-13)
    assert np.array_equal(I[perm][r1["order"]], I[r0["order"]])
    r2 = orc.solve(dict(pd, bandwidth_hz=40e6), I, p * 3, g * 0.1, a)
    assert r2["T_inf"] == r0["T_inf"] and r2["gamma"] == r0["gamma"]
    assert np.array_equal(r2["batch_end"], r0["batch_end"])
    Ts = [orc.solve(dict(pd, bandwidth_hz=B), I, p, g, a)["T"] for B in (5e6, 10e6, 20e6, 40e6)]
    assert all(x > y for x, y in zip(Ts, Ts[1:]))


def test_status_codes(orc):
    pd = scengen.params("68M-7B", K=3, gamma_min=1, gamma_max=2, O_max=32)
    r = orc.solve(pd, [1, 2, 3], [0.2] * 3, [1e-8] * 3, 1.0)
    assert r["status"] == 2 and math.isnan(r["T"]) and np.isfinite(r["T_com"]) and r["gamma"] == -1
    r = orc.solve(pd, [1, 0, 3], [0.2] * 3, [1e-8] * 3, 0.5)
    assert r["status"] == 3 and math.isnan(r["T"]) and math.isnan(r["T_com"])
    r = orc.solve(pd, [1, 2, 3], [0.2] * 3, [1e-8, -1.0, 1e-8], 0.5)
    assert r["status"] == 3
    r = orc.solve(pd, [1, 2, 3], [0.2] * 3, [1e-8] * 3, 0.5)
    assert r["status"] == 0 and r["M"] >= 1 and r["batch_end"][r["M"] - 1] == 3


def test_constraints_hold(orc):
    """P13: every output satisfies constraints (a)-(g) of problem P."""
    _, sc, _ = scengen.config("C3", 0, 40)
    pd = scengen.params("1.1B-7B", K=32, gamma_min=1, gamma_max=8)
    out = orc.solve_batch(pd, sc)
    if True:
        for s in range(40):
            assert out["status"][s] == 0
            M = out["M"][s]
            ends = out["batch_end"][s][:M]
            assert 1 <= M <= 32 and ends[-1] == 32 and np.all(np.diff(ends) > 0)
            assert np.all(out["batch_end"][s][M:] == 0)
            Is = sc["I"][s][out["order"][s]]
            st = 0
            for e in ends:
                mem = orc.param_memory(*pd["draft"]) + int(e - st) * orc.kv_memory_per_task(
                    pd["draft"][0], pd["draft"][1], int(Is[e - 1]), 2048)
                assert mem <= 16e9
                st = e
            assert abs(out["w"][s].sum() - 1) < 1e-12 and np.all(out["w"][s] >= 0)
            assert 1 <= out["gamma"][s] <= 8
            assert sorted(out["order"][s]) == list(range(32))
            T, Tc, Ti = out["lat"][s]
            assert T == Tc + Ti
