"""Pins for the oracle's paper-baseline policies (Sec. IV, P:818-826, P:903-911,
P:936-940), -m "not gpu".  SURVEY.md 8(f) NEXT-2."""
import math

import numpy as np
import pytest

import scengen

BW_UNIFORM = 1
NO_PIPE, NONE, STATIC, MAX, HEUR = 1, 2, 3, 4, 5


def rel(a, b):
    return abs(a - b) / abs(b)


def test_uniform_bandwidth_spec_example(orc):
    """uniform shares on the two-task example give max(lam 100 2 /(B 10),
    lam 300 2 /(B 5)) = lam 120 / B, strictly above t* = lam 70 / B."""
    pd = scengen.params("1.1B-7B", K=2, noise_w=1.0)
    lam, B = 98304, 20e6
    t_opt, _ = orc.bandwidth(pd, [100, 300], [1.0, 1.0], [1023.0, 31.0])
    t_uni, w = orc.bandwidth(dict(pd, bandwidth_policy=BW_UNIFORM), [100, 300], [1.0, 1.0], [1023.0, 31.0])
    assert rel(t_uni, lam * 120 / B) < 1e-14 and t_uni > t_opt
    assert list(w) == [0.5, 0.5]


def test_uniform_never_better_and_equal_when_symmetric(orc):
    rng = np.random.default_rng(31)
    pd = scengen.params("68M-7B", K=12)
    for _ in range(40):
        sc = scengen.generate(int(rng.integers(1 << 30)), 12, 0, 1)
        t_opt, _ = orc.bandwidth(pd, sc["I"][0], sc["p"][0], sc["g"][0])
        t_uni, _ = orc.bandwidth(dict(pd, bandwidth_policy=BW_UNIFORM), sc["I"][0], sc["p"][0], sc["g"][0])
        assert t_uni >= t_opt * (1 - 1e-12)
    # identical tasks: both schemes coincide (w* = 1/K)
    t_opt, _ = orc.bandwidth(pd, [100] * 12, [0.2] * 12, [1e-8] * 12)
    t_uni, _ = orc.bandwidth(dict(pd, bandwidth_policy=BW_UNIFORM), [100] * 12, [0.2] * 12, [1e-8] * 12)
    assert rel(t_uni, t_opt) < 1e-12


def test_nopipe_dp_is_exact(orc):
    """The SD-w/o-pipeline cost is additive over batches, so Algorithm 1's
    recursion is exact for it: equals brute force over contiguous partitions."""
    rng = np.random.default_rng(32)
    for K in (1, 2, 4, 6):
        for _ in range(6):
            pair = ["68M-7B", "1.1B-7B", "1.1B-13B"][int(rng.integers(3))]
            pd = scengen.params(pair, K=K, O_max=int(rng.choice([32, 300])))
            Is = np.sort(rng.integers(1, 513, K)).astype(np.int32)
            a = float(rng.uniform(0.5, 0.9))
            for g in (0, 2, 7):
                t, S, gap, W = orc.dp_nopipe(pd, Is, a, g)
                plan = orc.backtrack(S)
                assert rel(orc.eval_plan_nopipe(pd, Is, a, g, plan), t) < 1e-12
                best = math.inf
                for mask in range(1 << (K - 1)):
                    ends = [t_ + 1 for t_ in range(K - 1) if mask >> t_ & 1] + [K]
                    best = min(best, orc.eval_plan_nopipe(pd, Is, a, g, ends))
                assert rel(t, best) < 1e-12


def test_pipelining_dominance(orc):
    """For every plan, each step's pipelined makespan <= the sequential sum
    (P:505-517 vs P:820), with equality for a single batch."""
    rng = np.random.default_rng(33)
    pd = scengen.params("1.1B-13B", K=6, O_max=100)
    for _ in range(20):
        Is = np.sort(rng.integers(1, 513, 6)).astype(np.int32)
        a = float(rng.uniform(0.5, 0.9))
        g = int(rng.integers(0, 9))
        cuts = sorted(rng.choice(np.arange(1, 6), size=int(rng.integers(0, 5)), replace=False).tolist())
        ends = cuts + [6]
        assert orc.eval_plan(pd, Is, a, g, ends) <= orc.eval_plan_nopipe(pd, Is, a, g, ends) * (1 + 1e-12)
        assert rel(orc.eval_plan(pd, Is, a, g, [6]), orc.eval_plan_nopipe(pd, Is, a, g, [6])) < 1e-12


def test_fixed_plans(orc):
    Is = np.sort(np.random.default_rng(34).integers(1, 513, 13)).astype(np.int32)
    pd = scengen.params("68M-7B", K=13, O_max=64)
    assert orc.fixed_plan(dict(pd, batching_policy=NONE), Is, 0.7, 3) == list(range(1, 14))
    assert orc.fixed_plan(dict(pd, batching_policy=STATIC, static_batch=4), Is, 0.7, 3) == [4, 8, 12, 13]
    assert orc.fixed_plan(dict(pd, batching_policy=STATIC, static_batch=40), Is, 0.7, 3) == [13]
    # max batching: 68M never binds (b = K); 1.1B binds at 30 for I = 512
    assert orc.fixed_plan(dict(pd, batching_policy=MAX), Is, 0.7, 3) == [13]
    pd11 = scengen.params("1.1B-7B", K=70)
    Is512 = np.full(70, 512, np.int32)
    assert orc.fixed_plan(dict(pd11, batching_policy=MAX), Is512, 0.7, 3) == [30, 60, 70]
    assert orc.fixed_plan(dict(pd11, batching_policy=MAX, mem_capacity_bytes=10**9), Is512, 0.7, 3) == []


def test_heuristic_stopping_rule(orc):
    """Heuristic batching (reading B5): sizes 2, 3, ... while the pipelined
    latency (eq:time) keeps improving; the returned size is the last improving
    one -- checked against eval_plan of every equal-size plan."""
    rng = np.random.default_rng(35)
    for _ in range(25):
        K = int(rng.integers(2, 24))
        pair = ["68M-7B", "1.1B-7B"][int(rng.integers(2))]
        pd = dict(scengen.params(pair, K=K, O_max=int(rng.choice([64, 512]))), batching_policy=HEUR)
        Is = np.sort(rng.integers(1, 513, K)).astype(np.int32)
        a = float(rng.uniform(0.5, 0.9))
        g = int(rng.integers(1, 9))
        ends = orc.fixed_plan(pd, Is, a, g)

        def plan(b):
            return [e for e in range(b, K, b)] + [K]
        T = {b: orc.eval_plan(pd, Is, a, g, plan(b)) for b in range(2, K + 1)}
        b = 2
        while b + 1 <= K and T[b + 1] < T[b]:
            b += 1
        assert ends == plan(b)


def test_heuristic_from_two_batches(orc):
    """Reading B5': start from two batches, b = ceil(K/2), and grow b
    while eq:time keeps improving -- checked against eval_plan of every plan."""
    rng = np.random.default_rng(37)
    for _ in range(25):
        K = int(rng.integers(2, 24))
        pd = dict(scengen.params("1.1B-7B", K=K, O_max=int(rng.choice([64, 512]))), batching_policy=HEUR,
                  heuristic_start=1)
        Is = np.sort(rng.integers(1, 513, K)).astype(np.int32)
        a = float(rng.uniform(0.5, 0.9))
        g = int(rng.integers(1, 9))

        def plan(b):
            return [e for e in range(b, K, b)] + [K]
        b = (K + 1) // 2
        T = {q: orc.eval_plan(pd, Is, a, g, plan(q)) for q in range(b, K + 1)}
        while b + 1 <= K and T[b + 1] < T[b]:
            b += 1
        assert orc.fixed_plan(pd, Is, a, g) == plan(b)


def test_policy_solves_are_consistent(orc):
    """Every policy's T_inf equals the literal evaluation of its own plan and
    gamma; FSL is gamma_min = gamma_max = 7; ADS core is gamma = 0."""
    _, sc, _ = scengen.config("C3", 0, 6)
    for pol in (NO_PIPE, NONE, STATIC, MAX, HEUR):
        pd = dict(scengen.params("1.1B-7B", K=32, gamma_min=1, gamma_max=8), batching_policy=pol)
        out = orc.solve_batch(pd, sc)
        for s in range(6):
            assert out["status"][s] == 0
            Is = sc["I"][s][out["order"][s]]
            ends = list(out["batch_end"][s][: out["M"][s]])
            ev = orc.eval_plan_nopipe if pol == NO_PIPE else orc.eval_plan
            assert rel(ev(pd, Is, float(sc["alpha"][s]), int(out["gamma"][s]), ends), out["lat"][s, 2]) < 1e-12
    fsl = orc.solve_batch(scengen.params("68M-7B", K=32, gamma_min=7, gamma_max=7), sc)
    assert np.all(fsl["gamma"] == 7)


# ---------------------------------------------------------------- NEXT-1
def test_actual_output_evaluation(orc):
    """Actual-output evaluation: equals the planned
    evaluation when every O_k = O_max, never exceeds it, and a batch that has
    finished drops out of later steps."""
    rng = np.random.default_rng(36)
    pd = scengen.params("1.1B-7B", K=9, O_max=300)
    for _ in range(20):
        Is = np.sort(rng.integers(1, 513, 9)).astype(np.int32)
        Os = rng.integers(1, 301, 9).astype(np.int32)
        a = float(rng.uniform(0.5, 0.9))
        g = int(rng.integers(0, 9))
        cuts = sorted(rng.choice(np.arange(1, 9), size=int(rng.integers(0, 8)), replace=False).tolist())
        ends = cuts + [9]
        full = orc.eval_plan(pd, Is, a, g, ends)
        assert rel(orc.eval_actual(pd, Is, np.full(9, 300, np.int32), a, g, ends), full) < 1e-14
        assert orc.eval_actual(pd, Is, Os, a, g, ends) <= full * (1 + 1e-12)
    # two batches, n_1 = 2 and n_2 = 1: step 2 runs batch 1 alone
    pd2 = scengen.params("68M-7B", K=2, O_max=8)
    Is, a, g = np.array([100, 200], np.int32), 0.5, 1          # L = 1.5
    Os = np.array([3, 1], np.int32)                              # n = ceil(3/1.5) = 2, ceil(1/1.5) = 1
    L = orc.expected_tokens(a, g)
    td = [[orc.draft_time(pd2, 1, int(Is[m]), g, L, n) for m in range(2)] for n in (1, 2)]
    tv = [[orc.verify_time(pd2, 1, int(Is[m]), g, L, n) for m in range(2)] for n in (1, 2)]
    step1 = max(td[0][0] + td[0][1], td[0][0] + tv[0][0]) + tv[0][1]
    step2 = td[1][0] + tv[1][0]
    assert rel(orc.eval_actual(pd2, Is, Os, a, g, [1, 2]), step1 + step2) < 1e-14


def test_actual_output_nopipe(orc):
    """Under SD w/o pipeline the actual-output replay is sequential too, and
    equals the sequential planned evaluation when every O_k = O_max."""
    rng = np.random.default_rng(37)
    pd = dict(scengen.params("1.1B-7B", K=7, O_max=200), batching_policy=NO_PIPE)
    for _ in range(10):
        Is = np.sort(rng.integers(1, 513, 7)).astype(np.int32)
        a, g = float(rng.uniform(0.5, 0.9)), int(rng.integers(0, 9))
        ends = [2, 5, 7]
        assert rel(orc.eval_actual(pd, Is, np.full(7, 200, np.int32), a, g, ends),
                   orc.eval_plan_nopipe(pd, Is, a, g, ends)) < 1e-14


@pytest.mark.parametrize("pair", ["68M-7B", "1.1B-7B"])
def test_row_optimum_monotone_in_prefix(orc, pair):
    """T*(i), the optimal pipelined latency of the i shortest tasks (Algorithm 1's
    row value, eq:time), is non-decreasing in i: dropping the longest task from its
    batch shrinks the batch and cannot raise its padded length, so no stage time
    grows.  The GPU's gamma-level pruning rests on this; checked
    here on the oracle, prefix by prefix, with binding memory windows included."""
    K = 24
    base = scengen.params(pair, K=K, gamma_min=1, gamma_max=6)
    J, h1, h2 = scengen.MODELS[pair.split("-")[0]]
    tight = orc.param_memory(J, h1, h2) + 6 * orc.kv_memory_per_task(J, h1, 256, base["O_max"])
    sc = scengen.generate(77, K, 0, 6, I_max=1024)
    for pd in (base, dict(base, mem_capacity_bytes=int(tight))):
        for s in range(6):
            Is = np.sort(sc["I"][s])
            for gamma in (1, 3, 6):
                prev = 0.0
                for i in range(1, K + 1):
                    t = orc.dp(dict(pd, K=i), Is[:i], float(sc["alpha"][s]), gamma)[0]
                    if not np.isfinite(t):
                        break
                    assert t >= prev * (1 - 1e-12), (s, gamma, i, t, prev)
                    prev = t


@pytest.mark.parametrize("pair", ["68M-7B", "1.1B-7B"])
def test_t_inf_at_least_total_verify_work(orc, pair):
    """T_inf(gamma) >= sum_k vsl(I_k) + vc: every step's pipeline makespan is at
    least the verify stage's serial work (eq:time), a batch's verify time is affine
    in its size with a slope that grows with the padded length (eq:flops_v,
    eq:latency_b2), so each task pays at least its own length's slope and the
    last batch at least the intercept.  The GPU skips a gamma whose bound exceeds
    the best finished T_inf; this pins the bound on the oracle's
    literal DP and stage-time functions."""
    K = 12
    pd = scengen.params(pair, K=K, gamma_min=1, gamma_max=8, O_max=256)
    sc = scengen.generate(91, K, 0, 5)
    for s in range(5):
        Is = np.sort(sc["I"][s])
        alpha = float(sc["alpha"][s])
        for gamma in (1, 2, 5, 8):
            L = orc.expected_tokens(alpha, gamma)
            N = orc.decode_steps(pd["O_max"], L)
            t_inf = orc.dp(pd, Is, alpha, gamma)[0]
            lb = 0.0
            for n in range(1, N + 1):
                for I in Is:
                    t1 = orc.verify_time(pd, 1, int(I), gamma, L, n)
                    t2 = orc.verify_time(pd, 2, int(I), gamma, L, n)
                    lb += t2 - t1                                # this task's slope at its own length
                t1 = orc.verify_time(pd, 1, int(Is[-1]), gamma, L, n)
                t2 = orc.verify_time(pd, 2, int(Is[-1]), gamma, L, n)
                lb += 2 * t1 - t2                                # one intercept
            assert t_inf >= lb * (1 - 1e-12), (s, gamma, t_inf, lb)
            assert lb > 0.5 * t_inf or pair != "68M-7B"          # and it is not vacuous for a small draft


@pytest.mark.parametrize("pair", ["68M-7B", "1.1B-7B"])
def test_row_value_plus_remaining_verify_work(orc, pair):
    """Upsilon[K,0,0] >= Upsilon[i,0,0] + sum_{k>i} vsl(I_k) for every row i: each
    candidate of row i+1 either extends a candidate of row i by task i+1 (same
    predecessor state; its batch's verify time grows by at least that task's own
    slope, every other stage time can only grow -- eq:flops_v, eq:latency_b2,
    eq:time) or starts a new batch after row i's state (every step's completion
    is at least Upsilon1[i,n] plus the new batch's verify time).  The GPU stops a
    gamma at a tile end when this bound exceeds the best finished T_inf (DESIGN.md
    5.2e); pinned here on the oracle's literal DP (row values from orc_dp_trace)
    and stage-time functions, with binding memory windows for the 1.1B draft."""
    K = 14
    pd = scengen.params(pair, K=K, gamma_min=1, gamma_max=8, O_max=192)
    if pair == "1.1B-7B":
        J, h1, h2 = scengen.MODELS["1.1B"]
        pd = dict(pd, mem_capacity_bytes=orc.param_memory(J, h1, h2) + 5 * orc.kv_memory_per_task(J, h1, 300, 192))
    sc = scengen.generate(93, K, 0, 6)
    n_tight = 0
    for s in range(6):
        Is = np.sort(sc["I"][s])
        alpha = float(sc["alpha"][s])
        for gamma in (1, 3, 7):
            L = orc.expected_tokens(alpha, gamma)
            N = orc.decode_steps(pd["O_max"], L)
            t, S, gap, rb, rt, W = orc.dp_trace(pd, Is, alpha, gamma)
            if not np.isfinite(t):
                continue
            vsl = np.array([sum(orc.verify_time(pd, 2, int(I), gamma, L, n) - orc.verify_time(pd, 1, int(I), gamma, L, n)
                                for n in range(1, N + 1)) for I in Is])
            for i in range(1, K):
                bound = rt[i - 1] + vsl[i:].sum()
                assert t >= bound * (1 - 1e-12), (s, gamma, i, t, bound)
                n_tight += bound > 0.9 * t
            assert np.all(np.diff(rt) >= vsl[1:] * (1 - 1e-12) - 1e-12 * rt[1:])   # row by row
    assert n_tight > 0


@pytest.mark.parametrize("pair", ["68M-7B", "1.1B-7B", "1.1B-13B"])
def test_t_inf_at_least_draft_work(orc, pair):
    """T_inf(gamma) >= sum_k dsl(I_k) + vsl(I_K) + (gamma c2d + c2v) N: every step's
    makespan (eq:time) is at least the draft stage's serial work -- each batch's
    draft time is affine in its size with a slope growing with the padded length
    (eq:flops_d, eq:latency_b2, eq:d_latency), so each task pays at least its own
    length's slope and some batch the intercept -- plus the last batch's verify
    time, which holds task K.  The GPU uses max(this, the verify-side bound) to
    skip a gamma before its DP; pinned on the literal DP."""
    K = 10
    pd = scengen.params(pair, K=K, gamma_min=1, gamma_max=8, O_max=160)
    sc = scengen.generate(95, K, 0, 5)
    n_tight = 0
    for s in range(5):
        Is = np.sort(sc["I"][s])
        alpha = float(sc["alpha"][s])
        for gamma in (1, 3, 6):
            L = orc.expected_tokens(alpha, gamma)
            N = orc.decode_steps(pd["O_max"], L)
            t_inf = orc.dp(pd, Is, alpha, gamma)[0]
            lb = 0.0
            for n in range(1, N + 1):
                for I in Is:
                    lb += orc.draft_time(pd, 2, int(I), gamma, L, n) - orc.draft_time(pd, 1, int(I), gamma, L, n)
                d1 = orc.draft_time(pd, 1, int(Is[-1]), gamma, L, n)
                lb += 2 * d1 - orc.draft_time(pd, 2, int(Is[-1]), gamma, L, n)      # one draft intercept
                lb += orc.verify_time(pd, 1, int(Is[-1]), gamma, L, n)              # last batch's verify
            assert t_inf >= lb * (1 - 1e-12), (s, gamma, t_inf, lb)
            n_tight += lb > 0.6 * t_inf
    assert n_tight > 0 or pair == "68M-7B"


@pytest.mark.parametrize("pair", ["68M-7B", "1.1B-7B"])
def test_t_inf_at_least_verify_work_by_batch_count(orc, pair):
    """T_inf(gamma) >= min over the batch count M of the verify stage's serial work plus the first
    batch's draft work: M = 1 is the single batch's latency, M = 2 the best split into two
    memory-feasible batches (each padded to its last, longest task), M >= 3 at least every task's
    own verify slope plus 3 intercepts plus a one-task draft at the shortest length (eq:time: each
    step's makespan >= T^d_{n,1} + sum_m T^v_{n,m}; eq:flops_v, eq:flops_d, eq:latency_b2).  The GPU
    uses it to skip a gamma before its DP; pinned on the literal DP, with a
    binding memory window for the 1.1B draft."""
    K = 10
    pd = scengen.params(pair, K=K, gamma_min=1, gamma_max=8, O_max=160)
    if pair == "1.1B-7B":
        J, h1, h2 = scengen.MODELS["1.1B"]
        pd = dict(pd, mem_capacity_bytes=orc.param_memory(J, h1, h2) + 6 * orc.kv_memory_per_task(J, h1, 300, 160))
    sc = scengen.generate(97, K, 0, 6)
    n_bind = 0
    for s in range(6):
        Is = np.sort(sc["I"][s])
        alpha = float(sc["alpha"][s])
        for gamma in (1, 2, 5):
            L = orc.expected_tokens(alpha, gamma)
            N = orc.decode_steps(pd["O_max"], L)
            t_inf = orc.dp(pd, Is, alpha, gamma)[0]
            if not np.isfinite(t_inf):
                continue

            def vwork(b, I):           # sum_n T^v_n of one batch of b tasks padded to I
                return sum(orc.verify_time(pd, b, int(I), gamma, L, n) for n in range(1, N + 1))

            def dwork(b, I):           # sum_n T^d_n of one batch (the first batch's draft delays every verify)
                return sum(orc.draft_time(pd, b, int(I), gamma, L, n) for n in range(1, N + 1))

            def fits(b, I):
                return np.isfinite(orc.eval_plan(dict(pd, K=b), np.full(b, I, np.int32), alpha, gamma, [b]))
            own = sum(vwork(2, I) - vwork(1, I) for I in Is)
            vc = 2 * vwork(1, Is[-1]) - vwork(2, Is[-1])
            cands = [own + 3 * vc + dwork(1, Is[0])]
            if fits(K, Is[-1]):
                cands.append(vwork(K, Is[-1]) + dwork(K, Is[-1]))
                assert abs(cands[-1] - orc.eval_plan(pd, Is, alpha, gamma, [K])) <= 1e-12 * cands[-1]
            for sp in range(1, K):
                if fits(sp, Is[sp - 1]) and fits(K - sp, Is[-1]):
                    cands.append(vwork(sp, Is[sp - 1]) + vwork(K - sp, Is[-1]) + dwork(sp, Is[sp - 1]))
            lb = min(cands)
            assert t_inf >= lb * (1 - 1e-12), (s, gamma, t_inf, lb)
            n_bind += lb > own + vc
    assert n_bind > 0
