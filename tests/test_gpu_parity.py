"""-m gpu: the CUDA path (through the C ABI) against the oracle, element by
element on the same seeded inputs (tests/parity.py for the tolerances).

Sizes: C1/C2 in full; C3 on a sample spanning many CTAs and ragged rows;
C4 and C5 solved at FULL size in the bench's launch configuration and
checked on deterministic samples the oracle can compute one by one, plus
properties that hold at any size (self-consistency of the plan under the
literal eq:time evaluation, constraints (a)-(g))."""
import numpy as np
import pytest

import oracle
import scengen
from tests.parity import compare, gpu_solve, load_fixture, to_numpy

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ENV, DENSE = 0, 1


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2510_11331_b200 as sd
    sd.lib()
    oracle.build()


def _check(pd, sc, precision=0, algo=ENV, orc=None, idx=None):
    orc = orc if orc is not None else oracle.solve_batch(pd, sc)
    g = gpu_solve(pd, sc, precision=precision, algo=algo, idx=idx)
    return compare(pd, sc, g, orc, precision, oracle), orc, g


# ---------------------------------------------------------------- C1, C2
@pytest.mark.parametrize("pair", ["68M-7B", "1.1B-7B", "1.1B-13B"])
def test_c1_all(pair):
    pd, sc, _ = scengen.config("C1", pair=pair)
    orc = oracle.solve_batch(pd, sc)
    for prec, algo in ((0, ENV), (0, DENSE), (1, ENV), (1, DENSE)):
        res, _, g = _check(pd, sc, prec, algo, orc)
        assert res["failures"] == 0
    assert g["gamma"][0] == {"68M-7B": 4, "1.1B-7B": 3, "1.1B-13B": g["gamma"][0]}[pair]


def test_c1_against_brute_force():
    """Joint brute force over every contiguous partition and gamma (K = 4): the
    GPU never beats it, and matches it wherever Algorithm 1 is exact (P8)."""
    pd, sc, _ = scengen.config("C1", 0, 200, pair="1.1B-13B")
    g = gpu_solve(pd, sc)
    n_eq = 0
    for s in range(200):
        Is = sc["I"][s][g["order"][s]]
        bf, bg, plan = oracle.brute_force(pd, Is, float(sc["alpha"][s]), 0, 4)
        assert g["lat"][s, 2] >= bf * (1 - 1e-12)
        n_eq += abs(g["lat"][s, 2] - bf) <= 1e-12 * bf
    assert n_eq >= 150


def test_c2_heterogeneous_speeds():
    pd, sc, _ = scengen.config("C2")
    orc = oracle.solve_batch(pd, sc)
    for prec, algo in ((0, ENV), (0, DENSE), (1, ENV)):
        res, _, _ = _check(pd, sc, prec, algo, orc)
        assert res["failures"] == 0


# ---------------------------------------------------------------- C3
@pytest.mark.parametrize("pair", ["68M-7B", "1.1B-7B"])
def test_c3_sample(pair):
    _, sc, _ = scengen.config("C3", 0, 1500)
    pd = scengen.params(pair, K=32, gamma_min=1, gamma_max=8)
    orc = oracle.solve_batch(pd, sc)
    res, _, _ = _check(pd, sc, 0, ENV, orc)
    assert res["exact"] + res["exempt_same"] + res["replayed"] == 1500
    sub = {k: (v[:300] if v is not None else None) for k, v in sc.items()}
    orc_sub = {k: v[:300] if hasattr(v, "__len__") else v for k, v in orc.items()}
    _check(pd, sub, 0, DENSE, orc_sub)
    _check(pd, sub, 1, ENV, orc_sub)


# ---------------------------------------------------------------- C4 (bench config)
def _full(cfg, pair, precision=0):
    pd, sc, n = scengen.config(cfg, pair=pair)
    return pd, sc, n, gpu_solve(pd, sc, precision=precision)


@pytest.mark.parametrize("precision", [0, 1])
@pytest.mark.parametrize("pair", ["68M-7B", "1.1B-7B"])
def test_c4_full_size_sampled(pair, precision):
    """All 1e6 C4 scenarios in one call (the bench launch), fp64 and the fp32
    variant; the oracle's stored results on the deterministic sample (s = 0 mod
    500: 2000 scenarios for (68M,7B); s = 0 mod 2000 for (1.1B,7B); written by
    tools/make_oracle_fixtures.py from oracle/ only) with the north_star
    tolerances and the near-tie replay; invariants on every scenario."""
    name = f"c4_{pair}"
    _, _, idx, orc = load_fixture(name)
    pd, sc, n, g = _full("C4", pair, precision)
    res = compare(pd, sc, g, orc, precision, oracle, idx=idx, label=f"C4 {pair} full launch, sample {len(idx)}, "
                                                                   f"{'fp64' if precision == 0 else 'fp32'}")
    assert res["failures"] == 0
    assert np.all(g["status"] == 0)
    M = g["M"]
    assert np.all((M >= 1) & (M <= 128)) and np.all((g["gamma"] >= 1) & (g["gamma"] <= 16))
    assert np.all(g["batch_end"][np.arange(n), M - 1] == 128)
    assert np.all(g["lat"][:, 0] == g["lat"][:, 1] + g["lat"][:, 2])
    assert np.allclose(g["w"].sum(1), 1.0, rtol=0, atol=1e-12)
    # the trace backtracks to the plan on every scenario (a cheap full-size consistency check)
    tr, be = g["trace"], g["batch_end"]
    for s in range(0, n, 997):
        assert oracle.backtrack(tr[s]) == [int(x) for x in be[s][: M[s]]]


# ---------------------------------------------------------------- C5 (large K)
@pytest.mark.parametrize("K", [256, 512, 1024])
def test_c5_large_k(K):
    """Full 1e4-scenario launch at each K and the full gamma range 1..16; the
    oracle's stored results on the first scenarios (tools/make_oracle_fixtures.py)
    and the eq:time self-consistency of sampled GPU plans."""
    _, _, idx, orc = load_fixture(f"c5_{K}")
    pd, sc, n, g = _full(f"C5{K}", "68M-7B")
    assert np.all(g["status"] == 0)
    res = compare(pd, sc, g, orc, 0, oracle, idx=idx, label=f"C5 K={K} full launch, gamma 1..16")
    assert res["failures"] == 0
    rng = np.random.default_rng(K)
    for s in rng.choice(n, 6, replace=False):
        Is = sc["I"][s][g["order"][s]]
        ends = list(g["batch_end"][s][: g["M"][s]])
        v = oracle.eval_plan(pd, Is, float(sc["alpha"][s]), int(g["gamma"][s]), ends)
        assert abs(v - g["lat"][s, 2]) <= 1e-12 * v
    sub = {k: (v[:1] if v is not None else None) for k, v in sc.items()}
    pd2 = dict(pd, gamma_min=1, gamma_max={256: 4, 512: 2, 1024: 1}[K])
    _check(pd2, sub, 0, DENSE)


# ---------------------------------------------------------------- edge cases
def test_k1_and_single_step():
    for K, O in ((1, 2048), (5, 1), (7, 2)):
        pd = scengen.params("1.1B-7B", K=K, gamma_min=0, gamma_max=6, O_max=O)
        sc = scengen.generate(21, K, 0, 64)
        for algo in (ENV, DENSE):
            _check(pd, sc, 0, algo)


def test_memory_window_and_infeasible():
    pd = scengen.params("1.1B-7B", K=64, gamma_min=1, gamma_max=4)
    sc = scengen.generate(22, 64, 0, 40)
    sc["I"][:20] = np.maximum(sc["I"][:20], 400)  # windows bind hard
    _check(pd, sc, 0, ENV)
    pd_bad = dict(pd, mem_capacity_bytes=2_000_000_000)  # 1.1B weights + one KV barely / not fit
    res, orc, g = _check(pd_bad, sc, 0, ENV)
    assert np.any(g["status"] == 1)
    assert np.all(np.isinf(g["lat"][g["status"] == 1, 0]))


@pytest.mark.parametrize("pair", ["68M-7B", "1.1B-7B"])
@pytest.mark.parametrize("bmax", [2, 5, 9, 31])
def test_narrow_memory_windows(pair, bmax):
    """Memory windows narrower than a DP tile (Alg. 1 lines 10-13):
    with b_max < tile rows a row's window starts inside its own tile, so the
    tiled DP has no older predecessor for it and the warm start must not
    propose one.  Capacity = weights + b_max KV caches of a mid-length task."""
    K = 64
    pd = scengen.params(pair, K=K, gamma_min=1, gamma_max=8)
    J, h1, h2 = scengen.MODELS[pair.split("-")[0]]
    cap = oracle.param_memory(J, h1, h2) + bmax * oracle.kv_memory_per_task(J, h1, 256, pd["O_max"])
    pd = dict(pd, mem_capacity_bytes=int(cap))
    sc = scengen.generate(40 + bmax, K, 0, 300)
    for prec in (0, 1):
        res, orc, g = _check(pd, sc, prec, ENV)
        assert res["failures"] == 0
    ends = [np.diff(np.r_[0, g["batch_end"][s][: g["M"][s]]]).max() for s in range(300) if g["status"][s] == 0]
    assert len(ends) > 0 and max(ends) <= 2 * bmax + 2     # the windows really bind


@pytest.mark.parametrize("pair", ["68M-7B", "1.1B-13B"])
def test_high_acceptance_gamma_pruning(pair):
    """High acceptance rates (alpha in [0.9, 0.99)) move gamma* away from 1, so the
    gamma-level pruning works against a best found late and
    prunes in a different pattern; results must still match the oracle."""
    pd = scengen.params(pair, K=48, gamma_min=1, gamma_max=12)
    sc = scengen.generate(55, 48, 0, 200, alpha_lo=0.9, alpha_hi=0.99)
    res, orc, g = _check(pd, sc, 0, ENV)
    assert res["failures"] == 0
    assert len(set(int(x) for x in orc["gamma"])) > 2        # a spread of gamma*, not all 1


def test_invalid_scenarios_status():
    pd = scengen.params("68M-7B", K=8, gamma_min=1, gamma_max=3)
    sc = scengen.generate(23, 8, 0, 6)
    sc["alpha"][1] = 1.0
    sc["alpha"][2] = float("nan")
    sc["I"][3, 4] = 0
    sc["g"][4, 0] = -1e-9
    sc["p"][5, 7] = float("inf")
    res, orc, g = _check(pd, sc)
    assert list(g["status"]) == [0, 2, 2, 3, 3, 3]


def test_downlink_and_gamma0():
    pd = scengen.params("68M-7B", K=16, gamma_min=0, gamma_max=3, downlink_s=2.5e-3)
    sc = scengen.generate(24, 16, 0, 50)
    _check(pd, sc, 0, ENV)
    _check(pd, sc, 0, DENSE)


def test_exact_ties_largest_j():
    """All runtime coefficients zero: every candidate ties at exactly 0, so
    the '>=' rule (largest j) gives M = K singleton batches (reading A6)."""
    pd = scengen.params("68M-7B", K=12, gamma_min=1, gamma_max=2, c1_draft=0.0, c2_draft=0.0,
                        c1_verify=0.0, c2_verify=0.0)
    sc = scengen.generate(25, 12, 0, 8)
    g = gpu_solve(pd, sc)
    assert np.all(g["M"] == 12) and np.all(g["gamma"] == 1) and np.all(g["lat"][:, 2] == 0.0)
    orc = oracle.solve_batch(pd, sc)
    assert np.array_equal(orc["batch_end"], g["batch_end"])


def test_overflow_second_pass():
    """FLAG_TINY_POOL forces every multi-segment DP through the worst-case
    second pass; results must be identical to the normal path."""
    pd = scengen.params("1.1B-7B", K=64, gamma_min=1, gamma_max=8)
    _, sc, _ = scengen.config("C2")
    sc = dict(sc)
    a = gpu_solve(pd, sc)
    b = gpu_solve(dict(pd, flags=1), sc)
    for k in a:
        if a[k] is not None:
            assert np.array_equal(a[k], b[k]), k


def test_host_entry_point_and_determinism():
    import paper_2510_11331_b200 as sd
    pd, sc, _ = scengen.config("C3", 0, 3000)
    d1 = gpu_solve(pd, sc)
    d2 = gpu_solve(pd, sc)
    I = torch.from_numpy(sc["I"]).pin_memory()
    p = torch.from_numpy(sc["p"]).pin_memory()
    g = torch.from_numpy(sc["g"]).pin_memory()
    al = torch.from_numpy(sc["alpha"]).pin_memory()
    h = sd.solve_host(pd, I, p, g, al)
    torch.cuda.synchronize()
    h = to_numpy(h)
    for k in d1:
        assert np.array_equal(d1[k], d2[k]), k
    for k in h:                                      # the host entry has no trace output
        assert np.array_equal(d1[k], h[k]), k


def test_permutation_invariance():
    pd, sc, _ = scengen.config("C3", 0, 200)
    a = gpu_solve(pd, sc)
    rng = np.random.default_rng(3)
    perm = np.stack([rng.permutation(32) for _ in range(200)])
    sc2 = dict(sc, I=np.take_along_axis(sc["I"], perm, 1), p=np.take_along_axis(sc["p"], perm, 1),
               g=np.take_along_axis(sc["g"], perm, 1))
    b = gpu_solve(pd, sc2)
    assert np.allclose(a["lat"], b["lat"], rtol=1e-12, atol=0)
    assert np.array_equal(a["gamma"], b["gamma"]) and np.array_equal(a["batch_end"], b["batch_end"])


def test_wide_snr_range_bandwidth():
    """eq:opt_w over SNRs from 1e-14 to 1e14 (the kernel's own log2(1 + SNR) and 1/sigma^2):
    w* and T_com within 1e-12 of the oracle's libm log2, including SNRs whose 1 + SNR rounds to 1."""
    pd, sc, _ = scengen.config("C3", 0, 300)
    rng = np.random.default_rng(11)
    snr = 10.0 ** rng.uniform(-14, 14, size=sc["g"].shape)
    snr[:5, 0] = 1e-17                                   # 1 + SNR == 1: s_k = 0, t_com and w* infinite / NaN
    g = snr * pd["noise_w"] / sc["p"]
    sc2 = dict(sc, g=np.ascontiguousarray(g))
    part = lambda a, b: {k: (None if v is None else np.ascontiguousarray(v[a:b])) for k, v in sc2.items()}  # noqa: E731
    res, _, _ = _check(pd, part(5, 300))
    assert res["failures"] == 0
    gg, o = gpu_solve(pd, part(0, 5)), oracle.solve_batch(pd, part(0, 5))
    for s in range(5):                                    # same non-finite outcome as the oracle
        assert np.array_equal(np.isfinite(gg["lat"][s]), np.isfinite(o["lat"][s]))
        assert gg["status"][s] == o["status"][s]


@pytest.mark.parametrize("cfg,n", [("C3", 70000), ("C5256", 300)])
def test_host_compact_layout(cfg, n):
    """sdedge_solve_batch_host_compact returns exactly sdedge_solve_batch_host's results (uint16 order,
    batch ends as a bit mask; several pipeline chunks at C3 70000, a 256-bit mask per scenario at K = 256)."""
    import paper_2510_11331_b200 as sd
    pd, sc, _ = scengen.config(cfg, 0, n)
    host = {k: torch.from_numpy(np.ascontiguousarray(sc[k])).pin_memory() for k in ("I", "p", "g", "alpha")}
    full = sd.solve_host(pd, host["I"], host["p"], host["g"], host["alpha"])
    comp = sd.solve_host_compact(pd, host["I"], host["p"], host["g"], host["alpha"])
    torch.cuda.synchronize()
    u = sd.unpack_compact(comp)
    for k in ("lat", "gamma", "M", "batch_end", "order", "w", "status"):
        a, b = full[k].numpy(), u[k]
        assert np.array_equal(a, b, equal_nan=True), k


def test_streams_and_empty_call():
    import paper_2510_11331_b200 as sd
    pd, sc, _ = scengen.config("C3", 0, 500)
    I = torch.from_numpy(sc["I"]).cuda()
    p = torch.from_numpy(sc["p"]).cuda()
    g = torch.from_numpy(sc["g"]).cuda()
    al = torch.from_numpy(sc["alpha"]).cuda()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    o1 = sd.solve(pd, I, p, g, al, stream=s1)
    o2 = sd.solve(pd, I, p, g, al, stream=s2)
    torch.cuda.synchronize()
    for k in o1:
        if o1[k] is not None:
            assert torch.equal(o1[k], o2[k])
    e = sd.solve(pd, I[:0], p[:0], g[:0], al[:0])
    torch.cuda.synchronize()
    assert e["lat"].shape == (0, 3)
    assert sd.sdedge_last_launch_count() == 0


def test_pipe_peak_runs():
    import paper_2510_11331_b200 as sd
    ops, t = sd.sdedge_pipe_peak(False)
    assert ops > 1e12 and t > 0


def test_host_entry_point_chunked():
    """More than one 65536-scenario chunk through the pipelined host entry:
    identical bytes to the device entry point."""
    import paper_2510_11331_b200 as sd
    pd = scengen.params("68M-7B", K=32, gamma_min=1, gamma_max=8)
    sc = scengen.generate(3, 32, 0, 200_000)
    d = gpu_solve(pd, sc)
    h = sd.solve_host(pd, *(torch.from_numpy(sc[k]).pin_memory() for k in ("I", "p", "g", "alpha")))
    torch.cuda.synchronize()
    h = to_numpy(h)
    for k in h:
        assert np.array_equal(d[k], h[k]), k


# ---------------------------------------------------------------- paper baselines (NEXT-2)
@pytest.mark.parametrize("pol", [1, 2, 3, 4, 5, "5half"])
def test_batching_policies(pol):
    """SD w/o pipeline, no batching, static, max and heuristic batching (both
    readings B5 and B5') against the oracle."""
    _, sc, _ = scengen.config("C3", 0, 300)
    hs = 1 if pol == "5half" else 0
    pol = 5 if pol == "5half" else pol
    for pair in ("68M-7B", "1.1B-7B"):
        pd = dict(scengen.params(pair, K=32, gamma_min=1, gamma_max=8), batching_policy=pol, static_batch=5,
                  heuristic_start=hs)
        for algo in (ENV, DENSE):
            res, _, g = _check(pd, sc, 0, algo)
            assert res["failures"] == 0
    pd = dict(scengen.params("1.1B-7B", K=128, gamma_min=1, gamma_max=16), batching_policy=pol, static_batch=5,
              heuristic_start=hs)
    _, sc4, _ = scengen.config("C4", 0, 24)
    _check(pd, sc4, 0, ENV)


def test_uniform_bandwidth_policy():
    """Uniform w_k = 1/K: T_com never below the optimal t*_com,
    T_inf and the schedule unchanged (decoupling)."""
    pd, sc, _ = scengen.config("C3", 0, 500)
    a = gpu_solve(pd, sc)
    pu = dict(pd, bandwidth_policy=1)
    res, _, b = _check(pu, sc, 0, ENV)
    assert np.all(b["lat"][:, 1] >= a["lat"][:, 1] * (1 - 1e-12))
    assert np.array_equal(a["lat"][:, 2], b["lat"][:, 2]) and np.array_equal(a["batch_end"], b["batch_end"])
    assert np.all(b["w"] == 1.0 / 32)


# ---------------------------------------------------------------- actual outputs (NEXT-1)
@pytest.mark.parametrize("pol", [0, 1])
@pytest.mark.parametrize("cfg,pair,n", [("C3", "68M-7B", 2000), ("C3", "1.1B-7B", 2000), ("C2", None, 3),
                                        ("C4", "68M-7B", 64)])
def test_actual_output_evaluation(cfg, pair, n, pol):
    """sdedge_evaluate_actual on the GPU's own plans vs the oracle's literal
    replay (eq:step_n, M_n, eq:time) of the same plans with O_k ~ U{1..O_max}."""
    import paper_2510_11331_b200 as sd
    pd, sc, _ = scengen.config(cfg, 0, n, pair=pair)
    pd = dict(pd, batching_policy=pol)
    K = pd["K"]
    O = scengen.output_lengths(9, K, 0, n, pd["O_max"])
    dev = "cuda:0"
    t = {k: torch.from_numpy(np.ascontiguousarray(sc[k])).to(dev) for k in ("I", "p", "g", "alpha")}
    co = None if sc.get("coeffs") is None else torch.from_numpy(sc["coeffs"]).to(dev)
    plan = sd.solve(pd, t["I"], t["p"], t["g"], t["alpha"], co)
    act = sd.evaluate_actual(pd, t["I"], t["p"], t["g"], t["alpha"], torch.from_numpy(O).to(dev), plan, co)
    torch.cuda.synchronize()
    act = act.cpu().numpy()
    pl = to_numpy(plan)
    for s in range(n):
        Is = sc["I"][s][pl["order"][s]]
        Os = O[s][pl["order"][s]]
        ends = list(pl["batch_end"][s][: pl["M"][s]])
        cs = None if sc.get("coeffs") is None else sc["coeffs"][s]
        v = oracle.eval_actual(pd, Is, Os, float(sc["alpha"][s]), int(pl["gamma"][s]), ends, coeffs=cs)
        assert abs(act[s] - v) <= 1e-12 * v, (s, act[s], v)
        assert act[s] <= pl["lat"][s, 2] * (1 + 1e-12)
    # O_k = O_max reproduces the planned T_inf
    full = sd.evaluate_actual(pd, t["I"], t["p"], t["g"], t["alpha"],
                              torch.full((n, K), pd["O_max"], dtype=torch.int32, device=dev), plan, co)
    torch.cuda.synchronize()
    assert np.allclose(full.cpu().numpy(), pl["lat"][:, 2], rtol=1e-12, atol=0)


def test_overflow_second_pass_tiled():
    """The tiny first-pass pool at K = 128 (tiled DP) with the slow 1.1B draft
    (multi-segment envelopes): identical results through the worst-case pass."""
    pd = scengen.params("1.1B-7B", K=128, gamma_min=1, gamma_max=8, c1_draft=4 * 4.11e-13)
    _, sc, _ = scengen.config("C4", 0, 300)
    a = gpu_solve(pd, sc)
    b = gpu_solve(dict(pd, flags=1), sc)
    for k in a:
        if a[k] is not None:
            assert np.array_equal(a[k], b[k]), k
    idx = np.arange(0, 300, 60)
    sub = {k: (v[idx] if v is not None else None) for k, v in sc.items()}
    compare(pd, sc, a, oracle.solve_batch(pd, sub), 0, oracle, idx=idx)


# ---------------------------------------------------------------- per-batch gamma (NEXT-3)
@pytest.mark.parametrize("cfg,pair,n", [("C3", "68M-7B", 300), ("C3", "1.1B-7B", 300), ("C2", None, 3),
                                        ("C4", "1.1B-7B", 16), ("C1", "1.1B-13B", 200)])
def test_per_batch_gamma(cfg, pair, n):
    """SDEDGE_BATCH_PER_BATCH_GAMMA (an extension, PAPER.md:555 fixes one l) against
    the oracle's Algorithm 1 over (j, gamma) candidates: T, T_com, T_inf, every
    batch boundary and every batch's gamma; the plan re-evaluated by the oracle's
    literal active-set eq:time (orc_eval_plan_pbg) equals the GPU's T_inf."""
    pd, sc, _ = scengen.config(cfg, 0, n, pair=pair)
    pd = dict(pd, batching_policy=6, gamma_min=max(pd["gamma_min"], 1))
    orc = oracle.solve_batch(pd, sc)
    g = gpu_solve(pd, sc)
    res = compare(pd, sc, g, orc, 0, oracle, label=f"per-batch gamma {cfg} {pair}")
    assert res["failures"] == 0
    for s in range(0, n, max(1, n // 20)):
        M = int(g["M"][s])
        Is = sc["I"][s][g["order"][s]]
        co = None if sc.get("coeffs") is None else sc["coeffs"][s]
        v = oracle.eval_plan_pbg(pd, Is, float(sc["alpha"][s]), g["batch_end"][s][:M], g["batch_gamma"][s][:M],
                                 coeffs=co)
        assert abs(v - g["lat"][s, 2]) <= 1e-12 * v
        assert g["gamma"][s] == g["batch_gamma"][s][M - 1] and np.all(g["batch_gamma"][s][M:] == 0)


def test_actual_output_rejects_malformed_plans():
    """sdedge_evaluate_actual takes caller plans: malformed ones give NaN, never
    out-of-bounds reads (batch ends not increasing / beyond K / not ending at K,
    order entries outside 0..K-1)."""
    import paper_2510_11331_b200 as sd
    pd, sc, _ = scengen.config("C3", 0, 6)
    K = pd["K"]
    dev = "cuda:0"
    t = {k: torch.from_numpy(np.ascontiguousarray(sc[k])).to(dev) for k in ("I", "p", "g", "alpha")}
    plan = sd.solve(pd, t["I"], t["p"], t["g"], t["alpha"])
    O = torch.full((6, K), 100, dtype=torch.int32, device=dev)
    plan["batch_end"][1, plan["M"][1] - 1] = K + 5             # beyond K
    plan["M"][2] = 2
    plan["batch_end"][2, :2] = torch.tensor([5, 3], dtype=torch.int32)   # not increasing
    plan["M"][3] = 1
    plan["batch_end"][3, 0] = K - 1                            # does not end at K
    plan["order"][4, 7] = K                                    # order out of range
    act = sd.evaluate_actual(pd, t["I"], t["p"], t["g"], t["alpha"], O, plan).cpu().numpy()
    assert np.isfinite(act[0]) and np.isfinite(act[5])
    assert np.all(np.isnan(act[1:5]))
