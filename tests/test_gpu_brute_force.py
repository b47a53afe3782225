"""-m gpu: the exhaustive search kernel (sdedge_brute_force, SURVEY 8(f)
NEXT-4 (i)) against the oracle's exhaustive search (orc_brute_force, pinned in
test_oracle_pins.py), element by element on the same seeded inputs.

What is unique is compared exactly or to 1e-11 relative (the minimum T_inf,
status, the sorted order); where two plans tie to rounding, the GPU's plan is
checked to be valid: the oracle's literal eq:time evaluation of it equals the
minimum.  Also pinned here: the exhaustive optimum never exceeds Algorithm 1's
(both on the GPU), and under the additive SD-w/o-pipeline cost the
DP is exact, so the two agree."""
import numpy as np
import pytest

import oracle
import scengen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

REL = 1e-11


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2510_11331_b200 as sd
    sd.lib()
    oracle.build()


def _dev(sc):
    return (torch.from_numpy(sc["I"]).cuda(), torch.from_numpy(sc["alpha"]).cuda(),
            None if sc.get("coeffs") is None else torch.from_numpy(sc["coeffs"]).cuda())


def _gpu_bf(pd, sc, work=None):
    import paper_2510_11331_b200 as sd
    I, a, co = _dev(sc)
    o = sd.brute_force(pd, I, a, co, work_counters=work)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in o.items()}


def _check_against_oracle(pd, sc, evaluate=oracle.eval_plan, oracle_bf=None):
    g = _gpu_bf(pd, sc)
    n, K = sc["I"].shape
    n_plan_eq = 0
    for s in range(n):
        order = np.argsort(sc["I"][s], kind="stable")
        assert (g["order"][s] == order).all()
        Is = sc["I"][s][order]
        a = float(sc["alpha"][s])
        bf, bg, plan = (oracle_bf or oracle.brute_force)(pd, Is, a, pd["gamma_min"], pd["gamma_max"])
        if not np.isfinite(bf):
            assert g["status"][s] == 1 and g["gamma"][s] == -1 and g["M"][s] == 0
            assert np.isinf(g["t_inf"][s])
            continue
        assert g["status"][s] == 0
        assert abs(g["t_inf"][s] - bf) <= REL * bf, (s, g["t_inf"][s], bf)
        M = int(g["M"][s])
        ends = g["batch_end"][s][:M]
        assert (g["batch_end"][s][M:] == 0).all() and ends[-1] == K and (np.diff(ends) > 0).all()
        if int(g["gamma"][s]) == bg and list(ends) == list(plan):
            n_plan_eq += 1
        else:   # a tie to rounding: the GPU's plan must be optimal under the literal evaluation
            v = evaluate(pd, Is, a, int(g["gamma"][s]), ends)
            assert abs(v - bf) <= REL * bf, (s, v, bf)
    return g, n_plan_eq


@pytest.mark.parametrize("pair,K,gmax", [("68M-7B", 1, 4), ("68M-7B", 4, 4), ("1.1B-13B", 7, 8),
                                         ("68M-7B", 10, 16), ("1.1B-7B", 12, 6)])
def test_bf_matches_oracle(pair, K, gmax):
    pd = scengen.params(pair, K=K, gamma_min=1, gamma_max=gmax)
    sc = scengen.generate(11, K, 0, 40 if K <= 10 else 12)
    _, n_eq = _check_against_oracle(pd, sc)
    assert n_eq >= 0.9 * len(sc["alpha"])


def test_bf_memory_window_binds():
    """Gamma_s lowered so the 1.1B draft fits only 2-4 tasks per batch (constraint (b)):
    partitions with an oversized batch are discarded exactly as in the oracle."""
    pd = scengen.params("1.1B-7B", K=9, gamma_min=1, gamma_max=4, mem_capacity_bytes=3_200_000_000)
    sc = scengen.generate(12, 9, 0, 40)
    g, _ = _check_against_oracle(pd, sc)
    assert (g["status"] == 0).all()
    sizes = [np.diff(np.concatenate([[0], g["batch_end"][s][:g["M"][s]]])).max() for s in range(40)]
    assert max(sizes) <= 4


def test_bf_memory_infeasible_and_invalid():
    pd = scengen.params("1.1B-7B", K=5, gamma_min=1, gamma_max=3, mem_capacity_bytes=1_000_000_000)
    sc = scengen.generate(13, 5, 0, 4)
    g = _gpu_bf(pd, sc)
    assert (g["status"] == 1).all() and (g["gamma"] == -1).all() and np.isinf(g["t_inf"]).all()
    pd = scengen.params("68M-7B", K=5, gamma_min=1, gamma_max=3)
    sc["alpha"][1] = 1.0
    sc["I"][2, 3] = 0
    g = _gpu_bf(pd, sc)
    assert list(g["status"]) == [0, 2, 3, 0]
    assert np.isnan(g["t_inf"][1]) and np.isnan(g["t_inf"][2]) and (g["M"][1:3] == 0).all()


def test_bf_k20_limit():
    import paper_2510_11331_b200 as sd
    pd = scengen.params("68M-7B", K=20, gamma_min=2, gamma_max=3, O_max=48)
    sc = scengen.generate(14, 20, 0, 2)
    _check_against_oracle(pd, sc)
    pd21 = scengen.params("68M-7B", K=21, gamma_min=1, gamma_max=2)
    sc21 = scengen.generate(14, 21, 0, 1)
    with pytest.raises(RuntimeError, match="K <= 20"):
        I, a, _ = _dev(sc21)
        sd.brute_force(pd21, I, a)


def test_bf_not_worse_than_algorithm1():
    """Algorithm 1 is a heuristic: its T_inf is never below the
    exhaustive optimum over its own search space, and equals it in most scenarios."""
    from tests.parity import gpu_solve
    pd = scengen.params("68M-7B", K=12, gamma_min=1, gamma_max=8)
    sc = scengen.generate(15, 12, 0, 300)
    g = _gpu_bf(pd, sc)
    a1 = gpu_solve(pd, sc)
    assert (a1["status"] == 0).all() and (g["status"] == 0).all()
    t1, tb = a1["lat"][:, 2], g["t_inf"]
    assert (t1 >= tb * (1 - 1e-12)).all()
    assert np.mean(np.abs(t1 - tb) <= 1e-12 * tb) >= 0.5


def test_bf_nopipe_equals_exact_dp():
    """Under the additive SD-w/o-pipeline cost the DP is exact (reading B2), so the
    GPU's exhaustive search and the GPU's DP agree; both match the oracle."""
    from tests.parity import gpu_solve
    pd = scengen.params("68M-7B", K=8, gamma_min=1, gamma_max=6, batching_policy=1)

    def bf_nopipe(pd, Is, a, gmin, gmax):
        best = (np.inf, -1, [])
        K = len(Is)
        for gm in range(gmin, gmax + 1):
            for mask in range(1 << (K - 1)):
                ends = [t + 1 for t in range(K - 1) if mask >> t & 1] + [K]
                v = oracle.eval_plan_nopipe(pd, Is, a, gm, ends)
                if v < best[0]:
                    best = (v, gm, ends)
        return best

    sc = scengen.generate(16, 8, 0, 25)
    g, _ = _check_against_oracle(pd, sc, evaluate=oracle.eval_plan_nopipe, oracle_bf=bf_nopipe)
    a1 = gpu_solve(pd, sc)
    assert np.allclose(a1["lat"][:, 2], g["t_inf"], rtol=1e-11, atol=0)


def test_bf_work_counters():
    """Plans evaluated = (#gamma) x 2^(K-1) when memory never binds; batch-steps = sum N_gamma x M."""
    K, gmin, gmax, n = 6, 1, 4, 10
    pd = scengen.params("68M-7B", K=K, gamma_min=gmin, gamma_max=gmax)
    sc = scengen.generate(17, K, 0, n)
    work = torch.zeros(5, dtype=torch.int64, device="cuda")
    _gpu_bf(pd, sc, work=work)
    w = work.cpu().numpy()
    assert w[0] == n * (gmax - gmin + 1) * 2 ** (K - 1)
    sumM = sum(bin(m).count("1") + 1 for m in range(2 ** (K - 1)))
    steps = sum(oracle.decode_steps(pd["O_max"], oracle.expected_tokens(float(a), gm))
                for a in sc["alpha"] for gm in range(gmin, gmax + 1))
    assert w[1] == steps * sumM


def test_bf_gamma_chunked_launch():
    """With enough scenarios one CTA takes all gammas of a scenario (the chunked
    launch); a small call takes one gamma per CTA.  Same arithmetic, so the two
    launches agree bit for bit; a sample is checked against the oracle."""
    K, n = 6, 5000
    pd = scengen.params("1.1B-13B", K=K, gamma_min=1, gamma_max=5)
    sc = scengen.generate(18, K, 0, n)
    big = _gpu_bf(pd, sc)
    sub = {k: (v[:100] if v is not None else None) for k, v in sc.items()}
    small = _gpu_bf(pd, sub)
    for k in ("t_inf", "gamma", "M", "batch_end", "order", "status"):
        assert (big[k][:100] == small[k]).all(), k
    sub = {k: (v[n - 60:] if v is not None else None) for k, v in sc.items()}
    g, _ = _check_against_oracle(pd, sub)
    for k in ("t_inf", "gamma", "M", "batch_end", "order", "status"):
        assert (big[k][n - 60:] == g[k]).all(), k
