"""-m "not gpu": the parity harness itself (tests/parity.py) -- the near-tie
branching replay accepts a schedule that Algorithm 1 reaches by taking a
near-best candidate at a near tie, and rejects schedules that no branch
reaches, wrong latencies and differing schedules at non-tied scenarios.
"GPU" outputs are synthesised from the oracle's own forced chains
(orc_dp_trace), so no GPU is needed."""
import numpy as np

import scengen
from tests.parity import compare


def _as_gpu(res, K):
    """Oracle results reshaped like gpu_solve's output (trace filled by the tests)."""
    g = {k: np.array(v, copy=True) for k, v in res.items() if k in
         ("status", "gamma", "M", "lat", "order", "batch_end", "w")}
    g["trace"] = np.zeros((len(g["status"]), K), np.int32)
    return g


def _solve(orc_mod, pd, sc):
    r = orc_mod.solve_batch(pd, sc, nthreads=2)
    return r


def test_replay_accepts_a_tied_branch_and_rejects_others(orc):
    # all coefficients zero: every candidate of every row costs exactly 0 -> every row is an exact tie
    pd = scengen.params("68M-7B", K=6, gamma_min=1, gamma_max=1, c1_draft=0.0, c2_draft=0.0,
                        c1_verify=0.0, c2_verify=0.0, O_max=16)
    sc = scengen.generate(71, 6, 0, 2)
    r = _solve(orc, pd, sc)
    assert np.all(r["min_row_gap"] == 0.0)
    g = _as_gpu(r, pd["K"])
    # the oracle's own choices (largest j on ties: every task its own batch), as a trace
    Is = sc["I"][0][r["order"][0]]
    t, S, *_ = orc.dp_trace(pd, Is, float(sc["alpha"][0]), 1)
    g["trace"][0] = S
    g["trace"][1] = orc.dp_trace(pd, sc["I"][1][r["order"][1]], float(sc["alpha"][1]), 1)[1]
    assert compare(pd, sc, g, r, 0, orc, label='harness self-test (failures expected)')["exact"] == 0           # all exempt, identical
    # another branch: every row takes j = 1 (one batch) -- also cost 0, so a valid near-tie branch
    g["trace"][0] = np.ones(6, np.int32)
    g["batch_end"][0] = [6, 0, 0, 0, 0, 0]
    g["M"][0] = 1
    res = compare(pd, sc, g, r, 0, orc, label='harness self-test (failures expected)')
    assert res["replayed"] == 1 and res["failures"] == 0
    # a trace that does not backtrack to the reported plan is rejected
    g["trace"][0] = np.arange(1, 7, dtype=np.int32)
    try:
        compare(pd, sc, g, r, 0, orc, label='harness self-test (failures expected)')
        raise AssertionError("inconsistent trace accepted")
    except AssertionError as e:
        assert "does not backtrack" in str(e)


def test_replay_rejects_a_worse_branch_and_wrong_latency(orc):
    pd = scengen.params("1.1B-7B", K=5, gamma_min=1, gamma_max=3, O_max=128)
    sc = scengen.generate(72, 5, 0, 4)
    r = _solve(orc, pd, sc)
    s = int(np.argmax(r["min_row_gap"]))                          # the least tied scenario
    assert r["min_row_gap"][s] > 1e-6
    g = _as_gpu(r, pd["K"])
    # a schedule that differs where there is no near tie: rejected outright
    M = int(r["M"][s])
    alt = [5] if M > 1 else [1, 5]
    g["batch_end"][s] = alt + [0] * (5 - len(alt))
    g["M"][s] = len(alt)
    try:
        compare(pd, sc, g, r, 0, orc, label='harness self-test (failures expected)')
        raise AssertionError("differing schedule at a non-tie accepted")
    except AssertionError as e:
        assert "schedule differs" in str(e)
    # the right schedule with a latency off by 1e-9 relative: rejected at fp64's 1e-12
    g = _as_gpu(r, pd["K"])
    g["lat"][s, 2] *= 1 + 1e-9
    try:
        compare(pd, sc, g, r, 0, orc, label='harness self-test (failures expected)')
        raise AssertionError("latency error accepted")
    except AssertionError as e:
        assert "latency rel err" in str(e)
    # ... but accepted by the fp32 tolerance (1e-5)
    assert compare(pd, sc, g, r, 1, orc, label='harness self-test fp32')["failures"] == 0
