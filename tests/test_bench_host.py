"""Host-side pieces of bench.py (CPU): the clock summary of the timed region (B200_PROFILING.md clocks line)
keeps only samples inside the region, flags throttle reasons, and for a region shorter than the 20 ms sampling
period falls back to the samples within 50 ms of it, saying so."""
import bench


def _sampler(rows, t0, t1):
    c = bench.ClockSampler(None)
    c.rows = [[t] + r for t, r in rows]
    c.t0, c.t1 = t0, t1
    return c


OK = ["1965", "1965", "700", "Not Active", "Not Active", "Not Active", "Not Active"]
CAP = ["1800", "1965", "1000", "Not Active", "Not Active", "Not Active", "Active"]


def test_clock_summary_inside_region():
    c = _sampler([(0.5, CAP), (1.01, OK), (1.02, OK), (1.03, CAP), (2.0, CAP)], 1.0, 1.05)
    out = c.summary()
    assert out["samples"] == 3 and out["sm_max_mhz"] == 1965.0 and out["sm_mhz"] == 1965.0
    assert out["reasons"] == ["sw_power_cap"] and "note" not in out


def test_clock_summary_short_region_uses_neighbours():
    c = _sampler([(0.9, CAP), (1.012, OK), (1.2, CAP)], 1.000, 1.005)
    out = c.summary()
    assert out["samples"] == 1 and out["reasons"] == [] and "note" in out


def test_clock_summary_unsampled():
    c = _sampler([(0.1, OK)], 1.0, 1.005)
    assert c.summary()["reasons"] == ["unsampled"]
