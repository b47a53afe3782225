import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build()
    return oracle


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    """Exact / exempt / replayed counts of every parity comparison of the session
    (shown even under -q)."""
    try:
        from tests.parity import STATS
    except Exception:
        return
    if not STATS:
        return
    tr = terminalreporter
    tr.section("parity counts (exact | exempt, identical | near-tie replayed | failures)")
    tot = [0, 0, 0, 0, 0]
    for label, r in STATS:
        tr.write_line(f"{label:60s} n={r['n']:6d} exact={r['exact']:6d} exempt_same={r['exempt_same']:4d} "
                      f"replayed={r['replayed']:4d} failures={r['failures']} worst_rel={r['worst_rel']:.2e}")
        if "self-test" in label:         # injected faults of the harness's own tests: not parity results
            continue
        for q, k in enumerate(("n", "exact", "exempt_same", "replayed", "failures")):
            tot[q] += r[k]
    tr.write_line(f"{'TOTAL (without the harness self-tests)':60s} n={tot[0]:6d} exact={tot[1]:6d} exempt_same={tot[2]:4d} replayed={tot[3]:4d} "
                  f"failures={tot[4]}")
