"""-m "not gpu": the stored oracle results of the large-config parity samples
(tests/data/oracle_*.npz, written by tools/make_oracle_fixtures.py, which calls
only oracle/) are current: their input fingerprint matches scengen, and a few
stored scenarios re-solved by the oracle now give identical results."""
import os

import numpy as np
import pytest

from tests.parity import load_fixture

DATA = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data")
NAMES = ["c4_68M-7B", "c4_1.1B-7B", "c5_256", "c5_512", "c5_1024"]


@pytest.mark.parametrize("name", NAMES)
def test_fixture_current(orc, name):
    pd, sc, idx, res = load_fixture(name)           # fingerprint checked inside
    assert len(idx) == len(res["status"]) and np.all(res["status"] == 0)
    K = pd["K"]
    for a in range(len(idx)):
        M = int(res["M"][a])
        be = res["batch_end"][a]
        assert 1 <= M <= K and be[M - 1] == K and np.all(np.diff(be[:M]) > 0) and np.all(be[M:] == 0)
        assert sorted(res["order"][a]) == list(range(K))
        assert res["lat"][a, 0] == res["lat"][a, 1] + res["lat"][a, 2]
    if name.startswith("c4"):                        # re-solve two stored scenarios (~2 s each)
        for a in (0, len(idx) - 1):
            sub = {k: (v[a:a + 1] if v is not None else None) for k, v in sc.items()}
            r = orc.solve_batch(pd, sub, nthreads=1)
            for k in ("status", "gamma", "M", "lat", "order", "batch_end", "w", "min_row_gap", "gamma_gap", "W"):
                assert np.array_equal(r[k][0], res[k][a]), (name, a, k)
