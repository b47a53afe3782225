import os, sys, numpy as np
sys.path.insert(0, "/root/repo")
import scengen, oracle
from tests.parity import gpu_solve
pd, sc, _ = scengen.config("C2", 0, 3)
for s in range(3):
    for g in range(1, 9):
        p = dict(pd, gamma_min=g, gamma_max=g)
        sub = {k: (v[s:s+1] if v is not None else None) for k, v in sc.items()}
        out = gpu_solve(p, sub)
        r = oracle.solve(p, sc["I"][s], sc["p"][s], sc["g"][s], sc["alpha"][s], coeffs=sc["coeffs"][s])
        ok = abs(out["lat"][0][2] - r["T_inf"]) <= 1e-12 * r["T_inf"]
        if not ok:
            print("s", s, "gamma", g, "gpu", out["lat"][0][2], "orc", r["T_inf"], "M", out["M"][0], r["M"])
            print("  gpu ends", list(out["batch_end"][0][:out["M"][0]]))
            print("  orc ends", list(r["batch_end"][:r["M"]]))
print("done")
