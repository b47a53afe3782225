#!/usr/bin/env python
"""Paper-context numbers on the B200 solver.

Runs the proposed policy and the paper's baselines (Sec. IV) through the CUDA
solver on seeded synthetic scenarios with the paper's parameters (Tables I/II,
K = 100, alpha = 0.8, l_max = 10) and reports the mean latency reduction of the
proposed scheme, next to the figure the paper prints.  Latency = T_com +
T_inf, with T_inf both as planned (uniform O_max) and evaluated with the tasks'
actual output lengths O_k ~ U{1..O_max} (sdedge_evaluate_actual).  The paper's
seeds and plotted data are not available, so only the trend is comparable.

    python tools/paper_context.py [--n 2000] > profiles/rNN_paper_context.json
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2510_11331_b200 as sd  # noqa: E402
import scengen  # noqa: E402

PROPOSED, NO_PIPE, NONE, STATIC, MAX, HEUR = range(6)


def run(pd, sc, O, pol=PROPOSED, bw=0, gmin=1, gmax=10):
    d = "cuda:0"
    t = {k: torch.from_numpy(np.ascontiguousarray(sc[k])).to(d) for k in ("I", "p", "g", "alpha")}
    p = dict(pd, batching_policy=pol, bandwidth_policy=bw, gamma_min=gmin, gamma_max=gmax, static_batch=4)
    out = sd.solve(p, t["I"], t["p"], t["g"], t["alpha"])
    act = sd.evaluate_actual(p, t["I"], t["p"], t["g"], t["alpha"], torch.from_numpy(O).to(d), out)
    torch.cuda.synchronize()
    lat = out["lat"].cpu().numpy()
    ok = out["status"].cpu().numpy() == 0
    return dict(planned=lat[ok, 0], actual=lat[ok, 1] + act.cpu().numpy()[ok], gamma=out["gamma"].cpu().numpy()[ok])


def reduction(a, b):
    """Mean relative latency reduction of a (proposed) vs b (baseline)."""
    return float(np.mean((b - a) / b))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2000)
    args = ap.parse_args()
    sd.lib()
    n, res = args.n, {}

    def scen(K, I_max=512, O_max=2048, root=101, g0=1e-3):
        sc = scengen.generate(root, K, 0, n, I_max=I_max, g0=g0)
        sc["alpha"][:] = 0.8                                  # alpha = 0.8 in every quoted figure
        return sc, scengen.output_lengths(root, K, 0, n, O_max)

    # Fig. bandw: proposed vs uniform bandwidth, K = 100, B_w = 25 MHz
    for pair, paper in (("68M-7B", 44.9), ("1.1B-7B", 29.3), ("1.1B-13B", 25.2)):
        pd = scengen.params(pair, K=100, bandwidth_hz=25e6)
        sc, O = scen(100)
        a, b = run(pd, sc, O), run(pd, sc, O, bw=1)
        res[f"vs_uniform_bandwidth_{pair}"] = dict(paper_pct=paper, planned_pct=100 * reduction(a["planned"], b["planned"]),
                                                  actual_pct=100 * reduction(a["actual"], b["actual"]))
    # sensitivity to reading R2 (g0 = "-30 dBm"): read as 1e-6 instead of 1e-3
    for pair, paper in (("68M-7B", 44.9), ("1.1B-7B", 29.3), ("1.1B-13B", 25.2)):
        pd = scengen.params(pair, K=100, bandwidth_hz=25e6)
        sc, O = scen(100, g0=1e-6)
        a, b = run(pd, sc, O), run(pd, sc, O, bw=1)
        res[f"vs_uniform_bandwidth_{pair}_g0_1e-6"] = dict(paper_pct=paper,
                                                          planned_pct=100 * reduction(a["planned"], b["planned"]),
                                                          actual_pct=100 * reduction(a["actual"], b["actual"]))
    # Fig. serving_comparison: vs SD w/o pipeline, (1.1B,7B), I_max = 512 / O_max = 1792
    for name, kw, paper in (("I_max512", dict(I_max=512), 31.6), ("O_max1792", dict(O_max=1792), 30.7)):
        pd = scengen.params("1.1B-7B", K=100, O_max=kw.get("O_max", 2048))
        sc, O = scen(100, **kw)
        a, b = run(pd, sc, O), run(pd, sc, O, pol=NO_PIPE)
        res[f"vs_sd_without_pipeline_{name}"] = dict(paper_pct=paper,
                                                     planned_pct=100 * reduction(a["planned"], b["planned"]),
                                                     actual_pct=100 * reduction(a["actual"], b["actual"]))
    # Fig. batching_comparison: vs max batching at K = 90; vs heuristic batching
    pd = scengen.params("1.1B-7B", K=90)
    sc, O = scen(90)
    a, b = run(pd, sc, O), run(pd, sc, O, pol=MAX)
    res["vs_max_batching_K90"] = dict(paper_pct=21.4, planned_pct=100 * reduction(a["planned"], b["planned"]),
                                      actual_pct=100 * reduction(a["actual"], b["actual"]))
    for name, kw, paper in (("I_max1792", dict(I_max=1792), 19.6), ("O_max1024", dict(O_max=1024), 20.5)):
        pd = scengen.params("1.1B-7B", K=100, O_max=kw.get("O_max", 2048))
        sc, O = scen(100, **kw)
        a, b = run(pd, sc, O), run(pd, sc, O, pol=HEUR)
        res[f"vs_heuristic_batching_{name}"] = dict(paper_pct=paper,
                                                    planned_pct=100 * reduction(a["planned"], b["planned"]),
                                                    actual_pct=100 * reduction(a["actual"], b["actual"]))
    # Other baselines of Sec. IV-A (no printed percentage): no batching, FSL (l = 7), ADS core (gamma = 0)
    pd = scengen.params("1.1B-7B", K=100)
    sc, O = scen(100)
    a = run(pd, sc, O)
    for name, kw in (("no_batching", dict(pol=NONE)), ("fixed_speculation_length_7", dict(gmin=7, gmax=7)),
                     ("autoregressive_gamma0", dict(gmin=0, gmax=0)), ("static_batching_4", dict(pol=STATIC))):
        b = run(pd, sc, O, **kw)
        res[f"vs_{name}"] = dict(paper_pct=None, planned_pct=100 * reduction(a["planned"], b["planned"]),
                                 actual_pct=100 * reduction(a["actual"], b["actual"]))
    res["gamma_star_histogram_1.1B-7B_K100"] = {int(k): int(v) for k, v in zip(*np.unique(a["gamma"], return_counts=True))}
    res["scenarios_per_setting"] = n
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
