"""Throughput of the exhaustive-search kernel (sdedge_brute_force, SURVEY 8(f)
NEXT-4 (i)) and of Algorithm 1 on the same scenarios, with the heuristic gap.

Work model: per batch-step (one batch of one plan at one
decoding step) 7 fp64 lane-ops: each stage time b (a + s (n-1)) + c as one
add and one FMA (the slope term s (n-1) is per step, not per batch), then
the C^d add, the max and the add of eq:time; the kernel counts the
batch-steps it evaluated.  Timed with CUDA events on the
launching stream after warm-up; the oracle's exhaustive search is timed on
a few scenarios on the host for context.

usage: python tools/bench_brute_force.py [--K 12] [--gmax 8] [--n 2000]"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_11331_b200 as sd  # noqa: E402
import scengen  # noqa: E402

OPS_PER_BATCH_STEP = 7
PEAK = 148 * 64 * 1.965e9   # fp64 lane-ops/s, DESIGN.md 7


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--K", type=int, default=12)
    ap.add_argument("--gmax", type=int, default=8)
    ap.add_argument("--n", type=int, default=2000)
    ap.add_argument("--pair", default="68M-7B")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--mem", type=float, default=0, help="Gamma_s in bytes (0 = Table default)")
    ap.add_argument("--oracle", type=int, default=4, help="scenarios timed on the CPU oracle (0 = skip)")
    a = ap.parse_args()
    pd = scengen.params(a.pair, K=a.K, gamma_min=1, gamma_max=a.gmax)
    if a.mem > 0:
        pd["mem_capacity_bytes"] = int(a.mem)
    sc = scengen.generate(21, a.K, 0, a.n)
    I = torch.from_numpy(sc["I"]).cuda()
    al = torch.from_numpy(sc["alpha"]).cuda()
    p = torch.from_numpy(sc["p"]).cuda()
    g = torch.from_numpy(sc["g"]).cuda()
    st = torch.cuda.current_stream()
    work = torch.zeros(5, dtype=torch.int64, device="cuda")
    sd.brute_force(pd, I, al)                       # warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(a.reps):
        o = sd.brute_force(pd, I, al, work_counters=work)
    e1.record(st)
    torch.cuda.synchronize()
    t_bf = e0.elapsed_time(e1) / 1e3 / a.reps
    w = work.cpu().numpy() // a.reps
    sd.solve(pd, I, p, g, al, want_w=False)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(a.reps):
        s1 = sd.solve(pd, I, p, g, al, want_w=False)
    e1.record(st)
    torch.cuda.synchronize()
    t_a1 = e0.elapsed_time(e1) / 1e3 / a.reps
    tb = o["t_inf"].cpu().numpy()
    t1 = s1["lat"][:, 2].cpu().numpy()
    ok = (o["status"].cpu().numpy() == 0) & (s1["status"].cpu().numpy() == 0)
    gap = (t1[ok] - tb[ok]) / tb[ok]
    ops = w[1] * OPS_PER_BATCH_STEP
    res = dict(kernel="bf_item_kernel", K=a.K, mem_capacity_bytes=pd["mem_capacity_bytes"], gamma=[1, a.gmax], pair=a.pair, n=a.n,
               bf_scenarios_per_s=a.n / t_bf, bf_ms=t_bf * 1e3, plans_per_launch=int(w[0]),
               batch_steps_per_launch=int(w[1]),
               roofline=dict(bound="alu", achieved=ops / t_bf / 1e12, peak=PEAK / 1e12,
                             unit="T fp64-lane-ops/s", frac=ops / t_bf / PEAK),
               alg1_scenarios_per_s=a.n / t_a1,
               heuristic_gap=dict(exact_frac=float(np.mean(gap <= 1e-12)), mean=float(gap.mean()),
                                  p99=float(np.quantile(gap, 0.99)), max=float(gap.max()),
                                  min=float(gap.min())))
    if a.oracle:
        import oracle
        t0 = time.perf_counter()
        for s in range(a.oracle):
            Is = sc["I"][s][np.argsort(sc["I"][s], kind="stable")]
            oracle.brute_force(pd, Is, float(sc["alpha"][s]), 1, a.gmax)
        res["oracle_bf_scenarios_per_s_1core"] = a.oracle / (time.perf_counter() - t0)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
