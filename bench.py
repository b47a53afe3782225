#!/usr/bin/env python
"""Benchmark: scenarios solved per second (fp64) by the sm_100a solver.

Workload (BASELINE.json configs[3]): 1e6 independent
scenarios per GPU, K = 128 tasks, gamma 1..16, (LLaMA-68M, LLaMA-7B),
alpha ~ U[0.5, 0.9), Rayleigh channels -- synthetic, seeded (scengen).
One step = one sdedge_solve_batch over the rank's whole shard (every row of
SURVEY 8(a): staging, sort, bandwidth, per-gamma DP, gamma argmin,
backtrack).  Inputs (2.6 GB) exceed the 126 MB L2, so no flush is needed.

    python bench.py [--gpus N --steps K --warmup W] [--algo envelope|dense]
                    [--precision fp64|fp32] [--impl reference]
Under torchrun (N > 1) each rank solves its own 1e6-scenario shard (weak
scaling, no data-path collective); times are max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import scengen  # noqa: E402

# Nominal FP64 pipe peak of B200 derived from the unit counts and clock
# (B200_PROFILING.md: 148 SMs, clocks.max.sm 1965 MHz; 64 FP64 lanes/SM/clk):
# one FP64 instruction lane-op (DFMA counted once) per lane per clock.
FP64_LANES_PER_SM = 64
FP32_LANES_PER_SM = 128

# Algorithmic FP64 operations:
#  dense    4 per candidate-step (n >= 2): Td fma, +Upsilon0 (folded), max, accumulate
#           -> SURVEY 8(d): 4 W;  plus the per-candidate constant terms.
#  envelope per fully evaluated candidate 16 (stage-time constants, n = 1 term,
#           verify closed form, compare), per (candidate, predecessor segment) 10
#           (two end values, sign tests, trapezoid sum, accumulate), per pruned
#           candidate 3 (the lower bound: add, FMA, compare), per DP row 40.
OPS = {"dense": dict(cand=16, seg=0, step=4, row=40, pruned=0),
       "envelope": dict(cand=16, seg=10, step=0, row=40, pruned=3)}

# DRAM bytes (read + write) per scenario of the envelope kernel from the one
# `ncu --set full` capture of round 1 (profiles/r01_ncu_envelope_final_c4.md:
# 0.29 GB read + 0.91 GB written for a 1e5-scenario C4 launch), scaled to the
# launch.  The algorithmic bytes are 2568 in + 2084 out per scenario; the rest
# is the write-back of the tiled DP's global row store.
NCU_DRAM_BYTES_PER_SCENARIO = {("C4", "envelope", "fp64"): (0.29304576e9 + 0.912838656e9) / 1e5}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["cuda", "reference"], default="cuda")
    ap.add_argument("--algo", choices=["envelope", "dense"], default="envelope")
    ap.add_argument("--precision", choices=["fp64", "fp32"], default="fp64")
    ap.add_argument("--config", default="C4")
    ap.add_argument("--pair", default=None)
    ap.add_argument("--n", type=int, default=None, help="scenarios per rank (default: the config's)")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=None)
    return ap.parse_args()


def shard(rank: int, n_per_rank: int):
    """Weak scaling: rank r owns scenarios [r n, (r+1) n) of the counter-based stream."""
    return rank * n_per_rank, (rank + 1) * n_per_rank


def max_over_ranks(x: float, dist, device) -> float:
    """Max of a per-rank time over all ranks (the multi-GPU timing rule)."""
    import torch
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the
    timed region (B200_PROFILING.md clocks line)."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, uuid):
        self.uuid, self.rows, self.proc = uuid, [], None

    def __enter__(self):
        try:
            cmd = ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "50"]
            if self.uuid:
                cmd += ["-i", self.uuid]
            self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[q] for r in self.rows for q in range(4) if r[3 + q] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor()


def oracle_rate(pd, sc, nthreads):
    """Time the C oracle (as it stands) on a bounded sample; scenarios/s."""
    import oracle  # test infrastructure: only the cpu_baseline / reference legs use it
    oracle.build()
    t0 = time.perf_counter()
    oracle.solve_batch(pd, sc, nthreads=nthreads)
    return len(sc["alpha"]) / (time.perf_counter() - t0), time.perf_counter() - t0


def config_of(args, n_rank, ws):
    name = {"C4": "c4_1e6xK128_gamma1-16", "C3": "c3_1e5xK32_gamma1-8"}.get(args.config, args.config)
    return {"workload": name, "scenarios_per_gpu": n_rank, "total_scenarios": n_rank * ws,
            "K": None, "gamma": None, "pair": None, "algo": args.algo, "precision": args.precision,
            "l2": "no flush: inputs per step exceed the 126 MB L2",
            "parallelism": f"scenario-shard x{ws}"}


def run_reference(args):
    """--impl reference: the oracle, as it stands, timed on host cores (rank 0)."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    pd, _, n_total = scengen.config(args.config, 0, 1, pair=args.pair)
    cores = os.cpu_count() or 1
    per_step = args.cpu_sample or cores
    rates, times = [], []
    for st in range(args.warmup + args.steps):
        _, sc, _ = scengen.config(args.config, st * per_step, (st + 1) * per_step, pair=args.pair)
        r, t = oracle_rate(pd, sc, cores)
        if st >= args.warmup:
            rates.append(r)
            times.append(t)
    value = per_step * len(times) / sum(times)
    cfg = config_of(args, n_total, ws)
    cfg.update(K=pd["K"], gamma=[pd["gamma_min"], pd["gamma_max"]],
               pair=f"{scengen_pair(pd)}")
    line = {"impl": "reference", "metric": "scenarios solved/sec (fp64)", "value": value,
            "unit": "scenarios/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * float(np.mean(times)), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg,
            "cpu_baseline": {"value": value, "unit": "scenarios/s", "cores": cores, "kind": "oracle",
                             "cpu": cpu_model(),
                             "sample": f"{per_step} scenarios of {args.config} per step "
                                       f"(consecutive indices), {cores} threads"},
            "e2e": {"value": value, "unit": "scenarios/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def scengen_pair(pd):
    inv = {v: k for k, v in scengen.MODELS.items()}
    return f"{inv[tuple(pd['draft'])]}-{inv[tuple(pd['verify'])]}"


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist
    import paper_2510_11331_b200 as sd

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        # NCCL may print its version banner on stdout when the communicator is
        # created; keep stdout for the single JSON line.
        sys.stdout.flush()
        saved = os.dup(1)
        os.dup2(2, 1)
        try:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            dist.barrier()
        finally:
            sys.stdout.flush()
            os.dup2(saved, 1)
            os.close(saved)
    dev = torch.device("cuda", local)
    sd.lib()

    pd, _, n_total = scengen.config(args.config, 0, 1, pair=args.pair)
    n = args.n or n_total
    s0, _ = shard(rank, n)                                  # weak scaling: own shard per rank
    t_gen = time.perf_counter()
    _, sc, _ = scengen.config(args.config, s0, s0 + n, pair=args.pair)
    t_gen = time.perf_counter() - t_gen
    K = pd["K"]
    prec = 0 if args.precision == "fp64" else 1
    algo = sd.ALGO_ENVELOPE if args.algo == "envelope" else sd.ALGO_DENSE

    host = {k: torch.from_numpy(np.ascontiguousarray(sc[k])).pin_memory() for k in ("I", "p", "g", "alpha")}
    d = {k: v.to(dev, non_blocking=True) for k, v in host.items()}
    stream = torch.cuda.current_stream(dev)
    work = torch.zeros(5, dtype=torch.int64, device=dev)
    out = sd._alloc_out(torch, n, K, dev, True)

    def step(count=False):
        sd.solve(pd, d["I"], d["p"], d["g"], d["alpha"], None, out=out, stream=stream, precision=prec,
                 algo=algo, work_counters=work if count else None)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches_per_step = sd.sdedge_last_launch_count()

    uuid = None
    try:
        uuid = str(torch.cuda.get_device_properties(dev).uuid)
        uuid = uuid if uuid.startswith("GPU-") else "GPU-" + uuid
    except Exception:
        pass
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    work.zero_()
    with ClockSampler(uuid) as clk:
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            step(count=True)
        e1.record(stream)
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
    el = e0.elapsed_time(e1) * 1e-3
    el_max = max_over_ranks(el, dist, dev)
    wk = work.cpu().numpy().astype(np.float64) / args.steps    # per step (= per main launch)
    status_ok = int((out["status"] == 0).sum().item())

    # ---- end to end through the host entry point (pinned host in, pinned host out)
    e2e = None
    if not args.no_e2e:
        hout = sd._alloc_out(torch, n, K, None, True, pin=True)
        ksteps = args.e2e_steps or max(1, min(args.steps, 3))
        sd.solve_host(pd, host["I"], host["p"], host["g"], host["alpha"], out=hout, stream=stream,
                      precision=prec, algo=algo)
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        h0 = time.perf_counter()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(ksteps):
            sd.solve_host(pd, host["I"], host["p"], host["g"], host["alpha"], out=hout, stream=stream,
                          precision=prec, algo=algo)
        f1.record(stream)
        torch.cuda.synchronize()
        te = max_over_ranks(f0.elapsed_time(f1) * 1e-3, dist, dev)
        h2d = sum(v.numel() * v.element_size() for v in host.values())
        d2h = sum(v.numel() * v.element_size() for v in hout.values() if v is not None)
        e2e = {"value": n * ws * ksteps / te, "unit": "scenarios/s", "h2d_bytes_per_step": h2d * ws,
               "d2h_bytes_per_step": d2h * ws, "steps": ksteps, "entry": "sdedge_solve_batch_host"}

    # ---- roofline of the dominant kernel (solve_kernel<.., BIG=0>; the second
    # launch is the worst-case-pool pass, empty unless an envelope overflowed)
    props = torch.cuda.get_device_properties(dev)
    nsm = props.multi_processor_count
    lanes = FP64_LANES_PER_SM if prec == 0 else FP32_LANES_PER_SM
    peak = nsm * lanes * 1965e6
    o = OPS[args.algo]
    ops = (o["cand"] * wk[4] + o["seg"] * wk[1] + o["step"] * wk[2] + o["row"] * wk[3]
           + o["pruned"] * (wk[0] - wk[4]))
    t_launch = el / args.steps
    achieved = ops / t_launch
    clocks = clk.summary()

    if rank == 0:
        cpu = None
        if ws == 1 and not args.no_cpu_baseline:
            cores = os.cpu_count() or 1
            m = args.cpu_sample or 3 * cores   # ~15 s of oracle work on the box
            try:
                r, tt = oracle_rate(pd, {k: (v[:m] if v is not None else None) for k, v in sc.items()}, cores)
                cpu = {"value": r, "unit": "scenarios/s", "cores": cores, "kind": "oracle", "cpu": cpu_model(),
                       "sample": f"first {m} scenarios of the rank-0 shard ({tt:.1f} s, {cores} threads)"}
            except Exception as e:  # pragma: no cover
                cpu = {"value": None, "unit": "scenarios/s", "cores": cores, "kind": "oracle",
                       "sample": f"failed: {e}"}
        cfg = config_of(args, n, ws)
        cfg.update(K=K, gamma=[pd["gamma_min"], pd["gamma_max"]], pair=scengen_pair(pd))
        line = {
            "metric": "scenarios solved/sec (fp64)" if prec == 0 else "scenarios solved/sec (fp32 variant)",
            "value": n * ws / (el_max / args.steps),
            "unit": "scenarios/s",
            "n_gpus": ws,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": 1e3 * el_max / args.steps,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64" if prec == 0 else "f32",
            "data": "synthetic",
            "config": cfg,
            "roofline": {"bound": "alu", "achieved": achieved / 1e12, "peak": peak / 1e12,
                         "unit": "T fp64-lane-ops/s" if prec == 0 else "T fp32-lane-ops/s",
                         "frac": achieved / peak,
                         "traffic": (NCU_DRAM_BYTES_PER_SCENARIO[(args.config, args.algo, args.precision)] * n
                                     if (args.config, args.algo, args.precision) in NCU_DRAM_BYTES_PER_SCENARIO
                                     else None),
                         "traffic_unit": "DRAM bytes per launch (r01 ncu capture, per-scenario scaled)",
                         "algorithmic_bytes": (20 * K + 8 + 36 + 16 * K) * n,
                         "peak_source": f"derived: {nsm} SMs x {lanes} lanes x 1965 MHz (B200_PROFILING.md)",
                         "work_per_launch": {"candidates": wk[0], "full_evaluations": wk[4],
                                             "cand_segments": wk[1], "candidate_steps_W": wk[2],
                                             "rows": wk[3], "ops": ops},
                         "kernel": "solve_kernel (main pass)"},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
            "status_ok": status_ok,
            "gen_s": t_gen,
        }
        print(json.dumps(line))
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
