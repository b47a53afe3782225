"""ctypes wrapper around the plain-C oracle (oracle/sdedge_oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.  It does not
import, and is not imported by, the product package paper_2510_11331_b200.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "sdedge_oracle.c")
LIB = os.path.join(HERE, "libsdedge_oracle.so")
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-std=gnu11", "-fPIC", "-shared",
          "-pthread", "-Wall"]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no FMA contraction, no fast-math)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(
            os.path.getmtime(SRC), os.path.getmtime(os.path.join(HERE, "sdedge_oracle.h"))):
        subprocess.check_call(["gcc", *CFLAGS, "-o", LIB, SRC, "-lm"])
    return LIB


class Params(C.Structure):
    _fields_ = [("Jd", C.c_int32), ("h1d", C.c_int32), ("h2d", C.c_int32),
                ("Jv", C.c_int32), ("h1v", C.c_int32), ("h2v", C.c_int32),
                ("c1d", C.c_double), ("c2d", C.c_double), ("c1v", C.c_double), ("c2v", C.c_double),
                ("Bw", C.c_double), ("sigma2", C.c_double), ("lambda_", C.c_double),
                ("gamma_s", C.c_int64), ("K", C.c_int32), ("O_max", C.c_int32),
                ("gamma_min", C.c_int32), ("gamma_max", C.c_int32), ("downlink_s", C.c_double),
                ("bw_policy", C.c_int32), ("batch_policy", C.c_int32), ("static_batch", C.c_int32),
                ("heuristic_start", C.c_int32)]


class Result(C.Structure):
    _fields_ = [("status", C.c_int32), ("gamma", C.c_int32), ("M", C.c_int32),
                ("T", C.c_double), ("T_com", C.c_double), ("T_inf", C.c_double),
                ("min_row_gap", C.c_double), ("gap_gamma", C.c_int32), ("gap_row", C.c_int32),
                ("gamma_gap", C.c_double), ("W", C.c_int64)]


_lib = None
P_i32 = C.POINTER(C.c_int32)
P_f64 = C.POINTER(C.c_double)
P_i64 = C.POINTER(C.c_int64)


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        L.orc_expected_tokens.restype = C.c_double
        L.orc_expected_tokens.argtypes = [C.c_double, C.c_int]
        L.orc_decode_steps.restype = C.c_int32
        L.orc_decode_steps.argtypes = [C.c_int32, C.c_double]
        L.orc_param_memory.restype = C.c_int64
        L.orc_param_memory.argtypes = [C.c_int32] * 3
        L.orc_kv_memory_per_task.restype = C.c_int64
        L.orc_kv_memory_per_task.argtypes = [C.c_int32] * 4
        L.orc_flops_draft.restype = C.c_double
        L.orc_flops_draft.argtypes = [C.c_int32] * 3 + [C.c_double, C.c_double, C.c_int, C.c_int]
        L.orc_flops_verify.restype = C.c_double
        L.orc_flops_verify.argtypes = [C.c_int32] * 3 + [C.c_double, C.c_int, C.c_double, C.c_int]
        L.orc_runtime.restype = C.c_double
        L.orc_runtime.argtypes = [C.c_double] * 4
        for f in (L.orc_draft_time, L.orc_verify_time):
            f.restype = C.c_double
            f.argtypes = [C.POINTER(Params), P_f64, C.c_int, C.c_int32, C.c_int, C.c_double, C.c_int]
        L.orc_bandwidth.restype = C.c_double
        L.orc_bandwidth.argtypes = [C.POINTER(Params), P_i32, P_f64, P_f64, P_f64]
        L.orc_eval_plan.restype = C.c_double
        L.orc_eval_plan.argtypes = [C.POINTER(Params), P_f64, P_i32, C.c_double, C.c_int, C.c_int, P_i32]
        L.orc_dp.restype = C.c_double
        L.orc_dp.argtypes = [C.POINTER(Params), P_f64, P_i32, C.c_double, C.c_int, P_i32, P_f64,
                             P_i64, C.c_int, C.c_int]
        L.orc_dp_trace.restype = C.c_double
        L.orc_dp_trace.argtypes = [C.POINTER(Params), P_f64, P_i32, C.c_double, C.c_int, P_i32, P_i32, P_f64,
                                   P_f64, P_f64, P_i64]
        L.orc_eval_plan_nopipe.restype = C.c_double
        L.orc_eval_plan_nopipe.argtypes = [C.POINTER(Params), P_f64, P_i32, C.c_double, C.c_int, C.c_int, P_i32]
        L.orc_dp_nopipe.restype = C.c_double
        L.orc_dp_nopipe.argtypes = [C.POINTER(Params), P_f64, P_i32, C.c_double, C.c_int, P_i32, P_f64, P_i64]
        L.orc_fixed_plan.restype = C.c_int
        L.orc_fixed_plan.argtypes = [C.POINTER(Params), P_f64, P_i32, C.c_double, C.c_int, P_i32]
        L.orc_eval_actual.restype = C.c_double
        L.orc_eval_actual.argtypes = [C.POINTER(Params), P_f64, P_i32, P_i32, C.c_double, C.c_int, C.c_int, P_i32]
        L.orc_solve.restype = None
        L.orc_solve.argtypes = [C.POINTER(Params), P_i32, P_f64, P_f64, C.c_double, P_f64,
                                C.POINTER(Result), P_i32, P_i32, P_f64, P_f64, P_i32]
        L.orc_eval_plan_pbg.restype = C.c_double
        L.orc_eval_plan_pbg.argtypes = [C.POINTER(Params), P_f64, P_i32, C.c_double, C.c_int, P_i32, P_i32]
        L.orc_dp_pbg.restype = C.c_double
        L.orc_dp_pbg.argtypes = [C.POINTER(Params), P_f64, P_i32, C.c_double, P_i32, P_i32, P_f64, P_i64]
        L.orc_brute_force.restype = C.c_double
        L.orc_brute_force.argtypes = [C.POINTER(Params), P_f64, P_i32, C.c_double, C.c_int, C.c_int,
                                      P_i32, P_i32, P_i32]
        L.orc_solve_batch.restype = None
        L.orc_solve_batch.argtypes = [C.POINTER(Params), C.c_int64, P_i32, P_f64, P_f64, P_f64, P_f64,
                                      P_i32, P_i32, P_i32, P_f64, P_i32, P_i32, P_f64, P_f64, P_f64,
                                      P_i64, P_i32, C.c_int]
    return _lib


def make_params(d: dict) -> Params:
    """Marshal a scengen.params() dict into the oracle's own struct."""
    Jd, h1d, h2d = d["draft"]
    Jv, h1v, h2v = d["verify"]
    return Params(Jd, h1d, h2d, Jv, h1v, h2v, d["c1_draft"], d["c2_draft"], d["c1_verify"],
                  d["c2_verify"], d["bandwidth_hz"], d["noise_w"], d.get("lambda_bits", 0.0),
                  int(d["mem_capacity_bytes"]), d["K"], d["O_max"], d["gamma_min"], d["gamma_max"],
                  d.get("downlink_s", 0.0), d.get("bandwidth_policy", 0), d.get("batching_policy", 0),
                  d.get("static_batch", 4), d.get("heuristic_start", 0))


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t)) if a is not None else None


def _co(co):
    if co is None:
        return None
    co = np.ascontiguousarray(co, dtype=np.float64)
    return co


# ---------------------------------------------------------------- primitives
def expected_tokens(alpha, gamma):
    return lib().orc_expected_tokens(alpha, gamma)


def decode_steps(O, L):
    return lib().orc_decode_steps(O, L)


def param_memory(J, h1, h2):
    return lib().orc_param_memory(J, h1, h2)


def kv_memory_per_task(J, h1, I, O):
    return lib().orc_kv_memory_per_task(J, h1, I, O)


def flops_draft(model, Im, L, i, n):
    return lib().orc_flops_draft(*model, float(Im), float(L), i, n)


def flops_verify(model, Im, gamma, L, n):
    return lib().orc_flops_verify(*model, float(Im), gamma, float(L), n)


def runtime(c1, c2, F, b):
    return lib().orc_runtime(c1, c2, F, float(b))


def draft_time(pd, b, Im, gamma, L, n, coeffs=None):
    P = make_params(pd)
    co = _co(coeffs)
    return lib().orc_draft_time(C.byref(P), _p(co, C.c_double), b, Im, gamma, L, n)


def verify_time(pd, b, Im, gamma, L, n, coeffs=None):
    P = make_params(pd)
    co = _co(coeffs)
    return lib().orc_verify_time(C.byref(P), _p(co, C.c_double), b, Im, gamma, L, n)


def bandwidth(pd, I, p, g):
    P = make_params(dict(pd, K=len(I)))
    I = np.ascontiguousarray(I, dtype=np.int32)
    p = np.ascontiguousarray(p, dtype=np.float64)
    g = np.ascontiguousarray(g, dtype=np.float64)
    w = np.empty(len(I))
    t = lib().orc_bandwidth(C.byref(P), _p(I, C.c_int32), _p(p, C.c_double), _p(g, C.c_double),
                            _p(w, C.c_double))
    return t, w


def eval_plan(pd, Is, alpha, gamma, batch_end, coeffs=None):
    P = make_params(dict(pd, K=len(Is)))
    Is = np.ascontiguousarray(Is, dtype=np.int32)
    be = np.ascontiguousarray(batch_end, dtype=np.int32)
    co = _co(coeffs)
    return lib().orc_eval_plan(C.byref(P), _p(co, C.c_double), _p(Is, C.c_int32), alpha, gamma,
                               len(be), _p(be, C.c_int32))


def dp(pd, Is, alpha, gamma, coeffs=None, force_row=0, force_j=0):
    """Algorithm 1 for one gamma; returns (T_inf, S, row_gap, W)."""
    P = make_params(dict(pd, K=len(Is)))
    Is = np.ascontiguousarray(Is, dtype=np.int32)
    S = np.zeros(len(Is), np.int32)
    gap = np.full(len(Is), np.inf)
    W = C.c_int64(0)
    co = _co(coeffs)
    t = lib().orc_dp(C.byref(P), _p(co, C.c_double), _p(Is, C.c_int32), alpha, gamma,
                     _p(S, C.c_int32), _p(gap, C.c_double), C.byref(W), force_row, force_j)
    return t, S, gap, W.value


def dp_trace(pd, Is, alpha, gamma, force=None, coeffs=None):
    """Algorithm 1 for one gamma with row i taking j = force[i-1] where that is
    > 0 (near-tie branching replay, SURVEY 8(c) "T"); returns
    (T_inf, S, row_gap, row_best, row_taken, W)."""
    K = len(Is)
    P = make_params(dict(pd, K=K))
    Is = np.ascontiguousarray(Is, dtype=np.int32)
    f = None if force is None else np.ascontiguousarray(force, dtype=np.int32)
    S = np.zeros(K, np.int32)
    gap = np.full(K, np.inf)
    rb = np.full(K, np.nan)
    rt = np.full(K, np.nan)
    W = C.c_int64(0)
    co = _co(coeffs)
    t = lib().orc_dp_trace(C.byref(P), _p(co, C.c_double), _p(Is, C.c_int32), alpha, gamma, _p(f, C.c_int32),
                           _p(S, C.c_int32), _p(gap, C.c_double), _p(rb, C.c_double), _p(rt, C.c_double),
                           C.byref(W))
    return t, S, gap, rb, rt, W.value


def eval_plan_pbg(pd, Is, alpha, batch_end, gammas, coeffs=None):
    """Planned T_inf of a plan with a speculation length per batch (NEXT-3 extension)."""
    P = make_params(dict(pd, K=len(Is)))
    Is = np.ascontiguousarray(Is, dtype=np.int32)
    be = np.ascontiguousarray(batch_end, dtype=np.int32)
    gm = np.ascontiguousarray(gammas, dtype=np.int32)
    co = _co(coeffs)
    return lib().orc_eval_plan_pbg(C.byref(P), _p(co, C.c_double), _p(Is, C.c_int32), alpha, len(be),
                                   _p(be, C.c_int32), _p(gm, C.c_int32))


def dp_pbg(pd, Is, alpha, coeffs=None):
    """Algorithm 1 over (j, gamma) candidates; returns (T_inf, S, Gm, row_gap, W)."""
    K = len(Is)
    P = make_params(dict(pd, K=K))
    Is = np.ascontiguousarray(Is, dtype=np.int32)
    S = np.zeros(K, np.int32)
    Gm = np.zeros(K, np.int32)
    gap = np.full(K, np.inf)
    W = C.c_int64(0)
    co = _co(coeffs)
    t = lib().orc_dp_pbg(C.byref(P), _p(co, C.c_double), _p(Is, C.c_int32), alpha, _p(S, C.c_int32),
                         _p(Gm, C.c_int32), _p(gap, C.c_double), C.byref(W))
    return t, S, Gm, gap, W.value


def eval_plan_nopipe(pd, Is, alpha, gamma, batch_end, coeffs=None):
    P = make_params(dict(pd, K=len(Is)))
    Is = np.ascontiguousarray(Is, dtype=np.int32)
    be = np.ascontiguousarray(batch_end, dtype=np.int32)
    co = _co(coeffs)
    return lib().orc_eval_plan_nopipe(C.byref(P), _p(co, C.c_double), _p(Is, C.c_int32), alpha, gamma,
                                      len(be), _p(be, C.c_int32))


def eval_actual(pd, Is, Os, alpha, gamma, batch_end, coeffs=None):
    """Actual-output evaluation of a plan (Is, Os in sorted order)."""
    P = make_params(dict(pd, K=len(Is)))
    Is = np.ascontiguousarray(Is, dtype=np.int32)
    Os = np.ascontiguousarray(Os, dtype=np.int32)
    be = np.ascontiguousarray(batch_end, dtype=np.int32)
    co = _co(coeffs)
    return lib().orc_eval_actual(C.byref(P), _p(co, C.c_double), _p(Is, C.c_int32), _p(Os, C.c_int32), alpha,
                                 gamma, len(be), _p(be, C.c_int32))


def dp_nopipe(pd, Is, alpha, gamma, coeffs=None):
    P = make_params(dict(pd, K=len(Is)))
    Is = np.ascontiguousarray(Is, dtype=np.int32)
    S = np.zeros(len(Is), np.int32)
    gap = np.full(len(Is), np.inf)
    W = C.c_int64(0)
    co = _co(coeffs)
    t = lib().orc_dp_nopipe(C.byref(P), _p(co, C.c_double), _p(Is, C.c_int32), alpha, gamma,
                            _p(S, C.c_int32), _p(gap, C.c_double), C.byref(W))
    return t, S, gap, W.value


def fixed_plan(pd, Is, alpha, gamma, coeffs=None):
    P = make_params(dict(pd, K=len(Is)))
    Is = np.ascontiguousarray(Is, dtype=np.int32)
    ends = np.zeros(len(Is) + 1, np.int32)
    co = _co(coeffs)
    M = lib().orc_fixed_plan(C.byref(P), _p(co, C.c_double), _p(Is, C.c_int32), alpha, gamma, _p(ends, C.c_int32))
    return [int(x) for x in ends[:M]]


def backtrack(S):
    """Batch ends from a boundary vector S (reading A5)."""
    out, i = [], len(S)
    while i > 0:
        out.append(i)
        i = int(S[i - 1]) - 1
    return out[::-1]


def solve(pd, I, p, g, alpha, coeffs=None):
    K = len(I)
    P = make_params(dict(pd, K=K))
    I = np.ascontiguousarray(I, dtype=np.int32)
    p = np.ascontiguousarray(p, dtype=np.float64)
    g = np.ascontiguousarray(g, dtype=np.float64)
    co = _co(coeffs)
    R = Result()
    order = np.zeros(K, np.int32)
    be = np.zeros(K, np.int32)
    w = np.zeros(K)
    tg = np.zeros(pd["gamma_max"] - pd["gamma_min"] + 1)
    bg = np.zeros(K, np.int32)
    lib().orc_solve(C.byref(P), _p(I, C.c_int32), _p(p, C.c_double), _p(g, C.c_double), alpha,
                    _p(co, C.c_double), C.byref(R), _p(order, C.c_int32), _p(be, C.c_int32),
                    _p(w, C.c_double), _p(tg, C.c_double), _p(bg, C.c_int32))
    return dict(status=R.status, gamma=R.gamma, M=R.M, T=R.T, T_com=R.T_com, T_inf=R.T_inf,
                min_row_gap=R.min_row_gap, gap_gamma=R.gap_gamma, gap_row=R.gap_row,
                gamma_gap=R.gamma_gap, W=R.W, order=order, batch_end=be, w=w, tinf_gamma=tg,
                batch_gamma=bg)


def brute_force(pd, Is, alpha, gamma_min, gamma_max, coeffs=None):
    K = len(Is)
    P = make_params(dict(pd, K=K))
    Is = np.ascontiguousarray(Is, dtype=np.int32)
    co = _co(coeffs)
    bg, bm = C.c_int32(0), C.c_int32(0)
    ends = np.zeros(32, np.int32)
    t = lib().orc_brute_force(C.byref(P), _p(co, C.c_double), _p(Is, C.c_int32), alpha,
                              gamma_min, gamma_max, C.byref(bg), C.byref(bm), _p(ends, C.c_int32))
    return t, bg.value, list(ends[:bm.value])


def solve_batch(pd, sc, nthreads=None):
    """Solve every scenario of a scengen dict; returns SoA numpy results."""
    I = np.ascontiguousarray(sc["I"], dtype=np.int32)
    n, K = I.shape
    P = make_params(dict(pd, K=K))
    p = np.ascontiguousarray(sc["p"], dtype=np.float64)
    g = np.ascontiguousarray(sc["g"], dtype=np.float64)
    al = np.ascontiguousarray(sc["alpha"], dtype=np.float64)
    co = _co(sc.get("coeffs"))
    out = dict(status=np.zeros(n, np.int32), gamma=np.zeros(n, np.int32), M=np.zeros(n, np.int32),
               lat=np.zeros((n, 3)), order=np.zeros((n, K), np.int32),
               batch_end=np.zeros((n, K), np.int32), w=np.zeros((n, K)),
               min_row_gap=np.zeros(n), gamma_gap=np.zeros(n), W=np.zeros(n, np.int64),
               batch_gamma=np.zeros((n, K), np.int32))
    nthreads = nthreads or os.cpu_count() or 1
    lib().orc_solve_batch(C.byref(P), n, _p(I, C.c_int32), _p(p, C.c_double), _p(g, C.c_double),
                          _p(al, C.c_double), _p(co, C.c_double), _p(out["status"], C.c_int32),
                          _p(out["gamma"], C.c_int32), _p(out["M"], C.c_int32),
                          _p(out["lat"], C.c_double), _p(out["order"], C.c_int32),
                          _p(out["batch_end"], C.c_int32), _p(out["w"], C.c_double),
                          _p(out["min_row_gap"], C.c_double), _p(out["gamma_gap"], C.c_double),
                          _p(out["W"], C.c_int64), _p(out["batch_gamma"], C.c_int32), nthreads)
    out["nthreads"] = nthreads
    return out
