"""Thin Python binding of the sm_100a solver library (include/sdedge.h).

Argument marshalling only: every step of the solve runs inside
libsdedge.so's CUDA kernels.  PyTorch provides device memory and streams.
There is no CPU fallback: if the library is missing, import-time loading
raises.
"""
from __future__ import annotations

import ctypes as C
import os

from ._build import LIB, build  # noqa: F401

__all__ = ["sdedge_solve_batch", "sdedge_solve_batch_host", "sdedge_solve_batch_host_compact", "solve_host_compact", "sdedge_evaluate_actual", "evaluate_actual", "sdedge_brute_force", "brute_force", "sdedge_pipe_peak", "sdedge_last_error",
           "sdedge_last_launch_count", "sdedge_abi_version", "solve", "solve_host", "make_params",
           "ALGO_ENVELOPE", "ALGO_DENSE", "EXPORTED_SYMBOLS", "lib"]

ALGO_ENVELOPE, ALGO_DENSE = 0, 1
BW_OPTIMAL, BW_UNIFORM = 0, 1
BATCH_PROPOSED, BATCH_NO_PIPELINE, BATCH_NONE, BATCH_STATIC, BATCH_MAX, BATCH_HEURISTIC, BATCH_PER_BATCH_GAMMA = range(7)
FLAG_TINY_POOL, FLAG_HEURISTIC_HALF = 1, 2
EXPORTED_SYMBOLS = ("sdedge_solve_batch", "sdedge_solve_batch_host", "sdedge_solve_batch_host_compact",
                    "sdedge_evaluate_actual",
                    "sdedge_brute_force", "sdedge_last_launch_count", "sdedge_last_error",
                    "sdedge_abi_version", "sdedge_pipe_peak", "sdedge_ipc_export", "sdedge_ipc_open",
                    "sdedge_ipc_close", "sdedge_kernel_timing", "sdedge_kernel_times", "sdedge_copy_async")


class SdedgeCompactSchedule(C.Structure):
    _fields_ = [("gamma", C.c_void_p), ("num_batches", C.c_void_p), ("batch_end_mask", C.c_void_p),
                ("order", C.c_void_p), ("bw_share", C.c_void_p), ("status", C.c_void_p)]


class SdedgeModel(C.Structure):
    _fields_ = [("layers", C.c_int32), ("hidden", C.c_int32), ("ffn", C.c_int32)]


class SdedgeParams(C.Structure):
    _fields_ = [("draft", SdedgeModel), ("verify", SdedgeModel),
                ("c1_draft", C.c_double), ("c2_draft", C.c_double),
                ("c1_verify", C.c_double), ("c2_verify", C.c_double),
                ("bandwidth_hz", C.c_double), ("noise_w", C.c_double), ("lambda_bits", C.c_double),
                ("mem_capacity_bytes", C.c_int64), ("K", C.c_int32), ("O_max", C.c_int32),
                ("gamma_min", C.c_int32), ("gamma_max", C.c_int32), ("precision", C.c_int32),
                ("algo", C.c_int32), ("flags", C.c_int32), ("downlink_s", C.c_double),
                ("stream", C.c_void_p), ("bandwidth_policy", C.c_int32), ("batching_policy", C.c_int32),
                ("static_batch", C.c_int32), ("reserved", C.c_int32)]


class SdedgeScenarios(C.Structure):
    _fields_ = [("input_len", C.c_void_p), ("tx_power_w", C.c_void_p), ("gain", C.c_void_p),
                ("alpha", C.c_void_p), ("coeffs", C.c_void_p)]


class SdedgeSchedule(C.Structure):
    _fields_ = [("gamma", C.c_void_p), ("num_batches", C.c_void_p), ("batch_end", C.c_void_p),
                ("order", C.c_void_p), ("bw_share", C.c_void_p), ("status", C.c_void_p),
                ("work_counters", C.c_void_p), ("row_choice", C.c_void_p), ("batch_gamma", C.c_void_p)]


_lib = None


def lib() -> C.CDLL:
    """Load libsdedge.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise RuntimeError(f"{LIB} is missing: run __graft_entry__.build() "
                               "(there is no CPU fallback)")
        L = C.CDLL(LIB)
        for f in ("sdedge_solve_batch", "sdedge_solve_batch_host"):
            fn = getattr(L, f)
            fn.restype = C.c_int
            fn.argtypes = [C.POINTER(SdedgeScenarios), C.c_int64, C.POINTER(SdedgeParams), C.c_void_p,
                           C.POINTER(SdedgeSchedule)]
        L.sdedge_solve_batch_host_compact.restype = C.c_int
        L.sdedge_solve_batch_host_compact.argtypes = [C.POINTER(SdedgeScenarios), C.c_int64, C.POINTER(SdedgeParams),
                                                      C.c_void_p, C.POINTER(SdedgeCompactSchedule)]
        L.sdedge_evaluate_actual.restype = C.c_int
        L.sdedge_evaluate_actual.argtypes = [C.POINTER(SdedgeScenarios), C.c_void_p, C.c_int64,
                                             C.POINTER(SdedgeParams), C.POINTER(SdedgeSchedule), C.c_void_p]
        L.sdedge_brute_force.restype = C.c_int
        L.sdedge_brute_force.argtypes = [C.POINTER(SdedgeScenarios), C.c_int64, C.POINTER(SdedgeParams),
                                         C.c_void_p, C.POINTER(SdedgeSchedule)]
        L.sdedge_last_error.restype = C.c_char_p
        L.sdedge_last_launch_count.restype = C.c_int
        L.sdedge_abi_version.restype = C.c_int
        L.sdedge_ipc_export.restype = C.c_int
        L.sdedge_ipc_export.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64)]
        L.sdedge_ipc_open.restype = C.c_int
        L.sdedge_ipc_open.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_void_p)]
        L.sdedge_copy_async.restype = C.c_int
        L.sdedge_copy_async.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]
        L.sdedge_ipc_close.restype = C.c_int
        L.sdedge_ipc_close.argtypes = [C.c_void_p, C.c_uint64]
        L.sdedge_kernel_timing.restype = C.c_int
        L.sdedge_kernel_timing.argtypes = [C.c_int32]
        L.sdedge_kernel_times.restype = C.c_int
        L.sdedge_kernel_times.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_int32)]
        L.sdedge_pipe_peak.restype = C.c_int
        L.sdedge_pipe_peak.argtypes = [C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        _lib = L
    return _lib


def sdedge_last_error() -> str:
    return lib().sdedge_last_error().decode()


def sdedge_last_launch_count() -> int:
    return lib().sdedge_last_launch_count()


def sdedge_abi_version() -> int:
    return lib().sdedge_abi_version()


def make_params(d: dict, stream=None, precision: int | None = None, algo: int | None = None) -> SdedgeParams:
    """Marshal a parameter dict (scengen.params() layout) into sdedge_params."""
    st = 0
    if stream is not None:
        st = stream if isinstance(stream, int) else int(stream.cuda_stream)
    return SdedgeParams(SdedgeModel(*d["draft"]), SdedgeModel(*d["verify"]),
                        d["c1_draft"], d["c2_draft"], d["c1_verify"], d["c2_verify"],
                        d["bandwidth_hz"], d["noise_w"], d.get("lambda_bits", 0.0),
                        int(d["mem_capacity_bytes"]), d["K"], d["O_max"], d["gamma_min"], d["gamma_max"],
                        d.get("precision", 0) if precision is None else precision,
                        d.get("algo", ALGO_ENVELOPE) if algo is None else algo,
                        d.get("flags", 0) | (FLAG_HEURISTIC_HALF if d.get("heuristic_start", 0) else 0),
                        d.get("downlink_s", 0.0), st, d.get("bandwidth_policy", 0),
                        d.get("batching_policy", 0), d.get("static_batch", 4), 0)


def _ptr(t):
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return t.ctypes.data  # numpy (host entry point)


def _check(name, t, dtype, shape, device):
    """Marshalling guard: the C ABI takes raw pointers, so a wrong dtype, a
    non-contiguous view, a wrong device or shape would be read as garbage."""
    if t is None:
        return
    import torch
    if t.dtype != dtype or not t.is_contiguous() or tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: need a contiguous {dtype} tensor of shape {tuple(shape)}, "
                         f"got {t.dtype} {tuple(t.shape)} contiguous={t.is_contiguous()}")
    if device == "host" and t.is_cuda:
        raise ValueError(f"{name}: the host entry point takes host (pinned) tensors")
    if isinstance(device, torch.device) and t.device != device:
        raise ValueError(f"{name}: on {t.device}, expected {device}")


def _check_inputs(I, p, g, alpha, coeffs, device):
    import torch
    if I.dim() != 2:
        raise ValueError("I: need a [n, K] int32 tensor")
    n, K = I.shape
    _check("I", I, torch.int32, (n, K), device)
    _check("p", p, torch.float64, (n, K), device)
    _check("g", g, torch.float64, (n, K), device)
    _check("alpha", alpha, torch.float64, (n,), device)
    _check("coeffs", coeffs, torch.float64, (n, 4), device)
    return n, K


def _call(fn, I, p, g, alpha, coeffs, n, P, lat, gamma, M, bend, order, w, status, work=None, trace=None,
          bgam=None):
    sc = SdedgeScenarios(_ptr(I), _ptr(p), _ptr(g), _ptr(alpha), _ptr(coeffs))
    sch = SdedgeSchedule(_ptr(gamma), _ptr(M), _ptr(bend), _ptr(order), _ptr(w), _ptr(status), _ptr(work),
                         _ptr(trace), _ptr(bgam))
    rc = fn(C.byref(sc), n, C.byref(P), _ptr(lat), C.byref(sch))
    if rc != 0:
        raise RuntimeError(f"sdedge_solve_batch failed ({rc}): {sdedge_last_error()}")
    return rc


def sdedge_solve_batch(I, p, g, alpha, coeffs, n, params: SdedgeParams, out_latency, gamma, num_batches,
                       batch_end, order, bw_share, status, work_counters=None, row_choice=None, batch_gamma=None):
    """Direct C-ABI call on DEVICE tensors (all contiguous, see include/sdedge.h)."""
    return _call(lib().sdedge_solve_batch, I, p, g, alpha, coeffs, n, params, out_latency, gamma,
                 num_batches, batch_end, order, bw_share, status, work_counters, row_choice, batch_gamma)


def sdedge_solve_batch_host(I, p, g, alpha, coeffs, n, params: SdedgeParams, out_latency, gamma,
                            num_batches, batch_end, order, bw_share, status):
    """Direct C-ABI call on HOST buffers (numpy or pinned torch CPU tensors)."""
    return _call(lib().sdedge_solve_batch_host, I, p, g, alpha, coeffs, n, params, out_latency, gamma,
                 num_batches, batch_end, order, bw_share, status)


def sdedge_solve_batch_host_compact(I, p, g, alpha, coeffs, n, params: SdedgeParams, out_latency, gamma,
                                    num_batches, batch_end_mask, order, bw_share, status):
    """Direct C-ABI call on HOST buffers with the compact schedule layout (include/sdedge.h)."""
    sc = SdedgeScenarios(_ptr(I), _ptr(p), _ptr(g), _ptr(alpha), _ptr(coeffs))
    sch = SdedgeCompactSchedule(_ptr(gamma), _ptr(num_batches), _ptr(batch_end_mask), _ptr(order), _ptr(bw_share),
                                _ptr(status))
    rc = lib().sdedge_solve_batch_host_compact(C.byref(sc), n, C.byref(params), _ptr(out_latency), C.byref(sch))
    if rc != 0:
        raise RuntimeError(f"sdedge_solve_batch_host_compact failed ({rc}): {sdedge_last_error()}")
    return rc


def sdedge_evaluate_actual(I, p, g, alpha, coeffs, output_len, n, params: SdedgeParams, gamma, num_batches,
                           batch_end, order, status, out_t_inf):
    """Direct C-ABI call (DEVICE tensors): actual-output T_inf of solved plans."""
    sc = SdedgeScenarios(_ptr(I), _ptr(p), _ptr(g), _ptr(alpha), _ptr(coeffs))
    sch = SdedgeSchedule(_ptr(gamma), _ptr(num_batches), _ptr(batch_end), _ptr(order), None, _ptr(status), None)
    rc = lib().sdedge_evaluate_actual(C.byref(sc), _ptr(output_len), n, C.byref(params), C.byref(sch),
                                      _ptr(out_t_inf))
    if rc != 0:
        raise RuntimeError(f"sdedge_evaluate_actual failed ({rc}): {sdedge_last_error()}")
    return rc


def evaluate_actual(params: dict, I, p, g, alpha, output_len, plan: dict, coeffs=None, stream=None):
    """Actual-output T_inf [n] (CUDA tensor) of the plans in `plan` (solve() output)."""
    import torch
    n, K = _check_inputs(I, p, g, alpha, coeffs, I.device)
    _check("output_len", output_len, torch.int32, (n, K), I.device)
    if stream is None:
        stream = torch.cuda.current_stream(I.device)
    P = make_params(dict(params, K=K), stream=stream)
    out = torch.empty(n, dtype=torch.float64, device=I.device)
    sdedge_evaluate_actual(I, p, g, alpha, coeffs, output_len, n, P, plan["gamma"], plan["M"], plan["batch_end"],
                           plan["order"], plan["status"], out)
    return out


def sdedge_brute_force(I, alpha, coeffs, n, params: SdedgeParams, out_t_inf, gamma, num_batches, batch_end,
                       order, status, work_counters=None):
    """Direct C-ABI call (DEVICE tensors): exhaustive search over contiguous plans and gamma (K <= 20)."""
    sc = SdedgeScenarios(_ptr(I), None, None, _ptr(alpha), _ptr(coeffs))
    sch = SdedgeSchedule(_ptr(gamma), _ptr(num_batches), _ptr(batch_end), _ptr(order), None, _ptr(status),
                         _ptr(work_counters))
    rc = lib().sdedge_brute_force(C.byref(sc), n, C.byref(params), _ptr(out_t_inf), C.byref(sch))
    if rc != 0:
        raise RuntimeError(f"sdedge_brute_force failed ({rc}): {sdedge_last_error()}")
    return rc


def brute_force(params: dict, I, alpha, coeffs=None, stream=None, work_counters=None) -> dict:
    """Exact optimum over every contiguous plan and gamma for CUDA-resident
    scenarios (K <= 20); returns CUDA tensors t_inf, gamma, M, batch_end, order, status."""
    import torch
    n, K = I.shape
    _check("I", I, torch.int32, (n, K), I.device)
    _check("alpha", alpha, torch.float64, (n,), I.device)
    _check("coeffs", coeffs, torch.float64, (n, 4), I.device)
    if stream is None:
        stream = torch.cuda.current_stream(I.device)
    P = make_params(dict(params, K=K), stream=stream)
    kw = dict(device=I.device)
    o = dict(t_inf=torch.empty(n, dtype=torch.float64, **kw), gamma=torch.empty(n, dtype=torch.int32, **kw),
             M=torch.empty(n, dtype=torch.int32, **kw), batch_end=torch.empty((n, K), dtype=torch.int32, **kw),
             order=torch.empty((n, K), dtype=torch.int32, **kw), status=torch.empty(n, dtype=torch.int32, **kw))
    sdedge_brute_force(I, alpha, coeffs, n, P, o["t_inf"], o["gamma"], o["M"], o["batch_end"], o["order"],
                       o["status"], work_counters)
    return o


def sdedge_kernel_timing(enable: bool) -> None:
    lib().sdedge_kernel_timing(1 if enable else 0)


def sdedge_kernel_times() -> dict:
    """Summed ms and launch counts per kernel kind since sdedge_kernel_timing(True)."""
    ms = (C.c_double * 4)()
    cnt = (C.c_int32 * 4)()
    rc = lib().sdedge_kernel_times(ms, cnt)
    if rc != 0:
        raise RuntimeError(f"sdedge_kernel_times failed ({rc}): {sdedge_last_error()}")
    names = ("prep", "main", "big", "other")
    return {names[k]: (ms[k], cnt[k]) for k in range(4)}


def sdedge_pipe_peak(fp32: bool = False):
    ops, el = C.c_double(0), C.c_double(0)
    rc = lib().sdedge_pipe_peak(1 if fp32 else 0, C.byref(ops), C.byref(el))
    if rc != 0:
        raise RuntimeError(f"sdedge_pipe_peak failed ({rc}): {sdedge_last_error()}")
    return ops.value, el.value


def ipc_export(t) -> tuple[bytes, int]:
    """(64-byte CUDA IPC handle of t's allocation, byte offset of t in it)."""
    h = (C.c_ubyte * 64)()
    off = C.c_uint64(0)
    rc = lib().sdedge_ipc_export(t.data_ptr(), h, C.byref(off))
    if rc != 0:
        raise RuntimeError(f"sdedge_ipc_export failed ({rc}): {sdedge_last_error()}")
    return bytes(h), off.value


def ipc_open(handle: bytes, offset: int) -> int:
    """Map a peer allocation exported by ipc_export; returns the device address."""
    h = (C.c_ubyte * 64).from_buffer_copy(handle)
    p = C.c_void_p(0)
    rc = lib().sdedge_ipc_open(h, offset, C.byref(p))
    if rc != 0:
        raise RuntimeError(f"sdedge_ipc_open failed ({rc}): {sdedge_last_error()}")
    return p.value


def copy_async(dst: int, src: int, nbytes: int, stream) -> None:
    """Device-to-device copy on `stream` (torch stream or raw handle); peer pointers allowed."""
    st = stream if isinstance(stream, int) else int(stream.cuda_stream)
    rc = lib().sdedge_copy_async(dst, src, nbytes, st)
    if rc != 0:
        raise RuntimeError(f"sdedge_copy_async failed ({rc}): {sdedge_last_error()}")


def ipc_close(ptr: int, offset: int) -> None:
    rc = lib().sdedge_ipc_close(ptr, offset)
    if rc != 0:
        raise RuntimeError(f"sdedge_ipc_close failed ({rc}): {sdedge_last_error()}")


class Rows:
    """Raw device address of row `row` of a row-major [n, width] array of
    `itemsize`-byte elements (peer-mapped output arrays carry no torch tensor)."""

    def __init__(self, base: int, width: int, itemsize: int, row: int = 0):
        self.addr = base + row * width * itemsize

    def data_ptr(self) -> int:
        return self.addr


def _alloc_out(torch, n, K, device, want_w, pin=False):
    kw = dict(device=device) if device is not None else dict(pin_memory=pin)
    return dict(lat=torch.empty((n, 3), dtype=torch.float64, **kw),
                gamma=torch.empty(n, dtype=torch.int32, **kw),
                M=torch.empty(n, dtype=torch.int32, **kw),
                batch_end=torch.empty((n, K), dtype=torch.int32, **kw),
                order=torch.empty((n, K), dtype=torch.int32, **kw),
                w=torch.empty((n, K), dtype=torch.float64, **kw) if want_w else None,
                status=torch.empty(n, dtype=torch.int32, **kw))


def solve(params: dict, I, p, g, alpha, coeffs=None, want_w: bool = True, stream=None, out=None,
          precision: int | None = None, algo: int | None = None, work_counters=None, trace: bool = False) -> dict:
    """Solve scenarios held in CUDA tensors; returns CUDA output tensors
    (enqueued on `stream`, default torch's current stream).  trace=True adds
    out["trace"]: the [n, K] int32 row choices S of gamma* (debug export)."""
    import torch
    n, K = _check_inputs(I, p, g, alpha, coeffs, I.device)
    dev = I.device
    if stream is None:
        stream = torch.cuda.current_stream(dev)
    P = make_params(dict(params, K=K), stream=stream, precision=precision, algo=algo)
    o = out if out is not None else _alloc_out(torch, n, K, dev, want_w)
    if trace and o.get("trace") is None:
        o["trace"] = torch.empty((n, K), dtype=torch.int32, device=dev)
    if params.get("batching_policy", 0) == BATCH_PER_BATCH_GAMMA and o.get("batch_gamma") is None:
        o["batch_gamma"] = torch.empty((n, K), dtype=torch.int32, device=dev)
    for k, v in o.items():
        if hasattr(v, "is_contiguous"):
            _check(f"out[{k}]", v, v.dtype, v.shape, dev)
    sdedge_solve_batch(I, p, g, alpha, coeffs, n, P, o["lat"], o["gamma"], o["M"], o["batch_end"],
                       o["order"], o["w"], o["status"], work_counters, o.get("trace"), o.get("batch_gamma"))
    return o


def alloc_out_compact(torch, n, K, want_w=True):
    """Pinned host outputs of sdedge_solve_batch_host_compact."""
    kw = dict(pin_memory=True)
    return dict(lat=torch.empty((n, 3), dtype=torch.float64, **kw), gamma=torch.empty(n, dtype=torch.int32, **kw),
                M=torch.empty(n, dtype=torch.int32, **kw),
                batch_end_mask=torch.empty((n, (K + 31) // 32), dtype=torch.int32, **kw),   # uint32 bits
                order=torch.empty((n, K), dtype=torch.int16, **kw),                         # uint16 values
                w=torch.empty((n, K), dtype=torch.float64, **kw) if want_w else None,
                status=torch.empty(n, dtype=torch.int32, **kw))


def unpack_compact(o) -> dict:
    """numpy views of a compact result: order as uint16 -> int32, batch_end rebuilt from the mask."""
    import numpy as np
    order = o["order"].numpy().view(np.uint16).astype(np.int32)
    mask = o["batch_end_mask"].numpy().view(np.uint32)
    n, W = mask.shape
    K = order.shape[1]
    bits = ((mask[:, :, None] >> np.arange(32, dtype=np.uint32)) & 1).reshape(n, W * 32)[:, :K].astype(bool)
    bend = np.zeros((n, K), np.int32)
    for s in range(n):
        e = np.nonzero(bits[s])[0] + 1
        bend[s, :len(e)] = e
    return dict(lat=o["lat"].numpy(), gamma=o["gamma"].numpy(), M=o["M"].numpy(), batch_end=bend, order=order,
                w=None if o["w"] is None else o["w"].numpy(), status=o["status"].numpy())


def solve_host_compact(params: dict, I, p, g, alpha, coeffs=None, want_w: bool = True, stream=None, out=None,
                       precision: int | None = None, algo: int | None = None) -> dict:
    """solve_host() with the compact output layout (uint16 order, batch-end bit mask): fewer bytes back over
    PCIe; unpack_compact() gives the solve_host() arrays."""
    import torch
    n, K = _check_inputs(I, p, g, alpha, coeffs, "host")
    if stream is None:
        stream = torch.cuda.current_stream()
    P = make_params(dict(params, K=K), stream=stream, precision=precision, algo=algo)
    o = out if out is not None else alloc_out_compact(torch, n, K, want_w)
    sdedge_solve_batch_host_compact(I, p, g, alpha, coeffs, n, P, o["lat"], o["gamma"], o["M"], o["batch_end_mask"],
                                    o["order"], o["w"], o["status"])
    return o


def solve_host(params: dict, I, p, g, alpha, coeffs=None, want_w: bool = True, stream=None, out=None,
               precision: int | None = None, algo: int | None = None) -> dict:
    """Solve scenarios held in (pinned) host tensors through the host entry
    point; the copies run on `stream` (caller synchronises before reading)."""
    import torch
    n, K = _check_inputs(I, p, g, alpha, coeffs, "host")
    if stream is None:
        stream = torch.cuda.current_stream()
    P = make_params(dict(params, K=K), stream=stream, precision=precision, algo=algo)
    o = out if out is not None else _alloc_out(torch, n, K, None, want_w, pin=True)
    sdedge_solve_batch_host(I, p, g, alpha, coeffs, n, P, o["lat"], o["gamma"], o["M"], o["batch_end"],
                            o["order"], o["w"], o["status"])
    return o
