"""-m "not gpu": the C-ABI library builds/loads and exports every symbol that
include/sdedge.h declares; argument validation runs host-side (no compute)."""
import ctypes as C
import os
import re

import pytest

import paper_2510_11331_b200 as sd
import scengen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "sdedge.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(sdedge_\w+)\s*\(", txt, re.M)))


def test_header_declares_expected():
    assert declared_symbols() == sorted(sd.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol():
    sd.build()
    L = C.CDLL(sd.LIB)
    for name in declared_symbols():
        assert hasattr(L, name), name
    assert sd.sdedge_abi_version() == 3


def test_struct_layout_matches_header():
    # sdedge_params: 2 models (24 B) + 4 c + B_w + sigma + lambda (56) + int64 + 7 int32 + pad + double + ptr
    assert C.sizeof(sd.SdedgeParams) == 152
    assert C.sizeof(sd.SdedgeScenarios) == 40 and C.sizeof(sd.SdedgeSchedule) == 72


@pytest.mark.parametrize("bad", [dict(K=0), dict(K=1025), dict(gamma_min=3, gamma_max=2),
                                 dict(gamma_max=65), dict(O_max=0), dict(noise_w=0.0),
                                 dict(bandwidth_hz=-1.0), dict(c1_draft=float("nan")),
                                 dict(precision=2), dict(algo=7), dict(flags=4), dict(draft=(0, 768, 3072)),
                                 dict(verify=(32, 70000, 11008)), dict(downlink_s=-1.0),
                                 dict(bandwidth_policy=2), dict(batching_policy=7),
                                 dict(batching_policy=3, static_batch=0)])
def test_invalid_arguments_rejected_without_gpu(bad):
    pd = dict(scengen.params("68M-7B", K=4), **bad)
    P = sd.make_params(pd)
    sc = sd.SdedgeScenarios(1, 1, 1, 1, None)
    sch = sd.SdedgeSchedule(1, 1, 1, 1, None, 1, None)
    rc = sd.lib().sdedge_solve_batch(C.byref(sc), 1, C.byref(P), 1, C.byref(sch))
    assert rc == -1 and sd.sdedge_last_error()


def test_null_pointers_rejected():
    P = sd.make_params(scengen.params("68M-7B", K=4))
    sc = sd.SdedgeScenarios(None, 1, 1, 1, None)
    sch = sd.SdedgeSchedule(1, 1, 1, 1, None, 1, None)
    assert sd.lib().sdedge_solve_batch(C.byref(sc), 1, C.byref(P), 1, C.byref(sch)) == -1
    assert sd.lib().sdedge_solve_batch(None, 1, C.byref(P), 1, C.byref(sch)) == -1
    assert sd.lib().sdedge_solve_batch(C.byref(sc), -1, C.byref(P), 1, C.byref(sch)) == -1


def test_no_oracle_in_product_path():
    """The product package must not import or link anything under oracle/."""
    pkg = os.path.join(ROOT, "paper_2510_11331_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cuh", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                for pat in ("import oracle", "from oracle", "sdedge_oracle", "orc_", "liboracle"):
                    assert pat not in txt, (f, pat)
