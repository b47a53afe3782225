#!/usr/bin/env python
"""Record the DRAM traffic of the main solve launch from one `ncu --set full`
capture into profiles/ncu_traffic.json, keyed by workload and tagged with the
sha256 of csrc/sdedge.cu it was measured on (bench.py reports `traffic` only
while that sha matches the source).

    python tools/ncu_traffic.py REPORT.ncu-rep KEY N_SCENARIOS
    KEY = "<config>/<pair>/<algo>/<precision>", e.g. C4/68M-7B/envelope/fp64
"""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from ncu_summary import raw  # noqa: E402


def to_bytes(v, unit):
    f = float(v.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main():
    rep, key, n = sys.argv[1], sys.argv[2], int(sys.argv[3])
    kernels, units = raw(rep)
    ks = [k for k in kernels if "solve_kernel" in k.get("Kernel Name", "")]
    k = max(ks, key=lambda k: float(k["gpu__time_duration.sum"].replace(",", "")))
    rd = to_bytes(k["dram__bytes_read.sum"], units["dram__bytes_read.sum"])
    wr = to_bytes(k["dram__bytes_write.sum"], units["dram__bytes_write.sum"])
    src = open(os.path.join(ROOT, "paper_2510_11331_b200", "csrc", "sdedge.cu"), "rb").read()
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    db = json.load(open(path)) if os.path.exists(path) else {}
    db[key] = {"dram_bytes_per_scenario": (rd + wr) / n, "read": rd, "written": wr, "n_scenarios": n,
               "capture": os.path.basename(rep), "source_sha256": hashlib.sha256(src).hexdigest()}
    json.dump(db, open(path, "w"), indent=1, sort_keys=True)
    print(key, db[key])


if __name__ == "__main__":
    main()
