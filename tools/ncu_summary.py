#!/usr/bin/env python
"""Summarise an ncu --set full report (+ optional launch-list CSV) into markdown.

usage: python tools/ncu_summary.py REPORT.ncu-rep [LAUNCHES.csv] > profiles/rNN_....md
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__inst_executed.sum", "warp instructions executed"),
    ("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "thread DFMA executed"),
    ("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "thread DADD executed"),
    ("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", "thread DMUL executed"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__inst_executed_pipe_fp64.sum", "FP64-pipe warp instructions"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active %"),
    ("dram__bytes_read.sum", "DRAM bytes read"),
    ("dram__bytes_write.sum", "DRAM bytes written"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("l1tex__t_bytes.sum", "L1 bytes"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem / block"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "avg active threads / warp instr"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))


def main():
    rep = sys.argv[1]
    kernels, units = raw(rep)
    print(f"# ncu summary: `{rep.split('/')[-1]}`\n")
    for k in kernels:
        print(f"## {k.get('Kernel Name', '?')[:120]}\n")
        print("| metric | value | unit |\n|---|---|---|")
        for m, name in KEYS:
            if m in k:
                print(f"| {name} (`{m}`) | {k[m]} | {units.get(m, '')} |")
        st = {m.replace("smsp__pcsamp_warps_issue_stalled_", ""): k[m] for m in k
              if m.startswith("smsp__pcsamp_warps_issue_stalled_") and not m.endswith("not_issued")}
        tot = sum(float(v.replace(",", "")) for v in st.values() if v.replace(",", "").replace(".", "").isdigit())
        if tot:
            print("\nwarp-stall samples (share of all samples):\n")
            for m, v in sorted(st.items(), key=lambda x: -float(x[1].replace(",", "") or 0))[:10]:
                print(f"- {m}: {100 * float(v.replace(',', '')) / tot:.1f} %")
        print()
    if len(sys.argv) > 2:
        rows = [r for r in csv.reader(open(sys.argv[2])) if len(r) > 10 and not r[0].startswith("==")]
        hdr = rows[0]
        ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
        tot = {}
        for r in rows[1:]:
            name = r[ik].split("(")[0][:70]
            tot.setdefault(name, [0, 0.0])
            tot[name][0] += 1
            tot[name][1] += float(r[iv].replace(",", ""))
            unit = r[iu]
        s = sum(v[1] for v in tot.values())
        print("## launch list (`--metrics gpu__time_duration.sum`, cold-cache, serialised)\n")
        print("| kernel | launches | total time | share |\n|---|---|---|---|")
        for n, (c, t) in sorted(tot.items(), key=lambda x: -x[1][1]):
            print(f"| `{n}` | {c} | {t:.0f} {unit} | {100 * t / s:.2f} % |")


if __name__ == "__main__":
    main()
