#!/usr/bin/env python
"""Summarise an ncu report (--set full) for the sweep kernels: key throughput,
pipe, stall and instruction-mix numbers.  Usage: python tools/ncu_summary.py rep.ncu-rep"""
import collections
import csv
import io
import subprocess
import sys


def ncu(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep):
    rows = ncu(rep, "--page", "raw", "--csv")
    hdr, units = rows[0], rows[1]
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
            "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        print("==", d["Kernel Name"][:80])
        for k in keys:
            if k in d:
                print(f"   {k:66s} {d[k]:>18s} {units[hdr.index(k)]}")
        st = [(k, float(v)) for k, v in d.items()
              if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
              and v not in ("", "n/a")]
        st.sort(key=lambda kv: -kv[1])
        print("   stalls/issue:", ", ".join(f"{k[35:-27]}={v:.2f}" for k, v in st[:8]))
    src = ncu(rep, "--page", "source", "--csv", "--print-source", "sass")
    kern, sh, data = None, None, collections.defaultdict(list)
    for r in src:
        if r and r[0] == "Kernel Name":
            kern, sh = r[1], None
            continue
        if r and r[0] == "Address":
            sh = r
            continue
        if sh and kern:
            data[kern].append(dict(zip(sh, r)))
    for k, v in data.items():
        tot, ops = 0, collections.Counter()
        for d in v:
            n = int(d.get("Instructions Executed") or 0)
            tot += n
            f = d["Source"].strip().split()
            if not f:
                continue
            o = f[1] if f[0].startswith("@") else f[0]
            ops[o.split(".")[0]] += n
        print("== mix", k[:70], "total", tot)
        print("   " + ", ".join(f"{o}={n / tot * 100:.1f}%" for o, n in ops.most_common(22)))


if __name__ == "__main__":
    main(sys.argv[1])
