#!/usr/bin/env python
"""DRAM traffic per launch of the sweep kernels from `ncu --set full` captures
(tools/profile_r02.sh) -> profiles/ncu_traffic.json ({"<config>/<kernel>": {"bytes",
"quads", ...}}, read by bench.py for roofline.traffic) and a markdown summary.

    python tools/ncu_traffic.py gpurun_out/r02_sweep_*.raw.csv > profiles/r02_sweep_ncu.md
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1e-9,
        "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}


def raw(rep):
    """Raw page of a report (.ncu-rep) or of its saved CSV (.raw.csv)."""
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    while rows and (not rows[0] or rows[0][0] != "ID" and "Kernel Name" not in rows[0]):
        rows = rows[1:]
    return rows[0], rows[1], rows[2:]


def main(reps):
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        table = json.load(open(path))
    except (OSError, ValueError):
        table = {}
    table = {k: v for k, v in table.items() if isinstance(v, dict)}
    print("| config | kernel | time (ms) | DRAM read (GB) | DRAM write (GB) | algorithmic (GB) | "
          "traffic / algorithmic | lane-instr / view-cell | IPC | ALU % | FMA % | warps active % | regs |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    sys.path.insert(0, ROOT)
    import synth
    for rep in reps:
        m = re.search(r"sweep_(\w+?)x(\d+)\.(ncu-rep|raw\.csv)$", rep)
        cfgname, quads = m.group(1), int(m.group(2))
        cfg = synth.CONFIGS[cfgname]
        hdr, units, rows = raw(rep)
        for row in rows:
            d = dict(zip(hdr, row))
            u = dict(zip(hdr, units))
            name = d["Kernel Name"]
            # template arguments: <CPL, C64, BWD, ...> (sweep_kernel / stair_kernel)
            targs = re.search(r"_kernel<([^>]*)>", name).group(1).replace("(int)", "").replace("(bool)", "")
            targs = [a.strip() for a in targs.split(",")]
            bwd = targs[2] in ("1", "true")
            kern = "sweep_bwd_wta" if bwd else "sweep_fwd"

            def val(k):
                return float(d[k].replace(",", "")) * UNIT.get(u[k], 1)
            rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
            view_px = 4 * quads * cfg.W * cfg.H
            alg = view_px * (2 * cfg.D + (6 if bwd else 16))
            cells = view_px * cfg.D
            lane_instr = float(d["smsp__inst_executed.sum"].replace(",", "")) * 32 / cells
            table[f"{cfgname}x{quads}/{kern}"] = {"bytes": rd + wr, "read": rd, "write": wr, "quads": quads,
                                          "algorithmic": alg, "ncu_ms": val("gpu__time_duration.sum") * 1e3,
                                          "lane_instr_per_view_cell": lane_instr,
                                          "source": os.path.basename(rep)}
            print(f"| {cfgname} x{quads} | {kern} | {val('gpu__time_duration.sum') * 1e3:.3f} | {rd / 1e9:.3f} | "
                  f"{wr / 1e9:.3f} | {alg / 1e9:.3f} | {(rd + wr) / alg:.3f} | {lane_instr:.1f} | "
                  f"{d['sm__inst_executed.avg.per_cycle_active']} | "
                  f"{d['sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active']} | "
                  f"{d['sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active']} | "
                  f"{d['sm__warps_active.avg.pct_of_peak_sustained_active']} | {d['launch__registers_per_thread']} |")
    with open(path, "w") as f:
        json.dump(table, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:])
