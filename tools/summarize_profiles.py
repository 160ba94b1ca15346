#!/usr/bin/env python
"""Turn the round's gpurun_out/ artefacts into tracked summaries under profiles/:
  profiles/<tag>_launches.md       per-kernel share of a bench step (ncu launch list)
  profiles/<tag>_sweep_ncu.md      ncu --set full summary of the sweep kernels
  profiles/<tag>_eval_ncu.md       ncu --set full summary of the evaluation kernel (row f1)
  profiles/<tag>_flow_launches.md  per-kernel share of an optical-flow call (row f2)
  profiles/<tag>_flow_ncu.md       ncu --set full summary of the main flow kernels
  profiles/ncu_traffic.json        dram bytes per launch of those kernels (bench.py reads it)
  profiles/<tag>_bench.json        the bench JSON line
Usage: python tools/summarize_profiles.py <tag>"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def short(name):
    for k in ("ff_prop_kernel", "ff_knn_mma_kernel", "ff_knn_prep_kernel", "ff_knn_kernel", "ff_search_kernel",
              "ff_lift_kernel", "ff_init_kernel", "ff_quad_kernel", "ff_wht_kernel", "ff_downsample_kernel",
              "ff_consistency_kernel", "eval_kernel"):
        if k in name:
            return k
    for k in ("sweep_kernel<", "census_kernel", "lr_kernel", "combine_kernel", "cost_kernel", "wta_kernel"):
        if k in name:
            if k == "sweep_kernel<":
                args = name.split("sweep_kernel<")[1].split(">")[0]
                return "sweep_bwd_wta" if args.split(",")[2].strip() in ("1", "true", "(bool)1") else "sweep_fwd"
            return k
    return name[:40]


def launches(tag, src="launches.csv", out=None, title=None, cmd=None):
    rows = list(csv.reader(open(os.path.join(OUT, src))))
    hdr = None
    data = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                data.append(d)
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for d in data:
        k = short(d["Kernel Name"])
        v = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
                 "second": 1e6, "s": 1e6}
        v = v * scale.get(unit, 1.0)
        tot[k] += v
        cnt[k] += 1
    s = sum(tot.values())
    lines = [f"# {tag}: {title or 'kernel launch list'} (ncu gpu__time_duration, --clock-control none)", "",
             "Command: " + (cmd or "`python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph "
                                   "--no-stream --no-flow --no-eval` (8 Driving quads per step)") +
             "; ncu serialises launches and runs cold, so compare shares.", "",
             "| kernel | launches | total us | us/launch | share |", "|---|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        lines.append(f"| {k} | {cnt[k]} | {v:.1f} | {v / cnt[k]:.1f} | {100 * v / s:.1f}% |")
    open(os.path.join(PROF, out or f"{tag}_launches.md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def ncu_rows(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def full(tag, rep_name="prof_sweep_round.ncu-rep", out=None, title="the sweep kernels", cmd=None,
         traffic=None):
    rep = os.path.join(OUT, rep_name)
    if not os.path.exists(rep):
        print("missing", rep)
        return
    rows = ncu_rows(rep, "--page", "raw", "--csv")
    hdr, units = rows[0], rows[1]
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
            "sm__inst_executed.avg.per_cycle_active",
            "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__grid_size", "launch__block_size", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
    lines = [f"# {tag}: ncu --set full of {title}", "",
             "Command: " + (cmd or "`ncu --set full --clock-control none --import-source on -k regex:sweep_kernel "
                                   "-c 2 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph "
                                   "--no-stream --no-flow --no-eval` (launches of 32 Driving views = 8 quads)") + ".", ""]
    traffic = {} if traffic is None else traffic
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        name = short(d["Kernel Name"])
        lines += [f"## {name} (`{d['Kernel Name'][:90]}`)", "", "| metric | value | unit |", "|---|---|---|"]
        for k in keys:
            if k in d:
                lines.append(f"| {k} | {d[k]} | {units[hdr.index(k)]} |")
        st = [(k, float(v)) for k, v in d.items() if k.startswith("smsp__average_warps_issue_stalled_")
              and k.endswith("_per_issue_active.ratio") and v not in ("", "n/a")]
        st.sort(key=lambda kv: -kv[1])
        lines += ["", "Top stall reasons (warp cycles per issued instruction): " +
                  ", ".join(f"{k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]}={v:.2f}"
                            for k, v in st[:8]), ""]
        def gb(k):
            v = float(d[k].replace(",", ""))
            u = units[hdr.index(k)]
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        traffic[name] = gb("dram__bytes_read.sum") + gb("dram__bytes_write.sum")
    open(os.path.join(PROF, out or f"{tag}_sweep_ncu.md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    return traffic


if __name__ == "__main__":
    tag = sys.argv[1]
    os.makedirs(PROF, exist_ok=True)
    launches(tag)
    traffic = full(tag) or {}
    full(tag, "prof_eval_round.ncu-rep", f"{tag}_eval_ncu.md", "the evaluation kernel (row f1)",
         "`ncu --set full --clock-control none --import-source on -k regex:eval_kernel -c 1 python bench.py "
         "--steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-stream --no-flow` (8 Driving quads)",
         traffic)
    if os.path.exists(os.path.join(OUT, "flow_launches.csv")):
        launches(tag, "flow_launches.csv", f"{tag}_flow_launches.md", "optical-flow kernel launch list (row f2)",
                 "`python tools/flow_timing.py 8 3` (8 Driving pairs, 3 fields each, 3 levels; 8 calls)")
    full(tag, "prof_flow_round.ncu-rep", f"{tag}_flow_ncu.md", "the main optical-flow kernels (row f2)",
         "`ncu --set full --clock-control none --import-source on -k regex:\"ff_prop_kernel|ff_knn_mma_kernel\" "
         "-s 20 -c 3 python tools/flow_timing.py 8 3`", traffic)
    json.dump(traffic, open(os.path.join(PROF, "ncu_traffic.json"), "w"), indent=1)
    b = os.path.join(OUT, "bench_full.json")
    if os.path.exists(b):
        open(os.path.join(PROF, f"{tag}_bench.json"), "w").write(open(b).read())
