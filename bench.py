#!/usr/bin/env python
"""Benchmark of the hot path: SGM at t and t+1 + basic scene-flow combination + 3D.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

`--gpus N` with N > 1 re-launches itself under torch.distributed.run (one process per
GPU, NCCL); when the driver launches it under torchrun, WORLD_SIZE must equal N.

One step = the whole hot path (census x4, 4 SGM views, 2 LR checks, combine + 3D:
every row of SURVEY.md 8(a)) over this rank's share of the workload, inputs resident
in HBM.  Default workload = BASELINE.json configs[4]: 64 Driving-scale quads (seeds
1000..1063) split 64/N over the ranks (strong scaling; `--weak` keeps
`--quads-per-gpu` per rank instead).  After the compute-only timing, the same steps
are timed again with the NCCL gather of every rank's results (S, dP and both masks)
to rank 0 inside the timed region.

Prints ONE JSON line (rank 0).  Metric: BASELINE.json's "SGM cost-volume cells/s
(W*H*D/s)", counted once per LR-checked disparity map (2 per quad), plus frames/s.
See DESIGN.md section 7 for the roofline accounting.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "SGM cost-volume cells/s (W*H*D/s)"
UNIT = "cells/s"
BATCH_TOTAL = 64            # BASELINE.json configs[4]
SIDE_QUADS = 8              # quads of the side sections (stream / flow / densify / eval)
# the other single-GPU BASELINE configs, timed on rank 0 at N=1 (the "configs" block)
CONFIG_SET = (("tiny", 64), ("driving", 1), ("wide", 8), ("highres", 4))


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="batch", choices=["batch", "driving", "wide", "highres", "tiny"])
    ap.add_argument("--quads", type=int, default=BATCH_TOTAL,
                    help="total quads of the batch config, split over the ranks (strong scaling)")
    ap.add_argument("--weak", action="store_true", help="fixed --quads-per-gpu per rank instead")
    ap.add_argument("--quads-per-gpu", type=int, default=8)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-gather", action="store_true", help="skip the with-gather timing")
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config block")
    ap.add_argument("--no-eval", action="store_true", help="skip the evaluation-step timing")
    ap.add_argument("--no-stream", action="store_true", help="skip the streaming-mode timing")
    ap.add_argument("--no-flow", action="store_true", help="skip the optical-flow timing")
    ap.add_argument("--no-densify", action="store_true", help="skip the densification timing")
    ap.add_argument("--minimal", action="store_true", help="only the main step (+ e2e unless --no-e2e)")
    a = ap.parse_args(argv)
    if a.minimal:
        a.no_cpu_baseline = a.no_gather = a.no_configs = True
        a.no_eval = a.no_stream = a.no_flow = a.no_densify = True
    return a


# ---------------------------------------------------------------------------- launching
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_ranks(n):
    """Re-run this command as n ranks under torch.distributed.run (127.0.0.1 rendezvous)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


# ---------------------------------------------------------------------------- helpers
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region.  nvidia-smi is
    started (and waited for: its first sample can take a few hundred ms) before the timed
    region; only samples stamped between begin() and stop() are kept."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []                      # (monotonic time, fields)
        self.proc = None
        self.t_begin = None

    def start(self, wait_s=10.0):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
            return
        t0 = time.monotonic()
        while not self.rows and time.monotonic() - t0 < wait_s and self.proc.poll() is None:
            time.sleep(0.01)

    def begin(self):
        self.t_begin = time.monotonic()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.monotonic(), [c.strip() for c in line.split(",")]))

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        t_end = time.monotonic()
        time.sleep(0.03)                    # the sample in flight at the end of the region
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        t_begin = self.t_begin if self.t_begin is not None else 0.0
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for t, r in self.rows:
            if t < t_begin or t > t_end + 0.025:
                continue
            try:
                sm.append(float(r[1]))
                smax.append(float(r[2]))
            except (ValueError, IndexError):
                continue
            for n, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def ncu_traffic(config, kernel, quads):
    """DRAM bytes (read + write) per launch of `kernel` scaled to `quads` quads, from the
    committed `ncu --set full` capture (profiles/ncu_traffic.json: {"<config>x<quads>/<kernel>"
    or "<config>/<kernel>": {"bytes": per launch, "quads": quads of that launch}}; the capture
    of the same quad count first), else None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            table = json.load(f)
    except (OSError, ValueError):
        return None
    rec = table.get(f"{config}x{quads}/{kernel}") or table.get(f"{config}/{kernel}")
    if not isinstance(rec, dict) or not rec.get("quads"):
        return None
    return rec["bytes"] * quads / rec["quads"]


def pct(v, q):
    v = sorted(v)
    if not v:
        return None
    k = (len(v) - 1) * q
    lo = int(k)
    hi = min(lo + 1, len(v) - 1)
    return v[lo] + (v[hi] - v[lo]) * (k - lo)


def dist_stats(ms):
    return {"mean": sum(ms) / len(ms), "median": statistics.median(ms), "p10": pct(ms, 0.1),
            "p90": pct(ms, 0.9), "n": len(ms)}


# Algorithmic work per view-cell and sweep, in lane-operations:
# 16-bit min-plus ops count 1/2 (two per u16x2 lane-op), 32-bit ops count 1.
#   per path: min(L(d-1),L(d+1)), +P1, min with L(d), min with m+P2, +C, -m,
#             min-reduction contribution, accumulate            = 8 elementary -> 4
#   forward sweep: 4 paths + the Hamming cost (62-bit census: 2 xor, 2 popc, 1 add = 5;
#                  <= 32-bit census: 1 xor, 1 popc = 2)
#   backward sweep: 4 paths + S_fwd + S_bwd (1/2) + argmin (1); it computes no cost (it
#                  unpacks C from the S_fwd word the forward sweep stored)
def alu_ops_per_cell(c64, bwd):
    return 4 * 4 + 1.5 if bwd else 4 * 4 + (5 if c64 else 2)


def sweep_bytes(cfg, view_px, bwd):
    """Algorithmic HBM bytes of one sweep launch over `view_px` view-pixels: S_fwd (uint16
    per cell) written once by the forward sweep and read once by the backward sweep, plus
    the forward sweep's census reads (reference + match row, 16 B/px) and the backward
    sweep's raw WTA stores (int16 + float32, 6 B/px)."""
    return view_px * (2 * cfg.D + (6 if bwd else 16))


def roofline_block(cfg, quads, stage_avg, peaks, peak_src, tag):
    """ALU + HBM roofline of both sweep kernels for `quads` quads; the dominant one first."""
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    issue_peak = 148 * 128 * sm_mhz * 1e6          # lane-ops/s: 1 warp-instr/clk/SMSP
    hbm_peak = float(peaks.get("hbm_gbs", 6554.9))
    c64 = cfg.cw * cfg.ch - 1 > 32
    view_px = 4 * quads * cfg.W * cfg.H
    cells = view_px * cfg.D
    out = {}
    for kern, bwd in (("sweep_fwd", False), ("sweep_bwd_wta", True)):
        ms = stage_avg.get(kern)
        if not ms:
            continue
        ops = alu_ops_per_cell(c64, bwd) * cells
        ach = ops / (ms * 1e-3)
        b = sweep_bytes(cfg, view_px, bwd)
        gbs = b / (ms * 1e-3) / 1e9
        out[kern] = {
            "bound": "alu", "achieved": ach / 1e12, "peak": issue_peak / 1e12, "unit": "Tlane-op/s",
            "frac": ach / issue_peak, "traffic": ncu_traffic(tag, kern, quads),
            "launch_ms": ms, "ops_per_view_cell": alu_ops_per_cell(c64, bwd),
            "algorithmic_ops_per_launch": ops,
            "alu_pipe_ceiling": {"peak": issue_peak / 2e12, "frac": ach / (issue_peak / 2),
                                 "note": "VIMNMX / VIADDMNMX / VIMNMX3 / IADD3 / LOP3 issue at half "
                                         "rate (0.5 warp-instr/clk/SMSP, tools/pipe_probe.cu)"},
            "hbm": {"achieved_gbs": gbs, "peak_gbs": hbm_peak, "frac": gbs / hbm_peak,
                    "algorithmic_bytes_per_launch": b},
            "peak_source": f"148 SM x 128 lanes x {sm_mhz:.0f} MHz (sm_max_mhz, {peak_src})",
        }
    if not out:
        return None
    dom = max(out, key=lambda k: out[k]["launch_ms"])
    head = dict(out[dom])
    head["kernel"] = dom
    head["kernels"] = out
    return head


# ---------------------------------------------------------------------------- reference arm
def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def run_oracle_quads(quads, prm, cores):
    """The C oracle (oracle/, as it stands) on every quad, one quad per worker thread
    (ctypes releases the GIL), `cores` threads.  Returns the wall time."""
    from concurrent.futures import ThreadPoolExecutor
    import oracle
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=cores) as ex:
        list(ex.map(lambda q: oracle.run_quad(q, prm, threads=False), quads))
    return time.perf_counter() - t0


def run_reference(args, cfg, rank):
    """The oracle (oracle/, plain C, fp64) as it stands on all host cores: each step is a
    bounded sample of the same workload -- one quad per core, each cropped to 48 rows."""
    if rank != 0:
        return
    import numpy as np
    import oracle
    import synth
    oracle.build()
    cores = host_cores()
    rows = min(48, cfg.H)
    nq = min(cores, BATCH_TOTAL) if cfg.name == "batch" else 1
    use = cores if cfg.name == "batch" else 1
    quads = synth.make_batch(cfg, 0, nq, workers=min(nq, cores))
    crops = [{k: np.ascontiguousarray(q[k][:rows]) for k in ("il0", "ir0", "il1", "ir1", "flow")}
             for q in quads]
    prm = dict(synth.sgm_params(cfg), cy=(rows - 1) / 2.0)
    for _ in range(args.warmup):
        run_oracle_quads(crops, prm, use)
    dt = 0.0
    for _ in range(args.steps):
        dt += run_oracle_quads(crops, prm, use)
    cells = 2 * cfg.W * rows * cfg.D * nq * args.steps
    value = cells / dt
    sample = (f"{nq} quad(s) per step, each cropped to {cfg.W}x{rows} (2 LR-checked maps + "
              f"combine + 3D per quad), {use} thread(s), one quad per thread")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True,
            "scaling": "strong" if cfg.name == "batch" and not args.weak else "weak",
            "vs_baseline": None, "dtype": "int16/f64", "data": "synthetic",
            "config": {"workload": f"{cfg.name}: {sample} (D={cfg.D}, census {cfg.cw}x{cfg.ch}, "
                                   f"P1={cfg.P1}, P2={cfg.P2})"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": use, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(cfg, quads):
    """The oracle on a bounded sample of the workload: for the batch config one full quad
    per host core, all cores in parallel (~10-20 s); otherwise one quad, one thread."""
    import oracle
    import synth
    oracle.build()
    prm = synth.sgm_params(cfg)
    if cfg.name == "batch":
        cores = host_cores()
        sample = quads[:min(cores, len(quads))]
        use = min(cores, len(sample))
    else:
        sample, use = quads[:1], 1
    dt = run_oracle_quads(sample, prm, use)
    return {"value": len(sample) * 2 * cfg.W * cfg.H * cfg.D / dt, "unit": UNIT, "cores": use,
            "kind": "oracle",
            "sample": f"{len(sample)} full {cfg.name} quad(s) {cfg.W}x{cfg.H} D={cfg.D} (2 LR-checked "
                      f"maps, combine, 3D each), {use} thread(s), one quad per thread, {dt:.1f} s wall"}


# ---------------------------------------------------------------------------- our arm
class Runner:
    """One handle + inputs + outputs of a workload on this rank, with timing helpers."""

    def __init__(self, cfg, quads, dev, packed=False, graph=True):
        import torch
        from paper_1801_04720_b200 import SGM, Camera, stack_quads
        from paper_1801_04720_b200.dist import alloc_packed_outputs
        self.torch = torch
        self.cfg, self.quads, self.dev = cfg, quads, dev
        self.n = len(quads)
        self.sgm = SGM.from_config(cfg, max_batch=self.n, device=dev.index)
        self.imgs, self.flow = stack_quads(quads, self.sgm.pitch, dev)
        import synth
        prm = synth.sgm_params(cfg)
        self.cam = Camera(prm["f"], prm["B"], prm["cx"], prm["cy"])
        if packed:
            self.packed, self.out = alloc_packed_outputs(self.sgm, self.n)
        else:
            self.packed, self.out = None, self.sgm.alloc_outputs(self.n)
        self.stream = torch.cuda.Stream(dev)
        self.flush = torch.empty(int(256 * 2**20), dtype=torch.uint8, device=dev)   # > 126 MB L2
        self.flush_sum = torch.empty((), dtype=torch.int64, device=dev)
        self.graph = None
        with torch.cuda.stream(self.stream):
            for _ in range(3):
                self.step()
        self.stream.synchronize()
        if graph:
            try:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=self.stream):
                    self.step()
                self.stream.synchronize()
                g.replay()
                self.stream.synchronize()
                self.graph = g
            except Exception as e:  # pragma: no cover - reported, eager path still measured
                print(f"# CUDA graph capture failed ({e}); timing eager launches", file=sys.stderr)

    def step(self):
        self.sgm.scene_flow(self.imgs, self.flow, self.cam, self.out, stream=self.stream)

    def run_once(self):
        if self.graph is not None:
            self.graph.replay()
        else:
            self.step()

    def flush_l2(self):
        # write a buffer twice the L2 size, then read it back: the L2 then holds clean lines
        # of `flush` only, so the timed kernels neither hit their own data nor pay for
        # writing back the flush's dirty lines
        self.flush.fill_(1)
        self.torch.sum(self.flush.view(self.torch.int64), dim=0, out=self.flush_sum)

    def timed(self, fn, steps, warmup=0):
        """Per-step device times (ms) of fn() on the runner's stream, L2 flushed before each."""
        torch = self.torch
        ms = []
        with torch.cuda.stream(self.stream):
            for _ in range(warmup):
                fn()
            for _ in range(steps):
                self.flush_l2()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(self.stream)
                fn()
                e1.record(self.stream)
                e1.synchronize()
                ms.append(e0.elapsed_time(e1))
        return ms

    def stage_times(self, steps):
        """Per-kernel durations: the same steps launched eagerly with the library's CUDA
        events recorded on the launch stream around every kernel (graph replays cannot be
        split).  Returns ({stage: mean ms}, launches per step)."""
        torch = self.torch
        stage = {}
        self.sgm.set_timing(True)
        n0 = self.sgm.launch_count()
        with torch.cuda.stream(self.stream):
            for _ in range(steps):
                self.flush_l2()
                self.step()
                self.stream.synchronize()
                t = self.sgm.read_timing()
                if t:
                    for k, v in t.items():
                        stage.setdefault(k, []).append(v)
        self.sgm.set_timing(False)
        per_step = (self.sgm.launch_count() - n0) / max(steps, 1)
        return {k: sum(v) / len(v) for k, v in stage.items()}, per_step

    def close(self):
        self.sgm.close()


def config_entry(cfg, n, runner, steps, warmup, peaks, peak_src):
    ms = runner.timed(runner.run_once, steps, warmup=max(warmup, 3))
    st, lps = runner.stage_times(max(3, min(steps, 10)))
    m = statistics.mean(ms)
    return {"quads": n, "W": cfg.W, "H": cfg.H, "D": cfg.D,
            "ms_per_step": m, "ms": dist_stats(ms),
            "map_cells_per_s": 2 * n * cfg.W * cfg.H * cfg.D / (m * 1e-3),
            "frames_per_s": n / (m * 1e-3), "stage_ms": st, "launches_per_step": lps,
            "roofline": roofline_block(cfg, n, st, peaks, peak_src, cfg.name)}


def main():
    args = parse()
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus))
    world = int(env_world or "1")
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("SGM_BENCH_SHARE_GPU"):          # functional run: all ranks on cuda:0 (gloo)
        local = 0
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    import synth
    cfg = synth.CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg, rank)
        return

    # ---------------- workload of this rank (inputs generated before CUDA is initialised)
    from paper_1801_04720_b200.dist import split_even, shard_indices
    strong = cfg.name == "batch" and not args.weak
    if strong:
        if args.quads % world:
            print(f"bench.py: {args.quads} quads do not split over {world} ranks", file=sys.stderr)
            sys.exit(2)
        idx = split_even(args.quads, world, rank)
    else:
        per = args.quads_per_gpu
        idx = shard_indices(rank, world, per)
    F = len(idx)
    total = F * world
    cores = host_cores()
    gen_workers = max(1, min(F, cores // max(world, 1)))
    t_gen = time.perf_counter()
    quads = synth.make_batch(cfg, idx[0], F, workers=gen_workers)
    t_gen = time.perf_counter() - t_gen

    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_1801_04720_b200.dist import (init_distributed, max_over_ranks, gather_packed)

    if torch.cuda.device_count() <= local:
        print(f"bench.py: rank {rank} needs cuda:{local}, {torch.cuda.device_count()} visible",
              file=sys.stderr)
        sys.exit(2)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = init_distributed(world, rank)
    peaks, peak_src = measured_peaks()

    run = Runner(cfg, quads, dev, packed=True, graph=not args.no_graph)
    W, H, D = cfg.W, cfg.H, cfg.D

    # ---------------- main timed region: compute only
    clocks = ClockSampler(local)
    clocks.start()                          # before the barrier: nvidia-smi needs a moment
    if pg is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks.begin()
    step_ms = run.timed(run.run_once, args.steps, warmup=args.warmup)
    torch.cuda.synchronize(dev)
    if pg is not None:
        dist.barrier()
    clk = clocks.stop()
    total_ms = max_over_ranks(sum(step_ms), dev)
    ms_per_step = total_ms / args.steps
    maps = 2 * total
    value = maps * W * H * D / (ms_per_step * 1e-3)
    frames_per_s = total / (ms_per_step * 1e-3)
    stage_avg, launches_per_step = run.stage_times(args.steps)
    roof = roofline_block(cfg, F, stage_avg, peaks, peak_src, cfg.name)

    # ---------------- the same steps with the NCCL gather of the results to rank 0
    # (configs[4]: "results are gathered with NCCL").  Two timings: `serial` -- every step is
    # compute then gather, one after the other on the stream -- and `pipelined` -- step k's
    # payload is staged (one D2D copy) and gathered asynchronously while step k+1's kernels
    # run (dist.PipelinedGather); the K-step span ends when the last gather has landed.  At
    # and `direct` (peer-memory stores, below).  At N > 1 the headline value is the better of
    # the pipelined and the direct form: the gather is inside the timed step.
    gather = None
    compute_only = None
    if not args.no_gather:
        if world > 1:
            from paper_1801_04720_b200.dist import PipelinedGather
            recv = [torch.empty_like(run.packed) for _ in range(world)] if rank == 0 else None

            def step_gather():
                run.run_once()
                gather_packed(run.packed, recv, rank, world)
            if pg is not None:
                dist.barrier()
            torch.cuda.synchronize(dev)
            g_ms = run.timed(step_gather, args.steps, warmup=max(args.warmup, 1))
            torch.cuda.synchronize(dev)
            g_tot = max_over_ranks(sum(g_ms), dev) / args.steps
            del recv
            pipe = PipelinedGather(run.packed, rank, world)

            def step_pipe():
                run.run_once()
                pipe.submit(run.packed)
            with torch.cuda.stream(run.stream):
                for _ in range(max(args.warmup, 3)):
                    step_pipe()
                pipe.drain()
                run.stream.synchronize()
                dist.barrier()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(run.stream)
                for _ in range(args.steps):
                    step_pipe()
                pipe.drain()
                e1.record(run.stream)
                e1.synchronize()
                p_tot = e0.elapsed_time(e1)
            torch.cuda.synchronize(dev)
            dist.barrier()
            p_tot = max_over_ranks(p_tot, dev) / args.steps
            gather = {"ms_per_step": p_tot, "frames_per_s": total / (p_tot * 1e-3),
                      "value": maps * W * H * D / (p_tot * 1e-3),
                      "mode": "pipelined: step k's payload staged and gathered (async) while "
                              "step k+1 computes; span of K steps incl. the last gather; the "
                              "per-rank working set (> 5 GB) exceeds L2, no flush inside the span",
                      "serial": {"ms_per_step": g_tot, "frames_per_s": total / (g_tot * 1e-3),
                                 "value": maps * W * H * D / (g_tot * 1e-3)},
                      "bytes_to_rank0_per_step": int(run.packed.numel() * (world - 1)),
                      "payload": "S (u,v,d0,d1) f32x4 + dP f32x4 + valid_sf + valid_3d = 34 B/px",
                      "collective": "dist.gather (NCCL) of one packed uint8 buffer per rank"}
            # Peer-memory form: rank 0 owns the result buffers, the other ranks map them through
            # CUDA IPC (peer access over NVLink) and pass their slice to sgm_scene_flow as the
            # output, so the combination kernel's stores carry the payload to rank 0 (no
            # collective, no staging copy); one tiny all-reduce per step orders "all ranks
            # done" on the stream.  Two alternating slots, one CUDA graph each.
            direct = None
            try:
                from paper_1801_04720_b200.dist import DirectGather, unpack_results
                dg = DirectGather(run.packed.numel(), rank, world, dev, slots=2)
            except Exception as e:
                direct = {"unavailable": str(e)[:200]}
            else:
                outs = [unpack_results(dg.mine(sl), F, H, W) for sl in range(2)]

                def eager(sl):
                    run.sgm.scene_flow(run.imgs, run.flow, run.cam, outs[sl], stream=run.stream)
                with torch.cuda.stream(run.stream):
                    for sl in range(2):
                        eager(sl)
                    run.stream.synchronize()
                    graphs = []
                    if run.graph is not None:
                        for sl in range(2):
                            g = torch.cuda.CUDAGraph()
                            with torch.cuda.graph(g, stream=run.stream):
                                eager(sl)
                            graphs.append(g)

                    def step_direct(k):
                        if graphs:
                            graphs[k & 1].replay()
                        else:
                            eager(k & 1)
                        dg.fence()
                    for k in range(max(args.warmup, 3)):
                        step_direct(k)
                    run.stream.synchronize()
                    dist.barrier()
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(run.stream)
                    for k in range(args.steps):
                        step_direct(k)
                    e1.record(run.stream)
                    e1.synchronize()
                    d_tot = e0.elapsed_time(e1)
                torch.cuda.synchronize(dev)
                dist.barrier()
                d_tot = max_over_ranks(d_tot, dev) / args.steps
                direct = {"ms_per_step": d_tot, "frames_per_s": total / (d_tot * 1e-3),
                          "value": maps * W * H * D / (d_tot * 1e-3),
                          "mode": "peer memory: every rank's kernels store S, dP and the masks "
                                  "straight into rank 0's buffer (CUDA IPC mapping, NVLink), one "
                                  "1-word all-reduce per step as the completion fence"}
                dg.close()
            gather["direct"] = direct
            compute_only = {"ms_per_step": ms_per_step, "frames_per_s": frames_per_s, "value": value,
                            "ms": dist_stats(step_ms)}
            best = gather
            if direct and "value" in direct and direct["value"] > gather["value"]:
                best = direct
            gather["headline"] = "direct" if best is direct else "pipelined"
            ms_per_step, frames_per_s, value = best["ms_per_step"], best["frames_per_s"], best["value"]
        else:
            gather = {"ms_per_step": ms_per_step, "frames_per_s": frames_per_s, "value": value,
                      "bytes_to_rank0_per_step": 0,
                      "note": "N=1: the results are already on rank 0 (no collective)"}

    # ---------------- e2e through the public API with host buffers
    # Every step uploads its own inputs from pinned host memory and downloads its result
    # (S + mask, 3D motion dP + mask) through sgm_scene_flow_host; steps are issued back
    # to back (two alternating host buffer sets), so step k+1's upload and step k-1's
    # download overlap step k's kernels; the span of the K steps is timed on the stream.
    e2e = None
    if not args.no_e2e:
        sgm, stream = run.sgm, run.stream
        sets = []
        for _ in range(2):
            himg = torch.from_numpy(np.stack([[q[k] for k in ("il0", "ir0", "il1", "ir1")]
                                              for q in quads])).pin_memory()
            hflow = torch.from_numpy(np.stack([q["flow"] for q in quads])).pin_memory()
            hout = sgm.alloc_outputs(F, with_disp=False, pinned_host=True, with_p0=False)
            sets.append((himg, hflow, hout))
        h2d = sets[0][0].numel() + sets[0][1].numel() * 4
        d2h = sum(t.numel() * t.element_size() for t in sets[0][2].values())
        with torch.cuda.stream(stream):
            for k in range(max(args.warmup, 3)):
                himg, hflow, hout = sets[k & 1]
                sgm.scene_flow_host(himg, hflow, run.cam, hout, stream=stream)
            stream.synchronize()
            if pg is not None:
                dist.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for k in range(args.steps):
                himg, hflow, hout = sets[k & 1]
                sgm.scene_flow_host(himg, hflow, run.cam, hout, stream=stream)
            e1.record(stream)
            e1.synchronize()
            tot = e0.elapsed_time(e1)
        tot = max_over_ranks(tot, dev)
        e2e_ms = tot / args.steps
        e2e = {"value": maps * W * H * D / (e2e_ms * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": e2e_ms, "frames_per_s": total / (e2e_ms * 1e-3),
               "pipelined": "steps issued back to back; per-step upload/download overlap the "
                            "neighbouring steps' kernels"}
        del sets

    side = side_sections(args, cfg, run, quads[:SIDE_QUADS], dev, world, peaks)

    # ---------------- the other single-GPU BASELINE configs (rank 0 at N=1)
    configs = None
    if not args.no_configs and world == 1:
        configs = {}
        for name, n in CONFIG_SET:
            c = synth.CONFIGS[name]
            if name == cfg.name and n == F:
                continue
            qs = synth.make_batch(c, 0, n, workers=max(1, min(n, cores)))
            r = Runner(c, qs, dev, graph=not args.no_graph)
            configs[f"{name}x{n}"] = config_entry(c, n, r, args.steps, args.warmup, peaks, peak_src)
            r.close()
            del r, qs
            torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, quads)

    if rank == 0:
        scale = "strong" if strong else "weak"
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": scale, "vs_baseline": None, "dtype": "u16x2/int32 (f32 sub-pixel, 3D)",
            "data": "synthetic",
            "config": {"workload": f"{cfg.name}: {total} Driving-scale quads, {F} per GPU per step "
                                   f"({W}x{H}, D={D}, census {cfg.cw}x{cfg.ch}, P1={cfg.P1}, "
                                   f"P2={cfg.P2}, 8 paths, LR T={cfg.T})",
                       "global_batch": total, "quads_per_gpu": F, "W": W, "H": H, "D": D,
                       "parallelism": f"{scale} scaling: frame quads sharded over {world} GPU(s) "
                                      "(contiguous blocks), no collective between the kernels; at "
                                      "N > 1 the step includes the NCCL gather of the results "
                                      "to rank 0, pipelined ('gather'; 'compute_only' without it)",
                       "l2": "256 MiB buffer written then read between timed steps (flush)",
                       "graph": run.graph is not None, "input_gen_s": round(t_gen, 1)},
            "frames_per_s": frames_per_s,
            "ms": dist_stats(step_ms),
            "stage_ms": stage_avg,
            "gpu_launches": int(round(launches_per_step * args.steps)),
            "clocks": clk,
            "roofline": roof,
            "gather": gather,
            "compute_only": compute_only,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "geometry": run.sgm.geometry(),
            "configs": configs,
        }
        line.update(side)
        print(json.dumps(line), flush=True)
    run.close()
    if pg is not None:
        dist.destroy_process_group()


def side_sections(args, cfg, run, quads, dev, world, peaks):
    """Rows f1-f4 of SURVEY.md 8(f), each timed on its own over SIDE_QUADS quads."""
    import numpy as np
    import torch
    from paper_1801_04720_b200.dist import max_over_ranks
    from paper_1801_04720_b200 import stack_quads
    F = len(quads)
    W, H, D = cfg.W, cfg.H, cfg.D
    sgm, stream, cam = run.sgm, run.stream, run.cam
    imgs, flow = stack_quads(quads, sgm.pitch, dev)
    out = sgm.alloc_outputs(F)
    res = {"stream": None, "flow": None, "densify": None, "evaluate": None}

    def avg(fn, steps, warm=3):
        return max_over_ranks(sum(run.timed(fn, steps, warmup=warm)), dev) / steps

    def sf():
        sgm.scene_flow(imgs, flow, cam, out, stream=stream)

    # ---------------- row f3: streaming (video) mode -- F quads of one video (F+1 frames)
    if not args.no_stream:
        import synth
        from paper_1801_04720_b200 import stack_video
        video = synth.make_video(cfg, F, 0)
        vimgs, vflow = stack_video(video, sgm.pitch, dev)
        vout = sgm.alloc_outputs(F, stream_mode=True)
        quad_ms = avg(sf, args.steps)
        sv_ms = avg(lambda: sgm.scene_flow_stream(vimgs, vflow, cam, vout, stream=stream), args.steps)
        res["stream"] = {"workload": f"one video of {F + 1} frames = {F} quads per GPU "
                                     f"({F + 1} SGM pairs instead of {2 * F})",
                         "ms_per_step": sv_ms, "frames_per_s": F * world / (sv_ms * 1e-3),
                         "map_cells_per_s": (F + 1) * world * W * H * D / (sv_ms * 1e-3),
                         "quad_mode_ms_same_quads": quad_ms, "speedup_vs_quad_mode": quad_ms / sv_ms}
        del vimgs, vflow, vout

    # ---------------- row f2: the optical-flow step and the full method
    if not args.no_flow:
        from paper_1801_04720_b200 import FlowFields
        ffh = FlowFields(W, H, max_batch=F, device=dev.index)
        fa = imgs[:, 0, :, :W].contiguous()            # left frames t
        fb = imgs[:, 2, :, :W].contiguous()            # left frames t+1
        fo = ffh.flow(fa, fb, stream=stream)
        sfo = sgm.alloc_outputs(F, with_disp=False)
        fsteps = max(1, min(args.steps, 5))
        f_ms = avg(lambda: ffh.flow(fa, fb, out=fo, stream=stream), fsteps)
        full_ms = avg(lambda: (ffh.flow(fa, fb, out=fo, stream=stream),
                               sgm.scene_flow(imgs, fo["flow"], cam, sfo, flow_valid=fo["valid"],
                                              stream=stream)), fsteps, warm=1)
        with torch.cuda.stream(stream):
            ffh.set_timing(True)
            ffh.flow(fa, fb, out=fo, stream=stream)
            stream.synchronize()
            fstages = ffh.read_timing()
            ffh.set_timing(False)
        gtf = flow.cpu().numpy()
        estf = fo["flow"].cpu().numpy()
        fval = fo["valid"].cpu().numpy() > 0
        epe = np.hypot(estf[..., 0] - gtf[..., 0], estf[..., 1] - gtf[..., 1])
        # roofline of the propagation kernel (random search fused in): the method's work per
        # sweep is three candidate data terms per pixel (left/up or right/down + the random
        # one), (2r+1)^2 samples x 8 integer ops (4 bilinear multiply-adds, Q^2 a, subtract,
        # abs, accumulate); the kernel is a latency-bound wavefront
        P = ffh.params
        ops = 0.0
        lw, lh = W, H
        for _lvl in range(P.levels):
            for r in (P.patch_radius, P.patch_radius, P.patch_radius + 2):
                ops += F * lw * lh * P.sweeps * 3 * (2 * r + 1) ** 2 * 8
            lw, lh = (lw + 1) // 2, (lh + 1) // 2
        sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
        peak_ops = 148 * 128 * sm_mhz * 1e6
        prop_ms = fstages["prop"] if fstages else None
        res["flow"] = {
            "workload": f"{F} Driving pairs per GPU (left frames t, t+1), {P.levels} levels, r={P.patch_radius}, "
                        f"{P.sweeps} sweeps/level, kNN {P.knn} on {P.desc_window}x{P.desc_window} WHT, "
                        "forward + 2 inverse fields + consistency",
            "ms_per_step": f_ms, "pairs_per_s": F * world / (f_ms * 1e-3),
            "full_method_ms_per_step": full_ms,
            "full_method_frames_per_s": F * world / (full_ms * 1e-3),
            "stage_ms": fstages,
            "valid_fraction": float(fval.mean()),
            "epe_le_1px_on_valid": float((epe[fval] <= 1.0).mean()),
            "roofline": None if not prop_ms else {
                "bound": "alu", "kernel": "ff_prop_kernel", "achieved": ops / (prop_ms * 1e-3) / 1e12,
                "peak": peak_ops / 1e12, "unit": "Tlane-op/s", "frac": ops / (prop_ms * 1e-3) / peak_ops,
                "traffic": ncu_traffic("driving", "ff_prop_kernel", F), "algorithmic_ops_per_call": ops,
                "launch_ms_per_call": prop_ms,
                "note": "row-sequential wavefront (left/up dependency): latency-bound, not issue-bound"},
        }
        ffh.close()
        del sfo

    # ---------------- row f4: edge-aware densification of the step's scene flow
    dsf = None
    sf()
    if not args.no_densify:
        from paper_1801_04720_b200 import densify
        guide = imgs[:, 0, :, :W].contiguous()
        box = {}

        def dens():
            box["d"] = densify(out["sf"], out["valid_sf"], guide, stream=stream, count_certified=True)
        d_ms = avg(dens, max(1, min(args.steps, 10)))
        dsf, cert = box["d"]
        torch.cuda.synchronize(dev)
        gaps = int((out["valid_sf"] == 0).sum().item())
        from paper_1801_04720_b200.flow import DENSIFY_WINDOW
        res["densify"] = {"workload": f"{F} Driving scene flows (4 channels) per GPU, K=25, lambda=1, "
                                      f"guide = I_l^t, SPEC F-6 ranking, candidate window {DENSIFY_WINDOW}",
                          "ms_per_step": d_ms, "gap_pixels": gaps, "gap_fraction": gaps / float(F * W * H),
                          "gap_pixels_per_s": gaps * world / (d_ms * 1e-3),
                          "certified_fraction": int(cert.item()) / max(gaps, 1)}

    # ---------------- row f1: the evaluation step (KITTI outlier counts vs the generator's GT)
    if not args.no_eval:
        from paper_1801_04720_b200 import rates_from_counts
        gd0 = torch.from_numpy(np.stack([q["gt_d0"] for q in quads])).to(dev)
        gd1 = torch.from_numpy(np.stack([q["gt_d1w"] for q in quads])).to(dev)
        noc = torch.from_numpy(np.stack([q["gt_noc"] for q in quads])).to(dev)
        counts = torch.empty((F, 2, 6), dtype=torch.int64, device=dev)
        ev_ms = avg(lambda: sgm.evaluate(out["sf"], out["valid_sf"], gd0, gd1, flow, noc, counts=counts,
                                         stream=stream), args.steps)
        tot = counts.sum(0).cpu().tolist()
        all_rates = None
        if dsf is not None:                          # "All": the densified field, every pixel
            ones = torch.ones_like(out["valid_sf"])
            dc = sgm.evaluate(dsf, ones, gd0, gd1, flow, noc, stream=stream)
            torch.cuda.synchronize(dev)
            all_rates = rates_from_counts(dc.sum(0).cpu().tolist())
        px = F * W * H
        bytes_px = 16 + 1 + 4 + 4 + 8 + 1            # sf, valid_sf, gt_d0, gt_d1, gt_flow, gt_noc
        gbs = px * bytes_px / (ev_ms * 1e-3) / 1e9
        hbm_peak = float(peaks.get("hbm_gbs", 6554.9))
        res["evaluate"] = {"metric": "evaluated pixels/s", "value": px * world / (ev_ms * 1e-3),
                           "unit": "px/s", "ms_per_launch": ev_ms, "pixels_per_launch": px,
                           "roofline": {"bound": "hbm", "achieved": gbs, "peak": hbm_peak,
                                        "unit": "GB/s", "frac": gbs / hbm_peak,
                                        "traffic": ncu_traffic("driving", "eval_kernel", F),
                                        "algorithmic_bytes_per_px": bytes_px},
                           "counts_occ_noc": tot, "rates": rates_from_counts(tot),
                           "rates_densified_all": all_rates}
    del out, imgs, flow
    return res


if __name__ == "__main__":
    main()
