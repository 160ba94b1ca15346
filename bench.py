#!/usr/bin/env python
"""Benchmark of the hot path: SGM at t and t+1 + basic scene-flow combination + 3D.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one process per GPU, NCCL)

One step = the whole hot path (census x4, 4 SGM views, 2 LR checks, combine + 3D:
every row of SURVEY.md 8(a)) over a batch of Driving-scale frame quads
(BASELINE.json configs[1] parameters; the per-GPU shard of the configs[4]
batched sweep), inputs resident in HBM.  Weak scaling: each rank owns
`--quads-per-gpu` quads (global batch = N x that; N=8 at 8 quads/GPU is the
64-quad configs[4] sweep); no collective inside the timed region.

Prints ONE JSON line (rank 0).  Metric: BASELINE.json's "SGM cost-volume cells/s
(W*H*D/s)", counted once per LR-checked disparity map (2 per quad), plus
frames/s.  See DESIGN.md "Measurement" for the roofline accounting.
"""
from __future__ import annotations

import argparse
import json
import os
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="batch", choices=["batch", "driving", "wide", "highres", "tiny"])
    ap.add_argument("--quads-per-gpu", type=int, default=8)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-eval", action="store_true", help="skip the evaluation-step timing")
    ap.add_argument("--no-stream", action="store_true", help="skip the streaming-mode timing")
    ap.add_argument("--no-flow", action="store_true", help="skip the optical-flow timing")
    ap.add_argument("--no-densify", action="store_true", help="skip the densification timing")
    ap.add_argument("--gather", action="store_true", help="also time an NCCL gather of results")
    return ap.parse_args()


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


def ncu_traffic(kernel):
    """dram bytes per launch of `kernel` from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    try:
        with open(p) as f:
            return json.load(f).get(kernel)
    except (OSError, ValueError):
        return None


# Algorithmic work per view-cell, in lane-operations:
# 16-bit min-plus ops count 1/2 (two per u16x2 lane-op), 32-bit ops count 1.
#   per path: min(L(d-1),L(d+1)), +P1, min with L(d), min with m+P2, +C, -m,
#             min-reduction contribution, accumulate            = 8 elementary -> 4
#   Hamming of a 62-bit census: 2 xor + 2 popc + 1 add            = 5 (24-bit: 2)
#   backward sweep extra: S_fwd + S_bwd (1/2), argmin (1)
def alu_ops_per_cell(c64, bwd):
    ops = 4 * 4 + (5 if c64 else 2)
    if bwd:
        ops += 1.5
    return ops


def sweep_bytes_per_cell(bwd):
    # S_fwd uint16 written once by the forward sweep, read once by the backward sweep
    return 2.0


# ---------------------------------------------------------------------------- reference arm
def run_reference(args, cfg, rank, world):
    """The oracle (oracle/, plain C, fp64) as it stands on the host cores: each step is a
    bounded sample -- one quad cropped to 48 rows -- of the same workload."""
    if rank != 0:
        return
    import numpy as np
    import oracle
    import synth
    oracle.build()
    prm = synth.sgm_params(cfg)
    rows = 48
    quad = synth.make_quad(cfg, 0)
    crop = {k: np.ascontiguousarray(quad[k][:rows]) for k in ("il0", "ir0", "il1", "ir1", "flow")}
    prm = dict(prm, cy=(rows - 1) / 2.0)
    for _ in range(args.warmup):
        oracle.run_quad(crop, prm, threads=False)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.run_quad(crop, prm, threads=False)
    dt = time.perf_counter() - t0
    cells = 2 * cfg.W * rows * cfg.D * args.steps
    value = cells / dt
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int16/f64", "data": "synthetic",
            "config": {"workload": f"{cfg.name}: 1 quad cropped to {cfg.W}x{rows} per step "
                                   f"(D={cfg.D}, census {cfg.cw}x{cfg.ch}, P1={cfg.P1}, P2={cfg.P2})"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"{args.steps} x one {cfg.W}x{rows} crop of a quad "
                                       "(2 LR-checked maps + combine + 3D), single thread"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(cfg):
    """Oracle on one full quad of the workload, one thread (bounded: ~10-20 s)."""
    import oracle
    import synth
    oracle.build()
    prm = synth.sgm_params(cfg)
    q = synth.make_quad(cfg, 0)
    t0 = time.perf_counter()
    oracle.run_quad(q, prm, threads=False)
    dt = time.perf_counter() - t0
    return {"value": 2 * cfg.W * cfg.H * cfg.D / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"1 {cfg.name} quad {cfg.W}x{cfg.H} D={cfg.D} (2 LR-checked maps, combine, "
                      f"3D) single-threaded C oracle, {dt:.1f} s"}


# ---------------------------------------------------------------------------- our arm
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import synth
    cfg = synth.CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return

    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_1801_04720_b200 import SGM, Camera
    from paper_1801_04720_b200.dist import init_distributed, shard_indices, max_over_ranks

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = init_distributed(world, rank)
    F = args.quads_per_gpu
    idx = shard_indices(rank, world, F)
    quads = [synth.make_quad(cfg, i) for i in idx]
    sgm = SGM.from_config(cfg, max_batch=F, device=local)
    from paper_1801_04720_b200.sgm import stack_quads
    imgs, flow = stack_quads(quads, sgm.pitch, dev)
    prm = synth.sgm_params(cfg)
    cam = Camera(prm["f"], prm["B"], prm["cx"], prm["cy"])
    out = sgm.alloc_outputs(F)
    stream = torch.cuda.Stream(dev)
    flush = torch.empty(int(256 * 2**20), dtype=torch.uint8, device=dev)   # > 126 MB L2
    flush_sum = torch.empty((), dtype=torch.int64, device=dev)

    def flush_l2():
        # write a buffer twice the L2 size, then read it back: the L2 then holds clean
        # lines of `flush` only, so the timed kernels neither hit their own data nor pay
        # for writing back the flush's dirty lines
        flush.fill_(1)
        torch.sum(flush.view(torch.int64), dim=0, out=flush_sum)

    def step():
        sgm.scene_flow(imgs, flow, cam, out, stream=stream)

    graph = None
    with torch.cuda.stream(stream):
        for _ in range(max(args.warmup, 3)):
            step()
    stream.synchronize()
    if not args.no_graph:
        try:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream):
                step()
            stream.synchronize()
            graph.replay()
            stream.synchronize()
        except Exception as e:  # pragma: no cover - reported, eager path still measured
            print(f"# CUDA graph capture failed ({e}); timing eager launches", file=sys.stderr)
            graph = None

    def run_once():
        if graph is not None:
            graph.replay()
        else:
            step()

    launches_per_step = 5
    stage_ms = {}
    clocks = ClockSampler(local)
    clocks.start()                          # before the barrier: nvidia-smi needs a moment
    if pg is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks.begin()
    total_ms = 0.0
    with torch.cuda.stream(stream):
        for _ in range(args.steps):
            flush_l2()                                       # evict L2 between timed steps
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            run_once()
            e1.record(stream)
            e1.synchronize()
            total_ms += e0.elapsed_time(e1)
    torch.cuda.synchronize(dev)
    if pg is not None:
        dist.barrier()
    clk = clocks.stop()
    # per-kernel durations: the same steps launched eagerly with the library's CUDA events
    # recorded on the launch stream around every kernel (graph replays cannot be split)
    sgm.set_timing(True)
    with torch.cuda.stream(stream):
        for _ in range(args.steps):
            flush_l2()
            step()
            stream.synchronize()
            t = sgm.read_timing()
            if t:
                for k, v in t.items():
                    stage_ms.setdefault(k, []).append(v)
    sgm.set_timing(False)
    total_ms = max_over_ranks(total_ms, dev)
    ms_per_step = total_ms / args.steps
    W, H, D = cfg.W, cfg.H, cfg.D
    maps = 2 * F * world
    value = maps * W * H * D / (ms_per_step * 1e-3)
    frames_per_s = F * world / (ms_per_step * 1e-3)

    # ---------------- roofline of the dominant kernel (backward sweep + WTA)
    peaks, peak_src = measured_peaks()
    stage_avg = {k: sum(v) / len(v) for k, v in stage_ms.items()}
    dom = max(("sweep_fwd", "sweep_bwd_wta"), key=lambda k: stage_avg.get(k, 0.0))
    dom_ms = stage_avg.get(dom)
    c64 = cfg.cw * cfg.ch - 1 > 32
    geo = sgm.geometry()
    view_cells = 4 * F * W * H * D
    roof = None
    if dom_ms:
        ops = alu_ops_per_cell(c64, dom == "sweep_bwd_wta") * view_cells
        sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
        peak_ops = 148 * 128 * sm_mhz * 1e6                     # lane-ops/s, 1 issue/SMSP/clk
        achieved = ops / (dom_ms * 1e-3)
        hbm_achieved = sweep_bytes_per_cell(True) * view_cells / (dom_ms * 1e-3) / 1e9
        roof = {"bound": "alu", "kernel": dom, "achieved": achieved / 1e12,
                "peak": peak_ops / 1e12, "unit": "Tlane-op/s", "frac": achieved / peak_ops,
                "traffic": ncu_traffic(dom),
                "algorithmic_ops_per_launch": ops, "launch_ms": dom_ms,
                "peak_source": f"148 SM x 128 lanes x {sm_mhz:.0f} MHz (sm_max_mhz, {peak_src})",
                "hbm": {"achieved_gbs": hbm_achieved, "peak_gbs": peaks.get("hbm_gbs"),
                        "frac": hbm_achieved / float(peaks.get("hbm_gbs", 6554.9)),
                        "algorithmic_bytes_per_launch": sweep_bytes_per_cell(True) * view_cells}}

    # ---------------- e2e through the public API with host buffers
    # Every step uploads its own inputs from pinned host memory and downloads its result
    # (S + mask, 3D motion dP + mask) through sgm_scene_flow_host; steps are issued back
    # to back (two alternating host buffer sets), so step k+1's upload and step k-1's
    # download overlap step k's kernels; the span of the K steps is timed on the stream.
    e2e = None
    if not args.no_e2e:
        sets = []
        for _ in range(2):
            himg = torch.from_numpy(np.stack([[q[k] for k in ("il0", "ir0", "il1", "ir1")]
                                              for q in quads])).pin_memory()
            hflow = torch.from_numpy(np.stack([q["flow"] for q in quads])).pin_memory()
            hout = sgm.alloc_outputs(F, with_disp=False, pinned_host=True, with_p0=False)
            sets.append((himg, hflow, hout))
        h2d = sets[0][0].numel() + sets[0][1].numel() * 4
        d2h = sum(t.numel() * t.element_size() for t in sets[0][2].values())
        sgm.set_timing(False)
        with torch.cuda.stream(stream):
            for k in range(max(args.warmup, 3)):
                himg, hflow, hout = sets[k & 1]
                sgm.scene_flow_host(himg, hflow, cam, hout, stream=stream)
            stream.synchronize()
            if pg is not None:
                dist.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for k in range(args.steps):
                himg, hflow, hout = sets[k & 1]
                sgm.scene_flow_host(himg, hflow, cam, hout, stream=stream)
            e1.record(stream)
            e1.synchronize()
            tot = e0.elapsed_time(e1)
        tot = max_over_ranks(tot, dev)
        e2e_ms = tot / args.steps
        e2e = {"value": maps * W * H * D / (e2e_ms * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": e2e_ms, "frames_per_s": F * world / (e2e_ms * 1e-3),
               "pipelined": "steps issued back to back; per-step upload/download overlap the "
                            "neighbouring steps' kernels"}

    # ---------------- streaming (video) mode, timed on its own
    # F consecutive quads of one video (F+1 frames): each frame's map computed once.
    stream_res = None
    if not args.no_stream:
        from paper_1801_04720_b200 import stack_video
        video = synth.make_video(cfg, F, idx[0])
        vimgs, vflow = stack_video(video, sgm.pitch, dev)
        vout = sgm.alloc_outputs(F, stream_mode=True)
        with torch.cuda.stream(stream):
            for _ in range(max(args.warmup, 3)):
                sgm.scene_flow_stream(vimgs, vflow, cam, vout, stream=stream)
            sv_ms = 0.0
            for _ in range(args.steps):
                flush_l2()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                sgm.scene_flow_stream(vimgs, vflow, cam, vout, stream=stream)
                e1.record(stream)
                e1.synchronize()
                sv_ms += e0.elapsed_time(e1)
        sv_ms = max_over_ranks(sv_ms, dev) / args.steps
        stream_res = {"workload": f"one video of {F + 1} frames = {F} quads per GPU "
                                  f"({F + 1} SGM pairs instead of {2 * F})",
                      "ms_per_step": sv_ms, "frames_per_s": F * world / (sv_ms * 1e-3),
                      "map_cells_per_s": (F + 1) * world * W * H * D / (sv_ms * 1e-3),
                      "speedup_vs_quad_mode": ms_per_step / sv_ms}
        del vimgs, vflow, vout

    # ---------------- the optical-flow step (Flow Fields+-style
    # core) timed on its own, and the full method: flow estimated on the GPU, then the
    # scene-flow step with the estimated flow and its consistency mask.
    flow_res = None
    if not args.no_flow:
        from paper_1801_04720_b200 import FlowFields
        ffh = FlowFields(W, H, max_batch=F, device=local)
        fa = imgs[:, 0, :, :W].contiguous()            # left frames t
        fb = imgs[:, 2, :, :W].contiguous()            # left frames t+1
        fo = ffh.flow(fa, fb, stream=stream)
        sfo = sgm.alloc_outputs(F, with_disp=False)
        fsteps = max(1, min(args.steps, 5))
        with torch.cuda.stream(stream):
            for _ in range(max(args.warmup, 3)):
                ffh.flow(fa, fb, out=fo, stream=stream)
            stream.synchronize()

            def timed(fn):
                tot = 0.0
                for _ in range(fsteps):
                    flush_l2()
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    fn()
                    e1.record(stream)
                    e1.synchronize()
                    tot += e0.elapsed_time(e1)
                return max_over_ranks(tot, dev) / fsteps

            f_ms = timed(lambda: ffh.flow(fa, fb, out=fo, stream=stream))
            full_ms = timed(lambda: (ffh.flow(fa, fb, out=fo, stream=stream),
                                     sgm.scene_flow(imgs, fo["flow"], cam, sfo, flow_valid=fo["valid"],
                                                    stream=stream)))
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
                # two propagation candidates + the fused random-search candidate
                ops += F * lw * lh * P.sweeps * 3 * (2 * r + 1) ** 2 * 8
            lw, lh = (lw + 1) // 2, (lh + 1) // 2
        sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
        peak_ops = 148 * 128 * sm_mhz * 1e6
        prop_ms = fstages["prop"] if fstages else None
        flow_res = {
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
                "traffic": ncu_traffic("ff_prop_kernel"), "algorithmic_ops_per_call": ops,
                "launch_ms_per_call": prop_ms,
                "note": "row-sequential wavefront (left/up dependency): latency-bound, not issue-bound"},
        }
        ffh.close()
        del sfo

    # ---------------- edge-aware densification of the step's scene flow
    # (4 channels, guide = left frame t), timed on its own; its D1/D2/Fl/SF over all pixels
    # are reported by the evaluation section ("All" next to the sparse "Est").
    dens_res = None
    dsf = None
    if not args.no_densify:
        from paper_1801_04720_b200 import densify
        guide = imgs[:, 0, :, :W].contiguous()
        with torch.cuda.stream(stream):
            run_once()
            for _ in range(max(args.warmup, 3)):
                dsf = densify(out["sf"], out["valid_sf"], guide, stream=stream)
            d_ms = 0.0
            dsteps = max(1, min(args.steps, 10))
            for _ in range(dsteps):
                flush_l2()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                dsf = densify(out["sf"], out["valid_sf"], guide, stream=stream)
                e1.record(stream)
                e1.synchronize()
                d_ms += e0.elapsed_time(e1)
        d_ms = max_over_ranks(d_ms, dev) / dsteps
        gaps = int((out["valid_sf"] == 0).sum().item())
        dens_res = {"workload": f"{F} Driving scene flows (4 channels) per GPU, K=25, lambda=1, guide = I_l^t",
                    "ms_per_step": d_ms, "gap_pixels": gaps, "gap_fraction": gaps / float(F * W * H),
                    "gap_pixels_per_s": gaps * world / (d_ms * 1e-3)}

    # ---------------- the evaluation step, timed on its own
    # (not part of the step above): KITTI outlier counts of the step's scene flow
    # against the generator's ground truth, one sgm_evaluate launch per step.
    evaluation = None
    if not args.no_eval:
        from paper_1801_04720_b200 import rates_from_counts
        gd0 = torch.from_numpy(np.stack([q["gt_d0"] for q in quads])).to(dev)
        gd1 = torch.from_numpy(np.stack([q["gt_d1w"] for q in quads])).to(dev)
        noc = torch.from_numpy(np.stack([q["gt_noc"] for q in quads])).to(dev)
        counts = torch.empty((F, 2, 6), dtype=torch.int64, device=dev)
        with torch.cuda.stream(stream):
            run_once()
            for _ in range(max(args.warmup, 3)):
                sgm.evaluate(out["sf"], out["valid_sf"], gd0, gd1, flow, noc, counts=counts,
                             stream=stream)
            ev_ms = 0.0
            for _ in range(args.steps):
                flush_l2()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                sgm.evaluate(out["sf"], out["valid_sf"], gd0, gd1, flow, noc, counts=counts,
                             stream=stream)
                e1.record(stream)
                e1.synchronize()
                ev_ms += e0.elapsed_time(e1)
        ev_ms = max_over_ranks(ev_ms, dev) / args.steps
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
        evaluation = {"metric": "evaluated pixels/s", "value": px * world / (ev_ms * 1e-3),
                      "unit": "px/s", "ms_per_launch": ev_ms, "pixels_per_launch": px,
                      "roofline": {"bound": "hbm", "achieved": gbs, "peak": hbm_peak,
                                   "unit": "GB/s", "frac": gbs / hbm_peak,
                                   "traffic": ncu_traffic("eval_kernel"),
                                   "algorithmic_bytes_per_px": bytes_px},
                      "counts_occ_noc": tot, "rates": rates_from_counts(tot),
                      "rates_densified_all": all_rates}

    gather = None
    if args.gather and pg is not None:
        from paper_1801_04720_b200.dist import gather_results
        torch.cuda.synchronize(dev)
        dist.barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        gathered = gather_results(out, rank, world, dev)
        t1.record()
        t1.synchronize()
        gather = {"ms": max_over_ranks(t0.elapsed_time(t1), dev),
                  "bytes_to_rank0": int(sum(x.numel() * x.element_size() for x in gathered))
                  if gathered else 0}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(synth.CONFIGS["driving"] if cfg.name == "batch" else cfg)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u16x2/int32 (f32 sub-pixel, 3D)",
            "data": "synthetic",
            "config": {"workload": f"{cfg.name}: {F} Driving-scale quads per GPU per step "
                                   f"({W}x{H}, D={D}, census {cfg.cw}x{cfg.ch}, P1={cfg.P1}, "
                                   f"P2={cfg.P2}, 8 paths, LR T={cfg.T}); global batch {F * world}",
                       "quads_per_gpu": F, "global_batch": F * world, "W": W, "H": H, "D": D,
                       "parallelism": f"frames sharded over {world} GPU(s), no collective in step",
                       "l2": "256 MiB buffer written then read between timed steps (flush)",
                       "graph": graph is not None},
            "frames_per_s": frames_per_s,
            "stage_ms": stage_avg,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk,
            "roofline": roof,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "geometry": geo,
            "evaluate": evaluation,
            "stream": stream_res,
            "flow": flow_res,
            "densify": dens_res,
        }
        if gather:
            line["gather"] = gather
        print(json.dumps(line), flush=True)
    sgm.close()
    if pg is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
