"""Fidelity of the windowed densification against the SPEC's F-6 (every seed competes) on
full-size Driving scene flows: GPU sgm_densify with candidate windows 4..32 (time, certified
fraction) and, at sampled gap pixels, the oracle with window 0 (exact F-6) vs the windowed
result.  Run on the GPU box:  python tools/densify_gap.py [n_quads] [n_points]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_1801_04720_b200 import SGM, Camera, densify, stack_quads  # noqa: E402


def main():
    nq = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    npts = int(sys.argv[2]) if len(sys.argv) > 2 else 24
    cfg = synth.CONFIGS["driving"]
    prm = synth.sgm_params(cfg)
    quads = synth.make_batch(cfg, 0, nq, workers=nq)
    dev = torch.device("cuda", 0)
    g = SGM.from_config(cfg, max_batch=nq)
    imgs, flow = stack_quads(quads, g.pitch, dev)
    out = g.scene_flow(imgs, flow, Camera(prm["f"], prm["B"], prm["cx"], prm["cy"]))
    guide = imgs[:, 0, :, :cfg.W].contiguous()
    gaps = int((out["valid_sf"] == 0).sum().item())
    res = {}
    for window in (4, 8, 16, 32):
        densify(out["sf"], out["valid_sf"], guide, window=window)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d, cert = densify(out["sf"], out["valid_sf"], guide, window=window, count_certified=True)
        e1.record()
        e1.synchronize()
        res[window] = d[0].cpu().numpy()
        print(f"window {window:2d}: {e0.elapsed_time(e1):8.2f} ms for {nq} scene flows, "
              f"certified {int(cert.item()) / gaps:.3f} of {gaps} gap pixels", flush=True)
    sf = out["sf"][0].cpu().numpy()
    v = out["valid_sf"][0].cpu().numpy()
    gd = np.argwhere(v == 0)
    rng = np.random.default_rng(0)
    pick = gd[rng.choice(len(gd), npts, replace=False)]
    xy = np.stack([pick[:, 1], pick[:, 0]], 1).astype(np.int32)
    t0 = time.time()
    exact = oracle.densify_points(sf, v, quads[0]["il0"], xy, window=0)
    print(f"exact F-6 oracle at {npts} points: {time.time() - t0:.1f} s", flush=True)
    for window, d in res.items():
        got = d[pick[:, 0], pick[:, 1]].astype(np.float64)
        err = np.abs(got - exact)
        same = (err <= 1e-4 * np.maximum(1, np.abs(exact))).all(1)
        print(f"window {window:2d}: equal to exact F-6 at {same.sum()}/{npts} points; max |diff| "
              f"u,v {err[:, :2].max():.3f} px, d0,d1 {err[:, 2:].max():.3f} px; median "
              f"{np.median(err[~same]) if (~same).any() else 0:.4f}", flush=True)
    g.close()


if __name__ == "__main__":
    main()
