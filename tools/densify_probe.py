"""Time / profile sgm_densify on the scene flow of 8 Driving quads: python tools/densify_probe.py"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_1801_04720_b200 import SGM, Camera, densify, stack_quads  # noqa: E402

cfg = synth.CONFIGS["driving"]
prm = synth.sgm_params(cfg)
dev = torch.device("cuda", 0)
quads = [synth.make_quad(cfg, k) for k in range(8)]
g = SGM.from_config(cfg, max_batch=8)
imgs, flow = stack_quads(quads, g.pitch, dev)
out = g.scene_flow(imgs, flow, Camera(prm["f"], prm["B"], prm["cx"], prm["cy"]))
guide = imgs[:, 0, :, :cfg.W].contiguous()
for _ in range(3):
    d = densify(out["sf"], out["valid_sf"], guide)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    d = densify(out["sf"], out["valid_sf"], guide)
e1.record()
e1.synchronize()
v = out["valid_sf"].cpu().numpy()
print(f"densify: {e0.elapsed_time(e1) / 5:.3f} ms; gaps {int((v == 0).sum())}; "
      f"gap columns per row (mean) {(v == 0).sum(2).mean():.1f}")
