"""Digest of the scene-flow outputs of a tree for bitwise A/B comparison (run from the tree):
cd ab/<v> && python ../../tools/ab_dump.py <out.json>  (sha256 per output array)"""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1801_04720_b200 import SGM, Camera, stack_quads  # noqa: E402

res = {}
for name, n in (("driving", 3), ("wide", 1), ("highres", 1), ("tiny", 5), ("driving", 40)):
    cfg = synth.CONFIGS[name]
    prm = synth.sgm_params(cfg)
    quads = [synth.make_quad(cfg, 100 + i) for i in range(min(n, 3))]
    quads = [quads[i % len(quads)] for i in range(n)]
    g = SGM.from_config(cfg, max_batch=n, device=0)
    imgs, flow = stack_quads(quads, g.pitch, torch.device("cuda", 0))
    out = g.scene_flow(imgs, flow, Camera(prm["f"], prm["B"], prm["cx"], prm["cy"]))
    torch.cuda.synchronize()
    for k in ("disp_int", "disp_sub", "disp_valid", "sf", "valid_sf"):
        res[f"{name}{n}_{k}"] = hashlib.sha256(np.ascontiguousarray(out[k].cpu().numpy()).tobytes()).hexdigest()
    g.close()
json.dump(res, open(sys.argv[1], "w"), indent=1)
print("dumped", sys.argv[1])
