"""Time the optical-flow core on Driving-size pairs: python tools/flow_timing.py [n] [levels]"""
import hashlib
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import synth  # noqa: E402
from paper_1801_04720_b200 import FlowFields  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
levels = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = synth.CONFIGS["driving"]
quads = [synth.make_quad(cfg, k) for k in range(n)]
dev = torch.device("cuda", 0)
A = torch.from_numpy(np.stack([q["il0"] for q in quads])).to(dev)
B = torch.from_numpy(np.stack([q["il1"] for q in quads])).to(dev)
ff = FlowFields(cfg.W, cfg.H, levels=levels, max_batch=n)
out = ff.flow(A, B)
torch.cuda.synchronize()
for _ in range(2):
    ff.flow(A, B, out=out)
torch.cuda.synchronize()
t0 = time.perf_counter()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
reps = 5
for _ in range(reps):
    ff.flow(A, B, out=out)
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1) / reps
ff.set_timing(True)
ff.flow(A, B, out=out)
torch.cuda.synchronize()
print("stage ms", ff.read_timing())
ff.set_timing(False)
fl = out["flow"].cpu().numpy()
v = out["valid"].cpu().numpy() > 0
gt = np.stack([q["flow"] for q in quads])
epe = np.hypot(*(fl - gt).transpose(3, 0, 1, 2))
print(f"n={n} levels={levels}: {ms:.2f} ms per call, {ms / n:.3f} ms per pair; "
      f"valid {v.mean():.3f}; EPE<=1 on valid {(epe[v] <= 1).mean():.3f}; "
      f"launches/call {ff.launch_count() / (reps + 3):.0f}")
print("digest", hashlib.sha256(out["flow"].cpu().numpy().tobytes() + out["valid"].cpu().numpy().tobytes()).hexdigest()[:16])
