"""Per-pixel step latency of the propagation kernel: one field, one band (H=16) and a
full-height field, timed through sgm_flow_sweep (prop + search) with CUDA events."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import oracle  # noqa: E402
from paper_1801_04720_b200 import FlowFields  # noqa: E402

dev = torch.device("cuda", 0)
for (W, H) in [(1242, 16), (1242, 375), (311, 94)]:
    A, B = synth.translated_pair(W, H, 1, 3, 1)
    ff = FlowFields(W, H, search_radius=1)
    gA, gB = torch.from_numpy(A).to(dev), torch.from_numpy(B).to(dev)
    rng = np.random.default_rng(0)
    f0 = torch.from_numpy(rng.integers(-16, 17, size=(H, W, 2)).astype(np.int32)).to(dev)
    c0 = torch.full((H, W), 1 << 30, dtype=torch.int32, device=dev)
    ff.set_timing(False)
    for s in range(3):
        f, c = f0.clone(), c0.clone()
        ff.sweep(gA, gB, f, c, 0)
    torch.cuda.synchronize()
    ts = []
    for s in range(5):
        f, c = f0.clone(), c0.clone()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ff.sweep(gA, gB, f, c, 0)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts)
    print(f"{W}x{H}: sweep {ms:.3f} ms; per step (W+H) {ms * 1e6 / (W + H):.0f} ns")
    ff.close()
