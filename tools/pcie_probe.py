import time, torch
x = torch.empty(186_300_000, dtype=torch.uint8, device="cuda")
h = torch.empty(186_300_000, dtype=torch.uint8, pin_memory=True)
for _ in range(3):
    h.copy_(x, non_blocking=True); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); h.copy_(x, non_blocking=True); e1.record(); e1.synchronize()
print("D2H 186 MB pinned: %.2f ms  %.1f GB/s" % (e0.elapsed_time(e1), 186.3e6 / e0.elapsed_time(e1) / 1e6))
e0.record(); x.copy_(h, non_blocking=True); e1.record(); e1.synchronize()
print("H2D 186 MB pinned: %.2f ms  %.1f GB/s" % (e0.elapsed_time(e1), 186.3e6 / e0.elapsed_time(e1) / 1e6))
