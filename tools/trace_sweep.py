"""Timeline of the sweep CTAs/warps (debug): python tools/trace_sweep.py [quads]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1801_04720_b200 import SGM, Camera, stack_quads  # noqa: E402

F = int(sys.argv[1]) if len(sys.argv) > 1 else 8
cfg = synth.CONFIGS["batch"]
g = SGM.from_config(cfg, max_batch=F)
geo = g.geometry()
nw = geo["sweep_warps"]
nb = (cfg.H + geo["band_rows"] - 1) // geo["band_rows"]
ncta = 4 * F * nb
print("band rows", geo["band_rows"], "bands", nb)
tr = torch.zeros(4 * F * ((cfg.H + 9) // 10) * (nw + 1) * 4, dtype=torch.int64, device="cuda")
g.lib.sgm_debug_set_trace(g.h, ctypes.c_void_p(tr.data_ptr()))
quads = [synth.make_quad(cfg, i) for i in range(F)]
imgs, flow = stack_quads(quads, g.pitch, torch.device("cuda"))
prm = synth.sgm_params(cfg)
cam = Camera(prm["f"], prm["B"], prm["cx"], prm["cy"])
out = g.alloc_outputs(F)
for _ in range(3):
    g.scene_flow(imgs, flow, cam, out)
torch.cuda.synchronize()
t = tr.cpu().numpy()[:ncta * (nw + 1) * 4].reshape(ncta, nw + 1, 4).astype(np.float64)
# the backward sweep ran last: its timeline is in the buffer
t0 = t[:, :nw, 0][t[:, :nw, 0] > 0].min()
st = (t[:, :nw, 0] - t0) / 1e3
en = (t[:, :nw, 1] - t0) / 1e3
dur = en - st
valid = t[:, :nw, 0] > 0
print(f"CTAs {ncta}, warps/CTA {nw}; kernel span {en[valid].max():.1f} us")
print(f"warp loop duration us: median {np.median(dur[valid]):.1f}  min {dur[valid].min():.1f}  max {dur[valid].max():.1f}")
print(f"per-position period (median) ns: {np.median(dur[valid]) * 1e3 / cfg.W:.1f}")
cs = st[:, 0]
ce = en.max(axis=1)
print("CTA start us (first 10 tickets):", np.round(cs[:10], 1))
print("CTA start us by wave (ticket 148k):", np.round(cs[::148], 1))
print("warp start offsets within CTA 0 (us):", np.round(st[0] - st[0, 0], 2))
print("warp end offsets within CTA 0 (us):", np.round(en[0] - en[0, 0], 2))
conc = []
for tt in np.linspace(0, en[valid].max(), 20):
    conc.append(int(((cs <= tt) & (ce >= tt)).sum()))
print("resident CTAs over time:", conc)
sm = t[:, 0, 2].astype(int)
print("distinct SMs used:", len(set(sm.tolist())))
# --- per-CTA span vs per-warp work, per-row start lag, band start lag
span = en.max(axis=1) - st.min(axis=1)
print(f"CTA span median {np.median(span):.1f} us; warp loop median {np.median(dur[valid]):.1f} us")
rowlag = np.diff(st, axis=1)[:, :]
print(f"per-row start lag median {np.median(rowlag):.2f} us = {np.median(rowlag) * 1e3 / (np.median(dur[valid]) * 1e3 / cfg.W):.1f} positions")
nv = 4 * F
bandstart = st[:, 0].reshape(-1, nv)   # [band][view]
bl = np.diff(bandstart, axis=0)
print(f"band-to-band start lag median {np.median(bl):.2f} us")
# time when each SM was busy: union of CTA spans per SM (valid warps only)
stv = np.where(valid, st, np.inf).min(axis=1)
env = np.where(valid, en, -np.inf).max(axis=1)
ok = np.isfinite(stv) & np.isfinite(env)
busy = 0.0
sms = t[:, 0, 2].astype(int)
span = env[ok].max()
for smid in set(sms[ok].tolist()):
    sel = ok & (sms == smid)
    iv = sorted(zip(stv[sel], env[sel]))
    cur_s, cur_e = iv[0]
    for a, b in iv[1:]:
        if a > cur_e:
            busy += cur_e - cur_s
            cur_s, cur_e = a, b
        else:
            cur_e = max(cur_e, b)
    busy += cur_e - cur_s
nsm = len(set(sms[ok].tolist()))
print(f"SM busy fraction over the kernel span: {busy / (nsm * span):.3f}")
# per band index: mean warp-loop duration (includes waiting for the band above)
nb_ = ncta // (4 * F)
dur_c = np.where(valid, dur, np.nan)
mean_by_band = [np.nanmean(dur_c[b * 4 * F:(b + 1) * 4 * F]) for b in range(nb_)]
print("mean warp loop us by band:", np.round(mean_by_band, 0))
