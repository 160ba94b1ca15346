"""Seeded synthetic frame quadruples for the five BASELINE.json configs.

This module is the ONLY code shared by the oracle side (tests, bench
cpu_baseline) and the CUDA side: it renders inputs and holds none of the
method's arithmetic (no census, cost, aggregation, WTA, LR, warp or 3D).

The scenes stand in for the paper's KITTI Scene Flow frames, which are
not available here.  Recipe:

* layers: a background (Tiny: fronto-parallel plane d=1, G25; others: road
  plane d(y) = 5 + 85*y/(H-1), G26) plus N fronto-parallel boxes, nearer
  (larger disparity) layers occlude farther ones;
* each layer carries its own texture: U[0,255) noise, Gaussian sigma=1,
  min-max stretched to [0,255] (+ sparse strong edges: line segments of
  width 2 px, value 0 or 255, for the Driving-type configs);
* left view at t samples texture at the layer point; the right view at t
  samples the layer point seen at x_r + d (bilinear in the texture);
* frame t+1: Tiny shifts every layer by (3,1) and adds +1 to every disparity;
  the others apply an ego zoom s=1.02 about the principal point plus a
  per-box translation t_k ~ U[-20,20]^2 and scale every disparity by s (G27);
* flow F(x) = position at t+1 minus position at t of the layer visible at x
  in the left image at t (float32), dense;
* intensities are rounded half-up to uint8.

All randomness is numpy default_rng(seed) (PCG64); generation is float64.
"""
from __future__ import annotations

import dataclasses
import hashlib

import numpy as np
from scipy.ndimage import gaussian_filter

GENERATOR_VERSION = "synth-v1"


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    W: int
    H: int
    D: int
    cw: int
    ch: int
    P1: int
    P2: int
    T: int
    f: float
    B: float
    n_boxes: int
    box_d: tuple
    n_edges: int
    seed: int
    kind: str            # "tiny" or "driving"


CONFIGS = {
    # BASELINE.json configs[0]
    "tiny": Config("tiny", 64, 48, 16, 5, 5, 10, 120, 1, 720.0, 0.54, 3, (2, 5, 9), 0, 0, "tiny"),
    # configs[1]
    "driving": Config("driving", 1242, 375, 128, 9, 7, 7, 86, 1, 720.0, 0.54, 6, (20.0, 120.0),
                      40, 1, "driving"),
    # configs[2]
    "wide": Config("wide", 1242, 375, 256, 9, 7, 7, 86, 1, 720.0, 0.54, 6, (20.0, 250.0),
                   40, 2, "driving"),
    # configs[3]
    "highres": Config("highres", 2048, 1024, 192, 9, 7, 7, 86, 1, 720.0, 0.54, 12, (20.0, 120.0),
                      80, 3, "driving"),
    # configs[4]: 64 Driving-scale quads, seeds 1000..1063
    "batch": Config("batch", 1242, 375, 128, 9, 7, 7, 86, 1, 720.0, 0.54, 6, (20.0, 120.0),
                    40, 1000, "driving"),
}


def sgm_params(cfg: Config) -> dict:
    """Parameters of the method for a config (BASELINE.json; G19 principal point)."""
    return {"D": cfg.D, "cw": cfg.cw, "ch": cfg.ch, "P1": cfg.P1, "P2": cfg.P2, "T": cfg.T,
            "f": cfg.f, "B": cfg.B, "cx": (cfg.W - 1) / 2.0, "cy": (cfg.H - 1) / 2.0,
            "invalid": -1}


def _round_u8(v):
    return np.clip(np.floor(v + 0.5), 0, 255).astype(np.uint8)


def _texture(rng, h, w, n_edges):
    t = rng.uniform(0.0, 255.0, size=(h, w))
    t = gaussian_filter(t, sigma=1.0, mode="reflect")
    lo, hi = t.min(), t.max()
    t = (t - lo) * (255.0 / max(hi - lo, 1e-9))
    for _ in range(n_edges):
        x0, y0 = rng.uniform(0, w), rng.uniform(0, h)
        ang = rng.uniform(0, np.pi)
        length = rng.uniform(20, 120)
        val = 0.0 if rng.uniform() < 0.5 else 255.0
        n = int(length * 2) + 1
        ts = np.linspace(0.0, length, n)
        xs = x0 + np.cos(ang) * ts
        ys = y0 + np.sin(ang) * ts
        # width 2 px: stamp the segment and its +1 neighbour across the normal
        nx, ny = -np.sin(ang), np.cos(ang)
        for off in (0.0, 1.0):
            xi = np.floor(xs + nx * off).astype(int)
            yi = np.floor(ys + ny * off).astype(int)
            ok = (xi >= 0) & (xi < w) & (yi >= 0) & (yi < h)
            t[yi[ok], xi[ok]] = val
    return t


def _sample(tex, margin, u, v):
    """Bilinear texture lookup at layer coordinates (u, v) (texture origin at -margin)."""
    h, w = tex.shape
    uu = np.clip(u + margin, 0.0, w - 1.000001)
    vv = np.clip(v + margin, 0.0, h - 1.000001)
    x0 = np.floor(uu).astype(np.int64)
    y0 = np.floor(vv).astype(np.int64)
    fx = uu - x0
    fy = vv - y0
    a = tex[y0, x0]
    b = tex[y0, x0 + 1]
    c = tex[y0 + 1, x0]
    d = tex[y0 + 1, x0 + 1]
    return (a * (1 - fx) * (1 - fy) + b * fx * (1 - fy) + c * (1 - fx) * fy + d * fx * fy)


class _Layer:
    """A planar scene layer: footprint (left view, frame t), disparity model, motion."""

    def __init__(self, rect, d_const, plane, tex, margin, shift, zoom, dscale, dadd, centre):
        self.rect = rect            # (x0, y0, x1, y1) or None for the background
        self.d_const = d_const      # constant disparity (boxes / tiny background)
        self.plane = plane          # (a, b): d(y) = a + b*y for the road plane, else None
        self.tex = tex
        self.margin = margin
        self.shift = np.asarray(shift, np.float64)   # translation t_k at t+1
        self.zoom = zoom                              # ego zoom s at t+1
        self.dscale = dscale                          # disparity factor at t+1
        self.dadd = dadd                              # disparity offset at t+1
        self.c = np.asarray(centre, np.float64)

    # frame-t layer point p  <->  image point q of a frame with motion amount u (left
    # view): q = c + zoom^u (p - c) + u * shift.  u = 0 is frame t, u = 1 frame t+1 of a
    # quad; videos (make_video) visit u = 0, 1, 2, 1, 0, ...
    def to_t(self, qx, qy, frame):
        if frame == 0:
            return qx, qy
        s = self.zoom ** frame
        px = self.c[0] + (qx - self.c[0] - self.shift[0] * frame) / s
        py = self.c[1] + (qy - self.c[1] - self.shift[1] * frame) / s
        return px, py

    def from_t(self, px, py, frame):
        if frame == 0:
            return px, py
        s = self.zoom ** frame
        return (self.c[0] + s * (px - self.c[0]) + self.shift[0] * frame,
                self.c[1] + s * (py - self.c[1]) + self.shift[1] * frame)

    def covers(self, px, py):
        if self.rect is None:
            return np.ones(np.broadcast(px, py).shape, bool)
        x0, y0, x1, y1 = self.rect
        return (px >= x0) & (px < x1) & (py >= y0) & (py < y1)

    def disp_t(self, py):
        if self.plane is not None:
            return self.plane[0] + self.plane[1] * py
        return np.full(np.shape(py), float(self.d_const))

    def disp(self, py, frame):
        d = self.disp_t(py)
        return d if frame == 0 else d * self.dscale ** frame + self.dadd * frame


def _render(layers, W, H, frame):
    """Left and right images, GT disparity of the left view, visible-layer index."""
    ys, xs = np.mgrid[0:H, 0:W].astype(np.float64)
    best_d = np.full((H, W), -np.inf)
    left = np.zeros((H, W))
    lid = np.full((H, W), -1, np.int64)
    for k, L in enumerate(layers):
        px, py = L.to_t(xs, ys, frame)
        cov = L.covers(px, py)
        d = L.disp(py, frame)
        take = cov & (d > best_d)
        best_d = np.where(take, d, best_d)
        left = np.where(take, _sample(L.tex, L.margin, px, py), left)
        lid = np.where(take, k, lid)
    # right view: pixel x_r shows the nearest layer point whose left-view position is x_r + d
    best_r = np.full((H, W), -np.inf)
    right = np.zeros((H, W))
    for L in layers:
        # the row of a layer point is unchanged between views; its disparity depends on the
        # frame-t row only, so compute it from the left-view row y
        _, py_row = L.to_t(xs, ys, frame)
        d = L.disp(py_row, frame)
        xl = xs + d
        px, py = L.to_t(xl, ys, frame)
        cov = L.covers(px, py)
        take = cov & (d > best_r)
        best_r = np.where(take, d, best_r)
        right = np.where(take, _sample(L.tex, L.margin, px, py), right)
    return _round_u8(left), _round_u8(right), best_d.astype(np.float32), lid


def make_quad(cfg: Config | str, index: int = 0) -> dict:
    """One seeded frame quadruple (il0, ir0, il1, ir1 uint8 [H][W]; flow float32 [H][W][2];
    ground-truth disparities gt_d0, gt_d1 float32 [H][W] of the left views)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    seed = cfg.seed + index
    W, H = cfg.W, cfg.H
    layers = _build_layers(cfg, np.random.default_rng(seed))
    il0, ir0, gt_d0, lid0 = _render(layers, W, H, 0)
    il1, ir1, gt_d1, lid1 = _render(layers, W, H, 1)
    flow, gt_d1w, noc = _motion(layers, W, H, 0, 1, lid0, lid1)
    return {"il0": il0, "ir0": ir0, "il1": il1, "ir1": ir1,
            "flow": flow, "gt_d0": gt_d0, "gt_d1": gt_d1, "gt_d1w": gt_d1w, "gt_noc": noc,
            "config": cfg.name, "seed": seed}


def _build_layers(cfg: Config, rng) -> list:
    W, H = cfg.W, cfg.H
    centre = ((W - 1) / 2.0, (H - 1) / 2.0)
    dmax = cfg.D + 8
    margin = int(dmax + 64 + 0.05 * max(W, H))
    tw, th = W + 2 * margin, H + 2 * margin
    layers = []
    if cfg.kind == "tiny":
        shift, zoom, dscale, dadd = (3.0, 1.0), 1.0, 1.0, 1.0
        layers.append(_Layer(None, 1.0, None, _texture(rng, th, tw, 0), margin,
                             shift, zoom, dscale, dadd, centre))
        for dk in cfg.box_d:                      # painted far-to-near
            bw, bh = rng.integers(12, 25), rng.integers(10, 21)
            x0 = rng.integers(dk + 2, W - bw - 4)
            y0 = rng.integers(2, H - bh - 3)
            layers.append(_Layer((x0, y0, x0 + bw, y0 + bh), float(dk), None,
                                 _texture(rng, th, tw, 0), margin, shift, zoom, dscale, dadd,
                                 centre))
    else:
        zoom = 1.02
        layers.append(_Layer(None, None, (5.0, 85.0 / (H - 1)),
                             _texture(rng, th, tw, cfg.n_edges), margin, (0.0, 0.0), zoom,
                             zoom, 0.0, centre))
        boxes = []
        for _ in range(cfg.n_boxes):
            dk = rng.uniform(cfg.box_d[0], cfg.box_d[1])
            bw = rng.uniform(0.05, 0.2) * W
            bh = rng.uniform(0.1, 0.4) * H
            x0 = rng.uniform(0, W - bw)
            y0 = rng.uniform(0, H - bh)
            t = rng.uniform(-20.0, 20.0, size=2)
            boxes.append((dk, (x0, y0, x0 + bw, y0 + bh), t))
        boxes.sort(key=lambda b: b[0])
        for dk, rect, t in boxes:
            layers.append(_Layer(rect, dk, None, _texture(rng, th, tw, max(cfg.n_edges // 8, 1)),
                                 margin, t, zoom, zoom, 0.0, centre))
    return layers


def _motion(layers, W, H, ua, ub, lid_a, lid_b):
    """Flow from the frame with motion amount ua to the one with ub, the disparity at ub
    of the point seen at each pixel of ua, and the non-occluded mask."""
    ys, xs = np.mgrid[0:H, 0:W].astype(np.float64)
    flow = np.zeros((H, W, 2), np.float64)
    gt_d1w = np.zeros((H, W), np.float64)
    for k, L in enumerate(layers):
        m = lid_a == k
        px, py = L.to_t(xs[m], ys[m], ua)       # layer point seen at x in frame ua
        qx, qy = L.from_t(px, py, ub)
        flow[m, 0] = qx - xs[m]
        flow[m, 1] = qy - ys[m]
        gt_d1w[m] = L.disp(py, ub)              # disparity at ub of the point seen at x
    # non-occluded: the point seen at x lands inside the image in frame ub and is the
    # visible layer there (KITTI "noc" semantics, P:131 / Table 1 caption)
    qx = np.floor(xs + flow[..., 0] + 0.5).astype(np.int64)
    qy = np.floor(ys + flow[..., 1] + 0.5).astype(np.int64)
    inside = (qx >= 0) & (qx < W) & (qy >= 0) & (qy < H)
    noc = np.zeros((H, W), bool)
    noc[inside] = lid_b[qy[inside], qx[inside]] == lid_a[inside]
    return flow.astype(np.float32), gt_d1w.astype(np.float32), noc.astype(np.uint8)


# motion amount of video frame k (bounded, so disparities stay inside [0, D-1])
VIDEO_MOTION = (0, 1, 2, 1)


def make_video(cfg: Config | str, n_quads: int, index: int = 0) -> dict:
    """A seeded stereo video of n_quads + 1 frames for the streaming mode (SURVEY 8(f)
    rank 3): the scene of make_quad(cfg, index), with motion amount
    VIDEO_MOTION[k % 4] at frame k, so frames 0 and 1 are exactly that quad's.
    left, right uint8 [n+1][H][W]; flow float32 [n][H][W][2] (frame k -> k+1); gt_d
    float32 [n+1][H][W]; gt_d1w float32 [n][H][W] (disparity at k+1 of the point seen at
    x in frame k); gt_noc uint8 [n][H][W]."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    seed = cfg.seed + index
    W, H = cfg.W, cfg.H
    layers = _build_layers(cfg, np.random.default_rng(seed))
    us = [VIDEO_MOTION[k % len(VIDEO_MOTION)] for k in range(n_quads + 1)]
    frames = [_render(layers, W, H, u) for u in us]
    out = {"left": np.stack([f[0] for f in frames]), "right": np.stack([f[1] for f in frames]),
           "gt_d": np.stack([f[2] for f in frames]), "config": cfg.name, "seed": seed,
           "motion": us}
    flows, d1w, nocs = [], [], []
    for k in range(n_quads):
        f, d, m = _motion(layers, W, H, us[k], us[k + 1], frames[k][3], frames[k + 1][3])
        flows.append(f); d1w.append(d); nocs.append(m)
    out.update(flow=np.stack(flows), gt_d1w=np.stack(d1w), gt_noc=np.stack(nocs))
    return out


def video_quad(video: dict, k: int) -> dict:
    """Quad k of a video as a make_quad-style dict (frames k and k+1)."""
    return {"il0": video["left"][k], "ir0": video["right"][k], "il1": video["left"][k + 1],
            "ir1": video["right"][k + 1], "flow": video["flow"][k],
            "gt_d0": video["gt_d"][k], "gt_d1": video["gt_d"][k + 1],
            "gt_d1w": video["gt_d1w"][k], "gt_noc": video["gt_noc"][k]}


def make_batch(cfg: Config | str, start: int, count: int, workers: int = 1) -> list:
    """Quads start .. start+count-1 of a config; `workers` > 1 generates them in a process
    pool (forked, or spawned once CUDA is initialised in this process)."""
    idx = [start + i for i in range(count)]
    if workers <= 1 or count <= 1:
        return [make_quad(cfg, i) for i in idx]
    import multiprocessing as mp
    method = "fork"
    try:
        import torch
        if torch.cuda.is_initialized():
            method = "spawn"
    except Exception:  # pragma: no cover - torch is optional for the generator
        pass
    with mp.get_context(method).Pool(min(workers, count)) as pool:
        return pool.starmap(make_quad, [(cfg, i) for i in idx])


def manifest(quad: dict) -> dict:
    """SHA-256 of every array of a quad (generator version stamped)."""
    out = {"generator": GENERATOR_VERSION, "config": quad["config"], "seed": quad["seed"]}
    for k in ("il0", "ir0", "il1", "ir1", "flow"):
        out[k] = hashlib.sha256(np.ascontiguousarray(quad[k]).tobytes()).hexdigest()
    return out


# --- small inputs for parity tests (random images of arbitrary size) ---------------

def random_pair(W, H, seed, shift=None, smooth=True):
    """Smoothed-noise left image and a right image that is the left one shifted by
    ``shift`` px (integer) -- the constant-disparity pair of the north-star invariant
    -- or an independent smoothed-noise image when ``shift`` is None."""
    rng = np.random.default_rng(seed)
    pad = 0 if shift is None else int(shift)
    t = rng.uniform(0.0, 255.0, size=(H, W + pad))
    if smooth:
        t = gaussian_filter(t, sigma=1.0, mode="reflect")
        t = (t - t.min()) * (255.0 / max(t.max() - t.min(), 1e-9))
    if shift is None:
        left = _round_u8(t[:, :W])
        t2 = rng.uniform(0.0, 255.0, size=(H, W))
        if smooth:
            t2 = gaussian_filter(t2, sigma=1.0, mode="reflect")
            t2 = (t2 - t2.min()) * (255.0 / max(t2.max() - t2.min(), 1e-9))
        right = _round_u8(t2)
        return left, right
    # left(x) = t(x); right(x) = t(x + shift), so left(x) = right(x - shift):
    # every left pixel has disparity ``shift``
    left = _round_u8(t[:, 0:W])
    right = _round_u8(t[:, pad:pad + W])
    return left, right


def random_flow(W, H, seed, scale=8.0, integer=False):
    rng = np.random.default_rng(seed)
    f = rng.uniform(-scale, scale, size=(H, W, 2))
    if integer:
        f = np.round(f)
    return f.astype(np.float32)


def random_eval_instance(H, W, seed, n=None):
    """Seeded estimate + ground truth for the evaluation step ("random
    instances"): GT disparities in [0, 80), GT flow ~ N(0, 15); the estimate is the GT
    plus a per-channel error drawn from {0, N(0,1), N(0,4), N(0,30)} (40/30/20/10 %),
    so every outlier decision is exercised; ~80 % est-valid, ~90 % GT-valid, ~85 % of
    those non-occluded.  Leading batch axis ``n`` if given."""
    rng = np.random.default_rng(seed)
    shp = (H, W) if n is None else (n, H, W)
    gd0 = rng.uniform(0, 80, shp).astype(np.float32)
    gd1 = rng.uniform(0, 80, shp).astype(np.float32)
    gfl = rng.normal(0, 15, shp + (2,)).astype(np.float32)
    scale = rng.choice([0.0, 1.0, 4.0, 30.0], size=shp + (4,), p=[0.4, 0.3, 0.2, 0.1])
    sf = np.stack([gfl[..., 0], gfl[..., 1], gd0, gd1], -1) + \
        (scale * rng.normal(0, 1, shp + (4,))).astype(np.float32)
    v = (rng.random(shp) < 0.8).astype(np.uint8)
    gv = (rng.random(shp) < 0.9).astype(np.uint8)
    noc = ((rng.random(shp) < 0.85) & (gv > 0)).astype(np.uint8)
    return {"sf": sf.astype(np.float32), "valid_sf": v, "gt_d0": gd0, "gt_d1": gd1,
            "gt_flow": gfl, "gt_noc": noc, "gt_valid": gv}


def translated_pair(W, H, seed, tx, ty, sigma=1.0):
    """Frames A, B of a textured plane translated by the integer (tx, ty): the point at x
    in A appears at x + (tx, ty) in B, so the true flow A -> B is (tx, ty) wherever
    x + (tx, ty) is inside the image ("exact-translation recovery")."""
    rng = np.random.default_rng(seed)
    m = 16 + max(abs(tx), abs(ty))
    t = rng.uniform(0.0, 255.0, size=(H + 2 * m, W + 2 * m))
    t = gaussian_filter(t, sigma=sigma, mode="reflect")
    t = (t - t.min()) * (255.0 / max(t.max() - t.min(), 1e-9))
    A = _round_u8(t[m:m + H, m:m + W])
    B = _round_u8(t[m - ty:m - ty + H, m - tx:m - tx + W])
    return A, B
