"""ctypes marshalling for oracle/sgm_oracle.c (test infrastructure only).

No arithmetic of the method lives here: every function allocates numpy outputs,
passes pointers to the C oracle and returns the arrays.  See sgm_oracle.c for
the citations of each step.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sgm_oracle.c")
_SRCS = [_SRC, os.path.join(_HERE, "flow_oracle.c")]
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def lib_path() -> str:
    return _LIB


def build(force: bool = False) -> str:
    """Compile sgm_oracle.c with gcc -O2 -ffp-contract=off (no SIMD intrinsics)."""
    if force or not os.path.exists(_LIB) or \
            os.path.getmtime(_LIB) < max(os.path.getmtime(s) for s in _SRCS):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared",
                               "-std=c11", "-o", tmp, *_SRCS, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _get():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            P = ctypes.c_void_p
            I = ctypes.c_int
            L = ctypes.c_int64
            Dd = ctypes.c_double
            lib.orc_census.argtypes = [P, I, I, L, I, I, P]
            lib.orc_cost.argtypes = [P, P, I, I, I, I, I, P]
            lib.orc_path.argtypes = [P, I, I, I, I, I, I, I, P]
            lib.orc_aggregate.argtypes = [P, I, I, I, I, I, P]
            lib.orc_wta.argtypes = [P, I, I, I, P, P]
            lib.orc_lr_check.argtypes = [P, P, P, I, I, I, I, P, P, P]
            lib.orc_sgm_view.argtypes = [P, P, I, I, I, I, I, I, I, P, P, P, P]
            lib.orc_disparity.argtypes = [P, P, I, I, L, I, I, I, I, I, I, I,
                                          P, P, P, P, P, P, P]
            lib.orc_combine.argtypes = [P, P, P, P, P, P, I, I, I, P, P]
            lib.orc_reproject.argtypes = [P, P, I, I, Dd, Dd, Dd, Dd, P, P, P, P]
            U64 = ctypes.c_uint64
            lib.orc_ff_downsample.argtypes = [P, I, I, P]
            lib.orc_ff_wht.argtypes = [P, I, I, I, P]
            lib.orc_ff_patch_cost.argtypes = [P, P, I, I, I, I, I, I, I, I]
            lib.orc_ff_patch_cost.restype = ctypes.c_int32
            lib.orc_ff_knn_init.argtypes = [P, P, I, I, I, I, I, I, P, P, P]
            lib.orc_ff_rng.argtypes = [U64, I, I, I, I]
            lib.orc_ff_rng.restype = U64
            lib.orc_ff_sweep.argtypes = [P, P, I, I, I, I, I, I, I, U64, P, P]
            lib.orc_ff_lift.argtypes = [P, P, I, I, I, I, P, I, I, P, P]
            lib.orc_ff_field.argtypes = [P, P, I, I, I, I, I, I, I, I, I, U64, P, P]
            lib.orc_ff_consistency.argtypes = [P, P, P, I, I, I, P]
            lib.orc_ff_flow.argtypes = [P, P, I, I, I, I, I, I, I, I, I, U64, I, P, P]
            lib.orc_edge_distance.argtypes = [P, I, I, I, I, I, I, Dd]
            lib.orc_edge_distance.restype = Dd
            Fl = ctypes.c_float
            lib.orc_densify.argtypes = [P, P, P, I, I, I, I, Fl, I, P]
            lib.orc_densify.restype = ctypes.c_int
            lib.orc_densify_points.argtypes = [P, P, P, I, I, I, I, Fl, I, I, P, P]
            lib.orc_densify_points.restype = ctypes.c_int
            for fn in ("orc_ff_downsample", "orc_ff_wht", "orc_ff_knn_init", "orc_ff_sweep",
                       "orc_ff_lift", "orc_ff_field", "orc_ff_consistency", "orc_ff_flow"):
                getattr(lib, fn).restype = ctypes.c_int
            lib.orc_evaluate.argtypes = [P, P, P, P, P, P, P, I, I, ctypes.c_float, ctypes.c_float, P]
            for fn in ("orc_census", "orc_cost", "orc_path", "orc_aggregate", "orc_wta",
                       "orc_lr_check", "orc_sgm_view", "orc_disparity", "orc_combine",
                       "orc_reproject", "orc_evaluate"):
                getattr(lib, fn).restype = ctypes.c_int
            _lib = lib
    return _lib


def _p(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def _chk(rc, what):
    if rc != 0:
        raise ValueError(f"oracle {what} failed with code {rc}")


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def census(img, cw, ch):
    img = _c(img, np.uint8)
    H, W = img.shape
    out = np.empty((H, W), np.uint64)
    _chk(_get().orc_census(_p(img), W, H, W, cw, ch, _p(out)), "census")
    return out


def cost(cen_ref, cen_match, D, s, cmax):
    cen_ref = _c(cen_ref, np.uint64)
    cen_match = _c(cen_match, np.uint64)
    H, W = cen_ref.shape
    out = np.empty((H, W, D), np.uint8)
    _chk(_get().orc_cost(_p(cen_ref), _p(cen_match), W, H, D, s, cmax, _p(out)), "cost")
    return out


def path(cost_vol, P1, P2, rx, ry):
    cost_vol = _c(cost_vol, np.uint8)
    H, W, D = cost_vol.shape
    out = np.empty((H, W, D), np.int32)
    _chk(_get().orc_path(_p(cost_vol), W, H, D, P1, P2, rx, ry, _p(out)), "path")
    return out


def aggregate(cost_vol, P1, P2):
    cost_vol = _c(cost_vol, np.uint8)
    H, W, D = cost_vol.shape
    out = np.empty((H, W, D), np.uint32)
    _chk(_get().orc_aggregate(_p(cost_vol), W, H, D, P1, P2, _p(out)), "aggregate")
    return out


def wta(S):
    S = _c(S, np.uint32)
    H, W, D = S.shape
    di = np.empty((H, W), np.int16)
    ds = np.empty((H, W), np.float64)
    _chk(_get().orc_wta(_p(S), W, H, D, _p(di), _p(ds)), "wta")
    return di, ds


def lr_check(dl_int, dl_sub, dr_int, T, invalid=-1):
    dl_int = _c(dl_int, np.int16)
    dl_sub = _c(dl_sub, np.float64)
    dr_int = _c(dr_int, np.int16)
    H, W = dl_int.shape
    oi = np.empty((H, W), np.int16)
    os_ = np.empty((H, W), np.float64)
    v = np.empty((H, W), np.uint8)
    _chk(_get().orc_lr_check(_p(dl_int), _p(dl_sub), _p(dr_int), W, H, T, invalid,
                             _p(oi), _p(os_), _p(v)), "lr_check")
    return oi, os_, v


def sgm_view(cen_ref, cen_match, D, s, cmax, P1, P2, want_cost=False, want_S=False):
    cen_ref = _c(cen_ref, np.uint64)
    cen_match = _c(cen_match, np.uint64)
    H, W = cen_ref.shape
    di = np.empty((H, W), np.int16)
    ds = np.empty((H, W), np.float64)
    C = np.empty((H, W, D), np.uint8) if want_cost else None
    S = np.empty((H, W, D), np.uint32) if want_S else None
    _chk(_get().orc_sgm_view(_p(cen_ref), _p(cen_match), W, H, D, s, cmax, P1, P2,
                             _p(di), _p(ds), _p(C), _p(S)), "sgm_view")
    return di, ds, C, S


def disparity(left, right, D, cw, ch, P1, P2, T, invalid=-1):
    """Full SGM on one rectified pair.  Returns dict with LR-checked and raw maps."""
    left = _c(left, np.uint8)
    right = _c(right, np.uint8)
    H, W = left.shape
    out = {
        "d_int": np.empty((H, W), np.int16), "d_sub": np.empty((H, W), np.float64),
        "valid": np.empty((H, W), np.uint8),
        "dl_int": np.empty((H, W), np.int16), "dl_sub": np.empty((H, W), np.float64),
        "dr_int": np.empty((H, W), np.int16), "dr_sub": np.empty((H, W), np.float64),
    }
    _chk(_get().orc_disparity(_p(left), _p(right), W, H, W, D, cw, ch, P1, P2, T, invalid,
                              _p(out["d_int"]), _p(out["d_sub"]), _p(out["valid"]),
                              _p(out["dl_int"]), _p(out["dl_sub"]),
                              _p(out["dr_int"]), _p(out["dr_sub"])), "disparity")
    return out


def combine(d0, v0, d1, v1, flow, flow_valid=None, rule=0):
    d0 = _c(d0, np.float64)
    d1 = _c(d1, np.float64)
    v0 = _c(v0, np.uint8)
    v1 = _c(v1, np.uint8)
    flow = _c(flow, np.float32)
    fv = None if flow_valid is None else _c(flow_valid, np.uint8)
    H, W = d0.shape
    sf = np.empty((H, W, 4), np.float64)
    valid = np.empty((H, W), np.uint8)
    _chk(_get().orc_combine(_p(d0), _p(v0), _p(d1), _p(v1), _p(flow), _p(fv), W, H, rule,
                            _p(sf), _p(valid)), "combine")
    return sf, valid


def reproject(sf, valid_sf, f, B, cx, cy):
    sf = _c(sf, np.float64)
    valid_sf = _c(valid_sf, np.uint8)
    H, W, _ = sf.shape
    p0 = np.empty((H, W, 3), np.float64)
    p1 = np.empty((H, W, 3), np.float64)
    dp = np.empty((H, W, 3), np.float64)
    v3 = np.empty((H, W), np.uint8)
    _chk(_get().orc_reproject(_p(sf), _p(valid_sf), W, H, f, B, cx, cy,
                              _p(p0), _p(p1), _p(dp), _p(v3)), "reproject")
    return p0, p1, dp, v3


def evaluate(sf, valid_sf, gt_d0, gt_d1, gt_flow, gt_noc, gt_valid=None, tau_abs=3.0,
             tau_rel=0.05):
    """KITTI-style outlier counts (float32 decisions).  Returns int64 [2][6] =
    {n_gt, n_eval, n_d1, n_d2, n_fl, n_sf} for split 0 (all) and 1 (non-occluded)."""
    sf = _c(sf, np.float32)
    valid_sf = _c(valid_sf, np.uint8)
    gt_d0 = _c(gt_d0, np.float32)
    gt_d1 = _c(gt_d1, np.float32)
    gt_flow = _c(gt_flow, np.float32)
    gt_noc = _c(gt_noc, np.uint8)
    gv = None if gt_valid is None else _c(gt_valid, np.uint8)
    H, W = valid_sf.shape
    out = np.zeros((2, 6), np.int64)
    _chk(_get().orc_evaluate(_p(sf), _p(valid_sf), _p(gt_d0), _p(gt_d1), _p(gt_flow), _p(gv),
                             _p(gt_noc), W, H, tau_abs, tau_rel, _p(out)), "evaluate")
    return out


def run_quad(quad, prm, rule=0, threads=True):
    """The whole hot path on one frame quadruple: SGM at t and t+1,
    combination Eq. (4)/(5), 3D.  ``quad`` holds il0, ir0, il1, ir1, flow;
    ``prm`` holds D, cw, ch, P1, P2, T, f, B (and optional cx, cy)."""
    args = (prm["D"], prm["cw"], prm["ch"], prm["P1"], prm["P2"], prm["T"])
    res = {}

    def run(key, l, r):
        res[key] = disparity(l, r, *args)

    if threads:
        th = [threading.Thread(target=run, args=("t0", quad["il0"], quad["ir0"])),
              threading.Thread(target=run, args=("t1", quad["il1"], quad["ir1"]))]
        for t in th:
            t.start()
        for t in th:
            t.join()
    else:
        run("t0", quad["il0"], quad["ir0"])
        run("t1", quad["il1"], quad["ir1"])
    H, W = quad["il0"].shape
    cx = prm.get("cx", (W - 1) / 2.0)
    cy = prm.get("cy", (H - 1) / 2.0)
    sf, vsf = combine(res["t0"]["d_sub"], res["t0"]["valid"], res["t1"]["d_sub"],
                      res["t1"]["valid"], quad["flow"], None, rule)
    p0, p1, dp, v3 = reproject(sf, vsf, prm["f"], prm["B"], cx, cy)
    return {"disp0": res["t0"], "disp1": res["t1"], "sf": sf, "valid_sf": vsf,
            "p0": p0, "p1": p1, "dp": dp, "valid_3d": v3}


def run_stream(video, prm, rule=0, threads=True):
    """Streaming mode ("reuse"): a stereo video of n+1 frames
    gives n quads (frame k, frame k+1).  Every frame's LR-checked map is computed once and
    serves as D1 of quad k-1 and D0 of quad k; the combination and 3D are those of
    run_quad.  ``video`` holds left, right uint8 [n+1][H][W] and flow [n][H][W][2]."""
    left, right, flow = video["left"], video["right"], video["flow"]
    n = flow.shape[0]
    args = (prm["D"], prm["cw"], prm["ch"], prm["P1"], prm["P2"], prm["T"])
    maps = [None] * (n + 1)

    def run(k):
        maps[k] = disparity(left[k], right[k], *args)

    if threads:
        th = [threading.Thread(target=run, args=(k,)) for k in range(n + 1)]
        for t in th:
            t.start()
        for t in th:
            t.join()
    else:
        for k in range(n + 1):
            run(k)
    H, W = left.shape[1:]
    cx = prm.get("cx", (W - 1) / 2.0)
    cy = prm.get("cy", (H - 1) / 2.0)
    quads = []
    for k in range(n):
        sf, vsf = combine(maps[k]["d_sub"], maps[k]["valid"], maps[k + 1]["d_sub"],
                          maps[k + 1]["valid"], flow[k], None, rule)
        p0, p1, dp, v3 = reproject(sf, vsf, prm["f"], prm["B"], cx, cy)
        quads.append({"disp0": maps[k], "disp1": maps[k + 1], "sf": sf, "valid_sf": vsf,
                      "p0": p0, "p1": p1, "dp": dp, "valid_3d": v3})
    return {"maps": maps, "quads": quads}


# ---------------------------------------------------------------- optical flow (flow_oracle.c)
FQ = 8   # flow vectors are integers in 1/FQ px (reading FF1)

FF_DEFAULTS = {"levels": 3, "r": 4, "sweeps": 8, "R0": 8, "win": 8, "knn": 4, "penalty": 20,
               "seed": 1, "thr_q": 8}


def ff_downsample(img):
    img = _c(img, np.uint8)
    H, W = img.shape
    out = np.empty(((H + 1) // 2, (W + 1) // 2), np.uint8)
    _chk(_get().orc_ff_downsample(_p(img), W, H, _p(out)), "ff_downsample")
    return out


def ff_wht(img, win=8):
    img = _c(img, np.uint8)
    H, W = img.shape
    out = np.empty((H, W, 16), np.int32)
    _chk(_get().orc_ff_wht(_p(img), W, H, win, _p(out)), "ff_wht")
    return out


def ff_patch_cost(A, B, x, y, fu, fv, r=4, penalty=20):
    A = _c(A, np.uint8)
    B = _c(B, np.uint8)
    H, W = A.shape
    return int(_get().orc_ff_patch_cost(_p(A), _p(B), W, H, x, y, fu, fv, r, penalty))


def ff_knn_init(A, B, win=8, knn=4, r=4, penalty=20):
    A = _c(A, np.uint8)
    B = _c(B, np.uint8)
    H, W = A.shape
    flow = np.empty((H, W, 2), np.int32)
    cost = np.empty((H, W), np.int32)
    nn = np.empty((H, W, knn), np.int32)
    _chk(_get().orc_ff_knn_init(_p(A), _p(B), W, H, win, knn, r, penalty, _p(flow), _p(cost),
                                _p(nn)), "ff_knn_init")
    return flow, cost, nn


def ff_rng(seed, level, sweep, x, y):
    return int(_get().orc_ff_rng(seed, level, sweep, x, y))


def ff_sweep(A, B, flow, cost, sweep, level=0, r=4, penalty=20, R0=8, seed=1):
    """One propagation sweep + random search, in place on copies (returned)."""
    A = _c(A, np.uint8)
    B = _c(B, np.uint8)
    H, W = A.shape
    flow = np.array(flow, np.int32, copy=True)
    cost = np.array(cost, np.int32, copy=True)
    _chk(_get().orc_ff_sweep(_p(A), _p(B), W, H, r, penalty, sweep, level, R0, seed,
                             _p(flow), _p(cost)), "ff_sweep")
    return flow, cost


def ff_lift(A, B, coarse, r=4, penalty=20):
    A = _c(A, np.uint8)
    B = _c(B, np.uint8)
    coarse = _c(coarse, np.int32)
    H, W = A.shape
    Hc, Wc = coarse.shape[:2]
    flow = np.empty((H, W, 2), np.int32)
    cost = np.empty((H, W), np.int32)
    _chk(_get().orc_ff_lift(_p(A), _p(B), W, H, Wc, Hc, _p(coarse), r, penalty, _p(flow),
                            _p(cost)), "ff_lift")
    return flow, cost


def ff_field(A, B, levels=3, r=4, sweeps=8, R0=8, win=8, knn=4, penalty=20, seed=1):
    A = _c(A, np.uint8)
    B = _c(B, np.uint8)
    H, W = A.shape
    flow = np.empty((H, W, 2), np.int32)
    cost = np.empty((H, W), np.int32)
    _chk(_get().orc_ff_field(_p(A), _p(B), W, H, levels, r, sweeps, R0, win, knn, penalty, seed,
                             _p(flow), _p(cost)), "ff_field")
    return flow, cost


def ff_consistency(F, G1, G2, thr_q=8):
    F = _c(F, np.int32)
    G1 = _c(G1, np.int32)
    G2 = _c(G2, np.int32)
    H, W = F.shape[:2]
    v = np.empty((H, W), np.uint8)
    _chk(_get().orc_ff_consistency(_p(F), _p(G1), _p(G2), W, H, thr_q, _p(v)), "ff_consistency")
    return v


def ff_flow(A, B, levels=3, r=4, sweeps=8, R0=8, win=8, knn=4, penalty=20, seed=1, thr_q=8):
    """Forward field + two inverse fields + consistency.  Returns (flow int32
    [H][W][2] in 1/FQ px, valid uint8 [H][W])."""
    A = _c(A, np.uint8)
    B = _c(B, np.uint8)
    H, W = A.shape
    flow = np.empty((H, W, 2), np.int32)
    v = np.empty((H, W), np.uint8)
    _chk(_get().orc_ff_flow(_p(A), _p(B), W, H, levels, r, sweeps, R0, win, knn, penalty, seed,
                            thr_q, _p(flow), _p(v)), "ff_flow")
    return flow, v


# ---------------------------------------------------------------- densification (flow_oracle.c)
def edge_distance(guide, p, s, lam=1.0):
    guide = _c(guide, np.uint8)
    H, W = guide.shape
    return float(_get().orc_edge_distance(_p(guide), W, H, p[0], p[1], s[0], s[1], lam))


def densify(field, valid, guide, K=25, lam=1.0, window=0):
    """Fill the gaps of a C-channel field [H][W][C] (C <= 4): each gap pixel takes the
    1/d_e-weighted mean of its K valid seeds of smallest edge-aware distance d_e (SPEC
    F-6); window > 0 restricts the candidates to Chebyshev distance max(window, rho_K).
    lam is a float32 parameter (as in the C ABI).  Returns float64 [H][W][C]; raises if
    the image has no valid pixel (SPEC S:258 error)."""
    field = _c(field, np.float32)
    if field.ndim == 2:
        field = field[..., None]
    valid = _c(valid, np.uint8)
    guide = _c(guide, np.uint8)
    H, W, C = field.shape
    out = np.empty((H, W, C), np.float64)
    rc = _get().orc_densify(_p(field), _p(valid), _p(guide), W, H, C, K, lam, window, _p(out))
    if rc == 3:
        raise ValueError("densify: no valid pixel")
    _chk(rc, "densify")
    return out


def densify_points(field, valid, guide, xy, K=25, lam=1.0, window=0):
    """densify at the pixels xy [m][2] (x, y) only: float64 [m][C]."""
    field = _c(field, np.float32)
    if field.ndim == 2:
        field = field[..., None]
    valid = _c(valid, np.uint8)
    guide = _c(guide, np.uint8)
    xy = _c(xy, np.int32)
    H, W, C = field.shape
    out = np.empty((len(xy), C), np.float64)
    _chk(_get().orc_densify_points(_p(field), _p(valid), _p(guide), W, H, C, K, lam, window, len(xy),
                                   _p(xy), _p(out)), "densify_points")
    return out
