"""GPU parity: the CUDA path (called through the C ABI via the thin binding) against
the CPU oracle on the same seeded inputs.  Integers, masks and costs must be
bit-exact; sub-pixel disparities within 1e-4 px, scene-flow d1 within
1e-4*max(1,|d1|), 3D points within 1e-4 relative (BASELINE.json north_star, G22).
"""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

SUB_TOL = 1e-4


def _np(t):
    t = t.detach().cpu()
    if t.dtype == getattr(torch, "uint16", None):
        return t.view(torch.int16).numpy().view(np.uint16)
    if t.dtype == getattr(torch, "uint64", None):
        return t.view(torch.int64).numpy().view(np.uint64)
    return t.numpy()


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    return torch.device("cuda", 0)


def make_sgm(W, H, D, cw, ch, P1, P2, T=1, max_batch=1, rule=0):
    from paper_1801_04720_b200 import SGM
    return SGM(W, H, D, cw, ch, P1, P2, T, -1, rule, max_batch, 0)


# (W, H, D, cw, ch, P1, P2) -- tiles, ragged tails, padding of D, every CPL variant
SHAPES = [
    (64, 48, 16, 5, 5, 10, 120),      # Tiny (CPL=2, D < 64 padded)
    (97, 37, 64, 9, 7, 7, 86),        # ragged W/H, CPL=2 full
    (150, 70, 100, 9, 7, 7, 86),      # CPL=4 with padding (Dp=128)
    (300, 41, 128, 9, 7, 7, 86),      # Driving parameters, cropped
    (260, 33, 192, 9, 7, 7, 86),      # CPL=6
    (300, 29, 256, 9, 7, 7, 86),      # CPL=8
    (40, 20, 64, 5, 5, 3, 9),         # W < D (border everywhere)
    (33, 1, 32, 3, 3, 2, 20),         # single row
    (1, 9, 16, 3, 3, 2, 20),          # single column
    # edge cases of the parameters: one / two disparity levels, D just past a CPL step,
    # D = 255, a 3x1 census (2 bits), tall and wide census windows, P1 = P2 = 0
    (45, 17, 1, 5, 5, 4, 30),
    (45, 17, 2, 5, 5, 4, 30),
    (90, 19, 65, 9, 7, 7, 86),
    (280, 13, 255, 9, 7, 7, 86),
    (37, 15, 16, 3, 1, 1, 5),
    (61, 23, 32, 7, 9, 7, 86),
    (61, 23, 32, 13, 3, 5, 60),
    (48, 21, 24, 3, 3, 0, 0),
    # the band handoff in bytes (sweep_params h8): padded D at the clamp bound C_max + 2 P2 =
    # 254, an odd width with 6 cells per lane (byte rows rounded up to an even position
    # count), and P2 large enough (C_max + P2 + P1 > 255) to keep the u16 handoff
    (200, 40, 96, 9, 7, 7, 96),
    (261, 35, 192, 9, 7, 7, 86),
    (200, 40, 128, 9, 7, 10, 190),
]


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s[:3])))
def test_census_cost_aggregate_wta_lr(orc, dev, shape):
    W, H, D, cw, ch, P1, P2 = shape
    L, R = synth.random_pair(W, H, seed=W * 7 + H)
    g = make_sgm(W, H, D, cw, ch, P1, P2)
    gl, gr = g.upload_image(L), g.upload_image(R)
    cl, cr = g.census(gl), g.census(gr)
    ocl, ocr = orc.census(L, cw, ch), orc.census(R, cw, ch)
    assert np.array_equal(_np(cl), ocl)
    assert np.array_equal(_np(cr), ocr)
    cmax = cw * ch - 1
    raw = {}
    for view, s in ((0, -1), (1, +1)):
        ref, match = (ocl, ocr) if view == 0 else (ocr, ocl)
        di, ds, C, S = orc.sgm_view(ref, match, D, s, cmax, P1, P2, want_cost=True, want_S=True)
        gC = g.cost(cl, cr, view)
        assert np.array_equal(_np(gC), C), f"cost view {view}"
        gS = g.aggregate(cl, cr, view)
        torch.cuda.synchronize()
        assert np.array_equal(_np(gS).astype(np.uint32), S), f"aggregate view {view}"
        gdi, gds = g.wta(gS)
        assert np.array_equal(_np(gdi), di)
        assert np.abs(_np(gds) - ds).max() <= SUB_TOL
        raw[view] = (gdi, gds, di, ds)
    oi, osub, ov = orc.lr_check(raw[0][2], raw[0][3], raw[1][2], 1)
    gi, gsub, gv = g.lr_check(raw[0][0], raw[0][1], raw[1][0])
    assert np.array_equal(_np(gv), ov)
    assert np.array_equal(_np(gi), oi)
    assert np.abs(_np(gsub) - osub).max() <= SUB_TOL
    # fused production path == stage-wise composition, and == oracle
    fi, fsub, fv = g.disparity(gl, gr)
    assert np.array_equal(_np(fi), _np(gi)) and np.array_equal(_np(fv), _np(gv))
    assert np.array_equal(_np(fsub), _np(gsub))
    g.close()


# Widths around the row loop's unrolled block (CPL positions), its tail, and the backward
# sweep's WTA record period (32 positions; 30 for 6 cells per lane): W below one block, exact
# multiples, one more / one less, for every cells-per-lane variant; a few rows only (the
# oracle's cost grows with W H D).  The production path (fused sweeps, sub-pixel + store block
# at the block ends) is compared with the oracle's LR-checked maps.
WIDTHS = [
    (16, 2, (1, 2, 3, 31, 32, 33, 64, 65)),
    (128, 4, (1, 3, 4, 5, 31, 32, 33, 35, 36, 64, 67)),
    (192, 6, (1, 5, 6, 7, 29, 30, 31, 36, 59, 60, 61, 66, 90)),
    (256, 8, (1, 7, 8, 9, 31, 32, 33, 40, 63, 64, 65)),
]


@pytest.mark.parametrize("D,cpl,widths", WIDTHS, ids=lambda v: str(v) if isinstance(v, int) else "w")
def test_disparity_widths_around_block_and_period(orc, dev, D, cpl, widths):
    H = 5
    for W in widths:
        L, R = synth.random_pair(W, H, seed=1000 * cpl + W)
        g = make_sgm(W, H, D, 9, 7, 7, 86)
        assert g.geometry()["cells_per_lane"] == cpl
        fi, fsub, fv = g.disparity(g.upload_image(L), g.upload_image(R))
        ocl, ocr = orc.census(L, 9, 7), orc.census(R, 9, 7)
        dl, dls = orc.sgm_view(ocl, ocr, D, -1, 62, 7, 86)[:2]
        dr = orc.sgm_view(ocr, ocl, D, +1, 62, 7, 86)[0]
        oi, osub, ov = orc.lr_check(dl, dls, dr, 1)
        assert np.array_equal(_np(fv), ov), (D, W)
        assert np.array_equal(_np(fi), oi), (D, W)
        assert np.abs(_np(fsub) - osub).max() <= SUB_TOL, (D, W)
        g.close()


def test_aggregate_invariants_on_gpu(orc, dev):
    """P1 = P2 = 0 => S = 8C (north-star invariant) on the GPU path too."""
    W, H, D = 120, 40, 64
    L, R = synth.random_pair(W, H, seed=3)
    g = make_sgm(W, H, D, 9, 7, 0, 0)
    cl, cr = g.census(g.upload_image(L)), g.census(g.upload_image(R))
    C = _np(g.cost(cl, cr, 0)).astype(np.uint32)
    S = _np(g.aggregate(cl, cr, 0)).astype(np.uint32)
    assert np.array_equal(S, 8 * C)
    g.close()


def test_constant_disparity_pair_gpu(dev):
    d, W, H = 9, 256, 64
    L, R = synth.random_pair(W, H, seed=11, shift=d)
    g = make_sgm(W, H, 64, 9, 7, 7, 86)
    di, ds, v = g.disparity(g.upload_image(L), g.upload_image(R))
    inner = (slice(3, -3), slice(d + 4, -4))
    assert (_np(di)[inner] == d).all() and _np(v)[inner].all()
    g.close()


def test_determinism(dev):
    W, H = 300, 80
    L, R = synth.random_pair(W, H, seed=5)
    g = make_sgm(W, H, 128, 9, 7, 7, 86)
    gl, gr = g.upload_image(L), g.upload_image(R)
    first = [_np(t) for t in g.disparity(gl, gr)]
    for _ in range(5):
        again = [_np(t) for t in g.disparity(gl, gr)]
        for a, b in zip(first, again):
            assert np.array_equal(a, b)
    g.close()


def _combine_inputs(W, H, seed):
    rng = np.random.default_rng(seed)
    d0 = rng.uniform(0.5, 60, size=(H, W)).astype(np.float32)
    d1 = rng.uniform(0.5, 60, size=(H, W)).astype(np.float32)
    v0 = (rng.uniform(size=(H, W)) < 0.9).astype(np.uint8)
    v1 = (rng.uniform(size=(H, W)) < 0.9).astype(np.uint8)
    d0[v0 == 0] = -1
    d1[v1 == 0] = -1
    flow = rng.uniform(-12, 12, size=(H, W, 2)).astype(np.float32)
    flow[::7, ::5] = np.round(flow[::7, ::5])         # lattice targets
    flow[3, :, 0] = W                                  # leaves the image
    d0[5, :5] = 0.0                                    # d = 0 (G21)
    fv = (rng.uniform(size=(H, W)) < 0.97).astype(np.uint8)
    return d0, v0, d1, v1, flow, fv


@pytest.mark.parametrize("rule", [0, 1])
def test_combine_parity(orc, dev, rule):
    from paper_1801_04720_b200 import Camera
    W, H = 203, 77
    d0, v0, d1, v1, flow, fv = _combine_inputs(W, H, 8 + rule)
    g = make_sgm(W, H, 64, 9, 7, 7, 86, rule=rule)
    T = lambda a: torch.from_numpy(a).to(dev)  # noqa: E731
    cam = Camera(720.0, 0.54, (W - 1) / 2, (H - 1) / 2)
    r = g.combine_sceneflow(T(d0), T(v0), T(d1), T(v1), T(flow), T(fv), cam)
    sf, vsf = orc.combine(d0.astype(np.float64), v0, d1.astype(np.float64), v1, flow, fv, rule)
    p0, p1, dp, v3 = orc.reproject(sf, vsf, 720.0, 0.54, (W - 1) / 2, (H - 1) / 2)
    _check_sceneflow(r, sf, vsf, p0, p1, dp, v3)
    g.close()


def _check_sceneflow(r, sf, vsf, p0, p1, dp, v3):
    gv = _np(r["valid_sf"])
    assert np.array_equal(gv, vsf)
    gsf = _np(r["sf"]).astype(np.float64)
    m = vsf.astype(bool)
    assert (gsf[~m] == 0).all()
    assert np.array_equal(gsf[..., :2][m], sf[..., :2][m])           # u, v: exact copies
    # d0 is the float32 sub-pixel map on the GPU, fp64 in the oracle (1e-4 px, G22)
    assert np.abs(gsf[..., 2][m] - sf[..., 2][m]).max(initial=0) <= SUB_TOL
    err = np.abs(gsf[..., 3] - sf[..., 3])[m]
    assert (err <= SUB_TOL * np.maximum(1.0, np.abs(sf[..., 3][m]))).all()
    gv3 = _np(r["valid_3d"])
    assert np.array_equal(gv3, v3)
    m3 = v3.astype(bool)
    gp0 = _np(r["p0"])[..., :3].astype(np.float64)
    gdp = _np(r["dp"])[..., :3].astype(np.float64)
    n0 = np.linalg.norm(p0, axis=-1)
    n1 = np.linalg.norm(p1, axis=-1)
    assert (np.linalg.norm(gp0 - p0, axis=-1)[m3] <= 1e-4 * n0[m3]).all()
    assert (np.linalg.norm(gdp - dp, axis=-1)[m3] <= 1e-4 * np.maximum(n0, n1)[m3]).all()
    assert (gp0[~m3] == 0).all() and (gdp[~m3] == 0).all()


def _quad_parity(orc, g, quads, prm, dev):
    from paper_1801_04720_b200 import Camera, stack_quads
    imgs, flow = stack_quads(quads, g.pitch, dev)
    H, W = quads[0]["il0"].shape
    cam = Camera(prm["f"], prm["B"], prm["cx"], prm["cy"])
    out = g.scene_flow(imgs, flow, cam)
    torch.cuda.synchronize()
    for i, q in enumerate(quads):
        o = orc.run_quad(q, prm)
        for t, key in ((0, "disp0"), (1, "disp1")):
            assert np.array_equal(_np(out["disp_valid"][i, t]), o[key]["valid"])
            assert np.array_equal(_np(out["disp_int"][i, t]), o[key]["d_int"])
            assert np.abs(_np(out["disp_sub"][i, t]) - o[key]["d_sub"]).max() <= SUB_TOL
        r = {k: out[k][i] for k in ("sf", "valid_sf", "p0", "dp", "valid_3d")}
        _check_sceneflow(r, o["sf"], o["valid_sf"], o["p0"], o["p1"], o["dp"], o["valid_3d"])
    return out


def test_scene_flow_tiny(orc, dev):
    cfg = synth.CONFIGS["tiny"]
    prm = synth.sgm_params(cfg)
    from paper_1801_04720_b200 import SGM
    g = SGM.from_config(cfg, max_batch=2)
    quads = [synth.make_quad(cfg, 0), synth.make_quad(cfg, 1)]
    _quad_parity(orc, g, quads, prm, dev)
    g.close()


def test_identical_frames_zero_flow_gpu(dev):
    """Zero flow with identical frames gives D1 = D0 and d1 = d0 (north-star invariant)."""
    from paper_1801_04720_b200 import SGM, Camera, stack_quads
    cfg = synth.CONFIGS["tiny"]
    q = synth.make_quad(cfg, 0)
    q = dict(q, il1=q["il0"], ir1=q["ir0"], flow=np.zeros_like(q["flow"]))
    g = SGM.from_config(cfg)
    imgs, flow = stack_quads([q], g.pitch, dev)
    out = g.scene_flow(imgs, flow, Camera(720.0, 0.54, 31.5, 23.5))
    assert torch.equal(out["disp_sub"][0, 0], out["disp_sub"][0, 1])
    v = out["valid_sf"][0].bool()
    assert torch.equal(out["sf"][0][..., 2][v], out["sf"][0][..., 3][v])
    assert torch.equal(out["valid_sf"][0], out["disp_valid"][0, 0])
    g.close()


@pytest.mark.parametrize("name", ["driving", "wide", "highres"])
def test_scene_flow_full_size(orc, dev, name):
    """BASELINE.json configs[1..3] at full size, in the batched launch bench.py times,
    element by element against the oracle."""
    cfg = synth.CONFIGS[name]
    prm = synth.sgm_params(cfg)
    from paper_1801_04720_b200 import SGM
    g = SGM.from_config(cfg, max_batch=1)
    _quad_parity(orc, g, [synth.make_quad(cfg, 0)], prm, dev)
    g.close()


def oracle_many(orc, quads, prm):
    """The oracle on every quad, one quad per host thread (ctypes releases the GIL)."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    cores = len(os.sched_getaffinity(0))
    with ThreadPoolExecutor(max_workers=max(1, min(cores, len(quads)))) as ex:
        return list(ex.map(lambda q: orc.run_quad(q, prm, threads=False), quads))


def check_quad_outputs(out, i, o):
    """Every output field of quad i of a batched launch against the oracle's run_quad."""
    for t, key in ((0, "disp0"), (1, "disp1")):
        assert np.array_equal(_np(out["disp_valid"][i, t]), o[key]["valid"]), (i, key)
        assert np.array_equal(_np(out["disp_int"][i, t]), o[key]["d_int"]), (i, key)
        assert np.abs(_np(out["disp_sub"][i, t]) - o[key]["d_sub"]).max() <= SUB_TOL, (i, key)
    r = {k: out[k][i] for k in ("sf", "valid_sf", "p0", "dp", "valid_3d")}
    _check_sceneflow(r, o["sf"], o["valid_sf"], o["p0"], o["p1"], o["dp"], o["valid_3d"])


def test_batch_config_full(orc, dev):
    """configs[4]: 8 quads in one batched launch (the per-GPU shard at N=8, the bench's
    band geometry), EVERY quad and every output field (integer and LR-checked
    disparities, masks, S, P0, dP) element by element against the oracle, run on the
    host cores in parallel; a quad alone gives the same bytes as inside the batch."""
    cfg = synth.CONFIGS["batch"]
    prm = synth.sgm_params(cfg)
    from paper_1801_04720_b200 import SGM, Camera, stack_quads
    g = SGM.from_config(cfg, max_batch=8)
    quads = synth.make_batch(cfg, 0, 8, workers=8)
    imgs, flow = stack_quads(quads, g.pitch, dev)
    cam = Camera(prm["f"], prm["B"], prm["cx"], prm["cy"])
    out = g.scene_flow(imgs, flow, cam)
    torch.cuda.synchronize()
    for i, o in enumerate(oracle_many(orc, quads, prm)):
        check_quad_outputs(out, i, o)
    g1 = SGM.from_config(cfg, max_batch=1)
    one = g1.scene_flow(imgs[5:6].contiguous(), flow[5:6].contiguous(), cam)
    torch.cuda.synchronize()
    for k in ("sf", "valid_sf", "disp_int", "disp_sub", "p0", "dp"):
        assert torch.equal(one[k][0], out[k][5]), k
    g.close()
    g1.close()


def test_batch_config_64_quads(orc, dev):
    """configs[4] in full: all 64 quads (seeds 1000..1063) in the single launch the N=1 bench
    times, every quad and every output field against the oracle (host cores in parallel),
    and byte-identical to the eight 8-quad launches of the N=8 partition (SURVEY.md 8(e):
    gathered outputs equal the 1-GPU run)."""
    cfg = synth.CONFIGS["batch"]
    prm = synth.sgm_params(cfg)
    from paper_1801_04720_b200 import SGM, Camera, stack_quads
    quads = synth.make_batch(cfg, 0, 64, workers=16)
    cam = Camera(prm["f"], prm["B"], prm["cx"], prm["cy"])
    g = SGM.from_config(cfg, max_batch=64)
    imgs, flow = stack_quads(quads, g.pitch, dev)
    out = g.scene_flow(imgs, flow, cam)
    torch.cuda.synchronize()
    g8 = SGM.from_config(cfg, max_batch=8)
    for r in range(8):
        part = g8.scene_flow(imgs[8 * r:8 * r + 8].contiguous(), flow[8 * r:8 * r + 8].contiguous(), cam)
        torch.cuda.synchronize()
        for k in ("sf", "valid_sf", "p0", "dp", "valid_3d", "disp_int", "disp_sub", "disp_valid"):
            assert torch.equal(part[k], out[k][8 * r:8 * r + 8]), (r, k)
    g8.close()
    for i, o in enumerate(oracle_many(orc, quads, prm)):
        check_quad_outputs(out, i, o)
    g.close()


def test_host_entry_point_matches_device(dev):
    from paper_1801_04720_b200 import SGM, Camera, stack_quads
    cfg = synth.CONFIGS["tiny"]
    prm = synth.sgm_params(cfg)
    n = 5                                   # chunked pipeline: chunks of 2, last one partial
    g = SGM.from_config(cfg, max_batch=n)
    quads = [synth.make_quad(cfg, i) for i in range(n)]
    imgs, flow = stack_quads(quads, g.pitch, dev)
    cam = Camera(prm["f"], prm["B"], prm["cx"], prm["cy"])
    ref = g.scene_flow(imgs, flow, cam)
    torch.cuda.synchronize()
    himg = torch.from_numpy(np.stack([[q[k] for k in ("il0", "ir0", "il1", "ir1")]
                                      for q in quads])).pin_memory()
    hflow = torch.from_numpy(np.stack([q["flow"] for q in quads])).pin_memory()
    hout = g.alloc_outputs(n, pinned_host=True)
    g.scene_flow_host(himg, hflow, cam, hout)
    torch.cuda.synchronize()
    for k in hout:
        assert torch.equal(hout[k], ref[k].cpu()), k
    # back-to-back calls pipeline through the two staging slots: three calls with
    # different inputs, one synchronisation, every output intact
    sets = []
    for sel in ([0, 1], [2, 3], [4, 0]):
        hi = torch.from_numpy(np.stack([[quads[i][k] for k in ("il0", "ir0", "il1", "ir1")]
                                        for i in sel])).pin_memory()
        hf = torch.from_numpy(np.stack([quads[i]["flow"] for i in sel])).pin_memory()
        ho = g.alloc_outputs(2, pinned_host=True, with_p0=False)
        g.scene_flow_host(hi, hf, cam, ho)
        sets.append((sel, ho))
    torch.cuda.synchronize()
    for sel, ho in sets:
        for j, i in enumerate(sel):
            for k in ho:
                assert torch.equal(ho[k][j], ref[k][i].cpu()), (sel, k)
    # without disparity outputs the host entry stages none and runs the fused LR + combination
    # form (4 kernels + the re-pitch): same bytes
    hno = g.alloc_outputs(n, pinned_host=True, with_disp=False)
    n0 = g.launch_count()
    g.scene_flow_host(himg, hflow, cam, hno)
    torch.cuda.synchronize()
    assert g.launch_count() - n0 == 5
    for k in hno:
        assert torch.equal(hno[k], ref[k].cpu()), k
    g.close()


def test_timing_and_launch_count(dev):
    from paper_1801_04720_b200 import SGM, Camera, stack_quads
    cfg = synth.CONFIGS["tiny"]
    g = SGM.from_config(cfg)
    imgs, flow = stack_quads([synth.make_quad(cfg)], g.pitch, dev)
    cam = Camera(720.0, 0.54, 31.5, 23.5)
    g.set_timing(True)
    n0 = g.launch_count()
    g.scene_flow(imgs, flow, cam)
    torch.cuda.synchronize()
    t = g.read_timing()
    assert g.launch_count() - n0 == 5
    assert set(t) == {"census", "sweep_fwd", "sweep_bwd_wta", "lr_check", "combine"}
    assert all(v > 0 for v in t.values())
    g.close()


def test_invalid_device_arguments(dev):
    from paper_1801_04720_b200 import _lib
    cfg = synth.CONFIGS["tiny"]
    from paper_1801_04720_b200 import SGM
    g = SGM.from_config(cfg)
    img = torch.zeros((48, 65), dtype=torch.uint8, device=dev)   # pitch not a multiple of 16
    with pytest.raises(_lib.SgmError):
        g.census(img)
    g.close()


def test_random_small_instances(orc, dev):
    """SPEC acceptance: 50 random instances up to 16x16x8 -- random size,
    disparity range, census window and penalties -- with an exact integer match of the
    aggregated volume S and of the integer disparities of both views."""
    rng = np.random.default_rng(2024)
    for it in range(50):
        W, H = int(rng.integers(1, 17)), int(rng.integers(1, 17))
        D = int(rng.integers(1, 9))
        cw, ch = [(3, 3), (5, 5), (3, 1), (1, 3), (7, 5)][it % 5]
        cmax = cw * ch - 1
        P1 = int(rng.integers(0, 20))
        P2 = int(rng.integers(P1, min(255 - cmax, 120) + 1))
        img = rng.integers(0, 256, size=(H, W)).astype(np.uint8)
        shift = int(rng.integers(0, 4))
        L = img
        R = np.roll(img, -shift, axis=1)
        g = make_sgm(W, H, D, cw, ch, P1, P2)
        cl, cr = g.census(g.upload_image(L)), g.census(g.upload_image(R))
        ocl, ocr = orc.census(L, cw, ch), orc.census(R, cw, ch)
        for view, s in ((0, -1), (1, +1)):
            ref, match = (ocl, ocr) if view == 0 else (ocr, ocl)
            di, ds, C, S = orc.sgm_view(ref, match, D, s, cmax, P1, P2, want_S=True)
            gS = g.aggregate(cl, cr, view)
            torch.cuda.synchronize()
            assert np.array_equal(_np(gS).astype(np.uint32), S), (it, view, W, H, D)
        g.close()


@pytest.mark.parametrize("name,n,rule", [("tiny", 3, 0), ("tiny", 2, 1), ("driving", 2, 0), ("wide", 1, 0)])
def test_fused_lr_combination_equals_separate_kernels(dev, name, n, rule):
    """Without disparity outputs sgm_scene_flow fuses the LR check into the combination
    kernel (4 launches, the LR-checked maps never materialised); the results must equal, bit
    for bit, those of the 5-launch form (which the other tests compare with the oracle) --
    quad and streaming mode, both bilinear rules, with a flow mask."""
    from paper_1801_04720_b200 import SGM, Camera, stack_quads, stack_video
    cfg = synth.CONFIGS[name]
    prm = synth.sgm_params(cfg)
    g = SGM(cfg.W, cfg.H, cfg.D, cfg.cw, cfg.ch, cfg.P1, cfg.P2, cfg.T, -1, rule, n, 0)
    cam = Camera(prm["f"], prm["B"], prm["cx"], prm["cy"])
    quads = [synth.make_quad(cfg, 40 + k) for k in range(n)]
    imgs, flow = stack_quads(quads, g.pitch, dev)
    rng = np.random.default_rng(5)
    fmask = torch.from_numpy((rng.uniform(size=(n, cfg.H, cfg.W)) < 0.9).astype(np.uint8)).to(dev)
    keys = ("sf", "valid_sf", "p0", "dp", "valid_3d")
    for mask in (None, fmask):
        ref = g.scene_flow(imgs, flow, cam, flow_valid=mask)              # with disparity maps
        n0 = g.launch_count()
        out = g.scene_flow(imgs, flow, cam, g.alloc_outputs(n, with_disp=False), flow_valid=mask)
        torch.cuda.synchronize()
        assert g.launch_count() - n0 == 4
        for k in keys:
            assert torch.equal(out[k], ref[k]), (k, mask is not None)
    if name == "tiny":
        video = synth.make_video(cfg, n, 7)
        vi, vf = stack_video(video, g.pitch, dev)
        ref = g.scene_flow_stream(vi, vf, cam)
        out = g.scene_flow_stream(vi, vf, cam, g.alloc_outputs(n, with_disp=False, stream_mode=True))
        torch.cuda.synchronize()
        for k in keys:
            assert torch.equal(out[k], ref[k]), ("stream", k)
    g.close()
