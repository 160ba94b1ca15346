"""Pins for the CPU oracle (oracle/sgm_oracle.c) against what the paper, the spec
and mathematics fix -- never against the oracle itself.  CPU only.

Each test names the passage (P:n PAPER.md, S:n SPEC.md, G# DESIGN.md reading)
and the kind of pin: hand value, closed form, brute force, invariant.
"""
import itertools
import json
import os

import numpy as np
import pytest

import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
DIRS = [(1, 0), (-1, 0), (0, 1), (0, -1), (1, 1), (-1, -1), (-1, 1), (1, -1)]


# --------------------------------------------------------------------------- census
@pytest.mark.parametrize("ex", GOLD["census"], ids=lambda e: e["cite"][:5])
def test_census_hand_values(orc, ex):
    img = np.array(ex["img"], np.uint8)
    c = orc.census(img, ex["w"], ex["h"])
    x, y = ex["at"]
    assert int(c[y, x]) == ex["bits"], ex["cite"]


def test_census_monotone_invariance(orc):
    """Census depends only on the order of intensities (S:113 'neighbour < centre'):
    any strictly increasing remap leaves it unchanged; a constant image gives 0."""
    rng = np.random.default_rng(3)
    img = rng.integers(0, 120, size=(9, 11)).astype(np.uint8)
    remap = (np.arange(256) * 2 + 5).clip(0, 255).astype(np.uint8)  # strictly increasing on 0..119
    a = orc.census(img, 5, 5)
    b = orc.census(remap[img], 5, 5)
    assert np.array_equal(a, b)
    assert not orc.census(np.full((6, 7), 9, np.uint8), 9, 7).any()


def test_census_bit_length_and_width(orc):
    """A 9x7 window yields 62 bits (S:113 window^2-1 generalised, G2: 9 wide x 7 tall);
    a pixel darker-than-all neighbourhood pattern sets exactly w*h-1 bits."""
    img = np.full((7, 9), 200, np.uint8)
    img[3, 4] = 255
    c = orc.census(img, 9, 7)
    assert int(c[3, 4]) == (1 << 62) - 1
    # transposing the image and the window permutes bits but keeps the count
    rng = np.random.default_rng(4)
    im = rng.integers(0, 256, size=(12, 10)).astype(np.uint8)
    c1 = orc.census(im, 9, 7)
    c2 = orc.census(im.T.copy(), 7, 9).T
    cnt = np.vectorize(lambda v: bin(int(v)).count("1"))
    assert np.array_equal(cnt(c1), cnt(c2))


def test_census_even_window_rejected(orc):
    with pytest.raises(ValueError):
        orc.census(np.zeros((4, 4), np.uint8), 4, 3)  # S:115 even window is an error


# --------------------------------------------------------------------------- cost
def test_cost_hand_cases(orc):
    """identical -> C(.,.,0)=0; shift s -> C(x,y,s)=0 for x>=s;
    x<d -> descriptor length (C_max = w*h-1, G5)."""
    L, R = synth.random_pair(40, 12, 1, shift=5)
    cl, cr = orc.census(L, 5, 5), orc.census(R, 5, 5)
    C = orc.cost(cl, cl, 8, -1, 24)
    assert not C[:, :, 0].any()
    C = orc.cost(cl, cr, 8, -1, 24)
    # interior (away from the clamped image border by the census radius)
    assert not C[2:-2, 5 + 2:-2, 5].any()
    assert (C[:, 2, 7] == 24).all() and (C[:, 8, 7] != 24).any()
    # right reference: out of image when x + d > W-1 (G12)
    Cr = orc.cost(cr, cl, 8, +1, 24)
    assert (Cr[:, -1, 1:] == 24).all()


def test_cost_popcount_independent(orc):
    """The popcount primitive against Python's own bit count on random descriptors."""
    rng = np.random.default_rng(9)
    a = rng.integers(0, 2**62, size=(3, 17), dtype=np.uint64)
    b = rng.integers(0, 2**62, size=(3, 17), dtype=np.uint64)
    C = orc.cost(a, b, 4, -1, 62)
    for y in range(3):
        for x in range(17):
            for d in range(4):
                if x - d >= 0:
                    assert C[y, x, d] == bin(int(a[y, x]) ^ int(b[y, x - d])).count("1")
                else:
                    assert C[y, x, d] == 62


# --------------------------------------------------------------------------- aggregation
def _viterbi(costs, P1, P2):
    """Brute force: E_n(d) = min over all label sequences ending in d of
    sum C_i(d_i) + sum V(d_i, d_{i+1}),  V = 0 / P1 (|diff|=1) / P2 (else).
    Returns E_n and E_{n-1} (the energy of the path without its last pixel)."""
    n, D = costs.shape

    def V(a, b):
        return 0 if a == b else (P1 if abs(a - b) == 1 else P2)

    def energy(m):
        E = np.full(D, np.iinfo(np.int64).max, np.int64)
        for seq in itertools.product(range(D), repeat=m):
            e = sum(int(costs[i, seq[i]]) for i in range(m))
            e += sum(V(seq[i], seq[i + 1]) for i in range(m - 1))
            E[seq[-1]] = min(E[seq[-1]], e)
        return E

    return energy(n), (energy(n - 1) if n > 1 else None)


@pytest.mark.parametrize("seed", range(6))
def test_single_path_equals_explicit_dp(orc, seed):
    """BJ north_star: a single-path sweep equals an explicit dynamic program.
    The normalised recursion equals the exhaustive path energy minus the
    minimum energy of the path one pixel shorter (exact integers), in all 8
    directions, for random costs and 0 <= P1 <= P2 (G8)."""
    rng = np.random.default_rng(seed)
    H, W, D = 4, 5, 3
    C = rng.integers(0, 25, size=(H, W, D)).astype(np.uint8)
    P1 = int(rng.integers(0, 8))
    P2 = int(rng.integers(P1, 20))
    for rx, ry in DIRS:
        L = orc.path(C, P1, P2, rx, ry)
        for y in range(H):
            for x in range(W):
                seq = []
                px, py = x, y
                while 0 <= px < W and 0 <= py < H:
                    seq.append((py, px))
                    px, py = px - rx, py - ry
                seq.reverse()
                costs = np.array([C[p] for p in seq])
                En, Eprev = _viterbi(costs, P1, P2)
                expect = En if Eprev is None else En - Eprev.min()
                assert np.array_equal(L[y, x], expect), (rx, ry, x, y)


@pytest.mark.parametrize("ex", GOLD["aggregate_single_path"], ids=lambda e: e["cite"][:5])
def test_path_hand_example(orc, ex):
    C = np.array(ex["cost"], np.uint8)[None]            # 1 row, 2 pixels, D=2
    L = orc.path(C, ex["P1"], ex["P2"], 1, 0)
    assert list(L[0, -1]) == ex["L_last"]


def test_aggregate_invariants(orc):
    """BJ / S:134 / S:167: P1=P2=0 => S = 8C exactly (so WTA(S) = WTA(C));
    1x1 image => 8C; C + c => S + 8c; bounds 0 <= L <= C_max + P2 (G9)."""
    rng = np.random.default_rng(11)
    C = rng.integers(0, 63, size=(7, 9, 6)).astype(np.uint8)
    S = orc.aggregate(C, 0, 0)
    assert np.array_equal(S, 8 * C.astype(np.uint32))
    one = rng.integers(0, 63, size=(1, 1, 5)).astype(np.uint8)
    assert np.array_equal(orc.aggregate(one, 7, 86), 8 * one.astype(np.uint32))
    S1 = orc.aggregate(C, 7, 86)
    S2 = orc.aggregate(C + 3, 7, 86)
    assert np.array_equal(S2, S1 + 24)
    for rx, ry in DIRS:
        L = orc.path(C, 7, 86, rx, ry)
        assert L.min() >= 0 and L.max() <= 62 + 86
    assert S1.max() <= 8 * (62 + 86)


def test_aggregate_path_sum(orc):
    """S = sum of the 8 independent single-path recursions."""
    rng = np.random.default_rng(12)
    C = rng.integers(0, 25, size=(5, 6, 4)).astype(np.uint8)
    S = orc.aggregate(C, 3, 9)
    tot = sum(orc.path(C, 3, 9, rx, ry).astype(np.int64) for rx, ry in DIRS)
    assert np.array_equal(S.astype(np.int64), tot)


# --------------------------------------------------------------------------- WTA
@pytest.mark.parametrize("ex", GOLD["wta"], ids=lambda e: e["cite"][:5])
def test_wta_hand_values(orc, ex):
    S = np.array(ex["S"], np.uint32)[None, None]
    di, ds = orc.wta(S)
    assert ds[0, 0] == ex["d"]
    assert di[0, 0] == int(np.floor(ex["d"] + 0.5)) or di[0, 0] == int(ex["d"])


def test_wta_closed_form_and_ranges(orc):
    """Smallest-index argmin; parabola vertex of the 3 samples; the
    offset of 8C equals that of C bit-exactly (scale invariance); interior offsets lie
    in (-0.5, 0.5] under the smallest-index rule (G11)."""
    rng = np.random.default_rng(5)
    S = rng.integers(0, 300, size=(20, 30, 9)).astype(np.uint32)
    di, ds = orc.wta(S)
    ref = np.argmin(S, axis=2)                              # numpy: first minimum
    assert np.array_equal(di, ref)
    _, ds8 = orc.wta(8 * S)
    assert np.array_equal(ds, ds8)
    off = ds - di
    inner = (di > 0) & (di < 8)
    assert (off[~inner] == 0).all()
    assert (off[inner] > -0.5).all() and (off[inner] <= 0.5).all()
    # vertex of the parabola through (-1,a), (0,b), (1,c) -- closed form
    for y, x in zip(*np.nonzero(inner)):
        a, b, c = (float(v) for v in S[y, x, di[y, x] - 1:di[y, x] + 2])
        coef = np.polyfit([-1.0, 0.0, 1.0], [a, b, c], 2)
        assert abs(off[y, x] - (-coef[1] / (2 * coef[0]))) < 1e-12


# --------------------------------------------------------------------------- LR
@pytest.mark.parametrize("ex", GOLD["lr"], ids=lambda e: e["cite"][:5])
def test_lr_hand_values(orc, ex):
    W = 12
    dl = np.full((1, W), ex["dl"], np.int16)
    dr = np.full((1, W), ex["dr"], np.int16)
    oi, os_, v = orc.lr_check(dl, dl.astype(np.float64), dr, ex["T"])
    x = W - 1                                              # x - d >= 0
    assert bool(v[0, x]) == ex["valid"]
    assert oi[0, x] == (ex["dl"] if ex["valid"] else -1)
    assert os_[0, x] == (float(ex["dl"]) if ex["valid"] else -1.0)
    # x - d < 0 is always invalid (the right pixel is outside the image)
    if ex["dl"] > 0:
        assert not v[0, 0]


def test_right_view_equals_mirrored_left(orc):
    """G12: the right-reference view computed directly (match at x+d) is bit-identical
    to SPEC S-5: mirror both images, run the left pipeline, mirror back."""
    for (cw, ch, D) in [(5, 5, 16), (9, 7, 32)]:
        L, R = synth.random_pair(70, 21, 7)
        cl, cr = orc.census(L, cw, ch), orc.census(R, cw, ch)
        cmax = cw * ch - 1
        di, ds, _, S = orc.sgm_view(cr, cl, D, +1, cmax, 7, 86, want_S=True)
        Lm, Rm = L[:, ::-1].copy(), R[:, ::-1].copy()
        clm, crm = orc.census(Rm, cw, ch), orc.census(Lm, cw, ch)
        dim, dsm, _, Sm = orc.sgm_view(clm, crm, D, -1, cmax, 7, 86, want_S=True)
        assert np.array_equal(S, Sm[:, ::-1])
        assert np.array_equal(di, dim[:, ::-1])
        assert np.array_equal(ds, dsm[:, ::-1])


@pytest.mark.parametrize("d,cw,ch,D,P1,P2", [(6, 5, 5, 16, 10, 120), (5, 9, 7, 32, 7, 86),
                                             (11, 9, 7, 64, 7, 86)])
def test_constant_disparity_recovered(orc, d, cw, ch, D, P1, P2):
    """BJ north_star: a constant-disparity synthetic pair recovers its disparity exactly
    in the interior; the x < d band is LR-invalid (x - d* < 0)."""
    L, R = synth.random_pair(128, 48, 5 + d, shift=d)
    o = orc.disparity(L, R, D, cw, ch, P1, P2, 1)
    ry, rx = ch // 2, cw // 2
    inner = (slice(ry, -ry), slice(d + rx, -rx))
    assert (o["d_int"][inner] == d).all()
    assert o["valid"][inner].all()
    assert not o["valid"][:, : max(d - 1, 0)].any() or d <= 1


def test_identical_frames_zero_flow(orc):
    """BJ north_star / S:311: identical frames + zero flow => D1 = D0 exactly,
    d1 = d0 bit-exactly and valid_sf = valid(D0); d1 - d0 = 0 (static scene)."""
    q = synth.make_quad("tiny")
    prm = synth.sgm_params(synth.CONFIGS["tiny"])
    quad = {"il0": q["il0"], "ir0": q["ir0"], "il1": q["il0"], "ir1": q["ir0"],
            "flow": np.zeros_like(q["flow"])}
    r = orc.run_quad(quad, prm)
    assert np.array_equal(r["disp0"]["d_int"], r["disp1"]["d_int"])
    assert np.array_equal(r["disp0"]["d_sub"], r["disp1"]["d_sub"])
    assert np.array_equal(r["valid_sf"], r["disp0"]["valid"])
    v = r["valid_sf"].astype(bool)
    assert (r["sf"][..., 3][v] == r["sf"][..., 2][v]).all()
    v3 = r["valid_3d"].astype(bool)
    assert (r["dp"][v3] == 0).all()


# --------------------------------------------------------------------------- combine
def _cell_inputs(cell, W=4, H=4):
    d1 = np.zeros((H, W))
    d1[0:2, 0:2] = np.array(cell, np.float64)
    return d1


@pytest.mark.parametrize("ex", GOLD["bilinear"], ids=lambda e: e["cite"][:5])
def test_bilinear_hand_values(orc, ex):
    """Eq. (5) on the unit cell of S:57-58."""
    W = H = 4
    d1 = _cell_inputs(ex["cell"])
    flow = np.zeros((H, W, 2), np.float32)
    flow[0, 0] = ex["p"]
    ones = np.ones((H, W), np.uint8)
    sf, v = orc.combine(np.ones((H, W)), ones, d1, ones, flow)
    assert v[0, 0] == 1 and sf[0, 0, 3] == ex["value"]


@pytest.mark.parametrize("ex", GOLD["combine"], ids=lambda e: e["cite"][:5])
def test_combine_hand_value(orc, ex):
    W = H = 4
    d1 = _cell_inputs(ex["cell"])
    d0 = np.full((H, W), ex["d0"])
    flow = np.zeros((H, W, 2), np.float32)
    flow[0, 0] = ex["flow"]
    ones = np.ones((H, W), np.uint8)
    sf, v = orc.combine(d0, ones, d1, ones, flow)
    assert v[0, 0] == 1 and list(sf[0, 0]) == ex["S"]


def test_bilinear_exact_on_bilinear_functions(orc):
    """Eq. (5) reproduces a + b x + c y + d x y at every in-domain point (to 1e-6),
    is exact at lattice points, and is bounded by its footprint."""
    H, W = 9, 13
    ys, xs = np.mgrid[0:H, 0:W].astype(np.float64)
    a, b, c, d = 2.0, 0.5, -0.25, 0.125
    D1 = a + b * xs + c * ys + d * xs * ys
    rng = np.random.default_rng(0)
    flow = rng.uniform(-3, 3, size=(H, W, 2)).astype(np.float32)
    ones = np.ones((H, W), np.uint8)
    sf, v = orc.combine(np.ones((H, W)), ones, D1, ones, flow)
    xp = (xs.astype(np.float32) + flow[..., 0]).astype(np.float64)
    yp = (ys.astype(np.float32) + flow[..., 1]).astype(np.float64)
    inside = (xp >= 0) & (xp <= W - 1) & (yp >= 0) & (yp <= H - 1)
    assert np.array_equal(v.astype(bool), inside)
    exp = a + b * xp + c * yp + d * xp * yp
    assert np.abs(sf[..., 3][inside] - exp[inside]).max() < 1e-6
    # lattice flow => exact lookup
    flow_i = np.round(flow)
    sf2, v2 = orc.combine(np.ones((H, W)), ones, D1, ones, flow_i)
    m = v2.astype(bool)
    xi = (xs + flow_i[..., 0]).astype(int)
    yi = (ys + flow_i[..., 1]).astype(int)
    assert np.array_equal(sf2[..., 3][m], D1[yi[m], xi[m]])


def test_combine_validity_cases(orc):
    """Eq. (4): leaving Omega, an invalid D0(x) or an invalid tap of D1 makes
    the pixel undefined (0 + mask 0, G14); G17 clamps the +1 tap at the border;
    G18 rule 0 only requires taps with nonzero weight; rule 1 requires all four."""
    H, W = 6, 8
    ones = np.ones((H, W), np.uint8)
    d0 = np.full((H, W), 4.0)
    d1 = np.full((H, W), 3.0)
    flow = np.zeros((H, W, 2), np.float32)
    flow[0, 0] = (W, 0)                       # S:312 leaves the image
    flow[1, 1] = (W - 1 - 1, 0)               # exactly the last column: inside (G16/G17)
    flow[2, 2] = (0.5, 0.0)                   # tap (3,2) needed
    flow[3, 3] = (-3.0001, 0)                  # x' < 0 in float32
    flow[4, 4] = (np.nan, 0)                  # NaN is outside (G16)
    v1 = ones.copy()
    v1[2, 3] = 0
    sf, v = orc.combine(d0, ones, d1, v1, flow)
    assert v[0, 0] == 0 and (sf[0, 0] == 0).all()
    assert v[1, 1] == 1 and sf[1, 1, 3] == 3.0
    assert v[2, 2] == 0
    assert v[3, 3] == 0 and v[4, 4] == 0
    # rule 0 vs 1: fx = 0 needs only the (x0, .) taps under rule 0
    flow2 = np.zeros((H, W, 2), np.float32)
    v1b = ones.copy()
    v1b[1, 1] = 0                             # the (x0+1, y0+1) tap of pixel (0,0)
    _, va = orc.combine(d0, ones, d1, v1b, flow2, rule=0)
    _, vb = orc.combine(d0, ones, d1, v1b, flow2, rule=1)
    assert va[0, 0] == 1 and vb[0, 0] == 0
    v0 = ones.copy()
    v0[5, 5] = 0
    _, vc = orc.combine(d0, v0, d1, ones, flow2)
    assert vc[5, 5] == 0
    fv = ones.copy()
    fv[5, 6] = 0
    _, vd = orc.combine(d0, ones, d1, ones, flow2, flow_valid=fv)
    assert vd[5, 6] == 0 and vd[5, 7] == 1


# --------------------------------------------------------------------------- 3D
def test_triangulate_hand_values(orc):
    g = GOLD["triangulate"]
    sf = np.zeros((1, 1, 4))
    sf[0, 0] = (0, 0, g[0]["d"], g[0]["d"])
    p0, p1, dp, v = orc.reproject(sf, np.ones((1, 1), np.uint8), g[0]["f"], g[0]["B"], 0.0, 0.0)
    assert p0[0, 0, 2] == g[0]["Z"] and (dp == 0).all()
    e = g[1]
    sf[0, 0] = (e["uv"][0], e["uv"][1], e["d0"], e["d1"])
    p0, p1, dp, v = orc.reproject(sf, np.ones((1, 1), np.uint8), e["f"], e["B"], e["cx"], e["cy"])
    assert list(dp[0, 0]) == e["dP"]


def test_tiny_depths_and_signs(orc):
    """Z = f B / d (BJ north_star); Tiny depths f*B = 388.8; sign(dZ) = sign(d0 - d1)
    for u = v = 0; d <= 0 is skipped (G21)."""
    t = GOLD["tiny_depths"][0]
    n = len(t["d"])
    sf = np.zeros((1, n, 4))
    sf[0, :, 2] = t["d"]
    sf[0, :, 3] = t["d"]
    p0, p1, dp, v = orc.reproject(sf, np.ones((1, n), np.uint8), t["f"], t["B"], 0.0, 0.0)
    assert np.allclose(p0[0, :, 2], t["Z"], rtol=1e-12)
    rng = np.random.default_rng(2)
    sf = np.zeros((4, 5, 4))
    sf[..., 2] = rng.uniform(1, 50, size=(4, 5))
    sf[..., 3] = rng.uniform(1, 50, size=(4, 5))
    sf[0, 0, 3] = 0.0
    p0, p1, dp, v = orc.reproject(sf, np.ones((4, 5), np.uint8), 720.0, 0.54, 2.0, 1.5)
    assert v[0, 0] == 0
    m = v.astype(bool)
    assert (np.sign(dp[..., 2][m]) == np.sign(sf[..., 2] - sf[..., 3])[m]).all()
    # round trip: Z back to disparity
    assert np.allclose((720.0 * 0.54 / p0[..., 2])[m], sf[..., 2][m], rtol=1e-12)
    # principal ray: X = Y = 0 at (cx, cy)
    sf2 = np.zeros((3, 5, 4))
    sf2[..., 2:] = 10.0
    p0, _, _, _ = orc.reproject(sf2, np.ones((3, 5), np.uint8), 720.0, 0.54, 2.0, 1.0)
    assert p0[1, 2, 0] == 0 and p0[1, 2, 1] == 0


def test_census_window_orientation(orc):
    """G2/G4: for a 9x7 window a single darker pixel at (dx, dy) sets exactly bit
    k = (dy+3)*9 + (dx+4) (minus one past the centre); (dx, dy) = (0, 4) is outside."""
    ex = GOLD["census_orientation"][0]
    for dx, dy, k in ex["cases"]:
        img = np.full((15, 15), 100, np.uint8)
        img[7 + dy, 7 + dx] = 10
        assert int(orc.census(img, ex["w"], ex["h"])[7, 7]) == 1 << k, (dx, dy)
    img = np.full((15, 15), 100, np.uint8)
    img[7 + 4, 7] = 10
    assert int(orc.census(img, 9, 7)[7, 7]) == 0


def test_lr_row_hand_example(orc):
    ex = GOLD["lr_row"][0]
    dl = np.array([ex["dl"]], np.int16)
    dr = np.array([ex["dr"]], np.int16)
    oi, os_, v = orc.lr_check(dl, dl.astype(np.float64) + 0.25, dr, ex["T"])
    assert list(v[0]) == ex["valid"]
    assert list(oi[0]) == [d if ok else -1 for d, ok in zip(ex["dl"], ex["valid"])]
    assert list(os_[0]) == [d + 0.25 if ok else -1.0 for d, ok in zip(ex["dl"], ex["valid"])]


def test_stream_equals_independent_quads(orc):
    """Streaming mode: reusing frame k's map as D1 of quad
    k-1 and D0 of quad k changes nothing -- every quad is bit-identical to run_quad on
    (frame k, frame k+1)."""
    cfg = synth.CONFIGS["tiny"]
    prm = synth.sgm_params(cfg)
    v = synth.make_video(cfg, 4, 0)
    s = orc.run_stream(v, prm)
    assert len(s["maps"]) == 5 and len(s["quads"]) == 4
    for k in range(4):
        r = orc.run_quad(synth.video_quad(v, k), prm)
        for key in ("sf", "valid_sf", "p0", "dp", "valid_3d"):
            assert np.array_equal(s["quads"][k][key], r[key]), (k, key)
        for key in ("d_sub", "valid", "d_int"):
            assert np.array_equal(s["quads"][k]["disp0"][key], r["disp0"][key])
            assert np.array_equal(s["quads"][k]["disp1"][key], r["disp1"][key])


def test_video_generator_frames_match_quads():
    """make_video's frames 0/1 are make_quad's; later frames follow VIDEO_MOTION."""
    q = synth.make_quad("tiny", 2)
    v = synth.make_video("tiny", 3, 2)
    q0 = synth.video_quad(v, 0)
    for key in ("il0", "ir0", "il1", "ir1", "flow", "gt_d0", "gt_d1", "gt_d1w", "gt_noc"):
        assert np.array_equal(q[key], q0[key]), key
    # frame 3 has the motion amount of frame 1 (0, 1, 2, 1): identical images
    assert v["motion"] == [0, 1, 2, 1]
    assert np.array_equal(v["left"][1], v["left"][3]) and np.array_equal(v["right"][1], v["right"][3])
    # flows k -> k+1 and back cancel on the tiny pure translation
    assert np.allclose(v["flow"][1], -v["flow"][2])
