"""Pins for the optical-flow oracle (SPEC flow-fields
S:189-292).  Each SPEC worked example is checked, plus textbook facts (Walsh functions,
splitmix64), brute force on tiny inputs (exhaustive kNN by numpy, the scan-order sweep
re-run in Python) and the module's invariants."""
import numpy as np
import pytest
from scipy.linalg import hadamard

import synth

Q = 8


def _tex(W, H, seed):
    A, _ = synth.translated_pair(W, H, seed, 0, 0)
    return A


# ---------------------------------------------------------------- pyramid (FF2)
def test_downsample_hand_values(orc):
    img = np.array([[1, 2, 9], [3, 4, 9]], np.uint8)
    d = orc.ff_downsample(img)
    assert d.shape == (1, 2)
    assert d[0, 0] == 3          # (1+2+3+4+2) >> 2
    assert d[0, 1] == 9          # column 3 clamps to column 2
    one = orc.ff_downsample(np.array([[10, 13, 200]], np.uint8))
    assert list(one[0]) == [12, 200]   # rows clamp: (2*10 + 2*13 + 2) >> 2 = 12


# ---------------------------------------------------------------- WHT descriptors (FF3)
def _walsh_sequency(N):
    Hn = hadamard(N)
    changes = [(np.diff(r) != 0).sum() for r in Hn]
    return Hn[np.argsort(changes)]


@pytest.mark.parametrize("win", [4, 8, 16])
def test_wht_matches_matrix_transform(orc, win):
    """c(u,v) = (Wv P Wu^T) with scipy's Hadamard rows sorted by sign changes."""
    img = _tex(23, 19, 3)
    d = orc.ff_wht(img, win)
    Wm = _walsh_sequency(win)
    o = win // 2 - 1
    H, W = img.shape
    for (x, y) in [(0, 0), (11, 9), (22, 18), (5, 17)]:
        ys = np.clip(np.arange(y - o, y - o + win), 0, H - 1)
        xs = np.clip(np.arange(x - o, x - o + win), 0, W - 1)
        P = img[np.ix_(ys, xs)].astype(np.int64)
        C = Wm @ P @ Wm.T                          # C[v, u]
        assert np.array_equal(d[y, x], C[:4, :4].reshape(-1)), (x, y)


def test_wht_spec_examples(orc):
    c = 7
    for win in (4, 8, 16):
        d = orc.ff_wht(np.full((20, 20), c, np.uint8), win)
        assert d[10, 10, 0] == c * win * win and (d[10, 10, 1:] == 0).all()
    img = _tex(16, 16, 4)
    d1, d2 = orc.ff_wht(img, 8), orc.ff_wht(255 - img, 8)
    e0 = np.zeros(16, np.int64)
    e0[0] = 255 * 64
    assert (d2.astype(np.int64) == e0 - d1).all()                               # S:212 (affine)
    imp = np.zeros((8, 8), np.uint8)
    imp[2, 2] = 1                                   # patch of (3,3) starts at (2,2) for win 4
    d = orc.ff_wht(imp, 4)
    assert (np.abs(d[3, 3]) == 1).all()


# ---------------------------------------------------------------- data term (FF4)
def test_patch_cost_spec_examples(orc):
    A = _tex(30, 20, 5)
    assert orc.ff_patch_cost(A, A, 10, 10, 0, 0, r=4) == 0
    B = (A.astype(int) + 10).clip(0, 255).astype(np.uint8)
    A2 = (A // 2).astype(np.uint8)                  # no clipping: B2 = A2 + 10 exactly
    B2 = A2 + 10
    assert orc.ff_patch_cost(A2, B2, 10, 10, 0, 0, r=1) == 9 * 10 * Q * Q
    assert orc.ff_patch_cost(A, B, 10, 10, 1000 * Q, 0, r=1, penalty=20) == 9 * 20 * Q * Q
    assert orc.ff_patch_cost(A, B, 10, 10, 0, 0, r=0) == Q * Q * abs(int(A[10, 10]) - int(B[10, 10]))


def test_patch_cost_subpixel_on_ramp(orc):
    """B(x) = 2x: the bilinear sample at x + k/8 is 2x + k/4 exactly; A = B + 1 is met
    at the half-pixel flow (4/8, 0) with zero cost."""
    W, H = 40, 12
    B = np.tile((2 * np.arange(W)).astype(np.uint8), (H, 1))
    A = (B + 1).astype(np.uint8)
    assert orc.ff_patch_cost(A, B, 20, 6, 4, 0, r=3) == 0
    assert orc.ff_patch_cost(A, B, 20, 6, 2, 0, r=3) == 49 * 32       # |64 - 32| per sample
    A2, B2 = synth.translated_pair(40, 30, 6, 3, -2)
    assert orc.ff_patch_cost(A2, B2, 20, 15, 3 * Q, -2 * Q, r=4) == 0


# ---------------------------------------------------------------- kNN init (FF5)
def test_knn_exhaustive_brute_force(orc):
    A = _tex(9, 7, 7)
    B = _tex(9, 7, 8)
    flow, cost, nn = orc.ff_knn_init(A, B, win=4, knn=4, r=1)
    da = orc.ff_wht(A, 4).reshape(-1, 16).astype(np.int64)
    db = orc.ff_wht(B, 4).reshape(-1, 16).astype(np.int64)
    dist = ((da[:, None, :] - db[None, :, :]) ** 2).sum(-1)
    want = np.argsort(dist, axis=1, kind="stable")[:, :4]
    assert np.array_equal(nn.reshape(-1, 4), want)
    # the kept candidate is the first of minimal data term among the four
    W = 9
    for p in range(63):
        xa, ya = p % W, p // W
        cs = [orc.ff_patch_cost(A, B, xa, ya, (q % W - xa) * Q, (q // W - ya) * Q, r=1)
              for q in want[p]]
        k = int(np.argmin(cs))
        q = want[p][k]
        assert cost.reshape(-1)[p] == cs[k]
        assert tuple(flow.reshape(-1, 2)[p]) == ((q % W - xa) * Q, (q // W - ya) * Q)


def test_knn_spec_examples(orc):
    A = _tex(24, 18, 9)
    flow, cost, _ = orc.ff_knn_init(A, A, win=8, knn=4, r=2)
    assert (flow == 0).all()
    assert (cost[2:-2, 2:-2] == 0).all()            # interior: no sample leaves the image
    A, B = synth.translated_pair(40, 30, 10, 3, 0)
    flow, _, _ = orc.ff_knn_init(A, B, win=8, knn=4, r=3)
    inner = (slice(4, 26), slice(4, 33))
    ok = (flow[inner][..., 0] == 3 * Q) & (flow[inner][..., 1] == 0)
    assert ok.mean() >= 0.9
    two = np.array([[0, 255]], np.uint8)
    f, c, nn = orc.ff_knn_init(two, two, win=4, knn=1, r=0)
    assert f.shape == (1, 2, 2)


# ---------------------------------------------------------------- RNG (FF6)
def test_rng_is_splitmix64(orc):
    # key 0 -> the first output of SplitMix64 seeded with 0 (Steele, Lea & Flood 2014)
    assert orc.ff_rng(0, 0, 0, 0, 0) == 0xE220A8397B1DCDAF
    vals = {orc.ff_rng(5, 1, 2, x, y) for x in range(20) for y in range(20)}
    assert len(vals) == 400
    assert orc.ff_rng(5, 1, 2, 3, 4) == orc.ff_rng(5, 1, 2, 3, 4)


# ---------------------------------------------------------------- sweeps (FF7)
def _py_sweep(orc, A, B, flow, cost, s, level, r, penalty, R0, seed):
    """The sweep of S:231 written out in Python (scan order, strict acceptance), then the
    random search; costs from the oracle's data term."""
    H, W = A.shape
    flow, cost = flow.copy(), cost.copy()
    fwd = s % 2 == 0
    for jj in range(H):
        y = jj if fwd else H - 1 - jj
        for ii in range(W):
            x = ii if fwd else W - 1 - ii
            for (nx, ny) in ((x - 1, y), (x, y - 1)) if fwd else ((x + 1, y), (x, y + 1)):
                if 0 <= nx < W and 0 <= ny < H:
                    fu, fv = int(flow[ny, nx, 0]), int(flow[ny, nx, 1])
                    c = orc.ff_patch_cost(A, B, x, y, fu, fv, r, penalty)
                    if c < cost[y, x]:
                        cost[y, x] = c
                        flow[y, x] = (fu, fv)
    R = max(R0 >> s, 1)
    span = 2 * R * Q + 1
    for y in range(H):
        for x in range(W):
            z = orc.ff_rng(seed, level, s, x, y)
            fu = int(flow[y, x, 0]) + (z & 0xFFFFFFFF) % span - R * Q
            fv = int(flow[y, x, 1]) + (z >> 32) % span - R * Q
            c = orc.ff_patch_cost(A, B, x, y, fu, fv, r, penalty)
            if c < cost[y, x]:
                cost[y, x] = c
                flow[y, x] = (fu, fv)
    return flow, cost


@pytest.mark.parametrize("s", [0, 1, 2, 3])
def test_sweep_matches_python_scan(orc, s):
    A, B = synth.translated_pair(11, 8, 11, 2, 1)
    rng = np.random.default_rng(s)
    flow = rng.integers(-3 * Q, 3 * Q + 1, size=(8, 11, 2)).astype(np.int32)
    cost = np.array([[orc.ff_patch_cost(A, B, x, y, int(flow[y, x, 0]), int(flow[y, x, 1]), 1, 20)
                      for x in range(11)] for y in range(8)], np.int32)
    f1, c1 = orc.ff_sweep(A, B, flow, cost, s, level=1, r=1, penalty=20, R0=4, seed=77)
    f2, c2 = _py_sweep(orc, A, B, flow, cost, s, 1, 1, 20, 4, 77)
    assert np.array_equal(f1, f2) and np.array_equal(c1, c2)


def test_sweep_invariants(orc):
    A, B = synth.translated_pair(32, 24, 12, -2, 3)
    flow = np.zeros((24, 32, 2), np.int32)
    cost = np.array([[orc.ff_patch_cost(A, B, x, y, 0, 0) for x in range(32)] for y in range(24)],
                    np.int32)
    prev = cost
    for s in range(6):
        flow, cost = orc.ff_sweep(A, B, flow, cost, s)
        assert (cost <= prev).all()
        prev = cost
        for (x, y) in [(0, 0), (31, 23), (7, 19)]:
            assert cost[y, x] == orc.ff_patch_cost(A, B, x, y, int(flow[y, x, 0]), int(flow[y, x, 1]))
    # identical frames, zero field: already optimal -> unchanged
    A = _tex(20, 15, 13)
    f0 = np.zeros((15, 20, 2), np.int32)
    c0 = np.zeros((15, 20), np.int32)
    f1, c1 = orc.ff_sweep(A, A, f0, c0, 0)
    assert (f1 == 0).all() and (c1 == 0).all()


def test_propagation_spreads_a_seed(orc):
    """one correct seed in a wrong constant field spreads to >= 50 % of the pixels
    within 2 sweeps (random search with radius 1 px cannot reach the answer alone)."""
    A, B = synth.translated_pair(40, 30, 14, 5, 4)
    flow = np.full((30, 40, 2), -6 * Q, np.int32)
    flow[3, 3] = (5 * Q, 4 * Q)
    cost = np.array([[orc.ff_patch_cost(A, B, x, y, int(flow[y, x, 0]), int(flow[y, x, 1]))
                      for x in range(40)] for y in range(30)], np.int32)
    for s in range(2):
        flow, cost = orc.ff_sweep(A, B, flow, cost, s, R0=1)
    ok = (flow[..., 0] == 5 * Q) & (flow[..., 1] == 4 * Q)
    assert ok.mean() >= 0.5


# ---------------------------------------------------------------- lift (FF8)
def test_lift_spec_examples(orc):
    A = _tex(4, 4, 15)
    coarse = np.array([[[0, 0], [0, 0]], [[0, 0], [3 * Q, -Q]]], np.int32)     # (1,1) = (3,-1)
    f, c = orc.ff_lift(A, A, coarse, r=1)
    assert tuple(f[3, 3]) == (6 * Q, -2 * Q)
    assert tuple(f[2, 2]) == (6 * Q, -2 * Q) and tuple(f[1, 1]) == (0, 0)
    const = np.full((3, 5, 2), 5, np.int32)
    f, _ = orc.ff_lift(_tex(9, 6, 16), _tex(9, 6, 17), const, r=1)
    assert (f == 10).all()
    for (x, y) in [(0, 0), (8, 5)]:
        assert c.shape == (4, 4)


# ---------------------------------------------------------------- consistency (FF9)
def test_consistency_spec_examples(orc):
    z = np.zeros((6, 10, 2), np.int32)
    assert orc.ff_consistency(z, z, z).all()
    F = np.zeros((6, 10, 2), np.int32)
    F[2, 3] = (4 * Q, 0)
    G = np.zeros((6, 10, 2), np.int32)
    G[2, 7] = (-4 * Q, 0)
    v = orc.ff_consistency(F, G, G, thr_q=Q)
    assert v[2, 3] == 1
    G2 = G.copy()
    G2[2, 7] = (-1 * Q, 0)
    v = orc.ff_consistency(F, G, G2, thr_q=Q)
    assert v[2, 3] == 0                                                         # S:251 any field
    F[0, 9] = (Q, 0)                                                            # leaves the image
    assert orc.ff_consistency(F, G, G, thr_q=Q)[0, 9] == 0
    # bilinear inverse at a half-pixel target: G = -4 and -5 around -> mean -4.5 cancels F
    F = np.zeros((6, 10, 2), np.int32)
    F[1, 1] = (36, 0)                                                           # 4.5 px
    G = np.zeros((6, 10, 2), np.int32)
    G[1, 5] = (-32, 0)
    G[1, 6] = (-40, 0)
    assert orc.ff_consistency(F, G, G, thr_q=0)[1, 1] == 1


# ---------------------------------------------------------------- whole flow
def test_flow_translation_recovery(orc):
    for (tx, ty) in [(3, 0), (-5, 2), (8, -8)]:
        A, B = synth.translated_pair(64, 48, 20 + tx, tx, ty)
        f, v = orc.ff_flow(A, B, levels=2)
        inner = np.zeros(v.shape, bool)
        inner[8:40, 8:56] = True
        m = inner & (v > 0)
        assert m.sum() > 0.5 * inner.sum()
        epe = np.hypot(f[..., 0] / Q - tx, f[..., 1] / Q - ty)
        assert (epe[m] <= 0.5).mean() >= 0.9


def test_flow_filters_points_leaving_the_image(orc):
    tx, ty = 7, 0
    A, B = synth.translated_pair(64, 40, 31, tx, ty)
    f, v = orc.ff_flow(A, B, levels=2)
    leaving = np.zeros(v.shape, bool)
    leaving[:, 64 - tx:] = True                    # true correspondence outside B
    assert (v[leaving] == 0).mean() >= 0.95


def test_flow_deterministic(orc):
    A, B = synth.translated_pair(48, 32, 33, 2, 2)
    a = orc.ff_flow(A, B, levels=2, seed=5)
    b = orc.ff_flow(A, B, levels=2, seed=5)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
