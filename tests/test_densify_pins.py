"""Pins for the densification oracle (SPEC densify S:253-262, F-6;
readings DN1-DN4 in DESIGN.md): the SPEC's worked examples, hand-computed edge-aware
distances, the module invariants (S:259 seeds kept, idempotence) and a brute-force
Python re-implementation on tiny inputs."""
import math

import numpy as np
import pytest

import synth


def test_edge_distance_hand_values(orc):
    flat = np.full((5, 20), 77, np.uint8)
    assert orc.edge_distance(flat, (2, 2), (15, 2)) == pytest.approx(13.0)
    assert orc.edge_distance(flat, (0, 0), (3, 4)) == pytest.approx(5.0)
    step = np.zeros((5, 20), np.uint8)
    step[:, 10:] = 255
    # the segment (2,2) -> (15,2) crosses x = 9 and x = 10, each with |G(x+1) - G(x-1)| = 255
    assert orc.edge_distance(step, (2, 2), (15, 2)) == pytest.approx(13.0 + 2 * 255)
    assert orc.edge_distance(step, (2, 2), (8, 2)) == pytest.approx(6.0)
    assert orc.edge_distance(step, (2, 2), (15, 2), lam=0.5) == pytest.approx(13.0 + 255)
    # adjacent pixels have no interior samples
    assert orc.edge_distance(step, (9, 1), (10, 1)) == pytest.approx(1.0)


def test_fully_valid_is_identity(orc):
    rng = np.random.default_rng(0)
    f = rng.normal(0, 5, (12, 17, 2)).astype(np.float32)
    g = synth.translated_pair(17, 12, 1, 0, 0)[0]
    out = orc.densify(f, np.ones((12, 17), np.uint8), g)
    assert np.array_equal(out, f.astype(np.float64))


def test_single_seed_fills_everything(orc):
    f = np.zeros((9, 13, 2), np.float32)
    v = np.zeros((9, 13), np.uint8)
    f[4, 6] = (2.0, 3.0)
    v[4, 6] = 1
    out = orc.densify(f, v, np.full((9, 13), 100, np.uint8))
    assert np.allclose(out, np.array([2.0, 3.0]), rtol=0, atol=1e-12)


def test_two_seeds_across_an_edge(orc):
    H, W = 6, 24
    g = np.zeros((H, W), np.uint8)
    g[:, 12:] = 255
    f = np.zeros((H, W, 2), np.float32)
    v = np.zeros((H, W), np.uint8)
    f[3, 0] = (0.0, 0.0)
    f[3, 23] = (10.0, 0.0)
    v[3, 0] = v[3, 23] = 1
    out = orc.densify(f, v, g)
    assert (np.abs(out[:, :12, 0] - 0.0) < 0.5).all()
    assert (np.abs(out[:, 12:, 0] - 10.0) < 0.5).all()


def test_invariants(orc):
    rng = np.random.default_rng(1)
    H, W = 14, 19
    f = rng.normal(0, 8, (H, W, 4)).astype(np.float32)
    v = (rng.random((H, W)) < 0.3).astype(np.uint8)
    g = synth.translated_pair(W, H, 2, 0, 0)[0]
    out = orc.densify(f, v, g, K=7)
    m = v > 0
    assert np.array_equal(out[m], f[m].astype(np.float64))                     # seeds kept
    lo, hi = f[m].min(0), f[m].max(0)
    assert (out >= lo - 1e-9).all() and (out <= hi + 1e-9).all()               # convex weights
    again = orc.densify(out.astype(np.float32), np.ones((H, W), np.uint8), g)
    assert np.array_equal(again, out.astype(np.float32).astype(np.float64))   # idempotent on dense
    const = np.full((H, W, 1), 4.5, np.float32)
    assert np.allclose(orc.densify(const, v, g)[..., 0], 4.5, atol=1e-12)


def _py_densify(f, v, g, K, lam, window=0):
    """Independent re-implementation of SPEC F-6: every candidate seed's
    edge-aware distance by an explicit walk, the K smallest by numpy lexsort (ties to the
    smaller index), inverse-distance weights."""
    H, W, C = f.shape
    f = f.astype(np.float64)
    lam = float(np.float32(lam))                      # the ABI's float32 parameter
    seeds = np.flatnonzero(v.reshape(-1))
    sy, sx = seeds // W, seeds % W
    out = f.astype(np.float64).copy()
    gi = g.astype(np.int64)

    def grad(x, y):
        return (abs(gi[y, min(x + 1, W - 1)] - gi[y, max(x - 1, 0)]) +
                abs(gi[min(y + 1, H - 1), x] - gi[max(y - 1, 0), x]))

    for y in range(H):
        for x in range(W):
            if v[y, x]:
                continue
            ch = np.maximum(np.abs(sx - x), np.abs(sy - y))
            if window > 0:
                counts = np.bincount(ch, minlength=max(W, H) + 1).cumsum()
                rho = int(np.argmax(counts >= K)) if counts[-1] >= K else max(W, H)
                cand = np.flatnonzero(ch <= max(window, rho))
            else:
                cand = np.arange(len(seeds))
            de = []
            for q in cand:
                dx, dy = int(sx[q] - x), int(sy[q] - y)
                n = max(abs(dx), abs(dy))
                s = 0
                for k in range(1, n):
                    s += grad(x + math.floor(k * dx / n + 0.5), y + math.floor(k * dy / n + 0.5))
                de.append(math.sqrt(dx * dx + dy * dy) + lam * s)
            de = np.array(de)
            order = cand[np.lexsort((seeds[cand], de))][:K]
            dsel = de[np.lexsort((seeds[cand], de))][:K]
            w = 1.0 / dsel
            out[y, x] = (w[:, None] * f[sy[order], sx[order]]).sum(0) / w.sum()
    return out


@pytest.mark.parametrize("seed", range(3))
def test_brute_force(orc, seed):
    rng = np.random.default_rng(10 + seed)
    H, W = 9, 11
    f = rng.normal(0, 3, (H, W, 2)).astype(np.float32)
    v = (rng.random((H, W)) < 0.25).astype(np.uint8)
    v[0, 0] = 1
    g = (rng.random((H, W)) * 255).astype(np.uint8)
    out = orc.densify(f, v, g, K=5, lam=0.7)
    ref = _py_densify(f, v, g, 5, 0.7)
    assert np.allclose(out, ref, rtol=1e-12, atol=1e-12)
    outw = orc.densify(f, v, g, K=3, lam=0.7, window=2)
    refw = _py_densify(f, v, g, 3, 0.7, window=2)
    assert np.allclose(outw, refw, rtol=1e-12, atol=1e-12)


def test_edge_aware_ranking_not_euclidean(orc):
    """SPEC F-6 ranks seeds by the edge-aware distance, not by Euclidean distance: with
    K = 1, a gap pixel next to a strong edge takes the farther seed on its own side
    (d_e = 6) over the nearer one across the edge (d_e = 2 + 255)."""
    H, W = 5, 20
    g = np.zeros((H, W), np.uint8)
    g[:, 11:] = 255                                      # edge between x = 10 and x = 11
    f = np.zeros((H, W, 1), np.float32)
    v = np.zeros((H, W), np.uint8)
    v[2, 12], f[2, 12] = 1, 7.0                          # across the edge, |p - s| = 2
    v[2, 4], f[2, 4] = 1, -3.0                           # same side, |p - s| = 6
    out = orc.densify(f, v, g, K=1)
    assert out[2, 10, 0] == -3.0
    assert orc.edge_distance(g, (10, 2), (12, 2)) == pytest.approx(2.0 + 255)   # interior x = 11: g = 255
    assert orc.edge_distance(g, (10, 2), (4, 2)) == pytest.approx(6.0)          # interior x = 9..5: g = 0
    # both weights enter with K = 2: the closer-by-d_e seed dominates
    out2 = orc.densify(f, v, g, K=2)
    w_a, w_b = 1 / 6.0, 1 / (2.0 + 255)
    assert out2[2, 10, 0] == pytest.approx((w_a * -3.0 + w_b * 7.0) / (w_a + w_b), rel=1e-12)


def test_window_restricts_candidates(orc):
    """window > 0: only seeds within Chebyshev distance max(window, rho_K) compete."""
    H, W = 3, 30
    g = np.full((H, W), 50, np.uint8)                    # flat guide: d_e = Euclidean
    f = np.zeros((H, W, 1), np.float32)
    v = np.zeros((H, W), np.uint8)
    v[1, 0], f[1, 0] = 1, 1.0
    v[1, 29], f[1, 29] = 1, 2.0
    full = orc.densify(f, v, g, K=2)
    x = 3                                                # distances 3 and 26
    assert full[1, x, 0] == pytest.approx((1 / 3 * 1.0 + 1 / 26 * 2.0) / (1 / 3 + 1 / 26), rel=1e-12)
    win = orc.densify(f, v, g, K=2, window=5)            # rho_2 = 26 at x = 3: both still in
    assert win[1, x, 0] == full[1, x, 0]
    win1 = orc.densify(f, v, g, K=1, window=5)           # rho_1 = 3: the far seed is out
    assert win1[1, x, 0] == 1.0


def test_no_seed_is_an_error(orc):
    with pytest.raises(ValueError):
        orc.densify(np.zeros((4, 4, 2), np.float32), np.zeros((4, 4), np.uint8), np.zeros((4, 4), np.uint8))


def test_points_equal_full(orc):
    rng = np.random.default_rng(4)
    H, W = 13, 17
    f = rng.normal(0, 3, (H, W, 2)).astype(np.float32)
    v = (rng.random((H, W)) < 0.4).astype(np.uint8)
    g = synth.translated_pair(W, H, 5, 0, 0)[0]
    full = orc.densify(f, v, g, K=9)
    xy = np.stack([rng.integers(0, W, 30), rng.integers(0, H, 30)], 1)
    pts = orc.densify_points(f, v, g, xy, K=9)
    assert np.array_equal(pts, full[xy[:, 1], xy[:, 0]])
