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


def _py_densify(f, v, g, K, lam):
    """Independent re-implementation: numpy lexsort for the K nearest, explicit walk."""
    H, W, C = f.shape
    f = f.astype(np.float64)
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
            d2 = (sx - x) ** 2 + (sy - y) ** 2
            order = np.lexsort((seeds, d2))[:K]
            wsum, acc = 0.0, np.zeros(C)
            for q in order:
                dx, dy = int(sx[q] - x), int(sy[q] - y)
                n = max(abs(dx), abs(dy))
                s = 0
                for k in range(1, n):
                    s += grad(x + math.floor(k * dx / n + 0.5), y + math.floor(k * dy / n + 0.5))
                w = 1.0 / (math.hypot(dx, dy) + lam * s)
                wsum += w
                acc += w * f[sy[q], sx[q]]
            out[y, x] = acc / wsum
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
