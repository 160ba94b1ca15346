"""GPU parity of the densification (SPEC F-6): sgm_densify against
oracle.densify on the same seeded inputs, with every seed competing (window 0, the SPEC's
definition) and with a candidate window.  The seed ranking is bit-reproducible (fp64 keys
with one rounding each on both sides); the outputs are float32 on the GPU, fp64 in the
oracle: within 1e-4 * max(1, |value|)."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    return torch.device("cuda", 0)


def _close(a, b):
    return (np.abs(a - b) <= TOL * np.maximum(1.0, np.abs(b))).all()


@pytest.mark.parametrize("case", [(37, 23, 1, 0.05, 5, 1.0), (64, 48, 2, 0.3, 25, 1.0),
                                  (29, 31, 4, 0.9, 25, 0.5), (50, 9, 2, 0.02, 1, 0.0),
                                  (1, 40, 2, 0.2, 3, 1.0)], ids=str)
def test_densify_parity(orc, dev, case):
    from paper_1801_04720_b200 import densify
    W, H, C, dens, K, lam = case
    rng = np.random.default_rng(W * H + C)
    n = 2
    f = rng.normal(0, 6, (n, H, W, C)).astype(np.float32)
    v = (rng.random((n, H, W)) < dens).astype(np.uint8)
    v[:, 0, 0] = 1
    g = np.stack([synth.translated_pair(W, H, k, 0, 0)[0] for k in range(n)])
    T = lambda a: torch.from_numpy(a).to(dev)  # noqa: E731
    for window in (0, 3):
        out, cert = densify(T(f), T(v), T(g), K=K, lam=lam, window=window, count_certified=True)
        out = out.cpu().numpy()
        for i in range(n):
            ref = orc.densify(f[i], v[i], g[i], K=K, lam=lam, window=window)
            m = v[i] > 0
            assert np.array_equal(out[i][m], f[i][m])           # seeds kept bit for bit
            assert _close(out[i], ref), window
        if window == 0:                                         # every gap pixel is exact
            assert int(cert.item()) == int((v == 0).sum())


def test_densify_spec_examples_and_no_seed(dev):
    from paper_1801_04720_b200 import densify
    H, W = 6, 24
    g = np.zeros((H, W), np.uint8)
    g[:, 12:] = 255
    f = np.zeros((H, W, 2), np.float32)
    v = np.zeros((H, W), np.uint8)
    f[3, 23] = (10.0, 0.0)
    v[3, 0] = v[3, 23] = 1
    T = lambda a: torch.from_numpy(a).to(dev)  # noqa: E731
    out = densify(T(f), T(v), T(g)).cpu().numpy()
    assert (np.abs(out[:, :12, 0]) < 0.5).all() and (np.abs(out[:, 12:, 0] - 10) < 0.5).all()
    out, cnt = densify(T(f), T(np.zeros_like(v)), T(g), count_unfilled=True)
    assert int(cnt.item()) == H * W and (out == 0).all()


def test_densify_estimated_flow_full_size(orc, dev):
    """The GPU flow of a Driving pair (sparse after the consistency filter) densified with
    the left frame as guide, checked at sampled gap pixels against the exhaustive oracle."""
    from paper_1801_04720_b200 import FlowFields, densify
    q = synth.make_quad("driving", 0)
    H, W = q["il0"].shape
    ff = FlowFields(W, H, levels=3)
    A = torch.from_numpy(q["il0"][None]).to(dev)
    B = torch.from_numpy(q["il1"][None]).to(dev)
    fo = ff.flow(A, B)
    dense, cert = densify(fo["flow"], fo["valid"], A, count_certified=True)
    dense = dense.cpu().numpy()[0]
    flow = fo["flow"].cpu().numpy()[0]
    valid = fo["valid"].cpu().numpy()[0]
    gaps = np.argwhere(valid == 0)
    rng = np.random.default_rng(0)
    pick = gaps[rng.choice(len(gaps), 150, replace=False)]
    xy = np.stack([pick[:, 1], pick[:, 0]], 1)
    from paper_1801_04720_b200.flow import DENSIFY_WINDOW
    ref = orc.densify_points(flow, valid, q["il0"], xy, window=DENSIFY_WINDOW)
    assert _close(dense[pick[:, 0], pick[:, 1]], ref)
    assert np.array_equal(dense[valid > 0], flow[valid > 0])
    assert 0 <= int(cert.item()) <= len(gaps)
    ff.close()
