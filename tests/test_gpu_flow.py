"""GPU parity of the optical-flow core: every stage and
the whole flow through include/sgmflow.h against oracle/flow_oracle.c on the same seeded
inputs.  All arithmetic is integer on both sides, so the bar is bit-exact."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu
Q = 8


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    return torch.device("cuda", 0)


def _ff(W, H, **kw):
    from paper_1801_04720_b200 import FlowFields
    return FlowFields(W, H, **kw)


def _t(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


@pytest.mark.parametrize("win", [4, 8, 16])
def test_descriptors(orc, dev, win):
    img = synth.translated_pair(53, 29, win, 0, 0)[0]
    ff = _ff(53, 29, desc_window=win)
    d = ff.descriptors(_t(img, dev)).cpu().numpy()
    assert np.array_equal(d, orc.ff_wht(img, win))
    ff.close()


@pytest.mark.parametrize("r", [0, 1, 4, 7])
def test_patch_cost(orc, dev, r):
    A, B = synth.translated_pair(41, 33, 2 + r, 3, -2)
    rng = np.random.default_rng(r)
    q = np.stack([rng.integers(0, 41, 300), rng.integers(0, 33, 300),
                  rng.integers(-60 * Q, 60 * Q, 300), rng.integers(-40 * Q, 40 * Q, 300)], 1)
    q[:20, 2:] = rng.integers(-Q, Q, (20, 2))            # near-zero sub-pixel flows
    ff = _ff(41, 33)
    got = ff.patch_cost(_t(A, dev), _t(B, dev), torch.from_numpy(q.astype(np.int32)), radius=r)
    got = got.cpu().numpy()
    want = [orc.ff_patch_cost(A, B, *map(int, row), r=r) for row in q]
    assert np.array_equal(got, np.array(want, np.int32))
    ff.close()


@pytest.mark.parametrize("shape", [(23, 17), (64, 48), (129, 71)], ids=str)
def test_knn_init(orc, dev, shape):
    W, H = shape
    A, B = synth.translated_pair(W, H, W, 4, 1)
    ff = _ff(W, H, knn=4)
    f, c, nn = ff.knn_init(_t(A, dev), _t(B, dev), radius=3)
    of, oc, onn = orc.ff_knn_init(A, B, win=8, knn=4, r=3)
    assert np.array_equal(nn.cpu().numpy(), onn)
    assert np.array_equal(f.cpu().numpy(), of)
    assert np.array_equal(c.cpu().numpy(), oc)
    ff.close()


@pytest.mark.parametrize("shape", [(31, 9), (70, 37), (150, 64), (5, 40)], ids=str)
@pytest.mark.parametrize("sweep", [0, 1, 2, 5])
def test_sweep(orc, dev, shape, sweep):
    """One propagation sweep (scan order across rows, bands and CTAs) + random search."""
    W, H = shape
    A, B = synth.translated_pair(W, H, W + H, -3, 2)
    rng = np.random.default_rng(sweep)
    flow = rng.integers(-4 * Q, 4 * Q + 1, size=(H, W, 2)).astype(np.int32)
    flow[H // 2, W // 2] = (-3 * Q, 2 * Q)                 # one correct seed to propagate
    cost = np.array([[orc.ff_patch_cost(A, B, x, y, int(flow[y, x, 0]), int(flow[y, x, 1]), r=2)
                      for x in range(W)] for y in range(H)], np.int32)
    ff = _ff(W, H, search_radius=4)
    gf, gc = _t(flow, dev), _t(cost, dev)
    ff.sweep(_t(A, dev), _t(B, dev), gf, gc, sweep, level=1, seed=9, radius=2)
    of, oc = orc.ff_sweep(A, B, flow, cost, sweep, level=1, r=2, R0=4, seed=9)
    assert np.array_equal(gf.cpu().numpy(), of)
    assert np.array_equal(gc.cpu().numpy(), oc)
    ff.close()


@pytest.mark.parametrize("shape,levels", [((64, 48), 2), ((97, 61), 3), ((40, 150), 3)], ids=str)
def test_field(orc, dev, shape, levels):
    W, H = shape
    pairs = [synth.translated_pair(W, H, 100 + k, 2 + k, -1) for k in range(2)]
    A = np.stack([p[0] for p in pairs])
    B = np.stack([p[1] for p in pairs])
    ff = _ff(W, H, levels=levels, max_batch=2)
    f, c = ff.field(_t(A, dev), _t(B, dev), seed=3, radius=4)
    for k in range(2):
        of, oc = orc.ff_field(A[k], B[k], levels=levels, seed=3)
        assert np.array_equal(f[k].cpu().numpy(), of), k
        assert np.array_equal(c[k].cpu().numpy(), oc), k
    ff.close()


def test_flow_full(orc, dev):
    """Forward + two inverse fields + consistency on a synthetic quad's left frames."""
    q = synth.make_quad("tiny", 0)
    A, B = q["il0"][None], q["il1"][None]
    H, W = q["il0"].shape
    ff = _ff(W, H, levels=2)
    out = ff.flow(_t(A, dev), _t(B, dev), want_fields=True)
    of, ov = orc.ff_flow(A[0], B[0], levels=2)
    assert np.array_equal(out["fields_q"][0, 0].cpu().numpy(), of)
    assert np.array_equal(out["valid"][0].cpu().numpy(), ov)
    assert np.array_equal(out["flow"][0].cpu().numpy(), of.astype(np.float32) / Q)
    G1 = orc.ff_field(B[0], A[0], levels=2, seed=2)[0]
    G2 = orc.ff_field(B[0], A[0], levels=2, seed=3, r=6)[0]
    assert np.array_equal(out["fields_q"][0, 1].cpu().numpy(), G1)
    assert np.array_equal(out["fields_q"][0, 2].cpu().numpy(), G2)
    v = ff.consistency(_t(of, dev), _t(G1, dev), _t(G2, dev)).cpu().numpy()
    assert np.array_equal(v, ov)
    ff.close()


@pytest.mark.slow
def test_flow_driving_full_size(orc, dev):
    """BASELINE configs[1] size (1242x375) with 4 levels: every vector and mask bit."""
    q = synth.make_quad("driving", 0)
    H, W = q["il0"].shape
    ff = _ff(W, H, levels=4)
    out = ff.flow(_t(q["il0"][None], dev), _t(q["il1"][None], dev), want_fields=True)
    of, ov = orc.ff_flow(q["il0"], q["il1"], levels=4)
    assert np.array_equal(out["fields_q"][0, 0].cpu().numpy(), of)
    assert np.array_equal(out["valid"][0].cpu().numpy(), ov)
    ff.close()


def test_flow_deterministic_and_feeds_scene_flow(dev):
    from paper_1801_04720_b200 import SGM, Camera, stack_quads
    cfg = synth.CONFIGS["tiny"]
    prm = synth.sgm_params(cfg)
    quads = [synth.make_quad(cfg, k) for k in range(2)]
    A = torch.from_numpy(np.stack([q["il0"] for q in quads])).to(dev)
    B = torch.from_numpy(np.stack([q["il1"] for q in quads])).to(dev)
    ff = _ff(cfg.W, cfg.H, levels=2, max_batch=2)
    o1 = ff.flow(A, B)
    o2 = ff.flow(A, B)
    assert torch.equal(o1["flow"], o2["flow"]) and torch.equal(o1["valid"], o2["valid"])
    # estimated flow vs the generator's (Tiny is a pure (3,1) translation): most surviving
    # vectors are exact
    fl = o1["flow"].cpu().numpy()
    v = o1["valid"].cpu().numpy() > 0
    gt = np.stack([q["flow"] for q in quads])
    assert (np.abs(fl - gt).max(-1)[v] <= 0.5).mean() > 0.9
    # the estimated flow and its mask drive the combination (G23 flow mask)
    g = SGM.from_config(cfg, max_batch=2)
    imgs, _ = stack_quads(quads, g.pitch, dev)
    out = g.scene_flow(imgs, o1["flow"], Camera(prm["f"], prm["B"], prm["cx"], prm["cy"]),
                       flow_valid=o1["valid"])
    vs = out["valid_sf"].cpu().numpy() > 0
    assert not (vs & ~v).any()
    g.close()
    ff.close()


@pytest.mark.parametrize("shape,levels", [((1, 40), 3), ((40, 1), 3), ((3, 2), 2), ((2, 2), 1),
                                          ((17, 5), 4)], ids=str)
def test_flow_degenerate_shapes(orc, dev, shape, levels):
    """Single-row / single-column images, a 1x1 coarsest level, fewer pixels than kNN
    candidates' tiles: the whole flow stays bit-exact."""
    W, H = shape
    A, B = synth.translated_pair(W, H, 50 + W + H, 1, 0)
    ff = _ff(W, H, levels=levels, knn=4)
    out = ff.flow(_t(A[None], dev), _t(B[None], dev), want_fields=True)
    of, ov = orc.ff_flow(A, B, levels=levels)
    assert np.array_equal(out["fields_q"][0, 0].cpu().numpy(), of)
    assert np.array_equal(out["valid"][0].cpu().numpy(), ov)
    ff.close()


@pytest.mark.slow
def test_flow_highres_full_size(orc, dev):
    """BASELINE configs[3] size (2048x1024), 4 levels: every vector and mask bit."""
    q = synth.make_quad("highres", 0)
    H, W = q["il0"].shape
    ff = _ff(W, H, levels=4)
    out = ff.flow(_t(q["il0"][None], dev), _t(q["il1"][None], dev), want_fields=True)
    of, ov = orc.ff_flow(q["il0"], q["il1"], levels=4)
    assert np.array_equal(out["fields_q"][0, 0].cpu().numpy(), of)
    assert np.array_equal(out["valid"][0].cpu().numpy(), ov)
    ff.close()
