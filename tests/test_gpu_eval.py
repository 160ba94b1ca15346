"""GPU parity of the evaluation step: sgm_evaluate through
the C ABI against oracle.evaluate on the same seeded inputs.  The counts are
integers decided in float32 on both sides, so the bar is bit-exact."""
import json
import os

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    return torch.device("cuda", 0)


def _handle(W, H, max_batch):
    from paper_1801_04720_b200 import SGM
    return SGM(W, H, 16, 5, 5, 10, 120, 1, -1, 0, max_batch, 0)


def _dev(inst, dev, with_gv=True):
    keys = ("sf", "valid_sf", "gt_d0", "gt_d1", "gt_flow", "gt_noc")
    t = {k: torch.from_numpy(np.ascontiguousarray(inst[k])).to(dev) for k in keys}
    t["gt_valid"] = torch.from_numpy(inst["gt_valid"]).to(dev) if with_gv else None
    return t


def _gpu_counts(g, t, **kw):
    c = g.evaluate(t["sf"], t["valid_sf"], t["gt_d0"], t["gt_d1"], t["gt_flow"], t["gt_noc"],
                   t["gt_valid"], **kw)
    torch.cuda.synchronize()
    return c.cpu().numpy()


def _orc_counts(orc, inst, i, with_gv=True, **kw):
    return orc.evaluate(inst["sf"][i], inst["valid_sf"][i], inst["gt_d0"][i], inst["gt_d1"][i],
                        inst["gt_flow"][i], inst["gt_noc"][i],
                        inst["gt_valid"][i] if with_gv else None, **kw)


# (W, H, n): a single pixel, one partial tile, several tiles with a ragged tail, a
# Driving-sized frame, and a batch whose per-quad size is not a multiple of 4.
SHAPES = [(1, 1, 1), (37, 11, 2), (97, 37, 3), (1242, 375, 1), (333, 77, 8)]


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("with_gv", [True, False])
def test_evaluate_parity(orc, dev, shape, with_gv):
    W, H, n = shape
    inst = synth.random_eval_instance(H, W, seed=W + 31 * H + n, n=n)
    g = _handle(W, H, n)
    c = _gpu_counts(g, _dev(inst, dev, with_gv))
    for i in range(n):
        assert np.array_equal(c[i], _orc_counts(orc, inst, i, with_gv)), f"quad {i}"
    g.close()


def test_evaluate_misaligned_inputs(orc, dev):
    """Byte masks and GT maps that do not start on a 16-byte boundary take the scalar
    kernel; the counts are the same."""
    W, H, n = 61, 13, 3
    inst = synth.random_eval_instance(H, W, seed=99, n=n)
    g = _handle(W, H, n)
    t = _dev(inst, dev)

    def shifted(x):
        flat = x.reshape(-1)
        buf = torch.empty(flat.numel() + 1, dtype=x.dtype, device=dev)
        buf[1:] = flat
        return buf[1:].view(x.shape)

    for key in ("valid_sf", "gt_noc", "gt_valid", "gt_d0"):
        tt = dict(t)
        tt[key] = shifted(t[key])
        assert tt[key].data_ptr() % 16 != 0
        c = _gpu_counts(g, tt)
        for i in range(n):
            assert np.array_equal(c[i], _orc_counts(orc, inst, i)), key
    g.close()


def test_evaluate_thresholds(orc, dev):
    W, H, n = 64, 20, 2
    inst = synth.random_eval_instance(H, W, seed=7, n=n)
    g = _handle(W, H, n)
    t = _dev(inst, dev)
    for ta, tr in ((0.0, 0.0), (1.0, 0.01), (3.0, 0.05), (10.0, 0.5)):
        c = _gpu_counts(g, t, tau_abs=ta, tau_rel=tr)
        for i in range(n):
            assert np.array_equal(c[i], _orc_counts(orc, inst, i, tau_abs=ta, tau_rel=tr))
    g.close()


@pytest.mark.parametrize("ex", GOLD["outlier"], ids=lambda e: f"{e['err']}@{e['mag']}")
def test_outlier_rule_examples_gpu(dev, ex):
    """The SPEC worked examples on the device, one channel per pixel."""
    inst = {"sf": np.zeros((1, 1, 3, 4), np.float32), "valid_sf": np.ones((1, 1, 3), np.uint8),
            "gt_d0": np.full((1, 1, 3), 7.0, np.float32), "gt_d1": np.full((1, 1, 3), 7.0, np.float32),
            "gt_flow": np.zeros((1, 1, 3, 2), np.float32), "gt_noc": np.ones((1, 1, 3), np.uint8),
            "gt_valid": np.ones((1, 1, 3), np.uint8)}
    inst["sf"][..., 2:] = 7.0
    e, m = ex["err"], ex["mag"]
    inst["gt_d0"][0, 0, 0] = m; inst["sf"][0, 0, 0, 2] = m + e
    inst["gt_d1"][0, 0, 1] = m; inst["sf"][0, 0, 1, 3] = m + e
    inst["gt_flow"][0, 0, 2] = (m, 0.0); inst["sf"][0, 0, 2, 0] = m + e
    g = _handle(3, 1, 1)
    c = _gpu_counts(g, _dev(inst, dev))[0]
    w = int(ex["outlier"])
    assert list(c[0]) == [3, 3, w, w, w, 3 * w], ex["cite"]
    g.close()


def test_evaluate_deterministic_and_overwrites(dev):
    W, H, n = 200, 50, 4
    inst = synth.random_eval_instance(H, W, seed=3, n=n)
    g = _handle(W, H, n)
    t = _dev(inst, dev)
    counts = torch.full((n, 2, 6), 12345, dtype=torch.int64, device=dev)
    a = g.evaluate(t["sf"], t["valid_sf"], t["gt_d0"], t["gt_d1"], t["gt_flow"], t["gt_noc"],
                   t["gt_valid"], counts=counts).clone()
    b = g.evaluate(t["sf"], t["valid_sf"], t["gt_d0"], t["gt_d1"], t["gt_flow"], t["gt_noc"],
                   t["gt_valid"], counts=counts)
    assert torch.equal(a, b)
    assert int(a[:, 0, 0].sum()) == int(inst["gt_valid"].sum())
    g.close()


def test_evaluate_invalid_args(dev):
    from paper_1801_04720_b200._lib import SgmError
    W, H = 16, 4
    inst = synth.random_eval_instance(H, W, seed=1, n=1)
    g = _handle(W, H, 1)
    t = _dev(inst, dev)
    with pytest.raises(SgmError):
        g.evaluate(t["sf"], t["valid_sf"], t["gt_d0"], t["gt_d1"], t["gt_flow"], t["gt_noc"],
                   tau_abs=-1.0)
    with pytest.raises(SgmError):
        g.evaluate(t["sf"], t["valid_sf"], t["gt_d0"], t["gt_d1"], t["gt_flow"], t["gt_noc"],
                   tau_rel=float("nan"))
    big = {k: v.repeat(2, *([1] * (v.dim() - 1))) for k, v in t.items() if v is not None}
    with pytest.raises(SgmError):             # n > max_batch
        g.evaluate(big["sf"], big["valid_sf"], big["gt_d0"], big["gt_d1"], big["gt_flow"],
                   big["gt_noc"])
    g.close()


@pytest.mark.parametrize("name", ["tiny", "driving"])
def test_evaluate_end_to_end(orc, dev, name):
    """The whole path then the evaluation, on the generator's ground truth: the GPU
    counts equal the oracle's counts of the GPU's own scene flow (bit-exact), and
    differ from the counts of the oracle's scene flow only at pixels whose error
    lies within the 1e-4 px sub-pixel tolerance of a threshold."""
    from paper_1801_04720_b200 import SGM, Camera, stack_quads
    cfg = synth.CONFIGS[name]
    prm = synth.sgm_params(cfg)
    n = 2
    quads = [synth.make_quad(cfg, i) for i in range(n)]
    g = SGM.from_config(cfg, max_batch=n)
    imgs, flow = stack_quads(quads, g.pitch, dev)
    out = g.scene_flow(imgs, flow, Camera(prm["f"], prm["B"], prm["cx"], prm["cy"]))
    gd0 = torch.from_numpy(np.stack([q["gt_d0"] for q in quads])).to(dev)
    gd1 = torch.from_numpy(np.stack([q["gt_d1w"] for q in quads])).to(dev)
    noc = torch.from_numpy(np.stack([q["gt_noc"] for q in quads])).to(dev)
    c = g.evaluate(out["sf"], out["valid_sf"], gd0, gd1, flow, noc).cpu().numpy()
    sf = out["sf"].cpu().numpy()
    vsf = out["valid_sf"].cpu().numpy()
    for i, q in enumerate(quads):
        mine = orc.evaluate(sf[i], vsf[i], q["gt_d0"], q["gt_d1w"], q["flow"], q["gt_noc"])
        assert np.array_equal(c[i], mine)
        r = orc.run_quad(q, prm)
        ref = orc.evaluate(r["sf"].astype(np.float32), r["valid_sf"], q["gt_d0"], q["gt_d1w"],
                           q["flow"], q["gt_noc"])
        assert np.array_equal(c[i][:, :2], ref[:, :2])          # same masks -> same n_gt, n_eval
        assert np.abs(c[i] - ref).max() <= max(2, ref[0, 1] // 100000)
    g.close()
