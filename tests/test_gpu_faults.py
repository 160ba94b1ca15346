"""Failure detection: the sweeps' bounded cross-CTA waits report a
time-out through the handle's device fault word instead of silently producing output,
and every entry point runs on its handle's device."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    return torch.device("cuda", 0)


def _tiny(dev, n=1):
    from paper_1801_04720_b200 import SGM, Camera, stack_quads
    cfg = synth.CONFIGS["tiny"]
    prm = synth.sgm_params(cfg)
    g = SGM.from_config(cfg, max_batch=n)
    imgs, flow = stack_quads([synth.make_quad(cfg, i) for i in range(n)], g.pitch, dev)
    return g, imgs, flow, Camera(prm["f"], prm["B"], prm["cx"], prm["cy"])


def test_forced_timeout_is_reported_not_silent(dev):
    from paper_1801_04720_b200 import _lib
    g, imgs, flow, cam = _tiny(dev)
    ref = {k: v.clone() for k, v in g.scene_flow(imgs, flow, cam).items()}
    torch.cuda.synchronize()
    assert g.device_error() == 0
    g.set_debug_flags(4)                       # every bounded wait times out
    g.scene_flow(imgs, flow, cam)              # enqueues fine; the fault is asynchronous
    torch.cuda.synchronize()
    code = g.device_error()
    assert code in (1, 2)
    with pytest.raises(_lib.SgmError) as ei:   # sticky: the next call fails loudly
        g.scene_flow(imgs, flow, cam)
    assert ei.value.code == 3
    assert "device fault" in g.lib.sgm_last_error_string().decode()
    assert g.device_error(clear=True) == code
    g.set_debug_flags(0)
    out = g.scene_flow(imgs, flow, cam)
    torch.cuda.synchronize()
    assert g.device_error() == 0
    for k in ref:
        assert torch.equal(out[k], ref[k]), k
    g.close()


def test_two_handles_interleaved(dev):
    """Two handles used alternately give the same bytes as each used alone."""
    g1, imgs, flow, cam = _tiny(dev)
    g2, _, _, _ = _tiny(dev)
    a = {k: v.clone() for k, v in g1.scene_flow(imgs, flow, cam).items()}
    b = g2.scene_flow(imgs, flow, cam)
    c = g1.scene_flow(imgs, flow, cam)
    torch.cuda.synchronize()
    for k in a:
        assert torch.equal(a[k], b[k]) and torch.equal(a[k], c[k]), k
    g1.close()
    g2.close()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs two GPUs")
def test_handles_on_two_devices():  # pragma: no cover - single-GPU boxes skip it
    from paper_1801_04720_b200 import SGM, Camera, stack_quads
    cfg = synth.CONFIGS["tiny"]
    prm = synth.sgm_params(cfg)
    cam = Camera(prm["f"], prm["B"], prm["cx"], prm["cy"])
    q = [synth.make_quad(cfg, 0)]
    outs = []
    hs = [SGM.from_config(cfg, device=d) for d in (0, 1)]
    for d, g in enumerate(hs):
        imgs, flow = stack_quads(q, g.pitch, torch.device("cuda", d))
        with torch.cuda.device(d):
            outs.append(g.scene_flow(imgs, flow, cam, stream=torch.cuda.current_stream(d)))
    for d in (0, 1):
        torch.cuda.synchronize(d)
    for k in outs[0]:
        assert np.array_equal(outs[0][k].cpu().numpy(), outs[1][k].cpu().numpy()), k
    for g in hs:
        g.close()
