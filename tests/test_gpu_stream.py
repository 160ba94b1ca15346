"""GPU parity of the streaming (video) mode:
sgm_scene_flow_stream computes each frame's map once; every quad must equal, bit for
bit, sgm_scene_flow on (frame k, frame k+1), and match oracle.run_stream within the
tolerances of test_gpu_parity."""
import numpy as np
import pytest
import torch

import synth
from test_gpu_parity import SUB_TOL, _check_sceneflow, _np

pytestmark = pytest.mark.gpu

QUAD_KEYS = ("sf", "valid_sf", "p0", "dp", "valid_3d")


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    return torch.device("cuda", 0)


def _stream_vs_quads(g, video, cam, dev):
    from paper_1801_04720_b200 import stack_quads, stack_video
    n = video["flow"].shape[0]
    imgs, flow = stack_video(video, g.pitch, dev)
    launches = g.launch_count()
    out = g.scene_flow_stream(imgs, flow, cam)
    torch.cuda.synchronize()
    assert g.launch_count() - launches == 5
    quads = [synth.video_quad(video, k) for k in range(n)]
    qi, qf = stack_quads(quads, g.pitch, dev)
    ref = g.scene_flow(qi, qf, cam)
    torch.cuda.synchronize()
    for k in QUAD_KEYS:
        assert torch.equal(out[k], ref[k]), k
    for key in ("disp_int", "disp_sub", "disp_valid"):
        for f in range(n + 1):
            want = ref[key][f, 0] if f < n else ref[key][n - 1, 1]
            assert torch.equal(out[key][f], want), (key, f)
            if 0 < f < n:
                assert torch.equal(ref[key][f - 1, 1], ref[key][f, 0])
    return out


@pytest.mark.parametrize("name,n", [("tiny", 5), ("driving", 3),
                                    pytest.param("wide", 2, marks=pytest.mark.slow)])
def test_stream_parity(orc, dev, name, n):
    from paper_1801_04720_b200 import SGM, Camera
    cfg = synth.CONFIGS[name]
    prm = synth.sgm_params(cfg)
    video = synth.make_video(cfg, n, 0)
    g = SGM.from_config(cfg, max_batch=n)
    cam = Camera(prm["f"], prm["B"], prm["cx"], prm["cy"])
    out = _stream_vs_quads(g, video, cam, dev)
    s = orc.run_stream(video, prm)
    for f in range(n + 1):
        m = s["maps"][f]
        assert np.array_equal(_np(out["disp_valid"][f]), m["valid"])
        assert np.array_equal(_np(out["disp_int"][f]), m["d_int"])
        assert np.abs(_np(out["disp_sub"][f]) - m["d_sub"]).max() <= SUB_TOL
    for k in range(n):
        o = s["quads"][k]
        r = {key: out[key][k] for key in QUAD_KEYS}
        _check_sceneflow(r, o["sf"], o["valid_sf"], o["p0"], o["p1"], o["dp"], o["valid_3d"])
    g.close()


def test_stream_single_quad_and_ragged(dev):
    """n = 1 (two frames) equals sgm_scene_flow on one quad; a 97x37 video with D=64."""
    from paper_1801_04720_b200 import SGM, Camera
    cfg = synth.CONFIGS["tiny"]
    prm = synth.sgm_params(cfg)
    g = SGM.from_config(cfg, max_batch=1)
    cam = Camera(prm["f"], prm["B"], prm["cx"], prm["cy"])
    _stream_vs_quads(g, synth.make_video(cfg, 1, 3), cam, dev)
    g.close()


def test_stream_host_matches_device(dev):
    from paper_1801_04720_b200 import SGM, Camera, stack_video
    cfg = synth.CONFIGS["tiny"]
    prm = synth.sgm_params(cfg)
    n = 4
    g = SGM.from_config(cfg, max_batch=n)
    cam = Camera(prm["f"], prm["B"], prm["cx"], prm["cy"])
    videos = [synth.make_video(cfg, n, i) for i in range(3)]
    refs = []
    for v in videos:
        imgs, flow = stack_video(v, g.pitch, dev)
        refs.append({k: t.cpu() for k, t in g.scene_flow_stream(imgs, flow, cam).items()})
    torch.cuda.synchronize()
    outs = []
    for v in videos:                     # back to back through the two staging slots
        hi = torch.from_numpy(np.stack([v["left"], v["right"]], 1)).pin_memory()
        hf = torch.from_numpy(v["flow"]).pin_memory()
        ho = g.alloc_outputs(n, pinned_host=True, stream_mode=True)
        g.scene_flow_stream_host(hi, hf, cam, ho)
        outs.append(ho)
    torch.cuda.synchronize()
    for ho, ref in zip(outs, refs):
        for k in ho:
            assert torch.equal(ho[k], ref[k]), k
    g.close()


def test_stream_invalid(dev):
    from paper_1801_04720_b200 import SGM, Camera, stack_video
    from paper_1801_04720_b200._lib import SgmError
    cfg = synth.CONFIGS["tiny"]
    prm = synth.sgm_params(cfg)
    g = SGM.from_config(cfg, max_batch=2)
    cam = Camera(prm["f"], prm["B"], prm["cx"], prm["cy"])
    imgs, flow = stack_video(synth.make_video(cfg, 3, 0), g.pitch, dev)
    with pytest.raises(SgmError):        # n = 3 > max_batch
        g.scene_flow_stream(imgs, flow, cam)
    with pytest.raises(ValueError):      # frames != flows + 1
        g.scene_flow_stream(imgs[:3], flow, cam)
    g.close()
