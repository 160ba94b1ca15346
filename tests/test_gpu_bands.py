"""The sweep band geometry is chosen per call (band_geometry in csrc/api.cu: 10-17 rows
per band, heights spread evenly, K2).  Every band height must give bit-identical
results: each setting runs in its own process (SGM_BAND_ROWS is read once per process)
and the outputs' digests are compared with the default geometry's."""
import hashlib
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import hashlib, json, sys
import torch
sys.path.insert(0, sys.argv[1])
import synth
from paper_1801_04720_b200 import SGM, Camera, stack_quads
cfg = synth.CONFIGS["driving"]
prm = synth.sgm_params(cfg)
n = 2
g = SGM.from_config(cfg, max_batch=n)
quads = [synth.make_quad(cfg, 40 + i) for i in range(n)]
imgs, flow = stack_quads(quads, g.pitch, torch.device("cuda"))
out = g.scene_flow(imgs, flow, Camera(prm["f"], prm["B"], prm["cx"], prm["cy"]))
torch.cuda.synchronize()
res = {"band_rows": g.geometry()["band_rows"]}
for k in sorted(out):
    res[k] = hashlib.sha256(out[k].cpu().contiguous().view(torch.uint8).numpy().tobytes()).hexdigest()
print(json.dumps(res))
"""


def _run(rows, fine=None):
    env = dict(os.environ)
    env.pop("SGM_BAND_ROWS", None)
    env.pop("SGM_FINE_SYNC", None)
    if rows:
        env["SGM_BAND_ROWS"] = str(rows)
    if fine is not None:
        env["SGM_FINE_SYNC"] = str(fine)
    r = subprocess.run([sys.executable, "-c", CHILD, ROOT], env=env, capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_band_heights_bit_identical():
    ref = _run(0)
    for rows in (10, 13, 16, 17):
        got = _run(rows)
        for k, v in ref.items():
            if k != "band_rows":
                assert got[k] == v, (rows, k)


def test_sync_modes_bit_identical():
    """Latency mode (rows meet every position, chosen below two waves of CTAs: this 2-quad
    call) and throughput mode (every CPL positions) give the same bits, for two band heights."""
    for rows in (0, 16):
        a, b = _run(rows, fine=1), _run(rows, fine=0)
        for k, v in a.items():
            assert b[k] == v, (rows, k)
