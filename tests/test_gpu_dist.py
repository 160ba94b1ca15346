"""The frame-sharded multi-rank path of configs[4] end to end on one GPU:
two ranks (processes) each run their contiguous share of the quads through the C ABI,
write the payload (S, dP, both masks) into their packed buffer, and gather it to rank 0
(gloo over host copies here -- one GPU cannot host two NCCL ranks; bench.py uses the same
pack / gather code with NCCL).  Rank 0 checks the gathered bytes against a single-process
launch of the whole batch (byte-identical) and every quad against the oracle.  The ranks'
kernels never wait on each other."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import synth

pytestmark = pytest.mark.gpu

TOTAL = 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        import torch.distributed as dist
        from paper_1801_04720_b200 import SGM, Camera, stack_quads
        from paper_1801_04720_b200 import dist as sd
        dist.init_process_group("gloo", rank=rank, world_size=world)
        cfg = synth.CONFIGS["batch"]
        prm = synth.sgm_params(cfg)
        idx = sd.split_even(TOTAL, world, rank)
        quads = synth.make_batch(cfg, idx[0], len(idx))
        dev = torch.device("cuda", 0)
        g = SGM.from_config(cfg, max_batch=len(idx))
        imgs, flow = stack_quads(quads, g.pitch, dev)
        buf, out = sd.alloc_packed_outputs(g, len(idx))
        g.scene_flow(imgs, flow, Camera(prm["f"], prm["B"], prm["cx"], prm["cy"]), out)
        torch.cuda.synchronize()
        host = buf.cpu()
        recv = [torch.empty_like(host) for _ in range(world)] if rank == 0 else None
        sd.gather_packed(host, recv, rank, world)
        if rank == 0:
            torch.save(torch.cat(recv), q["path"])
        g.close()
        dist.destroy_process_group()
        q["res"].put({"rank": rank, "idx": idx})
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q["res"].put({"rank": rank, "error": repr(e)})


def test_two_ranks_gather_equals_single_launch_and_oracle(orc, tmp_path):
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    ctx = mp.get_context("spawn")
    q = {"res": ctx.Queue(), "path": str(tmp_path / "gathered.pt")}
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q["res"].get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    for r in res:
        assert "error" not in r, r
    gathered = torch.load(q["path"])

    from paper_1801_04720_b200 import SGM, Camera, stack_quads
    from paper_1801_04720_b200 import dist as sd
    cfg = synth.CONFIGS["batch"]
    prm = synth.sgm_params(cfg)
    quads = synth.make_batch(cfg, 0, TOTAL, workers=TOTAL)
    dev = torch.device("cuda", 0)
    g = SGM.from_config(cfg, max_batch=TOTAL)
    imgs, flow = stack_quads(quads, g.pitch, dev)
    buf, out = sd.alloc_packed_outputs(g, TOTAL)
    full = g.scene_flow(imgs, flow, Camera(prm["f"], prm["B"], prm["cx"], prm["cy"]),
                        dict(out, p0=torch.empty_like(out["sf"])))
    torch.cuda.synchronize()
    # per rank, the packed layout is [rank's quads][...] per field: unpack rank by rank
    per = TOTAL // 2
    n_bytes = sd.packed_bytes(per, cfg.H, cfg.W)
    for r in range(2):
        u = sd.unpack_results(gathered[r * n_bytes:(r + 1) * n_bytes], per, cfg.H, cfg.W)
        for k in sd.PACK_KEYS:
            assert torch.equal(u[k], full[k][r * per:(r + 1) * per].cpu()), (r, k)
    from test_gpu_parity import _check_sceneflow, oracle_many
    for i, o in enumerate(oracle_many(orc, quads, prm)):
        r = {k: full[k][i] for k in ("sf", "valid_sf", "p0", "dp", "valid_3d")}
        _check_sceneflow(r, o["sf"], o["valid_sf"], o["p0"], o["p1"], o["dp"], o["valid_3d"])
    g.close()
