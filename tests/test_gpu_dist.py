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


def _rank_direct(rank, world, port, q):
    """The peer-memory gather: rank 1's kernels write straight into rank 0's buffer (CUDA IPC;
    both processes share cuda:0 here, on a multi-GPU box the mapping is peer access)."""
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
        nbytes = sd.packed_bytes(len(idx), cfg.H, cfg.W)
        dg = sd.DirectGather(nbytes, rank, world, dev, slots=2)
        cam = Camera(prm["f"], prm["B"], prm["cx"], prm["cy"])
        for step in range(3):                              # slots 0, 1, 0
            slot = step & 1
            out = sd.unpack_results(dg.mine(slot), len(idx), cfg.H, cfg.W)
            g.scene_flow(imgs, flow, cam, out)
            dg.fence()
        if rank == 0:
            torch.save(torch.cat([b.clone() for b in dg.gathered(0)]).cpu(), q["path"])
            same = all(torch.equal(a, b) for a, b in zip(dg.gathered(0), dg.gathered(1)))
            q["res"].put({"rank": rank, "idx": idx, "slots_equal": same})
        dist.barrier()                                     # rank 0 has read: peers may unmap
        dg.close()
        g.close()
        if rank != 0:
            q["res"].put({"rank": rank, "idx": idx})
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q["res"].put({"rank": rank, "error": repr(e)})


def test_two_ranks_peer_memory_gather_equals_single_launch(tmp_path):
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    ctx = mp.get_context("spawn")
    q = {"res": ctx.Queue(), "path": str(tmp_path / "direct.pt")}
    port = _free_port()
    procs = [ctx.Process(target=_rank_direct, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q["res"].get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    for r in res:
        assert "error" not in r, r
    assert any(r.get("slots_equal") for r in res)
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
    full = g.scene_flow(imgs, flow, Camera(prm["f"], prm["B"], prm["cx"], prm["cy"]), out)
    torch.cuda.synchronize()
    per = TOTAL // 2
    n_bytes = sd.packed_bytes(per, cfg.H, cfg.W)
    for r in range(2):
        u = sd.unpack_results(gathered[r * n_bytes:(r + 1) * n_bytes], per, cfg.H, cfg.W)
        for k in sd.PACK_KEYS:
            assert torch.equal(u[k], full[k][r * per:(r + 1) * per].cpu()), (r, k)
    g.close()


def test_bench_two_ranks_functional():
    """bench.py's N = 2 code path end to end (self-spawned ranks, strong split, serial /
    pipelined / peer-memory gather inside the timed step) as a functional run: both ranks
    share cuda:0 and talk over gloo, so the numbers mean nothing -- the line's structure and
    the agreement of the ranks are what is checked."""
    import json
    import subprocess
    import sys
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SGM_DIST_BACKEND="gloo", SGM_BENCH_SHARE_GPU="1")
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--quads", "4",
                        "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--no-configs", "--no-eval",
                        "--no-stream", "--no-flow", "--no-densify", "--no-e2e"], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["global_batch"] == 4 and line["config"]["quads_per_gpu"] == 2
    g = line["gather"]
    assert g["bytes_to_rank0_per_step"] == 2 * 375 * 1242 * 34
    assert g["serial"]["ms_per_step"] > 0 and g["ms_per_step"] > 0
    assert "value" in g["direct"], g["direct"]
    assert g["headline"] in ("direct", "pipelined")
    best = g["direct"] if g["headline"] == "direct" else g
    assert line["value"] == best["value"] and line["ms_per_step"] == best["ms_per_step"]
    assert line["compute_only"]["ms_per_step"] > 0
    assert line["gpu_launches"] == 4 * 2      # census, 2 sweeps, combination with the LR check fused
