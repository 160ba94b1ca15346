"""Multi-process host logic of the frame-sharded path (paper_1801_04720_b200/dist.py),
world_size 2 over gloo on CPU: shard assignment, max-over-ranks timing, packing and
the gather of per-rank results to rank 0 (BASELINE.json configs[4])."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

from paper_1801_04720_b200 import dist as sd


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _stamp(fidx, H, W):
    """A stand-in per-quad "result" (no GPU needed): the frame index stamped into every
    field of the payload."""
    return {"sf": torch.full((H, W, 4), float(fidx)), "dp": torch.full((H, W, 4), -float(fidx)),
            "valid_sf": torch.full((H, W), fidx % 2, dtype=torch.uint8),
            "valid_3d": torch.full((H, W), (fidx + 1) % 2, dtype=torch.uint8)}


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        total, H, W = 6, 2, 3
        idx = sd.split_even(total, world, rank)       # configs[4]-style strong split
        n = len(idx)
        per = [_stamp(f, H, W) for f in idx]
        out = {k: torch.stack([p[k] for p in per]) for k in sd.PACK_KEYS}
        t = sd.max_over_ranks(10.0 * (rank + 1))
        got = sd.gather_results(out, rank, world)
        # the in-place variant: results written straight into the packed buffer
        buf = torch.empty(sd.packed_bytes(n, H, W), dtype=torch.uint8)
        views = sd.unpack_results(buf, n, H, W)
        for k in sd.PACK_KEYS:
            views[k].copy_(out[k])
        recv = [torch.empty_like(buf) for _ in range(world)] if rank == 0 else None
        sd.gather_packed(buf, recv, rank, world)
        res = {"rank": rank, "idx": idx, "tmax": t}
        if rank == 0:
            frames = []
            for r in range(world):
                assert torch.equal(got[r], recv[r])
                u = sd.unpack_results(recv[r], n, H, W)
                for k in range(n):
                    fidx = int(u["sf"][k, 0, 0, 0].item())
                    ref = _stamp(fidx, H, W)
                    for key in sd.PACK_KEYS:
                        assert torch.equal(u[key][k], ref[key]), (r, k, key)
                    frames.append(fidx)
            res["frames"] = frames
        else:
            assert got is None
        dist.destroy_process_group()
        q.put(res)
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put({"rank": rank, "error": repr(e)})


def test_shard_math():
    assert sd.shard_indices(0, 2, 4) == [0, 1, 2, 3]
    assert sd.shard_indices(1, 2, 4) == [4, 5, 6, 7]
    allx = sum((sd.split_even(64, 8, r) for r in range(8)), [])
    assert allx == list(range(64))
    with pytest.raises(ValueError):
        sd.split_even(64, 3, 0)
    with pytest.raises(ValueError):
        sd.shard_indices(2, 2, 4)


def test_pack_roundtrip():
    n, H, W = 2, 3, 5
    out = {"sf": torch.randn(n, H, W, 4), "dp": torch.randn(n, H, W, 4),
           "valid_sf": torch.randint(0, 2, (n, H, W), dtype=torch.uint8),
           "valid_3d": torch.randint(0, 2, (n, H, W), dtype=torch.uint8)}
    buf = sd.pack_results(out)
    assert buf.numel() == sd.packed_bytes(n, H, W) == n * H * W * 34
    u = sd.unpack_results(buf, n, H, W)
    for k in sd.PACK_KEYS:
        assert torch.equal(u[k], out[k]), k
    with pytest.raises(ValueError):
        sd.unpack_results(buf[:-1], n, H, W)


def test_bench_refuses_world_mismatch():
    """bench.py exits non-zero when WORLD_SIZE disagrees with --gpus, or when the 64-quad
    batch does not split evenly, before touching any GPU."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "1"], env=env,
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 2 and "WORLD_SIZE" in r.stderr
    env = dict(os.environ, WORLD_SIZE="3", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "3"], env=env,
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 2 and "split" in r.stderr


def test_gloo_world2_gather_and_max():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    res = {r["rank"]: r for r in res}
    for r in res.values():
        assert "error" not in r, r
    assert res[0]["idx"] == [0, 1, 2] and res[1]["idx"] == [3, 4, 5]
    assert res[0]["tmax"] == 20.0 and res[1]["tmax"] == 20.0
    assert res[0]["frames"] == [0, 1, 2, 3, 4, 5]


def _pipe_worker(rank, world, port, q):
    """Three pipelined steps: the payload of step k is overwritten (as the next step's
    kernels would) right after submit(); rank 0 must still receive step k's bytes."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        n, H, W = 2, 2, 3
        packed = torch.empty(sd.packed_bytes(n, H, W), dtype=torch.uint8)
        pipe = sd.PipelinedGather(packed, rank, world)
        seen = []
        for step in range(3):
            packed.fill_(10 * step + rank + 1)           # "compute" step k
            pipe.submit(packed)
            packed.fill_(255)                            # step k+1 starts overwriting
            if step == 1:                                # a reader between steps
                pipe.drain()
                if rank == 0:
                    seen.append([int(b[0]) for b in pipe.recv] + [int(b[-1]) for b in pipe.recv])
        pipe.drain()
        assert pipe.work is None
        if rank == 0:
            seen.append([int(b[0]) for b in pipe.recv] + [int(b[-1]) for b in pipe.recv])
            for b in pipe.recv:
                assert bool((b == b[0]).all())
        dist.destroy_process_group()
        q.put({"rank": rank, "seen": seen})
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put({"rank": rank, "error": repr(e)})


def test_gloo_world2_pipelined_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pipe_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    res = {r["rank"]: r for r in res}
    for r in res.values():
        assert "error" not in r, r
    # after step 1: payloads 11 (rank 0) and 12 (rank 1); after step 2: 21 and 22
    assert res[0]["seen"] == [[11, 12, 11, 12], [21, 22, 21, 22]]


def test_pipelined_gather_single_rank():
    packed = torch.arange(34 * 6, dtype=torch.uint8)
    pipe = sd.PipelinedGather(packed, 0, 1)
    pipe.submit(packed)
    packed.zero_()
    pipe.drain()
    assert torch.equal(pipe.recv[0], torch.arange(34 * 6, dtype=torch.uint8))
