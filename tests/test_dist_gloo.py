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


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        per = 3
        idx = sd.shard_indices(rank, world, per)
        # a stand-in "result" per rank: frame indices stamped into S (no GPU needed)
        n, H, W = per, 2, 3
        sf = torch.zeros((n, H, W, 4), dtype=torch.float32)
        for k, fidx in enumerate(idx):
            sf[k] = float(fidx)
        out = {"sf": sf, "valid_sf": torch.full((n, H, W), rank + 1, dtype=torch.uint8)}
        t = sd.max_over_ranks(10.0 * (rank + 1))
        got = sd.gather_results(out, rank, world)
        res = {"rank": rank, "idx": idx, "tmax": t}
        if rank == 0:
            frames = []
            for r, buf in enumerate(got):
                u = sd.unpack_results(buf, n, H, W)
                frames += [int(u["sf"][k, 0, 0, 0].item()) for k in range(n)]
                assert int(u["valid_sf"][0, 0, 0]) == r + 1
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
    sf = torch.randn(n, H, W, 4)
    v = torch.randint(0, 2, (n, H, W), dtype=torch.uint8)
    u = sd.unpack_results(sd.pack_results({"sf": sf, "valid_sf": v}), n, H, W)
    assert torch.equal(u["sf"], sf) and torch.equal(u["valid_sf"], v)


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
