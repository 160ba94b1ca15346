"""Multi-GPU plumbing: one process per GPU (torchrun), frame quads sharded over
ranks, no collective on the data path.  Independent frame
quads need no exchange, so the only collectives are a max-over-ranks of timers
and an optional gather of results to rank 0 (BASELINE.json configs[4]).

torch.distributed (NCCL on GPUs, gloo on CPU tests) is plumbing only.
"""
from __future__ import annotations

import datetime
import os

import torch
import torch.distributed as dist


def init_distributed(world: int, rank: int):
    """Initialise the default process group when world > 1 (NCCL if CUDA, else gloo)."""
    if world <= 1:
        return None
    if dist.is_initialized():
        return dist.group.WORLD
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    os.environ.setdefault("TORCH_NCCL_ASYNC_ERROR_HANDLING", "1")
    backend = "nccl" if torch.cuda.is_available() else "gloo"
    kw = {}
    if backend == "nccl":
        kw["device_id"] = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    dist.init_process_group(backend, rank=rank, world_size=world,
                            timeout=datetime.timedelta(seconds=300), **kw)
    return dist.group.WORLD


def shard_indices(rank: int, world: int, per_rank: int, base: int = 0):
    """Contiguous equal blocks of frame indices: rank r owns [r*per_rank, (r+1)*per_rank)."""
    if per_rank < 1 or not (0 <= rank < world):
        raise ValueError("bad shard request")
    start = base + rank * per_rank
    return list(range(start, start + per_rank))


def split_even(total: int, world: int, rank: int):
    """Strong-scaling split of `total` frames (configs[4]: 64 over 1/2/4/8 GPUs)."""
    if total % world:
        raise ValueError(f"{total} frames do not split evenly over {world} ranks")
    n = total // world
    return list(range(rank * n, (rank + 1) * n))


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (timings are reported as the slowest rank)."""
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    dev = device if (device is not None and dist.get_backend() == "nccl") else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


PACK_KEYS = ("sf", "valid_sf")


def pack_results(out: dict) -> torch.Tensor:
    """Flatten the per-rank scene flow (S float32 [n][H][W][4] + mask) into one byte tensor."""
    parts = [out[k].contiguous().view(torch.uint8).reshape(-1) for k in PACK_KEYS]
    return torch.cat(parts)


def unpack_results(buf: torch.Tensor, n: int, H: int, W: int) -> dict:
    sf_bytes = n * H * W * 4 * 4
    sf = buf[:sf_bytes].view(torch.float32).reshape(n, H, W, 4)
    v = buf[sf_bytes:sf_bytes + n * H * W].reshape(n, H, W)
    return {"sf": sf, "valid_sf": v}


def gather_results(out: dict, rank: int, world: int, device=None):
    """Gather every rank's packed results to rank 0 (one NCCL/gloo gather).  Returns the
    list of per-rank byte tensors on rank 0, None elsewhere."""
    buf = pack_results(out)
    if world <= 1:
        return [buf]
    if dist.get_backend() == "nccl":
        buf = buf.to(device)
    if rank == 0:
        bufs = [torch.empty_like(buf) for _ in range(world)]
        dist.gather(buf, gather_list=bufs, dst=0)
        return bufs
    dist.gather(buf, dst=0)
    return None
