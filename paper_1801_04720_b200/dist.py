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


# Per-rank result payload gathered to rank 0: S = (u, v, d0, d1) f32x4,
# dP = (dX, dY, dZ, 0) f32x4 and the two masks -- 34 bytes per pixel, in this order.
PACK_KEYS = ("sf", "dp", "valid_sf", "valid_3d")
_PACK_FMT = {"sf": (torch.float32, 4), "dp": (torch.float32, 4), "valid_sf": (torch.uint8, 1),
             "valid_3d": (torch.uint8, 1)}


def packed_bytes(n: int, H: int, W: int) -> int:
    return n * H * W * sum(torch.empty((), dtype=dt).element_size() * c for dt, c in _PACK_FMT.values())


def _views(buf: torch.Tensor, n: int, H: int, W: int) -> dict:
    out, off = {}, 0
    for k in PACK_KEYS:
        dt, c = _PACK_FMT[k]
        nbytes = n * H * W * c * torch.empty((), dtype=dt).element_size()
        v = buf[off:off + nbytes].view(dt)
        out[k] = v.reshape(n, H, W, c) if c > 1 else v.reshape(n, H, W)
        off += nbytes
    return out


def alloc_packed_outputs(sgm, n: int):
    """One uint8 buffer per rank holding the gathered outputs, and the output dict of
    sgm.scene_flow as views into it (S and dP 16-byte aligned), so the kernels write the
    payload in place and the gather needs no packing copy."""
    buf = torch.empty(packed_bytes(n, sgm.H, sgm.W), dtype=torch.uint8, device=sgm.device)
    return buf, _views(buf, n, sgm.H, sgm.W)


def pack_results(out: dict) -> torch.Tensor:
    """Flatten a rank's results (PACK_KEYS order) into one byte tensor."""
    parts = [out[k].contiguous().view(torch.uint8).reshape(-1) for k in PACK_KEYS]
    return torch.cat(parts)


def unpack_results(buf: torch.Tensor, n: int, H: int, W: int) -> dict:
    if buf.numel() != packed_bytes(n, H, W):
        raise ValueError("packed buffer size does not match n x H x W")
    return _views(buf, n, H, W)


def gather_packed(buf: torch.Tensor, recv, rank: int, world: int):
    """Gather every rank's packed buffer into rank 0's preallocated `recv` list (one
    collective; NCCL with device tensors, gloo with host tensors)."""
    if world <= 1:
        return
    if rank == 0:
        dist.gather(buf, gather_list=recv, dst=0)
    else:
        dist.gather(buf, dst=0)


def gather_results(out: dict, rank: int, world: int, device=None):
    """Gather every rank's packed results to rank 0 (one NCCL/gloo gather).  Returns the
    list of per-rank byte tensors on rank 0, None elsewhere."""
    buf = pack_results(out)
    if world <= 1:
        return [buf]
    if dist.get_backend() == "nccl":
        buf = buf.to(device)
    recv = [torch.empty_like(buf) for _ in range(world)] if rank == 0 else None
    gather_packed(buf, recv, rank, world)
    return recv


class PipelinedGather:
    """Gather of step k's packed results to rank 0, overlapped with step k+1's kernels.

    submit(packed) copies the step's payload into a staging buffer on the current stream
    and starts an asynchronous gather of it (NCCL runs it on its own stream, ordered after
    the copy); the next step's kernels, which overwrite `packed`, are then free to run while
    the payload travels.  The previous gather is awaited before the staging buffer is
    reused, so at most one collective is in flight.  drain() waits for the last one; after
    it rank 0's `recv[r]` holds rank r's payload of the most recent submit().
    """

    def __init__(self, packed: torch.Tensor, rank: int, world: int):
        self.rank, self.world = rank, world
        self.stage = torch.empty_like(packed)
        self.recv = [torch.empty_like(packed) for _ in range(world)] if rank == 0 else None
        self.work = None

    def submit(self, packed: torch.Tensor):
        self.drain()
        self.stage.copy_(packed, non_blocking=True)
        if self.world > 1:
            if self.rank == 0:
                self.work = dist.gather(self.stage, gather_list=self.recv, dst=0, async_op=True)
            else:
                self.work = dist.gather(self.stage, dst=0, async_op=True)
        elif self.recv is not None:
            self.recv[0].copy_(self.stage, non_blocking=True)

    def drain(self):
        if self.work is not None:
            self.work.wait()
            self.work = None
