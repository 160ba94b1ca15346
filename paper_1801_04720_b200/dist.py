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
    # SGM_DIST_BACKEND=gloo: functional runs of the multi-rank code on one GPU (two NCCL
    # ranks cannot share a device); device payloads are then staged through the host
    backend = os.environ.get("SGM_DIST_BACKEND") or ("nccl" if torch.cuda.is_available() else "gloo")
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
    if buf.is_cuda and dist.get_backend() != "nccl":       # gloo: stage through the host
        host = buf.cpu()
        hrecv = [torch.empty_like(host) for _ in range(world)] if rank == 0 else None
        gather_packed(host, hrecv, rank, world)
        if rank == 0:
            for d, h in zip(recv, hrecv):
                d.copy_(h)
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
        if self.world > 1 and self.stage.is_cuda and dist.get_backend() != "nccl":
            gather_packed(self.stage, self.recv, self.rank, self.world)   # gloo: synchronous
        elif self.world > 1:
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


class DirectGather:
    """Zero-copy gather over peer memory: rank 0 owns `slots` buffers of world x nbytes; every
    other rank maps them through CUDA IPC (peer access: NVLink / NVSwitch on a multi-GPU box)
    and hands its slice to sgm_scene_flow as the output buffer, so the combination kernel's
    own stores carry the payload to rank 0 -- no collective, no staging copy.  Rank 0 may
    read slot s once `fence()` of the step that wrote it has returned on every rank (one
    tiny all-reduce ordered after the step on the current stream).

    Only torch plumbing is used (torch.multiprocessing's CUDA IPC handles, sent with
    broadcast_object_list); construction is collective and either succeeds on every rank or
    raises on every rank (`ok` is agreed with an all-reduce).
    """

    def __init__(self, nbytes: int, rank: int, world: int, device, slots: int = 2):
        from torch.multiprocessing.reductions import reduce_tensor
        self.rank, self.world, self.nbytes = rank, world, nbytes
        # slices start 256-byte aligned (the kernels store float4)
        self.stride = stride = (nbytes + 255) // 256 * 256
        self.device = torch.device(device)
        self.bufs, err = None, None
        obj = [None]
        try:
            if rank == 0:
                self.bufs = [torch.empty(world * stride, dtype=torch.uint8, device=self.device)
                             for _ in range(slots)]
                torch.cuda.synchronize(self.device)
                obj = [[reduce_tensor(b) for b in self.bufs]]
        except Exception as e:  # agreed below
            err = e
        if world > 1:
            dist.broadcast_object_list(obj, src=0)
            if rank != 0 and obj[0] is not None:
                try:
                    with torch.cuda.device(self.device):
                        self.bufs = [fn(*args) for fn, args in obj[0]]
                except Exception as e:
                    err, self.bufs = e, None
        nccl = world > 1 and dist.get_backend() == "nccl"
        self._flag = torch.ones(1, dtype=torch.int32, device=self.device if nccl else "cpu")
        ok = torch.tensor([0 if (err is not None or self.bufs is None) else 1], dtype=torch.int32,
                          device=self._flag.device)
        if world > 1:
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()) == 0:
            self.bufs = None
            raise RuntimeError(f"peer-memory gather unavailable: {err!r}")

    def mine(self, slot: int) -> torch.Tensor:
        """This rank's slice of slot `slot` (memory of rank 0's device)."""
        b = self.bufs[slot]
        return b[self.rank * self.stride:self.rank * self.stride + self.nbytes]

    def gathered(self, slot: int):
        """Rank 0: the list of per-rank payloads of slot `slot` (views, no copy)."""
        if self.rank != 0:
            return None
        b = self.bufs[slot]
        return [b[r * self.stride:r * self.stride + self.nbytes] for r in range(self.world)]

    def fence(self):
        """Orders 'every rank's step has completed' after the work already enqueued on the
        current stream (NCCL) or after a device synchronize (gloo, CPU tests)."""
        if self.world <= 1:
            return
        if dist.get_backend() != "nccl":
            torch.cuda.synchronize(self.device)
        dist.all_reduce(self._flag, op=dist.ReduceOp.MAX)

    def close(self):
        self.bufs = None
