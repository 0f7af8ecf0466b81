"""One process per GPU over torch.distributed (NCCL on the B200 box, gloo in
the CPU tests).  The restoration path partitions into independent signals /
images, so ranks shard items with no data-path
collective; the only collectives are the barrier around the timed region,
the max-over-ranks of the step time, and optional result gathers."""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env_world():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def init(backend=None):
    rank, world, local = env_world()
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group(backend, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return rank, world, local


def shard(total: int, rank: int, world: int):
    """Contiguous balanced split of [0, total): (start, count)."""
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def barrier():
    if dist.is_initialized():
        dist.barrier()


def _dev():
    return torch.device("cuda") if torch.cuda.is_available() and \
        dist.is_initialized() and dist.get_backend() == "nccl" else torch.device("cpu")


def max_over_ranks(x: float) -> float:
    if not dist.is_initialized():
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=_dev())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float) -> float:
    if not dist.is_initialized():
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=_dev())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def gather_items(local: torch.Tensor, total: int) -> torch.Tensor | None:
    """Reassemble per-rank shards (leading axis = items, contiguous shard()
    order) on rank 0; other ranks get None."""
    if not dist.is_initialized():
        return local
    rank, world = dist.get_rank(), dist.get_world_size()
    counts = [shard(total, r, world)[1] for r in range(world)]
    dev = _dev()
    buf = local.to(dev).contiguous()
    if rank == 0:
        parts = [torch.empty((c,) + tuple(local.shape[1:]), dtype=local.dtype, device=dev)
                 for c in counts]
        parts[0].copy_(buf)
        for r in range(1, world):
            dist.recv(parts[r], src=r)
        return torch.cat(parts, 0)
    dist.send(buf, dst=0)
    return None


def finalize():
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()
