"""Host-side multi-rank plumbing for the data-parallel step (one process per GPU).

torch.distributed is used for process groups only: rendezvous, a symmetric-configuration
check before the collective context is created, and max-over-ranks timing.  The gradient
exchange itself never goes through torch.distributed: it is the ring kernel of libtem.so
 over NVLink peer memory.
"""
from __future__ import annotations

import hashlib
import json
import os
from dataclasses import asdict, is_dataclass

import torch
import torch.distributed as dist


def env_world():
    """(rank, world_size, local_rank) from the torchrun environment (defaults: single process)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init_from_env(backend: str = "nccl", device: torch.device | None = None):
    """Initialise the default process group from torchrun's env (MASTER_ADDR defaults to
    127.0.0.1: the container hostname may not resolve)."""
    rank, world, _ = env_world()
    if world <= 1 or dist.is_initialized():
        return rank, world
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    kw = {"device_id": device} if (backend == "nccl" and device is not None) else {}
    dist.init_process_group(backend, rank=rank, world_size=world, **kw)
    return rank, world


def config_digest(cfg) -> str:
    d = asdict(cfg) if is_dataclass(cfg) else dict(cfg)
    d = {k: (list(v) if isinstance(v, tuple) else v) for k, v in d.items() if k not in ("rank",)}
    return hashlib.sha256(json.dumps(d, sort_keys=True).encode()).hexdigest()


class ConfigMismatch(RuntimeError):
    pass


def check_symmetric(cfg, group=None):
    """Every rank must build the context with the same model / precision / lr / ring geometry
    ("all N workers call concurrently with equal K").  Raises on all ranks if not, before
    any kernel could wait on a peer that will never signal."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    mine = config_digest(cfg)
    allv = [None] * dist.get_world_size(group)
    dist.all_gather_object(allv, mine, group=group)
    if len(set(allv)) != 1:
        bad = [i for i, v in enumerate(allv) if v != allv[0]]
        raise ConfigMismatch(f"ranks {bad} disagree with rank 0 on the TEM configuration")


def max_over_ranks(value: float, group=None, device=None) -> float:
    """Max of a host scalar over ranks (bench timing: the slowest rank defines the step)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    dev = device if device is not None else (torch.device("cpu") if dist.get_backend(group) == "gloo"
                                           else torch.device("cuda", torch.cuda.current_device()))
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def shard_batch_indices(global_batch: int, world: int, rank: int):
    """P:113 data parallelism: rank r owns the contiguous videos [r*B, (r+1)*B) of the global
    batch (B = global_batch / world).  Raises if the batch does not split evenly."""
    if global_batch % world:
        raise ValueError("global batch must be a multiple of the world size")
    B = global_batch // world
    return range(rank * B, (rank + 1) * B)
