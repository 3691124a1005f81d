"""Multi-GPU plumbing for the server path.

Images are independent, so the work shards by batch with no data-path
collective: rank r serves images [lo, hi) of the global batch.  The only
exchange is optional: assembling every rank's compact payload (the valid
slots that go back to the client) on all ranks with one
all_gather over NVLink (NCCL) — or over gloo in the CPU tests.  Host logic
only; the per-rank compute is the library's kernels.
"""
from __future__ import annotations

from typing import Tuple

import torch
import torch.distributed as dist


def shard_range(total: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous, balanced split of `total` images over `world` ranks
    (the first total % world ranks get one extra image)."""
    if world < 1 or not 0 <= rank < world or total < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def gather_payload(local: torch.Tensor, total: int, group=None) -> torch.Tensor:
    """All-gather per-rank payloads [B_r, ...] (B_r from shard_range) into
    the global [total, ...] tensor in image order, on every rank."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi = shard_range(total, rank, world)
    assert local.shape[0] == hi - lo
    counts = [shard_range(total, r, world) for r in range(world)]
    width = max(h - l for l, h in counts)
    pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype,
                      device=local.device)
    pad[: hi - lo] = local
    out = torch.empty((world * width,) + tuple(local.shape[1:]),
                      dtype=local.dtype, device=local.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, pad, group=group)
    else:
        dist.all_gather(list(out.chunk(world)), pad, group=group)
    parts = [out[r * width: r * width + (h - l)] for r, (l, h) in enumerate(counts)]
    return torch.cat(parts, 0)
