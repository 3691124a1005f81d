"""Multi-GPU plumbing for the server path (north_star: "split
by output-channel ciphertext block and batch").

The path shards with no data-path collective: images are independent, and
given NTT(c0) so are the output-channel blocks of a Conv layer (Alg. 1 runs
one product per output block).  Two axes:

* batch (`shard_range`): rank r serves images [lo, hi) of the global batch,
  with a full replica of the filter spectra.  Weak scaling keeps the
  per-rank batch fixed; strong scaling splits one global batch.
* output block (`shard_out_blocks`, `sub_layer_weights`): when the batch is
  smaller than the world (config 2: one image, n_ob = 4), rank r evaluates
  output blocks [ob_lo, ob_hi) as a sub-layer of whole blocks -- the rows of
  W for channels ob_lo*c_ob .. ob_hi*c_ob, zero-padded to whole blocks.
  Its plan has the same s, c_ib, c_ob and t_n (channel n' of the sub-layer
  is n = n' + ob_lo*c_ob, and t_n depends on n mod c_ob), so its payload
  equals blocks [ob_lo, ob_hi) of the full layer's payload bit for bit, the
  padded channels included (product 0 + enc(phi1), as the full layer
  writes for channels past c_o).

The one exchange is optional: assembling every rank's compact payload (the
valid slots that go back to the client) on all ranks with one
all_gather (NCCL over NVLink, gloo in the CPU tests).  Host logic only; the
per-rank compute is the library's kernels.
"""
from __future__ import annotations

from typing import Tuple

import numpy as np
import torch
import torch.distributed as dist


def shard_range(total: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous, balanced split of `total` items over `world` ranks
    (the first total % world ranks get one extra item)."""
    if world < 1 or not 0 <= rank < world or total < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def choose_axis(batch: int, n_ob: int, world: int) -> str:
    """'batch' when every rank can get at least one image, else 'out_block'
    when the layer has at least as many output blocks as ranks, else
    'batch' (some ranks idle)."""
    if world <= batch or n_ob < world:
        return "batch"
    return "out_block"


def shard_out_blocks(n_ob: int, rank: int, world: int) -> Tuple[int, int]:
    """Output blocks [ob_lo, ob_hi) served by `rank` (balanced, contiguous)."""
    return shard_range(n_ob, rank, world)


def sub_layer_weights(W: np.ndarray, c_ob: int, ob_lo: int, ob_hi: int) -> np.ndarray:
    """Rows of W [c_o][c_i][f_w][f_h] for output blocks [ob_lo, ob_hi),
    zero-padded to (ob_hi - ob_lo) whole blocks of c_ob channels."""
    W = np.asarray(W)
    c_o = W.shape[0]
    k = ob_hi - ob_lo
    out = np.zeros((k * c_ob,) + W.shape[1:], dtype=W.dtype)
    lo, hi = ob_lo * c_ob, min(c_o, ob_hi * c_ob)
    if hi > lo:
        out[: hi - lo] = W[lo:hi]
    return out


def _gather_axis(local: torch.Tensor, total: int, axis: int, group=None) -> torch.Tensor:
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi = shard_range(total, rank, world)
    assert local.shape[axis] == hi - lo
    counts = [shard_range(total, r, world) for r in range(world)]
    width = max(h - l for l, h in counts)
    x = local.movedim(axis, 0)
    pad = torch.zeros((width,) + tuple(x.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: hi - lo] = x
    out = torch.empty((world * width,) + tuple(x.shape[1:]), dtype=local.dtype,
                      device=local.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, pad, group=group)
    else:
        dist.all_gather(list(out.chunk(world)), pad, group=group)
    parts = [out[r * width: r * width + (h - l)] for r, (l, h) in enumerate(counts)]
    return torch.cat(parts, 0).movedim(0, axis).contiguous()


def gather_payload(local: torch.Tensor, total: int, group=None) -> torch.Tensor:
    """All-gather per-rank payloads [B_r, ...] (B_r from shard_range) into
    the global [total, ...] tensor in image order, on every rank."""
    return _gather_axis(local, total, 0, group)


def gather_blocks(local: torch.Tensor, n_ob: int, group=None) -> torch.Tensor:
    """All-gather per-rank payloads [B][k_r][L][n_valid] (k_r output blocks
    from shard_out_blocks) into [B][n_ob][L][n_valid] in block order."""
    return _gather_axis(local, n_ob, 1, group)
