"""Row sharding of PQ layers across GPUs (north_star "splitting
output rows ... with an NCCL all-gather").

Rank r of N holds output rows [r*F_out/N, (r+1)*F_out/N) of every layer and
ALL codebooks (with input-axis subspaces every row uses every codebook).
After a sharded GEMV/GEMM each rank owns a contiguous column slice of y; the
slices are concatenated with one all-gather so every rank has the full
activation for the next layer.  Pure plumbing (torch.distributed); the
compute stays in libfasq.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def row_range(F_out: int, rank: int, world: int):
    """[r0, r1) output rows of `rank` (F_out must divide evenly)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if F_out % world:
        raise ValueError("F_out=%d not divisible by world=%d" % (F_out, world))
    rows = F_out // world
    return rank * rows, (rank + 1) * rows


def shard_indices(indices: torch.Tensor, rank: int, world: int) -> torch.Tensor:
    """Slice a logical index table [N_ss][F_out] to this rank's rows."""
    r0, r1 = row_range(indices.shape[1], rank, world)
    return indices[:, r0:r1].contiguous()


def gather_rows(local: torch.Tensor, full: torch.Tensor | None = None, group=None) -> torch.Tensor:
    """All-gather per-rank output slices y_r [B][F_out/N] into y [B][F_out]
    (rank-major column order).  NCCL: one all_gather_into_tensor on a
    rank-major staging buffer; gloo (CPU tests): list all_gather."""
    world = dist.get_world_size(group)
    B, rows = local.shape
    if full is None:
        full = torch.empty((B, rows * world), dtype=local.dtype, device=local.device)
    if world == 1:
        full.copy_(local)
        return full
    if B == 1:
        # [1][F_out] is already rank-major contiguous: gather straight into it
        if dist.get_backend(group) == "nccl":
            dist.all_gather_into_tensor(full.view(-1), local.reshape(-1), group=group)
        else:
            parts = list(full.view(world, rows).unbind(0))
            dist.all_gather(parts, local.reshape(-1).contiguous(), group=group)
            full.view(world, rows).copy_(torch.stack(parts))
        return full
    stage = torch.empty((world, B, rows), dtype=local.dtype, device=local.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(stage.view(-1), local.contiguous().view(-1), group=group)
    else:
        parts = [torch.empty_like(local) for _ in range(world)]
        dist.all_gather(parts, local.contiguous(), group=group)
        stage.copy_(torch.stack(parts))
    full.copy_(stage.permute(1, 0, 2).reshape(B, rows * world))
    return full
