"""Multi-GPU sharding along the natural shards of the DPM hot path.

* Batched AP solves (cfg4, and every BEP build): the RHS are independent units, sharded
  in contiguous blocks of ceil(B/p); no data-path collective.
* BEP build across ranks (C1): each rank computes a contiguous block of BEP columns
  (dpm_bep_columns), one all-gather assembles B (|γ_in| x K) on every rank, and every
  rank factors it redundantly (a K x K Cholesky is cheap; this avoids a broadcast).

The collective calls go through torch.distributed (NCCL on GPUs; gloo in the CPU tests).
The column computation is a callable so the host logic is testable without a GPU.
"""
from typing import Callable, Tuple

import torch
import torch.distributed as dist


def shard_range(total: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous block [b0, b1) of ceil(total/world) units for this rank (may be empty)."""
    per = -(-total // world) if world > 0 else total
    b0 = min(total, rank * per)
    return b0, min(total, b0 + per)


def allgather_columns(block: torch.Tensor, total_cols: int, world: int, rank: int) -> torch.Tensor:
    """All-gather row-blocks [ncols_r, m] (row r = BEP column) into [total_cols, m] on every rank.

    Blocks are padded to the common size ceil(K/p) so a single all_gather suffices."""
    per = -(-total_cols // world)
    m = block.shape[1]
    pad = torch.zeros((per, m), dtype=block.dtype, device=block.device)
    pad[: block.shape[0]] = block
    out = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(out, pad)
    full = torch.cat(out, dim=0)
    keep = []
    for r in range(world):
        c0, c1 = shard_range(total_cols, world, r)
        keep.append(full[r * per: r * per + (c1 - c0)])
    return torch.cat(keep, dim=0)


def distributed_bep(columns: Callable[[int, int], torch.Tensor], K: int, world: int, rank: int) -> torch.Tensor:
    """Assemble the full reduced-BEP matrix B ([K, |γ_in|], row c = column c) on every rank.

    `columns(c0, c1)` returns this rank's block [c1-c0, |γ_in|] (on GPUs: DPM.bep_columns)."""
    c0, c1 = shard_range(K, world, rank)
    blk = columns(c0, c1)
    if world == 1:
        return blk
    return allgather_columns(blk, K, world, rank)


def build_projection_distributed(ctx, world: int, rank: int):
    """GPU path: shard the K AP solves of a BEP build over ranks, all-gather B, factor locally."""
    B = distributed_bep(lambda a, b: ctx.bep_columns(a, b)[1], ctx.K, world, rank)
    ctx.bep_factor(B.contiguous())
    return B
