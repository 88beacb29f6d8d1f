"""Multi-GPU partitioning of the BWTA hot path (one process per GPU).

The paper is single-GPU.  The north star partitions

  * a BWTA linear along N (weight rows / output channels): rank r owns the
    packed weight rows [n0_r, n1_r) and their per-channel scales, computes
    Y_r^T = (s_W s_A dot)^T  [n_r x M] with bwta_gemm(y_transposed=True),
    and an all-gather of the Y_r^T blocks (NCCL over NVLink) yields Y^T
    [N x M] with no permute pass (rank-major concatenation = row-major Y^T);
  * attention along batch x heads: every (b, h) entry is independent, rank r
    owns a contiguous range of entries and the context blocks are gathered
    head-major.

Shards have equal padded size so a single all_gather_into_tensor suffices;
the pad rows are computed on zero weights and dropped.  Every per-element
result is identical to the single-GPU result (sharding N changes no
arithmetic), which tests/test_dist.py checks with world_size 2 over gloo.

Host-side logic only: the local compute is the library's (bwta_gemm /
bwta_attn_*), injectable for the CPU tests.
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple

import torch
import torch.distributed as dist


def shard_bounds(n: int, world: int, rank: int, align: int = 16) -> Tuple[int, int]:
    """Contiguous [start, stop) of rank's shard of n rows.

    Shards have size ceil(n / world) rounded up to `align` (so TMA boxes and
    all-gather blocks stay aligned); trailing ranks may get fewer or zero rows."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    per = -(-n // world)
    per = -(-per // align) * align if n >= align * world else per
    start = min(n, rank * per)
    stop = min(n, start + per)
    return start, stop


def padded_shard(n: int, world: int, align: int = 16) -> int:
    """Row count every rank contributes to the all-gather (max shard size)."""
    return max(shard_bounds(n, world, r, align)[1] - shard_bounds(n, world, r, align)[0] for r in range(world))


def shard_rows(t: Optional[torch.Tensor], n: int, world: int, rank: int, align: int = 16):
    """The rows of t ([n, ...]) owned by rank (a view), or None."""
    if t is None:
        return None
    s, e = shard_bounds(n, world, rank, align)
    return t[s:e]


def gather_rows(local: torch.Tensor, n: int, world: int, group=None, align: int = 16) -> torch.Tensor:
    """All-gather rank-major row blocks [n_r, ...] -> [n, ...].

    Each rank's block is padded to padded_shard() rows; one collective."""
    if world == 1 and local.shape[0] == n:
        return local  # nothing to gather
    per = padded_shard(n, world, align)
    if local.shape[0] > per:
        raise ValueError("local block larger than the padded shard")
    send = local
    if local.shape[0] != per:
        send = torch.zeros((per,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        send[: local.shape[0]] = local
    out = torch.empty((world * per,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    if world == 1:
        out.copy_(send)
    else:
        dist.all_gather_into_tensor(out, send.contiguous(), group=group)
    # rank r's rows live at [r * per, r * per + n_r); keep them in rank order
    pieces = []
    for r in range(world):
        s, e = shard_bounds(n, world, r, align)
        pieces.append(out[r * per: r * per + (e - s)])
    return torch.cat(pieces, 0) if world > 1 else out[:n]


def gemm_nshard(a, w_local, w_scale_local: Optional[torch.Tensor], a_scale: float, n_total: int,
                world: int, rank: int, group=None, out_dtype=torch.float16,
                local_gemm: Optional[Callable] = None, align: int = 16) -> torch.Tensor:
    """Y^T [N x M] of a BWTA linear whose weight rows are sharded across ranks.

    a: packed activations (replicated on every rank); w_local: this rank's packed
    weight rows (shard_bounds); returns the gathered Y^T on every rank."""
    if local_gemm is None:
        from . import bwta_gemm

        def local_gemm(a_, w_, s_, sa_, out_):
            return bwta_gemm(a_, w_, s_, sa_, out_dtype=out_.dtype, y_transposed=True, out=out_)
    s, e = shard_bounds(n_total, world, rank, align)
    m = a.ref.shape[-2]
    local = torch.empty((e - s, m), dtype=out_dtype, device=a.ref.device)
    if e > s:
        local_gemm(a, w_local, w_scale_local, a_scale, local)
    return gather_rows(local, n_total, world, group, align)


def heads_shard(bh: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous (batch x head) entries owned by rank for sharded attention."""
    return shard_bounds(bh, world, rank, align=1)


def gather_heads(local: torch.Tensor, bh: int, world: int, group=None) -> torch.Tensor:
    """All-gather per-rank [bh_r, T, D] context blocks -> [bh, T, D] (head-major)."""
    return gather_rows(local, bh, world, group, align=1)
