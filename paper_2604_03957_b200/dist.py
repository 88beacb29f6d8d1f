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
    # rank r's rows live at [r * per, r * per + n_r) and n_r = per for every rank but the
    # trailing ones (shard_bounds), so the rank-major prefix out[:n] IS the gathered matrix:
    # no re-copy
    return out[:n]


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


# ----------------------------------------------------------------------------
# Chunked N partition with the all-gather overlapped with the GEMM.
#
# The N rows (output channels) are cut into world x chunks blocks of nrc rows;
# block (c, r) -- global rows [(c * world + r) * nrc, +nrc) -- belongs to rank r.
# Chunk c of every rank together is the contiguous row range
# [c * world * nrc, (c + 1) * world * nrc) of Y^T, so each chunk's all-gather
# writes its final place in Y^T directly (in place: rank r's GEMM writes its
# block inside the gather buffer), and chunk c's gather runs on NCCL's stream
# while chunk c + 1's GEMM runs.  The owner of an output channel changes, not
# its arithmetic: the result equals the single-GPU Y^T bit for bit.
# ----------------------------------------------------------------------------
class NShardPlan:
    def __init__(self, n: int, world: int, rank: int, chunks: int = 1):
        if world < 1 or not (0 <= rank < world) or chunks < 1 or n < 0:
            raise ValueError("bad n/world/rank/chunks")
        self.n, self.world, self.rank, self.chunks = n, world, rank, chunks
        self.nrc = -(-n // (world * chunks)) if n else 0
        self.n_pad = self.nrc * world * chunks

    def block(self, c: int, r: Optional[int] = None) -> Tuple[int, int]:
        """Global rows [start, stop) of chunk c on rank r (clipped to n; may be empty)."""
        r = self.rank if r is None else r
        s = (c * self.world + r) * self.nrc
        return min(s, self.n), min(s + self.nrc, self.n)

    def local_rows(self) -> torch.Tensor:
        """Global row indices this rank owns, chunk-major (the rows of its local weight shard)."""
        idx = [torch.arange(*self.block(c)) for c in range(self.chunks)]
        return torch.cat(idx) if idx else torch.zeros(0, dtype=torch.int64)

    def local_span(self, c: int) -> Tuple[int, int]:
        """[start, stop) of chunk c inside the local shard (local_rows order)."""
        s = sum(self.block(i)[1] - self.block(i)[0] for i in range(c))
        b0, b1 = self.block(c)
        return s, s + (b1 - b0)


def gemm_nshard_overlap(a, w_local, w_scale_local: Optional[torch.Tensor], a_scale: float, plan: NShardPlan,
                        out: Optional[torch.Tensor] = None, group=None, out_dtype=torch.float16,
                        local_gemm: Optional[Callable] = None) -> torch.Tensor:
    """Y^T [N x M] of a BWTA linear N-sharded by `plan`, gathered on every rank.

    a: packed activations (replicated); w_local / w_scale_local: this rank's weight rows and
    scales in plan.local_rows() order; out: optional [plan.n_pad x M] buffer.  Chunk c's GEMM
    writes Y^T rows of block (c, rank) straight into `out`; its all-gather (async, NCCL stream)
    overlaps chunk c + 1's GEMM.  Returns out[:N] (a view)."""
    if local_gemm is None:
        from . import bwta_gemm

        def local_gemm(a_, w_, s_, sa_, out_):
            return bwta_gemm(a_, w_, s_, sa_, out_dtype=out_.dtype, y_transposed=True, out=out_)
    m = a.ref.shape[-2]
    if out is None:
        out = torch.empty((plan.n_pad, m), dtype=out_dtype, device=a.ref.device)
    if out.shape[0] < plan.n_pad or out.shape[1] != m or not out.is_contiguous():
        raise ValueError("out must be a contiguous [n_pad, M] buffer")
    works = []
    P, nrc = plan.world, plan.nrc
    for c in range(plan.chunks):
        g0, g1 = plan.block(c)
        l0, l1 = plan.local_span(c)
        if g1 > g0:
            w_c = _slice_packed(w_local, l0, l1) if hasattr(w_local, "sgn") else w_local[l0:l1]
            s_c = None if w_scale_local is None else w_scale_local[l0:l1]
            local_gemm(a, w_c, s_c, a_scale, out[g0:g1])
        if P > 1 or group is not None:   # (an explicit 1-rank group still runs the collective)
            blk = out[c * P * nrc:(c + 1) * P * nrc]
            mine = blk[plan.rank * nrc:(plan.rank + 1) * nrc]
            works.append(dist.all_gather_into_tensor(blk, mine, group=group, async_op=True))
    for w in works:
        w.wait()
    return out[:plan.n]


def _slice_packed(p, l0: int, l1: int):
    """Rows [l0, l1) of a Packed weight (a view of its planes)."""
    return type(p)(p.sgn[l0:l1], None if p.nz is None else p.nz[l0:l1], p.kind, p.cols)


# ----------------------------------------------------------------------------
# Fused all-gather over NVLink peer memory (the product path next to the NCCL baseline
# above): every rank maps every other rank's Y^T buffer into its address space once (CUDA IPC), and
# its GEMM epilogue stores each output tile of its N-shard block into all of them (bwta_gemm_peers)
# -- the gather overlaps the math tile by tile with no collective launch; one bwta_peer_barrier
# per step then makes all ranks' stores visible.  Y^T is double-buffered across steps, so a rank
# never overwrites a buffer a peer may still be reading: step s writes buffer s % 2, and reaching
# step s + 2's GEMM requires every peer to have passed step s + 1's barrier, i.e. to have finished
# everything it enqueued on step s's buffer before that.
# ----------------------------------------------------------------------------
class PeerLayout:
    """Byte layout of one rank's peer buffer: nbuf Y^T buffers [n_pad x M] (16-bit), then the
    `world` uint32 barrier flags, then (at count_off, never written by peers) the barrier count."""

    def __init__(self, plan: NShardPlan, m: int, nbuf: int = 2, elem: int = 2):
        if plan.chunks != 1:
            raise ValueError("the fused gather stores each rank's whole block from one GEMM (chunks = 1)")
        if m % 8:
            raise ValueError("M must be a multiple of 8 (16-byte Y^T rows for the TMA stores)")
        self.plan, self.m, self.nbuf, self.elem = plan, m, nbuf, elem
        self.y_bytes = -(-plan.n_pad * m * elem // 256) * 256
        self.flags_off = nbuf * self.y_bytes
        self.count_off = self.flags_off + 128
        self.total = self.flags_off + 256

    def block_offset(self, step: int) -> int:
        """Byte offset of this rank's Y^T block in buffer step % nbuf (the same in every rank's buffer)."""
        r0, _ = self.plan.block(0)
        return (step % self.nbuf) * self.y_bytes + r0 * self.m * self.elem


class PeerAllGather:
    """Y^T = gather over ranks of the N-sharded BWTA linear, stored by the GEMM epilogue straight
    into every rank's buffer.  group: the process group the IPC handles are exchanged over (any
    backend; the data path uses no collective).  One instance per (N, M) shape; close() unmaps."""

    def __init__(self, plan: NShardPlan, m: int, device, out_dtype=torch.float16, group=None, nbuf: int = 2):
        from . import ipc_handle, ipc_open
        self.lay = PeerLayout(plan, m, nbuf)
        self.plan, self.m, self.out_dtype, self.group = plan, m, out_dtype, group
        self.buf = torch.zeros(self.lay.total, dtype=torch.uint8, device=device)
        torch.cuda.synchronize(device)  # flags are zero before any peer can signal
        mine = ipc_handle(self.buf)
        world = plan.world
        allh = [None] * world
        if world > 1 or group is not None:
            dist.all_gather_object(allh, mine, group=group)
        else:
            allh = [mine]
        self._opened = []
        self.bases = []
        for r, (h, off) in enumerate(allh):
            if r == plan.rank:
                self.bases.append(self.buf.data_ptr())
            else:
                ptr = ipc_open(h, off)
                self._opened.append((ptr, off))
                self.bases.append(ptr)
        self.step = 0

    def out(self, step: int) -> torch.Tensor:
        """Y^T [N x M] of buffer step % nbuf (a view of this rank's buffer)."""
        b = step % self.lay.nbuf
        y = self.buf[b * self.lay.y_bytes:b * self.lay.y_bytes + self.plan.n_pad * self.m * 2]
        return y.view(self.out_dtype).view(self.plan.n_pad, self.m)[:self.plan.n]

    def __call__(self, a, w_local, w_scale_local: Optional[torch.Tensor], a_scale: float, stream=None,
                 design: str = "auto", tile=None) -> torch.Tensor:
        """One step: the local GEMM with its peer stores, then the barrier.  w_local: this rank's
        weight rows (plan.local_rows()).  Returns this step's gathered Y^T [N x M]."""
        from . import bwta_gemm_peers, bwta_peer_barrier
        g0, g1 = self.plan.block(0)
        off = self.lay.block_offset(self.step)
        if g1 > g0:
            peers = [b + off for r, b in enumerate(self.bases) if r != self.plan.rank]
            bwta_gemm_peers(a, w_local, w_scale_local, a_scale, self.bases[self.plan.rank] + off, self.m, peers,
                            out_dtype=self.out_dtype, y_transposed=True, design=design, stream=stream, tile=tile)
        bwta_peer_barrier([b + self.lay.flags_off for b in self.bases], self.plan.rank,
                          self.bases[self.plan.rank] + self.lay.count_off, stream=stream)
        y = self.out(self.step)
        self.step += 1
        return y

    def close(self):
        from . import ipc_close
        for ptr, off in self._opened:
            ipc_close(ptr, off)
        self._opened = []
