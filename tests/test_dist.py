"""Multi-process (world_size 2, gloo, CPU) checks of the N-sharded BWTA linear
and the head-sharded attention: shard bounds, padding, the all-gather layout,
and that the gathered result equals the single-process result exactly.  The
per-rank compute is the CPU oracle (the library needs a GPU); the host logic
under test is paper_2604_03957_b200.dist, the same code the GPU path runs."""
import os
import socket
import types

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2604_03957_b200 import dist as D


def test_shard_bounds_cover_and_align():
    for n in (1, 15, 16, 100, 768, 4096, 11008, 13824, 28672):
        for world in (1, 2, 3, 4, 8):
            spans = [D.shard_bounds(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (s0, e0), (s1, e1) in zip(spans, spans[1:]):
                assert e0 == s1 and s0 <= e0
            if n >= 16 * world:
                assert all((e - s) % 16 == 0 for s, e in spans[:-1])
            assert D.padded_shard(n, world) >= max(e - s for s, e in spans)
    assert D.shard_bounds(11008, 8, 3) == (3 * 1376, 4 * 1376)


def test_nshard_plan_blocks_tile_the_rows():
    """Chunk c of all ranks is one contiguous row range of Y^T (so each chunk's all-gather writes
    its final place), every row has one owner, padding only at the end."""
    for n in (1, 37, 100, 4096, 11008, 28672):
        for world in (1, 2, 4, 8):
            for chunks in (1, 2, 4):
                plans = [D.NShardPlan(n, world, r, chunks) for r in range(world)]
                p0 = plans[0]
                assert p0.n_pad >= n and p0.n_pad - n < world * chunks
                for c in range(chunks):
                    spans = [p.block(c) for p in plans]
                    assert spans[0][0] == min(n, c * world * p0.nrc)
                    for (s0, e0), (s1, e1) in zip(spans, spans[1:]):
                        assert e0 == s1
                owned = torch.cat([p.local_rows() for p in plans]).sort().values
                assert torch.equal(owned, torch.arange(n))
                for p in plans:
                    tot = 0
                    for c in range(chunks):
                        l0, l1 = p.local_span(c)
                        assert l0 == tot and l1 - l0 == p.block(c)[1] - p.block(c)[0]
                        tot = l1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outq):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(5)
        M, N, K = 37, 100, 300                      # ragged everywhere
        qa = rng.integers(-1, 2, (M, K)).astype(np.int8)
        qw = np.where(rng.integers(0, 2, (N, K)) == 1, 1, -1).astype(np.int8)
        s_w = rng.uniform(0.01, 0.05, N).astype(np.float32)
        s_a = 1.7
        s, e = D.shard_bounds(N, world, rank)
        a = types.SimpleNamespace(ref=torch.zeros((M, 1)))
        w_local = qw[s:e]

        def local_gemm(a_, w_, sw_, sa_, out_):
            y = oracle.gemm(qa, w_, sw_.numpy(), sa_, "f32")           # [M, n_r]
            out_.copy_(torch.from_numpy(np.ascontiguousarray(y.T)))
        yt = D.gemm_nshard(a, w_local, torch.from_numpy(s_w[s:e]), s_a, N, world, rank,
                           out_dtype=torch.float32, local_gemm=local_gemm)
        full = oracle.gemm(qa, qw, s_w, s_a, "f32").T
        ok_gemm = bool(np.array_equal(yt.numpy().view(np.uint32), np.ascontiguousarray(full).view(np.uint32)))

        # head-sharded attention: 5 (batch x head) entries over the ranks
        BH, T, Dh = 5, 9, 64
        qq = rng.integers(-1, 2, (BH, T, Dh)).astype(np.int8)
        kk = rng.integers(-1, 2, (BH, T, Dh)).astype(np.int8)
        h0, h1 = D.heads_shard(BH, world, rank)
        local = torch.from_numpy(oracle.attn_qk(qq[h0:h1], kk[h0:h1], 0.25, "f32")) if h1 > h0 else \
            torch.zeros((0, T, T), dtype=torch.float32)
        s_all = D.gather_heads(local, BH, world)
        ok_attn = bool(np.array_equal(s_all.numpy(), oracle.attn_qk(qq, kk, 0.25, "f32")))

        # chunked N partition with the in-place, overlapped per-chunk all-gathers
        ok_chunks = True
        for chunks in (1, 3, 7):
            plan = D.NShardPlan(N, world, rank, chunks)
            rows = plan.local_rows().numpy()
            yt2 = D.gemm_nshard_overlap(a, qw[rows], torch.from_numpy(s_w[rows]), s_a, plan,
                                        out_dtype=torch.float32, local_gemm=local_gemm)
            ok_chunks &= yt2.shape == (N, M) and bool(np.array_equal(
                yt2.numpy().view(np.uint32), np.ascontiguousarray(full).view(np.uint32)))
            # every global row is owned by exactly one rank
            owned = torch.from_numpy(rows.astype(np.int64))
            sizes = [None] * world
            dist.all_gather_object(sizes, owned.tolist())
            flat = sorted(i for r in sizes for i in r)
            ok_chunks &= flat == list(range(N))
        outq.put((rank, ok_gemm and ok_chunks, ok_attn))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_nshard_gemm_and_head_shard_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok_g and ok_a for _, ok_g, ok_a in res), res


def test_peer_layout_blocks_line_up():
    """The fused gather's byte layout: each rank's block offset in buffer s is its NShardPlan rows
    (the same offset in every rank's buffer, so peer stores land where the owner's would), 16-byte
    aligned, buffers disjoint, flags after them."""
    for n, m, world in ((1000, 256, 2), (11008, 2048, 8), (37, 8, 4), (4096, 2048, 1)):
        for r in range(world):
            plan = D.NShardPlan(n, world, r, 1)
            lay = D.PeerLayout(plan, m, nbuf=2)
            g0, g1 = plan.block(0)
            for step in range(4):
                off = lay.block_offset(step)
                assert off % 16 == 0
                assert off == (step % 2) * lay.y_bytes + g0 * m * 2
                assert off + (g1 - g0) * m * 2 <= (step % 2 + 1) * lay.y_bytes
            assert lay.y_bytes >= plan.n_pad * m * 2 and lay.flags_off == 2 * lay.y_bytes
            assert lay.total >= lay.flags_off + 4 * world
    with pytest.raises(ValueError):
        D.PeerLayout(D.NShardPlan(100, 2, 0, 2), 64)    # chunked plans are NCCL-only
    with pytest.raises(ValueError):
        D.PeerLayout(D.NShardPlan(100, 2, 0, 1), 12)    # 16-byte Y^T rows
