"""The fused all-gather (bwta_gemm_peers + bwta_peer_barrier) on the GPU.

Only one GPU is available, so:
  * single process: the "peers" are other buffers on the same GPU -- every output tile must land
    bit-identically in y and in each peer buffer, equal to the oracle (O10), for every tile class
    and orientation the epilogue takes;
  * two processes sharing GPU 0 (gloo only for the IPC-handle exchange): the real path -- CUDA IPC
    mappings of the other process's buffer, TMA stores into it from the epilogue, the system-scope
    flag barrier -- gathering an N-sharded linear over 2 ranks for several steps; each rank's Y^T
    must equal the oracle's full Y^T bit for bit.  (NCCL refuses two ranks on one device; IPC and
    the flag barrier do not care.)"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import bwta_inputs as gen
import oracle
from test_parity_gpu import B, assert_out_equal, storage  # noqa: F401

pytestmark = pytest.mark.gpu


def _ref_yt(x, w, s_a, mu, s_w, dt="f16"):
    qa = oracle.quantize_act(storage(x), "f16", s_a, "ternary")
    qw = oracle.binarize_weight(storage(w), "f16", mu=mu)
    ref = oracle.epilogue_linear(oracle.dot(qa, qw, threads=oracle.default_threads()), s_w.numpy(), s_a, dt)
    return np.ascontiguousarray(ref.T)


@pytest.mark.parametrize("M,N,K,tile", [(256, 384, 1000, None), (304, 517, 777, None), (2048, 640, 4096, None),
                                        (512, 1000, 2048, (128, 1)), (200, 3000, 1500, None),
                                        (1000, 96, 2500, (64, 2)),
                                        (2048, 4096, 2048, None)])  # >= 2 tile rounds: the 1-warp epilogue (E1)
def test_gemm_peers_stores_every_tile_to_every_peer(B, M, N, K, tile):
    seed = 9300 + M + N
    x = gen.activations((M, K), seed)
    w = gen.weights(N, K, seed + 1)
    s_a = gen.act_scale(x)
    mu, s_w = gen.weight_stats(w)
    a = B.bwta_pack_act(x.cuda(), s_a)
    wp = B.bwta_pack_weight(w.cuda(), mu=mu)
    bufs = [torch.full((N, M), float("nan"), dtype=torch.float16, device="cuda") for _ in range(3)]
    B.bwta_gemm_peers(a, wp, s_w.cuda(), s_a, bufs[0].data_ptr(), M, [bufs[1].data_ptr(), bufs[2].data_ptr()],
                      y_transposed=True, tile=tile)
    torch.cuda.synchronize()
    ref = _ref_yt(x, w, s_a, mu, s_w)
    for i, b in enumerate(bufs):
        assert_out_equal(b, ref, f"peer buffer {i}")
    # the same call through bwta_gemm (no peers) is the same kernel output
    y = B.bwta_gemm(a, wp, s_w.cuda(), s_a, y_transposed=True, tile=tile)
    assert torch.equal(y.view(torch.int16), bufs[0].view(torch.int16))


def test_gemm_peers_bf16_and_y_not_transposed(B):
    M, N, K = 384, 640, 1300
    x = gen.activations((M, K), 9400)
    w = gen.weights(N, K, 9401)
    s_a = gen.act_scale(x)
    mu, s_w = gen.weight_stats(w)
    a = B.bwta_pack_act(x.cuda(), s_a)
    wp = B.bwta_pack_weight(w.cuda(), mu=mu)
    y0 = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    y1 = torch.empty_like(y0)
    B.bwta_gemm_peers(a, wp, s_w.cuda(), s_a, y0.data_ptr(), N, [y1.data_ptr()], out_dtype=torch.bfloat16,
                      y_transposed=False)
    torch.cuda.synchronize()
    ref = _ref_yt(x, w, s_a, mu, s_w, "bf16").T
    assert_out_equal(y0, np.ascontiguousarray(ref), "bf16 y")
    assert torch.equal(y0.view(torch.int16), y1.view(torch.int16))


def test_gemm_peers_unsupported_shapes_enqueue_nothing(B):
    """Skinny products take the GEMV epilogue, which has no peer stores: UNSUPPORTED, buffers untouched."""
    M, N, K = 8, 4096, 1024
    x = gen.activations((M, K), 9500)
    w = gen.weights(N, K, 9501)
    a = B.bwta_pack_act(x.cuda(), 0.5)
    wp = B.bwta_pack_weight(w.cuda())
    y0 = torch.zeros((N, M), dtype=torch.float16, device="cuda")
    y1 = torch.zeros_like(y0)
    with pytest.raises(B.BwtaError, match="UNSUPPORTED"):
        B.bwta_gemm_peers(a, wp, None, 0.5, y0.data_ptr(), M, [y1.data_ptr()])
    torch.cuda.synchronize()
    assert not y0.any() and not y1.any()


def test_peer_barrier_single_rank_counts_in_device_memory(B):
    """The epoch is read from and written back to device memory: eager calls and CUDA-graph replays
    both advance it."""
    flags = torch.zeros(64, dtype=torch.int32, device="cuda")
    count = flags[32:]
    for _ in range(5):
        B.bwta_peer_barrier([flags.data_ptr()], 0, count.data_ptr())
    torch.cuda.synchronize()
    assert int(flags[0]) == 5 and int(count[0]) == 5
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        B.bwta_peer_barrier([flags.data_ptr()], 0, count.data_ptr(), stream=s)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert int(flags[0]) == 8 and int(count[0]) == 8


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _peer_worker(rank, world, port, M, N, K, steps, outq):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2604_03957_b200 as Bk
        from paper_2604_03957_b200 import dist as D
        torch.cuda.set_device(0)
        plan = D.NShardPlan(N, world, rank, 1)
        rows = plan.local_rows()
        pg = D.PeerAllGather(plan, M, "cuda", group=None if world == 1 else dist.group.WORLD)
        ok, msgs = True, []
        for step in range(steps):
            seed = 9600 + 10 * step
            x = gen.activations((M, K), seed)          # the same inputs on every rank
            w = gen.weights(N, K, seed + 1)
            s_a = gen.act_scale(x)
            mu, s_w = gen.weight_stats(w)
            a = Bk.bwta_pack_act(x.cuda(), s_a)
            wl = Bk.bwta_pack_weight(w[rows].contiguous().cuda(), mu=mu)
            yt = pg(a, wl, s_w[rows].contiguous().cuda(), s_a)
            torch.cuda.synchronize()
            ref = _ref_yt(x, w, s_a, mu, s_w)
            got = yt.cpu().view(torch.int16).numpy().view(np.uint16)
            same = got.shape == ref.shape and np.array_equal(got, ref)
            ok &= bool(same)
            if not same:
                msgs.append(f"rank {rank} step {step}: {int((got != ref).sum()) if got.shape == ref.shape else got.shape}"
                            " mismatches")
            dist.barrier()   # (test only) keep the steps in lockstep on the host too
        pg.close()
        outq.put((rank, ok, msgs))
    except Exception as e:  # report instead of hanging the parent
        outq.put((rank, False, [repr(e)]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("M,N,K,steps", [(256, 1000, 1000, 3), (512, 3000, 2048, 2)])
def test_peer_all_gather_two_processes_one_gpu(B, M, N, K, steps):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    world = 2
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, M, N, K, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        res = [q.get(timeout=240) for _ in range(world)]
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    assert all(ok for _, ok, _ in res), res
    for p in procs:
        assert p.exitcode == 0
