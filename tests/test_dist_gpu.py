"""The N-sharded linear through a real NCCL communicator on the GPU.

Only one GPU is available to the tests, and NCCL refuses two ranks on one
device, so this runs a 1-rank NCCL process group: the chunked, in-place,
async all_gather_into_tensor calls of dist.gemm_nshard_overlap execute on
NCCL's stream exactly as at N ranks (the multi-rank host logic is covered by
tests/test_dist.py with gloo, world size 2).  The gathered Y^T must equal the
oracle bit for bit (O10)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import bwta_inputs as gen
import oracle
from test_parity_gpu import B, assert_out_equal, storage  # noqa: F401

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl_group():
    assert torch.cuda.is_available()
    torch.cuda.set_device(0)
    if not dist.is_initialized():
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
        yield dist.group.WORLD
        dist.destroy_process_group()
    else:
        yield dist.group.WORLD


@pytest.mark.parametrize("chunks", [1, 3, 4])
def test_nshard_overlap_nccl_matches_oracle(B, nccl_group, chunks):
    from paper_2604_03957_b200 import dist as D
    M, K, N = 300, 1000, 517
    x = gen.activations((M, K), 9100)
    w = gen.weights(N, K, 9101)
    s_a = gen.act_scale(x)
    mu, s_w = gen.weight_stats(w)
    a = B.bwta_pack_act(x.cuda(), s_a)
    plan = D.NShardPlan(N, 1, 0, chunks)
    rows = plan.local_rows()
    wp = B.bwta_pack_weight(w[rows].contiguous().cuda(), mu=mu)
    out = torch.full((plan.n_pad, M), float("nan"), dtype=torch.float16, device="cuda")
    yt = D.gemm_nshard_overlap(a, wp, s_w[rows].contiguous().cuda(), s_a, plan, out=out, group=nccl_group)
    torch.cuda.synchronize()
    qa = oracle.quantize_act(storage(x), "f16", s_a, "ternary")
    qw = oracle.binarize_weight(storage(w), "f16", mu=mu)
    ref = oracle.epilogue_linear(oracle.dot(qa, qw, threads=oracle.default_threads()), s_w.numpy(), s_a, "f16")
    assert yt.shape == (N, M)
    assert_out_equal(yt, np.ascontiguousarray(ref.T), f"nccl nshard chunks={chunks}")


def test_gather_rows_nccl(B, nccl_group):
    """gather_rows / gather_heads through NCCL (padded shard) equal the local block."""
    from paper_2604_03957_b200 import dist as D
    t = torch.randn(37, 64, device="cuda")
    out = torch.empty_like(t)
    dist.all_gather_into_tensor(out, t, group=nccl_group)
    torch.cuda.synchronize()
    assert torch.equal(out, t)
    assert torch.equal(D.gather_rows(t, 37, 1, nccl_group), t)
