"""Skinny (decode) products: the skinny tcgen05 kernel vs the tile kernel with forced tiles (in-graph,
L2 flushed), M = 8 / 16 / 32 x K 8192 x N 28672 and LLaMA-7B shapes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bwta_inputs as gen
import paper_2604_03957_b200 as B
from quick_bench_util import timeit

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for (m, k, n) in [(16, 8192, 28672), (8, 8192, 28672), (32, 8192, 28672), (16, 4096, 11008), (16, 4096, 4096)]:
    x = gen.activations((m, k), 1).cuda()
    w = gen.weights(n, k, 2).cuda()
    s_a = gen.act_scale(x)
    mu, s_w = gen.weight_stats(w)
    s_w = s_w.cuda()
    a = B.bwta_pack_act(x, s_a)
    wp = B.bwta_pack_weight(w, mu=mu)
    y = torch.empty((m, n), dtype=torch.float16, device="cuda")
    r = {}
    for name, kw in (("auto", {}), ("t192x1", dict(tile=(192, 1))), ("t128x1", dict(tile=(128, 1))),
                     ("t64x1", dict(tile=(64, 1)))):
        r[name] = timeit(lambda: B.bwta_gemm(a, wp, s_w, s_a, out=y, **kw), flush=flush) * 1e3
    wb = n * k / 8
    print(f"{m}x{k}x{n}: " + " ".join(f"{k_}={v:.1f}us({wb / v / 1e3:.0f}GB/s)" for k_, v in r.items()), flush=True)
