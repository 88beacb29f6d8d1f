"""C3 / configs[4] GEMMs under every design-(b) tile (in-graph, L2 warm): the tile-choice and
TMEM A-ring experiments of round 2."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bwta_inputs as gen
import paper_2604_03957_b200 as B
from quick_bench_util import time_graph

TILES = [None, (128, 2), (192, 1), (192, 2)]
for (m, k, n) in [(2048, 4096, 4096), (2048, 4096, 11008), (2048, 8192, 28672), (4096, 768, 3072)]:
    x = gen.activations((m, k), 1).cuda()
    w = gen.weights(n, k, 2).cuda()
    s_a = gen.act_scale(x)
    mu, s_w = gen.weight_stats(w)
    s_w = s_w.cuda()
    a = B.bwta_pack_act(x, s_a)
    wp = B.bwta_pack_weight(w, mu=mu)
    y = torch.empty((m, n), dtype=torch.float16, device="cuda")
    r = {str(t): time_graph(lambda: B.bwta_gemm(a, wp, s_w, s_a, out=y, tile=t)) * 1e3 for t in TILES}
    print(f"{m}x{k}x{n}: " + " ".join(f"{t}={v:.2f}us({2*m*n*k/v/1e6:.0f}T)" for t, v in r.items()), flush=True)
