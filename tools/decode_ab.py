"""Decode GEMV A/B (BWTA_LIB selects the library build): per shape, the GEMM alone and pack + GEMM,
each as graph of 10 x [L2 flush, op] minus graph of 10 x [L2 flush] (cold weights, as the bench)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bwta_inputs as gen
import paper_2604_03957_b200 as B
from quick_bench_util import time_graph

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
fl = lambda: flush.view(torch.int64).max()
hbm = 6553.6e9
t_fl = time_graph(fl, reps=10)
SHAPES = [(1, 8192, 28672), (2, 8192, 28672), (1, 4096, 11008), (4, 8192, 28672), (16, 8192, 28672)]
if os.environ.get("DECODE_AB_SKINNY"):
    SHAPES = [(m, k, n) for m in (8, 16, 32) for (k, n) in ((4096, 4096), (4096, 11008), (11008, 4096), (8192, 28672))]
for (m, k, n) in SHAPES:
    w = gen.weights(n, k, 2).cuda()
    mu, s_w = gen.weight_stats(w)
    s_w = s_w.cuda()
    wp = B.bwta_pack_weight(w, mu=mu)
    x = gen.activations((m, k), 1).cuda()
    s_a = gen.act_scale(x)
    a = B.bwta_pack_act(x, s_a)
    y = torch.empty((m, n), dtype=torch.float16, device="cuda")
    g = lambda: B.bwta_gemm(a, wp, s_w, s_a, out=y)
    pg = lambda: B.bwta_gemm(B.bwta_pack_act(x, s_a), wp, s_w, s_a, out=y)
    t_g = (time_graph(lambda: (fl(), g()), reps=10) - t_fl) * 1e3
    t_pg = (time_graph(lambda: (fl(), pg()), reps=10) - t_fl) * 1e3
    byt = n * k / 8 + m * k / 4 + 4 * n + 2 * m * n
    print(f"M={m:2d} K={k} N={n}: gemm {t_g:6.2f}us ({byt / (t_g * 1e-6) / hbm:.2f} HBM)  pack+gemm {t_pg:6.2f}us "
          f"({byt / (t_pg * 1e-6) / hbm:.2f} HBM)", flush=True)
