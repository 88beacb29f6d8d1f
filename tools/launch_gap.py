"""What a lone tile-kernel launch costs beyond back-to-back replays (tools/cold_warm.py showed
~7.5 us at C3 N = 11008 with warm L2).  All in CUDA graphs of 20 repetitions, per-repetition
device time; 'after X' = graph of [X, gemm] minus graph of [X]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bwta_inputs as gen
import paper_2604_03957_b200 as B
from quick_bench_util import time_graph

m, k = 2048, 4096
x = gen.activations((m, k), 1).cuda()
s_a = gen.act_scale(x)
a = B.bwta_pack_act(x, s_a)
tiny = torch.zeros(16, device="cuda")
xs = gen.activations((128, 256), 3).cuda()
big_x = gen.activations((2048, 4096), 4).cuda()
for n in (4096, 11008):
    w = gen.weights(n, k, 2).cuda()
    mu, s_w = gen.weight_stats(w)
    s_w = s_w.cuda()
    wp = B.bwta_pack_weight(w, mu=mu)
    y = torch.empty((m, n), dtype=torch.float16, device="cuda")
    g = lambda: B.bwta_gemm(a, wp, s_w, s_a, out=y)
    ops = 2 * m * n * k
    res = {"b2b": time_graph(g)}
    preds = {
        "torch_tiny": lambda: tiny.add_(1.0),
        "pack_tiny": lambda: B.bwta_pack_act(xs, 1.0),
        "pack_x": lambda: B.bwta_pack_act(big_x, s_a),
        "sleep2us": lambda: torch.cuda._sleep(4000),
    }
    for name, pf in preds.items():
        t1 = time_graph(lambda: (pf(), g()))
        t0 = time_graph(pf)
        res["after_" + name] = t1 - t0
        res["pred_" + name] = t0
    print(f"N={n}: " + "  ".join(f"{kk}={v*1e3:.2f}us" for kk, v in res.items()), flush=True)
