"""Skinny (decode) GEMM timings: skinny tcgen05 kernel (auto) vs the general
tile kernel (forced tile) vs cuBLAS FP16, L2 flushed (development aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bwta_inputs as gen
import paper_2604_03957_b200 as B
from quick_bench_util import timeit, time_graph

flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
hbm = 6532e9
for (k, n) in [(4096, 4096), (4096, 11008), (11008, 4096), (5120, 13824), (8192, 28672)]:
    w = gen.weights(n, k, 2).cuda()
    mu, s_w = gen.weight_stats(w); s_w = s_w.cuda()
    wp = B.bwta_pack_weight(w, mu=mu)
    wh = w.half()
    for m in (1, 2, 4, 8, 16, 32):
        x = gen.activations((m, k), 1).cuda()
        s_a = gen.act_scale(x)
        a = B.bwta_pack_act(x, s_a)
        y = torch.empty((m, n), dtype=torch.float16, device="cuda")
        t_sk = timeit(lambda: B.bwta_gemm(a, wp, s_w, s_a, out=y), flush=flush)
        g_x = time_graph(lambda: B.bwta_gemm_x(x, s_a, wp, s_w)) if m <= 4 else float("nan")
        g_px = time_graph(lambda: B.bwta_gemm(B.bwta_pack_act(x, s_a), wp, s_w, s_a, out=y))
        t_gen = timeit(lambda: B.bwta_gemm(a, wp, s_w, s_a, out=y, design="tcgen05"), flush=flush)
        xh = x.half()
        t_cub = timeit(lambda: torch.nn.functional.linear(xh, wh), flush=flush)
        g_sk = time_graph(lambda: B.bwta_gemm(a, wp, s_w, s_a, out=y))
        g_cub = time_graph(lambda: torch.nn.functional.linear(xh, wh))
        byt = n * k / 8 + m * k / 4 + 4 * n + 2 * m * n
        print(f"M={m:2d} K={k} N={n}: skinny {t_sk*1e3:6.2f}us ({byt/t_sk/1e6:5.0f} GB/s, {byt/(t_sk*1e-3)/hbm:.2f} HBM)"
              f" | tcgen05 {t_gen*1e3:6.2f}us | cuBLAS fp16 {t_cub*1e3:6.2f}us | x{t_cub/t_sk:5.1f} vs cuBLAS"
              f" || graph (L2 warm): skinny {g_sk*1e3:6.2f}us pack+gemm {g_px*1e3:6.2f}us fused gemm_x {g_x*1e3:6.2f}us"
              f" cuBLAS {g_cub*1e3:6.2f}us", flush=True)
