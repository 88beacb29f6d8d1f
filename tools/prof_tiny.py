"""Tiny problems: fixed per-launch cost of each kernel (for ncu)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bwta_inputs as gen
import paper_2604_03957_b200 as B
for (m, k, n) in [(1, 256, 128), (128, 256, 128), (1, 8192, 128), (1, 256, 28672)]:
    w = gen.weights(n, k, 2).cuda()
    mu, s_w = gen.weight_stats(w)
    wp = B.bwta_pack_weight(w, mu=mu)
    x = gen.activations((m, k), 1).cuda()
    s_a = gen.act_scale(x)
    a = B.bwta_pack_act(x, s_a)
    y = torch.empty((m, n), dtype=torch.float16, device="cuda")
    for _ in range(2):
        B.bwta_gemm(a, wp, s_w.cuda(), s_a, out=y)
        B.bwta_gemm(a, wp, s_w.cuda(), s_a, out=y, tile=(64, 1))
torch.cuda.synchronize()
