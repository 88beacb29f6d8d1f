"""One decode shape, a few launches (for ncu)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bwta_inputs as gen
import paper_2604_03957_b200 as B
m, k, n = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (16, 8192, 28672)))
w = gen.weights(n, k, 2).cuda()
mu, s_w = gen.weight_stats(w)
wp = B.bwta_pack_weight(w, mu=mu)
x = gen.activations((m, k), 1).cuda()
s_a = gen.act_scale(x)
a = B.bwta_pack_act(x, s_a)
y = torch.empty((m, n), dtype=torch.float16, device="cuda")
for _ in range(3):
    B.bwta_gemm(a, wp, s_w.cuda(), s_a, out=y)
torch.cuda.synchronize()
