"""configs[2] grouped launch (both linears over the row-concatenated weights), a few launches (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bwta_inputs as gen
import paper_2604_03957_b200 as B

M, K, Ns = 2048, 4096, (4096, 11008)
x = gen.activations((M, K), 303).cuda()
s_a = gen.act_scale(x)
ws = [gen.weights(n, K, 304 + i) for i, n in enumerate(Ns)]
stats = [gen.weight_stats(w) for w in ws]
mu_cat = torch.cat([torch.full((n,), float(mu), dtype=torch.float32) for n, (mu, _) in zip(Ns, stats)]).cuda()
wp = B.bwta_pack_weight(torch.cat(ws).cuda(), mu=mu_cat)
sw = torch.cat([s for _, s in stats]).cuda()
y = torch.empty((M, sum(Ns)), dtype=torch.float16, device="cuda")
for _ in range(3):
    a = B.bwta_pack_act(x, s_a)
    B.bwta_gemm(a, wp, sw, s_a, out=y)
torch.cuda.synchronize()
