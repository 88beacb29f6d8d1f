import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bwta_inputs as gen, paper_2604_03957_b200 as B
m, k, n = 2048, 4096, int(sys.argv[1]) if len(sys.argv) > 1 else 11008
x = gen.activations((m, k), 1).cuda(); w = gen.weights(n, k, 2).cuda()
s_a = gen.act_scale(x); mu, s_w = gen.weight_stats(w); s_w = s_w.cuda()
a = B.bwta_pack_act(x, s_a); wp = B.bwta_pack_weight(w, mu=mu)
y = torch.empty((m, n), dtype=torch.float16, device="cuda")
for _ in range(3):
    B.bwta_pack_act(x, s_a); B.bwta_gemm(a, wp, s_w, s_a, out=y, design="tcgen05")
torch.cuda.synchronize()
