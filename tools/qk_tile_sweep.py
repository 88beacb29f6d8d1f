"""C4 attention QK^T: every design-(b) tile vs AUTO vs cuBLAS (in-graph)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bwta_inputs as gen, paper_2604_03957_b200 as B
from quick_bench_util import time_graph
b, h, t, d = 1, 32, 2048, 128
qp = B.bwta_pack_act(gen.activations((b, h, t, d), 3).cuda(), 1.6)
kp = B.bwta_pack_act(gen.activations((b, h, t, d), 4).cuda(), 1.6)
S = torch.empty((b, h, t, t), dtype=torch.float16, device="cuda")
q16 = gen.activations((b, h, t, d), 3).cuda(); k16 = gen.activations((b, h, t, d), 4).cuda()
print("cuBLAS", time_graph(lambda: torch.matmul(q16, k16.transpose(-1, -2))) * 1e3)
for tile in [None, (64, 1), (128, 1), (192, 1), (64, 2), (128, 2), (192, 2)]:
    print(tile, round(time_graph(lambda: B.bwta_attn_qk(qp, kp, 0.1, out=S, tile=tile)) * 1e3, 2))
