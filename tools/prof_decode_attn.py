"""One fused decode attention launch (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bwta_inputs as gen
import paper_2604_03957_b200 as B
b, h, tk, dh = 1, 32, 2048, 128
q = gen.activations((b, h, 1, dh), 1).cuda(); k = gen.activations((b, h, tk, dh), 2).cuda(); v = gen.activations((b, h, tk, dh), 3).cuda()
qp, kp, vt = B.bwta_pack_act(q, 1.6), B.bwta_pack_act(k, 1.6), B.bwta_pack_act(v, 1.6, transpose=True)
for _ in range(3):
    B.bwta_attn_decode(qp, kp, vt, 0.1, 2.0 / tk, 0.01)
torch.cuda.synchronize()
