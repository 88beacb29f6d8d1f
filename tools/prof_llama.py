"""One eager configs[2] step (pack X + both LLaMA-7B prefill linears) after warm-up, for the ncu
launch list:  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'tc_|pack_|gemv'
python tools/prof_llama.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bwta_inputs as gen
import paper_2604_03957_b200 as B

M, K = 2048, 4096
x = gen.activations((M, K), 303).cuda()
s_x = gen.act_scale(x)
ws = []
for i, n in enumerate((4096, 11008)):
    w = gen.weights(n, K, 304 + i)
    mu, s_w = gen.weight_stats(w)
    ws.append((B.bwta_pack_weight(w.cuda(), mu=mu), s_w.cuda(), torch.empty((M, n), dtype=torch.float16, device="cuda")))


def step():
    a = B.bwta_pack_act(x, s_x)
    for wp, sw, y in ws:
        B.bwta_gemm(a, wp, sw, s_x, out=y)


for _ in range(3):
    step()
torch.cuda.synchronize()
step()
torch.cuda.synchronize()
