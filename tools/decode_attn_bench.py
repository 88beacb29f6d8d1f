"""Fused decode attention (one launch) vs the unfused BWTA path (QK^T, fp16 P via torch softmax,
bool pack, PV: 4+ launches) vs cuBLAS/torch fp16 -- in-graph times, LLaMA-7B decode shapes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bwta_inputs as gen
import paper_2604_03957_b200 as B
from quick_bench_util import time_graph

for (b, h, tk, dh) in [(1, 32, 2048, 128), (8, 32, 2048, 128), (1, 32, 8192, 128)]:
    q = gen.activations((b, h, 1, dh), 1).cuda()
    k = gen.activations((b, h, tk, dh), 2).cuda()
    v = gen.activations((b, h, tk, dh), 3).cuda()
    sq, sk, sv = gen.act_scale(q), gen.act_scale(k), gen.act_scale(v)
    alpha = float(np.float32(sq * sk / np.sqrt(dh)))
    s_att = float(np.float32(2.0 / tk))
    beta = float(np.float32(s_att * sv))
    qp, kp = B.bwta_pack_act(q, sq), B.bwta_pack_act(k, sk)
    vt = B.bwta_pack_act(v, sv, transpose=True)
    t_f = time_graph(lambda: B.bwta_attn_decode(qp, kp, vt, alpha, s_att, beta))

    def unfused():
        s = B.bwta_attn_qk(qp, kp, alpha)
        p = torch.softmax(s.float(), -1).half()
        B.bwta_attn_pv(B.bwta_pack_act(p, s_att, "bool"), vt, beta)
    t_u = time_graph(unfused)
    t_t = time_graph(lambda: torch.softmax((q @ k.transpose(-1, -2)).float() * alpha, -1).half() @ v)
    print(f"B={b} H={h} Tk={tk} Dh={dh}: fused {t_f*1e3:6.2f} us | unfused BWTA {t_u*1e3:6.2f} us | "
          f"torch fp16 {t_t*1e3:6.2f} us", flush=True)
