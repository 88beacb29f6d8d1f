"""Fused prefill attention (bwta_attn_prefill) vs the unfused BWTA path (QK^T, bool pack of a
stored P, PV), torch fp16 attention (cuBLAS QK^T, fp32 softmax, PV) and flash-attn (fp16) at
configs[3] (32 heads x 2048 x 128) and the BERT layer's attention (32 x 12 heads x 128 x 64);
L2 flushed by a 256 MiB read between reps."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bwta_inputs as gen
import paper_2604_03957_b200 as B
from quick_bench_util import timeit

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
try:
    from flash_attn import flash_attn_func
except Exception:  # pragma: no cover
    flash_attn_func = None
for (b, h, t, d) in [(1, 32, 2048, 128), (32, 12, 128, 64), (4, 32, 2048, 128), (1, 32, 8192, 128)]:
    q = gen.activations((b, h, t, d), 1).cuda()
    k = gen.activations((b, h, t, d), 2).cuda()
    v = gen.activations((b, h, t, d), 3).cuda()
    sq, sk, sv = gen.act_scale(q), gen.act_scale(k), gen.act_scale(v)
    alpha = float(np.float32(sq * sk / np.sqrt(d)))
    s_att = float(np.float32(2.0 / t))
    beta = float(np.float32(s_att * sv))
    qp, kp = B.bwta_pack_act(q, sq), B.bwta_pack_act(k, sk)
    vt = B.bwta_pack_act(v, sv, transpose=True)
    O = torch.empty((b, h, t, d), dtype=torch.float16, device="cuda")
    fused = timeit(lambda: B.bwta_attn_prefill(qp, kp, vt, alpha, s_att, beta, out=O), flush=flush)
    packs = timeit(lambda: (B.bwta_pack_act(q, sq), B.bwta_pack_act(k, sk), B.bwta_pack_act(v, sv, transpose=True)),
                   flush=flush)
    res = {"fused_us": fused * 1e3, "qkv_packs_us": packs * 1e3}
    if b * h * t * t * 2 <= (1 << 31):
        S = torch.empty((b, h, t, t), dtype=torch.float16, device="cuda")
        P = gen.attention_probs((b, h, t, t), 4).cuda()
        pp = B.bwta_pack_act(P, s_att, "bool")
        res["unfused_bwta_us"] = 1e3 * (timeit(lambda: B.bwta_attn_qk(qp, kp, alpha, out=S), flush=flush) +
                                        timeit(lambda: B.bwta_pack_act(P, s_att, "bool"), flush=flush) +
                                        timeit(lambda: B.bwta_attn_pv(pp, vt, beta, out=O), flush=flush))
        res["torch_fp16_us"] = 1e3 * timeit(lambda: torch.matmul(torch.softmax(torch.matmul(q, k.transpose(-1, -2)).float()
                                                                               * alpha, -1).half(), v), flush=flush)
        del S, P, pp
    if flash_attn_func is not None:
        qf, kf, vf = (x.transpose(1, 2).contiguous() for x in (q, k, v))
        res["flash_attn_fp16_us"] = 1e3 * timeit(lambda: flash_attn_func(qf, kf, vf, softmax_scale=alpha), flush=flush)
    ops = 4 * b * h * t * t * d
    res["fused_TOPS"] = ops / (fused * 1e-3) / 1e12
    print(f"b{b} h{h} t{t} d{d}: " + " ".join(f"{k_}={v_:.1f}" for k_, v_ in res.items()), flush=True)
