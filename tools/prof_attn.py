"""One fused prefill attention launch at configs[3] (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bwta_inputs as gen
import paper_2604_03957_b200 as B

b, h, t, d = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (1, 32, 2048, 128)))
q, k, v = (gen.activations((b, h, t, d), s).cuda() for s in (1, 2, 3))
sq, sk, sv = gen.act_scale(q), gen.act_scale(k), gen.act_scale(v)
alpha = float(np.float32(sq * sk / np.sqrt(d)))
s_att = float(np.float32(2.0 / t))
beta = float(np.float32(s_att * sv))
qp, kp = B.bwta_pack_act(q, sq), B.bwta_pack_act(k, sk)
vt = B.bwta_pack_act(v, sv, transpose=True)
for _ in range(3):
    B.bwta_attn_prefill(qp, kp, vt, alpha, s_att, beta)
torch.cuda.synchronize()
