"""Every design-(b) tile (BN x CTA group) vs AUTO on the BERT layer's matmuls (in-graph, L2 warm)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bwta_inputs as gen
import paper_2604_03957_b200 as B
from quick_bench_util import time_graph

TILES = [None, (64, 1), (128, 1), (192, 1), (64, 2), (128, 2), (192, 2)]
for (m, k, n, kind) in [(4096, 768, 2304, "ternary"), (4096, 768, 768, "ternary"), (4096, 768, 3072, "ternary"),
                        (4096, 3072, 768, "bool"), (2048, 4096, 11008, "ternary")]:
    x = (gen.relu_activations if kind == "bool" else gen.activations)((m, k), 1).cuda()
    w = gen.weights(n, k, 2).cuda()
    s_a = gen.act_scale(x); mu, s_w = gen.weight_stats(w); s_w = s_w.cuda()
    a = B.bwta_pack_act(x, s_a, kind); wp = B.bwta_pack_weight(w, mu=mu)
    y = torch.empty((m, n), dtype=torch.float16, device="cuda")
    r = {str(t): time_graph(lambda: B.bwta_gemm(a, wp, s_w, s_a, out=y, tile=t)) * 1e3 for t in TILES}
    rp = {str(t): time_graph(lambda: B.bwta_gemm_pack(a, wp, s_w, s_a, 0.5, "bool", tile=t)) * 1e3 for t in TILES} \
        if (m, k, n) == (4096, 768, 3072) else {}
    print(f"{m}x{k}x{n} {kind}: " + " ".join(f"{t}={v:.2f}" for t, v in r.items()), flush=True)
    if rp:
        print(f"   fused pack: " + " ".join(f"{t}={v:.2f}" for t, v in rp.items()), flush=True)
b, h, t, d = 32, 12, 128, 64
pp = B.bwta_pack_act(gen.attention_probs((b, h, t, t), 3).cuda(), 2 / t, "bool")
vt = B.bwta_pack_act(gen.activations((b, h, t, d), 4).cuda(), 1.6, transpose=True)
qp = B.bwta_pack_act(gen.activations((b, h, t, d), 5).cuda(), 1.6)
O = torch.empty((b, h, t, d), dtype=torch.float16, device="cuda")
S = torch.empty((b, h, t, t), dtype=torch.float16, device="cuda")
print("pv: " + " ".join(f"{tt}={time_graph(lambda: B.bwta_attn_pv(pp, vt, 0.1, out=O, tile=tt)) * 1e3:.2f}" for tt in TILES))
print("qk: " + " ".join(f"{tt}={time_graph(lambda: B.bwta_attn_qk(qp, qp, 0.1, out=S, tile=tt)) * 1e3:.2f}" for tt in TILES))
