"""DEV A/B (historical): kernel-A codes in shared memory vs in TMEM; needs a build with the
BWTA_A_TMEM switch (removed once TMEM-A became the default: 2-7 % faster on every shape measured)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bwta_inputs as gen
import paper_2604_03957_b200 as B
from quick_bench_util import timeit, time_graph

flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for (m, k, n, kind) in [(4096, 768, 2304, "ternary"), (4096, 768, 768, "ternary"), (4096, 768, 3072, "ternary"),
                        (4096, 3072, 768, "bool"), (2048, 4096, 4096, "ternary"), (2048, 4096, 11008, "ternary")]:
    x = gen.activations((m, k), 1).cuda()
    if kind == "bool":
        x = torch.relu(x)
    w = gen.weights(n, k, 2).cuda()
    s_a = gen.act_scale(x); mu, s_w = gen.weight_stats(w); s_w = s_w.cuda()
    a = B.bwta_pack_act(x, s_a, kind); wp = B.bwta_pack_weight(w, mu=mu)
    y = torch.empty((m, n), dtype=torch.float16, device="cuda")
    res = {}
    for mode in ("0", "1"):
        os.environ["BWTA_A_TMEM"] = mode
        yy = B.bwta_gemm(a, wp, s_w, s_a, out=y).clone()
        res[mode] = (timeit(lambda: B.bwta_gemm(a, wp, s_w, s_a, out=y), flush=flush),
                     time_graph(lambda: B.bwta_gemm(a, wp, s_w, s_a, out=y)), yy)
    same = torch.equal(res["0"][2].view(torch.int16), res["1"][2].view(torch.int16))
    print(f"M={m} K={k} N={n} {kind}: smem-A {res['0'][0]*1e3:6.2f}us (graph {res['0'][1]*1e3:6.2f}) | "
          f"TMEM-A {res['1'][0]*1e3:6.2f}us (graph {res['1'][1]*1e3:6.2f}) | equal={same}", flush=True)
