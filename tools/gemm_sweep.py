"""Sweep design knobs on a few GEMM shapes (device time, amortised graphs)."""
import sys, os, statistics, subprocess, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import torch, bwta_inputs as gen, paper_2604_03957_b200 as B
    from bench import op_time_ms
    s = torch.cuda.Stream(); flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    res = {}
    for (m, k, n, kind) in [(4096, 768, 2304, "ternary"), (4096, 3072, 768, "bool"), (2048, 4096, 4096, "ternary"), (2048, 4096, 11008, "ternary")]:
        x = (gen.relu_activations if kind == "bool" else gen.activations)((m, k), 1).cuda(); w = gen.weights(n, k, 2).cuda()
        s_a = gen.act_scale(x); mu, s_w = gen.weight_stats(w); s_w = s_w.cuda()
        a = B.bwta_pack_act(x, s_a, kind); wp = B.bwta_pack_weight(w, mu=mu)
        y = torch.empty((m, n), dtype=torch.float16, device="cuda")
        res[f"{m}x{k}x{n}"] = op_time_ms(lambda: B.bwta_gemm(a, wp, s_w, s_a, out=y, design="tcgen05"), flush, s) * 1e3
    b, h, t, d = 32, 12, 128, 64
    pp = B.bwta_pack_act(gen.attention_probs((b, h, t, t), 3).cuda(), 2 / t, "bool")
    vt = B.bwta_pack_act(gen.activations((b, h, t, d), 4).cuda(), 1.6, transpose=True)
    qp = B.bwta_pack_act(gen.activations((b, h, t, d), 5).cuda(), 1.6)
    O = torch.empty((b, h, t, d), dtype=torch.float16, device="cuda"); S = torch.empty((b, h, t, t), dtype=torch.float16, device="cuda")
    res["pv_bert"] = op_time_ms(lambda: B.bwta_attn_pv(pp, vt, 0.1, out=O, design="tcgen05"), flush, s) * 1e3
    res["qk_bert"] = op_time_ms(lambda: B.bwta_attn_qk(qp, qp, 0.1, out=S, design="tcgen05"), flush, s) * 1e3
    print(json.dumps(res))
else:
    for env in [{}, {"BWTA_TC_SWAP": "0"}, {"BWTA_TC_SWAP": "1"}, {"BWTA_TC_CG": "1"}, {"BWTA_TC_TMA_STORE": "0"}]:
        out = subprocess.run([sys.executable, __file__, "child"], env=os.environ | env, capture_output=True, text=True)
        print(env, out.stdout.strip() or out.stderr[-500:])
