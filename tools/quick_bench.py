"""Quick kernel timings (development aid, not the bench contract)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bwta_inputs as gen
import paper_2604_03957_b200 as B

def timeit(fn, iters=20, warm=5, flush=None):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        if flush is not None: flush.zero_()
        torch.cuda._sleep(300000)   # keep the GPU busy while the CPU enqueues: time = device time only
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ts.sort(); return ts[len(ts)//2]

flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for (m, k, n) in [(2048, 4096, 4096), (2048, 4096, 11008), (4096, 768, 3072), (128, 768, 768), (16, 8192, 28672)]:
    x = gen.activations((m, k), 1).cuda(); w = gen.weights(n, k, 2).cuda()
    s_a = gen.act_scale(x); mu, s_w = gen.weight_stats(w); s_w = s_w.cuda()
    a = B.bwta_pack_act(x, s_a); wp = B.bwta_pack_weight(w, mu=mu)
    y = torch.empty((m, n), dtype=torch.float16, device="cuda")
    t_pack = timeit(lambda: B.bwta_pack_act(x, s_a), flush=flush)
    res = {}
    for d in ("tcgen05", "cuda_core"):
        if d == "cuda_core" and m * n * k > 2e11: continue
        res[d] = timeit(lambda: B.bwta_gemm(a, wp, s_w, s_a, out=y, design=d), flush=flush)
    xh = x.half(); wh = w.half()
    t_cub = timeit(lambda: torch.nn.functional.linear(xh, wh), flush=flush)
    ops = 2 * m * n * k
    print(f"M={m} K={k} N={n}: pack {t_pack*1e3:.1f}us ({(2*m*k+m*k/4)/t_pack/1e6:.0f} GB/s) | " +
          " | ".join(f"{d} {t*1e3:.1f}us {ops/t/1e9:.0f} TOPS" for d, t in res.items()) +
          f" | cuBLAS fp16 {t_cub*1e3:.1f}us {ops/t_cub/1e9:.0f} TFLOPS")
# attention C4
b, h, t, d = 1, 32, 2048, 128
q = gen.activations((b, h, t, d), 3).cuda(); kk = gen.activations((b, h, t, d), 4).cuda(); v = gen.activations((b, h, t, d), 5).cuda()
p = gen.attention_probs((b, h, t, t), 6).cuda()
qp = B.bwta_pack_act(q, 1.6); kp = B.bwta_pack_act(kk, 1.6); vt = B.bwta_pack_act(v, 1.6, transpose=True)
pp = B.bwta_pack_act(p, 2.0 / t, "bool")
S = torch.empty((b, h, t, t), dtype=torch.float16, device="cuda")
O = torch.empty((b, h, t, d), dtype=torch.float16, device="cuda")
ops = 2 * b * h * t * t * d
for dsg in ("tcgen05", "cuda_core"):
    tq = timeit(lambda: B.bwta_attn_qk(qp, kp, 0.1, out=S, design=dsg), flush=flush)
    tp = timeit(lambda: B.bwta_attn_pv(pp, vt, 0.1, out=O, design=dsg), flush=flush)
    print(f"C4 {dsg}: QK {tq*1e3:.1f}us ({ops/tq/1e9:.0f} TOPS) PV {tp*1e3:.1f}us ({ops/tp/1e9:.0f} TOPS)")
tpk = timeit(lambda: B.bwta_pack_act(p, 2.0 / t, "bool"), flush=flush)
tvt = timeit(lambda: B.bwta_pack_act(v, 1.6, transpose=True), flush=flush)
print(f"C4 pack P {tpk*1e3:.1f}us {(p.numel()*2.125)/tpk/1e6:.0f} GB/s; pack V^T {tvt*1e3:.1f}us {(v.numel()*2.25)/tvt/1e6:.0f} GB/s")
qh, kh, vh = q.half(), kk.half(), v.half()
print(f"C4 cuBLAS: QK {timeit(lambda: torch.matmul(qh, kh.transpose(-1,-2)), flush=flush)*1e3:.1f}us PV {timeit(lambda: torch.matmul(p, vh), flush=flush)*1e3:.1f}us")
