"""Design (a) CUDA-core vs design (b) tcgen05, per shape (device time, L2 flushed).
    python tools/design_sweep.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bwta_inputs as gen
import paper_2604_03957_b200 as B

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timeit(fn, iters=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        flush.zero_()
        torch.cuda._sleep(200000)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2] * 1e3


def gemm_case(m, k, n, kind="ternary"):
    x = gen.activations((m, k), 1).cuda()
    if kind == "bool":
        x = torch.relu(x)
    w = gen.weights(n, k, 2).cuda()
    a = B.bwta_pack_act(x, 1.6, kind=kind)
    wp = B.bwta_pack_weight(w)
    y = torch.empty((m, n), dtype=torch.float16, device="cuda")
    sw = torch.rand(n, device="cuda") * 0.05 + 0.01
    return {d: timeit(lambda d=d: B.bwta_gemm(a, wp, sw, 1.6, out=y, design=d)) for d in ("cuda_core", "tcgen05")}


def attn_case(bh, t, d):
    q = torch.randn(bh, t, d, device="cuda", dtype=torch.float16)
    k = torch.randn(bh, t, d, device="cuda", dtype=torch.float16)
    v = torch.randn(bh, t, d, device="cuda", dtype=torch.float16)
    p = torch.softmax(torch.randn(bh, t, t, device="cuda"), -1).half()
    qp, kp = B.bwta_pack_act(q, 1.6), B.bwta_pack_act(k, 1.6)
    pp = B.bwta_pack_act(p, 2.0 / t, kind="bool")
    vt = B.bwta_pack_act(v, 1.6, transpose=True)
    s = torch.empty(bh, t, t, device="cuda", dtype=torch.float16)
    o = torch.empty(bh, t, d, device="cuda", dtype=torch.float16)
    r = {}
    for dsn in ("cuda_core", "tcgen05"):
        r["qk_" + dsn] = timeit(lambda: B.bwta_attn_qk(qp, kp, 0.1, out=s, design=dsn))
        r["pv_" + dsn] = timeit(lambda: B.bwta_attn_pv(pp, vt, 0.1, out=o, design=dsn))
    return r


for (m, k, n, kind) in [(128, 768, 768, "ternary"), (4096, 768, 2304, "ternary"), (4096, 768, 768, "ternary"),
                        (4096, 768, 3072, "ternary"), (4096, 3072, 768, "bool"), (2048, 4096, 4096, "ternary"),
                        (16, 8192, 28672, "ternary"), (64, 4096, 11008, "ternary")]:
    r = gemm_case(m, k, n, kind)
    print(f"gemm M={m} K={k} N={n} {kind}: " + " ".join(f"{d} {t:.1f}us" for d, t in r.items()), flush=True)
for (bh, t, d) in [(384, 128, 64), (32, 2048, 128), (64, 512, 64)]:
    r = attn_case(bh, t, d)
    print(f"attn BH={bh} T={t} D={d}: " + " ".join(f"{n} {v:.1f}us" for n, v in r.items()), flush=True)
