"""Timeline of one tcgen05 GEMM launch (CTAs 0 and 1) from the -DBWTA_TRACE build.

    python paper_2604_03957_b200/build.py --trace
    BWTA_LIB=libbwta_trace.so python tools/trace_gemm.py M K N [ternary|bool]

Prints, per CTA, the clock64 (SM cycles, relative to the CTA's first event)
of every hook in gemm_tc.cu, and per-k-block intervals for the first tile."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bwta_inputs as gen
import paper_2604_03957_b200 as B

if sys.argv[1] == "qkvpack":   # BERT QKV projection emitting the per-head Q/K/V^T planes
    x = gen.activations((4096, 768), 1).cuda()
    w = gen.weights(2304, 768, 2).cuda()
    a = B.bwta_pack_act(x, 1.6)
    wp = B.bwta_pack_weight(w)
    run = lambda: B.bwta_gemm_pack_qkv(a, wp, None, 0.01, 32, 128, 12, 64, (0.5, 0.5, 0.5))
elif sys.argv[1] == "qk":   # attention QK^T: qk BH T D
    bh, t, d = (int(v) for v in sys.argv[2:5])
    qp = B.bwta_pack_act(torch.randn(bh, t, d, device="cuda", dtype=torch.float16), 1.6)
    kp = B.bwta_pack_act(torch.randn(bh, t, d, device="cuda", dtype=torch.float16), 1.6)
    s_ = torch.empty(bh, t, t, device="cuda", dtype=torch.float16)
    run = lambda: B.bwta_attn_qk(qp, kp, 0.1, out=s_, design="tcgen05")
else:
    m, k, n = (int(v) for v in sys.argv[1:4])
    kind = sys.argv[4] if len(sys.argv) > 4 else "ternary"
    x = gen.activations((m, k), 1).cuda()
    if kind == "bool":
        x = torch.relu(x)
    w = gen.weights(n, k, 2).cuda()
    a = B.bwta_pack_act(x, 1.6, kind=kind)
    wp = B.bwta_pack_weight(w)
    y = torch.empty((m, n), dtype=torch.float16, device="cuda")
    tile = tuple(int(v) for v in os.environ["BWTA_TILE"].split(",")) if os.environ.get("BWTA_TILE") else None
    run = lambda: B.bwta_gemm(a, wp, None, 1.0, out=y, design="tcgen05", tile=tile)
buf = np.zeros((2, 16, 64), np.uint64)
f = B.lib.bwta_trace_fetch
for it in range(3):
    torch.cuda.synchronize()
    f(buf.ctypes.data)
    run()
    torch.cuda.synchronize()
    f(buf.ctypes.data)
cnt = (buf != 0).sum(-1)
names = ["start", "tma_issue", "unp_full", "unp_done", "mma_bready", "epi_tfull", "epi_done", "end_work", "exit",
         "e_ld", "unpA_full", "unpA_done", "mma_pre", "mma_post", "unpA_math", "unpA_empty"]
for c in range(2):
    t0 = int(buf[c][0][0])
    print(f"CTA {c}: counts", dict(zip(names, cnt[c][:len(names)].tolist())))
    ev = {}
    for r, nm in enumerate(names):
        v = buf[c][r].astype(np.int64)
        v = v[buf[c][r] != 0] - t0
        ev[nm] = v
        if len(v):
            print(f"  {nm:11s}", " ".join(f"{x:6d}" for x in v[:24]))
    for a_, b_ in (("tma_issue", "unp_full"), ("unp_full", "unp_done"), ("unp_done", "mma_bready"),
                   ("tma_issue", "unpA_full"), ("unpA_full", "unpA_done"), ("unpA_done", "mma_bready"), ("mma_pre", "mma_bready"), ("mma_bready", "mma_post"), ("unpA_full", "unpA_math"), ("unpA_math", "unpA_empty"), ("unpA_empty", "unpA_done")):
        if len(ev[a_]) and len(ev[b_]):
            n_ = min(len(ev[a_]), len(ev[b_]))
            print(f"  {a_}->{b_}: median {np.median(ev[b_][:n_] - ev[a_][:n_]):.0f} cycles")
    for nm in ("tma_issue", "unp_done", "unpA_full", "unpA_done", "mma_pre", "mma_bready", "mma_post"):
        if len(ev[nm]) > 2:
            print(f"  {nm} period: median {np.median(np.diff(ev[nm])):.0f} cycles")
