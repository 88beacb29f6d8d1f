"""Timeline of one tcgen05 GEMM launch (CTAs 0/1) from the BWTA_TRACE build.
    BWTA_LIB=libbwta_trace.so python tools/trace_gemm.py M K N"""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, bwta_inputs as gen, paper_2604_03957_b200 as B
m, k, n = (int(v) for v in sys.argv[1:4])
x = gen.activations((m, k), 1).cuda(); w = gen.weights(n, k, 2).cuda()
a = B.bwta_pack_act(x, 1.6); wp = B.bwta_pack_weight(w)
y = torch.empty((m, n), dtype=torch.float16, device="cuda")
buf = np.zeros((2, 14, 1024), np.uint64); cnt = np.zeros((2, 14), np.int32)
f = B.lib.bwta_trace_fetch
for it in range(3):
    torch.cuda.synchronize(); f(buf.ctypes.data, cnt.ctypes.data)
    B.bwta_gemm(a, wp, None, 1.0, out=y, design="tcgen05"); torch.cuda.synchronize()
    f(buf.ctypes.data, cnt.ctypes.data)
names = ["start", "tma", "unpackB_in", "unpackB_out", "mma", "epi_in", "epi_out", "end", "unpackA_in", "unpackA_out", "a_lds", "a_wait_st_done", "a_st_issued", "b_math_done"]
for c in range(2):
    t0 = buf[c][0][0]   # per-CTA clock64 origin (SM-local counters)
    print(f"CTA {c}: counts", dict(zip(names, cnt[c].tolist())))
    for r, nm in enumerate(names):
        v = (buf[c][r][:min(cnt[c][r], 1024)].astype(np.int64) - int(t0)) / 1965.0  # cycles -> us at 1965 MHz
        if len(v): print(f"  {nm:10s}", " ".join(f"{x:7.2f}" for x in np.sort(v)[:40]))
