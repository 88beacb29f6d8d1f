"""Fixed vs per-k-block vs per-tile cost of the tcgen05 GEMM (device time)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bwta_inputs as gen, paper_2604_03957_b200 as B
from bench import op_time_ms
s = torch.cuda.Stream(); flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def run(m, k, n, out_dtype=torch.float16):
    x = gen.activations((m, k), 1).cuda(); w = gen.weights(n, k, 2).cuda()
    a = B.bwta_pack_act(x, 1.6); wp = B.bwta_pack_weight(w)
    y = torch.empty((m, n), dtype=out_dtype, device="cuda")
    return op_time_ms(lambda: B.bwta_gemm(a, wp, None, 1.0, out=y, design="tcgen05"), flush, s) * 1e3
for (m, k, n) in [(128, 128, 256), (256, 128, 256), (256, 1024, 256), (256, 4096, 256), (2048, 128, 2304), (2048, 768, 2304),
                  (2048, 3072, 2304), (4096, 128, 2304), (4096, 768, 2304), (1024, 4096, 4096), (2048, 4096, 4096)]:
    t = run(m, k, n); ti = run(m, k, n, torch.int32)
    print(f"M={m:5d} K={k:5d} N={n:5d}: {t:7.2f} us  (i32 out {ti:7.2f})  {2*m*n*k/t/1e6:7.0f} TOPS")
