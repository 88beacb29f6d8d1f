"""Pack kernels vs a plain torch copy of the same input (device time, graphs).
Per-op time = (graph of R x [flush, op] - graph of R x [flush]) / R, so the
graph-launch latency is amortised; two flush styles: write (zero_) and read (sum)."""
import sys, os, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bwta_inputs as gen, paper_2604_03957_b200 as B
s = torch.cuda.Stream(); fbuf = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
def graph(fn):
    with torch.cuda.stream(s): fn()
    torch.cuda.synchronize(); g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s): fn()
    return g
def tg(g, n=10):
    ts = []
    for _ in range(n):
        with torch.cuda.stream(s):
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(s); g.replay(); b.record(s)
        torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return statistics.median(ts)
R = 20
def per_op(fn, style):
    fl = (lambda: fbuf.zero_()) if style == "write" else ((lambda: fbuf.sum()) if style == "read" else (lambda: fbuf[:1].zero_()))
    def rep():
        for _ in range(R): fl(); fn()
    def fonly():
        for _ in range(R): fl()
    return (tg(graph(rep)) - tg(graph(fonly))) / R * 1e3
x3 = gen.activations((2048, 4096), 1).cuda(); xb = gen.activations((4096, 768), 2).cuda()
qkv = gen.activations((4096, 2304), 3).cuda(); P = gen.attention_probs((32, 12, 128, 128), 4).cuda()
Rr = gen.relu_activations((4096, 3072), 5).cuda(); Pc4 = gen.attention_probs((1, 32, 2048, 2048), 6).cuda()
v4 = gen.activations((1, 32, 2048, 128), 7).cuda()
hv = lambda j: qkv[:, j*768:(j+1)*768].view(32, 128, 12, 64).transpose(1, 2)
cases = [("C3 X 2048x4096", x3, lambda: B.bwta_pack_act(x3, 1.6)),
         ("C2 X 4096x768", xb, lambda: B.bwta_pack_act(xb, 1.6)),
         ("C2 Q heads view", hv(0), lambda: B.bwta_pack_act(hv(0), 1.6)),
         ("C2 V^T heads view", hv(2), lambda: B.bwta_pack_act(hv(2), 1.6, transpose=True)),
         ("C2 Q+K+V^T one launch", qkv, lambda: B.bwta_pack_act_batch([(hv(0), 1.6, "ternary", False),
                                                                         (hv(1), 1.6, "ternary", False),
                                                                         (hv(2), 1.6, "ternary", True)])),
         ("C2 P bool", P, lambda: B.bwta_pack_act(P, 2/128, "bool")),
         ("C2 R bool 4096x3072", Rr, lambda: B.bwta_pack_act(Rr, 0.8, "bool")),
         ("C4 P bool 32x2048^2", Pc4, lambda: B.bwta_pack_act(Pc4, 2/2048, "bool")),
         ("C4 V^T 32x2048x128", v4, lambda: B.bwta_pack_act(v4, 1.6, transpose=True))]
for name, x, fn in cases:
    nb = x.numel() * 2
    out = []
    for style in ("write", "none"):
        tp = per_op(fn, style); tc = per_op(lambda: x.clone(), style)
        out.append(f"[{style}-flush] pack {tp:6.2f}us {nb*1.125/tp/1e3:5.0f}GB/s clone {tc:6.2f}us {2*nb/tc/1e3:5.0f}GB/s")
    print(f"{name:22s} {nb/1e6:6.1f}MB " + " | ".join(out))
x = torch.zeros(1, device="cuda")
print("tiny kernel:", per_op(lambda: x.add_(1), "read"), "us")
