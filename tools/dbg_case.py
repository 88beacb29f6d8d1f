import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, bwta_inputs as gen, oracle, paper_2604_03957_b200 as B
def st(t):
    t = t.detach().cpu().contiguous(); return t.view(torch.int16).numpy().view(np.uint16)
for (m, n, k) in [(64, 300, 1000), (64, 300, 768), (64, 256, 128), (128, 256, 1024), (64, 300, 1024), (256, 300, 1000)]:
    x = gen.activations((m, k), 5); w = gen.weights(n, k, 6)
    a = B.bwta_pack_act(x.cuda(), 1.6); wp = B.bwta_pack_weight(w.cuda())
    y = B.bwta_gemm(a, wp, None, 1.0, out_dtype=torch.int32, design="tcgen05").cpu().numpy()
    d = oracle.dot(oracle.quantize_act(st(x), "f16", 1.6, "ternary"), oracle.binarize_weight(st(w), "f16"), threads=8)
    bad = np.argwhere(y != d)
    print((m, n, k), "bad", len(bad), bad[:5].tolist(), (y - d)[tuple(bad[:5].T)].tolist() if len(bad) else "")
