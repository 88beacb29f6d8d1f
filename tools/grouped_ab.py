"""configs[2] step as two GEMMs vs one GEMM over the row-concatenated weights [W_4096; W_11008]
(outputs = column blocks of one [2048 x 15104] Y): graph of 10 x [L2 flush, step] minus graph of
10 x [L2 flush]; cuBLAS FP16 the same two ways."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bwta_inputs as gen
import paper_2604_03957_b200 as B
from quick_bench_util import time_graph

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
fl = lambda: flush.view(torch.int64).max()
t_fl = time_graph(fl, reps=10)
M, K, Ns = 2048, 4096, (4096, 11008)
X = gen.activations((M, K), 303).cuda()
s_x = gen.act_scale(X)
ws = [gen.weights(n, K, 304 + i) for i, n in enumerate(Ns)]
stats = [gen.weight_stats(w) for w in ws]
wps = [B.bwta_pack_weight(w.cuda(), mu=mu) for w, (mu, _) in zip(ws, stats)]
sws = [s.cuda() for _, s in stats]
ys = [torch.empty((M, n), dtype=torch.float16, device="cuda") for n in Ns]
# concatenated: per-row mu -> a per-row mu vector keeps each block's own mu
mu_cat = torch.cat([torch.full((n,), float(mu), dtype=torch.float32) for n, (mu, _) in zip(Ns, stats)]).cuda()
wcat = B.bwta_pack_weight(torch.cat(ws).cuda(), mu=mu_cat)
swcat = torch.cat(sws)
ycat = torch.empty((M, sum(Ns)), dtype=torch.float16, device="cuda")
st = {}


def sep():
    st["xq"] = B.bwta_pack_act(X, s_x)
    for wp, sw, y in zip(wps, sws, ys):
        B.bwta_gemm(st["xq"], wp, sw, s_x, out=y)


def grp():
    st["xq"] = B.bwta_pack_act(X, s_x)
    B.bwta_gemm(st["xq"], wcat, swcat, s_x, out=ycat)


sep()
grp()
torch.cuda.synchronize()
assert torch.equal(ycat[:, :Ns[0]], ys[0]) and torch.equal(ycat[:, Ns[0]:], ys[1]), "grouped != separate"
ops = sum(2 * M * n * K for n in Ns)
for name, f in (("separate", sep), ("grouped", grp)):
    t = (time_graph(lambda: (fl(), f()), reps=10) - t_fl) * 1e3
    print(f"{name}: {t:.2f} us/step = {ops / t / 1e6:.0f} TOPS", flush=True)
Xh = X.half()
w16 = [w.cuda().half() for w in ws]
w16cat = torch.cat(w16)
t1 = (time_graph(lambda: (fl(), [torch.nn.functional.linear(Xh, w) for w in w16]), reps=10) - t_fl) * 1e3
t2 = (time_graph(lambda: (fl(), torch.nn.functional.linear(Xh, w16cat)), reps=10) - t_fl) * 1e3
print(f"cuBLAS fp16 separate {t1:.2f} us, concatenated {t2:.2f} us", flush=True)
