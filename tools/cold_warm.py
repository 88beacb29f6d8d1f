"""Where the cold-L2 time of the C3 GEMMs goes: the same bwta_gemm timed
(a) back to back in one CUDA graph (warm L2, PDL overlap of prologue and tail),
(b) single launch after an L2 flush (the bench's per-op condition),
(c) single launch, L2 warm (operands read by the previous run), no predecessor overlap,
(d) single launch after a flush followed by a torch read of exactly the operands (warm operands,
    the rest of L2 holds the flush buffer)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bwta_inputs as gen
import paper_2604_03957_b200 as B
from quick_bench_util import time_graph, timeit

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for (m, k, n) in [(2048, 4096, 4096), (2048, 4096, 11008)]:
    x = gen.activations((m, k), 1).cuda()
    w = gen.weights(n, k, 2).cuda()
    s_a = gen.act_scale(x)
    mu, s_w = gen.weight_stats(w)
    s_w = s_w.cuda()
    a = B.bwta_pack_act(x, s_a)
    wp = B.bwta_pack_weight(w, mu=mu)
    y = torch.empty((m, n), dtype=torch.float16, device="cuda")
    fn = lambda: B.bwta_gemm(a, wp, s_w, s_a, out=y)
    ops = 2 * m * n * k
    ta = time_graph(fn) * 1e3
    tb = timeit(fn, flush=flush) * 1e3
    tc = timeit(fn) * 1e3

    def touch():
        flush.view(torch.int64).max()
        for t in (a.sgn, a.nz, wp.sgn):
            t.view(torch.int32).max()
    # (d): flush, then read the operands, then the GEMM (timed alone)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        touch()
        torch.cuda._sleep(300000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    td = ts[len(ts) // 2] * 1e3
    # (e) the bench's per-op condition: graph of 20 x [flush, gemm] minus graph of 20 x [flush]
    fl = lambda: flush.view(torch.int64).max()
    te = (time_graph(lambda: (fl(), fn()), reps=10) - time_graph(fl, reps=10)) * 1e3
    # (f) in-graph: flush, torch read of the operands, gemm  minus  flush, torch read
    rd = lambda: [t.view(torch.int32).max() for t in (a.sgn, a.nz, wp.sgn)]
    tf = (time_graph(lambda: (fl(), rd(), fn()), reps=10) - time_graph(lambda: (fl(), rd()), reps=10)) * 1e3
    print(f"  in-graph flush+operands-read {tf:.2f}us ({ops/tf/1e6:.0f}T)")
    # (g) in-graph: flush, zero Y (Y's lines resident and dirty), gemm; (h) write another buffer of Y's size
    zy = lambda: y.zero_()
    tg = (time_graph(lambda: (fl(), zy(), fn()), reps=10) - time_graph(lambda: (fl(), zy()), reps=10)) * 1e3
    y2 = torch.empty_like(y)
    z2 = lambda: y2.zero_()
    th = (time_graph(lambda: (z2(), fn()), reps=10) - time_graph(z2, reps=10)) * 1e3
    print(f"  in-graph flush+zero(Y) {tg:.2f}us   in-graph zero(other {y.numel()*2/1e6:.0f} MB) {th:.2f}us")
    print(f"{m}x{k}x{n} (BWTA_L2_PREFETCH={os.environ.get('BWTA_PF_KB', 'default')}): graph-flushed {te:.2f}us ({ops/te/1e6:.0f}T)  graph-warm {ta:.2f}us ({ops/ta/1e6:.0f}T)  flushed {tb:.2f}us ({ops/tb/1e6:.0f}T)  "
          f"single-warm {tc:.2f}us ({ops/tc/1e6:.0f}T)  flush+operands-read {td:.2f}us ({ops/td/1e6:.0f}T)", flush=True)
