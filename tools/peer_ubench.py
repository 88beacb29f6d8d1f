"""Cost of the fused gather's flag barrier (bwta_peer_barrier) on one GPU: graphs of R barriers
alone, R GEMMs, R x (GEMM + barrier) -> per-call device time."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0] + "/tests")
import bwta_inputs as gen  # noqa: E402
import paper_2604_03957_b200 as B  # noqa: E402


def graph_ms(fn, reps=50):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            fn()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            g.replay()
            e1.record(s)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / reps * 1e3)
    return best


flags = torch.zeros(64, dtype=torch.int32, device="cuda")
M, K = 2048, 4096
x = gen.activations((M, K), 1).cuda()
a = B.bwta_pack_act(x, 0.5)
for N in (4096, 11008, 1376):
    w = gen.weights(N, K, 2).cuda()
    wp = B.bwta_pack_weight(w)
    y = torch.empty((N, M), dtype=torch.float16, device="cuda")
    bar = lambda: B.bwta_peer_barrier([flags.data_ptr()], 0, flags.data_ptr() + 128)
    gem = lambda: B.bwta_gemm(a, wp, None, 0.5, y_transposed=True, out=y)
    gp = lambda: B.bwta_gemm_peers(a, wp, None, 0.5, y.data_ptr(), M, [])
    both = lambda: (gp(), bar())
    print(f"N={N}: barrier {graph_ms(bar):.2f} us, gemm {graph_ms(gem):.2f} us, gemm_peers {graph_ms(gp):.2f} us, "
          f"gemm_peers+barrier {graph_ms(both):.2f} us")
