"""DEV A/B (historical, needs a build with the BWTA_SWAP switch): tile-kernel operand orientation on
plain GEMMs -- auto vs forced no-swap vs forced swap (in-graph)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bwta_inputs as gen, paper_2604_03957_b200 as B
from quick_bench_util import time_graph
shapes = [(4096, 768, 2304, "ternary"), (4096, 768, 768, "ternary"), (4096, 768, 3072, "ternary"), (4096, 3072, 768, "bool"), (2048, 4096, 4096, "ternary"), (2048, 4096, 11008, "ternary")]
gem = []
for (m, k, n, kind) in shapes:
    x = (gen.relu_activations if kind == "bool" else gen.activations)((m, k), 1).cuda(); w = gen.weights(n, k, 2).cuda()
    gem.append((B.bwta_pack_act(x, 1.6, kind), B.bwta_pack_weight(w), torch.empty((m, n), dtype=torch.float16, device="cuda")))
for mode in (None, "0", "1"):
    if mode is None: os.environ.pop("BWTA_SWAP", None)
    else: os.environ["BWTA_SWAP"] = mode
    print({None: "auto   ", "0": "no swap", "1": "swap   "}[mode], " ".join(f"{time_graph(lambda: B.bwta_gemm(a, wp, None, 1.0, out=y)) * 1e3:7.2f}" for a, wp, y in gem), flush=True)
