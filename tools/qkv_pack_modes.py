"""Step time of the bench's BERT layer for each way of producing the Q/K/V^T planes."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2604_03957_b200 as B

dev = torch.device("cuda")
stream = torch.cuda.Stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for mode in ("overlap", "overlap_sep", "group2", "separate", "group3"):
    W = bench.bert_layer(B, dev, qkv_packs=mode)
    W["step"]()
    torch.cuda.synchronize()
    g = bench.graph_of(W["step"], stream)
    ts = bench.time_graph(g, flush, 40, 5, stream)
    print(f"{mode:12s} step {statistics.median(ts) * 1e3:6.1f} us", flush=True)
    del W, g
