"""Variants of the bench step (FFN1 fused pack on/off, Q/K/V^T pack grouping),
CUDA graphs timed alternately in one process."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2604_03957_b200 as B

dev = torch.device("cuda")
stream = torch.cuda.Stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
variants = {"fused+group3": dict(fuse_ffn=True, qkv_packs="group3"),
            "fused+group2": dict(fuse_ffn=True, qkv_packs="group2"),
            "fused+separate": dict(fuse_ffn=True, qkv_packs="separate"),
            "unfused+group2": dict(fuse_ffn=False, qkv_packs="group2")}
graphs = {}
for name, kw in variants.items():
    W = bench.bert_layer(B, dev, **kw)
    ops = W["ops"]
    graphs[name] = (bench.graph_of(lambda ops=ops: [o.fn() for o in ops], stream), W)
for rnd in range(3):
    for name in variants:
        ts = bench.time_graph(graphs[name][0], flush, 30, 5, stream)
        print(f"round {rnd} {name:16s}: {statistics.median(ts) * 1e3:.1f} us", flush=True)
