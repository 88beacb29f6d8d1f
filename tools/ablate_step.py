"""Marginal in-graph cost of each op of the bench step: time the CUDA graph of
the whole step and of the step minus one op (its outputs stay from a full
run), L2 flushed before each replay.  python tools/ablate_step.py"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2604_03957_b200 as B

dev = torch.device("cuda")
W = bench.bert_layer(B, dev)
ops = W["ops"]
stream = torch.cuda.Stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for op in ops:
    op.fn()
torch.cuda.synchronize()


def t_of(fns, reps=30):
    g = bench.graph_of(lambda: [f() for f in fns], stream)
    ts = bench.time_graph(g, flush, reps, 5, stream)
    return statistics.median(ts) * 1e3


full = t_of([o.fn for o in ops])
print(f"full step {full:.1f} us")
for i, op in enumerate(ops):
    t = t_of([o.fn for j, o in enumerate(ops) if j != i])
    print(f"  without {op.name:10s} {t:6.1f} us  -> marginal {full - t:5.1f} us")
