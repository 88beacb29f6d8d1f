"""Run the bert_layer step a few times (for ncu launch lists / captures)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench, paper_2604_03957_b200 as B
W = bench.bert_layer(B, torch.device("cuda"))
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    for op in W["ops"]:
        op.fn()
torch.cuda.synchronize()
