"""Run one op of the bench's bert_layer step inside a cudaProfilerStart/Stop window
(for `ncu --profile-from-start off`): python tools/prof_op.py gemm_qkv"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench, paper_2604_03957_b200 as B
W = bench.bert_layer(B, torch.device("cuda"))
W["step"]()
torch.cuda.synchronize()
op = {o.name: o for o in W["ops"]}[sys.argv[1]]
torch.cuda.cudart().cudaProfilerStart()
op.fn()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
