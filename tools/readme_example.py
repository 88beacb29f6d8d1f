"""The README usage example, runnable: python tools/readme_example.py"""
import sys; import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2604_03957_b200 as B
x = torch.randn(2048, 4096, dtype=torch.float16, device="cuda")
w = torch.randn(11008, 4096, dtype=torch.float16, device="cuda") * 0.02
s_a = 2 * x.abs().mean().item()
wp = B.bwta_pack_weight(w, mu=w.float().mean().item())
a = B.bwta_pack_act(x, s_a, "ternary")
y = B.bwta_gemm(a, wp, w_scale=None, a_scale=s_a)
torch.cuda.synchronize(); print("snippet ok", tuple(y.shape), y.dtype)
