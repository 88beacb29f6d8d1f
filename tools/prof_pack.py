import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bwta_inputs as gen, paper_2604_03957_b200 as B
x = gen.activations((2048, 4096), 1).cuda()
qkv = gen.activations((4096, 2304), 2).cuda()
v = qkv[:, 1536:].view(32, 128, 12, 64).transpose(1, 2)
q = qkv[:, :768].view(32, 128, 12, 64).transpose(1, 2)
for _ in range(3):
    B.bwta_pack_act(x, 1.6)
    B.bwta_pack_act(q, 1.6)
    B.bwta_pack_act(v, 1.6, transpose=True)
torch.cuda.synchronize()
