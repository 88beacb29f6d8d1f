import sys, os
sys.path.insert(0, os.getcwd())
import torch, bwta_inputs as gen, paper_2604_03957_b200 as B
x = gen.activations((4096, 768), 1).cuda(); w = gen.weights(2304, 768, 2).cuda()
a = B.bwta_pack_act(x, 1.6); wp = B.bwta_pack_weight(w)
for _ in range(3):
    B.bwta_gemm_pack_qkv(a, wp, None, 0.01, 32, 128, 12, 64, (0.5, 0.5, 0.5))
torch.cuda.synchronize()
