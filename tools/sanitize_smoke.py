"""Small calls of every entry point, for compute-sanitizer (memcheck / racecheck / initcheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bwta_inputs as gen
import paper_2604_03957_b200 as B

x = gen.activations((130, 300), 1).cuda()
w = gen.weights(200, 300, 2).cuda()
a = B.bwta_pack_act(x, 1.6)
ab = B.bwta_pack_act(torch.relu(x), 1.6, "bool")
wp = B.bwta_pack_weight(w)
for d in ("cuda_core", "tcgen05"):
    B.bwta_gemm(a, wp, None, 1.0, design=d)
    B.bwta_gemm(ab, wp, None, 1.0, design=d, y_transposed=True)
    B.bwta_gemm(a, wp, None, 1.0, design=d, out_dtype=torch.int32)
q = gen.activations((2, 3, 37, 64), 3).cuda()
k = gen.activations((2, 3, 41, 64), 4).cuda()
v = gen.activations((2, 3, 41, 64), 5).cuda()
p = gen.attention_probs((2, 3, 37, 41), 6).cuda()
qp, kp = B.bwta_pack_act(q, 1.6), B.bwta_pack_act(k, 1.6)
vt = B.bwta_pack_act(v, 1.6, transpose=True)
pp = B.bwta_pack_act(p, 0.05, "bool")
g = B.bwta_pack_act_batch([(q, 1.6, "ternary", False), (v, 1.6, "ternary", True)])
for d in ("cuda_core", "tcgen05"):
    B.bwta_attn_qk(qp, kp, 0.1, design=d)
    B.bwta_attn_pv(pp, vt, 0.1, design=d)
B.bwta_gemm_pack(a, wp, None, 1.0, 0.5, "bool")
# the lean grouped row pack (Q + K of the BERT step) and the kind-specialised BN = 192 CTA-pair tiles
B.bwta_pack_act_batch([(q, 1.6, "ternary", False), (k, 1.3, "ternary", False)])
x2 = gen.activations((300, 517), 12).cuda()
w2 = B.bwta_pack_weight(gen.weights(400, 517, 13).cuda())
for kind in ("ternary", "bool"):
    a2 = B.bwta_pack_act(torch.relu(x2) if kind == "bool" else x2, 1.6, kind)
    B.bwta_gemm(a2, w2, None, 1.0, tile=(192, 2))
    B.bwta_gemm_pack(a2, w2, None, 1.0, 0.5, "ternary", tile=(192, 2))
B.bwta_attn_pv_pack(pp, vt, 0.1, 0.5, "ternary")
# decode paths: CUDA-core GEMV (M <= 4), skinny tcgen05 (M <= 32), fused pack GEMV, fused attention
for m in (1, 3, 16):
    xd = gen.activations((m, 1000), 7 + m).cuda()
    wd = B.bwta_pack_weight(gen.weights(300, 1000, 8).cuda())
    B.bwta_gemm(B.bwta_pack_act(xd, 1.6), wd, None, 1.0)
    B.bwta_gemm(B.bwta_pack_act(xd, 1.6), wd, None, 1.0, y_transposed=True, out_dtype=torch.float32)
    if m <= 4:
        B.bwta_gemm_x(xd, 1.6, wd, None)
q1 = B.bwta_pack_act(gen.activations((2, 3, 1, 64), 9).cuda(), 1.6)
kd = B.bwta_pack_act(gen.activations((2, 3, 300, 64), 10).cuda(), 1.6)
vd = B.bwta_pack_act(gen.activations((2, 3, 300, 64), 11).cuda(), 1.6, transpose=True)
B.bwta_attn_decode(q1, kd, vd, 0.1, 2.0 / 300, 0.01, return_p=True)
torch.cuda.synchronize()
print("ok")
# round-2 entry points: fused prefill attention (+ context pack), QKV head-split pack, W1A1, b1 prior art
qp2 = B.bwta_pack_act(gen.activations((2, 3, 130, 64), 20).cuda(), 1.6)
kp2 = B.bwta_pack_act(gen.activations((2, 3, 150, 64), 21).cuda(), 1.6)
vt2 = B.bwta_pack_act(gen.activations((2, 3, 150, 64), 22).cuda(), 1.6, transpose=True)
B.bwta_attn_prefill(qp2, kp2, vt2, 0.1, 2.0 / 150, 0.01, return_p=True)
B.bwta_attn_prefill_pack(qp2, kp2, vt2, 0.1, 2.0 / 150, 0.01, 0.5)
xq = B.bwta_pack_act(gen.activations((128, 300), 23).cuda(), 1.6)
wq = B.bwta_pack_weight(gen.weights(3 * 2 * 64, 300, 24).cuda())
B.bwta_gemm_pack_qkv(xq, wq, None, 1.0, 2, 64, 2, 64, (0.5, 0.5, 0.5))
ab = B.bwta_pack_act(x, 1.6, "binary")
for d in ("auto", "cuda_core", "mma_b1"):
    B.bwta_gemm(ab, wp, None, 1.0, design=d)
B.bwta_attn_pv(pp, B.bwta_pack_act(v, 1.0, "binary", transpose=True), 0.1)
torch.cuda.synchronize()
print("ok2")
