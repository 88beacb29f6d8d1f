"""Which part of the per-head packs is slow: strided head views vs contiguous
tensors of the same row length, padding words, transposed vs row mode."""
import os
import sys

sys.path.insert(0, os.getcwd())
exec(open('tools/pack_bench.py').read().split("cases = [")[0])
qc = qkv[:, :768].contiguous().view(32, 128, 12, 64).transpose(1, 2).contiguous()   # [32,12,128,64] dense
q2 = qc.view(-1, 128)                                                                 # 128-element rows
cases = [("Q head view [32,12,128,64] strided", lambda: B.bwta_pack_act(hv(0), 1.6)),
         ("Q dense [32,12,128,64]", lambda: B.bwta_pack_act(qc, 1.6)),
         ("same bytes as [24576,128]", lambda: B.bwta_pack_act(q2, 1.6)),
         ("X [4096,768]", lambda: B.bwta_pack_act(xb, 1.6)),
         ("V^T head view strided", lambda: B.bwta_pack_act(hv(2), 1.6, transpose=True)),
         ("V^T dense [32,12,128,64]", lambda: B.bwta_pack_act(qc, 1.6, transpose=True)),
         ("X^T [4096,768] transposed", lambda: B.bwta_pack_act(xb, 1.6, transpose=True))]
for name, fn in cases:
    print(f"{name:38s} write-flush {per_op(fn, 'write'):6.2f}us  no-flush {per_op(fn, 'none'):6.2f}us", flush=True)
