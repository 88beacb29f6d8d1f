import sys, os
sys.path.insert(0, os.getcwd())
exec(open('tools/pack_bench.py').read().split("cases = [")[0])
cases = [("Q", lambda: B.bwta_pack_act(hv(0), 1.6)),
         ("Q,K separate", lambda: (B.bwta_pack_act(hv(0), 1.6), B.bwta_pack_act(hv(1), 1.6))),
         ("Q+K group", lambda: B.bwta_pack_act_batch([(hv(0), 1.6, "ternary", False), (hv(1), 1.6, "ternary", False)])),
         ("V^T", lambda: B.bwta_pack_act(hv(2), 1.6, transpose=True)),
         ("V^T+V^T group", lambda: B.bwta_pack_act_batch([(hv(2), 1.6, "ternary", True), (hv(2), 1.6, "ternary", True)])),
         ("Q,K,V^T separate", lambda: (B.bwta_pack_act(hv(0), 1.6), B.bwta_pack_act(hv(1), 1.6), B.bwta_pack_act(hv(2), 1.6, transpose=True))),
         ("Q+K+V^T group", lambda: B.bwta_pack_act_batch([(hv(0), 1.6, "ternary", False), (hv(1), 1.6, "ternary", False), (hv(2), 1.6, "ternary", True)])),
         ("X+X+X group", lambda: B.bwta_pack_act_batch([(xb, 1.6, "ternary", False)] * 3)),
         ("X,X,X separate", lambda: [B.bwta_pack_act(xb, 1.6) for _ in range(3)])]
for name, fn in cases:
    print(f"{name:20s} write-flush {per_op(fn, 'write'):6.2f}us  no-flush {per_op(fn, 'none'):6.2f}us", flush=True)
