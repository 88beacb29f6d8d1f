"""bench.py -- BWTA hot path on B200: effective TOPS of the BWTA matmuls (and
bitpack GB/s) against cuBLAS FP16 on the same GPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl bwta|reference]
                    [--workload llama_prefill|bert_layer|llama_attn|bert_linear|...]

Metric (BASELINE.json): "BWTA GEMM effective TOPS and speedup vs cuBLAS FP16 on
B200; bitpack HBM GB/s".  Effective TOPS = 2*M*N*K / t (the paper's
convention), summed over every BWTA matmul of one step.

Default workload = BASELINE.json configs[2], the north star's target and the
largest single-GPU config: the LLaMA-7B prefill linears (M = 2048 tokens,
K = 4096, N = 4096 and 11008).  A step runs the hot path once over one batch:
the ternary pack of X (A1), then both BWTA linears (A4 + A5) on the packed X.
At N > 1 GPUs (torchrun, one process per GPU, NCCL) the same step is
N-sharded (A8): every rank packs its replica of X, computes its output
channels in chunks and all-gathers them (in place, overlapped with the next
chunk's GEMM) so every rank ends with the full Y^T; total work is fixed
("scaling": "strong").  `--workload bert_layer` (configs[1]) runs one BERT-base
layer (every §8(a) row incl. attention); at N > 1 it runs replicas (weak).

Timing: each step is one CUDA-graph replay of the library calls (N = 1;
eager launches at N > 1, where the step holds NCCL collectives), bracketed by
CUDA events on the launching stream; a 256 MiB buffer (> 126 MB L2) is read
between steps (outside the events), so every step starts L2-cold; time = max
over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bwta_inputs as gen  # noqa: E402

METRIC = "BWTA GEMM effective TOPS and speedup vs cuBLAS FP16 on B200; bitpack HBM GB/s"
UNIT = "TOPS"


# ----------------------------------------------------------------------------- utils
def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return None


def peaks():
    mp = measured_peaks()
    if mp:
        return {"hbm_gbs": mp["hbm_gbs"], "bf16_tflops": mp["bf16_tflops"],
                "bf16_tflops_sustained": mp.get("bf16_tflops_sustained"), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True,
                                         bufsize=1)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def graph_of(fn, stream, pre=None):
    """Capture fn (after one eager warm-up run) into a CUDA graph; pre() runs on the host before
    each of the two calls (e.g. to select which output buffer the captured call uses)."""
    with torch.cuda.stream(stream):
        if pre:
            pre()
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    if pre:
        pre()
    with torch.cuda.graph(g, stream=stream):
        fn()
    torch.cuda.synchronize()
    return g


def _trimmed_mean(v):
    """Mean of the middle 80 % of the samples: CUDA event timestamps inside a graph step in ~1 us
    quanta, so a median of a few tens of samples is quantized; the trimmed mean resolves below
    the quantum and still drops outliers."""
    v = sorted(v)
    k = len(v) // 10
    v = v[k:len(v) - k] if len(v) > 2 * k else v
    return sum(v) / len(v)


def flush_l2(buf):
    """Evict L2 by READING a buffer 2x its size.  A memset flush would leave the
    L2 full of dirty lines whose write-back then lands inside the next timed
    region (measured: +10-20 us on an otherwise HBM-bound kernel)."""
    buf.view(torch.int64).amax()


def time_graph(g, flush, reps, warmup, stream):
    """Median / list of per-replay device times (ms), L2 flushed before each replay.  g: a graph, or
    a runner whose replay() cycles several (the double-buffered fused gather)."""
    ts = []
    with torch.cuda.stream(stream):
        for i in range(warmup + reps):
            flush_l2(flush)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            g.replay()
            e1.record(stream)
            if i >= warmup:
                ts.append((e0, e1))
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in ts]


def op_time_ms(fn, flush, stream, reps=20, trials=5):
    """Device time of one call of fn, L2-cold: a graph of reps x [flush, fn] minus a
    graph of reps x [flush], so the graph-launch latency is amortised away."""
    def body():
        for _ in range(reps):
            flush_l2(flush)
            fn()

    def fl():
        for _ in range(reps):
            flush_l2(flush)
    g1, g0 = graph_of(body, stream), graph_of(fl, stream)
    t1 = statistics.median(time_graph(g1, flush[:8], trials, 1, stream))
    t0 = statistics.median(time_graph(g0, flush[:8], trials, 1, stream))
    return max(t1 - t0, 0.0) / reps


# ----------------------------------------------------------------------------- workloads
class Op:
    def __init__(self, name, kind, fn, ops=0, bytes_=0, cublas=None, launches=1, alts=None):
        self.name, self.kind, self.fn, self.ops, self.bytes, self.cublas = name, kind, fn, ops, bytes_, cublas
        self.launches = launches  # library kernels per call
        self.alts = alts or {}    # the same op through other designs (timed alongside, not in the step)


def bert_layer(B, dev, seed=202, batch=32, seq=128, hidden=768, heads=12, ffn=3072, fuse_ffn=True,
               qkv_packs="overlap", fuse_ctx=True, fused_attn=True, fuse_qkv=True):
    """configs[1]: BERT-base layer, seq 128, batch 32 (M = 4096 tokens)."""
    M, D = batch * seq, hidden // heads
    g = lambda s: s + seed  # noqa: E731
    X = gen.activations((M, hidden), g(0)).to(dev)
    Xf = gen.activations((M, hidden), g(1)).to(dev)          # LayerNorm output stand-in
    P = gen.attention_probs((batch, heads, seq, seq), g(3)).to(dev)  # softmax output stand-in
    Ws = {"qkv": gen.weights(3 * hidden, hidden, g(4)), "o": gen.weights(hidden, hidden, g(5)),
          "f1": gen.weights(ffn, hidden, g(6)), "f2": gen.weights(hidden, ffn, g(7))}
    packed, wsc, w16 = {}, {}, {}
    for k, w in Ws.items():
        mu, s_w = gen.weight_stats(w)
        packed[k] = B.bwta_pack_weight(w.to(dev), mu=mu)      # offline
        wsc[k] = s_w.to(dev)
        w16[k] = w.to(dev)
    s = {"x": gen.act_scale(X), "xf": gen.act_scale(Xf), "att": float(np.float32(2.0 / seq))}
    qkv = torch.empty((M, 3 * hidden), dtype=torch.float16, device=dev)
    S = torch.empty((batch, heads, seq, seq), dtype=torch.float16, device=dev)
    ctx = torch.empty((M, hidden), dtype=torch.float16, device=dev)
    y_o = torch.empty((M, hidden), dtype=torch.float16, device=dev)
    h1 = torch.empty((M, ffn), dtype=torch.float16, device=dev)
    y2 = torch.empty((M, hidden), dtype=torch.float16, device=dev)

    side = torch.cuda.Stream(device=dev)

    def heads_view(t, j):  # [B, H, T, D] view of the j-th third of qkv (no copy)
        return t[:, j * hidden:(j + 1) * hidden].view(batch, seq, heads, D).transpose(1, 2)
    ctx_v = ctx.view(batch, seq, heads, D).transpose(1, 2)

    # calibration pass (outside any timing): scales of Q, K, V and the context
    xq = B.bwta_pack_act(X, s["x"])
    B.bwta_gemm(xq, packed["qkv"], wsc["qkv"], s["x"], out=qkv)
    torch.cuda.synchronize()
    for j, n in enumerate("qkv"):
        s[n] = gen.act_scale(heads_view(qkv, j))
    s["alpha"] = float(np.float32(s["q"] * s["k"] / np.sqrt(D)))
    s["beta"] = float(np.float32(s["att"] * s["v"]))
    st = {}

    def op_pack_x():
        st["xq"] = B.bwta_pack_act(X, s["x"])

    def op_qkv():
        B.bwta_gemm(st["xq"], packed["qkv"], wsc["qkv"], s["x"], out=qkv)

    def op_qkv_pack():  # QKV projection emitting the per-head Q / K / V^T planes (N2; Y never written)
        st["qp"], st["kp"], st["vt"] = B.bwta_gemm_pack_qkv(st["xq"], packed["qkv"], wsc["qkv"], s["x"], batch, seq,
                                                            heads, D, (s["q"], s["k"], s["v"]))

    def op_pack_qkv():  # the per-head Q, K and V^T packs (one launch by default)
        qa, ka, va = ((heads_view(qkv, 0), s["q"], "ternary", False), (heads_view(qkv, 1), s["k"], "ternary", False),
                      (heads_view(qkv, 2), s["v"], "ternary", True))
        if qkv_packs in ("overlap", "overlap_sep"):
            # Q + K packs (one launch, or two) on the step's stream; the V^T pack -- needed only by
            # PV -- on a side stream, so it overlaps the Q/K packs and QK^T (joined before PV)
            cur = torch.cuda.current_stream()
            side.wait_stream(cur)
            if qkv_packs == "overlap":
                st["qp"], st["kp"] = B.bwta_pack_act_batch([qa, ka])
            else:
                st["qp"], st["kp"] = (B.bwta_pack_act(x[0], x[1]) for x in (qa, ka))
            with torch.cuda.stream(side):
                st["vt"] = B.bwta_pack_act(va[0], va[1], transpose=True)
            if st.get("defer_join"):
                st["vt_pending"] = True
            else:
                cur.wait_stream(side)
        elif qkv_packs == "group3":
            st["qp"], st["kp"], st["vt"] = B.bwta_pack_act_batch([qa, ka, va])
        elif qkv_packs == "group2":
            st["qp"], st["kp"] = B.bwta_pack_act_batch([qa, ka])
            st["vt"] = B.bwta_pack_act(va[0], va[1], transpose=True)
        else:
            st["qp"], st["kp"], st["vt"] = (B.bwta_pack_act(x[0], x[1], transpose=x[3]) for x in (qa, ka, va))

    def op_qk():
        B.bwta_attn_qk(st["qp"], st["kp"], s["alpha"], out=S)
        if st.pop("vt_pending", False):
            torch.cuda.current_stream().wait_stream(side)

    def op_pack_p():
        st["pp"] = B.bwta_pack_act(P, s["att"], "bool")

    def op_pv():
        B.bwta_attn_pv(st["pp"], st["vt"], s["beta"], out=ctx_v)

    def op_pv_pack():  # PV emitting the O-projection's ternary input planes (fused pack, no ctx write)
        st["cq"] = B.bwta_attn_pv_pack(st["pp"], st["vt"], s["beta"], s["ctx"], "ternary")

    def op_pack_ctx():
        st["cq"] = B.bwta_pack_act(ctx, s["ctx"])

    def op_attn():  # QK^T -> fp32 softmax -> bool P -> PV in one launch (N3), context into [B, T, H*D]
        if st.pop("vt_pending", False):   # the V^T pack (side stream) joins here
            torch.cuda.current_stream().wait_stream(side)
        B.bwta_attn_prefill(st["qp"], st["kp"], st["vt"], s["alpha"], s["att"], s["beta"], out=ctx_v)

    def op_attn_pack():  # ... with the O-projection's input pack fused into its epilogue (no ctx write)
        if st.pop("vt_pending", False):
            torch.cuda.current_stream().wait_stream(side)
        st["cq"] = B.bwta_attn_prefill_pack(st["qp"], st["kp"], st["vt"], s["alpha"], s["att"], s["beta"], s["ctx"])

    def op_o():
        B.bwta_gemm(st["cq"], packed["o"], wsc["o"], s["ctx"], out=y_o)

    def op_pack_xf():
        st["fq"] = B.bwta_pack_act(Xf, s["xf"])

    def op_f1():  # FFN1 emits FFN2's bool input planes directly (fused pack, no h1 write)
        st["rq"] = B.bwta_gemm_pack(st["fq"], packed["f1"], wsc["f1"], s["xf"], s["r"], "bool")

    def op_f1_unfused():  # the same planes through fp16 h1 + a standalone pack
        B.bwta_gemm(st["fq"], packed["f1"], wsc["f1"], s["xf"], out=h1)

    def op_pack_h1():
        st["rq"] = B.bwta_pack_act(h1, s["r"], "bool")

    def op_f2():
        B.bwta_gemm(st["rq"], packed["f2"], wsc["f2"], s["r"], out=y2)

    op_pack_x(); op_qkv(); op_pack_qkv()  # noqa: E702
    if fused_attn:
        op_attn()
    else:
        op_qk(); op_pack_p(); op_pv()  # noqa: E702
    torch.cuda.synchronize()
    s["ctx"] = gen.act_scale(ctx)   # calibration of the context scale (outside timing)
    # calibration of FFN2's input scale on the (unfused) FFN1 output: s_r = 2 mean relu(h1)
    op_pack_xf()
    B.bwta_gemm(st["fq"], packed["f1"], wsc["f1"], s["xf"], out=h1)
    torch.cuda.synchronize()
    R = torch.relu(h1)              # the post-ReLU FFN activations (cuBLAS baseline input)
    s["r"] = gen.act_scale(R)

    # cuBLAS FP16 baselines of the same matmuls (torch -> cuBLASLt)
    q16, k16, v16 = (heads_view(qkv, j) for j in range(3))
    cub = {
        "qkv": lambda: torch.nn.functional.linear(X, w16["qkv"]),
        "qk": lambda: torch.matmul(q16, k16.transpose(-1, -2)),
        "pv": lambda: torch.matmul(P, v16),
        # fp16 attention as torch runs it: cuBLAS QK^T, fp32 softmax, cuBLAS PV
        "attn": lambda: torch.matmul(torch.softmax(torch.matmul(q16, k16.transpose(-1, -2)).float() * s["alpha"], -1)
                                     .half(), v16),
        "o": lambda: torch.nn.functional.linear(ctx, w16["o"]),
        "f1": lambda: torch.nn.functional.linear(Xf, w16["f1"]),
        "f2": lambda: torch.nn.functional.linear(R, w16["f2"]),
    }
    mm = lambda m, n, k: 2 * m * n * k  # noqa: E731
    pk = lambda n_el, planes: 2 * n_el + n_el * planes / 8  # noqa: E731  fp16 in + planes out
    ops = [Op("pack_x", "pack", op_pack_x, 0, pk(M * hidden, 2))]
    if fuse_qkv:
        ops += [Op("gemm_qkv_pack", "gemm", op_qkv_pack, mm(M, 3 * hidden, hidden),
                   M * hidden / 4 + 3 * hidden * hidden / 8 + 3 * M * hidden / 4, cub["qkv"])]
    else:
        ops += [Op("gemm_qkv", "gemm", op_qkv, mm(M, 3 * hidden, hidden),
                   M * hidden / 4 + 3 * hidden * hidden / 8 + 2 * M * 3 * hidden, cub["qkv"]),
                Op("pack_qkv", "pack", op_pack_qkv, 0, 3 * pk(M * hidden, 2), launches=2)]
    if fused_attn and fuse_ctx:  # real softmax inside; no P stand-in, no S/P/context in memory
        ops += [Op("attn_prefill_pack", "attn", op_attn_pack, 2 * mm(batch * heads * seq, seq, D),
                   2 * batch * heads * seq * D / 4 + batch * heads * D * seq / 4 + M * hidden / 4, cub["attn"],
                   launches=1)]
    elif fused_attn:
        ops += [Op("attn_prefill", "attn", op_attn, 2 * mm(batch * heads * seq, seq, D),
                   2 * batch * heads * seq * D / 4 + batch * heads * D * seq / 4 + 2 * M * hidden, cub["attn"]),
                Op("pack_ctx", "pack", op_pack_ctx, 0, pk(M * hidden, 2))]
    else:
        ops += [
            Op("attn_qk", "qk", op_qk, mm(batch * heads * seq, seq, D),
               2 * batch * heads * seq * D / 4 + 2 * batch * heads * seq * seq, cub["qk"]),
            Op("pack_p", "pack", op_pack_p, 0, pk(batch * heads * seq * seq, 1)),
        ] + ([
            Op("attn_pv_pack", "pv", op_pv_pack, mm(batch * heads * seq, D, seq),
               batch * heads * seq * seq / 8 + batch * heads * D * seq / 4 + M * hidden / 4, cub["pv"]),
        ] if fuse_ctx else [
            Op("attn_pv", "pv", op_pv, mm(batch * heads * seq, D, seq),
               batch * heads * seq * seq / 8 + batch * heads * D * seq / 4 + 2 * M * hidden, cub["pv"]),
            Op("pack_ctx", "pack", op_pack_ctx, 0, pk(M * hidden, 2)),
        ])
    ops += [
        Op("gemm_o", "gemm", op_o, mm(M, hidden, hidden),
           M * hidden / 4 + hidden * hidden / 8 + 2 * M * hidden, cub["o"]),
        Op("pack_xf", "pack", op_pack_xf, 0, pk(M * hidden, 2)),
    ]
    if fuse_ffn:
        ops.append(Op("gemm_ffn1", "gemm", op_f1, mm(M, ffn, hidden),
                      M * hidden / 4 + ffn * hidden / 8 + M * ffn / 8, cub["f1"]))  # writes FFN2's bool planes
    else:
        ops += [Op("gemm_ffn1", "gemm", op_f1_unfused, mm(M, ffn, hidden),
                   M * hidden / 4 + ffn * hidden / 8 + 2 * M * ffn, cub["f1"]),
                Op("pack_h1", "pack", op_pack_h1, 0, pk(M * ffn, 1))]
    ops += [
        Op("gemm_ffn2", "gemm", op_f2, mm(M, hidden, ffn),
           M * ffn / 8 + hidden * ffn / 8 + 2 * M * hidden, cub["f2"]),
    ]
    host_inputs = {"X": X, "Xf": Xf} if fused_attn else {"X": X, "Xf": Xf, "P": P}
    cfg = CFGS["bert_layer"]()
    def step():  # the whole path; the V^T pack joins the step's stream after QK^T (see op_pack_qkv)
        st["defer_join"] = True
        for op in ops:
            op.fn()
        st["defer_join"] = False
    return {"ops": ops, "step": step, "inputs": host_inputs, "outputs": [y2], "cfg": cfg,
            "oracle_sample": dict(X=X, Xf=Xf, R=R, P=P, Ws=Ws, s=s, heads=heads, D=D, batch=batch, seq=seq)}


def llama_prefill(B, dev, seed=303, M=2048, K=4096, Ns=(4096, 11008), world=1, rank=0, chunks=2, group=None,
                  gather="peer", grouped=True):
    """configs[2]: LLaMA-7B prefill linears, M = 2048 tokens, K = 4096, N = 4096 / 11008.
    world > 1: each linear N-sharded over the ranks, Y^T gathered on every rank:
      gather "peer" (default): the GEMM epilogue stores every tile into each peer's Y^T over NVLink
        (bwta_gemm_peers, dist.PeerAllGather, double-buffered) + one flag barrier per linear;
      gather "nccl": dist.NShardPlan with `chunks` chunks per rank, NCCL all_gather_into_tensor of
        each chunk overlapped with the next chunk's GEMM (the baseline)."""
    from paper_2604_03957_b200 import dist as D
    X = gen.activations((M, K), seed).to(dev)
    s_x = gen.act_scale(X)
    ops, st, outs, ws16, pgs, alt_outs = [], {}, [], {}, [], []

    def op_pack():
        st["xq"] = B.bwta_pack_act(X, s_x)
    ops.append(Op("pack_x", "pack", op_pack, 0, 2 * M * K + M * K / 4))
    if grouped and world == 1 and group is None:
        # both linears in ONE launch over the row-concatenated weights [W_4096; W_11008] (per-row mu
        # keeps each block's own binarization; outputs = the two column blocks of one [M, 15104] Y):
        # the same products bit for bit (tests/test_parity_gpu_large.py), 632 tiles in 8.5 rounds of
        # the persistent grid instead of 2.4 + 6.3 rounds in two launches; cuBLAS gets the same
        # concatenated GEMM as its baseline
        ws = [gen.weights(N, K, seed + 1 + i) for i, N in enumerate(Ns)]
        stats = [gen.weight_stats(w) for w in ws]
        mu_cat = torch.cat([torch.full((N,), float(mu), dtype=torch.float32) for N, (mu, _) in zip(Ns, stats)])
        wp = B.bwta_pack_weight(torch.cat(ws).to(dev), mu=mu_cat.to(dev))    # offline
        sw = torch.cat([s for _, s in stats]).to(dev)
        NT = sum(Ns)
        y = torch.empty((M, NT), dtype=torch.float16, device=dev)

        def op_g():
            B.bwta_gemm(st["xq"], wp, sw, s_x, out=y)

        def op_b1():
            B.bwta_gemm(st["xq"], wp, sw, s_x, out=y, design="mma_b1")

        def op_cc():
            B.bwta_gemm(st["xq"], wp, sw, s_x, out=y, design="cuda_core")
        w16 = torch.cat(ws).to(dev).half()
        name = "gemm_n" + "+".join(str(N) for N in Ns)
        ops.append(Op(name, "gemm", op_g, 2 * M * NT * K, M * K / 4 + NT * K / 8 + 4 * NT + 2 * M * NT,
                      lambda: torch.nn.functional.linear(X, w16),
                      alts={"design_a_cuda_core": op_cc, "prior_art_mma_b1": op_b1}))
        op_pack()
        smp = dict(X=X.cpu(), s_x=s_x, Ws={N: w for N, w in zip(Ns, ws)}, seed=seed)
        return {"ops": ops, "inputs": {"X": X}, "outputs": [y], "cfg": CFGS["llama_prefill"](),
                "oracle_sample": smp, "scaling": "strong",
                "parallelism": "single GPU; both linears in one launch over the row-concatenated weights"}
    for i, N in enumerate(Ns):
        w = gen.weights(N, K, seed + 1 + i)
        mu, s_w = gen.weight_stats(w)
        if world == 1 and group is None:
            wp = B.bwta_pack_weight(w.to(dev), mu=mu)          # offline
            sw = s_w.to(dev)
            y = torch.empty((M, N), dtype=torch.float16, device=dev)

            def op_g(wp=wp, sw=sw, y=y):
                B.bwta_gemm(st["xq"], wp, sw, s_x, out=y)

            def op_b1(wp=wp, sw=sw, y=y):  # prior art: the paper's mma.sync b1 design on this GPU
                B.bwta_gemm(st["xq"], wp, sw, s_x, out=y, design="mma_b1")

            def op_cc(wp=wp, sw=sw, y=y):  # design (a): LOP3 + POPC on CUDA cores
                B.bwta_gemm(st["xq"], wp, sw, s_x, out=y, design="cuda_core")
        elif gather == "peer":
            op_b1 = op_cc = None
            plan = D.NShardPlan(N, world, rank, 1)
            rows = plan.local_rows()
            wp = B.bwta_pack_weight(w[rows].contiguous().to(dev), mu=mu)
            sw = s_w[rows].contiguous().to(dev)
            pg = D.PeerAllGather(plan, M, dev, group=group if group is not None else torch.distributed.group.WORLD)
            pgs.append(pg)
            y = pg.out(0)
            alt_outs.append(pg.out(1))

            def op_g(wp=wp, sw=sw, pg=pg):
                pg(st["xq"], wp, sw, s_x)
        else:
            op_b1 = op_cc = None
            plan = D.NShardPlan(N, world, rank, chunks)
            rows = plan.local_rows()
            wp = B.bwta_pack_weight(w[rows].contiguous().to(dev), mu=mu)
            sw = s_w[rows].contiguous().to(dev)
            y = torch.empty((plan.n_pad, M), dtype=torch.float16, device=dev)

            def op_g(wp=wp, sw=sw, y=y, plan=plan):
                D.gemm_nshard_overlap(st["xq"], wp, sw, s_x, plan, out=y, group=group)
        outs.append(y)
        ws16[N] = w
        ops.append(Op(f"gemm_n{N}", "gemm", op_g, 2 * M * N * K, M * K / 4 + N * K / 8 + 4 * N + 2 * M * N,
                      (lambda N=N: torch.nn.functional.linear(X, st["w16"][N])) if world == 1 and group is None
                      else None,
                      alts={"design_a_cuda_core": op_cc, "prior_art_mma_b1": op_b1} if op_b1 else None))
    st["w16"] = {N: w.to(dev) for N, w in ws16.items()} if world == 1 and group is None else {}
    op_pack()
    smp = dict(X=X.cpu(), s_x=s_x, Ws=ws16, seed=seed)
    sharded = world > 1 or group is not None
    W = {"ops": ops, "inputs": {"X": X}, "outputs": outs, "cfg": CFGS["llama_prefill"](),
         "oracle_sample": smp, "scaling": "strong",
         "parallelism": ("single GPU" if not sharded else
                         f"N-shard x{world}, all-gather fused into the GEMM epilogue (peer TMA stores over NVLink "
                         "+ flag barrier, no collective)" if gather == "peer" else
                         f"N-shard x{world} ({chunks} chunks/rank, NCCL all-gather in place, overlapped)")}
    if pgs:   # double-buffered Y^T: the step alternates buffers, so the bench alternates two graphs
        def set_parity(p):
            for pg in pgs:
                pg.step = p
        W.update(parities=2, set_parity=set_parity, outputs_par=[outs, alt_outs])
    return W


def llama_attn(B, dev, seed=404, heads=32, seq=2048, D=128):
    """configs[3]: LLaMA-7B ternary attention QK^T and PV, 32 heads, head_dim 128, seq 2048."""
    q = gen.activations((1, heads, seq, D), seed).to(dev)
    k = gen.activations((1, heads, seq, D), seed + 1).to(dev)
    v = gen.activations((1, heads, seq, D), seed + 2).to(dev)
    P = gen.attention_probs((1, heads, seq, seq), seed + 3).to(dev)
    sq, sk, sv = gen.act_scale(q), gen.act_scale(k), gen.act_scale(v)
    s_att = float(np.float32(2.0 / seq))
    alpha, beta = float(np.float32(sq * sk / np.sqrt(D))), float(np.float32(s_att * sv))
    S = torch.empty((1, heads, seq, seq), dtype=torch.float16, device=dev)
    O = torch.empty((1, heads, seq, D), dtype=torch.float16, device=dev)
    st = {}

    def op_pack_qkv():
        st["qp"], st["kp"] = B.bwta_pack_act(q, sq), B.bwta_pack_act(k, sk)
        st["vt"] = B.bwta_pack_act(v, sv, transpose=True)

    def op_qk():
        B.bwta_attn_qk(st["qp"], st["kp"], alpha, out=S)

    def op_pack_p():
        st["pp"] = B.bwta_pack_act(P, s_att, "bool")

    def op_pv():
        B.bwta_attn_pv(st["pp"], st["vt"], beta, out=O)

    def op_fused():   # QK^T -> fp32 softmax -> bool P -> PV in one launch (N3); S and P stay on chip
        B.bwta_attn_prefill(st["qp"], st["kp"], st["vt"], alpha, s_att, beta, out=O2)

    def op_causal():  # the decoder's causal mask: key blocks above the diagonal skipped
        B.bwta_attn_prefill(st["qp"], st["kp"], st["vt"], alpha, s_att, beta, out=O3, causal=True)
    O2 = torch.empty((1, heads, seq, D), dtype=torch.float16, device=q.device)
    O3 = torch.empty((1, heads, seq, D), dtype=torch.float16, device=q.device)
    cmask = torch.ones((seq, seq), dtype=torch.bool, device=q.device).triu(1)

    def torch_causal():
        s_ = torch.matmul(q, k.transpose(-1, -2)).float() * alpha
        return torch.matmul(torch.softmax(s_.masked_fill(cmask, float("-inf")), -1).half(), v)
    op_pack_qkv(); op_pack_p()  # noqa: E702
    n = heads * seq * D
    ops = [Op("pack_qkv", "pack", op_pack_qkv, 0, 3 * (2 * n + n / 4)),
           Op("attn_qk", "qk", op_qk, 2 * heads * seq * seq * D, 2 * n / 4 + 2 * heads * seq * seq,
              lambda: torch.matmul(q, k.transpose(-1, -2))),
           Op("pack_p", "pack", op_pack_p, 0, 2 * heads * seq * seq + heads * seq * seq / 8),
           Op("attn_pv", "pv", op_pv, 2 * heads * seq * seq * D, heads * seq * seq / 8 + n / 4 + 2 * n,
              lambda: torch.matmul(P, v)),
           # the fused op does both products (4 T^2 D ops); baseline: torch fp16 QK^T, fp32 softmax, PV
           Op("attn_prefill_fused", "attn", op_fused, 4 * heads * seq * seq * D, 2 * n / 4 + n / 4 + 2 * n,
              lambda: torch.matmul(torch.softmax(torch.matmul(q, k.transpose(-1, -2)).float() * alpha, -1).half(), v)),
           # causal: the products over the visible keys only (4 D per (query, visible key) pair)
           Op("attn_prefill_causal", "attn", op_causal, 4 * heads * (seq * (seq + 1) // 2) * D,
              2 * n / 4 + n / 4 + 2 * n, torch_causal)]
    cfg = {"workload": "llama_attn (configs[3]): ternary attention, 32 heads, head_dim 128, seq 2048 (step: Q/K/V^T "
                       "packs + the fused prefill attention; the unfused ops are timed alongside)",
           "heads": heads, "seq_len": seq, "head_dim": D}

    def step():
        op_pack_qkv()
        op_fused()
    return {"ops": ops, "inputs": {}, "outputs": [O2], "cfg": cfg, "oracle_sample": None, "step": step,
            "step_ops": ["pack_qkv", "attn_prefill_fused"]}


def decode_linear(B, dev, seed=505, shapes=((1, 8192, 28672), (16, 8192, 28672), (1, 4096, 11008))):
    """Decode-sized BWTA linears: M = 1 / 16 tokens against configs[4]'s largest
    weight (K = 8192, N = 28672) and LLaMA-7B's FFN (K = 4096, N = 11008); the weight stream
    (N K / 8 bytes) is the algorithmic traffic.  The activation pack is part of each op."""
    ops = []
    for i, (M, K, N) in enumerate(shapes):
        X = gen.activations((M, K), seed + 10 * i).to(dev)
        s_x = gen.act_scale(X)
        w = gen.weights(N, K, seed + 10 * i + 1)
        mu, s_w = gen.weight_stats(w)
        wp = B.bwta_pack_weight(w.to(dev), mu=mu)
        sw = s_w.to(dev)
        y = torch.empty((M, N), dtype=torch.float16, device=dev)
        w16 = w.to(dev)

        def op_g(X=X, s_x=s_x, wp=wp, sw=sw, y=y):
            # pack + GEMV (two launches): in a graph this beats bwta_gemm_x, whose every CTA
            # re-quantizes the activation row (tools/decode_bench.py)
            B.bwta_gemm(B.bwta_pack_act(X, s_x), wp, sw, s_x, out=y)
        ops.append(Op(f"m{M}_k{K}_n{N}", "gemm", op_g, 2 * M * N * K, 2 * M * K + M * K / 4 + N * K / 8 + 2 * M * N,
                      (lambda X=X, w16=w16: torch.nn.functional.linear(X, w16))))
    cfg = {"workload": "decode_linear: M = 1 / 16 tokens x (K 8192, N 28672) and (K 4096, N 11008)"}
    return {"ops": ops, "inputs": {}, "outputs": [], "cfg": cfg, "oracle_sample": None}


def decode_attn(B, dev, seed=606, shapes=((1, 32, 2048, 128), (8, 32, 2048, 128))):
    """Fused decode attention (Tq = 1), one launch per call: LLaMA-7B heads,
    a 2048-token context, batch 1 and 8; baseline = torch fp16 (cuBLAS QK^T, softmax, cuBLAS PV).
    Bytes = the K and V^T bit planes + the query + the output."""
    ops = []
    for i, (b, h, tk, dh) in enumerate(shapes):
        q = gen.activations((b, h, 1, dh), seed + 10 * i).to(dev)
        k = gen.activations((b, h, tk, dh), seed + 10 * i + 1).to(dev)
        v = gen.activations((b, h, tk, dh), seed + 10 * i + 2).to(dev)
        sq, sk, sv = gen.act_scale(q), gen.act_scale(k), gen.act_scale(v)
        alpha = float(np.float32(sq * sk / np.sqrt(dh)))
        s_att = float(np.float32(2.0 / tk))
        beta = float(np.float32(s_att * sv))
        qp, kp = B.bwta_pack_act(q, sq), B.bwta_pack_act(k, sk)
        vt = B.bwta_pack_act(v, sv, transpose=True)

        def op(qp=qp, kp=kp, vt=vt, alpha=alpha, s_att=s_att, beta=beta):
            B.bwta_attn_decode(qp, kp, vt, alpha, s_att, beta)
        n = b * h
        ops.append(Op(f"b{b}_h{h}_tk{tk}_d{dh}", "attn", op, 4 * n * tk * dh,
                      n * (tk * dh / 4 + dh * tk / 4 + dh / 4 + 2 * dh),
                      (lambda q=q, k=k, v=v, alpha=alpha: torch.softmax(
                          (q @ k.transpose(-1, -2)).float() * alpha, -1).half() @ v)))
    cfg = {"workload": "decode_attn: fused BWTA decode attention, 32 heads x 128, context 2048, batch 1 / 8"}
    return {"ops": ops, "inputs": {}, "outputs": [], "cfg": cfg, "oracle_sample": None}


def nshard_gemm(B, dev, seed=707, world=1, rank=0, chunks=2, group=None, gather="peer"):
    """configs[4]: the LLaMA-70B-shaped BWTA linear (K 8192, N 28672, M 2048 tokens) N-sharded across
    the ranks exactly like llama_prefill at N > 1 (strong scaling)."""
    W = llama_prefill(B, dev, seed, M=2048, K=8192, Ns=(28672,), world=world, rank=rank, chunks=chunks, group=group,
                      gather=gather)
    W["cfg"] = CFGS["nshard_gemm"]()
    W["oracle_sample"] = None
    return W


def bert_linear(B, dev, seed=101, world=1, rank=0):
    """configs[0]: single BWTA linear M=128 K=768 N=768."""
    W = llama_prefill(B, dev, seed, M=128, K=768, Ns=(768,), world=world, rank=rank, chunks=1)
    W["cfg"] = CFGS["bert_linear"]()
    W["oracle_sample"] = None
    return W


# the config dict of each workload: identical in the GPU arm and the reference (oracle) arm
CFGS = {
    "llama_prefill": lambda: {"workload": "llama_prefill (configs[2]): LLaMA-7B prefill linears, M=2048 tokens, "
                                          "K=4096, N=4096 and N=11008, fp16 activations packed in the step",
                              "tokens": 2048, "k": 4096, "n": [4096, 11008]},
    "bert_layer": lambda: {"workload": "bert_layer (configs[1]): BERT-base layer, batch 32 x seq 128, hidden 768, "
                                       "12 heads x 64, FFN 3072", "batch": 32, "seq_len": 128, "hidden": 768,
                           "heads": 12, "ffn": 3072, "tokens": 4096},
    "nshard_gemm": lambda: {"workload": "nshard_gemm (configs[4]): K=8192 N=28672 M=2048, weight rows N-sharded, "
                                        "Y^T all-gathered (NCCL)", "tokens": 2048, "k": 8192, "n": [28672]},
    "bert_linear": lambda: {"workload": "bert_linear (configs[0]): M=128 K=768 N=768", "tokens": 128, "k": 768,
                            "n": [768]},
}


WORKLOADS = {"bert_layer": bert_layer, "llama_prefill": llama_prefill, "llama_attn": llama_attn,
             "bert_linear": bert_linear, "decode_linear": decode_linear, "decode_attn": decode_attn,
             "nshard_gemm": nshard_gemm}


# ----------------------------------------------------------------------------- oracle (CPU) legs
def oracle_bert_layer_step(smp, threads, row_frac=1.0):
    """The BERT layer's BWTA path through the CPU oracle (quantize + dot + epilogue),
    on the same inputs; row_frac < 1 runs a stated row/head sample.  Returns ops done."""
    import oracle

    def st(t):
        t = t.detach().cpu().contiguous()
        return t.view(torch.int16).numpy().view(np.uint16) if t.dtype in (torch.float16, torch.bfloat16) else t.numpy()
    s, M = smp["s"], smp["X"].shape[0]
    rows = max(1, int(M * row_frac))
    ops = 0
    qx = oracle.quantize_act(st(smp["X"][:rows]), "f16", s["x"], "ternary")
    y_f1 = None
    for name, xin, sx, kind in (("qkv", None, s["x"], "ternary"), ("o", smp["X"], s["x"], "ternary"),
                                ("f1", smp["Xf"], s["xf"], "ternary"), ("f2", "f1", s["r"], "bool")):
        w = smp["Ws"][name]
        mu, s_w = gen.weight_stats(w)
        qw = oracle.binarize_weight(st(w), "f16", mu=mu)
        if xin is None:
            qa = qx
        elif isinstance(xin, str):   # FFN2 consumes bool(FFN1 output): relu(y) >= t <=> y >= t
            qa = oracle.quantize_act(y_f1, "f16", sx, kind)
        else:
            qa = oracle.quantize_act(st(xin[:rows]), "f16", sx, kind)
        y = oracle.gemm(qa, qw, s_w.numpy(), sx, "f16", threads=threads)
        if name == "f1":
            y_f1 = y
        ops += 2 * qa.shape[0] * qw.shape[0] * qw.shape[1]
    nbh = max(1, int(smp["batch"] * smp["heads"] * row_frac))
    b = max(1, nbh // smp["heads"])
    q = gen.activations((b, smp["heads"], smp["seq"], smp["D"]), 1)
    qq = oracle.quantize_act(st(q).reshape(-1, smp["seq"], smp["D"]), "f16", 1.0, "ternary")
    oracle.attn_qk(qq, qq, s["alpha"], "f16", threads=threads)
    pp = oracle.quantize_act(st(smp["P"][:b]).reshape(-1, smp["seq"], smp["seq"]), "f16", s["att"], "bool")
    oracle.attn_pv(pp, qq, s["beta"], "f16", threads=threads)
    ops += 2 * 2 * qq.shape[0] * smp["seq"] * smp["seq"] * smp["D"]
    return ops, f"{rows}/{M} token rows of each BWTA linear + {qq.shape[0]} (batch x head) attention entries"


def _st(t):
    t = t.detach().cpu().contiguous()
    return t.view(torch.int16).numpy().view(np.uint16) if t.dtype in (torch.float16, torch.bfloat16) else t.numpy()


class OracleLlamaPrefill:
    """configs[2]'s step through the CPU oracle: quantize a sample of X's token rows,
    the integer dot with both binarized weights (the naive triple loop), the R5 epilogue to fp16.
    Weights are binarized once up front (offline in the product too)."""

    def __init__(self, smp, threads):
        import oracle
        self.o, self.smp, self.threads = oracle, smp, threads
        self.qw = {}
        for N, w in smp["Ws"].items():
            mu, s_w = gen.weight_stats(w)
            self.qw[N] = (oracle.binarize_weight(_st(w), "f16", mu=mu), s_w.numpy())
        self.xs = _st(smp["X"])

    def step(self, rows: int):
        o, M = self.o, self.xs.shape[0]
        r0 = (self._i * rows) % M if hasattr(self, "_i") else 0
        self._i = getattr(self, "_i", 0) + 1
        idx = (np.arange(rows) + r0) % M
        qa = o.quantize_act(self.xs[idx], "f16", self.smp["s_x"], "ternary")
        ops = 0
        for N, (qw, s_w) in self.qw.items():
            o.gemm(qa, qw, s_w, self.smp["s_x"], "f16", threads=self.threads)
            ops += 2 * rows * qw.shape[0] * qw.shape[1]
        return ops


def _llama_inputs_cpu(seed=303, M=2048, K=4096, Ns=(4096, 11008)):
    X = gen.activations((M, K), seed)
    return dict(X=X, s_x=gen.act_scale(X), Ws={N: gen.weights(N, K, seed + 1 + i) for i, N in enumerate(Ns)})


def reference_arm(args):
    """--impl reference: the CPU oracle, as it stands, on the host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    oracle.build()
    threads = oracle.default_threads()
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))

    wl = args.workload
    if wl == "llama_prefill":
        orc = OracleLlamaPrefill(_llama_inputs_cpu(), threads)
        # size each step so the whole --steps/--warmup run takes about a minute of CPU time
        t0 = time.perf_counter()
        orc.step(32)
        t32 = time.perf_counter() - t0
        budget = 60.0 / max(1, args.steps + args.warmup)
        rows = int(min(2048, max(16, 32 * budget / max(t32, 1e-6))))
        for _ in range(args.warmup):
            orc.step(rows)
        t0 = time.perf_counter()
        tot_ops = sum(orc.step(rows) for _ in range(args.steps))
        dt = time.perf_counter() - t0
        sample = (f"{rows} of 2048 token rows per step (rotating) through both linears (N 4096 + 11008, K 4096): "
                  "quantize X rows + integer dot + fp16 epilogue; weights binarized once (offline)")
        scaling = "strong"
    elif wl == "bert_layer":
        smp = _bert_inputs_cpu()
        frac = args.ref_row_frac
        for _ in range(args.warmup):
            oracle_bert_layer_step(smp, threads, frac)
        t0 = time.perf_counter()
        tot_ops = 0
        for _ in range(args.steps):
            o, sample = oracle_bert_layer_step(smp, threads, frac)
            tot_ops += o
        dt = time.perf_counter() - t0
        scaling = "weak"
    else:
        print(json.dumps({"impl": "reference", "unavailable": f"reference arm implemented for llama_prefill and "
                                                             f"bert_layer only (asked {wl})"}))
        return 0
    val = tot_ops / dt / 1e12
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
            "dtype": "int32 (oracle integer dot, fp32 epilogue)",
            "data": "synthetic (seeded, recipe in DESIGN.md)", "config": CFGS[wl](),
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def _bert_inputs_cpu(seed=202, batch=32, seq=128, hidden=768, heads=12, ffn=3072):
    M = batch * seq
    g = lambda s: s + seed  # noqa: E731
    X = gen.activations((M, hidden), g(0))
    Xf = gen.activations((M, hidden), g(1))
    R = gen.relu_activations((M, ffn), g(2))  # stand-in for the FFN1 output (timing only)
    P = gen.attention_probs((batch, heads, seq, seq), g(3))
    Ws = {"qkv": gen.weights(3 * hidden, hidden, g(4)), "o": gen.weights(hidden, hidden, g(5)),
          "f1": gen.weights(ffn, hidden, g(6)), "f2": gen.weights(hidden, ffn, g(7))}
    s = {"x": gen.act_scale(X), "xf": gen.act_scale(Xf), "r": gen.act_scale(R), "att": float(np.float32(2.0 / seq)),
         "alpha": 0.125, "beta": float(np.float32(2.0 / seq))}
    return dict(X=X, Xf=Xf, R=R, P=P, Ws=Ws, s=s, heads=heads, D=hidden // heads, batch=batch, seq=seq)


# ----------------------------------------------------------------------------- main arm
def _spawn(args) -> int:
    """--gpus N > 1 without a torchrun environment: launch N ranks with torchrun on this node."""
    import socket
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def time_eager(step, flush, reps, stream):
    """Per-step device times (ms) of eager launches (N > 1: the step holds NCCL collectives)."""
    ts = []
    with torch.cuda.stream(stream):
        for _ in range(reps):
            flush_l2(flush)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            ts.append((e0, e1))
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in ts]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="bwta", choices=["bwta", "reference"])
    ap.add_argument("--workload", default="llama_prefill", choices=sorted(WORKLOADS))
    ap.add_argument("--no-extras", action="store_true", help="skip the secondary-workload side measurements")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline (oracle) leg")
    ap.add_argument("--ref-row-frac", type=float, default=1.0)
    ap.add_argument("--chunks", type=int, default=2, help="N-shard chunks per rank (N > 1 or --nshard)")
    ap.add_argument("--gather", default="peer", choices=["peer", "nccl"],
                    help="N-shard gather: peer = fused into the GEMM epilogue over NVLink, nccl = chunked NCCL "
                         "all-gathers (baseline)")
    ap.add_argument("--nshard", action="store_true",
                    help="run the N-sharded path with its NCCL all-gathers even at N = 1 (a 1-rank communicator)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return reference_arm(args)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return _spawn(args)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 or args.nshard:
        import torch.distributed as dist
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,TUNING")
        os.environ.setdefault("NCCL_DEBUG_FILE", os.path.join(ROOT, "gpurun_out", f"nccl_rank{rank}.log"))
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        if "MASTER_ADDR" not in os.environ:  # --nshard at N = 1 without torchrun
            import socket
            so = socket.socket()
            so.bind(("127.0.0.1", 0))
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(so.getsockname()[1]), RANK="0", WORLD_SIZE="1")
            so.close()
        # NCCL prints its version on stdout at communicator creation: keep stdout for the JSON line
        saved = os.dup(1)
        os.dup2(2, 1)
        try:
            dist.init_process_group("nccl", device_id=dev)
            dist.barrier()
        finally:
            sys.stdout.flush()
            os.dup2(saved, 1)
            os.close(saved)
    import paper_2604_03957_b200 as B

    pk = peaks()
    # the matmuls run on tcgen05.mma.kind::mxf4 (E2M1 codes): dense FP4 = 4x dense bf16 (nominal 9 / 2.25 PF)
    tc_peak = pk["bf16_tflops"] * 4.0
    stream = torch.cuda.Stream(device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    wl_fn = WORKLOADS[args.workload]
    import inspect
    kw = {}
    if "world" in inspect.signature(wl_fn).parameters:
        kw = {"world": world, "rank": rank}
        if args.nshard and "group" in inspect.signature(wl_fn).parameters:
            kw["group"] = torch.distributed.group.WORLD
        if "chunks" in inspect.signature(wl_fn).parameters:
            kw["chunks"] = args.chunks
        if "gather" in inspect.signature(wl_fn).parameters:
            kw["gather"] = args.gather
    W = wl_fn(B, dev, **kw)
    ops = W["ops"]
    scaling = W.get("scaling", "weak") if world > 1 or W.get("scaling") else "weak"
    sharded = (world > 1 or args.nshard) and scaling == "strong"

    def step():
        if W.get("step"):
            return W["step"]()
        for op in ops:
            op.fn()
    step_ops = W.get("step_ops")
    total_ops = sum(op.ops for op in ops if step_ops is None or op.name in step_ops)  # one replica / sharded job
    job_ops = total_ops * (world if (world > 1 and not sharded) else 1)

    # -------- device-time step (CUDA graph of the library calls at N = 1)
    # the step (incl. the NCCL all-gathers of the sharded path) is captured into a CUDA graph;
    # eager launches only if the capture fails (the host would otherwise bound the sharded step)
    use_graph = True
    par = {"i": 0, "n": W.get("parities", 1)}
    try:
        if par["n"] == 1:
            g_step = graph_of(step, stream)
        else:   # one graph per output buffer, replayed alternately (the fused gather's double buffer)
            gs = [graph_of(step, stream, pre=lambda p=p: W["set_parity"](p)) for p in range(par["n"])]

            class _Cycle:
                def replay(self):
                    par["i"] = (par["i"] + 1) % par["n"]
                    gs[par["i"]].replay()
            g_step = _Cycle()
    except Exception as exc:  # pragma: no cover
        print(f"bench: CUDA-graph capture failed ({exc!r}); eager launches", file=sys.stderr)
        torch.cuda.synchronize()
        use_graph, g_step = False, None
    run = (lambda: g_step.replay()) if use_graph else step
    l0 = B.lib.bwta_kernel_launches()
    with torch.cuda.stream(stream):
        step()
    torch.cuda.synchronize()
    launches_per_step = B.lib.bwta_kernel_launches() - l0

    clk = ClockSampler(local).__enter__()
    t_w = time.perf_counter()
    nw = 0
    while nw < args.warmup or time.perf_counter() - t_w < 0.5:   # >= W steps and >= 0.5 s under load
        with torch.cuda.stream(stream):
            flush_l2(flush)
            run()
        nw += 1
        if nw % 16 == 0:
            torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    times = time_graph(g_step, flush, args.steps, 0, stream) if use_graph else time_eager(step, flush, args.steps,
                                                                                          stream)
    torch.cuda.synchronize()
    clk.__exit__()
    if world > 1:
        torch.distributed.barrier()
    t_total = sum(times)  # ms, K steps
    if world > 1:
        t = torch.tensor([t_total], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        t_total = float(t.item())
    ms_step = t_total / args.steps
    value = job_ops * args.steps / (t_total / 1e3) / 1e12

    # -------- per-op device times and cuBLAS FP16 baselines (N = 1: graphs of one op)
    per_op, cub_ms = {}, {}
    if use_graph:
        for op in ops:
            per_op[op.name] = op_time_ms(op.fn, flush, stream)
            if op.cublas is not None:
                cub_ms[op.name] = op_time_ms(op.cublas, flush, stream)
    else:   # eager per-op times (compute + its gathers at N > 1)
        for op in ops:
            per_op[op.name] = statistics.median(time_eager(op.fn, flush, 10, stream))
    alt_ms = {}
    if world == 1:
        for op in ops:
            for an, fn in op.alts.items():
                alt_ms.setdefault(op.name, {})[an] = op_time_ms(fn, flush, stream, reps=5, trials=3)
    cublas_total = sum(cub_ms.values())
    bwta_mm_only = sum(per_op[n] for n in cub_ms)
    pack_ms = sum(per_op[o.name] for o in ops if o.kind == "pack")

    # -------- per-kernel device times INSIDE the step (the roofline's denominator): the step's op
    # sequence launched eagerly on the bench stream, L2 flushed before every step as in the timed
    # region, CUDA events recorded on that stream between consecutive ops; a device sleep ahead of
    # each step keeps the host's enqueue off the GPU timeline (no idle gaps inside the intervals)
    in_step, in_graph = {}, {}
    if world == 1 and not W.get("step") and W.get("parities", 1) == 1:
        samples = {op.name: [] for op in ops}
        with torch.cuda.stream(stream):
            for r in range(max(args.steps, 5) + 2):
                flush_l2(flush)
                torch.cuda._sleep(1_000_000)
                evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(ops) + 1)]
                evs[0].record(stream)
                for i, op in enumerate(ops):
                    op.fn()
                    evs[i + 1].record(stream)
                torch.cuda.synchronize()
                if r >= 2:
                    for i, op in enumerate(ops):
                        samples[op.name].append(evs[i].elapsed_time(evs[i + 1]))
        in_step = {k: _trimmed_mean(v) for k, v in samples.items()}
        # the same per-op intervals inside a CUDA graph of the step: external timing events captured
        # between the ops (each event node also stands between two kernels, so no PDL overlap across
        # it); replayed with the L2 flushed before every replay, as the timed steps are
        try:
            evs = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(len(ops) + 1)]

            def step_ev():
                evs[0].record(stream)
                for i, op in enumerate(ops):
                    op.fn()
                    evs[i + 1].record(stream)
            g_ev = graph_of(step_ev, stream)
            samples = {op.name: [] for op in ops}
            with torch.cuda.stream(stream):
                for r in range(max(args.steps, 5) + 2):
                    flush_l2(flush)
                    g_ev.replay()
                    torch.cuda.synchronize()
                    if r >= 2:
                        for i, op in enumerate(ops):
                            samples[op.name].append(evs[i].elapsed_time(evs[i + 1]))
            in_graph = {k: _trimmed_mean(v) for k, v in samples.items()}
        except Exception as exc:  # pragma: no cover
            print(f"bench: in-graph op timing unavailable ({exc!r})", file=sys.stderr)
            torch.cuda.synchronize()

    # -------- roofline of the dominant KERNEL: the single-launch op with the largest time
    cands = [o for o in ops if o.launches == 1]
    dom = max(cands, key=lambda o: per_op[o.name])
    t_dom = (in_graph.get(dom.name) or in_step.get(dom.name) or per_op[dom.name]) / 1e3
    if dom.kind == "pack" or args.workload.startswith("decode"):  # decode: the bit-plane stream bounds it
        roof = {"bound": "hbm", "achieved": dom.bytes / t_dom / 1e9, "peak": pk["hbm_gbs"], "unit": "GB/s"}
    else:
        roof = {"bound": "tensor", "achieved": dom.ops / t_dom / 1e12, "peak": tc_peak, "unit": "TOPS"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["kernel"] = dom.name
    roof["duration_us"] = t_dom * 1e6
    roof["timing"] = ("in-step, in-graph: CUDA events (external event nodes) on the launching stream around the "
                      "kernel inside a CUDA graph of the step, L2 flushed before every replay (trimmed mean "
                      "over the timed-step count)" if dom.name in in_graph else
                      "in-step: CUDA events on the launching stream around the kernel inside the L2-flushed step "
                      "sequence, eager launches (trimmed mean over the timed-step count)" if dom.name in in_step else
                      "isolated: graph of [L2 flush, kernel] x 20 minus graph of [L2 flush] x 20")
    roof["algorithmic"] = {"ops_per_launch": dom.ops, "bytes_per_launch": dom.bytes}
    roof["peak_source"] = (f"{pk['source']} bf16 {pk['bf16_tflops']} TFLOP/s x 4 (dense fp4/bf16 nominal ratio; "
                           "the path runs tcgen05.mma.kind::mxf4)"
                           if roof["unit"] == "TOPS" else f"{pk['source']} HBM copy")
    roof["traffic"] = _traffic(dom.name, args.workload)
    roof["traffic_l2"] = _traffic(dom.name, args.workload + "_lts_bytes")
    roof["traffic_source"] = ("profiles/ncu_traffic.json (ncu --set full, one launch): traffic = dram__bytes_read.sum + "
                              "dram__bytes_write.sum (the output write stays in L2 during the launch, so it is "
                              "undercounted); traffic_l2 = lts__t_sectors_srcunit_tex x 32 B")

    # -------- end to end through the public API with host buffers
    e2e = None
    if W["inputs"]:
        hosts = {k: v.detach().cpu().pin_memory() for k, v in W["inputs"].items()}
        outs = W.get("outputs") or []
        outs_h = [[torch.empty(o.shape, dtype=o.dtype).pin_memory() for o in outs] for _ in range(2)]
        h2d = sum(v.numel() * v.element_size() for v in hosts.values())
        d2h = sum(o.numel() * o.element_size() for o in outs)
        # Pipelined like a serving loop: step i's inputs go H2D (pinned -> device staging, copy
        # stream) while step i-1 computes; the compute stream moves them into the step's input
        # tensors (D2D), flushes L2, runs the step and stages the outputs; a second copy stream
        # reads them back D2H.  Every step's H2D and D2H is inside the timed region (from the
        # first H2D to the last D2H, pipeline fill and drain included).
        cin, cout = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        stage_in = [{k: torch.empty_like(v) for k, v in W["inputs"].items()} for _ in range(2)]
        stage_out = [[torch.empty_like(o) for o in outs] for _ in range(2)]
        ev_in_ready = [torch.cuda.Event() for _ in range(2)]
        ev_in_free = [torch.cuda.Event() for _ in range(2)]
        ev_out_ready = [torch.cuda.Event() for _ in range(2)]
        ev_out_free = [torch.cuda.Event() for _ in range(2)]

        def run_pipelined(nsteps):
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            if world > 1:
                torch.distributed.barrier()
            t0.record(cin)
            for i in range(nsteps):
                sl = i % 2
                with torch.cuda.stream(cin):
                    if i >= 2:
                        cin.wait_event(ev_in_free[sl])
                    for k, v in hosts.items():
                        stage_in[sl][k].copy_(v, non_blocking=True)
                    ev_in_ready[sl].record(cin)
                with torch.cuda.stream(stream):
                    stream.wait_event(ev_in_ready[sl])
                    for k in hosts:
                        W["inputs"][k].copy_(stage_in[sl][k], non_blocking=True)
                    ev_in_free[sl].record(stream)
                    flush_l2(flush)
                    run()
                    if outs:
                        if i >= 2:
                            stream.wait_event(ev_out_free[sl])
                        cur = W["outputs_par"][par["i"]] if (use_graph and "outputs_par" in W) else outs
                        for so, o in zip(stage_out[sl], cur):
                            so.copy_(o, non_blocking=True)
                        ev_out_ready[sl].record(stream)
                if outs:
                    with torch.cuda.stream(cout):
                        cout.wait_event(ev_out_ready[sl])
                        for oh, so in zip(outs_h[sl], stage_out[sl]):
                            oh.copy_(so, non_blocking=True)
                        ev_out_free[sl].record(cout)
            cout.wait_stream(stream)
            t1.record(cout)
            torch.cuda.synchronize()
            ms = t0.elapsed_time(t1)
            if world > 1:
                t = torch.tensor([ms], device=dev)
                torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
                ms = float(t.item())
            return ms

        run_pipelined(args.warmup)
        t_e2e = run_pipelined(args.steps)
        e2e = {"value": job_ops * args.steps / (t_e2e / 1e3) / 1e12, "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": t_e2e / args.steps,
               "pipelined": "H2D of step i overlaps the compute of step i-1 (two staging buffers); the outputs "
                            "are read back D2H every step; L2 flushed before every step; fill and drain inside "
                            "the timed region"}

    # -------- side measurements: the secondary workloads (N = 1, rank 0)
    extras = {}
    if not args.no_extras and world == 1:
        names = [n for n in ("llama_prefill", "bert_layer", "llama_attn", "decode_linear", "decode_attn")
                 if n != args.workload]
        for name in names:
            Wx = WORKLOADS[name](B, dev)
            res = {}
            if Wx.get("step"):          # a whole-step graph (bert_layer)
                def st_x():
                    Wx["step"]()
                gx = graph_of(st_x, stream)
                tx = statistics.median(time_graph(gx, flush, 20, 3, stream))
                ox = sum(o.ops for o in Wx["ops"])
                res["step"] = {"us": tx * 1e3, "TOPS": ox / (tx / 1e3) / 1e12}
                del gx
            for op in Wx["ops"]:
                t = op_time_ms(op.fn, flush, stream)
                r = {"us": t * 1e3}
                if op.kind == "pack":
                    r["GB/s"] = op.bytes / (t / 1e3) / 1e9
                elif name.startswith("decode"):  # HBM-bound: bytes (bit planes streamed + inputs + outputs)
                    r["GB/s"] = op.bytes / (t / 1e3) / 1e9
                    r["frac_hbm_peak"] = r["GB/s"] / pk["hbm_gbs"]
                else:
                    r["TOPS"] = op.ops / (t / 1e3) / 1e12
                    r["frac_tc_peak"] = r["TOPS"] / tc_peak
                if op.cublas is not None:
                    tc = op_time_ms(op.cublas, flush, stream)
                    r["cublas_fp16_us"] = tc * 1e3
                    r["speedup_vs_cublas_fp16"] = tc / t
                res[op.name] = r
            if "step" in res:
                cb = sum(r.get("cublas_fp16_us", 0) for r in res.values())
                res["step"]["speedup_vs_cublas_fp16_matmuls"] = cb / res["step"]["us"]
            extras[name] = res
            del Wx
        torch.cuda.empty_cache()

    # -------- CPU oracle baseline (rank 0, N = 1 only)
    cpu = None
    if not args.no_cpu and world == 1 and W.get("oracle_sample") is not None:
        import oracle
        oracle.build()
        threads = oracle.default_threads()
        if args.workload == "llama_prefill":
            orc = OracleLlamaPrefill(W["oracle_sample"], threads)
            t0 = time.perf_counter()
            o, n = 0, 0
            while n < 1 or time.perf_counter() - t0 < 10.0:       # >= one full step and >= 10 s of CPU work
                o += orc.step(2048)
                n += 1
            dt = time.perf_counter() - t0
            sample = (f"{n} full step(s) (all 2048 token rows through both linears: quantize X + integer dot + "
                      f"fp16 epilogue; weights binarized once, offline); {dt:.2f} s wall")
        else:
            t0 = time.perf_counter()
            o, sample = oracle_bert_layer_step(W["oracle_sample"], threads, 1.0)
            dt = time.perf_counter() - t0
            sample = f"one full step: {sample}; {dt:.2f} s wall"
        cpu = {"value": o / dt / 1e12, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample}

    if rank == 0:
        pack_gbs = {o.name: o.bytes / (per_op[o.name] / 1e3) / 1e9 for o in ops if o.kind == "pack"}
        speed = None
        if cub_ms:
            speed = {"matmuls_only": cublas_total / bwta_mm_only if bwta_mm_only else None,
                     "incl_activation_pack": cublas_total / (bwta_mm_only + pack_ms),
                     "whole_step": cublas_total / ms_step,
                     "per_op": {n: cub_ms[n] / per_op[n] for n in cub_ms}}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": scaling,
            "vs_baseline": None, "dtype": "fp4-e2m1 codes (tcgen05 kind::mxf4, f32 accumulate; fp16 in/out)",
            "data": "synthetic (seeded, recipe in DESIGN.md)",
            "config": W["cfg"],
            "parallelism": W.get("parallelism", f"replicas x{world}" if world > 1 else "single GPU"),
            "timing": {"l2": "256 MiB read (clean eviction) between steps, outside the timed events",
                       "launch": "CUDA graph of the step" if use_graph else "eager launches (NCCL in the step)",
                       "clock_window": "nvidia-smi every 20 ms over >= 0.5 s of warm-up load + the timed steps"},
            "clocks": clk.summary(), "gpu_launches": launches_per_step * args.steps,
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "speedup_vs_cublas_fp16": speed,
            "per_op_us": {k: v * 1e3 for k, v in per_op.items()},
            "in_step_us": {k: v * 1e3 for k, v in in_step.items()},
            "in_graph_us": {k: v * 1e3 for k, v in in_graph.items()},
            "cublas_fp16_us": {k: v * 1e3 for k, v in cub_ms.items()},
            "other_designs_us": {k: {a: t * 1e3 for a, t in v.items()} for k, v in alt_ms.items()},
            "pack_GBps": pack_gbs, "extras": extras,
        }
        if world > 1 or args.nshard:
            line["comm"] = {"backend": "nccl", "nccl_version": ".".join(map(str, torch.cuda.nccl.version())),
                            "collective": "all_gather_into_tensor (in place, async, per chunk)"}
        print(json.dumps(line))
    if world > 1 or args.nshard:
        torch.distributed.destroy_process_group()
    return 0


def _traffic(op_name, workload):
    """dram bytes per launch of the dominant op from the committed ncu summary, if any."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        return d.get(workload, {}).get(op_name)
    except Exception:
        return None


if __name__ == "__main__":
    sys.exit(main())
