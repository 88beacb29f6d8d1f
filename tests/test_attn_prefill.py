"""Fused prefill attention (bwta_attn_prefill) against the oracle's
composition of the paper's steps, row by row (oracle.attn_decode applied to every query
row: QK^T -> float64 softmax rounded to p_dt -> bool quantizer
 -> PV).  Reading R13: the kernel's softmax is fp32
(table of exp(alpha d) for the normaliser, R13's expression for the threshold), so a bit of
P may differ from the oracle's only where p lies within rounding distance of s_att / 2; the
test accepts exactly that, counts it, and requires O to be equal wherever P agrees."""
import ctypes

import numpy as np
import pytest
import torch

import bwta_inputs as gen
import oracle
from test_parity_gpu import B, DT, out_storage, storage, words  # noqa: F401

CASES = [  # b, h, tq, tk, dh, binary K, p dtype, alpha sign
    (1, 2, 128, 128, 128, False, torch.float16, 1),
    (2, 3, 130, 300, 64, False, torch.bfloat16, 1),
    (1, 1, 37, 41, 128, True, torch.float16, 1),
    (1, 2, 257, 1000, 96, False, torch.float32, 1),
    (2, 2, 300, 129, 16, False, torch.float16, 1),
    (1, 2, 200, 333, 128, False, torch.float16, -1),
    (1, 1, 5, 2100, 128, False, torch.float16, 1),
]


def _oracle_rows(oq, ok, ov, alpha, s_att, pname, beta, out, causal=False):
    """oracle.attn_decode over every query row (K and V^T repeated per row); causal: row i sees
    keys j <= i + Tk - Tq (the oracle's nkeys mask)."""
    bh, tq, dh = oq.shape
    tk = ok.shape[1]
    qq = oq.reshape(bh * tq, dh)
    kk = np.repeat(ok, tq, axis=0)
    vv = np.repeat(ov, tq, axis=0)
    nk = np.tile(np.arange(tq) + (tk - tq) + 1, bh) if causal else None
    return oracle.attn_decode(qq, kk, vv, alpha, s_att, pname, beta, out, threads=oracle.default_threads(), nkeys=nk)


@pytest.mark.gpu
@pytest.mark.parametrize("case", range(len(CASES)))
def test_attn_prefill_parity(B, case):
    b, h, tq, tk, dh, kbin, p_dt, sgn = CASES[case]
    seed = 9500 + 10 * case
    q = gen.activations((b, h, tq, dh), seed)
    k = gen.activations((b, h, tk, dh), seed + 1)
    v = gen.activations((b, h, tk, dh), seed + 2)
    sq, sk, sv = gen.act_scale(q), gen.act_scale(k), gen.act_scale(v)
    alpha = float(np.float32(sgn * sq * sk / np.sqrt(dh)))
    s_att = float(np.float32(2.0 / tk))
    beta = float(np.float32(s_att * sv))
    qp = B.bwta_pack_act(q.cuda(), sq, "ternary")
    if kbin:
        kb = B.bwta_pack_weight(k.reshape(-1, dh).cuda())
        kp = type(qp)(kb.sgn.reshape(b, h, tk, -1), None, "binary", dh)
    else:
        kp = B.bwta_pack_act(k.cuda(), sk, "ternary")
    vt = B.bwta_pack_act(v.cuda(), sv, "ternary", transpose=True)
    pname = DT[p_dt]
    o16, pbits = B.bwta_attn_prefill(qp, kp, vt, alpha, s_att, beta, torch.float16, p_dt, return_p=True)
    oi = B.bwta_attn_prefill(qp, kp, vt, alpha, s_att, beta, torch.int32, p_dt)
    oq = oracle.quantize_act(storage(q).reshape(b * h, tq, dh), "f16", sq, "ternary")
    if kbin:
        ok = oracle.binarize_weight(storage(k).reshape(-1, dh), "f16").reshape(b * h, tk, dh)
    else:
        ok = oracle.quantize_act(storage(k).reshape(b * h, tk, dh), "f16", sk, "ternary")
    ov = oracle.quantize_act(storage(v).reshape(b * h, tk, dh), "f16", sv, "ternary")
    ref_i, pb, p64 = _oracle_rows(oq, ok, ov, alpha, s_att, pname, beta, "i32")
    ref_16, _, _ = _oracle_rows(oq, ok, ov, alpha, s_att, pname, beta, "f16")
    got_bits = oracle.unpack(None, words(pbits).reshape(b * h * tq, -1), "bool", tk).astype(np.int8)
    diff = got_bits != pb
    t = s_att / 2
    assert np.all(np.abs(p64[diff] / t - 1.0) < 2.0 ** -8), "P differs away from the threshold"
    flips = diff.sum(axis=1)
    gi = oi.cpu().numpy().reshape(b * h * tq, dh)
    assert np.all(np.abs(gi - ref_i) <= flips[:, None])
    g16 = out_storage(o16).reshape(b * h * tq, dh)
    same = flips == 0
    assert np.array_equal(g16[same], ref_16[same])
    assert pb.sum() > 0 and flips.sum() <= max(2, pb.size // 10000)
    # the unfused library path on the same P bits gives the same O (exact integer PV)
    pp = type(qp)(None, pbits.reshape(b, h, tq, -1), "bool", tk)
    o_unf = B.bwta_attn_pv(pp, vt, beta, out_dtype=torch.int32)
    assert torch.equal(o_unf.reshape(-1, dh).cpu(), oi.reshape(-1, dh).cpu())


@pytest.mark.gpu
def test_attn_prefill_strided_heads_and_out_view(B):
    """Q/K/V as per-head views of a [B, T, 3*H*D] projection output; O written into the
    [B, T, H*D] context layout through a strided view."""
    Bsz, T, H, D = 2, 150, 3, 64
    qkv = gen.activations((Bsz, T, 3 * H * D), 9901).cuda()
    views = [qkv[..., j * H * D:(j + 1) * H * D].unflatten(-1, (H, D)).transpose(1, 2) for j in range(3)]
    s = [gen.act_scale(x) for x in views]
    qp, kp = B.bwta_pack_act(views[0], s[0]), B.bwta_pack_act(views[1], s[1])
    vt = B.bwta_pack_act(views[2], s[2], transpose=True)
    alpha = float(np.float32(s[0] * s[1] / 8.0))
    s_att = float(np.float32(2.0 / T))
    beta = float(np.float32(s_att * s[2]))
    ctx = torch.zeros((Bsz, T, H * D), dtype=torch.float16, device="cuda")
    ctx_v = ctx.view(Bsz, T, H, D).transpose(1, 2)
    B.bwta_attn_prefill(qp, kp, vt, alpha, s_att, beta, out=ctx_v)
    ref = B.bwta_attn_prefill(qp, kp, vt, alpha, s_att, beta)
    assert torch.equal(ctx_v.contiguous().view(torch.int16), ref.view(torch.int16))


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["ternary", "bool"])
@pytest.mark.parametrize("o_dtype", [torch.float16, torch.bfloat16])
def test_attn_prefill_pack_equals_prefill_then_pack(B, kind, o_dtype):
    """bwta_attn_prefill_pack == bwta_pack_act(context of bwta_attn_prefill) bit-exactly (the
    fused epilogue rounds to o_dtype exactly like the stored context), ragged Tq / Tk, Dh 32-128."""
    for i, (b, h, tq, tk, dh) in enumerate([(2, 3, 37, 41, 64), (1, 2, 130, 300, 128), (4, 12, 128, 128, 64),
                                            (1, 5, 200, 129, 32)]):
        seed = 9700 + 10 * i
        q, k, v = (gen.activations((b, h, t, dh), seed + j) for j, t in enumerate((tq, tk, tk)))
        sq, sk, sv = gen.act_scale(q), gen.act_scale(k), gen.act_scale(v)
        alpha = float(np.float32(sq * sk / np.sqrt(dh)))
        s_att = float(np.float32(2.0 / tk))
        beta = float(np.float32(s_att * sv))
        qp, kp = B.bwta_pack_act(q.cuda(), sq), B.bwta_pack_act(k.cuda(), sk)
        vt = B.bwta_pack_act(v.cuda(), sv, "ternary", transpose=True)
        o = B.bwta_attn_prefill(qp, kp, vt, alpha, s_att, beta, out_dtype=o_dtype)
        ctx = o.transpose(1, 2).reshape(b * tq, h * dh).contiguous()
        s_ctx = gen.act_scale(ctx) or 1.0
        ref = B.bwta_pack_act(ctx, s_ctx, kind)
        got = B.bwta_attn_prefill_pack(qp, kp, vt, alpha, s_att, beta, s_ctx, kind, o_dtype=o_dtype)
        assert torch.equal(got.nz, ref.nz), (b, h, tq, tk, dh)
        if kind == "ternary":
            assert torch.equal(got.sgn, ref.sgn), (b, h, tq, tk, dh)


def test_attn_prefill_validation():
    """Host validation before any device work (no GPU here)."""
    from paper_2604_03957_b200 import _native as N
    L = N.lib

    def pf(**kw):
        a = dict(qs=16, qn=32, ks=48, kn=64, vs=80, vn=96, b=1, h=2, tq=10, tk=100, dh=64, ldq=4, ldk=4, ldv=4,
                 alpha=0.1, s_att=0.02, p_dt=0, beta=0.1, o=112, o_dt=0, ld_o=64, pout=None, ldp=0)
        a.update(kw)
        return L.bwta_attn_prefill(a["qs"], a["qn"], a["ks"], a["kn"], a["vs"], a["vn"], a["b"], a["h"], a["tq"],
                                   a["tk"], a["dh"], a["ldq"], 0, 0, a["ldk"], 0, 0, a["ldv"], 0, 0,
                                   ctypes.c_float(a["alpha"]), ctypes.c_float(a["s_att"]), a["p_dt"],
                                   ctypes.c_float(a["beta"]), None, None, a["o"], a["o_dt"], a["ld_o"], 0, 0, a["pout"],
                                   a["ldp"],
                                   None)
    assert pf() == 4                     # valid, but no sm_100 device here
    assert pf(dh=129) == 4               # one 128-element tensor-core stage per row
    assert pf(tk=0) == 2                 # softmax over an empty row
    assert pf(ldv=0) == 2
    assert pf(ld_o=63) == 2
    assert pf(pout=128, ldp=0) == 2
    assert pf(ldk=5) == 3
    assert pf(ks=20) == 3
    assert pf(qs=None) == 1
    assert pf(o=None) == 1
    assert pf(s_att=0.0) == 1
    assert pf(alpha=float("inf")) == 1
    assert pf(p_dt=3) == 4
    assert pf(kn=None) == 4              # binary K is valid
    assert pf(b=0) == 0 and pf(tq=0) == 0

    def pfp(**kw):
        a = dict(qs=16, qn=32, ks=48, kn=64, vs=80, vn=96, b=1, h=2, tq=10, tk=100, dh=64, o_dt=0, s_o=1.0, kind=2,
                 os_=112, on=128, ldo=4)
        a.update(kw)
        return L.bwta_attn_prefill_pack(a["qs"], a["qn"], a["ks"], a["kn"], a["vs"], a["vn"], a["b"], a["h"], a["tq"],
                                        100, a["dh"], 4, 0, 0, 4, 0, 0, 4, 0, 0, ctypes.c_float(0.1),
                                        ctypes.c_float(0.02), 0, ctypes.c_float(0.1), None, None, a["o_dt"],
                                        ctypes.c_float(a["s_o"]),
                                        a["kind"], a["os_"], a["on"], a["ldo"], None)
    assert pfp() == 4                    # valid, but no sm_100 device here
    assert pfp(dh=48) == 4               # a head must own whole words of the context row
    assert pfp(o_dt=2) == 4              # the pack rounds to f16 / bf16
    assert pfp(kind=0) == 4
    assert pfp(on=None) == 1
    assert pfp(kind=1) == 1              # bool output has no sgn plane
    assert pfp(s_o=0.0) == 1
    assert pfp(ldo=0) == 2
    assert pfp(on=132) == 3


@pytest.mark.gpu
def test_attn_per_head_scales(B):
    """Per-head alpha / beta: one call with alpha_heads / beta_heads equals the
    per-head calls with the scalar alpha_h / beta_h bit for bit (prefill, prefill + context pack,
    decode), including a head with a negative alpha."""
    b, h, tq, tk, dh = 2, 4, 130, 300, 64
    q, k, v = (gen.activations((b, h, t, dh), 9900 + j) for j, t in enumerate((tq, tk, tk)))
    qp, kp = B.bwta_pack_act(q.cuda(), 1.3), B.bwta_pack_act(k.cuda(), 1.2)
    vt = B.bwta_pack_act(v.cuda(), 1.1, "ternary", transpose=True)
    s_att = float(np.float32(2.0 / tk))
    ah = [0.11, -0.07, 0.23, 0.05]
    bh = [0.01, 0.02, 0.015, 0.03]
    o = B.bwta_attn_prefill(qp, kp, vt, 1.0, s_att, 1.0, alpha_heads=ah, beta_heads=bh)
    for hh in range(h):
        sub = lambda P: type(P)(None if P.sgn is None else P.sgn[:, hh:hh + 1], P.nz[:, hh:hh + 1], P.kind, P.cols)
        ref = B.bwta_attn_prefill(sub(qp), sub(kp), sub(vt), ah[hh], s_att, bh[hh])
        assert torch.equal(o[:, hh:hh + 1].view(torch.int16), ref.view(torch.int16)), hh
    # decode (one query row per head)
    q1 = B.bwta_pack_act(gen.activations((b, h, 1, dh), 9950).cuda(), 1.3)
    od = B.bwta_attn_decode(q1, kp, vt, 1.0, s_att, 1.0, alpha_heads=ah, beta_heads=bh)
    for hh in range(h):
        sub = lambda P: type(P)(None if P.sgn is None else P.sgn[:, hh:hh + 1], P.nz[:, hh:hh + 1], P.kind, P.cols)
        ref = B.bwta_attn_decode(sub(q1), sub(kp), sub(vt), ah[hh], s_att, bh[hh])
        assert torch.equal(od[:, hh:hh + 1].view(torch.int16), ref.view(torch.int16)), hh
    # the fused context pack with per-head scales == pack of the per-head-scaled context
    ctx = o.transpose(1, 2).reshape(b * tq, h * dh).contiguous()
    s_ctx = gen.act_scale(ctx) or 1.0
    got = B.bwta_attn_prefill_pack(qp, kp, vt, 1.0, s_att, 1.0, s_ctx, alpha_heads=ah, beta_heads=bh)
    ref = B.bwta_pack_act(ctx, s_ctx)
    assert torch.equal(got.nz, ref.nz) and torch.equal(got.sgn, ref.sgn)


CAUSAL_CASES = [  # b, h, tq, tk, dh, binary K, p dtype
    (1, 2, 128, 128, 128, False, torch.float16),
    (2, 2, 300, 300, 64, False, torch.bfloat16),
    (1, 1, 130, 400, 128, True, torch.float16),
    (1, 2, 257, 1100, 96, False, torch.float32),
    (1, 1, 5, 2100, 128, False, torch.float16),
]


@pytest.mark.gpu
@pytest.mark.parametrize("case", range(len(CAUSAL_CASES)))
def test_attn_prefill_causal_parity(B, case):
    """causal = 1 (bwta_attn_prefill_ex): row i sees keys j <= i + Tk - Tq; against the oracle's
    masked composition under R13's counted tolerance, masked P bits exactly zero, O equal where P
    agrees, and the unfused PV of the kernel's own P bits equal to its O."""
    b, h, tq, tk, dh, kbin, p_dt = CAUSAL_CASES[case]
    seed = 9700 + 10 * case
    q = gen.activations((b, h, tq, dh), seed)
    k = gen.activations((b, h, tk, dh), seed + 1)
    v = gen.activations((b, h, tk, dh), seed + 2)
    sq, sk, sv = gen.act_scale(q), gen.act_scale(k), gen.act_scale(v)
    alpha = float(np.float32(sq * sk / np.sqrt(dh)))
    s_att = float(np.float32(2.0 / tk))
    beta = float(np.float32(s_att * sv))
    qp = B.bwta_pack_act(q.cuda(), sq, "ternary")
    if kbin:
        kb = B.bwta_pack_weight(k.reshape(-1, dh).cuda())
        kp = type(qp)(kb.sgn.reshape(b, h, tk, -1), None, "binary", dh)
    else:
        kp = B.bwta_pack_act(k.cuda(), sk, "ternary")
    vt = B.bwta_pack_act(v.cuda(), sv, "ternary", transpose=True)
    pname = DT[p_dt]
    o16, pbits = B.bwta_attn_prefill(qp, kp, vt, alpha, s_att, beta, torch.float16, p_dt, return_p=True, causal=True)
    oi = B.bwta_attn_prefill(qp, kp, vt, alpha, s_att, beta, torch.int32, p_dt, causal=True)
    oq = oracle.quantize_act(storage(q).reshape(b * h, tq, dh), "f16", sq, "ternary")
    if kbin:
        ok = oracle.binarize_weight(storage(k).reshape(-1, dh), "f16").reshape(b * h, tk, dh)
    else:
        ok = oracle.quantize_act(storage(k).reshape(b * h, tk, dh), "f16", sk, "ternary")
    ov = oracle.quantize_act(storage(v).reshape(b * h, tk, dh), "f16", sv, "ternary")
    ref_i, pb, p64 = _oracle_rows(oq, ok, ov, alpha, s_att, pname, beta, "i32", causal=True)
    ref_16, _, _ = _oracle_rows(oq, ok, ov, alpha, s_att, pname, beta, "f16", causal=True)
    got_bits = oracle.unpack(None, words(pbits).reshape(b * h * tq, -1), "bool", tk).astype(np.int8)
    rows = np.tile(np.arange(tq), b * h)
    masked = np.arange(tk)[None, :] > (rows + tk - tq)[:, None]
    assert got_bits[masked].sum() == 0, "a masked key got a P bit"
    diff = got_bits != pb
    t = s_att / 2
    assert np.all(np.abs(p64[diff] / t - 1.0) < 2.0 ** -8), "P differs away from the threshold"
    flips = diff.sum(axis=1)
    gi = oi.cpu().numpy().reshape(b * h * tq, dh)
    assert np.all(np.abs(gi - ref_i) <= flips[:, None])
    g16 = out_storage(o16).reshape(b * h * tq, dh)
    same = flips == 0
    assert np.array_equal(g16[same], ref_16[same])
    assert pb.sum() > 0 and flips.sum() <= max(2, pb.size // 10000)
    pp = type(qp)(None, pbits.reshape(b, h, tq, -1), "bool", tk)
    o_unf = B.bwta_attn_pv(pp, vt, beta, out_dtype=torch.int32)
    assert torch.equal(o_unf.reshape(-1, dh).cpu(), oi.reshape(-1, dh).cpu())


@pytest.mark.gpu
def test_attn_prefill_causal_rejects_tk_below_tq(B):
    q = B.bwta_pack_act(gen.activations((1, 1, 64, 64), 1).cuda(), 1.0)
    k = B.bwta_pack_act(gen.activations((1, 1, 32, 64), 2).cuda(), 1.0)
    vt = B.bwta_pack_act(gen.activations((1, 1, 32, 64), 3).cuda(), 1.0, transpose=True)
    with pytest.raises(B.BwtaError):
        B.bwta_attn_prefill(q, k, vt, 0.1, 0.05, 0.1, causal=True)
