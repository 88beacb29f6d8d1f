"""GPU parity on the paths the timed bench and the ABI actually take, at the
sizes where a mistake would hide from the small cases (round-2 additions):

  * R12: the tensor-core path accumulates E2M1 products in FP32 and
    relies on every partial sum being exact up to the ABI's K cap of 2^24.
    Random operands keep |dot| ~ sqrt(K); here operands are periodic with a
    bias towards agreement, so |dot| reaches K (all-agree / all-disagree rows)
    and odd values with every low bit set at every magnitude.  Expected values
    are the closed form of a periodic sum (no oracle call is needed at 2^24):
        dot = floor(K / L) * S(L) + S(K mod L),   S(n) = sum_{k<n} a[k mod P_A] w[k mod P_W]
    with L = lcm(P_A, P_W) -- checked against the oracle at small K first.
  * the lean grouped row pack (pack_group_rows_kernel) the BERT step uses;
  * configs[4]'s tile path (M 2048, K 8192, N 28672, Y^T) on sampled rows;
  * configs[3] (C4) QK^T / PV and configs[1]'s 384-entry QK^T on sampled entries.
"""
import math

import numpy as np
import pytest
import torch

import bwta_inputs as gen
import oracle
from test_parity_gpu import B, DT, assert_out_equal, inject_specials, storage, tie_scale, words  # noqa: F401

gpu = pytest.mark.gpu

PA, PW = 96, 160          # periods (elements) of the A and W patterns; multiples of 32
L = PA * PW // math.gcd(PA, PW)   # 480


def _bits_to_words(bits: np.ndarray) -> np.ndarray:
    """[R, 32*w] {0,1} -> uint32 [R, w], element c -> bit c % 32 of word c // 32 (R8)."""
    r, c = bits.shape
    b = bits.reshape(r, c // 32, 32).astype(np.uint64)
    return (b << np.arange(32, dtype=np.uint64)).sum(-1).astype(np.uint32)


def _periodic_planes(period_codes: np.ndarray, K: int, kind: str):
    """Planes (device int32 [R, ld]) of rows whose codes repeat period_codes [R, P] along K."""
    R, P = period_codes.shape
    ld = oracle.ld_words(K)
    nw = (K + 31) // 32
    pw = P // 32
    sgn_p = _bits_to_words(period_codes < 0)
    nz_p = _bits_to_words(period_codes != 0)
    idx = torch.arange(nw, device="cuda") % pw
    out = []
    for pat in ((sgn_p, nz_p) if kind == "ternary" else (sgn_p,)):
        t = torch.from_numpy(pat.view(np.int32)).cuda()[:, idx]
        if K % 32:
            t[:, -1] &= (1 << (K % 32)) - 1
        full = torch.zeros((R, ld), dtype=torch.int32, device="cuda")
        full[:, :nw] = t
        out.append(full)
    return out


def _periodic_case(M, N, seed):
    """A period codes [M, PA] (ternary) and W period codes [N, PW] (binary), biased so
    that some dots reach +-K and the rest spread over the whole range, odd and even."""
    rng = np.random.default_rng(seed)
    # a common sign pattern of period 32 = gcd(PA, PW): unmodified A and W rows agree everywhere
    base = np.where(rng.random(32) < 0.5, -1, 1).astype(np.int8)
    w = np.tile(base, (N, PW // 32))
    for j in range(N):
        f = [0.0, 0.0, 1.0, 0.5, 0.01, 0.1][j % 6] if j < 6 else rng.choice([0.0, 0.002, 0.02, 0.3, 0.5, 0.9, 1.0])
        flip = rng.random(PW) < f
        w[j, flip] *= -1
    # A rows: agree with base[:PA] except flips, with some zeros
    a = np.tile(base, (M, PA // 32))
    for i in range(M):
        if i < 4:
            zf, ff = 0.0, [0.0, 1.0, 0.0, 0.0][i]
            if i == 2:
                zf = 1.0 / PA        # exactly one zero per period -> odd dots
        else:
            zf = rng.choice([0.0, 0.0, 0.01, 0.05, 0.3, 0.6])
            ff = rng.choice([0.0, 0.0, 0.01, 0.1, 0.5, 1.0])
        z = rng.random(PA) < zf
        if i == 2:
            z[:] = False
            z[7] = True
        fl = rng.random(PA) < ff
        a[i, fl] *= -1
        a[i, z] = 0
    return a, w


def _closed_form_dot(a_per: np.ndarray, w_per: np.ndarray, K: int) -> np.ndarray:
    aL = np.tile(a_per, (1, L // PA)).astype(np.int64)
    wL = np.tile(w_per, (1, L // PW)).astype(np.int64)
    full, rem = divmod(K, L)
    d = full * (aL @ wL.T)
    if rem:
        d += aL[:, :rem] @ wL[:, :rem].T
    return d


def test_closed_form_matches_oracle_small_k():
    """The closed form used below equals the oracle's triple loop (K spans several periods + a tail)."""
    a, w = _periodic_case(9, 7, 11)
    for K in (1, 95, 480, 1000, 4097):
        qa = np.tile(a, (1, -(-K // PA)))[:, :K]
        qw = np.tile(w, (1, -(-K // PW)))[:, :K]
        assert np.array_equal(_closed_form_dot(a, w, K), oracle.dot(qa, qw).astype(np.int64)), K


R12_K = [8192, 11008, 65536, 1 << 20, (1 << 24) - 32]


@gpu
@pytest.mark.parametrize("K", R12_K)
def test_r12_large_k_accumulator_exact(B, K):
    """tcgen05 kind::mxf4 + FP32 accumulation reproduces the integer dot exactly up to the ABI's
    K cap: |dot| up to K (all-agree, all-disagree) and odd values near K, on every design-(b)
    tile / CTA-pair shape, both orientations, the skinny tcgen05 kernel and the CUDA-core GEMV."""
    M = N = 256
    a_per, w_per = _periodic_case(M, N, 1234 + K % 1000)
    ref = _closed_form_dot(a_per, w_per, K)
    assert np.abs(ref).max() == K                       # rows 0/1 x W row 0: all agree / all disagree
    assert (np.abs(ref) > K // 2).sum() > 1000 and (ref % 2 == 1).sum() > 1000
    a_sgn, a_nz = _periodic_planes(a_per, K, "ternary")
    (w_sgn,) = _periodic_planes(w_per, K, "binary")
    import paper_2604_03957_b200 as Bm
    A = Bm.Packed(a_sgn, a_nz, "ternary", K)
    W = Bm.Packed(w_sgn, None, "binary", K)
    ref32 = ref.astype(np.int32)
    for tile in [None, (64, 1), (128, 1), (192, 1), (64, 2), (128, 2), (192, 2)]:
        y = B.bwta_gemm(A, W, None, 1.0, out_dtype=torch.int32, design="tcgen05", tile=tile)
        assert np.array_equal(y.cpu().numpy(), ref32), (K, tile)
        del y
    # swapped orientation (A on the MMA N side): M > N
    Wn = Bm.Packed(w_sgn[:100], None, "binary", K)
    y = B.bwta_gemm(A, Wn, None, 1.0, out_dtype=torch.int32, design="tcgen05")
    assert np.array_equal(y.cpu().numpy(), ref32[:, :100]), (K, "swapped")
    # skinny: the <= 32-row tcgen05 kernel and the <= 4-row CUDA-core GEMV
    for m in (16, 32, 4, 1):
        As = Bm.Packed(a_sgn[:m], a_nz[:m], "ternary", K)
        for design in ("tcgen05", "auto"):
            y = B.bwta_gemm(As, W, None, 1.0, out_dtype=torch.int32, design=design)
            assert np.array_equal(y.cpu().numpy(), ref32[:m]), (K, m, design)
    # fp32 output: exact integer times 1.0 (R5)
    y = B.bwta_gemm(A, W, None, 1.0, out_dtype=torch.float32)
    assert np.array_equal(y.cpu().numpy(), ref.astype(np.float32)), (K, "f32")


# ----------------------------------------------------- lean grouped row pack ----
@gpu
@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16, torch.float32])
@pytest.mark.parametrize("kind", ["ternary", "bool"])
@pytest.mark.parametrize("n", [2, 3, 4])
def test_pack_group_lean_rows(B, dtype, kind, n):
    """bwta_pack_act_batch with 2-4 row packs of one kind (the one-body pack_group_rows_kernel the
    BERT step uses for Q + K) == the oracle, with ties / +-0 / +-inf / NaN / tiny values, per-head
    strided views (vector path) and an unaligned view set (scalar path), ragged columns."""
    Bsz, T, H, D = 2, 37, 3, 64
    for aligned in (True, False):
        extra = 0 if aligned else 1
        base = gen.activations((Bsz, T, 4 * H * D + extra), 1300 + n, dtype)
        s_list = [tie_scale(dtype, 1310 + j) for j in range(n)]
        base = inject_specials(base, s_list[0], 1320 + n)
        base = base.cuda()
        off = extra
        views = [base[:, :, off + j * H * D: off + (j + 1) * H * D].unflatten(-1, (H, D)).transpose(1, 2)
                 for j in range(n)]
        items = [(v, s, kind, False) for v, s in zip(views, s_list)]
        got = B.bwta_pack_act_batch(items)
        for (x, s, _, _), g in zip(items, got):
            sgn, nz, _ = oracle.pack_act(storage(x.contiguous()).reshape(-1, T, D), DT[dtype], s, kind)
            assert np.array_equal(words(g.nz).reshape(nz.shape), nz), (aligned, s)
            if kind == "ternary":
                assert np.array_equal(words(g.sgn).reshape(sgn.shape), sgn), (aligned, s)
    # ragged 2-D members (cols not a multiple of 32, different row counts)
    xs = [inject_specials(gen.activations((r, c), 1350 + r, dtype), 1.0, r).cuda()
          for r, c in [(5, 33), (70, 257), (3, 1000), (130, 129)][:n]]
    got = B.bwta_pack_act_batch([(x, 1.0, kind, False) for x in xs])
    for x, g in zip(xs, got):
        sgn, nz, _ = oracle.pack_act(storage(x), DT[dtype], 1.0, kind)
        assert np.array_equal(words(g.nz), nz)
        if kind == "ternary":
            assert np.array_equal(words(g.sgn), sgn)


@gpu
def test_pack_group_bert_qk_shape(B):
    """The exact Q + K group of the timed BERT step (32 x 12 heads x 128 x 64 views of the QKV output)."""
    Bsz, T, H, D = 32, 128, 12, 64
    qkv = gen.activations((Bsz * T, 3 * H * D), 1400).cuda()
    views = [qkv[:, j * H * D:(j + 1) * H * D].view(Bsz, T, H, D).transpose(1, 2) for j in range(2)]
    s = [gen.act_scale(v) for v in views]
    got = B.bwta_pack_act_batch([(views[0], s[0], "ternary", False), (views[1], s[1], "ternary", False)])
    for v, sc, g in zip(views, s, got):
        sgn, nz, _ = oracle.pack_act(storage(v.contiguous()).reshape(-1, T, D), "f16", sc, "ternary")
        assert np.array_equal(words(g.nz).reshape(nz.shape), nz)
        assert np.array_equal(words(g.sgn).reshape(sgn.shape), sgn)


# ------------------------------------------------------- configs[4] tile path ----
@gpu
def test_configs4_full_size_transposed_sampled(B):
    """configs[4]'s largest linear (M 2048, K 8192, N 28672) with Y^T output, exactly the launch the
    N-shard bench times at world 1: sampled weight rows (= rows of Y^T) against the oracle."""
    M, K, N = 2048, 8192, 28672
    x = gen.activations((M, K), 707)
    w = gen.weights(N, K, 708)
    s_a = gen.act_scale(x)
    mu, s_w = gen.weight_stats(w)
    a = B.bwta_pack_act(x.cuda(), s_a, "ternary")
    wp = B.bwta_pack_weight(w.cuda(), mu=mu)
    yt = B.bwta_gemm(a, wp, s_w.cuda(), s_a, out_dtype=torch.float16, y_transposed=True)
    yi = B.bwta_gemm(a, wp, s_w.cuda(), s_a, out_dtype=torch.int32, y_transposed=True)
    rows = np.concatenate([np.random.default_rng(7).choice(N, 48, replace=False), [0, 127, 128, N - 1]])
    qa = oracle.quantize_act(storage(x), "f16", s_a, "ternary")
    qw = oracle.binarize_weight(storage(w[torch.from_numpy(rows)]), "f16", mu=mu)
    d = oracle.dot(qw, qa, threads=oracle.default_threads())          # [rows, M] = (Y^T) rows
    assert np.array_equal(yi.cpu().numpy()[rows], d)
    ref = oracle.epilogue_linear(d.T.copy(), s_w.numpy()[rows], s_a, "f16").T
    assert_out_equal(yt[torch.from_numpy(rows).cuda()], np.ascontiguousarray(ref), "configs[4] Y^T")


# ----------------------------------------------------------- attention at size ----
def _att_inputs(b, h, t, dh, seed):
    q = gen.activations((b, h, t, dh), seed)
    k = gen.activations((b, h, t, dh), seed + 1)
    v = gen.activations((b, h, t, dh), seed + 2)
    return q, k, v, gen.act_scale(q), gen.act_scale(k), gen.act_scale(v)


@gpu
@pytest.mark.parametrize("cfg", ["c4", "c2"])
def test_attention_full_size_sampled(B, cfg):
    """configs[3] (C4: 32 heads, T 2048, Dh 128) and configs[1]'s attention (C2: 384 entries,
    T 128, Dh 64) in the bench's launch configuration; sampled (entry, query row) outputs of QK^T
    and PV against the oracle -- at C2 every one of the 384 entries is sampled."""
    b, h, t, dh = (1, 32, 2048, 128) if cfg == "c4" else (32, 12, 128, 64)
    q, k, v, sq, sk, sv = _att_inputs(b, h, t, dh, 404 if cfg == "c4" else 202)
    alpha = float(np.float32(sq * sk / np.sqrt(dh)))
    s_att = float(np.float32(2.0 / t))
    beta = float(np.float32(s_att * sv))
    p = gen.attention_probs((b, h, t, t), 405 if cfg == "c4" else 203)
    qp, kp = B.bwta_pack_act(q.cuda(), sq), B.bwta_pack_act(k.cuda(), sk)
    vt = B.bwta_pack_act(v.cuda(), sv, transpose=True)
    pp = B.bwta_pack_act(p.cuda(), s_att, "bool")
    S = B.bwta_attn_qk(qp, kp, alpha).reshape(b * h, t, t)
    O = B.bwta_attn_pv(pp, vt, beta).reshape(b * h, t, dh)
    rng = np.random.default_rng(9)
    ents = np.arange(b * h) if cfg == "c2" else rng.choice(b * h, 6, replace=False)
    nrow = 8 if cfg == "c2" else 40
    qs, ks, vs, ps = (storage(z).reshape(b * h, z.shape[-2], z.shape[-1]) for z in (q, k, v, p))
    S_h, O_h = S.cpu(), O.cpu()
    for e in ents:
        rows = np.concatenate([rng.choice(t, nrow, replace=False), [0, t - 1]])
        oq = oracle.quantize_act(qs[e][rows], "f16", sq, "ternary")
        ok = oracle.quantize_act(ks[e], "f16", sk, "ternary")
        ref = oracle.attn_qk(oq[None], ok[None], alpha, "f16", threads=4)[0]
        assert_out_equal(S_h[e][torch.from_numpy(rows)], ref, f"{cfg} qk entry {e}")
        op = oracle.quantize_act(ps[e][rows], "f16", s_att, "bool")
        ov = oracle.quantize_act(vs[e], "f16", sv, "ternary")
        ref = oracle.attn_pv(op[None], ov[None], beta, "f16", threads=4)[0]
        assert_out_equal(O_h[e][torch.from_numpy(rows)], ref, f"{cfg} pv entry {e}")


@gpu
def test_configs2_grouped_linears_sampled(B):
    """configs[2] exactly as bench.py times it: both LLaMA-7B prefill linears (N 4096, 11008) in ONE
    launch over the row-concatenated weights with a per-row mu vector (each block keeps its own
    binarization); the two column blocks of Y equal the two separate launches bit for bit, and
    sampled output channels of each block equal the oracle."""
    M, K, Ns = 2048, 4096, (4096, 11008)
    x = gen.activations((M, K), 303)
    s_a = gen.act_scale(x)
    ws = [gen.weights(n, K, 304 + i) for i, n in enumerate(Ns)]
    stats = [gen.weight_stats(w) for w in ws]
    a = B.bwta_pack_act(x.cuda(), s_a, "ternary")
    mu_cat = torch.cat([torch.full((n,), float(mu), dtype=torch.float32) for n, (mu, _) in zip(Ns, stats)])
    wcat = B.bwta_pack_weight(torch.cat(ws).cuda(), mu=mu_cat.cuda())
    ycat = B.bwta_gemm(a, wcat, torch.cat([s for _, s in stats]).cuda(), s_a, out_dtype=torch.float16)
    qa = oracle.quantize_act(storage(x), "f16", s_a, "ternary")
    off = 0
    for n, w, (mu, s_w) in zip(Ns, ws, stats):
        sep = B.bwta_gemm(a, B.bwta_pack_weight(w.cuda(), mu=mu), s_w.cuda(), s_a, out_dtype=torch.float16)
        assert torch.equal(ycat[:, off:off + n], sep), f"grouped block N={n} != separate launch"
        cols = np.concatenate([np.random.default_rng(n).choice(n, 24, replace=False), [0, n - 1]])
        qw = oracle.binarize_weight(storage(w[torch.from_numpy(cols)]), "f16", mu=mu)
        d = oracle.dot(qa, qw, threads=oracle.default_threads())          # [M, cols]
        ref = oracle.epilogue_linear(d, s_w.numpy()[cols], s_a, "f16")
        assert_out_equal(ycat[:, torch.from_numpy(off + cols).cuda()], ref, f"grouped N={n} vs oracle")
        off += n
