"""GPU parity: the CUDA path (through the C ABI via the thin binding) against
the CPU oracle, element by element, on the same seeded inputs.

Bar (BASELINE.json north_star): packed planes, row counts and integer dots
bit-exact; FP16/BF16/FP32 outputs within 1e-3 relative (asserted here as
bit-exact, which is stronger: both sides evaluate the same R5 expression).
"""
import numpy as np
import pytest
import torch

import bwta_inputs as gen
import oracle

pytestmark = pytest.mark.gpu

DT = {torch.float16: "f16", torch.bfloat16: "bf16", torch.float32: "f32"}


@pytest.fixture(scope="module")
def B():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2604_03957_b200 as B
    return B


def storage(x: torch.Tensor) -> np.ndarray:
    x = x.detach().cpu().contiguous()
    if x.dtype in (torch.float16, torch.bfloat16):
        return x.view(torch.int16).numpy().view(np.uint16)
    return x.numpy()


def words(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().contiguous().numpy().view(np.uint32)


def out_storage(y: torch.Tensor) -> np.ndarray:
    y = y.detach().cpu().contiguous()
    if y.dtype in (torch.float16, torch.bfloat16):
        return y.view(torch.int16).numpy().view(np.uint16)
    return y.numpy()


def assert_out_equal(got: torch.Tensor, ref: np.ndarray, what=""):
    g = out_storage(got)
    if got.dtype == torch.float32:
        gi, ri = g.view(np.uint32), ref.view(np.uint32)
    else:
        gi, ri = g, ref
    bad = np.nonzero(gi != ri)
    if bad[0].size:
        # report the relative error too (the north-star bar is 1e-3)
        idx = tuple(b[:5] for b in bad)
        raise AssertionError(f"{what}: {bad[0].size} mismatches, first at {idx}: got {gi[idx]} ref {ri[idx]}")


def _bump(v: torch.Tensor, away: bool) -> torch.Tensor:
    """Next representable value of the same dtype, away from / toward zero (v finite, non-zero)."""
    it = {torch.float16: torch.int16, torch.bfloat16: torch.int16, torch.float32: torch.int32}[v.dtype]
    b = v.reshape(1).clone().view(it)
    b += 1 if away else -1        # sign-magnitude encoding: +-1 on the magnitude bits
    return b.view(v.dtype).reshape(())


def inject_specials(x: torch.Tensor, s: float, seed: int) -> torch.Tensor:
    """Put exact ties (+-s/2), their neighbours, +-0, +-inf, NaN and tiny values at random places."""
    x = x.clone()
    flat = x.view(-1)
    n = flat.numel()
    g = torch.Generator().manual_seed(seed)
    dt = x.dtype
    vals = [torch.tensor(0.0, dtype=dt), torch.tensor(-0.0, dtype=dt), torch.tensor(float("inf"), dtype=dt),
            torch.tensor(float("-inf"), dtype=dt), torch.tensor(float("nan"), dtype=dt),
            torch.tensor(1e-7, dtype=dt), torch.tensor(-1e-7, dtype=dt)]
    if s > 0:
        half = torch.tensor(s / 2, dtype=torch.float64).to(dt)
        assert float(half) == s / 2
        vals += [half, -half, _bump(half, True), _bump(half, False), _bump(-half, True), _bump(-half, False)]
    k = min(n, 4 * len(vals))
    pos = torch.randperm(n, generator=g)[:k]
    for i, p in enumerate(pos.tolist()):
        flat[p] = vals[i % len(vals)]
    return x


def tie_scale(dt, seed):
    # a scale whose half is exactly representable in every storage type
    g = torch.Generator().manual_seed(seed)
    return float(torch.tensor(0.5 + torch.rand(1, generator=g).item(), dtype=torch.bfloat16).float() * 2)


# ----------------------------------------------------------------- pack ----
SHAPES = [(1, 1), (3, 31), (5, 33), (7, 64), (9, 257), (64, 768), (33, 1000), (130, 129)]


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16, torch.float32])
@pytest.mark.parametrize("kind", ["ternary", "bool"])
@pytest.mark.parametrize("transpose", [False, True])
def test_pack_act_parity(B, dtype, kind, transpose):
    for i, (r, c) in enumerate(SHAPES):
        seed = 1000 + i
        s = tie_scale(dtype, seed)
        x = inject_specials(gen.activations((2, r, c), seed, dtype), s, seed)
        p = B.bwta_pack_act(x.cuda(), s, kind, transpose=transpose, row_nnz=True)
        sgn, nz, nnz = oracle.pack_act(storage(x), DT[dtype], s, kind, transpose=transpose)
        assert np.array_equal(words(p.nz), nz), (r, c)
        if kind == "ternary":
            assert np.array_equal(words(p.sgn), sgn), (r, c)
        else:
            assert p.sgn is None
        assert np.array_equal(p.row_nnz.cpu().numpy(), nnz), (r, c)


@pytest.mark.parametrize("transpose", [False, True])
def test_pack_act_strided_heads_and_unaligned(B, transpose):
    Bsz, T, H, D = 2, 37, 3, 64
    qkv = gen.activations((Bsz, T, 3 * H * D), 77).cuda()
    qkv1 = gen.activations((Bsz, T, 3 * H * D + 1), 78).cuda()
    s = 1.3
    # [B, H, T, D] view of the K third (aligned rows), and a view whose rows are
    # not 16-byte aligned (odd element offset and row stride): the scalar path
    for view in (qkv[:, :, H * D:2 * H * D].unflatten(-1, (H, D)).transpose(1, 2),
                 qkv1[:, :, 1:1 + H * D].unflatten(-1, (H, D)).transpose(1, 2)):
        p = B.bwta_pack_act(view, s, "ternary", transpose=transpose)
        sgn, nz, _ = oracle.pack_act(storage(view.contiguous()).reshape(Bsz * H, T, D), "f16", s, "ternary",
                                     transpose=transpose)
        assert np.array_equal(words(p.nz).reshape(nz.shape), nz)
        assert np.array_equal(words(p.sgn).reshape(sgn.shape), sgn)


def test_pack_act_batch_matches_single_calls(B):
    """bwta_pack_act_batch (one launch) == the individual packs == the oracle:
    strided per-head Q, K (rows), V^T (transposed) and a bool P with ragged sizes."""
    Bsz, T, H, D = 2, 37, 3, 64
    qkv = gen.activations((Bsz, T, 3 * H * D), 91).cuda()
    P = gen.attention_probs((Bsz, H, T, T), 92).cuda()
    views = [qkv[:, :, j * H * D:(j + 1) * H * D].unflatten(-1, (H, D)).transpose(1, 2) for j in range(3)]
    items = [(views[0], 1.1, "ternary", False), (views[1], 0.9, "ternary", False),
             (views[2], 1.3, "ternary", True), (P, 2.0 / T, "bool", False)]
    got = B.bwta_pack_act_batch(items)
    for (x, s, kind, tr), g in zip(items, got):
        ref = B.bwta_pack_act(x, s, kind, transpose=tr)
        assert torch.equal(g.nz, ref.nz)
        sgn, nz, _ = oracle.pack_act(storage(x.contiguous()).reshape(-1, x.shape[-2], x.shape[-1]), "f16", s, kind,
                                     transpose=tr)
        assert np.array_equal(words(g.nz).reshape(nz.shape), nz)
        if kind == "ternary":
            assert torch.equal(g.sgn, ref.sgn)
            assert np.array_equal(words(g.sgn).reshape(sgn.shape), sgn)
    assert B.bwta_pack_act_batch([]) == []


def test_pack_act_tiny_and_huge_scales(B):
    x = gen.activations((4, 300), 5, torch.float16)
    x[0, :8] = torch.tensor([6e-8, -6e-8, 1e-5, -1e-5, 65504, -65504, 3e-8, -3e-8], dtype=torch.float16)
    for s in (1e-7, 1.2e-7, 3e-5, 131000.0, 1e30, 2.0 ** -130):
        p = B.bwta_pack_act(x.cuda(), s, "ternary")
        sgn, nz, _ = oracle.pack_act(storage(x), "f16", s, "ternary")
        assert np.array_equal(words(p.nz), nz) and np.array_equal(words(p.sgn), sgn), s


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16, torch.float32])
def test_pack_weight_parity(B, dtype):
    for n, k, seed in ((1, 1, 1), (5, 33, 2), (17, 768, 3), (64, 1000, 4)):
        w = gen.weights(n, k, seed, dtype)
        w = inject_specials(w, 0.0, seed)
        mu_s = float(torch.tensor(0.001, dtype=torch.float32))
        for mu, per_row in ((None, False), (mu_s, False), ("row", True)):
            if mu == "row":
                mu_t = gen.normal((n,), seed + 9, torch.float32, std=0.01)
                p = B.bwta_pack_weight(w.cuda(), mu=mu_t.cuda() if n > 1 else mu_t.cuda())
                ref = oracle.pack_weight(storage(w), DT[dtype], mu=mu_t.numpy(), mu_per_row=n > 1)
            else:
                p = B.bwta_pack_weight(w.cuda(), mu=mu)
                ref = oracle.pack_weight(storage(w), DT[dtype], mu=mu)
            assert np.array_equal(words(p.sgn), ref), (n, k, mu)


# ----------------------------------------------------------------- gemm ----
GEMM_SHAPES = [(1, 1, 1), (7, 5, 31), (33, 17, 33), (129, 130, 100), (200, 129, 768), (64, 300, 1000),
               (300, 257, 257), (16, 2048, 2048)]


def _gemm_case(B, m, n, k, seed, a_kind="ternary"):
    x = (gen.relu_activations if a_kind == "bool" else gen.activations)((m, k), seed)
    w = gen.weights(n, k, seed + 1)
    s_a = gen.act_scale(x) or 1.0     # an all-zero tiny ReLU input has mean 0
    mu, s_w = gen.weight_stats(w)
    a = B.bwta_pack_act(x.cuda(), s_a, a_kind)
    wp = B.bwta_pack_weight(w.cuda(), mu=mu)
    qa = oracle.quantize_act(storage(x), "f16", s_a, a_kind)
    qw = oracle.binarize_weight(storage(w), "f16", mu=mu)
    return a, wp, s_a, s_w, qa, qw


@pytest.mark.parametrize("design", ["cuda_core", "tcgen05", "mma_b1"])
def test_gemm_parity(B, design):
    for i, (m, n, k) in enumerate(GEMM_SHAPES):
        for a_kind in ("ternary", "bool"):
            a, wp, s_a, s_w, qa, qw = _gemm_case(B, m, n, k, 2000 + i, a_kind)
            d = oracle.dot(qa, qw, threads=oracle.default_threads())
            yi = B.bwta_gemm(a, wp, s_w.cuda(), s_a, out_dtype=torch.int32, design=design)
            assert np.array_equal(yi.cpu().numpy(), d), (m, n, k, a_kind)
            for dt, name in ((torch.float16, "f16"), (torch.bfloat16, "bf16"), (torch.float32, "f32")):
                y = B.bwta_gemm(a, wp, s_w.cuda(), s_a, out_dtype=dt, design=design)
                assert_out_equal(y, oracle.epilogue_linear(d, s_w.numpy(), s_a, name), f"{m}x{n}x{k} {name}")
            yt = B.bwta_gemm(a, wp, s_w.cuda(), s_a, out_dtype=torch.float16, y_transposed=True, design=design)
            assert_out_equal(yt, oracle.epilogue_linear(d, s_w.numpy(), s_a, "f16").T.copy(), "transposed")
            # no weight scale -> 1
            y1 = B.bwta_gemm(a, wp, None, s_a, out_dtype=torch.float32, design=design)
            assert_out_equal(y1, oracle.epilogue_linear(d, None, s_a, "f32"), "no w_scale")


@pytest.mark.parametrize("tile", [(64, 1), (128, 1), (192, 1), (64, 2), (128, 2), (192, 2)])
def test_gemm_parity_every_tile(B, tile):
    """Every design-(b) tile shape (tile_n x CTA group), both operand roles
    (M < N: activations expanded; M > N: roles swapped, D^T epilogue), ragged
    M/N/K tails, per-column / per-row scales, both output orientations."""
    for i, (m, n, k, a_kind) in enumerate([(300, 517, 421, "ternary"), (517, 300, 421, "bool"),
                                           (130, 1000, 2000, "bool"), (1000, 130, 300, "ternary"),
                                           (300, 517, 128, "ternary"), (517, 300, 97, "bool")]):  # 128-K stages
        a, wp, s_a, s_w, qa, qw = _gemm_case(B, m, n, k, 2500 + i, a_kind)
        d = oracle.dot(qa, qw, threads=oracle.default_threads())
        yi = B.bwta_gemm(a, wp, s_w.cuda(), s_a, out_dtype=torch.int32, design="tcgen05", tile=tile)
        assert np.array_equal(yi.cpu().numpy(), d), (m, n, k, a_kind, tile)
        ref = oracle.epilogue_linear(d, s_w.numpy(), s_a, "f16")
        y = B.bwta_gemm(a, wp, s_w.cuda(), s_a, out_dtype=torch.float16, design="tcgen05", tile=tile)
        assert_out_equal(y, ref, f"{m}x{n}x{k} {tile}")
        yt = B.bwta_gemm(a, wp, s_w.cuda(), s_a, out_dtype=torch.float16, y_transposed=True, design="tcgen05",
                         tile=tile)
        assert_out_equal(yt, ref.T.copy(), f"{m}x{n}x{k} {tile} transposed")
        yb = B.bwta_gemm(a, wp, s_w.cuda(), s_a, out_dtype=torch.bfloat16, design="tcgen05", tile=tile)
        assert_out_equal(yb, oracle.epilogue_linear(d, s_w.numpy(), s_a, "bf16"), f"{m}x{n}x{k} {tile} bf16")


@pytest.mark.parametrize("tile", [None, (64, 1), (192, 2)])
def test_gemm_pack_fused_equals_gemm_then_pack(B, tile):
    """bwta_gemm_pack == bwta_pack_act(bwta_gemm(...)) bit-exactly (and == the
    oracle's quantization of the oracle's Y), both operand orientations,
    ternary and bool outputs, f16 and bf16 rounding, ragged N (padding bits
    and padding words), with and without per-channel scales."""
    for i, (m, n, k, a_kind) in enumerate([(300, 517, 421, "ternary"), (517, 300, 421, "bool"),
                                           (1000, 130, 300, "ternary"), (64, 2000, 768, "bool")]):
        a, wp, s_a, s_w, qa, qw = _gemm_case(B, m, n, k, 2700 + i, a_kind)
        d = oracle.dot(qa, qw, threads=oracle.default_threads())
        for y_dt, name in ((torch.float16, "f16"), (torch.bfloat16, "bf16")):
            for sw in (s_w, None):
                y = B.bwta_gemm(a, wp, None if sw is None else sw.cuda(), s_a, out_dtype=y_dt)
                yref = oracle.epilogue_linear(d, None if sw is None else sw.numpy(), s_a, name)
                s_out = float(torch.tensor(2.0) * y.float().abs().mean()) or 1.0
                for kind in ("ternary", "bool"):
                    got = B.bwta_gemm_pack(a, wp, None if sw is None else sw.cuda(), s_a, s_out, kind, y_dt,
                                           design="tcgen05", tile=tile)
                    ref = B.bwta_pack_act(y, s_out, kind)
                    assert torch.equal(got.nz, ref.nz), (m, n, k, name, kind)
                    if kind == "ternary":
                        assert torch.equal(got.sgn, ref.sgn), (m, n, k, name, kind)
                    osg, onz, _ = oracle.pack_act(yref, name, s_out, kind)
                    assert np.array_equal(words(got.nz), onz), (m, n, k, name, kind, "oracle")


def test_gemm_pack_rounding_ties(B):
    """Outputs placed exactly on the f16/bf16 rounding midpoint below the
    quantization threshold (and one float ulp either side): the fused pack
    must round-to-nearest-even first, like bwta_gemm + bwta_pack_act."""
    m, n, k = 256, 192, 300
    a, wp, s_a, s_w, qa, qw = _gemm_case(B, m, n, k, 2800)
    d = oracle.dot(qa, qw)
    for y_dt, name, t in ((torch.float16, "f16", 1.0), (torch.float16, "f16", 1.0009765625),
                          (torch.bfloat16, "bf16", 1.0), (torch.bfloat16, "bf16", 1.0078125)):
        prev = float(torch.tensor(t, dtype=y_dt).view(torch.int16).sub(1).view(y_dt).float())
        mid = (prev + t) / 2
        for lo in (np.nextafter(np.float32(mid), np.float32(0)), np.float32(mid), np.nextafter(np.float32(mid), np.float32(2))):
            sw = torch.full((n,), float(lo) / 4.0, dtype=torch.float32)     # y = lo exactly where dot = 4
            assert (d == 4).sum() > 0
            for kind in ("ternary", "bool"):
                got = B.bwta_gemm_pack(a, wp, sw.cuda(), 1.0, 2.0 * t, kind, y_dt, design="tcgen05")
                y = B.bwta_gemm(a, wp, sw.cuda(), 1.0, out_dtype=y_dt)
                ref = B.bwta_pack_act(y, 2.0 * t, kind)
                assert torch.equal(got.nz, ref.nz), (name, t, float(lo), kind)
                _, onz, _ = oracle.pack_act(oracle.epilogue_linear(d, sw.numpy(), 1.0, name), name, 2.0 * t, kind)
                assert np.array_equal(words(got.nz), onz), (name, t, float(lo), kind)


def test_gemm_tiny_scales(B):
    """Per-channel scales in the subnormal product range still follow R5 exactly."""
    m, n, k = 200, 300, 256
    a, wp, s_a, s_w, qa, qw = _gemm_case(B, m, n, k, 2600)
    d = oracle.dot(qa, qw)
    s_w = s_w.clone()
    s_w[::7] = torch.tensor(3e-36)  # subnormal-range products
    for dt, name in ((torch.float16, "f16"), (torch.float32, "f32")):
        y = B.bwta_gemm(a, wp, s_w.cuda(), s_a, out_dtype=dt, design="tcgen05")
        assert_out_equal(y, oracle.epilogue_linear(d, s_w.numpy(), s_a, name), name)


def test_gemm_exhaustive_k6(B):
    """All 3^6 ternary x 2^6 binary (and bool) vectors at K=6, also shifted to
    straddle a word boundary (offset 29): dot equals the oracle's triple loop."""
    tern = np.stack(np.meshgrid(*[np.array([-1, 0, 1])] * 6, indexing="ij"), -1).reshape(-1, 6).astype(np.int8)
    binv = np.stack(np.meshgrid(*[np.array([-1, 1])] * 6, indexing="ij"), -1).reshape(-1, 6).astype(np.int8)
    for off in (0, 29):
        K = off + 6
        qa = np.zeros((tern.shape[0], K), np.int8)
        qa[:, off:] = tern
        qw = np.ones((binv.shape[0], K), np.int8)
        qw[:, off:] = binv
        sa, na = oracle.pack(qa)
        sw, _ = oracle.pack(qw, want_nz=False)
        import paper_2604_03957_b200 as Bm
        a = Bm.Packed(torch.from_numpy(sa.view(np.int32)).cuda(), torch.from_numpy(na.view(np.int32)).cuda(),
                      "ternary", K)
        w = Bm.Packed(torch.from_numpy(sw.view(np.int32)).cuda(), None, "binary", K)
        for design in ("cuda_core", "tcgen05", "mma_b1"):
            y = B.bwta_gemm(a, w, None, 1.0, out_dtype=torch.int32, design=design)
            assert np.array_equal(y.cpu().numpy(), oracle.dot(qa, qw)), (off, design)


def test_gemm_k_zero_and_empty(B):
    import paper_2604_03957_b200 as Bm
    # K = 0: planes must still be valid pointers (the ABI rejects NULL); nothing is read
    a = Bm.Packed(torch.zeros((3, 4), dtype=torch.int32, device="cuda"),
                  torch.zeros((3, 4), dtype=torch.int32, device="cuda"), "ternary", 0)
    w = Bm.Packed(torch.zeros((2, 4), dtype=torch.int32, device="cuda"), None, "binary", 0)
    y = B.bwta_gemm(a, w, None, 2.0, out_dtype=torch.float32)
    assert torch.equal(y.cpu(), torch.zeros(3, 2))
    a0 = Bm.Packed(torch.zeros((0, 4), dtype=torch.int32, device="cuda"),
                   torch.zeros((0, 4), dtype=torch.int32, device="cuda"), "ternary", 100)
    w0 = Bm.Packed(torch.zeros((2, 4), dtype=torch.int32, device="cuda"), None, "binary", 100)
    assert B.bwta_gemm(a0, w0, None, 1.0).shape == (0, 2)


# ------------------------------------------------------------ attention ----
ATT = [(1, 1, 1, 1, 64), (2, 3, 37, 41, 64), (1, 2, 128, 128, 128), (2, 2, 130, 129, 33), (1, 1, 256, 300, 128)]


@pytest.mark.parametrize("design", ["cuda_core", "tcgen05", "mma_b1"])
def test_attention_parity(B, design):
    for i, (b, h, tq, tk, dh) in enumerate(ATT):
        seed = 3000 + 10 * i
        q = gen.activations((b, h, tq, dh), seed)
        k = gen.activations((b, h, tk, dh), seed + 1)
        v = gen.activations((b, h, tk, dh), seed + 2)
        sq, sk, sv = gen.act_scale(q), gen.act_scale(k), gen.act_scale(v)
        alpha = float(np.float32(sq * sk / np.sqrt(dh)))
        qp = B.bwta_pack_act(q.cuda(), sq, "ternary")
        kp = B.bwta_pack_act(k.cuda(), sk, "ternary")
        oq = oracle.quantize_act(storage(q).reshape(b * h, tq, dh), "f16", sq, "ternary")
        ok = oracle.quantize_act(storage(k).reshape(b * h, tk, dh), "f16", sk, "ternary")
        for dt, name in ((torch.int32, "i32"), (torch.float16, "f16"), (torch.float32, "f32")):
            s = B.bwta_attn_qk(qp, kp, alpha, out_dtype=dt, design=design)
            ref = oracle.attn_qk(oq, ok, alpha, name, threads=4).reshape(b, h, tq, tk)
            assert_out_equal(s, ref, f"qk {b,h,tq,tk,dh} {name}")
        # binary K (nz == all ones)
        kb = B.bwta_pack_weight(k.reshape(-1, dh).cuda())
        kbp = type(kp)(kb.sgn.reshape(b, h, tk, -1), None, "binary", dh)
        s = B.bwta_attn_qk(qp, kbp, 1.0, out_dtype=torch.int32, design=design)
        okb = oracle.binarize_weight(storage(k).reshape(-1, dh), "f16").reshape(b * h, tk, dh)
        assert_out_equal(s, oracle.attn_qk(oq, okb, 1.0, "i32").reshape(b, h, tq, tk), "qk binary K")
        # PV: P bool from synthetic softmax probabilities, V^T via the transposed pack
        p = gen.attention_probs((b, h, tq, tk), seed + 3)
        s_att = float(np.float32(2.0 / tk))
        beta = float(np.float32(s_att * sv))
        pp = B.bwta_pack_act(p.cuda(), s_att, "bool")
        vt = B.bwta_pack_act(v.cuda(), sv, "ternary", transpose=True)
        op = oracle.quantize_act(storage(p).reshape(b * h, tq, tk), "f16", s_att, "bool")
        ov = oracle.quantize_act(storage(v).reshape(b * h, tk, dh), "f16", sv, "ternary")
        for dt, name in ((torch.int32, "i32"), (torch.float16, "f16"), (torch.bfloat16, "bf16")):
            o = B.bwta_attn_pv(pp, vt, beta, out_dtype=dt, design=design)
            ref = oracle.attn_pv(op, ov, beta, name, threads=4).reshape(b, h, tq, dh)
            assert_out_equal(o, ref, f"pv {b,h,tq,tk,dh} {name}")


def test_attention_strided_heads_from_qkv(B):
    """Q/K/V as per-head views of a [B, T, 3*H*D] projection output (no copies)."""
    Bsz, T, H, D = 3, 128, 4, 64
    qkv = gen.activations((Bsz, T, 3 * H * D), 99).cuda()
    q = qkv[..., :H * D].unflatten(-1, (H, D)).transpose(1, 2)
    k = qkv[..., H * D:2 * H * D].unflatten(-1, (H, D)).transpose(1, 2)
    sq, sk = gen.act_scale(q), gen.act_scale(k)
    qp = B.bwta_pack_act(q, sq, "ternary")
    kp = B.bwta_pack_act(k, sk, "ternary")
    s = B.bwta_attn_qk(qp, kp, 0.25, out_dtype=torch.int32)
    oq = oracle.quantize_act(storage(q.contiguous()).reshape(-1, T, D), "f16", sq, "ternary")
    ok = oracle.quantize_act(storage(k.contiguous()).reshape(-1, T, D), "f16", sk, "ternary")
    assert np.array_equal(s.cpu().numpy().reshape(-1, T, T), oracle.attn_qk(oq, ok, 1.0, "i32"))


# ------------------------------------------------- full-size (bench) shapes ----
@pytest.mark.parametrize("n", [4096, 11008])
def test_llama_prefill_full_size_sampled(B, n):
    """C3 at full size in the bench's launch configuration: every output row
    sampled is checked against the oracle (one row at a time)."""
    m, k = 2048, 4096
    x = gen.activations((m, k), 303)
    w = gen.weights(n, k, 304)
    s_a = gen.act_scale(x)
    mu, s_w = gen.weight_stats(w)
    a = B.bwta_pack_act(x.cuda(), s_a, "ternary")
    wp = B.bwta_pack_weight(w.cuda(), mu=mu)
    y = B.bwta_gemm(a, wp, s_w.cuda(), s_a, out_dtype=torch.float16)
    yi = B.bwta_gemm(a, wp, s_w.cuda(), s_a, out_dtype=torch.int32)
    rows = np.random.default_rng(1).choice(m, 12, replace=False)
    rows = np.concatenate([rows, [0, m - 1]])
    qa = oracle.quantize_act(storage(x[rows]), "f16", s_a, "ternary")
    qw = oracle.binarize_weight(storage(w), "f16", mu=mu)
    d = oracle.dot(qa, qw, threads=oracle.default_threads())
    assert np.array_equal(yi.cpu().numpy()[rows], d)
    assert_out_equal(y[torch.from_numpy(rows).cuda()], oracle.epilogue_linear(d, s_w.numpy(), s_a, "f16"), "C3")
    # planes of sampled rows
    sgn, nz, _ = oracle.pack_act(storage(x[rows]), "f16", s_a, "ternary")
    assert np.array_equal(words(a.nz)[rows], nz) and np.array_equal(words(a.sgn)[rows], sgn)


def test_nshard_gemm_single_rank_matches_full(B):
    """dist.gemm_nshard with world = 1 runs the real local path (bwta_gemm with
    y_transposed) and must reproduce the unsharded Y^T bit for bit; the rank
    logic itself is covered by tests/test_dist.py (gloo, world 2)."""
    from paper_2604_03957_b200 import dist as D
    a, wp, s_a, s_w, qa, qw = _gemm_case(B, 200, 300, 768, 4242)
    yt = D.gemm_nshard(a, wp, s_w.cuda(), s_a, 300, 1, 0, out_dtype=torch.float16)
    d = oracle.dot(qa, qw, threads=oracle.default_threads())
    assert_out_equal(yt, oracle.epilogue_linear(d, s_w.numpy(), s_a, "f16").T.copy(), "nshard")
    # two local shards computed on one GPU and concatenated equal the full output
    n = 300
    parts = []
    for r in range(2):
        s0, e0 = D.shard_bounds(n, 2, r)
        w_r = type(wp)(wp.sgn[s0:e0], None, "binary", wp.cols)
        parts.append(B.bwta_gemm(a, w_r, s_w[s0:e0].cuda(), s_a, out_dtype=torch.float16, y_transposed=True))
    assert torch.equal(torch.cat(parts, 0).cpu(), yt.cpu())


# --------------------------------------------------- skinny (decode) GEMM ----
# The smaller side has <= 32 rows -> the skinny tcgen05 kernel (gemv_tc.cu):
# kernel-A (the large side) codes in TMEM, the small side in shared memory.
# <= 4 rows: also the CUDA-core GEMV (gemv_cc.cu), the AUTO choice there.
SKINNY = [(1, 300, 1000, "ternary"), (5, 1000, 777, "bool"), (16, 1000, 2048, "ternary"),
          (17, 517, 300, "bool"), (32, 129, 3000, "ternary"), (2000, 9, 333, "ternary"),
          (3000, 32, 1000, "bool"), (1, 1, 40, "ternary"), (24, 4100, 96, "ternary"),
          (2, 777, 4100, "bool"), (3, 1030, 513, "ternary"), (4, 65, 8192, "ternary"), (1000, 3, 260, "bool"),
          (700, 1, 129, "ternary"), (1, 4100, 16384, "ternary"), (4, 333, 16384, "bool"), (2, 1000, 16385, "ternary"),
          (3, 4097, 4096, "ternary")]


@pytest.mark.parametrize("case", range(len(SKINNY)))
def test_gemm_skinny_parity(B, case):
    m, n, k, a_kind = SKINNY[case]
    a, wp, s_a, s_w, qa, qw = _gemm_case(B, m, n, k, 4000 + case, a_kind)
    d = oracle.dot(qa, qw, threads=oracle.default_threads())
    yi = B.bwta_gemm(a, wp, s_w.cuda(), s_a, out_dtype=torch.int32)
    assert np.array_equal(yi.cpu().numpy(), d), (m, n, k, a_kind)
    for dt, name in ((torch.float16, "f16"), (torch.bfloat16, "bf16"), (torch.float32, "f32")):
        y = B.bwta_gemm(a, wp, s_w.cuda(), s_a, out_dtype=dt)
        assert_out_equal(y, oracle.epilogue_linear(d, s_w.numpy(), s_a, name), f"{m}x{n}x{k} {name}")
    yt = B.bwta_gemm(a, wp, s_w.cuda(), s_a, out_dtype=torch.float16, y_transposed=True)
    assert_out_equal(yt, oracle.epilogue_linear(d, s_w.numpy(), s_a, "f16").T.copy(), "transposed")
    y1 = B.bwta_gemm(a, wp, None, s_a, out_dtype=torch.float32)
    assert_out_equal(y1, oracle.epilogue_linear(d, None, s_a, "f32"), "no w_scale")
    # every other path gives the same result: the general tile kernel (forced tile), the
    # tcgen05 skinny kernel, the CUDA-core path (GEMV when <= 4 rows)
    ref16 = B.bwta_gemm(a, wp, s_w.cuda(), s_a).view(torch.int16)
    for kw in (dict(tile=(64, 1)), dict(design="tcgen05"), dict(design="cuda_core")):
        yg = B.bwta_gemm(a, wp, s_w.cuda(), s_a, out_dtype=torch.float16, **kw)
        assert torch.equal(yg.view(torch.int16), ref16), kw
        yi2 = B.bwta_gemm(a, wp, s_w.cuda(), s_a, out_dtype=torch.int32, **kw)
        assert np.array_equal(yi2.cpu().numpy(), d), kw


def test_attention_decode_parity(B):
    """Decode attention (Tq = 1 and 3): QK^T and PV on the skinny kernel, batched heads."""
    for i, (b, h, tq, tk, dh) in enumerate([(2, 3, 1, 1000, 128), (1, 4, 3, 300, 64), (2, 2, 20, 333, 128)]):
        seed = 4500 + 10 * i
        q = gen.activations((b, h, tq, dh), seed)
        k = gen.activations((b, h, tk, dh), seed + 1)
        v = gen.activations((b, h, tk, dh), seed + 2)
        sq, sk, sv = gen.act_scale(q), gen.act_scale(k), gen.act_scale(v)
        alpha = float(np.float32(sq * sk / np.sqrt(dh)))
        qp = B.bwta_pack_act(q.cuda(), sq, "ternary")
        kp = B.bwta_pack_act(k.cuda(), sk, "ternary")
        oq = oracle.quantize_act(storage(q).reshape(b * h, tq, dh), "f16", sq, "ternary")
        ok = oracle.quantize_act(storage(k).reshape(b * h, tk, dh), "f16", sk, "ternary")
        for design in ("auto", "tcgen05", "cuda_core"):
            for dt, name in ((torch.int32, "i32"), (torch.float16, "f16")):
                s = B.bwta_attn_qk(qp, kp, alpha, out_dtype=dt, design=design)
                assert_out_equal(s, oracle.attn_qk(oq, ok, alpha, name, threads=4).reshape(b, h, tq, tk),
                                 f"qk {name} {design}")
        p = gen.attention_probs((b, h, tq, tk), seed + 3)
        s_att = float(np.float32(2.0 / tk))
        beta = float(np.float32(s_att * sv))
        pp = B.bwta_pack_act(p.cuda(), s_att, "bool")
        vt = B.bwta_pack_act(v.cuda(), sv, "ternary", transpose=True)
        op = oracle.quantize_act(storage(p).reshape(b * h, tq, tk), "f16", s_att, "bool")
        ov = oracle.quantize_act(storage(v).reshape(b * h, tk, dh), "f16", sv, "ternary")
        for design in ("auto", "tcgen05", "cuda_core"):
            for dt, name in ((torch.int32, "i32"), (torch.float16, "f16")):
                o = B.bwta_attn_pv(pp, vt, beta, out_dtype=dt, design=design)
                assert_out_equal(o, oracle.attn_pv(op, ov, beta, name, threads=4).reshape(b, h, tq, dh),
                                 f"pv {name} {design}")


@pytest.mark.parametrize("m", [1, 16])
def test_decode_full_size_sampled(B, m):
    """configs[4]-shaped decode linear at full size (K = 8192, N = 28672) in the
    bench's launch configuration; a random sample of 384 output columns (plus the
    first and last) is checked against the oracle."""
    k, n = 8192, 28672
    x = gen.activations((m, k), 5050 + m)
    w = gen.weights(n, k, 5051)
    s_a = gen.act_scale(x)
    mu, s_w = gen.weight_stats(w)
    a = B.bwta_pack_act(x.cuda(), s_a, "ternary")
    wp = B.bwta_pack_weight(w.cuda(), mu=mu)
    y = B.bwta_gemm(a, wp, s_w.cuda(), s_a, out_dtype=torch.float16)
    yi = B.bwta_gemm(a, wp, s_w.cuda(), s_a, out_dtype=torch.int32)
    cols = np.concatenate([np.random.default_rng(2).choice(n, 384, replace=False), [0, n - 1]])
    qa = oracle.quantize_act(storage(x), "f16", s_a, "ternary")
    qw = oracle.binarize_weight(storage(w[torch.from_numpy(cols)]), "f16", mu=mu)
    d = oracle.dot(qa, qw, threads=oracle.default_threads())
    assert np.array_equal(yi.cpu().numpy()[:, cols], d)
    assert_out_equal(y[:, torch.from_numpy(cols).cuda()].contiguous(),
                     oracle.epilogue_linear(d, s_w.numpy()[cols], s_a, "f16"), "decode")


# ------------------------------------------------ PV with the context pack fused ----
@pytest.mark.parametrize("kind", ["ternary", "bool"])
@pytest.mark.parametrize("o_dtype", [torch.float16, torch.bfloat16])
def test_attn_pv_pack_equals_pv_then_pack(B, kind, o_dtype):
    """bwta_attn_pv_pack == bwta_pack_act(context of bwta_attn_pv) bit-exactly, and == the
    oracle's quantization of the oracle's rounded context; the heads' words interleave in
    the token rows, ragged Tq/Tk, several tile shapes."""
    for i, (b, h, tq, tk, dh) in enumerate([(2, 3, 37, 41, 64), (1, 2, 130, 129, 128), (4, 12, 128, 128, 64),
                                            (1, 5, 200, 300, 32)]):
        seed = 6000 + 10 * i
        v = gen.activations((b, h, tk, dh), seed)
        p = gen.attention_probs((b, h, tq, tk), seed + 1)
        sv = gen.act_scale(v)
        s_att = float(np.float32(2.0 / tk))
        beta = float(np.float32(s_att * sv))
        pp = B.bwta_pack_act(p.cuda(), s_att, "bool")
        vt = B.bwta_pack_act(v.cuda(), sv, "ternary", transpose=True)
        o = B.bwta_attn_pv(pp, vt, beta, out_dtype=o_dtype)
        ctx = o.transpose(1, 2).reshape(b * tq, h * dh).contiguous()
        s_ctx = gen.act_scale(ctx) or 1.0
        ref = B.bwta_pack_act(ctx, s_ctx, kind)
        for tile in (None, (64, 1), (128, 2)):
            got = B.bwta_attn_pv_pack(pp, vt, beta, s_ctx, kind, o_dtype=o_dtype, tile=tile)
            assert torch.equal(got.nz, ref.nz), (b, h, tq, tk, dh, tile)
            if kind == "ternary":
                assert torch.equal(got.sgn, ref.sgn), (b, h, tq, tk, dh, tile)
        # oracle: PV in the oracle, rounded to o_dtype, quantized with the oracle's pack
        op = oracle.quantize_act(storage(p).reshape(b * h, tq, tk), "f16", s_att, "bool")
        ov = oracle.quantize_act(storage(v).reshape(b * h, tk, dh), "f16", sv, "ternary")
        name = DT[o_dtype]
        oo = oracle.attn_pv(op, ov, beta, name, threads=4).reshape(b, h, tq, dh)
        octx = np.ascontiguousarray(oo.transpose(0, 2, 1, 3).reshape(b * tq, h * dh))
        sgn, nz, _ = oracle.pack_act(octx, name, s_ctx, kind)
        assert np.array_equal(words(got.nz), nz)
        if kind == "ternary":
            assert np.array_equal(words(got.sgn), sgn)


# ---------------------------------------------------- fused decode attention ----
@pytest.mark.parametrize("case", range(4))
def test_attn_decode_parity(B, case):
    """bwta_attn_decode (one launch) against the oracle's composition: P bits equal except
    within rounding distance of the threshold (fp32 softmax vs the oracle's float64; none
    expected at these sizes, counted); O equal to the oracle where no P bit differs, and
    within one unit of the dot per differing bit otherwise."""
    b, h, tk, dh, kbin, p_dt = [(2, 3, 1000, 128, False, torch.float16), (1, 4, 37, 64, False, torch.bfloat16),
                                (2, 2, 4096, 128, True, torch.float16), (1, 2, 300, 96, False, torch.float32)][case]
    seed = 7000 + 10 * case
    q = gen.activations((b, h, 1, dh), seed)
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
    o16, pbits = B.bwta_attn_decode(qp, kp, vt, alpha, s_att, beta, torch.float16, p_dt, return_p=True)
    oi = B.bwta_attn_decode(qp, kp, vt, alpha, s_att, beta, torch.int32, p_dt)
    oq = oracle.quantize_act(storage(q).reshape(b * h, dh), "f16", sq, "ternary")
    if kbin:
        ok = oracle.binarize_weight(storage(k).reshape(-1, dh), "f16").reshape(b * h, tk, dh)
    else:
        ok = oracle.quantize_act(storage(k).reshape(b * h, tk, dh), "f16", sk, "ternary")
    ov = oracle.quantize_act(storage(v).reshape(b * h, tk, dh), "f16", sv, "ternary")
    ref_i, pb, p64 = oracle.attn_decode(oq, ok, ov, alpha, s_att, pname, beta, "i32", threads=4)
    ref_16, _, _ = oracle.attn_decode(oq, ok, ov, alpha, s_att, pname, beta, "f16", threads=4)
    got_bits = oracle.unpack(None, words(pbits), "bool", tk).astype(np.int8)
    diff = got_bits != pb
    t = s_att / 2
    assert np.all(np.abs(p64[diff] / t - 1.0) < 2.0 ** -8), "P differs away from the threshold"
    flips = diff.sum(axis=1)
    gi = oi.cpu().numpy().reshape(b * h, dh)
    assert np.all(np.abs(gi - ref_i) <= flips[:, None])
    g16 = out_storage(o16).reshape(b * h, dh)
    same = flips == 0
    assert np.array_equal(g16[same], ref_16[same])
    assert pb.sum() > 0 and flips.sum() <= max(2, pb.size // 10000)


# ------------------------------------------- decode GEMM with the pack fused ----
@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16, torch.float32])
@pytest.mark.parametrize("kind", ["ternary", "bool"])
def test_gemm_x_equals_pack_then_gemm(B, dtype, kind):
    """bwta_gemm_x (the activation pack inside the GEMV) == bwta_gemm(bwta_pack_act(x)) bit-exactly
    and == the oracle, incl. exact ties / +-0 / +-inf / NaN in x, ragged K, y transposed."""
    for i, (m, n, k) in enumerate([(1, 300, 1000), (2, 777, 4100), (3, 1030, 513), (4, 65, 8192), (1, 5, 7)]):
        seed = 8000 + 10 * i
        s = tie_scale(dtype, seed)
        x = inject_specials(gen.normal((m, k), seed, dtype), s, seed + 1)
        w = gen.weights(n, k, seed + 2)
        mu, s_w = gen.weight_stats(w)
        wp = B.bwta_pack_weight(w.cuda(), mu=mu)
        for yt in (False, True):
            got = B.bwta_gemm_x(x.cuda(), s, wp, s_w.cuda(), kind, torch.float16, y_transposed=yt)
            ref = B.bwta_gemm(B.bwta_pack_act(x.cuda(), s, kind), wp, s_w.cuda(), s, torch.float16, y_transposed=yt)
            assert torch.equal(got.view(torch.int16), ref.view(torch.int16)), (m, n, k, yt)
        gi = B.bwta_gemm_x(x.cuda(), s, wp, s_w.cuda(), kind, torch.int32)
        qa = oracle.quantize_act(storage(x), DT[dtype], s, kind)
        qw = oracle.binarize_weight(storage(w), "f16", mu=mu)
        assert np.array_equal(gi.cpu().numpy(), oracle.dot(qa, qw, threads=4)), (m, n, k)


# ------------------------------------------- QKV projection with the head-split packs fused ----
@pytest.mark.parametrize("kind", ["ternary", "bool"])
@pytest.mark.parametrize("y_dt", [torch.float16, torch.bfloat16])
def test_gemm_pack_qkv_equals_gemm_then_head_packs(B, kind, y_dt):
    """bwta_gemm_pack_qkv == bwta_pack_act of the per-head Q / K views and the transposed V view of
    the stored Y (bit-exact, incl. padding words), and == the oracle's quantization of its Y."""
    for i, (bsz, t, h, d, tile) in enumerate([(2, 64, 3, 64, None), (4, 128, 12, 64, None), (3, 96, 2, 96, None),
                                              (2, 160, 4, 32, (64, 1)), (1, 256, 2, 128, (192, 2))]):
        m, n, k = bsz * t, 3 * h * d, 300 + 37 * i
        a, wp, s_a, s_w, qa, qw = _gemm_case(B, m, n, k, 9800 + i)
        y = B.bwta_gemm(a, wp, s_w.cuda(), s_a, out_dtype=y_dt)
        views = [y[:, j * h * d:(j + 1) * h * d].reshape(bsz, t, h, d).transpose(1, 2) for j in range(3)]
        sc = [gen.act_scale(v) or 1.0 for v in views]
        got = B.bwta_gemm_pack_qkv(a, wp, s_w.cuda(), s_a, bsz, t, h, d, sc, kind, y_dt, tile=tile)
        for j, (g, v) in enumerate(zip(got, views)):
            ref = B.bwta_pack_act(v, sc[j], kind, transpose=(j == 2))
            assert torch.equal(g.nz, ref.nz), (i, j)
            if kind == "ternary":
                assert torch.equal(g.sgn, ref.sgn), (i, j)
        # oracle: Y from the oracle's dot + R5 epilogue, quantized per head with the oracle's pack
        name = DT[y_dt]
        yo = oracle.epilogue_linear(oracle.dot(qa, qw, threads=oracle.default_threads()), s_w.numpy(), s_a, name)
        for j in range(3):
            vj = np.ascontiguousarray(yo[:, j * h * d:(j + 1) * h * d].reshape(bsz, t, h, d).transpose(0, 2, 1, 3))
            sg, nz, _ = oracle.pack_act(vj.reshape(bsz * h, t, d), name, sc[j], kind, transpose=(j == 2))
            assert np.array_equal(words(got[j].nz).reshape(nz.shape), nz), (i, j, "oracle")


@pytest.mark.parametrize("kind", ["ternary", "bool"])
@pytest.mark.parametrize("m,k,n", [(200, 300, 130), (3, 4096, 1000), (1, 1000, 4099), (130, 2048, 77)])
def test_gemm_row_nnz_cuda_core(B, kind, m, k, n):
    """bwta_gemm_nnz (SURVEY §8(b) a_row_nnz): design (a)'s tile kernel takes popc(nz_a) from the
    pack's row_nnz instead of counting it (the other kernels ignore it); equal to the plain call and
    to the oracle element by element, through design (a) and AUTO (GEMV / tcgen05)."""
    x = gen.activations((m, k), 31)
    if kind == "bool":
        x = torch.relu(x)
    w = gen.weights(n, k, 32)
    mu, s_w = gen.weight_stats(w)
    a = B.bwta_pack_act(x.cuda(), 1.6, kind, row_nnz=True)
    a0 = B.bwta_pack_act(x.cuda(), 1.6, kind)
    wp = B.bwta_pack_weight(w.cuda(), mu=mu)
    for design in ("cuda_core", "auto"):
        y = B.bwta_gemm(a, wp, s_w.cuda(), 1.6, out_dtype=torch.int32, design=design)
        y0 = B.bwta_gemm(a0, wp, s_w.cuda(), 1.6, out_dtype=torch.int32, design=design)
        assert torch.equal(y, y0), design
    qa = oracle.quantize_act(storage(x), "f16", 1.6, kind)
    qw = oracle.binarize_weight(storage(w), "f16", mu=mu)
    assert np.array_equal(y.cpu().numpy(), oracle.dot(qa, qw, threads=oracle.default_threads()))
