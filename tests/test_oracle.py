"""Pins for the CPU oracle (oracle/), checked against things other than itself:
values the paper / SPEC hand examples fix (tests/golden/paper_examples.json),
closed forms, invariants, library routines (numpy float16, torch bfloat16,
numpy integer matmul) and brute force on tiny inputs.

A plausible mistake anywhere in the oracle (a dropped term, a wrong sign or
index, a transposed operand, a wrong tie rule, a wrong rounding) fails one of
these.  No GPU is needed.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))


def f16_bits(vals):
    return np.asarray(vals, np.float16).view(np.uint16)


# ------------------------------------------------------------ O1 decode ----
def test_decode_f16_all_patterns_match_numpy():
    bits = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    ours = oracle.decode(bits, "f16")
    ref = bits.view(np.float16).astype(np.float32)
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(ours), nan)
    assert np.array_equal(ours[~nan].view(np.uint32), ref[~nan].view(np.uint32))  # incl. -0.0


def test_decode_bf16_all_patterns_match_torch():
    bits = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    ours = oracle.decode(bits, "bf16")
    ref = torch.from_numpy(bits.view(np.int16)).view(torch.bfloat16).float().numpy()
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(ours), nan)
    assert np.array_equal(ours[~nan].view(np.uint32), ref[~nan].view(np.uint32))


# ------------------------------------------------------ O8 RNE converters --
def _probe_floats(n=400_000, seed=0):
    rng = np.random.default_rng(seed)
    raw = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32).view(np.float32)
    # values concentrated around the f16 / bf16 ranges, incl. subnormals and overflow
    a = (rng.standard_normal(n) * np.exp2(rng.integers(-30, 20, n))).astype(np.float32)
    # exact ties of f16: odd multiples of half an f16 ulp
    h = rng.integers(0, 0x7BFF, 20000).astype(np.uint16).view(np.float16).astype(np.float32)
    h2 = np.nextafter(h.astype(np.float16), np.float16(np.inf)).astype(np.float32)
    ties = ((h.astype(np.float64) + h2.astype(np.float64)) / 2).astype(np.float32)
    special = np.array([0.0, -0.0, 65504, 65519.996, 65520, -65520, 1e-8, 2.98e-8, 5.96e-8,
                        6.1e-5, np.inf, -np.inf, 3.4e38, 1e-40], np.float32)
    return np.concatenate([raw[np.isfinite(raw)], a, ties, special])


def test_f32_to_f16_matches_numpy_rne():
    y = _probe_floats()
    ours = oracle.f32_to_storage(y, "f16")
    ref = y.astype(np.float16).view(np.uint16)
    assert np.array_equal(ours, ref)


def test_f32_to_bf16_matches_torch_rne():
    y = _probe_floats(seed=1)
    # bf16 ties: float32 values whose low 16 bits are exactly 0x8000
    rng = np.random.default_rng(5)
    t = (rng.integers(0, 2**31, 20000, dtype=np.int64).astype(np.uint32) & 0xFFFF0000) | 0x8000
    y = np.concatenate([y, t.view(np.float32)[np.isfinite(t.view(np.float32))]])
    ours = oracle.f32_to_storage(y, "bf16")
    ref = torch.from_numpy(y).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(ours, ref)


def test_nan_encodes_as_nan():
    assert oracle.f32_to_f16(float("nan")) & 0x7C00 == 0x7C00
    assert oracle.f32_to_f16(float("nan")) & 0x03FF != 0
    assert oracle.f32_to_bf16(float("nan")) & 0x7F80 == 0x7F80
    assert oracle.f32_to_bf16(float("nan")) & 0x007F != 0


# ------------------------------------------------- quantizers & packing ----
def test_spec_pack_sign_example():
    g = GOLD["pack_sign"]
    sgn, _ = oracle.pack(np.array([g["q"]], np.int8), want_nz=False)
    assert int(sgn[0, 0]) == g["sgn_word0"]
    # sign of the weights themselves
    w = np.array([[-1.0, 1.0, 1.0, -1.0]], np.float32)
    assert int(oracle.pack_weight(w, "f32", mu=0.0)[0, 0]) == g["sgn_word0"]


def test_spec_pack_ternary_example():
    g = GOLD["pack_ternary"]
    x = f16_bits([g["x"]])
    q = oracle.quantize_act(x, "f16", g["s"], "ternary")
    assert q.tolist() == [g["q"]]
    sgn, nz, nnz = oracle.pack_act(x, "f16", g["s"], "ternary")
    assert int(nz[0, 0]) == g["nz_word0"] and int(sgn[0, 0]) == g["sgn_word0"]
    assert int(nnz[0]) == 3


def test_spec_pack_bool_example():
    g = GOLD["pack_bool"]
    x = f16_bits([g["x"]])
    sgn, nz, _ = oracle.pack_act(x, "f16", g["s"], "bool")
    assert sgn is None and int(nz[0, 0]) == g["nz_word0"]


def test_ternary_ties_and_special_values():
    g = GOLD["ternary_ties_specials"]
    x = np.array([g["x_f16_bits"]], np.uint16)
    assert oracle.quantize_act(x, "f16", 1.0, "ternary").tolist() == [g["q"]]
    sgn, nz, _ = oracle.pack_act(x, "f16", 1.0, "ternary")
    assert int(nz[0, 0]) == g["nz_word0"] and int(sgn[0, 0]) == g["sgn_word0"]
    gb = GOLD["bool_ties_specials"]
    assert oracle.quantize_act(x, "f16", 1.0, "bool").tolist() == [gb["q"]]
    _, nzb, _ = oracle.pack_act(x, "f16", 1.0, "bool")
    assert int(nzb[0, 0]) == gb["nz_word0"]


def test_tie_rule_is_not_odd_symmetric():
    # a/s = +0.5 -> +1 but a/s = -0.5 -> 0 (R1)
    for s in (1.0, 0.375, 3.0e-3, 1024.0):
        assert oracle.quant_act(0.5 * s, s, "ternary") == 1
        assert oracle.quant_act(-0.5 * s, s, "ternary") == 0
        assert oracle.quant_act(np.nextafter(np.float32(-0.5 * s), np.float32(-1e9)), s, "ternary") == -1
        assert oracle.quant_act(np.nextafter(np.float32(0.5 * s), np.float32(0)), s, "ternary") == 0
        assert oracle.quant_act(0.5 * s, s, "bool") == 1


def test_threshold_agrees_with_float_division_near_ties():
    # R2: the oracle decides a/s >= 0.5 exactly (a >= 0.5 s in double); for f32
    # a, s this agrees with IEEE float32 division (numpy), checked right at the
    # thresholds where any off-by-one-ulp mistake would show.
    rng = np.random.default_rng(17)
    s = rng.uniform(1e-3, 1e3, 3000).astype(np.float32)
    half = (s.astype(np.float64) * 0.5).astype(np.float32)
    xs = np.concatenate([half, np.nextafter(half, np.float32(np.inf)), np.nextafter(half, np.float32(0)),
                         -half, np.nextafter(-half, np.float32(-np.inf)), np.nextafter(-half, np.float32(0))])
    ss = np.tile(s, 6)
    r = xs / ss
    expect = np.where(r >= np.float32(0.5), 1, np.where(r < np.float32(-0.5), -1, 0))
    got = np.array([oracle.quant_act(float(x), float(t), "ternary") for x, t in zip(xs, ss)])
    assert np.array_equal(got, expect)


def test_weight_specials_ftz_trap():
    g = GOLD["weight_specials"]
    w = np.array([g["w_f32_bits"]], np.uint32).view(np.float32)
    q = oracle.binarize_weight(w, "f32", mu=0.0)
    assert q.tolist() == [g["q"]]
    assert int(oracle.pack_weight(w, "f32", mu=0.0)[0, 0]) == g["sgn_word0"]


def test_weight_mean_shift_per_row_and_scalar():
    rng = np.random.default_rng(3)
    w = rng.standard_normal((5, 40)).astype(np.float32)
    mu = rng.standard_normal(5).astype(np.float32)
    q = oracle.binarize_weight(w, "f32", mu=mu, mu_per_row=True)
    assert np.array_equal(q, np.where(w.astype(np.float64) - mu[:, None] >= 0, 1, -1))
    q0 = oracle.binarize_weight(w, "f32", mu=float(mu[0]))
    assert np.array_equal(q0, np.where(w >= mu[0], 1, -1))
    assert abs(oracle.mean(w, "f32") - float(np.mean(w.astype(np.float64)))) < 1e-12


def test_zero_projection_invariant():
    # |x| < s/2 quantizes to 0 (the paper's zero-point projection)
    rng = np.random.default_rng(4)
    s = 0.8
    x = (rng.uniform(-0.399, 0.399, (7, 300))).astype(np.float16)
    q = oracle.quantize_act(x.view(np.uint16), "f16", s, "ternary")
    assert not q.any()


def test_zero_fraction_matches_closed_form():
    g = GOLD["zero_fraction"]
    closed = 2 * 0.5 * (1 + math.erf(math.sqrt(2 / math.pi) / math.sqrt(2))) - 1
    assert abs(closed - g["value"]) < 1e-4
    rng = np.random.default_rng(11)
    x = rng.standard_normal((400, 2500)).astype(np.float16)
    s = 2 * float(np.mean(np.abs(x.astype(np.float64))))       # s_A^0 = (2/n)||A||_1
    q = oracle.quantize_act(x.view(np.uint16), "f16", s, "ternary")
    zf = float(np.mean(q == 0))
    assert abs(zf - closed) < 0.003
    assert abs(float(np.mean(q == 1)) - float(np.mean(q == -1))) < 0.003


@pytest.mark.parametrize("cols", [1, 31, 32, 33, 63, 64, 65, 127, 128, 129, 255, 256, 257])
def test_pack_unpack_roundtrip_and_padding(cols):
    rng = np.random.default_rng(cols)
    q = rng.integers(-1, 2, (6, cols)).astype(np.int8)
    sgn, nz = oracle.pack(q)
    ldw = oracle.ld_words(cols)
    assert sgn.shape == (6, ldw) and ldw % 4 == 0 and ldw * 32 >= cols
    assert np.array_equal(oracle.unpack(sgn, nz, "ternary", cols), q)
    # canonical: sgn subset of nz
    assert not np.any(sgn & ~nz)
    # padding bits/words are zero
    full = np.unpackbits(nz.view(np.uint8), bitorder="little").reshape(6, -1)
    assert not full[:, cols:].any()
    full_s = np.unpackbits(sgn.view(np.uint8), bitorder="little").reshape(6, -1)
    assert not full_s[:, cols:].any()
    # LSB-first element order, checked with numpy's bit unpacking (library routine)
    assert np.array_equal(full[:, :cols], (q != 0).astype(np.uint8))
    assert np.array_equal(full_s[:, :cols], (q < 0).astype(np.uint8))
    qb = (q != 0).astype(np.int8)
    _, nzb = oracle.pack(qb, want_sgn=False)
    assert np.array_equal(oracle.unpack(None, nzb, "bool", cols), qb)
    qw = np.where(q < 0, -1, 1).astype(np.int8)
    sw, _ = oracle.pack(qw, want_nz=False)
    assert np.array_equal(oracle.unpack(sw, None, "binary", cols), qw)


def test_transposed_pack_is_pack_of_transpose():
    rng = np.random.default_rng(9)
    x = rng.standard_normal((2, 70, 45)).astype(np.float16).view(np.uint16)
    sgn_t, nz_t, nnz_t = oracle.pack_act(x, "f16", 1.1, "ternary", transpose=True)
    assert sgn_t.shape == (2, 45, oracle.ld_words(70))
    xt = np.ascontiguousarray(np.swapaxes(x, 1, 2))
    sgn, nz, nnz = oracle.pack_act(xt, "f16", 1.1, "ternary")
    assert np.array_equal(sgn, sgn_t) and np.array_equal(nz, nz_t) and np.array_equal(nnz, nnz_t)


def test_scale_equivariance_powers_of_two():
    rng = np.random.default_rng(12)
    x = rng.standard_normal((4, 100)).astype(np.float16)
    base = oracle.pack_act(x.view(np.uint16), "f16", 0.75, "ternary")
    for e in (-3, 2, 5):
        x2 = (x.astype(np.float32) * 2.0 ** e).astype(np.float16)   # exact for these ranges
        assert np.array_equal(x2.astype(np.float32), x.astype(np.float32) * 2.0 ** e)
        got = oracle.pack_act(x2.view(np.uint16), "f16", 0.75 * 2.0 ** e, "ternary")
        for a, b in zip(base, got):
            assert np.array_equal(a, b)


def test_row_nnz_matches_numpy():
    rng = np.random.default_rng(2)
    q = rng.integers(-1, 2, (9, 77)).astype(np.int8)
    assert np.array_equal(oracle.row_nnz(q), np.count_nonzero(q, axis=1))


# ------------------------------------------------------------- O7 dot -----
def test_spec_case_examples():
    for key, a, b in (("case1", "a", "w"), ("case2", "att", "v"), ("case3", "q", "k")):
        g = GOLD[key]
        d = oracle.dot(np.array([g[a]], np.int8), np.array([g[b]], np.int8))
        assert int(d[0, 0]) == g["dot"]
    g = GOLD["gemm_int"]
    assert oracle.dot(np.array(g["a"], np.int8), np.array(g["b"], np.int8)).tolist() == g["dot"]


def test_word_boundary_k33_examples():
    g = GOLD["case1_k33"]
    K = 33
    a_nz = np.array([g["a_nz"] + [0, 0]], np.uint32)
    a_sgn = np.array([g["a_sgn"] + [0, 0]], np.uint32)
    w_sgn = np.array([g["w_sgn"] + [0, 0]], np.uint32)
    qa = oracle.unpack(a_sgn, a_nz, "ternary", K)
    qw = oracle.unpack(w_sgn, None, "binary", K)
    assert qa[0].tolist() == [(1, 0, -1, 1)[i % 4] for i in range(K)]
    assert qw[0].tolist() == [-1 if i % 5 == 0 else 1 for i in range(K)]
    assert int(oracle.row_nnz(qa)[0]) == g["nnz"]
    assert int(oracle.dot(qa, qw)[0, 0]) == g["dot"]
    g3 = GOLD["case3_k33"]
    qk = oracle.unpack(np.array([g3["k_sgn"] + [0, 0]], np.uint32),
                       np.array([g3["k_nz"] + [0, 0]], np.uint32), "ternary", K)
    assert int(oracle.dot(qa, qk)[0, 0]) == g3["dot"]
    assert int(np.count_nonzero(qa[0] * qk[0])) == g3["bound"]


def _all_vectors(values, k):
    grids = np.meshgrid(*([np.array(values, np.int8)] * k), indexing="ij")
    return np.stack([g.reshape(-1) for g in grids], axis=1).astype(np.int8)


def test_exhaustive_k6_equals_integer_matmul():
    tern = _all_vectors([-1, 0, 1], 6)     # 729
    binv = _all_vectors([-1, 1], 6)        # 64
    boolv = _all_vectors([0, 1], 6)        # 64
    for a, b in ((tern, binv), (tern, tern), (boolv, tern)):
        d = oracle.dot(a, b, threads=4)
        assert np.array_equal(d, a.astype(np.int64) @ b.astype(np.int64).T)


def test_dot_invariants():
    rng = np.random.default_rng(21)
    qa = rng.integers(-1, 2, (40, 301)).astype(np.int8)
    qw = np.where(rng.integers(0, 2, (30, 301)) == 1, 1, -1).astype(np.int8)
    d = oracle.dot(qa, qw, threads=3)
    nnz = np.count_nonzero(qa, axis=1)[:, None]
    assert np.all((d - nnz) % 2 == 0)                      # parity = popc(m) parity
    assert np.all(np.abs(d) <= nnz)                        # |dot| <= popc(m)
    ones = np.ones((1, 301), np.int8)
    assert np.array_equal(oracle.dot(qa, ones)[:, 0], qa.sum(axis=1))   # all-ones weights
    assert np.array_equal(oracle.dot(qa, -qw), -d)                     # weight negation
    dqq = oracle.dot(qa, qa)
    assert np.array_equal(np.diag(dqq), np.count_nonzero(qa, axis=1))  # Q = K diagonal
    # padding invariance: appending zero columns changes nothing
    pad = np.zeros((40, 31), np.int8)
    assert np.array_equal(oracle.dot(np.hstack([qa, pad]), np.hstack([qw, np.ones((30, 31), np.int8)])), d)


def _popc(x):
    return bin(int(x)).count("1")


def test_north_star_closed_form_on_planes():
    """dot = sum_w popc(nz) - 2 popc(nz & (sgn ^ w)) (north star; Case-1 P:324-325),
    and the xor form popc(w^A+) - popc(w^A-), against the oracle's
    unpack + integer dot, over random canonical planes."""
    rng = np.random.default_rng(8)
    for _ in range(200):
        words = int(rng.integers(1, 5))
        nz = rng.integers(0, 2**32, words, dtype=np.uint64).astype(np.uint32)
        sg = rng.integers(0, 2**32, words, dtype=np.uint64).astype(np.uint32) & nz
        w = rng.integers(0, 2**32, words, dtype=np.uint64).astype(np.uint32)
        K = words * 32
        qa = oracle.unpack(sg[None], nz[None], "ternary", K)
        qw = oracle.unpack(w[None], None, "binary", K)
        d = int(oracle.dot(qa, qw)[0, 0])
        cf = sum(_popc(nz[i]) - 2 * _popc(nz[i] & (sg[i] ^ w[i])) for i in range(words))
        ap = nz & ~sg
        an = sg
        xf = sum(_popc(w[i] ^ ap[i]) - _popc(w[i] ^ an[i]) for i in range(words))
        assert d == cf == xf


# -------------------------------------------------------- O8 epilogue -----
def test_epilogue_order_pin():
    g = GOLD["epilogue_order"]
    sw = np.array([g["s_w_bits"]], np.uint32).view(np.float32)
    sa = float(np.array([g["s_a_bits"]], np.uint32).view(np.float32)[0])
    d = np.array([[g["dot"]]], np.int32)
    y32 = oracle.epilogue_linear(d, sw, sa, "f32")
    assert float(y32[0, 0]) == g["y"]
    yb = oracle.epilogue_linear(d, sw, sa, "bf16")
    assert int(yb[0, 0]) == g["bf16_bits"]
    assert oracle.bf16_to_f32(int(yb[0, 0])) == g["bf16_value"]
    # the other association lands on a different bf16 (why R5 fixes the order)
    other = np.float32(np.float32(g["dot"]) * sw[0]) * np.float32(sa)
    assert float(torch.tensor(float(other)).to(torch.bfloat16)) == g["other_order_bf16_value"]


def test_epilogue_matches_numpy_float32():
    rng = np.random.default_rng(13)
    d = rng.integers(-4096, 4097, (33, 47)).astype(np.int32)
    sw = rng.uniform(0.001, 0.05, 47).astype(np.float32)
    sa = float(np.float32(rng.uniform(0.5, 3)))
    c = (sw * np.float32(sa)).astype(np.float32)
    ref = (d.astype(np.float32) * c[None, :]).astype(np.float32)
    y = oracle.epilogue_linear(d, sw, sa, "f32")
    assert np.array_equal(y.view(np.uint32), ref.view(np.uint32))
    assert np.array_equal(oracle.epilogue_linear(d, sw, sa, "f16"), ref.astype(np.float16).view(np.uint16))
    assert np.array_equal(oracle.epilogue_linear(d, sw, sa, "i32"), d)
    ys = oracle.epilogue_scalar(d, 0.125, "f16")
    assert np.array_equal(ys, (d.astype(np.float32) * np.float32(0.125)).astype(np.float16).view(np.uint16))
    assert oracle.epilogue_linear(np.zeros((1, 1), np.int32), sw[:1], sa, "f16")[0, 0] == 0  # +0.0


def test_spec_linear_tie_example():
    g = GOLD["linear_tie"]
    w = np.array(g["w"], np.float32)
    a = np.array(g["a"], np.float32)
    s_w = float(np.linalg.norm(w) / w.size)                 # ||W||_F / n_W
    s_a = float(2.0 / a.size * np.abs(a).sum())             # (2/n)||A||_1
    assert abs(s_w - g["s_w"]) < 1e-7 and s_a == g["s_a"]
    qa = oracle.quantize_act(a, "f32", s_a, "ternary")
    assert qa.tolist() == [g["q_a"]]
    qw = oracle.binarize_weight(w, "f32", mu=g["mu"])
    y = oracle.gemm(qa, qw, np.array([s_w], np.float32), s_a, "f32")
    assert abs(float(y[0, 0]) - g["y"]) < 1e-6
    assert abs(float(y[0, 0]) - g["y_spec_rule"]) > 1.0


def test_attention_oracles_reduce_to_matmul():
    rng = np.random.default_rng(31)
    q = rng.integers(-1, 2, (3, 9, 64)).astype(np.int8)
    k = rng.integers(-1, 2, (3, 11, 64)).astype(np.int8)
    s = oracle.attn_qk(q, k, 1.0, "f32")
    assert np.array_equal(s, np.einsum("bid,bjd->bij", q.astype(np.float32), k.astype(np.float32)))
    p = rng.integers(0, 2, (3, 9, 11)).astype(np.int8)
    v = rng.integers(-1, 2, (3, 11, 64)).astype(np.int8)
    o = oracle.attn_pv(p, v, 1.0, "f32")
    assert np.array_equal(o, np.einsum("bij,bjd->bid", p.astype(np.float32), v.astype(np.float32)))


def test_dot_threads_deterministic():
    rng = np.random.default_rng(41)
    a = rng.integers(-1, 2, (37, 200)).astype(np.int8)
    b = rng.integers(-1, 2, (23, 200)).astype(np.int8)
    assert np.array_equal(oracle.dot(a, b, 1), oracle.dot(a, b, 7))


# ---------------------------------------------- fused decode attention (N3) ----
def test_attn_decode_uniform_scores_give_column_sums():
    """alpha = 0: every score is 0, softmax is uniform 1/Tk; with s_att = 1/Tk every p
    clears the threshold 1/(2 Tk), so O = beta * (column sums of V) -- a closed form."""
    rng = np.random.default_rng(11)
    bh, tk, dh = 3, 50, 64
    qq = rng.integers(-1, 2, (bh, dh)).astype(np.int8)
    qk = rng.integers(-1, 2, (bh, tk, dh)).astype(np.int8)
    qv = rng.integers(-1, 2, (bh, tk, dh)).astype(np.int8)
    beta = 0.125
    o, pb, p = oracle.attn_decode(qq, qk, qv, 0.0, 1.0 / tk, "f16", beta, "f32")
    assert np.allclose(p, 1.0 / tk) and pb.all()
    assert np.array_equal(o, (qv.sum(axis=1).astype(np.float32) * np.float32(beta)).astype(np.float32))


def test_attn_decode_dominant_key_selects_its_value():
    """q = k_0 and every other key = -q: softmax is one-hot on key 0 (e^-80 elsewhere),
    so P = e_0 and O = beta * v_0 exactly."""
    rng = np.random.default_rng(12)
    dh, tk = 64, 20
    q = rng.integers(-1, 2, dh).astype(np.int8)
    q[:40] = 1                                  # >= 40 non-zeros
    qk = np.tile(-q, (tk, 1))
    qk[0] = q
    qv = rng.integers(-1, 2, (1, tk, dh)).astype(np.int8)
    o, pb, _ = oracle.attn_decode(q[None], qk[None], qv, 1.0, 0.5, "f16", 1.0, "i32")
    assert pb[0, 0] == 1 and pb[0, 1:].sum() == 0
    assert np.array_equal(o[0], qv[0, 0].astype(np.int32))


def test_attn_decode_key_permutation_invariance():
    """Permuting the (key, value) pairs permutes P and leaves O unchanged."""
    rng = np.random.default_rng(13)
    bh, tk, dh = 2, 300, 128
    qq = rng.integers(-1, 2, (bh, dh)).astype(np.int8)
    qk = rng.integers(-1, 2, (bh, tk, dh)).astype(np.int8)
    qv = rng.integers(-1, 2, (bh, tk, dh)).astype(np.int8)
    perm = rng.permutation(tk)
    o1, pb1, _ = oracle.attn_decode(qq, qk, qv, 0.09, 2.0 / tk, "f16", 0.01, "f16")
    o2, pb2, _ = oracle.attn_decode(qq, qk[:, perm], qv[:, perm], 0.09, 2.0 / tk, "f16", 0.01, "f16")
    assert np.array_equal(pb1[:, perm], pb2) and np.array_equal(o1, o2)
    assert 0 < pb1.sum() < pb1.size


def test_attn_causal_mask_uniform_scores_give_prefix_sums():
    """Causal mask (nkeys): alpha = 0 makes every visible score 0, so row b's softmax is uniform
    1 / n_b over its first n_b keys and 0 beyond; with s_att = 1 / n_max every visible p clears
    the threshold 1 / (2 n_max) and O = beta * (sum of the first n_b value rows) -- a closed form,
    independent of the unmasked path."""
    rng = np.random.default_rng(14)
    bh, tk, dh = 4, 40, 64
    nk = np.array([1, 7, 33, 40])
    qq = rng.integers(-1, 2, (bh, dh)).astype(np.int8)
    qk = rng.integers(-1, 2, (bh, tk, dh)).astype(np.int8)
    qv = rng.integers(-1, 2, (bh, tk, dh)).astype(np.int8)
    o, pb, p = oracle.attn_decode(qq, qk, qv, 0.0, 1.0 / tk, "f16", 0.25, "f32", nkeys=nk)
    for b in range(bh):
        assert np.allclose(p[b, :nk[b]], 1.0 / nk[b]) and np.all(p[b, nk[b]:] == 0)
        assert pb[b, :nk[b]].all() and pb[b, nk[b]:].sum() == 0
        ref = (qv[b, :nk[b]].sum(axis=0).astype(np.float32) * np.float32(0.25)).astype(np.float32)
        assert np.array_equal(o[b], ref)


def test_attn_causal_mask_is_truncation():
    """A row that sees its first n keys gives the same P (on those keys) and O as the unmasked
    composition on K[:n], V[:n] (masked keys are not keys); all keys visible == unmasked."""
    rng = np.random.default_rng(15)
    bh, tk, dh = 3, 200, 128
    qq = rng.integers(-1, 2, (bh, dh)).astype(np.int8)
    qk = rng.integers(-1, 2, (bh, tk, dh)).astype(np.int8)
    qv = rng.integers(-1, 2, (bh, tk, dh)).astype(np.int8)
    nk = np.array([5, 120, tk])
    o, pb, _ = oracle.attn_decode(qq, qk, qv, 0.09, 2.0 / 64, "f16", 0.01, "f16", nkeys=nk)
    for b in range(bh):
        n = nk[b]
        o1, pb1, _ = oracle.attn_decode(qq[b:b + 1], qk[b:b + 1, :n], qv[b:b + 1, :n], 0.09, 2.0 / 64, "f16", 0.01,
                                        "f16")
        assert np.array_equal(pb[b, :n], pb1[0]) and pb[b, n:].sum() == 0
        assert np.array_equal(o[b], o1[0])
    ou, pbu, _ = oracle.attn_decode(qq, qk, qv, 0.09, 2.0 / 64, "f16", 0.01, "f16")
    assert np.array_equal(o[2], ou[2]) and np.array_equal(pb[2], pbu[2])
