"""W1A1 variants (the paper's "Binary Linear" and "Binary A x V" kernels,
P:552-553): activations binarized by sign (Eq. sign; R4: +1 iff x >= 0, so -0.0 -> +1,
NaN -> -1), one sign plane per activation matrix.  Oracle: binarize_weight(x, mu = 0) is exactly
Eq. sign; the dot is the oracle's triple loop."""
import ctypes

import numpy as np
import pytest
import torch

import bwta_inputs as gen
import oracle
from test_parity_gpu import B, DT, assert_out_equal, inject_specials, storage, words  # noqa: F401

SHAPES = [(1, 1), (3, 31), (5, 33), (9, 257), (64, 768), (130, 129)]


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16, torch.float32])
@pytest.mark.parametrize("transpose", [False, True])
def test_pack_binary_activations(B, dtype, transpose):
    for i, (r, c) in enumerate(SHAPES):
        x = inject_specials(gen.activations((2, r, c), 1500 + i, dtype), 0.0, 1500 + i)
        p = B.bwta_pack_act(x.cuda(), 1.0, "binary", transpose=transpose)
        assert p.nz is None
        q = oracle.binarize_weight(storage(x).reshape(-1, c), DT[dtype]).reshape(2, r, c)
        if transpose:
            q = np.ascontiguousarray(np.swapaxes(q, -1, -2))
        sgn, _ = oracle.pack(q, want_nz=False)
        assert np.array_equal(words(p.sgn), sgn), (r, c, transpose)


@pytest.mark.gpu
def test_pack_binary_strided_heads(B):
    Bsz, T, H, D = 2, 37, 3, 64
    qkv = gen.activations((Bsz, T, 3 * H * D), 1600).cuda()
    view = qkv[:, :, H * D:2 * H * D].unflatten(-1, (H, D)).transpose(1, 2)
    for tr in (False, True):
        p = B.bwta_pack_act(view, 1.0, "binary", transpose=tr)
        q = oracle.binarize_weight(storage(view.contiguous()).reshape(-1, D), "f16").reshape(Bsz * H, T, D)
        if tr:
            q = np.ascontiguousarray(np.swapaxes(q, -1, -2))
        sgn, _ = oracle.pack(q, want_nz=False)
        assert np.array_equal(words(p.sgn).reshape(sgn.shape), sgn), tr


W1A1 = [(1, 300, 1000), (3, 65, 33), (16, 1000, 2048), (32, 129, 1), (200, 129, 768), (300, 517, 421),
        (1000, 130, 300), (130, 1000, 4100), (517, 300, 97)]


@pytest.mark.gpu
@pytest.mark.parametrize("case", range(len(W1A1)))
def test_gemm_w1a1_parity(B, case):
    """Binary Linear: binary activations x binary weights on every path (AUTO, the tcgen05 tile
    kernel with forced tiles / CTA pairs, the skinny kernel, design (a)); ragged K exercises the
    K-padding correction (each path multiplies its own padding as (+1)(+1))."""
    m, n, k = W1A1[case]
    x = gen.activations((m, k), 1700 + case)
    w = gen.weights(n, k, 1701 + case)
    s_a = gen.act_scale(x)
    mu, s_w = gen.weight_stats(w)
    a = B.bwta_pack_act(x.cuda(), s_a, "binary")
    wp = B.bwta_pack_weight(w.cuda(), mu=mu)
    qa = oracle.binarize_weight(storage(x), "f16")
    qw = oracle.binarize_weight(storage(w), "f16", mu=mu)
    d = oracle.dot(qa, qw, threads=oracle.default_threads())
    assert np.all(np.abs(d) <= k) and np.all((d - k) % 2 == 0)  # +-1 x +-1: dot = k - 2 (#disagree)
    for kw in (dict(), dict(design="tcgen05"), dict(tile=(64, 1)), dict(tile=(192, 2)), dict(tile=(128, 2)),
               dict(design="cuda_core"), dict(design="mma_b1")):
        yi = B.bwta_gemm(a, wp, s_w.cuda(), s_a, out_dtype=torch.int32, **kw)
        assert np.array_equal(yi.cpu().numpy(), d), (m, n, k, kw)
        y = B.bwta_gemm(a, wp, s_w.cuda(), s_a, out_dtype=torch.float16, **kw)
        assert_out_equal(y, oracle.epilogue_linear(d, s_w.numpy(), s_a, "f16"), f"{m}x{n}x{k} {kw}")
    yt = B.bwta_gemm(a, wp, s_w.cuda(), s_a, out_dtype=torch.bfloat16, y_transposed=True)
    assert_out_equal(yt, oracle.epilogue_linear(d, s_w.numpy(), s_a, "bf16").T.copy(), "transposed bf16")


@pytest.mark.gpu
@pytest.mark.parametrize("dims", [(2, 3, 37, 41, 64), (1, 2, 130, 300, 128), (1, 4, 3, 500, 64)])
def test_attn_pv_binary_v(B, dims):
    """Binary A x V: bool attention probabilities x binary V (V^T planes from the transposed binary
    pack); P's nz plane masks the key padding."""
    b, h, tq, tk, dh = dims
    seed = 1800 + tk
    v = gen.activations((b, h, tk, dh), seed)
    p = gen.attention_probs((b, h, tq, tk), seed + 1)
    s_att = float(np.float32(2.0 / tk))
    beta = float(np.float32(s_att * gen.act_scale(v)))
    pp = B.bwta_pack_act(p.cuda(), s_att, "bool")
    vt = B.bwta_pack_act(v.cuda(), 1.0, "binary", transpose=True)
    op = oracle.quantize_act(storage(p).reshape(b * h, tq, tk), "f16", s_att, "bool")
    ov = oracle.binarize_weight(storage(v).reshape(-1, dh), "f16").reshape(b * h, tk, dh)
    for design in ("auto", "tcgen05", "cuda_core"):
        for dt, name in ((torch.int32, "i32"), (torch.float16, "f16")):
            o = B.bwta_attn_pv(pp, vt, beta, out_dtype=dt, design=design)
            assert_out_equal(o, oracle.attn_pv(op, ov, beta, name, threads=4).reshape(b, h, tq, dh),
                             f"pv binary V {dims} {name} {design}")


def test_w1a1_validation():
    """Host validation of the binary kinds (no GPU here)."""
    from paper_2604_03957_b200 import _native as N
    L = N.lib

    def pk(kind, sgn, nz, rn=None):
        return L.bwta_pack_act(16, 0, 1, 1, 4, 64, 64, 0, 0, ctypes.c_float(1.0), kind, 0, sgn, nz, 4, 0, 0, rn, None)
    assert pk(0, 32, None) == 4          # binary: sgn only -- valid, no device here
    assert pk(0, 32, 48) == 1            # binary has no nz plane
    assert pk(0, None, None) == 1
    assert pk(0, 32, None, rn=64) == 1   # row counts are meaningless for binary
    assert pk(1, 32, 48) == 1            # bool has no sgn plane

    def gm(kind, a_sgn, a_nz):
        return L.bwta_gemm(a_sgn, a_nz, kind, 4, 4, 48, 8, 4, 100, None, ctypes.c_float(1.0), 64, 0, 8, 0, None, 0,
                           None, None)
    assert gm(0, 16, None) == 4          # binary A: valid
    assert gm(0, 16, 32) == 1
    assert gm(0, None, None) == 1
    assert gm(2, 16, None) == 1          # ternary needs nz
    # PV with binary V^T (vt_nz NULL) is valid
    assert L.bwta_attn_pv(None, 32, 48, None, 1, 1, 4, 100, 64, 4, 0, 0, 4, 0, 0, ctypes.c_float(0.1), 80, 0,
                          64, 0, 0, None, 0, None, None) == 4
