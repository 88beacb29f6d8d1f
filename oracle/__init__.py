"""BWTA CPU oracle (TEST INFRASTRUCTURE ONLY).

Plain, slow, obviously-correct implementation of what the BWTA inference hot
path computes, written from the paper (arxiv 2604.03957, /root/reference/PAPER.md
cited as P:<line>).  The arithmetic lives in ``bwta_oracle.c`` (plain C, fp64 /
exact where it decides an integer); this module only marshals numpy arrays.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline leg
and ``--impl reference``) may import this package.  The product package
``paper_2604_03957_b200`` never imports it and shares no code with it.

Pinning: every function here is pinned by tests/test_oracle.py against values
the paper / SPEC hand examples / closed forms / library routines fix.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bwta_oracle.c")
_LIB = os.path.join(_HERE, "liborc.so")
_lock = threading.Lock()
_lib = None

# dtype / kind codes of the oracle (own numbering, see bwta_oracle.c)
F16, BF16, F32, I32 = 0, 1, 2, 3
BINARY, BOOL, TERNARY = 0, 1, 2
_DT = {"f16": F16, "bf16": BF16, "f32": F32, "i32": I32}
_KIND = {"binary": BINARY, "bool": BOOL, "ternary": TERNARY}

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-fPIC",
          "-shared", "-pthread"]


def build(force: bool = False) -> str:
    """Compile bwta_oracle.c -> liborc.so with gcc (no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            P = ctypes.c_void_p
            i64 = ctypes.c_int64
            L.orc_f16_to_f32.restype = ctypes.c_float
            L.orc_f16_to_f32.argtypes = [ctypes.c_uint16]
            L.orc_bf16_to_f32.restype = ctypes.c_float
            L.orc_bf16_to_f32.argtypes = [ctypes.c_uint16]
            L.orc_f32_to_f16.restype = ctypes.c_uint16
            L.orc_f32_to_f16.argtypes = [ctypes.c_float]
            L.orc_f32_to_bf16.restype = ctypes.c_uint16
            L.orc_f32_to_bf16.argtypes = [ctypes.c_float]
            L.orc_decode.argtypes = [P, ctypes.c_int, i64, P]
            L.orc_quant_act.restype = ctypes.c_int
            L.orc_quant_act.argtypes = [ctypes.c_float, ctypes.c_float, ctypes.c_int]
            L.orc_sign_weight.restype = ctypes.c_int
            L.orc_sign_weight.argtypes = [ctypes.c_float, ctypes.c_float]
            L.orc_quantize_act.argtypes = [P, i64, i64, i64, ctypes.c_float, ctypes.c_int, P]
            L.orc_binarize_weight.argtypes = [P, i64, i64, i64, P, ctypes.c_int, P]
            L.orc_mean.restype = ctypes.c_double
            L.orc_mean.argtypes = [P, i64]
            L.orc_pack.argtypes = [P, i64, i64, i64, P, P]
            L.orc_unpack.argtypes = [P, P, ctypes.c_int, i64, i64, i64, P]
            L.orc_row_nnz.argtypes = [P, i64, i64, P]
            L.orc_dot.argtypes = [P, P, i64, i64, i64, P, ctypes.c_int]
            L.orc_epilogue_linear.argtypes = [P, i64, i64, P, ctypes.c_float, ctypes.c_int, P]
            L.orc_encode.argtypes = [P, i64, ctypes.c_int, P]
            L.orc_epilogue_scalar.argtypes = [P, i64, ctypes.c_float, ctypes.c_int, P]
            _lib = L
    return _lib


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _c(a: np.ndarray, dtype) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=dtype)


def default_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


# --------------------------------------------------------------------------
# Format contract (include/bwta.h "ld_words"): words per packed row.
# ceil(cols/32) words, rounded up to a multiple of 4 (16-byte rows).
# --------------------------------------------------------------------------
def ld_words(cols: int) -> int:
    words = (cols + 31) // 32
    return ((words + 3) // 4) * 4


# ---------------------------------------------------------------- scalars --
def f16_to_f32(h: int) -> float:
    return lib().orc_f16_to_f32(h)


def bf16_to_f32(h: int) -> float:
    return lib().orc_bf16_to_f32(h)


def f32_to_f16(f: float) -> int:
    return lib().orc_f32_to_f16(f)


def f32_to_bf16(f: float) -> int:
    return lib().orc_f32_to_bf16(f)


def quant_act(a: float, s: float, kind: str) -> int:
    return lib().orc_quant_act(a, s, _KIND[kind])


def sign_weight(w: float, mu: float) -> int:
    return lib().orc_sign_weight(w, mu)


# ---------------------------------------------------------------- arrays ---
def decode(x: np.ndarray, dt: str) -> np.ndarray:
    """Storage (uint16 bits for f16/bf16, float32 for f32) -> float32 values (O1)."""
    src = _c(x, np.float32 if dt == "f32" else np.uint16)
    out = np.empty(src.shape, np.float32)
    lib().orc_decode(_p(src), _DT[dt], src.size, _p(out))
    return out


def f32_to_storage(y: np.ndarray, dt: str) -> np.ndarray:
    """float32 -> f16/bf16 bits via the oracle's own RNE converter (O8)."""
    y = _c(y, np.float32)
    out = np.empty(y.shape, np.uint16)
    lib().orc_encode(_p(y), y.size, _DT[dt], _p(out))
    return out


def quantize_act(x: np.ndarray, dt: str, scale: float, kind: str) -> np.ndarray:
    """[..., rows, cols] storage -> int8 {-1,0,1} (ternary) / {0,1} (bool).  P:911-930."""
    vals = decode(x, dt)
    shp = vals.shape
    v2 = vals.reshape(-1, shp[-1])
    q = np.empty(v2.shape, np.int8)
    lib().orc_quantize_act(_p(v2), v2.shape[0], v2.shape[1], v2.shape[1],
                           ctypes.c_float(scale), _KIND[kind], _p(q))
    return q.reshape(shp)


def binarize_weight(w: np.ndarray, dt: str, mu=None, mu_per_row: bool = False) -> np.ndarray:
    """[N, K] storage -> int8 {-1,+1} = sign(W - mu).  P:901-909."""
    vals = decode(w, dt)
    n, k = vals.shape
    mu_arr = None if mu is None else _c(np.atleast_1d(np.asarray(mu, np.float32)), np.float32)
    q = np.empty((n, k), np.int8)
    lib().orc_binarize_weight(_p(vals), n, k, k, _p(mu_arr), int(bool(mu_per_row)), _p(q))
    return q


def mean(w: np.ndarray, dt: str) -> float:
    vals = decode(w, dt).reshape(-1)
    return lib().orc_mean(_p(vals), vals.size)


def pack(q: np.ndarray, ldw: int | None = None, want_sgn=True, want_nz=True):
    """int8 [..., rows, cols] -> (sgn, nz) uint32 [..., rows, ldw] (O6)."""
    q = _c(q, np.int8)
    shp = q.shape
    cols = shp[-1]
    ldw = ld_words(cols) if ldw is None else ldw
    q2 = q.reshape(-1, cols)
    sgn = np.empty((q2.shape[0], ldw), np.uint32) if want_sgn else None
    nz = np.empty((q2.shape[0], ldw), np.uint32) if want_nz else None
    lib().orc_pack(_p(q2), q2.shape[0], cols, ldw, _p(sgn), _p(nz))
    out_shape = shp[:-1] + (ldw,)
    return (None if sgn is None else sgn.reshape(out_shape),
            None if nz is None else nz.reshape(out_shape))


def unpack(sgn, nz, kind: str, cols: int) -> np.ndarray:
    ref = sgn if sgn is not None else nz
    shp = ref.shape
    ldw = shp[-1]
    s2 = None if sgn is None else _c(sgn, np.uint32).reshape(-1, ldw)
    n2 = None if nz is None else _c(nz, np.uint32).reshape(-1, ldw)
    rows = (s2 if s2 is not None else n2).shape[0]
    q = np.empty((rows, cols), np.int8)
    lib().orc_unpack(_p(s2), _p(n2), _KIND[kind], rows, cols, ldw, _p(q))
    return q.reshape(shp[:-1] + (cols,))


def row_nnz(q: np.ndarray) -> np.ndarray:
    q = _c(q, np.int8)
    q2 = q.reshape(-1, q.shape[-1])
    out = np.empty(q2.shape[0], np.int32)
    lib().orc_row_nnz(_p(q2), q2.shape[0], q2.shape[1], _p(out))
    return out.reshape(q.shape[:-1])


def pack_act(x: np.ndarray, dt: str, scale: float, kind: str, transpose: bool = False):
    """What bwta_pack_act must produce: (sgn|None, nz, row_nnz).

    x: storage [batch, rows, cols] (or [rows, cols]).  transpose=True packs the
    transposed matrix (planes [batch, cols, ld_words(rows)]), i.e. along rows.
    """
    q = quantize_act(x, dt, scale, kind)
    if transpose:
        q = np.ascontiguousarray(np.swapaxes(q, -1, -2))
    sgn, nz = pack(q, want_sgn=(kind == "ternary"))
    return sgn, nz, row_nnz(q)


def pack_weight(w: np.ndarray, dt: str, mu=None, mu_per_row: bool = False):
    q = binarize_weight(w, dt, mu, mu_per_row)
    sgn, _ = pack(q, want_nz=False)
    return sgn


def dot(a: np.ndarray, b: np.ndarray, threads: int = 1) -> np.ndarray:
    """int32 [M, N] = a[M, K] . b[N, K]^T over unpacked integers (O7)."""
    a = _c(a, np.int8)
    b = _c(b, np.int8)
    M, K = a.shape
    N, K2 = b.shape
    assert K == K2
    out = np.empty((M, N), np.int32)
    lib().orc_dot(_p(a), _p(b), M, N, K, _p(out), int(threads))
    return out


def epilogue_linear(d: np.ndarray, s_w, s_a: float, out_dt: str) -> np.ndarray:
    d = _c(d, np.int32)
    M, N = d.shape
    sw = None if s_w is None else _c(s_w, np.float32)
    out = np.empty((M, N), {"f16": np.uint16, "bf16": np.uint16, "f32": np.float32,
                            "i32": np.int32}[out_dt])
    lib().orc_epilogue_linear(_p(d), M, N, _p(sw), ctypes.c_float(s_a), _DT[out_dt], _p(out))
    return out


def epilogue_scalar(d: np.ndarray, alpha: float, out_dt: str) -> np.ndarray:
    d = _c(d, np.int32)
    out = np.empty(d.shape, {"f16": np.uint16, "bf16": np.uint16, "f32": np.float32,
                             "i32": np.int32}[out_dt])
    lib().orc_epilogue_scalar(_p(d), d.size, ctypes.c_float(alpha), _DT[out_dt], _p(out))
    return out


def gemm(qa: np.ndarray, qw: np.ndarray, s_w, s_a: float, out_dt: str, threads: int = 1):
    """linear(A) = s_W s_A (sign(W - mu) (x) quant(A^T, s_A)).

    qa: int8 [M, K] quantized activations, qw: int8 [N, K] signs.
    Returns Y [M, N] in out_dt storage.
    """
    return epilogue_linear(dot(qa, qw, threads), s_w, s_a, out_dt)


def attn_qk(qq: np.ndarray, qk: np.ndarray, alpha: float, out_dt: str, threads: int = 1):
    """Att_score = alpha * ternary(Q) (x) ternary(K)^T per (batch*head).

    qq: int8 [BH, Tq, D], qk: int8 [BH, Tk, D] -> [BH, Tq, Tk]."""
    outs = [epilogue_scalar(dot(qq[b], qk[b], threads), alpha, out_dt) for b in range(qq.shape[0])]
    return np.stack(outs)


def attn_pv(qp: np.ndarray, qv: np.ndarray, beta: float, out_dt: str, threads: int = 1):
    """Context = beta * bool(Att) (x) ternary(V) per (batch*head).

    qp: int8 [BH, Tq, Tk] in {0,1}, qv: int8 [BH, Tk, D] -> [BH, Tq, D]."""
    outs = []
    for b in range(qp.shape[0]):
        vt = np.ascontiguousarray(qv[b].T)       # [D, Tk] so that dot sums over Tk
        outs.append(epilogue_scalar(dot(qp[b], vt, threads), beta, out_dt))
    return np.stack(outs)


def attn_decode(qq: np.ndarray, qk: np.ndarray, qv: np.ndarray, alpha: float, s_att: float, p_dt: str,
                beta: float, out_dt: str, threads: int = 1, nkeys=None):
    """Fused decode attention, the composition of the paper's steps in order:
    S = alpha * (q . k_j) (R5 order, f32); P = softmax(S) over j in float64 (the paper
    keeps the softmax in high precision) then rounded to p_dt via f32 (O8 narrowing);
    bool quantization with s_att (R1-R2); O = beta * (P_bool . v) (R5).

    qq: int8 [BH, Dh], qk: int8 [BH, Tk, Dh], qv: int8 [BH, Tk, Dh].
    nkeys: optional int [BH]: entry b sees keys j < nkeys[b] only (a causal decoder's mask: a
    masked key is not a key -- it is out of the softmax, P = 0 and it adds nothing to PV).
    Returns (O storage [BH, Dh], P_bool int8 [BH, Tk], p float64 [BH, Tk])."""
    bh = qq.shape[0]
    s = np.stack([epilogue_scalar(dot(qq[b][None, :], qk[b], threads), alpha, "f32")[0] for b in range(bh)])
    s64 = s.astype(np.float64)
    if nkeys is not None:
        s64[np.arange(s64.shape[1])[None, :] >= np.asarray(nkeys)[:, None]] = -np.inf
    e = np.exp(s64 - s64.max(axis=1, keepdims=True))
    p = e / e.sum(axis=1, keepdims=True)
    if p_dt == "f32":
        pst = p.astype(np.float32)
    else:
        pst = f32_to_storage(p.astype(np.float32), p_dt)
    pb = quantize_act(pst, p_dt, s_att, "bool")
    o = np.stack([epilogue_scalar(dot(pb[b][None, :], np.ascontiguousarray(qv[b].T), threads), beta, out_dt)[0]
                  for b in range(bh)])
    return o, pb, p
