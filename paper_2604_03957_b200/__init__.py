"""B200-native BWTA inference hot path (arxiv 2604.03957).

Thin Python binding over the C ABI in ``include/bwta.h`` / ``libbwta.so``:
argument marshalling only (torch tensors -> device pointers, strides, the
current CUDA stream).  Every step of the path runs in the library's sm_100a
kernels; PyTorch only provides device memory and streams.  If the library is
missing, importing this package raises -- there is no fallback.

Functions carry the C names:
    bwta_pack_act, bwta_pack_weight, bwta_gemm, bwta_attn_qk, bwta_attn_pv
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import torch

from . import _native as N
from ._native import lib

__all__ = ["Packed", "BwtaError", "bwta_ld_words", "bwta_pack_act", "bwta_pack_weight",
           "bwta_pack_act_batch", "bwta_gemm", "bwta_gemm_pack", "bwta_attn_qk", "bwta_attn_pv", "bwta_attn_pv_pack", "bwta_attn_decode", "bwta_attn_prefill", "bwta_attn_prefill_pack", "bwta_gemm_pack_qkv", "bwta_gemm_x", "bwta_gemm_peers", "bwta_peer_barrier",
           "ipc_handle", "ipc_open", "ipc_close", "last_design", "lib"]


class BwtaError(RuntimeError):
    def __init__(self, status: int, where: str):
        msg = lib.bwta_status_string(status).decode()
        if status == 5:
            msg += f" (cudaError {lib.bwta_last_cuda_error()})"
        super().__init__(f"{where}: {msg}")
        self.status = status


def _check(st: int, where: str):
    if st != N.BWTA_OK:
        raise BwtaError(st, where)


_DT = {torch.float16: N.F16, torch.bfloat16: N.BF16, torch.float32: N.F32, torch.int32: N.I32}
_KIND = {"binary": N.BINARY, "bool": N.BOOL, "ternary": N.TERNARY}
_DESIGN = {"auto": N.DESIGN_AUTO, "cuda_core": N.DESIGN_CUDA_CORE, "cc": N.DESIGN_CUDA_CORE,
           "tcgen05": N.DESIGN_TCGEN05, "tc": N.DESIGN_TCGEN05, "mma_b1": N.DESIGN_MMA_B1}


def bwta_ld_words(cols: int) -> int:
    return int(lib.bwta_ld_words(cols))


def last_design() -> str:
    return {0: "none", 1: "cuda_core", 2: "tcgen05", 3: "mma_b1"}[lib.bwta_last_design()]


@dataclass
class Packed:
    """Bit planes of a quantized matrix (format: include/bwta.h).

    sgn / nz: int32 tensors [..., rows, ld] holding the uint32 words (either
    may be None: BOOL has no sgn, BINARY no nz).  ``cols`` is the number of
    elements along the packed axis."""
    sgn: Optional[torch.Tensor]
    nz: Optional[torch.Tensor]
    kind: str
    cols: int
    row_nnz: Optional[torch.Tensor] = None

    @property
    def ref(self) -> torch.Tensor:
        return self.sgn if self.sgn is not None else self.nz


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream) -> ctypes.c_void_p:
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _opts(design: str, tile=None):
    """tile: optional (tile_n, cta_group) override of design (b)'s tile choice."""
    o = N.Opts()
    o.design = _DESIGN[design]
    if tile is not None:
        o.tile_n, o.cta_group = int(tile[0]), int(tile[1])
    return ctypes.byref(o)


def _batch_dims(t: torch.Tensor):
    """(batch, heads, bstride, hstride) of a 2-, 3- or 4-D tensor's leading dims."""
    if t.dim() == 2:
        return 1, 1, 0, 0
    if t.dim() == 3:
        return t.shape[0], 1, t.stride(0), 0
    if t.dim() == 4:
        return t.shape[0], t.shape[1], t.stride(0), t.stride(1)
    raise ValueError("expected a 2-, 3- or 4-D tensor")


def _check_out(out: torch.Tensor, shape: tuple, device, what: str):
    """A caller-supplied output must have the result's shape, a supported dtype, live on the
    operands' device and have unit stride along its last dimension (the C ABI receives only the
    pointer and the leading strides; a wrong `out` would be written out of bounds)."""
    if tuple(out.shape) != tuple(shape):
        raise ValueError(f"{what}: out has shape {tuple(out.shape)}, expected {tuple(shape)}")
    if out.dtype not in _DT:
        raise ValueError(f"{what}: unsupported out dtype {out.dtype}")
    if out.device != torch.device(device):
        raise ValueError(f"{what}: out is on {out.device}, operands on {device}")
    if out.dim() and out.shape[-1] > 1 and out.stride(-1) != 1:
        raise ValueError(f"{what}: out must have unit stride in its last dimension")
    if out.dim() >= 2 and out.shape[-2] > 1 and out.stride(-2) < out.shape[-1]:
        raise ValueError(f"{what}: out rows overlap (row stride < row length)")


_WS: dict = {}


def _workspace(nbytes: int, device) -> tuple:
    if nbytes == 0:
        return None, 0
    key = (device, )
    buf = _WS.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=device)
        _WS[key] = buf
    return buf, buf.numel()


# ----------------------------------------------------------------------------
def _pack_desc(x: torch.Tensor, scale: float, kind: str, transpose: bool, row_nnz: bool):
    """(bwta_pack_desc_t, Packed) for one activation pack; allocates the planes."""
    if x.stride(-1) != 1:
        raise ValueError("x must have unit stride in its last dimension")
    if kind not in _KIND:
        raise ValueError(f"unknown kind {kind!r}")
    b, h, xbs, xhs = _batch_dims(x)
    rows, cols = x.shape[-2], x.shape[-1]
    out_rows, plen = (cols, rows) if transpose else (rows, cols)
    ldw = bwta_ld_words(plen)
    lead = tuple(x.shape[:-2])
    shape = lead + (out_rows, ldw)
    nz = torch.empty(shape, dtype=torch.int32, device=x.device) if kind != "binary" else None
    sgn = torch.empty(shape, dtype=torch.int32, device=x.device) if kind != "bool" else None
    rn = torch.empty(lead + (out_rows,), dtype=torch.int32, device=x.device) if row_nnz else None
    pbs = h * out_rows * ldw if x.dim() == 4 else out_rows * ldw
    phs = out_rows * ldw if x.dim() == 4 else 0
    if x.dim() == 2:
        pbs = 0
    d = N.PackDesc(_ptr(x), _DT[x.dtype], b, h, rows, cols, x.stride(-2), xbs, xhs, float(scale), _KIND[kind],
                   int(transpose), _ptr(sgn), _ptr(nz), ldw, pbs, phs, _ptr(rn))
    return d, Packed(sgn, nz, kind, plen, rn)


def bwta_pack_act(x: torch.Tensor, scale: float, kind: str = "ternary", transpose: bool = False,
                  row_nnz: bool = False, stream=None) -> Packed:
    """Quantize and bit-pack activations.  kind: "ternary" (sgn + nz planes), "bool"
    (nz), or "binary" (sgn only: sign(x) of Eq. sign, P:903-908 -- W1A1 activations; `scale` is
    then only the epilogue's s_A).

    x: CUDA tensor (f16/bf16/f32) [rows, cols], [B, rows, cols] or
    [B, H, rows, cols] (any batch/head/row strides, unit column stride).
    transpose=True packs along rows (planes of x^T; used for V^T in PV)."""
    d, out = _pack_desc(x, scale, kind, transpose, row_nnz)
    st = lib.bwta_pack_act(d.x, d.x_dt, d.batch, d.heads, d.rows, d.cols, d.ld_x, d.x_bstride, d.x_hstride,
                           ctypes.c_float(scale), d.kind, d.transpose, d.sgn, d.nz, d.ld_words, d.p_bstride,
                           d.p_hstride, d.row_nnz, _stream(stream))
    _check(st, "bwta_pack_act")
    return out


def bwta_pack_act_batch(items, stream=None) -> list:
    """Several bwta_pack_act calls in one kernel launch (<= 4; the per-head Q,
    K and V^T packs of an attention layer).  items: sequence of
    (x, scale, kind, transpose) tuples; returns the Packed results in order."""
    items = list(items)
    if len(items) > 4:
        raise ValueError("at most 4 packs per batch")
    descs, outs = [], []
    for x, scale, kind, transpose in items:
        d, o = _pack_desc(x, scale, kind, transpose, False)
        descs.append(d)
        outs.append(o)
    arr = (N.PackDesc * max(len(descs), 1))(*descs)
    _check(lib.bwta_pack_act_batch(ctypes.cast(arr, ctypes.c_void_p), len(descs), _stream(stream)),
           "bwta_pack_act_batch")
    return outs


def bwta_pack_weight(w: torch.Tensor, mu=None, stream=None) -> Packed:
    """sign(W - mu) bit-pack.  w: [N, K] CUDA tensor.
    mu: None (0), a python float, or a CUDA float32 tensor [1] or [N] (per row)."""
    if w.dim() != 2 or w.stride(-1) != 1:
        raise ValueError("w must be a 2-D tensor with unit column stride")
    n, k = w.shape
    ldw = bwta_ld_words(k)
    sgn = torch.empty((n, ldw), dtype=torch.int32, device=w.device)
    per_row = 0
    mu_t = None
    if mu is not None:
        mu_t = mu if isinstance(mu, torch.Tensor) else torch.tensor([float(mu)], dtype=torch.float32,
                                                                    device=w.device)
        mu_t = mu_t.to(device=w.device, dtype=torch.float32).contiguous()
        per_row = int(mu_t.numel() == n and n > 1)
    st = lib.bwta_pack_weight(_ptr(w), _DT[w.dtype], n, k, w.stride(0), _ptr(mu_t), per_row, _ptr(sgn),
                              ldw, _stream(stream))
    _check(st, "bwta_pack_weight")
    return Packed(sgn, None, "binary", k)


def bwta_gemm(a: Packed, w: Packed, w_scale: Optional[torch.Tensor], a_scale: float,
              out_dtype=torch.float16, y_transposed: bool = False, out: Optional[torch.Tensor] = None,
              design: str = "auto", stream=None, tile=None) -> torch.Tensor:
    """Y = s_W s_A (sign(W - mu) (x) quant(A^T, s_A)).

    a: Packed activations [M, lda] (ternary or bool); w: Packed weights [N, ldw].  When `a` carries
    the pack's row_nnz (bwta_pack_act(row_nnz=True)) it is passed on (bwta_gemm_nnz: design (a)'s tile
    kernel uses it instead of counting popc(nz_a)).
    Returns Y [M, N] (or Y^T [N, M] if y_transposed)."""
    if a.kind not in ("ternary", "bool", "binary") or w.kind != "binary" or a.cols != w.cols:
        raise ValueError("bwta_gemm expects ternary/bool/binary activations and binary weights of equal K")
    ar = a.ref
    m, n, k = ar.shape[-2], w.sgn.shape[-2], a.cols
    dev = ar.device
    if out is None:
        out = torch.empty((n, m) if y_transposed else (m, n), dtype=out_dtype, device=dev)
    else:
        _check_out(out, (n, m) if y_transposed else (m, n), dev, "bwta_gemm")
    o = _opts(design, tile)
    ws, wsb = _workspace(lib.bwta_gemm_workspace_size(m, n, k, o), dev)
    ws_scale = None if w_scale is None else w_scale.to(device=dev, dtype=torch.float32).contiguous()
    rn = a.row_nnz if (a.row_nnz is not None and a.row_nnz.dim() == 1 and a.row_nnz.numel() == m) else None
    st = lib.bwta_gemm_nnz(_ptr(a.sgn), _ptr(a.nz), _KIND[a.kind], m, ar.stride(-2), _ptr(rn), _ptr(w.sgn), n,
                           w.sgn.stride(-2), k, _ptr(ws_scale), ctypes.c_float(a_scale), _ptr(out),
                           _DT[out.dtype], out.stride(0), int(y_transposed), _ptr(ws), wsb, o, _stream(stream))
    _check(st, "bwta_gemm")
    return out


def bwta_gemm_peers(a: Packed, w: Packed, w_scale: Optional[torch.Tensor], a_scale: float, y_ptr: int, ld_y: int,
                    peer_ptrs, out_dtype=torch.float16, y_transposed: bool = True, design: str = "auto",
                    stream=None, tile=None) -> None:
    """bwta_gemm of one N-shard whose epilogue also stores every output tile into each peer's buffer
    (the fused all-gather, include/bwta.h bwta_gemm_peers).  y_ptr / peer_ptrs are device addresses
    (ints) of this shard's block in this GPU's / the peers' Y^T (row stride ld_y elements); the
    buffers are the caller's (paper_2604_03957_b200.dist.PeerAllGather owns them)."""
    if a.kind not in ("ternary", "bool", "binary") or w.kind != "binary" or a.cols != w.cols:
        raise ValueError("bwta_gemm_peers expects ternary/bool/binary activations and binary weights of equal K")
    if out_dtype not in (torch.float16, torch.bfloat16):
        raise ValueError("bwta_gemm_peers stores f16 / bf16")
    ar = a.ref
    m, n, k = ar.shape[-2], w.sgn.shape[-2], a.cols
    peers = list(peer_ptrs)
    arr = (ctypes.c_void_p * max(1, len(peers)))(*[ctypes.c_void_p(int(q)) for q in peers])
    ws_scale = None if w_scale is None else w_scale.to(device=ar.device, dtype=torch.float32).contiguous()
    st = lib.bwta_gemm_peers(_ptr(a.sgn), _ptr(a.nz), _KIND[a.kind], m, ar.stride(-2), _ptr(w.sgn), n,
                             w.sgn.stride(-2), k, _ptr(ws_scale), ctypes.c_float(a_scale), ctypes.c_void_p(int(y_ptr)),
                             _DT[out_dtype], int(ld_y), int(y_transposed), arr, len(peers), _opts(design, tile),
                             _stream(stream))
    _check(st, "bwta_gemm_peers")


def bwta_peer_barrier(flag_ptrs, rank: int, count_ptr: int, stream=None) -> None:
    """Cross-GPU barrier (include/bwta.h bwta_peer_barrier): flag_ptrs[r] = device address of rank r's
    uint32 flag array as mapped in this process; count_ptr = this rank's uint32 barrier count."""
    arr = (ctypes.c_void_p * len(flag_ptrs))(*[ctypes.c_void_p(int(q)) for q in flag_ptrs])
    _check(lib.bwta_peer_barrier(arr, len(flag_ptrs), int(rank), ctypes.c_void_p(int(count_ptr)), _stream(stream)),
           "bwta_peer_barrier")


def ipc_handle(t: torch.Tensor):
    """(handle bytes, byte offset) of the allocation holding t's storage (CUDA IPC)."""
    h = (ctypes.c_char * N.IPC_HANDLE_BYTES)()
    off = ctypes.c_int64(0)
    _check(lib.bwta_ipc_handle(ctypes.c_void_p(t.data_ptr()), h, ctypes.byref(off)), "bwta_ipc_handle")
    return bytes(h.raw), int(off.value)


def ipc_open(handle: bytes, offset: int) -> int:
    """Map another process's allocation (ipc_handle) into this one; returns the device address."""
    h = (ctypes.c_char * N.IPC_HANDLE_BYTES).from_buffer_copy(handle)
    ptr = ctypes.c_void_p(0)
    _check(lib.bwta_ipc_open(h, int(offset), ctypes.byref(ptr)), "bwta_ipc_open")
    return int(ptr.value)


def ipc_close(ptr: int, offset: int) -> None:
    _check(lib.bwta_ipc_close(ctypes.c_void_p(int(ptr)), int(offset)), "bwta_ipc_close")


def bwta_gemm_x(x: torch.Tensor, a_scale: float, w: Packed, w_scale: Optional[torch.Tensor], kind: str = "ternary",
                out_dtype=torch.float16, y_transposed: bool = False, stream=None) -> torch.Tensor:
    """bwta_gemm(bwta_pack_act(x, a_scale, kind), w, w_scale, a_scale) in one launch for <= 4
    activation rows (decode): the pack runs inside the GEMV.  x [M, K] values."""
    if kind not in ("ternary", "bool") or w.kind != "binary" or x.shape[-1] != w.cols or x.dim() != 2:
        raise ValueError("bwta_gemm_x expects x [M, K] and binary weights of equal K")
    if x.stride(-1) != 1:
        x = x.contiguous()
    m, k, n = x.shape[0], x.shape[1], w.sgn.shape[-2]
    out = torch.empty((n, m) if y_transposed else (m, n), dtype=out_dtype, device=x.device)
    ws_scale = None if w_scale is None else w_scale.to(device=x.device, dtype=torch.float32).contiguous()
    st = lib.bwta_gemm_x(_ptr(x), _DT[x.dtype], m, x.stride(0), ctypes.c_float(a_scale), _KIND[kind], _ptr(w.sgn), n,
                         w.sgn.stride(-2), k, _ptr(ws_scale), _ptr(out), _DT[out.dtype], out.stride(0),
                         int(y_transposed), _stream(stream))
    _check(st, "bwta_gemm_x")
    return out


def bwta_gemm_pack(a: Packed, w: Packed, w_scale: Optional[torch.Tensor], a_scale: float, out_scale: float,
                   out_kind: str = "ternary", y_dtype=torch.float16, design: str = "auto", stream=None,
                   tile=None) -> Packed:
    """bwta_pack_act(bwta_gemm(a, w, ...) in y_dtype, out_scale, out_kind) with the pack
    fused into the GEMM epilogue (Y is never written).  Returns the Packed planes
    of Y's rows [M, ld(N)] -- e.g. FFN1 emitting FFN2's bool input."""
    if a.kind not in ("ternary", "bool") or w.kind != "binary" or a.cols != w.cols:
        raise ValueError("bwta_gemm_pack expects ternary/bool activations and binary weights of equal K")
    if out_kind not in ("ternary", "bool"):
        raise ValueError("out_kind must be 'ternary' or 'bool'")
    ar = a.ref
    m, n, k = ar.shape[-2], w.sgn.shape[-2], a.cols
    dev = ar.device
    ldw = bwta_ld_words(n)
    nz = torch.empty((m, ldw), dtype=torch.int32, device=dev)
    sgn = torch.empty((m, ldw), dtype=torch.int32, device=dev) if out_kind == "ternary" else None
    ws_scale = None if w_scale is None else w_scale.to(device=dev, dtype=torch.float32).contiguous()
    st = lib.bwta_gemm_pack(_ptr(a.sgn), _ptr(a.nz), _KIND[a.kind], m, ar.stride(-2), _ptr(w.sgn), n,
                            w.sgn.stride(-2), k, _ptr(ws_scale), ctypes.c_float(a_scale), _DT[y_dtype],
                            ctypes.c_float(out_scale), _KIND[out_kind], _ptr(sgn), _ptr(nz), ldw,
                            _opts(design, tile), _stream(stream))
    _check(st, "bwta_gemm_pack")
    return Packed(sgn, nz, out_kind, n)


def bwta_gemm_pack_qkv(a: Packed, w: Packed, w_scale: Optional[torch.Tensor], a_scale: float, batch: int,
                       seq: int, heads: int, head_dim: int, out_scales, out_kind: str = "ternary",
                       y_dtype=torch.float16, design: str = "auto", stream=None, tile=None):
    """The QKV projection with the per-head packs fused (Y = [Q | K | V] never written): returns
    (Q, K, V^T) Packed planes [B, H, T, ld(D)], [B, H, T, ld(D)], [B, H, D, ld(T)] -- what
    bwta_pack_act of the per-head views (V transposed) of the stored Y would give."""
    if a.kind not in ("ternary", "bool") or w.kind != "binary" or a.cols != w.cols:
        raise ValueError("bwta_gemm_pack_qkv expects ternary/bool activations and binary weights of equal K")
    if out_kind not in ("ternary", "bool"):
        raise ValueError("out_kind must be 'ternary' or 'bool'")
    ar = a.ref
    m, n, k = ar.shape[-2], w.sgn.shape[-2], a.cols
    dev = ar.device
    ldd, ldt = bwta_ld_words(head_dim), bwta_ld_words(seq)

    def planes(shape):
        nz = torch.empty(shape, dtype=torch.int32, device=dev)
        sg = torch.empty(shape, dtype=torch.int32, device=dev) if out_kind == "ternary" else None
        return sg, nz
    qs, qn = planes((batch, heads, seq, ldd))
    ks, kn = planes((batch, heads, seq, ldd))
    vs, vn = planes((batch, heads, head_dim, ldt))
    sc = (ctypes.c_float * 3)(*[float(x) for x in out_scales])
    ws_scale = None if w_scale is None else w_scale.to(device=dev, dtype=torch.float32).contiguous()
    st = lib.bwta_gemm_pack_qkv(_ptr(a.sgn), _ptr(a.nz), _KIND[a.kind], m, ar.stride(-2), _ptr(w.sgn), n,
                                w.sgn.stride(-2), k, _ptr(ws_scale), ctypes.c_float(a_scale), _DT[y_dtype], batch, seq,
                                heads, head_dim, ctypes.cast(sc, ctypes.c_void_p), _KIND[out_kind], _ptr(qs), _ptr(qn),
                                ldd, _ptr(ks), _ptr(kn), ldd, _ptr(vs), _ptr(vn), ldt, _opts(design, tile),
                                _stream(stream))
    _check(st, "bwta_gemm_pack_qkv")
    return (Packed(qs, qn, out_kind, head_dim), Packed(ks, kn, out_kind, head_dim), Packed(vs, vn, out_kind, seq))


def bwta_attn_qk(q: Packed, k: Packed, alpha: float, out_dtype=torch.float16,
                 out: Optional[torch.Tensor] = None, design: str = "auto", stream=None, tile=None) -> torch.Tensor:
    """S = alpha * ternary(Q) (x) ternary(K)^T per (batch, head).

    q: Packed [B, H, Tq, ld] (or [B, Tq, ld] / [Tq, ld]); k: Packed ternary or binary
    with the same leading dims.  Returns S [..., Tq, Tk]."""
    qr, kr = q.ref, k.ref
    b, h, qbs, qhs = _batch_dims(qr)
    _, _, kbs, khs = _batch_dims(kr)
    tq, tk, dh = qr.shape[-2], kr.shape[-2], q.cols
    if k.cols != dh:
        raise ValueError("Q and K must have the same head dim")
    if out is None:
        out = torch.empty(tuple(qr.shape[:-2]) + (tq, tk), dtype=out_dtype, device=qr.device)
    else:
        _check_out(out, tuple(qr.shape[:-2]) + (tq, tk), qr.device, "bwta_attn_qk")
    _, _, obs, ohs = _batch_dims(out)
    o = _opts(design, tile)
    ws, wsb = _workspace(lib.bwta_attn_qk_workspace_size(b * h, tq, tk, dh, o), qr.device)
    k_nz = k.nz if k.kind == "ternary" else None
    st = lib.bwta_attn_qk(_ptr(q.sgn), _ptr(q.nz), _ptr(k.sgn), _ptr(k_nz), b, h, tq, tk, dh,
                          qr.stride(-2), qbs, qhs, kr.stride(-2), kbs, khs, ctypes.c_float(alpha),
                          _ptr(out), _DT[out.dtype], out.stride(-2), obs, ohs, _ptr(ws), wsb, o,
                          _stream(stream))
    _check(st, "bwta_attn_qk")
    return out


def bwta_attn_pv(p: Packed, vt: Packed, beta: float, out_dtype=torch.float16,
                 out: Optional[torch.Tensor] = None, design: str = "auto", stream=None, tile=None) -> torch.Tensor:
    """O = beta * bool(Att) (x) ternary(V) per (batch, head).

    p: Packed bool (or ternary) [..., Tq, ldp] over Tk; vt: Packed ternary
    [..., Dh, ldv] over Tk (bwta_pack_act(V, transpose=True)).  Returns O [..., Tq, Dh]."""
    pr, vr = p.ref, vt.ref
    b, h, pbs, phs = _batch_dims(pr)
    _, _, vbs, vhs = _batch_dims(vr)
    tq, dh, tk = pr.shape[-2], vr.shape[-2], p.cols
    if vt.cols != tk or vt.kind not in ("ternary", "binary") or p.kind not in ("bool", "ternary"):
        raise ValueError("V^T must be ternary or binary planes over the same Tk as P (bool or ternary)")
    if out is None:
        out = torch.empty(tuple(pr.shape[:-2]) + (tq, dh), dtype=out_dtype, device=pr.device)
    else:
        _check_out(out, tuple(pr.shape[:-2]) + (tq, dh), pr.device, "bwta_attn_pv")
    _, _, obs, ohs = _batch_dims(out)
    o = _opts(design, tile)
    ws, wsb = _workspace(lib.bwta_attn_pv_workspace_size(b * h, tq, tk, dh, o), pr.device)
    p_sgn = p.sgn if p.kind == "ternary" else None
    st = lib.bwta_attn_pv(_ptr(p_sgn), _ptr(p.nz), _ptr(vt.sgn), _ptr(vt.nz), b, h, tq, tk, dh,
                          pr.stride(-2), pbs, phs, vr.stride(-2), vbs, vhs, ctypes.c_float(beta),
                          _ptr(out), _DT[out.dtype], out.stride(-2), obs, ohs, _ptr(ws), wsb, o,
                          _stream(stream))
    _check(st, "bwta_attn_pv")
    return out


def _heads_vec(v, heads: int, dev):
    """Optional per-head scale vector -> a contiguous float32 device tensor [heads] (or None)."""
    if v is None:
        return None
    t = torch.as_tensor(v, dtype=torch.float32, device=dev).reshape(-1).contiguous()
    if t.numel() != heads:
        raise ValueError(f"expected {heads} per-head scales, got {t.numel()}")
    return t


def bwta_attn_decode(q: Packed, k: Packed, vt: Packed, alpha: float, s_att: float, beta: float,
                     out_dtype=torch.float16, p_dtype=torch.float16, return_p: bool = False, stream=None,
                     alpha_heads=None, beta_heads=None):
    """Fused decode attention, one launch (Tq = 1):
    O = beta * bool(round(softmax(alpha * ternary(q) (x) K^T), p_dtype) >= s_att / 2) (x) ternary(V).

    q: Packed ternary [B, H, 1, ld] (one query row per head); k: Packed ternary or binary
    [B, H, Tk, ld]; vt: Packed ternary [B, H, Dh, ld(Tk)] (bwta_pack_act(V, transpose=True)).
    Returns O [B, H, 1, Dh] (and the P planes [B*H, ld(Tk)] with return_p)."""
    qr, kr, vr = q.ref, k.ref, vt.ref
    if q.kind != "ternary" or vt.kind != "ternary" or k.cols != q.cols or vt.cols != kr.shape[-2]:
        raise ValueError("expects ternary q and V^T, K over the same head_dim, V^T over Tk")
    if qr.dim() != 4 or qr.shape[-2] != 1:
        raise ValueError("q must be Packed [B, H, 1, ld] (one query row per head)")
    b, h, qbs, qhs = _batch_dims(qr)
    _, _, kbs, khs = _batch_dims(kr)
    _, _, vbs, vhs = _batch_dims(vr)
    tk, dh = kr.shape[-2], vr.shape[-2]
    out = torch.empty((b, h, 1, dh), dtype=out_dtype, device=qr.device)
    ldp = bwta_ld_words(tk)
    pout = torch.empty((b * h, ldp), dtype=torch.int32, device=qr.device) if return_p else None
    k_nz = k.nz if k.kind == "ternary" else None
    ah, bh_ = _heads_vec(alpha_heads, h, qr.device), _heads_vec(beta_heads, h, qr.device)
    st = lib.bwta_attn_decode(_ptr(q.sgn), _ptr(q.nz), _ptr(k.sgn), _ptr(k_nz), _ptr(vt.sgn), _ptr(vt.nz), b, h, tk,
                              dh, qbs, qhs, kr.stride(-2), kbs, khs, vr.stride(-2), vbs, vhs, ctypes.c_float(alpha),
                              ctypes.c_float(s_att), _DT[p_dtype], ctypes.c_float(beta), _ptr(ah), _ptr(bh_), _ptr(out),
                              _DT[out_dtype],
                              h * dh, dh, _ptr(pout), ldp if return_p else 0, _stream(stream))
    _check(st, "bwta_attn_decode")
    return (out, pout) if return_p else out


def bwta_attn_prefill(q: Packed, k: Packed, vt: Packed, alpha: float, s_att: float, beta: float,
                      out_dtype=torch.float16, p_dtype=torch.float16, return_p: bool = False,
                      out: Optional[torch.Tensor] = None, stream=None, alpha_heads=None, beta_heads=None,
                      causal: bool = False):
    """Fused prefill attention, one launch:
    O = beta * bool(round(softmax(alpha * ternary(Q) (x) K^T), p_dtype) >= s_att / 2) (x) ternary(V).

    q: Packed ternary [B, H, Tq, ld] (or [B, Tq, ld] / [Tq, ld]); k: Packed ternary or binary
    [.., Tk, ld] over the same head_dim (<= 128); vt: Packed ternary [.., Dh, ld(Tk)]
    (bwta_pack_act(V, transpose=True)).  causal: row i sees keys j <= i + Tk - Tq only
    (bwta_attn_prefill_ex).  Returns O [.., Tq, Dh] (and the P planes [entries, Tq, ld(Tk)] with
    return_p)."""
    qr, kr, vr = q.ref, k.ref, vt.ref
    if q.kind != "ternary" or vt.kind != "ternary" or k.cols != q.cols or vt.cols != kr.shape[-2]:
        raise ValueError("expects ternary Q and V^T, K over the same head_dim, V^T over Tk")
    b, h, qbs, qhs = _batch_dims(qr)
    _, _, kbs, khs = _batch_dims(kr)
    _, _, vbs, vhs = _batch_dims(vr)
    tq, tk, dh = qr.shape[-2], kr.shape[-2], vr.shape[-2]
    if dh != q.cols:
        raise ValueError("V^T rows must equal the head_dim")
    shape = tuple(qr.shape[:-2]) + (tq, dh)
    if out is None:
        out = torch.empty(shape, dtype=out_dtype, device=qr.device)
    else:
        _check_out(out, shape, qr.device, "bwta_attn_prefill")
    _, _, obs, ohs = _batch_dims(out)
    ldp = bwta_ld_words(tk)
    pout = torch.empty((b * h, tq, ldp), dtype=torch.int32, device=qr.device) if return_p else None
    k_nz = k.nz if k.kind == "ternary" else None
    ah, bh_ = _heads_vec(alpha_heads, h, qr.device), _heads_vec(beta_heads, h, qr.device)
    st = lib.bwta_attn_prefill_ex(_ptr(q.sgn), _ptr(q.nz), _ptr(k.sgn), _ptr(k_nz), _ptr(vt.sgn), _ptr(vt.nz), b, h,
                                  tq, tk, dh, qr.stride(-2), qbs, qhs, kr.stride(-2), kbs, khs, vr.stride(-2), vbs, vhs,
                                  ctypes.c_float(alpha), ctypes.c_float(s_att), _DT[p_dtype], ctypes.c_float(beta),
                                  _ptr(ah), _ptr(bh_), _ptr(out), _DT[out.dtype], out.stride(-2), obs, ohs, _ptr(pout),
                                  ldp if return_p else 0, int(bool(causal)), _stream(stream))
    _check(st, "bwta_attn_prefill")
    return (out, pout) if return_p else out


def bwta_attn_prefill_pack(q: Packed, k: Packed, vt: Packed, alpha: float, s_att: float, beta: float,
                           out_scale: float, out_kind: str = "ternary", o_dtype=torch.float16,
                           p_dtype=torch.float16, stream=None, alpha_heads=None, beta_heads=None) -> Packed:
    """bwta_pack_act(C, out_scale, out_kind) of the attention context C[b*Tq + t, h*Dh + d] =
    round_{o_dtype}(O_{b,h}[t][d]) of bwta_attn_prefill, the pack fused into its epilogue (O is
    never written): the O-projection's input planes [B*Tq, ld(H*Dh)].  Dh % 32 == 0."""
    qr, kr, vr = q.ref, k.ref, vt.ref
    if out_kind not in ("ternary", "bool"):
        raise ValueError("out_kind must be 'ternary' or 'bool'")
    if q.kind != "ternary" or vt.kind != "ternary" or k.cols != q.cols or vt.cols != kr.shape[-2]:
        raise ValueError("expects ternary Q and V^T, K over the same head_dim, V^T over Tk")
    b, h, qbs, qhs = _batch_dims(qr)
    _, _, kbs, khs = _batch_dims(kr)
    _, _, vbs, vhs = _batch_dims(vr)
    tq, tk, dh = qr.shape[-2], kr.shape[-2], vr.shape[-2]
    ldo = bwta_ld_words(h * dh)
    nz = torch.empty((b * tq, ldo), dtype=torch.int32, device=qr.device)
    sgn = torch.empty((b * tq, ldo), dtype=torch.int32, device=qr.device) if out_kind == "ternary" else None
    k_nz = k.nz if k.kind == "ternary" else None
    ah, bh_ = _heads_vec(alpha_heads, h, qr.device), _heads_vec(beta_heads, h, qr.device)
    st = lib.bwta_attn_prefill_pack(_ptr(q.sgn), _ptr(q.nz), _ptr(k.sgn), _ptr(k_nz), _ptr(vt.sgn), _ptr(vt.nz), b, h,
                                    tq, tk, dh, qr.stride(-2), qbs, qhs, kr.stride(-2), kbs, khs, vr.stride(-2), vbs,
                                    vhs, ctypes.c_float(alpha), ctypes.c_float(s_att), _DT[p_dtype],
                                    ctypes.c_float(beta), _ptr(ah), _ptr(bh_), _DT[o_dtype], ctypes.c_float(out_scale), _KIND[out_kind],
                                    _ptr(sgn), _ptr(nz), ldo, _stream(stream))
    _check(st, "bwta_attn_prefill_pack")
    return Packed(sgn, nz, out_kind, h * dh)


def bwta_attn_pv_pack(p: Packed, vt: Packed, beta: float, out_scale: float, out_kind: str = "ternary",
                      o_dtype=torch.float16, design: str = "auto", stream=None, tile=None) -> Packed:
    """bwta_pack_act(C, out_scale, out_kind) of the attention context C[b, t, h*Dh + d] =
    round(O_{b,h}[t][d]) with the pack fused into the PV epilogue (O is never written):
    the O-projection's input planes [B*Tq, ld(H*Dh)].  p / vt as bwta_attn_pv, 4-D
    [B, H, ...] (or 3-D [H, ...] / 2-D)."""
    if out_kind not in ("ternary", "bool"):
        raise ValueError("out_kind must be 'ternary' or 'bool'")
    pr, vr = p.ref, vt.ref
    b, h, pbs, phs = _batch_dims(pr)
    _, _, vbs, vhs = _batch_dims(vr)
    tq, dh, tk = pr.shape[-2], vr.shape[-2], p.cols
    if vt.cols != tk or vt.kind != "ternary":
        raise ValueError("V^T must be ternary planes over the same Tk as P")
    ldo = bwta_ld_words(h * dh)
    nz = torch.empty((b * tq, ldo), dtype=torch.int32, device=pr.device)
    sgn = torch.empty((b * tq, ldo), dtype=torch.int32, device=pr.device) if out_kind == "ternary" else None
    p_sgn = p.sgn if p.kind == "ternary" else None
    st = lib.bwta_attn_pv_pack(_ptr(p_sgn), _ptr(p.nz), _ptr(vt.sgn), _ptr(vt.nz), b, h, tq, tk, dh,
                               pr.stride(-2), pbs, phs, vr.stride(-2), vbs, vhs, ctypes.c_float(beta),
                               _DT[o_dtype], ctypes.c_float(out_scale), _KIND[out_kind], _ptr(sgn), _ptr(nz), ldo,
                               _opts(design, tile), _stream(stream))
    _check(st, "bwta_attn_pv_pack")
    return Packed(sgn, nz, out_kind, h * dh)
