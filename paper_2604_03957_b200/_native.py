"""ctypes declarations of libbwta.so (include/bwta.h).  Loading fails loudly:
there is no fallback implementation anywhere in this package."""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, os.environ.get("BWTA_LIB", "libbwta.so"))  # BWTA_LIB: tools only

# enums (include/bwta.h)
BWTA_OK = 0
STATUS = {0: "BWTA_OK", 1: "BWTA_ERR_INVALID_VALUE", 2: "BWTA_ERR_SHAPE", 3: "BWTA_ERR_ALIGNMENT",
          4: "BWTA_ERR_UNSUPPORTED", 5: "BWTA_ERR_CUDA", 6: "BWTA_ERR_WORKSPACE"}
F16, BF16, F32, I32 = 0, 1, 2, 3
BINARY, BOOL, TERNARY = 0, 1, 2
DESIGN_AUTO, DESIGN_CUDA_CORE, DESIGN_TCGEN05, DESIGN_MMA_B1 = 0, 1, 2, 3

EXPORTS = ("bwta_ld_words", "bwta_status_string", "bwta_last_cuda_error", "bwta_last_design",
           "bwta_version", "bwta_kernel_launches", "bwta_pack_act", "bwta_pack_act_batch", "bwta_pack_weight",
           "bwta_gemm_workspace_size", "bwta_gemm_pack",
           "bwta_gemm", "bwta_gemm_nnz", "bwta_attn_qk_workspace_size", "bwta_attn_qk",
           "bwta_attn_pv_workspace_size", "bwta_attn_pv", "bwta_attn_pv_pack", "bwta_attn_decode", "bwta_gemm_x",
           "bwta_attn_prefill", "bwta_attn_prefill_ex", "bwta_attn_prefill_pack", "bwta_gemm_pack_qkv", "bwta_gemm_peers",
           "bwta_peer_barrier", "bwta_ipc_handle", "bwta_ipc_open", "bwta_ipc_close")
IPC_HANDLE_BYTES = 64


class Opts(ctypes.Structure):
    _fields_ = [("design", ctypes.c_int32), ("tile_n", ctypes.c_int32), ("cta_group", ctypes.c_int32),
                ("reserved", ctypes.c_int32 * 5)]


class PackDesc(ctypes.Structure):
    """bwta_pack_desc_t (include/bwta.h)."""
    _fields_ = [("x", ctypes.c_void_p), ("x_dt", ctypes.c_int32), ("batch", ctypes.c_int64),
                ("heads", ctypes.c_int64), ("rows", ctypes.c_int64), ("cols", ctypes.c_int64),
                ("ld_x", ctypes.c_int64), ("x_bstride", ctypes.c_int64), ("x_hstride", ctypes.c_int64),
                ("scale", ctypes.c_float), ("kind", ctypes.c_int32), ("transpose", ctypes.c_int32),
                ("sgn", ctypes.c_void_p), ("nz", ctypes.c_void_p), ("ld_words", ctypes.c_int64),
                ("p_bstride", ctypes.c_int64), ("p_hstride", ctypes.c_int64), ("row_nnz", ctypes.c_void_p)]


def _declare(L):
    P = ctypes.c_void_p
    i64 = ctypes.c_int64
    f32 = ctypes.c_float
    i32 = ctypes.c_int
    sz = ctypes.c_size_t
    OP = ctypes.POINTER(Opts)
    L.bwta_ld_words.restype = i64
    L.bwta_ld_words.argtypes = [i64]
    L.bwta_status_string.restype = ctypes.c_char_p
    L.bwta_status_string.argtypes = [i32]
    L.bwta_last_cuda_error.restype = i32
    L.bwta_last_cuda_error.argtypes = []
    L.bwta_last_design.restype = i32
    L.bwta_last_design.argtypes = []
    L.bwta_version.restype = i32
    L.bwta_version.argtypes = []
    L.bwta_kernel_launches.restype = ctypes.c_uint64
    L.bwta_kernel_launches.argtypes = []
    L.bwta_gemm_pack.restype = i32
    L.bwta_gemm_pack.argtypes = [P, P, i32, i64, i64, P, i64, i64, i64, P, f32, i32, f32, i32, P, P, i64, P, P]
    L.bwta_pack_act_batch.restype = i32
    L.bwta_pack_act_batch.argtypes = [P, i32, P]
    L.bwta_pack_act.restype = i32
    L.bwta_pack_act.argtypes = [P, i32, i64, i64, i64, i64, i64, i64, i64, f32, i32, i32,
                                P, P, i64, i64, i64, P, P]
    L.bwta_pack_weight.restype = i32
    L.bwta_pack_weight.argtypes = [P, i32, i64, i64, i64, P, i32, P, i64, P]
    L.bwta_gemm_workspace_size.restype = sz
    L.bwta_gemm_workspace_size.argtypes = [i64, i64, i64, OP]
    L.bwta_gemm.restype = i32
    L.bwta_gemm.argtypes = [P, P, i32, i64, i64, P, i64, i64, i64, P, f32, P, i32, i64, i32,
                            P, sz, OP, P]
    L.bwta_gemm_nnz.restype = i32
    L.bwta_gemm_nnz.argtypes = [P, P, i32, i64, i64, P, P, i64, i64, i64, P, f32, P, i32, i64, i32,
                                P, sz, OP, P]
    L.bwta_attn_qk_workspace_size.restype = sz
    L.bwta_attn_qk_workspace_size.argtypes = [i64, i64, i64, i64, OP]
    L.bwta_attn_qk.restype = i32
    L.bwta_attn_qk.argtypes = [P, P, P, P, i64, i64, i64, i64, i64, i64, i64, i64, i64, i64, i64,
                               f32, P, i32, i64, i64, i64, P, sz, OP, P]
    L.bwta_attn_pv_workspace_size.restype = sz
    L.bwta_attn_pv_workspace_size.argtypes = [i64, i64, i64, i64, OP]
    L.bwta_gemm_x.restype = i32
    L.bwta_gemm_x.argtypes = [P, i32, i64, i64, f32, i32, P, i64, i64, i64, P, P, i32, i64, i32, P]
    L.bwta_attn_decode.restype = i32
    L.bwta_attn_decode.argtypes = [P, P, P, P, P, P, i64, i64, i64, i64, i64, i64, i64, i64, i64, i64, i64, i64,
                                   f32, f32, i32, f32, P, P, P, i32, i64, i64, P, i64, P]
    L.bwta_attn_prefill.restype = i32
    L.bwta_attn_prefill.argtypes = [P, P, P, P, P, P] + [i64] * 14 + [f32, f32, i32, f32, P, P, P, i32, i64, i64, i64,
                                                                      P, i64, P]
    L.bwta_attn_prefill_ex.restype = i32
    L.bwta_attn_prefill_ex.argtypes = [P, P, P, P, P, P] + [i64] * 14 + [f32, f32, i32, f32, P, P, P, i32, i64, i64,
                                                                         i64, P, i64, i32, P]
    L.bwta_gemm_pack_qkv.restype = i32
    L.bwta_gemm_pack_qkv.argtypes = [P, P, i32, i64, i64, P, i64, i64, i64, P, f32, i32, i64, i64, i64, i64, P, i32,
                                     P, P, i64, P, P, i64, P, P, i64, OP, P]
    L.bwta_attn_prefill_pack.restype = i32
    L.bwta_attn_prefill_pack.argtypes = [P, P, P, P, P, P] + [i64] * 14 + [f32, f32, i32, f32, P, P, i32, f32, i32, P,
                                                                           P, i64, P]
    L.bwta_attn_pv_pack.restype = i32
    L.bwta_attn_pv_pack.argtypes = [P, P, P, P, i64, i64, i64, i64, i64, i64, i64, i64, i64, i64, i64,
                                    f32, i32, f32, i32, P, P, i64, P, P]
    L.bwta_gemm_peers.restype = i32
    L.bwta_gemm_peers.argtypes = [P, P, i32, i64, i64, P, i64, i64, i64, P, f32, P, i32, i64, i32,
                                  P, i32, OP, P]
    L.bwta_peer_barrier.restype = i32
    L.bwta_peer_barrier.argtypes = [P, i32, i32, P, P]
    L.bwta_ipc_handle.restype = i32
    L.bwta_ipc_handle.argtypes = [P, P, ctypes.POINTER(i64)]
    L.bwta_ipc_open.restype = i32
    L.bwta_ipc_open.argtypes = [P, i64, ctypes.POINTER(P)]
    L.bwta_ipc_close.restype = i32
    L.bwta_ipc_close.argtypes = [P, i64]
    L.bwta_attn_pv.restype = i32
    L.bwta_attn_pv.argtypes = [P, P, P, P, i64, i64, i64, i64, i64, i64, i64, i64, i64, i64, i64,
                               f32, P, i32, i64, i64, i64, P, sz, OP, P]
    return L


def load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run `python -m paper_2604_03957_b200.build` "
                          "(there is no fallback implementation)")
    return _declare(ctypes.CDLL(LIB_PATH))


lib = load()
