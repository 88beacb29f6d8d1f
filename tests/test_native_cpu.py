"""Host-side checks of the C-ABI library that need no GPU: it loads, exports
every symbol include/bwta.h declares, and validates arguments on the host
(returning the documented status without enqueueing anything)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bwta.h")


@pytest.fixture(scope="module")
def N():
    import __graft_entry__
    __graft_entry__._builder().build()
    from paper_2604_03957_b200 import _native
    return _native


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"BWTA_API\s+[\w\s\*]+?\b(bwta_\w+)\s*\(", text)))


def test_header_declares_the_five_entry_points():
    syms = declared_symbols()
    for s in ("bwta_pack_act", "bwta_pack_weight", "bwta_gemm", "bwta_attn_qk", "bwta_attn_pv"):
        assert s in syms
    # no torch types in the ABI
    assert "torch" not in open(HEADER).read().lower().replace("pytorch", "")


def test_library_exports_every_declared_symbol(N):
    out = subprocess.check_output(["nm", "-D", "--defined-only", N.LIB_PATH], text=True)
    exported = set(re.findall(r"\sT\s(bwta_\w+)", out))
    assert set(declared_symbols()) <= exported
    assert set(N.EXPORTS) == set(declared_symbols())
    L = N.lib
    for s in declared_symbols():
        assert hasattr(L, s)


def test_library_is_built_for_sm100a(N):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", N.LIB_PATH], text=True)
    assert "sm_100a" in out


def test_ld_words_and_strings(N):
    L = N.lib
    for cols, w in ((0, 0), (1, 4), (32, 4), (128, 4), (129, 8), (768, 24), (4096, 128), (11008, 344)):
        assert L.bwta_ld_words(cols) == w
    for st in range(7):
        assert L.bwta_status_string(st).decode().startswith(N.STATUS[st])
    assert L.bwta_version() >= 100


def _pack(L, **kw):
    a = dict(x=16, x_dt=0, batch=1, heads=1, rows=4, cols=64, ld_x=64, x_bs=0, x_hs=0, scale=1.0,
             kind=2, transpose=0, sgn=16, nz=32, ldw=4, p_bs=0, p_hs=0, row_nnz=None, stream=None)
    a.update(kw)
    return L.bwta_pack_act(a["x"], a["x_dt"], a["batch"], a["heads"], a["rows"], a["cols"], a["ld_x"],
                           a["x_bs"], a["x_hs"], ctypes.c_float(a["scale"]), a["kind"], a["transpose"],
                           a["sgn"], a["nz"], a["ldw"], a["p_bs"], a["p_hs"], a["row_nnz"], a["stream"])


def test_pack_act_validation(N):
    L = N.lib
    assert _pack(L, scale=0.0) == 1
    assert _pack(L, scale=-1.0) == 1
    assert _pack(L, scale=float("nan")) == 1
    assert _pack(L, scale=float("inf")) == 1
    assert _pack(L, x=None) == 1
    assert _pack(L, nz=None) == 1
    assert _pack(L, kind=1) == 1            # BOOL must not get a sgn plane
    assert _pack(L, sgn=None) == 1          # TERNARY needs one
    assert _pack(L, kind=0) == 1            # BINARY (W1A1 sign) has a sgn plane only, no nz
    assert _pack(L, x_dt=3) == 4            # I32 input unsupported
    assert _pack(L, rows=-1) == 2
    assert _pack(L, heads=0) == 2
    assert _pack(L, ld_x=63) == 2
    assert _pack(L, ldw=0) == 2
    assert _pack(L, ldw=6, cols=64) == 3    # ld % 4
    assert _pack(L, nz=36) == 3             # 16-byte alignment
    assert _pack(L, transpose=1, rows=200, ldw=4) == 2   # packs along rows -> needs 8 words
    # everything valid: the host checks pass and the device probe reports no sm_100 here
    assert _pack(L) == 4


def test_gemm_and_attention_validation(N):
    L = N.lib
    o = None

    def gemm(**kw):
        a = dict(a_sgn=16, a_nz=32, kind=2, m=4, lda=4, w=48, n=4, ldw=4, k=100, ws=None, s_a=1.0, y=64,
                 y_dt=0, ld_y=4, yt=0)
        a.update(kw)
        return L.bwta_gemm(a["a_sgn"], a["a_nz"], a["kind"], a["m"], a["lda"], a["w"], a["n"], a["ldw"], a["k"],
                           a["ws"], ctypes.c_float(a["s_a"]), a["y"], a["y_dt"], a["ld_y"], a["yt"], None, 0, o, None)
    assert gemm(k=(1 << 24) + 1) == 2
    assert gemm(lda=0) == 2
    assert gemm(lda=5, k=100) == 3 or gemm(lda=5, k=100) == 2
    assert gemm(a_sgn=None) == 1
    assert gemm(kind=1) == 1                 # BOOL activations have no sgn plane
    assert gemm(kind=0) == 1                 # BINARY activations have no nz plane
    assert gemm(y=None) == 1
    assert gemm(y_dt=7) == 4
    assert gemm(ld_y=3) == 2
    assert gemm(yt=1, ld_y=3) == 2
    assert gemm(s_a=float("nan")) == 1
    assert gemm(a_nz=40) == 3
    assert gemm() == 4                       # valid, but no sm_100 device here
    bad = N.Opts()
    bad.design = 9
    st = L.bwta_attn_qk(16, 32, 48, None, 1, 1, 4, 4, 64, 4, 0, 0, 4, 0, 0, ctypes.c_float(0.1), 64, 0, 4,
                        0, 0, None, 0, ctypes.byref(bad), None)
    assert st == 4   # device check comes before the opts check; opts validated on the device path
    assert L.bwta_attn_qk(16, 32, 48, None, 1, 1, 4, 4, 64, 1, 0, 0, 4, 0, 0, ctypes.c_float(0.1), 64, 0, 4,
                          0, 0, None, 0, None, None) == 2
    assert L.bwta_attn_qk(16, 32, 48, None, 70000, 1, 4, 4, 64, 4, 0, 0, 4, 0, 0, ctypes.c_float(0.1), 64, 0,
                          4, 0, 0, None, 0, None, None) == 2
    assert L.bwta_attn_pv(None, 32, 48, 64, 1, 1, 4, 100, 64, 4, 0, 0, 4, 0, 0, ctypes.c_float(0.1), 80, 0,
                          64, 0, 0, None, 0, None, None) == 4
    assert L.bwta_attn_pv(None, 32, 48, None, 1, 1, 4, 100, 64, 4, 0, 0, 4, 0, 0, ctypes.c_float(0.1), 80, 0,
                          64, 0, 0, None, 0, None, None) == 4   # binary V^T (vt_nz NULL): valid
    assert L.bwta_attn_pv(None, 32, None, 64, 1, 1, 4, 100, 64, 4, 0, 0, 4, 0, 0, ctypes.c_float(0.1), 80, 0,
                          64, 0, 0, None, 0, None, None) == 1   # V^T always has a sign plane
    assert L.bwta_attn_pv(None, 32, 48, 64, 1, 1, 4, 100, 64, 4, 0, 0, 4, 0, 0, ctypes.c_float(0.1), 80, 0,
                          63, 0, 0, None, 0, None, None) == 2


def test_pack_weight_validation(N):
    L = N.lib
    assert L.bwta_pack_weight(16, 0, 4, 64, 64, None, 0, 32, 4, None) == 4
    assert L.bwta_pack_weight(None, 0, 4, 64, 64, None, 0, 32, 4, None) == 1
    assert L.bwta_pack_weight(16, 0, 4, 64, 64, None, 1, 32, 4, None) == 1   # per-row mu needs mu
    assert L.bwta_pack_weight(16, 0, 4, 64, 63, None, 0, 32, 4, None) == 2
    assert L.bwta_pack_weight(16, 0, 4, 64, 64, None, 0, 36, 4, None) == 3


def test_product_package_never_touches_the_oracle():
    pkg = os.path.join(ROOT, "paper_2604_03957_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cuh", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "bwta_oracle" not in text and "liborc" not in text, f


def test_attn_pv_pack_validation(N):
    """bwta_attn_pv_pack: host validation before any device work (no GPU here)."""
    L = N.lib

    def pvp(**kw):
        a = dict(p_sgn=None, p_nz=32, vs=48, vn=64, b=1, h=2, tq=4, tk=100, dh=64, ldp=4, ldv=4, beta=0.1,
                 o_dt=0, s_o=1.0, kind=2, o_sgn=80, o_nz=96, ldo=4)
        a.update(kw)
        return L.bwta_attn_pv_pack(a["p_sgn"], a["p_nz"], a["vs"], a["vn"], a["b"], a["h"], a["tq"], a["tk"],
                                   a["dh"], a["ldp"], 0, 0, a["ldv"], 0, 0, ctypes.c_float(a["beta"]), a["o_dt"],
                                   ctypes.c_float(a["s_o"]), a["kind"], a["o_sgn"], a["o_nz"], a["ldo"], None, None)
    assert pvp() == 4                       # valid, but no sm_100 device here
    assert pvp(dh=48) == 4                  # a head must own whole words of the context row
    assert pvp(o_dt=2) == 4                 # fused pack rounds to f16 / bf16 only
    assert pvp(kind=0) == 4                 # the next layer's activations are ternary or bool
    assert pvp(o_nz=None) == 1
    assert pvp(kind=1) == 1                 # BOOL output has no sgn plane
    assert pvp(s_o=0.0) == 1
    assert pvp(s_o=float("inf")) == 1
    assert pvp(ldo=0) == 2                  # < bwta_ld_words(heads * dh)
    assert pvp(ldp=0) == 2
    assert pvp(o_nz=100) == 3               # 16-byte alignment
    assert pvp(b=0) == 0                    # empty problem


def test_attn_decode_validation(N):
    """bwta_attn_decode: host validation before any device work (no GPU here)."""
    L = N.lib

    def dec(**kw):
        a = dict(qs=16, qn=32, ks=48, kn=64, vs=80, vn=96, b=1, h=2, tk=100, dh=64, ldk=4, ldv=4, alpha=0.1,
                 s_att=0.02, p_dt=0, beta=0.1, o=112, o_dt=0, pout=None, ldp=0)
        a.update(kw)
        return L.bwta_attn_decode(a["qs"], a["qn"], a["ks"], a["kn"], a["vs"], a["vn"], a["b"], a["h"], a["tk"],
                                  a["dh"], 0, 0, a["ldk"], 0, 0, a["ldv"], 0, 0, ctypes.c_float(a["alpha"]),
                                  ctypes.c_float(a["s_att"]), a["p_dt"], ctypes.c_float(a["beta"]), None, None, a["o"],
                                  a["o_dt"], 0, 0, a["pout"], a["ldp"], None)
    assert dec() == 4                      # valid, but no sm_100 device here
    assert dec(tk=0) == 2                  # softmax over an empty row
    assert dec(dh=300) == 2                # head_dim <= 256
    assert dec(tk=20000) == 2              # tk <= 16384
    assert dec(ldv=0) == 2                 # < bwta_ld_words(tk)
    assert dec(pout=128, ldp=0) == 2
    assert dec(qs=None) == 1
    assert dec(o=None) == 1
    assert dec(s_att=0.0) == 1
    assert dec(alpha=float("nan")) == 1
    assert dec(p_dt=3) == 4                # P rounds to f16 / bf16 / f32
    assert dec(b=0) == 0
    # every plane is read with 16-byte vector loads: ld % 4 and 16-byte pointers
    assert dec(ldk=5) == 3
    assert dec(ldv=5) == 3
    assert dec(ks=20) == 3
    assert dec(qn=36) == 3
    assert dec(vs=84) == 3
    assert dec(kn=None) == 4               # binary K is valid
    assert dec(pout=132, ldp=4) == 3


def test_fused_pack_entry_points_validate_opts(N):
    """bwta_gemm_pack / bwta_attn_pv_pack reject bad tile overrides and designs on the host,
    before the padding memsets or any launch (a tile_n of 256 would otherwise launch a kernel
    whose TMA boxes and stages disagree)."""
    L = N.lib

    def opts(design=0, tile_n=0, cg=0):
        o = N.Opts()
        o.design, o.tile_n, o.cta_group = design, tile_n, cg
        return ctypes.byref(o)

    def gp(o):
        return L.bwta_gemm_pack(16, 32, 2, 8, 4, 48, 8, 4, 100, None, ctypes.c_float(1.0), 0, ctypes.c_float(1.0),
                                2, 64, 80, 4, o, None)

    def pvp(o):
        return L.bwta_attn_pv_pack(None, 32, 48, 64, 1, 2, 4, 100, 64, 4, 0, 0, 4, 0, 0, ctypes.c_float(0.1), 0,
                                   ctypes.c_float(1.0), 2, 80, 96, 4, o, None)
    for f in (gp, pvp):
        assert f(None) == 4                 # valid, but no sm_100 device here
        assert f(opts(tile_n=128, cg=2)) == 4
        for bad in (opts(tile_n=256), opts(tile_n=32), opts(tile_n=96), opts(cg=3), opts(cg=-1), opts(design=4),
                    opts(design=-1)):
            assert f(bad) == 1
        assert f(opts(design=1)) == 4       # fused pack: design (b) only
        assert f(opts(design=3)) == 4       # (nor the mma.sync b1 prior art)


def test_gemm_x_validation(N):
    """bwta_gemm_x: host validation before any device work (no GPU here)."""
    L = N.lib

    def gx(**kw):
        a = dict(x=16, x_dt=0, m=1, ld_x=100, s=1.0, kind=2, w=48, n=8, ldw=4, k=100, ws=None, y=64, y_dt=0,
                 ld_y=8, yt=0)
        a.update(kw)
        return L.bwta_gemm_x(a["x"], a["x_dt"], a["m"], a["ld_x"], ctypes.c_float(a["s"]), a["kind"], a["w"], a["n"],
                             a["ldw"], a["k"], a["ws"], a["y"], a["y_dt"], a["ld_y"], a["yt"], None)
    assert gx() == 4                        # valid, but no sm_100 device here
    assert gx(m=5) == 4                     # decode sizes only
    assert gx(kind=0) == 4
    assert gx(x_dt=3) == 4
    assert gx(x=None) == 1
    assert gx(s=0.0) == 1
    assert gx(ld_x=99) == 2
    assert gx(ldw=0) == 2
    assert gx(ld_y=7) == 2
    assert gx(w=40) == 3
    assert gx(m=0) == 0


def test_gemm_peers_and_barrier_validation(N):
    """bwta_gemm_peers / bwta_peer_barrier / IPC: host validation before any device work."""
    L = N.lib

    def peers_call(n_peers=1, peers=(80,), **kw):
        a = dict(a_sgn=16, a_nz=32, kind=2, m=64, lda=4, w=48, n=64, ldw=4, k=100, s_a=1.0, y=64, y_dt=0,
                 ld_y=64, yt=1)
        a.update(kw)
        arr = (ctypes.c_void_p * max(1, len(peers)))(*peers)
        return L.bwta_gemm_peers(a["a_sgn"], a["a_nz"], a["kind"], a["m"], a["lda"], a["w"], a["n"], a["ldw"],
                                 a["k"], None, ctypes.c_float(a["s_a"]), a["y"], a["y_dt"], a["ld_y"], a["yt"], arr,
                                 n_peers, None, None)
    assert peers_call(n_peers=8, peers=(80,) * 8) == 1    # at most 7 peers (8 GPUs)
    assert peers_call(n_peers=-1) == 1
    assert peers_call(peers=(0,)) == 1                    # NULL peer
    assert peers_call(peers=(72,)) == 3                   # peer not 16-byte aligned
    assert peers_call(y_dt=2) == 4                        # f32 is not a TMA-store epilogue class
    assert peers_call(y_dt=3) == 4
    assert peers_call(ld_y=68) == 3                       # 16-byte Y rows
    assert peers_call(y=72) == 3
    assert peers_call(a_sgn=None) == 1
    assert peers_call(k=(1 << 24) + 1) == 2
    assert peers_call() == 4                              # valid, but no sm_100 device here
    assert peers_call(n_peers=0, peers=()) == 4
    bad = N.Opts()
    bad.design = 1                                        # design (a) has no peer epilogue
    arr = (ctypes.c_void_p * 1)(80)
    assert L.bwta_gemm_peers(16, 32, 2, 64, 4, 48, 64, 4, 100, None, ctypes.c_float(1.0), 64, 0, 64, 1, arr, 1,
                             ctypes.byref(bad), None) == 4
    flags = (ctypes.c_void_p * 2)(64, 128)
    assert L.bwta_peer_barrier(flags, 2, 2, 256, None) == 1        # rank out of range
    assert L.bwta_peer_barrier(flags, 9, 0, 256, None) == 1        # world > 8
    assert L.bwta_peer_barrier(flags, 2, 0, None, None) == 1       # no count
    assert L.bwta_peer_barrier(flags, 2, 0, 258, None) == 3
    assert L.bwta_peer_barrier((ctypes.c_void_p * 2)(64, 130), 2, 0, 256, None) == 3
    assert L.bwta_peer_barrier(None, 2, 0, 256, None) == 1
    assert L.bwta_peer_barrier(flags, 2, 1, 256, None) == 4        # valid, no device
    assert L.bwta_ipc_handle(None, None, None) == 1
    assert L.bwta_ipc_open(None, 0, None) == 1
    assert L.bwta_ipc_close(None, 0) == 1
