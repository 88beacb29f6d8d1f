// gemm_tc.cu -- design (b): BWTA matmul on the 5th-generation tensor cores.
//
// sm_100a has no binary (b1) MMA (the paper's mma.sync b1 is
// emulated there through IMMA + MOVM), so the codes {-1, 0, +1} are fed to
// tcgen05.mma.kind::mxf4.block_scale as the E2M1 values 0xA / 0x0 / 0x2 with
// every UE8M0 block scale = 1.0: each product is exact and every partial sum
// is an integer of magnitude <= K <= 2^24, so the FP32 accumulator holds the
// integer dot exactly (DESIGN R12; tests/test_parity_gpu_large.py drives
// |dot| up to K = 2^24 - 32).  The dot is the same integer the paper's
// Case 1/2/3 instruction sequences compute; the epilogue applies
// c = fl32(scale[n] * scalar) (w_scale * a_scale, or alpha / beta) exactly as
// design (a).
//
// Operand roles.  The kernel computes D[i][j] = sum_k A[i][k] * B[j][k] with
// BOTH operands read as packed bit planes by TMA (box WPS words x rows: 2 bits
// per ternary element, 1 per bool/binary) and unpacked to E2M1 codes by 8
// unpack warps: kernel-B's into the UMMA 128B-swizzled K-major shared-memory
// layout, kernel-A's (256-K stages) into TMEM, where the MMA reads A.  No
// code image of either operand touches L2 or HBM: the L2 -> SM traffic is the
// bit planes only (measured on B200: an int8 operand image streamed by TMA
// capped the mainloop at ~740 cycles per 128-K stage against the 512-cycle
// int8 tensor floor).  The caller's A (M side) and W (N side) swap roles when
// that tiles the grid better; the epilogue then stores D^T (Y[m][n] = D[n][m]).
//
// CTA (one per SM, persistent over tiles of 128 x BN, or 256 x BN for a CTA
// pair), 20 warps:
//   warp 0     TMA producer: A and B bit-plane slices into a STAGES ring
//   warp 1     MMA issuer: KS/64 x tcgen05.mma (128|256 x BN x 64) per stage,
//              accumulators double-buffered in TMEM (2 x BN columns)
//   warp 2     TMEM allocator
//   warps 4-7, 12-15  epilogue (two warps per TMEM lane quarter, alternate
//              64-column chunks): tcgen05.ld -> fp32 scale -> fp16/bf16/fp32/
//              i32 -> smem staging (stmatrix) -> TMA tensor store (clips tails)
//   warps 8-11 unpack B rows, warps 16-19 unpack A rows: bits (smem) ->
//              E2M1 codes; B codes to smem (fence.proxy.async), A codes (256-K
//              stages) to TMEM with tcgen05.st -- the MMA reads A from TMEM
// Barriers: full (TMA tx), bready (8 unpack warps x CG), empty (MMA commit),
// tfull (accumulator ready), tempty (8 epilogue warps x CG drained TMEM).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "bwta_internal.h"
#include "sm100.cuh"
#include "tc_codes.cuh"

namespace bwta {
namespace {

using namespace sm100;

constexpr int BM = 128;     // MMA M (kernel-A rows per tile), cta_group::1
constexpr int UMMA_KB = 32; // bytes of K per tcgen05.mma (K = 64 four-bit elements)
constexpr int NT = 640;     // 20 warps (128-K stages)
// 256-K stages: two kernel-A unpack groups (warps 16-19, 20-23) take alternate stages
#ifndef BWTA_A_GROUPS
#define BWTA_A_GROUPS 2
#endif
constexpr int A_GROUPS = BWTA_A_GROUPS;
// (the fp16/bf16 TMA-store epilogue class only: the fused-pack and generic epilogues need more than
// the 80 registers a 768-thread CTA leaves and spill -- BERT FFN1 + pack 17.3 -> 20.4 us)
__host__ __device__ constexpr int a_groups(int ks, int eo) { return (ks == 256 && eo == 0) ? A_GROUPS : 1; }
// Epilogue warps per TMEM lane quarter: 2, or 1 (E1) for the fp16/bf16 TMA-store class when a tile's
// mainloop is long (K >= 2048): the epilogue's TMEM / shared-memory / issue bursts then slow the next
// tile's mainloop less (a timeline showed stage periods of 1.1-1.5 k instead of ~0.82 k cycles while
// the 8 epilogue warps drained a tile); the A groups then take warps 12-19 and the CTA has 20 warps.
// Short-K tiles (BERT, K = 768) are epilogue-bound and keep 2 (1 warp: 11.3 -> 13.3 us).
__host__ __device__ constexpr int epi_warps(int ks, int eo, bool e1) { return (e1 && ks == 256 && eo == 0) ? 1 : 2; }
__host__ __device__ constexpr int nt_of(int ks, int eo, bool e1) {
    return NT + 128 * (a_groups(ks, eo) - 1) - 128 * (2 - epi_warps(ks, eo, e1));
}
constexpr int OUT_BUF = 4096;
constexpr int OUT_NBUF = 2;  // staging buffers per epilogue warp (fast path: store k overlaps the staging of k + 1)

using namespace tc;

// barrier wait of the tile kernel; trace builds can switch the wait flavour (BWTA_DBG bits 5-6)
__device__ __forceinline__ void kwait(uint64_t* bar, uint32_t parity, int dbg) {
#ifdef BWTA_TRACE
    const int mode = (dbg >> 5) & 3;
    if (mode == 1) {
        mbar_wait(bar, parity);  // the hinted wait
        return;
    }
    if (mode == 2) {
        while (!mbar_test_wait(bar, parity)) {
        }
        return;
    }
#endif
    (void)dbg;
    // no suspend-time hint: measured 11 % faster per stage than the hinted wait on the C3 GEMM
    // (the hinted wait's wake-up latency sits on every barrier hand-off)
    while (!mbar_try_wait_nh(bar, parity)) {
    }
}

extern __shared__ __align__(16) uint8_t smem_raw[];  // dynamic shared memory of tc_gemm_kernel

// Timeline hooks (tools/trace_gemm.py; compiled only with -DBWTA_TRACE).
// Timestamps go to shared memory (a global store would be waited on by the
// next fence.proxy.async, i.e. MEMBAR.ALL.CTA, and distort the timeline);
// thread 0 copies them out at kernel exit for CTAs 0 and 1.
#ifdef BWTA_TRACE
constexpr int TRACE_EV = 16, TRACE_N = 64;
constexpr int TRACE_BYTES = TRACE_EV * TRACE_N * 8;
__device__ unsigned long long g_trace[2][TRACE_EV][TRACE_N];
#define TRACE_EPI(ev, idx, cond) \
    do {                         \
    } while (0)  // epilogue-internal hooks 12-15 (slots now used by the MMA issuer)
#define TRACE(ev, idx, cond)                                                                          \
    do {                                                                                              \
        if ((cond) && (idx) < TRACE_N)                                                                \
            reinterpret_cast<unsigned long long*>(smem_raw)[(ev) * TRACE_N + (idx)] = clock64();      \
    } while (0)
#else
constexpr int TRACE_BYTES = 0;  // (dynamic smem then starts with the operand ring)
#define TRACE(ev, idx, cond) \
    do {                     \
    } while (0)
#define TRACE_EPI(ev, idx, cond) \
    do {                         \
    } while (0)
#endif

struct TcParams {
    int64_t M, N;  // kernel rows (A side) / cols (B side) per entry
    int num_kb;
    int64_t nh, entries;
    int m_tiles, n_tiles;
    int a_kind, b_kind;  // B_BINARY / B_BOOL / B_TERNARY
    // epilogue
    void* y;
    int y_dt;
    int64_t ldy, y_bs, y_hs;  // elements (direct-store fallback)
    int out_trans;            // memory holds D^T
    int use_tma_store;
    int a_tmem;          // kernel-A codes in TMEM (tcgen05.st; MMA reads A from TMEM), KS = 256 only
    const float* scale;  // per kernel column (or per kernel row if scale_on_rows), may be null
    int scale_on_rows;
    float scalar;
    // fused pack of the output (MatmulArgs::pack_out)
    int pack_out, po_kind;
    uint32_t* po_sgn;
    uint32_t* po_nz;
    int64_t po_ld;
    int64_t po_bs, po_hs;  // words between the planes of consecutive batch / head entries
    float po_tp, po_tn;
    // head-split Q / K / V^T pack (MatmulArgs::po_heads); kernel rows = tokens (never swapped)
    int po_heads;
    int64_t ph_T, ph_H, ph_D;
    FastDiv fd_hd, fd_d, fd_t;  // / (H*D), / D, / T as 32-bit multiply-shift (the int64 divisions
                                // were subroutine calls, several per 32-column chunk)
    uint32_t* ph_sgn[3];
    uint32_t* ph_nz[3];
    int64_t ph_ld[3];
    float ph_tp[3], ph_tn[3];
    int n_peers;     // fused all-gather: the fast epilogue also stores every tile through PeerMaps::m[0 .. n_peers)
    float dot_bias;  // W1A1: K - K_processed (both operands binary; the generic epilogue adds it)
    FastDiv fd_tpe, fd_mt, fd_nh;  // tile -> (entry, m tile, n tile), entry -> (batch, head): 32-bit
                                   // multiply-shift (the int64 divisions were subroutine calls, ~1k
                                   // cycles per tile in the producer; total tiles < 2^31, host-checked)
    int pf_on;                // L2 prefetch of the operand planes at kernel start
    const void* pf_ptr[4];    // plane spans (A0, A1, B0, B1; null / 0 bytes: skip), 16-byte aligned
    uint64_t pf_bytes[4];
    int dbg;  // BWTA_TRACE builds only (tools/trace_gemm.py): 1 skip unpack math, 2 skip MMAs, 4 skip TMA, 8 skip A unpack, 16 skip B unpack, 32/64 wait flavour, 128 skip the B-code proxy fence
};

// output tensor maps of the peers' Y buffers (bwta_gemm_peers): the geometry of tmY at another base
struct PeerMaps {
    CUtensorMap m[MAX_PEERS];
};

__host__ __device__ constexpr int nplanes_of(int kind) { return kind == B_TERNARY ? 2 : 1; }

#ifndef BWTA_SMEM_BUDGET
#define BWTA_SMEM_BUDGET (210 * 1024 + 1280)
#endif
template <int BN, int CG, int KS = 256, int KK = 0>
struct Cfg {
    using S = Stage<KS>;
    // bit planes per operand: 2 unless the operand kinds are fixed at compile time (KK)
    static constexpr int AP = KK ? nplanes_of((KK - 1) / 3) : 2;
    static constexpr int BP = KK ? nplanes_of((KK - 1) % 3) : 2;
    static constexpr int BNC = BN / CG;          // kernel-B rows held (and unpacked) per CTA
    // E2M1 codes, 2 per byte; none for 256-K stages (kernel-A codes live in TMEM there), which
    // deepens the bit/B-code ring (the stage chain TMA -> unpack -> MMA -> commit is latency-bound)
    static constexpr int A_BYTES = KS == 256 ? 0 : BM * S::ROWB;
    static constexpr int B_BYTES = BNC * S::ROWB;
    static constexpr int ABITS = AP * BM * S::WPS * 4;  // AP planes x WPS words per row
    static constexpr int BBITS = BP * BNC * S::WPS * 4;
    static constexpr int STAGE = A_BYTES + B_BYTES + ABITS + BBITS;
    static constexpr int OUT_BYTES = 8 * OUT_NBUF * OUT_BUF;                // OUT_NBUF staging buffers per epilogue warp
    static constexpr int SCALE_COLS = BN;  // columns per epilogue warp (one warp per lane quarter: all BN)
    static constexpr int SCALE_BYTES = 8 * SCALE_COLS * 4;                  // per-warp column scales
    static constexpr int STAGES_FIT = (BWTA_SMEM_BUDGET - 1280 - OUT_BYTES - SCALE_BYTES - TRACE_BYTES) / STAGE;
    static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;
    static constexpr int BAR_BYTES = 256;
    static constexpr int SMEM = 1024 + STAGES * STAGE + OUT_BYTES + SCALE_BYTES + BAR_BYTES + TRACE_BYTES;
    // TMEM: two f32 accumulators of BN columns, then the UE8M0 scale factors
    // (all 1.0): SFA at SF_COL (4 columns used for M = 128), SFB at SF_COL + 8
    // (up to 8 columns).
    static constexpr int SF_COL = 2 * BN;
    // a_tmem mode: SA stages of kernel-A codes (32 columns = 256 K each) after the scale factors
    static constexpr int A_COL = 2 * BN + 16;
    static constexpr int SA_FIT = (512 - A_COL) / 32;
    static constexpr int SA0 = SA_FIT > 8 ? 8 : SA_FIT;
    static constexpr int SA = SA0 > STAGES ? STAGES : SA0;
    static constexpr int TMEM_COLS = 512;
    static_assert(SF_COL + 16 <= TMEM_COLS, "accumulators + scale factors exceed TMEM");
    static_assert(STAGES >= 2, "pipeline too shallow");
    static_assert(KS != 256 || SA <= STAGES, "the A code ring is released through empty[]");
    static_assert(BNC % 8 == 0, "swizzle atoms are 8 rows");
    static_assert(A_BYTES % 1024 == 0 && B_BYTES % 1024 == 0 && OUT_BYTES % 1024 == 0 && SCALE_BYTES % 128 == 0 &&
                      ABITS % 128 == 0 && BBITS % 128 == 0,
                  "smem region alignment");
};

__device__ __forceinline__ uint32_t fdiv_u32(uint32_t n, const FastDiv& f) { return (__umulhi(n, f.mul) + n) >> f.shift; }
struct TileCoord {
    int mt, nt, eb, eh;
};
__device__ __forceinline__ TileCoord tile_coord(const TcParams& p, int64_t t) {
    const uint32_t tu = uint32_t(t);
    const uint32_t e = fdiv_u32(tu, p.fd_tpe);
    const uint32_t r = tu - e * p.fd_tpe.d;
    const uint32_t nt = fdiv_u32(r, p.fd_mt);
    const uint32_t eb = fdiv_u32(e, p.fd_nh);
    return TileCoord{int(r - nt * p.fd_mt.d), int(nt), int(eb), int(e - eb * p.fd_nh.d)};
}

// f32 accumulator (the exact integer dot) -> dot / scaled output (R5)
__device__ __forceinline__ int32_t dot_of(uint32_t acc) { return __float2int_rn(__uint_as_float(acc)); }
__device__ __forceinline__ float scaled(uint32_t acc, float c) { return __fmul_rn(__uint_as_float(acc), c); }

__device__ __forceinline__ uint32_t pack2(int dt, float lo, float hi) {
    if (dt == DT_F16) {
        __half2 h = __halves2half2(__float2half_rn(lo), __float2half_rn(hi));
        return *reinterpret_cast<uint32_t*>(&h);
    }
    __nv_bfloat162 h = __halves2bfloat162(__float2bfloat16_rn(lo), __float2bfloat16_rn(hi));
    return *reinterpret_cast<uint32_t*>(&h);
}


// ---------------------------------------------------------------------------
// Epilogue.  8 warps: warp (h, q) (warps 4+q and 12+q) owns TMEM lane quarter
// q (kernel rows 32q..32q+31 of the CTA's 128) and the column chunks
// c = h, h+2, ... of CW = 128/ES columns (one 128-byte output row each).
// A chunk is staged in the warp's own 4 KB smem buffer and written by one
// TMA tensor store (which clips the M/N tails).
//
// Fast path (fp16/bf16 out, TMA store): tcgen05.ld.16x256b puts the
// accumulators in the mma.sync m16n8 fragment layout, two adjacent columns
// per register pair, so a pair converts to one f16x2 / bf16x2 word and
// stmatrix (.trans for D^T) writes 8x8 blocks -- 1 shared store per 8
// outputs per thread, no shuffles.  Scaling: the f32 accumulator is the
// exact dot, so y = fl(acc * c) is R5's fl(float(dot) * c) with one FMUL.
// ---------------------------------------------------------------------------

// generic tile: 32x32b loads, any output type, TMA or direct stores.  A
// chunk (one 128-byte output row per thread, CW columns) is processed in
// 32-column halves to bound register use.
template <int BN, int ES>
__device__ __forceinline__ void epi_tile_generic(const TcParams& p, const CUtensorMap& tmY, uint32_t tacc,
                                                 uint8_t* stg, int q, int h, int lane, int64_t mrow0, int nt,
                                                 int eb, int eh) {
    constexpr int CW = 128 / ES;
    const int64_t row = mrow0 + q * 32 + lane;  // kernel row of this thread
    const bool rok = row < p.M;
    float crow = p.scalar;
    if (p.scale_on_rows && p.scale) crow = __fmul_rn(__ldg(p.scale + (rok ? row : 0)), p.scalar);
    const bool col_scaled = !p.scale_on_rows && p.scale;
    const int64_t ybase = int64_t(eb) * p.y_bs + int64_t(eh) * p.y_hs;
    const uint32_t sbase = smem_u32(stg);
#pragma unroll 1
    for (int c0 = h * CW; c0 < BN; c0 += 2 * CW) {
        const int64_t n0 = int64_t(nt) * BN + c0;
        if (n0 >= p.N) break;
        if (p.use_tma_store) {
            if (lane == 0) bulk_wait_read<0>();
            __syncwarp();
        }
#pragma unroll 1
        for (int u = 0; u < CW / 32; ++u) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(tacc + (uint32_t(q * 32) << 16) + uint32_t(c0 + 32 * u), v);
            tmem_wait_ld();
            if (p.dot_bias != 0.f) {  // W1A1: remove the +1 x +1 products of the K padding (exact)
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__fadd_rn(__uint_as_float(v[j]), p.dot_bias));
            }
            const int64_t nl = n0 + 32 * u + lane;
            const float cl = col_scaled ? __fmul_rn(__ldg(p.scale + (nl < p.N ? nl : 0)), p.scalar) : crow;
            float f[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) f[j] = scaled(v[j], col_scaled ? __shfl_sync(0xffffffffu, cl, j) : crow);
            if (p.use_tma_store) {
                if (!p.out_trans) {
                    // row `lane` of a [32 rows x 128 B] box, 128B-swizzled (fp16/bf16: this half = 64 B)
                    if (ES == 2) {
                        uint32_t w[16];
#pragma unroll
                        for (int j = 0; j < 16; ++j) w[j] = pack2(p.y_dt, f[2 * j], f[2 * j + 1]);
#pragma unroll
                        for (int qq = 0; qq < 4; ++qq)
                            sts128(sbase + lane * 128 + (((4 * u + qq) ^ (lane & 7)) << 4), w[4 * qq], w[4 * qq + 1],
                                   w[4 * qq + 2], w[4 * qq + 3]);
                    } else {
#pragma unroll
                        for (int qq = 0; qq < 8; ++qq) {
                            uint32_t o[4];
#pragma unroll
                            for (int x = 0; x < 4; ++x)
                                o[x] = p.y_dt == DT_F32 ? __float_as_uint(f[4 * qq + x]) : uint32_t(dot_of(v[4 * qq + x]));
                            sts128(sbase + lane * 128 + ((qq ^ (lane & 7)) << 4), o[0], o[1], o[2], o[3]);
                        }
                    }
                } else {
                    // box [CW kernel-cols][32 kernel-rows]: lane is the contiguous index
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const uint32_t a = sbase + (32 * u + j) * 32 * ES + lane * ES;
                        if (ES == 2) {
                            const uint32_t h2 = pack2(p.y_dt, f[j], 0.f);
                            asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"(uint16_t(h2 & 0xffffu)) : "memory");
                        } else {
                            const uint32_t o = p.y_dt == DT_F32 ? __float_as_uint(f[j]) : uint32_t(dot_of(v[j]));
                            asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(o) : "memory");
                        }
                    }
                }
            } else {
                // direct stores (outputs whose layout TMA cannot describe)
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const int64_t n = n0 + 32 * u + j;
                    if (rok && n < p.N) {
                        const int64_t idx = ybase + (p.out_trans ? n * p.ldy + row : row * p.ldy + n);
                        if (p.y_dt == DT_F16) reinterpret_cast<__half*>(p.y)[idx] = __float2half_rn(f[j]);
                        else if (p.y_dt == DT_BF16) reinterpret_cast<__nv_bfloat16*>(p.y)[idx] = __float2bfloat16_rn(f[j]);
                        else if (p.y_dt == DT_F32) reinterpret_cast<float*>(p.y)[idx] = f[j];
                        else reinterpret_cast<int32_t*>(p.y)[idx] = dot_of(v[j]);
                    }
                }
            }
        }
        if (p.use_tma_store) {
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
                if (!p.out_trans) tma_store_4d(&tmY, stg, int(n0), int(mrow0 + q * 32), eh, eb);
                else tma_store_4d(&tmY, stg, int(mrow0 + q * 32), int(n0), eh, eb);
                bulk_commit();
            }
        }
    }
}

// fast tile: fp16/bf16 output through TMA (see above).  cs = this warp's
// column scales (c * 2^-12, 64 per chunk) when column-scaled; cr = the
// thread's four row scales (rows 16b + 8i + lane/4) when row-scaled.
template <int BN, bool BF16, int EPW = 2>
__device__ __forceinline__ void epi_tile_fast(const TcParams& p, const CUtensorMap& tmY, const PeerMaps& pm,
                                              uint32_t tacc, uint8_t* stg0,
                                              const float* cs, bool col_scaled, const float (&cr)[4], int q, int h,
                                              int lane, int64_t mrow0, int nt, int eb, int eh, int tix, int& nstore) {
    constexpr int CW = 64;
    const bool tr = h == 0 && q == 0 && lane == 0;
    (void)tr;
    (void)tix;
    const int t0 = lane & 3;
    // stmatrix addresses: matrix mi = lane/8 (column group offset mi/2, row half mi%2), line li = lane%8
    const int mi = lane >> 3, li = lane & 7;
#pragma unroll 1
    for (int i = 0, c0 = h * CW; c0 < BN; ++i, c0 += EPW * CW) {
        const int64_t n0 = int64_t(nt) * BN + c0;
        if (n0 >= p.N) break;
        uint8_t* stg = stg0 + (nstore % OUT_NBUF) * OUT_BUF;
        const uint32_t sbase = smem_u32(stg);
        ++nstore;
#pragma unroll
        for (int b = 0; b < 2; ++b) {  // 16-lane block b: rows 16b .. 16b+15 of the warp's 32
            uint32_t v[32];
            tmem_ld_16x256b_x8(tacc + (uint32_t(q * 32 + 16 * b) << 16) + uint32_t(c0), v);
            tmem_wait_ld();
            TRACE(9, tix * 8 + i * 2 + b, tr);
            // pk[2g + i2]: rows 16b + 8*i2 + lane/4, columns 8g + 2*t0, +1
            uint32_t pk[16];
#pragma unroll
            for (int g = 0; g < 8; ++g) {
                float ca = 0.f, cb = 0.f;
                if (col_scaled) {
                    const float2 c2 = *reinterpret_cast<const float2*>(cs + i * CW + 8 * g + 2 * t0);
                    ca = c2.x;
                    cb = c2.y;
                }
#pragma unroll
                for (int i2 = 0; i2 < 2; ++i2) {
                    const float c_lo = col_scaled ? ca : cr[2 * b + i2];
                    const float c_hi = col_scaled ? cb : cr[2 * b + i2];
                    const float f0 = scaled(v[4 * g + 2 * i2], c_lo);
                    const float f1 = scaled(v[4 * g + 2 * i2 + 1], c_hi);
                    pk[2 * g + i2] = pack2(BF16 ? DT_BF16 : DT_F16, f0, f1);
                }
            }
            if (b == 0) {
                TRACE_EPI(13, tix * 4 + i, tr);
                if (lane == 0) bulk_wait_read<OUT_NBUF - 1>();  // the store that last used this buffer has read it
                __syncwarp();
                TRACE_EPI(14, tix * 4 + i, tr);
            }
#pragma unroll
            for (int gp = 0; gp < 4; ++gp) {
                const int g = 2 * gp + (mi >> 1);
                const int r = 16 * b + 8 * (mi & 1);  // first row of this thread's matrix
                if (!p.out_trans) {
                    const int row = r + li;
                    stmatrix_x4(sbase + row * 128 + ((g ^ (row & 7)) << 4), pk[4 * gp], pk[4 * gp + 1],
                                pk[4 * gp + 2], pk[4 * gp + 3]);
                } else {
                    stmatrix_x4_trans(sbase + (8 * g + li) * 64 + r * 2, pk[4 * gp], pk[4 * gp + 1], pk[4 * gp + 2],
                                      pk[4 * gp + 3]);
                }
            }
            if (b == 0) TRACE_EPI(15, tix * 4 + i, tr);
        }
        fence_proxy_async_smem();
        __syncwarp();
        TRACE_EPI(12, tix * 4 + i, tr);
        if (lane == 0) {
            const int c0s = p.out_trans ? int(mrow0 + q * 32) : int(n0), c1s = p.out_trans ? int(n0) : int(mrow0 + q * 32);
            tma_store_4d(&tmY, stg, c0s, c1s, eh, eb);
            // fused all-gather: the same staged chunk to every peer's Y (NVLink writes), one bulk group
            for (int pi = 0; pi < p.n_peers; ++pi) tma_store_4d(&pm.m[pi], stg, c0s, c1s, eh, eb);
            bulk_commit();
        }
    }
}

// Fused next-layer pack: the tile's outputs y = fl32(dot * c) (R5) are
// quantized exactly as bwta_pack_act would quantize the stored Y (y rounded
// to fp16 / bf16, then R1-R3): the host turns the storage thresholds into fp32
// rounding boundaries (api.cu rounding_threshold), so +1 iff y >= po_tp and
// -1 iff y <= -po_tn on the fp32 value, NaN -> 0; the bits
// go straight into the next layer's planes (rows = the M rows of Y, bits
// along N).  32x32b TMEM loads: thread = kernel row, 32 kernel columns.
//  * not swapped (kernel row = m): a thread owns 32 consecutive n of its row
//    -> one word per plane per thread;
//  * swapped (kernel row = n): a warp's 32 lanes are 32 consecutive n ->
//    one __ballot_sync per kernel column (= output row m), lane j stores
//    the word of column j.
// smallest integer d (|d| <= 2^25) with fl32(d * c) >= t, for c > 0 finite
__device__ __forceinline__ float int_threshold_ge(float t, float c) {
    float d = ceilf(t / c);
    d = fminf(fmaxf(d, -33554432.f), 33554432.f);
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        if (__fmul_rn(d, c) < t) d += 1.f;
        else if (__fmul_rn(d - 1.f, c) >= t) d -= 1.f;
    }
    return d;
}

template <int BN>
__device__ __forceinline__ void epi_tile_pack(const TcParams& p, uint32_t tacc, uint8_t* scratch, int q, int h,
                                              int lane, int64_t mrow0, int nt, int64_t eoff) {
    const bool ternary = p.po_kind == K_TERNARY;
    const int64_t row = mrow0 + q * 32 + lane;  // kernel row of this thread
    const bool rok = row < p.M;
    float crow = p.scalar;
    if (p.scale_on_rows && p.scale) crow = __fmul_rn(__ldg(p.scale + (rok ? row : 0)), p.scalar);
    const bool col_scaled = !p.scale_on_rows && p.scale;
    // integer thresholds of the swapped orientation (per-lane scale), when every c > 0 is finite:
    // y >= tp <=> acc >= tpi;  y <= -tn <=> -acc*c >= tn <=> -acc >= tni' <=> acc <= tni
    const bool c_pos = !col_scaled && crow > 0.f && crow <= 3.4e38f;
    const bool ith = p.out_trans && __all_sync(0xffffffffu, c_pos);
    float tpi = 0.f, tni = 0.f;
    if (ith) {
        tpi = int_threshold_ge(p.po_tp, crow);
        tni = -int_threshold_ge(p.po_tn, crow);
    }
#pragma unroll 1
    for (int c0 = h * 32; c0 < BN; c0 += 64) {
        const int64_t n0 = int64_t(nt) * BN + c0;  // first kernel column (a multiple of 32)
        if (n0 >= p.N) break;
        uint32_t v[32];
        tmem_ld_32x32b_x32(tacc + (uint32_t(q * 32) << 16) + uint32_t(c0), v);
        tmem_wait_ld();
        float cl = crow;
        if (col_scaled) {
            const int64_t nl = n0 + lane;
            cl = __fmul_rn(__ldg(p.scale + (nl < p.N ? nl : 0)), p.scalar);
        }
        if (p.po_heads) {
            // chunk of Q / K / V (warp-uniform: H*D and D are multiples of 32); thread = token row
            const int reg = int(fdiv_u32(uint32_t(n0), p.fd_hd));
            const uint32_t nl = uint32_t(n0) - uint32_t(reg) * p.fd_hd.d;
            const int64_t hh = fdiv_u32(nl, p.fd_d), dcol = nl - uint32_t(hh) * p.fd_d.d;
            const float tp = p.ph_tp[reg], tn = p.ph_tn[reg];
            uint32_t* psg = p.ph_sgn[reg];
            uint32_t* pnz = p.ph_nz[reg];
            if (reg < 2) {  // Q / K: the thread's 32 columns are 32 consecutive head dims of its token
                uint32_t pos = 0, neg = 0;
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const float c = col_scaled ? __shfl_sync(0xffffffffu, cl, j) : crow;
                    const float y = scaled(v[j], c);
                    pos |= uint32_t(y >= tp) << j;
                    neg |= uint32_t(y <= -tn) << j;
                }
                if (rok) {
                    const int64_t b = fdiv_u32(uint32_t(row), p.fd_t), t = row - b * p.ph_T;
                    const int64_t off = ((b * p.ph_H + hh) * p.ph_T + t) * p.ph_ld[reg] + dcol / 32;
                    pnz[off] = ternary ? (pos | neg) : pos;
                    if (ternary) psg[off] = neg;
                    if (dcol + 32 == p.ph_D)  // the row's last data word: zero its padding words (R8)
                        for (int64_t w = 1; w < p.ph_ld[reg] - dcol / 32; ++w) {
                            pnz[off + w] = 0u;
                            if (ternary) psg[off + w] = 0u;
                        }
                }
            } else {        // V^T: the warp's 32 lanes are 32 consecutive tokens of one sequence
                uint32_t* sc = reinterpret_cast<uint32_t*>(scratch);
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const float c = col_scaled ? __shfl_sync(0xffffffffu, cl, j) : crow;
                    const float y = scaled(v[j], c);
                    sc[j] = __ballot_sync(0xffffffffu, rok && y >= tp);
                    if (ternary) sc[32 + j] = __ballot_sync(0xffffffffu, rok && y <= -tn);
                }
                __syncwarp();
                const uint32_t my_pos = sc[lane];
                const uint32_t my_neg = ternary ? sc[32 + lane] : 0u;
                __syncwarp();
                const int64_t m0 = mrow0 + q * 32;
                if (m0 < p.M) {
                    const int64_t b = fdiv_u32(uint32_t(m0), p.fd_t), t0 = m0 - b * p.ph_T;
                    const int64_t off = ((b * p.ph_H + hh) * p.ph_D + dcol + lane) * p.ph_ld[2] + t0 / 32;
                    pnz[off] = ternary ? (my_pos | my_neg) : my_pos;
                    if (ternary) psg[off] = my_neg;
                    if (t0 + 32 == p.ph_T)  // the row's last data word: zero its padding words (R8)
                        for (int64_t w = 1; w < p.ph_ld[2] - t0 / 32; ++w) {
                            pnz[off + w] = 0u;
                            if (ternary) psg[off + w] = 0u;
                        }
                }
            }
        } else if (!p.out_trans) {
            // this thread's 32 columns are 32 consecutive elements of its output row
            uint32_t pos = 0, neg = 0;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const float c = col_scaled ? __shfl_sync(0xffffffffu, cl, j) : crow;
                const float y = scaled(v[j], c);
                const bool valid = n0 + j < p.N;
                pos |= uint32_t(valid && y >= p.po_tp) << j;
                neg |= uint32_t(valid && y <= -p.po_tn) << j;
            }
            if (rok) {
                const int64_t off = eoff + row * p.po_ld + n0 / 32;
                p.po_nz[off] = ternary ? (pos | neg) : pos;
                if (ternary) p.po_sgn[off] = neg;
            }
        } else {
            // lanes are 32 consecutive elements (kernel rows) of output row n0 + j:
            // one ballot per column and plane; the (warp-uniform) ballot words go
            // through the warp's scratch so lane j picks up column j's word.
            // With a per-lane scale c > 0 the tests run on the exact integer
            // accumulator against integer thresholds (fl(d * c) is monotonic in d).
            uint32_t* sc = reinterpret_cast<uint32_t*>(scratch);
            if (ith) {
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const float acc = __uint_as_float(v[j]);
                    const uint32_t wp = __ballot_sync(0xffffffffu, rok && acc >= tpi);
                    sc[j] = wp;
                    if (ternary) sc[32 + j] = __ballot_sync(0xffffffffu, rok && acc <= tni);
                }
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const float c = col_scaled ? __shfl_sync(0xffffffffu, cl, j) : crow;
                    const float y = scaled(v[j], c);
                    sc[j] = __ballot_sync(0xffffffffu, rok && y >= p.po_tp);
                    if (ternary) sc[32 + j] = __ballot_sync(0xffffffffu, rok && y <= -p.po_tn);
                }
            }
            __syncwarp();
            const uint32_t my_pos = sc[lane];
            const uint32_t my_neg = ternary ? sc[32 + lane] : 0u;
            __syncwarp();
            // (a word past the last valid element is padding: zeroed by the host)
            if (n0 + lane < p.N && mrow0 + q * 32 < p.M) {
                const int64_t off = eoff + (n0 + lane) * p.po_ld + (mrow0 + q * 32) / 32;
                p.po_nz[off] = ternary ? (my_pos | my_neg) : my_pos;
                if (ternary) p.po_sgn[off] = my_neg;
            }
        }
    }
}

// EO = 0: the kernel only ever runs the fp16/bf16 TMA-store epilogue (the common case; the other
// variants are not compiled in, which shrinks the instruction footprint); EO = 2: only the fused
// next-layer pack; EO = 1: the generic epilogue (f32 / i32 outputs, layouts TMA cannot store).
template <int BN, int ES, int CG, int EO, int EPW = 2>
__device__ __forceinline__ void epilogue(const TcParams& p, const CUtensorMap& tmY, const PeerMaps& pm,
                                         uint32_t tmem_base, uint8_t* sOut,
                                         float* sScale, uint64_t* tfull, uint64_t* tempty, int q, int h, int lane,
                                         int64_t tiles_per_entry, int64_t total, int rank, int64_t t0,
                                         int64_t tstep) {
    uint8_t* stg = sOut + (h * 4 + q) * OUT_NBUF * OUT_BUF;
    int nstore = 0;  // fast path: chunks stored by this warp (selects the staging buffer)
    float* cs = sScale + (h * 4 + q) * Cfg<BN, CG>::SCALE_COLS;
    const bool fast_ok = ES == 2 && p.use_tma_store && p.dot_bias == 0.f;
    const bool col_scaled = !p.scale_on_rows && p.scale;
    int acc = 0;
    uint32_t acc_phase = 0;
    int tix = 0;
    for (int64_t t = t0; t < total; t += tstep, ++tix) {
        const TileCoord tc = tile_coord(p, t);
        const int mt = tc.mt, nt = tc.nt, eb = tc.eb, eh = tc.eh;
        const int64_t mrow0 = int64_t(mt) * BM * CG + rank * BM;  // first kernel row of this CTA
        // with an odd number of 64-column chunks the two warps of a lane
        // quarter alternate which of them takes the extra chunk
        const int hh = (EPW == 2 && ((BN / 64) & 1)) ? (h ^ (tix & 1)) : h;
        // scales of this tile (loaded before the accumulator is ready)
        const bool ok = fast_ok;
        float cr[4] = {0.f, 0.f, 0.f, 0.f};
        if (fast_ok) {
            if (col_scaled) {
                // this warp's chunks: columns nt*BN + (2i + h)*64 + [0, 64)
                for (int i = 0, c0 = hh * 64; c0 < BN; ++i, c0 += 64 * EPW) {
                    const int64_t n = int64_t(nt) * BN + c0 + 2 * lane;
                    const float a = __fmul_rn(__ldg(p.scale + (n < p.N ? n : 0)), p.scalar);
                    const float b = __fmul_rn(__ldg(p.scale + (n + 1 < p.N ? n + 1 : 0)), p.scalar);
                    *reinterpret_cast<float2*>(cs + i * 64 + 2 * lane) = make_float2(a, b);
                }
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    float c = p.scalar;
                    if (p.scale_on_rows && p.scale) {
                        const int64_t row = mrow0 + q * 32 + 16 * (k >> 1) + 8 * (k & 1) + (lane >> 2);
                        c = __fmul_rn(__ldg(p.scale + (row < p.M ? row : 0)), p.scalar);
                    }
                    cr[k] = c;
                }
            }
            __syncwarp();
        }
        kwait(&tfull[acc], acc_phase, p.dbg);
        tc_fence_after();
        TRACE(5, tix, h == 0 && q == 0 && lane == 0);
        const uint32_t tacc = tmem_base + uint32_t(acc * BN);
        if (EO == 2) {
            epi_tile_pack<BN>(p, tacc, reinterpret_cast<uint8_t*>(cs), q, hh, lane, mrow0, nt,
                              int64_t(eb) * p.po_bs + int64_t(eh) * p.po_hs);
        } else if (EO == 0 || (EO == 1 && ok)) {
            if (p.y_dt == DT_BF16)
                epi_tile_fast<BN, true, EPW>(p, tmY, pm, tacc, stg, cs, col_scaled, cr, q, hh, lane, mrow0, nt, eb, eh,
                                             tix, nstore);
            else
                epi_tile_fast<BN, false, EPW>(p, tmY, pm, tacc, stg, cs, col_scaled, cr, q, hh, lane, mrow0, nt, eb,
                                              eh, tix, nstore);
        } else if constexpr (EO == 1) {
            epi_tile_generic<BN, ES>(p, tmY, tacc, stg, q, hh, lane, mrow0, nt, eb, eh);
        }
        tc_fence_before();
        __syncwarp();
        TRACE(6, tix, h == 0 && q == 0 && lane == 0);
        if (lane == 0) {
            if (CG == 1) mbar_arrive(&tempty[acc]);
            else mbar_arrive_cluster(mapa_smem(&tempty[acc], 0));  // the leader owns the MMA
        }
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
    }
    if (lane == 0) bulk_wait_all();
}

// items [i0, rows * WPS/4) step `step` of one operand slice: item i = word quad i / rows of
// row i % rows (16 bytes per plane -> 4 x 16 bytes of codes); warp-uniform kind
template <int KIND, int KS>
__device__ __forceinline__ void unpack_quad(uint32_t p0addr, uint32_t p1addr, uint32_t rowaddr, int r, int h) {
    const int sw = KS == 256 ? (r & 7) : ((r >> 1) & 3);
    const uint4 w0 = lds128(p0addr + 16 * h);
    uint4 w1 = make_uint4(0, 0, 0, 0);
    if (KIND == B_TERNARY) w1 = lds128(p1addr + 16 * h);
    uint32_t x0[4] = {w0.x, w0.y, w0.z, w0.w};
    const uint32_t x1[4] = {w1.x, w1.y, w1.z, w1.w};
    if (KIND == B_TERNARY) {
#pragma unroll
        for (int g = 0; g < 4; ++g) x0[g] &= x1[g];  // canonical sgn (subset of nz)
    }
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        uint32_t o[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) o[j] = unpack_word<KIND>(x0[g], x1[g], j);
        sts128(rowaddr + (((4 * h + g) ^ sw) << 4), o[0], o[1], o[2], o[3]);
    }
}
template <int KS, int ROWS, int STEP>
__device__ __forceinline__ void unpack_quads(int kind, uint32_t bits, uint32_t dst, int i0) {
    // ROWS / STEP compile-time: the item -> (row, quad) split is a multiply-shift, not a division
    constexpr int RB = Stage<KS>::WPS * 4;  // bit bytes per row per plane
    constexpr int ROWB = Stage<KS>::ROWB;
    constexpr int ITEMS = ROWS * (Stage<KS>::WPS / 4);
    constexpr int PB = ROWS * RB;           // plane bytes
    if (kind == B_TERNARY) {
#pragma unroll
        for (int i = i0; i < ITEMS; i += STEP) {
            const int r = i % ROWS, h = i / ROWS;
            unpack_quad<B_TERNARY, KS>(bits + r * RB, bits + PB + r * RB, dst + r * ROWB, r, h);
        }
    } else if (kind == B_BOOL) {
#pragma unroll
        for (int i = i0; i < ITEMS; i += STEP) {
            const int r = i % ROWS, h = i / ROWS;
            unpack_quad<B_BOOL, KS>(bits + r * RB, 0, dst + r * ROWB, r, h);
        }
    } else {
#pragma unroll
        for (int i = i0; i < ITEMS; i += STEP) {
            const int r = i % ROWS, h = i / ROWS;
            unpack_quad<B_BINARY, KS>(bits + r * RB, 0, dst + r * ROWB, r, h);
        }
    }
}

// One 256-K operand row (8 words per plane) -> 32 TMEM columns (code word 4g + j
// in column 4g + j: the same K order as the shared-memory layout's 16-byte chunks).
template <int KIND>
__device__ __forceinline__ void unpack_row_tmem_k(uint32_t p0, uint32_t p1, uint32_t (&v)[32]) {
    uint32_t x0[8], x1[8];
    {
        const uint4 a = lds128(p0), b = lds128(p0 + 16);
        x0[0] = a.x; x0[1] = a.y; x0[2] = a.z; x0[3] = a.w; x0[4] = b.x; x0[5] = b.y; x0[6] = b.z; x0[7] = b.w;
    }
    if (KIND == B_TERNARY) {
        const uint4 a = lds128(p1), b = lds128(p1 + 16);
        x1[0] = a.x; x1[1] = a.y; x1[2] = a.z; x1[3] = a.w; x1[4] = b.x; x1[5] = b.y; x1[6] = b.z; x1[7] = b.w;
#pragma unroll
        for (int g = 0; g < 8; ++g) x0[g] &= x1[g];  // canonical sgn (subset of nz)
    } else {
#pragma unroll
        for (int g = 0; g < 8; ++g) x1[g] = 0;
    }
#pragma unroll
    for (int g = 0; g < 8; ++g)
#pragma unroll
        for (int j = 0; j < 4; ++j) v[4 * g + j] = unpack_word<KIND>(x0[g], x1[g], j);
}
// the codes of one 256-K kernel-A row in registers (stored to TMEM by the caller, one stage later)
__device__ __forceinline__ void unpack_row_regs(int kind, uint32_t p0, uint32_t p1, uint32_t (&v)[32]) {
    if (kind == B_TERNARY) unpack_row_tmem_k<B_TERNARY>(p0, p1, v);
    else if (kind == B_BOOL) unpack_row_tmem_k<B_BOOL>(p0, p1, v);
    else unpack_row_tmem_k<B_BINARY>(p0, p1, v);
}

// UMMA shared-memory descriptor of a K-major operand tile for the stage layout
template <int KS>
__device__ __forceinline__ uint64_t smem_desc_stage(uint32_t saddr) {
    if (KS == 256) return smem_desc_sw128(saddr);
    return smem_desc_sw64(saddr);
}

// KK = 0: operand kinds read from the parameters; KK = 1 + 3 * a_kind + b_kind: fixed at compile
// time (the common BWTA combinations), so the other unpack variants are not compiled in
template <int BN, int CG, int KS, int EO, int KK = 0, bool E1 = false>
__global__ void __launch_bounds__(nt_of(KS, EO, E1), 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmA1,
                   const __grid_constant__ CUtensorMap tmB0, const __grid_constant__ CUtensorMap tmB1,
                   const __grid_constant__ CUtensorMap tmY, const __grid_constant__ PeerMaps pm, TcParams p) {
    using C = Cfg<BN, CG, KS, KK>;
    constexpr int WPS = Stage<KS>::WPS;
    uint8_t* smem =
        reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw + TRACE_BYTES) + 1023) & ~uintptr_t(1023));
    // 1024-byte aligned regions first (SW128 operand tiles, SW128 output
    // staging), then the 128-byte aligned bit-plane stages, then barriers
    uint8_t* sA = smem;
    uint8_t* sB = sA + C::STAGES * C::A_BYTES;
    uint8_t* sOut = sB + C::STAGES * C::B_BYTES;
    float* sScale = reinterpret_cast<float*>(sOut + C::OUT_BYTES);
    uint8_t* sABits = sOut + C::OUT_BYTES + C::SCALE_BYTES;  // [stage][plane][128 rows][16 B]
    uint8_t* sBBits = sABits + C::STAGES * C::ABITS;         // [stage][plane][BNC rows][16 B]
    uint64_t* full = reinterpret_cast<uint64_t*>(sBBits + C::STAGES * C::BBITS);
    uint64_t* bready = full + C::STAGES;
    uint64_t* empty = bready + C::STAGES;
    uint64_t* tfull = empty + C::STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
#ifdef BWTA_TRACE
    for (int i = threadIdx.x; i < TRACE_EV * TRACE_N; i += blockDim.x) reinterpret_cast<unsigned long long*>(smem_raw)[i] = 0;
#endif

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int rank = CG == 2 ? int(cluster_ctarank()) : 0;
    const bool leader = rank == 0;
    const int a_kind_ = KK ? (KK - 1) / 3 : p.a_kind, b_kind_ = KK ? (KK - 1) % 3 : p.b_kind;
    const int a_planes = nplanes_of(a_kind_), b_planes = nplanes_of(b_kind_);

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA0);
        if (a_planes == 2) tma_prefetch_desc(&tmA1);
        tma_prefetch_desc(&tmB0);
        if (b_planes == 2) tma_prefetch_desc(&tmB1);
        if (p.use_tma_store) tma_prefetch_desc(&tmY);
        for (int pi = 0; pi < p.n_peers; ++pi) tma_prefetch_desc(&pm.m[pi]);
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&bready[s], 10 * CG);  // 4 A + 6 B unpack warps of every CTA of the pair
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 4 * epi_warps(KS, EO, E1) * CG);  // epilogue warps of every CTA of the pair
        }
        fence_barrier_init();
    }
    if (warp == 2) {
        if (CG == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
        else tmem_alloc2(tmem_slot, C::TMEM_COLS);
    }
    tc_fence_before();
    __syncthreads();               // CTA-local smem order (TMEM address slot, barrier inits)
    if (CG == 2) cluster_sync();   // the pair: relaxed arrive, tcgen05 fences order TMEM
    tc_fence_after();
    const uint32_t tmem_base_ = *tmem_slot;
    const uint32_t tmem_base = tmem_base_;
    if (warp >= 4 && warp < 8) {
        // UE8M0 scale factors = 1.0 (0x7F) in columns SF_COL .. SF_COL + 15 of every lane
        uint32_t ones[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) ones[i] = 0x7F7F7F7Fu;
        tmem_st_32x32b_x16(tmem_base + (uint32_t((warp & 3) * 32) << 16) + uint32_t(C::SF_COL), ones);
        tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();               // CTA-local smem order (TMEM address slot, barrier inits)
    if (CG == 2) cluster_sync();   // the pair: relaxed arrive, tcgen05 fences order TMEM
    tc_fence_after();
    const int64_t tiles_per_entry = int64_t(p.m_tiles) * p.n_tiles;
    const int64_t total = p.entries * tiles_per_entry;
    const int64_t t0 = blockIdx.x / CG, tstep = gridDim.x / CG;  // persistent over pair-tiles
    // L2 prefetch of the operand planes, each CTA one contiguous 1/gridDim share of every plane's
    // span: with cold operands the ring (STAGES slices in flight per CTA) would otherwise wait a
    // DRAM round trip per few slices; one bulk request per plane and CTA turns that latency chain
    // into a bandwidth-bound burst without adding per-row TMA work (tensor-box prefetches of the
    // 32-byte rows measured much slower: the TMA unit's row rate is a co-limit of the mainloop).
    // Issued before griddepcontrol.wait: a hint only (L2 is the coherence point).
    if (warp == 0 && lane == 0 && p.pf_on) {
#pragma unroll 1
        for (int i = 0; i < 4; ++i) {
            const uint64_t span = p.pf_bytes[i];
            if (!p.pf_ptr[i] || span == 0) continue;
            const uint64_t share = ((span + gridDim.x - 1) / gridDim.x + 15) & ~uint64_t(15);
            const uint64_t off = share * blockIdx.x;
            if (off >= span) continue;
            const uint64_t len = (span - off < share ? ((span - off) & ~uint64_t(15)) : share);
            if (len) bulk_prefetch_l2(static_cast<const uint8_t*>(p.pf_ptr[i]) + off, uint32_t(len));
        }
    }

    // prologue done (smem barriers, TMEM, descriptor prefetch): let the next
    // kernel start its own, then wait for our inputs (predecessor grid)
    pdl_launch_dependents();
    pdl_wait();
    TRACE(0, 0, threadIdx.x == 0);

    if (warp == 0) {
        // ------------------------------ TMA producer ------------------------------
        const uint32_t tx = uint32_t((a_planes * BM + b_planes * C::BNC) * WPS * 4);
        int stage = 0;
        uint32_t phase = 0;
        int it = 0;
        for (int64_t t = t0; t < total; t += tstep) {
            const TileCoord tc = tile_coord(p, t);
            const int mt = tc.mt, nt = tc.nt, eb = tc.eb, eh = tc.eh;
            const int arow = mt * BM * CG + rank * BM;
            const int brow = nt * BN + rank * C::BNC;
            for (int kb = 0; kb < p.num_kb; ++kb) {
#ifdef BWTA_TRACE
                if (!(p.dbg & 1024))
#endif
                kwait(&empty[stage], phase ^ 1, p.dbg);
                TRACE(1, it, lane == 0);
                ++it;
#ifdef BWTA_TRACE
                if (p.dbg & 4) {
                    if (lane == 0) mbar_arrive(&full[stage]);
                    __syncwarp();
                    if (++stage == C::STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                    continue;
                }
#endif
                if (lane == 0) {
                    mbar_arrive_expect_tx(&full[stage], tx);
                    uint8_t* ab = sABits + stage * C::ABITS;
                    tma_load_4d(ab, &tmA0, &full[stage], kb * WPS, arow, eh, eb);
                    if (a_planes == 2) tma_load_4d(ab + BM * WPS * 4, &tmA1, &full[stage], kb * WPS, arow, eh, eb);
                    uint8_t* bb = sBBits + stage * C::BBITS;
                    tma_load_4d(bb, &tmB0, &full[stage], kb * WPS, brow, eh, eb);
                    if (b_planes == 2)
                        tma_load_4d(bb + C::BNC * WPS * 4, &tmB1, &full[stage], kb * WPS, brow, eh, eb);
                }
                __syncwarp();
                if (++stage == C::STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------ MMA issuer (leader CTA) ------------------------------
        if (leader) {
            constexpr uint32_t idesc = idesc_mxf4(BM * CG, BN);
            const uint32_t tmem_base = __shfl_sync(0xffffffffu, tmem_base_, 0);  // warp-uniform
            const uint32_t sfa = tmem_base + uint32_t(C::SF_COL), sfb = tmem_base + uint32_t(C::SF_COL + 8);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            int it = 0;
            int sa = 0;  // a_tmem mode: A code stage
            for (int64_t t = t0; t < total; t += tstep) {
                kwait(&tempty[acc], acc_phase ^ 1, p.dbg);
                tc_fence_after();
                const uint32_t d = tmem_base + uint32_t(acc * BN);
                for (int kb = 0; kb < p.num_kb; ++kb) {
#ifdef BWTA_TRACE
                    TRACE(12, it, lane == 0);
                    if (!(p.dbg & 256))
#endif
                    kwait(&bready[stage], phase, p.dbg);
                    tc_fence_after();
                    TRACE(4, it, lane == 0);
                    ++it;
                    bool skip_mma = false;
#ifdef BWTA_TRACE
                    skip_mma = (p.dbg & 2) != 0;
#endif
                    const uint32_t b0 = smem_u32(sB + stage * C::B_BYTES);
                    if (KS == 256 && p.a_tmem) {
                        // the whole warp issues (elect.sync inside): operands stay in uniform registers
                        const uint32_t a0 = tmem_base + uint32_t(C::A_COL + sa * 32);
                        if (!skip_mma) {
#pragma unroll
                            for (int k = 0; k < Stage<KS>::NMMA; ++k) {
                                const uint64_t bd = smem_desc_stage<KS>(b0 + k * UMMA_KB);
                                if (CG == 1) mma_mxf4_ts_w(d, a0 + 8 * k, bd, idesc, sfa, sfb, (kb | k) != 0);
                                else mma_mxf4_ts_cg2_w(d, a0 + 8 * k, bd, idesc, sfa, sfb, (kb | k) != 0);
                            }
                        }
                        // (the A code stage is released by the same commit as the bit/B stage:
                        // the A unpack warps wait on empty[] of the stage SA back)
                        if (CG == 1) tc_commit_w(&empty[stage]);
                        else tc_commit2_mc_w(&empty[stage], 0x3);
                    } else {
                        if (lane == 0 && !skip_mma) {
                            const uint32_t a0 = smem_u32(sA + stage * C::A_BYTES);
#pragma unroll
                            for (int k = 0; k < Stage<KS>::NMMA; ++k) {
                                const uint64_t ad = smem_desc_stage<KS>(a0 + k * UMMA_KB);
                                const uint64_t bd = smem_desc_stage<KS>(b0 + k * UMMA_KB);
                                if (CG == 1) mma_mxf4(d, ad, bd, idesc, sfa, sfb, (kb | k) != 0);
                                else mma_mxf4_cg2(d, ad, bd, idesc, sfa, sfb, (kb | k) != 0);
                            }
                        }
                        if (lane == 0) {
                            if (CG == 1) tc_commit(&empty[stage]);
                            else tc_commit2_mc(&empty[stage], 0x3);
                        }
                    }
                    TRACE(13, it - 1, lane == 0);
                    __syncwarp();
                    if (++sa == C::SA) sa = 0;
                    if (++stage == C::STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if (CG == 1) tc_commit_w(&tfull[acc]);
                else tc_commit2_mc_w(&tfull[acc], 0x3);
                __syncwarp();
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
        }
    } else if (warp >= (epi_warps(KS, EO, E1) == 1 ? 12 : 16) && KS == 256 && p.a_tmem) {
        // ------------------------------ unpack kernel-A rows into TMEM (warps 16-23) ------------------------------
        // AG groups of 4 warps take alternate stages (group g: it = g mod AG): one group's
        // serial chain per stage (full wait, unpack, A-ring wait, tcgen05.st, wait::st, arrive) was the
        // mainloop's critical path.  Thread ut owns kernel-A row ut = TMEM lane ut (warp
        // w: lane quarter w & 3); A code stage it % SA.
        const int grp = (warp - (epi_warps(KS, EO, E1) == 1 ? 12 : 16)) >> 2;
        const int ut = (warp & 3) * 32 + lane;
        const int kind = a_kind_;
        const int plane_bytes = BM * WPS * 4;
        const uint32_t bready_addr0 = CG == 2 ? mapa_smem(&bready[0], 0) : 0u;
        const uint32_t lane_base = tmem_base + (uint32_t(32 * (warp & 3)) << 16);
        const int64_t n_it = ((total - t0 + tstep - 1) / tstep) * p.num_kb;
        uint32_t v[32];
        constexpr int AG = a_groups(KS, EO);
        for (int64_t it = grp; it < n_it; it += AG) {
            const int stage = int(it % C::STAGES);
            kwait(&full[stage], uint32_t((it / C::STAGES) & 1), p.dbg);
            TRACE(10, it, ut == 0);
            const uint32_t bits = smem_u32(sABits + stage * C::ABITS);
#ifdef BWTA_TRACE
            if (!(p.dbg & 9))
#endif
            unpack_row_regs(kind, bits + ut * 32, bits + plane_bytes + ut * 32, v);
            TRACE(14, it, ut == 0);
            // A code stage sa was last read by the MMAs of stage it - SA, whose commit completes
            // use (it - SA) / STAGES of empty[(it - SA) % STAGES] (one commit per stage frees both
            // rings; SA <= STAGES, and that barrier cannot complete its next phase before the MMAs
            // of stage it, which wait for these codes)
            const int sa = int(it % C::SA);
            if (it >= C::SA
#ifdef BWTA_TRACE
                && !(p.dbg & 512)
#endif
            ) {
                const int64_t pit = it - C::SA;
                kwait(&empty[pit % C::STAGES], uint32_t((pit / C::STAGES) & 1), p.dbg);
            }
            TRACE(15, it, ut == 0);
            tc_fence_after();
            tmem_st_32x32b_x32(lane_base + uint32_t(C::A_COL + sa * 32), v);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (CG == 1) mbar_arrive(&bready[stage]);
                else mbar_arrive_cluster(bready_addr0 + stage * 8);
            }
            TRACE(11, it, ut == 0);
        }
    } else if (warp >= 16 || (warp >= 8 && warp < 12) || warp == 2 || warp == 3) {
        // ------------------------------ unpack into shared memory ------------------------------
        // kernel-B: warps 2, 3, 8-11 (192 threads) over (row, 16-byte word quad) items;
        // kernel-A (128-K stages only): warps 16-19, one row per thread
        const bool is_a = warp >= 16;
        const int ut = is_a ? threadIdx.x - 512 : (warp < 4 ? (warp - 2) * 32 + lane : 64 + (warp - 8) * 32 + lane);
        const int kind = is_a ? a_kind_ : b_kind_;
        const int rows = is_a ? BM : C::BNC;
        const int plane_bytes = rows * WPS * 4;
        const uint32_t bready_addr0 = CG == 2 ? mapa_smem(&bready[0], 0) : 0u;
        int stage = 0;
        uint32_t phase = 0;
        int it = 0;
        for (int64_t t = t0; t < total; t += tstep) {
            for (int kb = 0; kb < p.num_kb; ++kb, ++it) {
                kwait(&full[stage], phase, p.dbg);
                TRACE(is_a ? 10 : 2, it, ut == 0);
                const uint32_t bits = is_a ? smem_u32(sABits + stage * C::ABITS) : smem_u32(sBBits + stage * C::BBITS);
                const uint32_t dst = is_a ? smem_u32(sA + stage * C::A_BYTES) : smem_u32(sB + stage * C::B_BYTES);
#ifdef BWTA_TRACE
                if (!(p.dbg & (is_a ? 9 : 17)))
#endif
                {
                    if (is_a) unpack_rows<KS>(kind, bits, plane_bytes, dst, ut, rows, 128);
                    else unpack_quads<KS, C::BNC, 192>(kind, bits, dst, ut);
                }
#ifdef BWTA_TRACE
                if (!(p.dbg & 128))
#endif
                fence_proxy_async_smem();
                __syncwarp();
                TRACE(is_a ? 11 : 3, it, ut == 0);
                if (lane == 0) {
                    if (CG == 1) mbar_arrive(&bready[stage]);
                    else mbar_arrive_cluster(bready_addr0 + stage * 8);
                }
                if (++stage == C::STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp >= 4) {
        // ------------------------------ epilogue (warps 4-7 and 12-15) ------------------------------
        const int q = warp & 3, h = warp >= 12 ? 1 : 0;
        if (EO != 1 || p.y_dt == DT_F16 || p.y_dt == DT_BF16)
            epilogue<BN, 2, CG, EO, epi_warps(KS, EO, E1)>(p, tmY, pm, tmem_base, sOut, sScale, tfull, tempty, q, h, lane, tiles_per_entry, total,
                                rank, t0, tstep);
        else
            if constexpr (EO == 1) epilogue<BN, 4, CG, EO>(p, tmY, pm, tmem_base, sOut, sScale, tfull, tempty, q, h, lane, tiles_per_entry, total,
                                rank, t0, tstep);
    }
    TRACE(7, 0, warp == 4 && lane == 0);
    tc_fence_before();
    __syncthreads();               // CTA-local smem order (TMEM address slot, barrier inits)
    if (CG == 2) cluster_sync();   // the pair: relaxed arrive, tcgen05 fences order TMEM
    TRACE(8, 0, threadIdx.x == 0);
#ifdef BWTA_TRACE
    __syncthreads();
    if (blockIdx.x < 2)
        for (int i = threadIdx.x; i < TRACE_EV * TRACE_N; i += blockDim.x)
            (&g_trace[blockIdx.x][0][0])[i] = reinterpret_cast<unsigned long long*>(smem_raw)[i];
#endif
    if (warp == 2) {
        tc_fence_after();
        if (CG == 1) tmem_dealloc(tmem_base, C::TMEM_COLS);
        else tmem_dealloc2(tmem_base, C::TMEM_COLS);
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
}  // namespace

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static std::once_flag g_encode_once;

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    std::call_once(g_encode_once, [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
        else
            cudaGetLastError();
    });
    return g_encode;
}

bool encode(CUtensorMap* m, CUtensorMapDataType dt, int rank, void* base, const uint64_t* dims,
            const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapSwizzle sw) {
    auto enc = encode_fn();
    if (!enc) return false;
    cuuint64_t d[5];
    cuuint64_t s[4];
    cuuint32_t b[5], es[5];
    for (int i = 0; i < rank; ++i) {
        d[i] = dims[i];
        b[i] = box[i];
        es[i] = 1;
        if (i + 1 < rank) s[i] = strides_bytes[i];
    }
    return enc(m, dt, rank, base, d, s, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int num_sms() { return device_sms(); }

int64_t kw4_of(int64_t K) { return ((K + 31) / 32 + 3) / 4 * 4; }

// A stride for a batch dimension of extent `count`: TMA needs a multiple of 16
// bytes even when the dimension is degenerate.
uint64_t bstride(int64_t count, int64_t stride_bytes, uint64_t fallback) {
    return (count <= 1 || stride_bytes <= 0) ? fallback : uint64_t(stride_bytes);
}

namespace {

struct Plan {
    bool swap;
    const uint32_t *a_sgn, *a_nz, *b_sgn, *b_nz;  // kernel operands
    int64_t Mk, Nk, lda, ldb, a_bs, a_hs, b_bs, b_hs;
    int bkind;
};

Plan make_plan(const MatmulArgs& a, bool swap) {
    Plan p{};
    p.swap = swap;
    if (!p.swap) {
        p.a_sgn = a.a_sgn; p.a_nz = a.a_nz; p.b_sgn = a.b_sgn; p.b_nz = a.b_nz;
        p.Mk = a.M; p.Nk = a.N; p.lda = a.lda; p.ldb = a.ldb;
        p.a_bs = a.a_bs; p.a_hs = a.a_hs; p.b_bs = a.b_bs; p.b_hs = a.b_hs;
    } else {
        p.a_sgn = a.b_sgn; p.a_nz = a.b_nz; p.b_sgn = a.a_sgn; p.b_nz = a.a_nz;
        p.Mk = a.N; p.Nk = a.M; p.lda = a.ldb; p.ldb = a.lda;
        p.a_bs = a.b_bs; p.a_hs = a.b_hs; p.b_bs = a.a_bs; p.b_hs = a.a_hs;
    }
    p.bkind = (p.b_sgn && p.b_nz) ? B_TERNARY : (p.b_nz ? B_BOOL : B_BINARY);
    return p;
}

// Tile shape: minimise (rounds of the persistent grid) x (per-tile cost).
// The mainloop is bound by shared-memory traffic (unpacked codes written
// and read back by the MMA), which per CTA and stage is proportional to the
// rows it unpacks: 128 A rows + BN / cg B rows; plus a fixed per-tile
// overhead (~64 rows' worth: fill, epilogue drain).
struct TileChoice {
    int bn, cg;
    double cost;
};
TileChoice choose_tile(int64_t Mk, int64_t Nk, int64_t entries) {
    TileChoice best{64, 1, 1e300};
    const int bns[3] = {192, 128, 64};
    for (int cg = 2; cg >= 1; --cg) {
        if (cg == 2 && Mk <= BM) continue;
        for (int bn : bns) {
            if (bn > 64 && Nk <= bn - 64) continue;  // a narrower tile covers N just as well
            const int64_t tiles = entries * ((Mk + BM * cg - 1) / (BM * cg)) * ((Nk + bn - 1) / bn);
            const int64_t slots = num_sms() / cg;
            const int64_t rounds = (tiles + slots - 1) / slots;
            const double cost = double(rounds) * (BM + bn / cg + 64);
            if (cost < best.cost - 1e-9) best = TileChoice{bn, cg, cost};
        }
    }
    return best;
}

template <int BN, int CG, int KS, int EO, int KK = 0, bool E1 = false>
cudaError_t launch_ks(const CUtensorMap& ma0, const CUtensorMap& ma1, const CUtensorMap& mb0, const CUtensorMap& mb1,
                      const CUtensorMap& my, const PeerMaps& pm, const TcParams& p, cudaStream_t s) {
    using C = Cfg<BN, CG, KS, KK>;
    auto kern = tc_gemm_kernel<BN, CG, KS, EO, KK, E1>;
    static std::atomic<uint64_t> optin{0};  // per device
    if (cudaError_t e = ensure_smem_optin(kern, C::SMEM, optin); e != cudaSuccess) return e;
    const int64_t tiles = p.entries * int64_t(p.m_tiles) * p.n_tiles;
    const int64_t slots = num_sms() / CG;
    const int grid = int((tiles < slots ? tiles : slots) * CG);
    return launch_pdl(kern, dim3(grid), dim3(nt_of(KS, EO, E1)), size_t(C::SMEM), s, CG, ma0, ma1, mb0, mb1, my, pm, p);
}

template <int BN, int CG>
cudaError_t launch_cfg(int ks, const CUtensorMap& ma0, const CUtensorMap& ma1, const CUtensorMap& mb0,
                       const CUtensorMap& mb1, const CUtensorMap& my, const PeerMaps& pm, const TcParams& p,
                       cudaStream_t s) {
    const bool fast = !p.pack_out && p.use_tma_store && (p.y_dt == DT_F16 || p.y_dt == DT_BF16) && p.dot_bias == 0.f;
    if (p.n_peers > 0 && !fast) return cudaErrorNotSupported;  // only the fast epilogue stores to peers
    // the heavy GEMM tiles (BN = 192, 256-K stages) get kinds fixed at compile time for the BWTA
    // linear's combinations: activations (ternary / bool) x binary weights, and the swapped pack
    const int kk = 1 + 3 * p.a_kind + p.b_kind;
    const bool spec = ks == 256 &&
                      (kk == 1 + 3 * B_TERNARY + B_BINARY || kk == 1 + 3 * B_BOOL + B_BINARY ||
                       kk == 1 + 3 * B_BINARY + B_TERNARY);
    if (fast) {
        if constexpr (BN == 192) if (spec) {
            // K >= 2048 and at least two rounds of tiles per CTA pair (a tile's epilogue then overlaps
            // the next tile's mainloop): one epilogue warp per lane quarter (E1).  A single round
            // (BERT FFN2: 64 tiles) leaves the epilogue exposed and keeps two (11.2 vs 11.8 us).
            const int64_t tiles_ = p.entries * int64_t(p.m_tiles) * p.n_tiles;
            if (p.num_kb >= 8 && tiles_ >= 2 * int64_t(num_sms() / CG)) {
                if (kk == 1 + 3 * B_TERNARY + B_BINARY) return launch_ks<BN, CG, 256, 0, 1 + 3 * B_TERNARY + B_BINARY, true>(ma0, ma1, mb0, mb1, my, pm, p, s);
                if (kk == 1 + 3 * B_BOOL + B_BINARY) return launch_ks<BN, CG, 256, 0, 1 + 3 * B_BOOL + B_BINARY, true>(ma0, ma1, mb0, mb1, my, pm, p, s);
                return launch_ks<BN, CG, 256, 0, 1 + 3 * B_BINARY + B_TERNARY, true>(ma0, ma1, mb0, mb1, my, pm, p, s);
            }
            if (kk == 1 + 3 * B_TERNARY + B_BINARY) return launch_ks<BN, CG, 256, 0, 1 + 3 * B_TERNARY + B_BINARY>(ma0, ma1, mb0, mb1, my, pm, p, s);
            if (kk == 1 + 3 * B_BOOL + B_BINARY) return launch_ks<BN, CG, 256, 0, 1 + 3 * B_BOOL + B_BINARY>(ma0, ma1, mb0, mb1, my, pm, p, s);
            return launch_ks<BN, CG, 256, 0, 1 + 3 * B_BINARY + B_TERNARY>(ma0, ma1, mb0, mb1, my, pm, p, s);
        }
        return ks == 128 ? launch_ks<BN, CG, 128, 0>(ma0, ma1, mb0, mb1, my, pm, p, s)
                         : launch_ks<BN, CG, 256, 0>(ma0, ma1, mb0, mb1, my, pm, p, s);
    }
    if (p.pack_out) {
        if constexpr (BN == 192) if (spec) {
            if (kk == 1 + 3 * B_TERNARY + B_BINARY) return launch_ks<BN, CG, 256, 2, 1 + 3 * B_TERNARY + B_BINARY>(ma0, ma1, mb0, mb1, my, pm, p, s);
            if (kk == 1 + 3 * B_BOOL + B_BINARY) return launch_ks<BN, CG, 256, 2, 1 + 3 * B_BOOL + B_BINARY>(ma0, ma1, mb0, mb1, my, pm, p, s);
            return launch_ks<BN, CG, 256, 2, 1 + 3 * B_BINARY + B_TERNARY>(ma0, ma1, mb0, mb1, my, pm, p, s);
        }
        return ks == 128 ? launch_ks<BN, CG, 128, 2>(ma0, ma1, mb0, mb1, my, pm, p, s)
                         : launch_ks<BN, CG, 256, 2>(ma0, ma1, mb0, mb1, my, pm, p, s);
    }
    return ks == 128 ? launch_ks<BN, CG, 128, 1>(ma0, ma1, mb0, mb1, my, pm, p, s)
                     : launch_ks<BN, CG, 256, 1>(ma0, ma1, mb0, mb1, my, pm, p, s);
}

}  // namespace

#ifdef BWTA_TRACE
// copy the timeline to the host and reset it (tools/trace_gemm.py)
extern "C" __attribute__((visibility("default"))) int bwta_trace_fetch(unsigned long long* buf) {
    if (cudaMemcpyFromSymbol(buf, g_trace, sizeof(g_trace)) != cudaSuccess) return 1;
    static unsigned long long zero[2][TRACE_EV][TRACE_N] = {};
    return cudaMemcpyToSymbol(g_trace, zero, sizeof(zero)) != cudaSuccess;
}
#endif

size_t matmul_tc_workspace(const MatmulArgs&) { return 0; }  // both operands are unpacked in-kernel

bool matmul_tc_supported(const MatmulArgs& a) {
    if (a.K < 1 || a.M < 1 || a.N < 1) return false;
    if (a.nb > (int64_t(1) << 31) || a.nh > (int64_t(1) << 31)) return false;
    if (a.M > (int64_t(1) << 31) || a.N > (int64_t(1) << 31)) return false;
    if (a.K > (int64_t(1) << 24)) return false;  // |dot| <= K must be exact in the f32 accumulator
    // both operands' bit planes are read by TMA: batch strides must be real strides
    if ((a.nb > 1 && (a.a_bs <= 0 || a.b_bs <= 0)) || (a.nh > 1 && (a.a_hs <= 0 || a.b_hs <= 0))) return false;
    return encode_fn() != nullptr;
}

// 4-D tensor map over a packed operand: dims {ld words, rows, heads, batch},
// box {wps words, box_rows, 1, 1} (one 32*wps-element K slice of box_rows rows)
bool encode_planes(CUtensorMap* m, const uint32_t* base, int64_t ld, int64_t rows, int64_t hs, int64_t bs,
                   int64_t nh, int64_t nb, int box_rows, int wps, CUtensorMapSwizzle sw) {
    const uint64_t row_b = uint64_t(ld) * 4;
    const uint64_t dims[4] = {uint64_t(ld), uint64_t(rows), uint64_t(nh), uint64_t(nb)};
    const uint64_t hsb = bstride(nh, hs * 4, row_b * rows);
    const uint64_t str[3] = {row_b, hsb, bstride(nb, bs * 4, hsb * nh)};
    const uint32_t box[4] = {uint32_t(wps), uint32_t(box_rows), 1, 1};
    return encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, const_cast<uint32_t*>(base), dims, str, box,
                  sw);
}
int kind_of(const uint32_t* sgn, const uint32_t* nz) { return (sgn && nz) ? B_TERNARY : (nz ? B_BOOL : B_BINARY); }

bool matmul_tc_peers_ok(const MatmulArgs& a) {
    // the 16-bit TMA-store epilogue of the tile kernel (launch_cfg's `fast` class) is the one that
    // stores to peers; W1A1 (dot_bias) and the fused packs take other epilogues
    const int es = 2;
    return a.n_peers >= 0 && a.n_peers <= MAX_PEERS && !matmul_gemv_eligible(a) && matmul_tc_supported(a) &&
           !a.pack_out && !a.po_heads && (a.y_dt == DT_F16 || a.y_dt == DT_BF16) && (a.a_nz || a.b_nz) &&
           reinterpret_cast<uintptr_t>(a.y) % 16 == 0 && (uint64_t(a.ldy) * es) % 16 == 0 &&
           (a.nb == 1 || (uint64_t(a.y_bs) * es) % 16 == 0) && (a.nh == 1 || (uint64_t(a.y_hs) * es) % 16 == 0);
}

cudaError_t launch_matmul_tc(const MatmulArgs& a, void*, size_t, cudaStream_t s) {
    if (a.n_peers > 0 && !matmul_tc_peers_ok(a)) return cudaErrorNotSupported;
    if (matmul_gemv_eligible(a)) return launch_matmul_gemv(a, s);
    const int64_t entries = a.nb * a.nh;
    const int64_t kw4 = kw4_of(a.K);
    // operand roles and tile shape: the caller's A on the MMA M side (kernel-A)
    // or swapped (W on the M side, the epilogue stores D^T), whichever tiles
    // the persistent grid better -- e.g. a skinny M = 16 goes on the N side
    const TileChoice t_ns = choose_tile(a.M, a.N, entries), t_sw = choose_tile(a.N, a.M, entries);
    // on a tie: plain outputs keep the caller's orientation (the non-transposed stmatrix/TMA epilogue
    // measured 5-11 % faster on the BERT GEMMs, tools/ab_swap.py); the fused pack swaps when M > N
    // (its ballot path with integer thresholds is 1.4x faster than the register-word path)
    const bool tie = !(t_ns.cost < t_sw.cost - 1e-9) && !(t_sw.cost < t_ns.cost - 1e-9);
    const bool swap = !a.po_heads && (t_sw.cost < t_ns.cost - 1e-9 || (tie && a.pack_out && a.M > a.N));
    const Plan pl = make_plan(a, swap);
    TileChoice tc = swap ? t_sw : t_ns;
    if (a.tile_n) tc.bn = a.tile_n;
    if (a.cta_group) tc.cg = a.cta_group;
    if (tc.cg == 2 && pl.Mk <= BM) tc.cg = 1;  // a pair needs two 128-row halves of kernel-A
    const int bn = tc.bn, cg = tc.cg;

    // stage depth along K: 128 when the whole reduction fits (attention, head_dim <= 128)
    const int ks = kw4 <= 4 ? 128 : 256;
    const int wps = ks / 32;
    // bit-plane tensor maps: plane 0 = sgn (binary/ternary) or nz (bool), plane 1 = nz (ternary)
    const int akind = kind_of(pl.a_sgn, pl.a_nz), bkind = kind_of(pl.b_sgn, pl.b_nz);
    CUtensorMap ma0, ma1, mb0, mb1, my;
    PeerMaps pm;
    {
        const uint32_t* a0 = akind == B_BOOL ? pl.a_nz : pl.a_sgn;
        const uint32_t* a1 = akind == B_TERNARY ? pl.a_nz : a0;
        const uint32_t* b0 = bkind == B_BOOL ? pl.b_nz : pl.b_sgn;
        const uint32_t* b1 = bkind == B_TERNARY ? pl.b_nz : b0;
        if (!encode_planes(&ma0, a0, pl.lda, pl.Mk, pl.a_hs, pl.a_bs, a.nh, a.nb, BM, wps) ||
            !encode_planes(&ma1, a1, pl.lda, pl.Mk, pl.a_hs, pl.a_bs, a.nh, a.nb, BM, wps) ||
            !encode_planes(&mb0, b0, pl.ldb, pl.Nk, pl.b_hs, pl.b_bs, a.nh, a.nb, bn / cg, wps) ||
            !encode_planes(&mb1, b1, pl.ldb, pl.Nk, pl.b_hs, pl.b_bs, a.nh, a.nb, bn / cg, wps))
            return cudaErrorInvalidValue;
    }
    TcParams p{};
    p.M = pl.Mk;
    p.N = pl.Nk;
    p.num_kb = int((kw4 + wps - 1) / wps);
    // W1A1 (both operands binary): the num_kb * ks K positions the kernel multiplies include the
    // zero-bit padding, each contributing (+1)(+1) -- subtract them in the epilogue
    if (!pl.a_nz && !pl.b_nz) p.dot_bias = float(a.K - int64_t(p.num_kb) * ks);
    p.entries = entries;
    p.nh = a.nh;
    p.m_tiles = int((pl.Mk + BM * cg - 1) / (BM * cg));
    p.n_tiles = int((pl.Nk + bn - 1) / bn);
    if (entries * int64_t(p.m_tiles) * p.n_tiles >= (int64_t(1) << 31)) return cudaErrorNotSupported;
    p.fd_tpe = make_fastdiv(uint32_t(int64_t(p.m_tiles) * p.n_tiles));
    p.fd_mt = make_fastdiv(uint32_t(p.m_tiles));
    p.fd_nh = make_fastdiv(uint32_t(a.nh));
    p.a_kind = akind;
    p.b_kind = bkind;
    p.y = a.y;
    p.y_dt = a.y_dt;
    p.ldy = a.ldy;
    p.y_bs = a.y_bs;
    p.y_hs = a.y_hs;
    p.out_trans = (pl.swap ? 1 : 0) ^ (a.y_trans ? 1 : 0);
    p.scale = a.col_scale;
    p.scale_on_rows = pl.swap ? 1 : 0;
    p.scalar = a.scalar;
    p.pack_out = a.pack_out;
    p.po_kind = a.po_kind;
    p.po_sgn = a.po_sgn;
    p.po_nz = a.po_nz;
    p.po_ld = a.po_ld;
    p.po_bs = a.po_bs;
    p.po_hs = a.po_hs;
    p.po_tp = a.po_tp;
    p.po_tn = a.po_tn;
    p.po_heads = a.po_heads;
    p.ph_T = a.ph_T;
    p.ph_H = a.ph_H;
    p.ph_D = a.ph_D;
    if (a.po_heads) {
        if (a.ph_H * a.ph_D >= (int64_t(1) << 31) || a.ph_T >= (int64_t(1) << 31) || pl.Mk >= (int64_t(1) << 31))
            return cudaErrorNotSupported;
        p.fd_hd = make_fastdiv(uint32_t(a.ph_H * a.ph_D));
        p.fd_d = make_fastdiv(uint32_t(a.ph_D));
        p.fd_t = make_fastdiv(uint32_t(a.ph_T));
    }
    for (int r = 0; r < 3; ++r) {
        p.ph_sgn[r] = a.ph_sgn[r];
        p.ph_nz[r] = a.ph_nz[r];
        p.ph_ld[r] = a.ph_ld[r];
        p.ph_tp[r] = a.ph_tp[r];
        p.ph_tn[r] = a.ph_tn[r];
    }
    // output tensor map (TMA store) when the layout allows it
    {
        const int es = (a.y_dt == DT_F16 || a.y_dt == DT_BF16) ? 2 : 4;
        const uint64_t ldb_ = uint64_t(a.ldy) * es;
        const int64_t inner = p.out_trans ? pl.Mk : pl.Nk, outer = p.out_trans ? pl.Nk : pl.Mk;
        const uint64_t hsb = bstride(a.nh, a.y_hs * es, ldb_ * outer);
        const uint64_t bsb = bstride(a.nb, a.y_bs * es, hsb * a.nh);
        bool ok = !a.pack_out && (reinterpret_cast<uintptr_t>(a.y) % 16 == 0) && ldb_ % 16 == 0 && hsb % 16 == 0 &&
                  bsb % 16 == 0 &&
                  ldb_ < (uint64_t(1) << 40) && hsb < (uint64_t(1) << 40) && bsb < (uint64_t(1) << 40);
        if (ok) {
            const uint64_t dims[4] = {uint64_t(inner), uint64_t(outer), uint64_t(a.nh), uint64_t(a.nb)};
            const uint64_t str[3] = {ldb_, hsb, bsb};
            const int cw = 128 / es;
            const uint32_t box_nt[4] = {uint32_t(cw), 32, 1, 1};
            const uint32_t box_t[4] = {32, uint32_t(cw), 1, 1};
            const CUtensorMapDataType dt = es == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16 : CU_TENSOR_MAP_DATA_TYPE_UINT32;
            ok = p.out_trans ? encode(&my, dt, 4, a.y, dims, str, box_t, CU_TENSOR_MAP_SWIZZLE_NONE)
                             : encode(&my, dt, 4, a.y, dims, str, box_nt, CU_TENSOR_MAP_SWIZZLE_128B);
        }
        p.use_tma_store = ok ? 1 : 0;
    // kernel-A codes go to TMEM (no shared-memory round trip for the 128-row operand) for 256-K
    // stages; measured 2-7 % faster than the shared-memory A path (tools/ab_atmem.py)
    p.a_tmem = ks == 256 ? 1 : 0;
    // L2 prefetch spans of the four plane maps (A0, A1, B0, B1): from the base to the end of the
    // last entry's last row; skipped when the span is more than twice the bytes the GEMM reads
    // (strided views into a larger tensor) -- BWTA_L2_PREFETCH=0 turns it off (tools/cold_warm.py)
    {
        static const int pf_env = [] {
            const char* e = getenv("BWTA_L2_PREFETCH");
            return e ? atoi(e) : 0;  // off by default: measured neutral on C3 (profiles/r02g_l2_prefetch_ab.txt)
        }();
        p.pf_on = pf_env;
        const uint32_t* bases[4] = {akind == B_BOOL ? pl.a_nz : pl.a_sgn, akind == B_TERNARY ? pl.a_nz : nullptr,
                                    bkind == B_BOOL ? pl.b_nz : pl.b_sgn, bkind == B_TERNARY ? pl.b_nz : nullptr};
        const int64_t lds[4] = {pl.lda, pl.lda, pl.ldb, pl.ldb}, rows[4] = {pl.Mk, pl.Mk, pl.Nk, pl.Nk};
        const int64_t bss[4] = {pl.a_bs, pl.a_bs, pl.b_bs, pl.b_bs}, hss[4] = {pl.a_hs, pl.a_hs, pl.b_hs, pl.b_hs};
        for (int i = 0; i < 4; ++i) {
            p.pf_ptr[i] = nullptr;
            p.pf_bytes[i] = 0;
            if (!bases[i] || reinterpret_cast<uintptr_t>(bases[i]) % 16 != 0) continue;
            const int64_t last = (a.nb - 1) * (a.nb > 1 ? bss[i] : 0) + (a.nh - 1) * (a.nh > 1 ? hss[i] : 0);
            const int64_t span_w = last + rows[i] * lds[i];
            const int64_t dense_w = a.nb * a.nh * rows[i] * lds[i];
            if (last < 0 || span_w > 2 * dense_w) continue;
            p.pf_ptr[i] = bases[i];
            p.pf_bytes[i] = uint64_t(span_w) * 4;
        }
    }
#ifdef BWTA_TRACE
    if (const char* dbg = getenv("BWTA_DBG")) p.dbg = atoi(dbg);
#endif
        if (!ok) my = ma0;  // unused
        if (a.n_peers > 0 && !ok) return cudaErrorNotSupported;
        // peers: the same map at each peer buffer's base (the all-gather destinations)
        p.n_peers = a.n_peers;
        for (int pi = 0; pi < a.n_peers; ++pi) {
            if (reinterpret_cast<uintptr_t>(a.y_peers[pi]) % 16 != 0) return cudaErrorInvalidValue;
            const uint64_t dims[4] = {uint64_t(inner), uint64_t(outer), uint64_t(a.nh), uint64_t(a.nb)};
            const uint64_t str[3] = {ldb_, hsb, bsb};
            const uint32_t box_nt[4] = {64, 32, 1, 1};
            const uint32_t box_t[4] = {32, 64, 1, 1};
            if (!(p.out_trans ? encode(&pm.m[pi], CU_TENSOR_MAP_DATA_TYPE_UINT16, 4, a.y_peers[pi], dims, str, box_t,
                                       CU_TENSOR_MAP_SWIZZLE_NONE)
                              : encode(&pm.m[pi], CU_TENSOR_MAP_DATA_TYPE_UINT16, 4, a.y_peers[pi], dims, str, box_nt,
                                       CU_TENSOR_MAP_SWIZZLE_128B)))
                return cudaErrorInvalidValue;
        }
    }
    if (cg == 2) {
        if (bn == 192) return launch_cfg<192, 2>(ks, ma0, ma1, mb0, mb1, my, pm, p, s);
        if (bn == 128) return launch_cfg<128, 2>(ks, ma0, ma1, mb0, mb1, my, pm, p, s);
        return launch_cfg<64, 2>(ks, ma0, ma1, mb0, mb1, my, pm, p, s);
    }
    if (bn == 192) return launch_cfg<192, 1>(ks, ma0, ma1, mb0, mb1, my, pm, p, s);
    if (bn == 128) return launch_cfg<128, 1>(ks, ma0, ma1, mb0, mb1, my, pm, p, s);
    return launch_cfg<64, 1>(ks, ma0, ma1, mb0, mb1, my, pm, p, s);
}

}  // namespace bwta
