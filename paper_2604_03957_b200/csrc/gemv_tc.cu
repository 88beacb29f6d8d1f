// gemv_tc.cu -- design (b) for skinny products: one operand has at most 32
// rows (decode: M = 1..32 tokens against a weight matrix).
//
// Same arithmetic as gemm_tc.cu (P:324-331 cases; R12: codes {-1, 0, +1} as
// E2M1 nibbles, every UE8M0 block scale 1.0, the f32 accumulator holds the
// integer dot exactly; R5 epilogue), different schedule.  With <= 32 rows on
// the MMA N side there is almost no tensor work per byte: the kernel must
// stream the large operand's bit planes at HBM rate and unpack them fast
// enough.  The general kernel is bound there by (i) its bit ring sharing the
// code stages (6 stages in flight -> Little's-law bound far below HBM rate)
// and (ii) shared-memory traffic of the unpacked codes (written, then read by
// the MMA: 1 B per element).  Here:
//   * the bit planes of the large operand (kernel-A, 128 rows per tile) flow
//     through a deep TMA ring (1024-K slices: one full 128-byte line per row
//     and plane, 128B-swizzled; ~160 KB in flight per SM) that is released by
//     the unpackers, not by the MMA.  (Measured: 32-byte-per-row boxes -- the
//     general kernel's 256-K slices -- cap a pure load loop at ~1.4 TB/s);
//   * kernel-A codes are written to TENSOR MEMORY with tcgen05.st and the MMA
//     reads A from TMEM (tcgen05.mma ... [a_tmem]) -- no shared-memory round
//     trip for the 128-row operand; only the <= 32-row operand is staged as
//     SW128 K-major codes in shared memory.
//
// CTA (persistent, one per SM, 16 warps):
//   warp 0      TMA producer (bit ring)
//   warp 1      MMA issuer: 4 x tcgen05.mma (128 x NB x 64) per 256-K unit
//   warp 2      TMEM allocator
//   warps 4-11  unpack, two groups of 4 warps taking alternate units: warp w
//               owns TMEM lane quarter w & 3, each thread one kernel-A row
//               (8 words -> 32 code words -> tcgen05.st), plus words of the
//               small operand
//   warps 12-15 epilogue: tcgen05.ld of the NB accumulator columns of the
//               warp's 32 rows -> scale (R5) -> direct global stores
// TMEM columns: [0, 2 NB) double-buffered accumulators, [64, 448) twelve A
// code stages of 32 columns, [448, 464) UE8M0 scale factors (all 1.0).
// The per-unit chain (unpack -> tcgen05.st -> MMA -> commit) is long, so the
// code ring is as deep as TMEM allows and the two unpack groups take
// alternate units.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include "bwta_internal.h"
#include "sm100.cuh"
#include "tc_codes.cuh"

namespace bwta {
namespace {

using namespace sm100;
using namespace tc;

constexpr int GV_BM = 128;      // kernel-A rows per tile (MMA M)
constexpr int GV_WPS = 8;       // packed words per row per plane per unit (256 K)
constexpr int GV_UPS = 4;       // units per bit stage: TMA boxes of 32 words = one 128-byte line per row
constexpr int GV_ROWB = 128;    // E2M1 code bytes per row per unit
// CTAs per SM: 1, or 2 when the problem has more tiles than SMs (each CTA then gets half the TMEM,
// shared memory and code stages; the per-unit chain is latency-bound, so two CTAs overlap two
// chains: M = 16 x K 8192 x N 28672 27.0 -> 22.1 us; with <= 1 tile per SM the halved rings are slower)
__host__ __device__ constexpr int gv_cst(int cps) { return cps == 2 ? 5 : 12; }  // code stages (A in TMEM, B in smem)
constexpr int GV_MAXRING = 40;  // bit-ring stages
constexpr int GV_NT = 512;      // 16 warps
constexpr int GV_ACOL = 64;     // first TMEM column of the A code stages
__host__ __device__ constexpr int gv_sfcol(int cps) { return GV_ACOL + gv_cst(cps) * 32; }
__host__ __device__ constexpr int gv_tmem_cols(int cps) { return cps == 2 ? 256 : 512; }
__host__ __device__ constexpr int gv_smem_max(int cps) { return cps == 2 ? 110 * 1024 : 200 * 1024; }

__device__ __forceinline__ uint32_t gv_fdiv(uint32_t n, const FastDiv& f) { return (__umulhi(n, f.mul) + n) >> f.shift; }
struct GvParams {
    float dot_bias;  // W1A1 (both operands binary): K - K_processed, added to every dot
    int64_t M, N;  // kernel-A rows / kernel-B rows (N <= NB) per entry
    int num_kb;
    int64_t nh, entries;
    int tiles_per_entry;
    FastDiv fd_tpe, fd_nh, fd_nsup;  // 32-bit multiply-shift decode of the tile index (host: total < 2^31)
    int a_kind, b_kind;
    int ring;                        // bit-ring depth
    int a_bits, b_bits;              // bytes per bit stage (all planes, 128 B per row per plane)
    void* y;
    int y_dt;
    int64_t y_rs, y_cs, y_bs, y_hs;  // element strides: kernel row, kernel col, batch, head
    const float* scale;              // caller's per-N scale (kernel rows if scale_on_rows), may be null
    int scale_on_rows;
    float scalar;
};

template <int NB>
struct GvCfg {
    static constexpr int B_BYTES = NB * GV_ROWB;  // one code stage of the small operand
    static_assert(B_BYTES % 1024 == 0, "SW128 atoms are 8 rows x 128 B");
};

// one packed word (32 elements, both planes) -> the 16-byte code chunk
template <int KIND>
__device__ __forceinline__ void unpack_chunk(uint32_t x0, uint32_t x1, uint32_t (&o)[4]) {
    if (KIND == B_TERNARY) x0 &= x1;  // canonical sgn (subset of nz)
#pragma unroll
    for (int j = 0; j < 4; ++j) o[j] = unpack_word<KIND>(x0, x1, j);
}

// the 8 words of one kernel-A row -> 32 TMEM columns (code word 4g + j)
// (q0, q1: the row's two 16-byte bit chunks of this unit; plane 1 at +poff)
template <int KIND>
__device__ __forceinline__ void unpack_a_row(uint32_t q0, uint32_t q1, uint32_t poff, uint32_t taddr) {
    uint32_t x0[8], x1[8];
    {
        const uint4 a = lds128(q0), b = lds128(q1);
        x0[0] = a.x; x0[1] = a.y; x0[2] = a.z; x0[3] = a.w; x0[4] = b.x; x0[5] = b.y; x0[6] = b.z; x0[7] = b.w;
    }
    if (KIND == B_TERNARY) {
        const uint4 a = lds128(q0 + poff), b = lds128(q1 + poff);
        x1[0] = a.x; x1[1] = a.y; x1[2] = a.z; x1[3] = a.w; x1[4] = b.x; x1[5] = b.y; x1[6] = b.z; x1[7] = b.w;
    } else {
#pragma unroll
        for (int g = 0; g < 8; ++g) x1[g] = 0;
    }
    uint32_t v[32];
#pragma unroll
    for (int g = 0; g < 8; ++g) {
        uint32_t o[4];
        unpack_chunk<KIND>(x0[g], x1[g], o);
#pragma unroll
        for (int j = 0; j < 4; ++j) v[4 * g + j] = o[j];
    }
    tmem_st_32x32b_x32(taddr, v);
}

__device__ __forceinline__ void store_out(const GvParams& p, int64_t off, float f, uint32_t acc) {
    if (p.y_dt == DT_F16) reinterpret_cast<__half*>(p.y)[off] = __float2half_rn(f);
    else if (p.y_dt == DT_BF16) reinterpret_cast<__nv_bfloat16*>(p.y)[off] = __float2bfloat16_rn(f);
    else if (p.y_dt == DT_F32) reinterpret_cast<float*>(p.y)[off] = f;
    else reinterpret_cast<int32_t*>(p.y)[off] = __float2int_rn(__uint_as_float(acc));
}

template <int NB, int CPS>
__global__ void __launch_bounds__(GV_NT, CPS)
    tc_gemv_kernel(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmA1,
                   const __grid_constant__ CUtensorMap tmB0, const __grid_constant__ CUtensorMap tmB1, GvParams p) {
    using C = GvCfg<NB>;
    constexpr int GV_CST_ = gv_cst(CPS), GV_SFCOL_ = gv_sfcol(CPS), GV_TMEM_COLS_ = gv_tmem_cols(CPS);
    extern __shared__ __align__(1024) uint8_t gv_smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(gv_smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sB = smem;                                   // [GV_CST_][NB rows][128 B] SW128 codes
    uint8_t* sBits = sB + GV_CST_ * C::B_BYTES;            // [ring][A planes | B planes]
    const int stage_bytes = p.a_bits + p.b_bits;
    uint64_t* bfull = reinterpret_cast<uint64_t*>(sBits + p.ring * stage_bytes);
    uint64_t* bempty = bfull + GV_MAXRING;
    uint64_t* cfull = bempty + GV_MAXRING;
    uint64_t* cempty = cfull + GV_CST_;
    uint64_t* afull = cempty + GV_CST_;
    uint64_t* aempty = afull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aempty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int a_planes = p.a_kind == B_TERNARY ? 2 : 1, b_planes = p.b_kind == B_TERNARY ? 2 : 1;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA0);
        if (a_planes == 2) tma_prefetch_desc(&tmA1);
        tma_prefetch_desc(&tmB0);
        if (b_planes == 2) tma_prefetch_desc(&tmB1);
        for (int s = 0; s < p.ring; ++s) {
            mbar_init(&bfull[s], 1);
            mbar_init(&bempty[s], 4 * GV_UPS);  // 4 warps per unit
        }
        for (int c = 0; c < GV_CST_; ++c) {
            mbar_init(&cfull[c], 4);
            mbar_init(&cempty[c], 1);  // MMA commit
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&afull[a], 1);
            mbar_init(&aempty[a], 4);  // epilogue warps
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, GV_TMEM_COLS_);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (warp >= 12) {
        uint32_t ones[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) ones[i] = 0x7F7F7F7Fu;  // UE8M0 1.0
        tmem_st_32x32b_x16(tmem_base + (uint32_t((warp & 3) * 32) << 16) + uint32_t(GV_SFCOL_), ones);
        tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_launch_dependents();
    pdl_wait();

    const int64_t total = p.entries * p.tiles_per_entry;
    if (warp == 0) {
        // ------------------------------ TMA producer ------------------------------
        if (lane == 0) {
            const uint32_t tx = uint32_t(stage_bytes);
            int s = 0;
            uint32_t ph = 0;
            for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
                const uint32_t e = gv_fdiv(uint32_t(t), p.fd_tpe);
                const int row = int(uint32_t(t) - e * p.fd_tpe.d) * GV_BM;
                const uint32_t eb_ = gv_fdiv(e, p.fd_nh);
                const int eb = int(eb_), eh = int(e - eb_ * p.fd_nh.d);
                const int nsup = (p.num_kb + GV_UPS - 1) / GV_UPS, rot = int(uint32_t(t) - gv_fdiv(uint32_t(t), p.fd_nsup) * uint32_t(nsup));
                for (int j = 0; j < p.num_kb; j += GV_UPS) {
                    mbar_wait(&bempty[s], ph ^ 1);
                    mbar_arrive_expect_tx(&bfull[s], tx);
                    uint8_t* st = sBits + s * stage_bytes;
                    // K slices in a per-tile rotated order: the CTAs then do not all read the
                    // same (small-operand) lines at once -- an L2 hot spot
                    const int js = j / GV_UPS + rot;
                    const int kw = (js < nsup ? js : js - nsup) * GV_UPS * GV_WPS;
                    tma_load_4d(st, &tmA0, &bfull[s], kw, row, eh, eb);
                    if (a_planes == 2) tma_load_4d(st + GV_BM * 128, &tmA1, &bfull[s], kw, row, eh, eb);
                    tma_load_4d(st + p.a_bits, &tmB0, &bfull[s], kw, 0, eh, eb);
                    if (b_planes == 2) tma_load_4d(st + p.a_bits + NB * 128, &tmB1, &bfull[s], kw, 0, eh, eb);
                    if (++s == p.ring) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------ MMA issuer ------------------------------
        // the whole warp issues (elect.sync inside the asm): operands stay in uniform registers
        constexpr uint32_t idesc = idesc_mxf4(GV_BM, NB);
        const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem_base, 0);
        const uint32_t sfa = tmem_u + uint32_t(GV_SFCOL_), sfb = tmem_u + uint32_t(GV_SFCOL_ + 8);
        int c = 0;
        uint32_t cph = 0;
        int acc = 0;
        uint32_t aph = 0;
        for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
            mbar_wait(&aempty[acc], aph ^ 1);
            tc_fence_after();
            const uint32_t d = tmem_u + uint32_t(acc * NB);
            for (int kb = 0; kb < p.num_kb; ++kb) {
                mbar_wait(&cfull[c], cph);
                tc_fence_after();
                {
                    const uint32_t a0 = tmem_u + uint32_t(GV_ACOL + c * 32);
                    const uint32_t b0 = smem_u32(sB + c * C::B_BYTES);
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        mma_mxf4_ts_w(d, a0 + 8 * k, smem_desc_sw128(b0 + 32 * k), idesc, sfa, sfb, (kb | k) != 0);
                    tc_commit_w(&cempty[c]);
                }
                __syncwarp();
                if (++c == GV_CST_) {
                    c = 0;
                    cph ^= 1;
                }
            }
            tc_commit_w(&afull[acc]);
            __syncwarp();
            acc ^= 1;
            if (acc == 0) aph ^= 1;
        }
    } else if (warp >= 4 && warp < 12) {
        // ------------------------------ unpack ------------------------------
        const int q = warp & 3, grp = (warp - 4) >> 2;
        const int arow = 32 * q + lane;        // kernel-A row within the tile (= TMEM lane)
        const int ut = (warp & 3) * 32 + lane; // 0..127 within the group: small-operand words ut, ut + 128
        const uint32_t lane_base = tmem_base + (uint32_t(32 * q) << 16) + uint32_t(GV_ACOL);
        int s = 0, c = 0;
        uint32_t ph = 0, cph = 0;
        int u = 0;  // unit counter (group grp takes u % 2 == grp), padded to whole bit stages
        for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
            const int nsup = (p.num_kb + GV_UPS - 1) / GV_UPS, rot = int(uint32_t(t) - gv_fdiv(uint32_t(t), p.fd_nsup) * uint32_t(nsup));
            for (int kb0 = 0; kb0 < p.num_kb; kb0 += GV_UPS) {
                const int js = kb0 / GV_UPS + rot;
                const int kb = (js < nsup ? js : js - nsup) * GV_UPS;  // first unit of this bit stage
#pragma unroll 1
                for (int sub = 0; sub < GV_UPS; ++sub, ++u) {
                    const bool real = kb + sub < p.num_kb;
                    if ((u & 1) == grp) {
                        mbar_wait(&bfull[s], ph);
                        if (real) {
                            mbar_wait(&cempty[c], cph ^ 1);
                            tc_fence_after();
                            const uint32_t st = smem_u32(sBits + s * stage_bytes);
                            // kernel-A: the 2 16-byte chunks (2 sub, 2 sub + 1) of row arow (128B swizzle)
                            // -> TMEM lane arow, the 32 columns of code stage c
                            const uint32_t pa = st + arow * 128;
                            const uint32_t ta = lane_base + uint32_t(c * 32);
                            const int c0 = (2 * sub) ^ (arow & 7), c1 = (2 * sub + 1) ^ (arow & 7);
                            if (p.a_kind == B_BINARY) unpack_a_row<B_BINARY>(pa + 16 * c0, pa + 16 * c1, 0, ta);
                            else if (p.a_kind == B_BOOL) unpack_a_row<B_BOOL>(pa + 16 * c0, pa + 16 * c1, 0, ta);
                            else unpack_a_row<B_TERNARY>(pa + 16 * c0, pa + 16 * c1, GV_BM * 128, ta);
                            // kernel-B: word bw of row brow (chunk 2 sub + bw / 4 of its swizzled 128-byte line)
                            // -> 16-byte code chunk (bw ^ (brow & 7)) of its SW128 code row
#pragma unroll
                            for (int i = 0; i < NB * 8 / 128; ++i) {
                                const int wi = ut + 128 * i, brow = wi >> 3, bw = wi & 7;
                                const uint32_t pb = st + p.a_bits + brow * 128 +
                                                    ((((2 * sub + (bw >> 2)) ^ (brow & 7))) << 4) + (bw & 3) * 4;
                                uint32_t x0, x1 = 0, o[4];
                                asm volatile("ld.shared.b32 %0, [%1];" : "=r"(x0) : "r"(pb));
                                if (p.b_kind == B_TERNARY)
                                    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(x1) : "r"(pb + NB * 128));
                                if (p.b_kind == B_BINARY) unpack_chunk<B_BINARY>(x0, x1, o);
                                else if (p.b_kind == B_BOOL) unpack_chunk<B_BOOL>(x0, x1, o);
                                else unpack_chunk<B_TERNARY>(x0, x1, o);
                                sts128(smem_u32(sB + c * C::B_BYTES) + brow * GV_ROWB + ((bw ^ (brow & 7)) << 4), o[0],
                                       o[1], o[2], o[3]);
                            }
                            tmem_wait_st();
                            fence_proxy_async_smem();
                            tc_fence_before();
                        }
                        __syncwarp();
                        if (lane == 0) {
                            mbar_arrive(&bempty[s]);
                            if (real) mbar_arrive(&cfull[c]);
                        }
                    }
                    if (real && ++c == GV_CST_) {
                        c = 0;
                        cph ^= 1;
                    }
                }
                if (++s == p.ring) {
                    s = 0;
                    ph ^= 1;
                }
            }
        }
    } else if (warp >= 12) {
        // ------------------------------ epilogue ------------------------------
        const int q = warp & 3;
        int acc = 0;
        uint32_t aph = 0;
        for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
            const uint32_t e = gv_fdiv(uint32_t(t), p.fd_tpe);
            const int64_t r = int64_t(uint32_t(t) - e * p.fd_tpe.d) * GV_BM + 32 * q + lane;
            const uint32_t eb_ = gv_fdiv(e, p.fd_nh);
            const int64_t eoff = int64_t(eb_) * p.y_bs + int64_t(e - eb_ * p.fd_nh.d) * p.y_hs;
            mbar_wait(&afull[acc], aph);
            tc_fence_after();
            uint32_t v[NB];
            if constexpr (NB == 16) tmem_ld_32x32b_x16(tmem_base + (uint32_t(32 * q) << 16) + uint32_t(acc * NB), v);
            else tmem_ld_32x32b_x32(tmem_base + (uint32_t(32 * q) << 16) + uint32_t(acc * NB), v);
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&aempty[acc]);
            acc ^= 1;
            if (acc == 0) aph ^= 1;
            if (r < p.M) {
                const float crow = p.scale && p.scale_on_rows ? __fmul_rn(__ldg(p.scale + r), p.scalar) : p.scalar;
                const int ncol = int(p.N);
#pragma unroll
                for (int j = 0; j < NB; ++j) {
                    if (j < ncol) {
                        const float cj = p.scale && !p.scale_on_rows ? __fmul_rn(__ldg(p.scale + j), p.scalar) : crow;
                        const uint32_t vj = __float_as_uint(__fadd_rn(__uint_as_float(v[j]), p.dot_bias));
                        store_out(p, eoff + r * p.y_rs + j * p.y_cs, __fmul_rn(__uint_as_float(vj), cj), vj);
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem_base, GV_TMEM_COLS_);
    }
}

template <int NB, int CPS>
cudaError_t launch_gemv_cps(const CUtensorMap& a0, const CUtensorMap& a1, const CUtensorMap& b0, const CUtensorMap& b1,
                        GvParams& p, cudaStream_t s) {
    using C = GvCfg<NB>;
    const int a_planes = p.a_kind == B_TERNARY ? 2 : 1, b_planes = p.b_kind == B_TERNARY ? 2 : 1;
    p.a_bits = a_planes * GV_BM * 128;
    p.b_bits = b_planes * NB * 128;
    const int stage = p.a_bits + p.b_bits;
    const int bar_bytes = (2 * GV_MAXRING + 2 * gv_cst(CPS) + 4) * 8 + 16;
    const int fixed = 1024 + gv_cst(CPS) * C::B_BYTES + bar_bytes;
    int ring = (gv_smem_max(CPS) - fixed) / stage;
    if (ring > GV_MAXRING) ring = GV_MAXRING;
    p.ring = ring;
    const int smem = fixed + ring * stage;
    auto kern = tc_gemv_kernel<NB, CPS>;
    static std::atomic<uint64_t> optin{0};  // per device
    if (cudaError_t e = ensure_smem_optin(kern, gv_smem_max(CPS), optin); e != cudaSuccess) return e;
    const int64_t total = p.entries * p.tiles_per_entry;
    const int64_t slots = int64_t(num_sms()) * CPS;
    const int grid = int(total < slots ? total : slots);
    return launch_pdl(kern, dim3(grid), dim3(GV_NT), size_t(smem), s, 1, a0, a1, b0, b1, p);
}
template <int NB>
cudaError_t launch_gemv(const CUtensorMap& a0, const CUtensorMap& a1, const CUtensorMap& b0, const CUtensorMap& b1,
                        GvParams& p, cudaStream_t s) {
    const int64_t total = p.entries * p.tiles_per_entry;
    if (total > num_sms()) return launch_gemv_cps<NB, 2>(a0, a1, b0, b1, p, s);
    return launch_gemv_cps<NB, 1>(a0, a1, b0, b1, p, s);
}

}  // namespace

// The skinny kernel serves any matmul whose smaller side has <= 32 rows.
bool matmul_gemv_eligible(const MatmulArgs& a) {
    if (a.pack_out || a.tile_n || a.cta_group) return false;  // fused pack / forced tiles: general kernel
    const int64_t small = a.M < a.N ? a.M : a.N;
    return small >= 1 && small <= 32;
}

cudaError_t launch_matmul_gemv(const MatmulArgs& a, cudaStream_t s) {
    // kernel-A = the large side (128-row tiles, codes in TMEM), kernel-B = the <= 32-row side
    const bool swap = a.M < a.N;  // caller's W / K / V^T side is the large one
    const uint32_t *ka_sgn = swap ? a.b_sgn : a.a_sgn, *ka_nz = swap ? a.b_nz : a.a_nz;
    const uint32_t *kb_sgn = swap ? a.a_sgn : a.b_sgn, *kb_nz = swap ? a.a_nz : a.b_nz;
    const int64_t Mk = swap ? a.N : a.M, Nk = swap ? a.M : a.N;
    const int64_t lda = swap ? a.ldb : a.lda, ldb = swap ? a.lda : a.ldb;
    const int64_t a_bs = swap ? a.b_bs : a.a_bs, a_hs = swap ? a.b_hs : a.a_hs;
    const int64_t b_bs = swap ? a.a_bs : a.b_bs, b_hs = swap ? a.a_hs : a.b_hs;
    const int akind = kind_of(ka_sgn, ka_nz), bkind = kind_of(kb_sgn, kb_nz);
    const int nb_rows = Nk <= 16 ? 16 : 32;

    CUtensorMap ma0, ma1, mb0, mb1;
    const uint32_t* pa0 = akind == B_BOOL ? ka_nz : ka_sgn;
    const uint32_t* pa1 = akind == B_TERNARY ? ka_nz : pa0;
    const uint32_t* pb0 = bkind == B_BOOL ? kb_nz : kb_sgn;
    const uint32_t* pb1 = bkind == B_TERNARY ? kb_nz : pb0;
    const int box_w = GV_WPS * GV_UPS;  // 32 words = 128 B per row
    const CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B;
    if (!encode_planes(&ma0, pa0, lda, Mk, a_hs, a_bs, a.nh, a.nb, GV_BM, box_w, sw) ||
        !encode_planes(&ma1, pa1, lda, Mk, a_hs, a_bs, a.nh, a.nb, GV_BM, box_w, sw) ||
        !encode_planes(&mb0, pb0, ldb, Nk, b_hs, b_bs, a.nh, a.nb, nb_rows, box_w, sw) ||
        !encode_planes(&mb1, pb1, ldb, Nk, b_hs, b_bs, a.nh, a.nb, nb_rows, box_w, sw))
        return cudaErrorInvalidValue;

    GvParams p{};
    p.M = Mk;
    p.N = Nk;
    p.num_kb = int((kw4_of(a.K) + GV_WPS - 1) / GV_WPS);
    p.fd_nsup = make_fastdiv(uint32_t((p.num_kb + GV_UPS - 1) / GV_UPS));
    if (!ka_nz && !kb_nz) p.dot_bias = float(a.K - int64_t(p.num_kb) * GV_WPS * 32);  // W1A1 padding
    p.nh = a.nh;
    p.entries = a.nb * a.nh;
    p.tiles_per_entry = int((Mk + GV_BM - 1) / GV_BM);
    if (int64_t(p.tiles_per_entry) * a.nb * a.nh >= (int64_t(1) << 31)) return cudaErrorNotSupported;
    p.fd_tpe = make_fastdiv(uint32_t(p.tiles_per_entry));
    p.fd_nh = make_fastdiv(uint32_t(a.nh));
    p.a_kind = akind;
    p.b_kind = bkind;
    p.y = a.y;
    p.y_dt = a.y_dt;
    // caller's Y[i][j] at i * ldy + j (or j * ldy + i when transposed); kernel row = j if swapped
    const int64_t si = a.y_trans ? 1 : a.ldy, sj = a.y_trans ? a.ldy : 1;
    p.y_rs = swap ? sj : si;
    p.y_cs = swap ? si : sj;
    p.y_bs = a.y_bs;
    p.y_hs = a.y_hs;
    p.scale = a.col_scale;
    p.scale_on_rows = swap ? 1 : 0;
    p.scalar = a.scalar;
    return nb_rows == 16 ? launch_gemv<16>(ma0, ma1, mb0, mb1, p, s) : launch_gemv<32>(ma0, ma1, mb0, mb1, p, s);
}

}  // namespace bwta
