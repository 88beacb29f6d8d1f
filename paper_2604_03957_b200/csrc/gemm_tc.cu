// gemm_tc.cu -- design (b): BWTA matmul on the 5th-generation tensor cores.
//
// sm_100a has no binary (b1) MMA (the paper's mma.sync b1 is
// emulated there through IMMA + MOVM), so the codes {-1, 0, +1} are fed to
// tcgen05.mma.kind::i8 (s8 x s8 -> s32, exact for |dot| <= 2^24).  The dot
// product is the same integer the paper's Case 1/2/3 instruction sequences
// compute; the epilogue applies c = fl32(scale[n] * scalar)
// (w_scale * a_scale, or alpha / beta) exactly as design (a).
//
// Operand roles.  The kernel computes D[i][j] = sum_k A8[i][k] * B[j][k] with
//   kernel-A : int8 image of the SMALLER operand, expanded once per call into
//              the workspace by expand_kernel (L2-resident), loaded by TMA;
//   kernel-B : the LARGER operand, read as packed bit planes by TMA (N*K/8
//              bytes for binary weights) and unpacked to int8 in shared memory
//              by 4 unpack warps, straight into the UMMA 128B-swizzled
//              K-major layout.  No int8 copy of it ever touches HBM.
// If the caller's A is the larger operand the roles swap and the epilogue
// stores D^T (Y[m][n] = D[n][m]).
//
// CTA (one per SM, persistent over tiles of 128 x BN), 12 warps:
//   warp 0     TMA producer: A8 tile (16 KB) + B bit tiles into a STAGES ring
//   warp 1     MMA issuer: 4 x tcgen05.mma (128 x BN x 32) per 128-K stage,
//              accumulators double-buffered in TMEM (2 x BN columns)
//   warp 2     TMEM allocator
//   warps 4-7  epilogue: tcgen05.ld 32x32b -> fp32 scale -> fp16/bf16/fp32/
//              i32 -> 128B-swizzled staging -> TMA tensor store (clips tails)
//   warps 8-11 unpack: bits (smem) -> int8 codes (smem), fence.proxy.async
// Barriers: full (TMA tx), bready (unpack done), empty (MMA commit),
// tfull (accumulator ready), tempty (epilogue drained TMEM).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "bwta_internal.h"
#include "sm100.cuh"

namespace bwta {
namespace {

using namespace sm100;

constexpr int BM = 128;     // MMA M (kernel-A rows per tile), cta_group::1
constexpr int BK = 128;     // K elements (= int8 bytes) per stage: one 128B swizzle row
constexpr int UMMA_K = 32;  // K per tcgen05.mma for 8-bit inputs
constexpr int NT = 384;     // 12 warps
constexpr int OUT_BUF = 4096;

enum BKind { B_BINARY = 0, B_BOOL = 1, B_TERNARY = 2 };

struct TcParams {
    int64_t M, N;  // kernel rows (A side) / cols (B side) per entry
    int num_kb;
    int64_t nh, entries;
    int m_tiles, n_tiles;
    // epilogue
    void* y;
    int y_dt;
    int64_t ldy, y_bs, y_hs;  // elements (direct-store fallback)
    int out_trans;            // memory holds D^T
    int use_tma_store;
    const float* scale;  // per kernel column (or per kernel row if scale_on_rows), may be null
    int scale_on_rows;
    float scalar;
};

template <int BN, int BKIND, int CG>
struct Cfg {
    static constexpr int BNC = BN / CG;          // kernel-B rows held (and unpacked) per CTA
    static constexpr int A_BYTES = BM * BK;
    static constexpr int B_BYTES = BNC * BK;
    static constexpr int PLANE_BYTES = BNC * 16;  // 4 words per row per stage
    static constexpr int NPLANES = BKIND == B_TERNARY ? 2 : 1;
    static constexpr int STAGE = A_BYTES + B_BYTES + NPLANES * PLANE_BYTES;
    static constexpr int OUT_BYTES = 4 * 2 * OUT_BUF;
    static constexpr int STAGES_FIT = (210 * 1024 - OUT_BYTES) / STAGE;
    static constexpr int STAGES = STAGES_FIT > 6 ? 6 : STAGES_FIT;
    static constexpr int BAR_BYTES = 256;
    static constexpr int SMEM = 1024 + STAGES * STAGE + OUT_BYTES + BAR_BYTES;
    static constexpr int TMEM_COLS = 2 * BN;
    static_assert(STAGES >= 2, "pipeline too shallow");
    static_assert(BNC % 8 == 0, "swizzle atoms are 8 rows");
};

// K order inside the int8 operand tiles.  Element k (0..31) of a packed word
// lands at byte 4*(k%8) + k/8 of its 32-byte group, i.e. code word j
// (j = 0..7) holds elements {j, 8+j, 16+j, 24+j}.  Both MMA operands use the
// same permutation (expand_kernel for A, the unpack warps for B), so every
// dot product is unchanged.
//
// Codes are scaled by 64 (int8 0x40 = +64, 0xC0 = -64, 0x00): the nz bit of
// element 8i+j moves to bit 6 of byte i and the sgn bit to bit 7 by LEFT
// shifts, which run as IMAD.SHL on the FMA pipe, so a code word costs ~2 FMA
// + 2 logic instructions instead of a nibble spread (measured in
// tools/ubench: 230 vs 313 cycles per 128-element ternary row per warp).  The
// s32 accumulator holds 4096 * dot exactly (|dot| <= K <= 2^18) and the
// epilogue recovers dot with an arithmetic shift by 12.
//   binary  (x0 = sgn):           0x40 | sgn << 7          -> +64 / -64
//   bool    (x0 = nz):            nz << 6                  -> 0 / +64
//   ternary (x0 = sgn, x1 = nz):  nz << 6 | sgn << 7       -> 0 / +64 / -64
// (ternary planes are canonical: sgn is a subset of nz, include/bwta.h)
constexpr int CODE_SHIFT = 12;  // log2(64 * 64)

__device__ __forceinline__ uint32_t shl_fma(uint32_t x, int k) {  // x << k as IMAD.SHL (FMA pipe)
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, 0;" : "=r"(r) : "r"(x), "r"(1u << k));
    return r;
}
__device__ __forceinline__ uint32_t to_bit6(uint32_t x, int j) { return j < 7 ? shl_fma(x, 6 - j) : (x >> 1); }

template <int KIND>
__device__ __forceinline__ uint32_t unpack_word(uint32_t x0, uint32_t x1, int j) {
    if (KIND == B_BINARY) return (shl_fma(x0, 7 - j) & 0x80808080u) | 0x40404040u;
    if (KIND == B_BOOL) return to_bit6(x0, j) & 0x40404040u;
    return (to_bit6(x1, j) & 0x40404040u) | (shl_fma(x0, 7 - j) & 0x80808080u);
}

// raw s32 accumulator (4096 * dot) -> dot
__device__ __forceinline__ int32_t dot_of(uint32_t acc) { return int32_t(acc) >> CODE_SHIFT; }
__device__ __forceinline__ float scaled(uint32_t acc, float c) { return __fmul_rn(__int2float_rn(dot_of(acc)), c); }

__device__ __forceinline__ uint32_t pack2(int dt, float lo, float hi) {
    if (dt == DT_F16) {
        __half2 h = __halves2half2(__float2half_rn(lo), __float2half_rn(hi));
        return *reinterpret_cast<uint32_t*>(&h);
    }
    __nv_bfloat162 h = __halves2bfloat162(__float2bfloat16_rn(lo), __float2bfloat16_rn(hi));
    return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

// Epilogue warp `ew` owns TMEM lanes 32*ew .. 32*ew+31 (kernel rows).  ES =
// output element size; a chunk is CW = 128/ES columns = one 128-byte row.
template <int BN, int ES, int CG>
__device__ __forceinline__ void epilogue(const TcParams& p, const CUtensorMap& tmY, uint32_t tmem_base, uint8_t* sOut,
                                         uint64_t* tfull, uint64_t* tempty, int ew, int lane,
                                         int64_t tiles_per_entry, int64_t total, int rank, int64_t t0,
                                         int64_t tstep) {
    constexpr int CW = 128 / ES;
    uint8_t* stg_base = sOut + ew * 2 * OUT_BUF;
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t nchunk = 0;
    for (int64_t t = t0; t < total; t += tstep) {
        const int64_t e = t / tiles_per_entry;
        const int64_t r = t % tiles_per_entry;
        const int mt = int(r % p.m_tiles), nt = int(r / p.m_tiles);
        const int eb = int(e / p.nh), eh = int(e % p.nh);
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        const int64_t mrow0 = int64_t(mt) * BM * CG + rank * BM;  // first kernel row of this CTA
        const int64_t row = mrow0 + ew * 32 + lane;               // kernel row of this thread
        const bool rok = row < p.M;
        float crow = p.scalar;
        if (p.scale_on_rows && p.scale) crow = __fmul_rn(__ldg(p.scale + (rok ? row : 0)), p.scalar);
        const bool col_scaled = !p.scale_on_rows && p.scale;
        const int64_t ybase = int64_t(eb) * p.y_bs + int64_t(eh) * p.y_hs;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += CW) {
            const int64_t n0 = int64_t(nt) * BN + c0;
            uint32_t v[CW];
            tmem_ld_32x32b_x32(tmem_base + (uint32_t(ew * 32) << 16) + uint32_t(acc * BN + c0),
                               *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
            if (CW == 64)
                tmem_ld_32x32b_x32(tmem_base + (uint32_t(ew * 32) << 16) + uint32_t(acc * BN + c0 + 32),
                                   *reinterpret_cast<uint32_t(*)[32]>(&v[CW == 64 ? 32 : 0]));
            tmem_wait_ld();
            if (n0 >= p.N) continue;
            // per-column scale: lane j holds the scale of column n0 + j (+ 32)
            float cl[CW / 32];
#pragma unroll
            for (int u = 0; u < CW / 32; ++u) {
                const int64_t n = n0 + 32 * u + lane;
                cl[u] = col_scaled ? __fmul_rn(__ldg(p.scale + (n < p.N ? n : 0)), p.scalar) : crow;
            }
            float f[CW];
#pragma unroll
            for (int j = 0; j < CW; ++j) {
                const float c = col_scaled ? __shfl_sync(0xffffffffu, cl[j / 32], j % 32) : crow;
                f[j] = scaled(v[j], c);
            }
            if (p.use_tma_store) {
                uint8_t* stg = stg_base + (nchunk & 1) * OUT_BUF;
                if (lane == 0) bulk_wait_read<1>();
                __syncwarp();
                const uint32_t sbase = smem_u32(stg);
                if (!p.out_trans) {
                    // row `lane` of a [32 rows x 128 B] box, 128B-swizzled
                    uint32_t w[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        if (ES == 2) w[j] = pack2(p.y_dt, f[2 * j], f[(2 * j + 1) % CW]);
                        else w[j] = p.y_dt == DT_F32 ? __float_as_uint(f[j]) : uint32_t(dot_of(v[j]));
                    }
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        sts128(sbase + lane * 128 + ((q ^ (lane & 7)) << 4), w[4 * q], w[4 * q + 1], w[4 * q + 2],
                               w[4 * q + 3]);
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        tma_store_4d(&tmY, stg, int(n0), int(mrow0 + ew * 32), eh, eb);
                        bulk_commit();
                    }
                } else {
                    // box [CW kernel-cols][32 kernel-rows]: lane is the contiguous index
#pragma unroll
                    for (int j = 0; j < CW; ++j) {
                        const uint32_t a = sbase + j * 32 * ES + lane * ES;
                        if (ES == 2) {
                            const uint32_t h2 = pack2(p.y_dt, f[j], 0.f);
                            asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"(uint16_t(h2 & 0xffffu)) : "memory");
                        } else {
                            const uint32_t o = p.y_dt == DT_F32 ? __float_as_uint(f[j]) : uint32_t(dot_of(v[j]));
                            asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(o) : "memory");
                        }
                    }
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        tma_store_4d(&tmY, stg, int(mrow0 + ew * 32), int(n0), eh, eb);
                        bulk_commit();
                    }
                }
                ++nchunk;
            } else {
                // direct stores (outputs whose layout TMA cannot describe)
#pragma unroll
                for (int j = 0; j < CW; ++j) {
                    const int64_t n = n0 + j;
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
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
            if (CG == 1) mbar_arrive(&tempty[acc]);
            else mbar_arrive_cluster(mapa_smem(&tempty[acc], 0));  // the leader owns the MMA
        }
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
    }
    if (lane == 0) bulk_wait_all();
}

template <int BN, int BKIND, int CG>
__global__ void __launch_bounds__(NT, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB0,
                   const __grid_constant__ CUtensorMap tmB1, const __grid_constant__ CUtensorMap tmY, TcParams p) {
    using C = Cfg<BN, BKIND, CG>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = sA + C::STAGES * C::A_BYTES;
    uint8_t* sBits = sB + C::STAGES * C::B_BYTES;  // [stage][plane][BNC rows][16 B]
    uint8_t* sOut = sBits + C::STAGES * C::NPLANES * C::PLANE_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sOut + C::OUT_BYTES);
    uint64_t* bready = full + C::STAGES;
    uint64_t* empty = bready + C::STAGES;
    uint64_t* tfull = empty + C::STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int rank = CG == 2 ? int(cluster_ctarank()) : 0;
    const bool leader = rank == 0;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB0);
        if (C::NPLANES == 2) tma_prefetch_desc(&tmB1);
        if (p.use_tma_store) tma_prefetch_desc(&tmY);
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&bready[s], 4 * CG);  // unpack warps of every CTA of the pair
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 4 * CG);  // epilogue warps of every CTA of the pair
        }
        fence_barrier_init();
    }
    if (warp == 2) {
        if (CG == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
        else tmem_alloc2(tmem_slot, C::TMEM_COLS);
    }
    tc_fence_before();
    if (CG == 2) cluster_sync();
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // prologue done (smem barriers, TMEM, descriptor prefetch): let the next
    // kernel start its own, then wait for our inputs (predecessor grid)
    pdl_launch_dependents();
    pdl_wait();

    const int64_t tiles_per_entry = int64_t(p.m_tiles) * p.n_tiles;
    const int64_t total = p.entries * tiles_per_entry;
    const int64_t t0 = blockIdx.x / CG, tstep = gridDim.x / CG;  // persistent over pair-tiles

    if (warp == 0) {
        // ------------------------------ TMA producer ------------------------------
        int stage = 0;
        uint32_t phase = 0;
        for (int64_t t = t0; t < total; t += tstep) {
            const int64_t e = t / tiles_per_entry;
            const int64_t r = t % tiles_per_entry;
            const int mt = int(r % p.m_tiles), nt = int(r / p.m_tiles);
            const int eb = int(e / p.nh), eh = int(e % p.nh);
            const int arow = mt * BM * CG + rank * BM;
            const int brow = nt * BN + rank * C::BNC;
            for (int kb = 0; kb < p.num_kb; ++kb) {
                mbar_wait(&empty[stage], phase ^ 1);
                if (lane == 0) {
                    mbar_arrive_expect_tx(&full[stage], C::A_BYTES + C::NPLANES * C::PLANE_BYTES);
                    tma_load_3d(sA + stage * C::A_BYTES, &tmA, &full[stage], kb * BK, arow, int(e));
                    uint8_t* bits = sBits + stage * C::NPLANES * C::PLANE_BYTES;
                    tma_load_4d(bits, &tmB0, &full[stage], kb * 4, brow, eh, eb);
                    if (C::NPLANES == 2) tma_load_4d(bits + C::PLANE_BYTES, &tmB1, &full[stage], kb * 4, brow, eh, eb);
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
            constexpr uint32_t idesc = idesc_i8(BM * CG, BN);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int64_t t = t0; t < total; t += tstep) {
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d = tmem_base + uint32_t(acc * BN);
                for (int kb = 0; kb < p.num_kb; ++kb) {
                    mbar_wait(&full[stage], phase);
                    mbar_wait(&bready[stage], phase);
                    tc_fence_after();
                    if (lane == 0) {
                        const uint32_t a0 = smem_u32(sA + stage * C::A_BYTES);
                        const uint32_t b0 = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
                        for (int k = 0; k < BK / UMMA_K; ++k) {
                            const uint64_t ad = smem_desc_sw128(a0 + k * UMMA_K), bd = smem_desc_sw128(b0 + k * UMMA_K);
                            if (CG == 1) mma_i8(d, ad, bd, idesc, (kb | k) != 0);
                            else mma_i8_cg2(d, ad, bd, idesc, (kb | k) != 0);
                        }
                        if (CG == 1) tc_commit(&empty[stage]);
                        else tc_commit2_mc(&empty[stage], 0x3);
                    }
                    __syncwarp();
                    if (++stage == C::STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if (lane == 0) {
                    if (CG == 1) tc_commit(&tfull[acc]);
                    else tc_commit2_mc(&tfull[acc], 0x3);
                }
                __syncwarp();
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
        }
    } else if (warp >= 8) {
        // ------------------------------ unpack ------------------------------
        const int ut = threadIdx.x - 256;  // 0..127
        const uint32_t bready_addr0 = CG == 2 ? mapa_smem(&bready[0], 0) : 0u;
        int stage = 0;
        uint32_t phase = 0;
        for (int64_t t = t0; t < total; t += tstep) {
            for (int kb = 0; kb < p.num_kb; ++kb) {
                mbar_wait(&full[stage], phase);
                const uint32_t bits = smem_u32(sBits + stage * C::NPLANES * C::PLANE_BYTES);
                const uint32_t bdst = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
                for (int i = 0; i < (C::BNC + 127) / 128; ++i) {
                    const int r = ut + 128 * i;
                    if (r < C::BNC) {
                        // plane 0: sgn (binary/ternary) or nz (bool); plane 1: nz (ternary)
                        const uint4 w0 = lds128(bits + r * 16);
                        uint4 w1 = make_uint4(0, 0, 0, 0);
                        if (BKIND == B_TERNARY) w1 = lds128(bits + C::PLANE_BYTES + r * 16);
                        const uint32_t p0[4] = {w0.x, w0.y, w0.z, w0.w};
                        const uint32_t p1[4] = {w1.x, w1.y, w1.z, w1.w};
                        const uint32_t rowaddr = bdst + r * 128;
#pragma unroll
                        for (int g = 0; g < 4; ++g) {  // 32-element group = one packed word
                            uint32_t o[8];
#pragma unroll
                            for (int j = 0; j < 8; ++j) o[j] = unpack_word<BKIND>(p0[g], p1[g], j);
                            sts128(rowaddr + (((2 * g) ^ (r & 7)) << 4), o[0], o[1], o[2], o[3]);
                            sts128(rowaddr + (((2 * g + 1) ^ (r & 7)) << 4), o[4], o[5], o[6], o[7]);
                        }
                    }
                }
                fence_proxy_async_smem();
                __syncwarp();
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
        // ------------------------------ epilogue ------------------------------
        if (p.y_dt == DT_F16 || p.y_dt == DT_BF16)
            epilogue<BN, 2, CG>(p, tmY, tmem_base, sOut, tfull, tempty, warp - 4, lane, tiles_per_entry, total, rank,
                                t0, tstep);
        else
            epilogue<BN, 4, CG>(p, tmY, tmem_base, sOut, tfull, tempty, warp - 4, lane, tiles_per_entry, total, rank,
                                t0, tstep);
    }
    tc_fence_before();
    if (CG == 2) cluster_sync();
    else __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        if (CG == 1) tmem_dealloc(tmem_base, C::TMEM_COLS);
        else tmem_dealloc2(tmem_base, C::TMEM_COLS);
    }
}

// ---------------------------------------------------------------------------
// Expand packed planes to an int8 image out[e][r][k'] of x64 codes in the
// unpack_word K order.  Kind from plane presence: sgn+nz ternary, nz only bool,
// sgn only binary (nz = the valid elements of the row).
// ---------------------------------------------------------------------------
struct ExpandArgs {
    const uint32_t* sgn;
    const uint32_t* nz;
    int64_t rows, K, ld, bs, hs, nh, entries;
    int64_t kw4;  // words per output row (Kp = 32 * kw4)
    int8_t* out;
    FastDiv div_kw4, div_rows, div_nh;
};

__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) { return (__umulhi(n, f.mul) + n) >> f.shift; }
__device__ __forceinline__ uint64_t fdiv(uint64_t n, const FastDiv& f) { return n / f.d; }

template <typename IDX>
__global__ void __launch_bounds__(256) expand_kernel(ExpandArgs a) {
    const IDX total = IDX(a.entries * a.rows * a.kw4);
    const IDX kw4 = IDX(a.kw4), rows = IDX(a.rows), nh = IDX(a.nh);
    pdl_launch_dependents();
    pdl_wait();  // no global memory access before the predecessor grid completed
    for (IDX i = IDX(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += IDX(gridDim.x) * blockDim.x) {
        const IDX rr = fdiv(i, a.div_kw4), w = i - rr * kw4;
        const IDX e = fdiv(rr, a.div_rows), r = rr - e * rows;
        const IDX eb = fdiv(e, a.div_nh), eh = e - eb * nh;
        const int64_t off = int64_t(eb) * a.bs + int64_t(eh) * a.hs + int64_t(r) * a.ld + int64_t(w);
        uint32_t nz = a.nz ? __ldg(a.nz + off) : 0xffffffffu;
        const uint32_t sg = a.sgn ? __ldg(a.sgn + off) & nz : 0u;
        if (!a.nz) {  // binary: element validity comes from K (no nz plane)
            const int64_t valid = a.K - int64_t(w) * 32;
            nz = valid >= 32 ? 0xffffffffu : (valid <= 0 ? 0u : ((1u << valid) - 1u));
        }
        uint32_t o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = unpack_word<B_TERNARY>(sg & nz, nz, j);
        uint4* dst = reinterpret_cast<uint4*>(a.out + int64_t(i) * 32);
        dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
        dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

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

int num_sms() {
    static int n = 0;
    if (n == 0) {
        int dev = 0, v = 148;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) v = 148;
        n = v;
    }
    return n;
}

int64_t kw4_of(int64_t K) { return ((K + 31) / 32 + 3) / 4 * 4; }
size_t round1k(size_t x) { return (x + 1023) & ~size_t(1023); }

// A stride for a batch dimension of extent `count`: TMA needs a multiple of 16
// bytes even when the dimension is degenerate.
uint64_t bstride(int64_t count, int64_t stride_bytes, uint64_t fallback) {
    return (count <= 1 || stride_bytes <= 0) ? fallback : uint64_t(stride_bytes);
}

struct Plan {
    bool swap;
    const uint32_t *a_sgn, *a_nz, *b_sgn, *b_nz;  // kernel operands
    int64_t Mk, Nk, lda, ldb, a_bs, a_hs, b_bs, b_hs;
    int bkind;
};

Plan make_plan(const MatmulArgs& a) {
    Plan p{};
    p.swap = a.M > a.N;
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

int pick_bn(int64_t N) { return N > 128 ? 256 : (N > 64 ? 128 : 64); }

template <int BN, int BKIND, int CG>
cudaError_t launch_cfg(const CUtensorMap& ma, const CUtensorMap& mb0, const CUtensorMap& mb1, const CUtensorMap& my,
                       const TcParams& p, cudaStream_t s) {
    using C = Cfg<BN, BKIND, CG>;
    auto kern = tc_gemm_kernel<BN, BKIND, CG>;
    static bool attr_set = false;  // benign race: the same value may be set twice
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    const int64_t tiles = p.entries * int64_t(p.m_tiles) * p.n_tiles;
    const int64_t slots = num_sms() / CG;
    const int grid = int((tiles < slots ? tiles : slots) * CG);
    return launch_pdl(kern, dim3(grid), dim3(NT), size_t(C::SMEM), s, CG, ma, mb0, mb1, my, p);
}

template <int BN, int CG>
cudaError_t launch_bn(int bkind, const CUtensorMap& ma, const CUtensorMap& mb0, const CUtensorMap& mb1,
                      const CUtensorMap& my, const TcParams& p, cudaStream_t s) {
    if (bkind == B_BINARY) return launch_cfg<BN, B_BINARY, CG>(ma, mb0, mb1, my, p, s);
    if (bkind == B_BOOL) return launch_cfg<BN, B_BOOL, CG>(ma, mb0, mb1, my, p, s);
    return launch_cfg<BN, B_TERNARY, CG>(ma, mb0, mb1, my, p, s);
}

}  // namespace

size_t matmul_tc_workspace(const MatmulArgs& a) {
    const Plan pl = make_plan(a);
    const size_t kp = size_t(kw4_of(a.K)) * 32;
    return round1k(size_t(a.nb * a.nh) * pl.Mk * kp);
}

bool matmul_tc_supported(const MatmulArgs& a) {
    if (a.K < 1 || a.M < 1 || a.N < 1) return false;
    if (a.nb * a.nh > 65535 || a.nb > (int64_t(1) << 31) || a.nh > (int64_t(1) << 31)) return false;
    if (a.M > (int64_t(1) << 31) || a.N > (int64_t(1) << 31)) return false;
    if (a.K > (int64_t(1) << 18)) return false;  // 4096 * |dot| must fit the s32 accumulator
    // the bit planes of kernel-B are read by TMA: batch strides must be real strides
    const Plan pl = make_plan(a);
    if ((a.nb > 1 && pl.b_bs <= 0) || (a.nh > 1 && pl.b_hs <= 0)) return false;
    return encode_fn() != nullptr;
}

cudaError_t launch_matmul_tc(const MatmulArgs& a, void* ws, size_t ws_bytes, cudaStream_t s) {
    const int64_t entries = a.nb * a.nh;
    const int64_t kw4 = kw4_of(a.K);
    const int64_t kp = kw4 * 32;
    const Plan pl = make_plan(a);
    if (ws_bytes < matmul_tc_workspace(a)) return cudaErrorInvalidValue;
    int8_t* wa = reinterpret_cast<int8_t*>(ws);

    // 1) expand kernel-A planes to an int8 image [entries][Mk][Kp]
    ExpandArgs ea{pl.a_sgn, pl.a_nz, pl.Mk, a.K, pl.lda, pl.a_bs, pl.a_hs, a.nh, entries, kw4, wa, {}, {}, {}};
    {
        const int64_t work = entries * pl.Mk * kw4;
        const int64_t blocks = (work + 255) / 256;
        const int grid = int(blocks > num_sms() * 8 ? num_sms() * 8 : blocks);
        const bool small = work + int64_t(grid) * 256 < (int64_t(1) << 31);
        ea.div_kw4 = make_fastdiv(uint32_t(small ? kw4 : 1));
        ea.div_rows = make_fastdiv(uint32_t(small ? pl.Mk : 1));
        ea.div_nh = make_fastdiv(uint32_t(small ? a.nh : 1));
        cudaError_t err = small ? launch_pdl(expand_kernel<uint32_t>, grid, 256, 0, s, 1, ea)
                                : launch_pdl(expand_kernel<uint64_t>, grid, 256, 0, s, 1, ea);
        if (err != cudaSuccess) return err;
    }

    // 2) tensor maps.  CTA pairs (cta_group::2, M = 256) whenever kernel-A has
    //    more than one 128-row block and kernel-B fills a 256-wide tile.
    const int bn = pick_bn(pl.Nk);
    const int cg = (pl.Mk > BM && bn == 256) ? 2 : 1;
    CUtensorMap ma, mb0, mb1, my;
    {
        const uint64_t dims[3] = {uint64_t(kp), uint64_t(pl.Mk), uint64_t(entries)};
        const uint64_t str[2] = {uint64_t(kp), uint64_t(kp) * pl.Mk};
        const uint32_t box[3] = {uint32_t(BK), uint32_t(BM), 1};
        if (!encode(&ma, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, wa, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B))
            return cudaErrorInvalidValue;
    }
    {
        const uint64_t row_b = uint64_t(pl.ldb) * 4;
        const uint64_t dims[4] = {uint64_t(pl.ldb), uint64_t(pl.Nk), uint64_t(a.nh), uint64_t(a.nb)};
        const uint64_t hsb = bstride(a.nh, pl.b_hs * 4, row_b * pl.Nk);
        const uint64_t str[3] = {row_b, hsb, bstride(a.nb, pl.b_bs * 4, hsb * a.nh)};
        const uint32_t box[4] = {4, uint32_t(bn / cg), 1, 1};
        const uint32_t* p0 = pl.bkind == B_BOOL ? pl.b_nz : pl.b_sgn;
        const uint32_t* p1 = pl.bkind == B_TERNARY ? pl.b_nz : p0;
        if (!encode(&mb0, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, const_cast<uint32_t*>(p0), dims, str, box,
                    CU_TENSOR_MAP_SWIZZLE_NONE) ||
            !encode(&mb1, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, const_cast<uint32_t*>(p1), dims, str, box,
                    CU_TENSOR_MAP_SWIZZLE_NONE))
            return cudaErrorInvalidValue;
    }
    TcParams p{};
    p.M = pl.Mk;
    p.N = pl.Nk;
    p.num_kb = int(kp / BK);
    p.entries = entries;
    p.nh = a.nh;
    p.m_tiles = int((pl.Mk + BM * cg - 1) / (BM * cg));
    p.n_tiles = int((pl.Nk + bn - 1) / bn);
    p.y = a.y;
    p.y_dt = a.y_dt;
    p.ldy = a.ldy;
    p.y_bs = a.y_bs;
    p.y_hs = a.y_hs;
    p.out_trans = (pl.swap ? 1 : 0) ^ (a.y_trans ? 1 : 0);
    p.scale = a.col_scale;
    p.scale_on_rows = pl.swap ? 1 : 0;
    p.scalar = a.scalar;
    // output tensor map (TMA store) when the layout allows it
    {
        const int es = (a.y_dt == DT_F16 || a.y_dt == DT_BF16) ? 2 : 4;
        const uint64_t ldb_ = uint64_t(a.ldy) * es;
        const int64_t inner = p.out_trans ? pl.Mk : pl.Nk, outer = p.out_trans ? pl.Nk : pl.Mk;
        const uint64_t hsb = bstride(a.nh, a.y_hs * es, ldb_ * outer);
        const uint64_t bsb = bstride(a.nb, a.y_bs * es, hsb * a.nh);
        bool ok = (reinterpret_cast<uintptr_t>(a.y) % 16 == 0) && ldb_ % 16 == 0 && hsb % 16 == 0 && bsb % 16 == 0 &&
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
        if (!ok) my = ma;  // unused
    }
    if (bn == 256 && cg == 2) return launch_bn<256, 2>(pl.bkind, ma, mb0, mb1, my, p, s);
    if (bn == 256) return launch_bn<256, 1>(pl.bkind, ma, mb0, mb1, my, p, s);
    if (bn == 128) return launch_bn<128, 1>(pl.bkind, ma, mb0, mb1, my, p, s);
    return launch_bn<64, 1>(pl.bkind, ma, mb0, mb1, my, p, s);
}

}  // namespace bwta
