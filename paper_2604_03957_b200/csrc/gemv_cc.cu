// gemv_cc.cu -- design (a) for decode-sized products: the smaller side has at
// most 4 rows (M = 1..4 tokens against a weight matrix, or one query row
// against a head's K / V^T planes).
//
// The large operand is streamed once at HBM rate; each 32-element word of it
// meets every small-side row with the paper's bit-serial identities (
// R10): with m = nz_small & nz_large (nz = all-ones for a binary operand),
//     dot += popc(m) - 2 popc(m & (sgn_small ^ sgn_large))
// and for a binary large operand the first term is hoisted (popc(nz_small) per
// row, counted once).  At <= 4 small rows this is 1-8 LOP3 + POPC per word,
// below the HBM byte rate of the tensor path's floor (the skinny tcgen05
// kernel is bound by ~100 cycles per tcgen05.mma instruction at N <= 128,
// tools/ubench/mxf4_ubench.cu), so CUDA cores win here.
//
// Warp task = RW consecutive large-side rows (4, halved when the large side is
// ternary); the loads of the next 32-quad iteration are in flight
// while the current one is counted.  Lane l owns word quads
// q = l, l + 32, ... (16-byte loads, coalesced 512 B per warp and row); for
// each quad it loads the small side's quad once (L1-resident, reused across
// the RW rows) and the RW large-side quads (RW independent 16-byte loads in
// flight).  The RW x MS partial counts are summed over the warp by recursive
// halving (NV - 1 + few shuffles for NV values).  Epilogue R5: c = fl32(scale * scalar), y = fl32(dot * c).
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "bwta_internal.h"

namespace bwta {
namespace {

constexpr int GC_NT = 256;    // 8 warps per CTA
// CTAs per SM: 3 (<= 85 registers) for 1-2 small rows -- more warps in flight and an even
// spread of the 4-row tasks -- and 2 (<= 128 registers) for 3-4 rows
__host__ __device__ constexpr int gc_ctas(int ms) { return ms <= 2 ? 3 : 2; }

struct GcParams {
    const uint32_t *l_sgn, *l_nz;  // large side (kernel rows): null plane = absent
    const uint32_t *s_sgn, *s_nz;  // small side (<= MS rows)
    int64_t L, S;                  // rows of each side per entry
    int64_t ldl, lds;              // words
    int64_t l_bs, l_hs, s_bs, s_hs;
    int64_t nh, entries;
    int nq;                        // word quads per row (ceil(ceil(K/32) / 4))
    void* y;
    int y_dt;
    int64_t y_rs, y_cs, y_bs, y_hs;  // element strides: large row, small row, batch, head
    const float* scale;              // caller's per-N scale (large rows if scale_on_rows)
    int scale_on_rows;
    float scalar;
};

__device__ __forceinline__ uint4 ldg_nc4(const uint32_t* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ uint4 ldg4(const uint32_t* p) { return __ldg(reinterpret_cast<const uint4*>(p)); }
__device__ __forceinline__ uint32_t w_of(const uint4& v, int i) { return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w; }

// Sum NV (a power of two <= 32) per-lane values over the warp with NV - 1 + (5 - log2 NV)
// shuffles (recursive halving): afterwards lane l holds the total of value l >> (5 - log2 NV).
template <int NV>
__device__ __forceinline__ int32_t warp_reduce_many(int32_t (&v)[NV], int lane) {
    int n = NV;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        if (n > 1) {
            const bool upper = lane & o;
#pragma unroll
            for (int i = 0; i < NV / 2; ++i) {
                if (i < n / 2) {
                    const int32_t send = upper ? v[i] : v[i + n / 2];
                    const int32_t keep = upper ? v[i + n / 2] : v[i];
                    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                }
            }
            n >>= 1;
        } else {
            v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
        }
    }
    return v[0];
}

__host__ __device__ constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x / 2); }

// LP / SP: large / small plane presence (bit 0 sgn, bit 1 nz); RW large rows per warp task
template <int MS, int LP, int SP>
__global__ void __launch_bounds__(GC_NT, gc_ctas(MS)) cc_gemv_kernel(GcParams p) {
    constexpr bool L_SGN = LP & 1, L_NZ = LP & 2, S_SGN = SP & 1, S_NZ = SP & 2;
    constexpr bool HOIST = !L_NZ;  // m = nz_small: popc(m) summed once per small row
    // rows per task: enough to reuse the small side's L1 loads, few enough for two iterations of
    // large-side loads in registers
    constexpr int RW = 4 / (L_NZ ? 2 : 1);
    constexpr int NV = RW * MS;
    pdl_launch_dependents();
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int64_t gw = (int64_t(blockIdx.x) * GC_NT + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * GC_NT) >> 5;
    const int64_t tasks_per_entry = (p.L + RW - 1) / RW;
    const int64_t total = p.entries * tasks_per_entry;
    const int nqi = (p.nq + 31) / 32;  // warp-uniform quad iterations
    for (int64_t task = gw; task < total; task += nwarps) {
        const int64_t e = task / tasks_per_entry;
        const int64_t r0 = (task % tasks_per_entry) * RW;
        const int64_t eb = e / p.nh, eh = e % p.nh;
        const int64_t loff = eb * p.l_bs + eh * p.l_hs, soff = eb * p.s_bs + eh * p.s_hs;
        int32_t cneg[NV], cpos[HOIST ? MS : NV];  // popc(m & (sgn ^ sgn)), popc(m)
#pragma unroll
        for (int i = 0; i < NV; ++i) cneg[i] = 0;
#pragma unroll
        for (int i = 0; i < (HOIST ? MS : NV); ++i) cpos[i] = 0;
        const uint32_t* lsg[RW];
        const uint32_t* lnz[RW];
#pragma unroll
        for (int r = 0; r < RW; ++r) {
            const int64_t o = loff + (r0 + r < p.L ? r0 + r : r0) * p.ldl;
            lsg[r] = L_SGN ? p.l_sgn + o : nullptr;
            lnz[r] = L_NZ ? p.l_nz + o : nullptr;
        }
        // large side quads of the RW rows for quad iteration qi (RW x 16 B in flight per plane);
        // the next iteration's loads are issued before the current one is consumed
        uint4 ls[RW], ln[RW];
        auto load_large = [&](int qi, uint4 (&s_)[RW], uint4 (&n_)[RW]) {
            const int q = qi * 32 + lane;
            const bool qok = q < p.nq;
#pragma unroll
            for (int r = 0; r < RW; ++r) {
                const bool ok = qok && r0 + r < p.L;
                s_[r] = L_SGN && ok ? ldg_nc4(lsg[r] + 4 * q) : make_uint4(0, 0, 0, 0);
                n_[r] = L_NZ && ok ? ldg_nc4(lnz[r] + 4 * q) : make_uint4(0, 0, 0, 0);
            }
        };
        load_large(0, ls, ln);
        for (int qi = 0; qi < nqi; ++qi) {
            const int q = qi * 32 + lane;
            const bool qok = q < p.nq;
            uint4 lsn[RW], lnn[RW];
            if (qi + 1 < nqi) load_large(qi + 1, lsn, lnn);
            // small side quads (the same for every large row of the task; L1-resident)
            uint4 ss[MS], sn[MS];
#pragma unroll
            for (int m = 0; m < MS; ++m) {
                const bool ok = qok && m < p.S;
                const int64_t o = soff + int64_t(m < p.S ? m : 0) * p.lds + 4 * q;
                ss[m] = S_SGN && ok ? ldg4(p.s_sgn + o) : make_uint4(0, 0, 0, 0);
                sn[m] = !ok ? make_uint4(0, 0, 0, 0) : S_NZ ? ldg4(p.s_nz + o) : make_uint4(~0u, ~0u, ~0u, ~0u);
            }
            if (HOIST) {
#pragma unroll
                for (int m = 0; m < MS; ++m)
#pragma unroll
                    for (int i = 0; i < 4; ++i) cpos[m] += __popc(w_of(sn[m], i));
            }
#pragma unroll
            for (int r = 0; r < RW; ++r)
#pragma unroll
                for (int m = 0; m < MS; ++m)
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const uint32_t mm = HOIST ? w_of(sn[m], i) : (w_of(sn[m], i) & w_of(ln[r], i));
                        cneg[r * MS + m] += __popc(mm & (w_of(ss[m], i) ^ w_of(ls[r], i)));
                        if (!HOIST) cpos[r * MS + m] += __popc(mm);
                    }
            if (qi + 1 < nqi) {
#pragma unroll
                for (int r = 0; r < RW; ++r) {
                    ls[r] = lsn[r];
                    ln[r] = lnn[r];
                }
            }
        }
        int32_t v[NV];
#pragma unroll
        for (int i = 0; i < NV; ++i) v[i] = (HOIST ? cpos[i % MS] : cpos[i]) - 2 * cneg[i];
        const int32_t mine = warp_reduce_many<NV>(v, lane);
        constexpr int SH = 5 - ilog2(NV);
        if ((lane & ((1 << SH) - 1)) == 0) {
            const int idx = lane >> SH, r = idx / MS, m = idx % MS;
            const int64_t row = r0 + r;
            if (row < p.L && m < p.S) {
                const int64_t off = eb * p.y_bs + eh * p.y_hs + row * p.y_rs + int64_t(m) * p.y_cs;
                if (p.y_dt == DT_I32) {
                    reinterpret_cast<int32_t*>(p.y)[off] = mine;
                } else {
                    const float c = p.scale ? __fmul_rn(__ldg(p.scale + (p.scale_on_rows ? row : m)), p.scalar)
                                            : p.scalar;
                    const float f = __fmul_rn(float(mine), c);  // exact int -> f32 (|dot| <= 2^24), R5
                    if (p.y_dt == DT_F16) reinterpret_cast<__half*>(p.y)[off] = __float2half_rn(f);
                    else if (p.y_dt == DT_BF16) reinterpret_cast<__nv_bfloat16*>(p.y)[off] = __float2bfloat16_rn(f);
                    else reinterpret_cast<float*>(p.y)[off] = f;
                }
            }
        }
    }
}

int g_sms = 0;

template <int MS, int LP>
cudaError_t launch_s(int sp, const GcParams& p, int grid, cudaStream_t s) {
    if (sp == 3) return launch_pdl(cc_gemv_kernel<MS, LP, 3>, dim3(grid), dim3(GC_NT), 0, s, 1, p);
    if (sp == 2) return launch_pdl(cc_gemv_kernel<MS, LP, 2>, dim3(grid), dim3(GC_NT), 0, s, 1, p);
    return launch_pdl(cc_gemv_kernel<MS, LP, 1>, dim3(grid), dim3(GC_NT), 0, s, 1, p);
}
template <int MS>
cudaError_t launch_l(int lp, int sp, const GcParams& p, int grid, cudaStream_t s) {
    if (lp == 3) return launch_s<MS, 3>(sp, p, grid, s);
    if (lp == 2) return launch_s<MS, 2>(sp, p, grid, s);
    return launch_s<MS, 1>(sp, p, grid, s);
}

}  // namespace

bool matmul_gemv_cc_eligible(const MatmulArgs& a) {
    const int64_t small = a.M < a.N ? a.M : a.N;
    if (small < 1 || small > 4 || a.pack_out) return false;
    if (!a.a_nz && !a.b_nz) return false;  // one side carries the nz plane (activations always do)
    // 16-byte word-quad loads: 16-byte aligned planes, leading dims and strides
    auto al = [](const uint32_t* q) { return q == nullptr || (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
    if (!al(a.a_sgn) || !al(a.a_nz) || !al(a.b_sgn) || !al(a.b_nz)) return false;
    if ((a.lda | a.ldb) & 3) return false;
    if ((a.nb > 1 && ((a.a_bs | a.b_bs) & 3)) || (a.nh > 1 && ((a.a_hs | a.b_hs) & 3))) return false;
    return true;
}

cudaError_t launch_matmul_gemv_cc(const MatmulArgs& a, cudaStream_t s) {
    const bool swap = a.M < a.N;  // large side = the caller's W / K / V^T rows
    GcParams p{};
    p.l_sgn = swap ? a.b_sgn : a.a_sgn;
    p.l_nz = swap ? a.b_nz : a.a_nz;
    p.s_sgn = swap ? a.a_sgn : a.b_sgn;
    p.s_nz = swap ? a.a_nz : a.b_nz;
    p.L = swap ? a.N : a.M;
    p.S = swap ? a.M : a.N;
    p.ldl = swap ? a.ldb : a.lda;
    p.lds = swap ? a.lda : a.ldb;
    p.l_bs = swap ? a.b_bs : a.a_bs;
    p.l_hs = swap ? a.b_hs : a.a_hs;
    p.s_bs = swap ? a.a_bs : a.b_bs;
    p.s_hs = swap ? a.a_hs : a.b_hs;
    p.nh = a.nh;
    p.entries = a.nb * a.nh;
    p.nq = int(((a.K + 31) / 32 + 3) / 4);
    p.y = a.y;
    p.y_dt = a.y_dt;
    const int64_t si = a.y_trans ? 1 : a.ldy, sj = a.y_trans ? a.ldy : 1;  // caller's Y[i][j]
    p.y_rs = swap ? sj : si;
    p.y_cs = swap ? si : sj;
    p.y_bs = a.y_bs;
    p.y_hs = a.y_hs;
    p.scale = a.col_scale;
    p.scale_on_rows = swap ? 1 : 0;
    p.scalar = a.scalar;
    const int lp = (p.l_sgn ? 1 : 0) | (p.l_nz ? 2 : 0), sp = (p.s_sgn ? 1 : 0) | (p.s_nz ? 2 : 0);
    if (g_sms == 0) {
        int dev = 0, v = 148;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) v = 148;
        g_sms = v;
    }
    const int64_t warps = p.entries * ((p.L + 3) / 4);
    int64_t grid = (warps + GC_NT / 32 - 1) / (GC_NT / 32);
    const int ms = p.S == 1 ? 1 : (p.S == 2 ? 2 : 4);
    if (grid > int64_t(g_sms) * gc_ctas(ms)) grid = int64_t(g_sms) * gc_ctas(ms);
    if (p.S == 1) return launch_l<1>(lp, sp, p, int(grid), s);
    if (p.S == 2) return launch_l<2>(lp, sp, p, int(grid), s);
    return launch_l<4>(lp, sp, p, int(grid), s);
}

}  // namespace bwta
