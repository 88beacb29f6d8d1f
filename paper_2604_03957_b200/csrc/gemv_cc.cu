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
#ifndef GC_CTAS_1
#define GC_CTAS_1 3
#endif
__host__ __device__ constexpr int gc_ctas(int ms) { return ms == 1 ? GC_CTAS_1 : ms <= 2 ? 3 : 2; }
// large rows per warp task: 4 (2 for a ternary large side); GC_RW_BIN for a binary large side and
// <= 2 small rows (more weight bytes in flight per warp)
#ifndef GC_RW_BIN
#define GC_RW_BIN 4
#endif
__host__ __device__ constexpr int gc_rw(int ms, bool l_nz) { return l_nz ? 2 : (ms <= 2 ? GC_RW_BIN : 4); }

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
    // fused activation pack (the paper's in-kernel bitpack): the small side given as
    // values [S rows x K] (f16 / bf16 / f32, row stride ld_sx elements), quantized by every CTA
    // into shared-memory planes before the main loop (q = +1 iff x >= s_tp, -1 iff x <= s_ntn; R1-R3)
    FastDiv div_tpe, div_nh;  // tasks per entry, heads (32-bit task indices: host checks total < 2^31)
    const void* sx;
    int sx_dt, s_kind;
    int64_t ld_sx, K;
    float s_tp, s_ntn;
};

__device__ __forceinline__ uint4 ldg_nc4(const uint32_t* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ uint32_t fdiv32(uint32_t n, const FastDiv& f) { return (__umulhi(n, f.mul) + n) >> f.shift; }
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
__device__ __forceinline__ float sx_value(const GcParams& p, int64_t i) {
    if (p.sx_dt == DT_F16) return __half2float(reinterpret_cast<const __half*>(p.sx)[i]);
    if (p.sx_dt == DT_BF16) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p.sx)[i]);
    return reinterpret_cast<const float*>(p.sx)[i];
}

template <int MS, int LP, int SP, bool SQ = false>
__global__ void __launch_bounds__(GC_NT, gc_ctas(MS)) cc_gemv_kernel(GcParams p) {
    constexpr bool L_SGN = LP & 1, L_NZ = LP & 2, S_SGN = SP & 1, S_NZ = SP & 2;
    constexpr bool HOIST = !L_NZ;  // m = nz_small: popc(m) summed once per small row
    // rows per task: enough to reuse the small side's L1 loads, few enough for two iterations of
    // large-side loads in registers
    constexpr int RW = gc_rw(MS, L_NZ);
    constexpr int NV = RW * MS;
    pdl_launch_dependents();
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int64_t gw = (int64_t(blockIdx.x) * GC_NT + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * GC_NT) >> 5;
    const int64_t tasks_per_entry = (p.L + RW - 1) / RW;
    const int64_t total = p.entries * tasks_per_entry;
    const int nqi = (p.nq + 31) / 32;  // warp-uniform quad iterations
    extern __shared__ uint4 gc_smem[];  // SQ: small-side planes [MS][4 nq] sgn, then nz
    uint32_t* sp_sgn = reinterpret_cast<uint32_t*>(gc_smem);
    uint32_t* sp_nz = sp_sgn + MS * 4 * p.nq;
    if (SQ) {  // quantize + pack the small side once per CTA (single entry)
        {   // first, start the HBM -> L2 stream of this warp's first task (it overlaps the pack)
            const int64_t task = gw;
            if (task < total) {
                const int64_t r0 = task * RW;
                for (int r = 0; r < RW; ++r)
                    if (r0 + r < p.L)
                        for (int q = lane; q < p.nq; q += 32)
                            asm volatile("prefetch.global.L2 [%0];" ::"l"(p.l_sgn + (r0 + r) * p.ldl + 4 * q));
            }
        }
        const int64_t ldw = 4 * int64_t(p.nq);
        const int es = p.sx_dt == DT_F32 ? 4 : 2;
        const bool vec = (reinterpret_cast<uintptr_t>(p.sx) % 16 == 0) && ((p.ld_sx * es) % 16 == 0);
        for (int64_t idx = threadIdx.x; idx < MS * ldw; idx += GC_NT) {
            const int m = int(idx / ldw);
            const int64_t w = idx - m * ldw;
            uint32_t pos = 0, neg = 0;
            if (m < p.S && 32 * w < p.K) {
                const int64_t base = m * p.ld_sx + 32 * w;
                if (vec && es == 2 && 32 * w + 32 <= p.K) {  // 4 x 16-byte loads, 8 values each
                    const uint4* src = reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(p.sx) + base);
                    uint4 v[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) v[u] = __ldg(src + u);
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const uint32_t h[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const uint16_t bits = uint16_t(h[i >> 1] >> (16 * (i & 1)));
                            const float x = p.sx_dt == DT_F16 ? __half2float(__ushort_as_half(bits))
                                                              : __uint_as_float(uint32_t(bits) << 16);
                            pos |= uint32_t(x >= p.s_tp) << (8 * u + i);
                            neg |= uint32_t(x <= p.s_ntn) << (8 * u + i);
                        }
                    }
                } else {
                    for (int i = 0; i < 32; ++i) {
                        const int64_t c = 32 * w + i;
                        if (c < p.K) {
                            const float x = sx_value(p, base + i);
                            pos |= uint32_t(x >= p.s_tp) << i;
                            neg |= uint32_t(x <= p.s_ntn) << i;
                        }
                    }
                }
            }
            sp_nz[idx] = p.s_kind == K_TERNARY ? (pos | neg) : pos;
            sp_sgn[idx] = p.s_kind == K_TERNARY ? neg : 0u;
        }
        __syncthreads();
    }
    // The warp's work is a stream of (task, quad iteration) steps; the large-side loads of the next
    // step -- possibly the next task's first -- are issued before the current step is counted, so
    // the weight stream never waits on a task's reduction and store (a warp's last task no longer
    // costs a full DRAM round trip of its own).
    struct Pos {
        int64_t r0, eb, eh;
    };
    auto pos_of = [&](int64_t task) {  // task -> (first large row, batch, head) without 64-bit divisions
        const uint32_t t = uint32_t(task);
        const uint32_t e = fdiv32(t, p.div_tpe);
        const uint32_t eb = fdiv32(e, p.div_nh);
        return Pos{int64_t(t - e * p.div_tpe.d) * RW, int64_t(eb), int64_t(e - eb * p.div_nh.d)};
    };
    auto large_ptrs = [&](const Pos& ps, const uint32_t* (&lsg)[RW], const uint32_t* (&lnz)[RW]) {
        const int64_t r0 = ps.r0;
        const int64_t loff = ps.eb * p.l_bs + ps.eh * p.l_hs;
#pragma unroll
        for (int r = 0; r < RW; ++r) {
            const int64_t o = loff + (r0 + r < p.L ? r0 + r : r0) * p.ldl;
            lsg[r] = L_SGN ? p.l_sgn + o : nullptr;
            lnz[r] = L_NZ ? p.l_nz + o : nullptr;
        }
    };
    auto load_large = [&](const Pos& ps, int qi, uint4 (&s_)[RW], uint4 (&n_)[RW]) {
        const uint32_t* lsg[RW];
        const uint32_t* lnz[RW];
        large_ptrs(ps, lsg, lnz);
        const int64_t r0 = ps.r0;
        const int q = qi * 32 + lane;
        const bool qok = q < p.nq;
#pragma unroll
        for (int r = 0; r < RW; ++r) {
            const bool ok = qok && r0 + r < p.L;
            s_[r] = L_SGN && ok ? ldg_nc4(lsg[r] + 4 * q) : make_uint4(0, 0, 0, 0);
            n_[r] = L_NZ && ok ? ldg_nc4(lnz[r] + 4 * q) : make_uint4(0, 0, 0, 0);
        }
    };
    int64_t task = gw;
    int qi = 0;
    uint4 ls[RW], ln[RW];
    Pos cur = pos_of(task < total ? task : 0);
    if (task < total) load_large(cur, 0, ls, ln);
    int32_t cneg[NV], cpos[HOIST ? MS : NV];  // popc(m & (sgn ^ sgn)), popc(m)
#pragma unroll
    for (int i = 0; i < NV; ++i) cneg[i] = 0;
#pragma unroll
    for (int i = 0; i < (HOIST ? MS : NV); ++i) cpos[i] = 0;
    while (task < total) {
        // the next step, and its loads in flight
        const bool last_q = qi + 1 >= nqi;
        const int64_t ntask = last_q ? task + nwarps : task;
        const int nqi_ = last_q ? 0 : qi + 1;
        uint4 lsn[RW], lnn[RW];
        const Pos nxt = last_q ? pos_of(ntask < total ? ntask : task) : cur;
        if (ntask < total) load_large(nxt, nqi_, lsn, lnn);
        const int64_t r0 = cur.r0, eb = cur.eb, eh = cur.eh;
        const int64_t soff = eb * p.s_bs + eh * p.s_hs;
        const int q = qi * 32 + lane;
        const bool qok = q < p.nq;
        // small side quads (the same for every large row of the task; L1-resident)
        uint4 ss[MS], sn[MS];
#pragma unroll
        for (int m = 0; m < MS; ++m) {
            const bool ok = qok && m < p.S;
            if (SQ) {
                const int64_t o = int64_t(m) * 4 * p.nq + 4 * q;
                ss[m] = ok ? *reinterpret_cast<const uint4*>(sp_sgn + o) : make_uint4(0, 0, 0, 0);
                sn[m] = ok ? *reinterpret_cast<const uint4*>(sp_nz + o) : make_uint4(0, 0, 0, 0);
            } else {
                const int64_t o = soff + int64_t(m < p.S ? m : 0) * p.lds + 4 * q;
                ss[m] = S_SGN && ok ? ldg4(p.s_sgn + o) : make_uint4(0, 0, 0, 0);
                sn[m] = !ok ? make_uint4(0, 0, 0, 0) : S_NZ ? ldg4(p.s_nz + o) : make_uint4(~0u, ~0u, ~0u, ~0u);
            }
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
        if (last_q) {
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
#pragma unroll
            for (int i = 0; i < NV; ++i) cneg[i] = 0;
#pragma unroll
            for (int i = 0; i < (HOIST ? MS : NV); ++i) cpos[i] = 0;
        }
#pragma unroll
        for (int r = 0; r < RW; ++r) {
            ls[r] = lsn[r];
            ln[r] = lnn[r];
        }
        task = ntask;
        qi = nqi_;
        cur = nxt;
    }
}


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

template <int MS>
cudaError_t launch_sq(const GcParams& p, int grid, cudaStream_t s) {
    const size_t smem = sizeof(uint32_t) * 2 * MS * 4 * size_t(p.nq);
    auto k = p.s_kind == K_TERNARY ? cc_gemv_kernel<MS, 1, 3, true> : cc_gemv_kernel<MS, 1, 2, true>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return e;
    }
    return launch_pdl(k, dim3(grid), dim3(GC_NT), smem, s, 1, p);
}

}  // namespace

// Y = bwta_gemm(bwta_pack_act(x), W) for <= 4 activation rows with the pack fused (one launch):
// x [m x k] values (row stride ld_x elements), binary W [n x ldw]; Y [m x n] (or Y^T).
cudaError_t launch_gemv_cc_fused(const void* x, int x_dt, int64_t ld_x, float tp, float ntn, int a_kind,
                                 const MatmulArgs& a, cudaStream_t s) {
    GcParams p{};
    p.l_sgn = a.b_sgn;
    p.l_nz = nullptr;
    p.L = a.N;
    p.S = a.M;
    p.ldl = a.ldb;
    p.nh = 1;
    p.entries = 1;
    p.nq = int(((a.K + 31) / 32 + 3) / 4);
    p.y = a.y;
    p.y_dt = a.y_dt;
    const int64_t si = a.y_trans ? 1 : a.ldy, sj = a.y_trans ? a.ldy : 1;
    p.y_rs = sj;  // large side = the caller's N
    p.y_cs = si;
    p.scale = a.col_scale;
    p.scale_on_rows = 1;
    p.scalar = a.scalar;
    p.sx = x;
    p.sx_dt = x_dt;
    p.s_kind = a_kind;
    p.ld_sx = ld_x;
    p.K = a.K;
    p.s_tp = tp;
    p.s_ntn = ntn;
    const int g_sms = device_sms();
    const int ms = p.S == 1 ? 1 : (p.S == 2 ? 2 : 4);
    if ((p.L + gc_rw(ms, false) - 1) / gc_rw(ms, false) >= (int64_t(1) << 31)) return cudaErrorInvalidValue;
    p.div_tpe = make_fastdiv(uint32_t((p.L + gc_rw(ms, false) - 1) / gc_rw(ms, false)));
    p.div_nh = make_fastdiv(1);
    int64_t grid = (p.L + gc_rw(ms, false) - 1) / gc_rw(ms, false) / (GC_NT / 32) + 1;
    if (grid > int64_t(g_sms) * gc_ctas(ms)) grid = int64_t(g_sms) * gc_ctas(ms);
    if (ms == 1) return launch_sq<1>(p, int(grid), s);
    if (ms == 2) return launch_sq<2>(p, int(grid), s);
    return launch_sq<4>(p, int(grid), s);
}

bool matmul_gemv_cc_eligible(const MatmulArgs& a) {
    const int64_t small = a.M < a.N ? a.M : a.N;
    if (small < 1 || small > 4 || a.pack_out) return false;
    if (!a.a_nz && !a.b_nz) return false;  // one side carries the nz plane (activations always do)
    const int64_t large = a.M < a.N ? a.N : a.M;
    if (a.nb * a.nh * ((large + 1) / 2) >= (int64_t(1) << 31)) return false;  // 32-bit task indices
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
    const int g_sms = device_sms();
    const int ms = p.S == 1 ? 1 : (p.S == 2 ? 2 : 4);
    const int rw = gc_rw(ms, p.l_nz != nullptr);
    const int64_t warps = p.entries * ((p.L + rw - 1) / rw);
    if (warps >= (int64_t(1) << 31) || p.nh >= (int64_t(1) << 31)) return cudaErrorInvalidValue;
    p.div_tpe = make_fastdiv(uint32_t((p.L + rw - 1) / rw));
    p.div_nh = make_fastdiv(uint32_t(p.nh));
    int64_t grid = (warps + GC_NT / 32 - 1) / (GC_NT / 32);
    if (grid > int64_t(g_sms) * gc_ctas(ms)) grid = int64_t(g_sms) * gc_ctas(ms);
    if (p.S == 1) return launch_l<1>(lp, sp, p, int(grid), s);
    if (p.S == 2) return launch_l<2>(lp, sp, p, int(grid), s);
    return launch_l<4>(lp, sp, p, int(grid), s);
}

}  // namespace bwta
