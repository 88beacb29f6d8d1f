// pack.cu -- activation / weight quantize + bit-pack kernels for sm_100a.
//
// What is computed (include/bwta.h; P:911-930 Eq. bool/ternary, P:901-909
// Eq. sign): per element a code q, packed LSB-first into uint32 planes
// nz (q != 0) and sgn (q < 0).
//
// B200 design (not the paper's in-register IPB, which fuses the
// pack into its MMA kernel): packing is a standalone HBM-streaming pass.
//   * Row mode: one warp reads 32 x 16 B fully-coalesced vectors per
//     "segment" (256 f16 / 128 f32 elements), SEGS segments in flight per
//     warp.  Each lane turns its 16 B into an E-bit chunk with packed-half
//     compares (HSET2 via __hge2_mask: 2 elements per instruction, exact,
//     no division), and 4 (f16/bf16) or 8 (f32) lanes OR their chunks into
//     one word with warp shuffles.
//   * Transposed mode (V^T for PV): a warp owns a 128-row x 32-col tile;
//     lane l packs row l of a 32-row group into a 32-bit word, and a 5-stage
//     shuffle butterfly transposes the 32x32 bit block so lane j ends up with
//     column j's word; 4 row groups give one 16-byte store per column.
// Exactness: x/s >= 0.5 <=> x >= s/2 <=> x >= tp, where tp is the smallest
// value of x's storage type >= s/2 (host-computed, api.cu); x/s < -0.5 <=>
// x <= -tn, tn = smallest storage value > s/2.  Compares of finite, infinite
// and subnormal halves are exact (set.* without .ftz); NaN compares false.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "bwta_internal.h"

namespace bwta {
namespace {

constexpr unsigned FULL = 0xffffffffu;

template <typename T> struct TypeInfo;
template <> struct TypeInfo<__half> { static constexpr int E = 8; };
template <> struct TypeInfo<__nv_bfloat16> { static constexpr int E = 8; };
template <> struct TypeInfo<float> { static constexpr int E = 4; };

// ---- 16-byte chunk -> E compare bits -------------------------------------
// Element 2j of a 32-bit word is its low half, 2j+1 the high half.  The
// selector keeps bit 2j of the low half and bit 17+2j of the high half so a
// final fold (v | v >> 16) yields element bits 0..7.
template <typename H2>
__device__ __forceinline__ void cmp8(const uint4& v, H2 tp, H2 ntn, uint32_t& pos, uint32_t& neg) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t ap = 0, an = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        H2 h = *reinterpret_cast<const H2*>(&w[j]);
        const uint32_t sel = (1u << (2 * j)) | (1u << (17 + 2 * j));
        ap |= __hge2_mask(h, tp) & sel;
        an |= __hle2_mask(h, ntn) & sel;
    }
    pos = (ap | (ap >> 16)) & 0xffu;
    neg = (an | (an >> 16)) & 0xffu;
}

template <typename T>
__device__ __forceinline__ void chunk_bits(const uint4& v, const Thresholds& th, uint32_t& pos, uint32_t& neg);

template <>
__device__ __forceinline__ void chunk_bits<__half>(const uint4& v, const Thresholds& th, uint32_t& pos, uint32_t& neg) {
    cmp8<__half2>(v, *reinterpret_cast<const __half2*>(&th.tp2), *reinterpret_cast<const __half2*>(&th.ntn2), pos, neg);
}
template <>
__device__ __forceinline__ void chunk_bits<__nv_bfloat16>(const uint4& v, const Thresholds& th, uint32_t& pos, uint32_t& neg) {
    cmp8<__nv_bfloat162>(v, *reinterpret_cast<const __nv_bfloat162*>(&th.tp2),
                         *reinterpret_cast<const __nv_bfloat162*>(&th.ntn2), pos, neg);
}
template <>
__device__ __forceinline__ void chunk_bits<float>(const uint4& v, const Thresholds& th, uint32_t& pos, uint32_t& neg) {
    const float f[4] = {__uint_as_float(v.x), __uint_as_float(v.y), __uint_as_float(v.z), __uint_as_float(v.w)};
    uint32_t p = 0, n = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        p |= (f[j] >= th.tpf ? 1u : 0u) << j;
        n |= (f[j] <= th.ntnf ? 1u : 0u) << j;
    }
    pos = p;
    neg = n;
}

// Weights: bit = 1 <=> !(w >= mu)  (sign(w - mu) = -1, NaN -> -1), compared in f32.
template <typename T>
__device__ __forceinline__ uint32_t chunk_lt_mu(const uint4& v, float mu);
template <>
__device__ __forceinline__ uint32_t chunk_lt_mu<float>(const uint4& v, float mu) {
    const float f[4] = {__uint_as_float(v.x), __uint_as_float(v.y), __uint_as_float(v.z), __uint_as_float(v.w)};
    uint32_t b = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) b |= (f[j] >= mu ? 0u : 1u) << j;
    return b;
}
template <typename T>
__device__ __forceinline__ float to_f32(T h);
template <> __device__ __forceinline__ float to_f32<__half>(__half h) { return __half2float(h); }
template <> __device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 h) { return __bfloat162float(h); }

template <typename T>
__device__ __forceinline__ uint32_t chunk_lt_mu(const uint4& v, float mu) {
    const T* e = reinterpret_cast<const T*>(&v);
    uint32_t b = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) b |= (to_f32<T>(e[j]) >= mu ? 0u : 1u) << j;
    return b;
}

// Load E elements starting at element `c` of a row (cols valid elements).
// Out-of-range elements read as +0 (which quantizes to 0 for bool/ternary).
template <typename T, bool VEC>
__device__ __forceinline__ uint4 load_chunk(const T* __restrict__ row, int64_t c, int64_t cols) {
    constexpr int E = TypeInfo<T>::E;
    if (VEC && c + E <= cols) {
        uint4 r;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                     : "l"(row + c));
        return r;
    }
    uint4 r = make_uint4(0, 0, 0, 0);
    T* e = reinterpret_cast<T*>(&r);
#pragma unroll
    for (int j = 0; j < E; ++j)
        if (c + j < cols) e[j] = row[c + j];
    return r;
}

__device__ __forceinline__ int64_t entry_off(int64_t e, int64_t nh, int64_t bs, int64_t hs) {
    return (e / nh) * bs + (e % nh) * hs;
}

// ---------------------------------------------------------------------------
// Row mode.  Work item = (entry, row, chunk of SEGS segments).
// ---------------------------------------------------------------------------
constexpr int SEGS = 4;

template <typename T, int KIND, bool VEC>
__global__ void __launch_bounds__(256) pack_rows_kernel(PackArgs p) {
    constexpr int E = TypeInfo<T>::E;     // elements per lane per segment
    constexpr int LPW = 32 / E;           // lanes per output word
    constexpr int WPS = E;                // words per segment
    const int lane = threadIdx.x & 31;
    const int64_t nseg = (p.ldw + WPS - 1) / WPS;
    const int64_t nchunk = (nseg + SEGS - 1) / SEGS;
    const int64_t items = p.nb * p.nh * p.rows * nchunk;
    const int64_t warp0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;

    for (int64_t it = warp0; it < items; it += nwarps) {
        const int64_t chunk = it % nchunk;
        const int64_t rr = it / nchunk;          // entry*rows + row
        const int64_t r = rr % p.rows;
        const int64_t e = rr / p.rows;
        const T* row = reinterpret_cast<const T*>(p.x) + entry_off(e, p.nh, p.x_bs, p.x_hs) + r * p.ld_x;
        const int64_t poff = entry_off(e, p.nh, p.p_bs, p.p_hs) + r * p.ldw;
        float mu = 0.f;
        if (KIND == K_BINARY && p.mu) mu = p.mu_per_row ? p.mu[r] : p.mu[0];

        uint4 v[SEGS];
#pragma unroll
        for (int s = 0; s < SEGS; ++s) {
            const int64_t seg = chunk * SEGS + s;
            const int64_t c = seg * (32 * E) + lane * E;
            v[s] = (seg < nseg) ? load_chunk<T, VEC>(row, c, p.cols) : make_uint4(0, 0, 0, 0);
        }
        uint32_t nnz = 0;
#pragma unroll
        for (int s = 0; s < SEGS; ++s) {
            const int64_t seg = chunk * SEGS + s;
            if (seg >= nseg) break;
            const int64_t c = seg * (32 * E) + lane * E;
            uint32_t pos, neg;
            if (KIND == K_BINARY) {
                // valid-element mask: elements >= cols must stay 0
                const int64_t nvalid = p.cols - c;
                const uint32_t valid = nvalid >= E ? ((1u << E) - 1) : (nvalid <= 0 ? 0u : ((1u << nvalid) - 1));
                neg = chunk_lt_mu<T>(v[s], mu) & valid;
                pos = 0;
            } else {
                chunk_bits<T>(v[s], p.th, pos, neg);
            }
            const int sh = E * (lane % LPW);
            // nz bits: ternary q != 0; bool q = 1 only for x >= t (binary: unused)
            uint32_t wn = (KIND == K_BOOL ? pos : (pos | neg)) << sh;
            uint32_t ws = neg << sh;           // sgn bits
#pragma unroll
            for (int o = 1; o < LPW; o <<= 1) {
                wn |= __shfl_xor_sync(FULL, wn, o);
                ws |= __shfl_xor_sync(FULL, ws, o);
            }
            const int64_t widx = seg * WPS + lane / LPW;
            if ((lane % LPW) == 0 && widx < p.ldw) {
                if (KIND == K_BINARY) {
                    p.sgn[poff + widx] = ws;
                } else {
                    p.nz[poff + widx] = wn;
                    if (KIND == K_TERNARY) p.sgn[poff + widx] = ws;
                    nnz += __popc(wn);
                }
            }
        }
        if (KIND != K_BINARY && p.row_nnz) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) nnz += __shfl_xor_sync(FULL, nnz, o);
            if (lane == 0 && nnz) atomicAdd(p.row_nnz + rr, int(nnz));
        }
    }
}

// ---------------------------------------------------------------------------
// Transposed mode.  Work item = (entry, 128-row tile, 32-col tile).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
    // 32x32 bit-matrix transpose across a warp: in, lane l holds row l
    // (bit c = column c); out, lane c holds column c (bit l = row l).
    const uint32_t masks[5] = {0x0000ffffu, 0x00ff00ffu, 0x0f0f0f0fu, 0x33333333u, 0x55555555u};
#pragma unroll
    for (int st = 0; st < 5; ++st) {
        const int j = 16 >> st;
        const uint32_t m = masks[st];
        const uint32_t o = __shfl_xor_sync(FULL, x, j);
        x = (lane & j) ? ((x & ~m) | ((o & ~m) >> j)) : ((x & m) | ((o & m) << j));
    }
    return x;
}

template <typename T, int KIND, bool VEC>
__global__ void __launch_bounds__(256) pack_cols_kernel(PackArgs p) {
    constexpr int E = TypeInfo<T>::E;
    constexpr int NV = 32 / E;            // 16-byte vectors per 32 columns
    const int lane = threadIdx.x & 31;
    const int64_t ntile_r = p.ldw / 4;    // 128-row tiles (ldw % 4 == 0)
    const int64_t ntile_c = (p.cols + 31) / 32;
    const int64_t items = p.nb * p.nh * ntile_r * ntile_c;
    const int64_t warp0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;

    for (int64_t it = warp0; it < items; it += nwarps) {
        const int64_t tc = it % ntile_c;
        const int64_t t2 = it / ntile_c;
        const int64_t tr = t2 % ntile_r;
        const int64_t e = t2 / ntile_r;
        const T* base = reinterpret_cast<const T*>(p.x) + entry_off(e, p.nh, p.x_bs, p.x_hs);
        const int64_t c0 = tc * 32;
        uint32_t nzw[4], sgw[4];
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            const int64_t r = tr * 128 + g * 32 + lane;
            uint32_t pos = 0, neg = 0;
            if (r < p.rows) {
                const T* row = base + r * p.ld_x;
                uint4 v[NV];
#pragma unroll
                for (int q = 0; q < NV; ++q) v[q] = load_chunk<T, VEC>(row, c0 + q * E, p.cols);
#pragma unroll
                for (int q = 0; q < NV; ++q) {
                    uint32_t pb, nb;
                    chunk_bits<T>(v[q], p.th, pb, nb);
                    pos |= pb << (q * E);
                    neg |= nb << (q * E);
                }
            }
            nzw[g] = transpose32(KIND == K_BOOL ? pos : (pos | neg), lane);
            sgw[g] = (KIND == K_TERNARY) ? transpose32(neg, lane) : 0u;
        }
        const int64_t col = c0 + lane;
        if (col < p.cols) {
            const int64_t poff = entry_off(e, p.nh, p.p_bs, p.p_hs) + col * p.ldw + tr * 4;
            *reinterpret_cast<uint4*>(p.nz + poff) = make_uint4(nzw[0], nzw[1], nzw[2], nzw[3]);
            if (KIND == K_TERNARY)
                *reinterpret_cast<uint4*>(p.sgn + poff) = make_uint4(sgw[0], sgw[1], sgw[2], sgw[3]);
            if (p.row_nnz) {
                const int n = __popc(nzw[0]) + __popc(nzw[1]) + __popc(nzw[2]) + __popc(nzw[3]);
                if (n) atomicAdd(p.row_nnz + e * p.cols + col, n);
            }
        }
    }
}

int grid_for(int64_t warp_items) {
    const int64_t blocks = (warp_items + 7) / 8;
    const int64_t cap = 148 * 16;
    return int(blocks < 1 ? 1 : (blocks > cap ? cap : blocks));
}

template <typename T>
cudaError_t rows_dispatch(const PackArgs& a, cudaStream_t s, int grid) {
#define BWTA_ROWS(KIND)                                                              \
    do {                                                                             \
        if (a.vec_ok) pack_rows_kernel<T, KIND, true><<<grid, 256, 0, s>>>(a);       \
        else pack_rows_kernel<T, KIND, false><<<grid, 256, 0, s>>>(a);               \
    } while (0)
    if (a.kind == K_BINARY) BWTA_ROWS(K_BINARY);
    else if (a.kind == K_BOOL) BWTA_ROWS(K_BOOL);
    else BWTA_ROWS(K_TERNARY);
#undef BWTA_ROWS
    return cudaGetLastError();
}

template <typename T>
cudaError_t cols_dispatch(const PackArgs& a, cudaStream_t s, int grid) {
#define BWTA_COLS(KIND)                                                              \
    do {                                                                             \
        if (a.vec_ok) pack_cols_kernel<T, KIND, true><<<grid, 256, 0, s>>>(a);       \
        else pack_cols_kernel<T, KIND, false><<<grid, 256, 0, s>>>(a);               \
    } while (0)
    if (a.kind == K_BOOL) BWTA_COLS(K_BOOL);
    else BWTA_COLS(K_TERNARY);
#undef BWTA_COLS
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_pack_rows(const PackArgs& a, cudaStream_t s) {
    const int E = (a.dt == DT_F32) ? 4 : 8;
    const int64_t nseg = (a.ldw + E - 1) / E;
    const int64_t items = a.nb * a.nh * a.rows * ((nseg + SEGS - 1) / SEGS);
    if (items == 0) return cudaSuccess;
    if (a.row_nnz && a.kind != K_BINARY) {
        cudaError_t err = cudaMemsetAsync(a.row_nnz, 0, sizeof(int32_t) * a.nb * a.nh * a.rows, s);
        if (err != cudaSuccess) return err;
    }
    const int grid = grid_for(items);
    switch (a.dt) {
        case DT_F16: return rows_dispatch<__half>(a, s, grid);
        case DT_BF16: return rows_dispatch<__nv_bfloat16>(a, s, grid);
        default: return rows_dispatch<float>(a, s, grid);
    }
}

cudaError_t launch_pack_cols(const PackArgs& a, cudaStream_t s) {
    const int64_t items = a.nb * a.nh * (a.ldw / 4) * ((a.cols + 31) / 32);
    if (items == 0) return cudaSuccess;
    if (a.row_nnz) {
        cudaError_t err = cudaMemsetAsync(a.row_nnz, 0, sizeof(int32_t) * a.nb * a.nh * a.cols, s);
        if (err != cudaSuccess) return err;
    }
    const int grid = grid_for(items);
    switch (a.dt) {
        case DT_F16: return cols_dispatch<__half>(a, s, grid);
        case DT_BF16: return cols_dispatch<__nv_bfloat16>(a, s, grid);
        default: return cols_dispatch<float>(a, s, grid);
    }
}

}  // namespace bwta
