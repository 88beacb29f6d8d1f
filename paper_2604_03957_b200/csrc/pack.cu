// pack.cu -- activation / weight quantize + bit-pack kernels for sm_100a.
//
// What is computed (include/bwta.h; P:911-930 Eq. bool/ternary, P:901-909
// Eq. sign): per element a code q, packed LSB-first into uint32 planes
// nz (q != 0) and sgn (q < 0).
//
// B200 design (not the paper's in-register IPB, which fuses the
// pack into its MMA kernel): packing is a standalone HBM-streaming pass.
//   * Row mode: the output words are walked as one flat list; one lane owns
//     one output word and reads its 32 elements as 16-byte vectors (64 B for
//     2-byte inputs), 2 words per lane in flight plus a prefetch of the next
//     pair.  Each 16 B vector becomes 8 compare bits through packed-half
//     compares (HSET2 via __hge2_mask: 2 elements per instruction, exact, no
//     division); no cross-lane traffic, and 32 lanes store 128 contiguous
//     bytes of plane.
//   * Transposed mode (V^T for PV): a warp owns a 32-row x 32-col tile; lane
//     l packs row l into a 32-bit word, a 5-stage shuffle butterfly transposes
//     the 32x32 bit block so lane j ends up with column j's word.
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

// Division by a launch constant: FastDiv on the 32-bit path, plain otherwise.
__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
    return (__umulhi(n, f.mul) + n) >> f.shift;
}
__device__ __forceinline__ uint64_t fdiv(uint64_t n, const FastDiv& f) { return n / f.d; }

// ---------------------------------------------------------------------------
// Row mode: one lane builds one output word.  The planes are walked as a
// flat list of words gw = (entry*rows + row)*ldw + w; lane gw reads the 32
// elements of its word as 16-byte vectors (64 B for 2-byte inputs, L1-
// allocating so the four quarter-line requests of a lane hit the same
// sectors), compares them with packed-half HSET2 and ORs the results into
// the word directly -- no cross-lane traffic; 32 lanes store 128 contiguous
// bytes.  Every lane keeps 2 words in flight and prefetches the next pair
// before computing.  Lanes own data words only (w < ceil(cols/32)); the lane of
// a row's last data word also zeroes its padding words (head_dim 64 rows: 2
// data + 2 padding words -- no lane idles on padding).
// ---------------------------------------------------------------------------
template <typename T> struct WplOf { static constexpr int v = sizeof(T) == 4 ? 1 : 2; };  // words per lane per iteration

// the 8 compare bits of one 16-byte vector, placed at bit offset `sh`
template <typename T>
__device__ __forceinline__ void vec_bits(const uint4& v, const Thresholds& th, int sh, uint32_t& pos, uint32_t& neg) {
    uint32_t pb, nb;
    chunk_bits<T>(v, th, pb, nb);
    pos |= pb << sh;
    neg |= nb << sh;
}

// Body of the row-mode pack for block `vb` of a grid of `vg` blocks (256 threads).
template <typename T, int KIND, bool VEC, typename IDX>
__device__ __forceinline__ void pack_rows_body(const PackArgs& p, unsigned vb, unsigned vg) {
    constexpr int E = TypeInfo<T>::E;  // elements per 16-byte vector
    constexpr int NV = 32 / E;         // vectors per word
    constexpr int WPL = WplOf<T>::v;
    const IDX ldw = IDX(p.ldw), rows = IDX(p.rows), nh = IDX(p.nh), nwd = IDX(p.nwd);
    const IDX total = IDX(p.nb * p.nh) * rows * nwd;  // data words; their lanes also zero the row's padding
    const IDX cols = IDX(p.cols);
    const IDX nthreads = IDX(vg) * blockDim.x;
    const IDX tid = IDX(vb) * blockDim.x + threadIdx.x;

    auto issue = [&](IDX gw0, uint4 (&v)[WplOf<T>::v][NV], IDX (&gr)[WplOf<T>::v], IDX (&gwv)[WplOf<T>::v]) {
#pragma unroll
        for (int u = 0; u < WPL; ++u) {
            const IDX gw = gw0 + IDX(u) * nthreads;
            const IDX r = fdiv(gw < total ? gw : IDX(0), p.div_nwd);  // flat row (entry*rows + row)
            gr[u] = r;
            gwv[u] = gw - r * nwd;
            const IDX c0 = gwv[u] * 32;
#pragma unroll
            for (int q = 0; q < NV; ++q) v[u][q] = make_uint4(0, 0, 0, 0);
            if (gw < total && c0 < cols) {
                const IDX e = fdiv(r, p.div_rows), rr = r - e * rows;
                const IDX eb = fdiv(e, p.div_nh), eh = e - eb * nh;
                const T* row = reinterpret_cast<const T*>(p.x) + int64_t(eb) * p.x_bs + int64_t(eh) * p.x_hs +
                               int64_t(rr) * p.ld_x;
                if (VEC && c0 + 32 <= cols) {
                    const uint4* src = reinterpret_cast<const uint4*>(row + c0);
#pragma unroll
                    for (int q = 0; q < NV; ++q) v[u][q] = __ldg(src + q);
                } else {
#pragma unroll
                    for (int q = 0; q < NV; ++q) v[u][q] = load_chunk<T, false>(row, int64_t(c0) + q * E, int64_t(cols));
                }
            }
        }
    };

    uint4 v[WPL][NV], vn[WPL][NV];
    IDX gr[WPL], gwv[WPL], grn[WPL], gwvn[WPL];
    const IDX step = nthreads * WPL;
    IDX gw0 = tid;
    if (gw0 < total) issue(gw0, vn, grn, gwvn);
    for (; gw0 < total; gw0 += step) {
#pragma unroll
        for (int u = 0; u < WPL; ++u) {
            gr[u] = grn[u];
            gwv[u] = gwvn[u];
#pragma unroll
            for (int q = 0; q < NV; ++q) v[u][q] = vn[u][q];
        }
        if (gw0 + step < total) issue(gw0 + step, vn, grn, gwvn);
#pragma unroll
        for (int u = 0; u < WPL; ++u) {
            const IDX gw = gw0 + IDX(u) * nthreads;
            if (gw >= total) break;
            uint32_t pos = 0, neg = 0;
            if (KIND == K_BINARY) {
                float mu = 0.f;
                if (p.mu) mu = p.mu_per_row ? p.mu[gr[u] - fdiv(gr[u], p.div_rows) * rows] : p.mu[0];
#pragma unroll
                for (int q = 0; q < NV; ++q) neg |= chunk_lt_mu<T>(v[u][q], mu) << (q * E);
                const int64_t nvalid = int64_t(cols) - int64_t(gwv[u]) * 32;
                neg &= nvalid >= 32 ? 0xffffffffu : (nvalid <= 0 ? 0u : ((1u << nvalid) - 1u));
            } else {
#pragma unroll
                for (int q = 0; q < NV; ++q) vec_bits<T>(v[u][q], p.th, q * E, pos, neg);
            }
            const uint32_t wn = KIND == K_BOOL ? pos : (pos | neg);  // nz: ternary q != 0, bool x >= t
            const IDX r = gr[u];
            int64_t poff;
            if (p.planes_dense) {
                poff = int64_t(r) * int64_t(ldw) + int64_t(gwv[u]);
            } else {
                const IDX e = fdiv(r, p.div_rows), rr = r - e * rows;
                const IDX eb = fdiv(e, p.div_nh), eh = e - eb * nh;
                poff = int64_t(eb) * p.p_bs + int64_t(eh) * p.p_hs + int64_t(rr) * p.ldw + int64_t(gwv[u]);
            }
            if (KIND == K_BINARY) {
                p.sgn[poff] = neg;
            } else {
                p.nz[poff] = wn;
                if (KIND == K_TERNARY) p.sgn[poff] = neg;
                if (p.row_nnz && wn) atomicAdd(p.row_nnz + r, __popc(wn));
            }
            if (gwv[u] + 1 == nwd) {  // the row's last data word: zero the padding words
                for (IDX w = nwd; w < ldw; ++w) {
                    const int64_t o = poff + int64_t(w - gwv[u]);
                    if (KIND == K_BINARY || KIND == K_TERNARY) p.sgn[o] = 0u;
                    if (KIND != K_BINARY) p.nz[o] = 0u;
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Transposed mode.  Work item = (entry, 32-row group, 32-col tile): lane l
// packs row l of the group into a 32-bit word (bit c = column c), a 5-stage
// shuffle butterfly transposes the 32x32 bit block, and lane c stores the
// word of column c.  Row groups up to ldw cover the zero padding.
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

// Body of the transposed pack for block `vb` of a grid of `vg` blocks.
// Work item = (entry, 32-column tile, 4 consecutive 32-row groups): lane l
// loads row 32*g + l of each of the 4 groups (4 x 64 B in flight per lane),
// packs and transposes each 32x32 bit block, and lane c then holds 4
// consecutive words of output row c, stored as one 16-byte vector per plane
// (ld is a multiple of 4 words, so the vector never crosses a row).
template <typename T, int KIND, bool VEC, typename IDX>
__device__ __forceinline__ void pack_cols_body(const PackArgs& p, unsigned vb, unsigned vg) {
    constexpr int E = TypeInfo<T>::E;
    constexpr int NV = 32 / E;  // 16-byte vectors per 32 columns
    constexpr int G = 4;        // row groups per item
    const int lane = threadIdx.x & 31;
    const IDX ngq = IDX(p.ldw / G);               // 128-row quads (ld covers the padding)
    const IDX ntile_c = IDX((p.cols + 31) / 32);
    const IDX nh = IDX(p.nh);
    const IDX items = IDX(p.nb * p.nh) * ngq * ntile_c;
    const IDX warp0 = (IDX(vb) * blockDim.x + threadIdx.x) >> 5;
    const IDX nwarps = (IDX(vg) * blockDim.x) >> 5;
    for (IDX it = warp0; it < items; it += nwarps) {
        const IDX tc = it % ntile_c, t2 = it / ntile_c;
        const IDX gq = t2 % ngq, e = t2 / ngq;
        const T* base = reinterpret_cast<const T*>(p.x) + int64_t(e / nh) * p.x_bs + int64_t(e % nh) * p.x_hs;
        // 2-byte inputs: all 4 groups' loads in flight at once; f32 (twice the
        // registers) one group at a time
        constexpr int GL = sizeof(T) == 4 ? 1 : G;
        uint32_t nzw[G], sgw[G];
#pragma unroll
        for (int g0 = 0; g0 < G; g0 += GL) {
            uint4 v[GL][NV];
#pragma unroll
            for (int g = 0; g < GL; ++g) {
                const int64_t r = (int64_t(gq) * G + g0 + g) * 32 + lane;
#pragma unroll
                for (int q = 0; q < NV; ++q) v[g][q] = make_uint4(0, 0, 0, 0);
                if (r < p.rows) {
                    const T* row = base + r * p.ld_x;
#pragma unroll
                    for (int q = 0; q < NV; ++q) v[g][q] = load_chunk<T, VEC>(row, int64_t(tc) * 32 + q * E, p.cols);
                }
            }
#pragma unroll
            for (int g = 0; g < GL; ++g) {
                uint32_t pos = 0, neg = 0;
                if (KIND == K_BINARY) {
                    // sign (Eq. sign; R4): -1 unless x >= 0 (NaN -> -1, -0.0 -> +1); rows past
                    // the end were loaded as +0 and columns past the end are dropped by the caller
                    const int64_t r = (int64_t(gq) * G + g0 + g) * 32 + lane;
#pragma unroll
                    for (int q = 0; q < NV; ++q) neg |= chunk_lt_mu<T>(v[g][q], 0.f) << (q * E);
                    if (r >= p.rows) neg = 0u;  // padding bits are 0 (R8)
                } else {
#pragma unroll
                    for (int q = 0; q < NV; ++q) {
                        uint32_t pb, nb;
                        chunk_bits<T>(v[g][q], p.th, pb, nb);
                        pos |= pb << (q * E);
                        neg |= nb << (q * E);
                    }
                }
                nzw[g0 + g] = KIND == K_BINARY ? 0u : transpose32(KIND == K_BOOL ? pos : (pos | neg), lane);
                sgw[g0 + g] = (KIND != K_BOOL) ? transpose32(neg, lane) : 0u;
            }
        }
        const int64_t col = int64_t(tc) * 32 + lane;
        if (col < p.cols) {
            const int64_t poff = int64_t(e / nh) * p.p_bs + int64_t(e % nh) * p.p_hs + col * p.ldw + int64_t(gq) * G;
            if (KIND != K_BINARY) *reinterpret_cast<uint4*>(p.nz + poff) = make_uint4(nzw[0], nzw[1], nzw[2], nzw[3]);
            if (KIND != K_BOOL)
                *reinterpret_cast<uint4*>(p.sgn + poff) = make_uint4(sgw[0], sgw[1], sgw[2], sgw[3]);
            if (KIND != K_BINARY && p.row_nnz) {
                const int c = __popc(nzw[0]) + __popc(nzw[1]) + __popc(nzw[2]) + __popc(nzw[3]);
                if (c) atomicAdd(p.row_nnz + int64_t(e) * p.cols + col, c);
            }
        }
    }
}

template <typename T, int KIND, bool VEC, typename IDX>
__global__ void __launch_bounds__(256, 2) pack_rows_kernel(PackArgs p) {
    pdl_launch_dependents();
    pdl_wait();  // no global memory access before the predecessor grid completed
    pack_rows_body<T, KIND, VEC, IDX>(p, blockIdx.x, gridDim.x);
}

template <typename T, int KIND, bool VEC, typename IDX>
__global__ void __launch_bounds__(256, 2) pack_cols_kernel(PackArgs p) {
    pdl_launch_dependents();
    pdl_wait();
    pack_cols_body<T, KIND, VEC, IDX>(p, blockIdx.x, gridDim.x);
}

// Several activation packs (same input dtype, 32-bit indexing) in one launch:
// block b runs the pack whose block range [end[d-1], end[d]) contains b.
// Saves the per-launch ramp and drain of the small per-head packs (Q, K and
// V^T of an attention layer).
struct PackGroup {
    PackArgs a[PACK_GROUP_MAX];
    int transpose[PACK_GROUP_MAX];
    int block_end[PACK_GROUP_MAX];
    int n;
};

template <typename T, int KIND, bool VEC>
__device__ __forceinline__ void group_body(const PackArgs& p, int transpose, unsigned vb, unsigned vg) {
    if (transpose) pack_cols_body<T, KIND, VEC, uint32_t>(p, vb, vg);
    else pack_rows_body<T, KIND, VEC, uint32_t>(p, vb, vg);
}

template <typename T>
__global__ void __launch_bounds__(256, 2) pack_group_kernel(const __grid_constant__ PackGroup g) {
    pdl_launch_dependents();
    pdl_wait();
    int d = 0;
    while (d + 1 < g.n && int(blockIdx.x) >= g.block_end[d]) ++d;
    const int b0 = d ? g.block_end[d - 1] : 0;
    const unsigned vb = blockIdx.x - b0, vg = g.block_end[d] - b0;
    const PackArgs& p = g.a[d];
    const int tr = g.transpose[d];
    if (p.kind == K_BOOL) {
        if (p.vec_ok) group_body<T, K_BOOL, true>(p, tr, vb, vg);
        else group_body<T, K_BOOL, false>(p, tr, vb, vg);
    } else {
        if (p.vec_ok) group_body<T, K_TERNARY, true>(p, tr, vb, vg);
        else group_body<T, K_TERNARY, false>(p, tr, vb, vg);
    }
}

// Lean variant: every pack of the group is a row pack of the same kind and vector path, so the
// kernel holds ONE body (the generic group kernel holds eight and is instruction-fetch bound:
// ncu 'no_instruction' 16 of 24 stall cycles on the Q+K packs of a BERT layer).
template <typename T, int KIND, bool VEC>
__global__ void __launch_bounds__(256, 2) pack_group_rows_kernel(const __grid_constant__ PackGroup g) {
    pdl_launch_dependents();
    pdl_wait();
    int d = 0;
    while (d + 1 < g.n && int(blockIdx.x) >= g.block_end[d]) ++d;
    const int b0 = d ? g.block_end[d - 1] : 0;
    pack_rows_body<T, KIND, VEC, uint32_t>(g.a[d], blockIdx.x - b0, g.block_end[d] - b0);
}

template <typename T>
cudaError_t launch_group_rows(const PackGroup& g, int kind, bool vec, int blocks, cudaStream_t s) {
    if (kind == K_BOOL)
        return vec ? launch_pdl(pack_group_rows_kernel<T, K_BOOL, true>, blocks, 256, 0, s, 1, g)
                   : launch_pdl(pack_group_rows_kernel<T, K_BOOL, false>, blocks, 256, 0, s, 1, g);
    return vec ? launch_pdl(pack_group_rows_kernel<T, K_TERNARY, true>, blocks, 256, 0, s, 1, g)
               : launch_pdl(pack_group_rows_kernel<T, K_TERNARY, false>, blocks, 256, 0, s, 1, g);
}

int num_sms_pack() { return device_sms(); }

// One resident wave (2 x 256-thread blocks per SM, <= 128 registers); warps loop with prefetch.
int grid_for(int64_t warp_items) {
    const int64_t blocks = (warp_items + 7) / 8;
    const int64_t cap = int64_t(num_sms_pack()) * 2;
    return int(blocks < 1 ? 1 : (blocks > cap ? cap : blocks));
}

template <typename T, typename IDX>
cudaError_t rows_dispatch(const PackArgs& a, cudaStream_t s, int grid) {
    cudaError_t err = cudaSuccess;
#define BWTA_ROWS(KIND)                                                                   \
    do {                                                                                  \
        if (a.vec_ok) err = launch_pdl(pack_rows_kernel<T, KIND, true, IDX>, grid, 256, 0, s, 1, a);  \
        else err = launch_pdl(pack_rows_kernel<T, KIND, false, IDX>, grid, 256, 0, s, 1, a);         \
    } while (0)
    if (a.kind == K_BINARY) BWTA_ROWS(K_BINARY);
    else if (a.kind == K_BOOL) BWTA_ROWS(K_BOOL);
    else BWTA_ROWS(K_TERNARY);
#undef BWTA_ROWS
    return err;
}

template <typename T, typename IDX>
cudaError_t cols_dispatch(const PackArgs& a, cudaStream_t s, int grid) {
    cudaError_t err = cudaSuccess;
#define BWTA_COLS(KIND)                                                                   \
    do {                                                                                  \
        if (a.vec_ok) err = launch_pdl(pack_cols_kernel<T, KIND, true, IDX>, grid, 256, 0, s, 1, a);  \
        else err = launch_pdl(pack_cols_kernel<T, KIND, false, IDX>, grid, 256, 0, s, 1, a);         \
    } while (0)
    if (a.kind == K_BOOL) BWTA_COLS(K_BOOL);
    else if (a.kind == K_BINARY) BWTA_COLS(K_BINARY);
    else BWTA_COLS(K_TERNARY);
#undef BWTA_COLS
    return err;
}

template <typename T>
cudaError_t rows_idx(const PackArgs& a, cudaStream_t s, int grid, bool small) {
    return small ? rows_dispatch<T, uint32_t>(a, s, grid) : rows_dispatch<T, uint64_t>(a, s, grid);
}
template <typename T>
cudaError_t cols_idx(const PackArgs& a, cudaStream_t s, int grid, bool small) {
    return small ? cols_dispatch<T, uint32_t>(a, s, grid) : cols_dispatch<T, uint64_t>(a, s, grid);
}

}  // namespace

cudaError_t launch_pack_rows(const PackArgs& a, cudaStream_t s) {
    const int64_t total_words = a.nb * a.nh * a.rows * a.nwd;
    if (total_words == 0) return cudaSuccess;
    if (a.row_nnz && a.kind != K_BINARY) {
        cudaError_t err = cudaMemsetAsync(a.row_nnz, 0, sizeof(int32_t) * a.nb * a.nh * a.rows, s);
        if (err != cudaSuccess) return err;
        count_launch();
    }
    const int grid = grid_for((total_words + 63) / 64);
    const bool small = total_words + 4 * int64_t(grid) * 256 < (int64_t(1) << 31) &&
                       a.cols + 32 < (int64_t(1) << 31);
    switch (a.dt) {
        case DT_F16: return rows_idx<__half>(a, s, grid, small);
        case DT_BF16: return rows_idx<__nv_bfloat16>(a, s, grid, small);
        default: return rows_idx<float>(a, s, grid, small);
    }
}

cudaError_t launch_pack_cols(const PackArgs& a, cudaStream_t s) {
    const int64_t items = a.nb * a.nh * (a.ldw / 4) * ((a.cols + 31) / 32);
    if (items == 0) return cudaSuccess;
    if (a.row_nnz) {
        cudaError_t err = cudaMemsetAsync(a.row_nnz, 0, sizeof(int32_t) * a.nb * a.nh * a.cols, s);
        if (err != cudaSuccess) return err;
        count_launch();
    }
    const int grid = grid_for(items);
    const bool small = items + int64_t(grid) * 8 < (int64_t(1) << 31);
    switch (a.dt) {
        case DT_F16: return cols_idx<__half>(a, s, grid, small);
        case DT_BF16: return cols_idx<__nv_bfloat16>(a, s, grid, small);
        default: return cols_idx<float>(a, s, grid, small);
    }
}

namespace {
int64_t pack_work(const PackArgs& a, int transpose) {
    return transpose ? a.nb * a.nh * a.ldw * ((a.cols + 31) / 32) * 32 : a.nb * a.nh * a.rows * a.nwd;
}
bool pack_small(const PackArgs& a, int transpose, int grid) {
    if (transpose) return pack_work(a, 1) / 32 + int64_t(grid) * 8 < (int64_t(1) << 31);
    return pack_work(a, 0) + 4 * int64_t(grid) * 256 < (int64_t(1) << 31) && a.cols + 32 < (int64_t(1) << 31);
}
}  // namespace

cudaError_t launch_pack_group(const PackArgs* a, const int* transpose, int n, cudaStream_t s) {
    // one pack, mixed dtypes or 64-bit indexing: ordinary launches, in order
    bool fuse = n > 1 && n <= PACK_GROUP_MAX;
    for (int i = 0; i < n && fuse; ++i)
        fuse = a[i].dt == a[0].dt && a[i].kind != K_BINARY && pack_small(a[i], transpose[i], 2 * num_sms_pack());
    if (!fuse) {
        for (int i = 0; i < n; ++i) {
            cudaError_t e = transpose[i] ? launch_pack_cols(a[i], s) : launch_pack_rows(a[i], s);
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    }
    PackGroup g{};
    g.n = n;
    int64_t total = 0, work[PACK_GROUP_MAX];
    for (int i = 0; i < n; ++i) {
        g.a[i] = a[i];
        g.transpose[i] = transpose[i];
        work[i] = pack_work(a[i], transpose[i]);
        total += work[i];
        if (a[i].row_nnz) {
            const int64_t cnt = a[i].nb * a[i].nh * (transpose[i] ? a[i].cols : a[i].rows);
            cudaError_t e = cudaMemsetAsync(a[i].row_nnz, 0, sizeof(int32_t) * cnt, s);
            if (e != cudaSuccess) return e;
            count_launch();
        }
    }
    // one resident wave shared in proportion to the words each pack writes
    const int wave = 2 * num_sms_pack();
    int end = 0;
    for (int i = 0; i < n; ++i) {
        int64_t b = total > 0 ? (work[i] * wave + total - 1) / total : 1;
        const int64_t need = transpose[i] ? (work[i] / 128 + 7) / 8 : (work[i] + 511) / 512;  // warp items
        if (b > need) b = need;
        end += int(b < 1 ? 1 : b);
        g.block_end[i] = end;
    }
    bool lean = true;  // all row packs of one kind and vector path -> the one-body kernel
    for (int i = 0; i < n; ++i)
        lean = lean && !transpose[i] && a[i].kind == a[0].kind && a[i].vec_ok == a[0].vec_ok;
    if (lean) {
        switch (a[0].dt) {
            case DT_F16: return launch_group_rows<__half>(g, a[0].kind, a[0].vec_ok, end, s);
            case DT_BF16: return launch_group_rows<__nv_bfloat16>(g, a[0].kind, a[0].vec_ok, end, s);
            default: return launch_group_rows<float>(g, a[0].kind, a[0].vec_ok, end, s);
        }
    }
    switch (a[0].dt) {
        case DT_F16: return launch_pdl(pack_group_kernel<__half>, end, 256, 0, s, 1, g);
        case DT_BF16: return launch_pdl(pack_group_kernel<__nv_bfloat16>, end, 256, 0, s, 1, g);
        default: return launch_pdl(pack_group_kernel<float>, end, 256, 0, s, 1, g);
    }
}

}  // namespace bwta
