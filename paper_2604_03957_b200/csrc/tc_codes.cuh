// tc_codes.cuh -- what the two tcgen05 kernels (gemm_tc.cu: general tiles;
// gemv_tc.cu: skinny problems) share: the E2M1 operand codes and the host-side
// TMA descriptor helpers.  Not part of the ABI.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdint.h>

#include "sm100.cuh"

namespace bwta {
namespace tc {

enum BKind { B_BINARY = 0, B_BOOL = 1, B_TERNARY = 2 };  // operand kinds (A or B)

// Operand codes: E2M1 nibbles, +1.0 = 0x2, -1.0 = 0xA, 0 = 0x0, fed to
// tcgen05.mma.kind::mxf4 with every UE8M0 block scale = 1.0 (0x7F), so each
// product is exactly q_a * q_w and the f32 accumulator holds the integer dot
// exactly (|dot| <= K <= 2^24).  K order inside a 32-element group: code word
// j (j = 0..3, 8 nibbles) holds elements {j, 4+j, ..., 28+j}, nibble i =
// element 4i + j, so the nz bit of element 4i+j moves to bit 4i+1 and the sgn
// bit to bit 4i+3 by one shift each (left shifts issued as IMAD.SHL on the FMA
// pipe).  Both operands use the same permutation, so every dot is unchanged.
//   binary  (x0 = sgn):           0x2 | sgn << 3            -> +1 / -1
//   bool    (x0 = nz):            nz << 1                   -> 0 / +1
//   ternary (x0 = sgn, x1 = nz):  nz << 1 | sgn << 3        -> 0 / +1 / -1
// (ternary sgn is masked to the canonical subset of nz)

__device__ __forceinline__ uint32_t shl_fma(uint32_t x, int k) {  // x << k as IMAD.SHL (FMA pipe)
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, 0;" : "=r"(r) : "r"(x), "r"(1u << k));
    return r;
}
// bit 4i+j -> bit 4i+1 (nz) / 4i+3 (sgn)
__device__ __forceinline__ uint32_t nz_to_bit1(uint32_t x, int j) { return j == 0 ? shl_fma(x, 1) : (j == 1 ? x : x >> (j - 1)); }
__device__ __forceinline__ uint32_t sg_to_bit3(uint32_t x, int j) { return j == 3 ? x : shl_fma(x, 3 - j); }

template <int KIND>
__device__ __forceinline__ uint32_t unpack_word(uint32_t x0, uint32_t x1, int j) {
    if (KIND == B_BINARY) return (sg_to_bit3(x0, j) & 0x88888888u) | 0x22222222u;
    if (KIND == B_BOOL) return nz_to_bit1(x0, j) & 0x22222222u;
    return (nz_to_bit1(x1, j) & 0x22222222u) | (sg_to_bit3(x0, j) & 0x88888888u);
}

__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

// ---- shared by the tcgen05 kernels (gemm_tc.cu, attn_prefill.cu) ----------------------------
// K elements per stage, KS = 256 (one 128-byte SW128 row of packed E2M1
// codes per operand row) or KS = 128 (a 64-byte SW64 row) for K <= 128 --
// attention with head_dim <= 128 -- so no stage is half padding.
template <int KS> struct Stage {
    static constexpr int ROWB = KS / 2;       // bytes per operand row per stage
    static constexpr int WPS = KS / 32;       // packed words per row per plane per stage
    static constexpr int NMMA = ROWB / 32;    // tcgen05.mma per stage (K = 64 each)
};
// One operand row (KS K-elements = KS/32 words per plane) -> KS/2 bytes of
// E2M1 codes at rowaddr in the UMMA K-major layout: packed word g becomes the
// 16-byte chunk g, placed by the 128B swizzle (chunk ^ (r & 7), 8-row atoms
// of 1024 B) or the 64B swizzle (chunk ^ ((r >> 1) & 3), 8-row atoms of 512 B).
// p0: sgn (binary, ternary) or nz (bool); p1: nz (ternary).
template <int KIND, int KS>
__device__ __forceinline__ void unpack_row(uint32_t p0addr, uint32_t p1addr, uint32_t rowaddr, int r) {
    const int sw = KS == 256 ? (r & 7) : ((r >> 1) & 3);
#pragma unroll
    for (int h = 0; h < Stage<KS>::WPS / 4; ++h) {  // words 4h .. 4h+3
        const uint4 w0 = sm100::lds128(p0addr + 16 * h);
        uint4 w1 = make_uint4(0, 0, 0, 0);
        if (KIND == B_TERNARY) w1 = sm100::lds128(p1addr + 16 * h);
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
}

// rows [r0, rows) step `step` of one operand slice (warp-uniform kind)
template <int KS>
__device__ __forceinline__ void unpack_rows(int kind, uint32_t bits, int plane_bytes, uint32_t dst, int r0, int rows,
                                            int step) {
    constexpr int RB = Stage<KS>::WPS * 4;  // bit bytes per row per plane
    constexpr int ROWB = Stage<KS>::ROWB;
    if (kind == B_TERNARY) {
        for (int r = r0; r < rows; r += step)
            unpack_row<B_TERNARY, KS>(bits + r * RB, bits + plane_bytes + r * RB, dst + r * ROWB, r);
    } else if (kind == B_BOOL) {
        for (int r = r0; r < rows; r += step) unpack_row<B_BOOL, KS>(bits + r * RB, 0, dst + r * ROWB, r);
    } else {
        for (int r = r0; r < rows; r += step) unpack_row<B_BINARY, KS>(bits + r * RB, 0, dst + r * ROWB, r);
    }
}


}  // namespace tc

// host helpers (gemm_tc.cu)
PFN_cuTensorMapEncodeTiled_v12000 encode_fn();
bool encode(CUtensorMap* m, CUtensorMapDataType dt, int rank, void* base, const uint64_t* dims,
            const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapSwizzle sw);
int num_sms();
int64_t kw4_of(int64_t K);
uint64_t bstride(int64_t count, int64_t stride_bytes, uint64_t fallback);
// 4-D tensor map over a packed operand: dims {ld words, rows, heads, batch},
// box {wps words, box_rows, 1, 1} (one 32*wps-element K slice of box_rows rows)
bool encode_planes(CUtensorMap* m, const uint32_t* base, int64_t ld, int64_t rows, int64_t hs, int64_t bs,
                   int64_t nh, int64_t nb, int box_rows, int wps,
                   CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_NONE);
int kind_of(const uint32_t* sgn, const uint32_t* nz);

}  // namespace bwta
