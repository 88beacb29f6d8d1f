// gemm_b1.cu -- the paper's own kernel design, as prior art measured on B200:
// the binarized warp-level MMA `mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc`
// (Sec. 5.2.3: "binary connective logic gates (and / xor) for bitwise multiplication
// and a popcount for accumulation").  sm_100a has no native b1 tensor path: ptxas lowers the
// instruction to MOVM.U4TO8 + IMMA -- this kernel measures what the A800/H800
// design costs here, next to design (b) (tcgen05 kind::mxf4).
//
// Case 1 / 2 / 3 with AND-popcount MMAs: with P = nz & ~sgn (the +1 elements) and N = nz & sgn
// (the -1 elements) of each operand (binary: P = ~sgn, N = sgn over the valid bits),
//   dot = popc(Pa & Pb) + popc(Na & Nb) - popc(Pa & Nb) - popc(Na & Pb)
// i.e. two accumulators of two MMAs each per 256-element K step.  Exact integers (int32).
// One warp computes a 32 x 32 output block (2 x 4 MMA tiles of 16 x 8); fragments are read
// straight from the bit planes (L1/L2-cached 32-bit loads, no shared memory).
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "bwta_internal.h"

namespace bwta {
namespace {

constexpr int B1_WM = 32, B1_WN = 32;  // outputs per warp
constexpr int B1_WARPS = 4;            // warps per CTA (a 64 x 64 block)

__device__ __forceinline__ void mma_b1(int32_t (&c)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc "
        "{%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, {%0, %1, %2, %3};"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// word w of row r of an operand as (P, N) masks; rows / words out of range read as 0
__device__ __forceinline__ void pn_word(const uint32_t* sgn, const uint32_t* nz, int64_t ld, int64_t r, int64_t rows,
                                        int64_t w, int64_t nw, uint32_t valid, uint32_t& P, uint32_t& N) {
    if (r >= rows || w >= nw) {
        P = N = 0u;
        return;
    }
    const uint32_t s = sgn ? __ldg(sgn + r * ld + w) : 0u;
    const uint32_t m = nz ? __ldg(nz + r * ld + w) : valid;  // absent nz: every valid bit is +-1
    P = m & ~s;
    N = m & s;
}

__global__ void __launch_bounds__(32 * B1_WARPS) matmul_b1_kernel(MatmulArgs p) {
    pdl_launch_dependents();
    pdl_wait();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t4 = lane & 3;  // groupID, threadID_in_group
    const int64_t e = blockIdx.z, eb = e / p.nh, eh = e % p.nh;
    const int64_t i0 = int64_t(blockIdx.y) * 64 + (warp >> 1) * B1_WM;
    const int64_t j0 = int64_t(blockIdx.x) * 64 + (warp & 1) * B1_WN;
    const uint32_t* As = p.a_sgn ? p.a_sgn + eb * p.a_bs + eh * p.a_hs : nullptr;
    const uint32_t* An = p.a_nz ? p.a_nz + eb * p.a_bs + eh * p.a_hs : nullptr;
    const uint32_t* Bs = p.b_sgn ? p.b_sgn + eb * p.b_bs + eh * p.b_hs : nullptr;
    const uint32_t* Bn = p.b_nz ? p.b_nz + eb * p.b_bs + eh * p.b_hs : nullptr;
    const int64_t nw = (p.K + 31) / 32;
    int32_t cpos[2][4][4], cneg[2][4][4];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
            for (int c = 0; c < 4; ++c) cpos[mi][ni][c] = cneg[mi][ni][c] = 0;
    for (int64_t k8 = 0; k8 < nw; k8 += 8) {  // one 256-element K step
        // A fragment (16 x 256, row-major): a0 row g, word t4; a1 row g+8; a2 / a3 words t4+4
        uint32_t aP[2][4], aN[2][4];
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int64_t r = i0 + 16 * mi + g + 8 * (q & 1);
                const int64_t w = k8 + t4 + 4 * (q >> 1);
                const uint32_t valid = w < nw - 1 ? 0xffffffffu : (p.K % 32 ? (1u << (p.K % 32)) - 1u : 0xffffffffu);
                pn_word(As, An, p.lda, r, p.M, w, nw, valid, aP[mi][q], aN[mi][q]);
            }
        // B fragment (256 x 8, column-major = B rows of the operand): b0 col g, word t4; b1 word t4+4
        uint32_t bP[4][2], bN[4][2];
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int64_t r = j0 + 8 * ni + g;
                const int64_t w = k8 + t4 + 4 * q;
                const uint32_t valid = w < nw - 1 ? 0xffffffffu : (p.K % 32 ? (1u << (p.K % 32)) - 1u : 0xffffffffu);
                pn_word(Bs, Bn, p.ldb, r, p.N, w, nw, valid, bP[ni][q], bN[ni][q]);
            }
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) {
                mma_b1(cpos[mi][ni], aP[mi], bP[ni]);
                mma_b1(cpos[mi][ni], aN[mi], bN[ni]);
                mma_b1(cneg[mi][ni], aP[mi], bN[ni]);
                mma_b1(cneg[mi][ni], aN[mi], bP[ni]);
            }
    }
    // C fragment (16 x 8): c0, c1 row g, cols 2 t4, 2 t4 + 1; c2, c3 row g + 8
    const int64_t ybase = eb * p.y_bs + eh * p.y_hs;
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int64_t i = i0 + 16 * mi + g + 8 * (c >> 1), j = j0 + 8 * ni + 2 * t4 + (c & 1);
                if (i >= p.M || j >= p.N) continue;
                const int32_t d = cpos[mi][ni][c] - cneg[mi][ni][c];
                const int64_t idx = ybase + (p.y_trans ? j * p.ldy + i : i * p.ldy + j);
                if (p.y_dt == DT_I32) {
                    reinterpret_cast<int32_t*>(p.y)[idx] = d;
                } else {
                    const float cs = p.col_scale ? __fmul_rn(__ldg(p.col_scale + j), p.scalar) : p.scalar;
                    const float f = __fmul_rn(float(d), cs);  // R5
                    if (p.y_dt == DT_F16) reinterpret_cast<__half*>(p.y)[idx] = __float2half_rn(f);
                    else if (p.y_dt == DT_BF16) reinterpret_cast<__nv_bfloat16*>(p.y)[idx] = __float2bfloat16_rn(f);
                    else reinterpret_cast<float*>(p.y)[idx] = f;
                }
            }
}

}  // namespace

cudaError_t launch_matmul_b1(const MatmulArgs& a, cudaStream_t s) {
    if (a.M == 0 || a.N == 0 || a.nb * a.nh == 0) return cudaSuccess;
    const dim3 grid(unsigned((a.N + 63) / 64), unsigned((a.M + 63) / 64), unsigned(a.nb * a.nh));
    return launch_pdl(matmul_b1_kernel, grid, dim3(32 * B1_WARPS), 0, s, 1, a);
}

}  // namespace bwta
