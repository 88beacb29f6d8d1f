// attn_decode.cu -- fused BWTA decode attention (Tq = 1):
//   s_j = fl32(float(q . k_j) * alpha)                      (Case 3 / binary K; R5)
//   p_j = softmax_j(s) in fp32, rounded to p_dt              (high-precision softmax)
//   b_j = [round(p_j) >= s_att / 2]                          (bool quantizer; R1, R2)
//   o_d = fl32(float(sum_j b_j v_jd) * beta)                 (Case 2; R5)
// in ONE launch: no S, P or P-plane round trip through memory.  One CTA of
// 1024 threads per (batch, head) entry -- or a cluster of 2-8 CTAs splitting its
// keys when there are few entries (their (max, sum) merged in rank order, their
// partial PV dots summed by rank 0 through distributed shared memory).  The two products are the paper's bit-serial
// identities on CUDA cores (R10): a decode query is a single row, far below a
// tensor-core tile.
//   pass 1: thread j-strided dots, online (max, sum of exp) per thread, merged
//           across the warp (shuffles) and the CTA (fixed warp order);
//   pass 2: the scores (kept in shared memory), p_j = exp(s_j - max) / sum, round to p_dt, compare,
//           __ballot_sync -> P word (32 consecutive j) in shared memory;
//   PV:     thread (d, slice): popc over a slice of V^T row d's words against
//           the P words; slices summed through shared memory.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "bwta_internal.h"
#include "sm100.cuh"

namespace bwta {
namespace {

constexpr int AD_WARPS = 32;  // 1024 threads per CTA
constexpr int AD_CMAX = 8;    // CTAs per entry (a cluster) when there are few (batch, head) entries

// cluster barrier with release / acquire semantics (the shared-memory data crosses it)
__device__ __forceinline__ void cluster_sync_acqrel() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t ld_cluster_u32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
constexpr int AD_QW = 8;  // head_dim <= 256

__device__ __forceinline__ float round_to(int dt, float p) {
    if (dt == DT_F16) return __half2float(__float2half_rn(p));
    if (dt == DT_BF16) return __bfloat162float(__float2bfloat16_rn(p));
    return p;
}

// K rows are 16-byte aligned (ld % 4 == 0): 16-byte loads, 4 words at a time
__device__ __forceinline__ int32_t qk_dot(const uint32_t (&qs)[AD_QW], const uint32_t (&qn)[AD_QW], int qw,
                                          const uint32_t* ks, const uint32_t* kn) {
    int32_t d = 0;
#pragma unroll
    for (int w4 = 0; w4 < AD_QW; w4 += 4) {
        if (w4 < qw) {
            const uint4 s4 = __ldg(reinterpret_cast<const uint4*>(ks + w4));
            const uint4 n4 = kn ? __ldg(reinterpret_cast<const uint4*>(kn + w4)) : make_uint4(~0u, ~0u, ~0u, ~0u);
            const uint32_t sv[4] = {s4.x, s4.y, s4.z, s4.w}, nv[4] = {n4.x, n4.y, n4.z, n4.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint32_t m = qn[w4 + i] & nv[i];  // q's padding words are 0
                d += __popc(m) - 2 * __popc(m & (qs[w4 + i] ^ sv[i]));
            }
        }
    }
    return d;
}

__global__ void __launch_bounds__(AD_WARPS * 32) attn_decode_kernel(DecodeArgs p) {
    pdl_launch_dependents();
    pdl_wait();
    extern __shared__ uint32_t ad_pw[];  // this CTA's P words, then partial PV sums
    __shared__ float red_m[AD_WARPS], red_z[AD_WARPS];
    __shared__ float cta_mz[2];          // this CTA's (max, sum) -- read by the cluster
    __shared__ int32_t cta_o[256];       // this CTA's partial O (head_dim <= 256) -- read by rank 0
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int cs = p.cs;                 // CTAs per entry (cluster size)
    const int rank = cs > 1 ? int(sm100::cluster_ctarank()) : 0;
    // (32-bit index arithmetic: the int64 divisions were subroutine calls; the host keeps
    // entries * cs, tk and nh below 2^31)
    const int e32 = int(blockIdx.x) / cs;
    const int64_t e = e32;
    // this CTA's keys: whole words [w_lo, w_hi) of the P row
    const int nw = int((p.tk + 31) / 32);
    const int64_t w_lo = int(int64_t(nw) * rank / cs), w_hi = int(int64_t(nw) * (rank + 1) / cs);
    const int64_t j_lo = 32 * w_lo, j_hi = 32 * w_hi < p.tk ? 32 * w_hi : p.tk;
    const int nh32 = int(p.nh);
    const int64_t eb = e32 / nh32, eh = e32 - (e32 / nh32) * nh32;
    const float alpha = p.alpha_h ? __ldg(p.alpha_h + eh) : p.alpha;  // per-head alpha (nullable)
    const int qw = int((p.dh + 31) / 32);
    uint32_t qs[AD_QW], qn[AD_QW];
    const uint32_t* q0 = p.q_nz + eb * p.q_bs + eh * p.q_hs;
    const uint32_t* q1 = p.q_sgn + eb * p.q_bs + eh * p.q_hs;
#pragma unroll
    for (int w4 = 0; w4 < AD_QW; w4 += 4) {  // q rows are 16-byte aligned, padding words 0
        const uint4 n4 = w4 < qw ? __ldg(reinterpret_cast<const uint4*>(q0 + w4)) : make_uint4(0, 0, 0, 0);
        const uint4 s4 = w4 < qw ? __ldg(reinterpret_cast<const uint4*>(q1 + w4)) : make_uint4(0, 0, 0, 0);
        qn[w4] = n4.x; qn[w4 + 1] = n4.y; qn[w4 + 2] = n4.z; qn[w4 + 3] = n4.w;
        qs[w4] = s4.x & n4.x; qs[w4 + 1] = s4.y & n4.y; qs[w4 + 2] = s4.z & n4.z; qs[w4 + 3] = s4.w & n4.w;
    }
    const uint32_t* kbase_s = p.k_sgn + eb * p.k_bs + eh * p.k_hs;
    const uint32_t* kbase_n = p.k_nz ? p.k_nz + eb * p.k_bs + eh * p.k_hs : nullptr;
    constexpr int NT = AD_WARPS * 32;
    // pass 1: max and sum of exp, online per thread, merged across the CTA
    float mx = -INFINITY, z = 0.f;
    // this CTA's scores, kept for pass 2 (after the P words and the PV partials)
    float* sc = reinterpret_cast<float*>(ad_pw + p.sc_off);
    for (int64_t j = j_lo + tid; j < j_hi; j += NT) {
        const int32_t d = qk_dot(qs, qn, qw, kbase_s + j * p.ldk, kbase_n ? kbase_n + j * p.ldk : nullptr);
        const float s = __fmul_rn(float(d), alpha);
        sc[j - j_lo] = s;
        if (s > mx) {
            z = z * expf(mx - s) + 1.f;
            mx = s;
        } else {
            z += expf(s - mx);
        }
    }
    auto merge = [](float& m1, float& z1, float m2, float z2) {
        const float m = fmaxf(m1, m2);
        z1 = (m1 == -INFINITY ? 0.f : z1 * expf(m1 - m)) + (m2 == -INFINITY ? 0.f : z2 * expf(m2 - m));
        m1 = m;
    };
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) merge(mx, z, __shfl_xor_sync(0xffffffffu, mx, o), __shfl_xor_sync(0xffffffffu, z, o));
    if (lane == 0) {
        red_m[warp] = mx;
        red_z[warp] = z;
    }
    __syncthreads();
    mx = red_m[0];
    z = red_z[0];
    for (int w = 1; w < AD_WARPS; ++w) merge(mx, z, red_m[w], red_z[w]);  // same order in every thread
    if (cs > 1) {  // merge the cluster's CTAs in rank order (identical in every CTA)
        if (tid == 0) {
            cta_mz[0] = mx;
            cta_mz[1] = z;
        }
        cluster_sync_acqrel();
        mx = __uint_as_float(ld_cluster_u32(sm100::mapa_smem(&cta_mz[0], 0)));
        z = __uint_as_float(ld_cluster_u32(sm100::mapa_smem(&cta_mz[1], 0)));
        for (int r = 1; r < cs; ++r)
            merge(mx, z, __uint_as_float(ld_cluster_u32(sm100::mapa_smem(&cta_mz[0], r))),
                  __uint_as_float(ld_cluster_u32(sm100::mapa_smem(&cta_mz[1], r))));
    }
    // pass 2: P words (warp w, round i covers j = NT i + 32 w + lane -> word (NT / 32) i + w)
    const int64_t lw = w_hi - w_lo;  // this CTA's words; ad_pw[i] = P word w_lo + i
    for (int64_t j0 = j_lo; j0 < j_hi; j0 += NT) {
        const int64_t j = j0 + tid;
        bool bit = false;
        if (j < j_hi) {
            const float s = sc[j - j_lo];  // written by this same thread in pass 1
            const float pj = __fdiv_rn(expf(s - mx), z);
            bit = round_to(p.p_dt, pj) >= p.p_t;
        }
        const uint32_t word = __ballot_sync(0xffffffffu, bit);
        const int64_t wi = (j0 - j_lo + 32 * warp) / 32;
        if (lane == 0 && wi < lw) ad_pw[wi] = word;
    }
    const int64_t lq = (lw + 3) / 4 + 1;  // local quads (+1: the slice may start mid-quad)
    for (int64_t wi = lw + tid; wi < 4 * lq; wi += NT) ad_pw[wi] = 0u;
    __syncthreads();
    if (p.p_out) {
        uint32_t* po = p.p_out + e * p.p_ld;
        for (int64_t wi = tid; wi < lw; wi += NT) po[w_lo + wi] = ad_pw[wi];
        if (rank == cs - 1)
            for (int64_t wi = nw + tid; wi < p.p_ld; wi += NT) po[wi] = 0u;
    }
    // PV: output d by NT / dh_groups threads, each a slice of the P words, partials through smem
    int32_t* part = reinterpret_cast<int32_t*>(ad_pw + 4 * lq);  // [NT]
    const int dpad = int((p.dh + 31) / 32) * 32;                    // threads per slice group
    const int nslice = NT / dpad > 0 ? NT / dpad : 1;
    const int dd = tid % dpad, sl = tid / dpad;
    int32_t acc = 0;
    if (sl < nslice && dd < p.dh) {
        // V^T words [w_lo, w_hi) of row d, in word quads aligned to the V^T row (16-byte loads);
        // the local P words are read at the matching (possibly unaligned) offsets
        const int64_t a0 = w_lo & ~int64_t(3);                 // first aligned word
        const int64_t nq = (w_hi - a0 + 3) / 4, q0 = nq * sl / nslice, q1 = nq * (sl + 1) / nslice;
        const uint4* vs = reinterpret_cast<const uint4*>(p.v_sgn + eb * p.v_bs + eh * p.v_hs + dd * p.ldv + a0);
        const uint4* vn = reinterpret_cast<const uint4*>(p.v_nz + eb * p.v_bs + eh * p.v_hs + dd * p.ldv + a0);
        auto pword = [&](int64_t w) -> uint32_t {  // P word a0 + w (0 outside this CTA's range)
            const int64_t g = a0 + w;
            return (g >= w_lo && g < w_hi) ? ad_pw[g - w_lo] : 0u;
        };
#pragma unroll 4
        for (int64_t qi = q0; qi < q1; ++qi) {
            const uint4 n4 = __ldg(vn + qi), s4 = __ldg(vs + qi);
            const uint4 p4 = make_uint4(pword(4 * qi), pword(4 * qi + 1), pword(4 * qi + 2), pword(4 * qi + 3));
            const uint32_t m0 = p4.x & n4.x, m1 = p4.y & n4.y, m2 = p4.z & n4.z, m3 = p4.w & n4.w;
            acc += __popc(m0) + __popc(m1) + __popc(m2) + __popc(m3) -
                   2 * (__popc(m0 & s4.x) + __popc(m1 & s4.y) + __popc(m2 & s4.z) + __popc(m3 & s4.w));
        }
    }
    part[tid] = acc;
    __syncthreads();
    int32_t dot = 0;
    if (tid < p.dh)
        for (int s2 = 0; s2 < nslice; ++s2) dot += part[s2 * dpad + tid];
    if (cs > 1) {  // rank 0 sums the cluster's partial dots (exact integers, any order)
        if (tid < p.dh) cta_o[tid] = dot;
        cluster_sync_acqrel();
        if (rank == 0 && tid < p.dh)
            for (int r = 1; r < cs; ++r) dot += int32_t(ld_cluster_u32(sm100::mapa_smem(&cta_o[tid], r)));
        cluster_sync_acqrel();  // no CTA leaves while its shared memory may still be read
        if (rank != 0) return;
    }
    if (tid < p.dh) {
        const int64_t off = eb * p.o_bs + eh * p.o_hs + tid;
        const float y = __fmul_rn(float(dot), p.beta_h ? __ldg(p.beta_h + eh) : p.beta);
        if (p.o_dt == DT_F16) reinterpret_cast<__half*>(p.o)[off] = __float2half_rn(y);
        else if (p.o_dt == DT_BF16) reinterpret_cast<__nv_bfloat16*>(p.o)[off] = __float2bfloat16_rn(y);
        else if (p.o_dt == DT_F32) reinterpret_cast<float*>(p.o)[off] = y;
        else reinterpret_cast<int32_t*>(p.o)[off] = dot;
    }
}

}  // namespace

cudaError_t launch_attn_decode(const DecodeArgs& a, cudaStream_t s) {
    const int64_t entries = a.nb * a.nh;
    // CTAs per entry: spread few entries over the SMs (cluster of up to 8), keeping >= 2 words each
    int cs = 1;
    while (cs < AD_CMAX && entries * cs * 2 <= 148 && (a.tk + 31) / 32 >= 2 * cs * 2) cs *= 2;
    DecodeArgs b = a;
    b.cs = cs;
    const int grid = int(entries * cs);
    const int64_t lw = ((a.tk + 31) / 32 + cs - 1) / cs;
    b.sc_off = 4 * ((lw + 3) / 4 + 1) + AD_WARPS * 32;               // words: P words, PV partials, scores
    const size_t smem = sizeof(uint32_t) * size_t(b.sc_off + 32 * lw);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(attn_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return e;
    }
    return launch_pdl(attn_decode_kernel, dim3(grid), dim3(AD_WARPS * 32), smem, s, cs, b);
}

}  // namespace bwta
