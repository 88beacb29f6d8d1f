// attn_prefill.cu -- fused BWTA prefill attention on the 5th-generation tensor
// cores, one launch for the whole layer's attention:
//   S  = Q . K^T                       integer dots, exact in the f32 accumulator   P:959-967 (R10, R12)
//   s  = fl32(dot * alpha)                                                           (R5)
//   p  = softmax over the keys in fp32, rounded to p_dt                              P:882-891 (R13)
//   b  = [round(p) >= s_att / 2]                                                     P:911-919 (R1, R2)
//   O  = fl32(float(b . V) * beta)     integer dots again                            P:969-975 (R5, R12)
// S and P never leave the SM: no T x T score matrix, no probability matrix and
// no P bit-plane pass through HBM (at configs[3] that is 268 MB of fp16 S plus
// the 285 MB P pack of the unfused path).
//
// The bool quantizer needs the row's softmax normaliser before any bit is
// known, so each 128-query tile makes two passes over its keys (the QK^T MMAs
// are cheap next to the softmax arithmetic):
//   pass 1: S blocks -> per-row max and sum of exp.  Every score is alpha times
//           an integer in [-Dh, Dh], so exp(s_j - s_max) is read from a table of
//           exp(alpha d), d in [-2 Dh, 0] (one shared-memory lookup per score,
//           no MUFU); the two half-row partial sums are merged in a fixed order.
//   threshold: p is monotone in the integer dot, so the row's bool decision is
//           dot >= d*_row for one integer d*_row, found by a binary search over
//           [-Dh, max] evaluating R13's exact expression
//           round_p_dt(fl32(expf(fl32(d alpha) - s_max) / z)) >= s_att/2 (the
//           decode kernel's per-score formula);
//   pass 2: S blocks again -> E2M1 codes of the bool P tile (0x2 / 0x0) written
//           to shared memory in the UMMA K-major layout -> O += P . V^T on the
//           tensor core (V^T planes unpacked like any operand), O in TMEM.
// alpha < 0 is folded into the Q codes (negated), so the code paths see |alpha|.
//
// CTA (persistent over (entry, 128-query tile) items), 24 warps:
//   warp 0      TMA producer: Q tile planes; per key block the K planes (+ V^T planes in pass 2)
//   warp 1      MMA issuer: QK^T (128 x 128 x Dh) into S[0/1]; PV (128 x Dh x 128) into O
//   warp 2      TMEM allocator           warp 3  exp table
//   warps 4-7   unpack Q / K / V^T bit planes -> E2M1 codes (shared memory)
//   warps 8-23  softmax + P codes + epilogue: warp (h, q) owns TMEM lane quarter q
//               (query rows 32q..32q+31) and the 32-key slice h of every S block
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <math.h>
#include <stdlib.h>

#include "bwta_internal.h"
#include "sm100.cuh"
#include "tc_codes.cuh"

namespace bwta {
namespace {

using namespace sm100;
using namespace tc;

constexpr int AP_SMW = 16;                 // softmax warps: AP_SMW / 4 per TMEM lane quarter
constexpr int AP_NH = AP_SMW / 4;          // key slices per S block (one per softmax warp of a quarter)
constexpr int AP_NT = 256 + 32 * AP_SMW;
constexpr int AP_S = 6;          // K stages in flight (bits + codes; freed by the QK^T commit)
constexpr int AP_VS = 4;         // V^T code stages (freed by the PV commit)
constexpr int AP_BQ = 128;       // query rows per tile (MMA M)
constexpr int AP_BK = 128;       // keys per block (QK MMA N, PV MMA K)
constexpr int AP_DH = 128;       // head_dim <= 128: one 128-K stage (2 MMAs of K = 64)
constexpr int AP_TBL = 2 * AP_DH + 1;
constexpr int AP_KW = 128 / AP_NH;         // keys of a block per softmax warp
constexpr int AP_NG = AP_KW / 32;          // 32-key chunks per softmax warp and block
constexpr int CODE_ROW = AP_DH / 2;               // 64 B of codes per operand row (SW64)
constexpr int Q_CODES = AP_BQ * CODE_ROW;         // 8 KB
constexpr int Q_BITS = 2 * AP_BQ * 16;            // 2 planes x 128 rows x 16 B
constexpr int K_CODES = AP_BK * CODE_ROW;         // 8 KB
constexpr int V_CODES = AP_DH * CODE_ROW;         // <= 8 KB (dhp rows)
constexpr int K_BITS = 2 * AP_BK * 16;
constexpr int STAGE_B = K_CODES + K_BITS;          // 12 KB
constexpr int VCH_W = 32;                          // V^T words (1024 keys) per chunk: 128-byte TMA rows
constexpr int VCH_BLK = VCH_W / 4;                 // key blocks per V^T chunk
constexpr int VCH_B = 2 * AP_DH * VCH_W * 4;       // both planes, <= 32 KB
constexpr int P_CODES = AP_BQ * CODE_ROW;         // 8 KB per P buffer
constexpr int SMEM_AP = 1024 + 2 * Q_CODES + AP_S * STAGE_B + AP_VS * V_CODES + 2 * VCH_B + 2 * P_CODES +
                        2 * Q_BITS + 4 * 1024 /*tables*/ + 2 * AP_NH * AP_BQ * 4 * 2 /*merge*/ + 512 /*barriers*/;
static_assert(SMEM_AP <= 227 * 1024, "shared memory");
constexpr int TM_S = 0, TM_O = 256, TM_SF = 384;  // TMEM columns: S[0], S[1], O, scale factors
#ifndef AP_REUSE
#define AP_REUSE 1  // items with one key block: pass 2 reuses pass 1's S (no second K load / unpack / QK^T)
#endif
__device__ __forceinline__ uint32_t ap_fdiv(uint32_t n, const FastDiv& f) { return (__umulhi(n, f.mul) + n) >> f.shift; }
// The item of loop slot tr (= round k * gridDim + CTA b).  Causal items differ in length (q tile
// i reads i + 1 key blocks when tq == tk), so they go heaviest first (q tiles descending, entries
// fastest) and alternate rounds assign them in reverse CTA order (a zigzag, which pairs a CTA's
// heavy item with a light one): every CTA ends up with about the same number of key blocks.
template <typename P>
__device__ __forceinline__ int64_t item_at(const P& p, int64_t tr) {
    if (!p.causal) return tr;
    const uint32_t g = gridDim.x, k = uint32_t(tr) / g, b = uint32_t(tr) - k * g;
    const uint32_t i = k * g + ((k & 1) ? g - 1 - b : b);
    if (i >= uint32_t(p.items)) return p.items;
    const uint32_t r = ap_fdiv(i, p.fd_ent);          // heaviness rank: q tile = Q - 1 - r
    const uint32_t e = i - r * p.fd_ent.d;
    return int64_t(e) * p.fd_qt.d + (p.fd_qt.d - 1 - r);
}
// key blocks an item reads: all of them, or (causal) those holding a key <= the tile's last row + coff
template <typename P>
__device__ __forceinline__ int item_blocks(const P& p, int64_t t) {
    if (!p.causal) return p.nblk;
    const int64_t q0 = int64_t(uint32_t(t) - ap_fdiv(uint32_t(t), p.fd_qt) * p.fd_qt.d) * 128;
    int64_t last = q0 + 127;
    if (last > p.tq - 1) last = p.tq - 1;
    const int64_t nb = (last + p.coff) / 128 + 1;
    return int(nb < p.nblk ? nb : p.nblk);
}

struct ApParams {
    FastDiv fd_qt, fd_nh;  // item -> (entry, q tile), entry -> (batch, head): 32-bit multiply-shift
    int causal;            // row i sees keys j <= i + coff only; key blocks past the tile's last row skipped
    FastDiv fd_ent;        // entries (causal schedule)
    int64_t coff;          // tk - tq
    int64_t nh, tq, tk;
    int dh, dhp;           // head_dim, rounded up to 16 (PV MMA N, V^T box rows)
    int q_tiles, nblk;
    int64_t items;
    int k_kind;            // B_TERNARY or B_BINARY
    int neg;               // alpha < 0: Q codes negated
    float alpha;           // |alpha|
    const float* alpha_h;  // per-head alpha [nh] (nullable; signed: negative heads negate their Q codes)
    const float* beta_h;   // per-head beta [nh] (nullable)
    float p_t;             // bool threshold as a p_dt storage value (R2)
    int p_dt;
    float beta;
    void* o;
    int o_dt;
    int64_t ld_o, o_bs, o_hs;  // elements
    int vec_o;                 // fp16/bf16 O with 16-byte aligned rows and strides
    int q_wide, k_wide;        // Q / K planes with ld == 4 and rows % 16 == 0: 256-byte TMA rows
    int dbg;  // BWTA_TRACE builds only: 1 skip pass-1 math, 2 skip pass-2 math, 4 skip MMAs, 8 skip unpack, 16 spin on S
    uint32_t* p_out;           // optional P planes [entries][tq][p_ld] (zeroed by the host)
    int64_t p_ld;
    // fused next-layer pack of the context (N2): instead of O, the planes of the [B*Tq, H*Dh]
    // context rows, head h owning words [h Dh/32, (h+1) Dh/32) of row b*Tq + t (Dh % 32 == 0);
    // +1 iff fl32(dot * beta) >= po_tp, -1 iff <= -po_tn (the o_dt rounding boundaries, R2)
    int pack_out, po_kind;
    uint32_t *po_sgn, *po_nz;
    int64_t po_ld;
    float po_tp, po_tn;
};

__device__ __forceinline__ float round_to(int dt, float p) {
    if (dt == DT_F16) return __half2float(__float2half_rn(p));
    if (dt == DT_BF16) return __bfloat162float(__float2bfloat16_rn(p));
    return p;
}
__device__ __forceinline__ float lds_f32(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void wait_bar(uint64_t* b, uint32_t parity) {
    while (!mbar_try_wait_nh(b, parity)) {
    }
}
__device__ __forceinline__ void wait_spin(uint64_t* b, uint32_t parity) {
    while (!mbar_test_wait(b, parity)) {
    }
}

// one 128-element row of Q (ternary): unpack like unpack_row<B_TERNARY, 128>, optionally negated
__device__ __forceinline__ void unpack_q_row(uint32_t sgn_addr, uint32_t nz_addr, uint32_t rowaddr, int r, bool neg) {
    const int sw = (r >> 1) & 3;
    const uint4 s4 = lds128(sgn_addr), n4 = lds128(nz_addr);
    const uint32_t sg[4] = {s4.x, s4.y, s4.z, s4.w}, nz[4] = {n4.x, n4.y, n4.z, n4.w};
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        const uint32_t x1 = nz[g], x0 = neg ? (nz[g] & ~sg[g]) : (sg[g] & nz[g]);
        uint32_t o[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) o[j] = unpack_word<B_TERNARY>(x0, x1, j);
        sts128(rowaddr + ((g ^ sw) << 4), o[0], o[1], o[2], o[3]);
    }
}

// bit(d): R13's expression for an integer dot d (|alpha|-scaled, the row's s_max and z)
__device__ __forceinline__ bool p_bit(const ApParams& p, float alpha, int d, float mx, float z) {
    const float s = __fmul_rn(float(d), alpha);
    return round_to(p.p_dt, __fdiv_rn(expf(__fsub_rn(s, mx)), z)) >= p.p_t;
}

__global__ void __launch_bounds__(AP_NT, 1)
    attn_prefill_kernel(const __grid_constant__ CUtensorMap tmQs, const __grid_constant__ CUtensorMap tmQn,
                        const __grid_constant__ CUtensorMap tmKs, const __grid_constant__ CUtensorMap tmKn,
                        const __grid_constant__ CUtensorMap tmVs, const __grid_constant__ CUtensorMap tmVn,
                        ApParams p) {
    extern __shared__ __align__(16) uint8_t ap_smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(ap_smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = sm;                                   // 2 x Q codes (double-buffered across items)
    uint8_t* sStage = sQ + 2 * Q_CODES;                 // [stage]{K codes, K bits}
    uint8_t* sVc = sStage + AP_S * STAGE_B;             // [stage] V^T codes
    uint8_t* sV = sVc + AP_VS * V_CODES;                // 2 V^T chunks (bits, 1024 keys)
    uint8_t* sP = sV + 2 * VCH_B;                       // 2 P code buffers
    uint8_t* sQb = sP + 2 * P_CODES;                    // 2 x Q bits (sgn plane, nz plane)
    float* tbl = reinterpret_cast<float*>(sQb + 2 * Q_BITS);     // exp(|alpha| (i - 2 Dh_max)), 2 KB
    // (per-head alphas: tbl[0..512) and tbl[512..1024) alternate between items)
    float* mrg = tbl + 1024;                                      // [2 parity][AP_NH slices][128 rows][R, z]
    uint64_t* bars = reinterpret_cast<uint64_t*>(mrg + 2 * AP_NH * AP_BQ * 2);
    uint64_t* k_full = bars;
    uint64_t* k_ready = k_full + AP_S;
    uint64_t* k_empty = k_ready + AP_S;
    uint64_t* v_ready = k_empty + AP_S;
    uint64_t* v_empty = v_ready + AP_VS;
    uint64_t* s_full = v_empty + AP_VS;
    uint64_t* s_free = s_full + 2;
    uint64_t* p_ready = s_free + 2;
    uint64_t* p_free = p_ready + 2;
    uint64_t* q_full = p_free + 2;
    uint64_t* q_ready = q_full + 2;
    uint64_t* q_empty = q_ready + 2;
    uint64_t* o_full = q_empty + 2;
    uint64_t* o_free = o_full + 1;
    uint64_t* vc_full = o_free + 1;
    uint64_t* vc_empty = vc_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(vc_empty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmQs);
        tma_prefetch_desc(&tmQn);
        tma_prefetch_desc(&tmKs);
        if (p.k_kind == B_TERNARY) tma_prefetch_desc(&tmKn);
        tma_prefetch_desc(&tmVs);
        tma_prefetch_desc(&tmVn);
        for (int s = 0; s < AP_S; ++s) {
            mbar_init(&k_full[s], 1);
            mbar_init(&k_ready[s], 4);
            mbar_init(&k_empty[s], 1);
        }
        for (int s = 0; s < AP_VS; ++s) {
            mbar_init(&v_ready[s], 4);
            mbar_init(&v_empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&s_full[b], 1);
            mbar_init(&s_free[b], AP_SMW);
            mbar_init(&p_ready[b], AP_SMW);
            mbar_init(&p_free[b], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&q_full[b], 1);
            mbar_init(&q_ready[b], 4);
            mbar_init(&q_empty[b], 1);
        }
        mbar_init(o_full, 1);
        mbar_init(o_free, AP_SMW);
        for (int b = 0; b < 2; ++b) {
            mbar_init(&vc_full[b], 1);
            mbar_init(&vc_empty[b], 4);
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, 512);
    if (warp == 3)
        for (int i = lane; i < AP_TBL; i += 32) tbl[i] = expf(__fmul_rn(float(i - 2 * AP_DH), p.alpha));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (warp >= 8 && warp < 12) {  // UE8M0 scale factors = 1.0 in columns TM_SF .. TM_SF + 15
        uint32_t ones[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) ones[i] = 0x7F7F7F7Fu;
        tmem_st_32x32b_x16(tmem + (uint32_t((warp & 3) * 32) << 16) + uint32_t(TM_SF), ones);
        tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_launch_dependents();
    pdl_wait();

    if (warp == 0) {
        // ------------------------------ TMA producer ------------------------------
        if (lane == 0) {
            const uint32_t kbytes = uint32_t((p.k_kind == B_TERNARY ? 2 : 1) * AP_BK * 16);
            const uint32_t vbytes = uint32_t(2 * p.dhp * VCH_W * 4);
            int g = 0, ic = 0, vc = 0;
            for (int64_t tr = blockIdx.x; tr - blockIdx.x < p.items; tr += gridDim.x, ++ic) {
            const int64_t t = item_at(p, tr);
            if (t >= p.items) continue;  // (only in the last round)
                const uint32_t e = ap_fdiv(uint32_t(t), p.fd_qt);
                const int q0 = int(uint32_t(t) - e * p.fd_qt.d) * AP_BQ;
                const uint32_t eb_ = ap_fdiv(e, p.fd_nh);
                const int eb = int(eb_), eh = int(e - eb_ * p.fd_nh.d);
                const int qb = ic & 1;
                wait_bar(&q_empty[qb], uint32_t((ic >> 1) & 1) ^ 1u);
                mbar_arrive_expect_tx(&q_full[qb], uint32_t(2 * AP_BQ * 16));
                // wide maps: [rows / 16][64 words] views of the contiguous 16-byte rows (box 8 x 256 B)
                const int qr = p.q_wide ? q0 / 16 : q0;
                uint8_t* qbits = sQb + qb * Q_BITS;
                tma_load_4d(qbits, &tmQs, &q_full[qb], 0, qr, eh, eb);
                tma_load_4d(qbits + AP_BQ * 16, &tmQn, &q_full[qb], 0, qr, eh, eb);
                const int nbi = item_blocks(p, t);
                const bool reuse = AP_REUSE && nbi == 1;  // one key block: pass 2 reuses pass 1's S
                for (int pass = 0; pass < 2; ++pass) {
                    for (int j = 0; j < nbi; ++j) {
                        if (pass && j % VCH_BLK == 0) {  // the next 1024 keys of V^T (both planes)
                            const int cb = vc & 1;
                            wait_bar(&vc_empty[cb], uint32_t((vc >> 1) & 1) ^ 1u);
                            uint8_t* vb = sV + cb * VCH_B;
                            mbar_arrive_expect_tx(&vc_full[cb], vbytes);
                            tma_load_4d(vb, &tmVs, &vc_full[cb], VCH_W * (j / VCH_BLK), 0, eh, eb);
                            tma_load_4d(vb + p.dhp * VCH_W * 4, &tmVn, &vc_full[cb], VCH_W * (j / VCH_BLK), 0, eh, eb);
                            ++vc;
                        }
                        if (pass && reuse) continue;  // no second K load
                        const int st = g % AP_S;
                        ++g;
                        wait_bar(&k_empty[st], uint32_t(((g - 1) / AP_S) & 1) ^ 1u);
                        uint8_t* kb = sStage + st * STAGE_B + K_CODES;
                        const int kr = p.k_wide ? j * (AP_BK / 16) : j * AP_BK;
                        mbar_arrive_expect_tx(&k_full[st], kbytes);
                        tma_load_4d(kb, &tmKs, &k_full[st], 0, kr, eh, eb);
                        if (p.k_kind == B_TERNARY) tma_load_4d(kb + AP_BK * 16, &tmKn, &k_full[st], 0, kr, eh, eb);
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------ MMA issuer ------------------------------
        const uint32_t idesc_qk = idesc_mxf4(AP_BQ, AP_BK), idesc_pv = idesc_mxf4(AP_BQ, p.dhp);
        // the whole warp issues (elect.sync inside the asm): operands stay in uniform registers
        const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem, 0);
        const uint32_t sf = tmem_u + uint32_t(TM_SF);
        int g = 0, sg = 0, pg = 0, ic = 0;
        // QK^T of K stage st into S buffer sb; the K stage is free again once these MMAs complete
        auto qk = [&](uint32_t qa, int st, int sb) {
            const uint32_t kc = smem_u32(sStage + st * STAGE_B);
            // K = head_dim in MMAs of 64 (the second is all zero codes when head_dim <= 64: skipped)
            if (!(p.dbg & 4))
#pragma unroll
            for (int k = 0; k < 2; ++k)
                if (k == 0 || p.dh > 64)
                    mma_mxf4_w(tmem_u + uint32_t(TM_S + sb * AP_BK), smem_desc_sw64(qa + 32 * k),
                               smem_desc_sw64(kc + 32 * k), idesc_qk, sf, sf + 8, k);
            tc_commit_w(&s_full[sb]);
            tc_commit_w(&k_empty[st]);
        };
        for (int64_t tr = blockIdx.x; tr - blockIdx.x < p.items; tr += gridDim.x, ++ic) {
            const int64_t t = item_at(p, tr);
            if (t >= p.items) continue;  // (only in the last round)
            const int nbi = item_blocks(p, t);
            const int qb = ic & 1;
            const uint32_t qa = smem_u32(sQ + qb * Q_CODES);
            wait_bar(&q_ready[qb], uint32_t((ic >> 1) & 1));
            tc_fence_after();
            // pass 1: S blocks for the row statistics
            for (int j = 0; j < nbi; ++j, ++g, ++sg) {
                const int st = g % AP_S, sb = sg & 1;
                wait_bar(&k_ready[st], uint32_t((g / AP_S) & 1));
                wait_bar(&s_free[sb], uint32_t((sg >> 1) & 1) ^ 1u);
                tc_fence_after();
                qk(qa, st, sb);
                __syncwarp();
            }
            // pass 2: QK^T of block j + 1 is issued before PV of block j (S is double-buffered); with
            // one key block pass 1's S is still in its buffer (the softmax warps hold it): no second QK^T
            const bool reuse = AP_REUSE && nbi == 1;
            if (reuse) tc_commit_w(&q_empty[qb]);  // the Q codes' last reader was pass 1's QK^T
            for (int j = 0; j <= nbi; ++j) {
                if (j < nbi && !reuse) {
                    const int gj = g + j, sgj = sg + j, st = gj % AP_S, sb = sgj & 1;
                    wait_bar(&k_ready[st], uint32_t((gj / AP_S) & 1));
                    wait_bar(&s_free[sb], uint32_t((sgj >> 1) & 1) ^ 1u);
                    tc_fence_after();
                    qk(qa, st, sb);
                    if (j == nbi - 1) tc_commit_w(&q_empty[qb]);  // the last read of this item's Q codes
                    __syncwarp();
                }
                if (j >= 1) {
                    const int jj = j - 1, pb = pg & 1, vs = pg % AP_VS;
                    wait_bar(&p_ready[pb], uint32_t((pg >> 1) & 1));
                    wait_bar(&v_ready[vs], uint32_t((pg / AP_VS) & 1));
                    if (jj == 0) wait_bar(o_free, uint32_t(ic & 1) ^ 1u);
                    tc_fence_after();
                    {
                        const uint32_t pa = smem_u32(sP + pb * P_CODES);
                        const uint32_t vcd = smem_u32(sVc + vs * V_CODES);
                        if (!(p.dbg & 4))
#pragma unroll
                        for (int k = 0; k < 2; ++k)
                            mma_mxf4_w(tmem_u + uint32_t(TM_O), smem_desc_sw64(pa + 32 * k), smem_desc_sw64(vcd + 32 * k),
                                       idesc_pv, sf, sf + 8, (jj | k) != 0);
                        tc_commit_w(&p_free[pb]);
                        tc_commit_w(&v_empty[vs]);
                        if (jj == nbi - 1) tc_commit_w(o_full);
                    }
                    __syncwarp();
                    ++pg;
                }
            }
            if (!reuse) {
                g += nbi;
                sg += nbi;
            }
        }
    } else if (warp >= 4 && warp < 8) {
        // ------------------------------ unpack (Q, K, V^T planes -> codes) ------------------------------
        const int ut = threadIdx.x - 128;
        int g = 0, ic = 0, vc = 0, pg = 0;
        for (int64_t tr = blockIdx.x; tr - blockIdx.x < p.items; tr += gridDim.x, ++ic) {
            const int64_t t = item_at(p, tr);
            if (t >= p.items) continue;  // (only in the last round)
            const int nbi = item_blocks(p, t);
            const int qb = ic & 1;
            wait_bar(&q_full[qb], uint32_t((ic >> 1) & 1));
            const uint32_t qbits = smem_u32(sQb + qb * Q_BITS);
            const uint32_t e_ = ap_fdiv(uint32_t(t), p.fd_qt);
            const bool negq = p.alpha_h ? (__ldg(p.alpha_h + (e_ - ap_fdiv(e_, p.fd_nh) * p.fd_nh.d)) < 0.f) : p.neg != 0;
            unpack_q_row(qbits + ut * 16, qbits + AP_BQ * 16 + ut * 16, smem_u32(sQ + qb * Q_CODES) + ut * CODE_ROW, ut,
                         negq);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&q_ready[qb]);
            const bool reuse = AP_REUSE && nbi == 1;
            for (int pass = 0; pass < 2; ++pass) {
                for (int j = 0; j < nbi; ++j) {
                    if (!(pass && reuse)) {  // (one key block: no second K unpack)
                        const int st = g % AP_S;
                        wait_bar(&k_full[st], uint32_t((g / AP_S) & 1));
                        ++g;
                        const uint32_t kc = smem_u32(sStage + st * STAGE_B);
                        if (!(p.dbg & 8)) unpack_rows<128>(p.k_kind, kc + K_CODES, AP_BK * 16, kc, ut, AP_BK, 128);
                        fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&k_ready[st]);
                    }
                    if (pass) {
                        const int cb = vc & 1, vs = pg % AP_VS;
                        if (j % VCH_BLK == 0) wait_bar(&vc_full[cb], uint32_t((vc >> 1) & 1));
                        wait_bar(&v_empty[vs], uint32_t((pg / AP_VS) & 1) ^ 1u);
                        // V^T rows of this block: words 4 (j % 8) .. + 3 of the chunk's 128-byte rows
                        const uint32_t ch = smem_u32(sV + cb * VCH_B) + 16 * (j % VCH_BLK);
                        const uint32_t vcd = smem_u32(sVc + vs * V_CODES);
                        for (int r = ut; r < p.dhp && !(p.dbg & 8); r += 128)
                            unpack_row<B_TERNARY, 128>(ch + r * VCH_W * 4, ch + (p.dhp + r) * VCH_W * 4,
                                                       vcd + r * CODE_ROW, r);
                        fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            mbar_arrive(&v_ready[vs]);
                            if (j % VCH_BLK == VCH_BLK - 1 || j == nbi - 1) mbar_arrive(&vc_empty[cb]);
                        }
                        if (j % VCH_BLK == VCH_BLK - 1 || j == nbi - 1) ++vc;
                        ++pg;
                    }
                }
            }
        }
    } else if (warp >= 8) {
        // ------------------------------ softmax, P codes, epilogue ------------------------------
        const int q = warp & 3, h = (warp - 8) >> 2;
        const int r = 32 * q + lane;                       // query row within the tile = TMEM lane
        const uint32_t lane_base = tmem + (uint32_t(32 * q) << 16);
        const float MAGIC = 12582912.f;                    // 1.5 * 2^23: float_as_int(x + MAGIC) = 0x4B400000 + x
        int sg = 0, pg = 0, ic = 0;
        for (int64_t tr = blockIdx.x; tr - blockIdx.x < p.items; tr += gridDim.x, ++ic) {
            const int64_t t = item_at(p, tr);
            if (t >= p.items) continue;  // (only in the last round)
            const int nbi = item_blocks(p, t);
            const uint32_t e = ap_fdiv(uint32_t(t), p.fd_qt);
            const int64_t qrow = int64_t(uint32_t(t) - e * p.fd_qt.d) * AP_BQ + r;
            const uint32_t eb_ = ap_fdiv(e, p.fd_nh);
            const int eb = int(eb_), eh = int(e - eb_ * p.fd_nh.d);
            // keys this row may see: all tk, or (causal) those <= qrow + coff (masked keys are not keys:
            // out of the max, the normaliser and P, exactly as keys past tk)
            const int64_t klim = p.causal ? (qrow + p.coff + 1 < p.tk ? qrow + p.coff + 1 : p.tk) : p.tk;
            float alpha = p.alpha, beta = p.beta;
            uint32_t tbl_s = smem_u32(tbl);
            if (p.alpha_h) {  // this head's |alpha|: its own exp table (double-buffered by item parity)
                alpha = fabsf(__ldg(p.alpha_h + eh));
                float* tb = tbl + 512 * (ic & 1);
                for (int i = threadIdx.x - 256; i < AP_TBL; i += 32 * AP_SMW)
                    tb[i] = expf(__fmul_rn(float(i - 2 * AP_DH), alpha));
                named_bar(5, 32 * AP_SMW);  // every softmax warp sees the table before using it
                tbl_s = smem_u32(tb);
            }
            if (p.beta_h) beta = __ldg(p.beta_h + eh);
            // ---- pass 1: R = running max of the integer dots (|alpha|-signed), z = sum exp(|alpha| (d - R))
            // (one key block: its S buffer is kept for pass 2 -- released after pass 2 reads it)
            const bool reuse = AP_REUSE && nbi == 1;
            float R = -INFINITY, z = 0.f;
            for (int j = 0; j < nbi; ++j, ++sg) {
                const int sb = sg & 1;
                if (p.dbg & 16) wait_spin(&s_full[sb], uint32_t((sg >> 1) & 1));
                else wait_bar(&s_full[sb], uint32_t((sg >> 1) & 1));
                tc_fence_after();
                const int64_t k0 = int64_t(j) * AP_BK + AP_KW * h;
                const int valid = klim - k0 >= AP_KW ? AP_KW : int(klim - k0 > 0 ? klim - k0 : 0);
#pragma unroll 1
                for (int gg = 0; gg < AP_NG; ++gg) {  // 32 keys at a time (register budget)
                    uint32_t v[32];
                    tmem_ld_32x32b_x32(lane_base + uint32_t(TM_S + sb * AP_BK + AP_KW * h + 32 * gg), v);
                    tmem_wait_ld();
                    if (gg == AP_NG - 1 && !reuse) {
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&s_free[sb]);
                    }
                    const int vg = (p.dbg & 1) ? 0 : valid - 32 * gg;
                    if (vg <= 0) continue;
                    float bm = -INFINITY;
                    if (vg >= 32) {
#pragma unroll
                        for (int c = 0; c < 32; ++c) bm = fmaxf(bm, __uint_as_float(v[c]));
                    } else {
#pragma unroll
                        for (int c = 0; c < 32; ++c)
                            if (c < vg) bm = fmaxf(bm, __uint_as_float(v[c]));
                    }
                    if (bm > R) {
                        if (R != -INFINITY) z *= lds_f32(tbl_s + 4 * (int(R - bm) + 2 * AP_DH));
                        R = bm;
                    }
                    // byte address of exp(|alpha| (d - R)): float_as_int(4 d + MAGIC) + (table + 4 (2 Dh) -
                    // float_as_int(4 R + MAGIC)) -- one FFMA and one IADD per score (4 |d| < 2^22: exact)
                    const uint32_t rb = tbl_s + 4 * 2 * AP_DH - uint32_t(__float_as_int(__fmaf_rn(R, 4.f, MAGIC)));
                    float zs = 0.f;
                    if (vg >= 32) {
#pragma unroll
                        for (int c = 0; c < 32; ++c)
                            zs += lds_f32(uint32_t(__float_as_int(__fmaf_rn(__uint_as_float(v[c]), 4.f, MAGIC))) + rb);
                    } else {
#pragma unroll
                        for (int c = 0; c < 32; ++c)
                            if (c < vg)
                                zs += lds_f32(uint32_t(__float_as_int(__fmaf_rn(__uint_as_float(v[c]), 4.f, MAGIC))) + rb);
                    }
                    z += zs;
                }
            }
            // ---- merge the row's key slices (fixed order h = 0, 1, ...)
            float* mb = mrg + (ic & 1) * (AP_NH * AP_BQ * 2);
            mb[(h * AP_BQ + r) * 2] = R;
            mb[(h * AP_BQ + r) * 2 + 1] = z;
            named_bar(1 + q, 32 * AP_NH);
            float Rm = -INFINITY;
#pragma unroll
            for (int hh = 0; hh < AP_NH; ++hh) Rm = fmaxf(Rm, mb[(hh * AP_BQ + r) * 2]);
            float zt = 0.f;
#pragma unroll
            for (int hh = 0; hh < AP_NH; ++hh) {
                const float Rh = mb[(hh * AP_BQ + r) * 2], zh = mb[(hh * AP_BQ + r) * 2 + 1];
                if (Rh != -INFINITY) zt += zh * lds_f32(tbl_s + 4 * (int(Rh - Rm) + 2 * AP_DH));
            }
            // ---- the row's integer threshold: bit(d) <=> d >= dthr (binary search over [-Dh, Rm + 1])
            const float mx = __fmul_rn(Rm, alpha);
            int lo = -p.dh, hi = int(Rm) + 1;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;  // floor for negatives too
                if (p_bit(p, alpha, mid, mx, zt)) hi = mid;
                else lo = mid + 1;
            }
            const float dthr = float(lo);
            // ---- pass 2: P codes of each block, then O += P . V^T on the tensor core
            if (reuse) --sg;  // the same S buffer and phase as pass 1
            for (int j = 0; j < nbi; ++j, ++sg, ++pg) {
                const int sb = sg & 1, pb = pg & 1;
                if (p.dbg & 16) wait_spin(&s_full[sb], uint32_t((sg >> 1) & 1));
                else wait_bar(&s_full[sb], uint32_t((sg >> 1) & 1));
                tc_fence_after();
                const int64_t k0 = int64_t(j) * AP_BK + AP_KW * h;
                const int valid = klim - k0 >= AP_KW ? AP_KW : int(klim - k0 > 0 ? klim - k0 : 0);
                uint32_t code[AP_NG][4], bits[AP_NG];
#pragma unroll
                for (int gg = 0; gg < AP_NG; ++gg) {
                    uint32_t v[32];
                    tmem_ld_32x32b_x32(lane_base + uint32_t(TM_S + sb * AP_BK + AP_KW * h + 32 * gg), v);
                    tmem_wait_ld();
                    uint32_t bw = 0;
                    if (!(p.dbg & 2))
#pragma unroll
                    for (int k = 0; k < 32; ++k) bw |= uint32_t(__uint_as_float(v[k]) >= dthr) << k;
                    const int vg = valid - 32 * gg;  // keys >= Tk (zero K rows) are not keys
                    bw &= vg >= 32 ? 0xffffffffu : (vg <= 0 ? 0u : (1u << vg) - 1u);
                    bits[gg] = bw;
                    // code word jw holds keys {jw, 4 + jw, ..., 28 + jw} of the group, nibble i = key 4i + jw
                    // (the tc_codes.cuh order), +1.0 = 0x2: one shift and mask per word
#pragma unroll
                    for (int jw = 0; jw < 4; ++jw) code[gg][jw] = ((bw >> jw) & 0x11111111u) << 1;
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&s_free[sb]);
                wait_bar(&p_free[pb], uint32_t((pg >> 1) & 1) ^ 1u);
                const uint32_t prow = smem_u32(sP + pb * P_CODES) + r * CODE_ROW;
                const int sw = (r >> 1) & 3;
#pragma unroll
                for (int gg = 0; gg < AP_NG; ++gg)
                    sts128(prow + (((AP_NG * h + gg) ^ sw) << 4), code[gg][0], code[gg][1], code[gg][2], code[gg][3]);
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&p_ready[pb]);
                if (p.p_out && qrow < p.tq) {
                    uint32_t* po = p.p_out + (e * p.tq + qrow) * p.p_ld;
#pragma unroll
                    for (int gg = 0; gg < AP_NG; ++gg)
                        if (valid > 32 * gg) po[k0 / 32 + gg] = bits[gg];
                }
            }
            // ---- epilogue: O (exact integer dots) -> fl32(dot * beta) -> o_dt
            wait_bar(o_full, uint32_t(ic & 1));
            tc_fence_after();
            const bool rok = qrow < p.tq;
            const int64_t obase = int64_t(eb) * p.o_bs + int64_t(eh) * p.o_hs + qrow * p.ld_o;
            if (p.pack_out) {  // 32-column chunks -> one word per plane per thread
                for (int c0 = 32 * h; c0 < p.dh; c0 += 32 * AP_NH) {
                    uint32_t o[32];
                    tmem_ld_32x32b_x32(lane_base + uint32_t(TM_O + c0), o);
                    tmem_wait_ld();
                    uint32_t pos = 0, neg = 0;
#pragma unroll
                    for (int c = 0; c < 32; ++c) {
                        const float y = __fmul_rn(__uint_as_float(o[c]), beta);  // R5
                        pos |= uint32_t(y >= p.po_tp) << c;
                        neg |= uint32_t(y <= -p.po_tn) << c;
                    }
                    if (rok) {
                        const int64_t off = (int64_t(eb) * p.tq + qrow) * p.po_ld + (int64_t(eh) * p.dh + c0) / 32;
                        p.po_nz[off] = p.po_kind == K_TERNARY ? (pos | neg) : pos;
                        if (p.po_kind == K_TERNARY) p.po_sgn[off] = neg;
                    }
                }
            } else
            for (int c0 = 16 * h; c0 < p.dhp; c0 += 16 * AP_NH) {
                uint32_t o[16];
                tmem_ld_32x32b_x16(lane_base + uint32_t(TM_O + c0), o);
                tmem_wait_ld();
                if (rok) {
                    if (p.vec_o && c0 + 16 <= p.dh) {  // fp16 / bf16, 16-byte aligned rows: two 16-byte stores
                        uint32_t w[8];
#pragma unroll
                        for (int c = 0; c < 8; ++c) {
                            const float y0 = __fmul_rn(__uint_as_float(o[2 * c]), beta);
                            const float y1 = __fmul_rn(__uint_as_float(o[2 * c + 1]), beta);
                            if (p.o_dt == DT_F16) {
                                __half2 hv = __halves2half2(__float2half_rn(y0), __float2half_rn(y1));
                                w[c] = *reinterpret_cast<uint32_t*>(&hv);
                            } else {
                                __nv_bfloat162 hv = __halves2bfloat162(__float2bfloat16_rn(y0), __float2bfloat16_rn(y1));
                                w[c] = *reinterpret_cast<uint32_t*>(&hv);
                            }
                        }
                        uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(p.o) + obase + c0);
                        dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
                        dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
                    } else {
#pragma unroll
                        for (int c = 0; c < 16; ++c) {
                            if (c0 + c < p.dh) {
                                const float acc = __uint_as_float(o[c]);
                                const float y = __fmul_rn(acc, beta);
                                const int64_t off = obase + c0 + c;
                                if (p.o_dt == DT_F16) reinterpret_cast<__half*>(p.o)[off] = __float2half_rn(y);
                                else if (p.o_dt == DT_BF16) reinterpret_cast<__nv_bfloat16*>(p.o)[off] = __float2bfloat16_rn(y);
                                else if (p.o_dt == DT_F32) reinterpret_cast<float*>(p.o)[off] = y;
                                else reinterpret_cast<int32_t*>(p.o)[off] = __float2int_rn(acc);
                            }
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(o_free);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

}  // namespace

bool attn_prefill_supported(const AttnPrefillArgs& a) {
    return a.dh >= 1 && a.dh <= AP_DH && a.tq >= 1 && a.tk >= 1 && encode_fn() != nullptr;
}

cudaError_t launch_attn_prefill(const AttnPrefillArgs& a, cudaStream_t s) {
    const int64_t entries = a.nb * a.nh;
    ApParams p{};
    p.nh = a.nh;
    p.tq = a.tq;
    p.tk = a.tk;
    p.dh = int(a.dh);
    p.dhp = int((a.dh + 15) / 16 * 16);
    p.q_tiles = int((a.tq + AP_BQ - 1) / AP_BQ);
    p.nblk = int((a.tk + AP_BK - 1) / AP_BK);
    p.items = entries * p.q_tiles;
    p.causal = a.causal;
    p.coff = a.tk - a.tq;
    p.fd_ent = make_fastdiv(uint32_t(entries));
    if (a.causal && a.tk < a.tq) return cudaErrorInvalidValue;  // every row needs at least one key
    if (p.items >= (int64_t(1) << 31) || a.nh >= (int64_t(1) << 31)) return cudaErrorNotSupported;
    p.fd_qt = make_fastdiv(uint32_t(p.q_tiles));
    p.fd_nh = make_fastdiv(uint32_t(a.nh));
    p.k_kind = a.k_nz ? B_TERNARY : B_BINARY;
    p.neg = a.alpha < 0.f ? 1 : 0;
    p.alpha = fabsf(a.alpha);
    p.p_t = a.p_t;
    p.p_dt = a.p_dt;
    p.beta = a.beta;
    p.alpha_h = a.alpha_h;
    p.beta_h = a.beta_h;
    p.o = a.o;
    p.o_dt = a.o_dt;
    p.ld_o = a.ld_o;
    p.o_bs = a.o_bs;
    p.o_hs = a.o_hs;
    p.p_out = a.p_out;
    p.p_ld = a.p_ld;
    p.pack_out = a.pack_out;
    p.po_kind = a.po_kind;
    p.po_sgn = a.po_sgn;
    p.po_nz = a.po_nz;
    p.po_ld = a.po_ld;
    p.po_tp = a.po_tp;
    p.po_tn = a.po_tn;
    p.vec_o = (a.o_dt == DT_F16 || a.o_dt == DT_BF16) && (reinterpret_cast<uintptr_t>(a.o) & 15) == 0 &&
              a.ld_o % 8 == 0 && a.o_bs % 8 == 0 && a.o_hs % 8 == 0;
    CUtensorMap qs, qn, ks, kn, vs, vn;
    // Q / K: 128 rows of 16 B per box -- as 8 rows of 256 B when the rows are contiguous (ld == 4,
    // rows % 16 == 0: TMA moves 256-byte rows far faster than 16-byte ones); V^T: chunks of 32
    // words (1024 keys) x dhp rows, 128-byte rows
#ifdef BWTA_TRACE
    if (const char* d = getenv("BWTA_DBG")) p.dbg = atoi(d);  // experiment switches (trace builds only)
#endif
    p.q_wide = a.ldq == 4 && a.tq % 16 == 0;
    p.k_wide = a.ldk == 4 && a.tk % 16 == 0;
    auto wide = [&](CUtensorMap* m, const uint32_t* base, int64_t rows, int64_t hs, int64_t bs) {
        const uint64_t dims[4] = {64, uint64_t(rows / 16), uint64_t(a.nh), uint64_t(a.nb)};
        const uint64_t hsb = bstride(a.nh, hs * 4, uint64_t(rows) * 16);
        const uint64_t str[3] = {256, hsb, bstride(a.nb, bs * 4, hsb * a.nh)};
        const uint32_t box[4] = {64, 8, 1, 1};
        return encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, const_cast<uint32_t*>(base), dims, str, box,
                      CU_TENSOR_MAP_SWIZZLE_NONE);
    };
    const bool ok_q = p.q_wide ? (wide(&qs, a.q_sgn, a.tq, a.q_hs, a.q_bs) && wide(&qn, a.q_nz, a.tq, a.q_hs, a.q_bs))
                               : (encode_planes(&qs, a.q_sgn, a.ldq, a.tq, a.q_hs, a.q_bs, a.nh, a.nb, AP_BQ, 4) &&
                                  encode_planes(&qn, a.q_nz, a.ldq, a.tq, a.q_hs, a.q_bs, a.nh, a.nb, AP_BQ, 4));
    const uint32_t* kn_base = a.k_nz ? a.k_nz : a.k_sgn;
    const bool ok_k = p.k_wide ? (wide(&ks, a.k_sgn, a.tk, a.k_hs, a.k_bs) && wide(&kn, kn_base, a.tk, a.k_hs, a.k_bs))
                               : (encode_planes(&ks, a.k_sgn, a.ldk, a.tk, a.k_hs, a.k_bs, a.nh, a.nb, AP_BK, 4) &&
                                  encode_planes(&kn, kn_base, a.ldk, a.tk, a.k_hs, a.k_bs, a.nh, a.nb, AP_BK, 4));
    if (!ok_q || !ok_k ||
        !encode_planes(&vs, a.v_sgn, a.ldv, a.dh, a.v_hs, a.v_bs, a.nh, a.nb, p.dhp, VCH_W) ||
        !encode_planes(&vn, a.v_nz, a.ldv, a.dh, a.v_hs, a.v_bs, a.nh, a.nb, p.dhp, VCH_W))
        return cudaErrorInvalidValue;
    static std::atomic<uint64_t> optin{0};  // per device
    if (cudaError_t e = ensure_smem_optin(attn_prefill_kernel, SMEM_AP, optin); e != cudaSuccess) return e;
    const int64_t grid = p.items < device_sms() ? p.items : device_sms();
    return launch_pdl(attn_prefill_kernel, dim3(unsigned(grid)), dim3(AP_NT), size_t(SMEM_AP), s, 1, qs, qn, ks, kn,
                      vs, vn, p);
}

}  // namespace bwta
