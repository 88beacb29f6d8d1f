// Internal declarations shared by the BWTA CUDA sources (not part of the ABI).
#pragma once
#include <cstdlib>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

namespace bwta {

// process-wide count of enqueued kernels / memsets (bwta_kernel_launches)
extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// Programmatic dependent launch (PDL).  Every library kernel is launched with
// programmatic stream serialization: it may start while its predecessor in
// the stream is still finishing, runs only prologue work (barrier init, TMEM
// allocation, descriptor prefetch) before pdl_wait(), and performs no global
// memory access before it.  pdl_wait() returns once the predecessor grid has
// completed and its memory is visible, so stream order is preserved.
// pdl_launch_dependents() lets the next kernel start its own prologue early.
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#endif

// cudaLaunchKernelEx with the PDL attribute (and an optional cluster size).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              int cluster, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    int n = 0;
    static const bool pdl_off = [] {  // BWTA_NO_PDL=1: plain stream order (A/B measurements only)
        const char* e = getenv("BWTA_NO_PDL");
        return e && atoi(e) != 0;
    }();
    if (!pdl_off) {
        attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[n].val.programmaticStreamSerializationAllowed = 1;
        ++n;
    }
    if (cluster > 1) {
        attr[n].id = cudaLaunchAttributeClusterDimension;
        attr[n].val.clusterDim.x = cluster;
        attr[n].val.clusterDim.y = 1;
        attr[n].val.clusterDim.z = 1;
        ++n;
    }
    cfg.attrs = attr;
    cfg.numAttrs = n;
    count_launch();
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// Per-device state.  One process may drive several GPUs: the SM count and every
// kernel's shared-memory opt-in are cached per device ordinal (lock-free atomics),
// not per process.
int device_sms();  // SM count of the current device (cached per device)
template <typename Kern>
inline cudaError_t ensure_smem_optin(Kern kernel, int bytes, std::atomic<uint64_t>& done_mask) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = (dev >= 0 && dev < 64) ? (uint64_t(1) << dev) : 0;
    if (bit && (done_mask.load(std::memory_order_acquire) & bit)) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess && bit) done_mask.fetch_or(bit, std::memory_order_release);
    return e;
}

enum Dt { DT_F16 = 0, DT_BF16 = 1, DT_F32 = 2, DT_I32 = 3 };
enum Kind { K_BINARY = 0, K_BOOL = 1, K_TERNARY = 2 };

// Thresholds in the storage type of x (see pack.cu: exact predicate rewrite).
//   q = +1  <=>  x >= tp        (tp = smallest storage value >= s/2)
//   q = -1  <=>  x <= ntn       (ntn = -(smallest storage value > s/2))
struct Thresholds {
    uint32_t tp2;   // f16/bf16: the 16-bit pattern of tp duplicated in both halves
    uint32_t ntn2;  // f16/bf16: the 16-bit pattern of ntn duplicated
    float tpf;      // f32 inputs
    float ntnf;
};

// n / d for 0 <= n < 2^31 with one IMAD.HI (Granlund-Montgomery round-up
// multiplier): q = (umulhi(n, mul) + n) >> shift.
struct FastDiv {
    uint32_t d, mul, shift;
};
inline FastDiv make_fastdiv(uint32_t d) {
    FastDiv f{d, 0, 0};
    while ((1ull << f.shift) < d) ++f.shift;
    f.mul = uint32_t(((1ull << 32) * ((1ull << f.shift) - d)) / d + 1);
    if (d == 1) f.mul = 0;
    return f;
}

struct PackArgs {
    const void* x;
    int dt;
    int64_t nb, nh, rows, cols, ld_x, x_bs, x_hs;  // elements
    int kind;
    uint32_t* sgn;
    uint32_t* nz;
    int64_t ldw, p_bs, p_hs;  // words
    int32_t* row_nnz;
    const float* mu;  // binary (weights) only
    int mu_per_row;
    Thresholds th;
    bool vec_ok;  // x rows are 16-byte aligned -> 128-bit loads
    bool planes_dense;  // planes are [entries][rows][ldw] contiguous -> word offset = flat index
    int64_t nwd;        // data words per packed row, max(1, ceil(cols / 32)); lanes own data words only
    FastDiv div_nwd, div_rows, div_nh;  // for the 32-bit index path
};

cudaError_t launch_pack_rows(const PackArgs& a, cudaStream_t s);
cudaError_t launch_pack_cols(const PackArgs& a, cudaStream_t s);
constexpr int PACK_GROUP_MAX = 4;
constexpr int MAX_PEERS = 7;  // bwta_gemm_peers: up to 8 GPUs of one NVSwitch node
// several activation packs in one launch (falls back to one launch each)
cudaError_t launch_pack_group(const PackArgs* a, const int* transpose, int n, cudaStream_t s);

// ---------------------------------------------------------------------------
// Bit-serial matmul (design (a)) and the generic matmul description shared by
// both designs.  Entry e = b*nh + h; operand X at base + b*X_bs + h*X_hs.
//   dot[i][j] = sum_w  popc(m) - 2 popc(m & (a_sgn ^ b_sgn)),  m = a_nz & b_nz
// with absent planes read as sgn = 0, nz = all-ones.
// Epilogue: c = col_scale ? fl32(col_scale[j] * scalar) : scalar
//           y = fl32(float(dot) * c) -> out_dt (I32: raw dot)
// ---------------------------------------------------------------------------
struct MatmulArgs {
    const uint32_t* a_sgn;
    const uint32_t* a_nz;
    const uint32_t* b_sgn;
    const uint32_t* b_nz;
    int64_t M, N, K;        // K in elements
    int64_t lda, ldb;       // words
    int64_t a_bs, a_hs, b_bs, b_hs;  // words
    int64_t nb, nh;
    void* y;
    int y_dt;
    int64_t ldy, y_bs, y_hs;  // elements
    int y_trans;              // store Y^T (y[j*ldy + i])
    const float* col_scale;   // [N] or null
    float scalar;
    int tile_n = 0, cta_group = 0;  // design (b) tile overrides (0 = auto)
    // popc of each A row's nz plane (bwta_pack_act's row_nnz): the CUDA-core kernels use
    // it instead of counting popc(nz_a) themselves when the other operand is binary (Case 1); null = count
    const int32_t* a_row_nnz = nullptr;
    // Both operands binary (W1A1, no nz plane on either side): every kernel multiplies its own K
    // padding (zero sign bits = +1 x +1) and subtracts that count from the dot in its epilogue
    // (dot_bias = K - K_processed, exact integer arithmetic).
    // fused next-layer pack (bwta_gemm_pack): instead of writing Y, quantize
    // round(Y to y_dt) with the next layer's thresholds and write its planes
    int pack_out = 0;
    int po_kind = 0;          // K_TERNARY / K_BOOL
    uint32_t* po_sgn = nullptr;
    uint32_t* po_nz = nullptr;
    int64_t po_ld = 0;        // words per packed row (rows = the M rows of Y)
    int64_t po_bs = 0, po_hs = 0;  // words between the planes of consecutive batch / head entries
    float po_tp = 0.f, po_tn = 0.f;  // +1 iff y >= po_tp; -1 iff y <= -po_tn (exact storage values)
    // head-split multi-output pack (bwta_gemm_pack_qkv): the columns of Y = [Q | K | V] (each H*D
    // wide) go to per-head planes: Q, K [B, H, T, ld] along D (region 0, 1), V^T [B, H, D, ld(T)]
    // along the tokens (region 2); the rows of Y are the B*T tokens
    int po_heads = 0;
    int64_t ph_T = 0, ph_H = 0, ph_D = 0;
    uint32_t* ph_sgn[3] = {nullptr, nullptr, nullptr};
    uint32_t* ph_nz[3] = {nullptr, nullptr, nullptr};
    int64_t ph_ld[3] = {0, 0, 0};
    float ph_tp[3] = {0.f, 0.f, 0.f}, ph_tn[3] = {0.f, 0.f, 0.f};
    // fused all-gather (bwta_gemm_peers): the epilogue also TMA-stores every output tile to the
    // same position of each of these n_peers buffers (peer GPUs' Y, mapped into this process)
    int n_peers = 0;
    void* y_peers[MAX_PEERS] = {};
};

cudaError_t launch_matmul_cc(const MatmulArgs& a, cudaStream_t s);
// the paper's own design (legacy mma.sync b1 AND-popcount; prior art measured on B200, gemm_b1.cu)
cudaError_t launch_matmul_b1(const MatmulArgs& a, cudaStream_t s);

// fused decode attention (attn_decode.cu): one query row per (batch, head) entry
struct DecodeArgs {
    const uint32_t *q_sgn, *q_nz;   // [entries][ldq words] (one row)
    const uint32_t *k_sgn, *k_nz;   // [entries][tk][ldk]; k_nz null: binary K
    const uint32_t *v_sgn, *v_nz;   // V^T [entries][dh][ldv]
    int64_t nb, nh, tk, dh;
    int64_t ldk, ldv;               // words
    int64_t q_bs, q_hs, k_bs, k_hs, v_bs, v_hs;  // words
    float alpha, p_t, beta;         // p_t: the bool threshold as a p_dt storage value (R2)
    const float *alpha_h, *beta_h;  // per-head alpha / beta [nh] (nullable)
    int p_dt;
    void* o;
    int o_dt;
    int64_t o_bs, o_hs;             // elements; O rows [dh] contiguous
    uint32_t* p_out;                // optional P planes [entries][p_ld]
    int64_t p_ld, pw_ld;            // words; pw_ld = ld_words(tk)
    int cs;                         // CTAs per entry (set by the launcher)
    int64_t sc_off;                 // shared-memory word offset of the kept scores (launcher)
};
cudaError_t launch_attn_decode(const DecodeArgs& a, cudaStream_t s);

// fused prefill attention on tcgen05 (attn_prefill.cu): Q tiles of 128 rows per (batch, head)
struct AttnPrefillArgs {
    const uint32_t *q_sgn, *q_nz;   // [entries][tq][ldq]
    const uint32_t *k_sgn, *k_nz;   // [entries][tk][ldk]; k_nz null: binary K
    const uint32_t *v_sgn, *v_nz;   // V^T [entries][dh][ldv]
    int64_t nb, nh, tq, tk, dh;
    int64_t ldq, ldk, ldv;          // words
    int64_t q_bs, q_hs, k_bs, k_hs, v_bs, v_hs;  // words
    float alpha, p_t, beta;         // p_t: the bool threshold as a p_dt storage value (R2)
    const float *alpha_h = nullptr, *beta_h = nullptr;  // per-head alpha / beta [nh] (nullable)
    int p_dt;
    void* o;
    int o_dt;
    int64_t ld_o, o_bs, o_hs;       // elements
    uint32_t* p_out;                // optional P planes [entries][tq][p_ld]
    int64_t p_ld;
    int pack_out = 0, po_kind = 0;  // fused pack of the [nb*tq, nh*dh] context (dh % 32 == 0)
    uint32_t *po_sgn = nullptr, *po_nz = nullptr;
    int64_t po_ld = 0;
    float po_tp = 0.f, po_tn = 0.f;
    int causal = 0;  // query row i attends to keys j <= i + (tk - tq) only (tk >= tq)
};
bool attn_prefill_supported(const AttnPrefillArgs& a);
cudaError_t launch_attn_prefill(const AttnPrefillArgs& a, cudaStream_t s);

// tcgen05 path (design (b)).  Returns cudaErrorNotSupported when the shape is
// outside what the tcgen05 kernels handle (the dispatcher then uses design (a)).
size_t matmul_tc_workspace(const MatmulArgs& a);
bool matmul_tc_supported(const MatmulArgs& a);
cudaError_t launch_matmul_tc(const MatmulArgs& a, void* ws, size_t ws_bytes, cudaStream_t s);
// a.n_peers > 0: the tile kernel with the 16-bit TMA-store epilogue is the only path that stores to peers
bool matmul_tc_peers_ok(const MatmulArgs& a);
cudaError_t launch_peer_barrier(uint32_t* const* flags, int world, int rank, uint32_t* count, cudaStream_t s);
// skinny products (smaller side <= 32 rows, gemv_tc.cu); launch_matmul_tc
// routes eligible shapes there
bool matmul_gemv_eligible(const MatmulArgs& a);
cudaError_t launch_matmul_gemv(const MatmulArgs& a, cudaStream_t s);
// decode-sized products (smaller side <= 4 rows) on CUDA cores (gemv_cc.cu)
bool matmul_gemv_cc_eligible(const MatmulArgs& a);
cudaError_t launch_matmul_gemv_cc(const MatmulArgs& a, cudaStream_t s);
cudaError_t launch_gemv_cc_fused(const void* x, int x_dt, int64_t ld_x, float tp, float ntn, int a_kind,
                                 const MatmulArgs& a, cudaStream_t s);

}  // namespace bwta
