/*
 * bwta.h -- C ABI of the B200-native BWTA inference hot path.
 *
 * BWTA = Binary Weights x Ternary Activations (arxiv 2604.03957,
 * /root/reference/PAPER.md cited as P:<line>).  The library implements the
 * paper's inference problem statement (App. B; Sec. 5):
 *
 *   bwta_pack_act    ternary / bool quantize + bit-pack of FP activations
 *                    (P:911-930 Eq. bool / ternary; Sec. 5.2.2)
 *   bwta_pack_weight sign(W - mu) bit-pack of weights, offline
 *                    (P:901-909 Eq. sign; P:934-939 Eq. bw)
 *   bwta_gemm        Y = s_W s_A (sign(W - mu) (x) quant(A^T, s_A))
 *                    (P:949-957 Eq. bwta_linear; Case 1 P:324-325)
 *   bwta_attn_qk     S = alpha (ternary(Q) (x) ternary(K)^T), alpha = s_Q s_K / sqrt(D)
 *                    (P:959-967 Eq. bwta_qk; Case 3 P:330-331)
 *   bwta_attn_pv     O = beta (bool(Att) (x) ternary(V)), beta = s_Att s_V
 *                    (Case 2 P:327-328)
 *
 * ---------------------------------------------------------------------------
 * Packed-plane format (bit-exact contract):
 *   A packed matrix [rows x cols] is `rows` rows of `ld` uint32 words each,
 *   ld >= bwta_ld_words(cols) and ld % 4 == 0 (16-byte rows).  Element
 *   (r, c) lives in word r*ld + c/32, bit c%32 (LSB first).  Planes:
 *     nz  : bit = 1  <=>  q != 0            (TERNARY, BOOL)
 *     sgn : bit = 1  <=>  q <  0            (TERNARY, BINARY)
 *   BINARY (weights, {-1,+1}) has only sgn; BOOL ({0,1}) has only nz;
 *   TERNARY ({-1,0,+1}) has both, canonical (sgn is a subset of nz).
 *   Every bit of an element index >= cols, and every word in
 *   [ceil(cols/32), ld), is 0.  The pack functions write them as 0; the
 *   matmul functions REQUIRE them to be 0.
 *
 * Quantization (App. B; readings R1-R3 in DESIGN.md):
 *   ternary(x, s) = +1 if x/s >= 0.5, -1 if x/s < -0.5, else 0
 *   bool(x, s)    =  1 if x/s >= 0.5, else 0
 *   decided EXACTLY (as x >= s/2 in real arithmetic; no division rounding).
 *   Ties: x = +s/2 -> +1, x = -s/2 -> 0 (the equation, not odd-symmetric).
 *   NaN -> 0, -0.0 -> 0, +-Inf -> +-1 (bool: +Inf -> 1).
 *   sign(w - mu) = +1 if w >= mu else -1 (NaN -> -1; -0.0 >= 0 -> +1).
 *
 * Epilogue (R5; INT32 -> float P:235):
 *   gemm:      c_n = fl32(w_scale[n] * a_scale);  y = fl32(float(dot) * c_n)
 *   attention: y = fl32(float(dot) * alpha)  (resp. beta)
 *   then round-to-nearest-even to FP16 / BF16 (overflow -> +-Inf), or FP32,
 *   or I32 = the raw integer dot (scales ignored).  |dot| <= K <= 2^24 so the
 *   int -> float conversion is exact.
 *
 * ---------------------------------------------------------------------------
 * Conventions for every entry point:
 *   - Every pointer argument is a DEVICE pointer owned by the caller unless
 *     stated otherwise.  The library never allocates device memory, never
 *     frees, and never synchronizes the stream.
 *   - Work is enqueued on `stream` (a cudaStream_t passed as void*, NULL =
 *     legacy default stream) and the call returns immediately.
 *   - Arguments are validated on the host first; on any error nothing is
 *     enqueued, outputs are untouched and a non-zero status is returned.
 *   - Outputs must not alias inputs.  Calls are thread-safe (no global
 *     mutable state except per-thread last-error detail).
 *   - Sizes are element counts; leading dimensions / strides of FP tensors
 *     are in elements, of packed planes in uint32 words.
 *   - Batched calls (pack_act, attn_qk, attn_pv) address entry
 *     e = b*heads + h  (0 <= b < batch, 0 <= h < heads) at
 *     base + b*bstride + h*hstride  for every tensor independently, so a
 *     [B, T, H*D] projection output can be used per head without copies.
 *   - Requires an sm_100 device (B200); otherwise BWTA_ERR_UNSUPPORTED.
 * ---------------------------------------------------------------------------
 */
#ifndef BWTA_H_
#define BWTA_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define BWTA_API __attribute__((visibility("default")))
#else
#define BWTA_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    BWTA_OK = 0,
    BWTA_ERR_INVALID_VALUE = 1, /* NULL pointer, scale not finite or <= 0, bad enum */
    BWTA_ERR_SHAPE = 2,         /* dim < 0, K > 2^24, ld / stride too small */
    BWTA_ERR_ALIGNMENT = 3,     /* packed planes not 16-byte aligned, ld % 4 != 0 */
    BWTA_ERR_UNSUPPORTED = 4,   /* dtype/kind combination, no sm_100 device */
    BWTA_ERR_CUDA = 5,          /* a CUDA call failed (detail: bwta_last_cuda_error) */
    BWTA_ERR_WORKSPACE = 6      /* workspace NULL or smaller than *_workspace_size() */
} bwta_status_t;

typedef enum { BWTA_F16 = 0, BWTA_BF16 = 1, BWTA_F32 = 2, BWTA_I32 = 3 } bwta_dtype_t;

typedef enum { BWTA_BINARY = 0, BWTA_BOOL = 1, BWTA_TERNARY = 2 } bwta_kind_t;

typedef enum {
    BWTA_DESIGN_AUTO = 0,      /* pick per shape */
    BWTA_DESIGN_CUDA_CORE = 1, /* design (a): LOP3 + POPC bit-serial on CUDA cores */
    BWTA_DESIGN_TCGEN05 = 2,   /* design (b): unpack to E2M1 codes + tcgen05.mma.kind::mxf4 (FP32 acc, exact) */
    BWTA_DESIGN_MMA_B1 = 3     /* prior art: the paper's warp-level mma.sync b1 AND-popcount design (
                                  ptxas emulates it on sm_100a with MOVM + IMMA); selectable, never AUTO */
} bwta_design_t;

/* Options for the matmul entry points; NULL = all defaults (zero-initialised). */
typedef struct {
    int32_t design;      /* bwta_design_t */
    int32_t tile_n;      /* design (b) only: 0 = auto, else the tile width 64 | 128 | 192 */
    int32_t cta_group;   /* design (b) only: 0 = auto, 1 = single CTA, 2 = CTA pair (cta_group::2) */
    int32_t reserved[5]; /* must be 0 */
} bwta_opts_t;

/* ---- helpers ------------------------------------------------------------ */

/* Words per packed row for `cols` elements: round_up(ceil(cols/32), 4). */
BWTA_API int64_t bwta_ld_words(int64_t cols);

/* Static string for a status code (never NULL). */
BWTA_API const char* bwta_status_string(bwta_status_t status);

/* Detail for the last BWTA_ERR_CUDA returned on this host thread:
 * the cudaError_t value (0 if none). */
BWTA_API int bwta_last_cuda_error(void);

/* Design used by the last successful matmul call on this host thread
 * (bwta_design_t; 0 before any call). */
BWTA_API int bwta_last_design(void);

/* Library version, e.g. 100 = 0.1.0. */
BWTA_API int bwta_version(void);

/* Number of device kernels (and memset nodes) this process has enqueued
 * through the library so far (all threads).  Used by benchmarks to report
 * how many of the library's kernels ran inside a timed region. */
BWTA_API uint64_t bwta_kernel_launches(void);

/* ---- activation pack ---------------------------------------------------- */
/*
 * Quantize and pack FP activations (Sec. 5.2.2).
 *
 * x      : [batch*heads] matrices of [rows x cols], dtype x_dt (F16 | BF16 | F32),
 *          row stride ld_x >= cols elements; entry e at x + b*x_bstride + h*x_hstride.
 * scale  : s_A > 0, finite (host value).  kind: BWTA_TERNARY, BWTA_BOOL, or BWTA_BINARY
 *          (W1A1 activations: q = sign(x) of Eq. sign P:903-908 -- +1 iff x >= 0,
 *          so -0.0 -> +1 and NaN -> -1 (R4); the scale does not enter the quantizer).
 * transpose = 0 : pack along cols -> planes [rows x ld_words], ld_words >= bwta_ld_words(cols)
 * transpose = 1 : pack along rows (the planes of X^T, used for V^T in PV)
 *                 -> planes [cols x ld_words], ld_words >= bwta_ld_words(rows)
 * sgn    : TERNARY / BINARY: output sign plane; BOOL: must be NULL.
 * nz     : TERNARY / BOOL: output non-zero plane; BINARY: must be NULL (every element is +-1).
 *          Plane entry e at plane + b*p_bstride + h*p_hstride (words).
 * row_nnz: nullable; int32 [batch*heads*out_rows], contiguous, = number of
 *          non-zero quantized values per packed row (out_rows = rows, or cols
 *          when transposed).
 * Alignment: sgn/nz 16-byte aligned, ld_words % 4 == 0, plane strides % 4 == 0.
 * x has no alignment requirement (aligned rows take a vectorised path).
 */
BWTA_API bwta_status_t bwta_pack_act(const void* x, bwta_dtype_t x_dt,
                            int64_t batch, int64_t heads, int64_t rows, int64_t cols,
                            int64_t ld_x, int64_t x_bstride, int64_t x_hstride,
                            float scale, bwta_kind_t kind, int transpose,
                            uint32_t* sgn, uint32_t* nz, int64_t ld_words,
                            int64_t p_bstride, int64_t p_hstride,
                            int32_t* row_nnz, void* stream);

/* ---- several activation packs in one launch ------------------------------ */
/*
 * bwta_pack_act_batch(descs, count, stream) == calling bwta_pack_act on
 * descs[0..count) in order (same arguments, same results, same errors), but
 * enqueued as ONE kernel launch when every desc has the same x_dt (otherwise
 * one launch per desc).  Intended for the per-head Q, K and V^T packs of an
 * attention layer, whose individual launches are latency-bound.
 * 0 <= count <= BWTA_PACK_BATCH_MAX; descs is a HOST array.  All descs are
 * validated before anything is enqueued.  The outputs of different descs
 * must not alias each other or any input.
 */
#define BWTA_PACK_BATCH_MAX 4
typedef struct {
    const void* x;
    bwta_dtype_t x_dt;
    int64_t batch, heads, rows, cols, ld_x, x_bstride, x_hstride;
    float scale;
    bwta_kind_t kind;
    int transpose;
    uint32_t* sgn;
    uint32_t* nz;
    int64_t ld_words, p_bstride, p_hstride;
    int32_t* row_nnz;
} bwta_pack_desc_t;

BWTA_API bwta_status_t bwta_pack_act_batch(const bwta_pack_desc_t* descs, int count, void* stream);

/* ---- weight pack (offline) ---------------------------------------------- */
/*
 * sgn[r] bit c = 1 <=> sign(W[r][c] - mu) = -1.
 * w      : [n x k] dtype w_dt (F16 | BF16 | F32), row stride ld_w >= k.
 * mu     : nullable device float; mu_per_row ? mu[n] : mu[0]; NULL -> 0.
 * sgn    : output [n x ld_words], ld_words >= bwta_ld_words(k), 16-byte aligned.
 */
BWTA_API bwta_status_t bwta_pack_weight(const void* w, bwta_dtype_t w_dt, int64_t n, int64_t k,
                               int64_t ld_w, const float* mu, int mu_per_row,
                               uint32_t* sgn, int64_t ld_words, void* stream);

/* ---- BWTA linear (Case 1 / bool x binary) -------------------------------- */
/*
 * Y[m][n] = fl32(float(dot[m][n]) * fl32(w_scale[n] * a_scale)),
 * dot[m][n] = sum_k qa[m][k] * qw[n][k].
 * A      : activations, a_kind = TERNARY (a_sgn, a_nz), BOOL (a_sgn NULL, a_nz) or BINARY
 *          (a_sgn, a_nz NULL: the W1A1 "Binary Linear"), planes [m x lda_words]
 *          (lda_words >= bwta_ld_words(k)).  With binary A every kernel multiplies its own K
 *          padding as (+1)(+1) and subtracts that count from the dot before the epilogue.
 * W      : weight sign plane [n x ldw_words] (ldw_words >= bwta_ld_words(k)).
 * w_scale: nullable device float [n] (NULL -> 1).  a_scale: host float.
 * y      : y_transposed = 0: Y [m x n] with row stride ld_y >= n;
 *          y_transposed = 1: Y^T [n x m] with row stride ld_y >= m.
 *          dtype y_dt in F16 | BF16 | F32 | I32.
 * workspace: device scratch of >= bwta_gemm_workspace_size(m, n, k, opts)
 *          bytes (may be NULL when that size is 0), 256-byte aligned.
 * 0 <= k <= 2^24.  m == 0 or n == 0: nothing to do, returns BWTA_OK without
 * looking at the pointers (empty tensors may have NULL data).
 */
BWTA_API size_t bwta_gemm_workspace_size(int64_t m, int64_t n, int64_t k, const bwta_opts_t* opts);

BWTA_API bwta_status_t bwta_gemm(const uint32_t* a_sgn, const uint32_t* a_nz, bwta_kind_t a_kind,
                        int64_t m, int64_t lda_words,
                        const uint32_t* w_sgn, int64_t n, int64_t ldw_words, int64_t k,
                        const float* w_scale, float a_scale,
                        void* y, bwta_dtype_t y_dt, int64_t ld_y, int y_transposed,
                        void* workspace, size_t workspace_bytes,
                        const bwta_opts_t* opts, void* stream);

/*
 * bwta_gemm with the activation rows' nonzero counts (SURVEY §8(b)'s a_row_nnz): a_row_nnz[i] =
 * popc of A row i's nz plane, as bwta_pack_act(row_nnz) writes it for the same planes (int32 [m],
 * device, 4-byte aligned; NULL = bwta_gemm).  The paper hoists this count out of the Case-1 inner
 * loop (dot = popc(nz_a) - 2 popc(nz_a & (sgn_a ^ w))); design (a)'s tile
 * kernel reads it instead of counting popc(nz_a) per word when A is TERNARY or BOOL; the other
 * kernels ignore it (the tensor-core kernels form the dot directly; the <= 4-row GEMV counts the
 * small side once per L1-resident quad -- a run-time switch there measured 15 % slower).  The counts are
 * trusted: counts that do not match the planes give wrong results.  Errors as bwta_gemm.
 */
BWTA_API bwta_status_t bwta_gemm_nnz(const uint32_t* a_sgn, const uint32_t* a_nz, bwta_kind_t a_kind,
                            int64_t m, int64_t lda_words, const int32_t* a_row_nnz,
                            const uint32_t* w_sgn, int64_t n, int64_t ldw_words, int64_t k,
                            const float* w_scale, float a_scale,
                            void* y, bwta_dtype_t y_dt, int64_t ld_y, int y_transposed,
                            void* workspace, size_t workspace_bytes,
                            const bwta_opts_t* opts, void* stream);

/* ---- N-sharded BWTA linear with the all-gather fused into the epilogue ---- */
/*
 * The north star's multi-GPU linear: rank r of `world` GPUs holds the weight rows of its N-shard
 * and computes its block of Y^T; with the NCCL all-gather as the baseline, here the GEMM's epilogue
 * itself stores every output tile both to y and to the same position of each peer's buffer
 * y_peers[0 .. n_peers) (device pointers valid in this process: peer GPUs' memory mapped with
 * bwta_ipc_open, reached over NVLink / NVSwitch), so the gather overlaps the math tile by tile
 * and no collective is launched.  Arguments and result as bwta_gemm (one shard: w_sgn / n / w_scale
 * are the local rows, y the local block inside the full Y^T, y_peers the same block in the peers'
 * Y^T), restricted to what the tile kernel's 16-bit TMA-store epilogue covers: y_dt F16 | BF16,
 * y and every y_peers[i] 16-byte aligned, ld_y % 8 == 0, design AUTO | TCGEN05, not W1A1 (binary
 * A with binary W), and a shape that takes the tile kernel (both m and n > 32) -- anything else
 * returns BWTA_ERR_UNSUPPORTED with nothing enqueued (gather those with a collective).
 * 0 <= n_peers <= 7.  The stores are complete when the kernel is; bwta_peer_barrier, enqueued after
 * it on every rank, makes all ranks' stores visible to the work that follows.  The caller keeps
 * the buffers alive and does not overwrite a buffer a peer may still be reading (double-buffer Y^T
 * across steps, or barrier before the GEMM too).
 */
BWTA_API bwta_status_t bwta_gemm_peers(const uint32_t* a_sgn, const uint32_t* a_nz, bwta_kind_t a_kind,
                                       int64_t m, int64_t lda_words,
                                       const uint32_t* w_sgn, int64_t n, int64_t ldw_words, int64_t k,
                                       const float* w_scale, float a_scale,
                                       void* y, bwta_dtype_t y_dt, int64_t ld_y, int y_transposed,
                                       void* const* y_peers, int n_peers,
                                       const bwta_opts_t* opts, void* stream);

/*
 * Cross-GPU barrier over flag arrays in device memory: flags[r] (host array of `world` device
 * pointers, valid in this process) is rank r's array of `world` uint32 slots; count is this rank's
 * own uint32 barrier count (device memory, not shared).  Both zero-initialised before the first
 * use.  One tiny kernel on `stream`: epoch = *count + 1; for every rank t a system-scope release
 * store flags[t][rank] = epoch after a system-scope fence (so every store of the work enqueued
 * before it on this stream -- e.g. bwta_gemm_peers' peer stores -- is visible to rank t), then
 * acquire loads until flags[rank][t] >= epoch for every t; then *count = epoch.  The epoch lives in
 * device memory, so a CUDA graph that captured the call advances it on every replay.  Every rank
 * makes the same sequence of calls.  1 <= world <= 8, 0 <= rank < world.  A rank that never
 * arrives traps the kernel after 30 s (sticky CUDA error) instead of hanging.
 */
BWTA_API bwta_status_t bwta_peer_barrier(uint32_t* const* flags, int world, int rank, uint32_t* count,
                                         void* stream);

/* CUDA IPC for the peer mappings: the handle (BWTA_IPC_HANDLE_BYTES bytes, host memory) of the
 * allocation holding device pointer ptr and ptr's byte offset in it; another process opens it with
 * bwta_ipc_open (-> a device pointer to the same bytes) and unmaps it with bwta_ipc_close(ptr,
 * offset).  One open per allocation per process. */
#define BWTA_IPC_HANDLE_BYTES 64
BWTA_API bwta_status_t bwta_ipc_handle(const void* ptr, void* handle, int64_t* offset);
BWTA_API bwta_status_t bwta_ipc_open(const void* handle, int64_t offset, void** ptr);
BWTA_API bwta_status_t bwta_ipc_close(void* ptr, int64_t offset);

/* ---- BWTA linear with the next layer's pack fused into the epilogue ------ */
/*
 * out = bwta_pack_act(Y, y_dt, out_scale, out_kind), Y = bwta_gemm(...) in
 * y_dt, BIT-EXACTLY -- without writing Y: the epilogue rounds each
 * y = fl32(dot * c) (R5) to y_dt (F16 | BF16) and quantizes it with the
 * exact thresholds of out_scale (R1-R3), writing the planes of Y's rows
 * (bits along n): out_nz (+ out_sgn for TERNARY) [m x out_ld_words],
 * out_ld_words >= bwta_ld_words(n), padding zero.  Typical use: the FFN1
 * linear emitting the BOOL planes FFN2 consumes (relu(y) >= t <=> y >= t
 * for t > 0), 2 bits instead of 16 per activation and no pack launch
 * (SURVEY §8(f) N2).  Design (b) only (opts->design CUDA_CORE ->
 * BWTA_ERR_UNSUPPORTED); no row_nnz.  Other arguments as bwta_gemm.
 */
BWTA_API bwta_status_t bwta_gemm_pack(const uint32_t* a_sgn, const uint32_t* a_nz, bwta_kind_t a_kind,
                                      int64_t m, int64_t lda_words,
                                      const uint32_t* w_sgn, int64_t n, int64_t ldw_words, int64_t k,
                                      const float* w_scale, float a_scale, bwta_dtype_t y_dt,
                                      float out_scale, bwta_kind_t out_kind,
                                      uint32_t* out_sgn, uint32_t* out_nz, int64_t out_ld_words,
                                      const bwta_opts_t* opts, void* stream);

/* ---- QKV projection with the per-head Q / K / V^T packs fused ---- */
/*
 * Y = bwta_gemm(A, W, w_scale, a_scale) rounded to y_dt (F16 | BF16) with Y = [Q | K | V] (n =
 * 3*heads*head_dim columns, the rows the m = batch*seq tokens), written only as the next operands'
 * planes, exactly as bwta_pack_act would pack the stored per-head views (R1-R3):
 *   Q, K planes [batch][heads][seq][ldq/ldk_words] (packed along head_dim, scale out_scale[0/1]),
 *   V^T planes  [batch][heads][head_dim][ldv_words] (packed along the tokens, out_scale[2]) --
 * the inputs of bwta_attn_qk / bwta_attn_pv / bwta_attn_prefill.  out_kind TERNARY | BOOL for all
 * three; padding words are zeroed by the kernel.  head_dim % 32 == 0 and seq % 32 == 0 (whole
 * words per head and per 32 tokens), design (b) only.  Other arguments and errors as bwta_gemm_pack.
 */
BWTA_API bwta_status_t bwta_gemm_pack_qkv(const uint32_t* a_sgn, const uint32_t* a_nz, bwta_kind_t a_kind,
                                          int64_t m, int64_t lda_words, const uint32_t* w_sgn, int64_t n,
                                          int64_t ldw_words, int64_t k, const float* w_scale, float a_scale,
                                          bwta_dtype_t y_dt, int64_t batch, int64_t seq, int64_t heads,
                                          int64_t head_dim, const float* out_scale /* host [3] */,
                                          bwta_kind_t out_kind, uint32_t* q_sgn, uint32_t* q_nz, int64_t ldq_words,
                                          uint32_t* k_sgn, uint32_t* k_nz, int64_t ldk_words,
                                          uint32_t* vt_sgn, uint32_t* vt_nz, int64_t ldv_words,
                                          const bwta_opts_t* opts, void* stream);

/* ---- attention QK^T (Case 3) -------------------------------------------- */
/*
 * S_e[i][j] = fl32(float(sum_d q[i][d] k[j][d]) * alpha)
 * Q planes [tq x ldq_words] (ternary: q_sgn, q_nz); K planes [tk x ldk_words]
 * ternary (k_sgn, k_nz) or binary (k_nz == NULL).  dh = reduction length.
 * S [tq x tk] per entry, row stride ld_s, dtype s_dt.
 */
BWTA_API size_t bwta_attn_qk_workspace_size(int64_t batch_heads, int64_t tq, int64_t tk, int64_t dh,
                                   const bwta_opts_t* opts);

BWTA_API bwta_status_t bwta_attn_qk(const uint32_t* q_sgn, const uint32_t* q_nz,
                           const uint32_t* k_sgn, const uint32_t* k_nz,
                           int64_t batch, int64_t heads, int64_t tq, int64_t tk, int64_t dh,
                           int64_t ldq_words, int64_t q_bstride, int64_t q_hstride,
                           int64_t ldk_words, int64_t k_bstride, int64_t k_hstride,
                           float alpha,
                           void* s, bwta_dtype_t s_dt, int64_t ld_s,
                           int64_t s_bstride, int64_t s_hstride,
                           void* workspace, size_t workspace_bytes,
                           const bwta_opts_t* opts, void* stream);

/* ---- attention PV (Case 2) ---------------------------------------------- */
/*
 * O_e[i][d] = fl32(float(sum_j p[i][j] v[j][d]) * beta)
 * P planes [tq x ldp_words]: bool (p_sgn == NULL, p_nz) or ternary.
 * V is given TRANSPOSED: planes [dh x ldv_words] over the tk axis, as
 * produced by bwta_pack_act(transpose = 1) of V [tk x dh]; ternary (vt_sgn, vt_nz) or binary
 * (vt_sgn, vt_nz NULL: the "Binary A x V" of P:553; P's nz plane masks the key padding).
 * O [tq x dh] per entry, row stride ld_o, dtype o_dt.
 */
BWTA_API size_t bwta_attn_pv_workspace_size(int64_t batch_heads, int64_t tq, int64_t tk, int64_t dh,
                                   const bwta_opts_t* opts);

BWTA_API bwta_status_t bwta_attn_pv(const uint32_t* p_sgn, const uint32_t* p_nz,
                           const uint32_t* vt_sgn, const uint32_t* vt_nz,
                           int64_t batch, int64_t heads, int64_t tq, int64_t tk, int64_t dh,
                           int64_t ldp_words, int64_t p_bstride, int64_t p_hstride,
                           int64_t ldv_words, int64_t v_bstride, int64_t v_hstride,
                           float beta,
                           void* o, bwta_dtype_t o_dt, int64_t ld_o,
                           int64_t o_bstride, int64_t o_hstride,
                           void* workspace, size_t workspace_bytes,
                           const bwta_opts_t* opts, void* stream);

/* ---- attention PV with the next layer's pack fused into the epilogue ----- */
/*
 * bwta_pack_act(C, out_scale, out_kind) of the attention context
 *   C[b, t, h*dh + d] = round_{o_dt}(O_{b,h}[t][d]),   O as bwta_attn_pv computes it
 * (P:969-975 then P:911-930): the O-projection's input planes come
 * straight out of the PV epilogue, O is never written.  Output planes: batch*tq rows
 * (token-major, b then t) of out_ld_words words, head h owning words
 * [h dh/32, (h+1) dh/32) of every row -- exactly the planes bwta_pack_act writes for
 * the [batch*tq, heads*dh] context.  Requires dh % 32 == 0, o_dt F16 | BF16,
 * out_kind TERNARY | BOOL, out_ld_words >= bwta_ld_words(heads*dh) (padding words are
 * zeroed by a memset on `stream`), design (b); the products the skinny kernels serve
 * (<= 32 rows on one side) return BWTA_ERR_UNSUPPORTED.  Other arguments and errors
 * as bwta_attn_pv.
 */
BWTA_API bwta_status_t bwta_attn_pv_pack(const uint32_t* p_sgn, const uint32_t* p_nz,
                           const uint32_t* vt_sgn, const uint32_t* vt_nz,
                           int64_t batch, int64_t heads, int64_t tq, int64_t tk, int64_t dh,
                           int64_t ldp_words, int64_t p_bstride, int64_t p_hstride,
                           int64_t ldv_words, int64_t v_bstride, int64_t v_hstride,
                           float beta, bwta_dtype_t o_dt, float out_scale, bwta_kind_t out_kind,
                           uint32_t* out_sgn, uint32_t* out_nz, int64_t out_ld_words,
                           const bwta_opts_t* opts, void* stream);

/* ---- decode linear with the activation pack fused ------------------------ */
/*
 * Y = bwta_gemm(bwta_pack_act(x, a_scale, a_kind), W, w_scale, a_scale) in ONE launch for
 * m <= 4 activation rows (decode): x [m x k] values (F16 | BF16 | F32, row stride ld_x
 * elements) are quantized (R1-R3) into shared-memory planes by every CTA of a
 * CUDA-core GEMV -- the paper's in-kernel bitpack -- then streamed against the
 * binary weight planes [n x ldw_words].  Outputs and errors as bwta_gemm; m > 4 returns
 * BWTA_ERR_UNSUPPORTED (pack + bwta_gemm there).
 */
BWTA_API bwta_status_t bwta_gemm_x(const void* x, bwta_dtype_t x_dt, int64_t m, int64_t ld_x, float a_scale,
                                   bwta_kind_t a_kind, const uint32_t* w_sgn, int64_t n, int64_t ldw_words,
                                   int64_t k, const float* w_scale, void* y, bwta_dtype_t y_dt, int64_t ld_y,
                                   int y_transposed, void* stream);

/* ---- fused prefill attention (tensor cores) ------------------------------ */
/*
 * The whole BWTA attention of a layer in ONE launch: per (batch b,
 * head h), with Q planes [tq x ldq_words] (ternary), K planes [tk x ldk_words] (ternary,
 * or binary with k_nz == NULL) and V^T planes [dh x ldv_words] (ternary, over tk, from
 * bwta_pack_act(V, transpose=1)):
 *   s_ij = fl32(float(q_i . k_j) * alpha)                     (R5)
 *   p_ij = softmax_j(s_i) in fp32, rounded to p_dt            (high-precision softmax)
 *   b_ij = [p_ij >= s_att / 2] on the rounded value           (bool quantizer; R1-R2)
 *   O_id = round_{o_dt}(fl32(float(sum_j b_ij v_jd) * beta))  (R5; I32: the raw dot)
 * S, P and the P planes never touch memory (QK^T and PV on tcgen05, the softmax in
 * registers).  Entry (b, h) of Q/K/V^T at b*X_bstride + h*X_hstride words;
 * O rows [dh] at b*o_bstride + h*o_hstride + i*ld_o elements.  p_out (nullable) receives the
 * P planes [batch*heads][tq][ldp_words] (tests; zeroed by a memset on `stream` first).
 * alpha_heads / beta_heads (nullable, device float [heads]): per-head alpha / beta replacing
 * alpha / beta for head h (the per-head scales of SURVEY §8(f) N4; a negative alpha_heads[h]
 * negates that head's scores).
 * 1 <= dh <= 128 (BWTA_ERR_UNSUPPORTED above), tk >= 1, tk <= 2^24.  Alignment: every
 * plane pointer 16-byte aligned, every ld / stride a multiple of 4 words (TMA).  As for
 * bwta_attn_decode, a bit of P may differ from an exact softmax only where p_ij lies
 * within rounding distance of s_att / 2 (R13).
 */
BWTA_API bwta_status_t bwta_attn_prefill(const uint32_t* q_sgn, const uint32_t* q_nz,
                           const uint32_t* k_sgn, const uint32_t* k_nz,
                           const uint32_t* vt_sgn, const uint32_t* vt_nz,
                           int64_t batch, int64_t heads, int64_t tq, int64_t tk, int64_t dh,
                           int64_t ldq_words, int64_t q_bstride, int64_t q_hstride,
                           int64_t ldk_words, int64_t k_bstride, int64_t k_hstride,
                           int64_t ldv_words, int64_t v_bstride, int64_t v_hstride,
                           float alpha, float s_att, bwta_dtype_t p_dt, float beta,
                           const float* alpha_heads, const float* beta_heads,
                           void* o, bwta_dtype_t o_dt, int64_t ld_o, int64_t o_bstride, int64_t o_hstride,
                           uint32_t* p_out, int64_t ldp_words, void* stream);

/*
 * bwta_attn_prefill with an optional causal mask (SURVEY §8(f) N3's causal tile skipping):
 * causal = 1: query row i attends to keys j <= i + (tk - tq) only (the decoder / LLaMA prefill
 * mask; requires tk >= tq, else BWTA_ERR_SHAPE); masked keys are not keys -- out of the row max,
 * the softmax normaliser, P and PV -- and key blocks past a query tile's last row are never loaded
 * or multiplied.  causal = 0 is bwta_attn_prefill.  Other arguments and errors as
 * bwta_attn_prefill.
 */
BWTA_API bwta_status_t bwta_attn_prefill_ex(const uint32_t* q_sgn, const uint32_t* q_nz,
                           const uint32_t* k_sgn, const uint32_t* k_nz,
                           const uint32_t* vt_sgn, const uint32_t* vt_nz,
                           int64_t batch, int64_t heads, int64_t tq, int64_t tk, int64_t dh,
                           int64_t ldq_words, int64_t q_bstride, int64_t q_hstride,
                           int64_t ldk_words, int64_t k_bstride, int64_t k_hstride,
                           int64_t ldv_words, int64_t v_bstride, int64_t v_hstride,
                           float alpha, float s_att, bwta_dtype_t p_dt, float beta,
                           const float* alpha_heads, const float* beta_heads,
                           void* o, bwta_dtype_t o_dt, int64_t ld_o, int64_t o_bstride, int64_t o_hstride,
                           uint32_t* p_out, int64_t ldp_words, int causal, void* stream);

/*
 * bwta_attn_prefill with the next layer's activation pack fused into its epilogue (SURVEY
 * §8(f) N2): instead of O, the planes of the [batch*tq, heads*dh] attention context
 * (round_{o_dt}(O), o_dt F16 | BF16) quantized with out_scale / out_kind (TERNARY | BOOL),
 * exactly as bwta_pack_act would quantize the stored context: row b*tq + t, head h owning words
 * [h dh/32, (h+1) dh/32) (dh % 32 == 0), out_ld_words >= bwta_ld_words(heads*dh) (padding words
 * zeroed by a memset on `stream`).  Other arguments and errors as bwta_attn_prefill.
 */
BWTA_API bwta_status_t bwta_attn_prefill_pack(const uint32_t* q_sgn, const uint32_t* q_nz,
                           const uint32_t* k_sgn, const uint32_t* k_nz,
                           const uint32_t* vt_sgn, const uint32_t* vt_nz,
                           int64_t batch, int64_t heads, int64_t tq, int64_t tk, int64_t dh,
                           int64_t ldq_words, int64_t q_bstride, int64_t q_hstride,
                           int64_t ldk_words, int64_t k_bstride, int64_t k_hstride,
                           int64_t ldv_words, int64_t v_bstride, int64_t v_hstride,
                           float alpha, float s_att, bwta_dtype_t p_dt, float beta,
                           const float* alpha_heads, const float* beta_heads,
                           bwta_dtype_t o_dt, float out_scale, bwta_kind_t out_kind,
                           uint32_t* out_sgn, uint32_t* out_nz, int64_t out_ld_words, void* stream);

/* ---- fused decode attention (one query row per entry) -------------------- */
/*
 * Per (batch b, head h), with one packed query row q (ternary; q_sgn/q_nz at
 * b*q_bstride + h*q_hstride words), K planes [tk x ldk_words] (ternary, or binary
 * with k_nz == NULL) and V^T planes [dh x ldv_words] (ternary, over tk):
 *   s_j = fl32(float(q . k_j) * alpha)                        (R5)
 *   p_j = softmax_j(s) in fp32, rounded to p_dt               (high-precision softmax)
 *   b_j = [p_j >= s_att / 2] on the rounded value             (bool quantizer; R1-R2)
 *   O[d] = round_{o_dt}(fl32(float(sum_j b_j v_jd) * beta))   (R5; I32: the raw dot)
 * in one launch (SURVEY §8(f) N3 for Tq = 1): S, P and the P planes never touch
 * memory.  O rows [dh] contiguous at b*o_bstride + h*o_hstride elements.  p_out
 * (nullable) receives the P planes [entries x ldp_words] (b-major, then h) -- for
 * tests.  1 <= tk <= 16384, dh <= 256.  The fp32 softmax is not bit-reproducible
 * against another summation order: a bit of P may differ from an exact softmax
 * only where p_j lies within rounding distance of s_att / 2.
 */
BWTA_API bwta_status_t bwta_attn_decode(const uint32_t* q_sgn, const uint32_t* q_nz,
                           const uint32_t* k_sgn, const uint32_t* k_nz,
                           const uint32_t* vt_sgn, const uint32_t* vt_nz,
                           int64_t batch, int64_t heads, int64_t tk, int64_t dh,
                           int64_t q_bstride, int64_t q_hstride,
                           int64_t ldk_words, int64_t k_bstride, int64_t k_hstride,
                           int64_t ldv_words, int64_t v_bstride, int64_t v_hstride,
                           float alpha, float s_att, bwta_dtype_t p_dt, float beta, const float* alpha_heads, const float* beta_heads,
                           void* o, bwta_dtype_t o_dt, int64_t o_bstride, int64_t o_hstride,
                           uint32_t* p_out, int64_t ldp_words, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* BWTA_H_ */
