// api.cu -- the extern "C" boundary (include/bwta.h): host-side validation,
// exact threshold derivation, design dispatch and kernel launches.
#include <cuda_runtime.h>

#include <atomic>
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>

#include "../../include/bwta.h"
#include "bwta_internal.h"

using namespace bwta;

namespace bwta {
std::atomic<uint64_t> g_launches{0};

namespace {
std::atomic<int> g_dev_sms[64];
}
int device_sms() {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return 148;
    }
    if (dev >= 0 && dev < 64 && (v = g_dev_sms[dev].load(std::memory_order_relaxed)) > 0) return v;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) {
        cudaGetLastError();
        v = 148;
    }
    if (dev >= 0 && dev < 64) g_dev_sms[dev].store(v, std::memory_order_relaxed);
    return v;
}
}  // namespace bwta

namespace {

thread_local int g_last_cuda_error = 0;
thread_local int g_last_design = 0;

constexpr int64_t KMAX = int64_t(1) << 24;

bwta_status_t cuda_fail(cudaError_t e) {
    g_last_cuda_error = int(e);
    return BWTA_ERR_CUDA;
}

// Per-device "is this an sm_100 part" cache (-1 unknown, 0 no, 1 yes).
std::atomic<int> g_dev_ok[64];

bwta_status_t check_device() {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) {
        cudaGetLastError();
        g_last_cuda_error = int(e);
        return BWTA_ERR_UNSUPPORTED;
    }
    if (dev >= 0 && dev < 64) {
        int v = g_dev_ok[dev].load(std::memory_order_relaxed);
        if (v == 1) return BWTA_OK;
        if (v == 2) return BWTA_ERR_UNSUPPORTED;
    }
    int major = 0, minor = 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess) {
        cudaGetLastError();
        return BWTA_ERR_UNSUPPORTED;
    }
    const bool ok = (major == 10 && minor == 0);
    if (dev >= 0 && dev < 64) g_dev_ok[dev].store(ok ? 1 : 2, std::memory_order_relaxed);
    return ok ? BWTA_OK : BWTA_ERR_UNSUPPORTED;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int64_t ldw_of(int64_t cols) {
    const int64_t w = (cols + 31) / 32;
    return (w + 3) / 4 * 4;
}

int esize(int dt) { return dt == DT_F32 ? 4 : 2; }

// ---- exact thresholds (see pack.cu) ----------------------------------------
double f16_value(uint16_t b) {  // positive patterns only
    const int e = (b >> 10) & 0x1f, m = b & 0x3ff;
    if (e == 31) return INFINITY;
    if (e == 0) return std::ldexp(double(m), -24);
    return std::ldexp(double(1024 + m), e - 25);
}
double bf16_value(uint16_t b) {
    const uint32_t u = uint32_t(b) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return double(f);
}
// smallest positive 16-bit pattern (<= inf pattern) whose value is >= t (strict: > t)
uint16_t smallest_pattern(double t, bool strict, bool bf16) {
    uint32_t lo = 0, hi = bf16 ? 0x7f80u : 0x7c00u;  // value(hi) = inf > t
    while (lo < hi) {
        const uint32_t mid = (lo + hi) / 2;
        const double v = bf16 ? bf16_value(uint16_t(mid)) : f16_value(uint16_t(mid));
        if (strict ? (v > t) : (v >= t)) hi = mid;
        else lo = mid + 1;
    }
    return uint16_t(lo);
}

// The smallest float f with RNE_to_y_dt(f) >= value(pattern) (pattern > 0):
// the epilogue of bwta_gemm_pack compares the fp32 product against it, which
// is exactly "round to f16/bf16, then compare with the storage threshold".
// The rounding boundary is the midpoint m of pattern and its predecessor (for
// the infinity pattern: max finite + half an ulp); a tie at m rounds to the
// even mantissa, so m itself qualifies iff the pattern's mantissa is even
// (for infinity: the virtual successor of max finite is even -> yes).
float rounding_threshold(uint16_t pattern, bool bf16) {
    const uint16_t inf = bf16 ? 0x7f80u : 0x7c00u;
    const double prev = bf16 ? bf16_value(uint16_t(pattern - 1)) : f16_value(uint16_t(pattern - 1));
    double m;
    bool inclusive;
    if (pattern >= inf) {
        const double ulp = bf16 ? std::ldexp(1.0, 127 - 7) : std::ldexp(1.0, 15 - 10);  // at max finite
        m = prev + ulp / 2;
        inclusive = true;
    } else {
        const double v = bf16 ? bf16_value(pattern) : f16_value(pattern);
        m = (prev + v) / 2;
        inclusive = (pattern & 1u) == 0;
    }
    const float lo = float(m);  // exact: at most one bit more than the 16-bit type
    return inclusive ? lo : std::nextafter(lo, INFINITY);
}

Thresholds make_thresholds(int dt, float scale) {
    Thresholds th{};
    const double t = 0.5 * double(scale);  // exact
    if (dt == DT_F32) {
        float f = float(t);
        float tp = (double(f) < t) ? std::nextafter(f, INFINITY) : f;
        float tn = (double(f) <= t) ? std::nextafter(f, INFINITY) : f;
        th.tpf = tp;
        th.ntnf = -tn;
    } else {
        const bool bf = (dt == DT_BF16);
        const uint32_t tp = smallest_pattern(t, false, bf);
        const uint32_t ntn = smallest_pattern(t, true, bf) | 0x8000u;
        th.tp2 = tp | (tp << 16);
        th.ntn2 = ntn | (ntn << 16);
    }
    return th;
}

bool scale_ok_pos(float s) { return std::isfinite(s) && s > 0.f; }

const bwta_opts_t* opts_or_default(const bwta_opts_t* o) {
    static const bwta_opts_t d{};
    return o ? o : &d;
}

// Every entry point taking bwta_opts_t validates it here, before anything is enqueued.
bwta_status_t check_opts(const bwta_opts_t* opts) {
    if (opts->design < 0 || opts->design > 3) return BWTA_ERR_INVALID_VALUE;
    for (int r : opts->reserved)
        if (r != 0) return BWTA_ERR_INVALID_VALUE;
    if (!(opts->tile_n == 0 || opts->tile_n == 64 || opts->tile_n == 128 || opts->tile_n == 192) ||
        opts->cta_group < 0 || opts->cta_group > 2)
        return BWTA_ERR_INVALID_VALUE;
    return BWTA_OK;
}

// Run a matmul description with the requested design.
bwta_status_t run_matmul(const MatmulArgs& a0, void* ws, size_t ws_bytes, const bwta_opts_t* opts,
                         cudaStream_t s) {
    opts = opts_or_default(opts);
    if (bwta_status_t st = check_opts(opts); st != BWTA_OK) return st;
    MatmulArgs a = a0;
    a.tile_n = opts->tile_n;
    a.cta_group = opts->cta_group;
    if (opts->design == BWTA_DESIGN_MMA_B1) {  // prior art: the paper's mma.sync b1 design (never AUTO)
        cudaError_t e = launch_matmul_b1(a, s);
        if (e != cudaSuccess) return cuda_fail(e);
        g_last_design = BWTA_DESIGN_MMA_B1;
        return BWTA_OK;
    }
    // decode-sized products (<= 4 rows on one side): the CUDA-core GEMV (design (a)
    // family) streams the large side at HBM rate; AUTO prefers it unless a tile
    // shape was forced
    if (matmul_gemv_cc_eligible(a) && (opts->design == BWTA_DESIGN_CUDA_CORE ||
                                       (opts->design == BWTA_DESIGN_AUTO && !a.tile_n && !a.cta_group))) {
        cudaError_t e = launch_matmul_gemv_cc(a, s);
        if (e != cudaSuccess) return cuda_fail(e);
        g_last_design = BWTA_DESIGN_CUDA_CORE;
        return BWTA_OK;
    }
    bool use_tc = false;
    if (opts->design == BWTA_DESIGN_TCGEN05) {
        if (!matmul_tc_supported(a)) return BWTA_ERR_UNSUPPORTED;
        use_tc = true;
    } else if (opts->design == BWTA_DESIGN_AUTO) {
        use_tc = matmul_tc_supported(a);
    }
    if (use_tc) {
        const size_t need = matmul_tc_workspace(a);
        if (need > 0 && (ws == nullptr || ws_bytes < need)) return BWTA_ERR_WORKSPACE;
        cudaError_t e = launch_matmul_tc(a, ws, ws_bytes, s);
        if (e != cudaSuccess) return cuda_fail(e);
        g_last_design = BWTA_DESIGN_TCGEN05;
        return BWTA_OK;
    }
    cudaError_t e = launch_matmul_cc(a, s);
    if (e != cudaSuccess) return cuda_fail(e);
    g_last_design = BWTA_DESIGN_CUDA_CORE;
    return BWTA_OK;
}

bool valid_out_dt(int dt) { return dt == BWTA_F16 || dt == BWTA_BF16 || dt == BWTA_F32 || dt == BWTA_I32; }

}  // namespace

extern "C" {

int64_t bwta_ld_words(int64_t cols) { return cols < 0 ? 0 : ldw_of(cols); }

const char* bwta_status_string(bwta_status_t st) {
    switch (st) {
        case BWTA_OK: return "BWTA_OK";
        case BWTA_ERR_INVALID_VALUE: return "BWTA_ERR_INVALID_VALUE: null pointer, bad scale or bad enum";
        case BWTA_ERR_SHAPE: return "BWTA_ERR_SHAPE: negative dimension, K > 2^24 or leading dimension too small";
        case BWTA_ERR_ALIGNMENT: return "BWTA_ERR_ALIGNMENT: packed planes must be 16-byte aligned with ld % 4 == 0";
        case BWTA_ERR_UNSUPPORTED: return "BWTA_ERR_UNSUPPORTED: dtype/kind combination or device is not sm_100";
        case BWTA_ERR_CUDA: return "BWTA_ERR_CUDA: a CUDA runtime call failed";
        case BWTA_ERR_WORKSPACE: return "BWTA_ERR_WORKSPACE: workspace missing or too small";
    }
    return "BWTA_ERR_UNKNOWN";
}

int bwta_last_cuda_error(void) { return g_last_cuda_error; }
int bwta_last_design(void) { return g_last_design; }
int bwta_version(void) { return 100; }
uint64_t bwta_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

namespace {
// Validate one activation pack and describe it; `empty` = nothing to write.
bwta_status_t prepare_pack(const bwta_pack_desc_t& d, PackArgs& a, bool& empty) {
    const void* x = d.x;
    const bwta_dtype_t x_dt = d.x_dt;
    const int64_t batch = d.batch, heads = d.heads, rows = d.rows, cols = d.cols, ld_x = d.ld_x;
    const int64_t x_bstride = d.x_bstride, x_hstride = d.x_hstride;
    const float scale = d.scale;
    const bwta_kind_t kind = d.kind;
    const int transpose = d.transpose;
    uint32_t* sgn = d.sgn;
    uint32_t* nz = d.nz;
    const int64_t ld_words = d.ld_words, p_bstride = d.p_bstride, p_hstride = d.p_hstride;
    if (x_dt != BWTA_F16 && x_dt != BWTA_BF16 && x_dt != BWTA_F32) return BWTA_ERR_UNSUPPORTED;
    if (kind != BWTA_TERNARY && kind != BWTA_BOOL && kind != BWTA_BINARY) return BWTA_ERR_UNSUPPORTED;
    if (!scale_ok_pos(scale)) return BWTA_ERR_INVALID_VALUE;
    if (transpose != 0 && transpose != 1) return BWTA_ERR_INVALID_VALUE;
    if (batch < 0 || heads < 1 || rows < 0 || cols < 0) return BWTA_ERR_SHAPE;
    if (x == nullptr) return BWTA_ERR_INVALID_VALUE;
    // planes: TERNARY sgn + nz, BOOL nz only, BINARY (W1A1 activations, sign(x)) sgn only
    if ((kind != BWTA_BOOL) != (sgn != nullptr) || (kind != BWTA_BINARY) != (nz != nullptr))
        return BWTA_ERR_INVALID_VALUE;
    if (kind == BWTA_BINARY && d.row_nnz) return BWTA_ERR_INVALID_VALUE;  // every element is non-zero
    const int64_t packed_len = transpose ? rows : cols;
    if (ld_x < cols || ld_words < ldw_of(packed_len)) return BWTA_ERR_SHAPE;
    if (x_bstride < 0 || x_hstride < 0 || p_bstride < 0 || p_hstride < 0) return BWTA_ERR_SHAPE;
    if (ld_words % 4 || p_bstride % 4 || p_hstride % 4 || (nz && !aligned16(nz)) || (sgn && !aligned16(sgn)))
        return BWTA_ERR_ALIGNMENT;
    // No packed rows at all -> nothing to write.  (Packed rows whose length
    // is 0 are all padding and are still written as zero words.)
    empty = batch == 0 || (transpose ? cols : rows) == 0;
    a = PackArgs{};
    a.x = x;
    a.dt = x_dt;
    a.nb = batch;
    a.nh = heads;
    a.rows = rows;
    a.cols = cols;
    a.ld_x = ld_x;
    a.x_bs = x_bstride;
    a.x_hs = x_hstride;
    a.kind = kind;  // BWTA_* and K_* share the numbering; K_BINARY with mu = 0 is sign(x) (Eq. sign, R4)
    a.sgn = sgn;
    a.nz = nz;
    a.mu = nullptr;
    a.ldw = ld_words;
    a.p_bs = p_bstride;
    a.p_hs = p_hstride;
    a.row_nnz = d.row_nnz;
    a.th = make_thresholds(x_dt, scale);
    const int es = esize(x_dt);
    a.vec_ok = aligned16(x) && (ld_x * es) % 16 == 0 && (x_bstride * es) % 16 == 0 && (x_hstride * es) % 16 == 0;
    const int64_t out_rows = transpose ? cols : rows;
    a.planes_dense = (heads == 1 || p_hstride == out_rows * ld_words) &&
                     (batch == 1 || p_bstride == heads * out_rows * ld_words);
    a.nwd = std::max<int64_t>(1, (cols + 31) / 32);
    a.div_nwd = make_fastdiv(uint32_t(a.nwd < (1ll << 31) ? a.nwd : 1));
    a.div_rows = make_fastdiv(uint32_t(rows > 0 && rows < (1ll << 31) ? rows : 1));
    a.div_nh = make_fastdiv(uint32_t(heads < (1ll << 31) ? heads : 1));
    return BWTA_OK;
}
}  // namespace

bwta_status_t bwta_pack_act(const void* x, bwta_dtype_t x_dt, int64_t batch, int64_t heads, int64_t rows,
                            int64_t cols, int64_t ld_x, int64_t x_bstride, int64_t x_hstride, float scale,
                            bwta_kind_t kind, int transpose, uint32_t* sgn, uint32_t* nz, int64_t ld_words,
                            int64_t p_bstride, int64_t p_hstride, int32_t* row_nnz, void* stream) {
    const bwta_pack_desc_t d{x,     x_dt,  batch, heads,     rows,     cols,      ld_x,      x_bstride, x_hstride,
                             scale, kind, transpose, sgn, nz, ld_words, p_bstride, p_hstride, row_nnz};
    PackArgs a;
    bool empty = false;
    bwta_status_t st = prepare_pack(d, a, empty);
    if (st != BWTA_OK) return st;
    st = check_device();
    if (st != BWTA_OK || empty) return st;
    cudaError_t e = transpose ? launch_pack_cols(a, (cudaStream_t)stream) : launch_pack_rows(a, (cudaStream_t)stream);
    return e == cudaSuccess ? BWTA_OK : cuda_fail(e);
}

bwta_status_t bwta_pack_act_batch(const bwta_pack_desc_t* descs, int count, void* stream) {
    if (count < 0 || count > BWTA_PACK_BATCH_MAX) return BWTA_ERR_INVALID_VALUE;
    if (count == 0) return BWTA_OK;
    if (descs == nullptr) return BWTA_ERR_INVALID_VALUE;
    PackArgs a[BWTA_PACK_BATCH_MAX];
    int tr[BWTA_PACK_BATCH_MAX];
    int n = 0;
    for (int i = 0; i < count; ++i) {  // validate everything before enqueueing anything
        bool empty = false;
        bwta_status_t st = prepare_pack(descs[i], a[n], empty);
        if (st != BWTA_OK) return st;
        if (!empty) tr[n++] = descs[i].transpose;
    }
    bwta_status_t st = check_device();
    if (st != BWTA_OK || n == 0) return st;
    cudaError_t e = launch_pack_group(a, tr, n, (cudaStream_t)stream);
    return e == cudaSuccess ? BWTA_OK : cuda_fail(e);
}

bwta_status_t bwta_pack_weight(const void* w, bwta_dtype_t w_dt, int64_t n, int64_t k, int64_t ld_w,
                               const float* mu, int mu_per_row, uint32_t* sgn, int64_t ld_words, void* stream) {
    if (w_dt != BWTA_F16 && w_dt != BWTA_BF16 && w_dt != BWTA_F32) return BWTA_ERR_UNSUPPORTED;
    if (n < 0 || k < 0) return BWTA_ERR_SHAPE;
    if (w == nullptr || sgn == nullptr) return BWTA_ERR_INVALID_VALUE;
    if (mu_per_row != 0 && mu_per_row != 1) return BWTA_ERR_INVALID_VALUE;
    if (mu_per_row && mu == nullptr) return BWTA_ERR_INVALID_VALUE;
    if (ld_w < k || ld_words < ldw_of(k)) return BWTA_ERR_SHAPE;
    if (ld_words % 4 || !aligned16(sgn)) return BWTA_ERR_ALIGNMENT;
    bwta_status_t st = check_device();
    if (st != BWTA_OK) return st;
    if (n == 0) return BWTA_OK;
    PackArgs a{};
    a.x = w;
    a.dt = w_dt;
    a.nb = 1;
    a.nh = 1;
    a.rows = n;
    a.cols = k;
    a.ld_x = ld_w;
    a.kind = K_BINARY;
    a.sgn = sgn;
    a.ldw = ld_words;
    a.mu = mu;
    a.mu_per_row = mu_per_row;
    a.vec_ok = aligned16(w) && (ld_w * esize(w_dt)) % 16 == 0;
    a.planes_dense = true;
    a.nwd = std::max<int64_t>(1, (k + 31) / 32);
    a.div_nwd = make_fastdiv(uint32_t(a.nwd < (1ll << 31) ? a.nwd : 1));
    a.div_rows = make_fastdiv(uint32_t(n > 0 && n < (1ll << 31) ? n : 1));
    a.div_nh = make_fastdiv(1);
    cudaError_t e = launch_pack_rows(a, (cudaStream_t)stream);
    return e == cudaSuccess ? BWTA_OK : cuda_fail(e);
}

size_t bwta_gemm_workspace_size(int64_t m, int64_t n, int64_t k, const bwta_opts_t* opts) {
    opts = opts_or_default(opts);
    if (m <= 0 || n <= 0 || k < 0 || opts->design == BWTA_DESIGN_CUDA_CORE) return 0;
    MatmulArgs a{};
    a.M = m;
    a.N = n;
    a.K = k;
    a.lda = a.ldb = ldw_of(k);
    a.nb = a.nh = 1;
    a.b_nz = nullptr;
    a.a_nz = reinterpret_cast<const uint32_t*>(16);
    a.a_sgn = reinterpret_cast<const uint32_t*>(16);
    a.y_dt = DT_F16;
    return matmul_tc_supported(a) ? matmul_tc_workspace(a) : 0;
}

bwta_status_t bwta_gemm(const uint32_t* a_sgn, const uint32_t* a_nz, bwta_kind_t a_kind, int64_t m, int64_t lda_words,
                        const uint32_t* w_sgn, int64_t n, int64_t ldw_words, int64_t k, const float* w_scale,
                        float a_scale, void* y, bwta_dtype_t y_dt, int64_t ld_y, int y_transposed, void* workspace,
                        size_t workspace_bytes, const bwta_opts_t* opts, void* stream) {
    return bwta_gemm_nnz(a_sgn, a_nz, a_kind, m, lda_words, nullptr, w_sgn, n, ldw_words, k, w_scale, a_scale, y, y_dt,
                         ld_y, y_transposed, workspace, workspace_bytes, opts, stream);
}

bwta_status_t bwta_gemm_nnz(const uint32_t* a_sgn, const uint32_t* a_nz, bwta_kind_t a_kind, int64_t m,
                            int64_t lda_words, const int32_t* a_row_nnz, const uint32_t* w_sgn, int64_t n,
                            int64_t ldw_words, int64_t k, const float* w_scale, float a_scale, void* y,
                            bwta_dtype_t y_dt, int64_t ld_y, int y_transposed, void* workspace, size_t workspace_bytes,
                            const bwta_opts_t* opts, void* stream) {
    if (a_kind != BWTA_TERNARY && a_kind != BWTA_BOOL && a_kind != BWTA_BINARY) return BWTA_ERR_UNSUPPORTED;
    if (!valid_out_dt(y_dt)) return BWTA_ERR_UNSUPPORTED;
    if (m < 0 || n < 0 || k < 0 || k > KMAX) return BWTA_ERR_SHAPE;
    if (m == 0 || n == 0) return BWTA_OK;  // empty product: nothing to read or write
    if (w_sgn == nullptr || y == nullptr) return BWTA_ERR_INVALID_VALUE;
    if ((a_kind != BWTA_BOOL) != (a_sgn != nullptr) || (a_kind != BWTA_BINARY) != (a_nz != nullptr))
        return BWTA_ERR_INVALID_VALUE;
    if (!std::isfinite(a_scale)) return BWTA_ERR_INVALID_VALUE;
    if (y_transposed != 0 && y_transposed != 1) return BWTA_ERR_INVALID_VALUE;
    const int64_t need = ldw_of(k);
    if (lda_words < need || ldw_words < need) return BWTA_ERR_SHAPE;
    if (ld_y < (y_transposed ? m : n)) return BWTA_ERR_SHAPE;
    if (lda_words % 4 || ldw_words % 4 || (a_nz && !aligned16(a_nz)) || (a_sgn && !aligned16(a_sgn)) ||
        !aligned16(w_sgn))
        return BWTA_ERR_ALIGNMENT;
    bwta_status_t st = check_device();
    if (st != BWTA_OK) return st;
    if (m == 0 || n == 0) return BWTA_OK;
    MatmulArgs a{};
    a.a_sgn = a_sgn;
    a.a_nz = a_nz;
    a.b_sgn = w_sgn;
    a.b_nz = nullptr;
    a.M = m;
    a.N = n;
    a.K = k;
    a.lda = lda_words;
    a.ldb = ldw_words;
    a.nb = a.nh = 1;
    a.y = y;
    a.y_dt = y_dt;
    a.ldy = ld_y;
    a.y_trans = y_transposed;
    a.col_scale = w_scale;
    a.scalar = a_scale;
    if (a_row_nnz) {
        if (reinterpret_cast<uintptr_t>(a_row_nnz) % 4) return BWTA_ERR_ALIGNMENT;
        if (a_kind != BWTA_BINARY) a.a_row_nnz = a_row_nnz;  // binary A has no nz plane to count
    }
    return run_matmul(a, workspace, workspace_bytes, opts, (cudaStream_t)stream);
}

bwta_status_t bwta_gemm_peers(const uint32_t* a_sgn, const uint32_t* a_nz, bwta_kind_t a_kind, int64_t m,
                              int64_t lda_words, const uint32_t* w_sgn, int64_t n, int64_t ldw_words, int64_t k,
                              const float* w_scale, float a_scale, void* y, bwta_dtype_t y_dt, int64_t ld_y,
                              int y_transposed, void* const* y_peers, int n_peers, const bwta_opts_t* opts,
                              void* stream) {
    if (n_peers < 0 || n_peers > MAX_PEERS || (n_peers > 0 && y_peers == nullptr)) return BWTA_ERR_INVALID_VALUE;
    if (y_dt != BWTA_F16 && y_dt != BWTA_BF16) return BWTA_ERR_UNSUPPORTED;
    const bwta_opts_t* o = opts_or_default(opts);
    if (bwta_status_t st = check_opts(o); st != BWTA_OK) return st;
    if (o->design != BWTA_DESIGN_AUTO && o->design != BWTA_DESIGN_TCGEN05) return BWTA_ERR_UNSUPPORTED;
    for (int i = 0; i < n_peers; ++i) {
        if (y_peers[i] == nullptr) return BWTA_ERR_INVALID_VALUE;
        if (!aligned16(y_peers[i])) return BWTA_ERR_ALIGNMENT;
    }
    if (a_kind != BWTA_TERNARY && a_kind != BWTA_BOOL && a_kind != BWTA_BINARY) return BWTA_ERR_UNSUPPORTED;
    if (m < 0 || n < 0 || k < 0 || k > KMAX) return BWTA_ERR_SHAPE;
    if (m == 0 || n == 0) return BWTA_OK;
    if (w_sgn == nullptr || y == nullptr) return BWTA_ERR_INVALID_VALUE;
    if ((a_kind != BWTA_BOOL) != (a_sgn != nullptr) || (a_kind != BWTA_BINARY) != (a_nz != nullptr))
        return BWTA_ERR_INVALID_VALUE;
    if (!std::isfinite(a_scale)) return BWTA_ERR_INVALID_VALUE;
    if (y_transposed != 0 && y_transposed != 1) return BWTA_ERR_INVALID_VALUE;
    const int64_t need = ldw_of(k);
    if (lda_words < need || ldw_words < need) return BWTA_ERR_SHAPE;
    if (ld_y < (y_transposed ? m : n)) return BWTA_ERR_SHAPE;
    if (lda_words % 4 || ldw_words % 4 || (a_nz && !aligned16(a_nz)) || (a_sgn && !aligned16(a_sgn)) ||
        !aligned16(w_sgn) || !aligned16(y) || ld_y % 8)
        return BWTA_ERR_ALIGNMENT;
    bwta_status_t st = check_device();
    if (st != BWTA_OK) return st;
    MatmulArgs a{};
    a.a_sgn = a_sgn;
    a.a_nz = a_nz;
    a.b_sgn = w_sgn;
    a.M = m;
    a.N = n;
    a.K = k;
    a.lda = lda_words;
    a.ldb = ldw_words;
    a.nb = a.nh = 1;
    a.y = y;
    a.y_dt = y_dt;
    a.ldy = ld_y;
    a.y_trans = y_transposed;
    a.col_scale = w_scale;
    a.scalar = a_scale;
    a.tile_n = o->tile_n;
    a.cta_group = o->cta_group;
    a.n_peers = n_peers;
    for (int i = 0; i < n_peers; ++i) a.y_peers[i] = y_peers[i];
    // only the tile kernel's 16-bit TMA-store epilogue stores to peers: skinny (GEMV) shapes and W1A1
    // take other epilogues -> the caller gathers those with a collective
    if (!matmul_tc_peers_ok(a)) return BWTA_ERR_UNSUPPORTED;
    cudaError_t e = launch_matmul_tc(a, nullptr, 0, (cudaStream_t)stream);
    if (e == cudaErrorNotSupported) return BWTA_ERR_UNSUPPORTED;
    if (e != cudaSuccess) return cuda_fail(e);
    g_last_design = BWTA_DESIGN_TCGEN05;
    return BWTA_OK;
}

bwta_status_t bwta_peer_barrier(uint32_t* const* flags, int world, int rank, uint32_t* count, void* stream) {
    if (flags == nullptr || count == nullptr || world < 1 || world > MAX_PEERS + 1 || rank < 0 || rank >= world)
        return BWTA_ERR_INVALID_VALUE;
    if (reinterpret_cast<uintptr_t>(count) % 4) return BWTA_ERR_ALIGNMENT;
    for (int r = 0; r < world; ++r) {
        if (flags[r] == nullptr) return BWTA_ERR_INVALID_VALUE;
        if (reinterpret_cast<uintptr_t>(flags[r]) % 4) return BWTA_ERR_ALIGNMENT;
    }
    bwta_status_t st = check_device();
    if (st != BWTA_OK) return st;
    cudaError_t e = launch_peer_barrier(flags, world, rank, count, (cudaStream_t)stream);
    return e == cudaSuccess ? BWTA_OK : cuda_fail(e);
}

bwta_status_t bwta_ipc_handle(const void* ptr, void* handle, int64_t* offset) {
    if (ptr == nullptr || handle == nullptr || offset == nullptr) return BWTA_ERR_INVALID_VALUE;
    static_assert(sizeof(cudaIpcMemHandle_t) == BWTA_IPC_HANDLE_BYTES, "IPC handle size");
    using GetRange = int (*)(unsigned long long*, size_t*, unsigned long long);  // cuMemGetAddressRange_v2
    static GetRange get_range = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<GetRange>(fn);
    }();
    if (get_range == nullptr) return BWTA_ERR_UNSUPPORTED;
    unsigned long long base = 0;
    size_t size = 0;
    if (get_range(&base, &size, reinterpret_cast<unsigned long long>(ptr)) != 0) return BWTA_ERR_INVALID_VALUE;
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
    if (e != cudaSuccess) return cuda_fail(e);
    std::memcpy(handle, &h, sizeof(h));
    *offset = int64_t(reinterpret_cast<unsigned long long>(ptr) - base);
    return BWTA_OK;
}

bwta_status_t bwta_ipc_open(const void* handle, int64_t offset, void** ptr) {
    if (handle == nullptr || ptr == nullptr || offset < 0) return BWTA_ERR_INVALID_VALUE;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    void* base = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_fail(e);
    *ptr = static_cast<char*>(base) + offset;
    return BWTA_OK;
}

bwta_status_t bwta_ipc_close(void* ptr, int64_t offset) {
    if (ptr == nullptr || offset < 0) return BWTA_ERR_INVALID_VALUE;
    cudaError_t e = cudaIpcCloseMemHandle(static_cast<char*>(ptr) - offset);
    return e == cudaSuccess ? BWTA_OK : cuda_fail(e);
}

bwta_status_t bwta_gemm_pack(const uint32_t* a_sgn, const uint32_t* a_nz, bwta_kind_t a_kind, int64_t m,
                             int64_t lda_words, const uint32_t* w_sgn, int64_t n, int64_t ldw_words, int64_t k,
                             const float* w_scale, float a_scale, bwta_dtype_t y_dt, float out_scale,
                             bwta_kind_t out_kind, uint32_t* out_sgn, uint32_t* out_nz, int64_t out_ld_words,
                             const bwta_opts_t* opts, void* stream) {
    if (a_kind != BWTA_TERNARY && a_kind != BWTA_BOOL) return BWTA_ERR_UNSUPPORTED;
    if (out_kind != BWTA_TERNARY && out_kind != BWTA_BOOL) return BWTA_ERR_UNSUPPORTED;
    if (y_dt != BWTA_F16 && y_dt != BWTA_BF16) return BWTA_ERR_UNSUPPORTED;
    if (m < 0 || n < 0 || k < 0 || k > KMAX) return BWTA_ERR_SHAPE;
    if (m == 0 || n == 0) return BWTA_OK;
    if (a_nz == nullptr || w_sgn == nullptr || out_nz == nullptr) return BWTA_ERR_INVALID_VALUE;
    if ((a_kind == BWTA_TERNARY) != (a_sgn != nullptr)) return BWTA_ERR_INVALID_VALUE;
    if ((out_kind == BWTA_TERNARY) != (out_sgn != nullptr)) return BWTA_ERR_INVALID_VALUE;
    if (!std::isfinite(a_scale) || !scale_ok_pos(out_scale)) return BWTA_ERR_INVALID_VALUE;
    const int64_t need = ldw_of(k);
    if (lda_words < need || ldw_words < need || out_ld_words < ldw_of(n)) return BWTA_ERR_SHAPE;
    if (lda_words % 4 || ldw_words % 4 || out_ld_words % 4 || !aligned16(a_nz) || (a_sgn && !aligned16(a_sgn)) ||
        !aligned16(w_sgn) || !aligned16(out_nz) || (out_sgn && !aligned16(out_sgn)))
        return BWTA_ERR_ALIGNMENT;
    const bwta_opts_t* o = opts_or_default(opts);
    if (bwta_status_t so = check_opts(o); so != BWTA_OK) return so;
    if (o->design == BWTA_DESIGN_CUDA_CORE || o->design == BWTA_DESIGN_MMA_B1)
        return BWTA_ERR_UNSUPPORTED;  // fused pack: design (b) only
    bwta_status_t st = check_device();
    if (st != BWTA_OK) return st;
    MatmulArgs a{};
    a.a_sgn = a_sgn;
    a.a_nz = a_nz;
    a.b_sgn = w_sgn;
    a.M = m;
    a.N = n;
    a.K = k;
    a.lda = lda_words;
    a.ldb = ldw_words;
    a.nb = a.nh = 1;
    a.y_dt = y_dt;
    a.col_scale = w_scale;
    a.scalar = a_scale;
    a.pack_out = 1;
    a.po_kind = out_kind;
    a.po_sgn = out_sgn;
    a.po_nz = out_nz;
    a.po_ld = out_ld_words;
    const double t = 0.5 * double(out_scale);  // exact
    const bool bf = y_dt == BWTA_BF16;
    a.po_tp = rounding_threshold(smallest_pattern(t, false, bf), bf);
    a.po_tn = rounding_threshold(smallest_pattern(t, true, bf), bf);
    a.tile_n = o->tile_n;
    a.cta_group = o->cta_group;
    if (!matmul_tc_supported(a)) return BWTA_ERR_UNSUPPORTED;
    cudaStream_t s = (cudaStream_t)stream;
    if (out_ld_words * 32 > n) {
        // words past ceil(n/32) are padding the kernel does not visit: zero the planes first
        cudaError_t e = cudaMemsetAsync(out_nz, 0, sizeof(uint32_t) * size_t(m) * size_t(out_ld_words), s);
        if (e == cudaSuccess && out_sgn)
            e = cudaMemsetAsync(out_sgn, 0, sizeof(uint32_t) * size_t(m) * size_t(out_ld_words), s);
        if (e != cudaSuccess) return cuda_fail(e);
        count_launch(out_sgn ? 2 : 1);
    }
    cudaError_t e = launch_matmul_tc(a, nullptr, 0, s);
    if (e != cudaSuccess) return cuda_fail(e);
    g_last_design = BWTA_DESIGN_TCGEN05;
    return BWTA_OK;
}

bwta_status_t bwta_gemm_pack_qkv(const uint32_t* a_sgn, const uint32_t* a_nz, bwta_kind_t a_kind, int64_t m,
                                 int64_t lda_words, const uint32_t* w_sgn, int64_t n, int64_t ldw_words, int64_t k,
                                 const float* w_scale, float a_scale, bwta_dtype_t y_dt, int64_t batch, int64_t seq,
                                 int64_t heads, int64_t head_dim, const float* out_scale, bwta_kind_t out_kind,
                                 uint32_t* q_sgn, uint32_t* q_nz, int64_t ldq_words, uint32_t* k_sgn, uint32_t* k_nz,
                                 int64_t ldk_words, uint32_t* vt_sgn, uint32_t* vt_nz, int64_t ldv_words,
                                 const bwta_opts_t* opts, void* stream) {
    if (a_kind != BWTA_TERNARY && a_kind != BWTA_BOOL) return BWTA_ERR_UNSUPPORTED;
    if (out_kind != BWTA_TERNARY && out_kind != BWTA_BOOL) return BWTA_ERR_UNSUPPORTED;
    if (y_dt != BWTA_F16 && y_dt != BWTA_BF16) return BWTA_ERR_UNSUPPORTED;
    if (m < 0 || n < 0 || k < 0 || k > KMAX || batch < 0 || seq < 0 || heads < 1 || head_dim < 1) return BWTA_ERR_SHAPE;
    if (m != batch * seq || n != 3 * heads * head_dim) return BWTA_ERR_SHAPE;
    if (m == 0) return BWTA_OK;
    if (head_dim % 32 || seq % 32) return BWTA_ERR_UNSUPPORTED;  // whole words per head / per 32 tokens
    if (a_nz == nullptr || w_sgn == nullptr || out_scale == nullptr || q_nz == nullptr || k_nz == nullptr ||
        vt_nz == nullptr)
        return BWTA_ERR_INVALID_VALUE;
    if ((a_kind == BWTA_TERNARY) != (a_sgn != nullptr)) return BWTA_ERR_INVALID_VALUE;
    const bool tern = out_kind == BWTA_TERNARY;
    if (tern != (q_sgn != nullptr) || tern != (k_sgn != nullptr) || tern != (vt_sgn != nullptr))
        return BWTA_ERR_INVALID_VALUE;
    if (!std::isfinite(a_scale)) return BWTA_ERR_INVALID_VALUE;
    for (int r = 0; r < 3; ++r)
        if (!scale_ok_pos(out_scale[r])) return BWTA_ERR_INVALID_VALUE;
    const int64_t need = ldw_of(k);
    if (lda_words < need || ldw_words < need || ldq_words < ldw_of(head_dim) || ldk_words < ldw_of(head_dim) ||
        ldv_words < ldw_of(seq))
        return BWTA_ERR_SHAPE;
    auto al = [](const void* q) { return q == nullptr || aligned16(q); };
    if (lda_words % 4 || ldw_words % 4 || ldq_words % 4 || ldk_words % 4 || ldv_words % 4 || !al(a_nz) || !al(a_sgn) ||
        !al(w_sgn) || !al(q_sgn) || !al(q_nz) || !al(k_sgn) || !al(k_nz) || !al(vt_sgn) || !al(vt_nz))
        return BWTA_ERR_ALIGNMENT;
    const bwta_opts_t* o = opts_or_default(opts);
    if (bwta_status_t so = check_opts(o); so != BWTA_OK) return so;
    if (o->design == BWTA_DESIGN_CUDA_CORE || o->design == BWTA_DESIGN_MMA_B1) return BWTA_ERR_UNSUPPORTED;
    bwta_status_t st = check_device();
    if (st != BWTA_OK) return st;
    MatmulArgs a{};
    a.a_sgn = a_sgn;
    a.a_nz = a_nz;
    a.b_sgn = w_sgn;
    a.M = m;
    a.N = n;
    a.K = k;
    a.lda = lda_words;
    a.ldb = ldw_words;
    a.nb = a.nh = 1;
    a.y_dt = y_dt;
    a.col_scale = w_scale;
    a.scalar = a_scale;
    a.pack_out = 1;
    a.po_kind = out_kind;
    a.po_heads = 1;
    a.ph_T = seq;
    a.ph_H = heads;
    a.ph_D = head_dim;
    uint32_t* sg[3] = {q_sgn, k_sgn, vt_sgn};
    uint32_t* nzp[3] = {q_nz, k_nz, vt_nz};
    const int64_t lds[3] = {ldq_words, ldk_words, ldv_words};
    const bool bf = y_dt == BWTA_BF16;
    for (int r = 0; r < 3; ++r) {
        a.ph_sgn[r] = sg[r];
        a.ph_nz[r] = nzp[r];
        a.ph_ld[r] = lds[r];
        const double t = 0.5 * double(out_scale[r]);  // exact
        a.ph_tp[r] = rounding_threshold(smallest_pattern(t, false, bf), bf);
        a.ph_tn[r] = rounding_threshold(smallest_pattern(t, true, bf), bf);
    }
    a.tile_n = o->tile_n;
    a.cta_group = o->cta_group;
    if (!matmul_tc_supported(a) || matmul_gemv_eligible(a)) return BWTA_ERR_UNSUPPORTED;
    cudaError_t e = launch_matmul_tc(a, nullptr, 0, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e);
    g_last_design = BWTA_DESIGN_TCGEN05;
    return BWTA_OK;
}

size_t bwta_attn_qk_workspace_size(int64_t batch_heads, int64_t tq, int64_t tk, int64_t dh, const bwta_opts_t* opts) {
    opts = opts_or_default(opts);
    if (batch_heads <= 0 || tq <= 0 || tk <= 0 || dh < 0 || opts->design == BWTA_DESIGN_CUDA_CORE) return 0;
    MatmulArgs a{};
    a.M = tq;
    a.N = tk;
    a.K = dh;
    a.lda = a.ldb = ldw_of(dh);
    a.nb = batch_heads;
    a.nh = 1;
    a.a_bs = a.b_bs = 4;  // any real stride: the size depends only on the shape
    a.a_nz = a.a_sgn = a.b_nz = a.b_sgn = reinterpret_cast<const uint32_t*>(16);
    a.y_dt = DT_F16;
    return matmul_tc_supported(a) ? matmul_tc_workspace(a) : 0;
}

static bwta_status_t check_batch(int64_t batch, int64_t heads) {
    if (batch < 0 || heads < 1) return BWTA_ERR_SHAPE;
    if (batch * heads > 65535) return BWTA_ERR_SHAPE;
    return BWTA_OK;
}

bwta_status_t bwta_attn_qk(const uint32_t* q_sgn, const uint32_t* q_nz, const uint32_t* k_sgn, const uint32_t* k_nz,
                           int64_t batch, int64_t heads, int64_t tq, int64_t tk, int64_t dh, int64_t ldq_words,
                           int64_t q_bstride, int64_t q_hstride, int64_t ldk_words, int64_t k_bstride,
                           int64_t k_hstride, float alpha, void* s, bwta_dtype_t s_dt, int64_t ld_s,
                           int64_t s_bstride, int64_t s_hstride, void* workspace, size_t workspace_bytes,
                           const bwta_opts_t* opts, void* stream) {
    if (!valid_out_dt(s_dt)) return BWTA_ERR_UNSUPPORTED;
    bwta_status_t st = check_batch(batch, heads);
    if (st != BWTA_OK) return st;
    if (tq < 0 || tk < 0 || dh < 0 || dh > KMAX) return BWTA_ERR_SHAPE;
    if (batch == 0 || tq == 0 || tk == 0) return BWTA_OK;
    if (q_sgn == nullptr || q_nz == nullptr || k_sgn == nullptr || s == nullptr) return BWTA_ERR_INVALID_VALUE;
    if (!std::isfinite(alpha)) return BWTA_ERR_INVALID_VALUE;
    const int64_t need = ldw_of(dh);
    if (ldq_words < need || ldk_words < need || ld_s < tk) return BWTA_ERR_SHAPE;
    if (q_bstride < 0 || q_hstride < 0 || k_bstride < 0 || k_hstride < 0 || s_bstride < 0 || s_hstride < 0)
        return BWTA_ERR_SHAPE;
    if (ldq_words % 4 || ldk_words % 4 || q_bstride % 4 || q_hstride % 4 || k_bstride % 4 || k_hstride % 4 ||
        !aligned16(q_sgn) || !aligned16(q_nz) || !aligned16(k_sgn) || (k_nz && !aligned16(k_nz)))
        return BWTA_ERR_ALIGNMENT;
    st = check_device();
    if (st != BWTA_OK) return st;
    if (batch == 0 || tq == 0 || tk == 0) return BWTA_OK;
    MatmulArgs a{};
    a.a_sgn = q_sgn;
    a.a_nz = q_nz;
    a.b_sgn = k_sgn;
    a.b_nz = k_nz;
    a.M = tq;
    a.N = tk;
    a.K = dh;
    a.lda = ldq_words;
    a.ldb = ldk_words;
    a.a_bs = q_bstride;
    a.a_hs = q_hstride;
    a.b_bs = k_bstride;
    a.b_hs = k_hstride;
    a.nb = batch;
    a.nh = heads;
    a.y = s;
    a.y_dt = s_dt;
    a.ldy = ld_s;
    a.y_bs = s_bstride;
    a.y_hs = s_hstride;
    a.scalar = alpha;
    return run_matmul(a, workspace, workspace_bytes, opts, (cudaStream_t)stream);
}

size_t bwta_attn_pv_workspace_size(int64_t batch_heads, int64_t tq, int64_t tk, int64_t dh, const bwta_opts_t* opts) {
    opts = opts_or_default(opts);
    if (batch_heads <= 0 || tq <= 0 || dh <= 0 || tk < 0 || opts->design == BWTA_DESIGN_CUDA_CORE) return 0;
    MatmulArgs a{};
    a.M = tq;
    a.N = dh;
    a.K = tk;
    a.lda = a.ldb = ldw_of(tk);
    a.nb = batch_heads;
    a.nh = 1;
    a.a_bs = a.b_bs = 4;  // any real stride: the size depends only on the shape
    a.a_nz = a.b_nz = a.b_sgn = reinterpret_cast<const uint32_t*>(16);
    a.y_dt = DT_F16;
    return matmul_tc_supported(a) ? matmul_tc_workspace(a) : 0;
}

bwta_status_t bwta_gemm_x(const void* x, bwta_dtype_t x_dt, int64_t m, int64_t ld_x, float a_scale, bwta_kind_t a_kind,
                          const uint32_t* w_sgn, int64_t n, int64_t ldw_words, int64_t k, const float* w_scale,
                          void* y, bwta_dtype_t y_dt, int64_t ld_y, int y_transposed, void* stream) {
    if (x_dt != BWTA_F16 && x_dt != BWTA_BF16 && x_dt != BWTA_F32) return BWTA_ERR_UNSUPPORTED;
    if (a_kind != BWTA_TERNARY && a_kind != BWTA_BOOL) return BWTA_ERR_UNSUPPORTED;
    if (!valid_out_dt(y_dt)) return BWTA_ERR_UNSUPPORTED;
    if (m < 0 || n < 0 || k < 0 || k > KMAX) return BWTA_ERR_SHAPE;
    if (m > 4) return BWTA_ERR_UNSUPPORTED;  // decode sizes only (pack + bwta_gemm otherwise)
    if (m == 0 || n == 0) return BWTA_OK;
    if (x == nullptr || w_sgn == nullptr || y == nullptr) return BWTA_ERR_INVALID_VALUE;
    if (!scale_ok_pos(a_scale)) return BWTA_ERR_INVALID_VALUE;
    if (ld_x < k || ldw_words < ldw_of(k) || ld_y < (y_transposed ? m : n)) return BWTA_ERR_SHAPE;
    if (ldw_words % 4 || !aligned16(w_sgn)) return BWTA_ERR_ALIGNMENT;
    bwta_status_t st = check_device();
    if (st != BWTA_OK) return st;
    // R2 thresholds as values of the input type: +1 iff x >= tp, -1 iff x <= ntn
    float tp, ntn;
    if (x_dt == BWTA_F32) {
        const Thresholds th = make_thresholds(DT_F32, a_scale);
        tp = th.tpf;
        ntn = th.ntnf;
    } else {
        const bool bf = x_dt == BWTA_BF16;
        const double t = 0.5 * double(a_scale);
        const uint16_t p1 = smallest_pattern(t, false, bf), p2 = smallest_pattern(t, true, bf);
        tp = float(bf ? bf16_value(p1) : f16_value(p1));
        ntn = -float(bf ? bf16_value(p2) : f16_value(p2));
    }
    MatmulArgs a{};
    a.b_sgn = w_sgn;
    a.M = m;
    a.N = n;
    a.K = k;
    a.ldb = ldw_words;
    a.nb = a.nh = 1;
    a.y = y;
    a.y_dt = y_dt;
    a.ldy = ld_y;
    a.y_trans = y_transposed ? 1 : 0;
    a.col_scale = w_scale;
    a.scalar = a_scale;
    cudaError_t e = launch_gemv_cc_fused(x, x_dt, ld_x, tp, ntn, a_kind, a, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e);
    g_last_design = BWTA_DESIGN_CUDA_CORE;
    return BWTA_OK;
}

bwta_status_t bwta_attn_decode(const uint32_t* q_sgn, const uint32_t* q_nz, const uint32_t* k_sgn,
                               const uint32_t* k_nz, const uint32_t* vt_sgn, const uint32_t* vt_nz, int64_t batch,
                               int64_t heads, int64_t tk, int64_t dh, int64_t q_bstride, int64_t q_hstride,
                               int64_t ldk_words, int64_t k_bstride, int64_t k_hstride, int64_t ldv_words,
                               int64_t v_bstride, int64_t v_hstride, float alpha, float s_att, bwta_dtype_t p_dt,
                               float beta, const float* alpha_heads, const float* beta_heads, void* o,
                               bwta_dtype_t o_dt, int64_t o_bstride, int64_t o_hstride, uint32_t* p_out,
                               int64_t ldp_words, void* stream) {
    if (!valid_out_dt(o_dt) || (p_dt != BWTA_F16 && p_dt != BWTA_BF16 && p_dt != BWTA_F32))
        return BWTA_ERR_UNSUPPORTED;
    bwta_status_t st = check_batch(batch, heads);
    if (st != BWTA_OK) return st;
    if (tk < 0 || dh < 0 || tk > (int64_t(1) << 14) || dh > 256) return BWTA_ERR_SHAPE;
    if (batch == 0 || dh == 0) return BWTA_OK;
    if (tk == 0) return BWTA_ERR_SHAPE;  // softmax over an empty row
    if (q_sgn == nullptr || q_nz == nullptr || k_sgn == nullptr || vt_sgn == nullptr || vt_nz == nullptr ||
        o == nullptr)
        return BWTA_ERR_INVALID_VALUE;
    if (!std::isfinite(alpha) || !std::isfinite(beta) || !scale_ok_pos(s_att)) return BWTA_ERR_INVALID_VALUE;
    if (ldk_words < ldw_of(dh) || ldv_words < ldw_of(tk) || (p_out && ldp_words < ldw_of(tk))) return BWTA_ERR_SHAPE;
    if (q_bstride < 0 || q_hstride < 0 || k_bstride < 0 || k_hstride < 0 || v_bstride < 0 || v_hstride < 0 ||
        o_bstride < 0 || o_hstride < 0)
        return BWTA_ERR_SHAPE;
    // every plane is read with 16-byte vector loads (attn_decode.cu)
    if (ldk_words % 4 || ldv_words % 4 || q_bstride % 4 || q_hstride % 4 || k_bstride % 4 || k_hstride % 4 ||
        v_bstride % 4 || v_hstride % 4 || (p_out && ldp_words % 4) || !aligned16(q_sgn) || !aligned16(q_nz) ||
        !aligned16(k_sgn) || (k_nz && !aligned16(k_nz)) || !aligned16(vt_sgn) || !aligned16(vt_nz) ||
        (p_out && !aligned16(p_out)))
        return BWTA_ERR_ALIGNMENT;
    st = check_device();
    if (st != BWTA_OK) return st;
    DecodeArgs a{};
    a.q_sgn = q_sgn;
    a.q_nz = q_nz;
    a.k_sgn = k_sgn;
    a.k_nz = k_nz;
    a.v_sgn = vt_sgn;
    a.v_nz = vt_nz;
    a.nb = batch;
    a.nh = heads;
    a.tk = tk;
    a.dh = dh;
    a.ldk = ldk_words;
    a.ldv = ldv_words;
    a.q_bs = q_bstride;
    a.q_hs = q_hstride;
    a.k_bs = k_bstride;
    a.k_hs = k_hstride;
    a.v_bs = v_bstride;
    a.v_hs = v_hstride;
    a.alpha = alpha;
    a.beta = beta;
    a.alpha_h = alpha_heads;
    a.beta_h = beta_heads;
    a.p_dt = p_dt;
    const double t = 0.5 * double(s_att);  // exact
    if (p_dt == BWTA_F32) {
        a.p_t = float(t);
    } else {
        const bool bf = p_dt == BWTA_BF16;
        const uint16_t tp = smallest_pattern(t, false, bf);  // smallest storage value >= s/2 (R2)
        a.p_t = float(bf ? bf16_value(tp) : f16_value(tp));
    }
    a.o = o;
    a.o_dt = o_dt;
    a.o_bs = o_bstride;
    a.o_hs = o_hstride;
    a.p_out = p_out;
    a.p_ld = ldp_words;
    a.pw_ld = ldw_of(tk);
    cudaError_t e = launch_attn_decode(a, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e);
    return BWTA_OK;
}

}  // extern "C"

namespace {
// bwta_attn_prefill (pack = 0: O) and bwta_attn_prefill_pack (pack = 1: the context planes)
bwta_status_t attn_prefill_impl(const uint32_t* q_sgn, const uint32_t* q_nz, const uint32_t* k_sgn,
                                const uint32_t* k_nz, const uint32_t* vt_sgn, const uint32_t* vt_nz, int64_t batch,
                                int64_t heads, int64_t tq, int64_t tk, int64_t dh, int64_t ldq_words,
                                int64_t q_bstride, int64_t q_hstride, int64_t ldk_words, int64_t k_bstride,
                                int64_t k_hstride, int64_t ldv_words, int64_t v_bstride, int64_t v_hstride,
                                float alpha, float s_att, bwta_dtype_t p_dt, float beta, const float* alpha_heads,
                                const float* beta_heads, void* o, bwta_dtype_t o_dt,
                                int64_t ld_o, int64_t o_bstride, int64_t o_hstride, uint32_t* p_out,
                                int64_t ldp_words, int pack, float out_scale, bwta_kind_t out_kind,
                                uint32_t* out_sgn, uint32_t* out_nz, int64_t out_ld_words, void* stream,
                                int causal = 0) {
    if (causal != 0 && causal != 1) return BWTA_ERR_INVALID_VALUE;
    if (causal && tk < tq) return BWTA_ERR_SHAPE;  // every query row needs at least one key
    if (pack) {
        if (o_dt != BWTA_F16 && o_dt != BWTA_BF16) return BWTA_ERR_UNSUPPORTED;  // the rounding being packed
        if (out_kind != BWTA_TERNARY && out_kind != BWTA_BOOL) return BWTA_ERR_UNSUPPORTED;
        if (dh % 32) return BWTA_ERR_UNSUPPORTED;  // a head must own whole words of the context row
    }
    if (!valid_out_dt(o_dt) || (p_dt != BWTA_F16 && p_dt != BWTA_BF16 && p_dt != BWTA_F32))
        return BWTA_ERR_UNSUPPORTED;
    bwta_status_t st = check_batch(batch, heads);
    if (st != BWTA_OK) return st;
    if (tq < 0 || tk < 0 || dh < 0 || tk > KMAX || tq > (int64_t(1) << 31)) return BWTA_ERR_SHAPE;
    if (dh > 128) return BWTA_ERR_UNSUPPORTED;  // one 128-element tensor-core stage per Q/K row
    if (batch == 0 || tq == 0 || dh == 0) return BWTA_OK;
    if (tk == 0) return BWTA_ERR_SHAPE;  // softmax over an empty row
    if (q_sgn == nullptr || q_nz == nullptr || k_sgn == nullptr || vt_sgn == nullptr || vt_nz == nullptr ||
        (!pack && o == nullptr) || (pack && (out_nz == nullptr || (out_kind == BWTA_TERNARY) != (out_sgn != nullptr))))
        return BWTA_ERR_INVALID_VALUE;
    if (pack && !scale_ok_pos(out_scale)) return BWTA_ERR_INVALID_VALUE;
    if (!std::isfinite(alpha) || !std::isfinite(beta) || !scale_ok_pos(s_att)) return BWTA_ERR_INVALID_VALUE;
    if (ldq_words < ldw_of(dh) || ldk_words < ldw_of(dh) || ldv_words < ldw_of(tk) || (!pack && ld_o < dh) ||
        (p_out && ldp_words < ldw_of(tk)) || (pack && out_ld_words < ldw_of(heads * dh)))
        return BWTA_ERR_SHAPE;
    if (q_bstride < 0 || q_hstride < 0 || k_bstride < 0 || k_hstride < 0 || v_bstride < 0 || v_hstride < 0 ||
        o_bstride < 0 || o_hstride < 0)
        return BWTA_ERR_SHAPE;
    // every plane is read by TMA: 16-byte aligned bases and row / batch / head strides
    if (ldq_words % 4 || ldk_words % 4 || ldv_words % 4 || q_bstride % 4 || q_hstride % 4 || k_bstride % 4 ||
        k_hstride % 4 || v_bstride % 4 || v_hstride % 4 || !aligned16(q_sgn) || !aligned16(q_nz) ||
        !aligned16(k_sgn) || (k_nz && !aligned16(k_nz)) || !aligned16(vt_sgn) || !aligned16(vt_nz) ||
        (p_out && (ldp_words % 4 || !aligned16(p_out))) ||
        (pack && (out_ld_words % 4 || !aligned16(out_nz) || (out_sgn && !aligned16(out_sgn)))))
        return BWTA_ERR_ALIGNMENT;
    st = check_device();
    if (st != BWTA_OK) return st;
    AttnPrefillArgs a{};
    a.causal = causal;
    a.q_sgn = q_sgn;
    a.q_nz = q_nz;
    a.k_sgn = k_sgn;
    a.k_nz = k_nz;
    a.v_sgn = vt_sgn;
    a.v_nz = vt_nz;
    a.nb = batch;
    a.nh = heads;
    a.tq = tq;
    a.tk = tk;
    a.dh = dh;
    a.ldq = ldq_words;
    a.ldk = ldk_words;
    a.ldv = ldv_words;
    a.q_bs = q_bstride;
    a.q_hs = q_hstride;
    a.k_bs = k_bstride;
    a.k_hs = k_hstride;
    a.v_bs = v_bstride;
    a.v_hs = v_hstride;
    a.alpha = alpha;
    a.beta = beta;
    a.alpha_h = alpha_heads;
    a.beta_h = beta_heads;
    a.p_dt = p_dt;
    const double t = 0.5 * double(s_att);  // exact
    if (p_dt == BWTA_F32) {
        a.p_t = float(t);                  // exact (halving a normal float)
    } else {
        const bool bf = p_dt == BWTA_BF16;
        const uint16_t tp = smallest_pattern(t, false, bf);  // smallest storage value >= s/2 (R2)
        a.p_t = float(bf ? bf16_value(tp) : f16_value(tp));
    }
    a.o = o;
    a.o_dt = o_dt;
    a.ld_o = ld_o;
    a.o_bs = o_bstride;
    a.o_hs = o_hstride;
    a.p_out = p_out;
    a.p_ld = ldp_words;
    if (pack) {
        a.pack_out = 1;
        a.po_kind = out_kind;
        a.po_sgn = out_sgn;
        a.po_nz = out_nz;
        a.po_ld = out_ld_words;
        const double tt = 0.5 * double(out_scale);  // exact
        const bool bf = o_dt == BWTA_BF16;
        a.po_tp = rounding_threshold(smallest_pattern(tt, false, bf), bf);
        a.po_tn = rounding_threshold(smallest_pattern(tt, true, bf), bf);
    }
    if (!attn_prefill_supported(a)) return BWTA_ERR_UNSUPPORTED;
    cudaStream_t s = (cudaStream_t)stream;
    if (pack && out_ld_words * 32 > heads * dh) {  // padding words of the context rows: no head writes them
        const size_t bytes = sizeof(uint32_t) * size_t(batch) * size_t(tq) * size_t(out_ld_words);
        cudaError_t e = cudaMemsetAsync(out_nz, 0, bytes, s);
        if (e == cudaSuccess && out_sgn) e = cudaMemsetAsync(out_sgn, 0, bytes, s);
        if (e != cudaSuccess) return cuda_fail(e);
        count_launch(out_sgn ? 2 : 1);
    }
    if (p_out) {  // the kernel writes the data words of P; padding words stay zero
        cudaError_t e = cudaMemsetAsync(p_out, 0, sizeof(uint32_t) * size_t(batch * heads) * size_t(tq) *
                                                        size_t(ldp_words), s);
        if (e != cudaSuccess) return cuda_fail(e);
        count_launch();
    }
    cudaError_t e = launch_attn_prefill(a, s);
    if (e != cudaSuccess) return cuda_fail(e);
    g_last_design = BWTA_DESIGN_TCGEN05;
    return BWTA_OK;
}
}  // namespace

extern "C" {

bwta_status_t bwta_attn_prefill(const uint32_t* q_sgn, const uint32_t* q_nz, const uint32_t* k_sgn,
                                const uint32_t* k_nz, const uint32_t* vt_sgn, const uint32_t* vt_nz, int64_t batch,
                                int64_t heads, int64_t tq, int64_t tk, int64_t dh, int64_t ldq_words,
                                int64_t q_bstride, int64_t q_hstride, int64_t ldk_words, int64_t k_bstride,
                                int64_t k_hstride, int64_t ldv_words, int64_t v_bstride, int64_t v_hstride,
                                float alpha, float s_att, bwta_dtype_t p_dt, float beta, const float* alpha_heads,
                                const float* beta_heads, void* o, bwta_dtype_t o_dt,
                                int64_t ld_o, int64_t o_bstride, int64_t o_hstride, uint32_t* p_out,
                                int64_t ldp_words, void* stream) {
    return attn_prefill_impl(q_sgn, q_nz, k_sgn, k_nz, vt_sgn, vt_nz, batch, heads, tq, tk, dh, ldq_words, q_bstride,
                             q_hstride, ldk_words, k_bstride, k_hstride, ldv_words, v_bstride, v_hstride, alpha, s_att,
                             p_dt, beta, alpha_heads, beta_heads, o, o_dt, ld_o, o_bstride, o_hstride, p_out,
                             ldp_words, 0, 0.f, BWTA_TERNARY, nullptr, nullptr, 0, stream);
}

bwta_status_t bwta_attn_prefill_ex(const uint32_t* q_sgn, const uint32_t* q_nz, const uint32_t* k_sgn,
                                   const uint32_t* k_nz, const uint32_t* vt_sgn, const uint32_t* vt_nz, int64_t batch,
                                   int64_t heads, int64_t tq, int64_t tk, int64_t dh, int64_t ldq_words,
                                   int64_t q_bstride, int64_t q_hstride, int64_t ldk_words, int64_t k_bstride,
                                   int64_t k_hstride, int64_t ldv_words, int64_t v_bstride, int64_t v_hstride,
                                   float alpha, float s_att, bwta_dtype_t p_dt, float beta, const float* alpha_heads,
                                   const float* beta_heads, void* o, bwta_dtype_t o_dt, int64_t ld_o,
                                   int64_t o_bstride, int64_t o_hstride, uint32_t* p_out, int64_t ldp_words,
                                   int causal, void* stream) {
    return attn_prefill_impl(q_sgn, q_nz, k_sgn, k_nz, vt_sgn, vt_nz, batch, heads, tq, tk, dh, ldq_words, q_bstride,
                             q_hstride, ldk_words, k_bstride, k_hstride, ldv_words, v_bstride, v_hstride, alpha, s_att,
                             p_dt, beta, alpha_heads, beta_heads, o, o_dt, ld_o, o_bstride, o_hstride, p_out,
                             ldp_words, 0, 0.f, BWTA_TERNARY, nullptr, nullptr, 0, stream, causal);
}

bwta_status_t bwta_attn_prefill_pack(const uint32_t* q_sgn, const uint32_t* q_nz, const uint32_t* k_sgn,
                                     const uint32_t* k_nz, const uint32_t* vt_sgn, const uint32_t* vt_nz, int64_t batch,
                                     int64_t heads, int64_t tq, int64_t tk, int64_t dh, int64_t ldq_words,
                                     int64_t q_bstride, int64_t q_hstride, int64_t ldk_words, int64_t k_bstride,
                                     int64_t k_hstride, int64_t ldv_words, int64_t v_bstride, int64_t v_hstride,
                                     float alpha, float s_att, bwta_dtype_t p_dt, float beta,
                                     const float* alpha_heads, const float* beta_heads, bwta_dtype_t o_dt,
                                     float out_scale, bwta_kind_t out_kind, uint32_t* out_sgn, uint32_t* out_nz,
                                     int64_t out_ld_words, void* stream) {
    return attn_prefill_impl(q_sgn, q_nz, k_sgn, k_nz, vt_sgn, vt_nz, batch, heads, tq, tk, dh, ldq_words, q_bstride,
                             q_hstride, ldk_words, k_bstride, k_hstride, ldv_words, v_bstride, v_hstride, alpha, s_att,
                             p_dt, beta, alpha_heads, beta_heads, nullptr, o_dt, 0, 0, 0, nullptr, 0, 1, out_scale,
                             out_kind, out_sgn, out_nz, out_ld_words, stream);
}

bwta_status_t bwta_attn_pv_pack(const uint32_t* p_sgn, const uint32_t* p_nz, const uint32_t* vt_sgn,
                                const uint32_t* vt_nz, int64_t batch, int64_t heads, int64_t tq, int64_t tk, int64_t dh,
                                int64_t ldp_words, int64_t p_bstride, int64_t p_hstride, int64_t ldv_words,
                                int64_t v_bstride, int64_t v_hstride, float beta, bwta_dtype_t o_dt, float out_scale,
                                bwta_kind_t out_kind, uint32_t* out_sgn, uint32_t* out_nz, int64_t out_ld_words,
                                const bwta_opts_t* opts, void* stream) {
    if (o_dt != BWTA_F16 && o_dt != BWTA_BF16) return BWTA_ERR_UNSUPPORTED;
    if (out_kind != BWTA_TERNARY && out_kind != BWTA_BOOL) return BWTA_ERR_UNSUPPORTED;
    bwta_status_t st = check_batch(batch, heads);
    if (st != BWTA_OK) return st;
    if (tq < 0 || tk < 0 || dh < 0 || tk > KMAX) return BWTA_ERR_SHAPE;
    if (batch == 0 || tq == 0 || dh == 0) return BWTA_OK;
    if (p_nz == nullptr || vt_sgn == nullptr || vt_nz == nullptr || out_nz == nullptr) return BWTA_ERR_INVALID_VALUE;
    if ((out_kind == BWTA_TERNARY) != (out_sgn != nullptr)) return BWTA_ERR_INVALID_VALUE;
    if (!std::isfinite(beta) || !scale_ok_pos(out_scale)) return BWTA_ERR_INVALID_VALUE;
    if (dh % 32) return BWTA_ERR_UNSUPPORTED;  // a head must own whole words of the context row
    const int64_t need = ldw_of(tk);
    if (ldp_words < need || ldv_words < need || out_ld_words < ldw_of(heads * dh)) return BWTA_ERR_SHAPE;
    if (p_bstride < 0 || p_hstride < 0 || v_bstride < 0 || v_hstride < 0) return BWTA_ERR_SHAPE;
    if (ldp_words % 4 || ldv_words % 4 || out_ld_words % 4 || p_bstride % 4 || p_hstride % 4 || v_bstride % 4 ||
        v_hstride % 4 || !aligned16(p_nz) || (p_sgn && !aligned16(p_sgn)) || !aligned16(vt_sgn) ||
        !aligned16(vt_nz) || !aligned16(out_nz) || (out_sgn && !aligned16(out_sgn)))
        return BWTA_ERR_ALIGNMENT;
    const bwta_opts_t* o = opts_or_default(opts);
    if (bwta_status_t so = check_opts(o); so != BWTA_OK) return so;
    if (o->design == BWTA_DESIGN_CUDA_CORE || o->design == BWTA_DESIGN_MMA_B1)
        return BWTA_ERR_UNSUPPORTED;  // fused pack: design (b) only
    st = check_device();
    if (st != BWTA_OK) return st;
    MatmulArgs a{};
    a.a_sgn = p_sgn;
    a.a_nz = p_nz;
    a.b_sgn = vt_sgn;
    a.b_nz = vt_nz;
    a.M = tq;
    a.N = dh;
    a.K = tk;
    a.lda = ldp_words;
    a.ldb = ldv_words;
    a.a_bs = p_bstride;
    a.a_hs = p_hstride;
    a.b_bs = v_bstride;
    a.b_hs = v_hstride;
    a.nb = batch;
    a.nh = heads;
    a.y_dt = o_dt;
    a.scalar = beta;
    a.pack_out = 1;
    a.po_kind = out_kind;
    a.po_sgn = out_sgn;
    a.po_nz = out_nz;
    a.po_ld = out_ld_words;           // one packed row per token (b, t): the heads' contexts concatenated
    a.po_bs = tq * out_ld_words;
    a.po_hs = dh / 32;                // head h owns words [h dh / 32, (h + 1) dh / 32) of the row
    const double t = 0.5 * double(out_scale);  // exact
    const bool bf = o_dt == BWTA_BF16;
    a.po_tp = rounding_threshold(smallest_pattern(t, false, bf), bf);
    a.po_tn = rounding_threshold(smallest_pattern(t, true, bf), bf);
    a.tile_n = o->tile_n;
    a.cta_group = o->cta_group;
    if (!matmul_tc_supported(a) || matmul_gemv_eligible(a)) return BWTA_ERR_UNSUPPORTED;
    cudaStream_t s = (cudaStream_t)stream;
    if (out_ld_words * 32 > heads * dh) {
        // padding words of the context rows: no head writes them
        const size_t bytes = sizeof(uint32_t) * size_t(batch) * size_t(tq) * size_t(out_ld_words);
        cudaError_t e = cudaMemsetAsync(out_nz, 0, bytes, s);
        if (e == cudaSuccess && out_sgn) e = cudaMemsetAsync(out_sgn, 0, bytes, s);
        if (e != cudaSuccess) return cuda_fail(e);
        count_launch(out_sgn ? 2 : 1);
    }
    cudaError_t e = launch_matmul_tc(a, nullptr, 0, s);
    if (e != cudaSuccess) return cuda_fail(e);
    g_last_design = BWTA_DESIGN_TCGEN05;
    return BWTA_OK;
}

bwta_status_t bwta_attn_pv(const uint32_t* p_sgn, const uint32_t* p_nz, const uint32_t* vt_sgn, const uint32_t* vt_nz,
                           int64_t batch, int64_t heads, int64_t tq, int64_t tk, int64_t dh, int64_t ldp_words,
                           int64_t p_bstride, int64_t p_hstride, int64_t ldv_words, int64_t v_bstride,
                           int64_t v_hstride, float beta, void* o, bwta_dtype_t o_dt, int64_t ld_o,
                           int64_t o_bstride, int64_t o_hstride, void* workspace, size_t workspace_bytes,
                           const bwta_opts_t* opts, void* stream) {
    if (!valid_out_dt(o_dt)) return BWTA_ERR_UNSUPPORTED;
    bwta_status_t st = check_batch(batch, heads);
    if (st != BWTA_OK) return st;
    if (tq < 0 || tk < 0 || dh < 0 || tk > KMAX) return BWTA_ERR_SHAPE;
    if (batch == 0 || tq == 0 || dh == 0) return BWTA_OK;
    // vt_nz == NULL: binary V (Binary A x V); P's nz plane masks the key padding
    if (p_nz == nullptr || vt_sgn == nullptr || o == nullptr) return BWTA_ERR_INVALID_VALUE;
    if (!std::isfinite(beta)) return BWTA_ERR_INVALID_VALUE;
    const int64_t need = ldw_of(tk);
    if (ldp_words < need || ldv_words < need || ld_o < dh) return BWTA_ERR_SHAPE;
    if (p_bstride < 0 || p_hstride < 0 || v_bstride < 0 || v_hstride < 0 || o_bstride < 0 || o_hstride < 0)
        return BWTA_ERR_SHAPE;
    if (ldp_words % 4 || ldv_words % 4 || p_bstride % 4 || p_hstride % 4 || v_bstride % 4 || v_hstride % 4 ||
        !aligned16(p_nz) || (p_sgn && !aligned16(p_sgn)) || !aligned16(vt_sgn) || (vt_nz && !aligned16(vt_nz)))
        return BWTA_ERR_ALIGNMENT;
    st = check_device();
    if (st != BWTA_OK) return st;
    if (batch == 0 || tq == 0 || dh == 0) return BWTA_OK;
    MatmulArgs a{};
    a.a_sgn = p_sgn;
    a.a_nz = p_nz;
    a.b_sgn = vt_sgn;
    a.b_nz = vt_nz;
    a.M = tq;
    a.N = dh;
    a.K = tk;
    a.lda = ldp_words;
    a.ldb = ldv_words;
    a.a_bs = p_bstride;
    a.a_hs = p_hstride;
    a.b_bs = v_bstride;
    a.b_hs = v_hstride;
    a.nb = batch;
    a.nh = heads;
    a.y = o;
    a.y_dt = o_dt;
    a.ldy = ld_o;
    a.y_bs = o_bstride;
    a.y_hs = o_hstride;
    a.scalar = beta;
    return run_matmul(a, workspace, workspace_bytes, opts, (cudaStream_t)stream);
}

}  // extern "C"
