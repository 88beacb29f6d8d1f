/*
 * bwta_oracle.c -- plain, slow, obviously-correct CPU oracle for the BWTA
 * inference hot path (arxiv 2604.03957, "BWTA: Accurate and Efficient
 * Binarized Transformer by Algorithm-Hardware Co-design").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2604_03957_b200/) never links, imports or calls it,
 * and it shares no code, header, table or constant with the CUDA path.
 *
 * Citations: "P:<line>" = /root/reference/PAPER.md line (section/equation in
 * parentheses).  Readings where the paper is silent or ambiguous are listed
 * in DESIGN.md section "Readings of the paper" and referenced here as R<n>.
 *
 * Every function follows the paper's definition step by step; there is no
 * blocking, no bit-parallel arithmetic (no popcount) and no reordering.
 * Compile with: gcc -O2 -ffp-contract=off -fno-fast-math -std=c11 -fPIC -shared
 * (no FMA contraction: every float multiply is a separately rounded IEEE op).
 *
 * Pinning status (see tests/test_oracle.py): every exported function is pinned
 * against values fixed by the paper / SPEC hand examples / closed forms /
 * library routines (numpy float16, integer matmul).  None is "parity unpinned".
 */
#define _GNU_SOURCE
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* dtype codes of this oracle (its own numbering; the Python wrapper maps) */
enum { ORC_F16 = 0, ORC_BF16 = 1, ORC_F32 = 2, ORC_I32 = 3 };
/* activation quantizer kinds */
enum { ORC_BINARY = 0, ORC_BOOL = 1, ORC_TERNARY = 2 };

/* ------------------------------------------------------------------------ */
/* O1. Decode FP16 / BF16 / FP32 storage to an exact float value.            */
/* IEEE-754 binary16: 1 sign, 5 exponent (bias 15), 10 fraction bits.        */
/* ------------------------------------------------------------------------ */
float orc_f16_to_f32(uint16_t h) {
    int sign = (h >> 15) & 1;
    int e = (h >> 10) & 0x1f;
    int m = h & 0x3ff;
    double v;
    if (e == 0)
        v = ldexp((double)m, -24);               /* subnormal: m * 2^-24 */
    else if (e == 31)
        v = m ? NAN : INFINITY;                  /* inf / nan */
    else
        v = ldexp((double)(1024 + m), e - 25);   /* (1 + m/2^10) * 2^(e-15) */
    return (float)(sign ? -v : v);
}

/* bfloat16 is by definition the high 16 bits of an IEEE binary32. */
float orc_bf16_to_f32(uint16_t b) {
    uint32_t u = (uint32_t)b << 16;
    float f;
    memcpy(&f, &u, sizeof f);
    return f;
}

void orc_decode(const void* x, int dt, int64_t count, float* out) {
    for (int64_t i = 0; i < count; ++i) {
        if (dt == ORC_F16)
            out[i] = orc_f16_to_f32(((const uint16_t*)x)[i]);
        else if (dt == ORC_BF16)
            out[i] = orc_bf16_to_f32(((const uint16_t*)x)[i]);
        else
            out[i] = ((const float*)x)[i];
    }
}

/* ------------------------------------------------------------------------ */
/* Round-to-nearest-even conversion of a float to a narrower binary format  */
/* with `mbits` fraction bits, exponent bias `bias`, exponent field max      */
/* `emax_field` (all-ones = inf/nan).  Done in exact double arithmetic:      */
/* scale the magnitude so that one unit-in-the-last-place is 1.0, round      */
/* with rint() (IEEE default mode = ties-to-even), re-assemble the fields.   */
/* ------------------------------------------------------------------------ */
static uint16_t rne_narrow(float f, int mbits, int bias, int emax_field, uint16_t qnan) {
    uint16_t sign = signbit(f) ? (uint16_t)(1u << 15) : 0;
    if (isnan(f)) return qnan;
    double a = fabs((double)f);
    uint16_t inf = (uint16_t)(sign | ((uint16_t)emax_field << mbits));
    if (isinf(a)) return inf;
    if (a == 0.0) return sign;
    int ex;
    frexp(a, &ex);            /* a = fr * 2^ex, fr in [0.5, 1) */
    int e = ex - 1;           /* a in [2^e, 2^(e+1)) */
    int emin = 1 - bias;      /* smallest normal exponent */
    double r;
    if (e < emin) {
        /* subnormal range: unit = 2^(emin - mbits) */
        r = rint(ldexp(a, -(emin - mbits)));
        /* r in [0, 2^mbits]; r == 2^mbits encodes the smallest normal */
        return (uint16_t)(sign | (uint16_t)r);
    }
    r = rint(ldexp(a, -(e - mbits)));     /* in [2^mbits, 2^(mbits+1)] */
    if (r == ldexp(1.0, mbits + 1)) {     /* rounded up to the next binade */
        r = ldexp(1.0, mbits);
        e += 1;
    }
    int efield = e + bias;
    if (efield >= emax_field) return inf; /* overflow -> inf (RNE semantics) */
    uint16_t frac = (uint16_t)((uint32_t)r - (1u << mbits));
    return (uint16_t)(sign | ((uint16_t)efield << mbits) | frac);
}

uint16_t orc_f32_to_f16(float f) { return rne_narrow(f, 10, 15, 31, 0x7e00); }
uint16_t orc_f32_to_bf16(float f) { return rne_narrow(f, 7, 127, 255, 0x7fc0); }

/* ------------------------------------------------------------------------ */
/* O3 / O4. Activation quantizers (App. B.1, Eq. bool / ternary). */
/*                                                                          */
/*   bool(a, s)    = 1 if a/s >= 0.5 ; 0 if a/s < 0.5  */
/*   ternary(a, s) = 1 if a/s >= 0.5 ; 0 if -0.5 <= a/s < 0.5 ;             */
/*                  -1 if a/s < -0.5  */
/*                                                                          */
/* R1: ties follow this equation literally (+0.5 -> +1, -0.5 -> 0).          */
/* R2: the predicate a/s >= 0.5 is decided exactly: for s > 0 it equals      */
/*     a >= 0.5*s, and 0.5*s of a float s is exact in double.                */
/* R3: NaN satisfies none of the comparisons -> the "otherwise" value 0.     */
/* ------------------------------------------------------------------------ */
int orc_quant_act(float a, float s, int kind) {
    double t = 0.5 * (double)s;          /* exact */
    double x = (double)a;                /* exact */
    if (kind == ORC_BOOL) return (x >= t) ? 1 : 0;
    if (x >= t) return 1;                /* a/s >= 0.5 */
    if (x < -t) return -1;               /* a/s < -0.5 */
    return 0;                            /* -0.5 <= a/s < 0.5 (and NaN, R3) */
}

/* ------------------------------------------------------------------------ */
/* A1 / A2. Weight binarisation (P:901-909 Eq. sign; P:934-939 Eq. bw):      */
/*   sign(w - mu) = +1 if (w - mu) >= 0, else -1.                           */
/* The difference of two floats taken in double has the sign of the exact   */
/* difference and is zero iff w == mu, so the comparison is exact.  NaN     */
/* falls in "otherwise" -> -1 (R3); -0.0 - 0 = -0.0 >= 0 -> +1 (R4).         */
/* ------------------------------------------------------------------------ */
int orc_sign_weight(float w, float mu) {
    double d = (double)w - (double)mu;
    return (d >= 0.0) ? 1 : -1;
}

/* Quantize a row-major [rows x cols] float matrix (leading dim ld). */
void orc_quantize_act(const float* x, int64_t rows, int64_t cols, int64_t ld,
                      float s, int kind, int8_t* q /* [rows x cols] */) {
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t c = 0; c < cols; ++c)
            q[r * cols + c] = (int8_t)orc_quant_act(x[r * ld + c], s, kind);
}

/* mu: NULL -> 0; mu_per_row -> mu[r], else mu[0] */
void orc_binarize_weight(const float* w, int64_t n, int64_t k, int64_t ld,
                         const float* mu, int mu_per_row, int8_t* q) {
    for (int64_t r = 0; r < n; ++r) {
        float m = mu ? (mu_per_row ? mu[r] : mu[0]) : 0.0f;
        for (int64_t c = 0; c < k; ++c)
            q[r * k + c] = (int8_t)orc_sign_weight(w[r * ld + c], m);
    }
}

/* Mean of a matrix in double (P:936 mu(W)); used by tests and the recipe. */
double orc_mean(const float* w, int64_t count) {
    double acc = 0.0;
    for (int64_t i = 0; i < count; ++i) acc += (double)w[i];
    return acc / (double)count;
}

/* ------------------------------------------------------------------------ */
/* O6. The packed-plane format (the bit-exact contract of include/bwta.h).  */
/* Element (r, c) of a [rows x cols] quantized matrix lives in row r, word  */
/* c/32, bit c%32 (LSB first).  Planes:                                     */
/*   nz  bit = 1  <=>  q != 0          (ternary / bool)                     */
/*   sgn bit = 1  <=>  q <  0          (ternary / binary; "negative   */
/*                                      numbers are stored as bit 1")       */
/* Each row holds ldw words; all bits of elements >= cols are 0.            */
/* sgn or nz may be NULL when not wanted.                                   */
/* ------------------------------------------------------------------------ */
void orc_pack(const int8_t* q, int64_t rows, int64_t cols, int64_t ldw,
              uint32_t* sgn, uint32_t* nz) {
    for (int64_t r = 0; r < rows; ++r) {
        for (int64_t w = 0; w < ldw; ++w) {
            if (sgn) sgn[r * ldw + w] = 0;
            if (nz) nz[r * ldw + w] = 0;
        }
        for (int64_t c = 0; c < cols; ++c) {
            int v = q[r * cols + c];
            uint32_t bit = (uint32_t)1 << (c % 32);
            if (nz && v != 0) nz[r * ldw + c / 32] |= bit;
            if (sgn && v < 0) sgn[r * ldw + c / 32] |= bit;
        }
    }
}

/* Inverse of orc_pack for a given kind (reads the format definition back):  */
/*   BINARY : q = sgn ? -1 : +1      BOOL : q = nz ? 1 : 0                  */
/*   TERNARY: q = nz ? (sgn ? -1 : +1) : 0                                  */
void orc_unpack(const uint32_t* sgn, const uint32_t* nz, int kind,
                int64_t rows, int64_t cols, int64_t ldw, int8_t* q) {
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t c = 0; c < cols; ++c) {
            int sb = sgn ? (int)((sgn[r * ldw + c / 32] >> (c % 32)) & 1u) : 0;
            int nb = nz ? (int)((nz[r * ldw + c / 32] >> (c % 32)) & 1u) : 0;
            int v;
            if (kind == ORC_BINARY) v = sb ? -1 : 1;
            else if (kind == ORC_BOOL) v = nb ? 1 : 0;
            else v = nb ? (sb ? -1 : 1) : 0;
            q[r * cols + c] = (int8_t)v;
        }
}

/* Per-row count of non-zero quantized values (row_nnz of bwta_pack_act). */
void orc_row_nnz(const int8_t* q, int64_t rows, int64_t cols, int32_t* out) {
    for (int64_t r = 0; r < rows; ++r) {
        int32_t n = 0;
        for (int64_t c = 0; c < cols; ++c) n += (q[r * cols + c] != 0);
        out[r] = n;
    }
}

/* ------------------------------------------------------------------------ */
/* O7. Integer dot products (P:949-957 Eq. bwta_linear).          */
/*   dot[m][n] = sum_k a[m][k] * b[n][k]      ("B pre-transposed")          */
/* A naive triple loop over unpacked integers.  Rows of the output are      */
/* split across `threads` POSIX threads (each output is still the same      */
/* sequential k-loop; integer addition makes the order irrelevant).         */
/* ------------------------------------------------------------------------ */
typedef struct {
    const int8_t* a; const int8_t* b; int32_t* out;
    int64_t m0, m1, n, k;
} dot_job;

static void* dot_worker(void* p) {
    dot_job* j = (dot_job*)p;
    for (int64_t m = j->m0; m < j->m1; ++m)
        for (int64_t n = 0; n < j->n; ++n) {
            int32_t acc = 0;
            for (int64_t kk = 0; kk < j->k; ++kk)
                acc += (int32_t)j->a[m * j->k + kk] * (int32_t)j->b[n * j->k + kk];
            j->out[m * j->n + n] = acc;
        }
    return NULL;
}

void orc_dot(const int8_t* a /* [M x K] */, const int8_t* b /* [N x K] */,
             int64_t M, int64_t N, int64_t K, int32_t* out /* [M x N] */, int threads) {
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    if (threads > M) threads = (int)(M > 0 ? M : 1);
    pthread_t tid[256];
    dot_job jobs[256];
    for (int t = 0; t < threads; ++t) {
        jobs[t].a = a; jobs[t].b = b; jobs[t].out = out;
        jobs[t].m0 = M * t / threads; jobs[t].m1 = M * (t + 1) / threads;
        jobs[t].n = N; jobs[t].k = K;
    }
    if (threads == 1) { dot_worker(&jobs[0]); return; }
    for (int t = 0; t < threads; ++t) pthread_create(&tid[t], NULL, dot_worker, &jobs[t]);
    for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
}

/* ------------------------------------------------------------------------ */
/* O8. Float epilogue (linear(A) = s_W * s_A * BWTA(...);         */
/*     INT32 results converted to floating point).             */
/* R5 evaluation order (fixed so both sides round identically):              */
/*   c_n = fl32(s_w[n] * s_a);  y = fl32(float(dot) * c_n);  out = RNE(y).   */
/* Attention uses c = alpha (= s_Q s_K / sqrt(D))    */
/* or beta (= s_Att s_V), passed in by the caller.                          */
/* ------------------------------------------------------------------------ */
static void store_out(void* out, int dt, int64_t idx, float y, int32_t dot) {
    if (dt == ORC_F16) ((uint16_t*)out)[idx] = orc_f32_to_f16(y);
    else if (dt == ORC_BF16) ((uint16_t*)out)[idx] = orc_f32_to_bf16(y);
    else if (dt == ORC_F32) ((float*)out)[idx] = y;
    else ((int32_t*)out)[idx] = dot;   /* raw integer output, scales ignored */
}

void orc_epilogue_linear(const int32_t* dot, int64_t M, int64_t N,
                         const float* s_w /* [N] or NULL -> 1 */, float s_a,
                         int out_dt, void* out) {
    for (int64_t m = 0; m < M; ++m)
        for (int64_t n = 0; n < N; ++n) {
            volatile float sw = s_w ? s_w[n] : 1.0f;
            volatile float c = sw * s_a;                 /* fl32(s_w * s_a) */
            volatile float y = (float)dot[m * N + n] * c; /* fl32(dot * c)  */
            store_out(out, out_dt, m * N + n, y, dot[m * N + n]);
        }
}

void orc_epilogue_scalar(const int32_t* dot, int64_t count, float alpha,
                         int out_dt, void* out) {
    for (int64_t i = 0; i < count; ++i) {
        volatile float y = (float)dot[i] * alpha;
        store_out(out, out_dt, i, y, dot[i]);
    }
}

/* Vector form of the RNE converters (used to build expected outputs). */
void orc_encode(const float* y, int64_t count, int dt, uint16_t* out) {
    for (int64_t i = 0; i < count; ++i)
        out[i] = (dt == ORC_F16) ? orc_f32_to_f16(y[i]) : orc_f32_to_bf16(y[i]);
}
