/*
 * starmm_oracle.c -- CPU restatement of the reference's semiring MM path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing under oracle/ is part of the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker or
 * as the timed CPU baseline.  The product path (paper_1911_05328_b200) never
 * links or calls it.
 *
 * Every function restates a reference function (paths relative to
 * /root/reference/pkg/src/starmm/):
 *
 *   oracle_mm_i64        _mm_int       semiring.py:22-32  (i-k-j, from 0, wraps mod 2^64)
 *   oracle_mm_f64        _mm_float     semiring.py:35-45  (i-k-j, from 0.0, separate mul+add)
 *   oracle_mm_minplus_f64 _mm_minplus  semiring.py:48-60  (from +inf, "if v < out" -> NaN
 *                                                          candidates ignored)
 *   oracle_fold_*        fold_add      semiring.py:116-117 (np.add), 126-127 (np.minimum,
 *                                                          NaN-propagating)
 *   oracle_serial_mm     co2/tar/sar/star at workers=1 (classic.py:117-236): the serial
 *                        depth-first 8-way recursion, leaf = b x b product from the
 *                        identity folded into C (ops.py:30-65, 68-101)
 *   oracle_co3_mm        co3 at workers=1 (classic.py:133-155, ops.py:108-155)
 *
 * New semiring ids of this build (SURVEY.md key finding 1) have no reference
 * kernel; their oracles follow the same loop structure:
 *   oracle_mm_minplus_f32  fp32 (min,+), fp32 adds, "if v < out"
 *   oracle_mm_minplus_i32  int32 (min,+) with INT32_MAX = +inf (absorbing for the
 *                          product), finite sums saturate to +inf above INT32_MAX-1
 *                          and to INT32_MIN below it.
 *
 * Compile with -O2 -ffp-contract=off (no FMA contraction, no fast-math): numba's
 * default (non-fastmath) LLVM pipeline does not contract a*b+c either, so the
 * float64 loops round exactly like the reference's.
 *
 * With par != 0 the products split their output rows across pthreads (one per
 * online core, or oracle_set_threads); each output element still sees the same
 * k order, so results are bitwise identical to the serial loops.  This exists
 * for the CPU-baseline timing legs.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#include <pthread.h>
#include <unistd.h>

#define I32_INF INT32_MAX

static int g_threads = 0;

void oracle_set_threads(int t) { g_threads = t; }

int oracle_num_threads(void) {
    if (g_threads > 0) return g_threads;
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    return n > 0 ? (int)n : 1;
}

/* Row-parallel driver: body(ctx, i0, i1) over [0, r). */
typedef void (*rows_fn)(const void* ctx, int64_t i0, int64_t i1);
typedef struct { rows_fn fn; const void* ctx; int64_t i0, i1; } rows_job;

static void* rows_thread(void* p) {
    rows_job* j = (rows_job*)p;
    j->fn(j->ctx, j->i0, j->i1);
    return NULL;
}

static void run_rows(rows_fn fn, const void* ctx, int64_t r, int par) {
    int t = par ? oracle_num_threads() : 1;
    if (t > r) t = (int)r;
    if (t <= 1) { fn(ctx, 0, r); return; }
    pthread_t th[256];
    rows_job jobs[256];
    if (t > 256) t = 256;
    for (int q = 0; q < t; ++q) {
        jobs[q].fn = fn; jobs[q].ctx = ctx;
        jobs[q].i0 = r * q / t; jobs[q].i1 = r * (q + 1) / t;
        pthread_create(&th[q], NULL, rows_thread, &jobs[q]);
    }
    for (int q = 0; q < t; ++q) pthread_join(th[q], NULL);
}

typedef struct {
    const void* A; const void* B; void* out;
    int64_t kk, c, lda, ldb, ldo;
} mm_args;

#define MM_WRAPPER(NAME, BODY_FN, TA, TO)                                            \
    void NAME(const TA* A, const TA* B, TO* out, int64_t r, int64_t kk, int64_t c,   \
              int64_t lda, int64_t ldb, int64_t ldo, int par) {                      \
        mm_args a = { A, B, out, kk, c, lda, ldb, ldo };                             \
        run_rows(BODY_FN, &a, r, par);                                               \
    }

/* ---- dense products from the additive identity (Semiring.matmul) ------- */

/* semiring.py:22-32.  Unsigned arithmetic gives numpy's wrap-around. */
static void oracle_mm_i64_rows(const void* ctx, int64_t i0, int64_t i1) {
    const mm_args* x = (const mm_args*)ctx;
    const int64_t* A = (const int64_t*)x->A; const int64_t* B = (const int64_t*)x->B; int64_t* out = (int64_t*)x->out;
    int64_t kk = x->kk, c = x->c, lda = x->lda, ldb = x->ldb, ldo = x->ldo;
    for (int64_t i = i0; i < i1; ++i) {
        uint64_t* o = (uint64_t*)(out + i * ldo);
        for (int64_t j = 0; j < c; ++j) o[j] = 0;
        for (int64_t k = 0; k < kk; ++k) {
            uint64_t aik = (uint64_t)A[i * lda + k];
            const uint64_t* b = (const uint64_t*)(B + k * ldb);
            for (int64_t j = 0; j < c; ++j) o[j] += aik * b[j];
        }
    }
}
MM_WRAPPER(oracle_mm_i64, oracle_mm_i64_rows, int64_t, int64_t)


/* semiring.py:35-45 */
static void oracle_mm_f64_rows(const void* ctx, int64_t i0, int64_t i1) {
    const mm_args* x = (const mm_args*)ctx;
    const double* A = (const double*)x->A; const double* B = (const double*)x->B; double* out = (double*)x->out;
    int64_t kk = x->kk, c = x->c, lda = x->lda, ldb = x->ldb, ldo = x->ldo;
    for (int64_t i = i0; i < i1; ++i) {
        double* o = out + i * ldo;
        for (int64_t j = 0; j < c; ++j) o[j] = 0.0;
        for (int64_t k = 0; k < kk; ++k) {
            double aik = A[i * lda + k];
            const double* b = B + k * ldb;
            for (int64_t j = 0; j < c; ++j) o[j] += aik * b[j];
        }
    }
}
MM_WRAPPER(oracle_mm_f64, oracle_mm_f64_rows, double, double)


/* semiring.py:48-60 */
static void oracle_mm_minplus_f64_rows(const void* ctx, int64_t i0, int64_t i1) {
    const mm_args* x = (const mm_args*)ctx;
    const double* A = (const double*)x->A; const double* B = (const double*)x->B; double* out = (double*)x->out;
    int64_t kk = x->kk, c = x->c, lda = x->lda, ldb = x->ldb, ldo = x->ldo;
    for (int64_t i = i0; i < i1; ++i) {
        double* o = out + i * ldo;
        for (int64_t j = 0; j < c; ++j) o[j] = INFINITY;
        for (int64_t k = 0; k < kk; ++k) {
            double aik = A[i * lda + k];
            const double* b = B + k * ldb;
            for (int64_t j = 0; j < c; ++j) {
                double v = aik + b[j];
                if (v < o[j]) o[j] = v;
            }
        }
    }
}
MM_WRAPPER(oracle_mm_minplus_f64, oracle_mm_minplus_f64_rows, double, double)


/* fp32 (min,+): same loop in float arithmetic (new id "tropical_f32"). */
static void oracle_mm_minplus_f32_rows(const void* ctx, int64_t i0, int64_t i1) {
    const mm_args* x = (const mm_args*)ctx;
    const float* A = (const float*)x->A; const float* B = (const float*)x->B; float* out = (float*)x->out;
    int64_t kk = x->kk, c = x->c, lda = x->lda, ldb = x->ldb, ldo = x->ldo;
    for (int64_t i = i0; i < i1; ++i) {
        float* o = out + i * ldo;
        for (int64_t j = 0; j < c; ++j) o[j] = INFINITY;
        for (int64_t k = 0; k < kk; ++k) {
            float aik = A[i * lda + k];
            const float* b = B + k * ldb;
            for (int64_t j = 0; j < c; ++j) {
                float v = aik + b[j];
                if (v < o[j]) o[j] = v;
            }
        }
    }
}
MM_WRAPPER(oracle_mm_minplus_f32, oracle_mm_minplus_f32_rows, float, float)


/* int32 (min,+) (new id "tropical_i32"): INT32_MAX is +inf. */
static inline int32_t i32_tropical_mul(int32_t a, int32_t b) {
    if (a == I32_INF || b == I32_INF) return I32_INF;
    int64_t s = (int64_t)a + (int64_t)b;
    if (s >= (int64_t)I32_INF) return I32_INF;
    if (s < (int64_t)INT32_MIN) return INT32_MIN;
    return (int32_t)s;
}

static void oracle_mm_minplus_i32_rows(const void* ctx, int64_t i0, int64_t i1) {
    const mm_args* x = (const mm_args*)ctx;
    const int32_t* A = (const int32_t*)x->A; const int32_t* B = (const int32_t*)x->B; int32_t* out = (int32_t*)x->out;
    int64_t kk = x->kk, c = x->c, lda = x->lda, ldb = x->ldb, ldo = x->ldo;
    for (int64_t i = i0; i < i1; ++i) {
        int32_t* o = out + i * ldo;
        for (int64_t j = 0; j < c; ++j) o[j] = I32_INF;
        for (int64_t k = 0; k < kk; ++k) {
            int32_t aik = A[i * lda + k];
            const int32_t* b = B + k * ldb;
            for (int64_t j = 0; j < c; ++j) {
                int32_t v = i32_tropical_mul(aik, b[j]);
                if (v < o[j]) o[j] = v;
            }
        }
    }
}
MM_WRAPPER(oracle_mm_minplus_i32, oracle_mm_minplus_i32_rows, int32_t, int32_t)


/* ---- fold_add: C <- C (+) D (semiring.py:96-98, 116-117, 126-127) ------ */

void oracle_fold_i64(int64_t* C, const int64_t* D, int64_t r, int64_t c,
                     int64_t ldc, int64_t ldd) {
    for (int64_t i = 0; i < r; ++i)
        for (int64_t j = 0; j < c; ++j)
            C[i * ldc + j] = (int64_t)((uint64_t)C[i * ldc + j] + (uint64_t)D[i * ldd + j]);
}

void oracle_fold_f64(double* C, const double* D, int64_t r, int64_t c,
                     int64_t ldc, int64_t ldd) {
    for (int64_t i = 0; i < r; ++i)
        for (int64_t j = 0; j < c; ++j) C[i * ldc + j] += D[i * ldd + j];
}

/* np.minimum(C, D): NaN if either operand is NaN; on a tie the SECOND operand wins
 * (np.minimum(+0.0, -0.0) == -0.0, np.minimum(-0.0, +0.0) == +0.0 -- MINPD order,
 * pinned by tests/golden/ref_signed_zero.npz). */
void oracle_fold_min_f64(double* C, const double* D, int64_t r, int64_t c,
                         int64_t ldc, int64_t ldd) {
    for (int64_t i = 0; i < r; ++i)
        for (int64_t j = 0; j < c; ++j) {
            double x = C[i * ldc + j], y = D[i * ldd + j];
            C[i * ldc + j] = (x != x || y != y) ? NAN : (x < y ? x : y);
        }
}

void oracle_fold_min_f32(float* C, const float* D, int64_t r, int64_t c,
                         int64_t ldc, int64_t ldd) {
    for (int64_t i = 0; i < r; ++i)
        for (int64_t j = 0; j < c; ++j) {
            float x = C[i * ldc + j], y = D[i * ldd + j];
            C[i * ldc + j] = (x != x || y != y) ? NAN : (x < y ? x : y);
        }
}

void oracle_fold_min_i32(int32_t* C, const int32_t* D, int64_t r, int64_t c,
                         int64_t ldc, int64_t ldd) {
    for (int64_t i = 0; i < r; ++i)
        for (int64_t j = 0; j < c; ++j) {
            int32_t x = C[i * ldc + j], y = D[i * ldd + j];
            C[i * ldc + j] = y < x ? y : x;
        }
}

/* ---- generic dispatch by semiring id ----------------------------------- */
/* Semiring ids shared with include/starmm_b200.h. */
enum { SR_INT64 = 0, SR_FP64 = 1, SR_TROP_F64 = 2, SR_TROP_F32 = 3, SR_TROP_I32 = 4 };

static size_t elem_size(int sr) { return (sr == SR_TROP_F32 || sr == SR_TROP_I32) ? 4 : 8; }

int oracle_matmul(int sr, const void* A, const void* B, void* out,
                  int64_t r, int64_t kk, int64_t c,
                  int64_t lda, int64_t ldb, int64_t ldo, int par) {
    switch (sr) {
    case SR_INT64: oracle_mm_i64(A, B, out, r, kk, c, lda, ldb, ldo, par); return 0;
    case SR_FP64: oracle_mm_f64(A, B, out, r, kk, c, lda, ldb, ldo, par); return 0;
    case SR_TROP_F64: oracle_mm_minplus_f64(A, B, out, r, kk, c, lda, ldb, ldo, par); return 0;
    case SR_TROP_F32: oracle_mm_minplus_f32(A, B, out, r, kk, c, lda, ldb, ldo, par); return 0;
    case SR_TROP_I32: oracle_mm_minplus_i32(A, B, out, r, kk, c, lda, ldb, ldo, par); return 0;
    }
    return 1;
}

int oracle_fold(int sr, void* C, const void* D, int64_t r, int64_t c,
                int64_t ldc, int64_t ldd) {
    switch (sr) {
    case SR_INT64: oracle_fold_i64(C, D, r, c, ldc, ldd); return 0;
    case SR_FP64: oracle_fold_f64(C, D, r, c, ldc, ldd); return 0;
    case SR_TROP_F64: oracle_fold_min_f64(C, D, r, c, ldc, ldd); return 0;
    case SR_TROP_F32: oracle_fold_min_f32(C, D, r, c, ldc, ldd); return 0;
    case SR_TROP_I32: oracle_fold_min_i32(C, D, r, c, ldc, ldd); return 0;
    }
    return 1;
}

/* C <- C (+) A (x) B over r x c output with inner dim kk (the sampled-tile oracle:
 * fold_add(C0_tile, matmul(A_panel, B_panel))). */
int oracle_gemm_fold(int sr, void* C, const void* A, const void* B,
                     int64_t r, int64_t kk, int64_t c,
                     int64_t ldc, int64_t lda, int64_t ldb, int par) {
    size_t e = elem_size(sr);
    void* tmp = malloc((size_t)r * (size_t)c * e);
    if (!tmp) return 2;
    int rc = oracle_matmul(sr, A, B, tmp, r, kk, c, lda, ldb, c, par);
    if (!rc) rc = oracle_fold(sr, C, tmp, r, c, ldc, c);
    free(tmp);
    return rc;
}

/* ---- serial schedules at workers=1 ------------------------------------- */
/*
 * classic.py:86-93 (_mm_children): children in order k-outer, then i, then j.
 * With one worker every schedule except co3 reduces to the same depth-first
 * walk with an in-place leaf C <- C (+) (A (x) B) (co2: ops.py:41-46; tar:
 * classic.py:160-167 product_into + accumulate_region; sar/star serial:
 * PairState Empty then FirstDone, both in place, classic.py:190-204).
 */
typedef struct { int sr; int64_t b; void* tmp; } ser_ctx;

static void* at(int sr, const void* base, int64_t ld, int64_t r, int64_t c) {
    return (char*)base + ((size_t)(r * ld + c)) * elem_size(sr);
}

static void serial_rec(ser_ctx* x, void* C, const void* A, const void* B,
                       int64_t m, int64_t ldc, int64_t lda, int64_t ldb) {
    if (m == x->b) {
        oracle_matmul(x->sr, A, B, x->tmp, m, m, m, lda, ldb, m, 0);
        oracle_fold(x->sr, C, x->tmp, m, m, ldc, m);
        return;
    }
    int64_t h = m / 2;
    for (int k = 0; k < 2; ++k)
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 2; ++j)
                serial_rec(x, at(x->sr, C, ldc, i * h, j * h),
                           at(x->sr, A, lda, i * h, k * h),
                           at(x->sr, B, ldb, k * h, j * h), h, ldc, lda, ldb);
}

int oracle_serial_mm(int sr, void* C, const void* A, const void* B, int64_t n, int64_t b) {
    if (b < 1 || n < b || (n & (n - 1)) || (b & (b - 1))) return 3;
    ser_ctx x = { sr, b, malloc((size_t)(b * b) * elem_size(sr)) };
    if (!x.tmp) return 2;
    serial_rec(&x, C, A, B, n, n, n, n);
    free(x.tmp);
    return 0;
}

/*
 * co3 at workers=1 (classic.py:141-155): per node a fresh temporary D (virgin:
 * first write stores), children k=0 -> C quadrants, k=1 -> D quadrants, run in
 * order, then merge_tasks(C, D) (ops.py:108-155: fold D into C; virgin targets
 * are stored, which only happens for targets inside a temporary).
 *
 * Virgin tracking is per b x b tile of each temporary, as in the reference
 * (TileExclusionTable.virgin, matrix.py:64-90).
 */
typedef struct {
    int sr; int64_t b;
    void* tmp;               /* b x b product scratch */
} co3_ctx;

/* A destination region: a buffer plus an optional virgin map over its b-tiles. */
typedef struct { void* base; int64_t ld; unsigned char* virgin; int64_t vtc; } dst_t;

static void leaf_store_or_fold(co3_ctx* x, dst_t d, int64_t r0, int64_t c0, const void* vals,
                               int64_t ldv) {
    void* C = at(x->sr, d.base, d.ld, r0, c0);
    int64_t b = x->b;
    if (d.virgin) {
        unsigned char* v = &d.virgin[(r0 / b) * d.vtc + (c0 / b)];
        if (*v) {
            size_t e = elem_size(x->sr);
            for (int64_t i = 0; i < b; ++i)
                memcpy((char*)C + (size_t)(i * d.ld) * e, (const char*)vals + (size_t)(i * ldv) * e,
                       (size_t)b * e);
            *v = 0;
            return;
        }
    }
    oracle_fold(x->sr, C, vals, b, b, d.ld, ldv);
}

static void co3_rec(co3_ctx* x, dst_t C, int64_t cr, int64_t cc,
                    const void* A, const void* B, int64_t m, int64_t lda, int64_t ldb) {
    int64_t b = x->b;
    if (m == b) {
        oracle_matmul(x->sr, A, B, x->tmp, b, b, b, lda, ldb, b, 0);
        leaf_store_or_fold(x, C, cr, cc, x->tmp, b);
        return;
    }
    int64_t h = m / 2;
    size_t e = elem_size(x->sr);
    int64_t vt = m / b;
    dst_t D = { malloc((size_t)(m * m) * e), m, malloc((size_t)(vt * vt)), vt };
    memset(D.virgin, 1, (size_t)(vt * vt));
    for (int k = 0; k < 2; ++k)
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 2; ++j) {
                const void* Aq = at(x->sr, A, lda, i * h, k * h);
                const void* Bq = at(x->sr, B, ldb, k * h, j * h);
                if (k == 0) co3_rec(x, C, cr + i * h, cc + j * h, Aq, Bq, h, lda, ldb);
                else co3_rec(x, D, i * h, j * h, Aq, Bq, h, lda, ldb);
            }
    /* merge_tasks: tile-by-tile (the recursion order does not matter for values:
     * each tile of C receives exactly one fold of the matching D tile). */
    for (int64_t ti = 0; ti < vt; ++ti)
        for (int64_t tj = 0; tj < vt; ++tj)
            leaf_store_or_fold(x, C, cr + ti * b, cc + tj * b,
                               at(x->sr, D.base, m, ti * b, tj * b), m);
    free(D.base);
    free(D.virgin);
}

int oracle_co3_mm(int sr, void* C, const void* A, const void* B, int64_t n, int64_t b) {
    if (b < 1 || n < b || (n & (n - 1)) || (b & (b - 1))) return 3;
    co3_ctx x = { sr, b, malloc((size_t)(b * b) * elem_size(sr)) };
    if (!x.tmp) return 2;
    dst_t Cd = { C, n, NULL, 0 };
    co3_rec(&x, Cd, 0, 0, A, B, n, n, n);
    free(x.tmp);
    return 0;
}

/* ==========================================================================
 * Input generator restatement (paper_1911_05328_b200/csrc/generate.cuh): the
 * counter-based panels the device generates, regenerated on the host so that
 * sampled output tiles of full-size runs can be checked.  Philox4x32-10 (Salmon
 * et al., SC'11; pinned by its published known-answer vectors in
 * tests/test_oracle.py), then + - * / and sqrt only, no FMA contraction (this file
 * is compiled with -ffp-contract=off), with the same correctly rounded constants.
 * ========================================================================== */
void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3], k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; ++r) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c0, p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static const double G_INV_ODD[12] = {
    0x1.0000000000000p+0, 0x1.5555555555555p-2, 0x1.999999999999ap-3, 0x1.2492492492492p-3,
    0x1.c71c71c71c71cp-4, 0x1.745d1745d1746p-4, 0x1.3b13b13b13b14p-4, 0x1.1111111111111p-4,
    0x1.e1e1e1e1e1e1ep-5, 0x1.af286bca1af28p-5, 0x1.8618618618618p-5, 0x1.642c8590b2164p-5};
static const double G_IFE[14] = {
    0x1.0000000000000p+0, 0x1.0000000000000p-1, 0x1.5555555555555p-5, 0x1.6c16c16c16c17p-10,
    0x1.a01a01a01a01ap-16, 0x1.27e4fb7789f5cp-22, 0x1.1eed8eff8d898p-29, 0x1.93974a8c07c9dp-37,
    0x1.ae7f3e733b81fp-45, 0x1.6827863b97d97p-53, 0x1.e542ba4020225p-62, 0x1.0ce396db7f853p-70,
    0x1.f2cf01972f578p-80, 0x1.88e85fc6a4e5ap-89};
static const double G_IFO[14] = {
    0x1.0000000000000p+0, 0x1.5555555555555p-3, 0x1.1111111111111p-7, 0x1.a01a01a01a01ap-13,
    0x1.71de3a556c734p-19, 0x1.ae64567f544e4p-26, 0x1.6124613a86d09p-33, 0x1.ae7f3e733b81fp-41,
    0x1.952c77030ad4ap-49, 0x1.2f49b46814157p-57, 0x1.71b8ef6dcf572p-66, 0x1.761b41316381ap-75,
    0x1.3f3ccdd165fa9p-84, 0x1.d1ab1c2dccea3p-94};

static double g_log(double x) {
    uint64_t bits;
    memcpy(&bits, &x, 8);
    int e = (int)((bits >> 52) & 0x7ff) - 1023;
    bits = (bits & 0x000fffffffffffffULL) | 0x3ff0000000000000ULL;
    double m;
    memcpy(&m, &bits, 8);
    if (m > 0x1.6a09e667f3bcdp+0) { m = m * 0.5; e += 1; }
    const double s = (m - 1.0) / (m + 1.0);
    const double s2 = s * s;
    double t = G_INV_ODD[11];
    for (int k = 10; k >= 0; --k) t = t * s2 + G_INV_ODD[k];
    const double lm = (2.0 * s) * t;
    return (double)e * 0x1.62e42fee00000p-1 + ((double)e * 0x1.a39ef35793c76p-33 + lm);
}

static double g_cos2pi(double u) {
    const double t = u * 4.0;
    const int q = (int)t;
    const double f = t - (double)q;
    const double a = f * 0x1.921fb54442d18p+0;
    const double a2 = a * a;
    double c = -G_IFE[13], sn = -G_IFO[13];
    for (int k = 12; k >= 0; --k) {
        const double ce = (k & 1) ? -G_IFE[k] : G_IFE[k];
        const double so = (k & 1) ? -G_IFO[k] : G_IFO[k];
        c = c * a2 + ce;
        sn = sn * a2 + so;
    }
    sn = sn * a;
    switch (q & 3) {
    case 0: return c;
    case 1: return -sn;
    case 2: return -c;
    default: return sn;
    }
}

/* value of element (i, j); *absent for a GRAPH non-edge */
static double g_value(int dist, double a, double b, double p, uint64_t seed, uint32_t stream,
                      int64_t i, int64_t j, int* absent) {
    uint32_t ctr[4] = {(uint32_t)j, (uint32_t)i, stream, 0u}, key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t x[4];
    oracle_philox4x32_10(ctr, key, x);
    *absent = 0;
    const double two_m53 = 1.1102230246251565e-16;
    if (dist == 0) {
        const uint64_t u53 = ((uint64_t)x[0] << 21) | (x[1] >> 11);
        return a + (b - a) * ((double)u53 * two_m53);
    }
    if (dist == 1) {
        const uint64_t ua = ((uint64_t)x[0] << 21) | (x[1] >> 11);
        const uint64_t ub = ((uint64_t)x[2] << 21) | (x[3] >> 11);
        const double u1 = (double)(ua + 1) * two_m53, u2 = (double)ub * two_m53;
        const double rad = sqrt(-2.0 * g_log(u1));
        return a + b * (rad * g_cos2pi(u2));
    }
    if (dist == 3) {
        const uint32_t thr = (uint32_t)(p * 4294967296.0);
        if (!(x[1] < thr)) { *absent = 1; return 0.0; }
    }
    const uint64_t span = (uint64_t)((int64_t)b - (int64_t)a + 1);
    return (double)((int64_t)a + (int64_t)(((uint64_t)x[0] * span) >> 32));
}

int oracle_generate(int sr, int dist, void* out, int64_t ld, int64_t rows, int64_t cols, int64_t row0,
                    int64_t col0, uint64_t seed, uint32_t stream, double a, double b, double p, int flags) {
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t c = 0; c < cols; ++c) {
            const int64_t i = row0 + r, j = col0 + c;
            int absent;
            const double v = g_value(dist, a, b, p, seed, stream, i, j, &absent);
            const int diag = (flags & 1) && i == j;
            switch (sr) {
            case SR_INT64: ((int64_t*)out)[r * ld + c] = diag ? 0 : (absent ? 0 : (int64_t)v); break;
            case SR_FP64: ((double*)out)[r * ld + c] = diag ? 0.0 : (absent ? 0.0 : v); break;
            case SR_TROP_F64: ((double*)out)[r * ld + c] = diag ? 0.0 : (absent ? INFINITY : v); break;
            case SR_TROP_F32: ((float*)out)[r * ld + c] = diag ? 0.0f : (absent ? INFINITY : (float)v); break;
            case SR_TROP_I32: ((int32_t*)out)[r * ld + c] = diag ? 0 : (absent ? I32_INF : (int32_t)v); break;
            default: return 1;
            }
        }
    return 0;
}
