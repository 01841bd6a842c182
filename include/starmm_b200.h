/*
 * starmm_b200.h -- C ABI of the B200-native semiring matrix-multiplication path.
 *
 * This is the drop-in boundary under the reference package's Python surface
 * (starmm, /root/reference/pkg/src/starmm).  No C++ types, no torch types:
 * plain device pointers, element strides and an opaque cudaStream_t passed
 * as void*.  Every function returns an int status (0 = ok); no C++ exception
 * crosses this boundary.  Status codes map 1:1 onto the reference exception
 * classes (errors.py:4-41).
 *
 * Which reference interface each entry point replaces (file:line relative to
 * /root/reference/pkg/src/starmm/):
 *
 *   starmm_plan_create   Executor.__init__(cfg) + Config (runtime.py:60-79,
 *                        matrix.py:32-61): binds semiring, schedule, base_dim,
 *                        workers and allocation mode; owns the block pool
 *                        (pool.py:67-88) as a device scratch arena.
 *   starmm_execute       registry.run_algorithm (registry.py:23-57) ->
 *                        classic._classic_root (classic.py:241-265) for
 *                        co2 / co3 / tar / sar / star: C <- C (+) A (x) B.
 *   starmm_plan_stats    Pool.snapshot_counts (pool.py:158-167) +
 *                        MetricsSnapshot (metrics.py:19-36) GPU analogues.
 *   starmm_plan_reset_stats  Pool.reset (pool.py:148-156).
 *   starmm_plan_destroy  Executor.close (runtime.py:83-93).
 *   starmm_matmul        Semiring.matmul (semiring.py:92-94; numba kernels
 *                        _mm_int / _mm_float / _mm_minplus, semiring.py:22-60):
 *                        out <- A (x) B from the additive identity.
 *   starmm_madd          kernels.madd (kernels.py:47-52) / Semiring.fold_add
 *                        (semiring.py:96-98, 116-117, 126-127): C <- C (+) D.
 *   starmm_atomic_accumulate  classic.atomic_accumulate (classic.py:268-284) /
 *                        ops.accumulate_region (ops.py:76-101): concurrent-safe
 *                        C <- C (+) P (hardware atomics / per-tile slots).
 *   starmm_strerror      str(exception) for the status taxonomy.
 *   STARMM_STRASSEN..    strassen_parallel / sar_strassen / star_strassen_1/2
 *                        (strassen.py:211-235) via starmm_execute.
 *
 * Matrices are row-major with a leading dimension in ELEMENTS (ld >= cols),
 * like MatrixRegion.row_stride (matrix.py:144-146).  The caller owns A, B and
 * C; the library reads A and B and updates C in place.  Calls are stream-
 * ordered on `stream` and, like the reference entry points, block until the
 * result is in C (STARMM_F_ASYNC opts out of the final synchronisation).
 */
#ifndef STARMM_B200_H_
#define STARMM_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STARMM_ABI_VERSION 3

/* ---- status codes (errors.py:4-41) ------------------------------------- */
enum starmm_status {
    STARMM_OK = 0,
    STARMM_DIM_MISMATCH = 1,          /* DimMismatch        errors.py:8  */
    STARMM_INVALID_SPLIT = 2,         /* InvalidSplit       errors.py:12 */
    STARMM_NOT_BASE_CASE = 3,         /* NotBaseCase        errors.py:16 */
    STARMM_ALLOC_FAILURE = 4,         /* AllocFailure       errors.py:20 */
    STARMM_CONTRACT_VIOLATION = 5,    /* ContractViolation  errors.py:24 */
    STARMM_ALIGNMENT_ERROR = 6,       /* AlignmentError     errors.py:28 */
    STARMM_NO_ADDITIVE_INVERSE = 7,   /* NoAdditiveInverse  errors.py:32 */
    STARMM_TOO_LARGE = 8,             /* TooLarge           errors.py:36 */
    STARMM_INTERNAL_ERROR = 9,        /* InternalError      errors.py:40 */
    STARMM_CUDA_ERROR = 100           /* 100 + cudaError_t passthrough   */
};

/* ---- semiring ids (semiring.py:130-145 + this build's 32-bit ids) ------- */
enum starmm_semiring {
    STARMM_SR_INT64 = 0,          /* "int": int64 (+,x), wraps mod 2^64          */
    STARMM_SR_FP64 = 1,           /* "float": float64 (+,x)                       */
    STARMM_SR_TROPICAL_F64 = 2,   /* "tropical": float64 (min,+), zero = +inf     */
    STARMM_SR_TROPICAL_F32 = 3,   /* "tropical_f32": float32 (min,+)              */
    STARMM_SR_TROPICAL_I32 = 4    /* "tropical_i32": int32 (min,+), INT32_MAX=+inf */
};

/* ---- schedules (registry.py:11-13 CLASSICAL + STRASSEN_FAMILY) ---------- */
enum starmm_algo {
    STARMM_CO2 = 0, STARMM_CO3 = 1, STARMM_TAR = 2, STARMM_SAR = 3, STARMM_STAR = 4,
    /* the fast family (strassen.py): rings only, OVERWRITES C with A (x) B */
    STARMM_STRASSEN = 5, STARMM_SAR_STRASSEN = 6, STARMM_STAR_STRASSEN_1 = 7,
    STARMM_STAR_STRASSEN_2 = 8
};

/* ---- allocation modes (registry.py:20,32-33) ---------------------------- */
enum starmm_alloc { STARMM_POOLED = 0, STARMM_RAW = 1 };

/* ---- flags ------------------------------------------------------------- */
#define STARMM_F_ASYNC          0x1  /* do not synchronise the stream at return        */
#define STARMM_F_NO_FASTPATH    0x2  /* disable range-guarded exact narrow paths       */
#define STARMM_F_INIT_IDENTITY  0x4  /* ignore incoming C: C <- A (x) B (k-split partials) */
#define STARMM_F_ALLOW_NONPOW2  0x8  /* accept any n >= 1 (divergence from matrix.py:57-61) */
#define STARMM_F_TIME_MAIN      0x10 /* CUDA-event time the tile kernel (stats.main_kernel_ns) */
#define STARMM_F_INT_TENSOR     0x20 /* opt-in: exact small-range int64 on tcgen05 kind::i8 */
#define STARMM_F_FP64_EMU       0x40 /* opt-in: fp64 (+,x) as Ozaki-II CRT over 16 int8 tcgen05 GEMMs
                                        (DESIGN.md §5d); non-finite inputs and k >= 2^17 stay on DMMA */

typedef struct starmm_plan starmm_plan;

typedef struct {
    /* pool (pool.py:158-167) */
    int64_t pool_total_allocated_bytes;
    int64_t pool_high_water_bytes;
    int64_t pool_fresh_count;
    int64_t pool_reuse_count;
    /* metrics (metrics.py:19-36) */
    int64_t tile_serializations;     /* write-backs through a tile slot / atomic-madd */
    int64_t pair_count;              /* SAR pair states created                       */
    int64_t pair_transitions;        /* Empty->FirstRunning + FirstRunning->FirstDone */
    int64_t lazy_temp_acquires;      /* SAR halves that found their sibling running   */
    int64_t raw_alloc_count;
    int64_t raw_alloc_bytes;
    /* plan / launch description */
    int64_t tasks;                   /* leaf tasks (output tile x k-slice) last run   */
    int64_t workers;                 /* persistent CTAs (GPU workers)                 */
    int64_t ksplit;                  /* k-slices per output tile                      */
    int64_t tar_levels;              /* split levels run with the TAR protocol        */
    int64_t kernel_launches;         /* launches issued by the last execute           */
    int64_t path;                    /* kernel path id of the last execute */
    int64_t executes;
    int64_t main_kernel_ns;          /* sum of tile-kernel event times (STARMM_F_TIME_MAIN) */
    int64_t main_kernel_launches;    /* launches that contributed to main_kernel_ns      */
    int64_t balanced_workers;        /* >0: tar/star ran balanced (uneven) k-slices over this
                                        many workers, shared tiles merged by atomic-madd  */
    int64_t live_leaves_max;         /* leaf gauge: most leaf tasks observed in flight at once
                                        (task_enter/base_enter, metrics.py:63-95)         */
    int64_t guard_syncs;             /* host waits on the range guard (0 once a plan has a
                                        verdict: the device decides)        */
    int64_t candidates;              /* paths queued behind the device-side verdict (1: none) */
    int64_t cluster_size;            /* > 0: the k-slices of a tile ran on one thread-block
                                        cluster and merged through DSMEM (DMMA path)      */
    int64_t k_chunks;                /* k-outer launches of the tile kernel (L2-sized panels) */
} starmm_stats;

/* The device's block pool (pool.py:67-167): one per device, shared by every plan and
 * one-shot call, surviving across calls until starmm_pool_reset.  Exact-size stacks,
 * LIFO reuse, blocks never cleared; reuse across streams is ordered on the device. */
typedef struct {
    int64_t allocated_bytes;     /* owned by the pool (issued + cached)              */
    int64_t cached_bytes;        /* on the free stacks                               */
    int64_t issued_bytes;        /* handed out now                                   */
    int64_t high_water_bytes;    /* max issued since the last reset                  */
    int64_t fresh_count;         /* acquisitions served by cudaMalloc                */
    int64_t reuse_count;         /* acquisitions served from a free stack            */
    int64_t cross_stream_waits;  /* reuses ordered by cudaStreamWaitEvent            */
    int64_t trims;               /* cached blocks returned to the driver             */
} starmm_pool_counts;

int  starmm_abi_version(void);
const char* starmm_strerror(int status);

/* n_rows x n_cols of C = m x n, inner dimension k.  The reference API is square
 * (m = n = k, power of two >= base_dim, matrix.py:57-61); the plan accepts
 * rectangles so the multi-GPU layer can run 2D output blocks and k-slices. */
int  starmm_plan_create(starmm_plan** plan, int semiring, int algo, int alloc_mode,
                        int64_t m, int64_t n, int64_t k, int base_dim, int workers,
                        int ksplit_log2 /* -1 = auto */, int device, int flags);
int  starmm_execute(starmm_plan* plan, void* C, int64_t ldc, const void* A, int64_t lda,
                    const void* B, int64_t ldb, void* stream);
/* Same computation with C, A and B in HOST memory (pinned for full overlap):
 * compute-bound problems first run k-outer chunks over all rows as A's column
 * chunks and B's row chunks arrive, then the rest of k in row blocks of
 * `block_rows` rows (0 = auto) whose results (C0 folded in) stream back while the
 * next block computes; PCIe-bound ones upload B, then stream A/C row blocks.
 * Blocking.  DESIGN.md §7b.  Classical schedules only (else
 * STARMM_CONTRACT_VIOLATION).  After starmm_plan_set_peers (a k-split rank of the
 * fused combine) only A and B stream in, in k-chunks, and C is not touched: the tile
 * kernels fold into the owners' rows, which the owners pre-load and read back.
 * The reference's entry points take host (numpy) matrices (classic.py:294-316);
 * this is their host-buffer form. */
int  starmm_execute_host(starmm_plan* plan, void* C, int64_t ldc, const void* A, int64_t lda,
                         const void* B, int64_t ldb, void* stream, int64_t block_rows);
/* Fused k-split combine across GPUs: when set, every output tile
 * is folded with the semiring's atomic-madd (red.min.s32 / red.add.f64 / red.add.u64,
 * CAS for float minima) directly into the OWNER's rows over NVLink peer memory:
 * rows [p*rows_per_part, (p+1)*rows_per_part) of this plan's output live at
 * bases[p] (leading dimension ld).  The owners pre-load C0 in their rows; the
 * reduce-scatter of the reference design disappears into the tile epilogue.
 * This is TAR's accumulate_region (ops.py:76-101) across GPUs.  nparts <= 8;
 * nparts = 0 restores local write-back.  Not valid for co3. */
int  starmm_plan_set_peers(starmm_plan* plan, int nparts, void* const* bases, int64_t ld,
                           int64_t rows_per_part);
/* CUDA IPC for the peer mapping (handles are 64 opaque bytes, exchanged by the host). */
int  starmm_ipc_handle(const void* dptr, void* handle_out);
int  starmm_ipc_open(const void* handle, void** dptr_out);
int  starmm_ipc_close(void* dptr);
/* Strassen family: recursion stops (classical tile kernel) once the half size would
 * drop below max(base_dim, leaf); default leaf 1024 keeps GPU leaves large.
 * Replaces strassen._strassen_root's "C.rows == ex.cfg.base_dim" test (strassen.py:184-207). */
int  starmm_plan_set_strassen_leaf(starmm_plan* plan, int64_t leaf);
int  starmm_plan_stats(starmm_plan* plan, starmm_stats* out);
int  starmm_plan_reset_stats(starmm_plan* plan);
void starmm_plan_destroy(starmm_plan* plan);

/* one-shot kernels */
int  starmm_matmul(int semiring, void* out, int64_t ldo, const void* A, int64_t lda,
                   const void* B, int64_t ldb, int64_t m, int64_t n, int64_t k,
                   void* stream, int flags);
int  starmm_madd(int semiring, void* C, int64_t ldc, const void* D, int64_t ldd,
                 int64_t rows, int64_t cols, void* stream, int flags);
int  starmm_atomic_accumulate(int semiring, void* C, int64_t ldc, const void* P, int64_t ldp,
                              int64_t rows, int64_t cols, void* stream, int flags);

/* device facts used by the Python layer for planning / reporting */
int  starmm_device_sm_count(int device);

/* the device block pool: Pool.acquire / release / reset / snapshot_counts
 * (pool.py:89-167).  acquire hands out an exact-size block (not cleared) usable on
 * `stream` (*fresh = 1 when it was newly allocated, like pool.py:99-111); release
 * returns it, fenced by the work queued on `stream` so far.
 * discipline: 0 LIFO (the reference), 1 FIFO (the negative control, pool.py:70-74). */
int  starmm_pool_acquire(int device, int64_t bytes, void* stream, void** out, int* fresh);
int  starmm_pool_release(int device, void* block, void* stream);
int  starmm_pool_counts_get(int device, starmm_pool_counts* out);
int  starmm_pool_reset(int device);
int  starmm_pool_set_discipline(int device, int fifo);
/* bytes the pool may own before it reuses a block that is still in use on another
 * stream (ordered by an event wait) or returns cached blocks to the driver; default
 * 3/4 of the device memory (env STARMM_POOL_LIMIT_MB); returns the previous limit in *old */
int  starmm_pool_set_limit(int device, int64_t bytes, int64_t* old);

/* ---- input generation -----------------------------------
 * Counter-based: element (i, j) of a matrix is a pure function of (seed, stream_id,
 * GLOBAL row i, GLOBAL column j) -- Philox4x32-10 on (j, i, stream_id, 0), key = seed --
 * so a rank generates exactly its own panel [row0, row0+rows) x [col0, col0+cols) with
 * no collective, and any panel can be regenerated on the host (the oracle restates it
 * bit for bit).  Stream-ordered on `stream`, does not block.  The reference's fixture
 * generator (matrix.py:196-214, numpy) is what the parity tests keep using; this is
 * the generator for inputs too large to ship (the BASELINE configs at full size).
 *   UNIFORM_REAL  a + (b - a) * u, u in [0, 1) (53 bits)       float semirings
 *   NORMAL        a + b * z, z ~ N(0, 1) (Box-Muller, + - * / and sqrt only)
 *   UNIFORM_INT   integer in [a, b]                            any semiring
 *   GRAPH         edge with probability p: weight UNIFORM_INT[a, b], else the
 *                 additive identity (+inf / INT32_MAX)
 * STARMM_GEN_ZERO_DIAG sets element (i, i) to 0. */
enum starmm_dist { STARMM_DIST_UNIFORM_REAL = 0, STARMM_DIST_NORMAL = 1, STARMM_DIST_UNIFORM_INT = 2,
                   STARMM_DIST_GRAPH = 3 };
#define STARMM_GEN_ZERO_DIAG 0x1
int  starmm_generate(int semiring, int dist, void* out, int64_t ld, int64_t rows, int64_t cols,
                     int64_t row0, int64_t col0, uint64_t seed, uint32_t stream_id, double a,
                     double b, double p, int gen_flags, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* STARMM_B200_H_ */
