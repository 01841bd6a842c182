// dmma_kernel.cuh -- fp64 (+,x) tile product on the FP64 tensor core (DMMA).
//
// Replaces the reference's _mm_float (semiring.py:35-45) + np.add fold
// (semiring.py:116-117) for the "float" semiring.  tcgen05.mma has no f64
// kind on sm_100a (SURVEY.md finding 6); the FP64 tensor core is reached via
// mma.sync.m8n8k4.f64, which ptxas lowers to DMMA.8x8x4 (measured: 37.1 TF/s
// chip peak, profiles/r01_peaks_microbench.json).
//
// CTA tile 128x128, k-stage 16, 8 warps (2 x 4), warp tile 64x32 (8 x 4 DMMA
// blocks, 64 fp64 accumulators per lane).  Operands are staged global->smem
// with 16-byte cp.async in a 4-deep ring; rows are padded so the 64-bit
// fragment loads are bank-conflict free.  Persistent CTAs (one per SM) walk
// the leaf-task list; the epilogue applies the schedule's write-back protocol.
#pragma once
#include "common.cuh"
#include "writeback.cuh"

namespace starmm {

namespace dmma {
constexpr int BM = 128, BN = 128, BK = 16;
constexpr int STAGES = 4;
constexpr int THREADS = 256;
constexpr int A_LD = BK + 4;      // 20 doubles = 160 B row pitch
constexpr int B_LD = BN + 4;      // 132 doubles = 1056 B row pitch
constexpr int A_STAGE = BM * A_LD;
constexpr int B_STAGE = BK * B_LD;
constexpr int SMEM_BYTES = STAGES * (A_STAGE + B_STAGE) * 8 + 64;
}  // namespace dmma

STARMM_DEV void cp_async16(void* smem, const void* gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
STARMM_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
STARMM_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

STARMM_DEV void dmma_884(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

struct DmmaParams {
    const double* A; long long lda;   // >= BM/BK padded, 16-byte aligned rows
    const double* B; long long ldb;
    TaskGrid g;
    WbParams w;
};

__global__ void __launch_bounds__(dmma::THREADS, 1) dmma_fp64_kernel(DmmaParams p) {
    using namespace dmma;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* As = reinterpret_cast<double*>(smem_raw);
    double* Bs = As + STAGES * A_STAGE;
    int* smem_word = reinterpret_cast<int*>(Bs + STAGES * B_STAGE);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp >> 2, wn = warp & 3;          // 2 x 4 warps
    const int gi = lane >> 2, ti = lane & 3;          // fragment coordinates
    const TaskGrid& g = p.g;
    const int nk = (int)(g.kslice / BK);

    for (int t = blockIdx.x; t < g.num_tasks; t += gridDim.x) {
        int tm, tn, s, tile;
        decode_task(g, t, tm, tn, s, tile);
        const int mode = task_mode(p.w, g, s);
        int pair_seen = PAIR_EMPTY;
        if (mode == WB_PAIR) pair_seen = pair_arrive(p.w, g, tile, s, smem_word);

        const double* Ag = p.A + (long long)tm * BM * p.lda + (long long)s * g.kslice;
        const double* Bg = p.B + (long long)s * g.kslice * p.ldb + (long long)tn * BN;

        auto load_stage = [&](int kt, int stage) {
            const double* a = Ag + (long long)kt * BK;
            double* as = As + stage * A_STAGE;
#pragma unroll
            for (int i = 0; i < 4; ++i) {           // 128 rows x 8 chunks
                int c = tid + i * THREADS;
                int r = c >> 3, q = c & 7;
                cp_async16(as + r * A_LD + q * 2, a + (long long)r * p.lda + q * 2);
            }
            const double* b = Bg + (long long)kt * BK * p.ldb;
            double* bs = Bs + stage * B_STAGE;
#pragma unroll
            for (int i = 0; i < 4; ++i) {           // 16 rows x 64 chunks
                int c = tid + i * THREADS;
                int r = c >> 6, q = c & 63;
                cp_async16(bs + r * B_LD + q * 2, b + (long long)r * p.ldb + q * 2);
            }
        };

        double acc[8][4][2];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
        for (int st = 0; st < STAGES - 1; ++st) {
            if (st < nk) load_stage(st, st);
            cp_async_commit();
        }
        for (int kt = 0; kt < nk; ++kt) {
            cp_async_wait<STAGES - 2>();
            __syncthreads();
            int nxt = kt + STAGES - 1;
            if (nxt < nk) load_stage(nxt, nxt % STAGES);
            cp_async_commit();
            const double* as = As + (kt % STAGES) * A_STAGE + (wm * 64 + gi) * A_LD + ti;
            const double* bs = Bs + (kt % STAGES) * B_STAGE + ti * B_LD + wn * 32 + gi;
#pragma unroll
            for (int kk = 0; kk < BK; kk += 4) {
                double a[8], b[4];
#pragma unroll
                for (int i = 0; i < 8; ++i) a[i] = as[i * 8 * A_LD + kk];
#pragma unroll
                for (int j = 0; j < 4; ++j) b[j] = bs[kk * B_LD + j * 8];
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) dmma_884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
            }
        }
        cp_async_wait<0>();
        __syncthreads();

        writeback<SrFp64, BM, BN>(p.w, g, tm, tn, s, tile, blockIdx.x, mode, pair_seen,
                                  [&](auto f) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    int r = wm * 64 + i * 8 + gi;
                    int c = wn * 32 + j * 8 + ti * 2;
                    f(r, c, acc[i][j][0]);
                    f(r, c + 1, acc[i][j][1]);
                }
        });
    }
}

}  // namespace starmm
