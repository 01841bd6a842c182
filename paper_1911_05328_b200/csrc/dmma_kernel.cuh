// dmma_kernel.cuh -- fp64 (+,x) tile product on the FP64 tensor core (DMMA).
//
// Replaces the reference's _mm_float (semiring.py:35-45) + np.add fold
// (semiring.py:116-117) for the "float" semiring.  tcgen05.mma has no f64
// kind on sm_100a (SURVEY.md finding 6); the FP64 tensor core is reached via
// mma.sync.m8n8k4.f64, which ptxas lowers to DMMA.8x8x4 (measured: 37.1 TF/s
// chip peak, profiles/r01_peaks_microbench.json).
//
// CTA tile BM x BN, k-stage BK, WM x WN warps (warp tile (BM/WM) x (BN/WN),
// 8x8 DMMA blocks, accumulators in registers).  Operands are staged
// global->smem with 16-byte cp.async in a STAGES-deep ring; rows are padded so
// the 64-bit fragment loads are bank-conflict free.  Persistent CTAs (one per
// SM) walk the leaf-task list; the epilogue applies the schedule's write-back
// protocol (writeback.cuh).
#pragma once
#include "common.cuh"
#include "writeback.cuh"

namespace starmm {

STARMM_DEV void cp_async16(void* smem, const void* gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
STARMM_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
STARMM_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

STARMM_DEV void dmma_884(double& c0, double& c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

template <int BM_, int BN_, int WM_, int WN_, int BK_, int STAGES_, int MINB_ = 1, bool DB_ = false>
struct DmmaCfg {
    static constexpr int BM = BM_, BN = BN_, BK = BK_, STAGES = STAGES_;
    static constexpr int MIN_BLOCKS = MINB_;                 // co-resident CTAs per SM
    static constexpr bool DB = DB_;                          // register double-buffered fragments
    static constexpr int WM = WM_, WN = WN_;
    static constexpr int THREADS = WM * WN * 32;
    static constexpr int WTM = BM / WM, WTN = BN / WN;      // warp tile
    static constexpr int MI = WTM / 8, NJ = WTN / 8;         // 8x8 blocks per warp
    static constexpr int A_LD = BK + 4;                      // padded row pitch (doubles)
    static constexpr int B_LD = BN + 4;
    static constexpr int A_STAGE = BM * A_LD;
    static constexpr int B_STAGE = BK * B_LD;
    static constexpr int SMEM_BYTES = STAGES * (A_STAGE + B_STAGE) * 8 + 16 * STAGES + 64;
    static_assert(BK % 4 == 0 && (BK * BM / 2) % THREADS == 0 && (BK * BN / 2) % THREADS == 0,
                  "cp.async chunking");
};

// The production configuration (selected by tools/sweep_dmma.cu on B200): one 256x64
// CTA per SM of 8 warps stacked along M (8 x 1) with 32x64 warp tiles, 4-stage
// mbarrier ring -- 36.3 TF/s vs 36.1 for 128x128 (4 x 2) and 35.4 for two 64x128 CTAs
// of 4 warps (profiles/r01l_sweep_dmma_128.jsonl, r01n_sweep_dmma_aspect.jsonl): the
// warps of one CTA drift across the ring's stages (no CTA-wide barrier), and the large
// tile halves the fragment loads per DMMA and the L2 traffic per flop.
using DmmaProd = DmmaCfg<256, 64, 8, 1, 16, 4, 1>;

struct DmmaParams {
    const double* A; long long lda;   // tile-aligned (padded if needed), 16-byte rows
    const double* B; long long ldb;
    TaskGrid g;
    WbParams w;
    unsigned* gate = nullptr;         // wave gate counter (zeroed per launch), GATE builds only
    Pred pr;                          // device-side path predicate (common.cuh)
};

template <class K>
__global__ void __launch_bounds__(K::THREADS, K::MIN_BLOCKS) dmma_fp64_kernel(DmmaParams p) {
    constexpr int BM = K::BM, BN = K::BN, BK = K::BK, STAGES = K::STAGES;
    constexpr int A_LD = K::A_LD, B_LD = K::B_LD, A_STAGE = K::A_STAGE, B_STAGE = K::B_STAGE;
    constexpr int THREADS = K::THREADS, MI = K::MI, NJ = K::NJ;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* As = reinterpret_cast<double*>(smem_raw);
    double* Bs = As + STAGES * A_STAGE;
    int* smem_word = reinterpret_cast<int*>(Bs + STAGES * B_STAGE);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp / K::WN, wn = warp % K::WN;
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
            constexpr int A_CH = BK / 2;                     // 16-byte chunks per A row
#pragma unroll
            for (int i = 0; i < BM * A_CH / THREADS; ++i) {
                int c = tid + i * THREADS;
                int r = c / A_CH, q = c % A_CH;
                cp_async16(as + r * A_LD + q * 2, a + (long long)r * p.lda + q * 2);
            }
            const double* b = Bg + (long long)kt * BK * p.ldb;
            double* bs = Bs + stage * B_STAGE;
            constexpr int B_CH = BN / 2;
#pragma unroll
            for (int i = 0; i < BK * B_CH / THREADS; ++i) {
                int c = tid + i * THREADS;
                int r = c / B_CH, q = c % B_CH;
                cp_async16(bs + r * B_LD + q * 2, b + (long long)r * p.ldb + q * 2);
            }
        };

        double acc[MI][NJ][2];
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

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
            const double* as = As + (kt % STAGES) * A_STAGE + (wm * K::WTM + gi) * A_LD + ti;
            const double* bs = Bs + (kt % STAGES) * B_STAGE + ti * B_LD + wn * K::WTN + gi;
            if constexpr (K::DB) {
                double a[2][MI], b[2][NJ];
#pragma unroll
                for (int i = 0; i < MI; ++i) a[0][i] = as[i * 8 * A_LD];
#pragma unroll
                for (int j = 0; j < NJ; ++j) b[0][j] = bs[j * 8];
#pragma unroll
                for (int kk = 0; kk < BK; kk += 4) {
                    const int cur = (kk / 4) & 1;
                    if (kk + 4 < BK) {
#pragma unroll
                        for (int i = 0; i < MI; ++i) a[cur ^ 1][i] = as[i * 8 * A_LD + kk + 4];
#pragma unroll
                        for (int j = 0; j < NJ; ++j) b[cur ^ 1][j] = bs[(kk + 4) * B_LD + j * 8];
                    }
#pragma unroll
                    for (int i = 0; i < MI; ++i)
#pragma unroll
                        for (int j = 0; j < NJ; ++j)
                            dmma_884(acc[i][j][0], acc[i][j][1], a[cur][i], b[cur][j]);
                }
            } else {
#pragma unroll
                for (int kk = 0; kk < BK; kk += 4) {
                    double a[MI], b[NJ];
#pragma unroll
                    for (int i = 0; i < MI; ++i) a[i] = as[i * 8 * A_LD + kk];
#pragma unroll
                    for (int j = 0; j < NJ; ++j) b[j] = bs[kk * B_LD + j * 8];
#pragma unroll
                    for (int i = 0; i < MI; ++i)
#pragma unroll
                        for (int j = 0; j < NJ; ++j) dmma_884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
                }
            }
        }
        cp_async_wait<0>();
        __syncthreads();

        writeback<SrFp64, BM, BN, K::THREADS, 0>(p.w, g, tm, tn, s, tile, blockIdx.x, mode, pair_seen,
                                  [&](auto f) {
#pragma unroll
            for (int i = 0; i < MI; ++i)
#pragma unroll
                for (int j = 0; j < NJ; ++j) {
                    int r = wm * K::WTM + i * 8 + gi;
                    int c = wn * K::WTN + j * 8 + ti * 2;
                    f(r, c, acc[i][j][0]);
                    f(r, c + 1, acc[i][j][1]);
                }
        });
    }
}

// ---- mbarrier-pipelined variant ------------------------------------------------
// Same tiles and fragments; the CTA-wide __syncthreads of every k-stage is replaced by
// two mbarriers per ring slot: full[s] completes when every thread's cp.async into the
// slot has landed (cp.async.mbarrier.arrive.noinc), empty[s] when every thread has read
// it.  Warps drift up to a stage apart instead of meeting at each stage boundary.
STARMM_DEV void mbar_init(unsigned long long* bar, unsigned count) {
    unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count));
}
STARMM_DEV void mbar_arrive(unsigned long long* bar) {
    unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}\n" ::"r"(a)
                 : "memory");
}
STARMM_DEV void mbar_cp_async_arrive(unsigned long long* bar) {
    unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(a) : "memory");
}
STARMM_DEV void mbar_wait(unsigned long long* bar, unsigned parity) {
    unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}\n" ::"r"(a), "r"(parity) : "memory");
}

// EPI = 1: the exclusive FOLD write-back reads its 2-double fragment pairs as 16-byte
// vectors, a whole fragment row (NJ pairs) in flight before any store (EPI = 0: the
// generic element-by-element writeback).  Other protocols always use the generic one.
// GATE = 1: wave gate -- a CTA starts its i-th tile only after every CTA has finished
// its (i-1)-th (one global counter; bounded wait, so a grid that is not fully
// co-resident cannot hang), keeping the persistent CTAs of a wave in step in k so the
// wave's A/B panel slices are shared in L2 instead of re-read from DRAM.
template <class K, int EPI = 0, int GATE = 0>
__global__ void __launch_bounds__(K::THREADS, K::MIN_BLOCKS) dmma_fp64_kernel_mb(DmmaParams p) {
    if (p.pr.off()) return;
    constexpr int BM = K::BM, BN = K::BN, BK = K::BK, STAGES = K::STAGES;
    constexpr int A_LD = K::A_LD, B_LD = K::B_LD, A_STAGE = K::A_STAGE, B_STAGE = K::B_STAGE;
    constexpr int THREADS = K::THREADS, MI = K::MI, NJ = K::NJ;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* As = reinterpret_cast<double*>(smem_raw);
    double* Bs = As + STAGES * A_STAGE;
    unsigned long long* full = reinterpret_cast<unsigned long long*>(Bs + STAGES * B_STAGE);
    unsigned long long* empty = full + STAGES;
    int* smem_word = reinterpret_cast<int*>(empty + STAGES);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp / K::WN, wn = warp % K::WN;
    const int gi = lane >> 2, ti = lane & 3;
    const TaskGrid& g = p.g;
    const int nk = (int)(g.kslice / BK);
    if (tid == 0) {
        for (int st = 0; st < STAGES; ++st) {
            mbar_init(&full[st], THREADS);
            mbar_init(&empty[st], THREADS);
        }
    }
    __syncthreads();
    long long gk = 0;   // global stage counter: slot = gk % STAGES, use = gk / STAGES

    int iter = 0;
    bool gate_on = true;      // (thread 0) a wait that hit the cap turns this CTA's gate off
    for (int t = blockIdx.x; t < g.num_tasks; t += gridDim.x, ++iter) {
        if constexpr (GATE >= 1) {
            if (iter > 0) {
                if (tid == 0 && gate_on) {
                    // slack: GATE 1 = none, 2 = a quarter wave, 3 = half a wave
                    const unsigned slack = GATE == 1 ? 0u : (GATE == 2 ? gridDim.x / 4 : gridDim.x / 2);
                    const unsigned need = (unsigned)iter * gridDim.x - slack;
                    const long long t0 = clock64();
                    unsigned v;
                    for (;;) {
                        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p.gate) : "memory");
                        if (v >= need) break;
                        if (clock64() - t0 > 4000000LL) { gate_on = false; break; }   // ~2 ms cap
                        __nanosleep(128);
                    }
                }
                __syncthreads();
            }
        }
        int tm, tn, s, tile;
        decode_task(g, t, tm, tn, s, tile);
        leaf_enter(p.w);
        const int mode = task_mode(p.w, g, s);
        int pair_seen = PAIR_EMPTY;
        if (mode == WB_PAIR) pair_seen = pair_arrive(p.w, g, tile, s, smem_word);

        const double* Ag = p.A + (long long)tm * BM * p.lda + (long long)s * g.kslice;
        const double* Bg = p.B + (long long)s * g.kslice * p.ldb + (long long)tn * BN;

        auto fill = [&](int kt) {   // k-stage kt of this task into slot (gk + kt) % STAGES
            const long long gidx = gk + kt;
            const int slot = (int)(gidx % STAGES);
            if (gidx >= STAGES) mbar_wait(&empty[slot], (unsigned)(((gidx / STAGES) - 1) & 1));
            const double* a = Ag + (long long)kt * BK;
            double* as = As + slot * A_STAGE;
            constexpr int A_CH = BK / 2;
#pragma unroll
            for (int i = 0; i < BM * A_CH / THREADS; ++i) {
                int c = tid + i * THREADS;
                int r = c / A_CH, q = c % A_CH;
                cp_async16(as + r * A_LD + q * 2, a + (long long)r * p.lda + q * 2);
            }
            const double* b = Bg + (long long)kt * BK * p.ldb;
            double* bs = Bs + slot * B_STAGE;
            constexpr int B_CH = BN / 2;
#pragma unroll
            for (int i = 0; i < BK * B_CH / THREADS; ++i) {
                int c = tid + i * THREADS;
                int r = c / B_CH, q = c % B_CH;
                cp_async16(bs + r * B_LD + q * 2, b + (long long)r * p.ldb + q * 2);
            }
            mbar_cp_async_arrive(&full[slot]);
        };

        double acc[MI][NJ][2];
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

        for (int st = 0; st < STAGES - 1 && st < nk; ++st) fill(st);
        for (int kt = 0; kt < nk; ++kt) {
            const long long gidx = gk + kt;
            const int slot = (int)(gidx % STAGES);
            mbar_wait(&full[slot], (unsigned)((gidx / STAGES) & 1));
            const double* as = As + slot * A_STAGE + (wm * K::WTM + gi) * A_LD + ti;
            const double* bs = Bs + slot * B_STAGE + ti * B_LD + wn * K::WTN + gi;
#pragma unroll
            for (int kk = 0; kk < BK; kk += 4) {
                double a[MI], b[NJ];
#pragma unroll
                for (int i = 0; i < MI; ++i) a[i] = as[i * 8 * A_LD + kk];
#pragma unroll
                for (int j = 0; j < NJ; ++j) b[j] = bs[kk * B_LD + j * 8];
#pragma unroll
                for (int i = 0; i < MI; ++i)
#pragma unroll
                    for (int j = 0; j < NJ; ++j) dmma_884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
            }
            mbar_arrive(&empty[slot]);
            const int nxt = kt + STAGES - 1;
            if (nxt < nk) fill(nxt);
        }
        gk += nk;

        if constexpr (EPI == 1) {
            const long long m0 = (long long)tm * BM, n0 = (long long)tn * BN;
            if (mode == WB_FOLD && m0 + BM <= p.w.M && n0 + BN <= p.w.N && (p.w.ldc & 1) == 0 &&
                (reinterpret_cast<uintptr_t>(p.w.C) & 15) == 0) {
                double* C = reinterpret_cast<double*>(p.w.C);
#pragma unroll
                for (int i = 0; i < MI; ++i) {
                    const long long r = m0 + wm * K::WTM + i * 8 + gi;
                    double2* row = reinterpret_cast<double2*>(C + r * p.w.ldc + n0 + wn * K::WTN + ti * 2);
                    double2 old[NJ];
#pragma unroll
                    for (int j = 0; j < NJ; ++j) old[j] = row[j * 4];
#pragma unroll
                    for (int j = 0; j < NJ; ++j)
                        row[j * 4] = make_double2(old[j].x + acc[i][j][0], old[j].y + acc[i][j][1]);
                }
                if constexpr (GATE >= 1) {
                    __syncthreads();
                    if (tid == 0) { __threadfence(); atomicAdd(p.gate, 1u); }
                }
                leaf_exit(p.w);
                continue;
            }
        }
        writeback<SrFp64, BM, BN, K::THREADS, 0>(p.w, g, tm, tn, s, tile, blockIdx.x, mode, pair_seen,
                                  [&](auto f) {
#pragma unroll
            for (int i = 0; i < MI; ++i)
#pragma unroll
                for (int j = 0; j < NJ; ++j) {
                    int r = wm * K::WTM + i * 8 + gi;
                    int c = wn * K::WTN + j * 8 + ti * 2;
                    f(r, c, acc[i][j][0]);
                    f(r, c + 1, acc[i][j][1]);
                }
        });
        leaf_exit(p.w);
        if constexpr (GATE >= 1) {
            __syncthreads();
            if (tid == 0) { __threadfence(); atomicAdd(p.gate, 1u); }
        }
    }
}

// ---- split-k on a thread-block cluster (DSMEM reduction) -------------------------
// The S k-slices of one output tile run on the S CTAs of one cluster (CS = S, 2..8):
// CTA rank r computes slice r into its registers, stages the partial tile in its own
// shared memory (the ring's A region: every stage of the task has been consumed), and
// after a cluster barrier each rank reduces a 1/S share of the tile's rows over the S
// partials read through distributed shared memory -- in rank order, so the sum is
// deterministic -- and folds it into C exclusively.  This is the reference's sibling
// k-halves (_mm_children pairs, classic.py:86-93) running concurrently with the
// accumulate_region merge (ops.py:76-101) done on chip: no global tile lock, no
// atomics and no global scratch round trip (the SAR lazy temporary, classic.py:190-204,
// is the sibling's shared-memory partial).  Persistent: cluster c walks tiles
// c, c + clusters, ...
namespace dsm {
STARMM_DEV unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
STARMM_DEV unsigned cluster_id_x() {
    unsigned r;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
    return r;
}
STARMM_DEV unsigned num_clusters_x() {
    unsigned r;
    asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
    return r;
}
STARMM_DEV void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n"
                 "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// shared::cta address of this CTA -> shared::cluster address of the same offset in `rank`
STARMM_DEV unsigned map_rank(const void* p, unsigned rank) {
    unsigned a = (unsigned)__cvta_generic_to_shared(p), r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
STARMM_DEV double2 ld_cluster_v2(unsigned addr) {
    double2 v;
    asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
    return v;
}
}  // namespace dsm

constexpr int DSM_PITCH = 72;   // doubles per staged partial row: a warp's 16-byte fragment
                                // stores hit 4 distinct 128-byte wavefronts (64 + 8)

template <class K, int CS>
__global__ void __launch_bounds__(K::THREADS, 1) dmma_fp64_cluster_kernel(DmmaParams p) {
    if (p.pr.off()) return;
    constexpr int BM = K::BM, BN = K::BN, BK = K::BK, STAGES = K::STAGES;
    constexpr int A_LD = K::A_LD, B_LD = K::B_LD, A_STAGE = K::A_STAGE, B_STAGE = K::B_STAGE;
    constexpr int THREADS = K::THREADS, MI = K::MI, NJ = K::NJ;
    static_assert(BM * DSM_PITCH <= STAGES * A_STAGE, "partial tile must fit the A ring");
    static_assert(BN == 64 && (BM / CS) * (BN / 2) % THREADS == 0, "reduction mapping");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* As = reinterpret_cast<double*>(smem_raw);
    double* Bs = As + STAGES * A_STAGE;
    unsigned long long* full = reinterpret_cast<unsigned long long*>(Bs + STAGES * B_STAGE);
    unsigned long long* empty = full + STAGES;
    double* part = As;                                   // staged partial tile [BM][DSM_PITCH]

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp / K::WN, wn = warp % K::WN;
    const int gi = lane >> 2, ti = lane & 3;
    const TaskGrid& g = p.g;
    const int nk = (int)(g.kslice / BK);
    const unsigned rank = dsm::cluster_rank();
    const int tiles = g.tiles_m * g.tiles_n;
    if (tid == 0) {
        for (int st = 0; st < STAGES; ++st) {
            mbar_init(&full[st], THREADS);
            mbar_init(&empty[st], THREADS);
        }
    }
    __syncthreads();
    long long gk = 0;
    const long long tile_bytes = (long long)BM * BN * 8;
    for (int tt = (int)dsm::cluster_id_x(); tt < tiles; tt += (int)dsm::num_clusters_x()) {
        int tm, tn, s_unused, tile;
        // decode the tile (k-slice 0 of the S-split task list): tile-major raster
        decode_task(g, tt << g.log2S, tm, tn, s_unused, tile);
        const int s = (int)rank;                          // this CTA's k-slice
        leaf_enter(p.w);
        const double* Ag = p.A + (long long)tm * BM * p.lda + (long long)s * g.kslice;
        const double* Bg = p.B + (long long)s * g.kslice * p.ldb + (long long)tn * BN;

        auto fill = [&](int kt) {
            const long long gidx = gk + kt;
            const int slot = (int)(gidx % STAGES);
            if (gidx >= STAGES) mbar_wait(&empty[slot], (unsigned)(((gidx / STAGES) - 1) & 1));
            const double* a = Ag + (long long)kt * BK;
            double* as = As + slot * A_STAGE;
            constexpr int A_CH = BK / 2;
#pragma unroll
            for (int i = 0; i < BM * A_CH / THREADS; ++i) {
                int c = tid + i * THREADS;
                int r = c / A_CH, q = c % A_CH;
                cp_async16(as + r * A_LD + q * 2, a + (long long)r * p.lda + q * 2);
            }
            const double* b = Bg + (long long)kt * BK * p.ldb;
            double* bs = Bs + slot * B_STAGE;
            constexpr int B_CH = BN / 2;
#pragma unroll
            for (int i = 0; i < BK * B_CH / THREADS; ++i) {
                int c = tid + i * THREADS;
                int r = c / B_CH, q = c % B_CH;
                cp_async16(bs + r * B_LD + q * 2, b + (long long)r * p.ldb + q * 2);
            }
            mbar_cp_async_arrive(&full[slot]);
        };

        double acc[MI][NJ][2];
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

        for (int st = 0; st < STAGES - 1 && st < nk; ++st) fill(st);
        for (int kt = 0; kt < nk; ++kt) {
            const long long gidx = gk + kt;
            const int slot = (int)(gidx % STAGES);
            mbar_wait(&full[slot], (unsigned)((gidx / STAGES) & 1));
            const double* as = As + slot * A_STAGE + (wm * K::WTM + gi) * A_LD + ti;
            const double* bs = Bs + slot * B_STAGE + ti * B_LD + wn * K::WTN + gi;
#pragma unroll
            for (int kk = 0; kk < BK; kk += 4) {
                double a[MI], b[NJ];
#pragma unroll
                for (int i = 0; i < MI; ++i) a[i] = as[i * 8 * A_LD + kk];
#pragma unroll
                for (int j = 0; j < NJ; ++j) b[j] = bs[kk * B_LD + j * 8];
#pragma unroll
                for (int i = 0; i < MI; ++i)
#pragma unroll
                    for (int j = 0; j < NJ; ++j) dmma_884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
            }
            mbar_arrive(&empty[slot]);
            const int nxt = kt + STAGES - 1;
            if (nxt < nk) fill(nxt);
        }
        gk += nk;

        // ---- stage the partial tile (every warp has consumed every slot of this task) ----
        __syncthreads();
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                const int r = wm * K::WTM + i * 8 + gi;
                const int c = wn * K::WTN + j * 8 + ti * 2;
                *reinterpret_cast<double2*>(&part[r * DSM_PITCH + c]) = make_double2(acc[i][j][0], acc[i][j][1]);
            }
        if (tid == 0 && rank != 0) {                      // the sibling's lazy temporary
            pool_acquire(p.w, blockIdx.x, tile_bytes);
            counter_add(p.w, CNT_LAZY_ACQUIRES, 1);
        }
        dsm::cluster_sync();                              // all S partials visible

        // ---- reduce rows [rank*BM/CS, (rank+1)*BM/CS) over the S partials, fold into C ----
        constexpr int ROWS = BM / CS, PER_ROW = BN / 2;   // double2 per row
        const long long m0 = (long long)tm * BM, n0 = (long long)tn * BN;
        double* C = reinterpret_cast<double*>(p.w.C);
        const long long ldc = p.w.ldc;
        const bool vec = ((ldc & 1) == 0) && ((reinterpret_cast<uintptr_t>(C) & 15) == 0);
#pragma unroll 4
        for (int e = tid; e < ROWS * PER_ROW; e += THREADS) {
            const int r = (int)rank * ROWS + e / PER_ROW, c2 = (e % PER_ROW) * 2;
            double2 sum = make_double2(0.0, 0.0);
#pragma unroll
            for (int q = 0; q < CS; ++q) {                // rank order: deterministic
                const double2 v = dsm::ld_cluster_v2(dsm::map_rank(&part[r * DSM_PITCH + c2], (unsigned)q));
                sum.x = q == 0 ? v.x : sum.x + v.x;
                sum.y = q == 0 ? v.y : sum.y + v.y;
            }
            const long long gr = m0 + r, gc = n0 + c2;
            if (gr >= p.w.M) continue;
            double* dst = C + gr * ldc + gc;
            if (vec && gc + 1 < p.w.N) {
                if (!p.w.init_identity) {
                    const double2 o = *reinterpret_cast<const double2*>(dst);
                    sum.x = o.x + sum.x;
                    sum.y = o.y + sum.y;
                }
                *reinterpret_cast<double2*>(dst) = sum;
            } else {
                if (gc < p.w.N) dst[0] = p.w.init_identity ? sum.x : dst[0] + sum.x;
                if (gc + 1 < p.w.N) dst[1] = p.w.init_identity ? sum.y : dst[1] + sum.y;
            }
        }
        if (tid == 0) {
            if (rank == 0) counter_add(p.w, CNT_SERIALIZATIONS, 1);   // one exclusive merge per tile
            else pool_release(p.w, tile_bytes);
        }
        leaf_exit(p.w);
        dsm::cluster_sync();                              // partials no longer read: ring reusable
    }
}


// ---- balanced slices ("stream-K") on the DMMA path ------------------------------------
// TAR with uneven k-slices (the SIMT kernels' balanced mode, simt_kernel.cuh): every
// persistent CTA gets the same share of the flattened (tile, k-stage) space; a tile a
// CTA covers whole is folded exclusively, the <= 2 pieces of a tile shared with a
// neighbouring CTA merge with the atomic-madd (red.add.f64, accumulate_region,
// ops.py:76-101).  Small problems (n = 2048: 256 tiles on 148 SMs = 1.73 waves) lose a
// quarter of the machine to the last wave otherwise.  Separate kernel: the production
// kernel's register allocation stays untouched.
template <class K>
__global__ void __launch_bounds__(K::THREADS, K::MIN_BLOCKS) dmma_fp64_balanced_kernel(DmmaParams p) {
    if (p.pr.off()) return;
    constexpr int BM = K::BM, BN = K::BN, BK = K::BK, STAGES = K::STAGES;
    constexpr int A_LD = K::A_LD, B_LD = K::B_LD, A_STAGE = K::A_STAGE, B_STAGE = K::B_STAGE;
    constexpr int THREADS = K::THREADS, MI = K::MI, NJ = K::NJ;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* As = reinterpret_cast<double*>(smem_raw);
    double* Bs = As + STAGES * A_STAGE;
    unsigned long long* full = reinterpret_cast<unsigned long long*>(Bs + STAGES * B_STAGE);
    unsigned long long* empty = full + STAGES;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp / K::WN, wn = warp % K::WN;
    const int gi = lane >> 2, ti = lane & 3;
    const TaskGrid& g = p.g;
    if (tid == 0) {
        for (int st = 0; st < STAGES; ++st) {
            mbar_init(&full[st], THREADS);
            mbar_init(&empty[st], THREADS);
        }
    }
    __syncthreads();
    long long gk = 0;
    TaskGrid g1 = g;
    g1.S = 1; g1.log2S = 0;
    const long long T = (long long)g.tiles_m * g.tiles_n * g.kstages;
    long long it = T * blockIdx.x / gridDim.x;
    const long long end = T * (blockIdx.x + 1) / gridDim.x;
    while (it < end) {
        const long long tl = it / g.kstages;
        const long long ks = it - tl * g.kstages;
        const long long ke = min(g.kstages, ks + (end - it));
        const int nk = (int)(ke - ks);
        int tm, tn, s0, tile;
        decode_task(g1, (int)tl, tm, tn, s0, tile);
        int mode = WB_RED;
        if (ks == 0 && ke == g.kstages && p.w.remote_parts == 0)
            mode = p.w.init_identity ? WB_STORE : WB_FOLD;
        leaf_enter(p.w);
        const double* Ag = p.A + (long long)tm * BM * p.lda + ks * BK;
        const double* Bg = p.B + ks * BK * p.ldb + (long long)tn * BN;

        auto fill = [&](int kt) {
            const long long gidx = gk + kt;
            const int slot = (int)(gidx % STAGES);
            if (gidx >= STAGES) mbar_wait(&empty[slot], (unsigned)(((gidx / STAGES) - 1) & 1));
            const double* a = Ag + (long long)kt * BK;
            double* as = As + slot * A_STAGE;
            constexpr int A_CH = BK / 2;
#pragma unroll
            for (int i = 0; i < BM * A_CH / THREADS; ++i) {
                int c = tid + i * THREADS;
                int r = c / A_CH, q = c % A_CH;
                cp_async16(as + r * A_LD + q * 2, a + (long long)r * p.lda + q * 2);
            }
            const double* b = Bg + (long long)kt * BK * p.ldb;
            double* bs = Bs + slot * B_STAGE;
            constexpr int B_CH = BN / 2;
#pragma unroll
            for (int i = 0; i < BK * B_CH / THREADS; ++i) {
                int c = tid + i * THREADS;
                int r = c / B_CH, q = c % B_CH;
                cp_async16(bs + r * B_LD + q * 2, b + (long long)r * p.ldb + q * 2);
            }
            mbar_cp_async_arrive(&full[slot]);
        };

        double acc[MI][NJ][2];
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

        for (int st = 0; st < STAGES - 1 && st < nk; ++st) fill(st);
        for (int kt = 0; kt < nk; ++kt) {
            const long long gidx = gk + kt;
            const int slot = (int)(gidx % STAGES);
            mbar_wait(&full[slot], (unsigned)((gidx / STAGES) & 1));
            const double* as = As + slot * A_STAGE + (wm * K::WTM + gi) * A_LD + ti;
            const double* bs = Bs + slot * B_STAGE + ti * B_LD + wn * K::WTN + gi;
#pragma unroll
            for (int kk = 0; kk < BK; kk += 4) {
                double a[MI], b[NJ];
#pragma unroll
                for (int i = 0; i < MI; ++i) a[i] = as[i * 8 * A_LD + kk];
#pragma unroll
                for (int j = 0; j < NJ; ++j) b[j] = bs[kk * B_LD + j * 8];
#pragma unroll
                for (int i = 0; i < MI; ++i)
#pragma unroll
                    for (int j = 0; j < NJ; ++j) dmma_884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
            }
            mbar_arrive(&empty[slot]);
            const int nxt = kt + STAGES - 1;
            if (nxt < nk) fill(nxt);
        }
        gk += nk;
        writeback<SrFp64, BM, BN, K::THREADS, 0>(p.w, g1, tm, tn, 0, tile, blockIdx.x, mode, PAIR_EMPTY,
                                  [&](auto f) {
#pragma unroll
            for (int i = 0; i < MI; ++i)
#pragma unroll
                for (int j = 0; j < NJ; ++j) {
                    int r = wm * K::WTM + i * 8 + gi;
                    int c = wn * K::WTN + j * 8 + ti * 2;
                    f(r, c, acc[i][j][0]);
                    f(r, c + 1, acc[i][j][1]);
                }
        });
        leaf_exit(p.w);
        it += nk;
    }
}

}  // namespace starmm
