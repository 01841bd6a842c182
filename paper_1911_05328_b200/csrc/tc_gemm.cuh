// tc_gemm.cuh -- persistent CTA-pair int8 x int8 -> int32 GEMM core on tcgen05.
//
// The exact-integer tensor-core engine behind two OPT-IN paths:
//   * small-range int64 (+,x): one pass, epilogue widens and folds into int64 C;
//   * fp64 (+,x) emulation (Ozaki scheme II): P passes, one per CRT modulus, over
//     stacked residue operands; the epilogue keeps each pass's residue and the last
//     pass reconstructs the exact integer product and folds it into fp64 C.
//
// Shape of one work unit: a 256 x 256 output tile computed by a CTA pair
// (cluster of 2, tcgen05.mma.cta_group::2, UMMA M = 256, N = 256, K = 32).
// CTA rank r of the pair owns output rows [128 r, 128 r + 128) of the tile, loads
// those 128 rows of A and 128 of the 256 B^T rows (columns of C) per k-stage, and
// holds its 128 x 256 s32 accumulator half in its own TMEM.
//
// Roles per CTA (320 threads):
//   warp 0 lane 0 : TMA producer (both CTAs; bytes land on the leader's full barrier)
//   warp 1        : TMEM owner (alloc/dealloc, cta_group::2); lane 0 of the LEADER
//                   issues the MMAs and commits (multicast) to both CTAs' barriers
//   warps 2..9    : epilogue -- TMEM lanes 32 (w % 4) .. + 31 are output rows; the
//                   two warps of a lane quarter take 128 columns each
// Pipelines: STAGES-deep smem ring (full: TMA -> MMA, empty: MMA -> TMA) and a
// 2-deep TMEM accumulator ring (acc_full: MMA -> epilogue of both CTAs, acc_empty:
// 16 epilogue warps of the pair -> MMA), so the epilogue of one work unit overlaps
// the mainloop of the next.  Work units are (pass, tile) in PASS-MAJOR order: all
// of a CTA pair's tiles for pass p, then pass p + 1, so each pass streams its own
// operand planes like one ordinary GEMM (tile-major order let the pairs drift
// across passes and thrashed L2: 218 GB of DRAM reads per 16-pass launch).
#pragma once
#include <cuda.h>
#include <cstdint>
#include "common.cuh"
#include "aux_kernels.cuh"

namespace starmm {
namespace tcg {
constexpr int BM = 128;                 // output rows per CTA (UMMA M = 256 per pair)
constexpr int BN = 256;                 // output columns per pair tile (UMMA N)
constexpr int BNH = BN / 2;             // B^T rows loaded per CTA
constexpr int BK = 128;                 // int8 elements (= bytes) per k-stage: one 128B swizzle atom
constexpr int STAGES = 6;
constexpr int EPI_WARPS = 8;           // 2 per TMEM lane quarter, each half the columns
constexpr int THREADS = 64 + 32 * EPI_WARPS;
constexpr int A_BYTES = BM * BK, B_BYTES = BNH * BK, STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int EPI_PITCH = 33;           // 4-byte words; per-warp 32 x 32 transpose buffer
constexpr int EPI_BYTES = EPI_WARPS * 32 * EPI_PITCH * 4;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + EPI_BYTES + 1024 /*align*/ + 256 /*barriers*/;
constexpr int ACC_COLS = BN;            // one s32 accumulator = 256 TMEM columns
constexpr int TMEM_COLS = 2 * ACC_COLS; // double-buffered: all 512 columns
// instruction descriptor: s32 accumulate (bits 4-5 = 2), A s8 (bit 7), B s8 (bit 10),
// both K-major, N >> 3 at bits 17-22, M >> 4 at bits 24-28
constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(256 >> 4) << 24);
}  // namespace tcg

struct TcgShape {
    int tiles_m, tiles_n, num_tiles, group_m;   // 256 x 256 pair tiles, grouped raster
    int nk;                                     // k-stages per pass
    int passes;                                 // stacked operand passes (1 or #moduli), pass-major
    int a_pass_rows, b_pass_rows;               // row offset of pass p in the stacked maps
    // bounded drift (optional): the producer of every CTA may start wave w + gate_depth
    // only after all CTAs issued every load of wave w (waves = pass x tile round), so
    // the pairs stay close enough in time to share each wave's panels in L2.  Meant
    // for a fully co-resident grid (cudaOccupancyMaxActiveClusters); a wait gives up
    // after 2 ms, so a partly resident grid is slower but cannot deadlock.
    unsigned* gate;                             // passes * rounds counters, zeroed; or null
    int gate_depth, rounds;
    Pred pr;                                    // device-side path predicate (common.cuh)
};

// ---------------------------------------------------------------------------
// PTX helpers (cluster-aware mbarriers, 2-CTA TMA, UMMA)
// ---------------------------------------------------------------------------
namespace tcgx {
STARMM_DEV uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
STARMM_DEV uint32_t cta_rank() {
    uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r;
}
STARMM_DEV void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
STARMM_DEV unsigned long long globaltimer_ns() {
    unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t;
}
STARMM_DEV unsigned ld_acquire(const unsigned* p) {
    unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
STARMM_DEV void mb_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
STARMM_DEV void mb_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
STARMM_DEV void mb_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "TCG_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra TCG_WAIT_%=;\n\t}" ::"r"(su32(b)), "r"(parity) : "memory");
}
// arrive on the same barrier in CTA `rank` of the cluster
STARMM_DEV void mb_arrive_cluster(uint64_t* b, uint32_t rank) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(su32(b)), "r"(rank));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
// 2-CTA TMA: data into this CTA's smem, completion bytes onto the LEADER's barrier
STARMM_DEV void tma_load_2sm(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
    const uint32_t mbar = su32(bar) & 0xFEFFFFFFu;   // peer bit cleared: CTA 0 of the pair
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];"
        ::"r"(su32(dst)), "l"((uint64_t)map), "r"(mbar), "r"(x), "r"(y) : "memory");
}
// UMMA smem descriptor: K-major, SWIZZLE_128B, 8-row core groups 1024 B apart
STARMM_DEV uint64_t desc_sw128(const void* smem) {
    uint64_t d = 0;
    d |= (uint64_t)((su32(smem) >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}
STARMM_DEV void umma2_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(tmem_d), "l"(da), "l"(db), "r"(tcg::IDESC), "r"(accumulate));
}
// arrive (once) on `bar` in both CTAs of the pair when all prior MMAs retire
STARMM_DEV void umma2_commit_both(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
        ::"r"(su32(bar)), "h"((uint16_t)0x3) : "memory");
}
STARMM_DEV void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]),
          "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]),
          "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
}  // namespace tcgx

STARMM_DEV void tcg_tile_coords(const TcgShape& s, int t, int& tm, int& tn) {
    const int width = s.group_m * s.tiles_n;
    const int grp = t / width;
    const int first_m = grp * s.group_m;
    const int gsize = min(s.tiles_m - first_m, s.group_m);
    const int r = t - grp * width;
    tm = first_m + r % gsize;
    tn = r / gsize;
}

// Epilogue context handed to the functor for one warp x 32-column chunk.
struct TcgChunk {
    int row0;        // first global output row of this warp's 32 rows
    int col0;        // first global output column of the chunk
    int pass;        // pass index (CRT modulus)
    int last;        // last pass of the tile
    int lane;
    uint32_t* stage; // this warp's 32 x EPI_PITCH word transpose buffer
    int warp_q;      // TMEM lane quarter (w % 4)
    int chunk;       // 0 .. BN/32-1
};

// Transpose helper: lane L holds row (row0 + L), columns col0 .. col0+31 in v[];
// afterwards lane L reads column (col0 + L) of row (row0 + r) from stage[r * PITCH + L].
STARMM_DEV void tcg_stage_rows(const TcgChunk& c, const uint32_t (&v)[32]) {
#pragma unroll
    for (int j = 0; j < 32; ++j) c.stage[c.lane * tcg::EPI_PITCH + j] = v[j];
    __syncwarp();
}

template <class Epi>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(tcg::THREADS, 1)
tcg_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
           TcgShape sh, Epi epi) {
    using namespace tcg;
    using namespace tcgx;
    if (sh.pr.off()) return;   // uniform over the cluster: both CTAs leave before any sync
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char* tiles = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint32_t* epi_stage = reinterpret_cast<uint32_t*>(tiles + STAGES * STAGE_BYTES);
    uint64_t* full = reinterpret_cast<uint64_t*>(tiles + STAGES * STAGE_BYTES + EPI_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* acc_full = empty + STAGES;      // [2]
    uint64_t* acc_empty = acc_full + 2;       // [2] (used in the leader only)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cta_rank();
    const bool leader = rank == 0;
    const int cluster_id = blockIdx.x >> 1, num_clusters = gridDim.x >> 1;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) { mb_init(&full[s], 1); mb_init(&empty[s], 1); }
        for (int b = 0; b < 2; ++b) { mb_init(&acc_full[b], 1); mb_init(&acc_empty[b], 2 * EPI_WARPS); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmap_a) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmap_b) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                     ::"r"(su32(tmem_slot)), "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    cluster_sync();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {   // ---- TMA producer (both CTAs) ----
            uint32_t it = 0;
            for (int p = 0; p < sh.passes; ++p) {
                for (int t = cluster_id; t < sh.num_tiles; t += num_clusters) {
                    int tm, tn;
                    tcg_tile_coords(sh, t, tm, tn);
                    const int w = p * sh.rounds + (t - cluster_id) / num_clusters;
                    if (sh.gate && w >= sh.gate_depth) {
                        const int wd = w - sh.gate_depth, rd = wd % sh.rounds;
                        const unsigned need = 2u * (unsigned)min(num_clusters, sh.num_tiles - rd * num_clusters);
                        // bounded wait: if the grid is not fully co-resident (another
                        // kernel holding SMs), give up after 2 ms instead of hanging
                        const unsigned long long t0 = globaltimer_ns();
                        while (ld_acquire(sh.gate + wd) < need && globaltimer_ns() - t0 < 2000000ull)
                            __nanosleep(128);
                    }
                    const int ay = p * sh.a_pass_rows + tm * 256 + (int)rank * BM;
                    const int by = p * sh.b_pass_rows + tn * BN + (int)rank * BNH;
                    for (int kt = 0; kt < sh.nk; ++kt, ++it) {
                        const uint32_t s = it % STAGES;
                        if (it >= STAGES) mb_wait(&empty[s], ((it / STAGES) - 1) & 1);
                        unsigned char* a = tiles + s * STAGE_BYTES;
                        if (leader) mb_expect_tx(&full[s], 2 * STAGE_BYTES);
                        tma_load_2sm(a, &tmap_a, &full[s], kt * BK, ay);
                        tma_load_2sm(a + A_BYTES, &tmap_b, &full[s], kt * BK, by);
                    }
                    if (sh.gate) {
                        __threadfence();
                        atomicAdd(sh.gate + w, 1u);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader && lane == 0) {   // ---- MMA issuer (leader CTA only) ----
            uint32_t it = 0, u = 0;
            for (int p = 0; p < sh.passes; ++p) {
                for (int t = cluster_id; t < sh.num_tiles; t += num_clusters, ++u) {
                    const uint32_t b = u & 1;
                    if (u >= 2) mb_wait(&acc_empty[b], ((u >> 1) - 1) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t acc = tmem + b * ACC_COLS;
                    for (int kt = 0; kt < sh.nk; ++kt, ++it) {
                        const uint32_t s = it % STAGES;
                        mb_wait(&full[s], (it / STAGES) & 1);
                        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                        const unsigned char* a = tiles + s * STAGE_BYTES;
                        const uint64_t da = desc_sw128(a), db = desc_sw128(a + A_BYTES);
#pragma unroll
                        for (int k = 0; k < BK / 32; ++k)
                            umma2_i8(acc, da + 2 * k, db + 2 * k, (kt | k) != 0);
                        umma2_commit_both(&empty[s]);
                    }
                    umma2_commit_both(&acc_full[b]);
                }
            }
        }
    } else {   // ---- epilogue warps 2..9 (both CTAs) ----
        const int q = warp & 3, half = (warp - 2) >> 2;
        uint32_t* stage = epi_stage + (warp - 2) * 32 * EPI_PITCH;
        uint32_t u = 0;
        for (int p = 0; p < sh.passes; ++p) {
            for (int t = cluster_id; t < sh.num_tiles; t += num_clusters, ++u) {
                int tm, tn;
                tcg_tile_coords(sh, t, tm, tn);
                const uint32_t b = u & 1;
                mb_wait(&acc_full[b], (u >> 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                TcgChunk c;
                c.row0 = tm * 256 + (int)rank * BM + q * 32;
                c.pass = p; c.last = p == sh.passes - 1; c.lane = lane; c.stage = stage;
                c.warp_q = q;
#pragma unroll 1
                for (int ch = half * (BN / 64); ch < (half + 1) * (BN / 64); ++ch) {
                    uint32_t v[32];
                    tmem_ld32(tmem + b * ACC_COLS + ((uint32_t)(q * 32) << 16) + ch * 32, v);
                    c.col0 = tn * BN + ch * 32;
                    c.chunk = ch;
                    epi(c, v);
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) mb_arrive_cluster(&acc_empty[b], 0);
            }
        }
    }
    __syncwarp();
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    cluster_sync();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
    }
}

// ---------------------------------------------------------------------------
// Epilogues
// ---------------------------------------------------------------------------
// int32 results straight to an int32 matrix (dev harness / tests of the core).
struct EpiStoreI32 {
    int* C; long long ldc; int M, N;
    STARMM_DEV void operator()(const TcgChunk& c, const uint32_t (&v)[32]) const {
        tcg_stage_rows(c, v);
        const int col = c.col0 + c.lane;
#pragma unroll 4
        for (int r = 0; r < 32; ++r) {
            const int row = c.row0 + r;
            if (row < M && col < N) C[(long long)row * ldc + col] = (int)c.stage[r * tcg::EPI_PITCH + c.lane];
        }
        __syncwarp();
    }
};

// Output-side fold shared by the tensor-core epilogues: plain store (INIT_IDENTITY),
// exclusive fold (each output element has one owner), or -- for the multi-GPU fused
// k-split combine (starmm_plan_set_peers) -- the atomic-madd into the owner's rows.
struct TcgOut {
    void* C; long long ldc; long long M, N; int init_identity;
    int remote_parts; long long remote_rows, remote_ld; void* remote_base[8];
};
template <class Sr>
STARMM_DEV void tcg_fold(const TcgOut& o, long long row, long long col, typename Sr::T d) {
    using T = typename Sr::T;
    if (o.remote_parts > 0) {
        const int part = (int)(row / o.remote_rows);
        void* base = o.remote_base[0];   // constant indices: no local-memory copy of the params
#pragma unroll
        for (int i = 1; i < 8; ++i) base = part == i ? o.remote_base[i] : base;
        T* q = (T*)base + (row - part * o.remote_rows) * o.remote_ld + col;
        Sr::atomic_fold(q, d);
        return;
    }
    T* q = (T*)o.C + row * o.ldc + col;
    *q = o.init_identity ? d : Sr::fold(*q, d);
}

// small-range int64 ring: widen (exact) and fold into / store to int64 C.  The C
// loads of a chunk are issued as one batch (16 rows in flight) before any store.
struct EpiFoldI64 {
    TcgOut o;
    int shift = 0;   // the accumulator's weight 2^shift (radix-256 digit groups); 0 otherwise
    STARMM_DEV void operator()(const TcgChunk& c, const uint32_t (&v)[32]) const {
        tcg_stage_rows(c, v);
        const long long col = c.col0 + c.lane;
        if (o.remote_parts > 0) {
            for (int r = 0; r < 32; ++r) {
                const long long row = c.row0 + r;
                if (row < o.M && col < o.N)
                    tcg_fold<SrInt64>(o, row, col, (long long)((unsigned long long)(long long)(int)
                                                               c.stage[r * tcg::EPI_PITCH + c.lane] << shift));
            }
        } else {
            long long* Cp = (long long*)o.C;
#pragma unroll
            for (int h = 0; h < 32; h += 16) {
                long long cv[16];
#pragma unroll
                for (int r = 0; r < 16; ++r) {
                    const long long row = c.row0 + h + r;
                    cv[r] = (!o.init_identity && row < o.M && col < o.N) ? Cp[row * o.ldc + col] : 0;
                }
#pragma unroll
                for (int r = 0; r < 16; ++r) {
                    const long long row = c.row0 + h + r;
                    if (row < o.M && col < o.N)
                        Cp[row * o.ldc + col] = (long long)((unsigned long long)cv[r] +
                            ((unsigned long long)(long long)(int)c.stage[(h + r) * tcg::EPI_PITCH + c.lane] << shift));
                }
            }
        }
        __syncwarp();
    }
};

// int64 (|x| <= 127 once the guard passes) -> int8, K-major [rows][kp], zero padded.
// A is already [m][k]; B ([k][n]) is transposed through a 32x32 shared-memory tile.
// Both fold the range guard into the same pass (RangeAcc, aux_kernels.cuh).
// grid: x over 8-element k-words of a row, y strides over rows (no divisions)
__global__ void pack_i8_rows_kernel(const long long* A, long long rows, long long kdim, long long lda,
                                    signed char* P, long long rowsp, long long kp,
                                    unsigned long long* range) {
    RangeAcc acc;
    const long long k0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 8;
    if (k0 < kp) {
        for (long long r = blockIdx.y; r < rowsp; r += gridDim.y) {
            long long v[8];
            const long long* src = A + r * lda + k0;
            if (r < rows && k0 + 8 <= kdim && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
#pragma unroll
                for (int e = 0; e < 8; e += 2) {          // 16-byte loads
                    const longlong2 x = *reinterpret_cast<const longlong2*>(src + e);
                    v[e] = x.x; v[e + 1] = x.y;
                }
            } else {
#pragma unroll
                for (int e = 0; e < 8; ++e) v[e] = (r < rows && k0 + e < kdim) ? src[e] : 0;
            }
            uint32_t w[2] = {0u, 0u};
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                acc.add(v[e]);
                w[e >> 2] |= (uint32_t)(unsigned char)(signed char)v[e] << (8 * (e & 3));
            }
            *reinterpret_cast<uint2*>(P + r * kp + k0) = make_uint2(w[0], w[1]);
        }
    }
    if (range) acc.flush(range);
}

// B [k][n] -> P [n][kp] int8.  Block (32, 8) covers 128 k x 32 columns: coalesced 256-byte
// row reads, then every warp writes one column's 128 k-bytes as 32 words (a full line).
__global__ void __launch_bounds__(256)
pack_i8_transpose_kernel(const long long* B, long long kdim, long long cols, long long ldb,
                         signed char* P, long long colsp, long long kp,
                         unsigned long long* range) {
    constexpr int TK = 128;
    __shared__ uint32_t tile[32][TK / 4 + 1];     // [column][k-word]
    RangeAcc acc;
    const long long k0 = (long long)blockIdx.y * TK, c0 = (long long)blockIdx.x * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;   // 32 x 8
    const long long c = c0 + tx;
    // thread (tx, ty) reads k = k0 + 4*ty + 32*i + e (e = 0..3) of column tx: packs one word
#pragma unroll
    for (int i = 0; i < TK / 32; ++i) {
        uint32_t w = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const long long k = k0 + 32 * i + 4 * ty + e;
            const long long v = (k < kdim && c < cols) ? B[k * ldb + c] : 0;
            acc.add(v);
            w |= (uint32_t)(unsigned char)(signed char)v << (8 * e);
        }
        tile[tx][8 * i + ty] = w;
    }
    if (range) acc.flush(range);
    __syncthreads();
    // warp ty writes columns ty, ty + 8, ty + 16, ty + 24: lane tx = k-word tx
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int col = ty + 8 * j;
        const long long cc = c0 + col, kk = k0 + 4 * tx;
        if (cc < colsp && kk < kp) *reinterpret_cast<uint32_t*>(P + cc * kp + kk) = tile[col][tx];
    }
}


// ---- opt-in general int64 on the int8 tensor cores: signed radix-256 digits ------------
// x = sum_i d_i 256^i (mod 2^64) with d_i in [-128, 127] (balanced digits, the carry out
// of the top digit dropped).  a*b mod 2^64 = sum_s 2^(8s) sum_{q<=s} d_q(a) d_{s-q}(b), so
// digit group s (s = 0..7) is ONE int8 GEMM over a (s+1)-times longer k: A's digits
// 0..s of each k against B's digits s..0.  Packed per K chunk (<= 8192, so every
// group's int32 sum (s+1) K 2^14 <= 2^30 is exact), limb-major within a row:
//   A: P[chunk][row][limb 0..7][Kc]      B^T: P[chunk][col][limb 7..0][Kc]
// so group s is a contiguous (s+1) Kc window of every row: columns [0, (s+1) Kc) of A,
// [(7-s) Kc, 8 Kc) of B^T -- one 2-D TMA map each (row stride 8 Kc bytes).
STARMM_DEV void i64_digits(long long x, signed char (&d)[8]) {
    unsigned long long u = (unsigned long long)x;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        int v = (int)(u & 0xffull);
        u >>= 8;
        if (v >= 128) { v -= 256; u += 1; }
        d[i] = (signed char)v;
    }
}

// A (rows x kdim) -> digit planes; thread per (row, 8 consecutive k)
// Both digit packers also run the range guard (RangeAcc): as a plan's first guess they
// are what tells the next call whether the single-GEMM int8 path would do.
__global__ void pack_limbs_rows_kernel(const long long* A, long long rows, long long kdim, long long lda,
                                       signed char* P, long long rowsp, long long kc, int nchunk,
                                       unsigned long long* range = nullptr, Pred pr = Pred()) {
    if (pr.off()) return;
    RangeAcc acc;
    const long long kw = (long long)blockIdx.x * blockDim.x + threadIdx.x;   // 8-k word within the padded k
    const long long kp_all = kc * nchunk;
    const bool live = kw * 8 < kp_all;
    for (long long r = blockIdx.y; live && r < rowsp; r += gridDim.y) {
        signed char d[8][8];   // [k][limb]
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const long long k = kw * 8 + e;
            const long long x = (r < rows && k < kdim) ? A[r * lda + k] : 0;
            acc.add(x);
            i64_digits(x, d[e]);
        }
        const long long k0 = kw * 8, ch = k0 / kc, kk = k0 - ch * kc;
        signed char* base = P + ((ch * rowsp + r) * 8) * kc + kk;
#pragma unroll
        for (int l = 0; l < 8; ++l) {
            unsigned long long w = 0;
#pragma unroll
            for (int e = 0; e < 8; ++e) w |= (unsigned long long)(unsigned char)d[e][l] << (8 * e);
            *reinterpret_cast<unsigned long long*>(base + l * kc) = w;
        }
    }
    if (range) acc.flush(range);   // every thread reaches the flush (full-warp shuffles)
}

// B (kdim x cols) -> B^T digit planes in reversed limb order; a 32-k x 32-col tile goes
// through shared memory (reads coalesced along columns, writes along k)
__global__ void pack_limbs_cols_kernel(const long long* B, long long kdim, long long cols, long long ldb,
                                       signed char* P, long long colsp, long long kc, int nchunk,
                                       unsigned long long* range = nullptr, Pred pr = Pred()) {
    if (pr.off()) return;
    __shared__ long long tile[32][33];
    RangeAcc acc;
    const long long c0 = (long long)blockIdx.x * 32, k0 = (long long)blockIdx.y * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;      // 32 x 8
    for (int i = ty; i < 32; i += 8) {
        const long long k = k0 + i, c = c0 + tx;
        tile[i][tx] = (k < kdim && c < cols) ? B[k * ldb + c] : 0;
        acc.add(tile[i][tx]);
    }
    if (range) acc.flush(range);
    __syncthreads();
    // thread (tx, ty): column c0 + (ty*4 .. ty*4+3), k = k0 + tx
    for (int j = ty; j < 32; j += 8) {
        const long long c = c0 + j, k = k0 + tx;
        if (c >= colsp || k >= kc * nchunk) continue;
        signed char d[8];
        i64_digits(tile[tx][j], d);
        const long long ch = k / kc, kk = k - ch * kc;
        signed char* base = P + ((ch * colsp + c) * 8) * kc + kk;
#pragma unroll
        for (int l = 0; l < 8; ++l) base[(7 - l) * kc] = d[l];
    }
}

}  // namespace starmm
