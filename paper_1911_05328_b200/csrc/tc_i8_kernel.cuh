// tc_i8_kernel.cuh -- OPT-IN exact int64 (+,x) on the 5th-generation tensor core.
//
// When every |x| <= 127 and K*max|a|*max|b| < 2^31 (the same range guard as the
// IDP.4A path), the int64 ring product equals an int8 x int8 product with int32
// accumulation -- exactly what tcgen05.mma kind::i8 computes.  This is an
// opt-in experiment (STARMM_F_INT_TENSOR): BASELINE's north star asks for a
// CUDA-core loop for exact-integer (+,x), which stays the default.
//
// Roles (one CTA per SM, persistent over 128 x 256 output tiles):
//   warp 0 lane 0 : TMA producer -- 128x128-byte A and 256x128-byte B boxes per
//                   k-stage (int8, K-major, SWIZZLE_128B) into a STAGES-deep ring
//   warp 1 lane 0 : MMA issuer -- 4 x tcgen05.mma.cta_group::1.kind::i8 (M=128,
//                   N=256, K=32) per stage into a 256-column s32 TMEM accumulator;
//                   tcgen05.commit frees ring slots and signals the epilogue
//   warps 2..5    : epilogue -- tcgen05.ld.32x32b (TMEM lane = output row), widen
//                   to int64, fold into C (or store, INIT_IDENTITY)
#pragma once
#include <cuda.h>
#include "common.cuh"
#include "aux_kernels.cuh"

namespace starmm {
namespace tci8 {
constexpr int BM = 128, BN = 256, BK = 128;          // BK in int8 elements (= bytes)
constexpr int STAGES = 4;
constexpr int THREADS = 192;
constexpr int A_BYTES = BM * BK, B_BYTES = BN * BK, STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
constexpr int TMEM_COLS = 256;
// instruction descriptor: s32 accumulate, s8 x s8, both K-major, N = 256, M = 128
constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);
}  // namespace tci8

struct TcI8Params {
    long long tiles_m, tiles_n, num_tiles;
    int nk;                      // k-stages (Kp / BK)
    int init_identity;
    long long* C; long long ldc; long long M, N;
};

STARMM_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

STARMM_DEV void mb_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
STARMM_DEV void mb_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
STARMM_DEV void mb_arrive1(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
STARMM_DEV void mb_wait_parity(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "TCI8_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra TCI8_WAIT_%=;\n\t}" ::"r"(smem_u32(b)), "r"(parity) : "memory");
}
STARMM_DEV void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];"
        ::"r"(smem_u32(dst)), "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(x), "r"(y) : "memory");
}
// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, 8-row atoms 1024 B apart
STARMM_DEV uint64_t umma_desc_sw128(const void* smem) {
    uint64_t d = 0;
    d |= (uint64_t)((smem_u32(smem) >> 4) & 0x3FFF);   // start address
    d |= (uint64_t)1 << 16;                            // LBO (unused for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;                  // SBO: next 8-row group
    d |= (uint64_t)1 << 46;                            // version (sm100)
    d |= (uint64_t)2 << 61;                            // SWIZZLE_128B
    return d;
}
STARMM_DEV void umma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(tmem_d), "l"(da), "l"(db), "r"(tci8::IDESC), "r"(accumulate));
}
STARMM_DEV void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 ::"r"(smem_u32(bar)) : "memory");
}

__global__ void __launch_bounds__(tci8::THREADS, 1)
tc_i8_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
             TcI8Params p) {
    using namespace tci8;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char* tiles = reinterpret_cast<unsigned char*>(          // SWIZZLE_128B: 1024-B aligned
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(tiles + STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* acc_full = empty + STAGES;
    uint64_t* acc_empty = acc_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) { mb_init(&full[s], 1); mb_init(&empty[s], 1); }
        mb_init(acc_full, 1);
        mb_init(acc_empty, 4);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmap_a) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmap_b) : "memory");
    }
    if (warp == 1) {   // TMEM: 256 columns x 128 lanes of s32
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     ::"r"(smem_u32(tmem_slot)), "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {   // ---- TMA producer ----
            long long it = 0;
            for (long long t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
                const int tm = (int)(t / p.tiles_n), tn = (int)(t % p.tiles_n);
                for (int kt = 0; kt < p.nk; ++kt, ++it) {
                    const int s = (int)(it % STAGES);
                    if (it >= STAGES) mb_wait_parity(&empty[s], (uint32_t)(((it / STAGES) - 1) & 1));
                    unsigned char* a = tiles + s * STAGE_BYTES;
                    mb_expect_tx(&full[s], STAGE_BYTES);
                    tma_load_2d(a, &tmap_a, &full[s], kt * BK, tm * BM);
                    tma_load_2d(a + A_BYTES, &tmap_b, &full[s], kt * BK, tn * BN);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {   // ---- MMA issuer ----
            long long it = 0, tile_no = 0;
            for (long long t = blockIdx.x; t < p.num_tiles; t += gridDim.x, ++tile_no) {
                if (tile_no > 0) mb_wait_parity(acc_empty, (uint32_t)((tile_no - 1) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                for (int kt = 0; kt < p.nk; ++kt, ++it) {
                    const int s = (int)(it % STAGES);
                    mb_wait_parity(&full[s], (uint32_t)((it / STAGES) & 1));
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const unsigned char* a = tiles + s * STAGE_BYTES;
                    const uint64_t da = umma_desc_sw128(a), db = umma_desc_sw128(a + A_BYTES);
#pragma unroll
                    for (int k = 0; k < BK / 32; ++k)   // 32 int8 = 32 bytes = 2 x 16B per step
                        umma_i8(tmem, da + 2 * k, db + 2 * k, (kt | k) != 0);
                    umma_commit(&empty[s]);             // slot free once these MMAs retire
                }
                umma_commit(acc_full);                  // accumulator complete
            }
        }
    } else {   // ---- epilogue warps 2..5: TMEM lanes 32*(warp%4) .. +32 ----
        const int lane_grp = warp & 3;
        long long tile_no = 0;
        for (long long t = blockIdx.x; t < p.num_tiles; t += gridDim.x, ++tile_no) {
            const int tm = (int)(t / p.tiles_n), tn = (int)(t % p.tiles_n);
            mb_wait_parity(acc_full, (uint32_t)(tile_no & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const long long row = (long long)tm * BM + lane_grp * 32 + lane;
            long long* crow = p.C + row * p.ldc + (long long)tn * BN;
#pragma unroll 1
            for (int chunk = 0; chunk < BN / 32; ++chunk) {
                uint32_t v[32];
                const uint32_t taddr = tmem + ((uint32_t)(lane_grp * 32) << 16) + chunk * 32;
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
                    "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                    "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                      "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
                      "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]),
                      "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                      "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
                      "=r"(v[30]), "=r"(v[31])
                    : "r"(taddr));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                const long long c0 = (long long)tn * BN + chunk * 32;
                if (row < p.M) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        if (c0 + j < p.N) {
                            long long* q = crow + chunk * 32 + j;
                            const long long d = (long long)(int)v[j];   // sign-extend: exact
                            *q = p.init_identity ? d
                                                 : (long long)((unsigned long long)*q + (unsigned long long)d);
                        }
                    }
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mb_arrive1(acc_empty);       // the MMA warp may overwrite TMEM
        }
    }
    __syncthreads();
    if (warp == 1) {
        __syncwarp();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
    }
}

// int64 (|x| <= 127 once the guard passes) -> int8, K-major [rows][kp], zero padded.
// A is already [m][k]; B ([k][n]) is transposed through a 32x32 shared-memory tile.
// Both fold the range guard into the same pass (RangeAcc, aux_kernels.cuh).
__global__ void pack_i8_rows_kernel(const long long* A, long long rows, long long kdim, long long lda,
                                    signed char* P, long long rowsp, long long kp,
                                    unsigned long long* range) {
    RangeAcc acc;
    long long total = rowsp * kp;
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        long long r = idx / kp, k = idx - r * kp;
        long long v = (r < rows && k < kdim) ? A[r * lda + k] : 0;
        acc.add(v);
        P[idx] = (signed char)v;
    }
    if (range) acc.flush(range);
}

__global__ void pack_i8_transpose_kernel(const long long* B, long long kdim, long long cols, long long ldb,
                                         signed char* P, long long colsp, long long kp,
                                         unsigned long long* range) {
    __shared__ signed char tile[32][33];
    RangeAcc acc;
    const long long k0 = (long long)blockIdx.y * 32, c0 = (long long)blockIdx.x * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;   // 32 x 8
    for (int i = ty; i < 32; i += 8) {
        long long k = k0 + i, c = c0 + tx;
        long long v = (k < kdim && c < cols) ? B[k * ldb + c] : 0;
        acc.add(v);
        tile[i][tx] = (signed char)v;
    }
    if (range) acc.flush(range);
    __syncthreads();
    for (int i = ty; i < 32; i += 8) {
        long long c = c0 + i, k = k0 + tx;
        if (c < colsp && k < kp) P[c * kp + k] = tile[tx][i];
    }
}

}  // namespace starmm
