// starmm_api.cu -- the C ABI of include/starmm_b200.h: plans, the device
// scratch arena (the LIFO block pool), path selection and launches.
//
// Reference mapping (relative to /root/reference/pkg/src/starmm/):
//   plan create/destroy ....... Executor(cfg) lifecycle (runtime.py:57-98)
//   execute validation ........ registry.run_algorithm (registry.py:23-57)
//   schedule dispatch ......... classic._classic_root (classic.py:241-265)
//   switch depth .............. classic.switch_depth (classic.py:78-83)
//   arena (pooled/raw temps) .. Executor.acquire_temp/release_temp (runtime.py:198-229)
//                               and Pool (pool.py:67-167): exact-size LIFO stacks,
//                               blocks never cleared, fresh/reuse/high-water counters
//   co3 merge ................. ops.merge_tasks (ops.py:108-155)
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <vector>
#include <type_traits>
#include <string>
#include <algorithm>
#include <cmath>
#include <limits>

#include "../../include/starmm_b200.h"
#include "common.cuh"
#include "writeback.cuh"
#include "dmma_kernel.cuh"
#include "simt_kernel.cuh"
#include "aux_kernels.cuh"
#include "tc_gemm.cuh"
#include "ozaki.cuh"
#include "simt_launch.h"

using namespace starmm;

namespace {

thread_local int g_last_cuda_error = 0;

int cuda_status(cudaError_t e) {
    if (e == cudaSuccess) return STARMM_OK;
    g_last_cuda_error = (int)e;
    if (e == cudaErrorMemoryAllocation) { cudaGetLastError(); return STARMM_ALLOC_FAILURE; }
    return STARMM_CUDA_ERROR + (int)e;
}

#define CK(x) do { cudaError_t _e = (x); if (_e != cudaSuccess) return cuda_status(_e); } while (0)
#define TRY(x) do { int _s = (x); if (_s != STARMM_OK) return _s; } while (0)

bool is_pow2(long long x) { return x >= 1 && (x & (x - 1)) == 0; }
long long round_up(long long x, long long m) { return (x + m - 1) / m * m; }

int elem_bytes(int sr) {
    return (sr == STARMM_SR_TROPICAL_F32 || sr == STARMM_SR_TROPICAL_I32) ? 4 : 8;
}

// classic.py:78-83: smallest k with 4**k >= p
int switch_depth(int p) {
    int k = 0;
    long long q = 1;
    while (q < p) { q *= 4; ++k; }
    return k;
}

// ---- the arena: exact-size LIFO free stacks (pool.py:89-132) -----------------
struct Arena {
    std::map<size_t, std::vector<void*>> free_stacks;
    std::vector<std::pair<void*, size_t>> owned;
    long long total_allocated = 0, issued = 0, high_water = 0, fresh = 0, reuse = 0;

    int acquire(size_t bytes, void** out, bool count_as_temp, long long* fresh_ctr,
                long long* reuse_ctr) {
        bytes = (size_t)round_up((long long)std::max<size_t>(bytes, 256), 256);
        auto& st = free_stacks[bytes];
        if (!st.empty()) {
            *out = st.back();             // LIFO pop (pool.py:97)
            st.pop_back();
            if (count_as_temp) ++*reuse_ctr;
        } else {
            void* p = nullptr;
            cudaError_t e = cudaMalloc(&p, bytes);
            if (e != cudaSuccess) return cuda_status(e);
            owned.push_back({p, bytes});
            total_allocated += (long long)bytes;
            *out = p;
            if (count_as_temp) ++*fresh_ctr;
        }
        issued += (long long)bytes;
        high_water = std::max(high_water, issued);
        return STARMM_OK;
    }
    void release(void* p, size_t bytes) {
        bytes = (size_t)round_up((long long)std::max<size_t>(bytes, 256), 256);
        free_stacks[bytes].push_back(p);  // blocks are not cleared (pool.py:4-6)
        issued -= (long long)bytes;
    }
    void destroy() {
        for (auto& o : owned) cudaFree(o.first);
        owned.clear();
        free_stacks.clear();
    }
};

struct Block { void* p = nullptr; size_t bytes = 0; };

}  // namespace

struct starmm_plan {
    int sr, algo, alloc, base_dim, workers, ksplit_req, device, flags;
    long long m, n, k;
    int sms = 0;
    Arena arena;
    // persistent device bookkeeping (from the arena, kept for the plan's life)
    unsigned long long* d_counters = nullptr;   // CNT__N
    unsigned long long* d_range = nullptr;      // 2 words
    // the guard's verdict is published to mapped pinned host memory by a 1-thread kernel
    // (zero-copy stores, no copy engine: a D2H memcpy here would queue behind the host
    // path's block downloads on the D2H engine)
    volatile unsigned long long* h_range = nullptr;
    unsigned long long* h_range_dev = nullptr;
    unsigned* d_worker_used = nullptr;          // per persistent worker
    unsigned* d_gate = nullptr;                 // DMMA wave-gate counter
    int dmma_gate = 1;                          // 0 inside the host path (overlapping launches)
    int max_workers = 0;
    starmm_stats st;
    long long ws_fresh = 0, ws_reuse = 0, ws_high_water = 0;
    long long raw_count = 0, raw_bytes = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;   // STARMM_F_TIME_MAIN
    int last_guarded_path = 0;                  // optimistic first guess for the next execute
    starmm_plan* twin = nullptr;                // host path: the second compute stream's plan
                                                // (own arena: staging reuse is stream-ordered)
    long long strassen_leaf = 1024;             // Strassen recursion stops at max(b, this)
    long long str_issued = 0;                   // Strassen temporaries currently issued
    // peer destinations of the fused k-split combine (starmm_plan_set_peers)
    int remote_parts = 0;
    long long remote_rows = 0, remote_ld = 0;
    void* remote_base[8] = {};
};

namespace {

// ---- kernel instantiation table: PathId in simt_launch.h ----------------------

// Tile / packing geometry of one kernel path (mirrors the device-side constants).
struct PathShape {
    int bm, bn, bk, per_sm;
    long long a_bytes_per_km;   // packed A bytes per (k, m) element, x1000 for dp4a's 1 byte
    long long b_bytes_per_kn;
};
template <class Pol>
PathShape simt_shape() {
    PathShape sh;
    sh.bm = simt::BM; sh.bn = simt::bn<Pol>(); sh.bk = Pol::BK; sh.per_sm = Pol::OCC;
    // bytes of packed operand per original (k, x) element
    sh.a_bytes_per_km = (long long)Pol::G * sizeof(typename Pol::Tp) * 1000 / Pol::KSTEP;
    sh.b_bytes_per_kn = (long long)Pol::G * sizeof(typename Pol::Tp) * 1000 / (Pol::KSTEP * Pol::OUTS);
    return sh;
}
PathShape path_shape(int path) {
    switch (path) {
    case PATH_DMMA_F64: {
        PathShape sh{DmmaProd::BM, DmmaProd::BN, DmmaProd::BK, DmmaProd::MIN_BLOCKS, 8000, 8000};
        return sh;
    }
    case PATH_SIMT_I64: return simt_shape<PolI64>();
    case PATH_SIMT_I64_NARROW: return simt_shape<PolI64Narrow>();
    case PATH_SIMT_F32_PAIR: return simt_shape<PolF32Pair>();
    case PATH_SIMT_I32_CARRIER: return simt_shape<PolF32Pair>();
    case PATH_SIMT_I32_VMIN: return simt_shape<PolI32Vmin>();
    case PATH_SIMT_I32_SAT: return simt_shape<PolI32Sat>();
    case PATH_SIMT_F64_MIN: return simt_shape<PolF64Min>();
    case PATH_SIMT_I64_DP4A: return simt_shape<PolI8Dp4a>();
    case PATH_SIMT_F32_S16X2: return simt_shape<PolS16x2Min>();
    case PATH_SIMT_I32_S16X2: return simt_shape<PolS16x2Min>();
    case PATH_SIMT_F64T_S16X2: return simt_shape<PolS16x2Min>();
    case PATH_SIMT_F64T_CARRIER: return simt_shape<PolF32Pair>();
    case PATH_TC_I8: {
        PathShape sh{2 * tcg::BM, tcg::BN, tcg::BK, 1, 1000, 1000};
        return sh;
    }
    case PATH_OZAKI_F64: {   // P residue planes of int8 per operand
        PathShape sh{2 * tcg::BM, tcg::BN, tcg::BK, 1, 1000LL * oz::P, 1000LL * oz::P};
        return sh;
    }
    }
    return simt_shape<PolI64>();
}

// mbarrier-pipelined k-loop (tools/sweep_dmma.cu: 35.4 vs 34.4 TF/s with per-stage
// __syncthreads), vectorised FOLD epilogue.  With `gate` (p.gate zeroed here) the
// wave gate with a quarter-wave slack keeps the persistent CTAs in step: DRAM reads
// per n=16384 launch 240-263 GB -> 51 GB at -0.1% (profiles/r01l_dmma_gate.md).
int launch_dmma(const DmmaParams& p, int grid, bool gate, cudaStream_t s) {
    using K = DmmaProd;
    static bool attr_done = false;
    if (!attr_done) {
        CK(cudaFuncSetAttribute(dmma_fp64_kernel_mb<K, 1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                K::SMEM_BYTES));
        CK(cudaFuncSetAttribute(dmma_fp64_kernel_mb<K, 1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                K::SMEM_BYTES));
        attr_done = true;
    }
    if (gate && p.gate) {
        CK(cudaMemsetAsync(p.gate, 0, sizeof(unsigned), s));
        dmma_fp64_kernel_mb<K, 1, 2><<<grid, K::THREADS, K::SMEM_BYTES, s>>>(p);
    } else {
        dmma_fp64_kernel_mb<K, 1, 0><<<grid, K::THREADS, K::SMEM_BYTES, s>>>(p);
    }
    CK(cudaGetLastError());
    return STARMM_OK;
}


template <class Sr>
int launch_madd(void* C, long long ldc, const void* D, long long ldd, long long rows, long long cols,
                int atomic, cudaStream_t s) {
    if (rows <= 0 || cols <= 0) return STARMM_OK;
    using T = typename Sr::T;
    madd_kernel<Sr><<<grid2d(rows, cols), 256, 0, s>>>((T*)C, ldc, (const T*)D, ldd, rows, cols,
                                                           atomic);
    CK(cudaGetLastError());
    return STARMM_OK;
}

int madd_dispatch(int sr, void* C, long long ldc, const void* D, long long ldd, long long rows,
                  long long cols, int atomic, cudaStream_t s) {
    switch (sr) {
    case STARMM_SR_INT64: return launch_madd<SrInt64>(C, ldc, D, ldd, rows, cols, atomic, s);
    case STARMM_SR_FP64: return launch_madd<SrFp64>(C, ldc, D, ldd, rows, cols, atomic, s);
    case STARMM_SR_TROPICAL_F64: return launch_madd<SrTropF64>(C, ldc, D, ldd, rows, cols, atomic, s);
    case STARMM_SR_TROPICAL_F32: return launch_madd<SrTropF32>(C, ldc, D, ldd, rows, cols, atomic, s);
    case STARMM_SR_TROPICAL_I32: return launch_madd<SrTropI32>(C, ldc, D, ldd, rows, cols, atomic, s);
    }
    return STARMM_CONTRACT_VIOLATION;
}

template <class Sr>
int launch_fill(void* C, long long rows, long long cols, long long ld, cudaStream_t s) {
    fill_kernel<Sr><<<grid2d(rows, cols), 256, 0, s>>>((typename Sr::T*)C, rows, cols, ld);
    CK(cudaGetLastError());
    return STARMM_OK;
}

int fill_dispatch(int sr, void* C, long long rows, long long cols, long long ld, cudaStream_t s) {
    switch (sr) {
    case STARMM_SR_INT64: return launch_fill<SrInt64>(C, rows, cols, ld, s);
    case STARMM_SR_FP64: return launch_fill<SrFp64>(C, rows, cols, ld, s);
    case STARMM_SR_TROPICAL_F64: return launch_fill<SrTropF64>(C, rows, cols, ld, s);
    case STARMM_SR_TROPICAL_F32: return launch_fill<SrTropF32>(C, rows, cols, ld, s);
    case STARMM_SR_TROPICAL_I32: return launch_fill<SrTropI32>(C, rows, cols, ld, s);
    }
    return STARMM_CONTRACT_VIOLATION;
}

template <class Tin, class Tp, int G, class Conv>
int launch_pack(const void* A, long long lda, const void* B, long long ldb, long long m,
                long long n, long long k, void* Ap, void* Bp, long long Mp, long long Np,
                long long Kp, Tp pad, cudaStream_t s, unsigned long long* range = nullptr) {
    dim3 ga((unsigned)(Kp / 32), (unsigned)(Mp / 32));
    pack_a_kernel<Tin, Tp, G, Conv><<<ga, dim3(32, 8), 0, s>>>((const Tin*)A, m, k, lda, (Tp*)Ap, Mp,
                                                              Kp, pad, range);
    CK(cudaGetLastError());
    pack_b_kernel<Tin, Tp, G, Conv><<<grid2d(Kp / G, Np), 256, 0, s>>>(
        (const Tin*)B, k, n, ldb, (Tp*)Bp, Np, Kp, pad, range);
    CK(cudaGetLastError());
    return STARMM_OK;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda needed)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                  CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                  CUtensorMapFloatOOBfill);
int make_i8_tmap(CUtensorMap* map, void* base, long long rows, long long kp, int box_rows) {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &q));
        if (!fn || q != cudaDriverEntryPointSuccess) return STARMM_INTERNAL_ERROR;
    }
    cuuint64_t dims[2] = {(cuuint64_t)kp, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)kp};
    cuuint32_t box[2] = {(cuuint32_t)tcg::BK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, base, dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? STARMM_OK : STARMM_INTERNAL_ERROR;
}

// The CTA-pair tensor-core GEMM over `passes` stacked int8 operand planes
// (A: passes x [Mp][Kp], B^T: passes x [Np][Kp]); Mp, Np multiples of 256.
// CTA pairs that can be co-resident (cluster 2x1x1, 1 CTA/SM): the persistent grid,
// which the drift gate requires to be fully resident
template <class Epi>
int tcg_max_clusters(int sms) {
    static int cached = -1;
    if (cached < 0) {
        auto kern = tcg_kernel<Epi>;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, tcg::SMEM_BYTES));
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3((unsigned)sms); lc.blockDim = dim3(tcg::THREADS); lc.dynamicSmemBytes = tcg::SMEM_BYTES;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        lc.attrs = at; lc.numAttrs = 1;
        int c = 0;
        if (cudaOccupancyMaxActiveClusters(&c, kern, &lc) != cudaSuccess || c < 1) {
            cudaGetLastError();
            c = std::max(1, sms / 2);
        }
        cached = c;
    }
    return cached;
}

// `acquire(bytes, &ptr)` hands out stream-ordered scratch (the plan's arena) for the
// drift-gate counters: one per (pass, tile round), zeroed before the launch.
template <class Epi, class Acquire>
int launch_tcg(const void* Ap, const void* Bp, long long Mp, long long Np, long long Kp, int passes,
               const Epi& epi, int sms, cudaStream_t s, Acquire&& acquire) {
    if ((long long)passes * Mp >= (1LL << 31) || (long long)passes * Np >= (1LL << 31)) return STARMM_TOO_LARGE;
    CUtensorMap ta, tb;
    TRY(make_i8_tmap(&ta, const_cast<void*>(Ap), Mp * passes, Kp, tcg::BM));
    TRY(make_i8_tmap(&tb, const_cast<void*>(Bp), Np * passes, Kp, tcg::BNH));
    auto kern = tcg_kernel<Epi>;
    const int clusters = tcg_max_clusters<Epi>(sms);
    TcgShape sh;
    sh.tiles_m = (int)(Mp / 256); sh.tiles_n = (int)(Np / 256); sh.num_tiles = sh.tiles_m * sh.tiles_n;
    sh.group_m = 8;
    sh.nk = (int)(Kp / tcg::BK); sh.passes = passes;
    sh.a_pass_rows = (int)Mp; sh.b_pass_rows = (int)Np;
    const int pairs = std::max(1, std::min(clusters, sh.num_tiles));
    const int grid = 2 * pairs;
    // bounded drift, one wave: 16-pass n=16384 DRAM reads 274 -> 69 GB, GEMM -17%
    // (tools/tc_gemm_dev.cu)
    sh.rounds = (sh.num_tiles + pairs - 1) / pairs;
    sh.gate_depth = 1;
    sh.gate = nullptr;
    if ((long long)passes * sh.rounds > 1) {
        void* g = nullptr;
        const size_t gb = (size_t)passes * sh.rounds * sizeof(unsigned);
        TRY(acquire(gb, &g));
        CK(cudaMemsetAsync(g, 0, gb, s));
        sh.gate = (unsigned*)g;
    }
    kern<<<grid, tcg::THREADS, tcg::SMEM_BYTES, s>>>(ta, tb, sh, epi);
    CK(cudaGetLastError());
    return STARMM_OK;
}

TcgOut tcg_out(const starmm_plan* P, void* C, long long ldc, bool init_identity) {
    TcgOut o;
    o.C = C; o.ldc = ldc; o.M = P->m; o.N = P->n; o.init_identity = init_identity ? 1 : 0;
    o.remote_parts = P->remote_parts; o.remote_rows = P->remote_rows; o.remote_ld = P->remote_ld;
    for (int i = 0; i < 8; ++i) o.remote_base[i] = P->remote_base[i];
    return o;
}

// CRT constants of the Ozaki-II moduli (exact, host side, 128-bit)
const OzCrt& ozaki_crt() {
    static OzCrt c;
    static bool done = false;
    if (done) return c;
    typedef unsigned __int128 u128;
    u128 M = 1;
    for (int p = 0; p < oz::P; ++p) M *= (u128)oz::MOD[p];
    for (int p = 0; p < oz::P; ++p) {
        const int m = oz::MOD[p];
        const u128 Mp = M / (u128)m;
        const int r = (int)(Mp % (u128)m);
        int inv = 1;
        while ((r * inv) % m != 1) ++inv;               // m <= 256: brute force is exact
        const u128 W = (Mp * (u128)inv) % M;
        for (int l = 0; l < 4; ++l) c.W[p][l] = (uint32_t)(W >> (32 * l));
    }
    const u128 H = M / 2;
    for (int l = 0; l < 4; ++l) { c.Ml[l] = (uint32_t)(M >> (32 * l)); c.Mh[l] = (uint32_t)(H >> (32 * l)); }
    c.invM = 1.0 / (double)M;
    done = true;
    return c;
}

// bits kept per scaled operand: M > 2 k 2^(2t) with a one-bit margin
int ozaki_bits(long long k) {
    double lm = 0;
    for (int p = 0; p < oz::P; ++p) lm += std::log2((double)oz::MOD[p]);
    int t = (int)std::floor((lm - std::log2((double)std::max(1LL, k)) - 2.0) / 2.0);
    return std::min(t, 62);
}

int occupancy_grid(starmm_plan* P, int per_sm, long long tasks) {
    long long g = (long long)P->sms * per_sm;
    return (int)std::max<long long>(1, std::min<long long>(g, tasks));
}

int ensure_bookkeeping(starmm_plan* P) {
    if (P->d_counters) return STARMM_OK;
    P->max_workers = P->sms * 2;
    long long fr = 0, ru = 0;
    void* p = nullptr;
    size_t bytes = CNT__N * 8 + 16 + (size_t)P->max_workers * 4 + 16;
    TRY(P->arena.acquire(bytes, &p, false, &fr, &ru));
    CK(cudaMemset(p, 0, bytes));
    P->d_counters = (unsigned long long*)p;
    P->d_range = P->d_counters + CNT__N;
    P->d_worker_used = (unsigned*)(P->d_range + 2);
    P->d_gate = P->d_worker_used + P->max_workers;
    void* h = nullptr;
    CK(cudaHostAlloc(&h, 16, cudaHostAllocMapped));
    P->h_range = (volatile unsigned long long*)h;
    CK(cudaHostGetDevicePointer((void**)&P->h_range_dev, h, 0));
    return STARMM_OK;
}

}  // namespace

// ============================================================================
int starmm_simt_launch(int path, const starmm::SimtParams& sp, int grid, int sms, cudaStream_t s) {
    switch (path) {
    case PATH_SIMT_I64: case PATH_SIMT_I64_NARROW: case PATH_SIMT_I64_DP4A:
        return starmm_simt_launch_int(path, sp, grid, sms, s);
    case PATH_SIMT_F32_PAIR: case PATH_SIMT_I32_CARRIER: case PATH_SIMT_F64T_CARRIER:
        return starmm_simt_launch_pair(path, sp, grid, sms, s);
    default:
        return starmm_simt_launch_min(path, sp, grid, sms, s);
    }
}

extern "C" {

int starmm_abi_version(void) { return STARMM_ABI_VERSION; }

const char* starmm_strerror(int status) {
    switch (status) {
    case STARMM_OK: return "ok";
    case STARMM_DIM_MISMATCH: return "DimMismatch: operands do not have compatible dimensions";
    case STARMM_INVALID_SPLIT: return "InvalidSplit: n must be a power of two >= base dimension";
    case STARMM_NOT_BASE_CASE: return "NotBaseCase: region is not base-sized";
    case STARMM_ALLOC_FAILURE: return "AllocFailure: device allocation failed";
    case STARMM_CONTRACT_VIOLATION: return "ContractViolation: invalid argument";
    case STARMM_ALIGNMENT_ERROR: return "AlignmentError: region not aligned to the base-tile grid";
    case STARMM_NO_ADDITIVE_INVERSE: return "NoAdditiveInverse";
    case STARMM_TOO_LARGE: return "TooLarge: problem exceeds supported size";
    case STARMM_INTERNAL_ERROR: return "InternalError";
    }
    if (status >= STARMM_CUDA_ERROR) return cudaGetErrorString((cudaError_t)(status - STARMM_CUDA_ERROR));
    return "unknown status";
}

int starmm_device_sm_count(int device) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
    return v;
}

int starmm_plan_create(starmm_plan** plan, int semiring, int algo, int alloc_mode, int64_t m,
                       int64_t n, int64_t k, int base_dim, int workers, int ksplit_log2, int device,
                       int flags) {
    if (!plan) return STARMM_CONTRACT_VIOLATION;
    *plan = nullptr;
    if (semiring < 0 || semiring > STARMM_SR_TROPICAL_I32) return STARMM_CONTRACT_VIOLATION;
    if (algo < STARMM_CO2 || algo > STARMM_STAR_STRASSEN_2) return STARMM_CONTRACT_VIOLATION;
    if (alloc_mode != STARMM_POOLED && alloc_mode != STARMM_RAW) return STARMM_CONTRACT_VIOLATION;
    if (alloc_mode == STARMM_RAW && algo != STARMM_CO3 && algo != STARMM_STRASSEN)
        return STARMM_CONTRACT_VIOLATION;                                     // registry.py:34-35
    // the fast family subtracts: rings only (registry.py:41-42)
    if (algo >= STARMM_STRASSEN && semiring != STARMM_SR_INT64 && semiring != STARMM_SR_FP64)
        return STARMM_NO_ADDITIVE_INVERSE;
    if (m < 1 || n < 1 || k < 1) return STARMM_DIM_MISMATCH;
    if (!is_pow2(base_dim) || workers < 1) return STARMM_CONTRACT_VIOLATION;          // matrix.py:44-47
    if (ksplit_log2 > 16) return STARMM_CONTRACT_VIOLATION;
    // Config.check_problem (matrix.py:57-61) unless the caller opted out.
    if (!(flags & STARMM_F_ALLOW_NONPOW2)) {
        if (!(m == n && n == k)) return STARMM_DIM_MISMATCH;
        if (!is_pow2(n) || n < base_dim) return STARMM_INVALID_SPLIT;
    }
    if (m > (1LL << 31) || n > (1LL << 31) || k > (1LL << 31)) return STARMM_TOO_LARGE;
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return STARMM_CONTRACT_VIOLATION;
    starmm_plan* P = new starmm_plan();
    P->sr = semiring; P->algo = algo; P->alloc = alloc_mode; P->base_dim = base_dim;
    P->workers = workers; P->ksplit_req = ksplit_log2; P->device = device; P->flags = flags;
    P->m = m; P->n = n; P->k = k;
    memset(&P->st, 0, sizeof(P->st));
    P->sms = starmm_device_sm_count(device);
    *plan = P;
    return STARMM_OK;
}

void starmm_plan_destroy(starmm_plan* P) {
    if (!P) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(P->device);
    cudaDeviceSynchronize();
    if (P->ev0) cudaEventDestroy(P->ev0);
    if (P->ev1) cudaEventDestroy(P->ev1);
    if (P->h_range) cudaFreeHost((void*)P->h_range);
    if (P->twin) starmm_plan_destroy(P->twin);
    P->arena.destroy();
    cudaSetDevice(prev);
    delete P;
}

int starmm_plan_reset_stats(starmm_plan* P) {
    if (!P) return STARMM_CONTRACT_VIOLATION;
    if (P->d_counters) {
        CK(cudaMemset(P->d_counters, 0, CNT__N * 8));
        CK(cudaMemset(P->d_worker_used, 0, (size_t)P->max_workers * 4));
    }
    memset(&P->st, 0, sizeof(P->st));
    P->ws_fresh = P->ws_reuse = P->ws_high_water = 0;
    P->raw_count = P->raw_bytes = 0;
    return STARMM_OK;
}

int starmm_plan_stats(starmm_plan* P, starmm_stats* out) {
    if (!P || !out) return STARMM_CONTRACT_VIOLATION;
    *out = P->st;
    unsigned long long c[CNT__N];
    memset(c, 0, sizeof(c));
    if (P->d_counters) CK(cudaMemcpy(c, P->d_counters, sizeof(c), cudaMemcpyDeviceToHost));
    out->tile_serializations = (int64_t)c[CNT_SERIALIZATIONS];
    out->pair_transitions = (int64_t)c[CNT_PAIR_TRANSITIONS];
    out->lazy_temp_acquires = (int64_t)c[CNT_LAZY_ACQUIRES];
    out->pool_fresh_count = (int64_t)c[CNT_POOL_FRESH] + P->ws_fresh;
    out->pool_reuse_count = (int64_t)(c[CNT_POOL_ACQUIRES] - c[CNT_POOL_FRESH]) + P->ws_reuse;
    out->pool_high_water_bytes = std::max<int64_t>((int64_t)c[CNT_POOL_HIGH_WATER], P->ws_high_water);
    out->pool_total_allocated_bytes = P->arena.total_allocated;
    out->raw_alloc_count = P->raw_count;
    out->raw_alloc_bytes = P->raw_bytes;
    return STARMM_OK;
}

static int execute_impl(starmm_plan* P, void* C, int64_t ldc, const void* A, int64_t lda,
                        const void* B, int64_t ldb, void* stream, bool force_async) {
    if (!P || !C || !A || !B) return STARMM_CONTRACT_VIOLATION;
    if (ldc < P->n || lda < P->k || ldb < P->n) return STARMM_DIM_MISMATCH;
    const int eb = elem_bytes(P->sr);
    if (((uintptr_t)C | (uintptr_t)A | (uintptr_t)B) % eb) return STARMM_ALIGNMENT_ERROR;
    int prev_dev = 0;
    CK(cudaGetDevice(&prev_dev));
    if (prev_dev != P->device) CK(cudaSetDevice(P->device));
    cudaStream_t s = (cudaStream_t)stream;
    TRY(ensure_bookkeeping(P));
    const bool init_identity = (P->flags & STARMM_F_INIT_IDENTITY) != 0;
    const bool fast_ok = !(P->flags & STARMM_F_NO_FASTPATH);
    int launches = 0;

    // ---- path selection -------------------------------------------------------
    // Range-guarded exact narrow paths are chosen optimistically: the operands are
    // packed for the fastest kernel while the packers reduce max|x| (and float
    // integrality) in the same pass; if the guard fails they are re-packed for the
    // path the observed range allows.
    int path = 0;
    bool guard_pending = false;
    if (P->sr == STARMM_SR_FP64) {
        // opt-in Ozaki-II emulation on the int8 tensor cores; the guard
        // (finite inputs) runs in the same pass that finds the per-row/column scales
        if (fast_ok && (P->flags & STARMM_F_FP64_EMU) && P->k < (1LL << 17)) {
            path = PATH_OZAKI_F64;
            guard_pending = true;
        } else {
            path = PATH_DMMA_F64;
        }
    }
    else if (P->sr == STARMM_SR_TROPICAL_F64) { path = fast_ok ? PATH_SIMT_F64T_S16X2 : PATH_SIMT_F64_MIN; guard_pending = fast_ok; }
    else if (P->sr == STARMM_SR_TROPICAL_F32) { path = fast_ok ? PATH_SIMT_F32_S16X2 : PATH_SIMT_F32_PAIR; guard_pending = fast_ok; }
    else if (P->sr == STARMM_SR_INT64) {
        path = fast_ok ? ((P->flags & STARMM_F_INT_TENSOR) ? PATH_TC_I8 : PATH_SIMT_I64_DP4A) : PATH_SIMT_I64;
        guard_pending = fast_ok;
    }
    else { path = fast_ok ? PATH_SIMT_I32_S16X2 : PATH_SIMT_I32_SAT; guard_pending = fast_ok; }
    // the previous execute's guard outcome is the better first guess (data ranges are
    // usually stable across calls); the guard itself still runs on every call
    if (guard_pending && P->last_guarded_path && P->sr != STARMM_SR_FP64) path = P->last_guarded_path;

    // geometry of the chosen path (re-derived if the guard changes the path)
    bool is_dmma = false;
    PathShape shape;
    int BK = 0, TBM = 0, TBN = 0, per_sm = 1, gpu_workers = 0, s_log2 = 0, S = 1, tar_levels = 0;
    bool balanced = false;
    long long tiles_m = 0, tiles_n = 0, tiles = 0, Mp = 0, Np = 0, Kp = 0, kslice = 0, ntasks = 0;
    TaskGrid g;
    auto plan_geometry = [&]() -> int {
        is_dmma = (path == PATH_DMMA_F64);
        shape = path_shape(path);
        BK = shape.bk; TBM = shape.bm; TBN = shape.bn; per_sm = shape.per_sm;
        tiles_m = (P->m + TBM - 1) / TBM; tiles_n = (P->n + TBN - 1) / TBN;
        tiles = tiles_m * tiles_n;
        gpu_workers = P->sms * per_sm;                  // persistent CTAs (the GPU workers)
        balanced = false;
        const bool simt_path = !is_dmma && path != PATH_TC_I8 && path != PATH_OZAKI_F64;
        const bool may_split = !(P->algo == STARMM_CO2 || path == PATH_TC_I8 || path == PATH_OZAKI_F64);
        if ((simt_path || is_dmma) && (P->ksplit_req < 0 || !may_split)) {
            // CUDA-core paths: pick (CTAs per SM, split depth) by a wave cost model
            //   time ~ ceil(tasks / CTAs) * (stages per task + overhead) / per-CTA rate
            // overhead = 4.5 stages of prologue/epilogue per task, plus the split write-back
            // (atomics: 2 stages; the CAS loop of the float minima: 20).  The kernels are
            // compiled for two CTAs per SM; launched at one per SM they run at 0.89 of a
            // full SM (tools/ksplit_ab.py, profiles/r01i_ksplit_c2.json).  Small problems
            // such as config 2 (1024 tiles = 3.46 waves of 296 CTAs) then prefer one CTA
            // per SM (co2: +5.5%) or a split to two.  co2 never splits (classic.py:125-128).
            // The split write-back's cost depends on the schedule's protocol (tools/ksplit_ab.py,
            // profiles/r01k_ksplit_*.json; DMMA n=2048: S=2/4 cost +6%/+1.6% for tar -- which the
            // model reproduces -- and +30%/+48% for sar): TAR atomic-madd 2 stages (20 for the CAS
            // of float minima), CO3 workspace + merge 3, SAR pair states + locks + lazy
            // temporaries 60 on DMMA (the sibling folds serialise under the tile lock; n=1024:
            // +40% at S=2) and 16 on the CUDA-core paths (2-4x longer stages, batched folds;
            // int64 n=1024: S=2 cost +23%);
            // STAR levels above switch_depth are TAR, deeper ones SAR.  The DMMA path always
            // runs two CTAs per SM.
            const bool cas_min = P->sr == STARMM_SR_TROPICAL_F32 || P->sr == STARMM_SR_TROPICAL_F64;
            const double pen_tar = cas_min ? 20.0 : 2.0, pen_sar = is_dmma ? 60.0 : 16.0;
            // (the SAR folds of one tile serialise under its lock: cost grows with the 2^sl
            // slices per tile -- tropical n=1024, S=8: -27% vs co2 with a flat penalty)
            auto split_pen = [&](int sl) -> double {
                if (sl == 0) return 0.0;
                const double sar = pen_sar * (double)(1 << sl) / 2.0;
                switch (P->algo) {
                case STARMM_TAR: return pen_tar;
                case STARMM_CO3: return 3.0;
                case STARMM_SAR: return sar;
                default: return sl <= switch_depth(P->workers) ? pen_tar : sar;   // star
                }
            };
            const double kst = (double)round_up(P->k, BK) / BK;
            int smax = 0;
            if (may_split)
                while (smax < 6 && (P->k >> (smax + 1)) >= std::max(P->base_dim, BK) &&
                       (tiles << smax) < 8LL * gpu_workers)
                    ++smax;
            double best = 0;
            int best_occ = per_sm, best_s = 0;
            for (int occ = per_sm; occ >= (is_dmma ? per_sm : 1); --occ) {
                const bool occ1_build = path == PATH_SIMT_I64_DP4A || path == PATH_SIMT_F32_PAIR ||
                                        path == PATH_SIMT_I32_CARRIER || path == PATH_SIMT_F64T_CARRIER ||
                                        path == PATH_SIMT_F32_S16X2 || path == PATH_SIMT_I32_S16X2 ||
                                        path == PATH_SIMT_F64T_S16X2;                // has_occ1_build
                const double rate1 = occ1_build ? 0.97 : 0.89;
                const double rate = occ == 1 ? (per_sm == 1 ? 1.0 : rate1) : 1.0 / occ;
                for (int sl = 0; sl <= smax; ++sl) {
                    const double waves = std::ceil((double)(tiles << sl) / ((double)P->sms * occ));
                    const double ovh = 4.5 + split_pen(sl);
                    const double c = waves * (kst / (double)(1 << sl) + ovh) / rate;
                    if (best == 0 || c < 0.99 * best) { best = c; best_occ = occ; best_s = sl; }
                }
            }
            // Balanced slices (TAR with uneven k-slices, "stream-K"): every worker gets the
            // same share of the flattened (tile, k-stage) space, pieces of shared tiles merge
            // with the atomic-madd.  Only for tar/star (their split write-back IS the
            // atomic-madd) and exact, cheap atomics (int64 red.add, int32 red.min).
            const char* benv = getenv("STARMM_NO_BALANCED");
            if (simt_path && may_split && (P->algo == STARMM_TAR || P->algo == STARMM_STAR) &&
                (P->sr == STARMM_SR_INT64 || P->sr == STARMM_SR_TROPICAL_I32) &&
                P->remote_parts == 0 && !(benv && benv[0] == '1')) {
                const double Gw = (double)P->sms * per_sm;
                const double c = ((double)tiles * (kst + 4.5) + Gw * (4.5 + 2.0)) / Gw * per_sm;
                if (c < 0.97 * best) { balanced = true; best_occ = per_sm; best_s = 0; }
            }
            per_sm = best_occ;
            gpu_workers = P->sms * per_sm;
            s_log2 = best_s;
        } else if (!may_split) {
            s_log2 = 0;            // k-halves serialised (classic.py:125-128): never split
                                   // (the opt-in tensor path keeps whole-K tiles too)
        } else if (P->ksplit_req >= 0) {
            s_log2 = P->ksplit_req;
        } else {
            // (the opt-in tcgen05 paths never reach here: they keep whole-K tiles)
            s_log2 = 0;
        }
        // a k-slice is at least one leaf (base_dim) and one k-stage; never more levels
        // than the recursion has (log2(k / b))
        while (s_log2 > 0 && ((P->k >> s_log2) < std::max(P->base_dim, BK) || (P->k >> s_log2) < 1))
            --s_log2;
        S = 1 << s_log2;
        tar_levels = 0;
        if (P->algo == STARMM_TAR) tar_levels = s_log2;
        if (P->algo == STARMM_STAR) tar_levels = std::min(switch_depth(P->workers), s_log2);
        Mp = tiles_m * TBM; Np = tiles_n * TBN;
        Kp = round_up(P->k, std::max<long long>(32, (long long)BK * S));
        kslice = Kp / S;
        g.tiles_m = (int)tiles_m; g.tiles_n = (int)tiles_n; g.S = S; g.log2S = s_log2;
        g.tar_levels = tar_levels; g.kslice = kslice;
        // raster groups sized so one wave of resident CTAs covers a near-square block of
        // tiles (minimises the A+B panels live in L2; tools/gsweep.sh: -42% DRAM bytes)
        g.group_m = is_dmma ? 4 : 12;   // DMMA: 4 x 256 rows (58 GB vs 61 GB at 6), SIMT 12 x 128
        g.balanced = balanced ? 1 : 0;
        g.kstages = Kp / std::max(1, BK);
        ntasks = tiles * S;
        if (ntasks > (1LL << 31) - 1) return STARMM_TOO_LARGE;
        g.num_tasks = (int)ntasks;
        return STARMM_OK;
    };

    // ---- staging buffers from the arena (not counted as algorithm temps) ----
    std::vector<Block> staged;
    auto stage_acquire = [&](size_t bytes, void** p) -> int {
        long long fr = 0, ru = 0;
        TRY(P->arena.acquire(bytes, p, false, &fr, &ru));
        staged.push_back({*p, bytes});
        return STARMM_OK;
    };
    int rc = STARMM_OK;
    unsigned long long *oz_rowmax = nullptr, *oz_colmax = nullptr;
    const void* opA = A; const void* opB = B;
    long long olda = lda, oldb = ldb;
    do {
      for (;;) {
        if ((rc = plan_geometry())) break;
        opA = A; opB = B; olda = lda; oldb = ldb;     // a re-plan starts from the caller's operands
        unsigned long long* rng = guard_pending ? P->d_range : nullptr;
        if (rng && (rc = cuda_status(cudaMemsetAsync(rng, 0, 2 * sizeof(unsigned long long), s)))) break;
        if (is_dmma) {
            bool direct = (P->m % TBM == 0) && (P->n % TBN == 0) && (P->k == Kp) &&
                          (((uintptr_t)A | (uintptr_t)B) % 16 == 0) && (lda % 2 == 0) && (ldb % 2 == 0);
            if (!direct) {
                void *pa, *pb;
                if ((rc = stage_acquire((size_t)(Mp * Kp * 8), &pa))) break;
                if ((rc = stage_acquire((size_t)(Kp * Np * 8), &pb))) break;
                pad_copy_kernel<double><<<grid2d(Mp, Kp), 256, 0, s>>>((const double*)A, P->m, P->k,
                                                                            lda, (double*)pa, Mp, Kp);
                pad_copy_kernel<double><<<grid2d(Kp, Np), 256, 0, s>>>((const double*)B, P->k, P->n,
                                                                            ldb, (double*)pb, Kp, Np);
                if ((rc = cuda_status(cudaGetLastError()))) break;
                launches += 2;
                opA = pa; opB = pb; olda = Kp; oldb = Np;
            }
        } else {
            void *pa, *pb;
            if ((rc = stage_acquire((size_t)(Mp * Kp * shape.a_bytes_per_km / 1000), &pa))) break;
            if ((rc = stage_acquire((size_t)(Kp * Np * shape.b_bytes_per_kn / 1000), &pb))) break;
            const float finf = std::numeric_limits<float>::infinity();
            const unsigned s16pad = 16383u | (16383u << 16);
            switch (path) {
            case PATH_SIMT_F32_PAIR:
                rc = launch_pack<float, float, 2, ConvIdentity>(A, lda, B, ldb, P->m, P->n, P->k, pa, pb,
                                                                 Mp, Np, Kp, finf, s, rng); break;
            case PATH_SIMT_I32_CARRIER:
                rc = launch_pack<int, float, 2, ConvI32ToF32>(A, lda, B, ldb, P->m, P->n, P->k, pa, pb,
                                                               Mp, Np, Kp, finf, s, rng); break;
            case PATH_SIMT_I32_VMIN:
                rc = launch_pack<int, int, 1, ConvI32Vmin>(A, lda, B, ldb, P->m, P->n, P->k, pa, pb, Mp,
                                                            Np, Kp, (1 << 30) - 1, s, rng); break;
            case PATH_SIMT_I32_SAT:
                rc = launch_pack<int, int, 1, ConvIdentity>(A, lda, B, ldb, P->m, P->n, P->k, pa, pb, Mp,
                                                             Np, Kp, 0x7fffffff, s, rng); break;
            case PATH_SIMT_I64:
                rc = launch_pack<long long, long long, 1, ConvIdentity>(A, lda, B, ldb, P->m, P->n, P->k,
                                                                         pa, pb, Mp, Np, Kp, 0LL, s, rng); break;
            case PATH_SIMT_I64_NARROW:
                rc = launch_pack<long long, int, 1, ConvI64ToI32>(A, lda, B, ldb, P->m, P->n, P->k, pa, pb,
                                                                   Mp, Np, Kp, 0, s, rng); break;
            case PATH_SIMT_F64_MIN: {
                const double dinf = std::numeric_limits<double>::infinity();
                rc = launch_pack<double, double, 1, ConvIdentity>(A, lda, B, ldb, P->m, P->n, P->k, pa,
                                                                   pb, Mp, Np, Kp, dinf, s, rng); break;
            }
            case PATH_SIMT_I64_DP4A:
                pack_a_s8x4_kernel<<<dim3((unsigned)((Kp / 4 + 31) / 32), (unsigned)(Mp / 32)), dim3(32, 8), 0, s>>>(
                    (const long long*)A, P->m, P->k, lda, (int*)pa, Mp, Kp, rng);
                pack_b_s8x4_kernel<<<grid2d(Kp / 4, Np / 2), 256, 0, s>>>(
                    (const long long*)B, P->k, P->n, ldb, (int*)pb, Np, Kp, rng);
                rc = cuda_status(cudaGetLastError());
                break;
            case PATH_TC_I8:
                pack_i8_rows_kernel<<<dim3((unsigned)((Kp / 8 + 255) / 256), (unsigned)std::min<long long>(Mp, 4096)), 256, 0, s>>>(
                    (const long long*)A, P->m, P->k, lda, (signed char*)pa, Mp, Kp, rng);
                pack_i8_transpose_kernel<<<dim3((unsigned)(Np / 32), (unsigned)((Kp + 127) / 128)), dim3(32, 8), 0, s>>>(
                    (const long long*)B, P->k, P->n, ldb, (signed char*)pb, Np, Kp, rng);
                rc = cuda_status(cudaGetLastError());
                break;
            case PATH_OZAKI_F64: {
                // scale pass (and the finiteness guard); residues are packed after it
                if ((rc = stage_acquire((size_t)Mp * 8, (void**)&oz_rowmax))) break;
                if ((rc = stage_acquire((size_t)Np * 8, (void**)&oz_colmax))) break;
                if ((rc = cuda_status(cudaMemsetAsync(oz_colmax, 0, (size_t)Np * 8, s)))) break;
                const int wpb = 8;
                oz_amax_rows_kernel<<<(unsigned)std::min<long long>((P->m + wpb - 1) / wpb, 148LL * 16), 32 * wpb, 0, s>>>(
                    (const double*)A, P->m, P->k, lda, oz_rowmax, rng + 1);
                oz_amax_cols_kernel<<<dim3((unsigned)((P->n + 31) / 32), (unsigned)((P->k + 255) / 256)), dim3(32, 8), 0, s>>>(
                    (const double*)B, P->k, P->n, ldb, oz_colmax, rng + 1);
                rc = cuda_status(cudaGetLastError());
                break;
            }
            case PATH_SIMT_F64T_CARRIER:
                rc = launch_pack<double, float, 2, ConvF64ToF32>(A, lda, B, ldb, P->m, P->n, P->k, pa, pb,
                                                                  Mp, Np, Kp, finf, s, rng); break;
            case PATH_SIMT_F32_S16X2:
            case PATH_SIMT_I32_S16X2:
            case PATH_SIMT_F64T_S16X2: {
                dim3 ga((unsigned)(Kp / 32), (unsigned)(Mp / 32));
                if (path == PATH_SIMT_F64T_S16X2) {
                    pack_a_kernel<double, unsigned, 1, ConvS16Dup><<<ga, dim3(32, 8), 0, s>>>(
                        (const double*)A, P->m, P->k, lda, (unsigned*)pa, Mp, Kp, s16pad, rng);
                    pack_b_s16x2_kernel<double><<<grid2d(Kp, Np / 2), 256, 0, s>>>(
                        (const double*)B, P->k, P->n, ldb, (unsigned*)pb, Np, Kp, rng);
                } else if (path == PATH_SIMT_F32_S16X2) {
                    pack_a_kernel<float, unsigned, 1, ConvS16Dup><<<ga, dim3(32, 8), 0, s>>>(
                        (const float*)A, P->m, P->k, lda, (unsigned*)pa, Mp, Kp, s16pad, rng);
                    pack_b_s16x2_kernel<float><<<grid2d(Kp, Np / 2), 256, 0, s>>>(
                        (const float*)B, P->k, P->n, ldb, (unsigned*)pb, Np, Kp, rng);
                } else {
                    pack_a_kernel<int, unsigned, 1, ConvS16Dup><<<ga, dim3(32, 8), 0, s>>>(
                        (const int*)A, P->m, P->k, lda, (unsigned*)pa, Mp, Kp, s16pad, rng);
                    pack_b_s16x2_kernel<int><<<grid2d(Kp, Np / 2), 256, 0, s>>>(
                        (const int*)B, P->k, P->n, ldb, (unsigned*)pb, Np, Kp, rng);
                }
                rc = cuda_status(cudaGetLastError());
                break;
            }
            }
            if (rc) break;
            launches += 2;
            opA = pa; opB = pb;
        }
        if (!guard_pending) break;
        // ---- the fused guard: decide the exact path the observed range allows ----
        unsigned long long h[2];
        publish_range_kernel<<<1, 32, 0, s>>>(P->d_range, P->h_range_dev);
        if ((rc = cuda_status(cudaGetLastError()))) break;
        if ((rc = cuda_status(cudaStreamSynchronize(s)))) break;
        h[0] = P->h_range[0];
        h[1] = P->h_range[1];
        ++launches;
        guard_pending = false;
        const unsigned long long mx = h[0];
        const bool bad = h[1] != 0;
        int actual = path;
        if (P->sr == STARMM_SR_FP64) {
            actual = bad ? PATH_DMMA_F64 : PATH_OZAKI_F64;   // NaN / inf: IEEE semantics via DMMA
        } else if (P->sr == STARMM_SR_INT64) {
            // exact iff every int32 partial sum fits: K * max|a| * max|b| < 2^31
            long double bound = (long double)P->k * (long double)mx * (long double)mx;
            if (mx <= 127 && bound < 2147483648.0L)
                actual = (P->flags & STARMM_F_INT_TENSOR) ? PATH_TC_I8 : PATH_SIMT_I64_DP4A;
            else if (mx < (1ull << 31) && bound < 2147483648.0L) actual = PATH_SIMT_I64_NARROW;
            else actual = PATH_SIMT_I64;
        } else if (P->sr == STARMM_SR_TROPICAL_F64) {
            // integer-valued float64: int16 when |x| <= 4096, else fp32 carrier while all
            // sums stay below 2^24 (exact), else the float64 kernel
            if (!bad && mx <= (unsigned long long)S16_FINITE_MAX) actual = PATH_SIMT_F64T_S16X2;
            else if (!bad && mx <= (1ull << 23)) actual = PATH_SIMT_F64T_CARRIER;
            else actual = PATH_SIMT_F64_MIN;
        } else if (P->sr == STARMM_SR_TROPICAL_F32) {
            // integer-valued with |x| <= 4096: int16 sums cannot overflow, exact
            actual = (!bad && mx <= (unsigned long long)S16_FINITE_MAX) ? PATH_SIMT_F32_S16X2
                                                                         : PATH_SIMT_F32_PAIR;
        } else {
            if (mx <= (unsigned long long)S16_FINITE_MAX) actual = PATH_SIMT_I32_S16X2;   // int16 exact
            else if (mx <= (1ull << 23)) actual = PATH_SIMT_I32_CARRIER;                 // fp32-exact sums
            else if (mx < (1ull << 28)) actual = PATH_SIMT_I32_VMIN;                     // no overflow
            else actual = PATH_SIMT_I32_SAT;
        }
        P->last_guarded_path = actual;
        if (actual == path) break;
        path = actual;                  // re-pack for the path the range allows
      }
      if (rc) break;
        if (path == PATH_OZAKI_F64) {   // residue planes for the scales the guard pass found
            const int t = ozaki_bits(P->k);
            oz_pack_rows_kernel<<<dim3((unsigned)((Kp / 4 + 255) / 256), (unsigned)std::min<long long>(Mp, 65535)), 256, 0, s>>>(
                (const double*)A, P->m, P->k, lda, oz_rowmax, t, (signed char*)opA, Mp, Kp);
            oz_pack_cols_kernel<<<dim3((unsigned)(Np / 32), (unsigned)(Kp / 64)), dim3(32, 8), 0, s>>>(
                (const double*)B, P->k, P->n, ldb, oz_colmax, t, (signed char*)opB, Np, Kp);
            if ((rc = cuda_status(cudaGetLastError()))) break;
            launches += 2;
        }

        // ---- per-run protocol state: slots (TileExclusionTable), pair states ----
        const bool need_slots = (S > 1) && (P->algo == STARMM_SAR || P->algo == STARMM_STAR);
        void* pstate = nullptr;
        size_t state_bytes = need_slots ? (size_t)(tiles + tiles * (S / 2)) * 4 : 0;
        if (need_slots) {
            if ((rc = stage_acquire(state_bytes, &pstate))) break;
            if ((rc = cuda_status(cudaMemsetAsync(pstate, 0, state_bytes, s)))) break;
        }
        // per-worker lazy-temp blocks (tile sized, for SAR/STAR pairs)
        void* wscratch = nullptr;
        const long long tile_elems = (long long)TBM * TBN;
        if (need_slots) {
            if ((rc = stage_acquire((size_t)(gpu_workers * tile_elems * eb), &wscratch))) break;
        }
        // co3 workspace D_1..D_{S-1}: pooled (arena, reused) or raw (fresh per call)
        void* W = nullptr;
        size_t wbytes = 0;
        if (P->algo == STARMM_CO3 && S > 1) {
            wbytes = (size_t)(S - 1) * (size_t)P->m * (size_t)P->n * eb;
            if (P->alloc == STARMM_POOLED) {
                if ((rc = P->arena.acquire(wbytes, &W, true, &P->ws_fresh, &P->ws_reuse))) break;
                staged.push_back({W, wbytes});
            } else {
                if ((rc = cuda_status(cudaMallocAsync(&W, wbytes, s)))) break;
                ++P->raw_count;
                P->raw_bytes += (long long)wbytes;
            }
            P->ws_high_water = std::max<long long>(P->ws_high_water, (long long)wbytes);
        }
        if (init_identity && (S > 1 || balanced) && P->algo != STARMM_CO3 && P->remote_parts == 0) {
            if ((rc = fill_dispatch(P->sr, C, P->m, P->n, ldc, s))) break;
            ++launches;
        }

        WbParams w;
        w.mode_base = P->algo; w.init_identity = init_identity ? 1 : 0;
        w.C = C; w.ldc = ldc; w.M = P->m; w.N = P->n;
        w.W = W; w.ldw = P->n; w.wstride = P->m * P->n;
        w.slots = (int*)pstate;
        w.pairs = pstate ? (int*)pstate + tiles : nullptr;
        w.counters = P->d_counters; w.worker_used = P->d_worker_used;
        w.scratch = wscratch; w.scratch_elems = tile_elems;
        w.remote_parts = P->remote_parts; w.remote_rows = P->remote_rows; w.remote_ld = P->remote_ld;
        for (int i = 0; i < 8; ++i) w.remote_base[i] = P->remote_base[i];

        int grid = occupancy_grid(P, per_sm, balanced ? ntasks * g.kstages : ntasks);
        const bool timed = (P->flags & STARMM_F_TIME_MAIN) != 0;
        if (timed) {
            if (!P->ev0) {
                if ((rc = cuda_status(cudaEventCreate(&P->ev0)))) break;
                if ((rc = cuda_status(cudaEventCreate(&P->ev1)))) break;
            }
            if ((rc = cuda_status(cudaEventRecord(P->ev0, s)))) break;
        }
        if (path == PATH_TC_I8) {
            EpiFoldI64 e;
            e.o = tcg_out(P, C, ldc, init_identity);
            rc = launch_tcg(opA, opB, Mp, Np, Kp, 1, e, P->sms, s, stage_acquire);
        } else if (path == PATH_OZAKI_F64) {
            void* planes = nullptr;
            if ((rc = stage_acquire((size_t)oz::P * Mp * Np, &planes))) break;
            EpiOzakiResidues e;
            e.R = (unsigned char*)planes; e.Mp = Mp; e.Np = Np;
            if ((rc = launch_tcg(opA, opB, Mp, Np, Kp, oz::P, e, P->sms, s, stage_acquire))) break;
            if (timed && (rc = cuda_status(cudaEventRecord(P->ev1, s)))) break;
            const long long groups = (P->n + OZ_CRT_W - 1) / OZ_CRT_W;
            oz_crt_kernel<<<dim3((unsigned)((groups + 127) / 128), (unsigned)std::min<long long>(P->m, 65535)), 128, 0, s>>>(
                (const unsigned char*)planes, Mp, Np, oz_rowmax, oz_colmax, ozaki_bits(P->k), ozaki_crt(),
                tcg_out(P, C, ldc, init_identity));
            rc = cuda_status(cudaGetLastError());
            ++launches;
        } else if (is_dmma) {
            DmmaParams dp;
            dp.A = (const double*)opA; dp.lda = olda; dp.B = (const double*)opB; dp.ldb = oldb;
            dp.g = g; dp.w = w;
            dp.gate = P->d_gate;
            // Wave gate: off by default since the one-CTA-per-SM 256x64 kernel keeps its
            // persistent CTAs close enough on its own (58 GB of DRAM reads per n=16384
            // launch without, 53 GB with, at -0.1..0.3%; the two-CTA 64x128 kernel needed
            // it: 250 -> 51 GB).  STARMM_DMMA_GATE=1 turns it on; it needs the whole grid
            // co-resident and pays only over several waves, and the host path's
            // overlapping launches never use it.
            const char* genv = getenv("STARMM_DMMA_GATE");
            const bool gate = genv && genv[0] == '1' && P->dmma_gate && ntasks >= 4LL * grid;
            rc = launch_dmma(dp, grid, gate, s);
        } else {
            SimtParams sp;
            sp.Ap = opA; sp.Bp = opB; sp.Mp = Mp; sp.Np = Np; sp.g = g; sp.w = w;
            // the CUDA-core tile kernels are instantiated in simt_launch_*.cu (parallel build)
            rc = cuda_status((cudaError_t)starmm_simt_launch(path, sp, grid, P->sms, s));
        }
        if (rc) break;
        ++launches;
        if (timed && path != PATH_OZAKI_F64) {   // (the Ozaki path records it after its GEMM)
            if ((rc = cuda_status(cudaEventRecord(P->ev1, s)))) break;
        }

        // ---- co3: merge the workspace bottom-up (merge_tasks, ops.py:108-155) ----
        if (P->algo == STARMM_CO3 && S > 1) {
            const long long slab = P->m * P->n;
            for (int lvl = s_log2; lvl >= 1 && !rc; --lvl) {
                int step = 1 << (s_log2 - lvl);
                for (int x = step; x < S && !rc; x += 2 * step) {
                    char* src = (char*)W + (size_t)(x - 1) * slab * eb;
                    int tgt = x - step;
                    if (tgt == 0) rc = madd_dispatch(P->sr, C, ldc, src, P->n, P->m, P->n, 0, s);
                    else rc = madd_dispatch(P->sr, (char*)W + (size_t)(tgt - 1) * slab * eb, P->n, src,
                                            P->n, P->m, P->n, 0, s);
                    ++launches;
                }
            }
            if (rc) break;
            if (P->alloc == STARMM_RAW) {
                if ((rc = cuda_status(cudaFreeAsync(W, s)))) break;
            }
        }
    } while (0);

    // staging buffers go back to their LIFO stacks; stream order protects reuse
    for (auto it = staged.rbegin(); it != staged.rend(); ++it) P->arena.release(it->p, it->bytes);
    if (rc) return rc;
    if (!(P->flags & STARMM_F_ASYNC) && !force_async) CK(cudaStreamSynchronize(s));
    if (P->flags & STARMM_F_TIME_MAIN) {
        CK(cudaEventSynchronize(P->ev1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, P->ev0, P->ev1));
        P->st.main_kernel_ns += (int64_t)((double)ms * 1e6);
        P->st.main_kernel_launches += 1;
    }

    P->st.tasks = ntasks;
    P->st.workers = std::min<long long>(ntasks, (long long)P->sms * per_sm);
    P->st.ksplit = S;
    P->st.balanced_workers = balanced ? std::min<long long>(ntasks * g.kstages, (long long)P->sms * per_sm) : 0;
    P->st.tar_levels = tar_levels;
    P->st.kernel_launches = launches;
    P->st.path = path;
    P->st.executes += 1;
    if (S > 1 && (P->algo == STARMM_SAR || P->algo == STARMM_STAR) && tar_levels < s_log2)
        P->st.pair_count += tiles * (S / 2);
    if (prev_dev != P->device) cudaSetDevice(prev_dev);
    return STARMM_OK;
}

// ============================================================================
// The Strassen family (strassen.py:1-235): C <- A (x) B over a ring, overwriting C.
// One building block, mm(C, A, B, mode) with mode = store / add / sub, recursed on the
// host; leaves are the tile kernels (CO2 plan on the sub-problem), operand sums and
// the signed assembly are ring_combine kernels.  The variants differ in temporaries
// exactly as the reference: the straightforward step materialises every operand sum
// and all seven products (<= 17 half-size blocks per level); the sar step owns three
// LIFO-reused blocks (S, T, P) and merges each product into the quadrants it feeds;
// star-strassen-1 runs classical 8-way levels above switch_depth(workers), -2 runs
// straightforward levels there; both use the sar step below.
namespace {

struct Combo { int r1, c1, op, r2, c2; };   // op: 0 bare quadrant, +1 add, -1 sub
// strassen.py:30-47
const Combo S_DEFS[8] = {{0, 0, 0, 0, 0}, {0, 0, 1, 1, 1}, {1, 0, 1, 1, 1}, {0, 0, 0, 0, 0},
                         {1, 1, 0, 0, 0}, {0, 0, 1, 0, 1}, {1, 0, -1, 0, 0}, {0, 1, -1, 1, 1}};
const Combo T_DEFS[8] = {{0, 0, 0, 0, 0}, {0, 0, 1, 1, 1}, {0, 0, 0, 0, 0}, {0, 1, -1, 1, 1},
                         {1, 0, -1, 0, 0}, {1, 1, 0, 0, 0}, {0, 0, 1, 0, 1}, {1, 0, 1, 1, 1}};
struct Term { int r, sign; };
// strassen.py:49-54 (C_FORMULAS), indexed [qi][qj]
const Term C_FORM[2][2][4] = {{{{1, 1}, {4, 1}, {5, -1}, {7, 1}}, {{3, 1}, {5, 1}, {0, 0}, {0, 0}}},
                              {{{2, 1}, {4, 1}, {0, 0}, {0, 0}}, {{1, 1}, {3, 1}, {2, -1}, {6, 1}}}};
enum MmMode { MM_STORE = 0, MM_ADD = 1, MM_SUB = 2 };

struct StrCtx {
    starmm_plan* P;
    cudaStream_t s;
    size_t eb;
    long long leaf;
    int k_switch;
    int launches;
};

char* quad(const void* base, long long ld, int i, int j, long long h, size_t eb) {
    return (char*)base + (size_t)((i * h) * ld + j * h) * eb;
}

int ring_combine(StrCtx& x, void* D, long long ldd, const void* X, long long ldx, const void* Y,
                 long long ldy, long long n, int beta, int ax, int ay) {
    const dim3 blocks = grid2d(n, n);
    if (x.P->sr == STARMM_SR_INT64)
        ring_combine_kernel<long long><<<blocks, 256, 0, x.s>>>((long long*)D, ldd, (const long long*)X,
                                                               ldx, (const long long*)Y, ldy, n, n,
                                                               beta, ax, ay);
    else
        ring_combine_kernel<double><<<blocks, 256, 0, x.s>>>((double*)D, ldd, (const double*)X, ldx,
                                                            (const double*)Y, ldy, n, n, beta, ax, ay);
    ++x.launches;
    return cuda_status(cudaGetLastError());
}

int str_acquire(StrCtx& x, long long n, void** out) {
    size_t bytes = (size_t)(n * n) * x.eb;
    if (x.P->alloc == STARMM_RAW) {
        CK(cudaMallocAsync(out, bytes, x.s));
        ++x.P->raw_count;
        x.P->raw_bytes += (long long)bytes;
    } else {
        TRY(x.P->arena.acquire(bytes, out, true, &x.P->ws_fresh, &x.P->ws_reuse));
    }
    x.P->str_issued += (long long)bytes;
    x.P->ws_high_water = std::max(x.P->ws_high_water, x.P->str_issued);
    return STARMM_OK;
}

void str_release(StrCtx& x, void* p, long long n) {
    size_t bytes = (size_t)(n * n) * x.eb;
    if (x.P->alloc == STARMM_RAW) cudaFreeAsync(p, x.s);
    else x.P->arena.release(p, bytes);   // LIFO: the next same-size acquire gets it back
    x.P->str_issued -= (long long)bytes;
}

// leaf: the classical tile kernel on an n x n sub-problem (CO2 protocol)
int str_leaf(StrCtx& x, int mode, void* C, long long ldc, const void* A, long long lda,
             const void* B, long long ldb, long long n) {
    starmm_plan* P = x.P;
    const int sv_algo = P->algo, sv_flags = P->flags, sv_alloc = P->alloc;
    const long long sv_m = P->m, sv_n = P->n, sv_k = P->k;
    void* tmp = nullptr;
    int rc = STARMM_OK;
    if (mode == MM_SUB && (rc = str_acquire(x, n, &tmp))) return rc;
    P->algo = STARMM_CO2; P->alloc = STARMM_POOLED;
    P->m = P->n = P->k = n;
    P->flags = (sv_flags | STARMM_F_ALLOW_NONPOW2) & ~STARMM_F_INIT_IDENTITY;
    if (mode != MM_ADD) P->flags |= STARMM_F_INIT_IDENTITY;
    if (mode == MM_SUB) rc = execute_impl(P, tmp, n, A, lda, B, ldb, x.s, true);
    else rc = execute_impl(P, C, ldc, A, lda, B, ldb, x.s, true);
    P->algo = sv_algo; P->flags = sv_flags; P->alloc = sv_alloc;
    P->m = sv_m; P->n = sv_n; P->k = sv_k;
    ++x.launches;
    if (!rc && mode == MM_SUB) rc = ring_combine(x, C, ldc, tmp, n, nullptr, 0, n, 1, -1, 0);
    if (tmp) str_release(x, tmp, n);
    return rc;
}

int str_mm(StrCtx& x, int depth, int mode, void* C, long long ldc, const void* A, long long lda,
           const void* B, long long ldb, long long n);

// materialise operand r of `defs` from quadrants of X (bare quadrants are used in place)
int str_operand(StrCtx& x, const Combo& d, const void* X, long long ldx, long long h, void** tmp,
                const void** op, long long* ld) {
    if (d.op == 0) {
        *op = quad(X, ldx, d.r1, d.c1, h, x.eb);
        *ld = ldx;
        *tmp = nullptr;
        return STARMM_OK;
    }
    TRY(str_acquire(x, h, tmp));
    TRY(ring_combine(x, *tmp, h, quad(X, ldx, d.r1, d.c1, h, x.eb), ldx,
                     quad(X, ldx, d.r2, d.c2, h, x.eb), ldx, h, 0, 1, d.op));
    *op = *tmp;
    *ld = h;
    return STARMM_OK;
}

// straightforward step (strassen.py:77-93)
int str_straightforward(StrCtx& x, int depth, int mode, void* C, long long ldc, const void* A,
                        long long lda, const void* B, long long ldb, long long n) {
    const long long h = n / 2;
    void* tS[8] = {}; void* tT[8] = {}; void* tP[8] = {};
    const void* S[8]; const void* T[8]; long long lS[8], lT[8];
    int rc = STARMM_OK;
    for (int r = 1; r <= 7 && !rc; ++r) rc = str_operand(x, S_DEFS[r], A, lda, h, &tS[r], &S[r], &lS[r]);
    for (int r = 1; r <= 7 && !rc; ++r) rc = str_operand(x, T_DEFS[r], B, ldb, h, &tT[r], &T[r], &lT[r]);
    for (int r = 1; r <= 7 && !rc; ++r) rc = str_acquire(x, h, &tP[r]);
    for (int r = 1; r <= 7 && !rc; ++r) rc = str_mm(x, depth + 1, MM_STORE, tP[r], h, S[r], lS[r], T[r], lT[r], h);
    // assemble each output quadrant from its signed products (ops.py:170-185)
    for (int qi = 0; qi < 2 && !rc; ++qi)
        for (int qj = 0; qj < 2 && !rc; ++qj) {
            char* Cq = quad(C, ldc, qi, qj, h, x.eb);
            const Term* t = C_FORM[qi][qj];
            const int flip = (mode == MM_SUB) ? -1 : 1;
            int beta = (mode == MM_STORE) ? 0 : 1;
            for (int u = 0; u < 4 && t[u].r && !rc; u += 2) {
                const bool pair = (u + 1 < 4) && t[u + 1].r;
                rc = ring_combine(x, Cq, ldc, tP[t[u].r], h, pair ? tP[t[u + 1].r] : nullptr, h, h, beta,
                                  flip * t[u].sign, pair ? flip * t[u + 1].sign : 0);
                beta = 1;
            }
        }
    for (int r = 7; r >= 1; --r) if (tP[r]) str_release(x, tP[r], h);
    for (int r = 7; r >= 1; --r) if (tT[r]) str_release(x, tT[r], h);
    for (int r = 7; r >= 1; --r) if (tS[r]) str_release(x, tS[r], h);
    return rc;
}

// sar step (strassen.py:120-145): per product S, T, P blocks, LIFO-reused across products
int str_sar(StrCtx& x, int depth, int mode, void* C, long long ldc, const void* A, long long lda,
            const void* B, long long ldb, long long n) {
    const long long h = n / 2;
    bool virgin[2][2] = {{mode == MM_STORE, mode == MM_STORE}, {mode == MM_STORE, mode == MM_STORE}};
    int rc = STARMM_OK;
    for (int r = 1; r <= 7 && !rc; ++r) {
        void *tS = nullptr, *tT = nullptr, *tP = nullptr;
        const void *Sop, *Top;
        long long lS, lT;
        rc = str_operand(x, S_DEFS[r], A, lda, h, &tS, &Sop, &lS);
        if (!rc) rc = str_operand(x, T_DEFS[r], B, ldb, h, &tT, &Top, &lT);
        if (!rc) rc = str_acquire(x, h, &tP);
        if (!rc) rc = str_mm(x, depth + 1, MM_STORE, tP, h, Sop, lS, Top, lT, h);
        // merge into every quadrant the product feeds (C_USES, strassen.py:56-59)
        for (int qi = 0; qi < 2 && !rc; ++qi)
            for (int qj = 0; qj < 2 && !rc; ++qj)
                for (int u = 0; u < 4; ++u) {
                    const Term& t = C_FORM[qi][qj][u];
                    if (t.r != r) continue;
                    const int sign = (mode == MM_SUB ? -1 : 1) * t.sign;
                    char* Cq = quad(C, ldc, qi, qj, h, x.eb);
                    rc = ring_combine(x, Cq, ldc, tP, h, nullptr, 0, h, virgin[qi][qj] ? 0 : 1, sign, 0);
                    virgin[qi][qj] = false;   // first touch stores (virgin tiles, ops.py:57-65)
                    break;
                }
        if (tP) str_release(x, tP, h);
        if (tT) str_release(x, tT, h);
        if (tS) str_release(x, tS, h);
    }
    return rc;
}

// classical 8-way level (star-strassen-1 above the switch, classic.py:86-93)
int str_classical(StrCtx& x, int depth, int mode, void* C, long long ldc, const void* A,
                  long long lda, const void* B, long long ldb, long long n) {
    const long long h = n / 2;
    int rc = STARMM_OK;
    for (int k = 0; k < 2 && !rc; ++k)
        for (int i = 0; i < 2 && !rc; ++i)
            for (int j = 0; j < 2 && !rc; ++j) {
                int m = (k == 0) ? mode : (mode == MM_SUB ? MM_SUB : MM_ADD);
                rc = str_mm(x, depth + 1, m, quad(C, ldc, i, j, h, x.eb), ldc, quad(A, lda, i, k, h, x.eb),
                            lda, quad(B, ldb, k, j, h, x.eb), ldb, h);
            }
    return rc;
}

int str_mm(StrCtx& x, int depth, int mode, void* C, long long ldc, const void* A, long long lda,
           const void* B, long long ldb, long long n) {
    const long long h = n / 2;
    if ((n & 1) || h < x.leaf) return str_leaf(x, mode, C, ldc, A, lda, B, ldb, n);
    switch (x.P->algo) {
    case STARMM_STRASSEN: return str_straightforward(x, depth, mode, C, ldc, A, lda, B, ldb, n);
    case STARMM_SAR_STRASSEN: return str_sar(x, depth, mode, C, ldc, A, lda, B, ldb, n);
    case STARMM_STAR_STRASSEN_1:
        if (depth < x.k_switch) return str_classical(x, depth, mode, C, ldc, A, lda, B, ldb, n);
        return str_sar(x, depth, mode, C, ldc, A, lda, B, ldb, n);
    default:   // STARMM_STAR_STRASSEN_2
        if (depth < x.k_switch) return str_straightforward(x, depth, mode, C, ldc, A, lda, B, ldb, n);
        return str_sar(x, depth, mode, C, ldc, A, lda, B, ldb, n);
    }
}

int strassen_execute(starmm_plan* P, void* C, int64_t ldc, const void* A, int64_t lda, const void* B,
                     int64_t ldb, void* stream) {
    if (!P || !C || !A || !B) return STARMM_CONTRACT_VIOLATION;
    if (P->m != P->n || P->n != P->k) return STARMM_DIM_MISMATCH;
    if (ldc < P->n || lda < P->k || ldb < P->n) return STARMM_DIM_MISMATCH;
    int prev_dev = 0;
    CK(cudaGetDevice(&prev_dev));
    if (prev_dev != P->device) CK(cudaSetDevice(P->device));
    TRY(ensure_bookkeeping(P));
    StrCtx x{P, (cudaStream_t)stream, (size_t)elem_bytes(P->sr),
             std::max<long long>(P->base_dim, P->strassen_leaf), switch_depth(P->workers), 0};
    int rc = str_mm(x, 0, MM_STORE, C, ldc, A, lda, B, ldb, P->n);
    if (!rc && !(P->flags & STARMM_F_ASYNC)) rc = cuda_status(cudaStreamSynchronize(x.s));
    P->st.kernel_launches = x.launches;
    P->st.executes += 1;
    if (prev_dev != P->device) cudaSetDevice(prev_dev);
    return rc;
}

}  // namespace

int starmm_execute(starmm_plan* P, void* C, int64_t ldc, const void* A, int64_t lda, const void* B,
                   int64_t ldb, void* stream) {
    if (P && P->algo >= STARMM_STRASSEN) return strassen_execute(P, C, ldc, A, lda, B, ldb, stream);
    return execute_impl(P, C, ldc, A, lda, B, ldb, stream, false);
}

int starmm_plan_set_strassen_leaf(starmm_plan* P, int64_t leaf) {
    if (!P || leaf < 1) return STARMM_CONTRACT_VIOLATION;
    P->strassen_leaf = leaf;
    return STARMM_OK;
}

int starmm_plan_set_peers(starmm_plan* P, int nparts, void* const* bases, int64_t ld,
                          int64_t rows_per_part) {
    if (!P || nparts < 0 || nparts > 8) return STARMM_CONTRACT_VIOLATION;
    if (nparts == 0) { P->remote_parts = 0; return STARMM_OK; }
    if (!bases || rows_per_part < 1 || ld < P->n) return STARMM_CONTRACT_VIOLATION;
    if (P->algo == STARMM_CO3) return STARMM_CONTRACT_VIOLATION;   // co3 merges its own workspace
    if ((long long)nparts * rows_per_part < P->m) return STARMM_DIM_MISMATCH;
    for (int i = 0; i < nparts; ++i) {
        if (!bases[i]) return STARMM_CONTRACT_VIOLATION;
        P->remote_base[i] = bases[i];
    }
    P->remote_parts = nparts;
    P->remote_rows = rows_per_part;
    P->remote_ld = ld;
    return STARMM_OK;
}

int starmm_ipc_handle(const void* dptr, void* handle_out) {
    if (!dptr || !handle_out) return STARMM_CONTRACT_VIOLATION;
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, const_cast<void*>(dptr)));
    memcpy(handle_out, &h, sizeof(h));
    return STARMM_OK;
}

int starmm_ipc_open(const void* handle, void** dptr_out) {
    if (!handle || !dptr_out) return STARMM_CONTRACT_VIOLATION;
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    CK(cudaIpcOpenMemHandle(dptr_out, h, cudaIpcMemLazyEnablePeerAccess));
    return STARMM_OK;
}

int starmm_ipc_close(void* dptr) {
    if (!dptr) return STARMM_CONTRACT_VIOLATION;
    CK(cudaIpcCloseMemHandle(dptr));
    return STARMM_OK;
}

// Host-buffer execution.  Two phases, so that the GPU computes from
// the first uploaded megabytes and the result streams back while it still computes:
//  1. k-outer prologue: k-chunks [kb_c, kb_{c+1}) of geometrically growing width
//     (k/32, k/16, ... while they cover at most half of k).  Chunk c needs only
//     A[:, chunk] and B[chunk, :]; it runs as ONE execute over all m rows into the
//     device C (the first chunk stores, C <- A(x)B, later ones fold).  Uploads of
//     chunk c+1 overlap chunk c's compute; only chunk 0's transfer is exposed.
//  2. row blocks: block i folds the remaining k range [kq, k) into its rows, then
//     C0 (uploaded meanwhile into a staging buffer) is folded in with madd and the
//     block streams back on its own copy stream while block i+1 computes.
// (+) and min are associative and commutative, so integers and (min,+) stay
// bit-exact; fp64 sums in a different order (tolerance, as every k-split).  When
// A aliases B (square, same ld) every element is uploaded once: chunk c adds the
// "cross" of row block c (columns >= kb_c) and column block c (rows >= kb_{c+1}),
// and the bottom-right square [kq, m) x [kq, n) completes the matrix before phase 2.
// STARMM_HOST_PHASE1=0 disables phase 1 (row blocks only, C0 uploaded in place).
// streams / events / the caller's device of a host-path call, released or restored on
// every return path
struct HostRes {
    std::vector<cudaStream_t> streams;
    std::vector<cudaEvent_t> events;
    int prev_dev = -1, dev = -1;
    ~HostRes() {
        for (auto x : streams) { cudaStreamSynchronize(x); cudaStreamDestroy(x); }
        for (auto x : events) cudaEventDestroy(x);
        if (prev_dev >= 0 && prev_dev != dev) cudaSetDevice(prev_dev);
    }
    int stream(cudaStream_t* out) {
        cudaError_t e = cudaStreamCreateWithFlags(out, cudaStreamNonBlocking);
        if (e != cudaSuccess) { *out = nullptr; return cuda_status(e); }
        streams.push_back(*out);
        return STARMM_OK;
    }
    int event(cudaEvent_t* out) {
        cudaError_t e = cudaEventCreateWithFlags(out, cudaEventDisableTiming);
        if (e != cudaSuccess) { *out = nullptr; return cuda_status(e); }
        events.push_back(*out);
        return STARMM_OK;
    }
};

// Phase 1 pays only when the problem is compute-bound over PCIe: the estimated compute
// time (a nominal per-semiring B200 rate) must exceed the H2D time (50 GB/s); PCIe-bound
// problems (config 2) upload B first and run row blocks only.  STARMM_HOST_PHASE1=0/1
// forces the choice.
static double host_nominal_ops(int sr) {
    switch (sr) {
    case STARMM_SR_FP64: return 35e12;     // DMMA
    case STARMM_SR_INT64: return 100e12;   // dp4a when the range guard passes
    default: return 60e12;                 // (min,+): VIADDMNMX.S16x2 / fp32 carrier
    }
}

static int host_phase1_chunks(long long m, long long n, long long k, int sr, double h2d_bytes,
                              std::vector<long long>& kb) {
    kb.assign(1, 0);
    const char* env = getenv("STARMM_HOST_PHASE1");
    if ((env && env[0] == '0') || m < 512 || k < 512) return 0;
    const double t_mm = 2.0 * (double)m * (double)n * (double)k / host_nominal_ops(sr);
    if (!(env && env[0] == '1') && t_mm < h2d_bytes / 50e9) return 0;
    // first chunk k/64 (k >= 8192) or k/32: its upload is the exposed head of the schedule
    const long long div = (k >= 8192 && sr == STARMM_SR_FP64) ? 64 : 32;   // DMMA calls have no packing / guard
    long long w = std::max<long long>(128, round_up((k + div - 1) / div, 128)), sum = 0;
    while (sum + w <= k / 2) {
        sum += w;
        kb.push_back(sum);
        w *= 2;
    }
    return (int)kb.size() - 1;
}

// Host path of a k-split rank with the fused combine (starmm_plan_set_peers): every
// tile kernel folds its partials straight into the owners' rows over peer memory, so
// there is no local C to upload or download -- only A and B stream in, in k-chunks of
// doubling width (k/32, k/16, ...), each chunk one execute over all rows as soon as its
// operands have landed (the owners pre-load C0 and download their rows themselves).
static int execute_host_remote(starmm_plan* P, const void* A, int64_t lda, const void* B, int64_t ldb,
                               void* stream) {
    HostRes res;
    CK(cudaGetDevice(&res.prev_dev));
    res.dev = P->device;
    if (res.prev_dev != P->device) CK(cudaSetDevice(P->device));
    const size_t eb = (size_t)elem_bytes(P->sr);
    const long long m = P->m, n = P->n, k = P->k;
    std::vector<long long> kb(1, 0);
    for (long long w = std::max<long long>(128, round_up((k + 31) / 32, 128)); kb.back() < k; w *= 2)
        kb.push_back(std::min(k, kb.back() + w));
    const int nq = (int)kb.size() - 1;
    cudaStream_t cs = (cudaStream_t)stream, up = nullptr;
    TRY(res.stream(&up));
    std::vector<cudaEvent_t> ev(nq);
    for (auto& e : ev) TRY(res.event(&e));
    void *dA = nullptr, *dB = nullptr;
    long long fr = 0, ru = 0;
    const size_t a_bytes = (size_t)m * k * eb, b_bytes = (size_t)k * n * eb;
    int rc = STARMM_OK;
    const int saved_flags = P->flags;
    do {
        if ((rc = P->arena.acquire(a_bytes, &dA, false, &fr, &ru))) break;
        if ((rc = P->arena.acquire(b_bytes, &dB, false, &fr, &ru))) break;
        for (int c = 0; c < nq && !rc; ++c) {
            const long long k0 = kb[c], kc = kb[c + 1] - kb[c];
            rc = cuda_status(cudaMemcpy2DAsync((char*)dB + k0 * n * eb, n * eb, (const char*)B + k0 * ldb * eb,
                                               ldb * eb, n * eb, kc, cudaMemcpyHostToDevice, up));
            if (!rc) rc = cuda_status(cudaMemcpy2DAsync((char*)dA + k0 * eb, k * eb, (const char*)A + k0 * eb,
                                                        lda * eb, kc * eb, m, cudaMemcpyHostToDevice, up));
            if (!rc) rc = cuda_status(cudaEventRecord(ev[c], up));
        }
        if (rc) break;
        P->flags = saved_flags & ~(STARMM_F_TIME_MAIN | STARMM_F_INIT_IDENTITY);
        for (int c = 0; c < nq && !rc; ++c) {
            const long long k0 = kb[c];
            if ((rc = cuda_status(cudaStreamWaitEvent(cs, ev[c], 0)))) break;
            P->k = kb[c + 1] - k0;
            // (C is not touched: every write-back goes to the peers)
            rc = execute_impl(P, dA, n, (char*)dA + k0 * eb, k, (char*)dB + k0 * n * eb, n, cs, true);
            P->k = k;
        }
        if (rc) break;
        rc = cuda_status(cudaStreamSynchronize(cs));
    } while (0);
    P->k = k; P->flags = saved_flags;
    cudaStreamSynchronize(up);
    cudaStreamSynchronize(cs);
    if (dB) P->arena.release(dB, b_bytes);
    if (dA) P->arena.release(dA, a_bytes);
    return rc;
}

int starmm_execute_host(starmm_plan* P, void* C, int64_t ldc, const void* A, int64_t lda,
                        const void* B, int64_t ldb, void* stream, int64_t block_rows) {
    if (!P || !C || !A || !B) return STARMM_CONTRACT_VIOLATION;
    // classical schedules only (the Strassen family overwrites C; host_mm checks the same);
    // with a fused peer combine the owners' rows live on the GPUs: execute_host_remote
    if (P->algo >= STARMM_STRASSEN) return STARMM_CONTRACT_VIOLATION;
    if (ldc < P->n || lda < P->k || ldb < P->n) return STARMM_DIM_MISMATCH;
    if (P->remote_parts > 0) return execute_host_remote(P, A, lda, B, ldb, stream);
    HostRes res;
    CK(cudaGetDevice(&res.prev_dev));
    res.dev = P->device;
    if (res.prev_dev != P->device) CK(cudaSetDevice(P->device));
    const size_t eb = (size_t)elem_bytes(P->sr);
    const long long m = P->m, n = P->n, k = P->k;
    const int saved_flags = P->flags;
    const bool user_init = (saved_flags & STARMM_F_INIT_IDENTITY) != 0;   // C <- A(x)B: C0 unused
    std::vector<long long> kb;
    const bool same_ab = (A == B) && (m == k) && (n == k) && (lda == ldb);
    const double h2d = (double)eb * ((double)m * k + (same_ab ? 0.0 : (double)k * n) +
                                     ((saved_flags & STARMM_F_INIT_IDENTITY) ? 0.0 : (double)m * n));
    const int nq = host_phase1_chunks(m, n, k, P->sr, h2d, kb);
    const long long kq = kb.back();
    // phase-2 row blocks: ~2.5e11 semiring ops each (>= ~7 ms of B200 work, so per-block
    // guards / packing stay negligible), at most 16, and at least 8 (m >= 1024) or 4
    // (m >= 512) so that small, PCIe-bound problems overlap uploads, compute and downloads
    const double ops2 = 2.0 * (double)m * (double)n * (double)(k - kq);
    const long long lo_blocks = m >= 1024 ? 8 : (m >= 512 ? 4 : 1);
    const long long auto_blocks = std::max<long long>(lo_blocks, std::min<long long>(16, (long long)(ops2 / 2.5e11)));
    long long R = block_rows > 0 ? block_rows
                                 : std::max<long long>(128, round_up((m + auto_blocks - 1) / auto_blocks, 128));
    R = std::min(R, m);
    // row-block starts; with the automatic size the last block is cut in quarters so the
    // download after the final kernel (the exposed tail) is a quarter block
    std::vector<long long> bst;
    for (long long r = 0; r < m; r += R) bst.push_back(r);
    if (block_rows <= 0 && bst.size() >= 4 && R >= 512) {
        const long long last = bst.back(), q = round_up((m - last + 3) / 4, 128);
        for (long long r = last + q; r < m; r += q) bst.push_back(r);
    }
    bst.push_back(m);
    const long long nblk = (long long)bst.size() - 1;
    const bool staged_c0 = nq > 0 && !user_init;    // phase 1 owns dC, C0 goes to a staging buffer
    cudaStream_t cs = (cudaStream_t)stream;
    cudaStream_t up = nullptr, down = nullptr, cs2 = nullptr;
    TRY(res.stream(&up));
    TRY(res.stream(&down));
    // Phase-2 row blocks alternate between two compute streams so that block i+1's CTAs
    // fill the SMs block i's last partial wave leaves idle (each block is its own
    // persistent launch).  The second stream runs on a twin plan with its own arena,
    // because staging buffers are reused in stream order only.
    const char* tsenv = getenv("STARMM_HOST_ONE_STREAM");
    const bool two_streams = nblk > 1 && !(tsenv && tsenv[0] == '1');
    if (two_streams) {
        if (!P->twin) {
            TRY(starmm_plan_create(&P->twin, P->sr, P->algo, P->alloc, P->m, P->n, P->k, P->base_dim,
                                   P->workers, P->ksplit_req, P->device, P->flags));
            P->twin->strassen_leaf = P->strassen_leaf;
        }
        P->twin->flags = P->flags;
        P->twin->ksplit_req = P->ksplit_req;
        TRY(res.stream(&cs2));
    }
    const starmm_stats twin_before = two_streams ? P->twin->st : starmm_stats{};
    struct GateOff {            // the schedule's launches overlap: no wave gate inside it
        starmm_plan* a; starmm_plan* b;
        ~GateOff() { a->dmma_gate = 1; if (b) b->dmma_gate = 1; }
    } gate_off{P, two_streams ? P->twin : nullptr};
    P->dmma_gate = 0;
    if (two_streams) P->twin->dmma_gate = 0;
    std::vector<cudaEvent_t> ev_q(nq), ev_a(nblk), ev_c(nblk), ev_done(nblk);
    cudaEvent_t ev_rest = nullptr, ev_p1 = nullptr;
    TRY(res.event(&ev_rest));
    TRY(res.event(&ev_p1));
    for (auto* v : {&ev_q, &ev_a, &ev_c, &ev_done})
        for (auto& e : *v) TRY(res.event(&e));
    // STARMM_HOST_TRACE=1: timing events on the three streams, printed as one JSON line
    // per event to stderr (label, ms since the start) -- the schedule's timeline
    const char* tenv = getenv("STARMM_HOST_TRACE");
    const bool tracing = tenv && tenv[0] == '1';
    std::vector<std::pair<std::string, cudaEvent_t>> trace;
    auto mark = [&](const std::string& label, cudaStream_t st) {
        if (!tracing) return;
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return;
        cudaEventRecord(e, st);
        trace.push_back({label, e});
    };
    mark("start", cs);
    if (tracing) {
        cudaStreamWaitEvent(up, trace[0].second, 0);
        cudaStreamWaitEvent(down, trace[0].second, 0);
    }
    void *dA = nullptr, *dB = nullptr, *dC = nullptr, *dC0 = nullptr;
    long long fr = 0, ru = 0;
    const size_t a_bytes = (size_t)m * k * eb, b_bytes = (size_t)k * n * eb, c_bytes = (size_t)m * n * eb;
    int rc = STARMM_OK;
    // host (src, ld_src) -> device (dst, ld_dst): the rows x cols block at (r0, c0)
    auto up_block = [&](void* dst, long long ld_dst, const void* src, long long ld_src, long long r0,
                        long long c0, long long rows, long long cols) {
        if (rows <= 0 || cols <= 0) return (int)STARMM_OK;
        return cuda_status(cudaMemcpy2DAsync((char*)dst + (r0 * ld_dst + c0) * eb, ld_dst * eb,
                                             (const char*)src + (r0 * ld_src + c0) * eb, ld_src * eb,
                                             cols * eb, rows, cudaMemcpyHostToDevice, up));
    };
    const char* k2env = getenv("STARMM_HOST_KSPLIT2");   // phase-2 k-split override (tuning)
    const int ks2 = k2env ? atoi(k2env) : -2;
    const int saved_ks = P->ksplit_req;
    auto run = [&](starmm_plan* Q, cudaStream_t st, void* Cd, const void* Ad, const void* Bd, long long rows,
                   long long kk, bool store) {
        Q->m = rows; Q->k = kk;
        if (kk == k - kq && ks2 >= -1) Q->ksplit_req = ks2;   // phase-2 split override (tuning)
        // (STARMM_F_TIME_MAIN would synchronise the host after every launch and serialise the
        // schedule, so the host path never times its kernels)
        const int f = saved_flags & ~STARMM_F_TIME_MAIN;
        Q->flags = store ? (f | STARMM_F_INIT_IDENTITY) : (f & ~STARMM_F_INIT_IDENTITY);
        int r = execute_impl(Q, Cd, n, Ad, k, Bd, n, st, true);
        Q->m = m; Q->k = k; Q->flags = saved_flags; Q->ksplit_req = saved_ks;
        return r;
    };
    do {
        if ((rc = P->arena.acquire(a_bytes, &dA, false, &fr, &ru))) break;
        if (!same_ab && (rc = P->arena.acquire(b_bytes, &dB, false, &fr, &ru))) break;
        if (same_ab) dB = dA;
        if ((rc = P->arena.acquire(c_bytes, &dC, false, &fr, &ru))) break;
        if (staged_c0 && (rc = P->arena.acquire(c_bytes, &dC0, false, &fr, &ru))) break;
        void* dCin = staged_c0 ? dC0 : dC;   // where C0's rows land
        // ---- uploads, in consumption order, all on `up` ----
        for (int c = 0; c < nq && !rc; ++c) {
            const long long k0 = kb[c], k1 = kb[c + 1];
            if (same_ab) {
                rc = up_block(dA, k, A, lda, k0, k0, k1 - k0, n - k0);             // row block c
                if (!rc) rc = up_block(dA, k, A, lda, k1, k0, m - k1, k1 - k0);    // column block c
            } else {
                rc = up_block(dB, n, B, ldb, k0, 0, k1 - k0, n);                   // B[chunk, :]
                if (!rc) rc = up_block(dA, k, A, lda, 0, k0, m, k1 - k0);          // A[:, chunk]
            }
            if (!rc) rc = cuda_status(cudaEventRecord(ev_q[c], up));
            mark("up_chunk" + std::to_string(c), up);
        }
        if (rc) break;
        if (same_ab) rc = up_block(dA, k, A, lda, kq, kq, m - kq, n - kq);         // bottom-right
        else rc = up_block(dB, n, B, ldb, kq, 0, k - kq, n);                       // B[kq:, :]
        if (!rc) rc = cuda_status(cudaEventRecord(ev_rest, up));
        mark("up_rest", up);
        for (long long b = 0; b < nblk && !rc; ++b) {
            const long long r0 = bst[b], rows = bst[b + 1] - bst[b];
            if (!same_ab) rc = up_block(dA, k, A, lda, r0, kq, rows, k - kq);      // A[blk, kq:]
            if (!rc) rc = cuda_status(cudaEventRecord(ev_a[b], up));
            mark("up_a" + std::to_string(b), up);
            if (!rc && !user_init) rc = up_block(dCin, n, C, ldc, r0, 0, rows, n); // C0[blk, :]
            if (!rc) rc = cuda_status(cudaEventRecord(ev_c[b], up));
            mark("up_c" + std::to_string(b), up);
        }
        if (rc) break;
        // ---- phase 1: k-outer chunks over all rows ----
        for (int c = 0; c < nq && !rc; ++c) {
            const long long k0 = kb[c], k1 = kb[c + 1];
            if ((rc = cuda_status(cudaStreamWaitEvent(cs, ev_q[c], 0)))) break;
            rc = run(P, cs, dC, (char*)dA + k0 * eb, (char*)dB + k0 * n * eb, m, k1 - k0, c == 0);
            mark("mm_chunk" + std::to_string(c), cs);
        }
        if (rc) break;
        // ---- phase 2: row blocks over [kq, k), C0 fold, download ----
        if ((rc = cuda_status(cudaStreamWaitEvent(cs, ev_rest, 0)))) break;
        if (two_streams) {
            if ((rc = cuda_status(cudaEventRecord(ev_p1, cs)))) break;     // phase 1 + B resident
            if ((rc = cuda_status(cudaStreamWaitEvent(cs2, ev_p1, 0)))) break;
        }
        for (long long b = 0; b < nblk && !rc; ++b) {
            const long long r0 = bst[b], rows = bst[b + 1] - bst[b];
            char* Cb = (char*)dC + r0 * n * eb;
            starmm_plan* Q = (two_streams && (b & 1)) ? P->twin : P;
            cudaStream_t sb = (two_streams && (b & 1)) ? cs2 : cs;
            // C0 is folded in BEFORE the block's tile kernel: a small kernel queued behind a
            // persistent launch on the other stream would wait for that launch to end
            if (staged_c0) {
                if ((rc = cuda_status(cudaStreamWaitEvent(sb, ev_c[b], 0)))) break;
                if ((rc = madd_dispatch(P->sr, Cb, n, (char*)dC0 + r0 * n * eb, n, rows, n, 0, sb))) break;
            }
            if (kq < k) {
                if ((rc = cuda_status(cudaStreamWaitEvent(sb, ev_a[b], 0)))) break;
                if (nq == 0 && (rc = cuda_status(cudaStreamWaitEvent(sb, ev_c[b], 0)))) break;
                rc = run(Q, sb, Cb, (char*)dA + (r0 * k + kq) * eb, (char*)dB + kq * n * eb, rows, k - kq,
                         nq == 0 && user_init);
                if (rc) break;
                mark("mm_blk" + std::to_string(b), sb);
            }
            if ((rc = cuda_status(cudaEventRecord(ev_done[b], sb)))) break;
            if ((rc = cuda_status(cudaStreamWaitEvent(down, ev_done[b], 0)))) break;
            rc = cuda_status(cudaMemcpy2DAsync((char*)C + r0 * ldc * eb, ldc * eb, Cb, n * eb, n * eb, rows,
                                               cudaMemcpyDeviceToHost, down));
            mark("down" + std::to_string(b), down);
        }
        if (rc) break;
        if ((rc = cuda_status(cudaStreamSynchronize(down)))) break;
        if (cs2 && (rc = cuda_status(cudaStreamSynchronize(cs2)))) break;
        rc = cuda_status(cudaStreamSynchronize(cs));
    } while (0);
    if (two_streams) {   // the twin's executes and launches count as this plan's
        const starmm_stats& t = P->twin->st;
        P->st.executes += t.executes - twin_before.executes;
        P->st.kernel_launches += t.kernel_launches;
        P->st.main_kernel_ns += t.main_kernel_ns - twin_before.main_kernel_ns;
        P->st.main_kernel_launches += t.main_kernel_launches - twin_before.main_kernel_launches;
    }
    P->m = m; P->k = k; P->flags = saved_flags;
    cudaStreamSynchronize(up);       // nothing may still read or write the arena blocks
    cudaStreamSynchronize(down);
    cudaStreamSynchronize(cs);
    if (cs2) cudaStreamSynchronize(cs2);
    for (auto& t : trace) {
        float ms = 0;
        cudaEventElapsedTime(&ms, trace[0].second, t.second);
        fprintf(stderr, "{\"host_trace\": \"%s\", \"ms\": %.3f}\n", t.first.c_str(), ms);
    }
    for (auto& t : trace) cudaEventDestroy(t.second);
    if (dC0) P->arena.release(dC0, c_bytes);
    if (dC) P->arena.release(dC, c_bytes);
    if (dB && !same_ab) P->arena.release(dB, b_bytes);
    if (dA) P->arena.release(dA, a_bytes);
    return rc;
}

int starmm_matmul(int semiring, void* out, int64_t ldo, const void* A, int64_t lda, const void* B,
                  int64_t ldb, int64_t m, int64_t n, int64_t k, void* stream, int flags) {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    starmm_plan* P = nullptr;
    TRY(starmm_plan_create(&P, semiring, STARMM_CO2, STARMM_POOLED, m, n, k, 1, 1, 0, dev,
                           (flags | STARMM_F_INIT_IDENTITY | STARMM_F_ALLOW_NONPOW2)));
    int rc = starmm_execute(P, out, ldo, A, lda, B, ldb, stream);
    starmm_plan_destroy(P);
    return rc;
}

int starmm_madd(int semiring, void* C, int64_t ldc, const void* D, int64_t ldd, int64_t rows,
                int64_t cols, void* stream, int flags) {
    if (!C || !D) return STARMM_CONTRACT_VIOLATION;
    if (ldc < cols || ldd < cols || rows < 0 || cols < 0) return STARMM_DIM_MISMATCH;
    cudaStream_t s = (cudaStream_t)stream;
    TRY(madd_dispatch(semiring, C, ldc, D, ldd, rows, cols, 0, s));
    if (!(flags & STARMM_F_ASYNC)) CK(cudaStreamSynchronize(s));
    return STARMM_OK;
}

int starmm_atomic_accumulate(int semiring, void* C, int64_t ldc, const void* P_, int64_t ldp,
                             int64_t rows, int64_t cols, void* stream, int flags) {
    if (!C || !P_) return STARMM_CONTRACT_VIOLATION;
    if (ldc < cols || ldp < cols || rows < 0 || cols < 0) return STARMM_DIM_MISMATCH;
    cudaStream_t s = (cudaStream_t)stream;
    TRY(madd_dispatch(semiring, C, ldc, P_, ldp, rows, cols, 1, s));
    if (!(flags & STARMM_F_ASYNC)) CK(cudaStreamSynchronize(s));
    return STARMM_OK;
}

}  // extern "C"
