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
//   device pool ............... Pool (pool.py:67-167) shared per device (arena.h)
//   range guard verdict ....... guard.h, on the device (select_path_kernel)
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
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
#include "ordered_kernel.cuh"
#include "generate.cuh"
#include "simt_launch.h"
#include "guard.h"
#include "arena.h"

using namespace starmm;
using starmm_host::DeviceCtx;
using starmm_host::FenceRef;

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

int current_device() {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess) { cudaGetLastError(); return 0; }
    return d;
}

// ---- per-device state: the shared block pool and mapped host words ------------
// Created on first use and never destroyed: the pools' blocks, events and mapped pages
// are the process's until exit (static destructors would run after the CUDA runtime
// has started tearing down, and a fence's destructor would touch a destroyed pool).
DeviceCtx* g_ctx[starmm_host::MAX_DEVICES] = {};
std::mutex g_ctx_mu;
// starmm_matmul's plan cache (per device, most recently used last)
std::mutex& g_mm_mu = *new std::mutex();
std::vector<starmm_plan*>* g_mm_cache = new std::vector<starmm_plan*>[starmm_host::MAX_DEVICES];

DeviceCtx* device_ctx(int dev) {
    if (dev < 0 || dev >= starmm_host::MAX_DEVICES) return nullptr;
    std::lock_guard<std::mutex> g(g_ctx_mu);
    if (!g_ctx[dev]) g_ctx[dev] = new DeviceCtx();
    DeviceCtx& c = *g_ctx[dev];
    if (c.device < 0) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        size_t fr = 0, tot = 0;
        int prev = current_device();
        if (prev != dev) cudaSetDevice(dev);
        if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) cudaGetLastError();
        if (prev != dev) cudaSetDevice(prev);
        // cached blocks are trimmed before the pool owns more than 3/4 of HBM
        // (STARMM_POOL_LIMIT_MB overrides; an allocation failure always trims and retries)
        const char* lim = getenv("STARMM_POOL_LIMIT_MB");
        c.arena.limit = lim ? atoll(lim) * (1LL << 20) : (long long)(tot / 4 * 3);
        c.arena.device = dev;
        c.sms = v;
        c.device = dev;
    }
    return &c;
}

// cudaSetDevice for the duration of a call, restored on every return path
struct DeviceGuard {
    int prev = -1, dev = -1;
    int set(int d) {
        CK(cudaGetDevice(&prev));
        dev = d;
        if (prev != d) CK(cudaSetDevice(d));
        return STARMM_OK;
    }
    ~DeviceGuard() { if (prev >= 0 && prev != dev) cudaSetDevice(prev); }
};

struct Block { void* p = nullptr; size_t bytes = 0; };

// per-candidate summary of one execute (the stats describe the path that ran)
struct CandInfo {
    int path = 0;
    long long tasks = 0, workers = 0, S = 1, tar_levels = 0, balanced_workers = 0, pair_count = 0;
    long long raw_count = 0, raw_bytes = 0;
    int s_log2 = 0;
    int cluster = 0;         // > 0: DMMA split-k merged on a cluster of this many CTAs
    int k_chunks = 1;        // k-outer chunks of a CUDA-core launch (simt_k_chunks)
};

}  // namespace

struct starmm_plan {
    int sr, algo, alloc, base_dim, workers, ksplit_req, device, flags;
    long long m, n, k;
    long long kofs = 0;                         // global k index of the first k (host path chunks)
    int sms = 0;
    DeviceCtx* ctx = nullptr;                   // the device's shared block pool
    // persistent device bookkeeping (one pool block, kept for the plan's life)
    void* book = nullptr;
    unsigned long long* d_counters = nullptr;   // CNT__N
    unsigned long long* d_range = nullptr;      // 2 words: max |x|, guard bits
    unsigned* d_sel = nullptr;                  // the device-side path verdict (Pred::sel)
    unsigned* d_worker_used = nullptr;          // per persistent worker
    unsigned* d_gate = nullptr;                 // DMMA wave-gate counter
    // mapped pinned host words (zero-copy; a D2H memcpy would queue behind the host
    // path's downloads on the copy engine): [0..1] range, [2] selected path, [3] the
    // narrowest allowed path (next call's first guess)
    unsigned long long* hs = nullptr;
    unsigned long long* hs_dev = nullptr;
    int dmma_gate = 1;                          // 0 inside the host path (overlapping launches)
    int max_workers = 0;
    starmm_stats st;
    long long total_allocated = 0;              // bytes this plan's acquisitions cudaMalloc'ed
    long long ws_fresh = 0, ws_reuse = 0, ws_high_water = 0;
    long long raw_count = 0, raw_bytes = 0;
    // STARMM_F_TIME_MAIN: each timed execute leaves one record (an event pair per queued
    // candidate); which candidate ran is known on the device, so with a device-side
    // verdict the select kernel writes it into a mapped ring slot.  Records are resolved
    // when the call blocks anyway, or lazily by starmm_plan_stats: an asynchronous timed
    // execute never waits (the bench's back-to-back steps leave no host gap).
    struct TimedRec {
        cudaEvent_t ev[6];
        int ncand, ran;             // ran < 0: read ring[slot]
        int path[3];
        int slot;
    };
    std::vector<TimedRec> timed;
    std::vector<cudaEvent_t> ev_pool;
    unsigned long long* ring = nullptr;         // mapped pinned: selected path per timed call
    unsigned long long* ring_dev = nullptr;
    int ring_next = 0;
    int hint = 0;                               // narrowest path the last guard allowed
    bool spec_used = false;                     // hs[3] carries a device-written hint
    starmm_plan* twin = nullptr;                // host path: the second compute stream's plan
    long long strassen_leaf = 1024;             // Strassen recursion stops at max(b, this)
    long long str_issued = 0;                   // Strassen temporaries currently issued
    // peer destinations of the fused k-split combine (starmm_plan_set_peers)
    int remote_parts = 0;
    long long remote_rows = 0, remote_ld = 0;
    void* remote_base[8] = {};
    // the last fence recorded on each stream this plan ran on (destroy waits for them)
    std::vector<FenceRef> fences;
};

static int resolve_timed(starmm_plan* P, bool block);

namespace {

// ---- the plan's view of the device pool ------------------------------------
int plan_acquire(starmm_plan* P, size_t bytes, cudaStream_t s, void** out, bool temp) {
    bool fresh = false;
    CK(P->ctx->arena.acquire(bytes, s, out, &fresh));
    if (fresh) P->total_allocated += (long long)starmm_host::DevArena::size_class(bytes);
    if (temp) { if (fresh) ++P->ws_fresh; else ++P->ws_reuse; }
    return STARMM_OK;
}

void plan_note_fence(starmm_plan* P, const FenceRef& f) {
    if (!f) return;
    for (auto& x : P->fences)
        if (x->st == f->st) { x = f; return; }
    P->fences.push_back(f);
}

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
    case PATH_TC_I8_LIMBS: { // 8 radix-256 digit planes of int8 per operand
        PathShape sh{2 * tcg::BM, tcg::BN, tcg::BK, 1, 8000, 8000};
        return sh;
    }
    case PATH_MIN_ORDERED: {  // reads A and B in place
        PathShape sh{ordered::TM, ordered::TN, ordered::TK, 1, 0, 0};
        return sh;
    }
    }
    return simt_shape<PolI64>();
}

// mbarrier-pipelined k-loop (tools/sweep_dmma.cu: 35.4 vs 34.4 TF/s with per-stage
// __syncthreads), vectorised FOLD epilogue.  With `gate` (p.gate zeroed here) the
// wave gate with a quarter-wave slack keeps the persistent CTAs in step: DRAM reads
// per n=16384 launch 240-263 GB -> 51 GB at -0.1% (profiles/r01l_dmma_gate.md).
// The >48 KB smem opt-in is a per-device (per-context) attribute: set once per device.
int launch_dmma(const DmmaParams& p, int grid, bool gate, cudaStream_t s) {
    using K = DmmaProd;
    static bool attr_done[starmm_host::MAX_DEVICES] = {};
    const int dev = current_device();
    if (!attr_done[dev]) {
        CK(cudaFuncSetAttribute(dmma_fp64_kernel_mb<K, 1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                K::SMEM_BYTES));
        CK(cudaFuncSetAttribute(dmma_fp64_kernel_mb<K, 1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                K::SMEM_BYTES));
        attr_done[dev] = true;
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


// ---- DMMA split-k on clusters (dmma_fp64_cluster_kernel) ------------------------------
// Cluster mode runs the S k-slices of a tile on the S CTAs of one cluster and merges
// them through DSMEM: for tar / sar / star on the DMMA path with S in {2, 4, 8}, local
// write-back.  STARMM_DMMA_CLUSTER=0 keeps the global-memory protocols (A/B evidence).
bool dmma_cluster_mode(const starmm_plan* P, int S) {
    if (S < 2 || S > 8 || P->remote_parts > 0) return false;
    if (!(P->algo == STARMM_TAR || P->algo == STARMM_SAR || P->algo == STARMM_STAR)) return false;
    const char* e = getenv("STARMM_DMMA_CLUSTER");
    return !(e && e[0] == '0');
}

template <int CS>
cudaError_t dmma_cluster_config(cudaLaunchConfig_t& lc, cudaLaunchAttribute* at, int* slots) {
    using K = DmmaProd;
    static bool attr_done[starmm_host::MAX_DEVICES] = {};
    static int cached[starmm_host::MAX_DEVICES] = {};
    const int dev = current_device();
    auto kern = dmma_fp64_cluster_kernel<K, CS>;
    if (!attr_done[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, K::SMEM_BYTES);
        if (e != cudaSuccess) return e;
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaLaunchConfig_t q = {};
        q.gridDim = dim3((unsigned)(sms / CS * CS)); q.blockDim = dim3(K::THREADS);
        q.dynamicSmemBytes = K::SMEM_BYTES;
        cudaLaunchAttribute qa[1];
        qa[0].id = cudaLaunchAttributeClusterDimension;
        qa[0].val.clusterDim.x = CS; qa[0].val.clusterDim.y = 1; qa[0].val.clusterDim.z = 1;
        q.attrs = qa; q.numAttrs = 1;
        int c = 0;
        if (cudaOccupancyMaxActiveClusters(&c, kern, &q) != cudaSuccess || c < 1) {
            cudaGetLastError();
            c = std::max(1, sms / CS);
        }
        cached[dev] = c;
        attr_done[dev] = true;
    }
    *slots = cached[dev];
    lc.blockDim = dim3(K::THREADS);
    lc.dynamicSmemBytes = K::SMEM_BYTES;
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CS; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    lc.attrs = at; lc.numAttrs = 1;
    return cudaSuccess;
}

// co-resident clusters of size S (the cluster mode's persistent slots)
int dmma_cluster_slots(int S) {
    cudaLaunchConfig_t lc = {};
    cudaLaunchAttribute at[1];
    int slots = 0;
    cudaError_t e = cudaSuccess;
    switch (S) {
    case 2: e = dmma_cluster_config<2>(lc, at, &slots); break;
    case 4: e = dmma_cluster_config<4>(lc, at, &slots); break;
    case 8: e = dmma_cluster_config<8>(lc, at, &slots); break;
    default: return 0;
    }
    if (e != cudaSuccess) { cudaGetLastError(); return 0; }
    return slots;
}

template <int CS>
int launch_dmma_cluster_cs(const DmmaParams& p, long long tiles, cudaStream_t s) {
    cudaLaunchConfig_t lc = {};
    cudaLaunchAttribute at[1];
    int slots = 0;
    CK(dmma_cluster_config<CS>(lc, at, &slots));
    const long long clusters = std::max<long long>(1, std::min<long long>(slots, tiles));
    lc.gridDim = dim3((unsigned)(clusters * CS));
    lc.stream = s;
    CK(cudaLaunchKernelEx(&lc, dmma_fp64_cluster_kernel<DmmaProd, CS>, p));
    return STARMM_OK;
}

int launch_dmma_cluster(const DmmaParams& p, int S, long long tiles, cudaStream_t s) {
    switch (S) {
    case 2: return launch_dmma_cluster_cs<2>(p, tiles, s);
    case 4: return launch_dmma_cluster_cs<4>(p, tiles, s);
    case 8: return launch_dmma_cluster_cs<8>(p, tiles, s);
    }
    return STARMM_INTERNAL_ERROR;
}

template <class Sr>
int launch_madd(void* C, long long ldc, const void* D, long long ldd, long long rows, long long cols,
                int atomic, cudaStream_t s, int rev = 0, Pred pr = Pred()) {
    if (rows <= 0 || cols <= 0) return STARMM_OK;
    using T = typename Sr::T;
    madd_kernel<Sr><<<grid2d(rows, cols), 256, 0, s>>>((T*)C, ldc, (const T*)D, ldd, rows, cols,
                                                           atomic, rev, pr);
    CK(cudaGetLastError());
    return STARMM_OK;
}

int madd_dispatch(int sr, void* C, long long ldc, const void* D, long long ldd, long long rows,
                  long long cols, int atomic, cudaStream_t s, int rev = 0, Pred pr = Pred()) {
    switch (sr) {
    case STARMM_SR_INT64: return launch_madd<SrInt64>(C, ldc, D, ldd, rows, cols, atomic, s, rev, pr);
    case STARMM_SR_FP64: return launch_madd<SrFp64>(C, ldc, D, ldd, rows, cols, atomic, s, rev, pr);
    case STARMM_SR_TROPICAL_F64: return launch_madd<SrTropF64>(C, ldc, D, ldd, rows, cols, atomic, s, rev, pr);
    case STARMM_SR_TROPICAL_F32: return launch_madd<SrTropF32>(C, ldc, D, ldd, rows, cols, atomic, s, rev, pr);
    case STARMM_SR_TROPICAL_I32: return launch_madd<SrTropI32>(C, ldc, D, ldd, rows, cols, atomic, s, rev, pr);
    }
    return STARMM_CONTRACT_VIOLATION;
}

template <class Sr>
int launch_fill(void* C, long long rows, long long cols, long long ld, cudaStream_t s, Pred pr) {
    fill_kernel<Sr><<<grid2d(rows, cols), 256, 0, s>>>((typename Sr::T*)C, rows, cols, ld, pr);
    CK(cudaGetLastError());
    return STARMM_OK;
}

int fill_dispatch(int sr, void* C, long long rows, long long cols, long long ld, cudaStream_t s,
                  Pred pr = Pred()) {
    switch (sr) {
    case STARMM_SR_INT64: return launch_fill<SrInt64>(C, rows, cols, ld, s, pr);
    case STARMM_SR_FP64: return launch_fill<SrFp64>(C, rows, cols, ld, s, pr);
    case STARMM_SR_TROPICAL_F64: return launch_fill<SrTropF64>(C, rows, cols, ld, s, pr);
    case STARMM_SR_TROPICAL_F32: return launch_fill<SrTropF32>(C, rows, cols, ld, s, pr);
    case STARMM_SR_TROPICAL_I32: return launch_fill<SrTropI32>(C, rows, cols, ld, s, pr);
    }
    return STARMM_CONTRACT_VIOLATION;
}

template <class Tin, class Tp, int G, class Conv>
int launch_pack(const void* A, long long lda, const void* B, long long ldb, long long m,
                long long n, long long k, void* Ap, void* Bp, long long Mp, long long Np,
                long long Kp, Tp pad, cudaStream_t s, unsigned long long* range, Pred pr) {
    const dim3 ga = pack_a_grid(Mp, Kp);
    pack_a_kernel<Tin, Tp, G, Conv><<<ga, dim3(32, 8), 0, s>>>((const Tin*)A, m, k, lda, (Tp*)Ap, Mp,
                                                              Kp, pad, range, pr);
    CK(cudaGetLastError());
    pack_b_kernel<Tin, Tp, G, Conv><<<grid2d(Kp / G, Np), 256, 0, s>>>(
        (const Tin*)B, k, n, ldb, (Tp*)Bp, Np, Kp, pad, range, pr);
    CK(cudaGetLastError());
    return STARMM_OK;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda needed)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                  CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                  CUtensorMapFloatOOBfill);
// row_stride: bytes between rows (0: kp, rows densely packed)
int make_i8_tmap(CUtensorMap* map, void* base, long long rows, long long kp, int box_rows,
                 long long row_stride = 0) {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &q));
        if (!fn || q != cudaDriverEntryPointSuccess) return STARMM_INTERNAL_ERROR;
    }
    cuuint64_t dims[2] = {(cuuint64_t)kp, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(row_stride > 0 ? row_stride : kp)};
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
// which the drift gate requires to be fully resident.  Cached per device (the smem
// attribute and the SM count are per device).
template <class Epi>
int tcg_max_clusters(int sms) {
    static int cached[starmm_host::MAX_DEVICES];
    static bool init[starmm_host::MAX_DEVICES] = {};
    const int dev = current_device();
    if (!init[dev]) {
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
        cached[dev] = c;
        init[dev] = true;
    }
    return cached[dev];
}

// `acquire(bytes, &ptr)` hands out stream-ordered scratch (the plan's arena) for the
// drift-gate counters: one per (pass, tile round), zeroed before the launch.
template <class Epi, class Acquire>
int launch_tcg(const void* Ap, const void* Bp, long long Mp, long long Np, long long Kp, int passes,
               const Epi& epi, int sms, cudaStream_t s, Acquire&& acquire, Pred pr,
               long long row_stride = 0) {
    if ((long long)passes * Mp >= (1LL << 31) || (long long)passes * Np >= (1LL << 31)) return STARMM_TOO_LARGE;
    CUtensorMap ta, tb;
    TRY(make_i8_tmap(&ta, const_cast<void*>(Ap), Mp * passes, Kp, tcg::BM, row_stride));
    TRY(make_i8_tmap(&tb, const_cast<void*>(Bp), Np * passes, Kp, tcg::BNH, row_stride));
    auto kern = tcg_kernel<Epi>;
    const int clusters = tcg_max_clusters<Epi>(sms);
    TcgShape sh;
    sh.tiles_m = (int)(Mp / 256); sh.tiles_n = (int)(Np / 256); sh.num_tiles = sh.tiles_m * sh.tiles_n;
    sh.group_m = 8;
    sh.nk = (int)(Kp / tcg::BK); sh.passes = passes;
    sh.a_pass_rows = (int)Mp; sh.b_pass_rows = (int)Np;
    sh.pr = pr;
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
    static std::once_flag once;
    std::call_once(once, []() {
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
    });
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

// One pool block per plan for its device-side words: counters, the range guard, the
// path verdict, per-worker flags, the DMMA gate; plus a mapped host slot.
int ensure_bookkeeping(starmm_plan* P, cudaStream_t s) {
    if (P->book) return STARMM_OK;
    P->max_workers = P->sms * 2;
    const size_t bytes = CNT__N * 8 + 16 + 16 + (size_t)P->max_workers * 4 + 16;
    void* p = nullptr;
    TRY(plan_acquire(P, bytes, s, &p, false));
    CK(cudaMemsetAsync(p, 0, bytes, s));
    P->book = p;
    P->d_counters = (unsigned long long*)p;
    P->d_range = P->d_counters + CNT__N;
    P->d_sel = (unsigned*)(P->d_range + 2);
    P->d_worker_used = (unsigned*)(P->d_range + 4);
    P->d_gate = P->d_worker_used + P->max_workers;
    CK(P->ctx->slots.get(&P->hs, &P->hs_dev));
    return STARMM_OK;
}

// The range guard's verdict on the device: the narrowest exact path for the observed
// range (guard.h), and the candidate that runs -- the first guess if it is exact for
// this data, else the ordered kernel (-0.0 in a float (min,+) operand) or the general
// kernel of the semiring.  Published to the plan's mapped host words as well.
__global__ void select_path_kernel(const unsigned long long* d_range, int sr, int flags, long long k,
                                   int first, int general, int ordered_ok, unsigned* d_sel,
                                   unsigned long long* h, unsigned long long* ring_slot) {
    if (threadIdx.x != 0) return;
    const unsigned long long mx = d_range[0], bits = d_range[1];
    const int nar = guard_narrowest(sr, flags, k, mx, bits, ordered_ok);
    const int sel = path_allowed(first, nar) ? first : (nar == PATH_MIN_ORDERED ? PATH_MIN_ORDERED : general);
    *d_sel = (unsigned)sel;
    h[0] = mx; h[1] = bits; h[2] = (unsigned long long)sel; h[3] = (unsigned long long)nar;
    if (ring_slot) *ring_slot = (unsigned long long)sel;
    __threadfence_system();
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
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
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
    if (device < 0 || device >= ndev || device >= starmm_host::MAX_DEVICES) return STARMM_CONTRACT_VIOLATION;
    DeviceCtx* ctx = device_ctx(device);
    if (!ctx) return STARMM_INTERNAL_ERROR;
    starmm_plan* P = new starmm_plan();
    P->sr = semiring; P->algo = algo; P->alloc = alloc_mode; P->base_dim = base_dim;
    P->workers = workers; P->ksplit_req = ksplit_log2; P->device = device; P->flags = flags;
    P->m = m; P->n = n; P->k = k;
    memset(&P->st, 0, sizeof(P->st));
    P->ctx = ctx;
    P->sms = ctx->sms;
    *plan = P;
    return STARMM_OK;
}

// Executor.close (runtime.py:83-93).  Waits only for this plan's own work (the fences
// of the streams it ran on), never for the device; its blocks go back to the device pool.
void starmm_plan_destroy(starmm_plan* P) {
    if (!P) return;
    DeviceGuard dg;
    dg.set(P->device);
    for (auto& f : P->fences)
        if (f && f->ev) cudaEventSynchronize(f->ev);
    P->fences.clear();
    for (auto& r : P->timed)
        for (int i = 0; i < 2 * r.ncand; ++i) cudaEventDestroy(r.ev[i]);
    for (auto e : P->ev_pool) cudaEventDestroy(e);
    if (P->ring) cudaFreeHost(P->ring);
    if (P->twin) starmm_plan_destroy(P->twin);
    if (P->book) P->ctx->arena.release(P->book, nullptr);
    if (P->hs) P->ctx->slots.put(P->hs, P->hs_dev);
    delete P;
}

int starmm_plan_reset_stats(starmm_plan* P) {
    if (!P) return STARMM_CONTRACT_VIOLATION;
    // timed records of earlier executes belong to the stats being discarded
    for (auto& r : P->timed) {
        cudaEventSynchronize(r.ev[2 * r.ncand - 1]);
        for (int i = 0; i < 2 * r.ncand; ++i) P->ev_pool.push_back(r.ev[i]);
    }
    P->timed.clear();
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
    {
        DeviceGuard dg;
        TRY(dg.set(P->device));
        TRY(resolve_timed(P, true));          // timed async executes: wait for their events
    }
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
    out->pool_total_allocated_bytes = P->total_allocated;
    out->raw_alloc_count = P->raw_count;
    out->raw_alloc_bytes = P->raw_bytes;
    out->live_leaves_max = (int64_t)c[CNT_LIVE_MAX];
    return STARMM_OK;
}

}  // extern "C"

// ============================================================================
// execute: path choice, packing, protocol state, tile kernel, co3 merge
// ============================================================================
namespace {

// Geometry of one kernel path on this plan's problem: tiles, occupancy, k-split.
struct Geom {
    int path = 0;
    bool is_dmma = false;
    PathShape shape{};
    int BK = 0, TBM = 0, TBN = 0, per_sm = 1, gpu_workers = 0, s_log2 = 0, S = 1, tar_levels = 0;
    bool balanced = false;
    long long tiles_m = 0, tiles_n = 0, tiles = 0, Mp = 0, Np = 0, Kp = 0, kslice = 0, ntasks = 0;
    TaskGrid g{};
};

int plan_geometry(const starmm_plan* P, int path, Geom& G) {
    G = Geom();
    G.path = path;
    G.is_dmma = (path == PATH_DMMA_F64);
    G.shape = path_shape(path);
    G.BK = G.shape.bk; G.TBM = G.shape.bm; G.TBN = G.shape.bn; G.per_sm = G.shape.per_sm;
    G.tiles_m = (P->m + G.TBM - 1) / G.TBM; G.tiles_n = (P->n + G.TBN - 1) / G.TBN;
    G.tiles = G.tiles_m * G.tiles_n;
    G.gpu_workers = P->sms * G.per_sm;                 // persistent CTAs (the GPU workers)
    if (path == PATH_MIN_ORDERED) {                    // k-serial, one CTA per output tile
        G.Mp = G.tiles_m * G.TBM; G.Np = G.tiles_n * G.TBN; G.Kp = P->k; G.kslice = P->k;
        G.ntasks = G.tiles;
        G.g.tiles_m = (int)G.tiles_m; G.g.tiles_n = (int)G.tiles_n; G.g.S = 1; G.g.num_tasks = (int)G.tiles;
        return G.tiles_m > 65535 ? STARMM_TOO_LARGE : STARMM_OK;
    }
    const bool is_dmma = G.is_dmma;
    const int BK = G.BK;
    const long long tiles = G.tiles;
    const bool tc_path = path == PATH_TC_I8 || path == PATH_OZAKI_F64 || path == PATH_TC_I8_LIMBS;
    const bool simt_path = !is_dmma && !tc_path;
    const bool may_split = !(P->algo == STARMM_CO2 || tc_path);
    int per_sm = G.per_sm, s_log2 = 0;
    bool balanced = false;
    if ((simt_path || is_dmma) && (P->ksplit_req < 0 || !may_split)) {
        // Pick (CTAs per SM, split depth) by a wave cost model
        //   time ~ ceil(tasks / CTAs) * (stages per task + overhead) / per-CTA rate
        // overhead = 4.5 stages of prologue/epilogue per task, plus the split write-back.
        // The CUDA-core kernels are compiled for two CTAs per SM; launched at one per SM
        // they run at 0.89 of a full SM, 0.97 for the policies with a one-CTA-per-SM build
        // (tools/ksplit_ab.py, profiles/r01i_ksplit_c2.json).  co2 never splits
        // (classic.py:125-128).  The split write-back's cost depends on the schedule's
        // protocol (tools/ksplit_ab.py, profiles/r01k_ksplit_*.json): TAR atomic-madd 2
        // stages (20 for the CAS of float minima), CO3 workspace + merge 3, SAR pair states
        // + locks + lazy temporaries 60 on DMMA (the sibling folds serialise under the tile
        // lock; measured on the round-1 two-CTA 64x128 DMMA kernel, kept for the one-CTA
        // 256x64 kernel whose longer stages make the same write-back relatively cheaper)
        // and 16 on the CUDA-core paths (int64 n=1024: S=2 cost +23%); STAR levels above
        // switch_depth are TAR, deeper ones SAR.  The DMMA path runs one CTA per SM.
        const bool cas_min = P->sr == STARMM_SR_TROPICAL_F32 || P->sr == STARMM_SR_TROPICAL_F64;
        const double pen_tar = cas_min ? 20.0 : 2.0, pen_sar = is_dmma ? 60.0 : 16.0;
        // (the SAR folds of one tile serialise under its lock: cost grows with the 2^sl
        // slices per tile -- tropical n=1024, S=8: -27% vs co2 with a flat penalty)
        auto split_pen = [&](int sl) -> double {
            if (sl == 0) return 0.0;
            // DMMA cluster mode: the S partials merge through DSMEM (~1.5 stages)
            if (is_dmma && dmma_cluster_mode(P, 1 << sl)) return 1.5;
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
                   (tiles << smax) < 8LL * G.gpu_workers)
                ++smax;
        double best = 0;
        int best_occ = per_sm, best_s = 0;
        const bool occ1_build = path == PATH_SIMT_I64_DP4A || path == PATH_SIMT_F32_PAIR ||
                                path == PATH_SIMT_I32_CARRIER || path == PATH_SIMT_F64T_CARRIER ||
                                path == PATH_SIMT_F32_S16X2 || path == PATH_SIMT_I32_S16X2 ||
                                path == PATH_SIMT_F64T_S16X2;                // has_occ1_build
        // (the dp4a policy's one-CTA build runs the cross-stage fragment ring and beats its
        // own two-CTA build: 137.2 vs 132.1 Tops/s at n = 8192, tools/sweep_simt.cu)
        const double rate1 = path == PATH_SIMT_I64_DP4A ? 1.03 : (occ1_build ? 0.97 : 0.89);
        // rate of ONE CTA, in units of a full SM running per_sm co-resident CTAs
        auto cta_rate = [&](int occ) { return occ == 1 ? (per_sm == 1 ? 1.0 : rate1) : 1.0 / occ; };
        for (int occ = per_sm; occ >= (is_dmma ? per_sm : 1); --occ) {
            const double rate = cta_rate(occ);
            for (int sl = 0; sl <= smax; ++sl) {
                double waves = std::ceil((double)(tiles << sl) / ((double)P->sms * occ));
                if (is_dmma && dmma_cluster_mode(P, 1 << sl)) {   // one tile per cluster at a time
                    const int slots = dmma_cluster_slots(1 << sl);
                    if (slots < 1) continue;
                    waves = std::ceil((double)tiles / (double)slots);
                }
                const double ovh = 4.5 + split_pen(sl);
                const double c = waves * (kst / (double)(1 << sl) + ovh) / rate;
                if (best == 0 || c < 0.99 * best) { best = c; best_occ = occ; best_s = sl; }
            }
        }
        // Balanced slices (TAR with uneven k-slices, "stream-K"): every worker gets the
        // same share of the flattened (tile, k-stage) space, pieces of shared tiles merge
        // with the atomic-madd.  Only for tar/star (their split write-back IS the
        // atomic-madd) and exact, cheap atomics (int64 red.add, int32 red.min).
        // On the DMMA path (fp64 red.add: order-dependent rounding, like every fp64 split)
        // it is TAR/STAR's atomic-madd for the <= 2 shared pieces per CTA.
        const char* benv = getenv("STARMM_NO_BALANCED");
        const bool bal_sr = simt_path ? (P->sr == STARMM_SR_INT64 || P->sr == STARMM_SR_TROPICAL_I32)
                                      : is_dmma;
        // STAR merges by atomic-madd only above its switch depth (classic.py:280-296): with
        // p workers too few to have a TAR level (switch_depth(p) == 0) it is pure SAR.
        const bool bal_algo = P->algo == STARMM_TAR ||
                              (P->algo == STARMM_STAR && switch_depth(P->workers) >= 1);
        if ((simt_path || is_dmma) && may_split && bal_algo &&
            bal_sr && P->remote_parts == 0 && !(benv && benv[0] == '1')) {
            for (int occ = per_sm; occ >= (is_dmma ? per_sm : 1); --occ) {
                const double Gw = (double)P->sms * occ;
                const double c = ((double)tiles * (kst + 4.5) + Gw * (4.5 + 2.0)) / Gw / cta_rate(occ);
                if (c < 0.97 * best) { balanced = true; best = c / 0.97; best_occ = occ; best_s = 0; }
            }
        }
        per_sm = best_occ;
        s_log2 = best_s;
    } else if (!may_split) {
        s_log2 = 0;            // k-halves serialised (classic.py:125-128): never split
                               // (the opt-in tensor path keeps whole-K tiles too)
    } else if (P->ksplit_req >= 0) {
        s_log2 = P->ksplit_req;
    }
    // a k-slice is at least one leaf (base_dim) and one k-stage; never more levels
    // than the recursion has (log2(k / b))
    while (s_log2 > 0 && ((P->k >> s_log2) < std::max(P->base_dim, BK) || (P->k >> s_log2) < 1))
        --s_log2;
    G.per_sm = per_sm;
    G.gpu_workers = P->sms * per_sm;
    G.s_log2 = s_log2;
    G.S = 1 << s_log2;
    G.balanced = balanced;
    G.tar_levels = 0;
    if (P->algo == STARMM_TAR) G.tar_levels = s_log2;
    if (P->algo == STARMM_STAR) G.tar_levels = std::min(switch_depth(P->workers), s_log2);
    G.Mp = G.tiles_m * G.TBM; G.Np = G.tiles_n * G.TBN;
    G.Kp = round_up(P->k, std::max<long long>(32, (long long)BK * G.S));
    G.kslice = G.Kp / G.S;
    TaskGrid& g = G.g;
    g.tiles_m = (int)G.tiles_m; g.tiles_n = (int)G.tiles_n; g.S = G.S; g.log2S = s_log2;
    g.tar_levels = G.tar_levels; g.kslice = G.kslice;
    // raster groups sized so one wave of resident CTAs covers a near-square block of
    // tiles (minimises the A+B panels live in L2; tools/gsweep.sh: -42% DRAM bytes)
    g.group_m = is_dmma ? 4 : 12;   // DMMA: 4 x 256 rows (58 GB vs 61 GB at 6), SIMT 12 x 128
    g.balanced = balanced ? 1 : 0;
    g.kstages = G.Kp / std::max(1, BK);
    G.ntasks = tiles * G.S;
    if (G.ntasks > (1LL << 31) - 1) return STARMM_TOO_LARGE;
    g.num_tasks = (int)G.ntasks;
    return STARMM_OK;
}

// packed k-group geometry of the CUDA-core paths (simt_kernel.cuh policies)
int simt_kstep(int path) {
    return path == PATH_SIMT_I64_DP4A ? 4 : 1;
}
int simt_g(int path) {
    return (path == PATH_SIMT_F32_PAIR || path == PATH_SIMT_I32_CARRIER || path == PATH_SIMT_F64T_CARRIER) ? 2 : 1;
}

// k-outer chunk count of a CUDA-core launch: 1 unless the panels one wave of persistent
// CTAs streams (group_m tile-rows of A, grid / group_m tile-columns of B, over all of k)
// exceed twice the L2; then enough chunks to bring them to ~96 MB.  Only for unsplit,
// unbalanced, local launches (every chunk is then a plain fold of whole tiles).
int simt_k_chunks(const starmm_plan* P, const Geom& G) {
    const char* e = getenv("STARMM_K_CHUNKS");
    if (G.S != 1 || G.balanced || P->remote_parts > 0 || G.path == PATH_MIN_ORDERED) return 1;
    if (e) return std::max(1, atoi(e));
    const long long waves_cols = std::max<long long>(1, (long long)P->sms * G.per_sm / G.g.group_m);
    const double bytes = ((double)std::min<long long>(G.g.group_m, G.tiles_m) * G.TBM * G.shape.a_bytes_per_km +
                          (double)std::min<long long>(waves_cols, G.tiles_n) * G.TBN * G.shape.b_bytes_per_kn) /
                         1000.0 * (double)G.Kp;
    if (bytes <= 2.0 * 126e6) return 1;
    const long long n = (long long)std::ceil(bytes / 96e6);
    return (int)std::max<long long>(1, std::min<long long>(n, G.Kp / std::max(4096, G.BK)));
}

// DMMA reads A and B in place when the tiles divide the problem and rows are 16-byte
// aligned; otherwise from zero-padded staging copies
bool dmma_direct(const starmm_plan* P, const Geom& G, const void* A, long long lda, const void* B,
                 long long ldb) {
    return (P->m % G.TBM == 0) && (P->n % G.TBN == 0) && (P->k == G.Kp) &&
           (((uintptr_t)A | (uintptr_t)B) % 16 == 0) && (lda % 2 == 0) && (ldb % 2 == 0);
}

// K chunking of the radix-256 digit path: chunks of <= 8192 k (every digit group's int32
// sum (s + 1) K 2^14 stays <= 2^30), multiples of the tcgen05 core's k-stage (tcg::BK)
void limb_chunks(long long Kp, long long* kc, int* nch) {
    const long long n = (Kp + 8191) / 8192;
    *kc = round_up((Kp + n - 1) / n, tcg::BK);
    *nch = (int)((Kp + *kc - 1) / *kc);
}

// staging bytes of the packed operands of a path (0: read in place)
void packed_bytes(const starmm_plan* P, const Geom& G, const void* A, long long lda, const void* B,
                  long long ldb, size_t* ab, size_t* bb) {
    *ab = *bb = 0;
    if (G.path == PATH_MIN_ORDERED) return;
    if (G.is_dmma) {
        if (dmma_direct(P, G, A, lda, B, ldb)) return;
        *ab = (size_t)(G.Mp * G.Kp * 8);
        *bb = (size_t)(G.Kp * G.Np * 8);
        return;
    }
    if (G.path == PATH_TC_I8_LIMBS) {
        long long kc; int nch;
        limb_chunks(G.Kp, &kc, &nch);
        *ab = (size_t)G.Mp * 8 * (size_t)(kc * nch);
        *bb = (size_t)G.Np * 8 * (size_t)(kc * nch);
        return;
    }
    *ab = (size_t)(G.Mp * G.Kp * G.shape.a_bytes_per_km / 1000);
    *bb = (size_t)(G.Kp * G.Np * G.shape.b_bytes_per_kn / 1000);
}

struct Exec {
    starmm_plan* P;
    cudaStream_t s;
    std::vector<Block> staged;
    int launches = 0;
    unsigned long long* oz_rowmax = nullptr;
    unsigned long long* oz_colmax = nullptr;
    int acquire(size_t bytes, void** p) {
        TRY(plan_acquire(P, bytes, s, p, false));
        staged.push_back({*p, bytes});
        return STARMM_OK;
    }
};

// Pack (or pad-copy) the operands of `G.path` into pa / pb.  rng: fold the range guard
// into the same pass.  Returns the operands the tile kernel reads.
int pack_operands(Exec& x, const Geom& G, const void* A, long long lda, const void* B, long long ldb,
                  void* pa, void* pb, unsigned long long* rng, Pred pr, const void** opA, long long* olda,
                  const void** opB, long long* oldb) {
    starmm_plan* P = x.P;
    cudaStream_t s = x.s;
    const long long Mp = G.Mp, Np = G.Np, Kp = G.Kp;
    *opA = A; *opB = B; *olda = lda; *oldb = ldb;
    int rc = STARMM_OK;
    if (G.path == PATH_MIN_ORDERED) return STARMM_OK;
    if (G.is_dmma) {
        if (dmma_direct(P, G, A, lda, B, ldb)) return STARMM_OK;
        pad_copy_kernel<double><<<grid2d(Mp, Kp), 256, 0, s>>>((const double*)A, P->m, P->k, lda,
                                                                (double*)pa, Mp, Kp, pr);
        pad_copy_kernel<double><<<grid2d(Kp, Np), 256, 0, s>>>((const double*)B, P->k, P->n, ldb,
                                                                (double*)pb, Kp, Np, pr);
        CK(cudaGetLastError());
        x.launches += 2;
        *opA = pa; *opB = pb; *olda = Kp; *oldb = Np;
        return STARMM_OK;
    }
    const float finf = std::numeric_limits<float>::infinity();
    const unsigned s16pad = 16383u | (16383u << 16);
    switch (G.path) {
    case PATH_SIMT_F32_PAIR:
        rc = launch_pack<float, float, 2, ConvIdentity>(A, lda, B, ldb, P->m, P->n, P->k, pa, pb,
                                                         Mp, Np, Kp, finf, s, rng, pr); break;
    case PATH_SIMT_I32_CARRIER:
        rc = launch_pack<int, float, 2, ConvI32ToF32>(A, lda, B, ldb, P->m, P->n, P->k, pa, pb,
                                                       Mp, Np, Kp, finf, s, rng, pr); break;
    case PATH_SIMT_I32_VMIN:
        rc = launch_pack<int, int, 1, ConvI32Vmin>(A, lda, B, ldb, P->m, P->n, P->k, pa, pb, Mp,
                                                    Np, Kp, (1 << 30) - 1, s, rng, pr); break;
    case PATH_SIMT_I32_SAT:
        rc = launch_pack<int, int, 1, ConvIdentity>(A, lda, B, ldb, P->m, P->n, P->k, pa, pb, Mp,
                                                     Np, Kp, 0x7fffffff, s, rng, pr); break;
    case PATH_SIMT_I64:
        rc = launch_pack<long long, long long, 1, ConvIdentity>(A, lda, B, ldb, P->m, P->n, P->k,
                                                                 pa, pb, Mp, Np, Kp, 0LL, s, rng, pr); break;
    case PATH_SIMT_I64_NARROW:
        rc = launch_pack<long long, int, 1, ConvI64ToI32>(A, lda, B, ldb, P->m, P->n, P->k, pa, pb,
                                                           Mp, Np, Kp, 0, s, rng, pr); break;
    case PATH_SIMT_F64_MIN: {
        const double dinf = std::numeric_limits<double>::infinity();
        rc = launch_pack<double, double, 1, ConvIdentity>(A, lda, B, ldb, P->m, P->n, P->k, pa,
                                                           pb, Mp, Np, Kp, dinf, s, rng, pr); break;
    }
    case PATH_SIMT_F64T_CARRIER:
        rc = launch_pack<double, float, 2, ConvF64ToF32>(A, lda, B, ldb, P->m, P->n, P->k, pa, pb,
                                                          Mp, Np, Kp, finf, s, rng, pr); break;
    // the narrow encodings below only ever run as a plan's first guess (never behind a
    // device-side verdict), so they take no predicate
    case PATH_SIMT_I64_DP4A:
        pack_a_s8x4_kernel<<<dim3((unsigned)((Kp / 4 + 31) / 32), (unsigned)(Mp / 32)), dim3(32, 8), 0, s>>>(
            (const long long*)A, P->m, P->k, lda, (int*)pa, Mp, Kp, rng);
        pack_b_s8x4_kernel<<<grid2d(Kp / 4, Np / 2), 256, 0, s>>>(
            (const long long*)B, P->k, P->n, ldb, (int*)pb, Np, Kp, rng);
        rc = cuda_status(cudaGetLastError());
        break;
    case PATH_TC_I8_LIMBS: {
        long long kc; int nch;
        limb_chunks(Kp, &kc, &nch);
        pack_limbs_rows_kernel<<<dim3((unsigned)((kc * nch / 8 + 255) / 256), (unsigned)std::min<long long>(Mp, 4096)), 256, 0, s>>>(
            (const long long*)A, P->m, P->k, lda, (signed char*)pa, Mp, kc, nch, rng, pr);
        pack_limbs_cols_kernel<<<dim3((unsigned)(Np / 32), (unsigned)((kc * nch + 31) / 32)), dim3(32, 8), 0, s>>>(
            (const long long*)B, P->k, P->n, ldb, (signed char*)pb, Np, kc, nch, rng, pr);
        rc = cuda_status(cudaGetLastError());
        break;
    }
    case PATH_TC_I8:
        pack_i8_rows_kernel<<<dim3((unsigned)((Kp / 8 + 255) / 256), (unsigned)std::min<long long>(Mp, 4096)), 256, 0, s>>>(
            (const long long*)A, P->m, P->k, lda, (signed char*)pa, Mp, Kp, rng);
        pack_i8_transpose_kernel<<<dim3((unsigned)(Np / 32), (unsigned)((Kp + 127) / 128)), dim3(32, 8), 0, s>>>(
            (const long long*)B, P->k, P->n, ldb, (signed char*)pb, Np, Kp, rng);
        rc = cuda_status(cudaGetLastError());
        break;
    case PATH_OZAKI_F64: {
        // scale pass (and the finiteness guard); residues are packed after the verdict
        TRY(x.acquire((size_t)Mp * 8, (void**)&x.oz_rowmax));
        TRY(x.acquire((size_t)Np * 8, (void**)&x.oz_colmax));
        CK(cudaMemsetAsync(x.oz_colmax, 0, (size_t)Np * 8, s));
        const int wpb = 8;
        oz_amax_rows_kernel<<<(unsigned)std::min<long long>((P->m + wpb - 1) / wpb, 148LL * 16), 32 * wpb, 0, s>>>(
            (const double*)A, P->m, P->k, lda, x.oz_rowmax, rng ? rng + 1 : nullptr);
        oz_amax_cols_kernel<<<dim3((unsigned)((P->n + 31) / 32), (unsigned)((P->k + 255) / 256)), dim3(32, 8), 0, s>>>(
            (const double*)B, P->k, P->n, ldb, x.oz_colmax, rng ? rng + 1 : nullptr);
        rc = cuda_status(cudaGetLastError());
        break;
    }
    case PATH_SIMT_F32_S16X2:
    case PATH_SIMT_I32_S16X2:
    case PATH_SIMT_F64T_S16X2: {
        const dim3 ga = pack_a_grid(Mp, Kp);
        if (G.path == PATH_SIMT_F64T_S16X2) {
            pack_a_kernel<double, unsigned, 1, ConvS16Dup><<<ga, dim3(32, 8), 0, s>>>(
                (const double*)A, P->m, P->k, lda, (unsigned*)pa, Mp, Kp, s16pad, rng);
            pack_b_s16x2_kernel<double><<<grid2d((Kp + 3) / 4, Np / 2), 256, 0, s>>>(
                (const double*)B, P->k, P->n, ldb, (unsigned*)pb, Np, Kp, rng);
        } else if (G.path == PATH_SIMT_F32_S16X2) {
            pack_a_kernel<float, unsigned, 1, ConvS16Dup><<<ga, dim3(32, 8), 0, s>>>(
                (const float*)A, P->m, P->k, lda, (unsigned*)pa, Mp, Kp, s16pad, rng);
            pack_b_s16x2_kernel<float><<<grid2d((Kp + 3) / 4, Np / 2), 256, 0, s>>>(
                (const float*)B, P->k, P->n, ldb, (unsigned*)pb, Np, Kp, rng);
        } else {
            pack_a_kernel<int, unsigned, 1, ConvS16Dup><<<ga, dim3(32, 8), 0, s>>>(
                (const int*)A, P->m, P->k, lda, (unsigned*)pa, Mp, Kp, s16pad, rng);
            pack_b_s16x2_kernel<int><<<grid2d((Kp + 3) / 4, Np / 2), 256, 0, s>>>(
                (const int*)B, P->k, P->n, ldb, (unsigned*)pb, Np, Kp, rng);
        }
        rc = cuda_status(cudaGetLastError());
        break;
    }
    }
    if (rc) return rc;
    x.launches += 2;
    *opA = pa; *opB = pb;
    return STARMM_OK;
}

template <class Sr>
int launch_ordered(const OrderedParams& op, long long tiles_m, long long tiles_n, cudaStream_t s) {
    const long long grid = std::max<long long>(1, std::min<long long>(tiles_m * tiles_n, 148LL * 6));
    minplus_ordered_kernel<Sr><<<(unsigned)grid, ordered::THREADS, 0, s>>>(op);
    CK(cudaGetLastError());
    return STARMM_OK;
}

// Everything after packing for one candidate path: Ozaki residues, protocol state
// (TileExclusionTable slots, pair states, lazy scratch, co3 workspace), identity fill,
// the tile kernel and the co3 merge -- every launch behind `pr`.  `ci` receives the
// candidate's stats.  ev: the candidate's timing pair (nullptr: untimed).
int launch_candidate(Exec& x, const Geom& G, void* C, long long ldc, const void* A, long long lda,
                     const void* B, long long ldb, const void* opA, long long olda, const void* opB,
                     long long oldb, Pred pr, cudaEvent_t* ev, CandInfo& ci) {
    starmm_plan* P = x.P;
    cudaStream_t s = x.s;
    const int eb = elem_bytes(P->sr);
    const bool init_identity = (P->flags & STARMM_F_INIT_IDENTITY) != 0;
    const int S = G.S, s_log2 = G.s_log2;
    const long long tiles = G.tiles, Mp = G.Mp, Np = G.Np, Kp = G.Kp;
    ci = CandInfo();
    ci.path = G.path;
    ci.tasks = G.ntasks;
    ci.S = S;
    ci.s_log2 = s_log2;
    ci.tar_levels = G.tar_levels;
    int rc = STARMM_OK;
    if (G.path == PATH_MIN_ORDERED) {
        OrderedParams op;
        op.A = A; op.lda = lda; op.B = B; op.ldb = ldb; op.C = C; op.ldc = ldc;
        op.M = P->m; op.N = P->n; op.K = P->k;
        op.blk = P->base_dim; op.kofs = P->kofs;
        op.init_identity = init_identity ? 1 : 0;
        op.pr = pr;
        if (ev && (rc = cuda_status(cudaEventRecord(ev[0], s)))) return rc;
        rc = P->sr == STARMM_SR_TROPICAL_F32 ? launch_ordered<SrTropF32>(op, G.tiles_m, G.tiles_n, s)
                                             : launch_ordered<SrTropF64>(op, G.tiles_m, G.tiles_n, s);
        if (rc) return rc;
        if (ev && (rc = cuda_status(cudaEventRecord(ev[1], s)))) return rc;
        ++x.launches;
        ci.workers = std::min<long long>(G.ntasks, (long long)P->sms * 8);
        return STARMM_OK;
    }
    if (G.path == PATH_OZAKI_F64) {   // residue planes for the scales the guard pass found
        const int t = ozaki_bits(P->k);
        oz_pack_rows_kernel<<<dim3((unsigned)((Kp / 4 + 255) / 256), (unsigned)std::min<long long>(Mp, 65535)), 256, 0, s>>>(
            (const double*)A, P->m, P->k, lda, x.oz_rowmax, t, (signed char*)opA, Mp, Kp, pr);
        oz_pack_cols_kernel<<<dim3((unsigned)(Np / 32), (unsigned)(Kp / 64)), dim3(32, 8), 0, s>>>(
            (const double*)B, P->k, P->n, ldb, x.oz_colmax, t, (signed char*)opB, Np, Kp, pr);
        CK(cudaGetLastError());
        x.launches += 2;
    }
    const bool cluster = G.is_dmma && dmma_cluster_mode(P, S);
    // ---- per-run protocol state: slots (TileExclusionTable), pair states ----
    const bool need_slots = !cluster && (S > 1) && (P->algo == STARMM_SAR || P->algo == STARMM_STAR);
    void* pstate = nullptr;
    const size_t state_bytes = need_slots ? (size_t)(tiles + tiles * (S / 2)) * 4 : 0;
    if (need_slots) {
        TRY(x.acquire(state_bytes, &pstate));
        CK(cudaMemsetAsync(pstate, 0, state_bytes, s));
    }
    // per-worker lazy-temp blocks (tile sized, for SAR/STAR pairs)
    void* wscratch = nullptr;
    const long long tile_elems = (long long)G.TBM * G.TBN;
    if (need_slots) TRY(x.acquire((size_t)(G.gpu_workers * tile_elems * eb), &wscratch));
    // co3 workspace D_1..D_{S-1}: pooled (the device pool, reused) or raw (fresh per call)
    void* W = nullptr;
    size_t wbytes = 0;
    if (P->algo == STARMM_CO3 && S > 1) {
        wbytes = (size_t)(S - 1) * (size_t)P->m * (size_t)P->n * eb;
        if (P->alloc == STARMM_POOLED) {
            TRY(plan_acquire(P, wbytes, s, &W, true));
            x.staged.push_back({W, wbytes});
        } else {
            CK(cudaMallocAsync(&W, wbytes, s));
            ci.raw_count = 1;
            ci.raw_bytes = (long long)wbytes;
        }
        P->ws_high_water = std::max<long long>(P->ws_high_water, (long long)wbytes);
    }
    if (init_identity && (S > 1 || G.balanced) && P->algo != STARMM_CO3 && P->remote_parts == 0 && !cluster) {
        TRY(fill_dispatch(P->sr, C, P->m, P->n, ldc, s, pr));
        ++x.launches;
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

    const int grid = occupancy_grid(P, G.per_sm, G.balanced ? G.ntasks * G.g.kstages : G.ntasks);
    if (ev && (rc = cuda_status(cudaEventRecord(ev[0], s)))) return rc;
    if (G.path == PATH_TC_I8) {
        EpiFoldI64 e;
        e.o = tcg_out(P, C, ldc, init_identity);
        TRY(launch_tcg(opA, opB, Mp, Np, Kp, 1, e, P->sms, s,
                       [&](size_t b, void** p) { return x.acquire(b, p); }, pr));
    } else if (G.path == PATH_TC_I8_LIMBS) {
        // per K chunk, the 8 digit groups: group s = one int8 GEMM over (s + 1) Kc of A's
        // digits 0..s against B's digits s..0, its int32 result folded as << 8s (mod 2^64)
        long long kc; int nch;
        limb_chunks(Kp, &kc, &nch);
        for (int ch = 0; ch < nch; ++ch)
            for (int sg = 0; sg < 8; ++sg) {
                EpiFoldI64 e;
                e.o = tcg_out(P, C, ldc, init_identity && ch == 0 && sg == 0);
                e.shift = 8 * sg;
                const signed char* a = (const signed char*)opA + (size_t)ch * Mp * 8 * kc;
                const signed char* b = (const signed char*)opB + (size_t)ch * Np * 8 * kc + (size_t)(7 - sg) * kc;
                TRY(launch_tcg(a, b, Mp, Np, (sg + 1) * kc, 1, e, P->sms, s,
                               [&](size_t bb, void** p) { return x.acquire(bb, p); }, pr, 8 * kc));
                if (ch || sg) ++x.launches;
            }
    } else if (G.path == PATH_OZAKI_F64) {
        void* planes = nullptr;
        TRY(x.acquire((size_t)oz::P * Mp * Np, &planes));
        EpiOzakiResidues e;
        e.R = (unsigned char*)planes; e.Mp = Mp; e.Np = Np;
        TRY(launch_tcg(opA, opB, Mp, Np, Kp, oz::P, e, P->sms, s,
                       [&](size_t b, void** p) { return x.acquire(b, p); }, pr));
        if (ev && (rc = cuda_status(cudaEventRecord(ev[1], s)))) return rc;
        const long long groups = (P->n + OZ_CRT_W - 1) / OZ_CRT_W;
        oz_crt_kernel<<<dim3((unsigned)((groups + 127) / 128), (unsigned)std::min<long long>(P->m, 65535)), 128, 0, s>>>(
            (const unsigned char*)planes, Mp, Np, x.oz_rowmax, x.oz_colmax, ozaki_bits(P->k), ozaki_crt(),
            tcg_out(P, C, ldc, init_identity), pr);
        CK(cudaGetLastError());
        ++x.launches;
    } else if (G.is_dmma) {
        DmmaParams dp;
        dp.A = (const double*)opA; dp.lda = olda; dp.B = (const double*)opB; dp.ldb = oldb;
        dp.g = G.g; dp.w = w;
        dp.gate = P->d_gate;
        dp.pr = pr;
        // Wave gate: off by default since the one-CTA-per-SM 256x64 kernel keeps its
        // persistent CTAs close enough on its own (58 GB of DRAM reads per n=16384
        // launch without, 53 GB with, at -0.1..0.3%; the two-CTA 64x128 kernel needed
        // it: 250 -> 51 GB).  STARMM_DMMA_GATE=1 turns it on; it needs the whole grid
        // co-resident and pays only over several waves, and the host path's
        // overlapping launches never use it.
        if (cluster) {
            TRY(launch_dmma_cluster(dp, S, tiles, s));
        } else if (G.balanced) {
            static bool bal_attr[starmm_host::MAX_DEVICES] = {};
            const int dev = current_device();
            if (!bal_attr[dev]) {
                CK(cudaFuncSetAttribute(dmma_fp64_balanced_kernel<DmmaProd>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, DmmaProd::SMEM_BYTES));
                bal_attr[dev] = true;
            }
            dmma_fp64_balanced_kernel<DmmaProd><<<grid, DmmaProd::THREADS, DmmaProd::SMEM_BYTES, s>>>(dp);
            CK(cudaGetLastError());
        } else {
            const char* genv = getenv("STARMM_DMMA_GATE");
            const bool gate = genv && genv[0] == '1' && P->dmma_gate && G.ntasks >= 4LL * grid;
            TRY(launch_dmma(dp, grid, gate, s));
        }
    } else {
        SimtParams sp;
        sp.Ap = opA; sp.Bp = opB; sp.Mp = Mp; sp.Np = Np; sp.g = G.g; sp.w = w;
        sp.pr = pr;
        // k-outer chunks: when the A and B panels one wave of persistent CTAs streams
        // exceed the L2 many times over, the CTAs drift apart in k and every wave re-reads
        // its panels from DRAM (config 5, n = 49152: 3.96 TB per launch for 38.6 GB of
        // operands, profiles/r02j_ncu_summary.md).  Running the k range as a few chunks,
        // each one launch over all tiles that folds into C (CO2's serialised k-halves,
        // classic.py:125-128, taken at the top level), keeps a wave's panels L2-sized for
        // the price of one C read-modify-write per chunk.
        const int nchunk = simt_k_chunks(P, G);
        if (nchunk <= 1) {
            // the CUDA-core tile kernels are instantiated in simt_launch_*.cu (parallel build)
            CK((cudaError_t)starmm_simt_launch(G.path, sp, grid, P->sms, s));
        } else {
            const int KSTEP = simt_kstep(G.path), GG = simt_g(G.path), OUTS = G.shape.bn / 128;
            const long long kc = round_up((Kp + nchunk - 1) / nchunk, G.BK);
            const size_t ea = (size_t)G.shape.a_bytes_per_km * KSTEP / 1000 / GG;   // bytes per packed element
            for (long long k0 = 0; k0 < Kp; k0 += kc) {
                const long long kl = std::min(kc, Kp - k0);
                SimtParams sc = sp;
                sc.Ap = (const char*)opA + (size_t)(k0 / KSTEP) * (size_t)Mp * GG * ea;
                sc.Bp = (const char*)opB + (size_t)(k0 / KSTEP) * (size_t)(Np / OUTS) * GG * ea;
                sc.g.kslice = kl;
                sc.g.kstages = kl / G.BK;
                if (k0 > 0) sc.w.init_identity = 0;           // later chunks fold
                CK((cudaError_t)starmm_simt_launch(G.path, sc, grid, P->sms, s));
                if (k0 > 0) ++x.launches;
            }
            ci.k_chunks = nchunk;
        }

    }
    ++x.launches;
    if (ev && G.path != PATH_OZAKI_F64 && (rc = cuda_status(cudaEventRecord(ev[1], s)))) return rc;

    // ---- co3: merge the workspace bottom-up (merge_tasks, ops.py:108-155) ----
    if (P->algo == STARMM_CO3 && S > 1) {
        const long long slab = P->m * P->n;
        for (int lvl = s_log2; lvl >= 1; --lvl) {
            const int step = 1 << (s_log2 - lvl);
            for (int xx = step; xx < S; xx += 2 * step) {
                char* src = (char*)W + (size_t)(xx - 1) * slab * eb;
                const int tgt = xx - step;
                if (tgt == 0) rc = madd_dispatch(P->sr, C, ldc, src, P->n, P->m, P->n, 0, s, 0, pr);
                else rc = madd_dispatch(P->sr, (char*)W + (size_t)(tgt - 1) * slab * eb, P->n, src,
                                        P->n, P->m, P->n, 0, s, 0, pr);
                if (rc) return rc;
                ++x.launches;
            }
        }
        if (P->alloc == STARMM_RAW) CK(cudaFreeAsync(W, s));
    }
    ci.workers = std::min<long long>(G.ntasks, (long long)P->sms * G.per_sm);
    if (cluster) ci.workers = std::min<long long>(tiles, dmma_cluster_slots(S)) * S;
    ci.cluster = cluster ? S : 0;
    ci.balanced_workers = G.balanced ? std::min<long long>(G.ntasks * G.g.kstages, (long long)P->sms * G.per_sm) : 0;
    if (G.balanced) ci.workers = ci.balanced_workers;    // every CTA of the grid owns a slice
    if (!cluster && S > 1 && (P->algo == STARMM_SAR || P->algo == STARMM_STAR) && G.tar_levels < s_log2)
        ci.pair_count = tiles * (S / 2);
    return STARMM_OK;
}

// widest exact path of the semiring (no range condition), and the fastest one to try first
int general_path(const starmm_plan* P) {
    switch (P->sr) {
    case STARMM_SR_FP64: return PATH_DMMA_F64;
    case STARMM_SR_INT64: return (P->flags & STARMM_F_INT_TENSOR) ? PATH_TC_I8_LIMBS : PATH_SIMT_I64;
    case STARMM_SR_TROPICAL_F64: return PATH_SIMT_F64_MIN;
    case STARMM_SR_TROPICAL_F32: return PATH_SIMT_F32_PAIR;
    default: return PATH_SIMT_I32_SAT;
    }
}
// the exact fallback queued behind a device-side verdict: cheap to launch predicated off.
// For int-tensor plans that is the CUDA-core 64-bit kernel (2 packers + 1 tile launch),
// not the radix-256 digit path (8 tcgen05 launches per K chunk, each with its own
// tensor maps and gate reset: ~30% of a small config-2 step when skipped); the next call
// starts from the digit path when the verdict says the data needs it.
int fallback_path(const starmm_plan* P) {
    if (P->sr == STARMM_SR_INT64) return PATH_SIMT_I64;
    return general_path(P);
}

int fastest_path(const starmm_plan* P) {
    const bool fast = !(P->flags & STARMM_F_NO_FASTPATH);
    if (!fast) return general_path(P);
    switch (P->sr) {
    case STARMM_SR_FP64: return (P->flags & STARMM_F_FP64_EMU) && P->k < (1LL << 17) ? PATH_OZAKI_F64 : PATH_DMMA_F64;
    case STARMM_SR_INT64: return (P->flags & STARMM_F_INT_TENSOR) ? PATH_TC_I8 : PATH_SIMT_I64_DP4A;
    case STARMM_SR_TROPICAL_F64: return PATH_SIMT_F64T_S16X2;
    case STARMM_SR_TROPICAL_F32: return PATH_SIMT_F32_S16X2;
    default: return PATH_SIMT_I32_S16X2;
    }
}
bool float_min(const starmm_plan* P) {
    return P->sr == STARMM_SR_TROPICAL_F64 || P->sr == STARMM_SR_TROPICAL_F32;
}
// does this call need the range guard?  (a fast path to confirm, or -0.0 to detect)
bool needs_guard(const starmm_plan* P) {
    if (fastest_path(P) != general_path(P)) return true;
    return float_min(P) && P->remote_parts == 0;
}

}  // namespace

// Resolve timed records: every one (block = true) or those already complete.
static int resolve_timed(starmm_plan* P, bool block) {
    size_t done = 0;
    for (; done < P->timed.size(); ++done) {
        auto& r = P->timed[done];
        const cudaEvent_t last = r.ev[2 * r.ncand - 1];
        if (block) CK(cudaEventSynchronize(last));
        else if (cudaEventQuery(last) != cudaSuccess) { cudaGetLastError(); break; }
        int ran = r.ran;
        if (ran < 0) {
            ran = 0;
            const int sel = (int)P->ring[r.slot];
            for (int c = 0; c < r.ncand; ++c)
                if (r.path[c] == sel) ran = c;
            P->st.path = sel;
        }
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, r.ev[2 * ran], r.ev[2 * ran + 1]));
        P->st.main_kernel_ns += (int64_t)((double)ms * 1e6);
        P->st.main_kernel_launches += 1;
        for (int i = 0; i < 2 * r.ncand; ++i) P->ev_pool.push_back(r.ev[i]);
    }
    P->timed.erase(P->timed.begin(), P->timed.begin() + (long)done);
    return STARMM_OK;
}

// force_async: the caller synchronises (host path, Strassen leaves).  host_guard: read
// the range guard on the host every call -- the host-buffer schedule, whose row blocks
// alternate between two compute streams: a predicated-off fallback TILE kernel still
// needs SM slots to start and exit, so queued behind the other stream's persistent
// kernel it would hold back this stream's downloads (config 3 e2e 54 -> 49.5 Tops/s);
// that schedule is a blocking call anyway.
static int execute_impl(starmm_plan* P, void* C, int64_t ldc, const void* A, int64_t lda,
                        const void* B, int64_t ldb, void* stream, bool force_async,
                        bool host_guard = false) {
    if (!P || !C || !A || !B) return STARMM_CONTRACT_VIOLATION;
    if (ldc < P->n || lda < P->k || ldb < P->n) return STARMM_DIM_MISMATCH;
    const int eb = elem_bytes(P->sr);
    if (((uintptr_t)C | (uintptr_t)A | (uintptr_t)B) % eb) return STARMM_ALIGNMENT_ERROR;
    DeviceGuard dg;
    TRY(dg.set(P->device));
    cudaStream_t s = (cudaStream_t)stream;
    TRY(ensure_bookkeeping(P, s));
    const bool async = (P->flags & STARMM_F_ASYNC) || force_async;
    const bool timed = (P->flags & STARMM_F_TIME_MAIN) != 0;
    starmm_plan::TimedRec rec{};
    if (timed) {
        TRY(resolve_timed(P, false));                  // recycle what has completed
        if (P->timed.size() >= 64) TRY(resolve_timed(P, true));
        if (!P->ring) {
            void* h = nullptr;
            CK(cudaHostAlloc(&h, 64 * sizeof(unsigned long long), cudaHostAllocMapped));
            P->ring = (unsigned long long*)h;
            CK(cudaHostGetDevicePointer((void**)&P->ring_dev, h, 0));
        }
        for (int i = 0; i < 6; ++i) {
            if (P->ev_pool.empty()) {
                cudaEvent_t e;
                CK(cudaEventCreate(&e));
                P->ev_pool.push_back(e);
            }
            rec.ev[i] = P->ev_pool.back();
            P->ev_pool.pop_back();
        }
        rec.slot = P->ring_next;
        P->ring_next = (P->ring_next + 1) % 64;
    }
    // an earlier call's device-side verdict (mapped host word; stale is fine: a hint)
    if (P->spec_used && P->hs[3]) P->hint = (int)P->hs[3];
    const bool ordered_ok = P->remote_parts == 0;

    // ---- path selection ------------------------------------------
    // Range-guarded exact narrow paths are chosen optimistically: the operands are
    // packed for the fastest path (or the one the last verdict allowed) while the
    // packers reduce max|x| (and float integrality / -0.0) in the same pass.  The
    // verdict is then taken ON THE DEVICE (select_path_kernel) and the exact fallback
    // candidates -- the semiring's general kernel, and for the float (min,+) semirings
    // the ordered kernel -- are queued behind it with a predicate; exactly one runs.
    // Only a plan's first blocking call (no verdict to go on yet) reads the guard on
    // the host, so that it picks the narrowest path at once.
    Exec x{P, s};
    int rc = STARMM_OK;
    CandInfo info[3];
    int ncand = 0;
    bool host_decided = true;
    const char* genv = getenv("STARMM_GUARD_SYNC");      // 1: always host-side, 0: never
    do {
        if (!needs_guard(P)) {
            Geom G;
            if ((rc = plan_geometry(P, general_path(P), G))) break;
            size_t ab, bb;
            packed_bytes(P, G, A, lda, B, ldb, &ab, &bb);
            void *pa = nullptr, *pb = nullptr;
            if (ab && (rc = x.acquire(ab, &pa))) break;
            if (bb && (rc = x.acquire(bb, &pb))) break;
            const void *opA, *opB;
            long long olda, oldb;
            if ((rc = pack_operands(x, G, A, lda, B, ldb, pa, pb, nullptr, Pred(), &opA, &olda, &opB, &oldb))) break;
            rc = launch_candidate(x, G, C, ldc, A, lda, B, ldb, opA, olda, opB, oldb, Pred(),
                                  timed ? &rec.ev[0] : nullptr, info[0]);
            ncand = 1;
            break;
        }
        int first = (P->hint && P->hint != PATH_MIN_ORDERED) ? P->hint : fastest_path(P);
        const bool host_sync = genv ? genv[0] == '1' : (host_guard || (!async && P->hint == 0));
        if (host_sync) {
            // ---- host-side verdict: pack, read the guard, re-pack if it disallows ----
            bool guard_pending = true;
            for (;;) {
                Geom G;
                if ((rc = plan_geometry(P, first, G))) break;
                size_t ab, bb;
                packed_bytes(P, G, A, lda, B, ldb, &ab, &bb);
                void *pa = nullptr, *pb = nullptr;
                if (ab && (rc = x.acquire(ab, &pa))) break;
                if (bb && (rc = x.acquire(bb, &pb))) break;
                unsigned long long* rng = guard_pending ? P->d_range : nullptr;
                if (rng && (rc = cuda_status(cudaMemsetAsync(rng, 0, 2 * sizeof(unsigned long long), s)))) break;
                const void *opA, *opB;
                long long olda, oldb;
                if ((rc = pack_operands(x, G, A, lda, B, ldb, pa, pb, rng, Pred(), &opA, &olda, &opB, &oldb))) break;
                if (guard_pending) {
                    publish_range_kernel<<<1, 32, 0, s>>>(P->d_range, P->hs_dev);
                    if ((rc = cuda_status(cudaGetLastError()))) break;
                    if ((rc = cuda_status(cudaStreamSynchronize(s)))) break;
                    ++x.launches;
                    ++P->st.guard_syncs;
                    guard_pending = false;
                    const int nar = guard_narrowest(P->sr, P->flags, P->k, P->hs[0], P->hs[1], ordered_ok);
                    P->hint = nar;
                    if (nar != first) { first = nar; continue; }   // re-pack for the allowed path
                }
                rc = launch_candidate(x, G, C, ldc, A, lda, B, ldb, opA, olda, opB, oldb, Pred(),
                                      timed ? &rec.ev[0] : nullptr, info[0]);
                ncand = 1;
                break;
            }
            break;
        }
        // ---- device-side verdict: first guess + predicated exact fallbacks ----
        host_decided = false;
        int cands[3] = {first, 0, 0};
        ncand = 1;
        const int general = fallback_path(P);
        if (general != first) cands[ncand++] = general;
        if (float_min(P) && ordered_ok) cands[ncand++] = PATH_MIN_ORDERED;
        Geom G[3];
        size_t abmax = 0, bbmax = 0;
        for (int c = 0; c < ncand && !rc; ++c) {
            rc = plan_geometry(P, cands[c], G[c]);
            size_t ab, bb;
            packed_bytes(P, G[c], A, lda, B, ldb, &ab, &bb);
            abmax = std::max(abmax, ab);
            bbmax = std::max(bbmax, bb);
        }
        if (rc) break;
        // every candidate packs into the same staging: a fallback's packers only run when
        // the first guess's kernel does not
        void *pa = nullptr, *pb = nullptr;
        if (abmax && (rc = x.acquire(abmax, &pa))) break;
        if (bbmax && (rc = x.acquire(bbmax, &pb))) break;
        if ((rc = cuda_status(cudaMemsetAsync(P->d_range, 0, 2 * sizeof(unsigned long long), s)))) break;
        const void *opA[3], *opB[3];
        long long olda[3], oldb[3];
        if ((rc = pack_operands(x, G[0], A, lda, B, ldb, pa, pb, P->d_range, Pred(), &opA[0], &olda[0],
                                &opB[0], &oldb[0]))) break;
        select_path_kernel<<<1, 32, 0, s>>>(P->d_range, P->sr, P->flags, P->k, first, general,
                                            ordered_ok ? 1 : 0, P->d_sel, P->hs_dev,
                                            timed ? P->ring_dev + rec.slot : nullptr);
        if ((rc = cuda_status(cudaGetLastError()))) break;
        ++x.launches;
        P->spec_used = true;
        for (int c = 0; c < ncand && !rc; ++c) {
            const Pred pr{P->d_sel, (unsigned)cands[c]};
            if (c > 0 && (rc = pack_operands(x, G[c], A, lda, B, ldb, pa, pb, nullptr, pr, &opA[c], &olda[c],
                                             &opB[c], &oldb[c]))) break;
            rc = launch_candidate(x, G[c], C, ldc, A, lda, B, ldb, opA[c], olda[c], opB[c], oldb[c], pr,
                                  timed ? &rec.ev[2 * c] : nullptr, info[c]);
        }
    } while (0);

    // staging blocks go back to the device pool, fenced by the work queued so far
    FenceRef fence = P->ctx->arena.fence(s);
    for (auto it = x.staged.rbegin(); it != x.staged.rend(); ++it) P->ctx->arena.release(it->p, fence);
    plan_note_fence(P, fence);
    if (rc) return rc;
    if (!async) CK(cudaStreamSynchronize(s));
    // which candidate ran: known now if the host decided or the call was blocking
    int ran = 0;
    if (!host_decided && !async) {
        const int sel = (int)P->hs[2];
        for (int c = 0; c < ncand; ++c)
            if (info[c].path == sel) ran = c;
        if (P->hs[3]) P->hint = (int)P->hs[3];
    }
    const CandInfo& ci = info[ran];
    if (timed) {
        rec.ncand = ncand;
        for (int c = 0; c < ncand; ++c) rec.path[c] = info[c].path;
        rec.ran = (host_decided || !async) ? ran : -1;
        for (int i = 2 * ncand; i < 6; ++i) P->ev_pool.push_back(rec.ev[i]);   // unused pairs
        P->timed.push_back(rec);
        if (!async) TRY(resolve_timed(P, true));
    }
    P->raw_count += ci.raw_count;
    P->raw_bytes += ci.raw_bytes;
    P->st.tasks = ci.tasks;
    P->st.workers = ci.workers;
    P->st.ksplit = ci.S;
    P->st.balanced_workers = ci.balanced_workers;
    P->st.tar_levels = ci.tar_levels;
    P->st.kernel_launches = x.launches;
    P->st.path = ci.path;
    P->st.executes += 1;
    P->st.pair_count += ci.pair_count;
    P->st.candidates = ncand;
    P->st.cluster_size = ci.cluster;
    P->st.k_chunks = ci.k_chunks;
    return STARMM_OK;
}

extern "C" {

// ============================================================================

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
        TRY(plan_acquire(x.P, bytes, x.s, out, true));
    }
    x.P->str_issued += (long long)bytes;
    x.P->ws_high_water = std::max(x.P->ws_high_water, x.P->str_issued);
    return STARMM_OK;
}

void str_release(StrCtx& x, void* p, long long n) {
    size_t bytes = (size_t)(n * n) * x.eb;
    if (x.P->alloc == STARMM_RAW) cudaFreeAsync(p, x.s);
    else x.P->ctx->arena.release(p, nullptr);   // LIFO: the next same-size acquire gets it back
                                                // (same stream: stream order protects it)
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
    DeviceGuard dg;
    TRY(dg.set(P->device));
    TRY(ensure_bookkeeping(P, (cudaStream_t)stream));
    StrCtx x{P, (cudaStream_t)stream, (size_t)elem_bytes(P->sr),
             std::max<long long>(P->base_dim, P->strassen_leaf), switch_depth(P->workers), 0};
    int rc = str_mm(x, 0, MM_STORE, C, ldc, A, lda, B, ldb, P->n);
    if (!rc && !(P->flags & STARMM_F_ASYNC)) rc = cuda_status(cudaStreamSynchronize(x.s));
    P->st.kernel_launches = x.launches;
    P->st.executes += 1;
    plan_note_fence(P, P->ctx->arena.fence(x.s));
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
                              long long base_dim, std::vector<long long>& kb) {
    kb.assign(1, 0);
    const char* env = getenv("STARMM_HOST_PHASE1");
    if ((env && env[0] == '0') || m < 512 || k < 512) return 0;
    const double t_mm = 2.0 * (double)m * (double)n * (double)k / host_nominal_ops(sr);
    if (!(env && env[0] == '1') && t_mm < h2d_bytes / 50e9) return 0;
    // first chunk k/64 (k >= 8192) or k/32: its upload is the exposed head of the schedule
    const long long div = (k >= 8192 && sr == STARMM_SR_FP64) ? 64 : 32;   // DMMA calls have no packing / guard
    // widths are multiples of the leaf size (and of 128): a leaf never straddles two
    // calls, so the ordered kernel's per-leaf minima are the reference's
    const long long cq = std::max<long long>(128, base_dim);
    long long w = std::max<long long>(cq, round_up((k + div - 1) / div, cq)), sum = 0;
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
    // chunk widths are multiples of the leaf size, so leaves never straddle two calls
    const long long cq = std::max<long long>(128, P->base_dim);
    for (long long w = std::max<long long>(cq, round_up((k + 31) / 32, cq)); kb.back() < k; w *= 2)
        kb.push_back(std::min(k, kb.back() + w));
    const int nq = (int)kb.size() - 1;
    cudaStream_t cs = (cudaStream_t)stream, up = nullptr;
    TRY(res.stream(&up));
    std::vector<cudaEvent_t> ev(nq);
    for (auto& e : ev) TRY(res.event(&e));
    // the uploads are ordered after everything already queued on the caller's stream
    // (it may still be producing the pinned inputs)
    cudaEvent_t ev_entry = nullptr;
    TRY(res.event(&ev_entry));
    CK(cudaEventRecord(ev_entry, cs));
    CK(cudaStreamWaitEvent(up, ev_entry, 0));
    void *dA = nullptr, *dB = nullptr;
    const size_t a_bytes = (size_t)m * k * eb, b_bytes = (size_t)k * n * eb;
    int rc = STARMM_OK;
    const int saved_flags = P->flags;
    do {
        if ((rc = plan_acquire(P, a_bytes, up, &dA, false))) break;
        if ((rc = plan_acquire(P, b_bytes, up, &dB, false))) break;
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
            P->kofs = k0;
            // (C is not touched: every write-back goes to the peers)
            rc = execute_impl(P, dA, n, (char*)dA + k0 * eb, k, (char*)dB + k0 * n * eb, n, cs, true, true);
            P->k = k;
            P->kofs = 0;
        }
        if (rc) break;
        rc = cuda_status(cudaStreamSynchronize(cs));
    } while (0);
    P->k = k; P->kofs = 0; P->flags = saved_flags;
    cudaStreamSynchronize(up);
    cudaStreamSynchronize(cs);
    if (dB) P->ctx->arena.release(dB, nullptr);
    if (dA) P->ctx->arena.release(dA, nullptr);
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
    const int nq = host_phase1_chunks(m, n, k, P->sr, h2d, P->base_dim, kb);
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
    // the copy streams start after everything already queued on the caller's stream
    // (it may still be producing the pinned inputs or reading C)
    cudaEvent_t ev_entry = nullptr;
    TRY(res.event(&ev_entry));
    CK(cudaEventRecord(ev_entry, cs));
    CK(cudaStreamWaitEvent(up, ev_entry, 0));
    CK(cudaStreamWaitEvent(down, ev_entry, 0));
    void *dA = nullptr, *dB = nullptr, *dC = nullptr, *dC0 = nullptr;
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
        Q->kofs = (long long)((const char*)Bd - (const char*)dB) / (long long)(n * eb);   // leaf alignment
        if (kk == k - kq && ks2 >= -1) Q->ksplit_req = ks2;   // phase-2 split override (tuning)
        // (STARMM_F_TIME_MAIN would synchronise the host after every launch and serialise the
        // schedule, so the host path never times its kernels)
        const int f = saved_flags & ~STARMM_F_TIME_MAIN;
        Q->flags = store ? (f | STARMM_F_INIT_IDENTITY) : (f & ~STARMM_F_INIT_IDENTITY);
        int r = execute_impl(Q, Cd, n, Ad, k, Bd, n, st, true, true);
        Q->m = m; Q->k = k; Q->kofs = 0; Q->flags = saved_flags; Q->ksplit_req = saved_ks;
        return r;
    };
    do {
        if ((rc = plan_acquire(P, a_bytes, up, &dA, false))) break;
        if (!same_ab && (rc = plan_acquire(P, b_bytes, up, &dB, false))) break;
        if (same_ab) dB = dA;
        if ((rc = plan_acquire(P, c_bytes, up, &dC, false))) break;
        if (staged_c0 && (rc = plan_acquire(P, c_bytes, up, &dC0, false))) break;
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
                // C0 comes first in the reference's fold sequence: Cb <- C0 (+) Cb
                if ((rc = madd_dispatch(P->sr, Cb, n, (char*)dC0 + r0 * n * eb, n, rows, n, 0, sb, 1))) break;
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
    // (every stream was synchronised above: the blocks are free on the device)
    if (dC0) P->ctx->arena.release(dC0, nullptr);
    if (dC) P->ctx->arena.release(dC, nullptr);
    if (dB && !same_ab) P->ctx->arena.release(dB, nullptr);
    if (dA) P->ctx->arena.release(dA, nullptr);
    return rc;
}

// Semiring.matmul (semiring.py:92-94): out <- A (x) B from the additive identity, one
// product over the whole K (the reference's numba kernel is one leaf: its first minimum
// over k wins, so the plan's leaf size is K rounded up to a power of two).  Plans are
// cached per device by shape and flags -- a call costs launches, not plan setup, and
// the range guard's verdict carries over from call to call.  A cached plan is taken out
// of the cache while a thread uses it.
int starmm_matmul(int semiring, void* out, int64_t ldo, const void* A, int64_t lda, const void* B,
                  int64_t ldb, int64_t m, int64_t n, int64_t k, void* stream, int flags) {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if (dev < 0 || dev >= starmm_host::MAX_DEVICES) return STARMM_CONTRACT_VIOLATION;
    const int pf = flags | STARMM_F_INIT_IDENTITY | STARMM_F_ALLOW_NONPOW2;
    int leaf = 1;
    while (leaf < k && leaf < (1 << 30)) leaf <<= 1;
    starmm_plan* P = nullptr;
    {
        std::lock_guard<std::mutex> g(g_mm_mu);
        auto& c = g_mm_cache[dev];
        for (size_t i = c.size(); i-- > 0;) {
            starmm_plan* q = c[i];
            if (q->sr == semiring && q->m == m && q->n == n && q->k == k && q->flags == pf) {
                P = q;
                c.erase(c.begin() + (long)i);
                break;
            }
        }
    }
    if (!P) TRY(starmm_plan_create(&P, semiring, STARMM_CO2, STARMM_POOLED, m, n, k, leaf, 1, 0, dev, pf));
    const int rc = starmm_execute(P, out, ldo, A, lda, B, ldb, stream);
    starmm_plan* evict = nullptr;
    {
        std::lock_guard<std::mutex> g(g_mm_mu);
        auto& c = g_mm_cache[dev];
        c.push_back(P);                                   // most recently used last
        if (c.size() > 32) { evict = c.front(); c.erase(c.begin()); }
    }
    if (evict) starmm_plan_destroy(evict);
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

// ---- the device block pool (pool.py:67-167) --------------------------------
int starmm_pool_acquire(int device, int64_t bytes, void* stream, void** out, int* fresh) {
    if (!out || bytes <= 0) return STARMM_CONTRACT_VIOLATION;
    *out = nullptr;
    DeviceCtx* c = device_ctx(device);
    if (!c) return STARMM_CONTRACT_VIOLATION;
    DeviceGuard dg;
    TRY(dg.set(device));
    bool f = false;
    CK(c->arena.acquire((size_t)bytes, (cudaStream_t)stream, out, &f));
    if (fresh) *fresh = f ? 1 : 0;
    return STARMM_OK;
}

int starmm_pool_release(int device, void* block, void* stream) {
    DeviceCtx* c = device_ctx(device);
    if (!c || !block) return STARMM_CONTRACT_VIOLATION;
    if (!c->arena.owns(block)) return STARMM_CONTRACT_VIOLATION;   // pool.py:120-127
    DeviceGuard dg;
    TRY(dg.set(device));
    c->arena.release(block, c->arena.fence((cudaStream_t)stream));
    return STARMM_OK;
}

int starmm_pool_counts_get(int device, starmm_pool_counts* out) {
    DeviceCtx* c = device_ctx(device);
    if (!c || !out) return STARMM_CONTRACT_VIOLATION;
    std::lock_guard<std::mutex> g(c->arena.mu);
    const starmm_host::PoolCounts& k = c->arena.c;
    out->allocated_bytes = k.allocated; out->cached_bytes = k.cached; out->issued_bytes = k.issued;
    out->high_water_bytes = k.high_water; out->fresh_count = k.fresh; out->reuse_count = k.reuse;
    out->cross_stream_waits = k.waits; out->trims = k.trims;
    return STARMM_OK;
}

int starmm_pool_reset(int device) {
    DeviceCtx* c = device_ctx(device);
    if (!c) return STARMM_CONTRACT_VIOLATION;
    DeviceGuard dg;
    TRY(dg.set(device));
    // cached one-shot matmul plans hold pool blocks: drop them first
    std::vector<starmm_plan*> drop;
    {
        std::lock_guard<std::mutex> g(g_mm_mu);
        drop.swap(g_mm_cache[device]);
    }
    for (auto* p : drop) starmm_plan_destroy(p);
    c->arena.reset();
    return STARMM_OK;
}

// ---- input generation (generate.cuh) ----------------------------------------
int starmm_generate(int semiring, int dist, void* out, int64_t ld, int64_t rows, int64_t cols,
                    int64_t row0, int64_t col0, uint64_t seed, uint32_t stream_id, double a,
                    double b, double p, int gen_flags, void* stream) {
    if (!out || rows < 0 || cols < 0 || ld < cols || row0 < 0 || col0 < 0) return STARMM_CONTRACT_VIOLATION;
    if (dist < STARMM_DIST_UNIFORM_REAL || dist > STARMM_DIST_GRAPH) return STARMM_CONTRACT_VIOLATION;
    if (row0 + rows > (1LL << 31) || col0 + cols > (1LL << 31)) return STARMM_TOO_LARGE;
    const bool fl = semiring == STARMM_SR_FP64 || semiring == STARMM_SR_TROPICAL_F64 ||
                    semiring == STARMM_SR_TROPICAL_F32;
    if ((dist == STARMM_DIST_UNIFORM_REAL || dist == STARMM_DIST_NORMAL) && !fl) return STARMM_CONTRACT_VIOLATION;
    if ((dist == STARMM_DIST_UNIFORM_INT || dist == STARMM_DIST_GRAPH) &&
        !(b >= a && b - a < 4294967296.0 && a == std::floor(a) && b == std::floor(b)))
        return STARMM_CONTRACT_VIOLATION;
    if (rows == 0 || cols == 0) return STARMM_OK;
    gen::Params g;
    g.dist = dist; g.flags = gen_flags; g.a = a; g.b = b; g.p = p; g.seed = seed; g.stream = stream_id;
    const dim3 grid = grid2d(rows, cols);
    cudaStream_t s = (cudaStream_t)stream;
    switch (semiring) {
    case STARMM_SR_INT64:
        gen::generate_kernel<SrInt64><<<grid, 256, 0, s>>>((long long*)out, ld, rows, cols, row0, col0, g); break;
    case STARMM_SR_FP64:
        gen::generate_kernel<SrFp64><<<grid, 256, 0, s>>>((double*)out, ld, rows, cols, row0, col0, g); break;
    case STARMM_SR_TROPICAL_F64:
        gen::generate_kernel<SrTropF64><<<grid, 256, 0, s>>>((double*)out, ld, rows, cols, row0, col0, g); break;
    case STARMM_SR_TROPICAL_F32:
        gen::generate_kernel<SrTropF32><<<grid, 256, 0, s>>>((float*)out, ld, rows, cols, row0, col0, g); break;
    case STARMM_SR_TROPICAL_I32:
        gen::generate_kernel<SrTropI32><<<grid, 256, 0, s>>>((int*)out, ld, rows, cols, row0, col0, g); break;
    default: return STARMM_CONTRACT_VIOLATION;
    }
    CK(cudaGetLastError());
    return STARMM_OK;
}

int starmm_pool_set_limit(int device, int64_t bytes, int64_t* old) {
    DeviceCtx* c = device_ctx(device);
    if (!c || bytes < 0) return STARMM_CONTRACT_VIOLATION;
    std::lock_guard<std::mutex> g(c->arena.mu);
    if (old) *old = c->arena.limit;
    c->arena.limit = bytes;
    return STARMM_OK;
}

int starmm_pool_set_discipline(int device, int fifo) {
    DeviceCtx* c = device_ctx(device);
    if (!c || (fifo != 0 && fifo != 1)) return STARMM_CONTRACT_VIOLATION;
    std::lock_guard<std::mutex> g(c->arena.mu);
    c->arena.fifo = fifo;
    return STARMM_OK;
}

}  // extern "C"
