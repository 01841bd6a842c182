// common.cuh -- semiring traits, task decode and the reductive write-back
// protocols shared by every tile kernel of libstarmm_b200.
//
// Reference mapping (paths relative to /root/reference/pkg/src/starmm/):
//   Semiring ops / identities ........ semiring.py:63-145
//   fold_add (np.add / np.minimum) ... semiring.py:116-117, 126-127
//   leaf store-or-fold ............... ops.py:30-65
//   accumulate_region (atomic-madd) .. ops.py:76-101  -> WB_RED / WB_LOCK
//   PairState lazy allocation ........ classic.py:42-75, 190-204 -> WB_PAIR
//   TileExclusionTable slots ......... matrix.py:64-90 -> per-tile lock words
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

#define STARMM_DEV __device__ __forceinline__

namespace starmm {

// Device-side path predicate.  The range guard's verdict is computed on the device
// (select_path_kernel, aux_kernels.cuh) into one word; every launch of a candidate
// path after it carries (sel, id) and returns at once unless *sel == id.  So the host
// queues the whole call without waiting for the guard (STARMM_F_ASYNC holds on every
// path) and exactly one candidate does the work.  sel == nullptr: unconditional.
struct Pred {
    const unsigned* sel = nullptr;
    unsigned id = 0;
    STARMM_DEV bool off() const { return sel != nullptr && *reinterpret_cast<const volatile unsigned*>(sel) != id; }
};

// ---------------------------------------------------------------------------
// Semiring traits over the OUTPUT element type (the C matrix type).
//   identity(): additive identity (semiring.py:130-145: 0 / 0.0 / +inf)
//   fold(c, d): c (+) d  with the reference's fold_add semantics
//   atomic_fold(p, d): concurrent-safe *p <- *p (+) d  (the atomic-madd)
// ---------------------------------------------------------------------------
struct SrInt64 {            // "int": int64, wraps mod 2^64 (semiring.py:5-9)
    using T = long long;
    static STARMM_DEV T identity() { return 0; }
    static STARMM_DEV T fold(T c, T d) {
        return (T)((unsigned long long)c + (unsigned long long)d);
    }
    static STARMM_DEV void atomic_fold(T* p, T d) {
        atomicAdd(reinterpret_cast<unsigned long long*>(p), (unsigned long long)d);
    }
};

struct SrFp64 {             // "float": float64 (+,x)
    using T = double;
    static STARMM_DEV T identity() { return 0.0; }
    static STARMM_DEV T fold(T c, T d) { return c + d; }
    static STARMM_DEV void atomic_fold(T* p, T d) { atomicAdd(p, d); }
};

// np.minimum(C, D) semantics (semiring.py:126-127): NaN if either operand is NaN, and
// on a tie the SECOND operand -- np.minimum(+0.0, -0.0) is -0.0 and
// np.minimum(-0.0, +0.0) is +0.0 (x86 MINPD order; measured, tests/golden/ref_signed_zero.npz).
template <class F>
STARMM_DEV F nan_min(F c, F d) {
    return (c != c || d != d) ? (c != c ? c : d) : (c < d ? c : d);
}

struct SrTropF64 {          // "tropical": float64 (min,+), +inf identity
    using T = double;
    static STARMM_DEV T identity() { return __longlong_as_double(0x7ff0000000000000ULL); }
    static STARMM_DEV T fold(T c, T d) { return nan_min(c, d); }
    static STARMM_DEV void atomic_fold(T* p, T d) {
        unsigned long long* q = reinterpret_cast<unsigned long long*>(p);
        unsigned long long old = *q, assumed;
        do {
            assumed = old;
            T nv = nan_min(__longlong_as_double((long long)assumed), d);
            unsigned long long nb = (unsigned long long)__double_as_longlong(nv);
            if (nb == assumed) return;
            old = atomicCAS(q, assumed, nb);
        } while (old != assumed);
    }
};

struct SrTropF32 {          // "tropical_f32": float32 (min,+)
    using T = float;
    static STARMM_DEV T identity() { return __int_as_float(0x7f800000); }
    static STARMM_DEV T fold(T c, T d) { return nan_min(c, d); }
    static STARMM_DEV void atomic_fold(T* p, T d) {
        unsigned* q = reinterpret_cast<unsigned*>(p);
        unsigned old = *q, assumed;
        do {
            assumed = old;
            T nv = nan_min(__uint_as_float(assumed), d);
            unsigned nb = __float_as_uint(nv);
            if (nb == assumed) return;
            old = atomicCAS(q, assumed, nb);
        } while (old != assumed);
    }
};

struct SrTropI32 {          // "tropical_i32": int32 (min,+), INT32_MAX = +inf
    using T = int;
    static STARMM_DEV T identity() { return 0x7fffffff; }
    static STARMM_DEV T fold(T c, T d) { return d < c ? d : c; }
    static STARMM_DEV void atomic_fold(T* p, T d) { atomicMin(p, d); }
};

// ---------------------------------------------------------------------------
// Task grid: a leaf task is (output tile, k-slice).  Tiles are rastered in
// column groups of `group_m` tile-rows so that co-resident CTAs share A row
// panels and B column panels in L2; the k-slices of one tile are adjacent in
// task order, so sibling halves run concurrently (the "all eight sub-products
// spawned" of TAR/SAR, classic.py:176-178, 207-218).
// ---------------------------------------------------------------------------
struct TaskGrid {
    int tiles_m, tiles_n;
    int S;                 // k-slices per output tile (2^ksplit_log2)
    int log2S;
    int tar_levels;        // top split levels that use the TAR protocol (STAR)
    int group_m;
    int num_tasks;
    long long kslice;      // k extent of one slice (multiple of the k-stage)
    // balanced slices (TAR with uneven k-slices, "stream-K"): worker b runs the
    // flattened (tile, k-stage) range [b*T/W, (b+1)*T/W) of T = tiles * kstages
    // iterations; a tile split between workers is merged with the atomic-madd
    int balanced;
    long long kstages;     // k-stages per tile (balanced mode)
};

STARMM_DEV void decode_task(const TaskGrid& g, int t, int& tm, int& tn, int& s, int& tile) {
    s = t & (g.S - 1);
    tile = t >> g.log2S;
    int width = g.group_m * g.tiles_n;
    int grp = tile / width;
    int first_m = grp * g.group_m;
    int gsize = min(g.tiles_m - first_m, g.group_m);
    int r = tile - grp * width;
    tm = first_m + r % gsize;
    tn = r / gsize;
    tile = tm * g.tiles_n + tn;   // canonical tile id for slot tables
}

// ---------------------------------------------------------------------------
// Write-back protocols.  One per schedule family:
//   WB_STORE  plain store (virgin target: co3 workspace slices, INIT_IDENTITY)
//   WB_FOLD   exclusive read-fold-write (co2: ops.py:41-46 direct fold)
//   WB_RED    hardware atomic-madd per element (tar: accumulate_region)
//   WB_LOCK   fold under the tile's exclusion slot (sar/star leaves, locked=True)
//   WB_PAIR   SAR pair-state protocol with lazy scratch (classic.py:190-204)
// ---------------------------------------------------------------------------
enum WbMode : int { WB_STORE = 0, WB_FOLD = 1, WB_RED = 2, WB_LOCK = 3, WB_PAIR = 4 };
enum PairSt : int { PAIR_EMPTY = 0, PAIR_FIRST_RUNNING = 1, PAIR_FIRST_DONE = 2 };

// Device-side counters (stats), one array of 64-bit words.
enum Counter : int {
    CNT_SERIALIZATIONS = 0, CNT_PAIR_TRANSITIONS, CNT_LAZY_ACQUIRES, CNT_POOL_ACQUIRES,
    CNT_POOL_FRESH, CNT_POOL_ISSUED, CNT_POOL_HIGH_WATER, CNT_PAIRS,
    CNT_LIVE, CNT_LIVE_MAX,          // leaf gauge: leaves in flight now / at most (metrics.py:63-95)
    CNT__N
};

struct WbParams {
    int mode_base;            // schedule: 0 co2, 1 co3, 2 tar, 3 sar, 4 star
    int init_identity;        // STARMM_F_INIT_IDENTITY
    void* C; long long ldc;
    long long M, N;           // valid output extent (masking)
    void* W; long long ldw; long long wstride;   // co3 workspace slices 1..S-1
    int* slots;               // per tile exclusion word
    int* pairs;               // per (tile, pair) state
    unsigned long long* counters;
    unsigned* worker_used;    // per worker: has this worker's scratch block been issued
    void* scratch; long long scratch_elems;      // per-worker lazy temp block (tile-sized)
    // k-split combine across GPUs (starmm_plan_set_peers): output row r is folded with
    // the atomic-madd into part p = r / remote_rows, which lives at remote_base[p]
    // (an NVLink-mapped peer buffer, or a local one), leading dimension remote_ld.
    int remote_parts;
    long long remote_rows, remote_ld;
    void* remote_base[8];
};

// Which protocol a given task uses (host mirrors this in DESIGN.md).
STARMM_DEV int task_mode(const WbParams& w, const TaskGrid& g, int s) {
    if (w.remote_parts > 0) return WB_RED;   // TAR across GPUs: every tile is atomic-madd'ed
    switch (w.mode_base) {
    case 0: return w.init_identity ? WB_STORE : WB_FOLD;                     // co2
    case 1: return (s == 0) ? (w.init_identity ? WB_STORE : WB_FOLD) : WB_STORE;  // co3
    case 2: return g.S == 1 ? (w.init_identity ? WB_STORE : WB_FOLD) : WB_RED;   // tar
    case 3: return g.S == 1 ? (w.init_identity ? WB_STORE : WB_FOLD) : WB_PAIR;  // sar
    default:                                                                      // star
        if (g.S == 1) return w.init_identity ? WB_STORE : WB_FOLD;
        return (g.tar_levels >= g.log2S) ? WB_RED : WB_PAIR;
    }
}

STARMM_DEV void counter_add(const WbParams& w, int c, unsigned long long v) {
    atomicAdd(&w.counters[c], v);
}

// Live leaf gauge, the GPU form of the reference's task_enter / base_enter
// (metrics.py:63-95): thread 0 of a CTA counts its leaf task (output tile x k-slice)
// in on entry and out on exit; the maximum observed is how many leaves really ran
// concurrently (not a formula of the grid).  One atomic pair per leaf.
STARMM_DEV void leaf_enter(const WbParams& w) {
    if (threadIdx.x == 0) {
        const unsigned long long now = atomicAdd(&w.counters[CNT_LIVE], 1ull) + 1ull;
        atomicMax(&w.counters[CNT_LIVE_MAX], now);
    }
}
STARMM_DEV void leaf_exit(const WbParams& w) {
    if (threadIdx.x == 0) atomicAdd(&w.counters[CNT_LIVE], ~0ull);   // -1
}

STARMM_DEV void lock_slot(int* slot) {
    int ns = 32;
    while (atomicCAS(slot, 0, 1) != 0) {
        __nanosleep(ns);
        if (ns < 1024) ns <<= 1;
    }
    __threadfence();
}

STARMM_DEV void unlock_slot(int* slot) {
    __threadfence();
    atomicExch(slot, 0);
}

// Per-worker LIFO scratch (pool.py:89-132).  Each persistent CTA owns one
// exact-size block; acquisitions nest at most one deep per worker, so the
// stack never grows beyond one block per worker and every acquisition after
// the first on a worker is a reuse.
STARMM_DEV void pool_acquire(const WbParams& w, int worker, long long bytes) {
    counter_add(w, CNT_POOL_ACQUIRES, 1);
    if (atomicExch(&w.worker_used[worker], 1u) == 0u) counter_add(w, CNT_POOL_FRESH, 1);
    unsigned long long now = atomicAdd(&w.counters[CNT_POOL_ISSUED], (unsigned long long)bytes) + bytes;
    atomicMax(&w.counters[CNT_POOL_HIGH_WATER], now);
}

STARMM_DEV void pool_release(const WbParams& w, long long bytes) {
    atomicAdd(&w.counters[CNT_POOL_ISSUED], (unsigned long long)(-bytes));
}

}  // namespace starmm
