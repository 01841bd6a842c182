// writeback.cuh -- the tile epilogue: applies one write-back protocol
// (common.cuh WbMode) to a CTA's accumulator fragment.
//
// `each(f)` must call f(r, c, v) once for every accumulator element the
// calling thread owns (r, c are tile-local; v is already converted to the
// output type).  All threads of the CTA must call writeback() together.
#pragma once
#include "common.cuh"

namespace starmm {

// Arrival on the pair state at task start (PairState.arrive, classic.py:62-68).
// Returns the state seen; thread 0 performs the CAS, the CTA shares it.
STARMM_DEV int pair_arrive(const WbParams& w, const TaskGrid& g, int tile, int s, int* smem_word) {
    if (threadIdx.x == 0) {
        int* st = &w.pairs[(long long)tile * (g.S >> 1) + (s >> 1)];
        int seen = atomicCAS(st, PAIR_EMPTY, PAIR_FIRST_RUNNING);
        if (seen == PAIR_EMPTY) counter_add(w, CNT_PAIR_TRANSITIONS, 1);
        *smem_word = seen;
    }
    __syncthreads();
    int seen = *smem_word;
    __syncthreads();
    return seen;
}

template <class Sr, int BM, int BN, class Each>
STARMM_DEV void writeback(const WbParams& w, const TaskGrid& g, int tm, int tn, int s, int tile,
                          int worker, int mode, int pair_seen, Each each) {
    using T = typename Sr::T;
    const long long m0 = (long long)tm * BM, n0 = (long long)tn * BN;
    T* C = reinterpret_cast<T*>(w.C);
    const long long ldc = w.ldc;
    const long long M = w.M, N = w.N;

    if (mode == WB_STORE) {
        T* dst = C;
        long long ld = ldc;
        if (w.mode_base == 1 && s > 0) {   // co3: slice s>0 lands in workspace D_s
            dst = reinterpret_cast<T*>(w.W) + (long long)(s - 1) * w.wstride;
            ld = w.ldw;
        }
        each([&](int r, int c, T v) {
            long long gr = m0 + r, gc = n0 + c;
            if (gr < M && gc < N) dst[gr * ld + gc] = v;
        });
        return;
    }
    if (mode == WB_FOLD) {
        each([&](int r, int c, T v) {
            long long gr = m0 + r, gc = n0 + c;
            if (gr < M && gc < N) {
                T* p = &C[gr * ldc + gc];
                *p = Sr::fold(*p, v);
            }
        });
        return;
    }
    const long long tile_bytes = (long long)BM * BN * (long long)sizeof(T);
    if (mode == WB_RED) {
        // TAR leaf (classic.py:160-167): the accumulator registers are this
        // worker's b x b block; merge it with per-element atomic-madd -- into the
        // local C, or (k-split across GPUs) straight into the owner GPU's rows over
        // NVLink peer memory: the combine is fused into the tile epilogue.
        if (threadIdx.x == 0) {
            pool_acquire(w, worker, tile_bytes);
            counter_add(w, CNT_SERIALIZATIONS, 1);
        }
        if (w.remote_parts > 0) {
            each([&](int r, int c, T v) {
                long long gr = m0 + r, gc = n0 + c;
                if (gr < M && gc < N) {
                    int part = (int)(gr / w.remote_rows);
                    T* dst = reinterpret_cast<T*>(w.remote_base[part]);
                    Sr::atomic_fold(&dst[(gr - part * w.remote_rows) * w.remote_ld + gc], v);
                }
            });
        } else {
            each([&](int r, int c, T v) {
                long long gr = m0 + r, gc = n0 + c;
                if (gr < M && gc < N) Sr::atomic_fold(&C[gr * ldc + gc], v);
            });
        }
        __syncthreads();
        if (threadIdx.x == 0) pool_release(w, tile_bytes);
        return;
    }
    // WB_LOCK / WB_PAIR: fold under the tile's exclusion slot.
    const bool lazy = (mode == WB_PAIR && pair_seen == PAIR_FIRST_RUNNING);
    T* tmp = reinterpret_cast<T*>(w.scratch) + (long long)worker * w.scratch_elems;
    if (lazy) {
        // Sibling is genuinely running: buy a temporary from this worker's
        // LIFO pool and compute into it (classic.py:193-200).
        if (threadIdx.x == 0) {
            pool_acquire(w, worker, tile_bytes);
            counter_add(w, CNT_LAZY_ACQUIRES, 1);
        }
        each([&](int r, int c, T v) { __stcg(&tmp[r * BN + c], v); });
    }
    __syncthreads();
    if (threadIdx.x == 0) lock_slot(&w.slots[tile]);
    __syncthreads();
    each([&](int r, int c, T v) {
        long long gr = m0 + r, gc = n0 + c;
        if (lazy) v = __ldcg(&tmp[r * BN + c]);
        if (gr < M && gc < N) {
            T* p = &C[gr * ldc + gc];
            __stcg(p, Sr::fold(__ldcg(p), v));
        }
    });
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        unlock_slot(&w.slots[tile]);
        counter_add(w, CNT_SERIALIZATIONS, 1);
        if (lazy) pool_release(w, tile_bytes);
        if (mode == WB_PAIR && pair_seen == PAIR_EMPTY) {
            // first half done: FirstRunning -> FirstDone (classic.py:70-75)
            atomicExch(&w.pairs[(long long)tile * (g.S >> 1) + (s >> 1)], PAIR_FIRST_DONE);
            counter_add(w, CNT_PAIR_TRANSITIONS, 1);
        }
    }
    __syncthreads();
}

}  // namespace starmm
