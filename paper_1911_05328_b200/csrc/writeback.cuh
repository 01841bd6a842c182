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

// Read-fold-write of the calling thread's NE elements, CH at a time: all CH loads of a
// chunk are issued before any store.  (Folding element by element, ptxas cannot hoist a
// load above the previous element's store -- rows are ldc apart, ldc unknown -- so every
// element paid a full HBM round trip: LDG DADD STG LDG DADD STG ... in the SASS.)
template <class Sr, int NE, int CH, class Each, class Addr>
STARMM_DEV void fold_batched(Each each, Addr addr, bool cg) {
    using T = typename Sr::T;
    static_assert(CH >= 1 && NE % CH == 0, "fold chunk");   // (FOLD_CH == 0 never gets here)
#pragma unroll
    for (int q = 0; q < NE / CH; ++q) {
        T old[CH];
        int idx = 0;
        each([&](int r, int c, T v) {
            if (idx / CH == q) {
                T* p = addr(r, c);
                old[idx % CH] = p ? (cg ? __ldcg(p) : *p) : v;
            }
            ++idx;
        });
        idx = 0;
        each([&](int r, int c, T v) {
            if (idx / CH == q) {
                T* p = addr(r, c);
                if (p) {
                    T x = Sr::fold(old[idx % CH], v);
                    if (cg) __stcg(p, x); else *p = x;
                }
            }
            ++idx;
        });
    }
}


// ---------------------------------------------------------------------------
// Vectorised exclusive epilogue (WB_FOLD / WB_STORE of full, 16-byte-aligned tiles).
//
// A CUDA-core thread owns FRAGMENTS of W consecutive output columns (FB = W * sizeof(T)
// bytes: 8, 16, 32 or 64), and the lanes tx, tx+1, ... of a row own adjacent fragments.
// Written element by element that is one 8-byte generic ST per lane at a 32-byte stride:
// every warp store touches 32 sectors and fills a quarter of each (ncu, int64 dp4a tile:
// 16.8 M L2 sectors requested for 4.2 M ideal, and ~11 us per tile boundary).  Here a
// fragment moves as 16-byte PIECES; when FB >= 32 the two lanes of an even/odd pair first
// swap pieces so that instruction k of the pair covers bytes [32k, 32k + 32) of the pair's
// 2*FB contiguous bytes -- every warp access reads or writes whole 32-byte sectors.
// ---------------------------------------------------------------------------
STARMM_DEV uint4 ldg16(const void* p) {
    uint4 v;
    asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(__cvta_generic_to_global(p)));
    return v;
}
STARMM_DEV void stg16(void* p, uint4 v) {
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};"
                 ::"l"(__cvta_generic_to_global(p)), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
STARMM_DEV uint2 ldg8(const void* p) {
    uint2 v;
    asm volatile("ld.global.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(__cvta_generic_to_global(p)));
    return v;
}
STARMM_DEV void stg8(void* p, uint2 v) {
    asm volatile("st.global.v2.u32 [%0], {%1,%2};" ::"l"(__cvta_generic_to_global(p)), "r"(v.x), "r"(v.y) : "memory");
}
STARMM_DEV uint4 shfl_xor1_16(uint4 v) {
    v.x = __shfl_xor_sync(0xffffffffu, v.x, 1);
    v.y = __shfl_xor_sync(0xffffffffu, v.y, 1);
    v.z = __shfl_xor_sync(0xffffffffu, v.z, 1);
    v.w = __shfl_xor_sync(0xffffffffu, v.w, 1);
    return v;
}
STARMM_DEV uint4 sel16(bool c, uint4 a, uint4 b) {
    return make_uint4(c ? a.x : b.x, c ? a.y : b.y, c ? a.z : b.z, c ? a.w : b.w);
}

// Lane parity b of a pair owns pieces b*NPL + i (i < NPL) of the pair's 2*NPL pieces;
// afterwards q[k] is pair piece 2k + b.  All 32 lanes must call.
template <int NPL>
STARMM_DEV void pair_exchange(uint4 (&q)[NPL], bool odd) {
    static_assert(NPL >= 2 && NPL % 2 == 0, "pieces per lane");
    uint4 out[NPL];
#pragma unroll
    for (int r = 0; r < NPL / 2; ++r) {
        const uint4 recv = shfl_xor1_16(sel16(odd, q[2 * r], q[2 * r + 1]));
        out[r] = sel16(odd, recv, q[2 * r]);
        out[NPL / 2 + r] = sel16(odd, q[2 * r + 1], recv);
    }
#pragma unroll
    for (int k = 0; k < NPL; ++k) q[k] = out[k];
}

template <class Sr>
STARMM_DEV uint4 fold16(uint4 old, uint4 v) {
    using T = typename Sr::T;
    constexpr int N = 16 / (int)sizeof(T);
    union U { uint4 q; T e[N]; } a, b;
    a.q = old; b.q = v;
#pragma unroll
    for (int x = 0; x < N; ++x) a.e[x] = Sr::fold(a.e[x], b.e[x]);
    return a.q;
}

// One thread's NF fragments of one output row: frag[f] holds W elements destined for
// gp[f][0..W) (16-byte aligned, or 8-byte when FB == 8).  fold: C <- fold(C, v), else
// plain store.  `odd`: parity of this lane within its even/odd pair (lane & 1); the
// partner's fragments are the next (odd) / previous (even) FB bytes.  Warp-collective.
template <class Sr, int W, int NF>
STARMM_DEV void epilogue_row_vec(typename Sr::T (&frag)[NF][W], typename Sr::T* (&gp)[NF], bool fold,
                                 bool odd) {
    using T = typename Sr::T;
    constexpr int FB = W * (int)sizeof(T);
    static_assert(FB == 8 || FB == 16 || FB == 32 || FB == 64, "fragment bytes");
    if constexpr (FB == 8) {
        union U { uint2 q; T e[W]; };
        U v[NF], old[NF];
#pragma unroll
        for (int f = 0; f < NF; ++f) {
#pragma unroll
            for (int x = 0; x < W; ++x) v[f].e[x] = frag[f][x];
            if (fold) old[f].q = ldg8(gp[f]);
        }
#pragma unroll
        for (int f = 0; f < NF; ++f) {
            if (fold) {
#pragma unroll
                for (int x = 0; x < W; ++x) v[f].e[x] = Sr::fold(old[f].e[x], v[f].e[x]);
            }
            stg8(gp[f], v[f].q);
        }
    } else {
        constexpr int NPL = FB / 16;
        constexpr int EPV = 16 / (int)sizeof(T);
        union U { uint4 q; T e[EPV]; };
        uint4 v[NF][NPL], old[NF][NPL];
        char* base[NF];
#pragma unroll
        for (int f = 0; f < NF; ++f) {
#pragma unroll
            for (int k = 0; k < NPL; ++k) {
                U u;
#pragma unroll
                for (int x = 0; x < EPV; ++x) u.e[x] = frag[f][k * EPV + x];
                v[f][k] = u.q;
            }
            base[f] = reinterpret_cast<char*>(gp[f]);
            if constexpr (NPL >= 2) {
                pair_exchange<NPL>(v[f], odd);
                base[f] += odd ? (16 - FB) : 0;      // pair base + 16*b; piece k at + 32*k
            }
            if (fold) {
#pragma unroll
                for (int k = 0; k < NPL; ++k) old[f][k] = ldg16(base[f] + (NPL >= 2 ? 32 : 16) * k);
            }
        }
#pragma unroll
        for (int f = 0; f < NF; ++f)
#pragma unroll
            for (int k = 0; k < NPL; ++k) {
                uint4 x = v[f][k];
                if (fold) x = fold16<Sr>(old[f][k], x);
                stg16(base[f] + (NPL >= 2 ? 32 : 16) * k, x);
            }
    }
}

// FOLD_CH: elements per batched read-fold-write chunk; 0 = element by element (the DMMA
// kernel, whose full aligned FOLD tiles take its own vectorised epilogue (EPI=1,
// dmma_kernel.cuh) -- this generic path only sees its ragged / protocol tiles; changes
// here shifted its register allocation and cost 1-3%, profiles/r01k_epilogue_ab.md)
template <class Sr, int BM, int BN, int NTHREADS, int FOLD_CH, class Each>
STARMM_DEV void writeback(const WbParams& w, const TaskGrid& g, int tm, int tn, int s, int tile,
                          int worker, int mode, int pair_seen, Each each) {
    constexpr int NE = BM * BN / NTHREADS;     // elements per thread
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
        if constexpr (FOLD_CH == 0) {
            each([&](int r, int c, T v) {
                long long gr = m0 + r, gc = n0 + c;
                if (gr < M && gc < N) {
                    T* p = &C[gr * ldc + gc];
                    *p = Sr::fold(*p, v);
                }
            });
        } else {
            fold_batched<Sr, NE, FOLD_CH>(each, [&](int r, int c) -> T* {
                long long gr = m0 + r, gc = n0 + c;
                return (gr < M && gc < N) ? &C[gr * ldc + gc] : nullptr;
            }, false);
        }
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
    auto fold_each = [&]() {
        each([&](int r, int c, T v) {
            long long gr = m0 + r, gc = n0 + c;
            if (lazy) v = __ldcg(&tmp[r * BN + c]);
            if (gr < M && gc < N) {
                T* p = &C[gr * ldc + gc];
                __stcg(p, Sr::fold(__ldcg(p), v));
            }
        });
    };
    if constexpr (FOLD_CH == 0) {
        fold_each();
    } else {
        if (lazy) {
            fold_each();
        } else {
            fold_batched<Sr, NE, FOLD_CH>(each, [&](int r, int c) -> T* {
                long long gr = m0 + r, gc = n0 + c;
                return (gr < M && gc < N) ? &C[gr * ldc + gc] : nullptr;
            }, true);
        }
    }
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
