// aux_kernels.cuh -- HBM-bound helpers around the tile products:
//   RangeAcc     range guard of the exact narrow paths, fused into the packers
//   pack_*       panel packing into the k-group-major layout of simt_kernel.cuh
//   pad_copy     zero-padded copy for the DMMA path when n is not tile aligned
//   fill         C <- identity (INIT_IDENTITY with split-k protocols)
//   madd / red   C <- C (+) D elementwise (kernels.madd, kernels.py:47-52; CO3
//                merge_tasks, ops.py:108-155) and its atomic variant
//                (accumulate_region, ops.py:76-101)
#pragma once
#include <algorithm>
#include "common.cuh"

namespace starmm {

// Running range guard fused into the packers (one read of A and B instead of two):
// out[0] = max |x| over the real (non-padding) elements read, +inf / INT32_MAX
// excluded; out[1] |= GUARD_BAD if a float is non-integral, NaN or -inf, and
// |= GUARD_NEG_ZERO if a float is -0.0 (the narrow encodings drop the sign of zero,
// and the reference's leaf order decides which zero survives: such operands take
// the ordered kernel, ordered_kernel.cuh).
constexpr unsigned GUARD_BAD = 1u, GUARD_NEG_ZERO = 2u;
struct RangeAcc {
    unsigned long long m = 0;
    unsigned bad = 0;
    STARMM_DEV void add(long long v) {
        unsigned long long a = v < 0 ? (unsigned long long)(-(v + 1)) + 1ull : (unsigned long long)v;
        m = a > m ? a : m;
    }
    STARMM_DEV void add(int v) {
        if (v == 0x7fffffff) return;
        unsigned long long a = (unsigned long long)(v < 0 ? -(long long)v : (long long)v);
        m = a > m ? a : m;
    }
    STARMM_DEV void add(float f) {
        if (f == __int_as_float(0x7f800000)) return;
        if (__float_as_uint(f) == 0x80000000u) { bad |= GUARD_NEG_ZERO; return; }
        if (!(f == rintf(f)) || fabsf(f) > 1e9f) { bad |= GUARD_BAD; return; }
        unsigned long long a = (unsigned long long)fabsf(f);
        m = a > m ? a : m;
    }
    STARMM_DEV void add(double d) {
        if (d == __longlong_as_double(0x7ff0000000000000LL)) return;
        if ((unsigned long long)__double_as_longlong(d) == 0x8000000000000000ull) { bad |= GUARD_NEG_ZERO; return; }
        if (!(d == rint(d)) || fabs(d) > 1e9) { bad |= GUARD_BAD; return; }
        unsigned long long a = (unsigned long long)fabs(d);
        m = a > m ? a : m;
    }
    // every thread of the launch must call flush (uses full-warp shuffles)
    STARMM_DEV void flush(unsigned long long* out) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            unsigned long long v = __shfl_xor_sync(0xffffffffu, m, o);
            m = v > m ? v : m;
            bad |= __shfl_xor_sync(0xffffffffu, bad, o);
        }
        // Skip the same-address atomic when the running maximum already covers this
        // warp (a stale read only costs a redundant atomic): 131K serialised atomics
        // on one L2 line were most of the int8 transpose packer's time.
        if ((threadIdx.x & 31) == 0) {
            if (m && m > *reinterpret_cast<volatile unsigned long long*>(&out[0])) atomicMax(&out[0], m);
            if (bad && (*reinterpret_cast<volatile unsigned long long*>(&out[1]) & bad) != bad)
                atomicOr(&out[1], (unsigned long long)bad);
        }
    }
};

// ---- packing ---------------------------------------------------------------
// Element conversion into the packed domain, with the pad value (annihilator
// of the product, so padded k terms contribute the additive identity).
struct ConvIdentity {   // same type
    template <class T> static STARMM_DEV T cvt(T x) { return x; }
};
struct ConvI32ToF32 {   // int32 tropical -> fp32 carrier, INT32_MAX -> +inf
    static STARMM_DEV float cvt(int x) {
        return x == 0x7fffffff ? __int_as_float(0x7f800000) : (float)x;
    }
};
struct ConvF64ToF32 {   // float64 tropical with integer values |x| <= 2^23 -> fp32 carrier (exact)
    static STARMM_DEV float cvt(double x) { return (float)x; }
};
struct ConvI32Vmin {    // int32 tropical -> VIADDMNMX encoding, INT32_MAX -> 2^30 - 1
    static STARMM_DEV int cvt(int x) { return x == 0x7fffffff ? (1 << 30) - 1 : x; }
};
struct ConvI64ToI32 {   // int64 ring, range-guarded narrow path
    static STARMM_DEV int cvt(long long x) { return (int)x; }
};
// (min,+) -> int16 encoding (+inf -> 16383), duplicated into both halves (A operand)
template <class T> STARMM_DEV unsigned s16_enc(T x);
template <> STARMM_DEV unsigned s16_enc<float>(float x) {
    return x == __int_as_float(0x7f800000) ? 16383u : ((unsigned)(int)x & 0xffffu);
}
template <> STARMM_DEV unsigned s16_enc<double>(double x) {
    return x == __longlong_as_double(0x7ff0000000000000LL) ? 16383u : ((unsigned)(int)x & 0xffffu);
}
template <> STARMM_DEV unsigned s16_enc<int>(int x) {
    return x == 0x7fffffff ? 16383u : ((unsigned)x & 0xffffu);
}
struct ConvS16Dup {
    template <class T> static STARMM_DEV unsigned cvt(T x) { unsigned e = s16_enc<T>(x); return e | (e << 16); }
};

// int64 ring -> s8x4 words along k: A (rows x kdim) -> P[kp/4][rowsp].  A 32-row x
// 128-k tile goes through shared memory so that both the int64 reads (32 B per
// thread, consecutive along a row) and the packed int32 writes are coalesced.
__global__ void pack_a_s8x4_kernel(const long long* A, long long rows, long long kdim, long long lda,
                                   int* P, long long rowsp, long long kp, unsigned long long* range) {
    __shared__ int tile[32][33];
    RangeAcc acc;
    const long long r0 = (long long)blockIdx.y * 32, w0 = (long long)blockIdx.x * 32;   // words
    const int tx = threadIdx.x, ty = threadIdx.y;                                       // 32 x 8
    // a thread's 4 int64 (32 B) as two 16-byte loads when the row allows it (4 separate
    // 8-byte loads per thread left each load instruction a quarter of its sectors)
    const bool vec = ((reinterpret_cast<uintptr_t>(A) | (uintptr_t)(lda * 8)) & 15) == 0;
    for (int i = ty; i < 32; i += 8) {
        const long long r = r0 + i, k = (w0 + tx) * 4;
        long long v[4] = {0, 0, 0, 0};
        if (r < rows) {
            if (vec && k + 3 < kdim) {
                const longlong2 x0 = *reinterpret_cast<const longlong2*>(A + r * lda + k);
                const longlong2 x1 = *reinterpret_cast<const longlong2*>(A + r * lda + k + 2);
                v[0] = x0.x; v[1] = x0.y; v[2] = x1.x; v[3] = x1.y;
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q) v[q] = k + q < kdim ? A[r * lda + k + q] : 0;
            }
        }
        unsigned w = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            acc.add(v[q]);
            w |= ((unsigned)(v[q] & 0xff)) << (8 * q);
        }
        tile[i][tx] = (int)w;
    }
    if (range) acc.flush(range);
    __syncthreads();
    for (int i = ty; i < 32; i += 8) {
        const long long kw = w0 + i, r = r0 + tx;
        if (kw < kp / 4 && r < rowsp) P[kw * rowsp + r] = tile[tx][i];
    }
}
// B (kdim x cols) -> P[kp/4][colsp].  2-D grid (x: column pairs, y: k-words), no 64-bit
// division per element (the grid-stride form spent 3x pack_a's time on it); two columns
// per thread with 16-byte loads when the rows allow it.
__global__ void __launch_bounds__(256, 8) pack_b_s8x4_kernel(const long long* B, long long kdim, long long cols, long long ldb,
                                   int* P, long long colsp, long long kp, unsigned long long* range) {
    RangeAcc acc;
    const bool vec = ((reinterpret_cast<uintptr_t>(B) | (uintptr_t)(ldb * 8)) & 15) == 0;
    for (long long kw = blockIdx.y; kw < kp / 4; kw += gridDim.y)
        for (long long c = 2 * ((long long)blockIdx.x * blockDim.x + threadIdx.x); c < colsp;
             c += 2 * (long long)gridDim.x * blockDim.x) {
            unsigned w0 = 0, w1 = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const long long k = kw * 4 + i;
                long long v0 = 0, v1 = 0;
                if (k < kdim) {
                    if (vec && c + 1 < cols) {
                        const longlong2 x = *reinterpret_cast<const longlong2*>(B + k * ldb + c);
                        v0 = x.x; v1 = x.y;
                    } else {
                        v0 = c < cols ? B[k * ldb + c] : 0;
                        v1 = c + 1 < cols ? B[k * ldb + c + 1] : 0;
                    }
                }
                acc.add(v0);
                acc.add(v1);
                w0 |= ((unsigned)(v0 & 0xff)) << (8 * i);
                w1 |= ((unsigned)(v1 & 0xff)) << (8 * i);
            }
            *reinterpret_cast<uint2*>(P + kw * colsp + c) = make_uint2(w0, w1);   // colsp is even
        }
    if (range) acc.flush(range);   // every thread reaches the flush (full-warp shuffles)
}
// (min,+) B (kdim x cols) -> P[kp][colsp/2] words (enc(B[k][2w]), enc(B[k][2w+1])).
// Four k rows per thread and pass, all eight loads issued before the first store: with
// one word per thread and pass only 16 KB per SM were in flight and the kernel ran at
// 2.3 TB/s (config 3: 172 us for its 268 MB panel).
template <class T>
__global__ void __launch_bounds__(256, 8) pack_b_s16x2_kernel(const T* B, long long kdim, long long cols, long long ldb,
                                    unsigned* P, long long colsp, long long kp, unsigned long long* range) {
    RangeAcc acc;
    const long long wpr = colsp / 2;
    for (long long k4 = (long long)blockIdx.y * 4; k4 < kp; k4 += (long long)gridDim.y * 4)   // 2-D grid, no division
        for (long long w = (long long)blockIdx.x * blockDim.x + threadIdx.x; w < wpr;
             w += (long long)gridDim.x * blockDim.x) {
            const long long c0 = 2 * w;
            T v0[4], v1[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const long long k = k4 + j;
                v0[j] = (k < kdim && c0 < cols) ? B[k * ldb + c0] : T(0);
                v1[j] = (k < kdim && c0 + 1 < cols) ? B[k * ldb + c0 + 1] : T(0);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const long long k = k4 + j;
                if (k >= kp) break;
                unsigned lo = 16383u, hi = 16383u;
                if (k < kdim && c0 < cols) { acc.add(v0[j]); lo = s16_enc<T>(v0[j]); }
                if (k < kdim && c0 + 1 < cols) { acc.add(v1[j]); hi = s16_enc<T>(v1[j]); }
                P[k * wpr + w] = lo | (hi << 16);
            }
        }
    if (range) acc.flush(range);
}

// A (rows x kdim, ld) -> P[kp/G][rowsp][G], transposing through a 32x32 smem tile
// so that both the global reads and the packed writes are coalesced.  (A 32 x 128 tile
// with 16 loads per thread before the barrier was slower -- 304 vs 211 us on config 3's
// A panel: fewer resident CTAs, longer bulk-synchronous phases.)
template <class Tin, class Tp, int G, class Conv>
__global__ void pack_a_kernel(const Tin* A, long long rows, long long kdim, long long lda,
                              Tp* P, long long rowsp, long long kp, Tp pad,
                              unsigned long long* range = nullptr, Pred pr = Pred()) {
    if (pr.off()) return;
    __shared__ Tp tile[32][33];
    RangeAcc acc;
    const int tx = threadIdx.x, ty = threadIdx.y;   // 32 x 8
    // grid-stride over 32 x 32 tiles (a bounded grid: a launch the path predicate turns
    // off costs a few microseconds instead of one empty CTA per tile)
    for (long long tr = blockIdx.y; tr * 32 < rowsp; tr += gridDim.y)
        for (long long tk = blockIdx.x; tk * 32 < kp; tk += gridDim.x) {
            const long long r0 = tr * 32, k0 = tk * 32;
            for (int i = ty; i < 32; i += 8) {
                long long r = r0 + i, k = k0 + tx;
                Tp v = pad;
                if (r < rows && k < kdim) {
                    Tin x = A[r * lda + k];
                    acc.add(x);
                    v = (Tp)Conv::cvt(x);
                }
                tile[i][tx] = v;
            }
            __syncthreads();
            // write: packed index for (k, r): ((k/G) * rowsp + r) * G + k%G
            for (int i = ty; i < 32; i += 8) {
                long long k = k0 + i;
                long long r = r0 + tx;
                if (k < kp && r < rowsp) P[((k / G) * rowsp + r) * G + (k % G)] = tile[tx][i];
            }
            __syncthreads();
        }
    if (range) acc.flush(range);
}

// bounded 2-D grid of pack_a_kernel: ~16 CTAs of 256 threads per SM
inline dim3 pack_a_grid(long long rowsp, long long kp) {
    const long long gx = std::max<long long>(1, std::min<long long>(kp / 32, 64));
    const long long gy = std::max<long long>(1, std::min<long long>(rowsp / 32, (148LL * 16 + gx - 1) / gx));
    return dim3((unsigned)gx, (unsigned)gy);
}

// B (kdim x cols, ld) -> P[kp/G][colsp][G]
template <class Tin, class Tp, int G, class Conv>
__global__ void __launch_bounds__(256, 8) pack_b_kernel(const Tin* B, long long kdim, long long cols, long long ldb,
                              Tp* P, long long colsp, long long kp, Tp pad,
                              unsigned long long* range = nullptr, Pred pr = Pred()) {
    if (pr.off()) return;
    RangeAcc acc;
    for (long long kg = blockIdx.y; kg < kp / G; kg += gridDim.y)   // 2-D grid, no division
        for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < colsp;
             c += (long long)gridDim.x * blockDim.x) {
#pragma unroll
            for (int g = 0; g < G; ++g) {
                long long k = kg * G + g;
                Tp v = pad;
                if (k < kdim && c < cols) {
                    Tin x = B[k * ldb + c];
                    acc.add(x);
                    v = (Tp)Conv::cvt(x);
                }
                P[(kg * colsp + c) * G + g] = v;
            }
        }
    if (range) acc.flush(range);
}

// Zero-padded copy (DMMA path): dst[rp x cp] from src[rows x cols, ld].
// the range guard's two words -> mapped pinned host memory (zero-copy stores)
__global__ void publish_range_kernel(const unsigned long long* d_range, unsigned long long* h_range) {
    if (threadIdx.x < 2) h_range[threadIdx.x] = d_range[threadIdx.x];
    __threadfence_system();
}

// 2-D grids (x: columns, y: rows, grid-stride in both) -- no 64-bit division per element
template <class T>
__global__ void pad_copy_kernel(const T* src, long long rows, long long cols, long long ld,
                                T* dst, long long rp, long long cp, Pred pr = Pred()) {
    if (pr.off()) return;
    for (long long r = blockIdx.y; r < rp; r += gridDim.y)
        for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < cp;
             c += (long long)gridDim.x * blockDim.x)
            dst[r * cp + c] = (r < rows && c < cols) ? src[r * ld + c] : (T)0;
}

template <class Sr>
__global__ void fill_kernel(typename Sr::T* C, long long rows, long long cols, long long ld, Pred pr = Pred()) {
    if (pr.off()) return;
    for (long long r = blockIdx.y; r < rows; r += gridDim.y)
        for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < cols;
             c += (long long)gridDim.x * blockDim.x)
            C[r * ld + c] = Sr::identity();
}

// C <- C (+) D.  atomic = 1 merges with the semiring's atomic-madd; rev = 1 folds in
// the other order, C <- D (+) C (D came first in k order: the host path's C0, whose
// place in the reference's fold sequence is before every leaf -- only the sign of a
// tied zero can tell the two orders apart, common.cuh nan_min).
template <class Sr>
__global__ void madd_kernel(typename Sr::T* C, long long ldc, const typename Sr::T* D, long long ldd,
                            long long rows, long long cols, int atomic, int rev = 0, Pred pr = Pred()) {
    if (pr.off()) return;
    for (long long r = blockIdx.y; r < rows; r += gridDim.y)
        for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < cols;
             c += (long long)gridDim.x * blockDim.x) {
            typename Sr::T d = D[r * ldd + c];
            typename Sr::T* p = &C[r * ldc + c];
            if (atomic) Sr::atomic_fold(p, d);
            else *p = rev ? Sr::fold(d, *p) : Sr::fold(*p, d);
        }
}

// launch shape for the 2-D elementwise kernels (256 threads, __launch_bounds__(256, 8) on
// the packers so that 8 CTAs per SM really are resident; x: 256-column blocks, y: rows, both
// grid-strided): at most one resident wave of CTAs (8 x 256 threads per SM), and the
// row dimension cut so that every CTA runs the same number of grid-stride iterations
// (1024 rows over 296 CTA-rows ran 3.46 -> 4 iterations on the slowest CTA: the int8
// B packer spent 14% of its time in that tail).
inline dim3 grid2d(long long rows, long long cols) {
    const long long bx = std::max<long long>(1, std::min<long long>((cols + 255) / 256, 64));
    const long long cap = std::max<long long>(1, (148LL * 8) / bx);
    const long long by0 = std::max<long long>(1, std::min<long long>(rows, cap));
    const long long iters = (rows + by0 - 1) / by0;
    const long long by = std::max<long long>(1, (rows + iters - 1) / std::max<long long>(1, iters));
    return dim3((unsigned)bx, (unsigned)by);
}

}  // namespace starmm

namespace starmm {

// ---- ring combinations for the Strassen family (strassen.py:29-58) ---------
// dst <- beta*dst + ax*X + ay*Y with coefficients in {-1, 0, 1}; int64 uses
// unsigned arithmetic so every step wraps mod 2^64 exactly like numpy's int64
// (the ring is Z/2^64, where Strassen's subtractions are exact).
template <class T> STARMM_DEV T ring_mac(T acc, int c, T x);
template <> STARMM_DEV long long ring_mac<long long>(long long acc, int c, long long x) {
    unsigned long long a = (unsigned long long)acc, v = (unsigned long long)x;
    return (long long)(c > 0 ? a + v : (c < 0 ? a - v : a));
}
template <> STARMM_DEV double ring_mac<double>(double acc, int c, double x) {
    return c > 0 ? acc + x : (c < 0 ? acc - x : acc);
}

template <class T>
__global__ void ring_combine_kernel(T* D, long long ldd, const T* X, long long ldx, const T* Y,
                                    long long ldy, long long rows, long long cols, int beta, int ax,
                                    int ay) {
    for (long long r = blockIdx.y; r < rows; r += gridDim.y)
        for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < cols;
             c += (long long)gridDim.x * blockDim.x) {
            T acc = beta ? D[r * ldd + c] : (T)0;
            if (beta < 0) acc = ring_mac<T>((T)0, -1, acc);
            if (ax) acc = ring_mac<T>(acc, ax, X[r * ldx + c]);
            if (ay) acc = ring_mac<T>(acc, ay, Y[r * ldy + c]);
            D[r * ldd + c] = acc;
        }
}

}  // namespace starmm
