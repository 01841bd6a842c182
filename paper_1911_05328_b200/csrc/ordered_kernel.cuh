// ordered_kernel.cuh -- float (min,+) in the reference's own evaluation order, for
// operands that hold -0.0.
//
// The reference's result for a tropical element is, bit for bit (pinned against the
// reference itself: tests/golden/ref_signed_zero.npz):
//   acc = C0;  for each leaf k-block [k0, k0 + b) in increasing k:
//       blk = +inf;  for k in block: v = a_ik + b_kj; if (v < blk) blk = v   (semiring.py:56-58)
//       acc = np.minimum(acc, blk)      (semiring.py:126-127: NaN wins, a tie keeps blk)
// For any two values that compare equal only the sign of zero can differ, and -0.0
// arises only as (-0.0) + (-0.0).  So when no operand is -0.0 every schedule and every
// kernel in this library gives the same bits; when one is, the sign of a zero result
// depends on the leaf size b and on the k order, which the packed fast kernels (and any
// k-split) do not keep.  The range guard flags -0.0 (GUARD_NEG_ZERO, aux_kernels.cuh)
// and such calls run this kernel: a plain smem-tiled k-serial loop that tracks the
// block minimum and folds it at every leaf boundary.  It is a correctness path (two
// FP32/FP64 instructions per term plus the boundary fold), not a fast one.
#pragma once
#include "common.cuh"

namespace starmm {

struct OrderedParams {
    const void* A; long long lda;
    const void* B; long long ldb;
    void* C; long long ldc;
    long long M, N, K;
    long long blk;          // leaf k-extent b (a power of two); >= K: one block
    long long kofs;         // global k index of this call's first k (leaf alignment)
    int init_identity;      // C <- A (x) B (the first leaf stores)
    Pred pr;
};

namespace ordered {
constexpr int TM = 64, TN = 64, TK = 32, THREADS = 256;   // 16 x 16 threads, 4 x 4 outputs each
}

template <class Sr>
__global__ void __launch_bounds__(ordered::THREADS) minplus_ordered_kernel(OrderedParams p) {
    using namespace ordered;
    using T = typename Sr::T;
    if (p.pr.off()) return;
    __shared__ T As[TK][TM + 1];
    __shared__ T Bs[TK][TN];
    const T inf = Sr::identity();
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const T* A = reinterpret_cast<const T*>(p.A);
    const T* B = reinterpret_cast<const T*>(p.B);
    T* C = reinterpret_cast<T*>(p.C);
    // grid-stride over the output tiles (a bounded grid: this kernel is launched behind
    // the device-side path verdict on every call of a float (min,+) plan, and one empty
    // CTA per tile cost config 3 36 us per step when the verdict turned it off)
    const long long tiles_n = (p.N + TN - 1) / TN, tiles = ((p.M + TM - 1) / TM) * tiles_n;
    for (long long t = blockIdx.x; t < tiles; t += gridDim.x) {
    const long long r0 = (t / tiles_n) * TM, c0 = (t % tiles_n) * TN;
    T acc[4][4], bl[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const long long r = r0 + ty + 16 * i, c = c0 + tx + 16 * j;
            acc[i][j] = (!p.init_identity && r < p.M && c < p.N) ? C[r * p.ldc + c] : inf;
            bl[i][j] = inf;
        }
    const long long bmask = p.blk - 1;
    for (long long k0 = 0; k0 < p.K; k0 += TK) {
        __syncthreads();
        for (int idx = tid; idx < TM * TK; idx += THREADS) {   // A tile, coalesced along k
            const int r = idx / TK, kk = idx % TK;
            const long long gr = r0 + r, gk = k0 + kk;
            As[kk][r] = (gr < p.M && gk < p.K) ? A[gr * p.lda + gk] : inf;
        }
        for (int idx = tid; idx < TK * TN; idx += THREADS) {   // B tile, coalesced along n
            const int kk = idx / TN, c = idx % TN;
            const long long gk = k0 + kk, gc = c0 + c;
            Bs[kk][c] = (gk < p.K && gc < p.N) ? B[gk * p.ldb + gc] : inf;
        }
        __syncthreads();
        const int kn = (int)min((long long)TK, p.K - k0);
        for (int kk = 0; kk < kn; ++kk) {
            const long long gk = k0 + kk;
            if (gk > 0 && ((p.kofs + gk) & bmask) == 0) {        // leaf boundary: fold the block
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) { acc[i][j] = Sr::fold(acc[i][j], bl[i][j]); bl[i][j] = inf; }
            }
            T a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const T v = a[i] + b[j];
                    bl[i][j] = v < bl[i][j] ? v : bl[i][j];      // the reference's "if v < out"
                }
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const long long r = r0 + ty + 16 * i, c = c0 + tx + 16 * j;
            if (r < p.M && c < p.N) C[r * p.ldc + c] = Sr::fold(acc[i][j], bl[i][j]);
        }
    }
}

}  // namespace starmm
