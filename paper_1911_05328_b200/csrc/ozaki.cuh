// ozaki.cuh -- OPT-IN fp64 (+,x) on the int8 tensor cores: Ozaki scheme II.
//
// The reference's float semiring computes C <- C + A @ B in float64
// (semiring.py:35-45, numba, separate mul and add).  B200 has no fp64 kind for
// tcgen05, and its DMMA path tops out at 37 TF/s; this path instead computes the
// product EXACTLY for integer-scaled operands and rounds once:
//
//   1. scale   A'_ik = rint(a_ik * 2^sig_i),  B'_kj = rint(b_kj * 2^tau_j)
//              sig_i = t - e_i with max_k |a_ik| < 2^e_i (per row of A; per column
//              of B likewise), so |A'|, |B'| <= 2^t.  This truncation is the ONLY
//              approximation: |a - A' 2^-sig| <= 2^(e_i - t - 1).
//   2. residues  A'_p = A' mod m_p (symmetric, int8) for P pairwise-coprime moduli
//              m_p <= 256, M = prod m_p > 2 k 2^(2t)  (t = 54 at k = 2^14, >= 53 up
//              to k < 2^17)
//   3. P int8 GEMMs on tcgen05 (tc_gemm.cuh): acc_p = A'_p B'_p exactly in int32
//              (|acc| <= k * 2^14 < 2^31)
//   4. CRT (oz_crt_kernel): X = sum_p rho_p W_p mod M, rho_p = acc_p mod m_p, centred into
//              (-M/2, M/2] -- the exact integer sum_k A'_ik B'_kj -- then one
//              correctly rounded int128 -> double conversion and an exact 2^-(sig+tau)
//              scaling, folded into C (one more rounding, as the reference's C + tmp).
//
// Error: |C_emu - C_exact| <= 2^(1-t) k max_k|a_ik| max_k|b_kj| + rounding, the same
// k * unit * magnitude form as DGEMM's gamma_k sum|a||b| bound.
// Non-finite inputs (NaN / inf) cannot be emulated: the guard sends them to DMMA.
#pragma once
#include <cstdint>
#include "common.cuh"
#include "tc_gemm.cuh"

namespace starmm {
namespace oz {
constexpr int P = 16;
// pairwise coprime, descending: M = prod = 2^125.38
constexpr int MOD[P] = {256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193};
constexpr int MOD_LAST = MOD[P - 1];
constexpr int PLANE = tcg::BM * tcg::BN;        // residue bytes per CTA-tile plane
}  // namespace oz

// sig = t - e with |x| < 2^e (e = frexp's exponent) from the bit pattern of |x|
// (finite: the guard sends inf / NaN elsewhere); an all-zero row or column -> 0
STARMM_DEV int oz_sigma(unsigned long long bits, int t) {
    if (bits == 0) return 0;
    const int ef = (int)(bits >> 52);
    const int e = ef ? ef - 1022 : 64 - __clzll((long long)bits) - 1074;   // normal : subnormal
    return t - e;
}

// x * 2^e, exact: one multiply by a constructed power of two in the normal range
// (scalbn's general path only for exponents outside it)
STARMM_DEV double oz_ldexp(double x, int e) {
    if (e >= -1022 && e <= 1023) return x * __hiloint2double((e + 1023) << 20, 0);
    return scalbn(x, e);
}

// Integer form for the packers: x = x2 2^42 + x1 2^21 + x0 (|x| <= 2^62, x0, x1 in
// [0, 2^21)), so x mod m = (x2 c2 + x1 c1 + x0) mod m with c_i = 2^(21 i) mod m: two
// IMADs into an int32 (|.| < 2^30), a non-negative offset, one constant modulo.
template <int m>
STARMM_DEV uint32_t oz_res_limbs(int x2, int x1, int x0) {
    if (m == 256) return (uint32_t)x0 & 0xff;                    // two's-complement low byte
    constexpr int c1 = (int)((1LL << 21) % m), c2 = (int)((1LL << 42) % m);
    constexpr int OFF = m * ((1 << 30) / m + 1);                 // makes the sum non-negative
    const uint32_t u = (uint32_t)(x2 * c2 + x1 * c1 + x0 + OFF) % (uint32_t)m;
    const int r = (int)u - ((int)u > (m - 1) / 2 ? m : 0);     // symmetric
    return (uint32_t)r & 0xff;
}

// The same residue on the FP64 pipe: q = rint(x / m) can be off by one (x/m rounds),
// the remainder fma(-m, q, x) is exact, and the symmetric fold is integer.
template <int m>
STARMM_DEV uint32_t oz_res_f64(double x) {
    const double q = rint(x * (1.0 / m));
    int r = (int)fma(-(double)m, q, x);
    r += (r < -((m - 1) / 2)) ? m : 0;
    r -= (r > (m - 1) / 2) ? m : 0;
    return (uint32_t)r & 0xff;
}

// All P residues of one scaled element, ORed into byte `shift` of each plane's word.
// Odd moduli go through the FP64 pipe, even ones through IMAD: the packers are
// math-pipe bound, and the two pipes issue in parallel.
template <int I = 0>
STARMM_DEV void oz_pack_element(double xd, long long x, int shift, uint32_t (&packed)[oz::P]) {
    if constexpr (I < oz::P) {
        uint32_t r;
        if constexpr (I % 2 == 1) {
            r = oz_res_f64<oz::MOD[I]>(xd);
        } else {
            const int x0 = (int)(x & 0x1FFFFF), x1 = (int)((x >> 21) & 0x1FFFFF), x2 = (int)(x >> 42);
            r = oz_res_limbs<oz::MOD[I]>(x2, x1, x0);
        }
        packed[I] |= r << shift;
        oz_pack_element<I + 1>(xd, x, shift, packed);
    }
}

// ---- scale pass: max |x| per row of A / per column of B (as ordered bit patterns) ---
// flag[0] |= 1 when any element is NaN or +-inf (the bit pattern of |x| >= +inf).
__global__ void oz_amax_rows_kernel(const double* A, long long m, long long k, long long lda,
                                    unsigned long long* rowmax, unsigned long long* flag) {
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long r = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < m; r += warps) {
        const double* a = A + r * lda;
        unsigned long long mx = 0;
        for (long long j = lane; j < k; j += 32) {
            const unsigned long long b = (unsigned long long)__double_as_longlong(a[j]) & 0x7fffffffffffffffULL;
            mx = b > mx ? b : mx;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const unsigned long long y = __shfl_xor_sync(0xffffffffu, mx, o);
            mx = y > mx ? y : mx;
        }
        if (lane == 0) {
            rowmax[r] = mx;
            if (mx >= 0x7ff0000000000000ULL) atomicOr(flag, 1ULL);
        }
    }
}

// block (32, 8): 32 columns x 256 rows of B; atomicMax into colmax (zeroed first)
__global__ void oz_amax_cols_kernel(const double* B, long long k, long long n, long long ldb,
                                    unsigned long long* colmax, unsigned long long* flag) {
    __shared__ unsigned long long red[8][32];
    const long long c = (long long)blockIdx.x * 32 + threadIdx.x;
    const long long k0 = (long long)blockIdx.y * 256;
    unsigned long long mx = 0;
    if (c < n) {
        for (long long i = k0 + threadIdx.y; i < k0 + 256 && i < k; i += 8) {
            const unsigned long long b = (unsigned long long)__double_as_longlong(B[i * ldb + c]) & 0x7fffffffffffffffULL;
            mx = b > mx ? b : mx;
        }
    }
    red[threadIdx.y][threadIdx.x] = mx;
    __syncthreads();
    if (threadIdx.y == 0 && c < n) {
        for (int y = 1; y < 8; ++y) mx = red[y][threadIdx.x] > mx ? red[y][threadIdx.x] : mx;
        atomicMax(&colmax[c], mx);
        if (mx >= 0x7ff0000000000000ULL) atomicOr(flag, 1ULL);
    }
}

// ---- residue packing -----------------------------------------------------------
// A [m][k] (row-major = K-major already) -> P planes [Mp][Kp] int8; each thread
// converts 4 consecutive k of one row and stores one 32-bit word per plane.
// Grid: x over the k-words of a row, y strides over rows (no divisions).
__global__ void oz_pack_rows_kernel(const double* A, long long m, long long k, long long lda,
                                    const unsigned long long* rowmax, int t, signed char* out,
                                    long long Mp, long long Kp, Pred pr = Pred()) {
    if (pr.off()) return;
    const long long plane = Mp * Kp;
    const long long k0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (k0 >= Kp) return;
    for (long long r = blockIdx.y; r < Mp; r += gridDim.y) {
        uint32_t packed[oz::P];
#pragma unroll
        for (int p = 0; p < oz::P; ++p) packed[p] = 0;
        if (r < m) {
            const int sig = oz_sigma(rowmax[r], t);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const long long kk = k0 + e;
                if (kk < k) {
                    const double xd = rint(oz_ldexp(A[r * lda + kk], sig));
                    oz_pack_element(xd, (long long)xd, 8 * e, packed);
                }
            }
        }
#pragma unroll
        for (int p = 0; p < oz::P; ++p)
            *reinterpret_cast<uint32_t*>(out + p * plane + r * Kp + k0) = packed[p];
    }
}

// B [k][n] -> P planes [Np][Kp] int8 (transposed to K-major through shared memory).
// Block (32, 8) covers 32 columns x 64 k: thread (tx, ty) converts k-words ty and
// ty + 8 (4 consecutive k each) of column tx -- coalesced row reads -- and packs one
// 32-bit word per plane; the planes leave through a 17-word-pitch transpose tile.
__global__ void __launch_bounds__(256)
oz_pack_cols_kernel(const double* B, long long k, long long n, long long ldb,
                    const unsigned long long* colmax, int t, signed char* out, long long Np, long long Kp,
                    Pred pr = Pred()) {
    if (pr.off()) return;
    constexpr int TK = 64, KW = TK / 4, PITCH = KW + 1;
    __shared__ uint32_t tile[oz::P][32][PITCH];
    const long long c0 = (long long)blockIdx.x * 32, k0 = (long long)blockIdx.y * TK;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const long long c = c0 + tx;
    const int tau = (c < n) ? oz_sigma(colmax[c], t) : 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int kw = ty + 8 * h;
        uint32_t packed[oz::P];
#pragma unroll
        for (int p = 0; p < oz::P; ++p) packed[p] = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const long long kk = k0 + kw * 4 + e;
            if (c < n && kk < k) {
                const double xd = rint(oz_ldexp(B[kk * ldb + c], tau));
                oz_pack_element(xd, (long long)xd, 8 * e, packed);
            }
        }
#pragma unroll
        for (int p = 0; p < oz::P; ++p) tile[p][tx][kw] = packed[p];
    }
    __syncthreads();
    const long long plane = Np * Kp;
    const int tid = ty * 32 + tx;
#pragma unroll 4
    for (int idx = tid; idx < oz::P * 32 * KW; idx += 256) {
        const int p = idx / (32 * KW), rem = idx - p * 32 * KW;
        const int col = rem / KW, wd = rem - col * KW;
        const long long cc = c0 + col, kk = k0 + wd * 4;
        if (cc < Np && kk < Kp)
            *reinterpret_cast<uint32_t*>(out + p * plane + cc * Kp + kk) = tile[p][col][wd];
    }
}

// ---- the CRT epilogue ------------------------------------------------------------
struct OzCrt {
    uint32_t W[oz::P][4];      // CRT weights (M/m_p) * ((M/m_p)^-1 mod m_p) mod M, 32-bit limbs
    uint32_t Ml[4];            // M
    uint32_t Mh[4];            // floor(M / 2)
    double invM;               // 1 / M (rounded)
};

template <int m>
STARMM_DEV void oz_pass_residues(const uint32_t (&v)[32], uint32_t (&packed)[8]) {
#pragma unroll
    for (int w = 0; w < 8; ++w) {
        uint32_t x = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int a = (int)v[w * 4 + e];
            int r = a % m;
            if (r < 0) r += m;
            x |= (uint32_t)r << (8 * e);
        }
        packed[w] = x;
    }
}

template <int I = 0>
STARMM_DEV void oz_pass_dispatch(int pass, const uint32_t (&v)[32], uint32_t (&packed)[8]) {
    if constexpr (I < oz::P) {
        if (pass == I) oz_pass_residues<oz::MOD[I]>(v, packed);
        else oz_pass_dispatch<I + 1>(pass, v, packed);
    }
}

// exact X = CRT(rho) centred into (-M/2, M/2], returned as a correctly rounded double
// d and a power-of-two exponent: X = d * 2^ex (d integral or 0)
STARMM_DEV double oz_reconstruct(const OzCrt& k, const uint32_t (&rho)[oz::P], int& ex) {
    unsigned long long a0 = 0, a1 = 0, a2 = 0, a3 = 0;     // limb columns, each < 2^44
#pragma unroll
    for (int p = 0; p < oz::P; ++p) {
        a0 += (unsigned long long)rho[p] * k.W[p][0];
        a1 += (unsigned long long)rho[p] * k.W[p][1];
        a2 += (unsigned long long)rho[p] * k.W[p][2];
        a3 += (unsigned long long)rho[p] * k.W[p][3];
    }
    // normalise S = sum rho_p W_p into 32-bit limbs s0..s4 (S < 2^140)
    uint32_t s0 = (uint32_t)a0;
    a1 += a0 >> 32;
    uint32_t s1 = (uint32_t)a1;
    a2 += a1 >> 32;
    uint32_t s2 = (uint32_t)a2;
    a3 += a2 >> 32;
    uint32_t s3 = (uint32_t)a3;
    uint32_t s4 = (uint32_t)(a3 >> 32);
    // q = floor(S / M), estimated in double (off by at most one either way)
    const double sd = ((double)s4 * 4294967296.0 + (double)s3) * 7.9228162514264338e28 /* 2^96 */ +
                      (double)s2 * 1.8446744073709552e19 /* 2^64 */;
    const double qd = floor(sd * k.invM);
    const uint32_t q = qd > 0.0 ? (uint32_t)qd : 0u;               // S / M < 2^15
    // R = S - q M in signed 64-bit limb arithmetic
    long long d;
    uint32_t r0, r1, r2, r3;
    d = (long long)s0 - (long long)((unsigned long long)q * (unsigned long long)k.Ml[0]);
    r0 = (uint32_t)d; d >>= 32;
    d += (long long)s1 - (long long)((unsigned long long)q * (unsigned long long)k.Ml[1]);
    r1 = (uint32_t)d; d >>= 32;
    d += (long long)s2 - (long long)((unsigned long long)q * (unsigned long long)k.Ml[2]);
    r2 = (uint32_t)d; d >>= 32;
    d += (long long)s3 - (long long)((unsigned long long)q * (unsigned long long)k.Ml[3]);
    r3 = (uint32_t)d; d >>= 32;
    d += (long long)s4;                                     // top: 0, or -1 if q was one too big
    if (d < 0) {                                            // R += M
        unsigned long long c = (unsigned long long)r0 + k.Ml[0]; r0 = (uint32_t)c; c >>= 32;
        c += (unsigned long long)r1 + k.Ml[1]; r1 = (uint32_t)c; c >>= 32;
        c += (unsigned long long)r2 + k.Ml[2]; r2 = (uint32_t)c; c >>= 32;
        c += (unsigned long long)r3 + k.Ml[3]; r3 = (uint32_t)c;
    } else {
        // R >= M (q one too small) -> R -= M
        const bool ge = d > 0 || r3 > k.Ml[3] ||
                        (r3 == k.Ml[3] && (r2 > k.Ml[2] || (r2 == k.Ml[2] && (r1 > k.Ml[1] ||
                        (r1 == k.Ml[1] && r0 >= k.Ml[0])))));
        if (ge) {
            long long b = (long long)r0 - k.Ml[0]; r0 = (uint32_t)b; b >>= 32;
            b += (long long)r1 - k.Ml[1]; r1 = (uint32_t)b; b >>= 32;
            b += (long long)r2 - k.Ml[2]; r2 = (uint32_t)b; b >>= 32;
            b += (long long)r3 - k.Ml[3]; r3 = (uint32_t)b;
        }
    }
    // centre: R > M/2 -> X = R - M < 0, |X| = M - R
    const bool neg = r3 > k.Mh[3] ||
                     (r3 == k.Mh[3] && (r2 > k.Mh[2] || (r2 == k.Mh[2] && (r1 > k.Mh[1] ||
                     (r1 == k.Mh[1] && r0 > k.Mh[0])))));
    if (neg) {
        long long b = (long long)k.Ml[0] - r0; r0 = (uint32_t)b; b >>= 32;
        b += (long long)k.Ml[1] - r1; r1 = (uint32_t)b; b >>= 32;
        b += (long long)k.Ml[2] - r2; r2 = (uint32_t)b; b >>= 32;
        b += (long long)k.Ml[3] - r3; r3 = (uint32_t)b;
    }
    const unsigned long long hi = ((unsigned long long)r3 << 32) | r2;
    const unsigned long long lo = ((unsigned long long)r1 << 32) | r0;
    double mag;
    if (hi == 0) {
        mag = __ull2double_rn(lo);
        ex = 0;
    } else {
        const int lz = __clzll((long long)hi);
        unsigned long long top = lz ? ((hi << lz) | (lo >> (64 - lz))) : hi;
        const unsigned long long rest = lz ? (lo << lz) : lo;
        top |= (rest != 0);                                 // sticky bit: one correct rounding
        mag = __ull2double_rn(top);
        ex = 64 - lz;
    }
    return neg ? -mag : mag;
}

// Epilogue of the P-pass residue GEMM: reduce each accumulator to its residue
// acc_p mod m_p (one byte) and store it to the residue planes R[P][Mp][Np]; TMEM is
// released as soon as a tile is read, so the epilogue never throttles the MMAs.
struct EpiOzakiResidues {
    unsigned char* R;
    long long Mp, Np;
    STARMM_DEV void operator()(const TcgChunk& c, const uint32_t (&v)[32]) const {
        uint32_t packed[8];
        oz_pass_dispatch(c.pass, v, packed);
        uint4* dst = reinterpret_cast<uint4*>(R + ((size_t)c.pass * Mp + (c.row0 + c.lane)) * Np + c.col0);
        dst[0] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
        dst[1] = make_uint4(packed[4], packed[5], packed[6], packed[7]);
    }
};

// CRT reconstruction, exact scaling and the fold into C.  One thread per 8 consecutive
// output columns of one row: per plane ONE 8-byte load of its 8 residue bytes (a warp
// reads 256 contiguous bytes of each plane -- with 4-byte loads of 16-column groups
// only a quarter of every sector was used and the kernel was L1/L2-throughput bound,
// ncu: 84% memory throughput at 2.2 TB/s of DRAM), then 2 groups of 4 columns.
constexpr int OZ_CRT_W = 8;
__global__ void __launch_bounds__(128)
oz_crt_kernel(const unsigned char* __restrict__ R, long long Mp, long long Np,
              const unsigned long long* __restrict__ rowmax, const unsigned long long* __restrict__ colmax,
              int t, const OzCrt crt, const TcgOut o, Pred pr = Pred()) {
    if (pr.off()) return;
    // grid: x over 8-column groups of a row, y strides over rows (no divisions)
    const long long c0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * OZ_CRT_W;
    if (c0 >= o.N) return;
    const size_t plane = (size_t)Mp * Np;
    for (long long row = blockIdx.y; row < o.M; row += gridDim.y) {
        const unsigned char* rbase = R + (size_t)row * Np + c0;   // 8-byte aligned (c0 % 8 == 0)
        const bool local = o.remote_parts == 0;
        const int ncol = (int)min((long long)OZ_CRT_W, o.N - c0);
        double* crow = (double*)o.C + row * o.ldc + c0;
        const int sig = oz_sigma(rowmax[row], t);
        uint2 word8[oz::P];                          // residue bytes of the 8 columns
#pragma unroll
        for (int p = 0; p < oz::P; ++p) word8[p] = __ldcs(reinterpret_cast<const uint2*>(rbase + p * plane));
        // 2 groups of 4 columns: the group loop stays rolled (code size: the body is
        // ~250 instructions per element); C loads lead the arithmetic
#pragma unroll 1
        for (int g = 0; g < OZ_CRT_W / 4; ++g) {
            double cv[4];
            int tau[4];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
                const int j = 4 * g + jj;
                cv[jj] = (local && !o.init_identity && j < ncol) ? crow[j] : 0.0;
                tau[jj] = j < ncol ? oz_sigma(colmax[c0 + j], t) : 0;
            }
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
                const int j = 4 * g + jj;
                uint32_t rho[oz::P];
#pragma unroll
                for (int p = 0; p < oz::P; ++p) {
                    const uint32_t w = g ? word8[p].y : word8[p].x;
                    rho[p] = (w >> (8 * jj)) & 0xff;
                }
                if (j < ncol) {
                    int ex;
                    const double d = oz_reconstruct(crt, rho, ex);
                    const double val = oz_ldexp(d, ex - sig - tau[jj]);
                    if (local) crow[j] = o.init_identity ? val : cv[jj] + val;
                    else tcg_fold<SrFp64>(o, row, c0 + j, val);
                }
            }
        }
    }
}

}  // namespace starmm
