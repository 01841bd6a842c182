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
//   4. CRT: X = sum_p rho_p W_p mod M, rho_p = acc_p mod m_p, centred into
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

// exponent e with |x| < 2^e for x = bits (non-negative double bit pattern); 0 row -> sig 0
STARMM_DEV int oz_sigma(unsigned long long bits, int t) {
    if (bits == 0) return 0;
    int e;
    frexp(__longlong_as_double((long long)bits), &e);
    return t - e;
}

// symmetric residue of an integral double |x| <= 2^62 modulo a constant m <= 256
template <int m>
STARMM_DEV int oz_res(double x) {
    if (m == 256) return (int)(signed char)(unsigned char)((unsigned long long)(long long)x & 0xff);
    const double q = rint(x * (1.0 / m));
    double r = fma(-(double)m, q, x);            // exact: the true remainder is small
    if (r > (m - 1) / 2) r -= m;
    else if (r < -((m - 1) / 2)) r += m;
    return (int)r;
}

template <int I = 0>
STARMM_DEV void oz_residues(double x, int (&r)[oz::P]) {
    if constexpr (I < oz::P) {
        r[I] = oz_res<oz::MOD[I]>(x);
        oz_residues<I + 1>(x, r);
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
__global__ void oz_pack_rows_kernel(const double* A, long long m, long long k, long long lda,
                                    const unsigned long long* rowmax, int t, signed char* out,
                                    long long Mp, long long Kp) {
    const long long words = Mp * (Kp / 4);
    const long long plane = Mp * Kp;
    for (long long w = (long long)blockIdx.x * blockDim.x + threadIdx.x; w < words;
         w += (long long)gridDim.x * blockDim.x) {
        const long long r = w / (Kp / 4), k0 = (w - r * (Kp / 4)) * 4;
        uint32_t packed[oz::P];
#pragma unroll
        for (int p = 0; p < oz::P; ++p) packed[p] = 0;
        if (r < m) {
            const int sig = oz_sigma(rowmax[r], t);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const long long kk = k0 + e;
                if (kk < k) {
                    const double x = rint(scalbn(A[r * lda + kk], sig));
                    int res[oz::P];
                    oz_residues(x, res);
#pragma unroll
                    for (int p = 0; p < oz::P; ++p) packed[p] |= (uint32_t)(res[p] & 0xff) << (8 * e);
                }
            }
        }
#pragma unroll
        for (int p = 0; p < oz::P; ++p)
            *reinterpret_cast<uint32_t*>(out + p * plane + r * Kp + k0) = packed[p];
    }
}

// B [k][n] -> P planes [Np][Kp] int8 (transposed to K-major through shared memory).
// Block (32, 8) covers 32 columns x 64 k.
__global__ void oz_pack_cols_kernel(const double* B, long long k, long long n, long long ldb,
                                    const unsigned long long* colmax, int t, signed char* out,
                                    long long Np, long long Kp) {
    constexpr int TK = 64, PITCH = TK + 4;   // bytes; 17-word pitch spreads banks
    __shared__ __align__(16) unsigned char tile[oz::P][32][PITCH];
    const long long c0 = (long long)blockIdx.x * 32, k0 = (long long)blockIdx.y * TK;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const long long c = c0 + tx;
    const int tau = (c < n) ? oz_sigma(colmax[c], t) : 0;
    for (int i = ty; i < TK; i += 8) {
        const long long kk = k0 + i;
        int res[oz::P];
        if (c < n && kk < k) {
            oz_residues(rint(scalbn(B[kk * ldb + c], tau)), res);
        } else {
#pragma unroll
            for (int p = 0; p < oz::P; ++p) res[p] = 0;
        }
#pragma unroll
        for (int p = 0; p < oz::P; ++p) tile[p][tx][i] = (unsigned char)(res[p] & 0xff);
    }
    __syncthreads();
    const long long plane = Np * Kp;
    const int tid = ty * 32 + tx;
#pragma unroll 1
    for (int p = 0; p < oz::P; ++p) {
        for (int idx = tid; idx < 32 * (TK / 4); idx += 256) {
            const int col = idx / (TK / 4), wd = idx % (TK / 4);
            const long long cc = c0 + col, kk = k0 + wd * 4;
            if (cc < Np && kk < Kp)
                *reinterpret_cast<uint32_t*>(out + p * plane + cc * Kp + kk) =
                    *reinterpret_cast<const uint32_t*>(&tile[p][col][wd * 4]);
        }
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
    long long q = (long long)floor(sd * k.invM);
    if (q < 0) q = 0;
    // R = S - q M in signed 64-bit limb arithmetic
    long long d;
    uint32_t r0, r1, r2, r3;
    d = (long long)s0 - (long long)((unsigned long long)q * k.Ml[0]);
    r0 = (uint32_t)d; d >>= 32;
    d += (long long)s1 - (long long)((unsigned long long)q * k.Ml[1]);
    r1 = (uint32_t)d; d >>= 32;
    d += (long long)s2 - (long long)((unsigned long long)q * k.Ml[2]);
    r2 = (uint32_t)d; d >>= 32;
    d += (long long)s3 - (long long)((unsigned long long)q * k.Ml[3]);
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

// Epilogue for the P-pass residue GEMM.  Every pass only reduces its accumulator to
// residues and stores them (this thread's row, 32 bytes per chunk) in a per-CTA,
// double-buffered scratch [2][P][128][256] bytes, so TMEM is released at once.  The
// CRT reconstruction of a tile is deferred: it runs in P column slices of 16, one
// after each pass epilogue of the CTA's next tile, hidden under that pass's mainloop.
// Every scratch byte is written and read by the same thread: no cross-thread hazard.
struct EpiOzakiF64 {
    static constexpr bool kDeferred = true;
    static constexpr size_t BUF_BYTES = (size_t)oz::P * oz::PLANE;
    TcgOut o;
    const unsigned long long* rowmax;   // per row of A
    const unsigned long long* colmax;   // per column of B
    int t;
    unsigned char* scratch;             // gridDim.x * 2 * BUF_BYTES bytes
    OzCrt crt;

    STARMM_DEV unsigned char* row_base(int buf, int rl) const {
        return scratch + ((size_t)blockIdx.x * 2 + buf) * BUF_BYTES + (size_t)rl * tcg::BN;
    }

    STARMM_DEV void operator()(const TcgChunk& c, const uint32_t (&v)[32]) const {
        uint32_t packed[8];
        oz_pass_dispatch(c.pass, v, packed);
        uint4* dst = reinterpret_cast<uint4*>(row_base(c.tile_slot & 1, c.warp_q * 32 + c.lane) +
                                              (size_t)c.pass * oz::PLANE + c.chunk * 32);
        dst[0] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
        dst[1] = make_uint4(packed[4], packed[5], packed[6], packed[7]);
    }

    // columns [16 slice, 16 slice + 16) of the previous tile, this thread's row
    STARMM_DEV void deferred(const TcgDeferred& d) const {
        constexpr int W = 16, PITCH = 17;
        const int rl = d.warp_q * 32 + d.lane;
        const unsigned char* base = row_base(d.buf, rl) + d.slice * W;
        uint4 res[oz::P];
#pragma unroll
        for (int p = 0; p < oz::P; ++p) res[p] = *reinterpret_cast<const uint4*>(base + (size_t)p * oz::PLANE);
        const long long row = d.row0 + d.lane;
        const int sig = row < o.M ? oz_sigma(rowmax[row], t) : 0;
        const long long c0 = d.colbase + d.slice * W;
        // this lane's 16 fold targets (two rows of 16 columns per warp step): their C
        // loads are issued now so the DRAM latency overlaps the reconstruction below
        const int half = d.lane >> 4, cl = d.lane & (W - 1);
        const long long col = c0 + cl;
        const bool local = o.remote_parts == 0;
        double cv[16];
#pragma unroll
        for (int rr = 0; rr < 16; ++rr) {
            const long long grow = d.row0 + 2 * rr + half;
            cv[rr] = (local && !o.init_identity && grow < o.M && col < o.N)
                         ? ((const double*)o.C)[grow * o.ldc + col] : 0.0;
        }
        const long long ctau = c0 + (d.lane & (W - 1));
        const int tau_mine = ctau < o.N ? oz_sigma(colmax[ctau], t) : 0;
        double* st = reinterpret_cast<double*>(d.stage);
#pragma unroll
        for (int j = 0; j < W; ++j) {
            uint32_t rho[oz::P];
#pragma unroll
            for (int p = 0; p < oz::P; ++p) {
                const uint32_t w = (j < 4) ? res[p].x : (j < 8) ? res[p].y : (j < 12) ? res[p].z : res[p].w;
                rho[p] = (w >> (8 * (j & 3))) & 0xff;
            }
            int ex;
            const double x = oz_reconstruct(crt, rho, ex);
            const int tau = __shfl_sync(0xffffffffu, tau_mine, j);
            st[d.lane * PITCH + j] = scalbn(x, ex - sig - tau);
        }
        __syncwarp();
        // coalesced fold: two rows of 16 columns (128 B each) per warp instruction
#pragma unroll
        for (int rr = 0; rr < 16; ++rr) {
            const int r = 2 * rr + half;
            const long long grow = d.row0 + r;
            if (grow < o.M && col < o.N) {
                const double x = st[r * PITCH + cl];
                if (local) ((double*)o.C)[grow * o.ldc + col] = o.init_identity ? x : cv[rr] + x;
                else tcg_fold<SrFp64>(o, grow, col, x);
            }
        }
        __syncwarp();
    }
};

}  // namespace starmm
