// generate.cuh -- counter-based input generation on the device.
//
// Every element is a pure function of (seed, stream id, GLOBAL row, GLOBAL column):
// Philox4x32-10 on the counter (col, row, stream, 0) with key (seed lo, seed hi), then
// a deterministic transform to the requested distribution.  So any rank generates its
// own panel of a matrix without receiving anything (no broadcast of A / B panels), any
// panel can be regenerated anywhere -- the CPU oracle regenerates the panels of sampled
// output tiles bit for bit (oracle/starmm_oracle.c oracle_generate restates this file) --
// and the values do not depend on how the matrix is cut into panels.
//
// Distributions (mirroring the BASELINE configs; the reference's own fixture generator
// is numpy-based, matrix.py:196-214, and stays the tests' generator):
//   UNIFORM_REAL  a + (b - a) * u,  u = 53 random bits * 2^-53 in [0, 1)
//   NORMAL        a + b * z, z by Box-Muller with a log and a cos built from + - * /
//                 only (no FMA: explicit _rn intrinsics), identical on host and device
//   UNIFORM_INT   integers in [a, b] (multiply-shift on 32 random bits)
//   GRAPH         edge with probability p (32-bit threshold): weight UNIFORM_INT[a, b],
//                 else the additive identity (+inf / INT32_MAX)
// Flag ZERO_DIAG: element (i, i) = 0 (the tropical one: "0 on the diagonal").
#pragma once
#include <cstdint>
#include "common.cuh"

namespace starmm {
namespace gen {

enum Dist : int { UNIFORM_REAL = 0, NORMAL = 1, UNIFORM_INT = 2, GRAPH = 3 };
constexpr int FLAG_ZERO_DIAG = 1;

struct Philox { uint32_t x[4]; };

STARMM_DEV Philox philox10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(M0, c0), lo0 = M0 * c0;
        const uint32_t hi1 = __umulhi(M1, c2), lo1 = M1 * c2;
        const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += W0; k1 += W1;
    }
    Philox p;
    p.x[0] = c0; p.x[1] = c1; p.x[2] = c2; p.x[3] = c3;
    return p;
}

// exact operations only (never contracted into an FMA), so the host restatement
// compiled with -ffp-contract=off rounds identically
STARMM_DEV double mul(double a, double b) { return __dmul_rn(a, b); }
STARMM_DEV double add(double a, double b) { return __dadd_rn(a, b); }
STARMM_DEV double sub(double a, double b) { return __dsub_rn(a, b); }
STARMM_DEV double dvd(double a, double b) { return __ddiv_rn(a, b); }

// correctly rounded coefficient tables (hex literals: the same bits on host and device)
__device__ __constant__ const double INV_ODD[12] = {   // 1/1, 1/3, ..., 1/23
    0x1.0000000000000p+0, 0x1.5555555555555p-2, 0x1.999999999999ap-3, 0x1.2492492492492p-3,
    0x1.c71c71c71c71cp-4, 0x1.745d1745d1746p-4, 0x1.3b13b13b13b14p-4, 0x1.1111111111111p-4,
    0x1.e1e1e1e1e1e1ep-5, 0x1.af286bca1af28p-5, 0x1.8618618618618p-5, 0x1.642c8590b2164p-5};
__device__ __constant__ const double INV_FACT_EVEN[14] = {   // 1/(2k)!
    0x1.0000000000000p+0, 0x1.0000000000000p-1, 0x1.5555555555555p-5, 0x1.6c16c16c16c17p-10,
    0x1.a01a01a01a01ap-16, 0x1.27e4fb7789f5cp-22, 0x1.1eed8eff8d898p-29, 0x1.93974a8c07c9dp-37,
    0x1.ae7f3e733b81fp-45, 0x1.6827863b97d97p-53, 0x1.e542ba4020225p-62, 0x1.0ce396db7f853p-70,
    0x1.f2cf01972f578p-80, 0x1.88e85fc6a4e5ap-89};
__device__ __constant__ const double INV_FACT_ODD[14] = {    // 1/(2k+1)!
    0x1.0000000000000p+0, 0x1.5555555555555p-3, 0x1.1111111111111p-7, 0x1.a01a01a01a01ap-13,
    0x1.71de3a556c734p-19, 0x1.ae64567f544e4p-26, 0x1.6124613a86d09p-33, 0x1.ae7f3e733b81fp-41,
    0x1.952c77030ad4ap-49, 0x1.2f49b46814157p-57, 0x1.71b8ef6dcf572p-66, 0x1.761b41316381ap-75,
    0x1.3f3ccdd165fa9p-84, 0x1.d1ab1c2dccea3p-94};

// natural log of x in (0, 1]: x = m * 2^e with m in [sqrt(1/2), sqrt(2)), then
// log m = 2 atanh(s), s = (m - 1) / (m + 1), |s| <= 0.1716 (series to s^23, Horner)
STARMM_DEV double det_log(double x) {
    long long bits = __double_as_longlong(x);
    int e = (int)((bits >> 52) & 0x7ff) - 1023;
    bits = (bits & 0x000fffffffffffffLL) | 0x3ff0000000000000LL;   // m in [1, 2)
    double m = __longlong_as_double(bits);
    if (m > 0x1.6a09e667f3bcdp+0) { m = mul(m, 0.5); e += 1; }     // sqrt(2)
    const double s = dvd(sub(m, 1.0), add(m, 1.0));
    const double s2 = mul(s, s);
    double t = INV_ODD[11];
#pragma unroll
    for (int k = 10; k >= 0; --k) t = add(mul(t, s2), INV_ODD[k]);
    const double lm = mul(mul(2.0, s), t);
    const double LN2_HI = 0x1.62e42fee00000p-1, LN2_LO = 0x1.a39ef35793c76p-33;
    return add(mul((double)e, LN2_HI), add(mul((double)e, LN2_LO), lm));
}

// cos(2 pi u) for u in [0, 1): quarter turn q and a = f * pi/2, f in [0, 1); Taylor
// series of cos a and sin a to a^27 (|a| < pi/2: truncation < 1e-19), Horner
STARMM_DEV double det_cos2pi(double u) {
    const double t = mul(u, 4.0);               // exact
    const int q = (int)t;
    const double f = sub(t, (double)q);         // exact
    const double a = mul(f, 0x1.921fb54442d18p+0);
    const double a2 = mul(a, a);
    double c = -INV_FACT_EVEN[13], sn = -INV_FACT_ODD[13];   // k = 13: odd, negative
#pragma unroll
    for (int k = 12; k >= 0; --k) {
        const double ce = (k & 1) ? -INV_FACT_EVEN[k] : INV_FACT_EVEN[k];
        const double so = (k & 1) ? -INV_FACT_ODD[k] : INV_FACT_ODD[k];
        c = add(mul(c, a2), ce);
        sn = add(mul(sn, a2), so);
    }
    sn = mul(sn, a);
    switch (q & 3) {
    case 0: return c;
    case 1: return -sn;
    case 2: return -c;
    default: return sn;
    }
}

struct Params {
    int dist, flags;
    double a, b, p;
    uint64_t seed;
    uint32_t stream;
};

// the value of element (i, j) as a double (exact for the integer distributions)
STARMM_DEV double value(const Params& g, long long i, long long j, bool* absent) {
    // counter (col, row, stream, 0): rows and columns stay below 2^31 (plan limit)
    const Philox r = philox10((uint32_t)j, (uint32_t)i, g.stream, 0u, (uint32_t)g.seed,
                              (uint32_t)(g.seed >> 32));
    *absent = false;
    switch (g.dist) {
    case UNIFORM_REAL: {
        const uint64_t u53 = ((uint64_t)r.x[0] << 21) | (r.x[1] >> 11);
        const double u = mul((double)u53, 1.1102230246251565e-16);   // 2^-53
        return add(g.a, mul(sub(g.b, g.a), u));
    }
    case NORMAL: {
        const uint64_t ua = ((uint64_t)r.x[0] << 21) | (r.x[1] >> 11);
        const uint64_t ub = ((uint64_t)r.x[2] << 21) | (r.x[3] >> 11);
        const double u1 = mul((double)(ua + 1), 1.1102230246251565e-16);   // (0, 1]
        const double u2 = mul((double)ub, 1.1102230246251565e-16);         // [0, 1)
        const double rad = __dsqrt_rn(mul(-2.0, det_log(u1)));
        return add(g.a, mul(g.b, mul(rad, det_cos2pi(u2))));
    }
    case UNIFORM_INT: {
        const uint64_t span = (uint64_t)((long long)g.b - (long long)g.a + 1);
        return (double)((long long)g.a + (long long)(((uint64_t)r.x[0] * span) >> 32));
    }
    default: {                                   // GRAPH
        const uint32_t thr = (uint32_t)(g.p * 4294967296.0);
        if (!(r.x[1] < thr)) { *absent = true; return 0.0; }
        const uint64_t span = (uint64_t)((long long)g.b - (long long)g.a + 1);
        return (double)((long long)g.a + (long long)(((uint64_t)r.x[0] * span) >> 32));
    }
    }
}

template <class Sr>
__global__ void generate_kernel(typename Sr::T* out, long long ld, long long rows, long long cols,
                                long long row0, long long col0, Params g) {
    using T = typename Sr::T;
    for (long long r = blockIdx.y; r < rows; r += gridDim.y)
        for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < cols;
             c += (long long)gridDim.x * blockDim.x) {
            const long long i = row0 + r, j = col0 + c;
            bool absent;
            const double v = value(g, i, j, &absent);
            T x = absent ? Sr::identity() : (T)v;
            if ((g.flags & FLAG_ZERO_DIAG) && i == j) x = (T)0;
            out[r * ld + c] = x;
        }
}

}  // namespace gen
}  // namespace starmm
