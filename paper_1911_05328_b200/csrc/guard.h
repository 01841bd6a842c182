// guard.h -- the range guard's verdict: which exact kernel path the observed operand
// range allows.  Shared by the host (first blocking call of a plan) and
// the device (select_path_kernel: every other call decides on the GPU, no host sync).
#pragma once
#include "../../include/starmm_b200.h"
#include "simt_launch.h"

#ifdef __CUDACC__
#define STARMM_HD __host__ __device__ __forceinline__
#else
#define STARMM_HD inline
#endif

namespace starmm {

constexpr unsigned long long GUARD_BITS_BAD = 1ull, GUARD_BITS_NEG_ZERO = 2ull;

// narrowest (fastest) exact path for operands with max |x| = mx and flag bits `bits`
// (GUARD_BITS_*: non-integral / NaN / -inf, and -0.0).  ordered_ok: the ordered kernel
// may run (local write-back); -0.0 operands of the float (min,+) semirings need it.
STARMM_HD int guard_narrowest(int sr, int flags, long long k, unsigned long long mx,
                              unsigned long long bits, int ordered_ok) {
    const bool fast = !(flags & STARMM_F_NO_FASTPATH);
    const bool bad = (bits & GUARD_BITS_BAD) != 0, negz = (bits & GUARD_BITS_NEG_ZERO) != 0;
    switch (sr) {
    case STARMM_SR_FP64:             // Ozaki-II needs finite inputs (its own guard word)
        return bits ? PATH_DMMA_F64 : PATH_OZAKI_F64;
    case STARMM_SR_INT64: {
        // opt-in tensor cores: small ranges as one int8 GEMM, anything else as radix-256
        // digit GEMMs (exact for every int64); CUDA cores otherwise
        const bool tc = (flags & STARMM_F_INT_TENSOR) != 0;
        if (!fast) return tc ? PATH_TC_I8_LIMBS : PATH_SIMT_I64;
        // exact iff every int32 partial sum fits: K * max|a| * max|b| < 2^31 (the double
        // product is exact below 2^53, so the comparison is exact where it matters)
        const double bound = (double)k * (double)mx * (double)mx;
        if (mx <= 127 && bound < 2147483648.0) return tc ? PATH_TC_I8 : PATH_SIMT_I64_DP4A;
        if (tc) return PATH_TC_I8_LIMBS;
        if (mx < (1ull << 31) && bound < 2147483648.0) return PATH_SIMT_I64_NARROW;
        return PATH_SIMT_I64;
    }
    case STARMM_SR_TROPICAL_F64:
        if (negz && ordered_ok) return PATH_MIN_ORDERED;
        if (!fast) return PATH_SIMT_F64_MIN;
        // integer-valued: int16 when |x| <= 4096, fp32 carrier while sums stay < 2^24
        if (!bad && mx <= 4096ull) return PATH_SIMT_F64T_S16X2;
        if (!bad && mx <= (1ull << 23)) return PATH_SIMT_F64T_CARRIER;
        return PATH_SIMT_F64_MIN;
    case STARMM_SR_TROPICAL_F32:
        if (negz && ordered_ok) return PATH_MIN_ORDERED;
        if (!fast) return PATH_SIMT_F32_PAIR;
        return (!bad && mx <= 4096ull) ? PATH_SIMT_F32_S16X2 : PATH_SIMT_F32_PAIR;
    default:                         // tropical_i32
        if (!fast) return PATH_SIMT_I32_SAT;
        if (mx <= 4096ull) return PATH_SIMT_I32_S16X2;           // int16 sums exact
        if (mx <= (1ull << 23)) return PATH_SIMT_I32_CARRIER;    // fp32-exact sums
        if (mx < (1ull << 28)) return PATH_SIMT_I32_VMIN;        // no overflow
        return PATH_SIMT_I32_SAT;
    }
}

// position in the semiring's chain, narrow (fast, small ranges) to wide (general)
STARMM_HD int path_rank(int path) {
    switch (path) {
    case PATH_TC_I8: case PATH_SIMT_I64_DP4A: case PATH_SIMT_F32_S16X2: case PATH_SIMT_I32_S16X2:
    case PATH_SIMT_F64T_S16X2: case PATH_OZAKI_F64: return 0;
    case PATH_SIMT_I64_NARROW: case PATH_SIMT_F64T_CARRIER: case PATH_SIMT_F32_PAIR:
    case PATH_SIMT_I32_CARRIER: case PATH_DMMA_F64: return 1;
    case PATH_SIMT_I64: case PATH_SIMT_F64_MIN: case PATH_SIMT_I32_VMIN: case PATH_TC_I8_LIMBS: return 2;
    case PATH_SIMT_I32_SAT: return 3;
    case PATH_MIN_ORDERED: return 9;
    }
    return 8;
}

// is `path` exact for data whose narrowest allowed path is `nar`?
STARMM_HD bool path_allowed(int path, int nar) {
    if (nar == PATH_MIN_ORDERED) return path == PATH_MIN_ORDERED;
    return path_rank(path) >= path_rank(nar);
}

}  // namespace starmm
