// simt_kernel.cuh -- CUDA-core semiring tile product for the semirings with
// no tensor-core path: (min,+) over fp32 / int32 / fp64 and exact int64 (+,x).
//
// Replaces the reference's numba kernels _mm_minplus / _mm_int
// (semiring.py:22-32, 48-60).  One kernel template, specialised by an inner
// "term" policy:
//
//   PolF32Pair   fp32 (min,+) on k-PAIRS: FADD2 (packed add of two k terms)
//                + FMNMX3 (3-input min)  -> 1 issue slot per inner term.
//                Also the exact carrier for int32 (min,+) when every finite
//                |x| <= 2^23 (range guard): sums stay exact in fp32.
//   PolI32Vmin   int32 (min,+): VIADDMNMX (min(a+b, c) in one DPX op); finite
//                |x| < 2^28 with +inf encoded as 2^30-1 (no overflow possible).
//   PolI32Sat    int32 (min,+) general: saturating semantics of the oracle.
//   PolF64Min    fp64 (min,+) (the reference's own "tropical"): DADD + DMNMX.
//   PolI64       int64 (+,x) mod 2^64: IMAD.WIDE + IMAD + IADD3 (4 SASS/term).
//   PolI64Narrow int64 (+,x) when K*max|a|*max|b| < 2^31 (range guard): IMAD
//                on int32 accumulators, sign-extended in the epilogue -- exact.
//
// Operands come from PACKED panels (aux_kernels.cuh pack_*): A and B are both
// laid out k-group-major, P[k/G][x][G] (x = m for A, n for B; G = 2 for the
// paired policy, else 1), padded to the tile grid with the product's
// annihilator, so a k-stage is a contiguous slab that 16-byte cp.async copies
// verbatim and every thread reads its operands with conflict-free LDS.128.
//
//   PolI8Dp4a    int64 (+,x) when |x| <= 127 and K*max|a|*max|b| < 2^31: IDP.4A
//                (dp4a) over four packed int8 k terms -- 4 terms per lane-op.
//   PolS16x2Min  integer-valued (min,+) with |x| <= 4096: VIADDMNMX.S16x2 on two
//                output columns per lane-op.
//
// CTA tile 128 x (128*OUTS), 256 threads, 8x8 accumulators per thread (each
// accumulator holds OUTS outputs), k-stage Pol::BK, cp.async ring of 3 stages (4 for
// the cross-stage fragment ring of the XSTAGE policies, see mainloop).  Warps
// are 4 (rows) x 8 (cols) threads so A reads broadcast across 8 lanes and B
// reads across 4.  The kernel is persistent: begin() / mainloop() / finish() per
// leaf task, the next task's first k-stages in flight before the write-back, and
// exclusive write-backs of full aligned tiles through the vectorised epilogue
// (writeback.cuh epilogue_row_vec).
#pragma once
#include <type_traits>
#include "common.cuh"
#include "writeback.cuh"
#include "dmma_kernel.cuh"   // cp.async helpers

namespace starmm {

// ---- inner term policies ---------------------------------------------------
struct PolF32Pair {        // packed element float, G = 2, accumulator float
    using Tp = float; using Acc = float;
    static constexpr int G = 2;
    static constexpr int KSTEP = 2, OUTS = 1, BK = 16;
    static constexpr int OCC = 2;   // CTAs per SM (tools/sweep_simt.cu)
    static STARMM_DEV Acc init() { return __int_as_float(0x7f800000); }
    // a = (A[i][k], A[i][k+1]), b = (B[k][j], B[k+1][j])
    static STARMM_DEV void term2(Acc& c, float2 a, float2 b) {
        float2 v = __fadd2_rn(a, b);
        c = fminf(fminf(c, v.x), v.y);
    }
};
struct PolF32Single {      // fp32 (min,+) one k at a time: FADD + FMNMX (ptxas may fuse k pairs)
    using Tp = float; using Acc = float;
    static constexpr int G = 1;
    static constexpr int KSTEP = 1, OUTS = 1, BK = 16;
    static constexpr int OCC = 1;   // CTAs per SM (tools/sweep_simt.cu)
    static STARMM_DEV Acc init() { return __int_as_float(0x7f800000); }
    static STARMM_DEV void term(Acc& c, Tp a, Tp b) { c = fminf(c, a + b); }
};
struct PolF32PairMin2 {    // FADD2 + two 2-input FMNMX
    using Tp = float; using Acc = float;
    static constexpr int G = 2;
    static constexpr int KSTEP = 2, OUTS = 1, BK = 16;
    static constexpr int OCC = 1;   // CTAs per SM (tools/sweep_simt.cu)
    static STARMM_DEV Acc init() { return __int_as_float(0x7f800000); }
    static STARMM_DEV void term2(Acc& c, float2 a, float2 b) {
        float2 v = __fadd2_rn(a, b);
        asm("min.f32 %0, %0, %1;" : "+f"(c) : "f"(v.x));
        asm("min.f32 %0, %0, %1;" : "+f"(c) : "f"(v.y));
    }
};
struct PolF64Min {
    using Tp = double; using Acc = double;
    static constexpr int G = 1;
    static constexpr int KSTEP = 1, OUTS = 1, BK = 16;
    static constexpr int OCC = 1;   // CTAs per SM (tools/sweep_simt.cu)
    // FP64-pipe bound (2 FP64 instructions per term), spare issue slots: the cross-stage
    // fragment ring gives +8..11% (profiles/r02z_sweep_xs_general.jsonl)
    static constexpr bool XSTAGE = true;
    static STARMM_DEV Acc init() { return __longlong_as_double(0x7ff0000000000000ULL); }
    // the reference's own rule (semiring.py:56-58): v = a + b; if v < out: out = v --
    // a NaN candidate never wins, and -0.0 does not replace +0.0 (fmin would, and costs
    // a DSETP+FSEL+SEL sequence on sm_100a: there is no DMNMX)
    static STARMM_DEV void term(Acc& c, Tp a, Tp b) {
        const double v = a + b;
        c = v < c ? v : c;
    }
};
struct PolI32Vmin {
    using Tp = int; using Acc = int;
    static constexpr int G = 1;
    static constexpr int KSTEP = 1, OUTS = 1, BK = 16;
    static constexpr int OCC = 2;   // CTAs per SM (tools/sweep_simt.cu)
    // generic element epilogue: with the vectorised one compiled in, this 128-register
    // build lost 1.8% in the main loop (34.08 vs 34.58 Tops/s raw at n = 8192)
    static constexpr bool NO_VEC_EPI = true;
    static STARMM_DEV Acc init() { return 0x7fffffff; }
    static STARMM_DEV void term(Acc& c, Tp a, Tp b) { c = __viaddmin_s32(a, b, c); }
};
struct PolI32Sat {
    using Tp = int; using Acc = int;
    static constexpr int G = 1;
    static constexpr int KSTEP = 1, OUTS = 1, BK = 16;
    static constexpr int OCC = 1;   // CTAs per SM (tools/sweep_simt.cu)
    static STARMM_DEV Acc init() { return 0x7fffffff; }
    static STARMM_DEV void term(Acc& c, Tp a, Tp b) {
        long long s = (long long)a + (long long)b;
        s = (a == 0x7fffffff || b == 0x7fffffff) ? 0x7fffffffLL : s;
        s = s > 0x7fffffffLL ? 0x7fffffffLL : (s < -0x80000000LL ? -0x80000000LL : s);
        c = min(c, (int)s);
    }
};
struct PolI64 {
    using Tp = long long; using Acc = unsigned long long;
    static constexpr int G = 1;
    static constexpr int KSTEP = 1, OUTS = 1, BK = 16;
    static constexpr int OCC = 1;   // CTAs per SM (tools/sweep_simt.cu)
    static STARMM_DEV Acc init() { return 0ull; }
    static STARMM_DEV void term(Acc& c, Tp a, Tp b) {
        c += (unsigned long long)a * (unsigned long long)b;
    }
};
struct PolI64Narrow {
    using Tp = int; using Acc = int;
    static constexpr int G = 1;
    static constexpr int KSTEP = 1, OUTS = 1, BK = 16;
    static constexpr int OCC = 2;   // CTAs per SM (tools/sweep_simt.cu)
    static STARMM_DEV Acc init() { return 0; }
    static STARMM_DEV void term(Acc& c, Tp a, Tp b) { c += a * b; }
};

// int64 (+,x) when every |x| <= 127 and K*max|a|*max|b| < 2^31 (range guard):
// four k terms per IDP.4A (dp4a: int8x4 dot + int32 accumulate) -- exact, and
// 4 terms per lane-instruction (255 terms/clk/SM measured, tools/microbench/packed.cu).
struct PolI8Dp4a {
    using Tp = int; using Acc = int;            // Tp packs A[i][4q..4q+3] / B[4q..4q+3][j] as s8x4
    static constexpr int G = 1, KSTEP = 4, OUTS = 1, BK = 64;
    static constexpr int OCC = 2;   // CTAs per SM (tools/sweep_simt.cu)
    static constexpr bool XSTAGE = true;   // half-rate pipe, spare issue slots: cross-stage prefetch
    static STARMM_DEV Acc init() { return 0; }
    static STARMM_DEV void term(Acc& c, Tp a, Tp b) { c = __dp4a(a, b, c); }
};
// (min,+) on integer-valued data with every finite |x| <= 4096 (range guard):
// VIADDMNMX.S16x2 computes min(a+b, c) for two output COLUMNS at once (a is
// duplicated into both halves at packing time); +inf is encoded 16383, so no
// sum can overflow int16 and any result > 8192 involved +inf.  127 terms/clk/SM.
struct PolS16x2Min {
    using Tp = unsigned; using Acc = unsigned;
    static constexpr int G = 1, KSTEP = 1, OUTS = 2, BK = 32;
    static constexpr int OCC = 2;   // CTAs per SM (tools/sweep_simt.cu)
    static STARMM_DEV Acc init() { return 0x7fff7fffu; }
    static STARMM_DEV void term(Acc& c, Tp a, Tp b) { c = __viaddmin_s16x2(a, b, c); }
};
constexpr int S16_INF_ENC = 16383, S16_FINITE_MAX = 4096, S16_INF_THRESHOLD = 8192;

// Accumulator -> output element conversion per (policy, output semiring).
template <class Pol, class Sr> struct Finish;
template <> struct Finish<PolF32Pair, SrTropF32> {
    static STARMM_DEV float out(float v) { return v; }
};
template <> struct Finish<PolF32Pair, SrTropI32> {   // fp32 carrier -> int32, +inf -> INT32_MAX
    static STARMM_DEV int out(float v) { return v == __int_as_float(0x7f800000) ? 0x7fffffff : (int)v; }
};
template <> struct Finish<PolF32Single, SrTropF32> {
    static STARMM_DEV float out(float v) { return v; }
};
template <> struct Finish<PolF32PairMin2, SrTropF32> {
    static STARMM_DEV float out(float v) { return v; }
};
template <> struct Finish<PolF64Min, SrTropF64> {
    static STARMM_DEV double out(double v) { return v; }
};
template <> struct Finish<PolI32Vmin, SrTropI32> {  // encoded sums >= 2^29 involve +inf
    static STARMM_DEV int out(int v) { return v >= (1 << 29) ? 0x7fffffff : v; }
};
template <> struct Finish<PolI32Sat, SrTropI32> {
    static STARMM_DEV int out(int v) { return v; }
};
template <> struct Finish<PolI64, SrInt64> {
    static STARMM_DEV long long out(unsigned long long v) { return (long long)v; }
};
template <> struct Finish<PolI64Narrow, SrInt64> {
    static STARMM_DEV long long out(int v) { return (long long)v; }
};
template <> struct Finish<PolI8Dp4a, SrInt64> {
    static STARMM_DEV long long out(int v) { return (long long)v; }
};
template <> struct Finish<PolS16x2Min, SrTropF32> {
    static STARMM_DEV float out2(unsigned v, int h) {
        int x = (int)(short)(h ? (v >> 16) : (v & 0xffffu));
        return x > S16_INF_THRESHOLD ? __int_as_float(0x7f800000) : (float)x;
    }
};
template <> struct Finish<PolS16x2Min, SrTropF64> {
    static STARMM_DEV double out2(unsigned v, int h) {
        int x = (int)(short)(h ? (v >> 16) : (v & 0xffffu));
        return x > S16_INF_THRESHOLD ? __longlong_as_double(0x7ff0000000000000LL) : (double)x;
    }
};
template <> struct Finish<PolF32Pair, SrTropF64> {   // fp32 carrier of integer-valued float64
    static STARMM_DEV double out(float v) { return (double)v; }
};
template <> struct Finish<PolS16x2Min, SrTropI32> {
    static STARMM_DEV int out2(unsigned v, int h) {
        int x = (int)(short)(h ? (v >> 16) : (v & 0xffffu));
        return x > S16_INF_THRESHOLD ? 0x7fffffff : x;
    }
};

namespace simt {
constexpr int BM = 128, BNW = 128, THREADS = 256;   // BNW: B positions per tile row
template <class Pol> constexpr int bn() { return BNW * Pol::OUTS; }   // output columns per tile
template <class Pol>
constexpr int stage_bytes() {
    return (BM + BNW) * (Pol::BK / Pol::KSTEP) * Pol::G * (int)sizeof(typename Pol::Tp);
}
// Cross-stage fragment prefetch (see mainloop): policies that set XSTAGE, in their
// one-CTA-per-SM build.  It runs a 4-stage ring (two stages resident at every barrier,
// copies issued three ahead); the stage-local loop keeps 3.
template <class P, class = void> struct HasXStage : std::false_type {};
template <class P> struct HasXStage<P, std::void_t<decltype(P::XSTAGE)>> : std::bool_constant<P::XSTAGE> {};
template <class P, class = void> struct NoVecEpi : std::false_type {};
template <class P> struct NoVecEpi<P, std::void_t<decltype(P::NO_VEC_EPI)>> : std::bool_constant<P::NO_VEC_EPI> {};
template <class Pol, int MINB> constexpr bool xstage() { return HasXStage<Pol>::value && MINB == 1; }
template <class Pol, int MINB> constexpr int stages() { return xstage<Pol, MINB>() ? 4 : 3; }
template <class Pol, int MINB>
constexpr int smem_bytes() { return stages<Pol, MINB>() * stage_bytes<Pol>() + 64; }
}  // namespace simt

struct SimtParams {
    const void* Ap;   // packed [Kp/KSTEP][Mp][G]
    const void* Bp;   // packed [Kp/KSTEP][Np/OUTS][G]
    long long Mp, Np; // padded extents (multiples of the tile)
    TaskGrid g;
    WbParams w;
    Pred pr;          // device-side path predicate (common.cuh)
};

template <class Pol, class Sr, int MINB = 1>
__global__ void __launch_bounds__(simt::THREADS, MINB) simt_mm_kernel(SimtParams p) {
    using namespace simt;
    using Tp = typename Pol::Tp;
    using Acc = typename Pol::Acc;
    using T = typename Sr::T;
    if (p.pr.off()) return;
    constexpr int G = Pol::G, KSTEP = Pol::KSTEP, OUTS = Pol::OUTS, BK = Pol::BK;
    constexpr int STAGES = stages<Pol, MINB>();
    constexpr bool XS = xstage<Pol, MINB>();
    constexpr int BN = BNW * OUTS;                      // output columns per tile
    constexpr int VEC = 16 / (G * (int)sizeof(Tp));     // positions per 16-byte load
    constexpr int NQ = 8 / VEC;                         // 16-byte loads per operand per k-group
    constexpr int KG = BK / KSTEP;                      // k-groups per stage
    constexpr int A_STAGE = KG * BM * G;                // elements
    constexpr int B_STAGE = KG * BNW * G;
    constexpr int CHUNK = 16 / (int)sizeof(Tp);         // elements per cp.async
    // Each thread copies the same PASSES 16-byte chunks of every k-stage: its global
    // source pointers advance by one stage per fill (fills are issued in k order), so the
    // steady-state loop carries two 64-bit adds instead of re-deriving the addresses
    // from the stage index (IMAD.WIDE chains, spilled in the 128-register builds).
    constexpr int ROW_CHUNKS = BM * G / CHUNK;          // == BNW * G / CHUNK
    constexpr int RPP = THREADS / ROW_CHUNKS;           // k-group rows per pass
    constexpr int PASSES = KG / RPP;
    static_assert(BM == BNW && KG % RPP == 0 && THREADS % ROW_CHUNKS == 0, "stage copy shape");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Tp* As = reinterpret_cast<Tp*>(smem_raw);
    Tp* Bs = As + STAGES * A_STAGE;
    int* smem_word = reinterpret_cast<int*>(Bs + STAGES * B_STAGE);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ty = (warp >> 1) * 4 + (lane >> 3);      // 0..15
    const int tx = (warp & 1) * 8 + (lane & 7);        // 0..15
    const TaskGrid& g = p.g;
    const long long Nw = p.Np / OUTS;
    const int r0 = tid / ROW_CHUNKS, q0 = tid % ROW_CHUNKS;
    const int s_off = r0 * BM * G + q0 * CHUNK;
    const long long a_pass = (long long)RPP * p.Mp * G, b_pass = (long long)RPP * Nw * G;
    const long long a_adv = (long long)KG * p.Mp * G, b_adv = (long long)KG * Nw * G;
    const Tp* pa = nullptr;      // this thread's next k-stage of A / B in global memory
    const Tp* pb = nullptr;

    auto load_next = [&](int stage) {
        Tp* as = As + stage * A_STAGE + s_off;
        Tp* bs = Bs + stage * B_STAGE + s_off;
#pragma unroll
        for (int i = 0; i < PASSES; ++i) {
            cp_async16(as + i * RPP * BM * G, pa + i * a_pass);
            cp_async16(bs + i * RPP * BNW * G, pb + i * b_pass);
        }
        pa += a_adv;
        pb += b_adv;
    };

    // begin(): point the stage copies at tile (tm, tn), k-stages [kst0, kst0 + nk), and
    // put the first STAGES - 1 of them in flight.  The shared-memory ring must be idle.
    // k-group row kg of A covers Mp*G contiguous elements, of B (Np/OUTS)*G.
    auto begin = [&](int tm, int tn, long long kst0, int nk) {
        const long long kg0 = kst0 * KG;
        pa = reinterpret_cast<const Tp*>(p.Ap) + (kg0 + r0) * p.Mp * G + (long long)tm * BM * G + q0 * CHUNK;
        pb = reinterpret_cast<const Tp*>(p.Bp) + (kg0 + r0) * Nw * G + (long long)tn * BNW * G + q0 * CHUNK;
#pragma unroll
        for (int st = 0; st < STAGES - 1; ++st) {
            if (st < nk) load_next(st);
            cp_async_commit();
        }
    };

    Acc acc[8][8];

    // mainloop(): the nk k-stages begin() addressed, into acc.  Leaves the ring idle.
    //
    // Cross-stage ring (XS; the pipe-bound dp4a policy at one CTA per SM -- the issue-bound
    // policies lose 1-5% to the extra registers and moves, profiles/r02z_sweep_xstage.jsonl,
    // and keep the stage-local loop below): at the top of iteration kt the stages kt and kt+1 are resident and
    // visible to every warp, and every warp has finished reading stage kt-1 -- so the
    // copy of stage kt+STAGES-1 (into stage kt-1's slot) is issued first, and the operand
    // fragments are double-buffered in registers ACROSS the stage boundary: the last
    // k-group of stage kt prefetches the first k-group of stage kt+1, and the first term
    // after the barrier issues without waiting on shared memory.  (With the fragments
    // fetched inside each stage only, every stage began with the barrier, the address
    // set-up and one LDS round trip in series: 6.8% of the in-loop samples of the dp4a
    // kernel, profiles/r02y_dp4a_occ1_regions.txt.)  The barrier sits at the END of the
    // iteration and waits for stage kt+2, copied at least one whole stage earlier.
    auto mainloop = [&](int nk) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = Pol::init();
        if constexpr (XS) {
            const Tp* as0 = As + ty * VEC * G;
            const Tp* bs0 = Bs + tx * VEC * G;
            Tp fa[2][8 * G], fb[2][8 * G];
            auto fetch = [&](int buf, int slot, int kg) {
                const Tp* as = as0 + slot * A_STAGE + kg * BM * G;
                const Tp* bs = bs0 + slot * B_STAGE + kg * BNW * G;
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    *reinterpret_cast<int4*>(&fa[buf][q * VEC * G]) =
                        *reinterpret_cast<const int4*>(as + q * 16 * VEC * G);
                    *reinterpret_cast<int4*>(&fb[buf][q * VEC * G]) =
                        *reinterpret_cast<const int4*>(bs + q * 16 * VEC * G);
                }
            };
            static_assert(KG % 2 == 0, "fragment double buffer parity");
            cp_async_wait<STAGES - 3>();
            __syncthreads();
            if (nk > 0) fetch(0, 0, 0);
            int ld_slot = STAGES - 1, cp_slot = 0;
            for (int kt = 0; kt < nk; ++kt) {
                if (kt + STAGES - 1 < nk) load_next(ld_slot);
                cp_async_commit();
                const int nx_slot = cp_slot == STAGES - 1 ? 0 : cp_slot + 1;
#pragma unroll
                for (int kg = 0; kg < KG; ++kg) {
                    // 8 row operands / 8 column operands, each G elements wide
                    if (kg + 1 < KG) {
                        fetch((kg + 1) & 1, cp_slot, kg + 1);
                    } else if (kt + 1 < nk) {
                        fetch(0, nx_slot, 0);
                    }
                    const Tp* a = fa[kg & 1];
                    const Tp* b = fb[kg & 1];
#pragma unroll
                    for (int i = 0; i < 8; ++i)
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            if constexpr (G == 2) {
                                Pol::term2(acc[i][j], make_float2(a[2 * i], a[2 * i + 1]),
                                           make_float2(b[2 * j], b[2 * j + 1]));
                            } else {
                                Pol::term(acc[i][j], a[i], b[j]);
                            }
                        }
                }
                cp_async_wait<STAGES - 3>();
                __syncthreads();
                ld_slot = ld_slot == STAGES - 1 ? 0 : ld_slot + 1;
                cp_slot = nx_slot;
            }
            cp_async_wait<0>();
        } else {
            const Tp* as0 = As + ty * VEC * G;
            const Tp* bs0 = Bs + tx * VEC * G;
            int ld_slot = STAGES - 1, cp_slot = 0;
            for (int kt = 0; kt < nk; ++kt) {
                cp_async_wait<STAGES - 2>();
                __syncthreads();
                if (kt + STAGES - 1 < nk) load_next(ld_slot);
                cp_async_commit();
                const Tp* as = as0 + cp_slot * A_STAGE;
                const Tp* bs = bs0 + cp_slot * B_STAGE;
#pragma unroll
                for (int kg = 0; kg < KG; ++kg) {
                    // 8 row operands / 8 column operands, each G elements wide
                    Tp a[8 * G], b[8 * G];
#pragma unroll
                    for (int q = 0; q < NQ; ++q) {
                        *reinterpret_cast<int4*>(&a[q * VEC * G]) =
                            *reinterpret_cast<const int4*>(as + kg * BM * G + q * 16 * VEC * G);
                        *reinterpret_cast<int4*>(&b[q * VEC * G]) =
                            *reinterpret_cast<const int4*>(bs + kg * BNW * G + q * 16 * VEC * G);
                    }
#pragma unroll
                    for (int i = 0; i < 8; ++i)
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            if constexpr (G == 2) {
                                Pol::term2(acc[i][j], make_float2(a[2 * i], a[2 * i + 1]),
                                           make_float2(b[2 * j], b[2 * j + 1]));
                            } else {
                                Pol::term(acc[i][j], a[i], b[j]);
                            }
                        }
                }
                ld_slot = ld_slot == STAGES - 1 ? 0 : ld_slot + 1;
                cp_slot = cp_slot == STAGES - 1 ? 0 : cp_slot + 1;
            }
            cp_async_wait<0>();
            __syncthreads();
        }
    };

    // finish(): acc -> C under write-back protocol `mode`.  Exclusive folds / stores of a
    // full tile whose rows are 16-byte aligned take the vectorised epilogue
    // (writeback.cuh epilogue_row_vec: whole 32-byte sectors per warp access); ragged
    // edges, unaligned targets and the k-split protocols take the generic one.
    auto finish = [&](int tm, int tn, int s, int tile, int mode, int pair_seen) {
        // (not for the policies with 64-bit accumulators -- general int64, general float64
        // (min,+): their 255-register one-CTA builds pay 3% in the main loop for the extra
        // epilogue code, and their tiles are ~10x longer, profiles/r02z_sweep_xs_general.jsonl)
        if constexpr (sizeof(Acc) < 8 && !NoVecEpi<Pol>::value) if (mode == WB_STORE || mode == WB_FOLD) {
            T* dst = reinterpret_cast<T*>(p.w.C);
            long long ld = p.w.ldc;
            if (mode == WB_STORE && p.w.mode_base == 1 && s > 0) {   // co3: slice s>0 -> workspace D_s
                dst = reinterpret_cast<T*>(p.w.W) + (long long)(s - 1) * p.w.wstride;
                ld = p.w.ldw;
            }
            const long long m0 = (long long)tm * BM, n0 = (long long)tn * BN;
            const bool vec_ok = m0 + BM <= p.w.M && n0 + BN <= p.w.N &&
                                (reinterpret_cast<unsigned long long>(dst) & 15) == 0 &&
                                (ld * (long long)sizeof(T)) % 16 == 0;
            if (vec_ok) {
                constexpr int W = VEC * OUTS;        // consecutive output columns per fragment
                // rows per batch (all loads of a batch are issued before its stores): the
                // one-CTA-per-SM builds have the registers for two rows in flight
                constexpr int RB = (MINB == 1 && W * (int)sizeof(T) <= 32) ? 2 : 1;
                const bool odd = (lane & 1) != 0;
#pragma unroll
                for (int ib = 0; ib < 8; ib += RB) {
                    T frag[RB * NQ][W];
                    T* gp[RB * NQ];
#pragma unroll
                    for (int ir = 0; ir < RB; ++ir) {
                        const int i = ib + ir;
                        const int r = (i / VEC) * 16 * VEC + ty * VEC + (i % VEC);
#pragma unroll
                        for (int jb = 0; jb < NQ; ++jb) {
#pragma unroll
                            for (int x = 0; x < W; ++x) {
                                if constexpr (OUTS == 1) {
                                    frag[ir * NQ + jb][x] = (T)Finish<Pol, Sr>::out(acc[i][jb * VEC + x]);
                                } else {
                                    frag[ir * NQ + jb][x] = (T)Finish<Pol, Sr>::out2(acc[i][jb * VEC + x / 2], x % 2);
                                }
                            }
                            gp[ir * NQ + jb] = dst + (m0 + r) * ld + n0 + (long long)(jb * 16 * VEC + tx * VEC) * OUTS;
                        }
                    }
                    epilogue_row_vec<Sr, W, RB * NQ>(frag, gp, mode == WB_FOLD, odd);
                }
                return;
            }
        }
        writeback<Sr, BM, BN, THREADS, 16>(p.w, g, tm, tn, s, tile, blockIdx.x, mode, pair_seen,
                              [&](auto f) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    int r = (i / VEC) * 16 * VEC + ty * VEC + (i % VEC);
                    int w = (j / VEC) * 16 * VEC + tx * VEC + (j % VEC);   // B position
                    if constexpr (OUTS == 1) {
                        f(r, w, (T)Finish<Pol, Sr>::out(acc[i][j]));
                    } else {
                        f(r, 2 * w, (T)Finish<Pol, Sr>::out2(acc[i][j], 0));
                        f(r, 2 * w + 1, (T)Finish<Pol, Sr>::out2(acc[i][j], 1));
                    }
                }
        });
    };

    if (g.balanced) {
        // Balanced slices (TAR with uneven k-slices): every worker gets the same number
        // of k-stages of the flattened (tile, k-stage) space; whole tiles fold (or store)
        // exclusively, pieces of a tile shared by workers merge with the atomic-madd.
        TaskGrid g1 = g;
        g1.S = 1; g1.log2S = 0;
        const long long Tn = (long long)g.tiles_m * g.tiles_n * g.kstages;
        long long it = Tn * blockIdx.x / gridDim.x;
        const long long end = Tn * (blockIdx.x + 1) / gridDim.x;
        while (it < end) {
            const long long tl = it / g.kstages;
            const long long ks = it - tl * g.kstages;
            const long long ke = min(g.kstages, ks + (end - it));
            int tm, tn, s0, tile;
            decode_task(g1, (int)tl, tm, tn, s0, tile);
            int mode = WB_RED;
            if (ks == 0 && ke == g.kstages && p.w.remote_parts == 0)
                mode = p.w.init_identity ? WB_STORE : WB_FOLD;
            leaf_enter(p.w);
            begin(tm, tn, ks, (int)(ke - ks));
            mainloop((int)(ke - ks));
            finish(tm, tn, 0, tile, mode, PAIR_EMPTY);
            leaf_exit(p.w);
            it += ke - ks;
        }
        return;
    }
    // Persistent task loop.  The next task's first k-stages are put in flight BEFORE this
    // task's write-back (the ring is idle by then), so the copy latency of a tile start
    // hides behind the epilogue of the previous tile.  SAR pair tasks announce themselves
    // (pair_arrive) when their leaf starts, so they begin after the write-back instead.
    const int nk = (int)(g.kslice / BK);
    int t = blockIdx.x;
    int tm = 0, tn = 0, s = 0, tile = 0, mode = 0;
    bool begun = false;
    if (t < g.num_tasks) {
        decode_task(g, t, tm, tn, s, tile);
        mode = task_mode(p.w, g, s);
    }
    while (t < g.num_tasks) {
        int pair_seen = PAIR_EMPTY;
        if (mode == WB_PAIR) pair_seen = pair_arrive(p.w, g, tile, s, smem_word);
        leaf_enter(p.w);
        if (!begun) begin(tm, tn, (long long)s * nk, nk);
        mainloop(nk);
        const int t2 = t + gridDim.x;
        int tm2 = 0, tn2 = 0, s2 = 0, tile2 = 0, mode2 = 0;
        begun = false;
        if (t2 < g.num_tasks) {
            decode_task(g, t2, tm2, tn2, s2, tile2);
            mode2 = task_mode(p.w, g, s2);
            if (mode2 != WB_PAIR) {
                begin(tm2, tn2, (long long)s2 * nk, nk);
                begun = true;
            }
        }
        finish(tm, tn, s, tile, mode, pair_seen);
        leaf_exit(p.w);
        t = t2; tm = tm2; tn = tn2; s = s2; tile = tile2; mode = mode2;
    }
}

}  // namespace starmm
