// Variant sweep for the CUDA-core semiring tile kernel (csrc/simt_kernel.cuh):
// inner-term policy x co-resident CTAs per SM, CO2 FOLD write-back, packed
// operands of zeros (throughput only), CUDA events, 1 warm-up + 3 timed.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -o tools/sweep_simt_bin tools/sweep_simt.cu
#include <cstdio>
#include "../paper_1911_05328_b200/csrc/simt_kernel.cuh"
using namespace starmm;

template <class Pol, class Sr, int MINB, bool MB = true>
void run(const char* name, int n, void* Ap, void* Bp, void* C, unsigned long long* cnt, int sms, int store = 0) {
    SimtParams p{};
    p.Ap = Ap; p.Bp = Bp; p.Mp = n; p.Np = n;
    TaskGrid& g = p.g;
    g.tiles_m = n / 128; g.tiles_n = n / simt::bn<Pol>(); g.S = 1; g.log2S = 0; g.group_m = 8; g.kslice = n;
    g.num_tasks = g.tiles_m * g.tiles_n;
    WbParams& w = p.w;
    w.mode_base = 0; w.init_identity = store; w.C = C; w.ldc = n; w.M = n; w.N = n; w.counters = cnt;
    auto kern = simt_mm_kernel<Pol, Sr, MINB>;   // (MB: the mbarrier ring variant was removed in round 2,
                                                  //  -1..-6%: profiles/r01n_sweep_simt_occ1_mbarrier.jsonl)
    constexpr int smem = simt::smem_bytes<Pol, MINB>();
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, simt::THREADS, smem);
    int grid = sms * (occ > 0 ? occ : 1);
    kern<<<grid, simt::THREADS, smem>>>(p);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int i = 0; i < 3; ++i) kern<<<grid, simt::THREADS, smem>>>(p);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 3;
    printf("{\"variant\":\"%s\",\"occ\":%d,\"ms\":%.3f,\"tops\":%.3f,\"err\":\"%s\"}\n", name, occ, ms,
           2.0 * n * (double)n * n / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    fflush(stdout);
}

// dp4a policy variants (k-stage depth)
struct PolI8Dp4aBK128 : PolI8Dp4a { static constexpr int BK = 128; };
struct PolI8Dp4aBK32 : PolI8Dp4a { static constexpr int BK = 32; };
template <> struct starmm::Finish<PolI8Dp4aBK128, SrInt64> : starmm::Finish<PolI8Dp4a, SrInt64> {};
template <> struct starmm::Finish<PolI8Dp4aBK32, SrInt64> : starmm::Finish<PolI8Dp4a, SrInt64> {};

struct PolI32VminNV : PolI32Vmin { static constexpr bool NO_VEC_EPI = true; };
template <> struct starmm::Finish<PolI32VminNV, SrTropI32> : starmm::Finish<PolI32Vmin, SrTropI32> {};
// cross-stage fragment ring on the one-CTA-per-SM general policies
struct PolF64MinXS : PolF64Min { static constexpr bool XSTAGE = true; };
struct PolI64XS : PolI64 { static constexpr bool XSTAGE = true; };
struct PolI32SatXS : PolI32Sat { static constexpr bool XSTAGE = true; };
template <> struct starmm::Finish<PolF64MinXS, SrTropF64> : starmm::Finish<PolF64Min, SrTropF64> {};
template <> struct starmm::Finish<PolI64XS, SrInt64> : starmm::Finish<PolI64, SrInt64> {};
template <> struct starmm::Finish<PolI32SatXS, SrTropI32> : starmm::Finish<PolI32Sat, SrTropI32> {};

int main(int argc, char** argv) {
    int n = argc > 1 ? atoi(argv[1]) : 8192;
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    void *A, *B, *C; unsigned long long* cnt;
    size_t bytes = (size_t)n * n * 8;
    cudaMalloc(&A, bytes); cudaMalloc(&B, bytes); cudaMalloc(&C, bytes); cudaMalloc(&cnt, 512);
    cudaMemset(A, 0, bytes); cudaMemset(B, 0, bytes); cudaMemset(C, 0, bytes);
    // (round 2: k-group unroll 2/4/8 and BK 128/256 at a 16-group unroll were swept on the
    //  stage-local fragment loop -- profiles/r02y_sweep_unroll_*.jsonl -- full unroll won)
    if (argc > 2 && argv[2][0] == 'a') {   // every production policy build (A/B against another revision)
        for (int rep = 0; rep < 2; ++rep) {
            run<PolI64Narrow, SrInt64, 2, false>("narrow_occ2", n, A, B, C, cnt, sms);
            run<PolI32Vmin, SrTropI32, 2, false>("i32vmin_occ2", n, A, B, C, cnt, sms);
            run<PolF32Pair, SrTropF32, 1, false>("f32pair_f32_occ1", n, A, B, C, cnt, sms);
            run<PolF32Pair, SrTropF32, 2, false>("f32pair_f32_occ2", n, A, B, C, cnt, sms);
            run<PolF32Pair, SrTropI32, 1, false>("f32pair_i32_occ1", n, A, B, C, cnt, sms);
            run<PolF32Pair, SrTropI32, 2, false>("f32pair_i32_occ2", n, A, B, C, cnt, sms);
            run<PolI32Sat, SrTropI32, 1, false>("i32sat_occ1", n, A, B, C, cnt, sms);
            run<PolS16x2Min, SrTropF32, 1, false>("s16x2_occ1", n, A, B, C, cnt, sms);
            run<PolS16x2Min, SrTropF32, 2, false>("s16x2_occ2", n, A, B, C, cnt, sms);
            run<PolI8Dp4a, SrInt64, 1, false>("dp4a_occ1", n, A, B, C, cnt, sms);
            run<PolI8Dp4a, SrInt64, 2, false>("dp4a_occ2", n, A, B, C, cnt, sms);
            run<PolF64Min, SrTropF64, 1, false>("f64min_occ1", n, A, B, C, cnt, sms);
            run<PolI64, SrInt64, 1, false>("i64_occ1", n, A, B, C, cnt, sms);
        }
        return 0;
    }
    if (argc > 2 && argv[2][0] == 'v') {
        for (int rep = 0; rep < 2; ++rep) {
            run<PolI32Vmin, SrTropI32, 2, false>("i32vmin_occ2", n, A, B, C, cnt, sms);
            run<PolI32VminNV, SrTropI32, 2, false>("i32vmin_novec_occ2", n, A, B, C, cnt, sms);
        }
        return 0;
    }
    if (argc > 2 && argv[2][0] == 'x') {   // cross-stage ring on the general one-CTA policies
        for (int rep = 0; rep < 2; ++rep) {
            run<PolF64Min, SrTropF64, 1, false>("f64min_occ1", n, A, B, C, cnt, sms);
            run<PolF64MinXS, SrTropF64, 1, false>("f64min_xs_occ1", n, A, B, C, cnt, sms);
            run<PolI64, SrInt64, 1, false>("i64_occ1", n, A, B, C, cnt, sms);
            run<PolI64XS, SrInt64, 1, false>("i64_xs_occ1", n, A, B, C, cnt, sms);
            run<PolI32Sat, SrTropI32, 1, false>("i32sat_occ1", n, A, B, C, cnt, sms);
            run<PolI32SatXS, SrTropI32, 1, false>("i32sat_xs_occ1", n, A, B, C, cnt, sms);
        }
        return 0;
    }
    if (argc > 2 && argv[2][0] == 'd') {   // dp4a k-stage depth
        for (int rep = 0; rep < 2; ++rep) {
            run<PolI8Dp4a, SrInt64, 2, false>("i64_dp4a_bk64_occ2", n, A, B, C, cnt, sms);
            run<PolI8Dp4aBK128, SrInt64, 2, false>("i64_dp4a_bk128_occ2", n, A, B, C, cnt, sms);
            run<PolI8Dp4aBK32, SrInt64, 2, false>("i64_dp4a_bk32_occ2", n, A, B, C, cnt, sms);
        }
        return 0;
    }
    run<PolI8Dp4a, SrInt64, 1, false>("i64_dp4a_occ1", n, A, B, C, cnt, sms);
    run<PolI8Dp4a, SrInt64, 1, false>("i64_dp4a_occ1_store", n, A, B, C, cnt, sms, 1);
    run<PolI8Dp4a, SrInt64, 2, false>("i64_dp4a_occ2", n, A, B, C, cnt, sms);
    run<PolS16x2Min, SrTropF32, 1, false>("minplus_s16x2_occ1", n, A, B, C, cnt, sms);
    run<PolS16x2Min, SrTropF32, 2, false>("minplus_s16x2_occ2", n, A, B, C, cnt, sms);
    run<PolF32Pair, SrTropI32, 1, false>("i32_carrier_occ1", n, A, B, C, cnt, sms);
    run<PolF32Pair, SrTropI32, 2, false>("i32_carrier_occ2", n, A, B, C, cnt, sms);
    return 0;
}
