// Variant sweep for the fp64 DMMA tile kernel (csrc/dmma_kernel.cuh): times each
// (warps, BK, stages) configuration on an n^3 fp64 product with the CO2 FOLD
// write-back, CUDA events, 1 warm-up + 3 timed launches.  Used to choose DmmaProd.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/sweep tools/sweep_dmma.cu
#include <cstdio>
#include <vector>
#include "../paper_1911_05328_b200/csrc/dmma_kernel.cuh"
using namespace starmm;

template <class K, bool MB = false, int EPI = 0, int GATE = 0>
void run(const char* name, int n, double* A, double* B, double* C, unsigned long long* cnt, int sms,
         int group_m = 8, bool persistent = true) {
    DmmaParams p{};
    p.A = A; p.lda = n; p.B = B; p.ldb = n;
    TaskGrid& g = p.g;
    g.tiles_m = n / K::BM; g.tiles_n = n / K::BN; g.S = 1; g.log2S = 0; g.tar_levels = 0;
    g.group_m = group_m; g.kslice = n; g.num_tasks = g.tiles_m * g.tiles_n;
    WbParams& w = p.w;
    w.mode_base = 0; w.init_identity = 0; w.C = C; w.ldc = n; w.M = n; w.N = n;
    w.counters = cnt;
    auto kern = MB ? dmma_fp64_kernel_mb<K, EPI, GATE> : dmma_fp64_kernel<K>;
    static unsigned* gate = nullptr;
    if (!gate) cudaMalloc(&gate, 4);
    p.gate = gate;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, K::SMEM_BYTES);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, K::THREADS, K::SMEM_BYTES);
    int grid = sms * (occ > 0 ? occ : 1);
    if (grid > g.num_tasks || !persistent) grid = g.num_tasks;
    cudaMemset(gate, 0, 4);
    kern<<<grid, K::THREADS, K::SMEM_BYTES>>>(p);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int i = 0; i < 3; ++i) { cudaMemsetAsync(gate, 0, 4); kern<<<grid, K::THREADS, K::SMEM_BYTES>>>(p); }
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 3;
    cudaError_t e = cudaGetLastError();
    printf("{\"variant\":\"%s\",\"occ\":%d,\"smem\":%d,\"ms\":%.3f,\"tflops\":%.3f,\"err\":\"%s\"}\n", name, occ,
           K::SMEM_BYTES, ms, 2.0 * n * (double)n * n / (ms * 1e-3) / 1e12, cudaGetErrorString(e));
    fflush(stdout);
}

int main(int argc, char** argv) {
    int n = argc > 1 ? atoi(argv[1]) : 16384;
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *A, *B, *C; unsigned long long* cnt;
    cudaMalloc(&A, (size_t)n * n * 8); cudaMalloc(&B, (size_t)n * n * 8); cudaMalloc(&C, (size_t)n * n * 8);
    cudaMalloc(&cnt, 64 * 8);
    cudaMemset(A, 0, (size_t)n * n * 8); cudaMemset(B, 0, (size_t)n * n * 8); cudaMemset(C, 0, (size_t)n * n * 8);
    using P = DmmaCfg<64, 128, 2, 2, 16, 4, 2>;
    run<P>("sync_64x128_s4", n, A, B, C, cnt, sms, 24, true);
    run<P, true>("mbar_64x128_s4", n, A, B, C, cnt, sms, 24, true);
    run<DmmaCfg<64, 128, 2, 2, 16, 3, 2>, true>("mbar_64x128_s3", n, A, B, C, cnt, sms, 24, true);
    run<DmmaCfg<64, 128, 2, 2, 32, 2, 2>, true>("mbar_64x128_bk32_s2", n, A, B, C, cnt, sms, 24, true);
    run<DmmaCfg<64, 128, 2, 2, 16, 4, 2, true>, true>("mbar_64x128_s4_db", n, A, B, C, cnt, sms, 24, true);
    if (argc > 2 && argv[2][0] == 'k') {   // 256x64 8x1: k-stage depth vs ring depth at ~200 KB
        for (int rep = 0; rep < 2; ++rep) {
            run<DmmaCfg<256, 64, 8, 1, 16, 4, 1>, true, 1, 0>("q256_bk16_s4", n, A, B, C, cnt, sms, 4, true);
            run<DmmaCfg<256, 64, 8, 1, 16, 4, 1, true>, true, 1, 0>("q256_bk16_s4_db", n, A, B, C, cnt, sms, 4, true);
        }
        return 0;
    }
    if (argc > 2 && argv[2][0] == 'r') {   // 256x64 refinements: warp tile shape, raster group
        for (int rep = 0; rep < 2; ++rep) {
            run<DmmaCfg<256, 64, 8, 1, 16, 4, 1>, true, 1, 0>("q256x64_8x1_g6", n, A, B, C, cnt, sms, 6, true);
            run<DmmaCfg<256, 64, 8, 1, 16, 4, 1>, true, 1, 0>("q256x64_8x1_g4", n, A, B, C, cnt, sms, 4, true);
            run<DmmaCfg<256, 64, 8, 1, 16, 4, 1>, true, 1, 0>("q256x64_8x1_g12", n, A, B, C, cnt, sms, 12, true);
            run<DmmaCfg<256, 64, 4, 2, 16, 4, 1>, true, 1, 0>("q256x64_4x2_g6", n, A, B, C, cnt, sms, 6, true);
            run<DmmaCfg<256, 64, 8, 1, 16, 4, 1>, true, 1, 2>("q256x64_8x1_g6_gate", n, A, B, C, cnt, sms, 6, true);
        }
        return 0;
    }
    if (argc > 2 && argv[2][0] == 'a') {   // aspect ratios of the 8-warp, 1-CTA/SM design
        for (int rep = 0; rep < 2; ++rep) {
            run<DmmaCfg<128, 128, 4, 2, 16, 4, 1>, true, 1, 0>("q128x128_4x2_s4", n, A, B, C, cnt, sms, 12, true);
            run<DmmaCfg<128, 128, 4, 2, 16, 3, 1>, true, 1, 0>("q128x128_4x2_s3", n, A, B, C, cnt, sms, 12, true);
            run<DmmaCfg<256, 64, 8, 1, 16, 4, 1>, true, 1, 0>("q256x64_8x1_s4", n, A, B, C, cnt, sms, 6, true);
            run<DmmaCfg<64, 256, 2, 4, 16, 4, 1>, true, 1, 0>("q64x256_2x4_s4", n, A, B, C, cnt, sms, 24, true);
        }
        return 0;
    }
    if (argc > 2 && argv[2][0] == 'n') {   // the 128x128 4x2 candidate: gate / raster group
        using Q = DmmaCfg<128, 128, 4, 2, 16, 4, 1>;
        for (int rep = 0; rep < 2; ++rep) {
            run<Q, true, 1, 0>("q128_g12_nogate", n, A, B, C, cnt, sms, 12, true);
            run<Q, true, 1, 2>("q128_g12_gate", n, A, B, C, cnt, sms, 12, true);
            run<Q, true, 1, 2>("q128_g8_gate", n, A, B, C, cnt, sms, 8, true);
            run<Q, true, 1, 2>("q128_g16_gate", n, A, B, C, cnt, sms, 16, true);
        }
        return 0;
    }
    if (argc > 2 && argv[2][0] == 'b') {   // one 128x128 CTA of 8 warps (32x64), mbarrier ring
        for (int rep = 0; rep < 2; ++rep) {
            run<P, true, 1, 0>("prod_64x128_2x2_s4_occ2", n, A, B, C, cnt, sms, 24, true);
            run<DmmaCfg<128, 128, 4, 2, 16, 4, 1>, true, 1, 0>("mbar_128x128_4x2_s4_occ1", n, A, B, C, cnt, sms, 12, true);
            run<DmmaCfg<128, 128, 4, 2, 16, 5, 1>, true, 1, 0>("mbar_128x128_4x2_s5_occ1", n, A, B, C, cnt, sms, 12, true);
            run<DmmaCfg<128, 128, 2, 4, 16, 4, 1>, true, 1, 0>("mbar_128x128_2x4_s4_occ1", n, A, B, C, cnt, sms, 12, true);
        }
        return 0;
    }
    if (argc > 2 && argv[2][0] == 'c') {   // cuBLAS-like: 64x64 tiles, 4 warps of 32x32, 3 CTAs/SM
        for (int rep = 0; rep < 2; ++rep) {
            run<P, true, 1, 0>("prod_64x128_2x2_s4_occ2", n, A, B, C, cnt, sms, 24, true);
            run<DmmaCfg<64, 64, 2, 2, 16, 3, 3>, true, 1, 0>("mbar_64x64_2x2_s3_occ3", n, A, B, C, cnt, sms, 24, true);
            run<DmmaCfg<64, 64, 2, 2, 16, 4, 3>, true, 1, 0>("mbar_64x64_2x2_s4_occ3", n, A, B, C, cnt, sms, 24, true);
            run<DmmaCfg<64, 64, 2, 2, 16, 3, 3>, true, 1, 0>("mbar_64x64_2x2_s3_occ3_g48", n, A, B, C, cnt, sms, 48, true);
        }
        return 0;
    }
    if (argc > 2 && argv[2][0] == 'g') {   // wave gate A/B
        for (int rep = 0; rep < 2; ++rep) {
            run<P, true, 1, 0>("mbar_s4_epi1_nogate", n, A, B, C, cnt, sms, 24, true);
            run<P, true, 1, 1>("mbar_s4_epi1_gate", n, A, B, C, cnt, sms, 24, true);
            run<P, true, 1, 2>("mbar_s4_epi1_gate_q", n, A, B, C, cnt, sms, 24, true);
            run<P, true, 1, 3>("mbar_s4_epi1_gate_h", n, A, B, C, cnt, sms, 24, true);
        }
        return 0;
    }
    if (argc > 2 && argv[2][0] == 'w') {   // 8 warps of 32x32 (4 warps per SMSP at 2 CTAs/SM)
        for (int rep = 0; rep < 2; ++rep) {
            run<P, true, 1>("mbar_64x128_2x2_s4_epi1", n, A, B, C, cnt, sms, 24, true);
            run<DmmaCfg<64, 128, 2, 4, 16, 4, 2>, true, 1>("mbar_64x128_2x4_s4_epi1", n, A, B, C, cnt, sms, 24, true);
            run<DmmaCfg<128, 128, 4, 4, 16, 3, 1>, true, 1>("mbar_128x128_4x4_s3_occ1", n, A, B, C, cnt, sms, 24, true);
        }
        return 0;
    }
    if (argc > 2 && argv[2][0] == 'e') {   // epilogue A/B: generic vs vectorised batched FOLD
        for (int rep = 0; rep < 2; ++rep) {
            run<P, true, 0>("mbar_64x128_s4_epi0", n, A, B, C, cnt, sms, 24, true);
            run<P, true, 1>("mbar_64x128_s4_epi1", n, A, B, C, cnt, sms, 24, true);
        }
        return 0;
    }
    if (argc > 2) {   // round-1 follow-up: k-stage depth vs stage count at the 2-CTA smem budget
        run<DmmaCfg<64, 128, 2, 2, 20, 3, 2>, true>("mbar_64x128_bk20_s3", n, A, B, C, cnt, sms, 24, true);
        run<DmmaCfg<64, 128, 2, 2, 12, 5, 2>, true>("mbar_64x128_bk12_s5", n, A, B, C, cnt, sms, 24, true);
        run<DmmaCfg<64, 128, 2, 2, 8, 8, 2>, true>("mbar_64x128_bk8_s8", n, A, B, C, cnt, sms, 24, true);
        run<P, true>("mbar_64x128_s4_g48", n, A, B, C, cnt, sms, 48, true);
        run<P, true>("mbar_64x128_s4_g12", n, A, B, C, cnt, sms, 12, true);
    }
    return 0;
}
