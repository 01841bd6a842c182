// Dev harness for the CTA-pair tcgen05 int8 GEMM core (csrc/tc_gemm.cuh).
//   tc_gemm_dev M N K [reps]  -> checks C = A * B^T (int32) against a CUDA-core
//   reference on sampled rows, then times the core alone (CUDA events).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cstring>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../paper_1911_05328_b200/csrc/tc_gemm.cuh"
#include "../paper_1911_05328_b200/csrc/ozaki.cuh"

using namespace starmm;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1); } } while (0)

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static void make_map(CUtensorMap* m, void* base, long long rows, long long kp, int box_rows) {
    static EncodeFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &q));
    }
    cuuint64_t dims[2] = {(cuuint64_t)kp, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)kp};
    cuuint32_t box[2] = {(cuuint32_t)tcg::BK, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, base, dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("tmap encode failed %d\n", (int)r); exit(1); }
}

__global__ void ref_rows(const signed char* A, const signed char* B, int* R, int K, int N, const int* rows, int nr) {
    int i = blockIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nr || j >= N) return;
    const signed char* a = A + (long long)rows[i] * K;
    const signed char* b = B + (long long)j * K;
    int s = 0;
    for (int k = 0; k < K; ++k) s += (int)a[k] * (int)b[k];
    R[(long long)i * N + j] = s;
}

__global__ void fill_rand(signed char* p, long long n, unsigned seed) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        unsigned x = (unsigned)(i * 2654435761u) ^ seed;
        x ^= x >> 13; x *= 0x5bd1e995; x ^= x >> 15;
        p[i] = (signed char)(x & 0xff);
    }
}

int main(int argc, char** argv) {
    int M = argc > 1 ? atoi(argv[1]) : 4096, N = argc > 2 ? atoi(argv[2]) : 4096, K = argc > 3 ? atoi(argv[3]) : 4096;
    int reps = argc > 4 ? atoi(argv[4]) : 10;
    int passes = argc > 5 ? atoi(argv[5]) : 1;
    int group_m = argc > 6 ? atoi(argv[6]) : 8;
    const char* epi_kind = argc > 7 ? argv[7] : "i32";   // i32 | oz (Ozaki CRT epilogue, timing only)
    int gate_depth = argc > 8 ? atoi(argv[8]) : 0;     // 0: no drift gating
    // M, N multiples of 256, K multiple of 128 (dev harness)
    signed char *A, *B; int* C;
    CK(cudaMalloc(&A, (size_t)M * K * passes)); CK(cudaMalloc(&B, (size_t)N * K * passes));
    CK(cudaMalloc(&C, (size_t)M * N * 4));
    fill_rand<<<1024, 256>>>(A, (long long)M * K * passes, 1234u);
    fill_rand<<<1024, 256>>>(B, (long long)N * K * passes, 999u);
    CUtensorMap ta, tb;
    make_map(&ta, A, (long long)M * passes, K, tcg::BM);
    make_map(&tb, B, (long long)N * passes, K, tcg::BNH);
    TcgShape sh;
    sh.tiles_m = M / 256; sh.tiles_n = N / 256; sh.num_tiles = sh.tiles_m * sh.tiles_n; sh.group_m = group_m;
    sh.nk = K / tcg::BK; sh.passes = passes; sh.a_pass_rows = M; sh.b_pass_rows = N;
    sh.gate = nullptr; sh.gate_depth = gate_depth; sh.rounds = 1;
    EpiStoreI32 epi;
    epi.C = C; epi.ldc = N; epi.M = M; epi.N = N;
    auto kern = tcg_kernel<EpiStoreI32>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, tcg::SMEM_BYTES));
    int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    int clusters = 0;
    {
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(sms); lc.blockDim = dim3(tcg::THREADS); lc.dynamicSmemBytes = tcg::SMEM_BYTES;
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        lc.attrs = at; lc.numAttrs = 1;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, tcg::SMEM_BYTES));
        CK(cudaOccupancyMaxActiveClusters(&clusters, kern, &lc));
    }
    int grid = 2 * std::min(clusters, sh.num_tiles);
    sh.rounds = (sh.num_tiles + grid / 2 - 1) / (grid / 2);
    unsigned* gate = nullptr;
    if (gate_depth > 0) {
        CK(cudaMalloc(&gate, (size_t)sh.rounds * passes * 4 * 64));
        sh.gate = gate;
    }
    auto reset_gate = [&]() { if (gate) cudaMemsetAsync(gate, 0, (size_t)sh.rounds * passes * 4); };
    printf("{\"max_active_clusters\": %d}\n", clusters);
    reset_gate();
    kern<<<grid, tcg::THREADS, tcg::SMEM_BYTES>>>(ta, tb, sh, epi);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    // check sampled rows (last pass only is in C: passes overwrite)
    const int nr = 64;
    std::vector<int> rows(nr);
    for (int i = 0; i < nr; ++i) rows[i] = (int)(((long long)i * 7919 + 13) % M);
    int *drows, *R;
    CK(cudaMalloc(&drows, nr * 4)); CK(cudaMalloc(&R, (size_t)nr * N * 4));
    CK(cudaMemcpy(drows, rows.data(), nr * 4, cudaMemcpyHostToDevice));
    const signed char* Al = A + (size_t)(passes - 1) * M * K;
    const signed char* Bl = B + (size_t)(passes - 1) * N * K;
    ref_rows<<<dim3((N + 127) / 128, nr), 128>>>(Al, Bl, R, K, N, drows, nr);
    CK(cudaDeviceSynchronize());
    std::vector<int> hr((size_t)nr * N), hc((size_t)N);
    CK(cudaMemcpy(hr.data(), R, hr.size() * 4, cudaMemcpyDeviceToHost));
    long long bad = 0;
    for (int i = 0; i < nr; ++i) {
        CK(cudaMemcpy(hc.data(), C + (size_t)rows[i] * N, N * 4, cudaMemcpyDeviceToHost));
        for (int j = 0; j < N; ++j) if (hc[j] != hr[(size_t)i * N + j]) { if (bad < 5) printf("mismatch r%d c%d %d vs %d\n", rows[i], j, hc[j], hr[(size_t)i*N+j]); ++bad; }
    }
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    if (epi_kind[0] == 'o') {   // Ozaki residue epilogue (timing only)
        unsigned char* Rb;
        CK(cudaMalloc(&Rb, (size_t)passes * M * N));
        EpiOzakiResidues eo;
        eo.R = Rb; eo.Mp = M; eo.Np = N;
        auto ko = tcg_kernel<EpiOzakiResidues>;
        CK(cudaFuncSetAttribute(ko, cudaFuncAttributeMaxDynamicSharedMemorySize, tcg::SMEM_BYTES));
        reset_gate();
        ko<<<grid, tcg::THREADS, tcg::SMEM_BYTES>>>(ta, tb, sh, eo);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        for (int r = 0; r < reps; ++r) { reset_gate(); ko<<<grid, tcg::THREADS, tcg::SMEM_BYTES>>>(ta, tb, sh, eo); }
        cudaEventRecord(e1);
    } else {
        cudaEventRecord(e0);
        for (int r = 0; r < reps; ++r) { reset_gate(); kern<<<grid, tcg::THREADS, tcg::SMEM_BYTES>>>(ta, tb, sh, epi); }
        cudaEventRecord(e1);
    }
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
    double ops = 2.0 * M * (double)N * K * passes;
    printf("{\"M\":%d,\"N\":%d,\"K\":%d,\"passes\":%d,\"grid\":%d,\"mismatches\":%lld,\"ms\":%.4f,\"tops\":%.1f}\n",
           M, N, K, passes, grid, bad, ms, ops / ms / 1e9);
    return bad ? 2 : 0;
}
