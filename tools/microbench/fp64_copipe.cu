// Do DMMA (FP64 tensor) and DFMA (FP64 CUDA core) share hardware on B200?
// Warps with (warp % 2 == 0) run DMMA chains, odd warps run DFMA chains; compare the
// combined flop rate with DMMA-only and DFMA-only runs of the same launch shape.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int NCH = 8;
__global__ void mixed(double* out, int iters, int mode) {  // mode 0 dmma, 1 dfma, 2 split
    int w = threadIdx.x >> 5;
    bool do_dmma = mode == 0 || (mode == 2 && (w & 1) == 0);
    double a = threadIdx.x * 1e-9, b = 1.0 + threadIdx.x * 1e-9;
    double c[NCH][2];
    for (int i = 0; i < NCH; i++) c[i][0] = c[i][1] = i;
    if (do_dmma) {
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int i = 0; i < NCH; i++)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    } else {
        for (int it = 0; it < iters * 8; ++it)           // 8 DFMA per lane ~ 1 DMMA.8x8x4 per lane
#pragma unroll
            for (int i = 0; i < NCH; i++) c[i][0] = fma(a, b, c[i][0]);
    }
    double s = 0;
    for (int i = 0; i < NCH; i++) s += c[i][0] + c[i][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* buf; cudaMalloc(&buf, 64 << 20);
    int iters = 4000, threads = 256, blocks = sms * 4;
    for (int mode = 0; mode < 3; ++mode) {
        mixed<<<blocks, threads>>>(buf, iters, mode);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        mixed<<<blocks, threads>>>(buf, iters, mode);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double warps = (double)blocks * threads / 32;
        double dmma_w = mode == 0 ? warps : (mode == 2 ? warps / 2 : 0);
        double dfma_w = warps - dmma_w;
        double flops = dmma_w * iters * NCH * 512.0 + dfma_w * 32 * iters * 8.0 * NCH * 2.0;
        printf("{\"mode\":\"%s\",\"ms\":%.3f,\"tflops\":%.2f}\n", mode == 0 ? "dmma" : mode == 1 ? "dfma" : "split",
               ms, flops / (ms * 1e-3) / 1e12);
    }
    return 0;
}
