// FP64 mma.sync shapes on sm_100a: m8n8k4 (DMMA.884, the production kernel's) vs the
// sm_90+ m16n8k4 / m16n8k8 / m16n8k16 shapes.  NCH independent accumulators per warp,
// reported as TF/s (2 flops per FMA).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench/dmma_shapes tools/microbench/dmma_shapes.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NCH = 8;

__global__ void k884(double* out, int iters) {
    double a = threadIdx.x * 1e-9, b = 1.0 + threadIdx.x * 1e-9;
    double c[NCH][2];
#pragma unroll
    for (int i = 0; i < NCH; i++) c[i][0] = c[i][1] = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NCH; i++)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < NCH; i++) s += c[i][0] + c[i][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k1684(double* out, int iters) {
    double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-3, b = 1.0 + threadIdx.x * 1e-9;
    double c[NCH][4];
#pragma unroll
    for (int i = 0; i < NCH; i++) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NCH; i++)
            asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                         : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < NCH; i++) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k1688(double* out, int iters) {
    double a[4], b[2];
#pragma unroll
    for (int i = 0; i < 4; i++) a[i] = threadIdx.x * 1e-9 + i;
    b[0] = 1.0; b[1] = 2.0;
    double c[NCH][4];
#pragma unroll
    for (int i = 0; i < NCH; i++) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NCH; i++)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                         : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < NCH; i++) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k16816(double* out, int iters) {
    double a[8], b[4];
#pragma unroll
    for (int i = 0; i < 8; i++) a[i] = threadIdx.x * 1e-9 + i;
#pragma unroll
    for (int i = 0; i < 4; i++) b[i] = 1.0 + i;
    double c[NCH][4];
#pragma unroll
    for (int i = 0; i < NCH; i++) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NCH; i++)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                         : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                         : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                           "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < NCH; i++) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class F>
void run(const char* name, F kern, double flops_per_mma, double* out, int sms, int warps_per_sm) {
    const int threads = 128, blocks = sms * warps_per_sm / 4, iters = 2000;
    kern<<<blocks, threads>>>(out, 10);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double fl = (double)blocks * (threads / 32) * iters * NCH * flops_per_mma;
    printf("{\"shape\":\"%s\",\"warps_per_sm\":%d,\"tflops\":%.2f,\"err\":\"%s\"}\n", name, warps_per_sm,
           fl / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out; cudaMalloc(&out, (size_t)sms * 64 * 128 * 8);
    for (int w : {4, 8, 16}) {
        run("m8n8k4", k884, 2.0 * 8 * 8 * 4, out, sms, w);
        run("m16n8k4", k1684, 2.0 * 16 * 8 * 4, out, sms, w);
        run("m16n8k8", k1688, 2.0 * 16 * 8 * 8, out, sms, w);
        run("m16n8k16", k16816, 2.0 * 16 * 8 * 16, out, sms, w);
    }
    return 0;
}
