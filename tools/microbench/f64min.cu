// Inner-term candidates for the reference's float64 (min,+) (semiring.py:48-60,
// `v = a + b; if v < out: out = v`) on sm_100a, which has no DMNMX:
//   ref    DADD + DSETP + 2 FSEL          (PolF64Min today)
//   dadd   DADD only                      (the FP64-pipe ceiling of any exact form)
//   u64    DADD + 64-bit unsigned min on the bit pattern: exact when every operand
//          is +0.0 / positive / +inf (non-negative data, a range guard)
//   i64    DADD + signed 64-bit min (same order for non-negative doubles)
// NCH independent chains per thread; terms/s reported.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench/f64min tools/microbench/f64min.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NCH = 16;

template <int V>
__global__ void k(double* out, const double* in, int iters) {
    double a[4], b[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) { a[i] = in[i] + threadIdx.x; b[i] = in[4 + i] + blockIdx.x; }
    double c[NCH];
#pragma unroll
    for (int i = 0; i < NCH; ++i) c[i] = 1e300;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NCH; ++i) {
            double v = a[i & 3] + b[(i >> 2) & 3];
            if (V == 0) c[i] = v < c[i] ? v : c[i];
            if (V == 1) c[i] += v;
            if (V == 2) {
                unsigned long long x = __double_as_longlong(v), y = __double_as_longlong(c[i]);
                c[i] = __longlong_as_double((long long)(x < y ? x : y));
            }
            if (V == 3) {
                long long x = __double_as_longlong(v), y = __double_as_longlong(c[i]);
                c[i] = __longlong_as_double(min(x, y));
            }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) { a[i] += 1.0; b[i] -= 0.5; }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < NCH; ++i) s += c[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int V>
void run(const char* name, double* out, const double* in, int sms) {
    const int iters = 4096, blocks = sms * 4, threads = 256;
    k<V><<<blocks, threads>>>(out, in, 16);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<V><<<blocks, threads>>>(out, in, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double terms = (double)blocks * threads * iters * NCH;
    printf("{\"variant\":\"%s\",\"terms_per_s\":%.4e,\"semiring_tops\":%.2f}\n", name, terms / (ms * 1e-3),
           2 * terms / (ms * 1e-3) / 1e12);
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out, *in;
    cudaMalloc(&out, (size_t)sms * 4 * 256 * 8); cudaMalloc(&in, 64);
    double h[8] = {1, 2, 3, 4, 5, 6, 7, 8};
    cudaMemcpy(in, h, 64, cudaMemcpyHostToDevice);
    run<0>("ref_dadd_dsetp_fsel", out, in, sms);
    run<1>("dadd_only", out, in, sms);
    run<2>("dadd_u64min", out, in, sms);
    run<3>("dadd_i64min", out, in, sms);
    return 0;
}
