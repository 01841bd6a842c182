// Throughput of packed (two terms per lane) candidates vs the 1-term ops, to see which
// inner loops can pass the 64 terms/clk/SM dispatch ceiling of the 16-lane pipes.
// terms/s counts semiring inner terms (one (x) + one (+)).
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
constexpr int NCH = 8;

__global__ void k_vmin16x2(unsigned* out, int iters) {           // min(a+b, c) on 2 x s16
    unsigned b[NCH], c[NCH];
    for (int i = 0; i < NCH; i++) { b[i] = ((volatile unsigned*)out)[threadIdx.x + 32 * i] | 0x00010001u; c[i] = 0x7fff7fffu - i; }
    for (int it = 0; it < iters; ++it) {
        unsigned x = c[0];
#pragma unroll
        for (int i = 0; i < NCH; i++) c[i] = __viaddmin_s16x2(x, b[i], c[i]);
    }
    unsigned s = 0;
    for (int i = 0; i < NCH; i++) s += c[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma2(float* out, int iters) {                 // 2 FMA per lane
    float2 b[NCH], c[NCH];
    for (int i = 0; i < NCH; i++) { b[i] = make_float2(out[threadIdx.x + i], out[threadIdx.x + 2 * i]); c[i] = make_float2(i, i + 1); }
    for (int it = 0; it < iters; ++it) {
        float2 x = c[0];
#pragma unroll
        for (int i = 0; i < NCH; i++) c[i] = __ffma2_rn(x, b[i], c[i]);
    }
    float s = 0;
    for (int i = 0; i < NCH; i++) s += c[i].x + c[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma(float* out, int iters) {
    float b[NCH], c[NCH];
    for (int i = 0; i < NCH; i++) { b[i] = out[threadIdx.x + i]; c[i] = i; }
    for (int it = 0; it < iters; ++it) {
        float x = c[0];
#pragma unroll
        for (int i = 0; i < NCH; i++) c[i] = fmaf(x, b[i], c[i]);
    }
    float s = 0;
    for (int i = 0; i < NCH; i++) s += c[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_hmin2(unsigned* out, int iters) {              // HADD2 + HMNMX2: 2 terms/lane
    __half2 b[NCH], c[NCH];
    for (int i = 0; i < NCH; i++) { b[i] = __halves2half2(__int2half_rn(threadIdx.x & 7), __int2half_rn(i)); c[i] = __halves2half2(__int2half_rn(1000), __int2half_rn(1000 + i)); }
    for (int it = 0; it < iters; ++it) {
        __half2 x = c[0];
#pragma unroll
        for (int i = 0; i < NCH; i++) c[i] = __hmin2(c[i], __hadd2(x, b[i]));
    }
    float s = 0;
    for (int i = 0; i < NCH; i++) s += __low2float(c[i]) + __high2float(c[i]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = (unsigned)s;
}
__global__ void k_imad16(unsigned* out, int iters) {             // 16x2 dot-style: IDP? use __dp2a? (int8/16 dot)
    unsigned b[NCH]; int c[NCH];
    for (int i = 0; i < NCH; i++) { b[i] = ((volatile unsigned*)out)[threadIdx.x + 32 * i] | 0x00010001u; c[i] = i; }
    for (int it = 0; it < iters; ++it) {
        unsigned x = (unsigned)c[0];
#pragma unroll
        for (int i = 0; i < NCH; i++) c[i] = __dp2a_lo((int)x, (int)b[i], c[i]);  // 2 x (s16*s8) + acc
    }
    int s = 0;
    for (int i = 0; i < NCH; i++) s += c[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dp4a(unsigned* out, int iters) {               // 4 x (s8*s8) + acc
    int b[NCH], c[NCH];
    for (int i = 0; i < NCH; i++) { b[i] = ((volatile int*)out)[threadIdx.x + 32 * i] | 0x01010101; c[i] = i; }
    for (int it = 0; it < iters; ++it) {
        int x = c[0];
#pragma unroll
        for (int i = 0; i < NCH; i++) c[i] = __dp4a(x, b[i], c[i]);
    }
    int s = 0;
    for (int i = 0; i < NCH; i++) s += c[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class F> float timeit(F f) {
    f(); cudaDeviceSynchronize();
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); return ms;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    void* buf; cudaMalloc(&buf, 64 << 20); cudaMemset(buf, 0, 64 << 20);
    int iters = 20000, threads = 256, blocks = sms * 8;
    double lanes = (double)blocks * threads;
    auto rep = [&](const char* name, float ms, double terms_per_lane_op) {
        double t = lanes * NCH * (double)iters * terms_per_lane_op / (ms * 1e-3);
        printf("{\"op\":\"%s\",\"terms_per_s\":%.4e,\"terms_per_clk_sm_at_1965\":%.1f}\n", name, t, t / sms / 1.965e9);
    };
    rep("viaddmnmx_s16x2 (2 terms)", timeit([&] { k_vmin16x2<<<blocks, threads>>>((unsigned*)buf, iters); }), 2);
    rep("ffma2 (2 terms)", timeit([&] { k_ffma2<<<blocks, threads>>>((float*)buf, iters); }), 2);
    rep("ffma (1 term)", timeit([&] { k_ffma<<<blocks, threads>>>((float*)buf, iters); }), 1);
    rep("hadd2+hmnmx2 (2 terms / 2 ops)", timeit([&] { k_hmin2<<<blocks, threads>>>((unsigned*)buf, iters); }), 2);
    rep("dp2a (2 terms)", timeit([&] { k_imad16<<<blocks, threads>>>((unsigned*)buf, iters); }), 2);
    rep("dp4a (4 terms)", timeit([&] { k_dp4a<<<blocks, threads>>>((unsigned*)buf, iters); }), 4);
    return 0;
}
