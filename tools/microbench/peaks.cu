// Instruction-throughput microbenchmarks used to fix the roofline denominators
// (DESIGN.md §Roofline).  Each kernel runs NCHAIN independent dependency chains
// per thread so the pipe, not latency, limits throughput.  Reported as
// "terms/s" (one semiring inner term = one (x) and one (+)) and derived ops/s.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

constexpr int NCH = 8;

__global__ void k_dmma(double* out, int iters){
  double a = threadIdx.x*1e-9, b = 1.0 + threadIdx.x*1e-9;
  double c[NCH][2];
  #pragma unroll
  for(int i=0;i<NCH;i++){c[i][0]=0; c[i][1]=0;}
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int i=0;i<NCH;i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(c[i][0]),"+d"(c[i][1]) : "d"(a),"d"(b));
  }
  double s=0;
  #pragma unroll
  for(int i=0;i<NCH;i++) s+=c[i][0]+c[i][1];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
__global__ void k_dfma(double* out, int iters){
  double a = threadIdx.x*1e-9, b = 1.0 + threadIdx.x*1e-9;
  double c[NCH];
  #pragma unroll
  for(int i=0;i<NCH;i++) c[i]=i;
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int i=0;i<NCH;i++) c[i] = fma(a, b, c[i]);
  }
  double s=0;
  #pragma unroll
  for(int i=0;i<NCH;i++) s+=c[i];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}

// Operands are fed back from the previous iteration (x = c[0]) so ptxas can
// neither hoist nor algebraically collapse the inner term.
__global__ void k_viaddmin(int* out, int iters){
  int b[NCH], c[NCH];
  #pragma unroll
  for(int i=0;i<NCH;i++){ b[i]=threadIdx.x+i; c[i]=1000000+i; }
  for(int it=0; it<iters; ++it){
    int x = c[0];
    #pragma unroll
    for(int i=0;i<NCH;i++) c[i] = __viaddmin_s32(x, b[i], c[i]);
  }
  int s=0;
  #pragma unroll
  for(int i=0;i<NCH;i++) s+=c[i];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
__global__ void k_faddmin(int* out, int iters){
  float b[NCH], c[NCH];
  #pragma unroll
  for(int i=0;i<NCH;i++){ b[i]=threadIdx.x+i; c[i]=1e6f+i; }
  for(int it=0; it<iters; ++it){
    float x = c[0];
    #pragma unroll
    for(int i=0;i<NCH;i++) c[i] = fminf(c[i], x + b[i]);
  }
  float s=0;
  #pragma unroll
  for(int i=0;i<NCH;i++) s+=c[i];
  out[blockIdx.x*blockDim.x+threadIdx.x]=(int)s;
}
// two k-terms per step: FADD2 (packed) + FMNMX3
__global__ void k_fadd2min3(int* out, int iters){
  float2 b[NCH]; float c[NCH];
  #pragma unroll
  for(int i=0;i<NCH;i++){ b[i]=make_float2(threadIdx.x+i, threadIdx.x+2*i); c[i]=1e6f+i; }
  for(int it=0; it<iters; ++it){
    float2 x = make_float2(c[0], c[1]);
    #pragma unroll
    for(int i=0;i<NCH;i++){
      float2 v = __fadd2_rn(x, b[i]);
      c[i] = fminf(fminf(c[i], v.x), v.y);
    }
  }
  float s=0;
  #pragma unroll
  for(int i=0;i<NCH;i++) s+=c[i];
  out[blockIdx.x*blockDim.x+threadIdx.x]=(int)s;
}
__global__ void k_imad32(int* out, int iters){
  int b[NCH], c[NCH];
  #pragma unroll
  for(int i=0;i<NCH;i++){ b[i]=((volatile int*)out)[threadIdx.x+64*i]|1; c[i]=i+1; }
  for(int it=0; it<iters; ++it){
    int x = c[0];
    #pragma unroll
    for(int i=0;i<NCH;i++) c[i] += x * b[i];
  }
  int s=0;
  #pragma unroll
  for(int i=0;i<NCH;i++) s+=c[i];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
__global__ void k_imad64(long long* out, int iters){
  long long b[NCH], c[NCH];
  #pragma unroll
  for(int i=0;i<NCH;i++){ b[i]=((volatile long long*)out)[threadIdx.x+64*i]|1; c[i]=i+1; }
  for(int it=0; it<iters; ++it){
    long long x = c[0];
    #pragma unroll
    for(int i=0;i<NCH;i++) c[i] += x * b[i];
  }
  long long s=0;
  #pragma unroll
  for(int i=0;i<NCH;i++) s+=c[i];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}

template<typename F>
float timeit(F f){
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  f(); cudaDeviceSynchronize();
  cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms,e0,e1); return ms;
}

int main(){
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,0));
  int sms = p.multiProcessorCount;
  printf("{\"device\":\"%s\",\"sms\":%d", p.name, sms);
  void* buf; CK(cudaMalloc(&buf, 64<<20));
  int iters = 20000;
  int threads = 256;
  for (int bps : {4, 8}) {
    int blocks = sms*bps;
    double lanes = (double)blocks*threads;
    float ms;
    // DMMA: each m8n8k4 = 8*8*4 = 256 FMA terms per warp (8 per lane)
    ms = timeit([&]{ k_dmma<<<blocks,threads>>>((double*)buf, iters); });
    printf(",\"dmma_terms_per_s_b%d\":%.4e", bps, lanes/32*256*NCH*(double)iters/(ms*1e-3));
    ms = timeit([&]{ k_dfma<<<blocks,threads>>>((double*)buf, iters); });
    printf(",\"dfma_terms_per_s_b%d\":%.4e", bps, lanes*NCH*(double)iters/(ms*1e-3));
    ms = timeit([&]{ k_viaddmin<<<blocks,threads>>>((int*)buf, iters); });
    printf(",\"viaddmnmx_terms_per_s_b%d\":%.4e", bps, lanes*NCH*(double)iters/(ms*1e-3));
    ms = timeit([&]{ k_faddmin<<<blocks,threads>>>((int*)buf, iters); });
    printf(",\"fadd_fmnmx_terms_per_s_b%d\":%.4e", bps, lanes*NCH*(double)iters/(ms*1e-3));
    ms = timeit([&]{ k_fadd2min3<<<blocks,threads>>>((int*)buf, iters); });
    printf(",\"fadd2_fmnmx3_terms_per_s_b%d\":%.4e", bps, lanes*NCH*2*(double)iters/(ms*1e-3));
    ms = timeit([&]{ k_imad32<<<blocks,threads>>>((int*)buf, iters); });
    printf(",\"imad32_terms_per_s_b%d\":%.4e", bps, lanes*NCH*(double)iters/(ms*1e-3));
    ms = timeit([&]{ k_imad64<<<blocks,threads>>>((long long*)buf, iters); });
    printf(",\"imad64_terms_per_s_b%d\":%.4e", bps, lanes*NCH*(double)iters/(ms*1e-3));
  }
  printf("}\n");
  CK(cudaGetLastError());
  return 0;
}
