// simt_launch.h -- kernel path ids (shared by the plan code and the launch units) and
// the dispatcher of the CUDA-core tile kernels, whose template instantiations live in
// simt_launch_int.cu / simt_launch_pair.cu / simt_launch_min.cu so that the library
// builds in parallel (make -j).
#pragma once
#include <cuda_runtime.h>

namespace starmm { struct SimtParams; }

enum PathId : int {
    PATH_DMMA_F64 = 1, PATH_SIMT_I64 = 2, PATH_SIMT_I64_NARROW = 3, PATH_SIMT_F32_PAIR = 4,
    PATH_SIMT_I32_CARRIER = 5, PATH_SIMT_I32_VMIN = 6, PATH_SIMT_I32_SAT = 7, PATH_SIMT_F64_MIN = 8,
    PATH_SIMT_I64_DP4A = 9, PATH_SIMT_F32_S16X2 = 10, PATH_SIMT_I32_S16X2 = 11,
    PATH_SIMT_F64T_S16X2 = 12, PATH_SIMT_F64T_CARRIER = 13, PATH_TC_I8 = 14, PATH_OZAKI_F64 = 15,
    PATH_MIN_ORDERED = 16,  // float (min,+) in the reference's leaf order (ordered_kernel.cuh)
    PATH_TC_I8_LIMBS = 17   // opt-in: any int64 as signed radix-256 digits on tcgen05 kind::i8
};

// Launch the persistent CUDA-core tile kernel of `path` (grid CTAs; grid <= sms selects the
// one-CTA-per-SM build where the policy has one).  Returns a cudaError_t value
// (cudaErrorInvalidValue for a path that is not a CUDA-core path).
int starmm_simt_launch(int path, const starmm::SimtParams& sp, int grid, int sms, cudaStream_t s);
int starmm_simt_launch_int(int path, const starmm::SimtParams& sp, int grid, int sms, cudaStream_t s);
int starmm_simt_launch_pair(int path, const starmm::SimtParams& sp, int grid, int sms, cudaStream_t s);
int starmm_simt_launch_min(int path, const starmm::SimtParams& sp, int grid, int sms, cudaStream_t s);
