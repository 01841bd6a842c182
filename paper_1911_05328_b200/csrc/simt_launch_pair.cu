// simt_launch_pair.cu -- CUDA-core tile kernel instantiations: fp32-pair / fp32-carrier (min,+).
#include "simt_launch_impl.cuh"

int starmm_simt_launch_pair(int path, const starmm::SimtParams& sp, int grid, int sms, cudaStream_t s) {
    switch (path) {
    case PATH_SIMT_F32_PAIR: return launch_simt<PolF32Pair, SrTropF32>(sp, grid, sms, s);
    case PATH_SIMT_I32_CARRIER: return launch_simt<PolF32Pair, SrTropI32>(sp, grid, sms, s);
    case PATH_SIMT_F64T_CARRIER: return launch_simt<PolF32Pair, SrTropF64>(sp, grid, sms, s);
    }
    return (int)cudaErrorInvalidValue;
}
