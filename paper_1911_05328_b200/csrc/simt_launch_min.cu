// simt_launch_min.cu -- CUDA-core tile kernel instantiations: s16x2 / int32 / float64 (min,+).
#include "simt_launch_impl.cuh"

int starmm_simt_launch_min(int path, const starmm::SimtParams& sp, int grid, int sms, cudaStream_t s) {
    switch (path) {
    case PATH_SIMT_F32_S16X2: return launch_simt<PolS16x2Min, SrTropF32>(sp, grid, sms, s);
    case PATH_SIMT_I32_S16X2: return launch_simt<PolS16x2Min, SrTropI32>(sp, grid, sms, s);
    case PATH_SIMT_F64T_S16X2: return launch_simt<PolS16x2Min, SrTropF64>(sp, grid, sms, s);
    case PATH_SIMT_I32_VMIN: return launch_simt<PolI32Vmin, SrTropI32>(sp, grid, sms, s);
    case PATH_SIMT_I32_SAT: return launch_simt<PolI32Sat, SrTropI32>(sp, grid, sms, s);
    case PATH_SIMT_F64_MIN: return launch_simt<PolF64Min, SrTropF64>(sp, grid, sms, s);
    }
    return (int)cudaErrorInvalidValue;
}
