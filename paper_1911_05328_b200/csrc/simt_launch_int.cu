// simt_launch_int.cu -- CUDA-core tile kernel instantiations: int64 (+,x).
#include "simt_launch_impl.cuh"

int starmm_simt_launch_int(int path, const starmm::SimtParams& sp, int grid, int sms, cudaStream_t s) {
    switch (path) {
    case PATH_SIMT_I64: return launch_simt<PolI64, SrInt64>(sp, grid, sms, s);
    case PATH_SIMT_I64_NARROW: return launch_simt<PolI64Narrow, SrInt64>(sp, grid, sms, s);
    case PATH_SIMT_I64_DP4A: return launch_simt<PolI8Dp4a, SrInt64>(sp, grid, sms, s);
    }
    return (int)cudaErrorInvalidValue;
}
