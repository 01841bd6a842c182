// simt_launch_impl.cuh -- the launch template shared by the simt_launch_*.cu units.
#pragma once
#include <type_traits>
#include "common.cuh"
#include "writeback.cuh"
#include "simt_kernel.cuh"
#include "simt_launch.h"

namespace {
#define SL_CK(x) do { cudaError_t _e = (x); if (_e != cudaSuccess) return (int)_e; } while (0)
using namespace starmm;

// Policies that also ship a one-CTA-per-SM build (register budget 255 instead of 128):
// the planner's occupancy-1 choice then runs at 0.97 of a full SM instead of 0.89
// (tools/sweep_simt.cu; config 2 = 1024 tiles, 6.9 waves of 148 CTAs).
template <class Pol> constexpr bool has_occ1_build() {
    return std::is_same<Pol, PolI8Dp4a>::value || std::is_same<Pol, PolF32Pair>::value ||
           std::is_same<Pol, PolS16x2Min>::value;
}

// The >48 KB dynamic-smem opt-in is an attribute of the function in the CURRENT
// device's context: remembered per device, not per process.
constexpr int SL_MAX_DEV = 64;
inline int sl_device() {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess) { cudaGetLastError(); return 0; }
    return d < SL_MAX_DEV ? d : SL_MAX_DEV - 1;
}

template <class Pol, class Sr>
int launch_simt(const SimtParams& p, int grid, int sms, cudaStream_t s) {
    const int dev = sl_device();
    if constexpr (has_occ1_build<Pol>() && Pol::OCC > 1) {
        if (grid <= sms) {
            auto k1 = simt_mm_kernel<Pol, Sr, 1>;
            constexpr int smem = simt::smem_bytes<Pol, 1>();
            static bool attr1[SL_MAX_DEV] = {};
            if (!attr1[dev]) {
                SL_CK(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
                attr1[dev] = true;
            }
            k1<<<grid, simt::THREADS, smem, s>>>(p);
            SL_CK(cudaGetLastError());
            return (int)cudaSuccess;
        }
    }
    auto kern = simt_mm_kernel<Pol, Sr, Pol::OCC>;
    constexpr int smem = simt::smem_bytes<Pol, Pol::OCC>();
    static bool attr_done[SL_MAX_DEV] = {};
    if (!attr_done[dev]) {
        SL_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr_done[dev] = true;
    }
    kern<<<grid, simt::THREADS, smem, s>>>(p);
    SL_CK(cudaGetLastError());
    return (int)cudaSuccess;
}

}  // namespace
