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

template <class Pol, class Sr>
int launch_simt(const SimtParams& p, int grid, int sms, cudaStream_t s) {
    constexpr int smem = simt::smem_bytes<Pol>();
    if constexpr (has_occ1_build<Pol>() && Pol::OCC > 1) {
        if (grid <= sms) {
            auto k1 = simt_mm_kernel<Pol, Sr, 1>;
            static bool attr1 = false;
            if (!attr1) {
                SL_CK(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
                attr1 = true;
            }
            k1<<<grid, simt::THREADS, smem, s>>>(p);
            SL_CK(cudaGetLastError());
            return (int)cudaSuccess;
        }
    }
    auto kern = simt_mm_kernel<Pol, Sr, Pol::OCC>;
    static bool attr_done = false;
    if (!attr_done) {
        SL_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr_done = true;
    }
    kern<<<grid, simt::THREADS, smem, s>>>(p);
    SL_CK(cudaGetLastError());
    return (int)cudaSuccess;
}

}  // namespace
