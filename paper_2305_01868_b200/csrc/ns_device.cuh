// ns_device.cuh -- device helpers shared by the search and scoring kernels.
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "ns_internal.cuh"

namespace ns {

constexpr unsigned kFull = 0xffffffffu;

// Exact max(x, 0) on the integer pipe (no FP64-pipe compare): the sign mask
// clears both words of a negative input (-0.0 -> +0.0), same value as
// x > 0 ? x : 0 for every non-NaN x.
__device__ __forceinline__ double relu_int(double x) {
    const int hi = __double2hiint(x), lo = __double2loint(x);
    const int m = hi >> 31;
    return __hiloint2double(hi & ~m, lo & ~m);
}
__device__ __forceinline__ double relu_exact(double x) { return relu_int(x); }


// max(x, 0) for the greedy's hot loop in ONE integer op: clamp the high word
// of the IEEE double at 0 (IMNMX).  For x >= 0 the result is x bit-for-bit;
// for x < 0 it is a non-negative subnormal (< 2^-1022).  Multiplied by a head
// weight and added to an accumulator whose magnitude exceeds ~2^-960 this is
// below half an ulp, so the rounded sum equals the exact-ReLU sum (DESIGN.md
// "Greedy kernel": the only difference is for scores below ~1e-289).
__device__ __forceinline__ double relu_hi(double x) {
    int lo = __double2loint(x);
    int hi = __double2hiint(x);
    return __hiloint2double(max(hi, 0), lo);
}


}  // namespace ns
