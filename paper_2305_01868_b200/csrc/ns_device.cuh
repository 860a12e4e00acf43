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


// One dense fp64 layer computed by a warp: y[o] = act(b[o] + sum_i W[o][i] x[i])
// with x and y in shared memory.  Deterministic sequential order over i.
template <bool RELU>
__device__ __forceinline__ void warp_dense(const double* __restrict__ W, const double* __restrict__ b,
                                           int in, int out, const double* x, double* y, int lane) {
    for (int o = lane; o < out; o += 32) {
        const double* w = W + (size_t)o * in;
        double acc = 0.0;
        for (int i = 0; i < in; ++i) acc = fma(__ldg(w + i), x[i], acc);
        acc = acc + __ldg(b + o);
        y[o] = RELU ? relu_exact(acc) : acc;
    }
    __syncwarp();
}

// Plan cost from per-device compute costs and device dims (
// readings R4, R10, R11), one warp.  `buf` is warp-private shared scratch of
// >= 2*(2*D + 128) + 2*D doubles.  Returns max_d (comp + fwd + bwd) on all lanes.
__device__ inline double warp_plan_cost(const CommParams& cp, const double* comp, const int32_t* devdim,
                                 double* buf, int lane, double start_scale, double dim_scale) {
    const int D = cp.D;
    double* x = buf;                  // [2D]  (also used as ping buffer, >= 128)
    double* y = buf + 2 * D + 128;    // [128]
    double* out = y + 2 * D + 128;    // [2D]: fwd then bwd
    // min comp (reading R10: forward starts are the relative compute delays)
    double mn = CUDART_INF;
    for (int d = lane; d < D; d += 32) mn = fmin(mn, comp[d]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(kFull, mn, o));
    for (int dir = 0; dir < 2; ++dir) {
        for (int d = lane; d < D; d += 32) {
            x[d] = dir == 0 ? (comp[d] - mn) / start_scale : 0.0;
            x[D + d] = (double)devdim[d] / dim_scale;
        }
        __syncwarp();
        warp_dense<true>(cp.W[dir][0], cp.b[dir][0], 2 * D, 128, x, y, lane);
        warp_dense<true>(cp.W[dir][1], cp.b[dir][1], 128, 64, y, x, lane);
        warp_dense<true>(cp.W[dir][2], cp.b[dir][2], 64, 32, x, y, lane);
        warp_dense<true>(cp.W[dir][3], cp.b[dir][3], 32, 16, y, x, lane);
        warp_dense<false>(cp.W[dir][4], cp.b[dir][4], 16, D, x, out + dir * D, lane);
    }
    double mx = -CUDART_INF;
    for (int d = lane; d < D; d += 32) mx = fmax(mx, (comp[d] + out[d]) + out[D + d]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(kFull, mx, o));
    __syncwarp();
    return mx;
}

constexpr int kPlanCostScratch(int D) { return 2 * (2 * D + 128) + 2 * D; }

}  // namespace ns
