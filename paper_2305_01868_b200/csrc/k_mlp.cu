// k_mlp.cu -- kernel N5: plan cost f = max_d(comp_d + fwd_d + bwd_d) for a
// batch of rows (trajectories of the search, or explicit plans of
// ns_score_plans), with the two communication-cost MLPs
// (2D -> 128 -> 64 -> 32 -> 16 -> D, "128-64-32-16"; "two
// separate models") evaluated on the FP64 tensor cores.
//
// The MLP over a batch of rows is a chain of dense GEMMs
// [rows x K] . W^T [K x N]; it runs as DMMA (mma.sync m8n8k4 .f64): fp64
// products and fp64 accumulation, so plan costs keep the oracle's precision
// (tcgen05 has no fp64 kind).  One warp owns 16 rows (two m8 tiles); the
// activations of its rows stay in shared memory between layers (ping-pong
// buffers padded so the A-fragment loads are bank-conflict free); weights
// are read as B fragments through L1 (the whole comm model is <= 0.6 MB and
// shared by every warp); bias + ReLU are fused into the accumulator epilogue.
// Forward starts are comp - min(comp) (reading R10), backward starts 0,
// inputs scaled by division exactly like the oracle (R10).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <math_constants.h>

#include "ns_device.cuh"
#include "ns_internal.cuh"

namespace ns {

struct PlanCostArgs {
    long long row_begin, row_end;   // rows [row_begin, row_end) of the arrays below
    int D;
    const uint8_t* feas;            // [rows] or nullptr (all feasible)
    const double* comp;             // [rows][D]
    const int32_t* devdim;          // [rows][D]
    double* cost;                   // [rows]
    CommParams cp;
    double start_scale, dim_scale;
    double inv_dim_scale;           // 1 / dim_scale when dim_scale is a power of two (exact), else 0
    int ldx, ldy;                   // smem row strides (doubles)
    int ldy2;                       // large D: row stride of the per-warp layer-2 / layer-4 outputs
    uint32_t rflags;                // NS_R10_ABS_STARTS / NS_R11_SUM_OF_MAX
    const int32_t* list;            // optional: rows = list[i], i < *list_n (then row_begin = 0, row_end = capacity)
    const int32_t* list_n;
};

constexpr unsigned kFullMlp = 0xffffffffu;

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

// Y[16 x N] = act(X[16 x K] . W^T + b) for the warp's 16 rows.
// W is [N][K] row-major (torch Linear), K % 4 == 0 except the first layer
// (guarded), N arbitrary (guarded).  RELU selects the hidden-layer epilogue.
template <bool RELU, bool UNROLL = false>
__device__ __forceinline__ void warp_layer(const double* __restrict__ W, const double* __restrict__ bias, int K,
                                           int N, const double* X, int ldx, double* Y, int ldy, int lane) {
    const int g = lane >> 2, t = lane & 3;
    const int K4 = (K + 3) >> 2, N8 = (N + 7) >> 3;
    for (int nc = 0; nc < N8; nc += 4) {
        double acc[2][4][2];
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[m][j][0] = acc[m][j][1] = 0.0;
        auto kstep = [&](int kt) {
            const int k = 4 * kt + t;
            const double a0 = X[g * ldx + k];
            const double a1 = X[(8 + g) * ldx + k];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int nt = nc + j;
                if (nt < N8) {   // warp-uniform
                    const int n = 8 * nt + g;
                    const double b = (n < N && k < K) ? __ldg(W + (size_t)n * K + k) : 0.0;
                    dmma(acc[0][j], a0, b);
                    dmma(acc[1][j], a1, b);
                }
            }
        };
        if constexpr (UNROLL) {
#pragma unroll 4
            for (int kt = 0; kt < K4; ++kt) kstep(kt);
        } else {
            for (int kt = 0; kt < K4; ++kt) kstep(kt);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int nt = nc + j;
            if (nt >= N8) continue;
            const int col = 8 * nt + 2 * t;
#pragma unroll
            for (int m = 0; m < 2; ++m) {
                const int r = 8 * m + g;
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int cc = col + e;
                    if (cc < N) {
                        double v = bias ? acc[m][j][e] + __ldg(bias + cc) : acc[m][j][e];
                        if (RELU) v = v > 0.0 ? v : 0.0;
                        Y[r * ldy + cc] = v;
                    }
                }
            }
        }
    }
    __syncwarp();
}

// Two warps own 16 rows, one per model direction (fwd / bwd run
// concurrently: half the dependent DMMA chain per row block, which is what
// bounds a single-task search's few hundred rows).  Layers 1 and 2 (2D -> 128 -> 64) are fused over
// four 32-unit chunks of the 128-wide hidden layer: each chunk is staged in
// shared memory and folded into the layer-2 accumulators (registers) at once,
// so no 16 x 128 activation buffer is needed (15 KB per warp instead of 27 KB
// -> 1.5x the resident warps).  Layers 3-5 use warp_layer.
#ifndef NS_PC_BLOCKS
#define NS_PC_BLOCKS 4
#endif
// BIG (D > 16, e.g. C5's 128 devices): the wide layers' weights stream from L2;
// their k-loops are unrolled so several B-fragment loads are in flight
template <bool BIG>
__global__ void __launch_bounds__(128, BIG ? 2 : NS_PC_BLOCKS) k_plan_cost_dmma(const PlanCostArgs a) {
    extern __shared__ double psm[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int D = a.D, K0 = 2 * D, K0p = (K0 + 3) & ~3;
    const int ldx = a.ldx, ldh = a.ldy;
    const int rb = w >> 1, dir = w & 1;   // row block of the CTA, model direction
    const int nrb = nwarps >> 1;
    const int per_warp = 16 * (ldx + ldh);
    const int per_rb = 16 * 2 * D + 32;
    double *X, *Hc, *O, *mn, *Y;
    long long* rid;
    if constexpr (BIG) {
        // one input tile per row block, read by both models (the bwd model
        // masks its start inputs); per warp Hc and Y; the outputs O overlay
        // the input tile after layer 1 -- 60 KB per CTA, 3 CTAs per SM
        const size_t rbw = (size_t)16 * ldx + 2 * 16 * (ldh + a.ldy2) + 64;
        X = psm + (size_t)rb * rbw;          // [16][ldx]: input, then O [16][2D]
        Hc = X + 16 * ldx + (size_t)dir * 16 * (ldh + a.ldy2);   // [16][ldh]: layer-1 chunk, layer-3 out
        Y = Hc + 16 * ldh;                   // [16][ldy2]: layer-2 out (64), layer-4 out (16)
        O = X;
        mn = X + 16 * ldx + 2 * 16 * (ldh + a.ldy2);
        rid = (long long*)(mn + 16);
    } else {
        X = psm + (size_t)w * per_warp;      // [16][ldx]: input, layer-2 out (64), layer-4 out (16)
        Hc = X + 16 * ldx;                   // [16][ldh]: layer-1 chunk (32), layer-3 out (32)
        Y = X;
        O = psm + (size_t)nwarps * per_warp + (size_t)rb * per_rb;   // [16][2D]: fwd, bwd
        mn = O + 16 * 2 * D;                 // [16] min comp per row
        rid = (long long*)(mn + 16);
    }
    const int ldyy = BIG ? a.ldy2 : ldx;     // row stride of Y
    const long long base = a.row_begin + ((long long)blockIdx.x * nrb + rb) * 16;
    const long long end = a.list ? a.row_begin + *a.list_n : a.row_end;
    const bool rows = base < end;
    // row ids (lane r < 16 of the fwd warp owns row r) and the per-row min
    // comp (min is exact in any order): small D one lane per row, large D
    // the fwd warp's lanes over the devices
    if (rows && dir == 0) {
        if (lane < 16) {
            const long long i = base + lane;
            long long r = -1;
            if (i < end) r = a.list ? (long long)a.list[i] : i;
            rid[lane] = r;
            if constexpr (!BIG) {
                double m = 0.0;
                if (r >= 0) {
                    m = CUDART_INF;
                    for (int d = 0; d < D; ++d) m = fmin(m, a.comp[r * D + d]);
                }
                mn[lane] = (a.rflags & NS_R10_ABS_STARTS) ? 0.0 : m;   // R10: relative (default) or absolute starts
            }
        }
        if constexpr (BIG) {
            __syncwarp();
            for (int r = 0; r < 16; ++r) {
                const long long row = rid[r];
                double m = CUDART_INF;
                if (row >= 0)
                    for (int d = lane; d < D; d += 32) m = fmin(m, a.comp[row * D + d]);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) m = fmin(m, __shfl_xor_sync(kFullMlp, m, o));
                if (lane == 0) mn[r] = (row < 0 || (a.rflags & NS_R10_ABS_STARTS)) ? 0.0 : m;
            }
        }
    }
    __syncthreads();
    if (rows) {
        // input rows [starts / start_scale (D), devdim / dim_scale (D)], zero
        // padded; a power-of-two dim_scale divides exactly by its reciprocal
        auto input = [&](int r, int c) {
            const long long row = rid[r];
            double v = 0.0;
            if (row >= 0 && c < K0) {
                if (c < D) {
                    v = (dir == 0 || BIG) ? (a.comp[row * D + c] - mn[r]) / a.start_scale : 0.0;
                } else {
                    const double dd = (double)a.devdim[row * D + (c - D)];
                    v = a.inv_dim_scale != 0.0 ? dd * a.inv_dim_scale : dd / a.dim_scale;
                }
            }
            X[r * ldx + c] = v;
        };
        if constexpr (BIG) {   // the shared tile: each warp builds 8 of its rows
            for (int r = 8 * dir; r < 8 * dir + 8; ++r)
                for (int c = lane; c < K0p; c += 32) input(r, c);
            __syncthreads();   // (BIG: one row block per CTA, rows is CTA-uniform)
        } else {
            for (int i = lane; i < 16 * K0p; i += 32) input(i / K0p, i % K0p);
        }
        __syncwarp();
        const double* W1 = a.cp.W[dir][0];
        const double* b1 = a.cp.b[dir][0];
        const double* W2 = a.cp.W[dir][1];
        // ---- layers 1+2: y2 = ReLU(W2 ReLU(W1 x + b1) + b2), 128 -> 64
        double acc2[2][8][2];
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
            for (int q = 0; q < 8; ++q) acc2[m][q][0] = acc2[m][q][1] = 0.0;
#pragma unroll 1
        for (int hc = 0; hc < 4; ++hc) {
            double acc1[2][4][2];
#pragma unroll
            for (int m = 0; m < 2; ++m)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc1[m][q][0] = acc1[m][q][1] = 0.0;
            // (unrolled: the B-fragment loads of several k-steps are in
            // flight together -- for large D the 2D x 128 layer-1 weights
            // stream from L2 and a one-step loop exposes its latency per step)
            auto l1_step = [&](int kt) {
                const int k = 4 * kt + t;
                const bool zs = BIG && dir == 1 && k < D;   // bwd: start inputs are 0
                const double a0 = zs ? 0.0 : X[g * ldx + k], a1 = zs ? 0.0 : X[(8 + g) * ldx + k];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int n = hc * 32 + 8 * q + g;
                    const double bv = k < K0 ? __ldg(W1 + (size_t)n * K0 + k) : 0.0;
                    dmma(acc1[0][q], a0, bv);
                    dmma(acc1[1][q], a1, bv);
                }
            };
            if constexpr (BIG) {   // (2 CTAs/SM by shared memory: registers for 16 steps of loads in flight)
                // bwd: the start inputs are 0, their products +-0 leave the
                // accumulators (+0 from the start) unchanged -- skip them
#pragma unroll 16
                for (int kt = dir == 1 ? D / 4 : 0; kt < K0p / 4; ++kt) l1_step(kt);
            } else {
                for (int kt = 0; kt < K0p / 4; ++kt) l1_step(kt);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int col = 8 * q + 2 * t;
                const double c0 = __ldg(b1 + hc * 32 + col), c1 = __ldg(b1 + hc * 32 + col + 1);
#pragma unroll
                for (int m = 0; m < 2; ++m) {
                    double2 hv;
                    hv.x = relu_exact(acc1[m][q][0] + c0);
                    hv.y = relu_exact(acc1[m][q][1] + c1);
                    *reinterpret_cast<double2*>(Hc + (8 * m + g) * ldh + col) = hv;
                }
            }
            __syncwarp();
#pragma unroll 2
            for (int kt = 0; kt < 8; ++kt) {
                const int k = 4 * kt + t;
                const double a0 = Hc[g * ldh + k], a1 = Hc[(8 + g) * ldh + k];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const double bv = __ldg(W2 + (size_t)(8 * q + g) * 128 + hc * 32 + k);
                    dmma(acc2[0][q], a0, bv);
                    dmma(acc2[1][q], a1, bv);
                }
            }
            __syncwarp();
        }
        {
            const double* b2 = a.cp.b[dir][1];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int col = 8 * q + 2 * t;
                const double c0 = __ldg(b2 + col), c1 = __ldg(b2 + col + 1);
#pragma unroll
                for (int m = 0; m < 2; ++m) {
                    double2 yv;
                    yv.x = relu_exact(acc2[m][q][0] + c0);
                    yv.y = relu_exact(acc2[m][q][1] + c1);
                    *reinterpret_cast<double2*>(Y + (8 * m + g) * ldyy + col) = yv;
                }
            }
        }
        __syncwarp();
        if constexpr (BIG) __syncthreads();   // both models are done with the input tile O overlays
        warp_layer<true, BIG>(a.cp.W[dir][2], a.cp.b[dir][2], 64, 32, Y, ldyy, Hc, ldh, lane);
        warp_layer<true, BIG>(a.cp.W[dir][3], a.cp.b[dir][3], 32, 16, Hc, ldh, Y, ldyy, lane);
        warp_layer<false, BIG>(a.cp.W[dir][4], a.cp.b[dir][4], 16, D, Y, ldyy, O + dir * D, 2 * D, lane);
    }
    __syncthreads();
    if (rows && dir == 0 && lane < 16) {
        const long long row = rid[lane];
        if (row >= 0) {
            double c = CUDART_INF;
            if (!a.feas || a.feas[row]) {
                c = -CUDART_INF;
                if (a.rflags & NS_R11_SUM_OF_MAX) {   // alternative R11: sum of the per-term maxima
                    double mc = -CUDART_INF, mf = -CUDART_INF, mb = -CUDART_INF;
                    for (int d = 0; d < D; ++d) {
                        mc = fmax(mc, a.comp[row * D + d]);
                        mf = fmax(mf, O[lane * 2 * D + d]);
                        mb = fmax(mb, O[lane * 2 * D + D + d]);
                    }
                    c = (mc + mf) + mb;
                } else {
                    for (int d = 0; d < D; ++d)
                        c = fmax(c, (a.comp[row * D + d] + O[lane * 2 * D + d]) + O[lane * 2 * D + D + d]);
                }
            }
            a.cost[row] = c;
        }
    }
}

// ---------------------------------------------------------------------------
// N1 on the FP64 tensor cores: per-table cached cost-model precompute.
// For every row (table g, split depth j): x = featurise(table, dim >> j)
// (R1), e = ReLU(W2 ReLU(W1 x + b1) + b2) (encoder "128-32",
// P:688; R2), v = H1 e (hoisted first head layer: H1 sum_t e_t + hb1 =
// hb1 + sum_t v_t), C({t}) = H2 ReLU(v + hb1) + hb2.  The encoder and the
// projection are a GEMM chain over rows; one warp owns 16 rows.
struct PreDmmaArgs {
    const ns_table_desc* desc;
    long long n_rows;        // n_tables * nj
    int jlo, nj;
    const double* enc1W;
    const double* enc1b;
    const double* enc2W;
    const double* enc2b;
    const double* H1;
    HeadParams head;
    double* feat;
    double* V;
    double* C;
    int32_t* vdim;
    int64_t* vbytes;
    int ldx, ldy;
    const int32_t* list;     // optional: rows r = list[1 + i], i < list[0] (valid deep variants only)
};

// One warp owns 16 rows.  The 128-wide hidden layer is produced in four
// 32-column chunks and folded into the layer-2 accumulators (kept in
// registers) immediately, so only a 16x32 chunk is ever staged in shared
// memory (11 KB per warp instead of 21 KB -> 2.5x the resident warps).  v
// leaves the accumulator fragments straight to HBM; the single-table cost is
// reduced from the same fragments.
#define PRE_RELU relu_int
#ifndef NS_PRE_BLOCKS
#define NS_PRE_BLOCKS 5
#endif
// shared-memory weight layout (NS_PRE_WSM): padded rows, stride == 4 mod 16
// doubles so a warp's B fragments fall on distinct banks
constexpr int kPW1 = 20, kPW2 = 132, kPW3 = 36;              // row strides of W1 [128][5], W2 [32][128], H1 [64][32]
constexpr int kPO1 = 0, kPO2 = kPO1 + 128 * kPW1, kPO3 = kPO2 + 32 * kPW2;
constexpr int kPOb1 = kPO3 + 64 * kPW3, kPOb2 = kPOb1 + 128, kPOhb1 = kPOb2 + 32, kPOH2 = kPOhb1 + 64;
constexpr int kPWTotal = kPOH2 + 64;                          // doubles
// WSM: encoder / projection weights resident in shared memory, one 16-warp CTA
// per SM (batches: the weights are staged once per SM and every B fragment is
// a conflict-free shared-memory load); otherwise B fragments through L1 with
// 4-warp CTAs (a few hundred rows: no staging latency).
template <bool WSM>
#ifndef NS_PRE_WSM_WARPS
#define NS_PRE_WSM_WARPS 16   // warps of the batched (shared-memory weights) precompute CTA
#endif
__global__ void __launch_bounds__(WSM ? 32 * NS_PRE_WSM_WARPS : 128, WSM ? 1 : NS_PRE_BLOCKS) k_precompute_dmma(const PreDmmaArgs a) {
    extern __shared__ double qsm[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int ldx = a.ldx, ldh = a.ldy;             // x and e stride / h-chunk stride
    double* const sw = qsm;   // WSM: weights (kPWTotal doubles) then the per-warp buffers
    if constexpr (WSM) {
        for (int i = threadIdx.x; i < 128 * kPW1; i += blockDim.x) {
            const int n = i / kPW1, k = i % kPW1;
            sw[kPO1 + i] = k < kF ? a.enc1W[n * kF + k] : 0.0;
        }
        for (int i = threadIdx.x; i < 32 * kPW2; i += blockDim.x) {
            const int n = i / kPW2, k = i % kPW2;
            sw[kPO2 + i] = k < kH ? a.enc2W[n * kH + k] : 0.0;
        }
        for (int i = threadIdx.x; i < 64 * kPW3; i += blockDim.x) {
            const int n = i / kPW3, k = i % kPW3;
            sw[kPO3 + i] = k < kE ? a.H1[n * kE + k] : 0.0;
        }
        for (int i = threadIdx.x; i < 128; i += blockDim.x) sw[kPOb1 + i] = a.enc1b[i];
        for (int i = threadIdx.x; i < 32; i += blockDim.x) sw[kPOb2 + i] = a.enc2b[i];
        for (int i = threadIdx.x; i < 64; i += blockDim.x) {
            sw[kPOhb1 + i] = a.head.hb1[i];
            sw[kPOH2 + i] = a.head.H2[i];
        }
        __syncthreads();
    }
#define PW1(n, k) (WSM ? sw[kPO1 + (n) * kPW1 + (k)] : ((k) < kF ? __ldg(a.enc1W + (n) * kF + (k)) : 0.0))
#define PB1(i) (WSM ? sw[kPOb1 + (i)] : __ldg(a.enc1b + (i)))
#define PW2(n, k) (WSM ? sw[kPO2 + (n) * kPW2 + (k)] : __ldg(a.enc2W + (n) * kH + (k)))
#define PB2(i) (WSM ? sw[kPOb2 + (i)] : __ldg(a.enc2b + (i)))
#define PH1(n, k) (WSM ? sw[kPO3 + (n) * kPW3 + (k)] : __ldg(a.H1 + (n) * kE + (k)))
#define PHB1(i) (WSM ? sw[kPOhb1 + (i)] : a.head.hb1[i])
#define PH2(i) (WSM ? sw[kPOH2 + (i)] : a.head.H2[i])
    // per warp: X [16][ldx] features (zero padded), Hc [16][ldh] hidden chunk,
    // E [16][ldh] table representation e (WSM: reuses the chunk buffer), row ids
    const int per_warp = WSM ? 16 * (ldx + ldh) + 16 : 16 * (ldx + ldh + ldh) + 16;
    double* X = qsm + (WSM ? kPWTotal : 0) + (size_t)w * per_warp;
    double* Hc = X + 16 * ldx;
    double* E = WSM ? Hc : Hc + 16 * ldh;
    long long* rowid = (long long*)(E + 16 * ldh);
    const long long n_rows = a.list ? (long long)__ldg(a.list) : a.n_rows;
    for (long long base = ((long long)blockIdx.x * nwarps + w) * 16; base < n_rows;
         base += (long long)gridDim.x * nwarps * 16) {
        // ---- features of the 16 rows (lane r < 16 owns row r); invalid variants -> zeros
        if (lane < 16) {
            const long long r = (a.list && base + lane < n_rows) ? (long long)__ldg(a.list + 1 + base + lane) : base + lane;
            double x[kF] = {0, 0, 0, 0, 0};
            long long row = -1;
            if (base + lane < n_rows) {
                const long long gtab = r / a.nj;
                const int j = a.jlo + (int)(r % a.nj);
                const ns_table_desc td = a.desc[gtab];
                bool ok = true;
                int dim = td.dim;
                for (int k = 0; k < j; ++k) {
                    if (dim % 8 != 0) ok = false;
                    dim >>= 1;
                }
                row = gtab * kDepth + j;
                if (ok) {
                    x[0] = (double)dim / 128.0;
                    x[1] = log10((double)td.hash_size) / 8.0;
                    x[2] = td.pooling_factor / 50.0;
                    x[3] = td.skew / 2.0;
                    x[4] = (double)td.hash_size * (double)dim * 4.0 / 1073741824.0;
                    for (int f = 0; f < kF; ++f) a.feat[row * kF + f] = x[f];
                    a.vdim[row] = dim;
                    a.vbytes[row] = td.hash_size * (long long)dim * 4;
                } else {
                    a.vdim[row] = 0;
                    row = -1;   // no v / cost for a variant that cannot exist
                }
            }
            rowid[lane] = row;
#pragma unroll
            for (int f = 0; f < kF; ++f) X[lane * ldx + f] = x[f];
            for (int f = kF; f < 8; ++f) X[lane * ldx + f] = 0.0;
        }
        __syncwarp();
        // ---- layers 1+2 fused over 4 chunks of 32 hidden units
        double e_acc[2][4][2];
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
            for (int q = 0; q < 4; ++q) e_acc[m][q][0] = e_acc[m][q][1] = 0.0;
#pragma unroll 1
        for (int hc = 0; hc < kH / 32; ++hc) {
            // h chunk = ReLU(x W1[hc*32 .. +32]^T + b1)   (K = 5, padded to 8)
            double hacc[2][4][2];
#pragma unroll
            for (int m = 0; m < 2; ++m)
#pragma unroll
                for (int q = 0; q < 4; ++q) hacc[m][q][0] = hacc[m][q][1] = 0.0;
#pragma unroll
            for (int kt = 0; kt < 2; ++kt) {
                const int k = 4 * kt + t;
                const double a0 = X[g * ldx + k], a1 = X[(8 + g) * ldx + k];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int n = hc * 32 + 8 * q + g;
                    const double bv = PW1(n, k);
                    dmma(hacc[0][q], a0, bv);
                    dmma(hacc[1][q], a1, bv);
                }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int col = 8 * q + 2 * t;
                const double b0 = PB1(hc * 32 + col), b1 = PB1(hc * 32 + col + 1);
#pragma unroll
                for (int m = 0; m < 2; ++m) {
                    double2 hv;
                    hv.x = PRE_RELU(hacc[m][q][0] + b0);
                    hv.y = PRE_RELU(hacc[m][q][1] + b1);
                    *reinterpret_cast<double2*>(Hc + (8 * m + g) * ldh + col) = hv;
                }
            }
            __syncwarp();
            // e_acc += h_chunk W2[:, hc*32 .. +32]^T    (K = 32 per chunk)
#pragma unroll
            for (int kt = 0; kt < 8; ++kt) {
                const int k = 4 * kt + t;
                const double a0 = Hc[g * ldh + k], a1 = Hc[(8 + g) * ldh + k];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int n = 8 * q + g;
                    const double bv = PW2(n, hc * 32 + k);
                    dmma(e_acc[0][q], a0, bv);
                    dmma(e_acc[1][q], a1, bv);
                }
            }
            __syncwarp();
        }
        // ---- e = ReLU(e_acc + b2) -> smem
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int col = 8 * q + 2 * t;
            const double b0 = PB2(col), b1 = PB2(col + 1);
#pragma unroll
            for (int m = 0; m < 2; ++m) {
                double2 ev;
                ev.x = PRE_RELU(e_acc[m][q][0] + b0);
                ev.y = PRE_RELU(e_acc[m][q][1] + b1);
                *reinterpret_cast<double2*>(E + (8 * m + g) * ldh + col) = ev;
            }
        }
        __syncwarp();
        // ---- v = H1 e (64 outputs, K = 32), straight from the fragments to HBM,
        //      and the single-table cost C({t}) = hb2 + sum_k H2_k ReLU(v_k + hb1_k)
        double cpart[2] = {0.0, 0.0};
        const long long row0 = rowid[g], row1 = rowid[8 + g];
#pragma unroll
        for (int nc = 0; nc < 2; ++nc) {
            double vacc[2][4][2];
#pragma unroll
            for (int m = 0; m < 2; ++m)
#pragma unroll
                for (int q = 0; q < 4; ++q) vacc[m][q][0] = vacc[m][q][1] = 0.0;
#pragma unroll
            for (int kt = 0; kt < 8; ++kt) {
                const int k = 4 * kt + t;
                const double a0 = E[g * ldh + k], a1 = E[(8 + g) * ldh + k];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int n = nc * 32 + 8 * q + g;
                    const double bv = PH1(n, k);
                    dmma(vacc[0][q], a0, bv);
                    dmma(vacc[1][q], a1, bv);
                }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int col = nc * 32 + 8 * q + 2 * t;
#pragma unroll
                for (int m = 0; m < 2; ++m) {
                    const long long row = m ? row1 : row0;
                    const double v0 = vacc[m][q][0], v1 = vacc[m][q][1];
                    if (row >= 0) *reinterpret_cast<double2*>(a.V + row * kV + col) = make_double2(v0, v1);
                    cpart[m] = fma(PH2(col), PRE_RELU(v0 + PHB1(col)), cpart[m]);
                    cpart[m] = fma(PH2(col + 1), PRE_RELU(v1 + PHB1(col + 1)), cpart[m]);
                }
            }
        }
        // reduce the 4 lanes of each row (fixed xor order -> deterministic)
#pragma unroll
        for (int m = 0; m < 2; ++m) {
            cpart[m] += __shfl_xor_sync(kFull, cpart[m], 1);
            cpart[m] += __shfl_xor_sync(kFull, cpart[m], 2);
        }
        if (t == 0) {
            if (row0 >= 0) a.C[row0] = a.head.hb2 + cpart[0];
            if (row1 >= 0) a.C[row1] = a.head.hb2 + cpart[1];
        }
        __syncwarp();
    }
}
#undef PW1
#undef PB1
#undef PW2
#undef PB2
#undef PH1
#undef PHB1
#undef PH2

static int ld_pad(int width) { return ((width + 15) / 16) * 16 + 4; }   // == 4 (mod 16): conflict-free A frags

ns_status launch_plan_cost(ns_ctx* ctx, long long rb, long long re, const uint8_t* feas, const double* comp,
                           const int32_t* devdim, double* cost, const int32_t* list, const int32_t* list_n) {
    if (re <= rb) return NS_OK;
    PlanCostArgs a;
    a.list = list;
    a.list_n = list_n;
    a.row_begin = rb;
    a.row_end = re;
    a.D = ctx->model.D;
    a.rflags = ctx->rflags;
    a.feas = feas;
    a.comp = comp;
    a.devdim = devdim;
    a.cost = cost;
    a.cp = comm_params(ctx);
    a.start_scale = ctx->model.start_scale;
    a.dim_scale = ctx->model.dim_scale;
    {
        int e;
        a.inv_dim_scale = (a.dim_scale > 0.0 && std::frexp(a.dim_scale, &e) == 0.5) ? 1.0 / a.dim_scale : 0.0;
    }
    const int K0p = (2 * a.D + 3) & ~3;
    a.ldx = ld_pad(K0p > 64 ? K0p : 64);
    a.ldy = ld_pad(32);
    a.ldy2 = ld_pad(64);
    const size_t per_warp = (size_t)16 * (a.ldx + a.ldy) * sizeof(double);
    const size_t per_rb = (size_t)(16 * 2 * a.D + 32) * sizeof(double);
    int wpb = 4;   // warps per CTA: two per 16-row block (fwd, bwd)
    while (wpb > 2 && per_warp * wpb + per_rb * (wpb / 2) > 72 * 1024) wpb >>= 1;
    size_t smem = per_warp * wpb + per_rb * (wpb / 2);
    if (a.D > 16) {   // large D: one row block per CTA with a shared input tile (k_plan_cost_dmma<true>)
        wpb = 2;
        smem = ((size_t)16 * a.ldx + 2 * 16 * (a.ldy + a.ldy2) + 64) * sizeof(double);
    }
    if (a.D > 16)
        cudaFuncSetAttribute(k_plan_cost_dmma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    else
        cudaFuncSetAttribute(k_plan_cost_dmma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const long long rows = re - rb;
    const long long blocks = (rows + 8LL * wpb - 1) / (8LL * wpb);   // 16 rows per warp pair
    prof_begin(ctx, PK_FINALIZE);
    if (a.D > 16)
        k_plan_cost_dmma<true><<<(unsigned)blocks, wpb * 32, smem, ctx->stream>>>(a);
    else
        k_plan_cost_dmma<false><<<(unsigned)blocks, wpb * 32, smem, ctx->stream>>>(a);
    prof_end(ctx);
    NS_LAUNCHED(ctx);
    return NS_OK;
}

// Deep variants (depth >= 1): only a table whose dims stay divisible by 8
// can be halved j times (the dim % 8 rule of the candidates), so the
// rows that cannot exist get vdim = 0 here and the DMMA kernel runs over the
// compacted list of the others (about 2/5 of them for dims uniform in
// multiples of 4).  Row order in the list does not matter: every row's
// arithmetic is independent of its 16-row block.
__global__ void k_pre_compact(const ns_table_desc* desc, long long n_rows, int jlo, int nj, int32_t* vdim,
                              int32_t* list) {
    for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < n_rows;
         r += (long long)gridDim.x * blockDim.x) {
        const long long g = r / nj;
        const int j = jlo + (int)(r % nj);
        int dim = desc[g].dim;
        bool ok = true;
        for (int k = 0; k < j; ++k) {
            if (dim % 8 != 0) ok = false;
            dim >>= 1;
        }
        if (ok)
            list[1 + atomicAdd(list, 1)] = (int32_t)r;
        else
            vdim[g * kDepth + j] = 0;
    }
}

void launch_precompute(ns_ctx* ctx, const ns_tables* t, int jlo, int jhi) {
    PreDmmaArgs a;
    a.desc = t->d_desc;
    a.nj = jhi - jlo + 1;
    a.jlo = jlo;
    a.n_rows = (long long)t->n_tables * a.nj;
    a.enc1W = ctx->model.enc1W;
    a.enc1b = ctx->model.enc1b;
    a.enc2W = ctx->model.enc2W;
    a.enc2b = ctx->model.enc2b;
    a.H1 = ctx->model.H1;
    a.head = ctx->model.head;
    a.feat = t->d_feat;
    a.V = t->d_V;
    a.C = t->d_C;
    a.vdim = t->d_vdim;
    a.vbytes = t->d_vbytes;
    a.ldx = ld_pad(8);    // x (8 features, zero padded)
    a.ldy = ld_pad(32);   // hidden chunk and e (32)
    a.list = nullptr;
    if (jlo >= 1 && t->d_plist && a.n_rows >= 16LL * 16 * ctx->sm_count && !getenv("NS_PRE_ALL_ROWS")) {
        cudaMemsetAsync(t->d_plist, 0, sizeof(int32_t), ctx->stream);
        const long long cb = std::min<long long>((a.n_rows + 255) / 256, (long long)ctx->sm_count * 16);
        k_pre_compact<<<(unsigned)cb, 256, 0, ctx->stream>>>(a.desc, a.n_rows, a.jlo, a.nj, a.vdim, t->d_plist);
        ctx->launches++;
        a.list = t->d_plist;
    }
    // batches stage the weights once per SM; a few hundred rows (a single
    // task) read them through L1 instead of paying the staging latency
    const bool wsm = a.n_rows >= 16LL * 16 * ctx->sm_count;
    const int wpb = wsm ? NS_PRE_WSM_WARPS : 4;
    const size_t smem = wsm ? ((size_t)kPWTotal + (size_t)wpb * (16 * (a.ldx + a.ldy) + 16)) * sizeof(double)
                            : (size_t)wpb * (16 * (a.ldx + 2 * a.ldy) + 16) * sizeof(double);
    if (wsm)
        cudaFuncSetAttribute(k_precompute_dmma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    else
        cudaFuncSetAttribute(k_precompute_dmma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    long long blocks = (a.n_rows + 16LL * wpb - 1) / (16LL * wpb);
    const long long cap = (long long)ctx->sm_count * (wsm ? 1 : 16);
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    prof_begin(ctx, PK_PRECOMPUTE);
    if (wsm)
        k_precompute_dmma<true><<<(unsigned)blocks, wpb * 32, smem, ctx->stream>>>(a);
    else
        k_precompute_dmma<false><<<(unsigned)blocks, wpb * 32, smem, ctx->stream>>>(a);
    prof_end(ctx);
    ctx->launches++;
}

}  // namespace ns
