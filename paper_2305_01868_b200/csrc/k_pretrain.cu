// k_pretrain.cu -- SURVEY §8(f) row F2: pre-training the neural cost models on
// the GPU (§3.1-3.2, App. B Alg. 3-5, App. C, App. F).
//
//  * sample generation: Alg. 3 augmentation is the index map (pool table t,
//    dimension j) -> augmented table t * n_dims + j; Alg. 4 combinations and
//    the subsets / uniforms of Alg. 5 are drawn by the caller (random numbers
//    are inputs); k_pt_compute_samples featurises every table of every
//    combination (reading R1) and labels the combination, k_pt_place runs
//    Alg. 5 lines 6-16 (sort by dimension, greedy-with-probability-p
//    placement over memory-feasible devices) and labels the placement;
//  * labels: SPEC.md's analytic cost model (constants S:113) stands
//    in for the paper's GPU micro-benchmarks (reading F2-L);
//  * training: one MSE/Adam step (App. C, App. F: Adam lr 1e-3, torch
//    defaults) = a fused forward + backward kernel per model that writes one
//    partial gradient per CTA (deterministic, no atomics) and a fused
//    reduce + Adam kernel.  Everything is fp64 (the precision the search uses:
//    trained weights load straight into ns_load_cost_models).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "ns_device.cuh"
#include "ns_internal.cuh"

namespace ns {
namespace {

// SPEC.md:113 OracleParams defaults
constexpr double kKappaW = 2.5e-3, kOverhead = 0.15, kLaunch = 0.5, kGamma = 0.3, kDimExp = 0.8,
                 kHashCoef = 0.05, kSkewCoef = 0.3, kLatency = 1.0, kBetaF = 0.010, kBetaB = 0.012;

// SPEC.md:121 work(t), operation order of the oracle (left to right)
__device__ double pt_work(int dim, long long hash, double pool, double skew) {
    const double a = __dmul_rn(kKappaW, pool);
    const double b = __dmul_rn(a, pow((double)dim, kDimExp));
    const double c = __dmul_rn(b, __dadd_rn(1.0, __dmul_rn(kHashCoef, log10((double)hash))));
    return __dmul_rn(c, __dsub_rn(1.0, __ddiv_rn(__dmul_rn(kSkewCoef, fmin(skew, 2.0)), 2.0)));
}

// Alg. 3: augmented table a -> (pool table, dimension)
struct AugView {
    const ns_table_desc* pool;
    const int32_t* dims;
    int n_dims;
    __device__ ns_table_desc get(int a) const {
        ns_table_desc d = pool[a / n_dims];
        d.dim = dims[a % n_dims];
        return d;
    }
};

// One warp per combination: features of its tables (R1), label.
__global__ void __launch_bounds__(256) k_pt_compute_samples(AugView av, const int32_t* off, const int32_t* idx, int n,
                                                            double* feats, double* labels) {
    const int lane = threadIdx.x & 31;
    for (int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < n; s += (gridDim.x * blockDim.x) >> 5) {
        const int r0 = off[s], r1 = off[s + 1];
        for (int r = r0 + lane; r < r1; r += 32) {
            const ns_table_desc td = av.get(idx[r]);
            double* x = feats + (size_t)r * kF;
            x[0] = (double)td.dim / 128.0;
            x[1] = log10((double)td.hash_size) / 8.0;
            x[2] = td.pooling_factor / 50.0;
            x[3] = td.skew / 2.0;
            x[4] = (double)td.hash_size * (double)td.dim * 4.0 / 1073741824.0;
        }
        if (lane == 0) {
            double lab;
            if (r1 - r0 == 1) {
                const ns_table_desc td = av.get(idx[r0]);
                lab = __dadd_rn(kLaunch + kOverhead, pt_work(td.dim, td.hash_size, td.pooling_factor, td.skew));
            } else {
                double acc = 0.0;   // sum_t (gamma * overhead + work(t)) in list order
                for (int r = r0; r < r1; ++r) {
                    const ns_table_desc td = av.get(idx[r]);
                    acc = __dadd_rn(acc, __dadd_rn(kGamma * kOverhead,
                                                   pt_work(td.dim, td.hash_size, td.pooling_factor, td.skew)));
                }
                lab = __dadd_rn(kLaunch, acc);
            }
            labels[s] = lab;
        }
    }
}

// One thread per placement: Alg. 5 lines 6-16 and the comm labels
// of both directions.
constexpr int kPtMaxT = 256;
__global__ void __launch_bounds__(128) k_pt_place(AugView av, int D, long long cap, const int32_t* off,
                                                  const int32_t* idx, const double* p, const double* u,
                                                  const double* r, const double* starts, int n, double* x_out,
                                                  double* yf_out, double* yb_out, int8_t* assign_out,
                                                  uint8_t* valid_out, long long* dd_scratch) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const int r0 = off[s], T = off[s + 1] - off[s];
    long long* dd = dd_scratch + (size_t)s * 2 * D;   // device dims, then bytes
    long long* mem = dd + D;
    for (int d = 0; d < D; ++d) dd[d] = mem[d] = 0;
    // stable sort of the sampled tables by descending dimension (line 6)
    short ord[kPtMaxT];
    for (int i = 0; i < T; ++i) {
        const int di = av.get(idx[r0 + i]).dim;
        int k = i;
        while (k > 0 && av.get(idx[r0 + ord[k - 1]]).dim < di) {
            ord[k] = ord[k - 1];
            --k;
        }
        ord[k] = (short)i;
    }
    bool valid = true;
    for (int k = 0; k < T; ++k) {
        const int i = ord[k];
        const ns_table_desc td = av.get(idx[r0 + i]);
        const long long bt = td.hash_size * (long long)td.dim * 4;
        int ncand = 0, best = -1;
        for (int d = 0; d < D; ++d)
            if (mem[d] + bt <= cap) {   // line 10: no memory error
                ++ncand;
                if (best < 0 || dd[d] < dd[best]) best = d;   // lowest device dim, lowest index on ties
            }
        if (ncand == 0) {
            valid = false;
            break;
        }
        int dsel = best;   // line 12
        if (!(u[r0 + k] <= p[s])) {   // line 14: candidate floor(r * |cand|) in device order
            int c = (int)floor(r[r0 + k] * (double)ncand);
            if (c > ncand - 1) c = ncand - 1;
            for (int d = 0; d < D; ++d)
                if (mem[d] + bt <= cap) {
                    if (c == 0) {
                        dsel = d;
                        break;
                    }
                    --c;
                }
        }
        assign_out[r0 + i] = (int8_t)dsel;
        dd[dsel] += td.dim;
        mem[dsel] += bt;
    }
    valid_out[s] = valid ? 1 : 0;
    // labels: T_end = max starts + latency + beta * max dims
    const double* st = starts + (size_t)s * D;
    double smax = -INFINITY;
    long long dmax = 0;
    for (int d = 0; d < D; ++d) {
        smax = fmax(smax, st[d]);
        dmax = dd[d] > dmax ? dd[d] : dmax;
    }
    const double tf = __dadd_rn(__dadd_rn(smax, kLatency), __dmul_rn(kBetaF, (double)dmax));
    const double tb = __dadd_rn(__dadd_rn(smax, kLatency), __dmul_rn(kBetaB, (double)dmax));
    for (int d = 0; d < D; ++d) {
        x_out[(size_t)s * 2 * D + d] = st[d] / 20.0;                  // reading R10 input scaling
        x_out[(size_t)s * 2 * D + D + d] = (double)dd[d] / 1024.0;
        yf_out[(size_t)s * D + d] = __dsub_rn(tf, st[d]);
        yb_out[(size_t)s * D + d] = __dsub_rn(tb, st[d]);
    }
}

// ---------------------------------------------------------------- training
// Flat parameter layout (torch order): per layer W [out][in] row-major, then b.

// Computation cost model, fused forward + backward over SPB samples per CTA
// (<= kPtRows table rows): encoder rows in parallel, per-sample sum, head,
// backward through head and encoder; the CTA's gradient partial (sum over its
// samples) goes to part[blockIdx.x][P].
constexpr int kPtRows = 64;
__global__ void __launch_bounds__(256) k_pt_compute_grad(const double* __restrict__ th, const double* feats,
                                                         const int32_t* off, const int32_t* list,
                                                         const double* labels, int B, int spb, double* part,
                                                         double* loss_part) {
    constexpr int P = 128 * 5 + 128 + 32 * 128 + 32 + 64 * 32 + 64 + 64 + 1;
    const int o1 = 0, ob1 = 640, o2 = 768, ob2 = 4864, o3 = 4896, ob3 = 6944, o4 = 7008, ob4 = 7072;
    extern __shared__ __align__(16) double sm[];
    double* X = sm;                           // [kPtRows][5]
    double* H = X + kPtRows * 5;              // [kPtRows][128] h1 (post-ReLU), later dh1
    double* E = H + kPtRows * 128;            // [kPtRows][32] e, later de
    double* S = E + kPtRows * 32;             // [spb][32]
    double* A = S + 16 * 32;                  // [spb][64] a (post-ReLU)
    double* dA = A + 16 * 64;                 // [spb][64]
    double* dS = dA + 16 * 64;                // [spb][32]
    double* err = dS + 16 * 32;               // [spb]
    double* sW1 = err + 16;                   // weights staged in shared memory (conflict-free layouts):
    double* sb1 = sW1 + 640;                  //   W1 [128][5], b1
    double* sW2 = sb1 + 128;                  //   W2 [32][128] (dh1 = W2^T de: lanes over inputs)
    double* sW2T = sW2 + 4096;                //   W2^T [128][32] (z2 = W2 h1: lanes over outputs)
    double* sb2 = sW2T + 4096;
    double* sH1 = sb2 + 32;                   //   H1 [64][32] (dS = H1^T dA)
    double* sH1T = sH1 + 2048;                //   H1^T [32][64] (za = H1 s)
    double* shb1 = sH1T + 2048;
    double* sH2 = shb1 + 64;                  //   H2 [64], hb2
    int* rs = (int*)(sH2 + 64 + 2);           // [kPtRows] sample (local) of each row
    __shared__ int s_r0[17];
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int i = tid; i < 640; i += nt) sW1[i] = __ldg(th + o1 + i);
    for (int i = tid; i < 128; i += nt) sb1[i] = __ldg(th + ob1 + i);
    for (int i = tid; i < 4096; i += nt) {
        const double wv = __ldg(th + o2 + i);
        sW2[i] = wv;
        sW2T[(i & 127) * 32 + (i >> 7)] = wv;
    }
    for (int i = tid; i < 32; i += nt) sb2[i] = __ldg(th + ob2 + i);
    for (int i = tid; i < 2048; i += nt) {
        const double wv = __ldg(th + o3 + i);
        sH1[i] = wv;
        sH1T[(i & 31) * 64 + (i >> 5)] = wv;
    }
    for (int i = tid; i < 64; i += nt) {
        shb1[i] = __ldg(th + ob3 + i);
        sH2[i] = __ldg(th + o4 + i);
    }
    if (tid == 0) sH2[64] = __ldg(th + ob4);
    const int s0 = blockIdx.x * spb, ns_ = min(spb, B - s0);
    if (tid == 0) {
        int acc = 0;
        for (int k = 0; k < ns_; ++k) {
            s_r0[k] = acc;
            const int sg = list[s0 + k];
            acc += off[sg + 1] - off[sg];
        }
        s_r0[ns_] = acc;
    }
    __syncthreads();
    const int R = s_r0[ns_];
    for (int e = tid; e < R * 5; e += nt) {
        const int rr = e / 5;
        int k = 0;
        while (s_r0[k + 1] <= rr) ++k;
        const int sg = list[s0 + k];
        X[e] = feats[(size_t)(off[sg] + rr - s_r0[k]) * 5 + e % 5];
        if (e % 5 == 0) rs[rr] = k;
    }
    __syncthreads();
    // h1 = ReLU(W1 x + b1)
    for (int e = tid; e < R * 128; e += nt) {
        const int rr = e >> 7, o = e & 127;
        double z = 0.0;
        for (int i = 0; i < 5; ++i) z = fma(sW1[o * 5 + i], X[rr * 5 + i], z);
        H[e] = relu_exact(z + sb1[o]);
    }
    __syncthreads();
    // e = ReLU(W2 h1 + b2)
    for (int e = tid; e < R * 32; e += nt) {
        const int rr = e >> 5, o = e & 31;
        double z = 0.0;
        for (int i = 0; i < 128; ++i) z = fma(sW2T[i * 32 + o], H[rr * 128 + i], z);
        E[e] = relu_exact(z + sb2[o]);
    }
    __syncthreads();
    // per-sample sum (row order)
    for (int e = tid; e < ns_ * 32; e += nt) {
        const int k = e >> 5, j = e & 31;
        double acc = 0.0;
        for (int rr = s_r0[k]; rr < s_r0[k + 1]; ++rr) acc += E[rr * 32 + j];
        S[e] = acc;
    }
    __syncthreads();
    // a = ReLU(H1 s + hb1)
    for (int e = tid; e < ns_ * 64; e += nt) {
        const int k = e >> 6, o = e & 63;
        double z = 0.0;
        for (int i = 0; i < 32; ++i) z = fma(sH1T[i * 64 + o], S[k * 32 + i], z);
        A[e] = relu_exact(z + shb1[o]);
    }
    __syncthreads();
    // y = H2 a + hb2; err; dA
    for (int k = tid >> 5; k < ns_; k += nt >> 5) {   // one warp per sample
        const int l = tid & 31;
        double z = fma(sH2[l], A[k * 64 + l], 0.0);
        z = fma(sH2[32 + l], A[k * 64 + 32 + l], z);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) z += __shfl_xor_sync(kFull, z, o);
        if (l == 0) err[k] = (z + sH2[64]) - labels[list[s0 + k]];
    }
    __syncthreads();
    for (int e = tid; e < ns_ * 64; e += nt) {
        const int k = e >> 6, o = e & 63;
        const double dy = 2.0 * err[k] / (double)B;
        dA[e] = A[e] > 0.0 ? dy * sH2[o] : 0.0;
    }
    __syncthreads();
    // dS = H1^T dA
    for (int e = tid; e < ns_ * 32; e += nt) {
        const int k = e >> 5, j = e & 31;
        double z = 0.0;
        for (int o = 0; o < 64; ++o) z = fma(sH1[o * 32 + j], dA[k * 64 + o], z);
        dS[e] = z;
    }
    __syncthreads();
    double* g = part + (size_t)blockIdx.x * P;
    // head gradients (sums over the CTA's samples in order)
    for (int e = tid; e < 64 * 32 + 64 + 64 + 1; e += nt) {
        double acc = 0.0;
        if (e < 2048) {
            const int o = e >> 5, i = e & 31;
            for (int k = 0; k < ns_; ++k) acc = fma(dA[k * 64 + o], S[k * 32 + i], acc);
            g[o3 + e] = acc;
        } else if (e < 2048 + 64) {
            const int o = e - 2048;
            for (int k = 0; k < ns_; ++k) acc += dA[k * 64 + o];
            g[ob3 + o] = acc;
        } else if (e < 2048 + 128) {
            const int o = e - 2048 - 64;
            for (int k = 0; k < ns_; ++k) acc = fma(2.0 * err[k] / (double)B, A[k * 64 + o], acc);
            g[o4 + o] = acc;
        } else {
            for (int k = 0; k < ns_; ++k) acc += 2.0 * err[k] / (double)B;
            g[ob4] = acc;
        }
    }
    // de = dS[sample] * [e > 0]
    for (int e = tid; e < R * 32; e += nt) {
        const int rr = e >> 5, j = e & 31;
        E[e] = E[e] > 0.0 ? dS[rs[rr] * 32 + j] : 0.0;
    }
    __syncthreads();
    // dW2 = sum_rows de h1^T, db2 = sum_rows de
    for (int e = tid; e < 32 * 128 + 32; e += nt) {
        double acc = 0.0;
        if (e < 4096) {
            const int o = e >> 7, i = e & 127;
            for (int rr = 0; rr < R; ++rr) acc = fma(E[rr * 32 + o], H[rr * 128 + i], acc);
            g[o2 + e] = acc;
        } else {
            const int o = e - 4096;
            for (int rr = 0; rr < R; ++rr) acc += E[rr * 32 + o];
            g[ob2 + o] = acc;
        }
    }
    __syncthreads();
    // dh1 = (W2^T de) * [h1 > 0]  (in place of h1)
    for (int e = tid; e < R * 128; e += nt) {
        const int rr = e >> 7, i = e & 127;
        double z = 0.0;
        for (int o = 0; o < 32; ++o) z = fma(sW2[o * 128 + i], E[rr * 32 + o], z);
        H[e] = H[e] > 0.0 ? z : 0.0;
    }
    __syncthreads();
    // dW1 = sum_rows dh1 x^T, db1 = sum_rows dh1
    for (int e = tid; e < 128 * 5 + 128; e += nt) {
        double acc = 0.0;
        if (e < 640) {
            const int o = e / 5, i = e % 5;
            for (int rr = 0; rr < R; ++rr) acc = fma(H[rr * 128 + o], X[rr * 5 + i], acc);
            g[o1 + e] = acc;
        } else {
            const int o = e - 640;
            for (int rr = 0; rr < R; ++rr) acc += H[rr * 128 + o];
            g[ob1 + o] = acc;
        }
    }
    if (tid == 0) {
        double l = 0.0;
        for (int k = 0; k < ns_; ++k) l += err[k] * err[k] / (double)B;
        loss_part[blockIdx.x] = l;
    }
    (void)P;
}

// Communication cost model 2D -> 128 -> 64 -> 32 -> 16 -> D (ReLU hidden),
// SPB samples per CTA, weights through L1/L2 (any D).
constexpr int kPtCommSpb = 8;
__global__ void __launch_bounds__(256) k_pt_comm_grad(const double* __restrict__ th, int D, const double* x,
                                                      const double* y, const int32_t* list, int B, double* part,
                                                      double* loss_part) {
    extern __shared__ __align__(16) double sm[];
    const int w[6] = {2 * D, 128, 64, 32, 16, D};
    int wo[5], bo[5];
    int P = 0;
    for (int l = 0; l < 5; ++l) {
        wo[l] = P;
        P += w[l] * w[l + 1];
        bo[l] = P;
        P += w[l + 1];
    }
    const int tid = threadIdx.x, nt = blockDim.x;
    const int s0 = blockIdx.x * kPtCommSpb, ns_ = min(kPtCommSpb, B - s0);
    // activations h_l [spb][w_l] for l = 0..5 (h_0 = x, hidden post-ReLU, h_5 = output); deltas share the layout
    int ho[7];
    ho[0] = 0;
    for (int l = 0; l < 6; ++l) ho[l + 1] = ho[l] + kPtCommSpb * w[l];
    double* h = sm;
    double* dz = sm + ho[6];   // [spb][w_l] per layer, same offsets
    for (int e = tid; e < ns_ * w[0]; e += nt) {
        const int k = e / w[0], i = e % w[0];
        h[ho[0] + k * w[0] + i] = x[(size_t)list[s0 + k] * w[0] + i];
    }
    __syncthreads();
    for (int l = 0; l < 5; ++l) {
        const int in = w[l], out = w[l + 1];
        for (int e = tid; e < ns_ * out; e += nt) {
            const int k = e / out, o = e % out;
            double z = 0.0;
            for (int i = 0; i < in; ++i) z = fma(__ldg(th + wo[l] + o * in + i), h[ho[l] + k * in + i], z);
            z = z + __ldg(th + bo[l] + o);
            h[ho[l + 1] + k * out + o] = l < 4 ? relu_exact(z) : z;
        }
        __syncthreads();
    }
    // output delta: 2 (pred - y) / (B D)
    for (int e = tid; e < ns_ * D; e += nt) {
        const int k = e / D, o = e % D;
        dz[ho[5] + k * D + o] = 2.0 * (h[ho[5] + k * D + o] - y[(size_t)list[s0 + k] * D + o]) / ((double)B * D);
    }
    __syncthreads();
    if (tid == 0) {
        double l = 0.0;
        for (int k = 0; k < ns_; ++k)
            for (int o = 0; o < D; ++o) {
                const double e = h[ho[5] + k * D + o] - y[(size_t)list[s0 + k] * D + o];
                l += e * e / ((double)B * D);
            }
        loss_part[blockIdx.x] = l;
    }
    double* g = part + (size_t)blockIdx.x * P;
    for (int l = 4; l >= 0; --l) {
        const int in = w[l], out = w[l + 1];
        // dW_l = sum_k dz_{l+1} h_l^T, db_l = sum_k dz_{l+1}
        for (int e = tid; e < out * in + out; e += nt) {
            double acc = 0.0;
            if (e < out * in) {
                const int o = e / in, i = e % in;
                for (int k = 0; k < ns_; ++k) acc = fma(dz[ho[l + 1] + k * out + o], h[ho[l] + k * in + i], acc);
                g[wo[l] + e] = acc;
            } else {
                const int o = e - out * in;
                for (int k = 0; k < ns_; ++k) acc += dz[ho[l + 1] + k * out + o];
                g[bo[l] + o] = acc;
            }
        }
        if (l > 0) {   // dz_l = (W_l^T dz_{l+1}) * [h_l > 0]
            for (int e = tid; e < ns_ * in; e += nt) {
                const int k = e / in, i = e % in;
                double z = 0.0;
                for (int o = 0; o < out; ++o) z = fma(__ldg(th + wo[l] + o * in + i), dz[ho[l + 1] + k * out + o], z);
                dz[ho[l] + k * in + i] = h[ho[l] + k * in + i] > 0.0 ? z : 0.0;
            }
        }
        __syncthreads();
    }
}

// Sum of the CTA partials (in CTA order) + Adam (torch defaults).
__global__ void __launch_bounds__(256) k_pt_adam(const double* part, int nblk, int P, double* th, double* m,
                                                 double* v, double bc1, double bc2, double lr, double b1, double b2,
                                                 double eps, const double* loss_part, double* loss_out) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p == 0 && loss_out) {
        double l = 0.0;
        for (int k = 0; k < nblk; ++k) l += loss_part[k];
        *loss_out = l;
    }
    if (p >= P) return;
    double gsum = 0.0;
    for (int k = 0; k < nblk; ++k) gsum += part[(size_t)k * P + p];
    const double mm = b1 * m[p] + (1.0 - b1) * gsum;
    const double vv = b2 * v[p] + (1.0 - b2) * gsum * gsum;
    m[p] = mm;
    v[p] = vv;
    th[p] = th[p] - lr * (mm / bc1) / (sqrt(vv / bc2) + eps);
}

size_t comm_smem(int D) { return (size_t)2 * kPtCommSpb * (2 * D + 128 + 64 + 32 + 16 + D) * sizeof(double); }

}  // namespace

ns_status pt_adam(ns_ctx* ctx, const double* part, int nblk, int P, double* th, double* m, double* v, int64_t t,
                  double lr, const double* loss_part, double* loss_out) {
    const double b1 = 0.9, b2 = 0.999, eps = 1e-8;
    const double bc1 = 1.0 - std::pow(b1, (double)t), bc2 = 1.0 - std::pow(b2, (double)t);
    prof_begin(ctx, PK_OTHER);
    k_pt_adam<<<(P + 255) / 256, 256, 0, ctx->stream>>>(part, nblk, P, th, m, v, bc1, bc2, lr, b1, b2, eps, loss_part,
                                                        loss_out);
    prof_end(ctx);
    NS_LAUNCHED(ctx);
    return NS_OK;
}

}  // namespace ns

using namespace ns;

extern "C" {

ns_status ns_pretrain_compute_samples(ns_ctx* ctx, const ns_table_desc* pool, int32_t n_pool, const int32_t* aug_dims,
                                      int32_t n_dims, const int32_t* comb_off, const int32_t* comb_idx, int32_t n,
                                      double* feats_out, double* labels_out) {
    if (!ctx) return NS_ERR_ARG;
    if (!pool || n_pool < 1 || !aug_dims || n_dims < 1 || !comb_off || !comb_idx || n < 1 || !feats_out ||
        !labels_out)
        return set_err(ctx, NS_ERR_ARG, "ns_pretrain_compute_samples: bad argument");
    for (const void* q : {(const void*)pool, (const void*)aug_dims, (const void*)comb_off, (const void*)comb_idx,
                          (const void*)feats_out, (const void*)labels_out})
        if (!is_device_ptr(q)) return set_err(ctx, NS_ERR_ARG, "ns_pretrain_*: pointers must be device memory");
    cudaSetDevice(ctx->device);
    AugView av{pool, aug_dims, n_dims};
    const unsigned blocks = (unsigned)std::min<long long>(((long long)n + 7) / 8, (long long)ctx->sm_count * 16);
    prof_begin(ctx, PK_OTHER);
    k_pt_compute_samples<<<blocks, 256, 0, ctx->stream>>>(av, comb_off, comb_idx, n, feats_out, labels_out);
    prof_end(ctx);
    NS_LAUNCHED(ctx);
    return NS_OK;
}

ns_status ns_pretrain_comm_samples(ns_ctx* ctx, const ns_table_desc* pool, int32_t n_pool, const int32_t* aug_dims,
                                   int32_t n_dims, int32_t D, int64_t mem_cap, const int32_t* off, const int32_t* idx,
                                   const double* p, const double* u, const double* r, const double* starts, int32_t n,
                                   double* x_out, double* yf_out, double* yb_out, int8_t* assign_out,
                                   uint8_t* valid_out) {
    if (!ctx) return NS_ERR_ARG;
    if (!pool || n_pool < 1 || !aug_dims || n_dims < 1 || D < 1 || D > kMaxD || !off || !idx || !p || !u || !r ||
        !starts || n < 1 || !x_out || !yf_out || !yb_out || !assign_out || !valid_out)
        return set_err(ctx, NS_ERR_ARG, "ns_pretrain_comm_samples: bad argument");
    for (const void* q : {(const void*)pool, (const void*)aug_dims, (const void*)off, (const void*)idx, (const void*)p,
                          (const void*)u, (const void*)r, (const void*)starts, (const void*)x_out,
                          (const void*)yf_out, (const void*)yb_out, (const void*)assign_out, (const void*)valid_out})
        if (!is_device_ptr(q)) return set_err(ctx, NS_ERR_ARG, "ns_pretrain_*: pointers must be device memory");
    cudaSetDevice(ctx->device);
    const size_t need = (size_t)n * 2 * D * sizeof(long long) + 256;
    long long* scratch = (long long*)arena_get(ctx, need);
    if (!scratch) return arena_error(ctx, "placements", need);
    AugView av{pool, aug_dims, n_dims};
    prof_begin(ctx, PK_OTHER);
    k_pt_place<<<(n + 127) / 128, 128, 0, ctx->stream>>>(av, D, mem_cap, off, idx, p, u, r, starts, n, x_out, yf_out,
                                                         yb_out, assign_out, valid_out, scratch);
    prof_end(ctx);
    NS_LAUNCHED(ctx);
    return NS_OK;
}

ns_status ns_pretrain_compute_step(ns_ctx* ctx, double* theta, double* adam_m, double* adam_v, int64_t t, double lr,
                                   const double* feats, const int32_t* off, const double* labels,
                                   const int32_t* batch, int32_t B, int32_t max_rows, double* loss_out) {
    if (!ctx) return NS_ERR_ARG;
    if (!theta || !adam_m || !adam_v || t < 1 || !feats || !off || !labels || !batch || B < 1 || max_rows < 1 ||
        max_rows > kPtRows)
        return set_err(ctx, NS_ERR_ARG, "ns_pretrain_compute_step: bad argument (1 <= max_rows <= 64)");
    for (const void* q : {(const void*)theta, (const void*)adam_m, (const void*)adam_v, (const void*)feats,
                          (const void*)off, (const void*)labels, (const void*)batch})
        if (!is_device_ptr(q)) return set_err(ctx, NS_ERR_ARG, "ns_pretrain_*: pointers must be device memory");
    if (loss_out && !is_device_ptr(loss_out)) return set_err(ctx, NS_ERR_ARG, "loss_out must be device memory");
    cudaSetDevice(ctx->device);
    constexpr int P = 7073;
    const int spb = std::max(1, std::min(16, kPtRows / max_rows));
    const int nblk = (B + spb - 1) / spb;
    const size_t need = ((size_t)nblk * P + nblk + 64) * sizeof(double);
    double* part = (double*)arena_get(ctx, need);
    if (!part) return arena_error(ctx, "pretrain", need);
    double* loss_part = part + (size_t)nblk * P;
    const size_t smem = ((size_t)kPtRows * (5 + 128 + 32) + 16 * (32 + 64 + 64 + 32) + 16 + 640 + 128 + 2 * 4096 + 32 +
                         2 * 2048 + 64 + 64 + 2) * sizeof(double) + kPtRows * sizeof(int);
    // (per call: the attribute is per device, a process may drive several)
    cudaFuncSetAttribute(k_pt_compute_grad, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    prof_begin(ctx, PK_OTHER);
    k_pt_compute_grad<<<nblk, 256, smem, ctx->stream>>>(theta, feats, off, batch, labels, B, spb, part, loss_part);
    prof_end(ctx);
    NS_LAUNCHED(ctx);
    return pt_adam(ctx, part, nblk, P, theta, adam_m, adam_v, t, lr, loss_part, loss_out);
}

ns_status ns_pretrain_comm_step(ns_ctx* ctx, int32_t D, double* theta, double* adam_m, double* adam_v, int64_t t,
                                double lr, const double* x, const double* y, const int32_t* batch, int32_t B,
                                double* loss_out) {
    if (!ctx) return NS_ERR_ARG;
    if (D < 1 || D > kMaxD || !theta || !adam_m || !adam_v || t < 1 || !x || !y || !batch || B < 1)
        return set_err(ctx, NS_ERR_ARG, "ns_pretrain_comm_step: bad argument");
    for (const void* q : {(const void*)theta, (const void*)adam_m, (const void*)adam_v, (const void*)x,
                          (const void*)y, (const void*)batch})
        if (!is_device_ptr(q)) return set_err(ctx, NS_ERR_ARG, "ns_pretrain_*: pointers must be device memory");
    if (loss_out && !is_device_ptr(loss_out)) return set_err(ctx, NS_ERR_ARG, "loss_out must be device memory");
    cudaSetDevice(ctx->device);
    const int w[6] = {2 * D, 128, 64, 32, 16, D};
    int P = 0;
    for (int l = 0; l < 5; ++l) P += w[l] * w[l + 1] + w[l + 1];
    const int nblk = (B + kPtCommSpb - 1) / kPtCommSpb;
    const size_t need = ((size_t)nblk * P + nblk + 64) * sizeof(double);
    double* part = (double*)arena_get(ctx, need);
    if (!part) return arena_error(ctx, "pretrain", need);
    double* loss_part = part + (size_t)nblk * P;
    const size_t smem = comm_smem(D);
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_pt_comm_grad, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    prof_begin(ctx, PK_OTHER);
    k_pt_comm_grad<<<nblk, 256, smem, ctx->stream>>>(theta, D, x, y, batch, B, part, loss_part);
    prof_end(ctx);
    NS_LAUNCHED(ctx);
    return pt_adam(ctx, part, nblk, P, theta, adam_m, adam_v, t, lr, loss_part, loss_out);
}

}  // extern "C"
