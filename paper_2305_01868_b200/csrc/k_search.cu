// k_search.cu -- the search hot path: kernels N3 (level candidates / column
// plans), order, N4 (greedy placement), N5 (finalize: plan cost), N6 (grid
// argmin, beam top-K, global best), and the host drivers for
// ns_shard_tablewise (Alg. 2) and ns_shard_columnwise (Alg. 1 + Alg. 2).
//
// Everything runs on the device; the host only enqueues a fixed sequence of
// launches (5 per beam level) without synchronising, then copies results.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <algorithm>
#include <cstdlib>
#include <climits>
#include <cmath>
#include <cstring>
#include <vector>

#include "ns_device.cuh"
#include "ns_internal.cuh"

#ifndef NS_WGRP_CTAS
#define NS_WGRP_CTAS 4   // resident CTAs per SM of k_greedy_wgrp88 (launch bounds and persistent grid; 128 registers with spills: 2 -> 3 -> 4 each +1-2% at 1024-1536 C5 tasks, 5 slower)
#endif
#ifndef NS_MERGE_THREADS
#define NS_MERGE_THREADS 256   // threads per column plan of k_merge_order (its rank-sort fallback included; 512: 2.04 vs 1.58 ms per step)
#endif
#ifndef NS_SELECT_THREADS
#define NS_SELECT_THREADS 256   // threads per task of k_select
#endif
#ifndef NS_EXPAND_THREADS
#define NS_EXPAND_THREADS 128   // threads per (task, beam) of k_expand (256: 3.08 vs 2.00 ms per 1536-task step)
#endif
#ifndef NS_EXPAND_COUNT_MAX
#define NS_EXPAND_COUNT_MAX 256   // k_expand: lists up to this length select candidates by rank counting
#endif
#ifndef NS_WGRP_MIN_CP
#define NS_WGRP_MIN_CP 148   // column plans per launch from which large D uses the grouped kernel
#endif

namespace ns {

struct WgrpQueue;   // k_greedy_wgrp88 work queue counters
struct P2Hdr;       // phase-2 item header (k_greedy_p2)

// ======================================================================
// Device buffers of one search call (carved from the ctx arena).
// "cp" = column-plan slot (one GreedyGridSearch call of Alg. 1 line 11);
// "traj" = (cp, grid point m), the unit of data parallelism.
// ======================================================================
struct SearchBufs {
    int n_tasks, D, M, K, N2, Lcap, Tpm, S, n_traj;
    long long n_rows_lin;   // variant rows bound (n_tasks * T_max * kDepth): Brow capacity
    uint32_t greedy_mode;   // NS_GREEDY_*
    // per cp
    int32_t* cp_task;
    int32_t* cp_valid;
    int32_t* cp_len;
    int32_t* cp_plan;    // [S][Lcap]
    int32_t* cp_Tp;
    double* vmin;        // [n_tasks][64] smallest v_k over the task's variant rows (linear-regime certificate)
    double* Brow;        // [rows] sum_k H2_k v_rk (k_task_lin)
    int ord_b, ord_e;    // column plans whose cost order this rank builds (its greedy block; others get cp_Tp only)
    int prev_b, prev_e;  // the previous level's ord_b / ord_e (k_merge_order: parents this rank ordered)
    int32_t* ord_row2;   // the previous level's cost orders (swapped with ord_row / ord_meta per level)
    int4* ord_meta2;
    int32_t* beam_slot;  // [n_tasks][K] slot (previous level's numbering) of each beam
    int32_t* ord_row;    // [S][Tpm]  variant row of the p-th table in cost order
    int4* ord_meta;      // [S][Tpm]  {dim, list index, bytes lo, bytes hi} of the p-th table (grouped greedy stream)
    // per traj
    int8_t* assign;      // [n_traj][Tpm]
    double* comp;        // [n_traj][D]
    int32_t* devdim;     // [n_traj][D]
    uint8_t* feas;       // [n_traj]
    uint32_t* work;      // [n_traj]
    double* tcost;       // [n_traj]
    int32_t* dup_of;     // [n_traj] grouped greedy: tau whose plan this one duplicates, or -1
    int32_t* uniq;       // [n_traj] compacted list of trajectories carrying a distinct feasible plan
    int32_t* n_uniq;     // [1]
    unsigned int* next_cp;   // [1] grouped-greedy work queue
    double* wsnap;       // large-D grouped greedy (k_greedy_wgrp88): fork snapshots [S * M][wsnap_doubles]
    bool wgrp;           // k_greedy_wgrp88 buffers carved
    size_t wsnap_doubles;   // per slot
    WgrpQueue* wq;
    int wgrp_cp_cap;     // column plans per launch the item buffers hold (a rank's block)
    int32_t* witem_cp;   // [S * M] fork items
    int32_t* witem_step;
    unsigned long long* witem_mask;
    int32_t* witem_ready;
    // phase 2 of the large-D grouped greedy (k_greedy_p2):
    // items handed over by k_greedy_wgrp88 once every device holds the
    // linear certificate, plus the forks phase 2 makes; frozen u of the
    // hand-offs; representatives whose u is replayed (k_greedy_replay)
    int p2_cap, uf_cap, rp_ctas;
    P2Hdr* p2_hdr;       // [p2_cap]
    uint32_t* p2_work;   // [p2_cap][64] work of each member so far
    double* p2_A;        // [p2_cap][128] per-device A_d
    long long* p2_room;  // [p2_cap][128] per-device memory headroom
    int32_t* p2_dsum;    // [p2_cap][128] per-device dim sum
    int32_t* p2_ready;   // [p2_cap] publication flags of phase-2 forks
    unsigned int* p2_q;  // [8] counters: next, forks, completed, n_init, uf used, replay entries
    double* uf_buf;      // [uf_cap][64][128] frozen u of the hand-offs
    int32_t* rp_ord;     // [p2_cap] replay order of the families (roots bucketed by column plan, k_rp_sort)
    int32_t* p2_first;   // [p2_cap] first fork of an item (-1: none), forks in step order
    int32_t* p2_next;    // [p2_cap] next fork of the same parent (-1: last)
    int32_t* p2_rtau;    // [p2_cap] an item's final representative (local tau)
    uint8_t* p2_alive;   // [p2_cap] 1: the item ended feasible (its representative needs comp)
    double* rp_snap;     // [replay CTAs][M][128][64] DFS snapshots of u at fork steps
    double* gscratch;    // grouped greedy group states
    int8_t* ghist;       // grouped greedy group histories [gscratch_warps][M][Tpm]
    int gscratch_warps;
    // per task
    int32_t* capdim;     // [n_tasks][M]
    int32_t* beam_plan;  // [n_tasks][K][Lcap]
    int32_t* beam_cnt;   // [n_tasks]
    double* best_cost;   // [n_tasks]
    int32_t* best_m;
    int32_t* best_ncol;
    int32_t* best_plan;  // [n_tasks][Lcap]
    int8_t* best_assign; // [n_tasks][Tpm]
    uint64_t* n_scores;  // [n_tasks]
    uint64_t* rank_keys; // [n_tasks][4] multi-rank consistency keys
    // column plans [own_cb, own_ce) of the current level were computed by this
    // rank (all of them with one rank or emulated ranks): only their
    // assignment rows are valid here (multi-rank: the others are not exchanged)
    int own_cb, own_ce;
    int r14;             // NS_R14_SPLITTABLE: rank only splittable tables as candidates
};

struct TaskView {   // read-only table arrays of the batch
    const int32_t* off;
    const int64_t* cap;
    const double* V;
    const double* C;
    const int32_t* vdim;
    const int64_t* vbytes;
};

// ---------------------------------------------------------------- helpers
// Post-split table list of a column plan: entry i is a variant row
// (table g, depth j) = g * kDepth + j.  The first half stays at c_i, the
// second is appended.  Every kernel that needs the list builds it in shared
// memory: rows in parallel, then the splits in plan order by one thread.

// ======================================================================
// Level setup kernels
// ======================================================================
__global__ void k_setup_level0(SearchBufs b) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= b.n_tasks) return;
    b.cp_task[q] = q;
    b.cp_valid[q] = 1;
    b.cp_len[q] = 0;
    b.best_cost[q] = CUDART_INF;
    b.best_m[q] = -1;
    b.best_ncol[q] = 0;
    b.n_scores[q] = 0;
    b.beam_cnt[q] = 0;
}

// N3: candidates of every beam plan (Alg. 1 line 8; reading
// R14): top-N by single-table cost (-C, index) then top-N by bytes
// (-bytes, index) not already listed, minus tables with dim % 8 != 0.  Child
// column plans = parent + [candidate], generation index (beam rank b,
// candidate rank j) -> slot (q*K + b)*2N + j.
__global__ void k_expand(SearchBufs b, TaskView tv, int level) {
    extern __shared__ int32_t sh[];
    const int q = blockIdx.x / b.K, bb = blockIdx.x % b.K;
    const int slot0 = (q * b.K + bb) * b.N2;
    const int plen = level - 1;
    const int T = tv.off[q + 1] - tv.off[q];
    const int Tp = T + plen;
    double* keyc = (double*)sh;                         // [Tpm] single cost of entry i
    long long* keyb = (long long*)(keyc + b.Tpm);       // [Tpm] bytes of entry i
    int32_t* rows = (int32_t*)(keyb + b.Tpm);           // [Tpm]
    int32_t* selc = rows + b.Tpm;       // [N] by cost rank -> index
    int32_t* sels = selc + b.N2;        // [N] by size rank -> index
    __shared__ int ncand;
    if (bb >= b.beam_cnt[q]) {
        for (int j = threadIdx.x; j < b.N2; j += blockDim.x) b.cp_valid[slot0 + j] = 0;
        return;
    }
    const int32_t* pplan = b.beam_plan + ((size_t)q * b.K + bb) * b.Lcap;
    {   // post-split table list, built in parallel then split in order
        const int base = tv.off[q];
        for (int i = threadIdx.x; i < T; i += blockDim.x) rows[i] = (base + i) * kDepth;
        __syncthreads();
        if (threadIdx.x == 0)
            for (int k = 0; k < plen; ++k) {
                const int c = pplan[k];
                rows[c] += 1;
                rows[T + k] = rows[c];
            }
    }
    const int N = b.N2 / 2;
    for (int j = threadIdx.x; j < b.N2; j += blockDim.x) selc[j] = sels[j] = -1;
    __syncthreads();
    for (int i = threadIdx.x; i < Tp; i += blockDim.x) {
        keyc[i] = tv.C[rows[i]];
        keyb[i] = tv.vbytes[rows[i]];
        if (b.r14 && (tv.vdim[rows[i]] % 8 != 0 || rows[i] % kDepth >= kDepth - 1)) {
            keyc[i] = -CUDART_INF;   // R14 alternative: unsplittable tables rank last
            keyb[i] = LLONG_MIN;     // (and are dropped by the filter below)
        }
    }
    __syncthreads();
    if (Tp <= NS_EXPAND_COUNT_MAX) {
        // short lists: ranks by counting, stopped once both reach N
        for (int i = threadIdx.x; i < Tp; i += blockDim.x) {
            const double ci = keyc[i];
            const long long bi = keyb[i];
            int rc = 0, rs = 0;
            for (int k = 0; k < Tp && (rc < N || rs < N); ++k) {
                const double ck = keyc[k];
                const long long bk = keyb[k];
                rc += (ck > ci) || (ck == ci && k < i);
                rs += (bk > bi) || (bk == bi && k < i);
            }
            if (rc < N) selc[rc] = i;
            if (rs < N) sels[rs] = i;
        }
        __syncthreads();
    }
    // long lists -- top-N by cost and top-N by bytes: N rounds of a block-wide
    // argmax; round r takes the largest entry below round r-1's pick in the
    // total order (key descending, list index ascending), nothing is marked
    __shared__ double s_kc[32];
    __shared__ long long s_kb[32];
    __shared__ int s_ic[32], s_ib[32];
    double pc = CUDART_INF;   // previous picks (+inf / INT_MIN: nothing picked yet)
    long long pb = LLONG_MAX;
    int pic = -1, pib = -1;
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    for (int r = 0; r < (Tp > NS_EXPAND_COUNT_MAX ? N : 0); ++r) {
        double bc = -CUDART_INF;
        long long bbv = LLONG_MIN;
        int ic = -1, ib = -1;
        for (int i = threadIdx.x; i < Tp; i += blockDim.x) {
            const double ci = keyc[i];
            const long long bi = keyb[i];
            // eligible: strictly after the previous pick in (key desc, index asc)
            const bool ec = ci < pc || (ci == pc && i > pic);
            const bool eb = bi < pb || (bi == pb && i > pib);
            if (ec && (ic < 0 || ci > bc || (ci == bc && i < ic))) {
                bc = ci;
                ic = i;
            }
            if (eb && (ib < 0 || bi > bbv || (bi == bbv && i < ib))) {
                bbv = bi;
                ib = i;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double oc = __shfl_xor_sync(kFull, bc, o);
            const int oic = __shfl_xor_sync(kFull, ic, o);
            const long long ob = __shfl_xor_sync(kFull, bbv, o);
            const int oib = __shfl_xor_sync(kFull, ib, o);
            if (oic >= 0 && (ic < 0 || oc > bc || (oc == bc && oic < ic))) {
                bc = oc;
                ic = oic;
            }
            if (oib >= 0 && (ib < 0 || ob > bbv || (ob == bbv && oib < ib))) {
                bbv = ob;
                ib = oib;
            }
        }
        if (lane == 0) {
            s_kc[wi] = bc;
            s_ic[wi] = ic;
            s_kb[wi] = bbv;
            s_ib[wi] = ib;
        }
        __syncthreads();
        bc = -CUDART_INF;
        bbv = LLONG_MIN;
        ic = ib = -1;
        for (int k = 0; k < nwarp; ++k) {   // every thread reduces the warp winners (same order)
            if (s_ic[k] >= 0 && (ic < 0 || s_kc[k] > bc || (s_kc[k] == bc && s_ic[k] < ic))) {
                bc = s_kc[k];
                ic = s_ic[k];
            }
            if (s_ib[k] >= 0 && (ib < 0 || s_kb[k] > bbv || (s_kb[k] == bbv && s_ib[k] < ib))) {
                bbv = s_kb[k];
                ib = s_ib[k];
            }
        }
        if (threadIdx.x == 0) {
            selc[r] = ic;
            sels[r] = ib;
        }
        pc = bc;
        pic = ic;
        pb = bbv;
        pib = ib;
        if (ic < 0) {   // fewer than N entries: later rounds select nothing
            pc = -CUDART_INF;
            pic = INT_MAX;
        }
        if (ib < 0) {
            pb = LLONG_MIN;
            pib = INT_MAX;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        int n = 0;
        int32_t* cand = sels + b.N2;    // [2N]
        for (int r = 0; r < N; ++r)
            if (selc[r] >= 0) cand[n++] = selc[r];
        const int nc = n;
        for (int r = 0; r < N; ++r) {
            const int i = sels[r];
            if (i < 0) continue;
            bool dup = false;
            for (int k = 0; k < nc; ++k) dup |= (cand[k] == i);
            if (!dup) cand[n++] = i;
        }
        int m = 0;
        for (int k = 0; k < n; ++k)
            if (tv.vdim[rows[cand[k]]] % 8 == 0 && rows[cand[k]] % kDepth < kDepth - 1) cand[m++] = cand[k];
        ncand = m;
    }
    __syncthreads();
    const int32_t* cand = sels + b.N2;
    for (int j = threadIdx.x; j < b.N2; j += blockDim.x) {
        const int g = slot0 + j;
        if (j < ncand) {
            b.cp_valid[g] = 1;
            b.cp_task[g] = q;
            b.cp_len[g] = level;
            int32_t* cpl = b.cp_plan + (size_t)g * b.Lcap;
            for (int k = 0; k < plen; ++k) cpl[k] = pplan[k];
            cpl[plen] = cand[j];
        } else {
            b.cp_valid[g] = 0;
        }
    }
}

// Alg. 2 lines 2-3: build the T' column-sharded tables and
// sort them by descending predicted single-table cost, ties by list index
// (reading R13): ascending order of the distinct keys (-C_i, i), fp64.  Long
// lists (T' > 256): one CTA per column plan, bitonic sort in shared memory
// over the next power of two (padding keys (+inf, INT_MAX) sort last).
__host__ __device__ inline int pow2_ceil(int x) {
    int n = 1;
    while (n < x) n <<= 1;
    return n;
}

// One 16-byte record per cost-order position: the grouped greedy stages it
// with a single copy instead of three gathers (dim, list index, bytes).
__device__ __forceinline__ int4 pack_meta(const TaskView& tv, int row, int i) {
    const unsigned long long by = (unsigned long long)tv.vbytes[row];
    return make_int4(tv.vdim[row], i, (int)(unsigned)(by & 0xffffffffull), (int)(unsigned)(by >> 32));
}

// The bitonic rank sort of column plan g (list of T + len entries) into
// ord_row / ord_meta (one CTA, shared memory as k_build_order sizes it).
__device__ void sort_order(const SearchBufs& b, const TaskView& tv, int g, int base, int T, int len,
                           unsigned char* bsm) {
    const int Tp = T + len;
    const int n = pow2_ceil(b.Tpm);
    double* key = (double*)bsm;              // [n]  -C
    int32_t* id = (int32_t*)(key + n);       // [n]  list index
    int32_t* rows = id + n;                  // [Tpm]
    for (int i = threadIdx.x; i < T; i += blockDim.x) rows[i] = (base + i) * kDepth;
    __syncthreads();
    if (threadIdx.x == 0) {
        const int32_t* plan = b.cp_plan + (size_t)g * b.Lcap;
        for (int k = 0; k < len; ++k) {   // halve c_k in place, append the other half
            const int c = plan[k];
            rows[c] += 1;
            rows[T + k] = rows[c];
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        key[i] = i < Tp ? -tv.C[rows[i]] : CUDART_INF;
        id[i] = i < Tp ? i : INT_MAX;
    }
    __syncthreads();
    for (int k = 2; k <= n; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const double ka = key[i], kb = key[ixj];
                    const int ia = id[i], ib = id[ixj];
                    const bool a_gt_b = ka > kb || (ka == kb && ia > ib);
                    if (((i & k) == 0) == a_gt_b) {   // ascending block: out of order if a > b
                        key[i] = kb;
                        key[ixj] = ka;
                        id[i] = ib;
                        id[ixj] = ia;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int r = threadIdx.x; r < Tp; r += blockDim.x) {
        const int i = id[r];
        b.ord_row[(size_t)g * b.Tpm + r] = rows[i];
        b.ord_meta[(size_t)g * b.Tpm + r] = pack_meta(tv, rows[i], i);
    }
}

__global__ void k_build_order(SearchBufs b, TaskView tv) {
    extern __shared__ __align__(16) unsigned char bsm[];
    const int g = blockIdx.x;
    if (!b.cp_valid[g]) return;
    const int q = b.cp_task[g];
    const int len = b.cp_len[g];
    const int base = tv.off[q], T = tv.off[q + 1] - base;
    if (threadIdx.x == 0) b.cp_Tp[g] = T + len;
    if (g < b.ord_b || g >= b.ord_e) return;   // another rank's greedy block (multi-rank)
    sort_order(b, tv, g, base, T, len, bsm);
}

// Beam levels, long lists: a child column plan is its parent's (a beam of the
// previous level, whose cost order that level built) plus one split c, so its
// order is the parent's with entry c removed and the two halves (-C_h, c) and
// (-C_h, T'_parent) merged in -- the same unique ascending order of the
// distinct keys (-C_i, i) the rank sort produces (reading R13), in one pass:
// parent entry r moves to r - [r > pos(c)] + [e1 < key_r] + [e2 < key_r], and
// e1 / e2 land after the entries below them.  The previous level's orders sit
// in ord_row2 / ord_meta2 (swapped per level); a parent another rank ordered
// (multi-rank block boundary) falls back to the rank sort.
__global__ void k_merge_order(SearchBufs b, TaskView tv, int level) {
    extern __shared__ __align__(16) unsigned char bsm[];
    __shared__ int s_pc, s_rowc, s_lt1, s_lt2;
    const int g = blockIdx.x;
    if (!b.cp_valid[g]) return;
    const int q = b.cp_task[g];
    const int len = b.cp_len[g];
    const int base = tv.off[q], T = tv.off[q + 1] - base;
    const int Tp = T + len, Tpp = Tp - 1;
    if (threadIdx.x == 0) b.cp_Tp[g] = Tp;
    if (g < b.ord_b || g >= b.ord_e) return;   // another rank's greedy block (multi-rank)
    const int bb = (g / b.N2) % b.K;
    const int gp = level == 1 ? q : b.beam_slot[q * b.K + bb];
    if (gp < b.prev_b || gp >= b.prev_e) {   // the parent's order lives on another rank
        sort_order(b, tv, g, base, T, len, bsm);
        return;
    }
    const int c = b.cp_plan[(size_t)g * b.Lcap + len - 1];
    const int32_t* prow = b.ord_row2 + (size_t)gp * b.Tpm;
    const int4* pmeta = b.ord_meta2 + (size_t)gp * b.Tpm;
    if (threadIdx.x == 0) {
        s_lt1 = 0;
        s_lt2 = 0;
    }
    for (int r = threadIdx.x; r < Tpp; r += blockDim.x)
        if (__ldg(&pmeta[r].y) == c) {
            s_pc = r;
            s_rowc = __ldg(prow + r);
        }
    __syncthreads();
    const int pc = s_pc, rowh = s_rowc + 1;   // both halves are the next variant row
    const double kh = -tv.C[rowh];
    int32_t* orow = b.ord_row + (size_t)g * b.Tpm;
    int4* ometa = b.ord_meta + (size_t)g * b.Tpm;
    int lt1 = 0, lt2 = 0;
    for (int r = threadIdx.x; r < Tpp; r += blockDim.x) {
        if (r == pc) continue;
        const int row = __ldg(prow + r);
        const int4 m = __ldg(pmeta + r);
        const double kr = -tv.C[row];
        const bool b1 = kh < kr || (kh == kr && c < m.y);   // e1 = (-C_h, c) sorts before entry r
        const bool b2 = kh < kr;                            // e2 = (-C_h, Tpp): Tpp > every parent index
        const int np = r - (r > pc ? 1 : 0) + (b1 ? 1 : 0) + (b2 ? 1 : 0);
        orow[np] = row;
        ometa[np] = m;
        lt1 += b1 ? 0 : 1;
        lt2 += b2 ? 0 : 1;
    }
    atomicAdd(&s_lt1, lt1);
    atomicAdd(&s_lt2, lt2);
    __syncthreads();
    if (threadIdx.x == 0) {
        const int p1 = s_lt1, p2 = s_lt2 + 1;
        orow[p1] = rowh;
        ometa[p1] = pack_meta(tv, rowh, c);
        orow[p2] = rowh;
        ometa[p2] = pack_meta(tv, rowh, Tpp);
    }
}

// Warp-per-column-plan form of k_build_order for short lists (Tpm <= 256):
// same rank sort, no CTA-wide barriers.  At level 0 it also initialises the
// per-task search state (column plan [] of task q in slot q) and the task's
// M grid caps floor(max_dim_m) (Alg. 2 line 4; operation order of
// reading R8 with explicit IEEE roundings).
// hi < 0: NS_NO_DIM_CAP ("w/o greedy grid search", Table 3, reading
// R8b): no dimension threshold at all, only the memory cap constrains.
__device__ __forceinline__ int32_t grid_cap(long long sumdim, int D, int M, int m, double hi) {
    if (hi < 0.0) return 2000000000;
    const double Ms = __ddiv_rn((double)sumdim, (double)D);
    double md = Ms;
    if (M > 1) {
        const double Me = __dmul_rn(hi, Ms);
        const double step = __ddiv_rn(__dsub_rn(Me, Ms), (double)(M - 1));
        md = __dadd_rn(Ms, __dmul_rn((double)m, step));
    }
    const double f = floor(md);
    return f > 2.0e9 ? 2000000000 : (int32_t)f;
}

__global__ void __launch_bounds__(256) k_order_warp(SearchBufs b, TaskView tv, int n_cp, int level0,
                                                    const int64_t* sumdim, double hi) {
    extern __shared__ __align__(16) unsigned char wsm[];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const int ri = (b.Tpm + 1) & ~1;
    int32_t* rows = (int32_t*)(wsm + (size_t)wl * (ri * 4 + b.Tpm * 8));
    double* key = (double*)(rows + ri);
    for (int g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; g < n_cp; g += (gridDim.x * blockDim.x) >> 5) {
        if (level0) {
            if (lane == 0) {
                b.cp_task[g] = g;
                b.cp_valid[g] = 1;
                b.cp_len[g] = 0;
                b.best_cost[g] = CUDART_INF;
                b.best_m[g] = -1;
                b.best_ncol[g] = 0;
                b.n_scores[g] = 0;
                b.beam_cnt[g] = 0;
            }
            for (int m = lane; m < b.M; m += 32) b.capdim[g * b.M + m] = grid_cap(sumdim[g], b.D, b.M, m, hi);
        } else if (!b.cp_valid[g]) {
            continue;
        }
        const int q = level0 ? g : b.cp_task[g];
        const int len = level0 ? 0 : b.cp_len[g];
        const int base = tv.off[q], T = tv.off[q + 1] - base, Tp = T + len;
        for (int i = lane; i < T; i += 32) rows[i] = (base + i) * kDepth;
        __syncwarp();
        if (lane == 0) {
            const int32_t* plan = b.cp_plan + (size_t)g * b.Lcap;
            for (int k = 0; k < len; ++k) {   // halve c_k in place, append the other half
                const int c = plan[k];
                rows[c] += 1;
                rows[T + k] = rows[c];
            }
            b.cp_Tp[g] = Tp;
        }
        __syncwarp();
        if (g < b.ord_b || g >= b.ord_e) continue;   // another rank's greedy block (multi-rank)
        for (int i = lane; i < Tp; i += 32) key[i] = tv.C[rows[i]];
        __syncwarp();
        if (Tp <= 64) {
            // items lane and lane + 32 ranked in one pass over the keys (each
            // key load serves both comparisons; no second, mostly idle pass)
            const int i0 = lane, i1 = lane + 32;
            const double c0 = i0 < Tp ? key[i0] : 0.0, c1 = i1 < Tp ? key[i1] : 0.0;
            int r0 = 0, r1 = 0;
            for (int k = 0; k < Tp; ++k) {
                const double ck = key[k];
                r0 += (ck > c0) || (ck == c0 && k < i0);
                r1 += (ck > c1) || (ck == c1 && k < i1);
            }
            if (i0 < Tp) {
                b.ord_row[(size_t)g * b.Tpm + r0] = rows[i0];
                b.ord_meta[(size_t)g * b.Tpm + r0] = pack_meta(tv, rows[i0], i0);
            }
            if (i1 < Tp) {
                b.ord_row[(size_t)g * b.Tpm + r1] = rows[i1];
                b.ord_meta[(size_t)g * b.Tpm + r1] = pack_meta(tv, rows[i1], i1);
            }
        } else {
            for (int i = lane; i < Tp; i += 32) {
                const double ci = key[i];
                int r = 0;
                for (int k = 0; k < Tp; ++k) {
                    const double ck = key[k];
                    r += (ck > ci) || (ck == ci && k < i);
                }
                b.ord_row[(size_t)g * b.Tpm + r] = rows[i];
                b.ord_meta[(size_t)g * b.Tpm + r] = pack_meta(tv, rows[i], i);
            }
        }
        __syncwarp();
    }
}

// ======================================================================
// N4: greedy placement (Alg. 2 lines 6-20, PAPER.md:289 step 3) -- the hot loop.
//
// LPD lanes per (trajectory or group, device); each lane keeps FPL = 64/LPD
// features of the hoisted head pre-activation u_d = hb1 + sum_{t on d} v_t and
// of the head weights H2 in registers (fp64).  For table t (cost order) every
// feasible device scores C(S_d + {t}) = hb2 + H2 . ReLU(u_d + v_t) (reading
// R5: cost after insertion): each lane computes its partial dot product and a
// butterfly over the LPD lanes joins them.  A shuffle argmin picks d* (lowest
// d on ties, R13); the lanes of d* add their slice of v_t.  Feasible:
// bytes_d + bytes_t <= cap and dim_d + dim_t <= floor(max_dim_m) (R6, R7); no
// feasible device strands the trajectory (R9).
//
// Why several lanes per device: with all 64 features in one lane, u plus the
// 64 head weights exceed the register budget and the compiler spills the
// weights.  Three kernels share this scheme: k_greedy_cta (latency mode,
// every trajectory in its own lane segment), k_greedy_dedup (throughput mode,
// one warp per column plan, identical trajectories grouped) and k_greedy_wide88
// (D > 16: one trajectory per CTA, one thread per device).
// ======================================================================
struct GreedyArgs {
    int traj_begin, traj_end, M, D, Tpm;
    long long n_rows;
    const int32_t* cp_valid;
    const int32_t* cp_task;
    const int32_t* cp_Tp;
    const int32_t* ord_row;
    const int4* ord_meta;
    const int32_t* capdim;
    const int64_t* cap;
    const double* V;
    const int32_t* vdim;
    const int64_t* vbytes;
    const double* vmin;   // [n_tasks][64] (k_task_lin)
    const double* Brow;   // [rows] (k_task_lin)
    int8_t* assign;
    double* comp;
    int32_t* devdim;
    uint8_t* feas;
    uint32_t* work;
    unsigned long long* computed;   // ctx stats counter: scores the kernel evaluated
    HeadParams head;
};

// Features per lane FPL = 64 / LPD (LPD = lanes per device).
template <bool SMEM>
__device__ __forceinline__ double2 ld_v2(const double2* p) {
    if constexpr (SMEM) return *p;
    else return __ldg(p);
}

// Partial dot product sum_{k<FPL} w[k] ReLU(u[k] + v[k]) with (up to) 4
// accumulators, v streamed in chunks of (up to) 8 doubles.
template <int FPL, bool SMEM>
__device__ __forceinline__ double part_score(const double (&u)[FPL], const double (&w)[FPL],
                                             const double2* __restrict__ v2) {
    constexpr int CH = FPL < 8 ? FPL : 8;   // doubles per chunk
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int c = 0; c < FPL / CH; ++c) {
        double2 vv[CH / 2];
#pragma unroll
        for (int i = 0; i < CH / 2; ++i) vv[i] = ld_v2<SMEM>(v2 + c * (CH / 2) + i);
#pragma unroll
        for (int i = 0; i < CH / 2; ++i) {
            const int k = c * CH + 2 * i;
            acc[(2 * i) & 3] = fma(w[k], relu_hi(u[k] + vv[i].x), acc[(2 * i) & 3]);
            acc[(2 * i + 1) & 3] = fma(w[k + 1], relu_hi(u[k + 1] + vv[i].y), acc[(2 * i + 1) & 3]);
        }
    }
    return (acc[0] + acc[1]) + (acc[2] + acc[3]);
}

// u += v (only the chosen device's lanes execute it)
template <int FPL, bool SMEM>
__device__ __forceinline__ void part_add(double (&u)[FPL], const double2* __restrict__ v2) {
#pragma unroll
    for (int i = 0; i < FPL / 2; ++i) {
        const double2 vv = ld_v2<SMEM>(v2 + i);
        u[2 * i] += vv.x;
        u[2 * i + 1] += vv.y;
    }
}

template <int FPL>
__device__ __forceinline__ double part_head(const double (&u)[FPL], const double (&w)[FPL]) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int k = 0; k < FPL; ++k) acc[k & 3] = fma(w[k], relu_exact(u[k]), acc[k & 3]);
    return (acc[0] + acc[1]) + (acc[2] + acc[3]);
}

// Sum of the LPD partials of one device (xor butterfly; IEEE addition is
// commutative so every lane of the device holds the identical value).
template <int LPD>
__device__ __forceinline__ double lane_group_sum(double x) {
#pragma unroll
    for (int o = LPD / 2; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
    return x;
}

__device__ __forceinline__ void argmin_step(double& bs, int& bd, int o) {
    const double os = __shfl_xor_sync(kFull, bs, o);
    const int od = __shfl_xor_sync(kFull, bd, o);
    if (os < bs || (os == bs && od < bd)) {
        bs = os;
        bd = od;
    }
}

// Per-lane slice of hb1 (initial u) and H2 (head weights); the weights are
// made opaque so the compiler keeps them in registers instead of
// re-loading them from the constant bank with a lane-dependent address.
template <int FPL>
__device__ __forceinline__ void load_lane_head(const HeadParams& hp, int part, double (&u)[FPL], double (&w)[FPL]) {
#pragma unroll
    for (int k = 0; k < FPL; ++k) {
        double hu = hp.hb1[k], hw = hp.H2[k];
#pragma unroll
        for (int q = 1; q < kV / FPL; ++q)
            if (part == q) {
                hu = hp.hb1[q * FPL + k];
                hw = hp.H2[q * FPL + k];
            }
        u[k] = hu;
        w[k] = hw;
        asm volatile("" : "+d"(w[k]));
    }
}


// Staged greedy: one CTA per (column plan, chunk of grid points).  All
// trajectories of a column plan consume the same cost-ordered table stream,
// so the CTA stages the v rows (and dim / bytes / list index) of the next
// kRing tables into shared memory once and every lane reads its slice from
// there (broadcast within a segment; the LPD slices of a row are padded
// 16 B apart so they fall on different banks) instead of each warp walking
// the order and the rows through L1/L2.
#ifndef NS_REDUX_ARGMIN
#define NS_REDUX_ARGMIN 1   // greedy kernels (grouped fast path, per-warp latency kernel): device argmin by two 32-bit warp reductions of an order key
#endif
constexpr int kRing = 40;   // tables staged per chunk (C2: the whole task)

template <int SEG, int LPD>
__global__ void __launch_bounds__(256) k_greedy_cta(const GreedyArgs a, int mchunk, int nchunk) {
    constexpr int FPL = kV / LPD;
    constexpr int PSTR = FPL + 2;            // slice stride (doubles)
    constexpr int RSTR = LPD * PSTR;         // row stride (doubles)
    __shared__ __align__(16) double s_v[kRing * RSTR];
    __shared__ int s_dim[kRing];
    __shared__ long long s_bytes[kRing];
    __shared__ int s_idx[kRing];
    constexpr unsigned SEGMASK = SEG == 32 ? kFull : ((1u << SEG) - 1u);
    const int g = blockIdx.x / nchunk, chunk = blockIdx.x % nchunk;
    const int lane = threadIdx.x & 31;
    const int j = threadIdx.x / SEG;                      // local trajectory
    const int seg = lane / SEG;
    const int ls = threadIdx.x % SEG;
    const int d = ls / LPD, part = ls % LPD;
    const int m = chunk * mchunk + j;
    const long long tau = (long long)g * a.M + m;
    const bool in_range = j < mchunk && m < a.M && tau >= a.traj_begin && tau < a.traj_end;
    const bool valid = a.cp_valid[g] != 0;
    bool alive = in_range && valid;
    int Tp = 0, capd = 0;
    long long cap = 0;
    if (valid) {
        const int q = a.cp_task[g];
        Tp = a.cp_Tp[g];
        cap = a.cap[q];
        if (in_range) capd = a.capdim[q * a.M + m];
    }
    const bool dev = d < a.D;
    double u[FPL], w[FPL];
    load_lane_head<FPL>(a.head, part, u, w);
    int dsum = 0;
    long long bsum = 0;
    uint32_t work = 0;
    const int32_t* orow = a.ord_row + (size_t)g * a.Tpm;
    const int4* ometa = a.ord_meta + (size_t)g * a.Tpm;
    int8_t* asg = a.assign + (size_t)(in_range ? tau : 0) * a.Tpm;
    const int Tmax = valid ? Tp : 0;   // uniform over the CTA
    for (int p0 = 0; p0 < Tmax; p0 += kRing) {
        const int np = min(kRing, Tmax - p0);
        __syncthreads();   // previous chunk fully consumed
        for (int i = threadIdx.x; i < np * (kV / 2); i += blockDim.x) {
            const int r = i / (kV / 2), c2 = i % (kV / 2);
            const int row = __ldg(orow + p0 + r);
            const double2 v = __ldg(reinterpret_cast<const double2*>(a.V + (size_t)row * kV) + c2);
            const int k = 2 * c2;
            *reinterpret_cast<double2*>(s_v + r * RSTR + (k / FPL) * PSTR + (k % FPL)) = v;
        }
        for (int r = threadIdx.x; r < np; r += blockDim.x) {
            const int4 mt = __ldg(ometa + p0 + r);
            s_dim[r] = mt.x;
            s_bytes[r] = (long long)(((unsigned long long)(unsigned)mt.w << 32) | (unsigned)mt.z);
            s_idx[r] = mt.y;
        }
        __syncthreads();
#pragma unroll 1
        for (int r = 0; r < np; ++r) {
            const bool act = alive;   // p0 + r < Tp == Tmax
            const int dt = s_dim[r];
            const long long bt = s_bytes[r];
            const bool f = act && dev && (bsum + bt <= cap) && (dsum + dt <= capd);
            const double2* v2 = reinterpret_cast<const double2*>(s_v + r * RSTR + part * PSTR);
            double ps = 0.0;
            if (f) ps = part_score<FPL, true>(u, w, v2);
            double bs = a.head.hb2 + lane_group_sum<LPD>(ps);
            int bd = d;
            if constexpr (SEG == 32 && NS_REDUX_ARGMIN) {
                // one trajectory per warp: the grouped kernel's order-key
                // argmin (two REDUX; lowest device among equal scores)
                const long long sb = __double_as_longlong(bs + 0.0);
                const unsigned long long key =
                    f ? (unsigned long long)(sb ^ ((sb >> 63) | (long long)0x8000000000000000ULL)) : ~0ULL;
                const unsigned khi = (unsigned)(key >> 32), klo = (unsigned)key;
                const unsigned mhi = __reduce_min_sync(kFull, khi);
                const unsigned mlo = __reduce_min_sync(kFull, khi == mhi ? klo : 0xFFFFFFFFu);
                const unsigned hit = __ballot_sync(kFull, f && part == 0 && khi == mhi && klo == mlo);
                if (hit == 0u) bs = CUDART_INF;
                bd = (__ffs(hit) - 1) / LPD;
            } else {
                if (!f) bs = CUDART_INF;
#pragma unroll
                for (int o = SEG / 2; o >= LPD; o >>= 1) argmin_step(bs, bd, o);
            }
            const unsigned bal = __ballot_sync(kFull, f && part == 0);
            if (act) {
                work += __popc((bal >> (seg * SEG)) & SEGMASK);
                if (bs == CUDART_INF) alive = false;   // R9: stranded -> grid point infeasible
            }
            if (act && bs != CUDART_INF) {
                if (d == bd) {
                    part_add<FPL, true>(u, v2);
                    dsum += dt;
                    bsum += bt;
                }
                if (ls == 0) asg[s_idx[r]] = (int8_t)bd;
            }
        }
    }
    const double hc = a.head.hb2 + lane_group_sum<LPD>(part_head<FPL>(u, w));
    if (in_range) {
        if (dev && part == 0) {
            a.comp[tau * a.D + d] = dsum > 0 ? hc : 0.0;   // reading R4
            a.devdim[tau * a.D + d] = dsum;
        }
        if (ls == 0) {
            a.feas[tau] = alive ? 1 : 0;
            a.work[tau] = work;
        }
    }
}

// cp.async (LDGSTS) helpers: the grouped greedy streams the next kStages
// tables' v rows into a per-warp shared-memory ring so the HBM/L2 latency of
// the row fetch is hidden behind kStages - 1 steps of work.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

#ifndef NS_KSTAGES
#define NS_KSTAGES 8
#endif
constexpr int kStages = NS_KSTAGES;   // row-stream ring depth (large-D greedy)
#ifndef NS_DSTAGES
#define NS_DSTAGES 3
#endif
#ifndef NS_PAIR_STAGE
#define NS_PAIR_STAGE 2   // tables staged per cp.async group in the grouped greedy (0: one per step)
#endif
constexpr int kDStages = NS_PAIR_STAGE ? 2 * NS_PAIR_STAGE : NS_DSTAGES;   // row-stream ring depth of the grouped greedy
#ifndef NS_G1SM
#define NS_G1SM 1   // group 1 of the grouped greedy in shared memory (typed pass)
#endif

// ---------------------------------------------------------------------------
// Grouped greedy (used for D <= 16): one WARP per column plan, all M grid
// trajectories of that column plan handled together.
//
// The M grid points differ only in the max_dim cap, so their greedy
// runs coincide until a cap binds: trajectories with the same assignment
// history have the same device states and therefore the same candidate
// scores C(S_d + {t}); only their feasible sets differ (by the dim cap).  The
// kernel keeps one device state per GROUP of identical trajectories, scores
// the D devices once per group, and lets every member take its own argmin
// over its own feasible set; members that choose a different device than the
// group's lowest member split off into a new group (state copied before the
// update).  This is the data-parallel form of the paper's life-long cache
// ("if we only make small changes to ... max_dim, the cost model will be
// very likely to be asked to predict the cost for the same set of tables",
// PAPER.md:291): every score the algorithm asks for is answered -- the work
// count W (O12) counts each member's feasible devices -- but each distinct
// (state, table) score is computed once.  Results are identical to running
// the M trajectories separately (same arithmetic on the same state).
//
// Lane layout: lane = (device d, part) with LPD = 32 / pow2(D) lanes per
// device and FPL = 64 / LPD features per lane.  Group 0 (which holds the
// loosest caps and lives the longest) keeps its whole state in registers
// (pre-activations, per-device dim/bytes, cap range, uniform work); later
// groups live in a per-warp global scratch (L1/L2).  Member and group
// bookkeeping lives in shared memory with compile-time extents (MC >= M).
// Device choices are recorded once per GROUP and step (a per-group history
// by list index, plus the parent and step of each split); at the end the
// histories are completed in creation order and only each group's
// representative (its lowest live member) gets an assignment row, comp /
// devdim row and dup_of = -1 -- the other members point at it through dup_of
// (plan cost and selection read representatives only).
// ---------------------------------------------------------------------------
struct DedupArgs {
    long long tau_base;    // absolute trajectory index of the first column plan (dup_of holds absolute taus)
    int n_cp;              // column plans of this launch: [0, n_cp) relative to the GreedyArgs pointers
    int mmax;              // M (<= the kernel's MC)
    double* scratch;       // [total_warps][M][D][64] group states (groups >= 1)
    int8_t* hist;          // [total_warps][M][Tpm] per-group device choices by list index
    int total_warps;
    int32_t* dup_of;       // [n_traj] tau of the member whose plan this one duplicates, or -1
    unsigned int* next_cp; // dynamic queue counter (zeroed before the launch)
};

// Per-warp shared-memory bookkeeping of the grouped greedy.  Every array has
// a compile-time extent (MC >= M grid points), so each field is a constant
// offset from one base register.
template <int LPD, int MC>
struct __align__(16) DedupSmem {
    static constexpr int FPL = kV / LPD;
    static constexpr int DPW = 32 / LPD;      // device slots per warp
    static constexpr int SS = FPL * 8 + 16;   // ring slice stride (bytes): +16 B keeps the LPD
    static constexpr int RS = LPD * SS;       //   slices of a row on distinct banks
    unsigned char ring[kDStages][RS];          // staged v rows of the next tables
#if NS_G1SM
    double g1[32][FPL + 2];                   // group 1's state (per-lane slices, 16 B pad)
#endif
    long long gb[MC][DPW];                    // group memory headroom cap - bytes per device (groups >= 1)
    int4 meta[kDStages];                       // staged {dim, list index, bytes lo, bytes hi}
    double sc[DPW];                           // scores of the current group
    int gd[MC][DPW];                          // group dims per device (groups >= 1)
    int mgroup[MC];                           // member -> group (-1 stranded)
    int mcap[MC];                             // member dim cap
    int mpick[MC];
    int gcap[MC];                             // loosest cap among a group's live members
    int gmin[MC];                             // tightest cap among a group's live members
    int gpar[MC];                             // group it split from
    int gstep[MC];                            // step (cost-order position) of the split
    uint32_t mwork[MC];
    uint32_t gwork[MC];                       // work of the group's uniform steps
    int sdv[DPW];                             // dim after insertion
    int sok[DPW];                             // device scored
};

template <int LPD, int MC>
#ifndef NS_DEDUP_BLOCKS8
#define NS_DEDUP_BLOCKS8 5   // CTAs per SM for LPD >= 8 (D <= 4): 96 registers, no spills
#endif
#ifndef NS_DEDUP_WPB
#define NS_DEDUP_WPB 4   // warps (column plans in flight) per CTA
#endif
__global__ void __launch_bounds__(NS_DEDUP_WPB * 32, (LPD >= 8 ? NS_DEDUP_BLOCKS8 : (LPD == 4 ? 2 : 1))) k_greedy_dedup(const GreedyArgs a, const DedupArgs x) {
    using SM = DedupSmem<LPD, MC>;
    constexpr int FPL = SM::FPL, DPW = SM::DPW, SS = SM::SS;
    extern __shared__ __align__(16) unsigned char dsm[];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int M = x.mmax, D = a.D;
    const int d = lane / LPD, part = lane % LPD;
    const bool dev = d < D;
    SM& s = reinterpret_cast<SM*>(dsm)[wl];
    // this lane's 16-byte chunk of a staged v row (slot 0; + slot * RS)
    unsigned char* const ring_lane = &s.ring[0][(lane / (FPL / 2)) * SS + (lane % (FPL / 2)) * 16];
    // hb1 (the empty-device pre-activation) is re-read from shared memory at
    // every column plan instead of occupying FPL registers for the whole kernel
    __shared__ double s_hb1[kV];
    for (int k = threadIdx.x; k < kV; k += blockDim.x) s_hb1[k] = a.head.hb1[k];
    // head weights as per-part slices padded 16 B apart (the LPD slices of one
    // load fall on distinct banks): FPL fewer register pairs per lane
    __shared__ __align__(16) double s_wp[LPD][FPL + 2];
    for (int k = threadIdx.x; k < kV; k += blockDim.x) s_wp[k / FPL][k % FPL] = a.head.H2[k];
#define GW(k) s_wp[part][k]
    __syncthreads();
    double u0[FPL];
    const long long gw = (long long)blockIdx.x * nw + wl;
    double* scr = x.scratch + (size_t)gw * M * D * kV;   // this warp's group states
    // state slice of group gr >= 1 owned by this lane (its device, part)
    double* const scr_l = scr + (size_t)(dev ? d : 0) * kV + part * FPL;
    auto gptr = [&](int gr) -> double* { return scr_l + (size_t)gr * D * kV; };
#if NS_G1SM
    // group 1's state in shared memory (this lane's slice, padded 16 B apart)
    double* const g1_l = &s.g1[(dev ? d : 0) * LPD + part][0];
#endif
    int8_t* hist = x.hist + (size_t)gw * M * a.Tpm;       // this warp's group histories
    // dynamic column-plan queue (column plans differ in length and in how many
    // groups they split into; a static stride leaves a long tail)
    long long g = gw;
    for (; g < x.n_cp;) {
        const bool valid = a.cp_valid[g] != 0;
        const long long tau0 = g * M;
        if (!valid) {
#pragma unroll
            for (int m0 = 0; m0 < MC; m0 += 32) {
                const int m = m0 + lane;
                if (m < M) {
                    a.feas[tau0 + m] = 0;
                    a.work[tau0 + m] = 0;
                    x.dup_of[tau0 + m] = -1;
                }
            }
            long long nx = 0;
            if (lane == 0) nx = x.total_warps + (long long)atomicAdd(x.next_cp, 1u);
            g = __shfl_sync(kFull, nx, 0);
            continue;
        }
        const int q = a.cp_task[g];
        const int Tp = a.cp_Tp[g];
        const long long cap = a.cap[q];
        // group 0 (all members at the start; keeps the loosest-cap members)
        // lives in registers: per-device dim / bytes in the device's lanes,
        // cap range and uniform work warp-uniform
        int cmax = 0, cmin = INT_MAX;
#pragma unroll
        for (int m0 = 0; m0 < MC; m0 += 32) {
            const int m = m0 + lane;
            if (m < M) {
                const int c = a.capdim[q * M + m];
                s.mgroup[m] = 0;
                s.mcap[m] = c;
                s.mwork[m] = 0;
                cmax = max(cmax, c);
                cmin = min(cmin, c);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            cmax = max(cmax, __shfl_xor_sync(kFull, cmax, o));
            cmin = min(cmin, __shfl_xor_sync(kFull, cmin, o));
        }
        int r_dsum = 0, r_gcap = cmax, r_gmin = cmin;
        long long r_bhr = cap;   // group 0: per-device memory headroom cap - bytes_d (this lane's device)
        uint32_t r_gwork = 0;
#pragma unroll
        for (int k = 0; k < FPL; ++k) u0[k] = s_hb1[part * FPL + k];
        int ng = 1;
        __syncwarp();
        const int32_t* orow = a.ord_row + (size_t)g * a.Tpm;
        const int4* ometa = a.ord_meta + (size_t)g * a.Tpm;
        // row-index window: the next 32 entries of the cost order in one register per lane
        int oc_cur = lane < Tp ? __ldg(orow + lane) : 0;
        int oc_nxt = 32 + lane < Tp ? __ldg(orow + 32 + lane) : 0;
#if !NS_PAIR_STAGE
        // ring slots rotate with counters (no modulo): table pp goes to slot
        // pp % kDStages == sl_w at its issue
        int sl_w = 0;
        auto issue = [&](int pp) {   // stage table pp of the cost order into ring slot sl_w
            if (pp < Tp) {
                if (pp > 0 && (pp & 31) == 0) {
                    oc_cur = oc_nxt;
                    oc_nxt = pp + 32 + lane < Tp ? __ldg(orow + pp + 32 + lane) : 0;
                }
                const int r = __shfl_sync(kFull, oc_cur, pp & 31);
                cp_async16(ring_lane + sl_w * SM::RS, a.V + (size_t)r * kV + 2 * lane);
                if (lane == 0) cp_async16(&s.meta[sl_w], ometa + pp);
            }
            cp_async_commit();   // one group per step, empty past the end
            sl_w = sl_w + 1 == kDStages ? 0 : sl_w + 1;
        };
#else
        // group staging: G = NS_PAIR_STAGE consecutive tables of the cost order
        // go into slots pp % 2G as ONE cp.async group, issued every G-th step
        // (1/G of the issue / wait / warp-sync overhead per step); the ring
        // holds the G tables in use and the G in flight
        constexpr int G = NS_PAIR_STAGE;
        auto stage1 = [&](int pp) {
            if (pp < Tp) {
                if (pp > 0 && (pp & 31) == 0) {
                    oc_cur = oc_nxt;
                    oc_nxt = pp + 32 + lane < Tp ? __ldg(orow + pp + 32 + lane) : 0;
                }
                const int r = __shfl_sync(kFull, oc_cur, pp & 31);
                cp_async16(ring_lane + (pp % (2 * G)) * SM::RS, a.V + (size_t)r * kV + 2 * lane);
                if (lane == 0) cp_async16(&s.meta[pp % (2 * G)], ometa + pp);
            }
        };
#endif
        // one group's pass over table t (G0: group 0, register-resident state)
        auto pass = [&](auto g0tag, const int gr, const auto& vcd, const int dt, const long long bt, const int idx,
                        const int p) {
            constexpr int KIND = decltype(g0tag)::value;   // 0: group 0, 1: group 1 (smem), 2: others
            constexpr bool G0 = KIND == 0;
            // ---- score the D devices once for the whole group (R5: after insertion)
            const int gcap_gr = G0 ? r_gcap : s.gcap[gr];
            if (gcap_gr < 0) return;   // group without live members
            const int dsum = G0 ? r_dsum : (dev ? s.gd[gr][d] : 0);
            const long long bhr = G0 ? r_bhr : (dev ? s.gb[gr][d] : 0);   // memory headroom
            const bool f = dev && (bt <= bhr) && (dsum + dt <= gcap_gr);
#if NS_G1SM
            double* ug = KIND == 1 ? g1_l : gptr(gr);   // valid for gr >= 1
#else
            double* ug = gptr(gr);   // valid for gr >= 1
#endif
            double ps = 0.0;
            if (f) {
                double acc[4] = {0.0, 0.0, 0.0, 0.0};
                if (G0) {
#pragma unroll
                    for (int k = 0; k < FPL; ++k) acc[k & 3] = fma(GW(k), relu_hi(u0[k] + vcd[k]), acc[k & 3]);
                } else {
#pragma unroll
                    for (int k = 0; k < FPL; ++k) acc[k & 3] = fma(GW(k), relu_hi(ug[k] + vcd[k]), acc[k & 3]);
                }
                ps = (acc[0] + acc[1]) + (acc[2] + acc[3]);
            }
            const double sco = a.head.hb2 + lane_group_sum<LPD>(ps);
            const int gmin_gr = G0 ? r_gmin : s.gmin[gr];
            // ---- fast path: every live member's cap admits every scored
            //      device -> all members see the same feasible set and take
            //      the group argmin (no split, uniform work)
            {
                // (one warp vote: every scored device fits the tightest member cap)
                if (__all_sync(kFull, !f || dsum + dt <= gmin_gr)) {
                    // device argmin: butterfly minimum, then the lowest device
                    // attaining it (R13) from one ballot
#if NS_REDUX_ARGMIN
                    // order key of the score (unsigned compare == double
                    // compare for non-NaN values; + 0.0 folds -0.0 into +0.0
                    // so equal scores keep equal keys); infeasible = all ones.
                    // min over the warp = high-word min, then low-word min
                    // among the lanes holding it (two REDUX, no 64-bit shuffles)
                    const long long sb = __double_as_longlong(sco + 0.0);
                    const unsigned long long key =
                        f ? (unsigned long long)(sb ^ ((sb >> 63) | (long long)0x8000000000000000ULL)) : ~0ULL;
                    const unsigned khi = (unsigned)(key >> 32), klo = (unsigned)key;
                    const unsigned mhi = __reduce_min_sync(kFull, khi);
                    const unsigned mlo = __reduce_min_sync(kFull, khi == mhi ? klo : 0xFFFFFFFFu);
                    const unsigned nf = __popc(__ballot_sync(kFull, f && part == 0));
                    const unsigned hit = __ballot_sync(kFull, f && part == 0 && khi == mhi && klo == mlo);
                    const int bd = (__ffs(hit) - 1) / LPD;
                    if (hit == 0u) {   // nothing feasible: the whole group strands (R9)
#else
                    const double own = f ? sco : CUDART_INF;
                    double bs = own;
#pragma unroll
                    for (int o = 16; o >= LPD; o >>= 1) {
                        // plain select (scores are never NaN): no fmin NaN fix-ups
                        const double ob = __shfl_xor_sync(kFull, bs, o);
                        bs = ob < bs ? ob : bs;
                    }
                    const unsigned nf = __popc(__ballot_sync(kFull, f && part == 0));
                    const unsigned hit = __ballot_sync(kFull, f && part == 0 && own == bs);
                    const int bd = (__ffs(hit) - 1) / LPD;
                    if (bs == CUDART_INF) {   // nothing feasible: the whole group strands (R9)
#endif
                        const uint32_t gwk = G0 ? r_gwork : s.gwork[gr];
#pragma unroll
                        for (int m0 = 0; m0 < MC; m0 += 32) {
                            const int m = m0 + lane;
                            if (m < M && s.mgroup[m] == gr) {
                                s.mwork[m] += gwk;
                                s.mgroup[m] = -1;
                            }
                        }
                        if (G0) r_gcap = -1;
                        __syncwarp();
                        if (!G0 && lane == 0) s.gcap[gr] = -1;
                        __syncwarp();
                        return;
                    }
                    if (d == bd) {
                        if (G0) {
#pragma unroll
                            for (int k = 0; k < FPL; ++k) u0[k] += vcd[k];
                        } else {
#pragma unroll
                            for (int k = 0; k < FPL; ++k) ug[k] += vcd[k];
                        }
                    }
                    if (lane == 0) hist[(size_t)gr * a.Tpm + idx] = (int8_t)bd;
                    if (G0) {
                        if (d == bd) {
                            r_dsum += dt;
                            r_bhr -= bt;
                        }
                        r_gwork += nf;
                    } else {
                        if (lane == 0) {
                            s.gd[gr][bd] += dt;
                            s.gb[gr][bd] -= bt;
                            s.gwork[gr] += nf;
                        }
                        __syncwarp();
                    }
                    return;
                }
            }
            if (part == 0 && d < DPW) {
                s.sc[d] = sco;
                s.sdv[d] = dsum + dt;
                s.sok[d] = f ? 1 : 0;
            }
            __syncwarp();
            // ---- every member takes its own argmin over its own feasible set
            //      (dim cap of its grid point; lowest device on ties, R13)
            const uint32_t gwk = G0 ? r_gwork : s.gwork[gr];
            int first = M;
            bool left = false;
#pragma unroll
            for (int m0 = 0; m0 < MC; m0 += 32) {
                const int m = m0 + lane;
                int pick = -2;
                if (m < M && s.mgroup[m] == gr) {
                    double best = CUDART_INF;
                    int bd = -1;
                    uint32_t cnt = 0;
                    const int cm = s.mcap[m];
#pragma unroll
                    for (int dd = 0; dd < DPW; ++dd) {   // DPW >= D device slots, unrolled
                        if (dd < D && s.sok[dd] && s.sdv[dd] <= cm) {
                            ++cnt;
                            const double sv = s.sc[dd];
                            if (sv < best) {
                                best = sv;
                                bd = dd;
                            }
                        }
                    }
                    s.mwork[m] += cnt;
                    if (bd < 0) {
                        s.mwork[m] += gwk;
                        s.mgroup[m] = -1;   // R9: stranded -> grid point infeasible
                        pick = -1;
                    } else {
                        pick = bd;
                    }
                }
                if (m < M) s.mpick[m] = pick;
                const unsigned live = __ballot_sync(kFull, pick >= 0);
                left |= __any_sync(kFull, pick == -1);
                // the group keeps the pick of its LOOSEST-cap live member (highest m):
                // tight caps bind first, so the splitting members are the few
                // tight ones and the majority stays in the register-resident group
                if (live) first = m0 + 31 - __clz(live);
            }
            __syncwarp();
            if (first == M) {   // every member stranded
                if (G0) r_gcap = -1;
                else if (lane == 0) s.gcap[gr] = -1;
                __syncwarp();
                return;
            }
            const int main_pick = s.mpick[first];
            bool split = false;
#pragma unroll
            for (int m0 = 0; m0 < MC; m0 += 32) {
                const int m = m0 + lane;
                split |= __any_sync(kFull, m < M && s.mpick[m] >= 0 && s.mpick[m] != main_pick);
            }
            // ---- members choosing another device split off (state before the update)
            if (split) {
                for (int dd = 0; dd < D; ++dd) {
                    if (dd == main_pick) continue;
                    int any = 0, c2 = -1, c2min = INT_MAX;
#pragma unroll
                    for (int m0 = 0; m0 < MC; m0 += 32) {
                        const int m = m0 + lane;
                        const bool mine = m < M && s.mpick[m] == dd;
                        if (mine) {
                            s.mgroup[m] = ng;
                            s.mwork[m] += gwk;   // bank the old group's uniform work
                            c2 = max(c2, s.mcap[m]);
                            c2min = min(c2min, s.mcap[m]);
                        }
                        any |= __any_sync(kFull, mine);
                    }
                    if (!any) continue;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        c2 = max(c2, __shfl_xor_sync(kFull, c2, o));
                        c2min = min(c2min, __shfl_xor_sync(kFull, c2min, o));
                    }
                    // new group ng = state(gr) + v_t on device dd
                    if (dev) {
#if NS_G1SM
                        if (ng == 1) {
#pragma unroll
                            for (int k = 0; k < FPL; ++k) {
                                double val = G0 ? u0[k] : ug[k];
                                if (d == dd) val += vcd[k];
                                g1_l[k] = val;
                            }
                        } else
#endif
                        {
                            double* un = gptr(ng);
#pragma unroll
                            for (int k = 0; k < FPL; ++k) {
                                double val = G0 ? u0[k] : ug[k];
                                if (d == dd) val += vcd[k];
                                un[k] = val;
                            }
                        }
                        if (part == 0) {
                            s.gd[ng][d] = dsum + (d == dd ? dt : 0);
                            s.gb[ng][d] = bhr - (d == dd ? bt : 0);
                        }
                    }
                    if (lane == 0) {
                        s.gcap[ng] = c2;
                        s.gmin[ng] = c2min;
                        s.gwork[ng] = 0;
                        s.gpar[ng] = gr;
                        s.gstep[ng] = p;
                        hist[(size_t)ng * a.Tpm + idx] = (int8_t)dd;
                    }
                    ++ng;
                    __syncwarp();
                }
            }
            // ---- the group itself takes main_pick
            if (d == main_pick) {
                if (G0) {
#pragma unroll
                    for (int k = 0; k < FPL; ++k) u0[k] += vcd[k];
                } else {
#pragma unroll
                    for (int k = 0; k < FPL; ++k) ug[k] += vcd[k];
                }
            }
            int c3 = gcap_gr, c3min = gmin_gr;
            if (split || left) {   // members left: tighten the group's cap range
                c3 = -1;
                c3min = INT_MAX;
#pragma unroll
                for (int m0 = 0; m0 < MC; m0 += 32) {
                    const int m = m0 + lane;
                    if (m < M && s.mgroup[m] == gr) {
                        c3 = max(c3, s.mcap[m]);
                        c3min = min(c3min, s.mcap[m]);
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    c3 = max(c3, __shfl_xor_sync(kFull, c3, o));
                    c3min = min(c3min, __shfl_xor_sync(kFull, c3min, o));
                }
            }
            if (lane == 0) hist[(size_t)gr * a.Tpm + idx] = (int8_t)main_pick;
            if (G0) {
                if (d == main_pick) {
                    r_dsum += dt;
                    r_bhr -= bt;
                }
                r_gcap = c3;
                r_gmin = c3min;
                __syncwarp();
            } else {
                __syncwarp();
                if (lane == 0) {
                    s.gd[gr][main_pick] += dt;
                    s.gb[gr][main_pick] -= bt;
                    s.gcap[gr] = c3;
                    s.gmin[gr] = c3min;
                }
                __syncwarp();
            }
                };
        auto process = [&](const auto& vcd, const int dt, const long long bt, const int idx, const int p) {
            const int ng0 = ng;
            pass(std::integral_constant<int, 0>{}, 0, vcd, dt, bt, idx, p);
#if NS_G1SM
            if (ng0 > 1) pass(std::integral_constant<int, 1>{}, 1, vcd, dt, bt, idx, p);
#pragma unroll 1
            for (int gr = 2; gr < ng0; ++gr) pass(std::integral_constant<int, 2>{}, gr, vcd, dt, bt, idx, p);
#else
#pragma unroll 1
            for (int gr = 1; gr < ng0; ++gr) pass(std::integral_constant<int, 2>{}, gr, vcd, dt, bt, idx, p);
#endif
        };
#pragma unroll 1
#if NS_PAIR_STAGE
#pragma unroll
        for (int j = 0; j < G; ++j) stage1(j);
        cp_async_commit();
#pragma unroll 1
        for (int p = 0; p < Tp; ++p) {
            const int sl = p % (2 * G);
            if (p % G == 0) {
                __syncwarp();              // tables p - G .. p - 1 (slots being refilled) consumed
#pragma unroll
                for (int j = 0; j < G; ++j) stage1(p + G + j);
                cp_async_commit();
                cp_async_wait<1>();        // tables p .. p + G - 1 have landed (this lane's copies)
                __syncwarp();              // ... and every lane's
            }
#else
        for (int pp = 0; pp < kDStages - 1; ++pp) issue(pp);
        int sl = 0;   // slot of table p
#pragma unroll 1
        for (int p = 0; p < Tp; ++p, sl = sl + 1 == kDStages ? 0 : sl + 1) {
            __syncwarp();                  // slot (p - 1) % kDStages fully consumed
            issue(p + kDStages - 1);
            cp_async_wait<kDStages - 1>();  // table p has landed (this lane's copies)
            __syncwarp();                  // ... and every lane's
#endif
            double vcd[FPL];
            const double2* src = reinterpret_cast<const double2*>(&s.ring[sl][part * SS]);
#pragma unroll
            for (int i2 = 0; i2 < FPL / 2; ++i2) {
                const double2 xv = src[i2];
                vcd[2 * i2] = xv.x;
                vcd[2 * i2 + 1] = xv.y;
            }
            const int4 mt = s.meta[sl];
            process(vcd, mt.x, (long long)(((unsigned long long)(unsigned)mt.w << 32) | (unsigned)mt.z), mt.y, p);
        }
        cp_async_wait<0>();
        // ---- group 0's register state to shared memory for the epilogue
        if (part == 0 && dev) s.gd[0][d] = r_dsum;
        if (lane == 0) s.gwork[0] = r_gwork;
        __syncwarp();
        // ---- complete the group histories in creation order: a group shares
        //      its parent's choices before the step it split off
        for (int gg = 1; gg < ng; ++gg) {
            const int par = s.gpar[gg], st = s.gstep[gg];
            for (int p2 = lane; p2 < st; p2 += 32) {
                const int i = __ldg(&ometa[p2].y);
                hist[(size_t)gg * a.Tpm + i] = hist[(size_t)par * a.Tpm + i];
            }
            __syncwarp();
        }
        // ---- outputs: per member feasibility, work, and its group's device costs
        for (int gr = 0; gr < ng; ++gr) {
            double hp;
            double w[FPL];
#pragma unroll
            for (int k = 0; k < FPL; ++k) w[k] = GW(k);
            if (gr == 0) {
                hp = part_head<FPL>(u0, w);
            } else {
                double tu[FPL];
#if NS_G1SM
                const double* ug = gr == 1 ? g1_l : gptr(gr);
#else
                const double* ug = gptr(gr);
#endif
#pragma unroll
                for (int k = 0; k < FPL; ++k) tu[k] = ug[k];
                hp = part_head<FPL>(tu, w);
            }
            const double hc = a.head.hb2 + lane_group_sum<LPD>(hp);
            if (part == 0 && dev) s.sc[d] = hc;
            __syncwarp();
            // members of this group: the first one carries the plan, others duplicate it
            int rep = -1;
#pragma unroll
            for (int m0 = 0; m0 < MC; m0 += 32) {
                const unsigned mem = __ballot_sync(kFull, m0 + lane < M && s.mgroup[m0 + lane] == gr);
                if (rep < 0 && mem) rep = m0 + __ffs(mem) - 1;
            }
            if (rep < 0) continue;   // group without live members (uniform)
            // plan cost (N5) and selection read the representative's row only
            for (int dd = lane; dd < D; dd += 32) {
                const int dsum = s.gd[gr][dd];
                a.comp[(tau0 + rep) * D + dd] = dsum > 0 ? s.sc[dd] : 0.0;   // reading R4
                a.devdim[(tau0 + rep) * D + dd] = dsum;
            }
#pragma unroll
            for (int m0 = 0; m0 < MC; m0 += 32) {
                const int m = m0 + lane;
                if (m < M && s.mgroup[m] == gr) x.dup_of[tau0 + m] = (m == rep) ? -1 : (int32_t)(x.tau_base + tau0 + rep);
            }
            // the representative carries the plan (duplicates are read through dup_of)
            int8_t* arow = a.assign + (size_t)(tau0 + rep) * a.Tpm;
            const int8_t* hrow = hist + (size_t)gr * a.Tpm;
            for (int i = lane; i < Tp; i += 32) arow[i] = hrow[i];
            __syncwarp();
        }
#pragma unroll
        for (int m0 = 0; m0 < MC; m0 += 32) {
            const int m = m0 + lane;
            if (m < M) {
                const int mg = s.mgroup[m];
                a.feas[tau0 + m] = mg >= 0 ? 1 : 0;
                a.work[tau0 + m] = s.mwork[m] + (mg >= 0 ? s.gwork[mg] : 0);
                if (mg < 0) x.dup_of[tau0 + m] = -1;
            }
        }
        __syncwarp();
        long long nx = 0;
        if (lane == 0) nx = x.total_warps + (long long)atomicAdd(x.next_cp, 1u);
        g = __shfl_sync(kFull, nx, 0);
    }
}

#undef GW

struct WgrpQueue {
    unsigned int next;        // items claimed
    unsigned int forks;       // items published beyond the n_cp initial ones
    unsigned int completed;   // items finished
    unsigned int pad;
};

struct WgrpArgs {
    int n_cp;                  // column plans of this launch (local slots 0 .. n_cp-1) = initial items
    int n_items;               // item capacity n_cp * M (forks <= n_cp * (M - 1))
    WgrpQueue* q;              // zeroed before the launch
    int32_t* item_cp;          // fork items i >= n_cp: column plan, start step, member mask
    int32_t* item_step;
    unsigned long long* item_mask;
    int32_t* item_ready;       // publication flags (zeroed before the launch)
    double* snap;              // fork snapshots, slot i - n_cp of fork item i
    int32_t* dup_of;           // local trajectory indexing, global tau values
    long long tau_base;        // global tau of local trajectory 0
    // phase-2 hand-off (see SearchBufs)
    int p2_cap, uf_cap, rp_ctas;
    P2Hdr* p2_hdr;
    uint32_t* p2_work;
    double* p2_A;
    long long* p2_room;
    int32_t* p2_dsum;
    int32_t* p2_ready;
    unsigned int* p2_q;
    double* uf_buf;
    int32_t* rp_ord;
    int32_t* p2_first;
    int32_t* p2_next;
    int32_t* p2_rtau;
    uint8_t* p2_alive;
    double* rp_snap;
};

struct P2Hdr {   // 32 bytes
    int g, p, rep, uf;
    int p_sw, pad;
    unsigned long long mask;
};

// ----------------------------------------------------------------------
// 8 x 8 lane layout of the large-D greedy (k_greedy_wide88 / k_greedy_wgrp88).
// A warp owns 32 devices.  Lane l holds feature group fg = l & 7 (features
// 8 fg .. 8 fg + 7) of the 8 devices of device group dg = l >> 3 (devices
// 32 w + 8 dg + j, j = 0..7): u is 64 doubles per lane as with one thread per
// device, but
//  * a lane reads only its 8 features of the staged v row (4 LDS.128, the
//    8 groups padded 16 B apart: one wavefront each) instead of all 64
//    (32 broadcast LDS.128 -- shared-memory wavefronts were the step's
//    bottleneck); the winner's update re-reads them on the 8
//    lanes that hold the winner (4 LDS.128 instead of 32);
//  * the head weights of its 8 features live in registers;
//  * a transposed butterfly over the 8 feature-group lanes (xor 4, 2, 1)
//    leaves lane l with the full score of device 32 w + l, so the argmin,
//    feasibility and work counts stay one device per lane.
// Score order (identical in both kernels): per (device, feature group) one
// accumulator over the 8 features in order, then the butterfly tree over the
// feature groups, then + hb2.
constexpr int kG8 = 8;                  // features per lane
constexpr int kSlot88 = 8 * (kG8 + 2);  // staged row: 8 groups of 8 doubles, padded by 2

// per-lane partials of the 8 devices: sum_{k<8} w_k ReLU(u_jk + v_k), one
// accumulator per device (features in order k = 0..7; the 8 devices are the
// independent chains), v streamed pairwise from the staged slot (register
// pressure: u alone is 128 registers)
template <typename W>
__device__ __forceinline__ void part88(const double (&u)[8][kG8], const double* slot, int fg, const W& w,
                                       double (&p)[8]) {
    const double2* s2 = reinterpret_cast<const double2*>(slot + fg * (kG8 + 2));
#pragma unroll
    for (int j = 0; j < 8; ++j) p[j] = 0.0;
#pragma unroll
    for (int q = 0; q < kG8 / 2; ++q) {
        const double2 vv = s2[q];
        const double w0 = w[2 * q], w1 = w[2 * q + 1];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            p[j] = fma(w0, relu_hi(u[j][2 * q] + vv.x), p[j]);
            p[j] = fma(w1, relu_hi(u[j][2 * q + 1] + vv.y), p[j]);
        }
    }
}

// the final per-device head partials sum_k w_k ReLU(u_jk) (exact ReLU), same order
template <typename W>
__device__ __forceinline__ void head88(const double (&u)[8][kG8], const W& w, double (&p)[8]) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        double a = 0.0;
#pragma unroll
        for (int k = 0; k < kG8; ++k) a = fma(w[k], relu_exact(u[j][k]), a);
        p[j] = a;
    }
}

// Transposed butterfly over the 8 feature-group lanes: at each level a lane
// keeps the half of its device values whose index bit matches its own fg bit
// and adds the partner's copy (IEEE addition commutes, so the lane pair
// computes one well-defined sum).  Returns the sum over the 8 groups of p[fg].
__device__ __forceinline__ double bfly88(double (&p)[8], int fg) {
    {
        const bool hi = fg & 4;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const double send = hi ? p[i] : p[i + 4], keep = hi ? p[i + 4] : p[i];
            p[i] = keep + __shfl_xor_sync(kFull, send, 4);
        }
    }
    {
        const bool hi = fg & 2;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const double send = hi ? p[i] : p[i + 2], keep = hi ? p[i + 2] : p[i];
            p[i] = keep + __shfl_xor_sync(kFull, send, 2);
        }
    }
    const bool hi = fg & 1;
    const double send = hi ? p[0] : p[1], keep = hi ? p[1] : p[0];
    return keep + __shfl_xor_sync(kFull, send, 1);
}

// warp 0 lane l copies features 2l, 2l + 1 of a row into the padded slot
__device__ __forceinline__ double* stage_dst88(double* slot, int lane) {
    return slot + (lane >> 2) * (kG8 + 2) + 2 * (lane & 3);
}

// the winner's update u_j += v on the 8 lanes holding device (dg*, j*): the
// lane's 8 features of the row re-read from the staged slot
__device__ __forceinline__ void add88(double (&u)[8][kG8], const double* slot, int fg, int j) {
    const double2* s2 = reinterpret_cast<const double2*>(slot + fg * (kG8 + 2));
#pragma unroll
    for (int jj = 0; jj < 8; ++jj)
        if (jj == j) {
#pragma unroll
            for (int q = 0; q < kG8 / 2; ++q) {
                const double2 vv = s2[q];
                u[jj][2 * q] += vv.x;
                u[jj][2 * q + 1] += vv.y;
            }
        }
}

// Linear-regime certificate (exact).  vmin_k is the smallest v_tk over every
// variant row the search can stream for the task (k_task_vmin).  If
// u_dk + vmin_k >= 0 for all 64 features then every pre-activation
// fl(u_dk + v_tk) of any later table is >= 0 (rounding is monotone), ReLU is
// the identity, and C(S_d + {t}) = hb2 + sum_k H2_k (u_dk + v_tk) =
// hb2 + (A_d + B_t), A_d = sum_k H2_k u_dk, B_t = sum_k H2_k v_tk -- the same
// real number the literal form computes, evaluated in another order (as the
// hoisting of H1 already is).  A warp whose 32 devices all hold the
// certificate skips part88 / bfly88 and scores its devices as hb2 + (A_d +
// B_t); otherwise it runs the literal form for all of them.  With monotone
// cost models (non-negative v) a device holds it from its first table on
// (92% of the C5 warp steps); with signed weights it never
// triggers.  A_d starts from lin_init88 (a fresh trajectory, u = hb1) and
// grows by B_t with every table the device takes (A_d + B_t is the real sum
// of the new u); the flag is re-checked on the winner's updated u.  Fork
// snapshots carry A_d and the flag, so the grouped and the per-trajectory
// kernels stay bit-identical.

// A_d and the certificate of the lane's own device (32 w + lane) for every
// device of the warp at once: per device j of the lane's group the 8-feature
// partial, the transposed butterfly (bfly88), one ballot per j for the flags
template <typename W>
__device__ __forceinline__ void lin_init88(const double (&u)[8][kG8], const W& w, const double* vm, int fg, int dg,
                                           bool dev, double& A, bool& lin) {
    double pa[8];
    unsigned okm = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        double x = 0.0;
        bool ok = true;
#pragma unroll
        for (int k = 0; k < kG8; ++k) {
            x = fma(w[k], u[j][k], x);
            ok &= (u[j][k] + vm[k] >= 0.0);
        }
        pa[j] = x;
        okm |= (ok ? 1u : 0u) << j;
    }
    A = bfly88(pa, fg);
    bool mine = true;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const unsigned bal = __ballot_sync(kFull, (okm >> j) & 1u);
        if (j == fg) mine = ((bal >> (8 * dg)) & 0xFFu) == 0xFFu;
    }
    lin = mine || !dev;
}

// the winner's update u_j += v (as add88) and its certificate check on the 8
// lanes holding it: returns whether this lane's 8 features of u_j now satisfy
// u + vmin >= 0 (true on every other lane)
__device__ __forceinline__ bool add88_lin(double (&u)[8][kG8], const double* slot, int fg, int j, const double* vm) {
    const double2* s2 = reinterpret_cast<const double2*>(slot + fg * (kG8 + 2));
    bool ok = true;
#pragma unroll
    for (int jj = 0; jj < 8; ++jj)
        if (jj == j) {
#pragma unroll
            for (int q = 0; q < kG8 / 2; ++q) {
                const double2 vv = s2[q];
                u[jj][2 * q] += vv.x;
                u[jj][2 * q + 1] += vv.y;
                ok &= (u[jj][2 * q] + vm[2 * q] >= 0.0) & (u[jj][2 * q + 1] + vm[2 * q + 1] >= 0.0);
            }
        }
    return ok;
}

// the certificate check of add88_lin without the update (a fork's device):
// whether this lane's 8 features of u_j + v satisfy u_j + v + vmin >= 0,
// the sums rounded as the update rounds them
__device__ __forceinline__ bool chk88(const double (&u)[8][kG8], const double* slot, int fg, int j, const double* vm) {
    const double2* s2 = reinterpret_cast<const double2*>(slot + fg * (kG8 + 2));
    bool ok = true;
#pragma unroll
    for (int jj = 0; jj < 8; ++jj)
        if (jj == j) {
#pragma unroll
            for (int q = 0; q < kG8 / 2; ++q) {
                const double2 vv = s2[q];
                const double x0 = u[jj][2 * q] + vv.x, x1 = u[jj][2 * q + 1] + vv.y;
                ok &= (x0 + vm[2 * q] >= 0.0) & (x1 + vm[2 * q + 1] >= 0.0);
            }
        }
    return ok;
}

// Per task: vmin_k over the variant rows a search can stream (depth <
// depths; invalid variants, vdim 0, skipped), and per such row
// B_r = sum_k H2_k v_rk (the linear-regime table term; lane l adds features
// 2l, 2l + 1, then a xor butterfly).  One CTA of 8 warps per task, a warp per
// row at a time.
__global__ void __launch_bounds__(256) k_task_lin(TaskView tv, int depths, HeadParams hp, double* vmin,
                                                  double* Brow) {
    __shared__ double s_min[8][kV];
    const int q = blockIdx.x, lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    const double w0 = hp.H2[2 * lane], w1 = hp.H2[2 * lane + 1];
    double m0 = CUDART_INF, m1 = CUDART_INF;
    const int r0 = tv.off[q] * kDepth, r1 = tv.off[q + 1] * kDepth;
    for (int r = r0 + wi; r < r1; r += 8) {
        if (r % kDepth >= depths || __ldg(tv.vdim + r) == 0) continue;
        const double2 v = __ldg(reinterpret_cast<const double2*>(tv.V + (size_t)r * kV) + lane);
        m0 = fmin(m0, v.x);
        m1 = fmin(m1, v.y);
        double b = fma(w1, v.y, w0 * v.x);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) b += __shfl_xor_sync(kFull, b, o);
        if (lane == 0) Brow[r] = b;
    }
    s_min[wi][2 * lane] = m0;
    s_min[wi][2 * lane + 1] = m1;
    __syncthreads();
    if (threadIdx.x < kV) {
        double m = s_min[0][threadIdx.x];
        for (int k = 1; k < 8; ++k) m = fmin(m, s_min[k][threadIdx.x]);
        vmin[(size_t)q * kV + threadIdx.x] = m;
    }
}

// Large D, latency mode (one trajectory per CTA) in the 8 x 8 layout; the
// step is as in k_greedy_wide88: one CTA argmin per table (warp REDUX argmin,
// then the warps' records through shared memory, double-buffered by step
// parity), cp.async ring of the cost-ordered v rows.
__global__ void __launch_bounds__(128, 2) k_greedy_wide88(const GreedyArgs a) {
    constexpr int kLook = kStages - 2;
    constexpr int kRingW = kStages;
    __shared__ __align__(16) double ring[kRingW][kSlot88];
    __shared__ unsigned long long s_key[2][4];
    __shared__ int s_dv[2][4];
    __shared__ int s_cnt[2][4];
    __shared__ int4 smeta[kRingW];
    __shared__ __align__(16) double ringB[kRingW];   // B_t of the staged rows (k_task_lin)
    __shared__ __align__(16) double s_vmin[kV];
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int fg = lane & 7, dg = lane >> 3;
    const long long tau = a.traj_begin + blockIdx.x;
    if (tau >= a.traj_end) return;
    const int g = (int)(tau / a.M), m = (int)(tau % a.M);
    const int d = threadIdx.x;   // this lane's device after the butterfly
    bool alive = a.cp_valid[g] != 0;
    int Tp = 0, capd = 0, q = 0;
    long long cap = 0;
    if (alive) {
        q = a.cp_task[g];
        Tp = a.cp_Tp[g];
        cap = a.cap[q];
        capd = a.capdim[q * a.M + m];
    }
    const bool dev = d < a.D;
    double u[8][kG8], w[kG8];
#pragma unroll
    for (int k = 0; k < kG8; ++k) {
        w[k] = a.head.H2[kG8 * fg + k];
        const double h = a.head.hb1[kG8 * fg + k];
#pragma unroll
        for (int j = 0; j < 8; ++j) u[j][k] = h;
    }
    for (int k2 = threadIdx.x; k2 < kV; k2 += blockDim.x) s_vmin[k2] = a.vmin[(size_t)q * kV + k2];
    __syncthreads();
    const double* vmq = s_vmin + kG8 * fg;   // this lane's 8 features of vmin
    double A = 0.0;   // linear-regime certificate of the lane's device (lin_init88)
    bool lin = false;
    lin_init88(u, w, vmq, fg, dg, dev, A, lin);
    int dsum = 0;
    long long bsum = 0;
    uint32_t work = 0;
    const int32_t* orow = a.ord_row + (size_t)g * a.Tpm;
    const int4* ometa = a.ord_meta + (size_t)g * a.Tpm;
    int8_t* asg = a.assign + (size_t)tau * a.Tpm;
    const int T = alive ? Tp : 0;
    auto issue = [&](int pp) {
        if (pp < T) {
            const int r = __ldg(orow + pp);
            const int slot = pp % kRingW;
            cp_async16(stage_dst88(ring[slot], lane), a.V + (size_t)r * kV + 2 * lane);
            if (lane == 0) cp_async16(smeta + slot, ometa + pp);
            if (lane == 1) cp_async8(ringB + slot, a.Brow + r);
        }
        cp_async_commit();
    };
    if (wi == 0)
        for (int pp = 0; pp < kLook; ++pp) issue(pp);
#pragma unroll 1
    for (int p = 0; p < T; ++p) {
        const int par = p & 1;
        if (wi == 0) {
            issue(p + kLook);
            cp_async_wait<kLook>();   // table p landed
        }
        __syncthreads();              // ... visible to every warp
        const int sl = p % kRingW;
        const int4 mt = smeta[sl];
        const int dt = mt.x;
        const long long bt = (long long)(((unsigned long long)(unsigned)mt.w << 32) | (unsigned)mt.z);
        const bool f = dev && (bsum + bt <= cap) && (dsum + dt <= capd);
        const double Bt = ringB[sl];
        double sco;
        if (__all_sync(kFull, lin)) {   // every device of the warp holds the certificate
            sco = a.head.hb2 + (A + Bt);
        } else {
            double pp8[8];
            part88(u, ring[sl], fg, w, pp8);
            sco = a.head.hb2 + bfly88(pp8, fg);
        }
        const long long sb = __double_as_longlong(sco + 0.0);
        unsigned long long key = f ? (unsigned long long)(sb ^ ((sb >> 63) | (long long)0x8000000000000000ULL)) : ~0ULL;
        unsigned khi = (unsigned)(key >> 32), klo = (unsigned)key;
        unsigned mhi = __reduce_min_sync(kFull, khi);
        unsigned mlo = __reduce_min_sync(kFull, khi == mhi ? klo : 0xFFFFFFFFu);
        unsigned hit = __ballot_sync(kFull, f && khi == mhi && klo == mlo);
        const unsigned bal = __ballot_sync(kFull, f);
        if (lane == 0) {
            s_key[par][wi] = ((unsigned long long)mhi << 32) | mlo;
            s_dv[par][wi] = wi * 32 + (hit ? __ffs(hit) - 1 : 0);
            s_cnt[par][wi] = __popc(bal);
        }
        __syncthreads();
        key = lane < nw ? s_key[par][lane] : ~0ULL;
        khi = (unsigned)(key >> 32);
        klo = (unsigned)key;
        mhi = __reduce_min_sync(kFull, khi);
        mlo = __reduce_min_sync(kFull, khi == mhi ? klo : 0xFFFFFFFFu);
        hit = __ballot_sync(kFull, lane < nw && khi == mhi && klo == mlo);
        const int cnt = __reduce_add_sync(kFull, lane < nw ? s_cnt[par][lane] : 0);
        const int bd = s_dv[par][hit ? __ffs(hit) - 1 : 0];
        work += cnt;
        if ((mhi & mlo) == 0xFFFFFFFFu) {   // nothing feasible (uniform across the CTA)
            alive = false;
            break;
        }
        if (wi == (bd >> 5)) {   // the winner's update and certificate (whole warp: ballot)
            const bool mine = dg == ((bd >> 3) & 3);
            const bool ok = mine ? add88_lin(u, ring[sl], fg, bd & 7, vmq) : true;
            const unsigned okm = __ballot_sync(kFull, ok);
            if (d == bd) {
                A += Bt;
                lin = ((okm >> (8 * dg)) & 0xFFu) == 0xFFu;
            }
        }
        if (d == bd) {
            dsum += dt;
            bsum += bt;
        }
        if (threadIdx.x == 0) asg[mt.y] = (int8_t)bd;
    }
    if (wi == 0) cp_async_wait<0>();
    double hp[8];
    head88(u, w, hp);
    const double hc = a.head.hb2 + bfly88(hp, fg);
    if (dev) {
        a.comp[tau * a.D + d] = dsum > 0 ? hc : 0.0;   // reading R4
        a.devdim[tau * a.D + d] = dsum;
    }
    if (threadIdx.x == 0) {
        a.feas[tau] = alive ? 1 : 0;
        a.work[tau] = work;
        if (work) atomicAdd(a.computed, (unsigned long long)work);
    }
}

// Large D, throughput mode: k_greedy_wgrp88 -- the M grid trajectories of a
// column plan share their scores while they make identical decisions (the
// paper's life-long cache, as data parallelism; on C5 26-33% of the
// algorithmic scores are distinct).  A work item is a GROUP of
// identical trajectories of one column plan from some step on; a CTA runs it
// in the 8 x 8 lane layout (part88 / bfly88), so its scores are bit-identical
// to k_greedy_wide88's:
//  * a step scores every device that passes the memory cap and the group's
//    largest dim cap; one CTA argmin gives (d*, x* = dim_d* + dim_t);
//  * fast path: x* <= the group's smallest cap -> every member picks d*
//    (each member's feasible set is nested in the largest one and holds d*);
//  * otherwise the members split: repeatedly, the argmin under the largest
//    remaining member cap c is taken by every remaining member whose cap
//    admits it (nested sets again); members with no feasible device strand
//    (R9).  The subgroup holding the largest cap continues; every other one
//    becomes a new work item (FORK): its state (u, dim and byte sums with its
//    own choice applied) goes to the item's snapshot slot and any CTA picks it
//    up from the global queue (persistent CTAs; the queue also balances
//    column plans of different lengths);
//  * W of every member (|F_m| per step, O12) is the group's count when every
//    device fits the smallest cap (one register for the whole group), else one
//    ballot per member; it travels with the members through forks;
//  * the assignment is written to ONE row per group (its lowest member's) and
//    copied to the other members' rows when they leave (fork) or finish;
//  * at the end the lowest member is the representative (comp, devdim) and
//    the others point to it (dup_of), as in k_greedy_dedup.
// One barrier per step: warp 0 waits for the NEXT row before the barrier that
// publishes the warps' argmin keys (double-buffered by step parity).  Caps are
// non-decreasing in m (R8), so a member set's extreme caps are its lowest /
// highest member.
__global__ void __launch_bounds__(128, NS_WGRP_CTAS) k_greedy_wgrp88(const GreedyArgs a, const WgrpArgs x) {
    constexpr int kLook = kStages - 2;
    constexpr int kRingW = kStages;
    constexpr int NWM = 4;
    constexpr int MMAX = 64;
    __shared__ __align__(16) double ring[kRingW][kSlot88];
    __shared__ __align__(16) double s_w88[kSlot88];
    __shared__ __align__(16) double s_vmin[kV];
    __shared__ __align__(16) double ringB[kRingW];   // B_t of the staged rows (k_task_lin)
    __shared__ int4 smeta[kRingW];
    // per warp and step parity: {key lo, key hi, device | x_winner << 7, max x} -- one 16-byte record
    // (dim sums < 2^25: T' * 128 < 2^24 is checked on the host)
    __shared__ uint4 s_rec[2][NWM];
    __shared__ unsigned long long r_key[NWM];   // slow-path rounds
    __shared__ int r_dv[NWM], r_xw[NWM];
    __shared__ int s_cap[MMAX];
    __shared__ unsigned s_work[MMAX];
    __shared__ unsigned long long s_sub_mask[MMAX];
    __shared__ int s_sub_dev[MMAX], s_sub_item[MMAX];
    __shared__ int s_nsub;
    __shared__ unsigned long long s_dead, s_remain;
    __shared__ int s_item;
    __shared__ int s_h, s_h2;   // phase-2 hand-off slots
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int nth = blockDim.x;
    const int fg = lane & 7, dg = lane >> 3;
    const int d = threadIdx.x;   // this lane's device after the butterfly (bfly88)
    const bool dev = d < a.D;
    // head weights of the lane's feature group from shared memory (padded like
    // the row slots: conflict-free), registers are the scarce resource here
    for (int q = threadIdx.x; q < kV; q += blockDim.x) s_w88[(q / kG8) * (kG8 + 2) + q % kG8] = a.head.H2[q];
    const double* w = s_w88 + fg * (kG8 + 2);
    const int M = a.M;
    // snapshot layout: u as [8 devices x 8 features][nth] doubles, then dsum, memory headroom,
    // A_d, certificate flag [nth] --
    // coalesced per thread index
    const size_t snap_doubles = (size_t)nth * (kV + 4);
    unsigned long long computed = 0, steps = 0;   // executed scores / group-steps (ns_stats)
    unsigned lin_sc = 0;                          // this thread's scores taken in the closed linear form
#ifdef NS_WGRP_TIMING   // debug build: clock64 per step phase of thread 0, printed by CTAs 0-3
    unsigned long long tph[7] = {0, 0, 0, 0, 0, 0, 0}, nlin = 0, town = 0, nown = 0;
    long long tlast = clock64();
#define NS_TMARK(k)                                  \
    {                                                \
        const long long tn = clock64();              \
        tph[k] += (unsigned long long)(tn - tlast);  \
        tlast = tn;                                  \
    }
#else
#define NS_TMARK(k)
#endif
    volatile unsigned int* vq = reinterpret_cast<volatile unsigned int*>(x.q);
    volatile int32_t* vready = x.item_ready;
    // copy assignment row src -> dst (list positions [0, n)); rows written by
    // other CTAs are read past L1
    auto copy_row = [&](long long src, long long dst, int n) {
        const int8_t* sp = a.assign + (size_t)src * a.Tpm;
        int8_t* dp = a.assign + (size_t)dst * a.Tpm;
        for (int i = threadIdx.x; i < n; i += nth) dp[i] = __ldcg(sp + i);
    };
    // sum of cf over the CTA (every member's common work |F_max| summed over the steps so far)
    auto block_sum = [&](unsigned v) -> unsigned {
        v = __reduce_add_sync(kFull, v);
        if (lane == 0) r_xw[wi] = (int)v;
        __syncthreads();
        unsigned t = __reduce_add_sync(kFull, lane < nw ? (unsigned)r_xw[lane] : 0u);
        __syncthreads();
        return t;
    };
    for (;;) {
        // ---- claim the next item (waits for a fork to be published, or for the end)
        if (threadIdx.x == 0) {
            const int i = (int)atomicAdd(&x.q->next, 1u);
            int got = -1;
            if (i < x.n_cp) {
                got = i;
            } else if (i < x.n_items) {   // beyond n_items nothing can ever be published
                unsigned ns_sleep = 128, it = 0;   // exponential backoff: a waiting CTA shares its SM with a working one
                for (;;) {
                    if (vready[i]) {
                        got = i;
                        break;
                    }
                    // all published items finished -> nothing can be published any more.
                    // Read `completed` BEFORE `forks`: an item publishes its forks
                    // before it completes, so completed == n_cp + forks (in this order)
                    // means no item was running when `completed` was read.  (Rarely:
                    // the fence invalidates the L1 the SM's working CTA uses.)
                    if ((++it & 7u) == 0) {
                        const unsigned done = vq[2];
                        __threadfence();
                        const unsigned pub = (unsigned)x.n_cp + vq[1];
                        if (done == pub && (unsigned)i >= pub) break;
                    }
                    __nanosleep(ns_sleep);
                    if (ns_sleep < 8192) ns_sleep <<= 1;
                }
                __threadfence();
            }
            s_item = got;
        }
        __syncthreads();
        const int item = s_item;
        if (item < 0) break;
        int g, p0;
        unsigned long long mask;
        if (item < x.n_cp) {
            g = item;
            p0 = 0;
            mask = a.cp_valid[g] ? (M >= 64 ? ~0ULL : ((1ULL << M) - 1)) : 0ULL;
        } else {
            // written by another CTA during this launch: read past L1
            g = __ldcg(x.item_cp + item);
            p0 = __ldcg(x.item_step + item);
            mask = __ldcg(x.item_mask + item);
        }
        const long long tau0 = (long long)g * M;   // local trajectory index of member 0
        const int q = a.cp_task[g];
        const int Tp = mask ? a.cp_Tp[g] : 0;
        const long long cap = mask ? a.cap[q] : 0;   // (fresh items start with room = cap)
        for (int m = threadIdx.x; m < M; m += blockDim.x) {
            s_cap[m] = mask ? a.capdim[q * M + m] : 0;
            if (item < x.n_cp) {   // a column plan starts: every member unplaced, no work yet
                s_work[m] = 0;
                a.feas[tau0 + m] = 0;
                x.dup_of[tau0 + m] = -1;
                if (!mask) a.work[tau0 + m] = 0;
            } else {
                s_work[m] = ((mask >> m) & 1ULL) ? __ldcg(a.work + tau0 + m) : 0u;
            }
        }
        double u[8][kG8];
        int dsum = 0;
        long long room = 0;   // memory headroom cap - bytes on this device (R7)
        if (item < x.n_cp) {
#pragma unroll
            for (int q = 0; q < kG8; ++q) {
                const double h = a.head.hb1[kG8 * fg + q];
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) u[jj][q] = h;
            }
            room = cap;
        } else {
            const double* sp = x.snap + (size_t)(item - x.n_cp) * snap_doubles;
#pragma unroll
            for (int jj = 0; jj < 8; ++jj)
#pragma unroll
                for (int q = 0; q < kG8; ++q) u[jj][q] = __ldcg(sp + (size_t)(jj * kG8 + q) * nth + threadIdx.x);
            dsum = __double2loint(__ldcg(sp + (size_t)kV * nth + threadIdx.x));
            room = __double_as_longlong(__ldcg(sp + (size_t)(kV + 1) * nth + threadIdx.x));
        }
        bool vpos = true;
        for (int k2 = threadIdx.x; k2 < kV; k2 += blockDim.x) {
            s_vmin[k2] = a.vmin[(size_t)q * kV + k2];
            vpos = vpos && s_vmin[k2] >= 0.0;
        }
        // vmin >= 0 (monotone cost models): a device's certificate, once
        // held, holds for good (u only grows), so a linear warp never needs
        // u again before the item ends -- the winner's u update is deferred
        // past the next record publication (off the step's critical path)
        const bool vmin_ok = __syncthreads_and(vpos) != 0;
        const double* vmq = s_vmin + kG8 * fg;   // this lane's 8 features of vmin
        int pend_j = -1, pend_sl = 0;            // deferred u update (owner lanes)
        double A = 0.0;   // linear-regime certificate of the lane's device
        bool lin = false;
        if (item < x.n_cp) {
            lin_init88(u, w, vmq, fg, dg, dev, A, lin);
        } else {
            const double* sp = x.snap + (size_t)(item - x.n_cp) * snap_doubles;
            A = __ldcg(sp + (size_t)(kV + 2) * nth + threadIdx.x);
            lin = __double2loint(__ldcg(sp + (size_t)(kV + 3) * nth + threadIdx.x)) != 0;
        }
        const int32_t* orow = a.ord_row + (size_t)g * a.Tpm;
        const int4* ometa = a.ord_meta + (size_t)g * a.Tpm;
        // warp 0 stages row pp with its index r (loaded a step ahead: rnext)
        auto stage_r = [&](int pp, int r) {
            if (pp < Tp) {
                const int sl = pp % kRingW;
                cp_async16(stage_dst88(ring[sl], lane), a.V + (size_t)r * kV + 2 * lane);
                if (lane == 0) cp_async16(smeta + sl, ometa + pp);
                if (lane == 1) cp_async8(ringB + sl, a.Brow + r);
            }
        };
        int rnext = 0;
        if (wi == 0) {
            for (int pp = p0; pp < p0 + kLook; ++pp) {
                stage_r(pp, pp < Tp ? __ldg(orow + pp) : 0);
                cp_async_commit();
            }
            rnext = p0 + kLook < Tp ? __ldg(orow + p0 + kLook) : 0;
            cp_async_wait<kLook - 1>();   // row p0 landed
        }
        __syncthreads();
        unsigned cf = 0;                  // steps this lane's device was scored
        bool handed = false;              // the item went on to phase 2
        int rep = mask ? __ffsll((long long)mask) - 1 : 0;   // the row holding the group's history
        bool alive = mask != 0;
        int pend = p0;   // steps run = pend - p0
        // the group's extreme caps (members ordered by cap, R8); they change only at forks
        int cmin = mask ? s_cap[__ffsll((long long)mask) - 1] : 0;
        int cmax = mask ? s_cap[63 - __clzll((long long)mask)] : 0;
#pragma unroll 1
        for (int p = p0; p < Tp; ++p) {
            NS_TMARK(5)
            pend = p + 1;
            const int par = p & 1;
            const int sl = p % kRingW;
            const int4 mt = smeta[sl];
            const int dt = mt.x;
            const long long bt = (long long)(((unsigned long long)(unsigned)mt.w << 32) | (unsigned)mt.z);
            const bool memok = dev && (bt <= room);
            const int xv = dsum + dt;
            const bool f = memok && xv <= cmax;
            // every device scores (no divergent branch); an infeasible
            // device's finite score is masked by its key ~0
            const double Bt = ringB[sl];
            double sco;
            const bool wlin = __all_sync(kFull, lin);
            if (wlin) {   // every device of the warp holds the certificate
#ifdef NS_WGRP_TIMING
                ++nlin;
#endif
                sco = a.head.hb2 + (A + Bt);
            } else {
                double pp8[8];
                part88(u, ring[sl], fg, w, pp8);
                sco = a.head.hb2 + bfly88(pp8, fg);
            }
            NS_TMARK(0)
            const long long sb = __double_as_longlong(sco + 0.0);
            const unsigned long long key =
                f ? (unsigned long long)(sb ^ ((sb >> 63) | (long long)0x8000000000000000ULL)) : ~0ULL;
            // warp: min key (two REDUX), lowest device holding it, its x,
            // feasible count, max x over memory-feasible devices
            {
                const unsigned khi = (unsigned)(key >> 32), klo = (unsigned)key;
                const unsigned mh = __reduce_min_sync(kFull, khi);
                const unsigned ml = __reduce_min_sync(kFull, khi == mh ? klo : 0xFFFFFFFFu);
                const unsigned hit = __ballot_sync(kFull, f && khi == mh && klo == ml);
                const unsigned xm = __reduce_max_sync(kFull, f ? (unsigned)xv : 0u);
                const int hl = hit ? __ffs(hit) - 1 : 0;
                const int xw = __shfl_sync(kFull, xv, hl);
                if (lane == 0)   // bit 31: every device of the warp held the certificate
                    s_rec[par][wi] = make_uint4(ml, mh,
                                                (unsigned)(wi * 32 + hl) | ((unsigned)xw << 7) |
                                                    (wlin ? 0x80000000u : 0u),
                                                xm);
            }
            NS_TMARK(1)
            // warp 0: row p + 1 lands before the barrier that publishes it (rows
            // up to p + kLook - 1 are in flight); row p + kLook is issued after
            // the barrier, off the warps' critical path
            if (pend_j >= 0) {   // last step's deferred winner update (the ring slot is still intact)
                add88(u, ring[pend_sl], fg, pend_j);
                pend_j = -1;
            }
            if (wi == 0) cp_async_wait<kLook - 2>();
            __syncthreads();
            if (wi == 0) {   // slot (p + kLook) % kRingW held row p - 2, read at step p - 2 at the latest
                stage_r(p + kLook, rnext);
                rnext = p + kLook + 1 < Tp ? __ldg(orow + p + kLook + 1) : 0;   // consumed next step
                cp_async_commit();
            }
            NS_TMARK(2)
            int bd, xstar;
            unsigned xmax;
            bool none, alllin;
            {
                const uint4 rc = lane < nw ? s_rec[par][lane] : make_uint4(~0u, ~0u, 0x80000000u, 0u);
                const unsigned mh = __reduce_min_sync(kFull, rc.y);
                const unsigned ml = __reduce_min_sync(kFull, rc.y == mh ? rc.x : 0xFFFFFFFFu);
                const unsigned hit = __ballot_sync(kFull, lane < nw && rc.y == mh && rc.x == ml);
                xmax = __reduce_max_sync(kFull, rc.w);
                none = (mh & ml) == 0xFFFFFFFFu;
                alllin = __all_sync(kFull, (rc.z >> 31) != 0u);
                const unsigned dx = __shfl_sync(kFull, rc.z, hit ? __ffs(hit) - 1 : 0);
                bd = (int)(dx & 127u);
                xstar = (int)((dx >> 7) & 0xFFFFFFu);
            }
            NS_TMARK(3)
            // ---- work W per member (O12): |F_m| = #{memory-feasible d : x_d <= cap_m}
            // = |F_max| (this thread's device counts in cf) minus the devices
            // with cap_m < x_d <= cap_max, counted only for the members whose
            // cap is below the largest feasible x (xmax)
            cf += (f) ? 1u : 0u;
            lin_sc += (f && wlin) ? 1u : 0u;
            if (xmax > (unsigned)cmin) {
                for (unsigned long long mm = mask; mm; mm &= mm - 1) {
                    const int m = __ffsll((long long)mm) - 1;
                    if ((unsigned)s_cap[m] >= xmax) break;   // caps non-decreasing in m
                    const unsigned b = __ballot_sync(kFull, f && xv > s_cap[m]);
                    if (lane == 0 && b) atomicSub(&s_work[m], (unsigned)__popc(b));
                }
            }
            if (none) {   // nothing feasible even under the largest cap: the group strands
                alive = false;
                break;
            }
            NS_TMARK(4)
            if (xstar > cmin) {
                // ---- slow path: members split by the caps that admit the winners
                __syncthreads();   // per-member work atomics done
                if (threadIdx.x == 0) {
                    unsigned long long take = 0;
                    for (unsigned long long mm = mask; mm; mm &= mm - 1) {
                        const int m = __ffsll((long long)mm) - 1;
                        if (s_cap[m] >= xstar) take |= 1ULL << m;
                    }
                    s_nsub = 1;
                    s_sub_mask[0] = take;
                    s_sub_dev[0] = bd;
                    s_remain = mask & ~take;
                    s_dead = 0;
                }
                __syncthreads();
                while (s_remain) {
                    const unsigned long long rem = s_remain;
                    const int c = s_cap[63 - __clzll((long long)rem)];
                    const bool fc = f && xv <= c;
                    const unsigned long long kc = fc ? key : ~0ULL;
                    const unsigned khi = (unsigned)(kc >> 32), klo = (unsigned)kc;
                    const unsigned mh = __reduce_min_sync(kFull, khi);
                    const unsigned ml = __reduce_min_sync(kFull, khi == mh ? klo : 0xFFFFFFFFu);
                    const unsigned hit = __ballot_sync(kFull, fc && khi == mh && klo == ml);
                    const int hl = hit ? __ffs(hit) - 1 : 0;
                    const int xw = __shfl_sync(kFull, xv, hl);
                    if (lane == 0) {
                        r_key[wi] = ((unsigned long long)mh << 32) | ml;
                        r_dv[wi] = wi * 32 + hl;
                        r_xw[wi] = xw;
                    }
                    __syncthreads();
                    if (threadIdx.x == 0) {
                        unsigned long long bk = ~0ULL;
                        int bdv = 0, bx = 0;
                        for (int k = 0; k < nw; ++k)
                            if (r_key[k] < bk) {   // strict: the lowest warp (device) keeps ties
                                bk = r_key[k];
                                bdv = r_dv[k];
                                bx = r_xw[k];
                            }
                        if (bk == ~0ULL) {
                            s_dead = rem;   // no feasible device under these members' caps
                            s_remain = 0;
                        } else {
                            unsigned long long take = 0;
                            for (unsigned long long mm = rem; mm; mm &= mm - 1) {
                                const int m = __ffsll((long long)mm) - 1;
                                if (s_cap[m] >= bx) take |= 1ULL << m;
                            }
                            s_sub_mask[s_nsub] = take;
                            s_sub_dev[s_nsub] = bdv;
                            s_nsub++;
                            s_remain = rem & ~take;
                        }
                    }
                    __syncthreads();
                }
                // ---- fork every subgroup but the first into a new work item
                const int nsub = s_nsub;
                const unsigned gw = block_sum(cf);
                if (threadIdx.x == 0)
                    for (int k = 1; k < nsub; ++k) s_sub_item[k] = x.n_cp + (int)atomicAdd(&x.q->forks, 1u);
                __syncthreads();
                for (int k = 1; k < nsub; ++k) {
                    const int dk = s_sub_dev[k];
                    const int it = s_sub_item[k];
                    double* sp = x.snap + (size_t)(it - x.n_cp) * snap_doubles;
                    const bool mine = d == dk;
                    const bool owner = wi == (dk >> 5) && dg == ((dk >> 3) & 3);
                    const double* vs = ring[sl] + fg * (kG8 + 2);
#pragma unroll
                    for (int jj = 0; jj < 8; ++jj)
#pragma unroll
                        for (int q = 0; q < kG8; ++q) {
                            double val = u[jj][q];
                            if (owner && jj == (dk & 7)) val += vs[q];
                            __stcg(sp + (size_t)(jj * kG8 + q) * nth + threadIdx.x, val);
                        }
                    sp[(size_t)kV * nth + threadIdx.x] = __hiloint2double(0, mine ? dsum + dt : dsum);
                    sp[(size_t)(kV + 1) * nth + threadIdx.x] = __longlong_as_double(mine ? room - bt : room);
                    {   // A_d and the certificate with dk's choice applied (as the update below does)
                        const bool ok = owner ? chk88(u, ring[sl], fg, dk & 7, vmq) : true;
                        const unsigned okm = __ballot_sync(kFull, ok);
                        const bool kl = ((okm >> (8 * dg)) & 0xFFu) == 0xFFu;
                        sp[(size_t)(kV + 2) * nth + threadIdx.x] = mine ? A + Bt : A;
                        sp[(size_t)(kV + 3) * nth + threadIdx.x] = __hiloint2double(0, mine ? (kl ? 1 : 0) : (lin ? 1 : 0));
                    }
                    // the subgroup's history row: the group's history so far + its choice
                    const unsigned long long km = s_sub_mask[k];
                    const int krep = __ffsll((long long)km) - 1;
                    copy_row(tau0 + rep, tau0 + krep, Tp);
                    for (int m = threadIdx.x; m < M; m += blockDim.x)
                        if ((km >> m) & 1ULL) a.work[tau0 + m] = s_work[m] + gw;   // work travels with the members
                }
                const unsigned long long dead = s_dead;
                for (int m = threadIdx.x; m < M; m += blockDim.x)
                    if ((dead >> m) & 1ULL) a.work[tau0 + m] = s_work[m] + gw;   // stranded (feas stays 0)
                __syncthreads();   // row copies done before the choices below land in them
                if (threadIdx.x < nsub && threadIdx.x > 0) {
                    const unsigned long long km = s_sub_mask[threadIdx.x];
                    a.assign[(size_t)(tau0 + __ffsll((long long)km) - 1) * a.Tpm + mt.y] = (int8_t)s_sub_dev[threadIdx.x];
                }
                mask = s_sub_mask[0];
                bd = s_sub_dev[0];
                cmin = s_cap[__ffsll((long long)mask) - 1];
                cmax = s_cap[63 - __clzll((long long)mask)];
                const int nrep = __ffsll((long long)mask) - 1;
                if (nrep != rep) {
                    copy_row(tau0 + rep, tau0 + nrep, Tp);
                    rep = nrep;
                }
                __threadfence();
                __syncthreads();
                if (threadIdx.x == 0)
                    for (int k = 1; k < nsub; ++k) {
                        const int it = s_sub_item[k];
                        x.item_cp[it] = g;
                        x.item_step[it] = p + 1;
                        x.item_mask[it] = s_sub_mask[k];
                        __threadfence();
                        atomicExch(&x.item_ready[it], 1);   // publish
                    }
            }
            NS_TMARK(6)
            // ---- the group's choice
            if (wi == (bd >> 5)) {   // the winner's update and certificate (whole warp: ballot)
#ifdef NS_WGRP_TIMING
                const long long to0 = clock64();
#endif
                const bool mine = dg == ((bd >> 3) & 3);
                if (vmin_ok && __all_sync(kFull, lin)) {
                    // linear warp: the certificate persists; u's update waits
                    if (mine) {
                        pend_j = bd & 7;
                        pend_sl = sl;
                    }
                    if (d == bd) A += Bt;
                } else {
                    const bool ok = mine ? add88_lin(u, ring[sl], fg, bd & 7, vmq) : true;
                    const unsigned okm = __ballot_sync(kFull, ok);
                    if (d == bd) {
                        A += Bt;
                        lin = ((okm >> (8 * dg)) & 0xFFu) == 0xFFu;
                    }
                }
#ifdef NS_WGRP_TIMING
                town += (unsigned long long)(clock64() - to0);
                ++nown;
#endif
            }
            if (d == bd) {
                dsum += dt;
                room -= bt;
            }
            if (threadIdx.x == 0) a.assign[(size_t)(tau0 + rep) * a.Tpm + mt.y] = (int8_t)bd;
            // ---- hand-off to phase 2 (k_greedy_p2): every device held the
            // certificate at this step (so it holds for good, vmin >= 0); the
            // rest of the trajectory needs only (A_d, dim sum, headroom) per
            // device -- phase 2 runs it with one warp per group, the frozen u
            // is kept for the representative's final replay
            if (alllin && vmin_ok && p + 2 < Tp) {
                if (threadIdx.x == 0) {
                    const unsigned ufs = atomicAdd(x.p2_q + 4, 1u);
                    s_h = ufs < (unsigned)x.uf_cap ? (int)ufs : -1;
                    s_h2 = s_h >= 0 ? (int)atomicAdd(x.p2_q + 3, 1u) : -1;
                }
                __syncthreads();
                const int uf = s_h, slot = s_h2;
                if (uf >= 0) {
                    if (pend_j >= 0) {
                        add88(u, ring[pend_sl], fg, pend_j);
                        pend_j = -1;
                    }
                    double* up = x.uf_buf + (size_t)uf * kV * 128;
#pragma unroll
                    for (int jj = 0; jj < 8; ++jj)
#pragma unroll
                        for (int q2 = 0; q2 < kG8; ++q2) __stcg(up + (size_t)(jj * kG8 + q2) * 128 + threadIdx.x, u[jj][q2]);
                    if (dev) {
                        x.p2_A[(size_t)slot * 128 + d] = A;
                        x.p2_room[(size_t)slot * 128 + d] = room;
                        x.p2_dsum[(size_t)slot * 128 + d] = dsum;
                    }
                    const unsigned gwh = block_sum(cf);
                    for (int m = threadIdx.x; m < M; m += blockDim.x)
                        if ((mask >> m) & 1ULL) x.p2_work[(size_t)slot * 64 + m] = s_work[m] + gwh;
                    if (threadIdx.x == 0) {
                        P2Hdr h;
                        h.g = g;
                        h.p = p + 1;
                        h.rep = rep;
                        h.uf = uf;
                        h.p_sw = p + 1;
                        h.pad = 0;
                        h.mask = mask;
                        x.p2_hdr[slot] = h;
                    }
                    computed += gwh;
                    steps += (unsigned long long)(p + 1 - p0);
                    handed = true;
                    break;
                }
            }
        }
        if (pend_j >= 0) {   // the last step's deferred winner update
            add88(u, ring[pend_sl], fg, pend_j);
            pend_j = -1;
        }
        if (wi == 0) cp_async_wait<0>();
        __syncthreads();   // the representative row is complete
        if (!handed) {
        const unsigned gw = block_sum(cf);
        computed += gw;
        steps += (unsigned long long)(pend - p0);
        // ---- item end: members' work and rows; representative's per-device costs, links of the others
        for (int m = threadIdx.x; m < M; m += blockDim.x)
            if ((mask >> m) & 1ULL) a.work[tau0 + m] = s_work[m] + gw;
        if (alive) {
            double hp[8];
            head88(u, w, hp);
            const double hc = a.head.hb2 + bfly88(hp, fg);
            if (dev) {
                a.comp[(tau0 + rep) * a.D + d] = dsum > 0 ? hc : 0.0;   // reading R4
                a.devdim[(tau0 + rep) * a.D + d] = dsum;
            }
            for (int m = threadIdx.x; m < M; m += blockDim.x)
                if ((mask >> m) & 1ULL) {
                    a.feas[tau0 + m] = 1;
                    x.dup_of[tau0 + m] = m == rep ? -1 : (int32_t)(x.tau_base + tau0 + rep);
                }
            for (unsigned long long mm = mask & ~(1ULL << rep); mm; mm &= mm - 1)
                copy_row(tau0 + rep, tau0 + __ffsll((long long)mm) - 1, Tp);
        }
        }   // !handed
        __threadfence();
        __syncthreads();   // ring and shared state are reused by the next item
        if (threadIdx.x == 0) atomicAdd(&x.q->completed, 1u);
    }
#ifdef NS_WGRP_TIMING
    if ((threadIdx.x & 31) == 0 && blockIdx.x < 2 && steps)
        printf("wgrp cta %d warp %d steps %llu cycles/step: score %.0f key+warp %.0f stage+bar %.0f xwarp %.0f W %.0f "
               "slow %.0f update+loop %.0f linear %.3f owner-update %.0f (%.2f of steps)\n",
               blockIdx.x, threadIdx.x >> 5, steps, (double)tph[0] / steps, (double)tph[1] / steps, (double)tph[2] / steps,
               (double)tph[3] / steps, (double)tph[4] / steps, (double)tph[6] / steps, (double)tph[5] / steps, (double)nlin / steps,
               nown ? (double)town / nown : 0.0, (double)nown / steps);
#endif
#undef NS_TMARK
    if (threadIdx.x == 0 && computed) atomicAdd(a.computed, computed);
    if (threadIdx.x == 0 && steps) atomicAdd(a.computed + 1, steps);
    const unsigned lsum = __reduce_add_sync(kFull, lin_sc);
    if ((threadIdx.x & 31) == 0 && lsum) atomicAdd(a.computed + 2, (unsigned long long)lsum);
}


// u_j += v from registers (phase-2 replay)
__device__ __forceinline__ void addv88(double (&u)[8][kG8], const double (&v)[kG8], int j) {
#pragma unroll
    for (int jj = 0; jj < 8; ++jj)
        if (jj == j) {
#pragma unroll
            for (int k = 0; k < kG8; ++k) u[jj][k] += v[k];
        }
}

// ----------------------------------------------------------------------
// Phase 2 of the large-D grouped greedy (k_greedy_p2).  Once every device
// of a group holds the linear certificate (and vmin >= 0, so it holds for
// good), a step needs only (A_d, dim sum, headroom) per device: the score is
// hb2 + (A_d + B_t), the winner's update A += B_t (the same operations
// k_greedy_wgrp88 and k_greedy_wide88 perform).  k_greedy_wgrp88 hands such
// a group over (frozen u, per-device states, member work so far); here ONE
// warp runs it -- each lane holds devices lane + 32 j (j < 4), every argmin is
// a warp reduction, no barrier, ~40 registers, so many groups are resident
// per SM.  The member splits (slow path) run inside the warp: the subgroup
// holding the largest cap continues, every other one becomes a phase-2 fork
// (tiny record) published on this kernel's queue.  Work counts, history rows
// and links are written as k_greedy_wgrp88 writes them; the representative's
// final per-device cost needs u, so it is queued for k_greedy_replay.
__device__ __forceinline__ int p2_cap_of(int cap0, int cap1, int m) {
    const int c0 = __shfl_sync(kFull, cap0, m & 31), c1 = __shfl_sync(kFull, cap1, m & 31);
    return m < 32 ? c0 : c1;
}

#ifndef NS_P2_CTAS
#define NS_P2_CTAS 3   // resident 8-warp CTAs per SM of k_greedy_p2 (80 registers, a few spills: +3% over 2)
#endif
__global__ void __launch_bounds__(256, NS_P2_CTAS) k_greedy_p2(const GreedyArgs a, const WgrpArgs x) {
    const int lane = threadIdx.x & 31;
    const int M = a.M, D = a.D;
    volatile unsigned int* vq = x.p2_q;   // [0] claimed [1] forks [2] completed [3] hand-offs [4] frozen u [5] replays
    volatile int32_t* vready = x.p2_ready;
    const unsigned n_init = __ldcg(x.p2_q + 3);
    unsigned long long computed = 0, nsteps = 0;
#ifdef NS_WGRP_TIMING
    unsigned long long t_loop = 0, t_claim = 0, n_items = 0, t_key = 0, t_w = 0, n_fk = 0;
    double fk_pos = 0.0, fk_rem = 0.0;
    long long tc0 = clock64();
#endif
    for (;;) {
        // ---- claim an item (a hand-off, or a fork once published)
        int item = -1;
        if (lane == 0) {
            const unsigned i = atomicAdd(x.p2_q + 0, 1u);
            if (i < n_init) {
                item = (int)i;
            } else if (i < (unsigned)x.p2_cap) {
                // a waiting warp polls its slot's flag (L2) and sleeps; the
                // fenced termination test runs rarely -- a fence invalidates the
                // SM's L1, which the working warps on the SM depend on
                unsigned ns = 256, it = 0;
                for (;;) {
                    if (vready[i]) {
                        item = (int)i;
                        break;
                    }
                    if ((++it & 7u) == 0) {
                        const unsigned done = vq[2];   // completed before published (see k_greedy_wgrp88)
                        __threadfence();
                        const unsigned pub = n_init + vq[1];
                        if (done == pub && i >= pub) break;
                    }
                    __nanosleep(ns);
                    if (ns < 16384) ns <<= 1;
                }
                __threadfence();
            }
        }
        item = __shfl_sync(kFull, item, 0);
#ifdef NS_WGRP_TIMING
        const long long tc1 = clock64();
        t_claim += (unsigned long long)(tc1 - tc0);
        ++n_items;
#endif
        if (item < 0) break;
        const long long* hp = reinterpret_cast<const long long*>(x.p2_hdr + item);
        P2Hdr h;
        {
            long long hv[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) hv[k] = __ldcg(hp + k);
            h = *reinterpret_cast<P2Hdr*>(hv);
        }
        const int g = h.g, uf = h.uf, p_sw = h.p_sw;
        int rep = h.rep;
        unsigned long long mask = h.mask;
        const long long tau0 = (long long)g * M;
        const int q = a.cp_task[g];
        const int Tp = a.cp_Tp[g];
        const int cap0 = lane < M ? a.capdim[q * M + lane] : INT_MAX;
        const int cap1 = lane + 32 < M ? a.capdim[q * M + lane + 32] : INT_MAX;
        unsigned wk0 = (lane < M && ((mask >> lane) & 1ULL)) ? __ldcg(x.p2_work + (size_t)item * 64 + lane) : 0u;
        unsigned wk1 = (lane + 32 < M && ((mask >> (lane + 32)) & 1ULL))
                           ? __ldcg(x.p2_work + (size_t)item * 64 + lane + 32) : 0u;
        double A4[4];
        int ds4[4];
        long long rm4[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int dd = lane + 32 * j;
            const bool v = dd < D;
            A4[j] = v ? __ldcg(x.p2_A + (size_t)item * 128 + dd) : 0.0;
            ds4[j] = v ? __ldcg(x.p2_dsum + (size_t)item * 128 + dd) : 0;
            rm4[j] = v ? __ldcg(x.p2_room + (size_t)item * 128 + dd) : -1;   // no device: no room
        }
        int cmin = p2_cap_of(cap0, cap1, __ffsll((long long)mask) - 1);
        int cmax = p2_cap_of(cap0, cap1, 63 - __clzll((long long)mask));
        int last_fork = -1;   // this item's latest fork (the replay walks forks in step order)
        const int32_t* orow = a.ord_row + (size_t)g * a.Tpm;
        const int4* ometa = a.ord_meta + (size_t)g * a.Tpm;
        auto copy_row = [&](long long src, long long dst, int n) {
            const int8_t* sp = a.assign + (size_t)src * a.Tpm;
            int8_t* dp = a.assign + (size_t)dst * a.Tpm;
            for (int i = lane; i < n; i += 32) dp[i] = __ldcg(sp + i);
            __syncwarp();
        };
        bool alive = true;
        // the step stream in chunks of 32 steps, lane l holding step c + l:
        // chunk c in (cm, cB), chunk c + 32 in flight (nm, nB), the row indices
        // of chunk c + 64 in flight (nr) -- one load latency per 32 steps
        const int c0 = h.p;
        auto ld_m = [&](int pp) { return pp < Tp ? __ldg(ometa + pp) : make_int4(0, 0, 0, 0); };
        auto ld_r = [&](int pp) { return pp < Tp ? __ldg(orow + pp) : 0; };
        int4 cm = ld_m(c0 + lane);
        double cB = __ldg(a.Brow + ld_r(c0 + lane));
        int nr0 = ld_r(c0 + 32 + lane);
        int4 nm = ld_m(c0 + 32 + lane);
        double nB = __ldg(a.Brow + nr0);
        int nr = ld_r(c0 + 64 + lane);
        // the group's choices of the chunk's steps: lane l keeps step c + l's and
        // writes it when the chunk ends (one store per 32 steps); the members'
        // work gains |F_max| per step, summed in csum until a split or the end
        int mybd = -1;
        int8_t* hrow = a.assign + (size_t)(tau0 + rep) * a.Tpm;
        unsigned csum = 0;
        auto flush_hist = [&]() {
            if (mybd >= 0) hrow[cm.y] = (int8_t)mybd;
            mybd = -1;
            __syncwarp();
        };
        auto flush_work = [&]() {
            if (lane < M && ((mask >> lane) & 1ULL)) wk0 += csum;
            if (lane + 32 < M && ((mask >> (lane + 32)) & 1ULL)) wk1 += csum;
            csum = 0;
        };
#pragma unroll 1
        for (int p = h.p; p < Tp; ++p) {
            const int k32 = (p - c0) & 31;
            if (k32 == 0 && p > c0) {   // next chunk
                flush_hist();
                cm = nm;
                cB = nB;
                nm = ld_m(p + 32 + lane);
                nB = __ldg(a.Brow + nr);
                nr = ld_r(p + 64 + lane);
            }
            const int dt = __shfl_sync(kFull, cm.x, k32);
            const unsigned btl = (unsigned)__shfl_sync(kFull, cm.z, k32), bth = (unsigned)__shfl_sync(kFull, cm.w, k32);
            const double Bt = __shfl_sync(kFull, cB, k32);
#ifdef NS_WGRP_TIMING
            const long long tk0 = clock64();
#endif
            const long long bt = (long long)(((unsigned long long)bth << 32) | btl);
            // scores hb2 + (A_d + B_t) of the lane's 4 devices; devices >= D have room -1
            int xj[4];
            bool fj[4];
            double bs = CUDART_INF;
            int bj = 0, cfl = 0;
            unsigned xm = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                xj[j] = ds4[j] + dt;
                fj[j] = (bt <= rm4[j]) & (xj[j] <= cmax);
                const double s = a.head.hb2 + (A4[j] + Bt);
                if (fj[j] & (s < bs)) {   // strict: the lane's lowest device keeps ties (-0 == +0)
                    bs = s;
                    bj = j;
                }
                xm = fj[j] ? max(xm, (unsigned)xj[j]) : xm;
                cfl += fj[j] ? 1 : 0;
            }
            unsigned long long best = ~0ULL;
            if (bs < CUDART_INF) {   // order-preserving key of the lane's best (+0.0: -0 and +0 alike)
                const long long sb = __double_as_longlong(bs + 0.0);
                best = (unsigned long long)(sb ^ ((sb >> 63) | (long long)0x8000000000000000ULL));
            }
            const unsigned khi = (unsigned)(best >> 32), klo = (unsigned)best;
            const unsigned mh = __reduce_min_sync(kFull, khi);
            const unsigned ml = __reduce_min_sync(kFull, khi == mh ? klo : 0xFFFFFFFFu);
            const bool none = (mh & ml) == 0xFFFFFFFFu;
            const unsigned dmin =
                __reduce_min_sync(kFull, (khi == mh && klo == ml) ? (unsigned)(32 * bj + lane) : 0xFFFFFFFFu);
            const unsigned xmax = __reduce_max_sync(kFull, xm);
            const unsigned cfc = __reduce_add_sync(kFull, (unsigned)cfl);
            const int bd = none ? 0 : (int)dmin;
            const int jb = bd >> 5, ob = bd & 31;   // the winner's slot and owner lane (warp-uniform)
            const int dsb = jb == 0 ? ds4[0] : jb == 1 ? ds4[1] : jb == 2 ? ds4[2] : ds4[3];
            const int xstar = __shfl_sync(kFull, dsb, ob) + dt;
            computed += cfc;
            csum += cfc;
            ++nsteps;
#ifdef NS_WGRP_TIMING
            const long long tk1 = clock64();
            t_key += (unsigned long long)(tk1 - tk0);
#endif
            // ---- work W per member (O12): |F_max| (csum) minus the devices with cap_m < x_d
            if (xmax > (unsigned)cmin) {
                for (unsigned long long mm = mask; mm; mm &= mm - 1) {
                    const int m = __ffsll((long long)mm) - 1;
                    const int cmm = p2_cap_of(cap0, cap1, m);
                    if ((unsigned)cmm >= xmax) break;   // caps non-decreasing in m
                    int c = 0;
#pragma unroll
                    for (int j = 0; j < 4; ++j) c += (fj[j] & (xj[j] > cmm)) ? 1 : 0;
                    const unsigned cnt = __reduce_add_sync(kFull, (unsigned)c);
                    if (lane == (m & 31)) {
                        if (m < 32) wk0 -= cnt;
                        else wk1 -= cnt;
                    }
                }
            }
#ifdef NS_WGRP_TIMING
            t_w += (unsigned long long)(clock64() - tk1);
#endif
            if (none) {   // nothing feasible even under the largest cap: the group strands
                alive = false;
                break;
            }
            if (xstar > cmin) {
                // ---- slow path: members split by the caps that admit the winners
                flush_work();
                flush_hist();
                const int li = __shfl_sync(kFull, cm.y, k32);
                unsigned long long take0 = 0;
                for (unsigned long long mm = mask; mm; mm &= mm - 1) {
                    const int m = __ffsll((long long)mm) - 1;
                    if (p2_cap_of(cap0, cap1, m) >= xstar) take0 |= 1ULL << m;
                }
                unsigned long long rem = mask & ~take0, dead = 0;
                while (rem) {
                    const int c = p2_cap_of(cap0, cap1, 63 - __clzll((long long)rem));
                    unsigned long long b2 = ~0ULL;
                    int bj2 = 0;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const long long sb = __double_as_longlong(a.head.hb2 + (A4[j] + Bt) + 0.0);
                        const unsigned long long kj = (fj[j] && xj[j] <= c)
                                                          ? (unsigned long long)(sb ^ ((sb >> 63) | (long long)0x8000000000000000ULL))
                                                          : ~0ULL;
                        if (kj < b2) {
                            b2 = kj;
                            bj2 = j;
                        }
                    }
                    const unsigned h2 = (unsigned)(b2 >> 32), l2 = (unsigned)b2;
                    const unsigned mh2 = __reduce_min_sync(kFull, h2);
                    const unsigned ml2 = __reduce_min_sync(kFull, h2 == mh2 ? l2 : 0xFFFFFFFFu);
                    if ((mh2 & ml2) == 0xFFFFFFFFu) {   // no feasible device under these members' caps
                        dead = rem;
                        break;
                    }
                    const int dk = (int)__reduce_min_sync(kFull, (h2 == mh2 && l2 == ml2) ? (unsigned)(32 * bj2 + lane)
                                                                                         : 0xFFFFFFFFu);
                    const int xb2 = bj2 == 0 ? xj[0] : bj2 == 1 ? xj[1] : bj2 == 2 ? xj[2] : xj[3];
                    const int xk = __shfl_sync(kFull, xb2, dk & 31);
                    unsigned long long take = 0;
                    for (unsigned long long mm = rem; mm; mm &= mm - 1) {
                        const int m = __ffsll((long long)mm) - 1;
                        if (p2_cap_of(cap0, cap1, m) >= xk) take |= 1ULL << m;
                    }
                    rem &= ~take;
#ifdef NS_WGRP_TIMING
                    ++n_fk;
                    fk_pos += (double)(p - p_sw) / (double)(Tp - p_sw);
                    fk_rem += (double)(Tp - p);
#endif
                    // fork: the subgroup with its own choice, as a phase-2 item
                    int slot = 0;
                    if (lane == 0) slot = (int)(n_init + atomicAdd(x.p2_q + 1, 1u));
                    slot = __shfl_sync(kFull, slot, 0);
                    const int krep = __ffsll((long long)take) - 1;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int dd = lane + 32 * j;
                        if (dd < D) {
                            const bool mine = dd == dk;
                            x.p2_A[(size_t)slot * 128 + dd] = mine ? A4[j] + Bt : A4[j];
                            x.p2_dsum[(size_t)slot * 128 + dd] = mine ? ds4[j] + dt : ds4[j];
                            x.p2_room[(size_t)slot * 128 + dd] = mine ? rm4[j] - bt : rm4[j];
                        }
                    }
                    if (lane < M && ((take >> lane) & 1ULL)) x.p2_work[(size_t)slot * 64 + lane] = wk0;
                    if (lane + 32 < M && ((take >> (lane + 32)) & 1ULL)) x.p2_work[(size_t)slot * 64 + lane + 32] = wk1;
                    copy_row(tau0 + rep, tau0 + krep, Tp);   // the group's history so far
                    if (lane == 0) {
                        if (last_fork < 0) x.p2_first[item] = slot;
                        else x.p2_next[last_fork] = slot;
                        a.assign[(size_t)(tau0 + krep) * a.Tpm + li] = (int8_t)dk;   // + its choice
                        P2Hdr fh;
                        fh.g = g;
                        fh.p = p + 1;
                        fh.rep = krep;
                        fh.uf = uf;
                        fh.p_sw = p_sw;
                        fh.pad = 0;
                        fh.mask = take;
                        x.p2_hdr[slot] = fh;
                        __threadfence();
                        atomicExch(x.p2_ready + slot, 1);   // publish
                    }
                    last_fork = slot;
                    __syncwarp();
                }
                // stranded members (feas stays 0): their work
                if (lane < M && ((dead >> lane) & 1ULL)) a.work[tau0 + lane] = wk0;
                if (lane + 32 < M && ((dead >> (lane + 32)) & 1ULL)) a.work[tau0 + lane + 32] = wk1;
                mask = take0;
                cmin = p2_cap_of(cap0, cap1, __ffsll((long long)mask) - 1);
                cmax = p2_cap_of(cap0, cap1, 63 - __clzll((long long)mask));
                const int nrep = __ffsll((long long)mask) - 1;
                if (nrep != rep) {
                    copy_row(tau0 + rep, tau0 + nrep, Tp);
                    rep = nrep;
                    hrow = a.assign + (size_t)(tau0 + rep) * a.Tpm;
                }
            }
            // ---- the group's choice: the owner lane updates its slot jb; this
            // lane records it if step p is its slot of the chunk
            if (lane == ob) {
                switch (jb) {
                    case 0: A4[0] += Bt; ds4[0] += dt; rm4[0] -= bt; break;
                    case 1: A4[1] += Bt; ds4[1] += dt; rm4[1] -= bt; break;
                    case 2: A4[2] += Bt; ds4[2] += dt; rm4[2] -= bt; break;
                    default: A4[3] += Bt; ds4[3] += dt; rm4[3] -= bt; break;
                }
            }
            mybd = lane == k32 ? bd : mybd;
        }
        flush_hist();
        flush_work();
#ifdef NS_WGRP_TIMING
        tc0 = clock64();
        t_loop += (unsigned long long)(tc0 - tc1);
#endif
        // ---- item end: members' work; representative's dims, links of the others, replay entry
        if (lane < M && ((mask >> lane) & 1ULL)) a.work[tau0 + lane] = wk0;
        if (lane + 32 < M && ((mask >> (lane + 32)) & 1ULL)) a.work[tau0 + lane + 32] = wk1;
        if (alive) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int dd = lane + 32 * j;
                if (dd < D) a.devdim[(tau0 + rep) * D + dd] = ds4[j];
            }
            for (int m = lane; m < M; m += 32)
                if ((mask >> m) & 1ULL) {
                    a.feas[tau0 + m] = 1;
                    x.dup_of[tau0 + m] = m == rep ? -1 : (int32_t)(x.tau_base + tau0 + rep);
                }
            __syncwarp();
            for (unsigned long long mm = mask & ~(1ULL << rep); mm; mm &= mm - 1)
                copy_row(tau0 + rep, tau0 + __ffsll((long long)mm) - 1, Tp);
        }
        if (lane == 0) {   // for the replay: the item's representative row and whether it needs comp
            x.p2_rtau[item] = (int32_t)(tau0 + rep);
            x.p2_alive[item] = alive ? 1 : 0;
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(x.p2_q + 2, 1u);   // completed
    }
#ifdef NS_WGRP_TIMING
    if (lane == 0 && (blockIdx.x < 8))
        printf("p2 cta %d warp %d: items %llu steps %llu cycles/step %.0f (keys %.0f W %.0f) claim-wait cycles %llu (n_init %u) "
               "forks %llu at %.2f of the phase-2 span, %.0f steps left\n",
               blockIdx.x, threadIdx.x >> 5, n_items, nsteps, nsteps ? (double)t_loop / nsteps : 0.0,
               nsteps ? (double)t_key / nsteps : 0.0, nsteps ? (double)t_w / nsteps : 0.0, t_claim, n_init, n_fk,
               n_fk ? fk_pos / n_fk : 0.0, n_fk ? fk_rem / n_fk : 0.0);
#endif
    if (lane == 0 && computed) atomicAdd(a.computed, computed);
    if (lane == 0 && computed) atomicAdd(a.computed + 2, computed);   // every phase-2 score is linear
    if (lane == 0 && nsteps) atomicAdd(a.computed + 1, nsteps);
}

// Replay order: the queue's entries bucketed by column plan (counting sort,
// one CTA), so the CTAs replaying at the same time read the same tasks' V rows
// and those stay in L2.  The order within a bucket is immaterial: every
// representative is replayed independently.
constexpr int kRpBuckets = 8192;
__global__ void __launch_bounds__(1024) k_rp_sort(const GreedyArgs a, const WgrpArgs x) {
    __shared__ int cnt[kRpBuckets];
    const unsigned n = __ldcg(x.p2_q + 3);   // families: one per hand-off
    const long long ncp = x.n_cp > 0 ? x.n_cp : 1;
    for (int i = threadIdx.x; i < kRpBuckets; i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    auto bucket = [&](unsigned e) {
        const long long g = x.p2_hdr[e].g;
        return (int)(ncp <= kRpBuckets ? g : g * kRpBuckets / ncp);
    };
    for (unsigned e = threadIdx.x; e < n; e += blockDim.x) atomicAdd(&cnt[bucket(e)], 1);
    __syncthreads();
    // exclusive scan: each thread owns kRpBuckets / 1024 consecutive buckets
    constexpr int per = kRpBuckets / 1024;
    int loc[per], tot = 0;
#pragma unroll
    for (int k = 0; k < per; ++k) {
        loc[k] = cnt[threadIdx.x * per + k];
        tot += loc[k];
    }
    __shared__ int wsum[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        int v = wsum[lane], iv = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(kFull, iv, o);
            if (lane >= o) iv += y;
        }
        wsum[lane] = iv - v;
    }
    __syncthreads();
    int run = wsum[wid] + incl - tot;
#pragma unroll
    for (int k = 0; k < per; ++k) {
        cnt[threadIdx.x * per + k] = run;
        run += loc[k];
    }
    __syncthreads();
    for (unsigned e = threadIdx.x; e < n; e += blockDim.x) x.rp_ord[atomicAdd(&cnt[bucket(e)], 1)] = (int)e;
}

// The representatives of phase-2 groups: u = the frozen u of the hand-off +
// every later placement replayed in step order (the same additions, in the
// same order, the per-trajectory kernel makes), then the head in the order
// of k_greedy_wide88 / k_greedy_wgrp88.  One CTA (NS_RP_WARPS warps) per family -- a
// hand-off and the items forked from it, which share the history before
// their fork step -- walked depth-first: an item's rows are added up to its
// next fork step f, u is saved (snapshot slot of the depth), the fork's
// subtree is walked from f with its own history, u is restored and the item
// continues; an item that ended feasible gets its comp at Tp.  Every
// representative's u is therefore the frozen u plus its own history's rows
// in step order, bit for bit, while the shared prefixes are added once.
// u for all devices lives in shared memory, device-major with a 16-byte
// aligned row stride (kUS); a walk over steps [s0, s1):
//  1. the steps' (row, device) go to shared memory;
//  2. warp w owns the devices d = w (mod NS_RP_WARPS) and lists its steps in order
//     (ballots over the device bytes); it adds each row to u_d with the 32
//     lanes on 2 features each (one coalesced 512-byte row per instruction),
//     the next rows' loads in flight while the current ones are added -- a
//     device's rows stay in step order, so every feature sums in the same
//     order as the sequential greedy.
// The head, one thread per device, is the 8 x 8 order written out -- per
// feature group fg an FMA chain over its 8 features (head88), then the tree
// bfly88 builds for device index j = d & 7:
// ((P_j + P_j^4) + (P_j^2 + P_j^6)) + ((P_j^1 + P_j^5) + (P_j^3 + P_j^7)).
constexpr int kUS = kV + 2;
#ifndef NS_RP_BATCH
#define NS_RP_BATCH 4   // rows in flight per warp of the replay (sweep at 1536 tasks: 8 warps x 4 best; 4 warps x 8: -2%, 16 warps x 2: -1.4%)
#endif
constexpr int kRpBatch = NS_RP_BATCH;
#ifndef NS_RP_WARPS
#define NS_RP_WARPS 8   // warps per replay CTA (devices d = w mod NS_RP_WARPS per warp; 128 registers, small spills)
#endif
constexpr int kRpWarps = NS_RP_WARPS;
// dynamic shared memory of k_greedy_replay; phase 2 is off (no hand-offs)
// when it exceeds the opt-in maximum (Tpm above ~12k column tables)
inline size_t replay_smem(int Tpm) {
    return (size_t)128 * kUS * sizeof(double) + (size_t)Tpm * (sizeof(int2) + 2 * sizeof(int) + 1);
}
constexpr size_t kSmemOptin = 232448;

#ifdef NS_WGRP_TIMING
__device__ unsigned long long g_rp_t[8];   // replay phase cycles summed over CTAs (thread 0)
#define RP_CLK(k, t0) do { if (threadIdx.x == 0) { const long long t1_ = clock64(); atomicAdd(&g_rp_t[k], (unsigned long long)(t1_ - t0)); t0 = t1_; } } while (0)
#else
#define RP_CLK(k, t0) do { } while (0)
#endif
// rows of steps [s0, s1) of one history (hist) added to s_u (CTA-wide); the
// family's row and table index of every step are in srow / stab (indexed by
// step).  Warp w takes the steps whose device is w (mod 4): it counts them,
// then (offsets from the four counts) lists them in step order as (row,
// device offset in s_u) pairs; the devices are gathered from hist twice
// (the second time from L1).
__device__ __forceinline__ void rp_walk(const GreedyArgs& a, double* s_u, const int* srow, const int* stab, int2* slst,
                                        uint8_t* sdev, int* s_wcnt, const int8_t* hist, int s0, int s1) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#ifdef NS_WGRP_TIMING
    long long tq = clock64();
#endif
    __syncthreads();   // the previous walk's lists are consumed
    for (int i0 = s0 + (int)threadIdx.x; i0 < s1; i0 += 4 * blockDim.x) {   // the walk's devices (4 loads in flight)
        int8_t v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int i = i0 + k * blockDim.x;
            v[k] = i < s1 ? __ldcg(hist + stab[i]) : (int8_t)0;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int i = i0 + k * blockDim.x;
            if (i < s1) sdev[i] = (uint8_t)v[k];
        }
    }
    __syncthreads();
    int cnt = 0;
    for (int i = s0 + lane; i - lane < s1; i += 32)
        cnt += __popc(__ballot_sync(kFull, i < s1 && (sdev[i] & (kRpWarps - 1)) == w));
    if (lane == 0) s_wcnt[w] = cnt;
    __syncthreads();
    RP_CLK(1, tq);
    int2* lst = slst;
    for (int v = 0; v < w; ++v) lst += s_wcnt[v];
    {
        int c = 0;
        for (int i = s0 + lane; i - lane < s1; i += 32) {
            const int dv = i < s1 ? (int)sdev[i] : -1;
            const bool mine = i < s1 && (dv & (kRpWarps - 1)) == w;
            const unsigned bm = __ballot_sync(kFull, mine);
            if (mine) lst[c + __popc(bm & ((1u << lane) - 1u))] = make_int2(srow[i], dv * kUS);
            c += __popc(bm);
        }
    }
    __syncwarp();
    RP_CLK(2, tq);
    double2 cur[kRpBatch];
#pragma unroll
    for (int k = 0; k < kRpBatch; ++k)
        if (k < cnt) cur[k] = __ldg(reinterpret_cast<const double2*>(a.V + (size_t)lst[k].x * kV) + lane);
    for (int b0 = 0; b0 < cnt; b0 += kRpBatch) {
        double2 nxt[kRpBatch];
#pragma unroll
        for (int k = 0; k < kRpBatch; ++k)
            if (b0 + kRpBatch + k < cnt)
                nxt[k] = __ldg(reinterpret_cast<const double2*>(a.V + (size_t)lst[b0 + kRpBatch + k].x * kV) + lane);
#pragma unroll
        for (int k = 0; k < kRpBatch; ++k)
            if (b0 + k < cnt) {
                double2* p = reinterpret_cast<double2*>(s_u + lst[b0 + k].y) + lane;
                double2 t = *p;
                t.x += cur[k].x;
                t.y += cur[k].y;
                *p = t;
            }
#pragma unroll
        for (int k = 0; k < kRpBatch; ++k) cur[k] = nxt[k];
    }
    RP_CLK(3, tq);
    __syncthreads();
    RP_CLK(4, tq);
}

// u (s_u rows) <-> a snapshot slot [128][64] in global memory (CTA-wide, coalesced)
__device__ __forceinline__ void rp_save(const double* s_u, double* snap) {
    __syncthreads();
    for (int i = threadIdx.x; i < 128 * kV / 2; i += blockDim.x) {
        const int d = i / (kV / 2), k2 = i % (kV / 2);
        __stcg(reinterpret_cast<double2*>(snap) + i, reinterpret_cast<const double2*>(s_u + d * kUS)[k2]);
    }
}
__device__ __forceinline__ void rp_load(double* s_u, const double* snap) {
    __syncthreads();
    constexpr int KL = 64 / kRpWarps;   // loads in flight per thread (16 at 4 warps)
    for (int i0 = threadIdx.x; i0 < 128 * kV / 2; i0 += KL * blockDim.x) {
        double2 v[KL];
#pragma unroll
        for (int k = 0; k < KL; ++k) {
            const int i = i0 + k * blockDim.x;
            if (i < 128 * kV / 2) v[k] = __ldcg(reinterpret_cast<const double2*>(snap) + i);
        }
#pragma unroll
        for (int k = 0; k < KL; ++k) {
            const int i = i0 + k * blockDim.x;
            if (i < 128 * kV / 2) reinterpret_cast<double2*>(s_u + (i / (kV / 2)) * kUS)[i % (kV / 2)] = v[k];
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(32 * kRpWarps, 2) k_greedy_replay(const GreedyArgs a, const WgrpArgs x) {
    // [128][kUS] u, then [Tpm] (row, device offset) step lists, [Tpm] rows and [Tpm] table indices of the steps
    extern __shared__ __align__(16) double s_u[];
    __shared__ int stk_item[64], stk_pos[64], stk_fork[64];   // DFS stack: item, step reached, its next fork
    __shared__ int s_wcnt[kRpWarps];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const unsigned n = __ldcg(x.p2_q + 3);   // families (hand-offs)
    unsigned long long rows = 0, reps = 0;   // ns_stats: rows replayed, representatives
    int2* slst = reinterpret_cast<int2*>(s_u + 128 * kUS);
    int* srow = reinterpret_cast<int*>(slst + a.Tpm);
    int* stab = srow + a.Tpm;
    uint8_t* sdev = reinterpret_cast<uint8_t*>(stab + a.Tpm);   // indexed by step
    double* snap = x.rp_snap + (size_t)blockIdx.x * a.M * 128 * kV;
    __shared__ unsigned s_claim;
#ifdef NS_WGRP_TIMING
    long long t_start = clock64(), t_busy = 0;
    unsigned n_fam = 0;
#endif
    for (;;) {
        __syncthreads();   // the previous family's head has read s_u, s_claim consumed
        if (tid == 0) s_claim = atomicAdd(x.p2_q + 6, 1u);   // families claimed in order (dynamic balance)
        __syncthreads();
        const unsigned e0 = s_claim;
        if (e0 >= n) break;
        const int root = __ldcg(x.rp_ord + e0);
        if (!__ldcg(x.p2_alive + root) && __ldcg(x.p2_first + root) < 0) continue;   // stranded, no forks
        const P2Hdr h = x.p2_hdr[root];
        const int g = h.g;
        const int Tp = a.cp_Tp[g];
        const int32_t* orow = a.ord_row + (size_t)g * a.Tpm;
        const int4* ometa = a.ord_meta + (size_t)g * a.Tpm;
#ifdef NS_WGRP_TIMING
        const long long tf0 = clock64();
        ++n_fam;
#endif
        // the family's steps (shared by all its items): V row and table index
        for (int i = h.p_sw + tid; i < Tp; i += blockDim.x) {
            srow[i] = __ldg(orow + i);
            stab[i] = __ldg(ometa + i).y;
        }
        {
            // frozen u: uf_buf element (j = jd * 8 + q, c = 32 wgi + 8 dgi + fg) is feature
            // 8 fg + q of device 32 wgi + 8 dgi + jd; a warp instruction covers one device's 32 features
            const double* up = x.uf_buf + (size_t)h.uf * kV * 128;
            const int q = lane & 7, fgl = lane >> 3;
            constexpr int KK = 128 / kRpWarps;   // loads in flight per thread
            for (int it0 = w; it0 < 256; it0 += kRpWarps * KK) {
                double vv[KK];
#pragma unroll
                for (int k = 0; k < KK; ++k) {
                    const int it = it0 + kRpWarps * k, d = it >> 1, fg = 4 * (it & 1) + fgl;
                    vv[k] = __ldcg(up + (size_t)((d & 7) * 8 + q) * 128 + (d & ~7) + fg);
                }
#pragma unroll
                for (int k = 0; k < KK; ++k) {
                    const int it = it0 + kRpWarps * k, d = it >> 1, fg = 4 * (it & 1) + fgl;
                    s_u[d * kUS + 8 * fg + q] = vv[k];
                }
            }
        }
        int item = root, pos = h.p_sw, fork = __ldcg(x.p2_first + root), depth = 0;
        for (;;) {
            const bool alive = __ldcg(x.p2_alive + item) != 0;
            const int target = fork >= 0 ? x.p2_hdr[fork].p - 1 : (alive ? Tp : pos);
            const long long rtau = __ldcg(x.p2_rtau + item);
            if (target > pos) {
                rp_walk(a, s_u, srow, stab, slst, sdev, s_wcnt, a.assign + (size_t)rtau * a.Tpm, pos, target);
                rows += (unsigned long long)(target - pos);
                pos = target;
            }
            if (fork >= 0) {   // descend: save u at the fork step, walk the fork from there
#ifdef NS_WGRP_TIMING
                long long tq = clock64();
#endif
                rp_save(s_u, snap + (size_t)depth * 128 * kV);
                RP_CLK(5, tq);
                if (tid == 0) {
                    stk_item[depth] = item;
                    stk_pos[depth] = pos;
                    stk_fork[depth] = __ldcg(x.p2_next + fork);
                }
                ++depth;
                item = fork;
                fork = __ldcg(x.p2_first + item);
                continue;
            }
            if (alive) {   // head, one thread per device
                __syncthreads();
                const int d = tid;
                if (d < a.D) {
                    const double* ud = s_u + d * kUS;
                    double P[8];
#pragma unroll
                    for (int fg = 0; fg < 8; ++fg) {
                        double acc = 0.0;
#pragma unroll
                        for (int q2 = 0; q2 < kG8; ++q2) acc = fma(a.head.H2[kG8 * fg + q2], relu_exact(ud[kG8 * fg + q2]), acc);
                        P[fg] = acc;
                    }
                    const int jd = d & 7;
                    double t[8];   // t[b] = P_{j ^ b}: three rounds of register swaps (no local memory)
#pragma unroll
                    for (int b = 0; b < 8; ++b) t[b] = P[b];
#pragma unroll
                    for (int bit = 1; bit < 8; bit <<= 1) {
                        const bool sw = (jd & bit) != 0;
#pragma unroll
                        for (int b = 0; b < 8; ++b)
                            if (!(b & bit)) {
                                const double lo = t[b], hi = t[b | bit];
                                t[b] = sw ? hi : lo;
                                t[b | bit] = sw ? lo : hi;
                            }
                    }
                    const double s3 = ((t[0] + t[4]) + (t[2] + t[6])) + ((t[1] + t[5]) + (t[3] + t[7]));
                    const int ds = a.devdim[rtau * a.D + d];
                    a.comp[rtau * a.D + d] = ds > 0 ? a.head.hb2 + s3 : 0.0;   // reading R4
                }
                ++reps;
            }
            if (depth == 0) break;
            // ascend: the parent's u at the fork step, its next fork
            --depth;
            __syncthreads();   // stack entries written by thread 0 are visible
            item = stk_item[depth];
            pos = stk_pos[depth];
            fork = stk_fork[depth];
#ifdef NS_WGRP_TIMING
            long long tq = clock64();
#endif
            rp_load(s_u, snap + (size_t)depth * 128 * kV);
            RP_CLK(6, tq);
        }
#ifdef NS_WGRP_TIMING
        t_busy += clock64() - tf0;
#endif
    }
#ifdef NS_WGRP_TIMING
    if (tid == 0 && (blockIdx.x % 37) == 0)
        printf("replay cta %d: families %u rows %llu reps %llu busy %lld of %lld cycles\n", blockIdx.x, n_fam, rows, reps,
               t_busy, clock64() - t_start);
    if (tid == 0 && blockIdx.x == 0) {   // sums of the previous launch (this one is still running)
        printf("replay phases (all CTAs, prev launch): sync0 %llu fill %llu lists %llu adds %llu sync1 %llu save %llu load %llu\n",
               g_rp_t[0], g_rp_t[1], g_rp_t[2], g_rp_t[3], g_rp_t[4], g_rp_t[5], g_rp_t[6]);
    }
#endif
    if (tid == 0 && (reps || rows)) {
        atomicAdd(a.computed + 3, rows);
        atomicAdd(a.computed + 4, reps);
    }
}

// ======================================================================
// N6: per task, grid argmin of every child column plan (Alg. 2 lines 16-18,
// reading R12: lowest m on ties), work totals, global best with strict < in
// generation order (Alg. 1 lines 13-16), next beam = K lowest (cost, gen)
// (Alg. 1 line 20; R13, R16).  One CTA per task.
// ======================================================================
// Level 0 (one column plan per task, C = 1): one warp per task.  The grid
// argmin (lowest m on ties, R12) is reduced with shuffles; level 0 always
// installs [] as the initial global best (R15).
// Pack per-task results into the contiguous staging layout.
struct OutStage {
    double* cost;
    int32_t* n_col;
    int32_t* col_plan;   // [n][Lout]
    int8_t* assign;      // [n][astride]: columns >= Tpm are -1
    int astride;
    int32_t* grid;
    uint64_t* scores;
    // which fields point straight at the caller's device buffers (no copy in deliver)
    bool d_cost, d_ncol, d_plan, d_assign, d_grid, d_scores;
};

// final_out (table-wise search, L = 0): level 0 is the whole search, so the
// warp also packs the task's outputs (k_write_out's job) -- one launch less.
__global__ void __launch_bounds__(256) k_select0(SearchBufs b, OutStage o, int final_out) {
    const int lane = threadIdx.x & 31;
    for (int q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < b.n_tasks; q += (gridDim.x * blockDim.x) >> 5) {
        unsigned long long wsum = 0;
        double best = CUDART_INF;
        int bm = INT_MAX;
        for (int m = lane; m < b.M; m += 32) {
            const long long tau = (long long)q * b.M + m;
            wsum += b.work[tau];
            const long long src = b.dup_of[tau] >= 0 ? (long long)b.dup_of[tau] : tau;
            const double c = b.feas[tau] ? b.tcost[src] : CUDART_INF;
            if (c < best) {   // m increases per lane: strict < keeps the lowest m
                best = c;
                bm = m;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            wsum += __shfl_xor_sync(kFull, wsum, o);
            const double ob = __shfl_xor_sync(kFull, best, o);
            const int om = __shfl_xor_sync(kFull, bm, o);
            if (ob < best || (ob == best && om < bm)) {
                best = ob;
                bm = om;
            }
        }
        if (best == CUDART_INF) bm = -1;
        if (lane == 0) {
            const unsigned long long sc = b.n_scores[q] + wsum;
            b.n_scores[q] = sc;
            b.best_cost[q] = best;
            b.best_m[q] = bm;
            b.best_ncol[q] = 0;
            b.beam_cnt[q] = 1;   // C_p <- {[]}
            if (final_out) {
                o.cost[q] = best;
                o.n_col[q] = 0;
                o.grid[q] = bm;
                o.scores[q] = sc;
                o.col_plan[q] = -1;   // Lout = 1 slot, no split
            }
        }
        const int Tp = b.cp_Tp[q];
        long long src = -1;
        if (bm >= 0) {
            const long long tau = (long long)q * b.M + bm;
            src = b.dup_of[tau] >= 0 ? (long long)b.dup_of[tau] : tau;
        }
        // multi-rank: another rank owns the row -> -128 here, the int8
        // allreduce-max after the search fills in the owner's values
        const bool own = q >= b.own_cb && q < b.own_ce;
        if (final_out) {
            for (int i = lane; i < o.astride; i += 32)
                o.assign[(size_t)q * o.astride + i] =
                    (src >= 0 && i < Tp && i < b.Tpm) ? (own ? b.assign[src * b.Tpm + i] : (int8_t)-128) : (int8_t)-1;
        } else {
            for (int i = lane; i < b.Tpm; i += 32)
                b.best_assign[(size_t)q * b.Tpm + i] =
                    (src >= 0 && i < Tp) ? (own ? b.assign[src * b.Tpm + i] : (int8_t)-128) : (int8_t)-1;
        }
    }
}

__global__ void __launch_bounds__(256) k_select(SearchBufs b, int C, int level, int Kbeam, int staged) {
    extern __shared__ unsigned char ssm[];
    const int q = blockIdx.x;
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double* ccost = (double*)ssm;                    // [C]
    int32_t* cm = (int32_t*)(ccost + C);             // [C]
    int32_t* cval = cm + C;                          // [C]
    double* tc = (double*)(cval + C + (C & 1));      // [C][M] trajectory costs (staged mode)
    __shared__ unsigned long long s_work[32];
    __shared__ double s_bc[32];
    __shared__ int s_bj[32], s_nv[32];
    __shared__ int s_best, s_nvalid;
    // ---- grid argmin of every child column plan: one warp per child, lanes over m
    unsigned long long wsum = 0;
    if (staged) {
        // every (child, m) cost gathered in parallel first (the dependent
        // dup_of -> tcost loads of all trajectories in flight at once)
        const long long t0 = (long long)q * C * b.M;
        for (int e = threadIdx.x; e < C * b.M; e += blockDim.x) {
            const long long tau = t0 + e;
            double c = CUDART_INF;
            if (b.cp_valid[q * C + e / b.M]) {
                wsum += b.work[tau];
                const long long src = b.dup_of[tau] >= 0 ? (long long)b.dup_of[tau] : tau;
                if (b.feas[tau]) c = b.tcost[src];
            }
            tc[e] = c;
        }
        __syncthreads();
    }
    double wbc = CUDART_INF;   // this warp's lexicographic (cost, generation) minimum over valid children
    int wbj = INT_MAX, wnv = 0;
    for (int j = wi; j < C; j += nw) {
        const int g = q * C + j;
        const int v = b.cp_valid[g];
        double best = CUDART_INF;
        int bm = INT_MAX;
        if (v) {
            for (int m = lane; m < b.M; m += 32) {
                double c;
                if (staged) {
                    c = tc[j * b.M + m];
                } else {
                    const long long tau = (long long)g * b.M + m;
                    wsum += b.work[tau];
                    const long long src = b.dup_of[tau] >= 0 ? (long long)b.dup_of[tau] : tau;
                    c = b.feas[tau] ? b.tcost[src] : CUDART_INF;
                }
                if (c < best) {   // m increases per lane: strict < keeps the lowest m
                    best = c;
                    bm = m;
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(kFull, best, o);
            const int om = __shfl_xor_sync(kFull, bm, o);
            if (ob < best || (ob == best && om < bm)) {
                best = ob;
                bm = om;
            }
        }
        if (best == CUDART_INF) bm = -1;
        if (lane == 0) {
            ccost[j] = best;
            cm[j] = bm;
            cval[j] = v;
        }
        if (v) {
            ++wnv;
            if (best < wbc || (best == wbc && j < wbj)) {
                wbc = best;
                wbj = j;
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) wsum += __shfl_xor_sync(kFull, wsum, o);
    if (lane == 0) {
        s_work[wi] = wsum;
        s_bc[wi] = wbc;
        s_bj[wi] = wbj;
        s_nv[wi] = wnv;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long work = 0;
        int arg = INT_MAX, nvalid = 0;
        double ac = CUDART_INF;
        for (int k = 0; k < nw; ++k) {
            work += s_work[k];
            nvalid += s_nv[k];
            if (s_bj[k] != INT_MAX && (s_bc[k] < ac || (s_bc[k] == ac && s_bj[k] < arg))) {
                ac = s_bc[k];
                arg = s_bj[k];
            }
        }
        b.n_scores[q] += work;
        s_nvalid = nvalid;
        // lexicographic (cost, gen) minimum of the level == the first strict
        // improvement in generation order
        s_best = -1;
        if (arg != INT_MAX && (level == 0 || ccost[arg] < b.best_cost[q])) {
            // level 0 always installs [] as the initial global best (R15)
            s_best = arg;
            b.best_cost[q] = ccost[arg];
            b.best_m[q] = cm[arg];
            b.best_ncol[q] = level;
            const int g = q * C + arg;
            for (int k = 0; k < level; ++k) b.best_plan[(size_t)q * b.Lcap + k] = b.cp_plan[(size_t)g * b.Lcap + k];
        }
        if (level == 0) b.beam_cnt[q] = 1;   // C_p <- {[]}
    }
    __syncthreads();
    if (s_best >= 0) {
        const int g = q * C + s_best;
        const int Tp = b.cp_Tp[g];
        const int mm = cm[s_best];
        long long src = -1;
        if (mm >= 0) {
            const long long tau = (long long)g * b.M + mm;
            src = b.dup_of[tau] >= 0 ? (long long)b.dup_of[tau] : tau;
        }
        const bool own = g >= b.own_cb && g < b.own_ce;
        for (int i = threadIdx.x; i < b.Tpm; i += blockDim.x)
            b.best_assign[(size_t)q * b.Tpm + i] =
                (src >= 0 && i < Tp) ? (own ? b.assign[src * b.Tpm + i] : (int8_t)-128) : (int8_t)-1;
    }
    if (level > 0) {
        // next beam: rank among valid children by (cost, gen); one warp per child
        for (int j = wi; j < C; j += nw) {
            if (!cval[j]) continue;
            const double cj = ccost[j];
            int r = 0;
            for (int k0 = 0; k0 < C; k0 += 32) {
                const int k = k0 + lane;
                const bool less = k < C && cval[k] && (ccost[k] < cj || (ccost[k] == cj && k < j));
                r += __popc(__ballot_sync(kFull, less));
            }
            if (r < Kbeam) {
                const int g = q * C + j;
                for (int k = lane; k < level; k += 32)
                    b.beam_plan[((size_t)q * b.K + r) * b.Lcap + k] = b.cp_plan[(size_t)g * b.Lcap + k];
                if (lane == 0) b.beam_slot[q * b.K + r] = g;   // its cost order: the next level's parent
            }
        }
        if (threadIdx.x == 0) b.beam_cnt[q] = s_nvalid < Kbeam ? s_nvalid : Kbeam;
    }
}

// Grid of max_dim caps (reading R8): M_s = sum(dim)/D,
// M_e = hi*M_s, step = (M_e - M_s)/(M-1), cap_m = floor(M_s + m*step).  Each
// operation is one IEEE-rounded fp64 op (explicit _rn intrinsics, no
// contraction), the operation order stated in DESIGN.md R8.
__global__ void k_grid_caps(const int64_t* sumdim, int n_tasks, int D, int M, double hi, int32_t* capdim) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_tasks * M) return;
    const int q = i / M, m = i % M;
    if (hi < 0.0) {   // NS_NO_DIM_CAP
        capdim[i] = 2000000000;
        return;
    }
    const double Ms = __ddiv_rn((double)sumdim[q], (double)D);
    double md = Ms;
    if (M > 1) {
        const double Me = __dmul_rn(hi, Ms);
        const double step = __ddiv_rn(__dsub_rn(Me, Ms), (double)(M - 1));
        md = __dadd_rn(Ms, __dmul_rn((double)m, step));
    }
    const double f = floor(md);
    capdim[i] = f > 2.0e9 ? 2000000000 : (int32_t)f;
}


// Multi-rank consistency check: per task the packed key
// (order-preserving bits of the best cost, FNV-1a hash of (column plan, grid
// index)) and its complement; after an allreduce-min over the ranks, key ==
// min and ~key == min(~key) (i.e. key == max) on every rank iff all ranks
// selected the same plan.  mode 0 builds the keys, mode 1 checks them.
__device__ __forceinline__ unsigned long long order_key64(double c) {
    const long long sb = __double_as_longlong(c + 0.0);
    return (unsigned long long)(sb ^ ((sb >> 63) | (long long)0x8000000000000000ULL));
}

__global__ void k_rank_check(SearchBufs b, int mode, int32_t* flag) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= b.n_tasks) return;
    const unsigned long long k0 = order_key64(b.best_cost[q]);
    unsigned long long h = 1469598103934665603ULL;
    auto mix = [&](unsigned long long v) {
        for (int i = 0; i < 4; ++i) {
            h ^= (v >> (16 * i)) & 0xffffULL;
            h *= 1099511628211ULL;
        }
    };
    const int nc = b.best_ncol[q];
    mix((unsigned long long)(unsigned)nc);
    mix((unsigned long long)(unsigned)b.best_m[q]);
    for (int k = 0; k < nc; ++k) mix((unsigned long long)(unsigned)b.best_plan[(size_t)q * b.Lcap + k]);
    uint64_t* key = b.rank_keys + 4 * (size_t)q;
    if (mode == 0) {
        key[0] = k0;
        key[1] = h;
        key[2] = ~k0;
        key[3] = ~h;
    } else if (key[0] != k0 || key[1] != h || key[2] != ~k0 || key[3] != ~h) {
        atomicOr(flag, 2);
    }
}

__global__ void __launch_bounds__(256) k_write_out(SearchBufs b, OutStage o, int Lout) {
    const int lane = threadIdx.x & 31;
    for (int q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < b.n_tasks; q += (gridDim.x * blockDim.x) >> 5) {
        const bool feasible = b.best_cost[q] < CUDART_INF;
        const int ncol = b.best_ncol[q];
        if (lane == 0) {
            o.cost[q] = b.best_cost[q];
            o.n_col[q] = ncol;
            o.grid[q] = feasible ? b.best_m[q] : -1;
            o.scores[q] = b.n_scores[q];
        }
        for (int k = lane; k < Lout; k += 32)
            o.col_plan[(size_t)q * Lout + k] = k < ncol ? b.best_plan[(size_t)q * b.Lcap + k] : -1;
        for (int i = lane; i < o.astride; i += 32)
            o.assign[(size_t)q * o.astride + i] =
                (feasible && i < b.Tpm) ? b.best_assign[(size_t)q * b.Tpm + i] : (int8_t)-1;
    }
}

// ======================================================================
// Host driver
// ======================================================================
namespace {

struct Carver {
    char* base;
    size_t off = 0;
    template <typename T>
    T* take(size_t n) {
        off = (off + 255) & ~size_t(255);
        T* p = base ? (T*)(base + off) : nullptr;
        off += n * sizeof(T);
        return p;
    }
};

static unsigned int* base_counter(int32_t* pair) { return reinterpret_cast<unsigned int*>(pair + 1); }

void carve(Carver& c, SearchBufs& b, OutStage& o, int Lout) {
    b.cp_task = c.take<int32_t>(b.S);
    b.cp_valid = c.take<int32_t>(b.S);
    b.cp_len = c.take<int32_t>(b.S);
    b.cp_plan = c.take<int32_t>((size_t)b.S * b.Lcap);
    b.cp_Tp = c.take<int32_t>(b.S);
    b.ord_row = c.take<int32_t>((size_t)b.S * b.Tpm);
    b.ord_meta = c.take<int4>((size_t)b.S * b.Tpm);
    // the second order buffer of the incremental (merge) orders: long lists, beam levels
    const bool merge_orders = b.Tpm > 256 && b.Lcap > 0 && b.S > b.n_tasks;
    b.ord_row2 = merge_orders ? c.take<int32_t>((size_t)b.S * b.Tpm) : nullptr;
    b.ord_meta2 = merge_orders ? c.take<int4>((size_t)b.S * b.Tpm) : nullptr;
    b.beam_slot = c.take<int32_t>((size_t)b.n_tasks * b.K);
    b.assign = c.take<int8_t>((size_t)b.n_traj * b.Tpm);
    b.comp = c.take<double>((size_t)b.n_traj * b.D);
    b.devdim = c.take<int32_t>((size_t)b.n_traj * b.D);
    b.feas = c.take<uint8_t>(b.n_traj);
    b.work = c.take<uint32_t>(b.n_traj);
    b.tcost = c.take<double>(b.n_traj);
    b.dup_of = c.take<int32_t>(b.n_traj);
    b.uniq = c.take<int32_t>(b.n_traj);
    {   // the two per-launch counters are adjacent: one memset clears both
        int32_t* ctr = c.take<int32_t>(2);
        b.n_uniq = ctr;
        b.next_cp = base_counter(ctr);
    }
    b.gscratch = c.take<double>((size_t)b.gscratch_warps * b.M * b.D * kV);
    {
        const size_t items = b.wgrp ? (size_t)b.wgrp_cp_cap * b.M : 0;
        b.wsnap = c.take<double>(items * b.wsnap_doubles);
        b.wq = reinterpret_cast<WgrpQueue*>(c.take<unsigned int>(4));
        b.witem_cp = c.take<int32_t>(items);
        b.witem_step = c.take<int32_t>(items);
        b.witem_mask = c.take<unsigned long long>(items);
        b.witem_ready = c.take<int32_t>(items);
        b.p2_cap = (int)items;
        b.uf_cap = b.wgrp && replay_smem(b.Tpm) <= kSmemOptin ? 2 * b.wgrp_cp_cap : 0;
        b.p2_hdr = reinterpret_cast<P2Hdr*>(c.take<long long>((size_t)b.p2_cap * 4));
        b.p2_work = c.take<uint32_t>((size_t)b.p2_cap * 64);
        b.p2_A = c.take<double>((size_t)b.p2_cap * 128);
        b.p2_room = c.take<long long>((size_t)b.p2_cap * 128);
        b.p2_dsum = c.take<int32_t>((size_t)b.p2_cap * 128);
        b.p2_ready = c.take<int32_t>((size_t)b.p2_cap);
        b.p2_q = c.take<unsigned int>(8);
        b.uf_buf = c.take<double>((size_t)b.uf_cap * kV * 128);
        b.rp_ord = c.take<int32_t>((size_t)b.p2_cap);
        b.p2_first = c.take<int32_t>((size_t)b.p2_cap);
        b.p2_next = c.take<int32_t>((size_t)b.p2_cap);
        b.p2_rtau = c.take<int32_t>((size_t)b.p2_cap);
        b.p2_alive = c.take<uint8_t>((size_t)b.p2_cap);
        b.rp_snap = c.take<double>(b.uf_cap ? (size_t)b.rp_ctas * b.M * 128 * kV : 0);
    }
    b.ghist = c.take<int8_t>((size_t)b.gscratch_warps * b.M * b.Tpm);
    b.capdim = c.take<int32_t>((size_t)b.n_tasks * b.M);
    b.vmin = c.take<double>((size_t)b.n_tasks * kV);
    b.Brow = c.take<double>((size_t)b.n_rows_lin);
    b.beam_plan = c.take<int32_t>((size_t)b.n_tasks * b.K * b.Lcap);
    b.beam_cnt = c.take<int32_t>(b.n_tasks);
    b.best_cost = c.take<double>(b.n_tasks);
    b.best_m = c.take<int32_t>(b.n_tasks);
    b.best_ncol = c.take<int32_t>(b.n_tasks);
    b.best_plan = c.take<int32_t>((size_t)b.n_tasks * b.Lcap);
    b.best_assign = c.take<int8_t>((size_t)b.n_tasks * b.Tpm);
    b.n_scores = c.take<uint64_t>(b.n_tasks);
    b.rank_keys = c.take<uint64_t>((size_t)b.n_tasks * 4);
    o.cost = c.take<double>(b.n_tasks);
    o.n_col = c.take<int32_t>(b.n_tasks);
    o.col_plan = c.take<int32_t>((size_t)b.n_tasks * Lout);
    o.assign = c.take<int8_t>((size_t)b.n_tasks * b.Tpm);
    o.astride = b.Tpm;
    o.grid = c.take<int32_t>(b.n_tasks);
    o.scores = c.take<uint64_t>(b.n_tasks);
}

TaskView task_view(const ns_tables* t) {
    TaskView tv;
    tv.off = t->d_off;
    tv.cap = t->d_cap;
    tv.V = t->d_V;
    tv.C = t->d_C;
    tv.vdim = t->d_vdim;
    tv.vbytes = t->d_vbytes;
    return tv;
}

size_t order_smem(int Tpm) { return ((size_t)((Tpm + 1) & ~1)) * 4 + (size_t)Tpm * 8; }

ns_status launch_greedy(ns_ctx* ctx, const SearchBufs& b, const ns_tables* t, long long tb, long long te) {
    // one memset per (greedy, finalize) pair: the grouped greedy's queue
    // counter and the compaction counter of the finalize that follows
    NS_CUDA(ctx, cudaMemsetAsync(b.n_uniq, 0, 2 * sizeof(int32_t), ctx->stream));
    if (te <= tb) return NS_OK;
    GreedyArgs a;
    a.traj_begin = (int)tb;
    a.traj_end = (int)te;
    a.n_rows = (long long)t->n_tables * kDepth;
    a.M = b.M;
    a.D = b.D;
    a.Tpm = b.Tpm;
    a.cp_valid = b.cp_valid;
    a.cp_task = b.cp_task;
    a.cp_Tp = b.cp_Tp;
    a.ord_row = b.ord_row;
    a.ord_meta = b.ord_meta;
    a.capdim = b.capdim;
    a.cap = t->d_cap;
    a.V = t->d_V;
    a.vdim = t->d_vdim;
    a.vbytes = t->d_vbytes;
    a.vmin = b.vmin;
    a.Brow = b.Brow;
    a.assign = b.assign;
    a.comp = b.comp;
    a.devdim = b.devdim;
    a.feas = b.feas;
    a.work = b.work;
    a.computed = ctx->d_stats;
    a.head = ctx->model.head;
    ctx->trajectories += (uint64_t)(te - tb);
    const long long n = te - tb;
    int dp = 1;
    while (dp < b.D) dp <<= 1;
    const long long n_cp_launch = (te - tb) / b.M;
    // Latency mode: with few column plans (a single-task column-wise search)
    // one warp per column plan leaves most SMs idle and the step chain is the
    // critical path, so every trajectory runs in its own lane segment
    // (k_greedy_cta).  Throughput mode (many column plans): grouped greedy.
    // Both kernels split a device's 64 features over the same LPD = 32 / dp
    // lanes and sum them in the same order, so their scores -- hence their
    // decisions and plan costs -- are bit-identical: a task's result does not
    // depend on the batch (kernel) it runs in.
    const bool latency_mode =
        dp <= 16 && (b.greedy_mode == NS_GREEDY_LANES || b.M > 64 ||   // grouped kernel: M <= 64
                     (b.greedy_mode == NS_GREEDY_AUTO && n_cp_launch * 4 < (long long)ctx->sm_count * 16));
    if (latency_mode) {
        const int seg = 32;   // one trajectory per warp, LPD = 32 / dp lanes per device
        const int mchunk = std::min(b.M, 256 / seg);
        const int nchunk = (b.M + mchunk - 1) / mchunk;
        const int threads = ((mchunk * seg + 31) / 32) * 32;
        const long long g0 = tb / b.M, g1 = (te - 1) / b.M + 1;
        GreedyArgs a2 = a;
        a2.ord_row = b.ord_row + (size_t)g0 * b.Tpm;
        a2.ord_meta = b.ord_meta + (size_t)g0 * b.Tpm;
        a2.cp_valid = b.cp_valid + g0;
        a2.cp_task = b.cp_task + g0;
        a2.cp_Tp = b.cp_Tp + g0;
        a2.traj_begin = (int)(tb - g0 * b.M);
        a2.traj_end = (int)(te - g0 * b.M);
        a2.assign = b.assign + (size_t)g0 * b.M * b.Tpm;
        a2.comp = b.comp + (size_t)g0 * b.M * b.D;
        a2.devdim = b.devdim + (size_t)g0 * b.M * b.D;
        a2.feas = b.feas + (size_t)g0 * b.M;
        a2.work = b.work + (size_t)g0 * b.M;
        const unsigned blocks = (unsigned)((g1 - g0) * nchunk);
        prof_begin(ctx, PK_GREEDY);
        switch (dp) {
            case 1: k_greedy_cta<32, 32><<<blocks, threads, 0, ctx->stream>>>(a2, mchunk, nchunk); break;
            case 2: k_greedy_cta<32, 16><<<blocks, threads, 0, ctx->stream>>>(a2, mchunk, nchunk); break;
            case 4: k_greedy_cta<32, 8><<<blocks, threads, 0, ctx->stream>>>(a2, mchunk, nchunk); break;
            case 8: k_greedy_cta<32, 4><<<blocks, threads, 0, ctx->stream>>>(a2, mchunk, nchunk); break;
            default: k_greedy_cta<32, 2><<<blocks, threads, 0, ctx->stream>>>(a2, mchunk, nchunk); break;
        }
        prof_end(ctx);
        NS_CUDA(ctx, cudaMemsetAsync(b.dup_of + tb, 0xff, (size_t)n * sizeof(int32_t), ctx->stream));
    } else if (dp <= 16 && b.M <= 64) {
        // grouped greedy: one warp per column plan (trajectories [tb, te) are
        // whole column plans: tb, te multiples of M)
        const long long g0 = tb / b.M, g1 = te / b.M;
        GreedyArgs a2 = a;
        a2.ord_row = b.ord_row + (size_t)g0 * b.Tpm;
        a2.ord_meta = b.ord_meta + (size_t)g0 * b.Tpm;
        a2.cp_valid = b.cp_valid + g0;
        a2.cp_task = b.cp_task + g0;
        a2.cp_Tp = b.cp_Tp + g0;
        a2.assign = b.assign + (size_t)g0 * b.M * b.Tpm;
        a2.comp = b.comp + (size_t)g0 * b.M * b.D;
        a2.devdim = b.devdim + (size_t)g0 * b.M * b.D;
        a2.feas = b.feas + (size_t)g0 * b.M;
        a2.work = b.work + (size_t)g0 * b.M;
        DedupArgs x;
        x.n_cp = (int)(g1 - g0);
        x.mmax = b.M;
        x.scratch = b.gscratch;
        x.hist = b.ghist;
        x.total_warps = (int)std::min<long long>(x.n_cp, (long long)b.gscratch_warps);
        x.dup_of = b.dup_of + (size_t)g0 * b.M;
        x.tau_base = g0 * b.M;
        x.next_cp = b.next_cp;
        const int lpd = 32 / dp;
        const int mc = b.M <= 16 ? 16 : 64;
        const int wpb = NS_DEDUP_WPB;
        unsigned blocks = 0;
        prof_begin(ctx, PK_GREEDY);
        switch (lpd * 1000 + mc) {
#define NS_DEDUP(L, MC)                                                                                  \
    case L * 1000 + MC: {                                                                                \
        const size_t smem = sizeof(DedupSmem<L, MC>) * wpb;                                              \
        blocks = (unsigned)((x.total_warps + wpb - 1) / wpb);                                            \
        x.total_warps = (int)blocks * wpb; /* every launched warp strides the column plans */            \
        if (smem + 2048 > 48 * 1024) /* + the static s_hb1, s_wp */                                     \
            cudaFuncSetAttribute(k_greedy_dedup<L, MC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        k_greedy_dedup<L, MC><<<blocks, wpb * 32, smem, ctx->stream>>>(a2, x);                           \
        break;                                                                                           \
    }
            NS_DEDUP(2, 16)
            NS_DEDUP(4, 16)
            NS_DEDUP(8, 16)
            NS_DEDUP(16, 16)
            NS_DEDUP(32, 16)
            NS_DEDUP(2, 64)
            NS_DEDUP(4, 64)
            NS_DEDUP(8, 64)
            NS_DEDUP(16, 64)
            NS_DEDUP(32, 64)
#undef NS_DEDUP
            default: return set_err(ctx, NS_ERR_INTERNAL, "bad greedy lane split");
        }
        prof_end(ctx);
    } else if (b.wgrp &&
               (b.greedy_mode == NS_GREEDY_GROUPED || n_cp_launch >= NS_WGRP_MIN_CP)) {
        // large D, many column plans: grouped trajectories (k_greedy_wgrp88)
        const int threads = ((b.D + 31) / 32) * 32;   // one warp per 32 devices (8 x 8 layout)
        const long long g0 = tb / b.M, g1 = te / b.M;
        GreedyArgs a2 = a;
        a2.ord_row = b.ord_row + (size_t)g0 * b.Tpm;
        a2.ord_meta = b.ord_meta + (size_t)g0 * b.Tpm;
        a2.cp_valid = b.cp_valid + g0;
        a2.cp_task = b.cp_task + g0;
        a2.cp_Tp = b.cp_Tp + g0;
        a2.assign = b.assign + (size_t)g0 * b.M * b.Tpm;
        a2.comp = b.comp + (size_t)g0 * b.M * b.D;
        a2.devdim = b.devdim + (size_t)g0 * b.M * b.D;
        a2.feas = b.feas + (size_t)g0 * b.M;
        a2.work = b.work + (size_t)g0 * b.M;
        WgrpArgs x;
        x.n_cp = (int)(g1 - g0);
        x.q = b.wq;
        x.item_cp = b.witem_cp;
        x.item_step = b.witem_step;
        x.item_mask = b.witem_mask;
        x.item_ready = b.witem_ready;
        x.snap = b.wsnap;
        x.dup_of = b.dup_of + (size_t)g0 * b.M;
        x.tau_base = g0 * b.M;
        const size_t n_items = (size_t)x.n_cp * b.M;
        x.n_items = (int)n_items;
        x.p2_cap = b.p2_cap;
        x.uf_cap = b.uf_cap;
        x.rp_ctas = b.rp_ctas;
        x.p2_hdr = b.p2_hdr;
        x.p2_work = b.p2_work;
        x.p2_A = b.p2_A;
        x.p2_room = b.p2_room;
        x.p2_dsum = b.p2_dsum;
        x.p2_ready = b.p2_ready;
        x.p2_q = b.p2_q;
        x.uf_buf = b.uf_buf;
        x.rp_ord = b.rp_ord;
        x.p2_first = b.p2_first;
        x.p2_next = b.p2_next;
        x.p2_rtau = b.p2_rtau;
        x.p2_alive = b.p2_alive;
        x.rp_snap = b.rp_snap;
        NS_CUDA(ctx, cudaMemsetAsync(b.wq, 0, sizeof(WgrpQueue), ctx->stream));
        NS_CUDA(ctx, cudaMemsetAsync(b.witem_ready, 0, n_items * sizeof(int32_t), ctx->stream));
        NS_CUDA(ctx, cudaMemsetAsync(b.p2_q, 0, 8 * sizeof(unsigned int), ctx->stream));
        NS_CUDA(ctx, cudaMemsetAsync(b.p2_ready, 0, (size_t)b.p2_cap * sizeof(int32_t), ctx->stream));
        NS_CUDA(ctx, cudaMemsetAsync(b.p2_first, 0xff, (size_t)b.p2_cap * sizeof(int32_t), ctx->stream));
        NS_CUDA(ctx, cudaMemsetAsync(b.p2_next, 0xff, (size_t)b.p2_cap * sizeof(int32_t), ctx->stream));
        const int ctas = (int)std::min<long long>((long long)n_items, (long long)ctx->sm_count * NS_WGRP_CTAS);
        prof_begin(ctx, PK_GREEDY);
        k_greedy_wgrp88<<<(unsigned)ctas, threads, 0, ctx->stream>>>(a2, x);
#ifdef NS_SPLIT_PROF   // diagnosis: phase 2 and the replays timed as "other"
        prof_end(ctx);
        prof_begin(ctx, PK_OTHER);
#endif
        // phase 2 (one warp per group, 3 CTAs of 8 warps per SM) and the representatives' replays
        k_greedy_p2<<<(unsigned)(ctx->sm_count * NS_P2_CTAS), 256, 0, ctx->stream>>>(a2, x);
#ifdef NS_SPLIT_PROF   // diagnosis: the replays timed as "score"
        prof_end(ctx);
        prof_begin(ctx, PK_SCORE);
#endif
        {
            const size_t rsm = replay_smem(b.Tpm);
            if (rsm > 48 * 1024)
                NS_CUDA(ctx, cudaFuncSetAttribute(k_greedy_replay, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm));
            k_rp_sort<<<1, 1024, 0, ctx->stream>>>(a2, x);
            k_greedy_replay<<<(unsigned)b.rp_ctas, 32 * kRpWarps, rsm, ctx->stream>>>(a2, x);
        }
        NS_LAUNCHED(ctx);   // p2, sort, replay (the caller counts wgrp88)
        NS_LAUNCHED(ctx);
        NS_LAUNCHED(ctx);
        prof_end(ctx);
    } else {
        const int threads = ((b.D + 31) / 32) * 32;
        prof_begin(ctx, PK_GREEDY);
        k_greedy_wide88<<<(unsigned)n, threads, 0, ctx->stream>>>(a);
        prof_end(ctx);
        // no grouping: every trajectory carries its own plan
        NS_CUDA(ctx, cudaMemsetAsync(b.dup_of + tb, 0xff, (size_t)n * sizeof(int32_t), ctx->stream));
    }
    NS_LAUNCHED(ctx);
    return NS_OK;
}

// Distinct feasible plans of [tb, te): duplicates (grouped greedy members
// that ended with the plan of an earlier member) read the representative's
// cost in k_select, infeasible trajectories are +inf there.
__global__ void k_compact(const uint8_t* feas, const int32_t* dup_of, long long tb, long long te, int32_t* list,
                          int32_t* n) {
    for (long long t = tb + (long long)blockIdx.x * blockDim.x + threadIdx.x; t < te;
         t += (long long)gridDim.x * blockDim.x) {
        if (feas[t] && dup_of[t] < 0) list[atomicAdd(n, 1)] = (int32_t)t;
    }
}

ns_status launch_finalize(ns_ctx* ctx, const SearchBufs& b, long long tb, long long te) {
    if (te <= tb) return NS_OK;
    // (n_uniq was cleared with the greedy queue counter by launch_greedy)
    const long long n = te - tb;
    prof_begin(ctx, PK_OTHER);
    k_compact<<<(unsigned)std::min<long long>((n + 255) / 256, 2048), 256, 0, ctx->stream>>>(b.feas, b.dup_of, tb, te,
                                                                                           b.uniq, b.n_uniq);
    prof_end(ctx);
    NS_LAUNCHED(ctx);
    return launch_plan_cost(ctx, 0, n, nullptr, b.comp, b.devdim, b.tcost, b.uniq, b.n_uniq);
}

// One level's trajectories: the n_cp column plans are split into equal
// contiguous blocks over the ranks (whole column plans, so grouped
// trajectories stay together); each rank runs N4 + N5 on its block, then the
// per-trajectory results (cost, feasibility, work, duplicate link, assignment)
// are allgathered in place so every rank runs the identical N6 selection
// (SURVEY §8(e)).  Single rank: plain launches.
ns_status run_level_trajectories(ns_ctx* ctx, SearchBufs& b, const ns_tables* t, long long n_cp) {
    const long long R = ctx->nranks;
    const long long per = (n_cp + R - 1) / R;
    ns_status s;
    b.own_cb = ctx->emulated ? 0 : (int)std::min(n_cp, ctx->rank * per);
    b.own_ce = ctx->emulated ? (int)n_cp : (int)std::min(n_cp, (long long)b.own_cb + per);
    // emulated ranks (test hook, ns_comm_init with id == NULL): this process
    // computes every rank's block into the shared buffers, the allgather is
    // the identity
    const long long r0 = ctx->emulated ? 0 : ctx->rank, r1 = ctx->emulated ? R : ctx->rank + 1;
    for (long long rk = r0; rk < r1; ++rk) {
        const long long cb = std::min(n_cp, rk * per), ce = std::min(n_cp, cb + per);
        if (ce > cb) {
            if ((s = launch_greedy(ctx, b, t, cb * b.M, ce * b.M)) != NS_OK) return s;
            if ((s = launch_finalize(ctx, b, cb * b.M, ce * b.M)) != NS_OK) return s;
        }
    }
    if (!comm_collective(ctx) || ctx->emulated) return NS_OK;
    const long long rk = ctx->rank;
    const size_t blk = (size_t)per * b.M;   // trajectories per rank block
    // the per-trajectory keys selection needs; assignment rows stay on their
    // rank (the winner's reaches the others by the int8 allreduce-max)
    struct {
        void* base;
        size_t elem;
    } arrs[] = {{b.tcost, sizeof(double)}, {b.feas, 1}, {b.work, sizeof(uint32_t)}, {b.dup_of, sizeof(int32_t)}};
    for (auto& ar : arrs) {
        char* recv = (char*)ar.base;
        const size_t bytes = blk * ar.elem;
        if ((s = comm_allgather(ctx, recv + (size_t)rk * bytes, recv, bytes)) != NS_OK) return s;
    }
    return NS_OK;
}

// Outputs the caller passed as device pointers are written by k_write_out
// directly (assign with the caller's stride, -1 padded); the others go
// through the staging buffers and are copied by deliver.
void bind_outputs(OutStage& o, const ns_plan_batch* out, int n, int Lout) {
    o.d_cost = out->cost && is_device_ptr(out->cost);
    o.d_ncol = out->n_col && is_device_ptr(out->n_col);
    o.d_plan = out->col_plan && Lout > 0 && is_device_ptr(out->col_plan);
    o.d_assign = out->assign && is_device_ptr(out->assign);
    o.d_grid = out->grid_index && is_device_ptr(out->grid_index);
    o.d_scores = out->n_scores && is_device_ptr(out->n_scores);
    (void)n;
    if (o.d_cost) o.cost = out->cost;
    if (o.d_ncol) o.n_col = out->n_col;
    if (o.d_plan) o.col_plan = out->col_plan;
    if (o.d_assign) {
        o.assign = out->assign;
        o.astride = out->assign_stride;
    }
    if (o.d_grid) o.grid = out->grid_index;
    if (o.d_scores) o.scores = (uint64_t*)out->n_scores;
}

// Copy staged results to the caller's (host) pointers.
ns_status deliver(ns_ctx* ctx, const ns_tables* t, const OutStage& o, int Lout, int Tpm, ns_plan_batch* out,
                  bool async) {
    const int n = t->n_tasks;
    cudaStream_t st = ctx->stream;
    // NS_SEARCH_ASYNC with host outputs: the result copies go to the output
    // stream once the search is done, so they overlap the caller's next batch
    // (its search waits for them before rewriting the staging; run_search)
    const bool host_out = (out->n_col && !o.d_ncol) || (out->col_plan && Lout > 0 && !o.d_plan) ||
                          (out->assign && !o.d_assign) || (out->grid_index && !o.d_grid) ||
                          (out->n_scores && !o.d_scores) || (out->cost && !o.d_cost);
    if (async && host_out) {
        NS_CUDA(ctx, ensure_copy_stream(ctx));
        NS_CUDA(ctx, cudaEventRecord(ctx->out_ready, ctx->stream));
        NS_CUDA(ctx, cudaStreamWaitEvent(ctx->out_stream, ctx->out_ready, 0));
        st = ctx->out_stream;
    }
    auto cp = [&](void* dst, const void* src, size_t bytes) -> cudaError_t {
        if (!dst) return cudaSuccess;
        return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st);
    };
    if (!o.d_ncol) NS_CUDA(ctx, cp(out->n_col, o.n_col, n * sizeof(int32_t)));
    if (out->col_plan && Lout > 0 && !o.d_plan)
        NS_CUDA(ctx, cp(out->col_plan, o.col_plan, (size_t)n * Lout * sizeof(int32_t)));
    if (out->assign && !o.d_assign) {
        // columns [Tpm, stride) are -1 (the copy below fills [0, Tpm))
        if (out->assign_stride > Tpm) {
            for (int q = 0; q < n; ++q)
                std::memset(out->assign + (size_t)q * out->assign_stride + Tpm, 0xff, out->assign_stride - Tpm);
        }
        NS_CUDA(ctx, cudaMemcpy2DAsync(out->assign, out->assign_stride, o.assign, Tpm, Tpm, n, cudaMemcpyDefault, st));
    }
    if (!o.d_grid) NS_CUDA(ctx, cp(out->grid_index, o.grid, n * sizeof(int32_t)));
    if (!o.d_scores) NS_CUDA(ctx, cp(out->n_scores, o.scores, n * sizeof(uint64_t)));
    if (async) {   // NS_SEARCH_ASYNC: no wait; the validation flag is checked by ns_synchronize
        if (!o.d_cost) NS_CUDA(ctx, cp(out->cost, o.cost, n * sizeof(double)));
        if (host_out) {
            NS_CUDA(ctx, cudaEventRecord(ctx->out_done, ctx->out_stream));
            ctx->out_pending = true;
        }
        return record_async_flag(ctx, t->d_flag);
    }
    // costs always pass through pinned host memory: the status needs them
    double* hcost = (double*)pinned_get(ctx, n * sizeof(double) + 64);
    if (!hcost) return set_err(ctx, NS_ERR_NOMEM, "pinned staging");
    int32_t* hflag = (int32_t*)(hcost + n);
    NS_CUDA(ctx, cudaMemcpyAsync(hcost, o.cost, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    NS_CUDA(ctx, cudaMemcpyAsync(hflag, t->d_flag, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    if (!o.d_cost) NS_CUDA(ctx, cp(out->cost, o.cost, n * sizeof(double)));
    NS_CUDA(ctx, cudaStreamSynchronize(st));
    prof_collect(ctx);
    ns_status fs = check_tables_flag(ctx, t, hflag);
    if (fs != NS_OK) return fs;
    for (int q = 0; q < n; ++q)
        if (!std::isfinite(hcost[q])) return NS_INFEASIBLE;
    return NS_OK;
}

// Buffer shapes of one search call (everything but the pointers): a function
// of the batch shape (tasks, longest table list), D, the search parameters
// and the ctx (ranks, SM count) only -- ns_search_workspace_bytes uses it too.
static void search_layout(const ns_ctx* ctx, int n_tasks, int T_max, int D, const ns_search_params* p,
                          bool columnwise, SearchBufs& b) {
    b = SearchBufs{};
    b.r14 = (p->flags & NS_R14_SPLITTABLE) ? 1 : 0;
    b.n_tasks = n_tasks;
    b.n_rows_lin = (long long)n_tasks * T_max * kDepth;
    b.greedy_mode = p->flags & 3u;
    b.D = D;
    b.M = p->M;
    const int L = columnwise ? p->L : 0;
    b.K = columnwise ? p->K : 1;
    b.N2 = columnwise ? 2 * p->N : 1;
    b.Lcap = L > 0 ? L : 1;
    b.Tpm = T_max + L;
    const int C = (columnwise && L > 0) ? b.K * b.N2 : 1;
    b.S = b.n_tasks * C;
    {
        // trajectory capacity: rank blocks of whole column plans (allgather needs
        // equal blocks), level 0 has n_tasks column plans, beam levels S
        const long long R = ctx->nranks;
        const long long per0 = (b.n_tasks + R - 1) / R, per = ((long long)b.S + R - 1) / R;
        b.n_traj = (int)(std::max(per0, per) * R * b.M);
    }
    {
        int dp = 1;
        while (dp < D) dp <<= 1;
        const long long max_cp = (long long)b.S;
        const size_t per = (size_t)b.M * D * kV * sizeof(double);
        // one resident wave of grouped-greedy warps (they pull column plans from a queue)
        constexpr int W = NS_DEDUP_WPB;
        long long warps = std::min<long long>(max_cp, (long long)ctx->sm_count * W * NS_DEDUP_BLOCKS8);
        warps = std::max<long long>(W, std::min<long long>(warps, (long long)((512ull << 20) / per)));
        b.gscratch_warps = dp <= 16 ? (int)(((warps + W - 1) / W) * W) : 0;
        // large D: fork snapshots of k_greedy_wgrp88 (one set of M - 1 slots per resident CTA)
        // (k_greedy_wgrp88 packs dim sums in 25 bits: T' * 128 < 2^24)
        b.wgrp = dp > 16 && b.M <= 64 && b.greedy_mode != NS_GREEDY_LANES && (long long)b.Tpm * kMaxDim < (1 << 24);
        {   // a launch covers one rank's block of column plans (level 0: tasks; beam levels: S)
            const long long R = ctx->nranks;
            b.wgrp_cp_cap = (int)std::max<long long>((b.n_tasks + R - 1) / R, ((long long)b.S + R - 1) / R);
        }
        const int nth = ((D + 31) / 32) * 32;   // 8 x 8 layout: 64 doubles of u per lane
        b.wsnap_doubles = (size_t)nth * (kV + 4);   // + dsum, headroom, A_d, certificate
        // phase-2 replay: 2 CTAs per SM, M DFS snapshot slots (64 KiB) each, within 512 MiB
        b.rp_ctas = (int)std::max<long long>(
            ctx->sm_count, std::min<long long>(2LL * ctx->sm_count, (512LL << 20) / ((long long)b.M * 128 * kV * 8)));
    }
}

ns_status run_search(ns_ctx* ctx, const ns_tables* t, int D, const ns_search_params* p, ns_plan_batch* out,
                     bool columnwise) {
    const double grid_hi = (p->flags & NS_NO_DIM_CAP) ? -1.0 : p->grid_hi_factor;
    ctx->rflags = p->flags & (NS_R10_ABS_STARTS | NS_R11_SUM_OF_MAX);
    SearchBufs b;
    search_layout(ctx, t->n_tasks, t->T_max, D, p, columnwise, b);
    const int L = columnwise ? p->L : 0;
    const int Lout = L;
    const int C = (columnwise && L > 0) ? b.K * b.N2 : 1;
    OutStage o{};
    Carver probe{nullptr};
    carve(probe, b, o, Lout > 0 ? Lout : 1);
    char* base = (char*)arena_get(ctx, probe.off + 256);
    if (!base) return arena_error(ctx, "search", probe.off + 256);
    Carver cv{base};
    carve(cv, b, o, Lout > 0 ? Lout : 1);
    ns_status s;
    const TaskView tv = task_view(t);
    // linear-regime bound of the large-D greedy: rows a table-wise search
    // streams are depth 0, a column-wise one any depth
    if (D > 16) {
        k_task_lin<<<b.n_tasks, 256, 0, ctx->stream>>>(tv, columnwise ? kDepth : 1, ctx->model.head, b.vmin,
                                                       b.Brow);
        NS_LAUNCHED(ctx);
    }
    const size_t osm = order_smem(b.Tpm);                                        // per warp (k_order_warp)
    const size_t bsm = (size_t)pow2_ceil(b.Tpm) * 12 + (size_t)b.Tpm * 4 + 16;   // k_build_order
    if (bsm > 48 * 1024) cudaFuncSetAttribute(k_build_order, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm);
    // short lists: one warp per column plan (8 per CTA); long lists: one CTA
    const bool warp_order = b.Tpm <= 256;
    const size_t wsm = 8 * osm;
    if (bsm > 48 * 1024) cudaFuncSetAttribute(k_merge_order, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm);
    const bool merge_orders = b.ord_row2 != nullptr && !getenv("NS_SORT_ORDERS");
    auto launch_order = [&](int n_cp, int level0, int level) {
        // only this rank's greedy block needs the cost order (the same
        // contiguous blocks as run_level_trajectories)
        const long long R = ctx->emulated ? 1 : ctx->nranks;
        const long long per = ((long long)n_cp + R - 1) / R;
        b.prev_b = b.ord_b;
        b.prev_e = b.ord_e;
        b.ord_b = ctx->emulated ? 0 : (int)std::min<long long>(n_cp, ctx->rank * per);
        b.ord_e = ctx->emulated ? n_cp : (int)std::min<long long>(n_cp, (long long)b.ord_b + per);
        prof_begin(ctx, PK_ORDER);
        if (warp_order) {
            const unsigned blocks = (unsigned)std::max(1, std::min((n_cp + 7) / 8, ctx->sm_count * 8));
            k_order_warp<<<blocks, 256, wsm, ctx->stream>>>(b, tv, n_cp, level0, t->d_sumdim, grid_hi);
        } else if (merge_orders && level > 0) {
            std::swap(b.ord_row, b.ord_row2);   // the previous level's orders become the parents
            std::swap(b.ord_meta, b.ord_meta2);
            k_merge_order<<<n_cp, NS_MERGE_THREADS, bsm, ctx->stream>>>(b, tv, level);
        } else {
            k_build_order<<<n_cp, 512, bsm, ctx->stream>>>(b, tv);
        }
        prof_end(ctx);
        NS_LAUNCHED(ctx);
    };
    // ---- level 0: the empty column plan (tablewise = this level only)
    if (!warp_order) {
        prof_begin(ctx, PK_OTHER);
        k_grid_caps<<<(b.n_tasks * b.M + 255) / 256, 256, 0, ctx->stream>>>(t->d_sumdim, b.n_tasks, b.D, b.M,
                                                                            grid_hi, b.capdim);
        k_setup_level0<<<(b.n_tasks + 255) / 256, 256, 0, ctx->stream>>>(b);
        prof_end(ctx);
        NS_LAUNCHED(ctx);
        NS_LAUNCHED(ctx);
    }
    launch_order(b.n_tasks, warp_order ? 1 : 0, 0);
    if ((s = run_level_trajectories(ctx, b, t, b.n_tasks)) != NS_OK) return s;
    // table-wise (L = 0): the level-0 selection also packs the outputs
    const bool final0 = L == 0;
    if (final0) bind_outputs(o, out, b.n_tasks, Lout);
    prof_begin(ctx, PK_SELECT);
    k_select0<<<(unsigned)std::max(1, std::min((b.n_tasks + 7) / 8, ctx->sm_count * 8)), 256, 0, ctx->stream>>>(
        b, o, final0 ? 1 : 0);
    prof_end(ctx);
    NS_LAUNCHED(ctx);
    // ---- beam levels (Alg. 1 lines 6-22)
    for (int level = 1; level <= L; ++level) {
        static const char* kLevelNames[] = {"level 1", "level 2", "level 3", "level 4", "level 5", "level 6",
                                            "level 7", "level 8", "level 9", "level 10", "level > 10"};
        NvtxRange nvtx_level(kLevelNames[level <= 10 ? level - 1 : 10]);
        const size_t esm = (size_t)b.Tpm * 20 + (size_t)b.N2 * 4 * 2 + (size_t)b.N2 * 4 + 64;
        if (esm > 48 * 1024)
            cudaFuncSetAttribute(k_expand, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)esm);
        prof_begin(ctx, PK_EXPAND);
        k_expand<<<b.n_tasks * b.K, NS_EXPAND_THREADS, esm, ctx->stream>>>(b, tv, level);
        prof_end(ctx);
        NS_LAUNCHED(ctx);
        launch_order(b.S, 0, level);
        if ((s = run_level_trajectories(ctx, b, t, b.S)) != NS_OK) return s;
        prof_begin(ctx, PK_SELECT);
        size_t ssel = (size_t)C * 16 + 8;
        const int staged = ssel + (size_t)C * b.M * 8 <= 160 * 1024 ? 1 : 0;
        if (staged) ssel += (size_t)C * b.M * 8;
        if (ssel > 40 * 1024) cudaFuncSetAttribute(k_select, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssel);
        k_select<<<b.n_tasks, NS_SELECT_THREADS, ssel, ctx->stream>>>(b, C, level, b.K, staged);
        prof_end(ctx);
        NS_LAUNCHED(ctx);
    }
    if (comm_collective(ctx) && !ctx->emulated) {
        // the winning assignment from its owner rank, then the consistency keys
        if (final0) {
            if ((s = comm_allreduce_max_i8(ctx, o.assign, (size_t)b.n_tasks * o.astride)) != NS_OK) return s;
        } else if ((s = comm_allreduce_max_i8(ctx, b.best_assign, (size_t)b.n_tasks * b.Tpm)) != NS_OK) {
            return s;
        }
        const unsigned kb = (unsigned)((b.n_tasks + 127) / 128);
        k_rank_check<<<kb, 128, 0, ctx->stream>>>(b, 0, t->d_flag);
        NS_LAUNCHED(ctx);
        if ((s = comm_allreduce_min_u64(ctx, b.rank_keys, (size_t)b.n_tasks * 4)) != NS_OK) return s;
        k_rank_check<<<kb, 128, 0, ctx->stream>>>(b, 1, t->d_flag);
        NS_LAUNCHED(ctx);
    }
    if (!final0) {
        bind_outputs(o, out, b.n_tasks, Lout);
        prof_begin(ctx, PK_OTHER);
        k_write_out<<<(unsigned)std::max(1, std::min((b.n_tasks + 7) / 8, ctx->sm_count * 8)), 256, 0, ctx->stream>>>(
            b, o, Lout > 0 ? Lout : 1);
        prof_end(ctx);
        NS_LAUNCHED(ctx);
    }
    return deliver(ctx, t, o, Lout, b.Tpm, out, (p->flags & NS_SEARCH_ASYNC) != 0);
}

}  // namespace

size_t search_workspace(const ns_ctx* ctx, int n_tasks, int T_max, int D, const ns_search_params* p,
                        bool columnwise) {
    SearchBufs b;
    search_layout(ctx, n_tasks, T_max, D, p, columnwise, b);
    OutStage o{};
    Carver probe{nullptr};
    const int L = columnwise ? p->L : 0;
    carve(probe, b, o, L > 0 ? L : 1);
    return probe.off + 256;
}

ns_status run_tablewise(ns_ctx* ctx, const ns_tables* t, int D, const ns_search_params* p, ns_plan_batch* out) {
    return run_search(ctx, t, D, p, out, false);
}

ns_status run_columnwise(ns_ctx* ctx, const ns_tables* t, int D, const ns_search_params* p, ns_plan_batch* out) {
    return run_search(ctx, t, D, p, out, true);
}

}  // namespace ns
