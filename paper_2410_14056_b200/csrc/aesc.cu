// TGT+ all-edges spanning centrality (aesc.hpp) on sm_100a.
//
// Per batch of up to S = 64 sources (one float64 column each):
//   K3a aesc_init      depth-0 state: p_0 = e_src, g_hat = 1/d_i + bip
//                      (aesc.hpp:577, 290-301)
//   K3b aesc_check     per-source crossover test of advance_to_switch
//                      (aesc.hpp:391-394): l < tau_src, cap, and
//                      support_degree_sum >= source_budget_sum(l) with the
//                      reference's repeated-addition budget (exact fallback
//                      whenever the fast bound cannot decide), freezing
//                      the source at tau~ = l
//   K3c/d aesc_rho_expand  rho = p_tau~ * inv_deg for the sources frozen at
//                      this depth (aesc.hpp:597-602), then the sparse frontier
//                      growth: candidate rows of depth l+1
//   K3e aesc_pull      p_{l+1}(x) = sum_{v in N(x)} p_l(v)/d(v) for all 64
//                      columns at once (row = 512 B, lane = 2 columns), the
//                      support masks (support(l+1) = N(support(l)),
//                      aesc.hpp:313-325) and the exact support degree sums
//   K3f aesc_hook_check g_hat[s] += p_l(i)/d_i - p_l(j)/d_j (aesc.hpp:581-588),
//                      fused with K3b of the next depth (block per column)
//   K4s sort_coarse_count / sort_coarse_scatter / sort_fine
//                      SABA bucketing of each (slot, side) seed set by its top
//                      seed bits, ~32 walks per bucket (PAPER Alg. 3), as a
//                      segment-local counting sort
//   K4  aesc_walk_sorted two-way walk pairs (aesc.hpp:448-525): warps walk 32
//                      adjacent seeds of one (slot, side), scoring rho in
//                      step order; aesc_pair_reduce folds (a_k - b_k) / n_req
//                      per 2048-pair tile with a fixed tree
//   K4b aesc_slot_reduce  per directed slot: tile partials folded in tile
//                      order, g_hat[s] += acc (aesc.hpp:624)
//   K5  aesc_symmetrise s_hat[e] = g_hat[u->v] + g_hat[v->u] (aesc.hpp:702-706)
//
// Exactness: tau, tau~ and n_req are integers decided exactly as the
// reference decides them (host plan restated bit-for-bit; the support degree
// sums are exact integers; budgets use the same float64 operations). The
// float64 values differ from the reference only by summation order (pull in
// ascending-neighbour order vs push in discovery order; tree vs left fold),
// far inside the 1e-9 relative contract. Every column's arithmetic is
// independent of which other sources share its batch (rows outside a
// column's support hold exact +0.0) and of the GPU count, so results are
// run-to-run and shard-count invariant.
//
// Buffer invariant: outside the rows a batch touches, P/Q/M/R are all zero.
// Double buffering keeps it within a batch (support(l+2) contains
// support(l)), and aesc_clear restores it between batches.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <exception>
#include <memory>
#include <thread>
#include <atomic>
#include <cmath>
#include <vector>

#include "device_graph.cuh"
#include "plan_host.hpp"
#include "saba_hash.cuh"
#include "walk_common.cuh"

namespace saba_cu {

constexpr int kCols = 64;           // sources per propagation batch
// propagation depths per CUDA-graph replay (even); SABA_DEPTHS_PER_GRAPH
// overrides (tuning knob)
int depths_per_graph() {
    static const int d = [] {
        const char* e = getenv("SABA_DEPTHS_PER_GRAPH");
        const int v = e ? atoi(e) : 8;
        return std::max(2, v + (v & 1));
    }();
    return d;
}

// SABA_PULL_SKIP=0|1 forces the dense or the column-sparse pull (tuning
// knob; -1 = decided per depth from the support degree sums)
int pull_skip_force() {
    static const int f = [] {
        const char* e = getenv("SABA_PULL_SKIP");
        return e ? atoi(e) : -1;
    }();
    return f;
}

struct AescState {
    uint32_t n_cap = 0;
    DevBuf P[2], Q[2], M[2], R;          // n x 64 doubles / uint64 masks / 64 x n rho
    DevBuf bits;                         // 64 x ceil(n/32) support bitmaps of R (sparse batches)
    DevBuf ulist[2], ucount, flag, tflag, tlist, tcount;
    DevBuf col_src, col_tau, degsum[2], tt, ctrl;  // per-column state
    DevBuf tau_slot, slot_edge_d, g_hat, s_hat, rho1;
    DevBuf tiles, slots, partials, groups, keys[2], vals[2], score, sort_tmp;
    DevBuf sort_segs, cb_seg, cb_cnt, cb_start, cb_cursor, coarse_tiles;  // K4s walk bucketing
    DevBuf heavy_rows, piece_off, pieces, part, part_mask;  // hub-row split (static per graph)
    uint32_t nheavy = 0, npieces = 0;
    DevBuf light_order;  // light rows by descending degree (dense depths)
    DevBuf recs;         // per-vertex walk records of the batch's columns (aesc_walk_rec)
    DevBuf tile_next;    // aesc_walk_hub's tile hand-out counter
    uint32_t nlight = 0;
    bool heavy_built = false;
    cudaStream_t stream = nullptr;       // propagation (and everything else)
    cudaStream_t stream_walk = nullptr;  // walk phase of the batch workers
    uint64_t* h_ctrl = nullptr;  // pinned mirror of the control block
    bool slot_edge_ready = false;  // slot_edge_d holds the slot -> edge map (K5)
    cudaEvent_t ev_walk[2] = {nullptr, nullptr};  // around each walk-kernel launch (report)
    ~AescState() {
        for (cudaEvent_t e : ev_walk)
            if (e) cudaEventDestroy(e);
        if (stream) cudaStreamDestroy(stream);
        if (stream_walk) cudaStreamDestroy(stream_walk);
        if (h_ctrl) cudaFreeHost(h_ctrl);
    }
};

constexpr int kWorkspaces = 2;  // batches in flight (one host thread + stream each)

// tau of a directed slot on the host: one value for a uniform plan, else a
// caller-owned per-slot array
struct SlotTau {
    const uint32_t* v = nullptr;
    uint32_t uni = 0;
    uint32_t operator[](uint64_t slot) const { return v ? v[slot] : uni; }
};

void release_aesc_state(saba_cu_graph* g) {
    delete[] g->aesc;
    g->aesc = nullptr;
}

namespace {

// Control block (device): active mask, frozen-at-this-depth mask, dense flag.
enum { kActive = 0, kFrozenNow = 1, kDense = 2, kDenseReq = 3, kDepth = 4, kRowNext = 5, kFrozenAcc = 6,
       kDone = 7, kEdgeVisits = 8, kCtrlWords = 9 };

struct AescParams {
    double eps, delta, log_term;  // log_term = log(4m/delta) (aesc.hpp:109)
    double bip_init;
    int64_t cap;
    uint32_t n;
    uint64_t m;
    int uniform_tau;
    uint32_t tau_uniform;
};

// walks_needed_raw (aesc.hpp:103-110) with the host's log term: the same
// IEEE operations in the same order (device code is built with --fmad=false).
__device__ __forceinline__ double walks_needed(int64_t tau_eff, double eps, double log_term,
                                               uint32_t deg) {
    if (tau_eff <= 0) return 0.0;
    const double scale = 0.5 * eps * double(deg);
    const double t = double(tau_eff);
    return ceil((2.0 * t * t / (scale * scale)) * log_term);
}

// source_budget_sum (aesc.hpp:362-374): repeated addition over the slots.
__device__ double budget_exact(const AescParams& p, const uint2* csr, const uint32_t* tau_slot,
                               uint32_t src, uint32_t l) {
    const uint2 r = csr[src];
    double total = 0.0;
    for (uint32_t s = r.x; s < r.x + r.y; ++s)
        total += walks_needed(int64_t(tau_slot[s]) - int64_t(l), p.eps, p.log_term, r.y);
    return total;
}

// (double)degsum >= budget, decided exactly. With a uniform tau the budget is
// `deg` additions of one value x; |fl-sum - deg*x| <= deg^2 * x * 2^-53, so
// the product decides the comparison unless degsum falls inside that band.
__device__ bool budget_reached(const AescParams& p, const uint2* csr, const uint32_t* tau_slot,
                               uint32_t src, uint32_t l, uint64_t degsum) {
    const double ds = double(degsum);  // aesc.hpp:392
    if (p.uniform_tau) {
        const uint32_t deg = csr[src].y;
        const double x = walks_needed(int64_t(p.tau_uniform) - int64_t(l), p.eps, p.log_term, deg);
        const double est = double(deg) * x;
        const double band = double(deg) * double(deg) * x * 0x1.0p-50;
        if (ds >= est + band) return true;
        if (ds < est - band) return false;
    }
    return ds >= budget_exact(p, csr, tau_slot, src, l);
}

__global__ void aesc_init(const uint32_t* __restrict__ col_src, int ncols,
                          const uint2* __restrict__ csr, AescParams p, double* __restrict__ P,
                          double* __restrict__ Q, unsigned long long* __restrict__ M,
                          uint32_t* __restrict__ ulist, uint32_t* __restrict__ ucount,
                          uint32_t* __restrict__ tflag, uint32_t* __restrict__ tlist,
                          uint32_t* __restrict__ tcount, unsigned long long* __restrict__ degsum,
                          uint32_t* __restrict__ tt, unsigned long long* __restrict__ ctrl,
                          double* __restrict__ g_hat) {
    const int c = threadIdx.x;
    if (c < ncols) {
        const uint32_t v = col_src[c];
        const uint2 r = csr[v];
        P[size_t(v) * kCols + c] = 1.0;
        Q[size_t(v) * kCols + c] = 1.0 / double(r.y);  // share = val / deg (aesc.hpp:314)
        M[v] = 1ull << c;  // the sources of a batch are distinct vertices
        ulist[c] = v;
        tflag[v] = 1;
        tlist[c] = v;
        degsum[c] = r.y;  // aesc.hpp:300
        tt[c] = 0xffffffffu;
        const double init = 1.0 / double(r.y) + p.bip_init;  // inv_deg + bip (aesc.hpp:577, 656)
        for (uint32_t s = r.x; s < r.x + r.y; ++s) g_hat[s] = init;
    }
    if (c == 0) {
        *ucount = ncols;
        *tcount = ncols;
        ctrl[kActive] = ncols == 64 ? ~0ull : ((1ull << ncols) - 1);
        ctrl[kFrozenNow] = 0;
        ctrl[kDense] = 0;
        ctrl[kDenseReq] = 0;
        ctrl[kDepth] = 0;
        ctrl[kFrozenAcc] = 0;
        ctrl[kDone] = 0;
    }
}

// One thread per column.
// The depth l lives in ctrl[kDepth] (so one captured graph serves every
// depth); the check advances it and resets the next frontier count.
__global__ void aesc_check(uint32_t* __restrict__ ucount_next, const uint32_t* __restrict__ col_src,
                           const uint32_t* __restrict__ col_tau, const uint2* __restrict__ csr,
                           const uint32_t* __restrict__ tau_slot, AescParams p,
                           const unsigned long long* __restrict__ degsum_cur,
                           unsigned long long* __restrict__ degsum_next, uint32_t* __restrict__ tt,
                           unsigned long long* __restrict__ ctrl, unsigned long long* __restrict__ edge_visits) {
    __shared__ unsigned long long frozen;
    const int c = threadIdx.x;
    const uint32_t l = uint32_t(ctrl[kDepth]);
    if (c == 0) frozen = 0;
    __syncthreads();
    const unsigned long long active = ctrl[kActive];
    degsum_next[c] = 0;
    if ((active >> c) & 1ull) {
        const uint32_t src = col_src[c];
        bool stop = l >= col_tau[c] || (p.cap >= 0 && int64_t(l) >= p.cap);
        if (!stop) stop = budget_reached(p, csr, tau_slot, src, l, degsum_cur[c]);
        if (stop) {
            tt[c] = l;
            atomicOr(&frozen, 1ull << c);
        } else {  // edge-visits of the push l -> l+1 (aesc.hpp:306-326)
            atomicAdd(edge_visits, degsum_cur[c]);
        }
    }
    __syncthreads();
    if (c == 0) {
        ctrl[kFrozenNow] = frozen;
        ctrl[kActive] = active & ~frozen;
        // dense mode switches only between depths, so every kernel of one
        // depth sees the same mode
        if (ctrl[kDenseReq]) ctrl[kDense] = 1;
        ctrl[kDepth] = l + 1;
        ctrl[kRowNext] = 0;  // dense pull: next item of the degree-ordered work list
        *ucount_next = 0;
    }
}

// rho for the columns frozen at this depth; rows outside the support hold
// exact zeros in P and therefore in R.
__device__ __forceinline__ void rho_body(const double* __restrict__ P, const uint2* __restrict__ csr,
                                         const uint32_t* __restrict__ ulist, const uint32_t* __restrict__ ucount,
                                         const unsigned long long* __restrict__ ctrl, uint32_t n,
                                         double* __restrict__ R, uint32_t* __restrict__ bits, uint32_t words) {
    const unsigned long long fz = ctrl[kFrozenNow];
    if (!fz) return;
    const bool dense = ctrl[kDense] != 0;
    const uint32_t rows = dense ? n : *ucount;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += gridDim.x * blockDim.x) {
        const uint32_t v = dense ? i : ulist[i];
        const double inv = 1.0 / double(csr[v].y);
        unsigned long long f = fz;
        while (f) {
            const int c = __ffsll(f) - 1;
            f &= f - 1;
            const double r = P[size_t(v) * kCols + c] * inv;  // p * inv_deg (aesc.hpp:599)
            R[size_t(c) * n + v] = r;
            if (r != 0.0) atomicOr(bits + size_t(c) * words + (v >> 5), 1u << (v & 31));
        }
    }
}

// list[count++] = x for every lane with `take`, one atomic per warp (all 32
// lanes must call).
__device__ __forceinline__ void warp_append(uint32_t* __restrict__ list, uint32_t* __restrict__ count,
                                            uint32_t x, bool take, uint32_t lane, uint32_t cap) {
    const uint32_t m = __ballot_sync(0xffffffffu, take);
    if (!m) return;
    uint32_t base = 0;
    if (lane == uint32_t(__ffs(m) - 1)) base = atomicAdd(count, uint32_t(__popc(m)));
    base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
    SABA_DCHECK(base + uint32_t(__popc(m)) <= cap);  // every row is appended at most once per list
    (void)cap;
    if (take) list[base + __popc(m & ((1u << lane) - 1u))] = x;
}

// Sparse frontier growth: rows of depth l+1 = N(rows of depth l that still
// carry an active column). Warp per row; the order of the new list is
// irrelevant (every row is computed independently).
__device__ __forceinline__ void expand_body(const uint2* __restrict__ csr, const uint32_t* __restrict__ adj,
                                            const unsigned long long* __restrict__ M,
                                            const uint32_t* __restrict__ ulist, const uint32_t* __restrict__ ucount,
                                            uint32_t* __restrict__ ulist_next, uint32_t* __restrict__ ucount_next,
                                            uint32_t* __restrict__ flag, uint32_t* __restrict__ tflag,
                                            uint32_t* __restrict__ tlist, uint32_t* __restrict__ tcount,
                                            const unsigned long long* __restrict__ ctrl, uint32_t n) {
    const unsigned long long active = ctrl[kActive];
    if (!active || ctrl[kDense]) return;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t rows = *ucount;
    for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < rows;
         i += (gridDim.x * blockDim.x) >> 5) {
        const uint32_t v = ulist[i];
        if (!(M[v] & active)) continue;
        const uint2 r = csr[v];
        for (uint32_t s0 = r.x; s0 < r.x + r.y; s0 += 32) {
            const uint32_t s = s0 + lane;
            uint32_t x = 0;
            bool claim = false;
            if (s < r.x + r.y) {
                x = adj[s];
                claim = !flag[x] && !atomicExch(flag + x, 1u);
            }
            // appends are warp-aggregated: one counter atomic per warp, not
            // per row (a single global counter serialises in L2)
            warp_append(ulist_next, ucount_next, x, claim, lane, n);
            bool fresh = false;
            if (claim && !tflag[x]) {  // x is claimed by exactly one thread per depth
                tflag[x] = 1;
                fresh = true;
            }
            warp_append(tlist, tcount, x, fresh, lane, n);
        }
    }
}

// K3c + K3d in one launch (one fewer kernel per depth): rho of the columns
// frozen at this depth (reads P_l) and the sparse frontier growth (reads the
// support masks) touch disjoint data, so one grid does both in turn.
__global__ void aesc_rho_expand(const double* __restrict__ P, const uint2* __restrict__ csr,
                                const uint32_t* __restrict__ adj, const unsigned long long* __restrict__ M,
                                const uint32_t* __restrict__ ulist, const uint32_t* __restrict__ ucount,
                                uint32_t* __restrict__ ulist_next, uint32_t* __restrict__ ucount_next,
                                uint32_t* __restrict__ flag, uint32_t* __restrict__ tflag,
                                uint32_t* __restrict__ tlist, uint32_t* __restrict__ tcount,
                                const unsigned long long* __restrict__ ctrl, uint32_t n, double* __restrict__ R,
                                uint32_t* __restrict__ bits, uint32_t words) {
    rho_body(P, csr, ulist, ucount, ctrl, n, R, bits, words);
    expand_body(csr, adj, M, ulist, ucount, ulist_next, ucount_next, flag, tflag, tlist, tcount, ctrl, n);
}

// Rows with more than kHeavy neighbours are split into fixed pieces of
// kHeavy neighbours (warp per piece) whose partial sums are combined in piece
// order: a deterministic function of the row alone, and no hub row sits on
// one warp's critical path.
constexpr uint32_t kHeavy = 256;
#ifndef SABA_PULL_UNROLL
#define SABA_PULL_UNROLL 6
#endif
constexpr int kPullUnroll = SABA_PULL_UNROLL;  // Q-row gathers in flight per warp

// Sum of Q rows (2 columns per lane) and OR of support masks over the
// neighbour slots [b, e), in slot order; kPullUnroll gathers in flight per warp.
__device__ __forceinline__ void pull_range(const uint32_t* __restrict__ adj,
                                           const double* __restrict__ Qc,
                                           const unsigned long long* __restrict__ Mc, uint32_t b,
                                           uint32_t e, uint32_t lane, bool need, double& a0, double& a1,
                                           unsigned long long& mask) {
    // need = one of the lane's two columns is still active: lanes of frozen
    // columns skip their half-sector of every Q row (their sums are zeroed
    // by pull_store anyway), so late depths move fewer L2 sectors.
    constexpr int U = kPullUnroll;
    for (uint32_t s0 = b; s0 < e; s0 += 32) {
        const uint32_t cnt = min(32u, e - s0);
        const uint32_t mine = lane < cnt ? adj[s0 + lane] : 0u;
        uint32_t k = 0;
        for (; k + U <= cnt; k += U) {
            double2 q[U];
            unsigned long long mm[U];
#pragma unroll
            for (int j = 0; j < U; ++j) {
                const uint32_t v = __shfl_sync(0xffffffffu, mine, k + j);
                mm[j] = Mc[v];
                q[j] = need ? reinterpret_cast<const double2*>(Qc + size_t(v) * kCols)[lane] : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int j = 0; j < U; ++j) {
                mask |= mm[j];
                a0 += q[j].x;
                a1 += q[j].y;
            }
        }
        for (; k < cnt; ++k) {
            const uint32_t v = __shfl_sync(0xffffffffu, mine, k);
            mask |= Mc[v];
            const double2 q = need ? reinterpret_cast<const double2*>(Qc + size_t(v) * kCols)[lane]
                                   : make_double2(0.0, 0.0);
            a0 += q.x;
            a1 += q.y;
        }
    }
}

// Column-sparse form of pull_range for depths where the columns' supports
// cover a small part of the graph (shallow plans such as cfg5, tau~ ~ 2, whose
// 64-source union frontier still goes dense): the 32 neighbour masks of a
// chunk are gathered first (one per lane), then each lane reads Q[v] for its
// two columns only when v is in the support of one of them. Rows outside a
// column's support hold exact +0.0 there, so a skipped load adds nothing and
// the sums are bit-identical to pull_range's.
__device__ __forceinline__ void pull_range_skip(const uint32_t* __restrict__ adj,
                                                const double* __restrict__ Qc,
                                                const unsigned long long* __restrict__ Mc, uint32_t b,
                                                uint32_t e, uint32_t lane, bool need, double& a0, double& a1,
                                                unsigned long long& mask) {
    constexpr int U = 4;  // the neighbour masks stay in registers: fewer Q loads in flight
    const unsigned long long mine_bits = 3ull << (2 * lane);
    for (uint32_t s0 = b; s0 < e; s0 += 32) {
        const uint32_t cnt = min(32u, e - s0);
        const uint32_t mine = lane < cnt ? adj[s0 + lane] : 0u;
        const unsigned long long mine_mask = lane < cnt ? Mc[mine] : 0ull;
        uint32_t k = 0;
        for (; k + U <= cnt; k += U) {
            double2 q[U];
#pragma unroll
            for (int j = 0; j < U; ++j) {
                const uint32_t v = __shfl_sync(0xffffffffu, mine, k + j);
                const unsigned long long mm = __shfl_sync(0xffffffffu, mine_mask, k + j);
                mask |= mm;
                q[j] = need && (mm & mine_bits) ? reinterpret_cast<const double2*>(Qc + size_t(v) * kCols)[lane]
                                                : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int j = 0; j < U; ++j) {
                a0 += q[j].x;
                a1 += q[j].y;
            }
        }
        for (; k < cnt; ++k) {
            const uint32_t v = __shfl_sync(0xffffffffu, mine, k);
            const unsigned long long mm = __shfl_sync(0xffffffffu, mine_mask, k);
            mask |= mm;
            const double2 q = need && (mm & mine_bits) ? reinterpret_cast<const double2*>(Qc + size_t(v) * kCols)[lane]
                                                       : make_double2(0.0, 0.0);
            a0 += q.x;
            a1 += q.y;
        }
    }
}

// Column-sparse depth? The useful fraction of a dense pull's Q reads for
// column c is degsum_c / 2m (the slots pointing into its support); below a
// quarter on average over the active columns the mask-first form wins.
// SABA_PULL_SKIP=0|1 forces either form (tuning knob; results identical).
__device__ __forceinline__ bool columns_sparse(const unsigned long long* __restrict__ degsum_cur,
                                               unsigned long long active, uint64_t two_m, int force) {
    if (force >= 0) return force != 0;
    unsigned long long tot = 0;
    uint32_t na = 0;
    for (int c = 0; c < kCols; ++c)
        if ((active >> c) & 1ull) {
            tot += degsum_cur[c];
            ++na;
        }
    return tot * 4 < two_m * na;
}

// Write one finished row of depth l+1 (P, Q = P / d, support mask) and
// account its degree into the support degree sums of its columns.
__device__ __forceinline__ void pull_store(uint32_t x, uint32_t deg, double a0, double a1,
                                           unsigned long long mask, unsigned long long active,
                                           uint32_t lane, double* __restrict__ Pn,
                                           double* __restrict__ Qn, unsigned long long* __restrict__ Mn,
                                           unsigned long long& ds0, unsigned long long& ds1) {
    const unsigned long long lo_mask = 1ull << (2 * lane), hi_mask = 1ull << (2 * lane + 1);
    mask &= active;
    if (!(active & lo_mask)) a0 = 0.0;
    if (!(active & hi_mask)) a1 = 0.0;
    const double dx = double(deg);
    reinterpret_cast<double2*>(Pn + size_t(x) * kCols)[lane] = make_double2(a0, a1);
    reinterpret_cast<double2*>(Qn + size_t(x) * kCols)[lane] = make_double2(a0 / dx, a1 / dx);
    if (lane == 0) Mn[x] = mask;
    if (mask & lo_mask) ds0 += deg;
    if (mask & hi_mask) ds1 += deg;
}

// Support degree sums: warp lanes -> shared memory -> one global atomic per
// column per block (same-address global atomics from every warp serialise in
// L2 and dominated the pull kernel).
__device__ __forceinline__ void flush_degsum(unsigned long long* sm, unsigned long long ds0,
                                             unsigned long long ds1, uint32_t lane,
                                             unsigned long long* __restrict__ degsum_next) {
    if (ds0) atomicAdd(sm + 2 * lane, ds0);
    if (ds1) atomicAdd(sm + 2 * lane + 1, ds1);
    __syncthreads();
    if (threadIdx.x < kCols && sm[threadIdx.x]) atomicAdd(degsum_next + threadIdx.x, sm[threadIdx.x]);
}

struct HeavyPiece {
    uint32_t row, begin, end, pad;
};

// Pull SpMM over the candidate rows (sparse) or all rows (dense) with at
// most kHeavy neighbours. Warp per row, lane = columns {2 lane, 2 lane + 1}.
#ifndef SABA_PULL_MINB
#define SABA_PULL_MINB 4  // 64 registers: 32 warps per SM keep more Q-row gathers in flight
#endif
__global__ void __launch_bounds__(256, SABA_PULL_MINB)
    aesc_pull(const uint2* __restrict__ csr, const uint32_t* __restrict__ adj,
              const double* __restrict__ Qc, const unsigned long long* __restrict__ Mc,
              double* __restrict__ Pn, double* __restrict__ Qn, unsigned long long* __restrict__ Mn,
              const uint32_t* __restrict__ ulist_next, const uint32_t* __restrict__ ucount_next,
              uint32_t* __restrict__ flag, unsigned long long* __restrict__ degsum_next,
              unsigned long long* __restrict__ ctrl, uint32_t n,
              const uint32_t* __restrict__ light_order, uint32_t nlight,
              const HeavyPiece* __restrict__ pieces, uint32_t npieces, double* __restrict__ part,
              unsigned long long* __restrict__ part_mask, const unsigned long long* __restrict__ degsum_cur,
              uint64_t two_m, int skip_force) {
    __shared__ unsigned long long bds[kCols];
    __shared__ bool s_skip;
    const unsigned long long active = ctrl[kActive];
    if (!active) return;
    if (threadIdx.x < kCols) bds[threadIdx.x] = 0;
    if (threadIdx.x == 0) s_skip = columns_sparse(degsum_cur, active, two_m, skip_force);
    __syncthreads();
    const bool skip = s_skip;
    const bool dense = ctrl[kDense] != 0;
    const uint32_t lane = threadIdx.x & 31;
    const bool need = ((active >> (2 * lane)) & 3ull) != 0;
    unsigned long long ds0 = 0, ds1 = 0;
    if (dense && light_order) {
        // dense depths: one work list of hub-row pieces, then light rows in
        // descending degree order, handed out one item at a time (longest
        // first, so no warp is left with a long tail); the next item is
        // claimed before the current one is summed, which hides the counter
        // atomic's round trip; aesc_pull_combine folds the pieces after
        const uint32_t total = npieces + nlight;
        uint32_t i = 0;
        if (lane == 0) i = uint32_t(atomicAdd(ctrl + kRowNext, 1ull));
        i = __shfl_sync(0xffffffffu, i, 0);
        while (i < total) {
            uint32_t nxt = 0;
            if (lane == 0) nxt = uint32_t(atomicAdd(ctrl + kRowNext, 1ull));
            double a0 = 0.0, a1 = 0.0;
            unsigned long long mask = 0;
            SABA_DCHECK(i < total);
            if (i < npieces) {
                const HeavyPiece pc = pieces[i];
                if (skip)
                    pull_range_skip(adj, Qc, Mc, pc.begin, pc.end, lane, need, a0, a1, mask);
                else
                    pull_range(adj, Qc, Mc, pc.begin, pc.end, lane, need, a0, a1, mask);
                reinterpret_cast<double2*>(part + size_t(i) * kCols)[lane] = make_double2(a0, a1);
                if (lane == 0) part_mask[i] = mask;
            } else {
                const uint32_t x = light_order[i - npieces];
                const uint2 r = csr[x];
                if (skip)
                    pull_range_skip(adj, Qc, Mc, r.x, r.x + r.y, lane, need, a0, a1, mask);
                else
                    pull_range(adj, Qc, Mc, r.x, r.x + r.y, lane, need, a0, a1, mask);
                pull_store(x, r.y, a0, a1, mask, active, lane, Pn, Qn, Mn, ds0, ds1);
            }
            i = __shfl_sync(0xffffffffu, nxt, 0);
        }
        flush_degsum(bds, ds0, ds1, lane, degsum_next);
        return;
    }
    const uint32_t rows = dense ? n : *ucount_next;
    for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < rows;
         i += (gridDim.x * blockDim.x) >> 5) {
        const uint32_t x = dense ? i : ulist_next[i];
        const uint2 r = csr[x];
        if (r.y > kHeavy) continue;  // pieces + combine
        double a0 = 0.0, a1 = 0.0;
        unsigned long long mask = 0;
        if (skip)
            pull_range_skip(adj, Qc, Mc, r.x, r.x + r.y, lane, need, a0, a1, mask);
        else
            pull_range(adj, Qc, Mc, r.x, r.x + r.y, lane, need, a0, a1, mask);
        pull_store(x, r.y, a0, a1, mask, active, lane, Pn, Qn, Mn, ds0, ds1);
        if (lane == 0 && !dense) flag[x] = 0;
    }
    flush_degsum(bds, ds0, ds1, lane, degsum_next);  // integer sums: order-free
    // switch to dense rows once the frontier covers a quarter of the graph
    if (!dense && blockIdx.x == 0 && threadIdx.x == 0 && rows > n / 4) ctrl[kDenseReq] = 1;
}


// Warp per piece of a heavy row that is a candidate at this depth.
__global__ void __launch_bounds__(256)
    aesc_pull_pieces(const HeavyPiece* __restrict__ pieces, uint32_t npieces,
                     const uint32_t* __restrict__ adj, const double* __restrict__ Qc,
                     const unsigned long long* __restrict__ Mc, const uint32_t* __restrict__ flag,
                     double* __restrict__ part, unsigned long long* __restrict__ part_mask,
                     const unsigned long long* __restrict__ ctrl, uint32_t dynamic,
                     const unsigned long long* __restrict__ degsum_cur, uint64_t two_m, int skip_force) {
    const unsigned long long active = ctrl[kActive];
    if (!active) return;
    const bool dense = ctrl[kDense] != 0;
    if (dense && dynamic) return;  // aesc_pull takes the pieces in dense depths
    __shared__ bool s_skip;
    if (threadIdx.x == 0) s_skip = columns_sparse(degsum_cur, active, two_m, skip_force);
    __syncthreads();
    const bool skip = s_skip;
    const uint32_t lane = threadIdx.x & 31;
    const bool need = ((active >> (2 * lane)) & 3ull) != 0;
    for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < npieces;
         i += (gridDim.x * blockDim.x) >> 5) {
        const HeavyPiece pc = pieces[i];
        if (!dense && !flag[pc.row]) continue;
        double a0 = 0.0, a1 = 0.0;
        unsigned long long mask = 0;
        if (skip)
            pull_range_skip(adj, Qc, Mc, pc.begin, pc.end, lane, need, a0, a1, mask);
        else
            pull_range(adj, Qc, Mc, pc.begin, pc.end, lane, need, a0, a1, mask);
        reinterpret_cast<double2*>(part + size_t(i) * kCols)[lane] = make_double2(a0, a1);
        if (lane == 0) part_mask[i] = mask;
    }
}

// Warp per heavy row: fold its pieces in order and store the row.
__global__ void aesc_pull_combine(const uint32_t* __restrict__ heavy_rows,
                                  const uint32_t* __restrict__ piece_off, uint32_t nheavy,
                                  const uint2* __restrict__ csr, const double* __restrict__ part,
                                  const unsigned long long* __restrict__ part_mask,
                                  double* __restrict__ Pn, double* __restrict__ Qn,
                                  unsigned long long* __restrict__ Mn, uint32_t* __restrict__ flag,
                                  unsigned long long* __restrict__ degsum_next,
                                  const unsigned long long* __restrict__ ctrl) {
    __shared__ unsigned long long bds[kCols];
    const unsigned long long active = ctrl[kActive];
    if (!active) return;
    if (threadIdx.x < kCols) bds[threadIdx.x] = 0;
    __syncthreads();
    const bool dense = ctrl[kDense] != 0;
    const uint32_t lane = threadIdx.x & 31;
    unsigned long long ds0 = 0, ds1 = 0;
    for (uint32_t h = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; h < nheavy;
         h += (gridDim.x * blockDim.x) >> 5) {
        const uint32_t x = heavy_rows[h];
        if (!dense && !flag[x]) continue;
        const uint32_t p0 = piece_off[h], p1 = piece_off[h + 1];
        double2 a = reinterpret_cast<const double2*>(part + size_t(p0) * kCols)[lane];
        unsigned long long mask = part_mask[p0];
        for (uint32_t p = p0 + 1; p < p1; ++p) {
            const double2 b = reinterpret_cast<const double2*>(part + size_t(p) * kCols)[lane];
            a.x += b.x;
            a.y += b.y;
            mask |= part_mask[p];
        }
        pull_store(x, csr[x].y, a.x, a.y, mask, active, lane, Pn, Qn, Mn, ds0, ds1);
        __syncwarp();
        if (lane == 0 && !dense) flag[x] = 0;
    }
    flush_degsum(bds, ds0, ds1, lane, degsum_next);
}


// K3f + K3b of the next depth in one launch (block per column): the hook of
// depth l+1 for the columns that stepped, then the crossover check of depth
// l+1 (aesc_check's per-column test); the last block to finish publishes the
// new active / frozen masks and advances the depth. Thread 0 of each block
// stages the control words in shared memory and the block passes a barrier
// before that thread counts the block as done, so no thread of any block can
// read ctrl after the last block rewrites it: the hook and the checks see the
// masks of depth l exactly as the separate kernels did, by construction.
__global__ void __launch_bounds__(128)
    aesc_hook_check(const uint32_t* __restrict__ col_src, const uint32_t* __restrict__ col_tau,
                    const uint2* __restrict__ csr, const uint32_t* __restrict__ adj,
                    const uint32_t* __restrict__ tau_slot, const double* __restrict__ Pn, AescParams p,
                    const unsigned long long* __restrict__ degsum_cur, unsigned long long* __restrict__ degsum_next,
                    uint32_t* __restrict__ tt, uint32_t* __restrict__ ucount_next, unsigned long long* ctrl,
                    double* __restrict__ g_hat, unsigned long long* __restrict__ edge_visits) {
    __shared__ bool last;
    __shared__ unsigned long long s_active, s_depth;
    const int c = blockIdx.x;
    if (threadIdx.x == 0) {
        s_active = ctrl[kActive];
        s_depth = ctrl[kDepth];
    }
    __syncthreads();
    const unsigned long long active = s_active;
    const uint32_t depth = uint32_t(s_depth);  // l + 1
    if ((active >> c) & 1ull) {  // hook (aesc.hpp:581-588)
        const uint32_t src = col_src[c];
        const uint2 r = csr[src];
        const double pi = Pn[size_t(src) * kCols + c] * (1.0 / double(r.y));
        for (uint32_t s = r.x + threadIdx.x; s < r.x + r.y; s += blockDim.x) {
            if (depth > tau_slot[s]) continue;
            const uint32_t j = adj[s];
            SABA_DCHECK(j < p.n);
            g_hat[s] += pi - Pn[size_t(j) * kCols + c] * (1.0 / double(csr[j].y));
        }
    }
    if (threadIdx.x == 0) {  // check of depth l + 1 (aesc.hpp:391-394)
        degsum_next[c] = 0;
        if ((active >> c) & 1ull) {
            const uint32_t src = col_src[c];
            bool stop = depth >= col_tau[c] || (p.cap >= 0 && int64_t(depth) >= p.cap);
            if (!stop) stop = budget_reached(p, csr, tau_slot, src, depth, degsum_cur[c]);
            if (stop) {
                tt[c] = depth;
                atomicOr(ctrl + kFrozenAcc, 1ull << c);
            } else {  // the push of depth l+1 -> l+2 visits every support slot
                atomicAdd(edge_visits, degsum_cur[c]);
            }
        }
        __threadfence();
        last = atomicAdd(ctrl + kDone, 1ull) == gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        const unsigned long long frozen = atomicExch(ctrl + kFrozenAcc, 0ull);
        ctrl[kFrozenNow] = frozen;
        ctrl[kActive] = active & ~frozen;
        if (ctrl[kDenseReq]) ctrl[kDense] = 1;  // mode switches only between depths
        ctrl[kDepth] = depth + 1;
        ctrl[kRowNext] = 0;
        *ucount_next = 0;
        ctrl[kDone] = 0;
    }
}

// Restore the all-zero invariant on every row a sparse batch touched.
__global__ void aesc_clear(const uint32_t* __restrict__ tlist, const uint32_t* __restrict__ tcount,
                           double* P0, double* P1, double* Q0, double* Q1,
                           unsigned long long* M0, unsigned long long* M1, double* R, uint32_t n,
                           uint32_t* tflag, int ncols, uint32_t* bits, uint32_t words) {
    const uint32_t rows = *tcount;
    const uint32_t lane = threadIdx.x & 31;
    for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < rows;
         i += (gridDim.x * blockDim.x) >> 5) {
        const uint32_t x = tlist[i];
        const double2 z = make_double2(0.0, 0.0);
        reinterpret_cast<double2*>(P0 + size_t(x) * kCols)[lane] = z;
        reinterpret_cast<double2*>(P1 + size_t(x) * kCols)[lane] = z;
        reinterpret_cast<double2*>(Q0 + size_t(x) * kCols)[lane] = z;
        reinterpret_cast<double2*>(Q1 + size_t(x) * kCols)[lane] = z;
        for (int c = lane; c < ncols; c += 32) {
            R[size_t(c) * n + x] = 0.0;
            bits[size_t(c) * words + (x >> 5)] = 0;  // the whole word is cleared anyway
        }
        if (lane == 0) {
            M0[x] = 0;
            M1[x] = 0;
            tflag[x] = 0;
        }
    }
}

// Walk phase layout. A slot's n_req pairs are split into groups of at most
// kGroupPairs pairs; a chunk holds whole groups (<= kChunkWalks walks, both
// sides). Walk w of a chunk is (group, side, k) in that order, so every
// (group, side) "segment" is a contiguous range of walk ids.
//
// SABA bouquets (PAPER Alg. 3 + §3.3; walker.hpp:436-439): within each
// segment the walks are bucketed by the top bits of their seeds, about 32
// walks per bucket, so a warp walks 32 adjacent seeds of one (slot, side) —
// the bouquet over the slot's whole seed set, not just a tile. The order is
// a performance device only: every walk's score depends on its own seed and
// lands in score[w], so any permutation gives identical results. That lets
// the bucketing be a segment-local counting sort (K4s) instead of a global
// radix sort: segments up to kFineDirect walks are bucketed by one CTA in
// one pass; larger ones first split by their top d1 seed bits into coarse
// buckets of about kCoarseTarget walks (count, scan, scatter), which the
// same one-pass CTA then buckets by the next bits.
constexpr uint32_t kGroupPairs = 1u << 24;
constexpr uint64_t kChunkWalks = uint64_t(1) << 28;
constexpr uint32_t kPairTile = 2048;       // pairs per deterministic reduction tile
constexpr uint32_t kFineDirect = 8192;     // segments up to this size skip the coarse split
constexpr uint32_t kCoarseTarget = 6144;   // expected walks per coarse bucket (<= kFineStage)
constexpr uint32_t kFineBitsMax = 11;      // <= 2048 fine buckets per coarse bucket
constexpr uint32_t kCoarseTile = 8192;     // walks per CTA in the coarse passes
constexpr uint32_t kCoarseBitsMax = 11;

struct WalkGroup {
    uint64_t edge_seed;  // substream(src_seed, slot) (aesc.hpp:622)
    uint64_t k0;         // first pair index of the group within its slot
    uint32_t pairs;      // pairs in this group
    uint32_t walk_off;   // side-0 walks at [walk_off, +pairs), side 1 after them
    uint32_t vi, vj;     // side 0 / side 1 start vertices (aesc.hpp:518-521)
    uint32_t len;        // tau_eff + 1 vertices
    uint32_t col;        // rho column
};

struct PairTile {
    double inv_n;  // 1 / n_req (aesc.hpp:512)
    uint32_t group, p0, count, out;
};

struct SlotWork {
    uint32_t t0, t1;  // global tile range of the slot, in pair order
    uint32_t slot;    // directed slot receiving the estimate
    uint32_t pad;
};

// One (group, side) segment of a chunk and its coarse buckets
// [cb, cb + 2^d1) in the chunk's coarse-bucket table.
struct SortSeg {
    uint32_t group, side, start, size, d1, cb;
};
struct CoarseTile {
    uint32_t seg, t0, count, pad;
};

// walk seed counter_hash(edge_seed, 2k+side) >> 32 (aesc.hpp:485) of walk w
__device__ __forceinline__ uint32_t seed_of(const WalkGroup& G, uint32_t w) {
    const uint32_t local = w - G.walk_off;
    const uint32_t side = local >= G.pairs;
    return walk_seed(G.edge_seed, 2 * (G.k0 + (local - side * G.pairs)) + side);
}

__device__ __forceinline__ uint32_t top_bits(uint32_t x, uint32_t skip, uint32_t bits) {
    return bits ? uint32_t((uint64_t(x) << skip) & 0xffffffffull) >> (32 - bits) : 0u;
}

// K4s-1: per coarse tile, histogram of the top d1 seed bits (smem), flushed
// with one global add per non-empty digit.
__global__ void __launch_bounds__(512)
    sort_coarse_count(const CoarseTile* __restrict__ tiles, const SortSeg* __restrict__ segs,
                      const WalkGroup* __restrict__ groups, uint32_t* __restrict__ cnt) {
    __shared__ uint32_t hist[1u << kCoarseBitsMax];
    const CoarseTile T = tiles[blockIdx.x];
    const SortSeg S = segs[T.seg];
    const WalkGroup G = groups[S.group];
    const uint32_t nd = 1u << S.d1;
    for (uint32_t d = threadIdx.x; d < nd; d += blockDim.x) hist[d] = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < T.count; i += blockDim.x)
        atomicAdd(hist + top_bits(seed_of(G, S.start + T.t0 + i), 0, S.d1), 1u);
    __syncthreads();
    for (uint32_t d = threadIdx.x; d < nd; d += blockDim.x)
        if (hist[d]) atomicAdd(cnt + S.cb + d, hist[d]);
}

// K4s-2: same tiles; reserve one run per non-empty digit from the bucket
// cursors, then place the tile's walk ids (order within a run is free).
__global__ void __launch_bounds__(512)
    sort_coarse_scatter(const CoarseTile* __restrict__ tiles, const SortSeg* __restrict__ segs,
                        const WalkGroup* __restrict__ groups, uint32_t* __restrict__ cursor,
                        uint32_t* __restrict__ tmp) {
    __shared__ uint32_t hist[1u << kCoarseBitsMax], base[1u << kCoarseBitsMax];
    const CoarseTile T = tiles[blockIdx.x];
    const SortSeg S = segs[T.seg];
    const WalkGroup G = groups[S.group];
    const uint32_t nd = 1u << S.d1;
    for (uint32_t d = threadIdx.x; d < nd; d += blockDim.x) hist[d] = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < T.count; i += blockDim.x)
        atomicAdd(hist + top_bits(seed_of(G, S.start + T.t0 + i), 0, S.d1), 1u);
    __syncthreads();
    for (uint32_t d = threadIdx.x; d < nd; d += blockDim.x) {
        base[d] = hist[d] ? atomicAdd(cursor + S.cb + d, hist[d]) : 0u;
        hist[d] = 0;
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < T.count; i += blockDim.x) {
        const uint32_t w = S.start + T.t0 + i;
        const uint32_t d = top_bits(seed_of(G, w), 0, S.d1);
        const uint32_t at = base[d] + atomicAdd(hist + d, 1u);
        SABA_DCHECK(at >= S.start && at < S.start + S.size);  // coarse buckets stay inside their segment
        tmp[at] = w;
    }
}

// K4s-3: one CTA per coarse bucket (a whole small segment, or one coarse
// digit of a large one): counting sort by the next fine bits, about 32 walks
// per fine bucket; writes the walk id and its group at the sorted position.
// Buckets up to kFineStage walks are permuted in shared memory and written
// out coalesced; the group id is the same for the whole bucket (a fill).
constexpr uint32_t kFineStage = 9216;
__global__ void __launch_bounds__(256)
    sort_fine(const uint32_t* __restrict__ cb_seg, const SortSeg* __restrict__ segs,
              const WalkGroup* __restrict__ groups, const uint32_t* __restrict__ cnt,
              const uint32_t* __restrict__ start, const uint32_t* __restrict__ tmp,
              uint32_t* __restrict__ out_w, uint32_t* __restrict__ out_g) {
    using Scan = cub::BlockScan<uint32_t, 256>;
    constexpr uint32_t kB = 1u << kFineBitsMax, kPer = kB / 256;
    __shared__ uint32_t hist[kB];
    __shared__ uint32_t stage[kFineStage];
    __shared__ typename Scan::TempStorage scan_tmp;
    const uint32_t b = blockIdx.x;
    const uint32_t count = cnt[b];
    if (count == 0) return;
    const SortSeg S = segs[cb_seg[b]];
    const WalkGroup G = groups[S.group];
    const uint32_t at = start[b];
    // about 32 walks per fine bucket
    uint32_t fb = 0;
    while (fb < kFineBitsMax && (32u << fb) < count) ++fb;
    const uint32_t nf = 1u << fb;
    for (uint32_t d = threadIdx.x; d < kB; d += blockDim.x) hist[d] = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < count; i += blockDim.x) {
        const uint32_t w = S.d1 ? tmp[at + i] : S.start + i;
        atomicAdd(hist + top_bits(seed_of(G, w), S.d1, fb), 1u);
    }
    __syncthreads();
    // exclusive scan of hist[0, nf): kPer consecutive digits per thread
    uint32_t v[kPer], run = 0;
#pragma unroll
    for (uint32_t j = 0; j < kPer; ++j) {
        const uint32_t d = threadIdx.x * kPer + j;
        v[j] = d < nf ? hist[d] : 0u;
        run += v[j];
    }
    uint32_t excl;
    Scan(scan_tmp).ExclusiveSum(run, excl);
    __syncthreads();
#pragma unroll
    for (uint32_t j = 0; j < kPer; ++j) {
        const uint32_t d = threadIdx.x * kPer + j;
        if (d < nf) hist[d] = excl;
        excl += v[j];
    }
    __syncthreads();
    const bool staged = count <= kFineStage;
    for (uint32_t i = threadIdx.x; i < count; i += blockDim.x) {
        const uint32_t w = S.d1 ? tmp[at + i] : S.start + i;
        const uint32_t r = atomicAdd(hist + top_bits(seed_of(G, w), S.d1, fb), 1u);
        SABA_DCHECK(r < count && w >= G.walk_off && w < G.walk_off + 2 * G.pairs);
        if (staged)
            stage[r] = w;
        else
            out_w[at + r] = w;
    }
    if (staged) __syncthreads();
    for (uint32_t i = threadIdx.x; i < count; i += blockDim.x) {
        if (staged) out_w[at + i] = stage[i];
        out_g[at + i] = S.group;
    }
}

// K4: warps walk consecutive sorted entries (WPT per lane); the score of
// walk w = sum of rho over steps 1..len-1 in step order (aesc.hpp:491-493).
// BITMAP: rho is non-zero only on the landing support; a 1-bit-per-vertex
// check (64x smaller than rho, L2-resident) skips gathers of exact zeros
// (adding +0.0 is the identity, so scores are unchanged).
// FAT: slots carry the neighbour's {id, base, degree} (L2-resident graphs),
// so a step is one dependent gather (plus the rho gather, which feeds nothing).
// WPT walks per lane, MINB resident blocks per SM (register budget): short
// walks are prologue/latency bound and want many warps with 2 walks each
// (32 registers), long ones 4 walks per lane (48 registers); see run_tiles.
template <bool PACKED, int WPT, bool BITMAP, bool FAT, int MINB, bool F16 = false>
__global__ void __launch_bounds__(256, MINB)
    aesc_walk_sorted(const uint32_t* __restrict__ gidx, const uint32_t* __restrict__ vals,
                     uint32_t nwalks, const WalkGroup* __restrict__ groups,
                     const uint2* __restrict__ csr, const uint32_t* __restrict__ adj,
                     const uint64_t* __restrict__ adjp, const double* __restrict__ R, uint32_t n,
                     const uint32_t* __restrict__ bits, uint32_t words, uint64_t mult,
                     const uint64_t* __restrict__ fat, uint32_t fat_idb, uint32_t fat_sh,
                     const uint4* __restrict__ fat16, double* __restrict__ score) {

    // Software-pipelined score side: the walk chain (csr -> adj, or one fat
    // gather) is the only dependency carried from step to step; the support
    // bit of x_l is loaded right after x_l is known, the rho gather of x_l is
    // issued at step l+1 and added at step l+2, so neither stalls the chain.
    // Additions still happen in step order (aesc.hpp:491-493).
    const uint64_t idmask = (uint64_t(1) << fat_idb) - 1, bmask = (uint64_t(1) << (fat_sh - fat_idb)) - 1;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    for (uint64_t base = uint64_t(warp) * 32 * WPT; base < nwalks; base += uint64_t(nwarps) * 32 * WPT) {
        uint32_t cur[WPT], seed[WPT], len[WPT], col[WPT], bcol[WPT], bw[WPT];
        double sc[WPT], rv[WPT];
        uint32_t maxlen = 1;
#pragma unroll
        for (int r = 0; r < WPT; ++r) {
            const uint64_t e = base + uint64_t(r) * 32 + lane;
            len[r] = 1;
            sc[r] = 0.0;
            rv[r] = 0.0;
            bw[r] = 0;
            cur[r] = 0;
            seed[r] = 0;
            col[r] = 0;
            bcol[r] = 0;
            if (e < nwalks) {
                const uint32_t w = vals[e];
                const WalkGroup G = groups[gidx[e]];
                const uint32_t local = w - G.walk_off;
                const uint32_t side = local >= G.pairs;
                seed[r] = walk_seed(G.edge_seed, 2 * (G.k0 + (local - side * G.pairs)) + side);
                cur[r] = side ? G.vj : G.vi;
                len[r] = G.len;
                col[r] = G.col * n;  // 32-bit element offsets: kCols * n < 2^32 (checked by the host)
                bcol[r] = G.col * words;
            }
            maxlen = max(maxlen, len[r]);
        }
        maxlen = __reduce_max_sync(0xffffffffu, maxlen);
        uint2 rec[WPT];
        if constexpr (FAT || F16) {
#pragma unroll
            for (int r = 0; r < WPT; ++r) rec[r] = len[r] > 1 ? ldg_csr(csr + cur[r]) : make_uint2(0, 1);
        }
        for (uint32_t l = 1; l < maxlen + 2; ++l) {
            const StepHash shs = step_hash(mult, l);
            if constexpr (!FAT && !F16) {  // critical load of step l first
#pragma unroll
                for (int r = 0; r < WPT; ++r)
                    if (l < len[r]) rec[r] = ldg_csr(csr + cur[r]);
            }
#pragma unroll
            for (int r = 0; r < WPT; ++r) {
                sc[r] += rv[r];  // step l-2 (0.0 when it was not a support step)
                // step l-1: cur is still x_{l-1}; bw holds its support bit
                const bool hit = BITMAP ? ((bw[r] >> (cur[r] & 31)) & 1u) != 0 : bw[r] != 0;
                rv[r] = hit ? __ldg(R + (col[r] + cur[r])) : 0.0;  // col[r] = column * n
            }
#pragma unroll
            for (int r = 0; r < WPT; ++r)
                if (l < len[r]) {
                    const uint32_t raw = seed[r] ^ hash_state_fast(shs, cur[r]);
                    if constexpr (F16) {
                        const uint4 f = __ldg(fat16 + (rec[r].x + scaled_index(raw, rec[r].y)));
                        cur[r] = f.x;
                        rec[r] = make_uint2(f.y, f.z);
                    } else if constexpr (FAT) {
                        const uint64_t f = __ldg(reinterpret_cast<const unsigned long long*>(fat) + rec[r].x +
                                                 scaled_index(raw, rec[r].y));
                        cur[r] = uint32_t(f & idmask);
                        rec[r] = make_uint2(uint32_t((f >> fat_idb) & bmask), uint32_t(f >> fat_sh));
                    } else {
                        cur[r] = adj_at<PACKED>(adj, adjp, rec[r].x + scaled_index(raw, rec[r].y));
                    }
                    SABA_DCHECK(cur[r] < n);
                    if constexpr (BITMAP)
                        bw[r] = __ldg(bits + (bcol[r] + (cur[r] >> 5)));
                    else
                        bw[r] = 1u;
                } else {
                    bw[r] = 0u;
                }
        }
#pragma unroll
        for (int r = 0; r < WPT; ++r) {  // walk ids are re-read (one register less per walk)
            const uint64_t e = base + uint64_t(r) * 32 + lane;
            if (e < nwalks) score[vals[e]] = sc[r];
        }
    }
}

// K4 for long walks on L2-resident graphs, with the rho values of the
// highest-degree vertices in shared memory. aesc_walk_sorted on such graphs
// is bound by the SM's L1-miss request rate (one request per clock; ncu:
// l1tex2xbar 93%): a fat gather and a rho gather per step, of which the rho
// gathers of hubs are the cacheable half. Here a 1024-thread block takes
// tiles of consecutive sorted walks from a device counter; consecutive walks
// belong to one (slot, side) segment and consecutive segments to one source,
// so a tile has one rho column almost always. The block keeps rho of that
// column for the nhub highest-degree vertices in shared memory (reloaded
// when the tile's column changes) and the fat record carries the neighbour's
// hub slot in its spare high bits, so the rho of a hub is a shared-memory
// load and only the tail (and the walks of a tile's second column, if any)
// gathers R. Same walks, seeds and step-order sums as aesc_walk_sorted.
template <int WPT, int THREADS>
__global__ void __launch_bounds__(THREADS)
    aesc_walk_hub(const uint32_t* __restrict__ gidx, const uint32_t* __restrict__ vals, uint32_t nwalks,
                  const WalkGroup* __restrict__ groups, const uint2* __restrict__ csr,
                  const double* __restrict__ R, uint32_t n, uint64_t mult, const uint64_t* __restrict__ fat,
                  uint32_t fat_idb, uint32_t fat_sh, uint32_t hub_shift,
                  const uint32_t* __restrict__ hub_vertex, uint32_t nhub, unsigned int* __restrict__ tile_next,
                  double* __restrict__ score) {
    extern __shared__ double rho_s[];
    __shared__ uint32_t s_tile, s_col;
    constexpr uint32_t TILE = THREADS * WPT;
    const uint32_t ntiles = (nwalks + TILE - 1) / TILE;
    const uint64_t idmask = (uint64_t(1) << fat_idb) - 1, bmask = (uint64_t(1) << (fat_sh - fat_idb)) - 1;
    const uint32_t dmask = (1u << (hub_shift - fat_sh)) - 1;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t cached_col = UINT32_MAX;  // block-uniform: column whose hub rho is in rho_s
    for (;;) {
        if (threadIdx.x == 0) {
            s_tile = atomicAdd(tile_next, 1u);
            if (s_tile < ntiles) s_col = groups[gidx[uint64_t(s_tile) * TILE]].col;
        }
        __syncthreads();
        const uint32_t tile = s_tile;
        if (tile >= ntiles) break;
        const uint32_t tcol = s_col;
        if (tcol != cached_col) {
            const double* __restrict__ Rc = R + size_t(tcol) * n;
            for (uint32_t h = threadIdx.x; h < nhub; h += THREADS) rho_s[h] = __ldg(Rc + __ldg(hub_vertex + h));
            cached_col = tcol;
            __syncthreads();
        }
        const uint64_t base = uint64_t(tile) * TILE + uint64_t(warp) * 32 * WPT;
        uint32_t cur[WPT], seed[WPT], len[WPT], col[WPT], hs[WPT];
        bool mine[WPT], stepped[WPT];
        double sc[WPT], rv[WPT];
        uint2 rec[WPT];
        uint32_t maxlen = 1;
#pragma unroll
        for (int r = 0; r < WPT; ++r) {
            const uint64_t e = base + uint64_t(r) * 32 + lane;
            len[r] = 1;
            sc[r] = 0.0;
            rv[r] = 0.0;
            stepped[r] = false;
            cur[r] = 0;
            seed[r] = 0;
            col[r] = 0;
            hs[r] = 0;
            mine[r] = false;
            if (e < nwalks) {
                const uint32_t w = vals[e];
                const WalkGroup G = groups[gidx[e]];
                const uint32_t local = w - G.walk_off;
                const uint32_t side = local >= G.pairs;
                seed[r] = walk_seed(G.edge_seed, 2 * (G.k0 + (local - side * G.pairs)) + side);
                cur[r] = side ? G.vj : G.vi;
                len[r] = G.len;
                col[r] = G.col * n;  // 32-bit element offsets: kCols * n < 2^32 (checked by the host)
                mine[r] = G.col == tcol;
            }
            rec[r] = len[r] > 1 ? ldg_csr(csr + cur[r]) : make_uint2(0, 1);
            maxlen = max(maxlen, len[r]);
        }
        maxlen = __reduce_max_sync(0xffffffffu, maxlen);
        for (uint32_t l = 1; l < maxlen + 2; ++l) {
            const StepHash shs = step_hash(mult, l);
#pragma unroll
            for (int r = 0; r < WPT; ++r) {
                sc[r] += rv[r];  // step l-2 (0.0 when there was none)
                // step l-1: cur is still x_{l-1}, hs its hub slot
                rv[r] = 0.0;
                if (stepped[r]) {
                    SABA_DCHECK(hs[r] <= nhub);
                    rv[r] = hs[r] != 0 && mine[r] ? rho_s[hs[r] - 1] : __ldg(R + (col[r] + cur[r]));
                }
            }
#pragma unroll
            for (int r = 0; r < WPT; ++r) {
                stepped[r] = l < len[r];
                if (stepped[r]) {
                    const uint32_t raw = seed[r] ^ hash_state_fast(shs, cur[r]);
                    const uint64_t f = __ldg(reinterpret_cast<const unsigned long long*>(fat) + rec[r].x +
                                             scaled_index(raw, rec[r].y));
                    cur[r] = uint32_t(f & idmask);
                    rec[r] = make_uint2(uint32_t((f >> fat_idb) & bmask), uint32_t(f >> fat_sh) & dmask);
                    hs[r] = uint32_t(f >> hub_shift);
                    SABA_DCHECK(cur[r] < n);
                }
            }
        }
#pragma unroll
        for (int r = 0; r < WPT; ++r) {
            const uint64_t e = base + uint64_t(r) * 32 + lane;
            if (e < nwalks) score[vals[e]] = sc[r];
        }
        __syncthreads();  // every warp is done with s_tile / s_col / rho_s before the next tile
    }
}

// Per-vertex walk records of one batch (beyond-L2 graphs): column c's
// record of vertex v is {base, degree, rho_c(v)} in 16 B, so the step from
// x_{l-1} loads ONE record that carries both what the selection needs and the
// score term of x_{l-1} (aesc.hpp:491-493) — two dependent gathers per step
// (record, neighbour id) instead of three (csr, neighbour id, rho). rho_c is
// exact zero outside column c's support, as in R.
__global__ void aesc_build_records(const uint2* __restrict__ csr, const double* __restrict__ R, uint32_t n,
                                   uint32_t ncols, uint4* __restrict__ recs) {
    const uint64_t total = uint64_t(ncols) * n;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t v = uint32_t(i % n);
        const uint2 r = csr[v];
        const double rho = __ldcs(R + i);
        recs[i] = make_uint4(r.x, r.y, uint32_t(__double_as_longlong(rho)),
                             uint32_t(uint64_t(__double_as_longlong(rho)) >> 32));
    }
}

// K4 over per-vertex records (see aesc_build_records). Same walks, same
// seeds, same step-order score sum as aesc_walk_sorted: the record loaded to
// leave x_{l-1} adds rho(x_{l-1}) for l >= 2, and x_{len-1}'s record is
// loaded once after the loop.
template <bool PACKED, int WPT, int MINB>
__global__ void __launch_bounds__(256, MINB)
    aesc_walk_rec(const uint32_t* __restrict__ gidx, const uint32_t* __restrict__ vals, uint32_t nwalks,
                  const WalkGroup* __restrict__ groups, const uint4* __restrict__ recs,
                  const uint32_t* __restrict__ adj, const uint64_t* __restrict__ adjp, uint32_t n, uint64_t mult,
                  double* __restrict__ score) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    for (uint64_t base = uint64_t(warp) * 32 * WPT; base < nwalks; base += uint64_t(nwarps) * 32 * WPT) {
        uint32_t cur[WPT], seed[WPT], len[WPT], col[WPT];  // col = column * n (< 2^32, host-checked)
        double sc[WPT];
        uint32_t maxlen = 1;
#pragma unroll
        for (int r = 0; r < WPT; ++r) {
            const uint64_t e = base + uint64_t(r) * 32 + lane;
            len[r] = 1;
            sc[r] = 0.0;
            cur[r] = 0;
            seed[r] = 0;
            col[r] = 0;
            if (e < nwalks) {
                const uint32_t w = vals[e];
                const WalkGroup G = groups[gidx[e]];
                const uint32_t local = w - G.walk_off;
                const uint32_t side = local >= G.pairs;
                seed[r] = walk_seed(G.edge_seed, 2 * (G.k0 + (local - side * G.pairs)) + side);
                cur[r] = side ? G.vj : G.vi;
                len[r] = G.len;
                col[r] = G.col * n;
            }
            maxlen = max(maxlen, len[r]);
        }
        maxlen = __reduce_max_sync(0xffffffffu, maxlen);
        for (uint32_t l = 1; l < maxlen; ++l) {
            const StepHash shs = step_hash(mult, l);
            uint4 q[WPT];
#pragma unroll
            for (int r = 0; r < WPT; ++r)
                if (l < len[r]) q[r] = __ldg(recs + (col[r] + cur[r]));
#pragma unroll
            for (int r = 0; r < WPT; ++r)
                if (l < len[r]) {
                    if (l >= 2) sc[r] += __hiloint2double(int(q[r].w), int(q[r].z));  // rho(x_{l-1})
                    const uint32_t raw = seed[r] ^ hash_state_fast(shs, cur[r]);
                    cur[r] = adj_at<PACKED>(adj, adjp, q[r].x + scaled_index(raw, q[r].y));
                    SABA_DCHECK(cur[r] < n && q[r].y > 0);
                }
        }
#pragma unroll
        for (int r = 0; r < WPT; ++r) {
            if (len[r] > 1) {  // rho(x_{len-1})
                const uint4 q = __ldg(recs + (col[r] + cur[r]));
                sc[r] += __hiloint2double(int(q.w), int(q.z));
            }
            const uint64_t e = base + uint64_t(r) * 32 + lane;
            if (e < nwalks) score[vals[e]] = sc[r];
        }
    }
}

// (a_k - b_k) / n_req over a tile of pair indices, thread-sequential then a
// fixed block tree (aesc.hpp:522 folds left; only the order differs).
__global__ void __launch_bounds__(256)
    aesc_pair_reduce(const PairTile* __restrict__ tiles, uint32_t ntiles,
                     const WalkGroup* __restrict__ groups, const double* __restrict__ score,
                     double* __restrict__ partials) {
    using Reduce = cub::BlockReduce<double, 256, cub::BLOCK_REDUCE_WARP_REDUCTIONS>;
    __shared__ typename Reduce::TempStorage tmp;
    constexpr uint32_t IPT = kPairTile / 256;
    for (uint32_t ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
        const PairTile T = tiles[ti];
        const WalkGroup G = groups[T.group];
        double x = 0.0;
#pragma unroll
        for (uint32_t i = 0; i < IPT; ++i) {
            const uint32_t p = threadIdx.x * IPT + i;
            if (p < T.count) {
                const uint32_t k = G.walk_off + T.p0 + p;
                x += (score[k] - score[k + G.pairs]) * T.inv_n;
            }
        }
        const double tot = Reduce(tmp).Sum(x);
        if (threadIdx.x == 0) partials[T.out] = tot;
        __syncthreads();
    }
}

__global__ void aesc_slot_reduce(const SlotWork* __restrict__ sw, uint32_t nslots,
                                 const double* __restrict__ partials, double* __restrict__ g_hat) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nslots; i += gridDim.x * blockDim.x) {
        const SlotWork w = sw[i];
        double acc = 0.0;
        for (uint32_t t = w.t0; t < w.t1; ++t) acc += partials[t];
        g_hat[w.slot] += acc;
    }
}

__global__ void aesc_symmetrise(const uint2* __restrict__ csr, const uint32_t* __restrict__ adj,
                                const uint32_t* __restrict__ slot_edge, uint32_t n,
                                const double* __restrict__ g_hat, double* __restrict__ s_hat) {
    for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x) {
        const uint2 r = csr[u];
        for (uint32_t s = r.x; s < r.x + r.y; ++s) {
            const uint32_t v = adj[s];
            if (v <= u) continue;
            const uint2 rv = csr[v];
            uint32_t lo = rv.x, hi = rv.x + rv.y;
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (adj[mid] < u) lo = mid + 1; else hi = mid;
            }
            s_hat[slot_edge[s]] = g_hat[s] + g_hat[lo];
        }
    }
}

// ------------------------------------------------------------------ host

template <class T>
T* buf(DevBuf& b, size_t count) {
    return static_cast<T*>(b.ensure(sizeof(T) * (count ? count : 1)));
}

struct Engine {
    saba_cu_graph* g;
    AescState* st;
    cudaStream_t s;
    AescParams p{};
    SlotTau tau_slot;  // tau per directed slot (host side)
    uint32_t launches = 0;
    uint64_t pairs = 0, steps = 0;
    cudaGraphExec_t depth_graph = nullptr;  // depths_per_graph() captured depths

    ~Engine() {
        if (depth_graph) cudaGraphExecDestroy(depth_graph);
    }

    explicit Engine(saba_cu_graph* g_, int workspace = 0) : g(g_) {
        if (!g->aesc) g->aesc = new AescState[kWorkspaces];
        st = &g->aesc[workspace];
        if (!st->stream) {
            // two batches in flight contend for the SMs: the propagation is a
            // serial chain of short kernels, the walk phase a few long ones,
            // so propagation runs on a high-priority stream and the walks on
            // a low-priority one (SABA_AESC_PRIO=0: one default stream)
            int lo = 0, hi = 0;
            SABA_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            const char* e = getenv("SABA_AESC_PRIO");
            if (e && atoi(e) == 0) lo = hi = 0;
            SABA_CUDA_CHECK(cudaStreamCreateWithPriority(&st->stream, cudaStreamNonBlocking, hi));
            SABA_CUDA_CHECK(cudaStreamCreateWithPriority(&st->stream_walk, cudaStreamNonBlocking, lo));
            SABA_CUDA_CHECK(cudaHostAlloc(&st->h_ctrl, sizeof(uint64_t) * kCtrlWords, cudaHostAllocDefault));
            for (cudaEvent_t& e : st->ev_walk) SABA_CUDA_CHECK(cudaEventCreate(&e));
        }
        s = st->stream;
        const uint32_t n = g->n;
        // the walk kernel addresses the rho block with 32-bit element offsets
        check_data(uint64_t(kCols) * n < (uint64_t(1) << 32),
                   "graph too large for the AESC batch layout (n must be < 2^26)");
        if (st->n_cap < n) {
            const size_t rows = size_t(n) * kCols;
            for (int b = 0; b < 2; ++b) {
                SABA_CUDA_CHECK(cudaMemsetAsync(buf<double>(st->P[b], rows), 0, sizeof(double) * rows, s));
                SABA_CUDA_CHECK(cudaMemsetAsync(buf<double>(st->Q[b], rows), 0, sizeof(double) * rows, s));
                SABA_CUDA_CHECK(cudaMemsetAsync(buf<uint64_t>(st->M[b], n), 0, sizeof(uint64_t) * n, s));
                buf<uint32_t>(st->ulist[b], n);
            }
            SABA_CUDA_CHECK(cudaMemsetAsync(buf<double>(st->R, rows), 0, sizeof(double) * rows, s));
            SABA_CUDA_CHECK(cudaMemsetAsync(buf<uint32_t>(st->bits, size_t(kCols) * words()), 0,
                                            sizeof(uint32_t) * kCols * words(), s));
            SABA_CUDA_CHECK(cudaMemsetAsync(buf<uint32_t>(st->flag, n), 0, sizeof(uint32_t) * n, s));
            SABA_CUDA_CHECK(cudaMemsetAsync(buf<uint32_t>(st->tflag, n), 0, sizeof(uint32_t) * n, s));
            buf<uint32_t>(st->tlist, n);
            st->n_cap = n;
        }
        if (!st->heavy_built) build_heavy();
        buf<uint32_t>(st->ucount, 2);
        buf<uint32_t>(st->tcount, 1);
        buf<uint32_t>(st->col_src, kCols);
        buf<uint32_t>(st->col_tau, kCols);
        buf<uint64_t>(st->degsum[0], kCols);
        buf<uint64_t>(st->degsum[1], kCols);
        buf<uint32_t>(st->tt, kCols);
        // kEdgeVisits accumulates over the batches of one estimator call
        SABA_CUDA_CHECK(cudaMemsetAsync(buf<uint64_t>(st->ctrl, kCtrlWords), 0, sizeof(uint64_t) * kCtrlWords, s));
    }

    // Rows with degree > kHeavy and their fixed pieces of kHeavy neighbours.
    void build_heavy() {
        std::vector<uint32_t> rows, poff{0};
        std::vector<HeavyPiece> pcs;
        for (uint32_t v = 0; v < g->n; ++v) {
            const uint32_t b = g->h_off[v], e = g->h_off[v + 1];
            if (e - b <= kHeavy) continue;
            rows.push_back(v);
            for (uint32_t s = b; s < e; s += kHeavy) pcs.push_back({v, s, std::min(e, s + kHeavy), 0});
            poff.push_back(uint32_t(pcs.size()));
        }
        st->nheavy = uint32_t(rows.size());
        st->npieces = uint32_t(pcs.size());
        SABA_CUDA_CHECK(cudaMemcpyAsync(buf<uint32_t>(st->heavy_rows, rows.size()), rows.data(),
                                        sizeof(uint32_t) * rows.size(), cudaMemcpyHostToDevice, s));
        SABA_CUDA_CHECK(cudaMemcpyAsync(buf<uint32_t>(st->piece_off, poff.size()), poff.data(),
                                        sizeof(uint32_t) * poff.size(), cudaMemcpyHostToDevice, s));
        SABA_CUDA_CHECK(cudaMemcpyAsync(buf<HeavyPiece>(st->pieces, pcs.size()), pcs.data(),
                                        sizeof(HeavyPiece) * pcs.size(), cudaMemcpyHostToDevice, s));
        buf<double>(st->part, size_t(pcs.size()) * kCols);
        buf<uint64_t>(st->part_mask, pcs.size());
        std::vector<uint32_t> light;
        light.reserve(g->n);
        for (uint32_t v = 0; v < g->n; ++v)
            if (g->h_off[v + 1] - g->h_off[v] <= kHeavy) light.push_back(v);
        std::stable_sort(light.begin(), light.end(), [&](uint32_t a, uint32_t b) { return deg(a) > deg(b); });
        st->nlight = getenv("SABA_PULL_STATIC") ? 0u : uint32_t(light.size());
        if (!light.empty())
            SABA_CUDA_CHECK(cudaMemcpyAsync(buf<uint32_t>(st->light_order, light.size()), light.data(),
                                            sizeof(uint32_t) * light.size(), cudaMemcpyHostToDevice, s));
        SABA_CUDA_CHECK(cudaStreamSynchronize(s));  // host vectors go out of scope
        st->heavy_built = true;
    }

    // a per-slot array must outlive the engine; a uniform plan is filled on the device
    void upload_tau(const SlotTau& t) {
        tau_slot = t;
        const size_t slots = 2 * g->m;
        uint32_t* d = buf<uint32_t>(st->tau_slot, slots);
        if (t.v == nullptr)
            fill_u32(d, t.uni, slots, s);
        else
            copy_h2d(d, t.v, sizeof(uint32_t) * slots, s);
    }

    uint32_t deg(uint32_t v) const { return g->h_off[v + 1] - g->h_off[v]; }
    uint32_t words() const { return (g->n + 31) / 32; }
    bool last_dense = false;  // did the last batch switch to dense rows

    uint64_t read_ctrl(int word) {
        SABA_CUDA_CHECK(cudaMemcpyAsync(st->h_ctrl + word, st->ctrl.as<uint64_t>() + word,
                                        sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
        SABA_CUDA_CHECK(cudaStreamSynchronize(s));
        return st->h_ctrl[word];
    }

    // Propagation of one batch (advance_to_switch for every column); returns
    // tau~ per column. *parity = index of the P buffer holding p_tau~.
    std::vector<uint32_t> propagate(const std::vector<uint32_t>& cols, double* g_hat_dev,
                                    int* parity = nullptr) {
        const int nc = int(cols.size());
        const uint32_t n = g->n;
        std::vector<uint32_t> ctau(nc);
        uint32_t lmax = 0;
        for (int c = 0; c < nc; ++c) {
            uint32_t t = 0;
            for (uint32_t sl = g->h_off[cols[c]]; sl < g->h_off[cols[c] + 1]; ++sl)
                t = std::max(t, tau_slot[sl]);
            ctau[c] = t;  // tau_src (aesc.hpp:386-388)
            lmax = std::max(lmax, t);
        }
        if (p.cap >= 0) lmax = uint32_t(std::min<int64_t>(lmax, p.cap));
        SABA_CUDA_CHECK(cudaMemcpyAsync(st->col_src.p, cols.data(), sizeof(uint32_t) * nc, cudaMemcpyHostToDevice, s));
        SABA_CUDA_CHECK(cudaMemcpyAsync(st->col_tau.p, ctau.data(), sizeof(uint32_t) * nc, cudaMemcpyHostToDevice, s));
        double* P[2] = {st->P[0].as<double>(), st->P[1].as<double>()};
        double* Q[2] = {st->Q[0].as<double>(), st->Q[1].as<double>()};
        unsigned long long* M[2] = {st->M[0].as<unsigned long long>(), st->M[1].as<unsigned long long>()};
        uint32_t* UL[2] = {st->ulist[0].as<uint32_t>(), st->ulist[1].as<uint32_t>()};
        uint32_t* UC = st->ucount.as<uint32_t>();
        unsigned long long* DS[2] = {st->degsum[0].as<unsigned long long>(),
                                     st->degsum[1].as<unsigned long long>()};
        auto* ctrl = st->ctrl.as<unsigned long long>();
        const uint2* csr = g->d_csr;
        const uint32_t* adj = g->d_adj;
        const uint32_t* tsl = st->tau_slot.as<uint32_t>();
        uint32_t* flag = st->flag.as<uint32_t>();
        uint32_t* tflag = st->tflag.as<uint32_t>();
        uint32_t* tlist = st->tlist.as<uint32_t>();
        uint32_t* tcount = st->tcount.as<uint32_t>();
        uint32_t* ttd = st->tt.as<uint32_t>();
        aesc_init<<<1, kCols, 0, s>>>(st->col_src.as<uint32_t>(), nc, csr, p, P[0], Q[0], M[0], UL[0],
                                      UC, tflag, tlist, tcount, DS[0], ttd, ctrl, g_hat_dev);
        ++launches;
        const int grid = g->sm_count * 8;
        auto occ_grid = [&](auto kernel) {
            int occ = 0;
            SABA_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, 256, 0));
            return g->sm_count * std::max(occ, 1);
        };
        const int grid_pull = occ_grid(aesc_pull), grid_comb = occ_grid(aesc_pull_combine);
        // One depth (aesc.hpp:391-397 + hook): every argument except the
        // buffer parity is fixed, the depth itself lives on the device.
        // The check of depth 0 runs once here; every depth ends with the hook
        // and the check of the next depth fused (aesc_hook_check).
        aesc_check<<<1, kCols, 0, s>>>(UC + 1, st->col_src.as<uint32_t>(), st->col_tau.as<uint32_t>(), csr, tsl,
                                       p, DS[0], DS[1], ttd, ctrl, ctrl + kEdgeVisits);
        ++launches;
        auto enqueue_depth = [&](int cur) {
            aesc_rho_expand<<<grid, 256, 0, s>>>(P[cur], csr, adj, M[cur], UL[cur], UC + cur, UL[cur ^ 1],
                                                 UC + (cur ^ 1), flag, tflag, tlist, tcount, ctrl, n,
                                                 st->R.as<double>(), st->bits.as<uint32_t>(), words());
            // sparse depths: pieces of candidate hub rows; dense depths: the
            // pull kernel takes the pieces into its dynamic work list
            if (st->npieces)
                aesc_pull_pieces<<<grid, 256, 0, s>>>(st->pieces.as<HeavyPiece>(), st->npieces, adj,
                                                      Q[cur], M[cur], flag, st->part.as<double>(),
                                                      st->part_mask.as<unsigned long long>(), ctrl,
                                                      st->nlight, DS[cur], 2 * g->m, pull_skip_force());
            aesc_pull<<<grid_pull, 256, 0, s>>>(csr, adj, Q[cur], M[cur], P[cur ^ 1], Q[cur ^ 1], M[cur ^ 1],
                                           UL[cur ^ 1], UC + (cur ^ 1), flag, DS[cur ^ 1], ctrl, n,
                                           st->nlight ? st->light_order.as<uint32_t>() : nullptr, st->nlight,
                                           st->pieces.as<HeavyPiece>(), st->npieces, st->part.as<double>(),
                                           st->part_mask.as<unsigned long long>(), DS[cur], 2 * g->m,
                                           pull_skip_force());
            if (st->npieces)
                aesc_pull_combine<<<grid_comb, 256, 0, s>>>(
                    st->heavy_rows.as<uint32_t>(), st->piece_off.as<uint32_t>(), st->nheavy, csr,
                    st->part.as<double>(), st->part_mask.as<unsigned long long>(), P[cur ^ 1],
                    Q[cur ^ 1], M[cur ^ 1], flag, DS[cur ^ 1], ctrl);
            aesc_hook_check<<<kCols, 128, 0, s>>>(st->col_src.as<uint32_t>(), st->col_tau.as<uint32_t>(), csr, adj,
                                                  tsl, P[cur ^ 1], p, DS[cur ^ 1], DS[cur], ttd, UC + cur, ctrl,
                                                  g_hat_dev, ctrl + kEdgeVisits);
        };
        const uint32_t per_depth = st->npieces ? 5 : 3;
        if (!depth_graph) {
            // depths_per_graph() depths (even, so the buffer parity returns to 0)
            // captured once per estimator call and replayed for every batch
            cudaGraph_t graph;
            SABA_CUDA_CHECK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
            for (int d = 0; d < depths_per_graph(); ++d) enqueue_depth(d & 1);
            SABA_CUDA_CHECK(cudaStreamEndCapture(s, &graph));
            SABA_CUDA_CHECK(cudaGraphInstantiate(&depth_graph, graph, 0));
            SABA_CUDA_CHECK(cudaGraphDestroy(graph));
        }
        // columns freeze at the latest when l reaches tau_src <= lmax; extra
        // depths of the last replay only run early-exiting kernels
        for (uint32_t l = 0; l <= lmax; l += depths_per_graph()) {
            SABA_CUDA_CHECK(cudaGraphLaunch(depth_graph, s));
            launches += per_depth * depths_per_graph();
            if (read_ctrl(kActive) == 0) break;
        }
        // Columns frozen by the check fused into a replay's last depth get
        // their rho from the next depth's first kernel, which no replay runs:
        // run it here (a replay has an even number of depths, so that depth
        // has parity 0; the expansion half exits, nothing is active).
        aesc_rho_expand<<<grid, 256, 0, s>>>(P[0], csr, adj, M[0], UL[0], UC, UL[1], UC + 1, flag, tflag, tlist,
                                             tcount, ctrl, n, st->R.as<double>(), st->bits.as<uint32_t>(), words());
        ++launches;
        SABA_CUDA_CHECK(cudaGetLastError());
        if (parity) *parity = 0;
        last_dense = read_ctrl(kDense) != 0;
        std::vector<uint32_t> tt(nc);
        SABA_CUDA_CHECK(cudaMemcpyAsync(tt.data(), ttd, sizeof(uint32_t) * nc, cudaMemcpyDeviceToHost, s));
        SABA_CUDA_CHECK(cudaStreamSynchronize(s));
        return tt;
    }

    void clear_batch(int nc) {
        const uint32_t n = g->n;
        if (read_ctrl(kDense)) {  // dense batches touched every row
            const size_t rows = size_t(n) * kCols;
            for (int b = 0; b < 2; ++b) {
                SABA_CUDA_CHECK(cudaMemsetAsync(st->P[b].p, 0, sizeof(double) * rows, s));
                SABA_CUDA_CHECK(cudaMemsetAsync(st->Q[b].p, 0, sizeof(double) * rows, s));
                SABA_CUDA_CHECK(cudaMemsetAsync(st->M[b].p, 0, sizeof(uint64_t) * n, s));
            }
            SABA_CUDA_CHECK(cudaMemsetAsync(st->R.p, 0, sizeof(double) * size_t(n) * nc, s));
            SABA_CUDA_CHECK(cudaMemsetAsync(st->bits.p, 0, sizeof(uint32_t) * size_t(words()) * nc, s));
            SABA_CUDA_CHECK(cudaMemsetAsync(st->tflag.p, 0, sizeof(uint32_t) * n, s));
            return;
        }
        aesc_clear<<<g->sm_count * 8, 256, 0, s>>>(
            st->tlist.as<uint32_t>(), st->tcount.as<uint32_t>(), st->P[0].as<double>(),
            st->P[1].as<double>(), st->Q[0].as<double>(), st->Q[1].as<double>(),
            st->M[0].as<unsigned long long>(), st->M[1].as<unsigned long long>(), st->R.as<double>(),
            n, st->tflag.as<uint32_t>(), nc, st->bits.as<uint32_t>(), words());
        SABA_CUDA_CHECK(cudaGetLastError());
        ++launches;
    }
};

void validate_cfg(const saba_cu_aesc_config& c) {
    // aesc.hpp:637-641 (same order)
    check_arg(c.epsilon > 0.0 && c.epsilon < 1.0, "aesc: epsilon must be in (0,1)");
    check_arg(c.delta > 0.0 && c.delta < 1.0, "aesc: delta must be in (0,1)");
    check_arg(c.power_iterations >= 1, "aesc: omega must be >= 1");
    check_arg(c.lanes >= 1 && c.lanes <= 64 && (c.lanes & (c.lanes - 1)) == 0,
              "aesc: lanes must be a power of two in [1, 64]");
    check_arg(c.mode == SABA_MODE_HASH || c.mode == SABA_MODE_SABA,
              "aesc: mode not supported on GPU (naive/vector-mod are CPU LCG baselines)");
}

// Host plan of one walk phase: slots -> groups -> chunks, tiles in pair order.
struct TileBuilder {
    struct Chunk {
        std::vector<WalkGroup> groups;
        std::vector<PairTile> tiles;
        uint32_t walks = 0;
        uint64_t steps = 0;  // walk steps of the chunk (both sides)
    };
    std::vector<Chunk> chunks;
    std::vector<SlotWork> slots;
    uint32_t ntiles = 0;

    void clear() {
        chunks.clear();
        slots.clear();
        ntiles = 0;
    }
    bool empty() const { return slots.empty(); }

    void add(uint32_t slot, uint32_t vi, uint32_t vj, uint32_t len, uint64_t n_req, uint64_t edge_seed,
             uint32_t col) {
        SlotWork w{ntiles, 0, slot, 0};
        const double inv_n = 1.0 / double(n_req);
        for (uint64_t k0 = 0; k0 < n_req; k0 += kGroupPairs) {
            const uint32_t pairs = uint32_t(std::min<uint64_t>(kGroupPairs, n_req - k0));
            if (chunks.empty() || chunks.back().walks + 2ull * pairs > kChunkWalks) chunks.emplace_back();
            Chunk& c = chunks.back();
            const uint32_t gi = uint32_t(c.groups.size());
            c.groups.push_back({edge_seed, k0, pairs, c.walks, vi, vj, len, col});
            for (uint32_t p0 = 0; p0 < pairs; p0 += kPairTile)
                c.tiles.push_back({inv_n, gi, p0, std::min(kPairTile, pairs - p0), ntiles++});
            c.walks += 2 * pairs;
            c.steps += 2ull * pairs * (len - 1);
        }
        w.t1 = ntiles;
        slots.push_back(w);
    }
};


// Walk phase: per chunk keygen -> radix sort (group, seed top bits) -> sorted
// walks -> pair tiles; then the per-slot fold into g_hat.
// Short walks beyond L2 (plan max tau below kShortWalk) step through 16-byte
// {id, base, degree} records: one dependent gather per step instead of csr
// then adjacency. Measured: cfg5 (tau 15) walks 4% faster; cfg4 (tau 127,
// long walks) 12% slower, as the 4x footprint costs L2 hits on hub lists.
// SABA_AESC_FAT16=0 disables.
constexpr uint32_t kShortWalk = 20;
#ifndef SABA_SHORT_WPT
#define SABA_SHORT_WPT 1
#endif
#ifndef SABA_SHORT_MINB
#define SABA_SHORT_MINB 8
#endif
constexpr int kShortWpt = SABA_SHORT_WPT, kShortMinb = SABA_SHORT_MINB;  // short-walk variant
bool aesc_fat16_enabled() {
    static const bool on = [] {
        const char* e = getenv("SABA_AESC_FAT16");
        return !e || atoi(e) != 0;
    }();
    return on;
}
bool aesc_fat_enabled() {  // SABA_AESC_FAT=0 disables (default: on when L2-resident)
    static const bool on = [] {
        const char* e = getenv("SABA_AESC_FAT");
        return !e || atoi(e) != 0;
    }();
    return on;
}

// Per-vertex records (aesc_walk_rec): 0 = off (default), 1 = on for the
// compact path (graphs beyond L2 without 16-byte slot records), 2 = for every
// batch (tuning knob SABA_AESC_REC). Measured and rejected as the default:
// one 16 B record gather per step in place of the csr + rho pair was slower
// on every config (walk phase cfg4 3.27 vs 2.93 s per 64 sources, cfg5 1.78
// vs 1.60 s per 512, cfg3 11.6 vs 10.6 s; profiles/r02_aesc_rec_experiment.txt):
// the dependent chain stays two gathers long and the 2.4 GB of per-column
// records (cfg4) cost more L2 capacity than the rho gather they replace.
int aesc_rec_mode() {
    static const int m = [] {
        const char* e = getenv("SABA_AESC_REC");
        return e ? atoi(e) : 0;
    }();
    return m;
}

// K4s host side: segments of the chunk, coarse tiles and the coarse-bucket
// table (a segment up to kFineDirect walks is one bucket), then count ->
// exclusive scan -> scatter -> fine bucketing into (out_w, out_g).
struct SortScratch {  // host side of one chunk's bucketing; lives until the chunk's sync
    std::vector<SortSeg> segs;
    std::vector<CoarseTile> ct;
    std::vector<uint32_t> cnt0, cb_seg;  // initial counts (whole small segments), owner segment
};
void bucket_walks(AescState* st, cudaStream_t s, const TileBuilder::Chunk& c, const WalkGroup* dg,
                  SortScratch& h, uint32_t* out_w, uint32_t* out_g, uint32_t* launches) {
    const uint32_t nw = c.walks;
    auto& segs = h.segs;
    auto& ct = h.ct;
    auto& cnt0 = h.cnt0;
    auto& cb_seg = h.cb_seg;
    segs.clear();
    ct.clear();
    cnt0.clear();
    cb_seg.clear();
    segs.reserve(2 * c.groups.size());
    for (uint32_t gi = 0; gi < uint32_t(c.groups.size()); ++gi) {
        const WalkGroup& G = c.groups[gi];
        for (uint32_t side = 0; side < 2; ++side) {
            SortSeg S{gi, side, G.walk_off + side * G.pairs, G.pairs, 0, uint32_t(cnt0.size())};
            if (S.size > kFineDirect) {
                while (S.d1 < kCoarseBitsMax && (uint64_t(kCoarseTarget) << S.d1) < S.size) ++S.d1;
                for (uint32_t t0 = 0; t0 < S.size; t0 += kCoarseTile)
                    ct.push_back({uint32_t(segs.size()), t0, std::min(kCoarseTile, S.size - t0), 0});
            }
            const uint32_t nb = 1u << S.d1;
            cnt0.insert(cnt0.end(), nb, S.d1 ? 0u : S.size);
            cb_seg.insert(cb_seg.end(), nb, uint32_t(segs.size()));
            segs.push_back(S);
        }
    }
    const uint32_t ncb = uint32_t(cnt0.size()), nseg = uint32_t(segs.size()), nct = uint32_t(ct.size());
    auto* d_seg = static_cast<SortSeg*>(st->sort_segs.ensure(sizeof(SortSeg) * nseg));
    auto* d_cbs = static_cast<uint32_t*>(st->cb_seg.ensure(sizeof(uint32_t) * ncb));
    auto* d_cnt = static_cast<uint32_t*>(st->cb_cnt.ensure(sizeof(uint32_t) * ncb));
    auto* d_start = static_cast<uint32_t*>(st->cb_start.ensure(sizeof(uint32_t) * ncb));
    SABA_CUDA_CHECK(cudaMemcpyAsync(d_seg, segs.data(), sizeof(SortSeg) * nseg, cudaMemcpyHostToDevice, s));
    SABA_CUDA_CHECK(cudaMemcpyAsync(d_cbs, cb_seg.data(), sizeof(uint32_t) * ncb, cudaMemcpyHostToDevice, s));
    SABA_CUDA_CHECK(cudaMemcpyAsync(d_cnt, cnt0.data(), sizeof(uint32_t) * ncb, cudaMemcpyHostToDevice, s));
    uint32_t* tmp = nullptr;
    if (nct) {
        auto* d_ct = static_cast<CoarseTile*>(st->coarse_tiles.ensure(sizeof(CoarseTile) * nct));
        SABA_CUDA_CHECK(cudaMemcpyAsync(d_ct, ct.data(), sizeof(CoarseTile) * nct, cudaMemcpyHostToDevice, s));
        sort_coarse_count<<<nct, 512, 0, s>>>(d_ct, d_seg, dg, d_cnt);
        SABA_CUDA_CHECK(cudaGetLastError());
        ++*launches;
    }
    size_t scan_bytes = 0;
    SABA_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, d_cnt, d_start, int(ncb), s));
    SABA_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(st->sort_tmp.ensure(scan_bytes), scan_bytes, d_cnt, d_start,
                                                  int(ncb), s));
    ++*launches;
    if (nct) {
        auto* d_cur = static_cast<uint32_t*>(st->cb_cursor.ensure(sizeof(uint32_t) * ncb));
        SABA_CUDA_CHECK(cudaMemcpyAsync(d_cur, d_start, sizeof(uint32_t) * ncb, cudaMemcpyDeviceToDevice, s));
        tmp = static_cast<uint32_t*>(st->vals[1].ensure(sizeof(uint32_t) * nw));
        sort_coarse_scatter<<<nct, 512, 0, s>>>(st->coarse_tiles.as<CoarseTile>(), d_seg, dg, d_cur, tmp);
        SABA_CUDA_CHECK(cudaGetLastError());
        ++*launches;
    }
    sort_fine<<<ncb, 256, 0, s>>>(d_cbs, d_seg, dg, d_cnt, d_start, tmp, out_w, out_g);
    SABA_CUDA_CHECK(cudaGetLastError());
    ++*launches;
}

struct Launch {
    const uint32_t *out_g, *out_w;
    uint32_t nw;
    const WalkGroup* dg;
    const saba_cu_graph* g;
    const double* R;
    const uint32_t* bits;
    uint32_t words;
    uint64_t mult;
    double* score;
    cudaStream_t s;
    const uint4* recs;  // per-vertex records of the batch (aesc_walk_rec), or null
};

template <bool P, int WPT, bool B, bool F, int MINB, bool F16 = false>
void walk_launch(const Launch& L) {
    auto k = aesc_walk_sorted<P, WPT, B, F, MINB, F16>;
    int occ = 0;
    SABA_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 256, 0));
    const int grid = int(std::min<uint64_t>((uint64_t(L.nw) + 32 * WPT - 1) / (32 * WPT) * 32 / 256 + 1,
                                            uint64_t(L.g->sm_count) * std::max(occ, 1)));
    k<<<grid, 256, 0, L.s>>>(L.out_g, L.out_w, L.nw, L.dg, L.g->d_csr, L.g->d_adj, L.g->d_adj_packed, L.R,
                             L.g->n, L.bits, L.words, L.mult, L.g->d_adj_fat, L.g->fat_idb, L.g->fat_sh,
                             L.g->d_adj_fat16, L.score);
}

template <bool P, int WPT, int MINB>
void rec_launch(const Launch& L) {
    auto k = aesc_walk_rec<P, WPT, MINB>;
    int occ = 0;
    SABA_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 256, 0));
    const int grid = int(std::min<uint64_t>((uint64_t(L.nw) + 32 * WPT - 1) / (32 * WPT) * 32 / 256 + 1,
                                            uint64_t(L.g->sm_count) * std::max(occ, 1)));
    k<<<grid, 256, 0, L.s>>>(L.out_g, L.out_w, L.nw, L.dg, L.recs, L.g->d_adj, L.g->d_adj_packed, L.g->n, L.mult,
                             L.score);
}

template <int WPT, int MINB>
void walk_dispatch(const Launch& L, bool fat, bool packed, bool f16) {
    if (L.recs) {
        if (packed) rec_launch<true, WPT, MINB>(L); else rec_launch<false, WPT, MINB>(L);
        return;
    }
    const bool b = L.bits != nullptr;
    if (f16) {
        if (b) walk_launch<false, WPT, true, false, MINB, true>(L); else walk_launch<false, WPT, false, false, MINB, true>(L);
    } else if (fat) {
        if (b) walk_launch<false, WPT, true, true, MINB>(L); else walk_launch<false, WPT, false, true, MINB>(L);
    } else if (packed) {
        if (b) walk_launch<true, WPT, true, false, MINB>(L); else walk_launch<true, WPT, false, false, MINB>(L);
    } else {
        if (b) walk_launch<false, WPT, true, false, MINB>(L); else walk_launch<false, WPT, false, false, MINB>(L);
    }
}

// SABA_AESC_L2WIN (experiment): pin what the walk kernel gathers per vertex in
// the persisting part of L2 while a chunk runs, so that the neighbour gathers
// streaming through L2 cannot evict it. 1 = the rho columns of the chunk's
// sources, 2 = the csr records. SABA_AESC_L2WIN_MB sizes the set-aside
// (default: the device maximum); `share` = walk streams that hold a window.
struct L2Window {
    int mode = 0;
    size_t setaside = 0, max_window = 0;
};
const L2Window& l2_window(int device) {
    static L2Window w[64];
    static std::once_flag once[64];
    std::call_once(once[device], [&] {
        const char* e = getenv("SABA_AESC_L2WIN");
        L2Window& x = w[device];
        x.mode = e ? atoi(e) : 0;
        if (!x.mode) return;
        int v = 0;
        SABA_CUDA_CHECK(cudaDeviceGetAttribute(&v, cudaDevAttrMaxPersistingL2CacheSize, device));
        x.setaside = size_t(v);
        if (const char* m = getenv("SABA_AESC_L2WIN_MB")) x.setaside = std::min(x.setaside, size_t(atoi(m)) << 20);
        SABA_CUDA_CHECK(cudaDeviceGetAttribute(&v, cudaDevAttrMaxAccessPolicyWindowSize, device));
        x.max_window = size_t(v);
        SABA_CUDA_CHECK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, x.setaside));
        if (getenv("SABA_TRACE"))
            fprintf(stderr, "[saba] aesc L2 window mode %d: set-aside %zu MB, max window %zu MB\n", x.mode,
                    x.setaside >> 20, x.max_window >> 20);
    });
    return w[device];
}
void set_l2_window(cudaStream_t s, const void* base, size_t bytes, const L2Window& w, int share) {
    cudaStreamAttrValue a{};
    a.accessPolicyWindow.base_ptr = const_cast<void*>(base);
    a.accessPolicyWindow.num_bytes = std::min(bytes, w.max_window);
    a.accessPolicyWindow.hitRatio =
        bytes ? std::min(1.0f, float(double(w.setaside) / double(share) / double(a.accessPolicyWindow.num_bytes))) : 0.f;
    a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    SABA_CUDA_CHECK(cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &a));
}

// SABA_AESC_HUB=N (experiment, default off): rho of the N highest-degree
// vertices in shared memory for long walks on the fat path (aesc_walk_hub).
// Measured on cfg3 (profiles/r02_aesc_hub_rho_experiment.txt): the walk
// kernels get ~7% faster with two workers, but a 1024-thread block with a
// 96 KB table leaves the other worker's propagation kernels less of each SM
// (propagation +20%), and with one worker nothing changes: the rho gathers of
// hubs were L1 hits already. 9.21 s without, 9.27-9.48 s with.
uint32_t aesc_hub_count() {
    static const uint32_t v = [] {
        const char* e = getenv("SABA_AESC_HUB");
        return e ? uint32_t(atoi(e)) : 0u;
    }();
    return v;
}

void run_tiles(saba_cu_graph* g, AescState* st, cudaStream_t s, TileBuilder& tb, const double* R,
               const uint32_t* bits, uint64_t mult, double* g_hat_dev, uint32_t* launches,
               const uint4* recs = nullptr, float* walk_kernel_ms = nullptr) {
    const uint32_t words = (g->n + 31) / 32;
    if (tb.empty()) return;
    double* part = static_cast<double*>(st->partials.ensure(sizeof(double) * std::max(tb.ntiles, 1u)));
    const bool packed = g->d_adj_packed != nullptr;
    // the fat adjacency is built (main thread) before any batch worker runs
    const bool fat = g->d_adj_fat != nullptr && fat_fits_l2(g) && aesc_fat_enabled();
    const bool f16 = !fat && g->d_adj_fat16 != nullptr && aesc_fat16_enabled();  // built for short plans only
    SortScratch scratch;
    for (TileBuilder::Chunk& c : tb.chunks) {
        const uint32_t ng = uint32_t(c.groups.size()), nw = c.walks, nt = uint32_t(c.tiles.size());
        auto* dg = static_cast<WalkGroup*>(st->groups.ensure(sizeof(WalkGroup) * ng));
        auto* dt = static_cast<PairTile*>(st->tiles.ensure(sizeof(PairTile) * nt));
        SABA_CUDA_CHECK(cudaMemcpyAsync(dg, c.groups.data(), sizeof(WalkGroup) * ng, cudaMemcpyHostToDevice, s));
        SABA_CUDA_CHECK(cudaMemcpyAsync(dt, c.tiles.data(), sizeof(PairTile) * nt, cudaMemcpyHostToDevice, s));
        uint32_t* out_g = static_cast<uint32_t*>(st->keys[0].ensure(sizeof(uint32_t) * nw));
        uint32_t* out_w = static_cast<uint32_t*>(st->vals[0].ensure(sizeof(uint32_t) * nw));
        double* score = static_cast<double*>(st->score.ensure(sizeof(double) * nw));
        bucket_walks(st, s, c, dg, scratch, out_w, out_g, launches);
        // walk shape of the chunk: mean steps per walk decides the variant
        // (measured on cfg5, ~12 steps, two workers: 1 walk/lane x 8 blocks
        // 1.53 s, 2 x 8 1.63, 2 x 6 1.62, 3 x 6 1.80, 4 x 5 1.88 per 768
        // sources; cfg3/cfg4, 24-73 steps: 4 x 5 is best by 3-4%)
        static const uint64_t short_steps = [] {  // SABA_SHORT_STEPS overrides (tuning knob)
            const char* e = getenv("SABA_SHORT_STEPS");
            return e ? uint64_t(atoi(e)) : uint64_t(kShortWalk);
        }();
        const bool short_walks = c.steps < short_steps * nw;
        const Launch L{out_g, out_w, nw, dg, g, R, bits, words, mult, score, s, recs};
        const L2Window& lw = l2_window(g->device);
        const bool windowed = lw.mode != 0 && !fat && !recs;
        if (windowed) {
            static const int share = [] {
                const char* e = getenv("SABA_AESC_WORKERS");
                return e && atoi(e) == 1 ? 1 : 2;
            }();
            if (lw.mode == 2) {
                set_l2_window(s, g->d_csr, sizeof(uint2) * g->n, lw, share);
            } else {
                uint32_t lo = UINT32_MAX, hi = 0;
                for (const WalkGroup& G : c.groups) {
                    lo = std::min(lo, G.col);
                    hi = std::max(hi, G.col);
                }
                set_l2_window(s, R + size_t(lo) * g->n, sizeof(double) * g->n * (size_t(hi) - lo + 1), lw, share);
            }
        }
        if (walk_kernel_ms) SABA_CUDA_CHECK(cudaEventRecord(st->ev_walk[0], s));
        const bool hub = fat && !short_walks && !recs && !bits && g->d_adj_fat_hub != nullptr;
        if (hub) {
            constexpr int T = 1024, WPT = 4;
            auto k = aesc_walk_hub<WPT, T>;
            const size_t smem = sizeof(double) * g->fat_hub_count;
            SABA_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            auto* ctr = static_cast<unsigned int*>(st->tile_next.ensure(sizeof(unsigned int), s));
            SABA_CUDA_CHECK(cudaMemsetAsync(ctr, 0, sizeof(unsigned int), s));
            const uint32_t ntiles = (nw + T * WPT - 1) / (T * WPT);
            k<<<std::min<uint32_t>(ntiles, uint32_t(g->sm_count)), T, smem, s>>>(
                out_g, out_w, nw, dg, g->d_csr, R, g->n, mult, g->d_adj_fat_hub, g->fat_idb, g->fat_sh,
                g->fat_hub_shift, g->d_fat_hub_vertex, g->fat_hub_count, ctr, score);
        } else if (short_walks)
            walk_dispatch<kShortWpt, kShortMinb>(L, fat, packed, f16);
        else
            walk_dispatch<4, 5>(L, fat, packed, false);
        SABA_CUDA_CHECK(cudaGetLastError());
        if (walk_kernel_ms) SABA_CUDA_CHECK(cudaEventRecord(st->ev_walk[1], s));
        if (windowed) set_l2_window(s, nullptr, 0, lw, 1);
        aesc_pair_reduce<<<int(std::min<uint32_t>(nt, g->sm_count * 8)), 256, 0, s>>>(dt, nt, dg, score, part);
        SABA_CUDA_CHECK(cudaGetLastError());
        *launches += 2;
        // the chunk's host metadata must outlive its uploads
        SABA_CUDA_CHECK(cudaStreamSynchronize(s));
        if (walk_kernel_ms) {
            float ms = 0.f;
            SABA_CUDA_CHECK(cudaEventElapsedTime(&ms, st->ev_walk[0], st->ev_walk[1]));
            *walk_kernel_ms += ms;
        }
    }
    const uint32_t nsw = uint32_t(tb.slots.size());
    auto* ds = static_cast<SlotWork*>(st->slots.ensure(sizeof(SlotWork) * nsw));
    SABA_CUDA_CHECK(cudaMemcpyAsync(ds, tb.slots.data(), sizeof(SlotWork) * nsw, cudaMemcpyHostToDevice, s));
    aesc_slot_reduce<<<(nsw + 127) / 128, 128, 0, s>>>(ds, nsw, part, g_hat_dev);
    SABA_CUDA_CHECK(cudaGetLastError());
    ++*launches;
    SABA_CUDA_CHECK(cudaStreamSynchronize(s));
}

// Power-iteration SpMV of the truncation plan (aesc.hpp:160-170) on the
// device, rounding exactly like the host loop: y[u] = (sum in slot order of
// x[a] * isd[a]) * isd[u], one multiply then one add per neighbour. The
// sequential reductions stay on the host, so lambda_hat is bit-identical.
// xs[a] = x[a] * isd[a], the rounded product every neighbour slot adds
__global__ void plan_scale_kernel(const double* __restrict__ x, const double* __restrict__ isd,
                                  double* __restrict__ xs, uint32_t n) {
    for (uint32_t a = blockIdx.x * blockDim.x + threadIdx.x; a < n; a += gridDim.x * blockDim.x)
        xs[a] = __dmul_rn(x[a], isd[a]);
}

// Warp per row: the lanes gather 32 neighbour products at a time (coalesced
// adjacency, independent loads) and every lane then adds them one by one in
// slot order, so the float64 sum is exactly the host loop's left fold while
// no thread serialises a dependent load per neighbour.
__global__ void plan_spmv_kernel(const uint2* __restrict__ csr, const uint32_t* __restrict__ adj,
                                 const double* __restrict__ xs, const double* __restrict__ isd,
                                 double* __restrict__ y, uint32_t n) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n; u += nwarps) {
        const uint2 r = csr[u];
        const uint32_t e = r.x + r.y;
        double acc = 0.0;
        for (uint32_t s0 = r.x; s0 < e; s0 += 32) {
            const uint32_t s = s0 + lane;
            const double prod = s < e ? xs[adj[s]] : 0.0;
            const uint32_t cnt = min(32u, e - s0);
            for (uint32_t j = 0; j < cnt; ++j) acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, prod, j));
        }
        if (lane == 0) y[u] = __dmul_rn(acc, isd[u]);
    }
}

struct DeviceSpmv {
    saba_cu_graph* g;
    DevBuf x, isd, y, xs;
    bool isd_up = false;
    SpmvFn fn() {
        return [this](const std::vector<double>& hx, const std::vector<double>& hisd, std::vector<double>& hy) {
            const uint32_t n = g->n;
            const size_t bytes = sizeof(double) * n;
            if (!isd_up) {
                copy_h2d(isd.ensure(bytes), hisd.data(), bytes, 0);
                isd_up = true;
            }
            copy_h2d(x.ensure(bytes), hx.data(), bytes, 0);
            const uint32_t grid = std::min<uint32_t>((n + 255) / 256, g->sm_count * 8);
            double* d_xs = static_cast<double*>(xs.ensure(bytes));
            plan_scale_kernel<<<grid, 256>>>(x.as<double>(), isd.as<double>(), d_xs, n);
            plan_spmv_kernel<<<g->sm_count * 16, 256>>>(g->d_csr, g->d_adj, d_xs, isd.as<double>(),
                                            static_cast<double*>(y.ensure(bytes)), n);
            SABA_CUDA_CHECK(cudaGetLastError());
            copy_d2h(hy.data(), y.p, bytes, 0);
        };
    }
};

}  // namespace

// The distinct sources of one shard. A repeated source is idempotent in the
// reference's per-source loop (each aesc_source call rewrites its own g_hat
// slots, aesc.hpp:572-577), but one batch column per occurrence would add its
// estimate twice, so the list is deduplicated first. Shards are cut
// cost-stratified: with a uniform tau the walk work of source v is
// sum_slots n_req * tau ~ tau^3 / d(v) (aesc.hpp:103-110, 478-496) and falls
// with degree, while tau~ grows as the degree falls (the ~85x spread of
// SURVEY §7); sources in ascending-degree order (ties by id) are dealt to the
// shards in snake order 0..N-1, N-1..0, so every shard gets the same degree
// profile. Each source runs on exactly one shard, so the sum over shards is
// exact and results are identical for any shard count.
std::vector<uint32_t> shard_sources(const uint32_t* off, uint32_t n, const uint32_t* sources, uint64_t count,
                                    uint32_t shard_index, uint32_t shard_count) {
    std::vector<uint32_t> all;
    if (sources) {
        all.assign(sources, sources + count);
        for (uint32_t v : all) check_arg(v < n, "source out of range");
        std::sort(all.begin(), all.end());
        all.erase(std::unique(all.begin(), all.end()), all.end());
    } else {
        all.resize(n);
        for (uint32_t v = 0; v < n; ++v) all[v] = v;
    }
    if (shard_count <= 1) return all;
    auto deg = [&](uint32_t v) { return off[v + 1] - off[v]; };
    std::stable_sort(all.begin(), all.end(), [&](uint32_t a, uint32_t b) { return deg(a) < deg(b); });
    std::vector<uint32_t> mine;
    mine.reserve(all.size() / shard_count + 1);
    for (uint64_t i = 0; i < all.size(); ++i) {
        const uint64_t r = i % (2ull * shard_count);
        const uint64_t shard = r < shard_count ? r : 2ull * shard_count - 1 - r;
        if (shard == shard_index) mine.push_back(all[i]);
    }
    return mine;
}

namespace {

AescParams make_params(const saba_cu_graph* g, double eps, double delta, int64_t cap) {
    AescParams p{};
    p.eps = eps;
    p.delta = delta;
    p.log_term = std::log(4.0 * double(g->m) / delta);  // aesc.hpp:109
    p.cap = cap;
    p.n = g->n;
    p.m = g->m;
    return p;
}

// K5 on `st`: s_hat[e] = g_hat[u->v] + g_hat[v->u] (aesc.hpp:702-706). The
// slot -> edge map is uploaded once per handle.
void enqueue_symmetrise(saba_cu_graph* g, const double* d_g, double* d_s, cudaStream_t st) {
    if (!g->aesc) g->aesc = new AescState[kWorkspaces];
    AescState& a = g->aesc[0];
    if (!a.slot_edge_ready) {
        const IdVec& se = slot_edges(g);
        uint32_t* d_se = static_cast<uint32_t*>(a.slot_edge_d.ensure(sizeof(uint32_t) * 2 * g->m, st));
        copy_h2d(d_se, se.data(), sizeof(uint32_t) * 2 * g->m, st);
        a.slot_edge_ready = true;
    }
    aesc_symmetrise<<<g->sm_count * 4, 256, 0, st>>>(g->d_csr, g->d_adj, a.slot_edge_d.as<uint32_t>(), g->n,
                                                     d_g, d_s);
    SABA_CUDA_CHECK(cudaGetLastError());
}

// One estimator call: the plan (once, on the first replica), then this
// shard's sources in batches of 64 over every replica of the handle (one
// multi-device handle = one shard per replica) and every batch worker of a
// replica, handed out dynamically (a shared batch counter: per-source cost
// varies ~85x), and finally one combine of the replicas' g_hat on
// the first replica. A column's arithmetic never depends on its batch, its
// worker or its replica, so the result is identical for any device count.
struct AescRun {
    Plan plan;
    std::vector<saba_cu_graph*> reps;
    std::vector<double*> d_g;       // per replica: its g_hat (2m), combined into d_g[0]
    std::vector<uint32_t> tt_all;   // tau~ per vertex (0 outside this call's sources)
    uint64_t pairs = 0, steps = 0, edge_visits = 0, nsources = 0;
    float prop_ms = 0.f, walk_ms = 0.f;
    double walk_kernel_ms = 0.0;
    double setup_seconds = 0.0;  // plan end -> first batch (per-call, not per-source, work)
    int workers = 1;
    uint32_t launches = 0;
    double seconds = 0.0, plan_seconds = 0.0;
    cudaStream_t root_stream = nullptr;
    const char* combine = "none";
};

void fill_aesc_report(const AescRun& run, saba_cu_aesc_report* rep) {
    saba_cu_aesc_report r{};
    r.seconds = run.seconds;
    r.plan_seconds = run.plan_seconds;
    r.propagation_ms = run.prop_ms;
    r.walk_ms = run.walk_ms;
    r.total_walk_pairs = run.pairs;
    r.total_walk_steps = run.steps;
    r.edge_visits = run.edge_visits;
    r.sources = run.nsources;
    r.lambda_hat = run.plan.lambda_hat;
    r.bipartite = run.plan.bipartite;
    r.clamped = run.plan.clamped;
    r.max_tau = run.plan.max_tau;
    r.launches = run.launches;
    r.replicas = uint32_t(run.reps.size());
    r.workers = uint32_t(run.workers);
    r.walk_kernel_ms = run.walk_kernel_ms;
    r.setup_seconds = run.setup_seconds;
    *rep = r;
}

void aesc_run(saba_cu_graph* g, const saba_cu_aesc_config& cfg, const uint32_t* sources, uint64_t source_count,
              uint32_t shard_index, uint32_t shard_count, bool need_slot_edges, AescRun& out) {
    const bool trace = getenv("SABA_TRACE") != nullptr;
    auto T = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
        if (!trace) return;
        const auto T1 = std::chrono::steady_clock::now();
        fprintf(stderr, "[saba] aesc %-26s %9.2f ms\n", what, std::chrono::duration<double, std::milli>(T1 - T).count());
        T = T1;
    };
    const auto t_plan0 = std::chrono::steady_clock::now();
    const auto& hadj = host_adj(g);
    lap("host adjacency");
    const HostCsr h{g->n, g->m, g->h_off.data(), hadj.data()};
    check_data(host_is_connected(h), "aesc: spanning centrality requires a connected graph");
    lap("connectivity");
    // slot -> edge ids: only per-edge plans and the s_hat symmetrisation need them
    const uint32_t* se = cfg.per_edge_tau || need_slot_edges ? slot_edges(g).data() : nullptr;
    lap("slot edges");
    // aesc.hpp:649: the plan is built for epsilon / 2
    DeviceSpmv dev{g};
    const SpmvFn spmv = dev.fn();
    out.plan = host_truncated_lengths(h, se, cfg.epsilon / 2.0, cfg.power_iterations, cfg.max_truncation,
                                      cfg.per_edge_tau != 0, &spmv);
    const Plan& plan = out.plan;
    const auto t_plan1 = std::chrono::steady_clock::now();
    out.plan_seconds = std::chrono::duration<double>(t_plan1 - t_plan0).count();
    lap("truncation plan");
    const uint32_t n = g->n;
    const uint64_t m = g->m;
    std::vector<uint32_t> list = shard_sources(g->h_off.data(), n, sources, source_count, shard_index, shard_count);
    out.nsources = list.size();
    // batches by descending degree (tau~ correlates with degree; batching
    // never changes a column's arithmetic)
    std::stable_sort(list.begin(), list.end(), [&](uint32_t a, uint32_t b) {
        return g->h_off[a + 1] - g->h_off[a] > g->h_off[b + 1] - g->h_off[b];
    });
    // tau per directed slot: a constant for a uniform plan (the default)
    std::vector<uint32_t> ts_v;
    SlotTau ts{nullptr, plan.tau.empty() ? 0u : plan.tau[0]};
    if (!plan.uniform) {
        ts_v.resize(2 * m);
#pragma omp parallel for schedule(static)
        for (int64_t sl = 0; sl < int64_t(2 * m); ++sl) ts_v[sl] = plan.tau[se[sl]];
        ts.v = ts_v.data();
    }
    lap("tau per slot");
    out.reps = replicas_of(g);
    const uint32_t R = uint32_t(out.reps.size());
    static const int workers_env = [] {  // SABA_AESC_WORKERS=1|2 overrides
        const char* e = getenv("SABA_AESC_WORKERS");
        return e ? std::max(1, std::min(kWorkspaces, atoi(e))) : 0;
    }();
    const size_t nbatches = (list.size() + kCols - 1) / kCols;
    // (measured: 3 workers gain nothing on cfg3/cfg4; 2 beat 1 on cfg3 and,
    // since the walk phase got cheaper, on the shallow cfg5 plan too: -11%)
    const int nworkers = cfg.workers > 0 ? std::min(cfg.workers, kWorkspaces)
                         : workers_env ? workers_env : (nbatches > R ? kWorkspaces : 1);
    out.workers = nworkers;
    std::vector<std::unique_ptr<Engine>> engines;  // replica-major: engines[r * nworkers + w]
    std::vector<std::unique_lock<std::recursive_mutex>> locks;
    out.d_g.assign(R, nullptr);
    for (uint32_t r = 0; r < R; ++r) {
        saba_cu_graph* rg = out.reps[r];
        if (r) locks.emplace_back(rg->mu);  // replica 0 is g (held by the caller)
        DeviceScope scope(rg->device);
        if (fat_fits_l2(rg) && aesc_fat_enabled()) {
            ensure_fat(rg);  // before the workers start
            if (aesc_hub_count() && plan.max_tau >= kShortWalk) ensure_fat_hub(rg, aesc_hub_count());
        }
        else if (plan.max_tau < kShortWalk && aesc_fat16_enabled())
            ensure_fat16(rg);
        for (int w = 0; w < nworkers; ++w) {
            engines.emplace_back(new Engine(rg, w));
            Engine& E = *engines.back();
            E.p = make_params(rg, cfg.epsilon, cfg.delta, cfg.switch_depth_cap);
            E.p.bip_init = plan.bipartite ? 1.0 / (2.0 * double(m)) : 0.0;  // aesc.hpp:657
            E.p.uniform_tau = plan.uniform ? 1 : 0;
            E.p.tau_uniform = plan.tau.empty() ? 0 : plan.tau[0];
            E.upload_tau(ts);
        }
        Engine& E0 = *engines[size_t(r) * nworkers];
        double* d_g = static_cast<double*>(E0.st->g_hat.ensure(sizeof(double) * 2 * m, E0.s));
        SABA_CUDA_CHECK(cudaMemsetAsync(d_g, 0, sizeof(double) * 2 * m, E0.s));
        out.d_g[r] = d_g;
        for (int w = 0; w < nworkers; ++w) SABA_CUDA_CHECK(cudaStreamSynchronize(engines[size_t(r) * nworkers + w]->s));
    }
    out.root_stream = engines[0]->s;
    lap("workers ready");
    out.tt_all.assign(n, 0);
    const size_t nthreads = engines.size();
    std::vector<float> prop_ms(nthreads, 0.f), walk_ms(nthreads, 0.f), walk_kms(nthreads, 0.f);
    std::vector<std::exception_ptr> failure(nthreads);
    std::atomic<size_t> next_batch{0};
    const auto t0 = std::chrono::steady_clock::now();
    out.setup_seconds = std::chrono::duration<double>(t0 - t_plan1).count();
    auto worker = [&](size_t wi) {
        try {
            Engine& W = *engines[wi];
            saba_cu_graph* rg = W.g;
            double* d_g = out.d_g[wi / nworkers];
            SABA_CUDA_CHECK(cudaSetDevice(rg->device));
            cudaEvent_t e0, e1, e2;
            SABA_CUDA_CHECK(cudaEventCreate(&e0));
            SABA_CUDA_CHECK(cudaEventCreate(&e1));
            SABA_CUDA_CHECK(cudaEventCreate(&e2));
            TileBuilder tb;
            for (size_t bi = next_batch++; bi < nbatches; bi = next_batch++) {
                const size_t b0 = bi * kCols;
                const std::vector<uint32_t> cols(list.begin() + b0, list.begin() + std::min(list.size(), b0 + kCols));
                const auto h0 = std::chrono::steady_clock::now();
                SABA_CUDA_CHECK(cudaEventRecord(e0, W.s));
                const std::vector<uint32_t> tt = W.propagate(cols, d_g);
                SABA_CUDA_CHECK(cudaEventRecord(e1, W.s));
                const auto h1 = std::chrono::steady_clock::now();
                tb.clear();
                for (size_t c = 0; c < cols.size(); ++c) {
                    const uint32_t src = cols[c];
                    out.tt_all[src] = tt[c];  // distinct sources: one writer per entry
                    const uint32_t lo = g->h_off[src], hi = g->h_off[src + 1], deg_i = hi - lo;
                    bool any = false;  // aesc.hpp:592-594
                    for (uint32_t sl = lo; sl < hi && !any; ++sl) any = ts[sl] > tt[c];
                    if (!any) continue;
                    const uint64_t src_seed = substream(substream(cfg.master_seed, kAescTag), src);
                    for (uint32_t sl = lo; sl < hi; ++sl) {
                        const int64_t tau_eff = int64_t(ts[sl]) - int64_t(tt[c]);
                        if (tau_eff <= 0) continue;
                        const uint64_t n_req = walk_budget(uint32_t(tau_eff), cfg.epsilon, cfg.delta, deg_i, m);
                        check_arg(cfg.switch_depth_cap < 0 || n_req * uint64_t(tau_eff) <= (uint64_t(1) << 26),
                                  "aesc: walk budget infeasible (switch_depth_cap too aggressive for epsilon)");
                        tb.add(sl, src, hadj[sl], uint32_t(tau_eff + 1), n_req, substream(src_seed, sl), uint32_t(c));
                        W.pairs += n_req;
                        W.steps += 2 * n_req * uint64_t(tau_eff);
                    }
                }
                // sparse supports: skip rho gathers of exact zeros via the bitmap
                static const int bitmap_mode = [] {  // 0 off, 1 on, 2 auto
                    const char* e = getenv("SABA_AESC_BITMAP");
                    return e ? atoi(e) : 2;
                }();
                // auto: supports of a few propagation steps are small even
                // when the batch's union frontier went dense
                const uint32_t tt_max = *std::max_element(tt.begin(), tt.end());
                const bool use_bits = bitmap_mode == 1 || (bitmap_mode == 2 && tt_max <= 4);
                const auto h2 = std::chrono::steady_clock::now();
                // the propagation above ended with a host sync, and run_tiles
                // returns after its own, so the two streams never overlap
                // within one worker
                const bool fat_path = rg->d_adj_fat != nullptr && fat_fits_l2(rg) && aesc_fat_enabled();
                const bool f16_path = !fat_path && rg->d_adj_fat16 != nullptr && aesc_fat16_enabled();
                const int rec_mode = aesc_rec_mode();
                const bool use_rec = !tb.empty() && (rec_mode == 2 || (rec_mode == 1 && !fat_path && !f16_path));
                const uint4* recs = nullptr;
                if (use_rec) {
                    cudaStream_t ws = W.st->stream_walk;
                    uint4* rb = static_cast<uint4*>(W.st->recs.ensure(sizeof(uint4) * size_t(n) * cols.size(), ws));
                    const uint64_t total = uint64_t(n) * cols.size();
                    const int grid = int(std::min<uint64_t>((total + 255) / 256, uint64_t(rg->sm_count) * 16));
                    aesc_build_records<<<grid, 256, 0, ws>>>(rg->d_csr, W.st->R.as<double>(), n,
                                                             uint32_t(cols.size()), rb);
                    SABA_CUDA_CHECK(cudaGetLastError());
                    ++W.launches;
                    recs = rb;
                }
                run_tiles(rg, W.st, W.st->stream_walk, tb, W.st->R.as<double>(),
                          use_bits && !use_rec ? W.st->bits.as<uint32_t>() : nullptr, cfg.hash_multiplier, d_g,
                          &W.launches, recs, &walk_kms[wi]);
                SABA_CUDA_CHECK(cudaEventRecord(e2, W.s));
                const auto h3 = std::chrono::steady_clock::now();
                W.clear_batch(int(cols.size()));
                SABA_CUDA_CHECK(cudaEventSynchronize(e2));
                float ta = 0.f, tw = 0.f;
                SABA_CUDA_CHECK(cudaEventElapsedTime(&ta, e0, e1));
                SABA_CUDA_CHECK(cudaEventElapsedTime(&tw, e1, e2));
                prop_ms[wi] += ta;
                walk_ms[wi] += tw;
                if (trace) {
                    const auto h4 = std::chrono::steady_clock::now();
                    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
                    fprintf(stderr, "[saba] aesc r%d w%zu batch %zu: propagate %.2f ms (device %.2f), tiles %.2f, "
                            "run_tiles %.2f (device walk %.2f), clear+sync %.2f\n", rg->device, wi, bi, ms(h0, h1), ta,
                            ms(h1, h2), ms(h2, h3), tw, ms(h3, h4));
                }
            }
            SABA_CUDA_CHECK(cudaStreamSynchronize(W.s));
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
            cudaEventDestroy(e2);
        } catch (...) {
            failure[wi] = std::current_exception();
            next_batch = nbatches;  // stop the other workers early
        }
    };
    std::vector<std::thread> threads;
    for (size_t w = 1; w < nthreads; ++w) threads.emplace_back(worker, w);
    worker(0);
    for (auto& t : threads) t.join();
    SABA_CUDA_CHECK(cudaSetDevice(g->device));
    for (auto& f : failure)
        if (f) std::rethrow_exception(f);
    lap("batches");
    for (size_t w = 0; w < nthreads; ++w) {
        Engine& E = *engines[w];
        DeviceScope scope(E.g->device);
        out.pairs += E.pairs;
        out.steps += E.steps;
        out.launches += E.launches;
        out.edge_visits += E.read_ctrl(kEdgeVisits);
        out.prop_ms += prop_ms[w];
        out.walk_ms += walk_ms[w];
        out.walk_kernel_ms += walk_kms[w];
    }
    // one combine of the replicas' g_hat (single writer per slot: exact)
    std::vector<void*> ptrs(out.d_g.begin(), out.d_g.end());
    std::vector<cudaStream_t> streams;
    for (uint32_t r = 0; r < R; ++r) streams.push_back(engines[size_t(r) * nworkers]->s);
    reduce_to_root(out.reps, ptrs, 2 * m, ReduceType::F64, streams);
    out.combine = last_combine_kind();
    lap("combine");
    out.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace
}  // namespace saba_cu

using namespace saba_cu;

extern "C" {

int saba_cu_truncated_lengths(saba_cu_graph* g, double epsilon, uint32_t power_iterations,
                              uint32_t max_truncation, int per_edge, uint32_t* tau_out,
                              double* lambda_hat, int* clamped) {
    return guard([&] {
        check_arg(g && tau_out && lambda_hat && clamped, "null argument");
        std::lock_guard<std::recursive_mutex> lock(g->mu);
        DeviceScope scope(g->device);
        const HostCsr h{g->n, g->m, g->h_off.data(), host_adj(g).data()};
        DeviceSpmv dev{g};
        const SpmvFn spmv = dev.fn();
        const Plan p = host_truncated_lengths(h, per_edge ? slot_edges(g).data() : nullptr, epsilon, power_iterations,
                                              max_truncation, per_edge != 0, &spmv);
        std::copy(p.tau.begin(), p.tau.end(), tau_out);
        *lambda_hat = p.lambda_hat;
        *clamped = p.clamped ? 1 : 0;
    });
}

int saba_cu_aesc(saba_cu_graph* g, const saba_cu_aesc_config* cfg, const uint32_t* sources,
                 uint64_t source_count, uint32_t shard_index, uint32_t shard_count,
                 double* g_hat_out, double* s_hat_out, uint32_t* tau_out, uint32_t* tau_tilde_out,
                 saba_cu_aesc_report* rep) {
    return guard([&] {
        check_arg(g && cfg && g_hat_out && tau_out && tau_tilde_out, "null argument");
        validate_cfg(*cfg);
        check_arg(shard_count >= 1 && shard_index < shard_count, "bad shard index/count");
        std::lock_guard<std::recursive_mutex> lock(g->mu);
        DeviceScope scope(g->device);
        const bool full = sources == nullptr && shard_count == 1;
        AescRun run;
        aesc_run(g, *cfg, sources, source_count, shard_index, shard_count, full && s_hat_out, run);
        saba_cu_graph* root = run.reps[0];
        cudaStream_t s = run.root_stream;
        const uint64_t m = g->m;
        const auto t_out0 = std::chrono::steady_clock::now();
        if (full && s_hat_out) {
            double* d_s = static_cast<double*>(root->aesc[0].s_hat.ensure(sizeof(double) * m, s));
            enqueue_symmetrise(root, run.d_g[0], d_s, s);
            ++run.launches;
            copy_d2h(s_hat_out, d_s, sizeof(double) * m, s);
        }
        copy_d2h(g_hat_out, run.d_g[0], sizeof(double) * 2 * m, s);
        run.seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - t_out0).count();
        std::copy(run.plan.tau.begin(), run.plan.tau.end(), tau_out);
        std::copy(run.tt_all.begin(), run.tt_all.end(), tau_tilde_out);
        if (rep) fill_aesc_report(run, rep);
    });
}

int saba_cu_aesc_device(saba_cu_graph* g, const saba_cu_aesc_config* cfg, const uint32_t* sources,
                        uint64_t source_count, uint32_t shard_index, uint32_t shard_count, double* g_hat_dev,
                        uint32_t* tau_out, uint32_t* tau_tilde_out, void* stream, saba_cu_aesc_report* rep) {
    return guard([&] {
        check_arg(g && cfg && g_hat_dev, "null argument");
        validate_cfg(*cfg);
        check_arg(shard_count >= 1 && shard_index < shard_count, "bad shard index/count");
        std::lock_guard<std::recursive_mutex> lock(g->mu);
        DeviceScope scope(g->device);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        AescRun run;
        aesc_run(g, *cfg, sources, source_count, shard_index, shard_count, false, run);
        // the result is complete (aesc_run synchronised); the copy is ordered
        // on the caller's stream like every later use of g_hat_dev
        SABA_CUDA_CHECK(cudaMemcpyAsync(g_hat_dev, run.d_g[0], sizeof(double) * 2 * g->m,
                                        cudaMemcpyDeviceToDevice, st));
        SABA_CUDA_CHECK(cudaStreamSynchronize(st));  // run's workspace may be reused by the next call
        if (tau_out) std::copy(run.plan.tau.begin(), run.plan.tau.end(), tau_out);
        if (tau_tilde_out) std::copy(run.tt_all.begin(), run.tt_all.end(), tau_tilde_out);
        if (rep) fill_aesc_report(run, rep);
    });
}

int saba_cu_symmetrise(saba_cu_graph* g, const double* g_hat_dev, double* s_hat_dev, void* stream) {
    return guard([&] {
        check_arg(g && g_hat_dev && s_hat_dev, "null argument");
        std::lock_guard<std::recursive_mutex> lock(g->mu);
        DeviceScope scope(g->device);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        g->enter(st);
        enqueue_symmetrise(g, g_hat_dev, s_hat_dev, st);
        g->leave(st);
    });
}

int saba_aesc_shard_sources(const uint32_t* offsets, uint32_t n, const uint32_t* sources,
                            uint64_t source_count, uint32_t shard_index, uint32_t shard_count, uint32_t* out,
                            uint64_t* out_count) {
    return guard([&] {
        check_arg(offsets && out_count, "null argument");
        check_arg(source_count == 0 || sources, "null sources");
        check_arg(shard_count >= 1 && shard_index < shard_count, "bad shard index/count");
        const std::vector<uint32_t> mine =
            shard_sources(offsets, n, sources, sources ? source_count : 0, shard_index, shard_count);
        if (out) std::copy(mine.begin(), mine.end(), out);
        *out_count = mine.size();
    });
}

int saba_cu_propagate(saba_cu_graph* g, uint32_t source, const uint32_t* tau, double epsilon,
                      double delta, int64_t cap, double* prob_out, uint32_t* depth_out) {
    return guard([&] {
        check_arg(g && tau && prob_out && depth_out, "null argument");
        check_arg(source < g->n, "LandingPropagator: source out of range");
        std::lock_guard<std::recursive_mutex> lock(g->mu);
        DeviceScope scope(g->device);
        const HostCsr h{g->n, g->m, g->h_off.data(), host_adj(g).data()};
        check_data(host_is_connected(h), "propagate_landing_probabilities: graph must be connected");
        const auto& se = slot_edges(g);
        Engine E(g);
        E.p = make_params(g, epsilon, delta, cap);
        E.p.uniform_tau = 0;  // caller-supplied tau: exact budget loop
        std::vector<uint32_t> ts_v(2 * g->m);
#pragma omp parallel for schedule(static)
        for (int64_t s = 0; s < int64_t(2 * g->m); ++s) ts_v[s] = tau[se[s]];
        E.upload_tau(SlotTau{ts_v.data(), 0});
        double* d_g = static_cast<double*>(E.st->g_hat.ensure(sizeof(double) * std::max<uint64_t>(2 * g->m, 1)));
        const std::vector<uint32_t> tt = E.propagate({source}, d_g);
        // column 0 of P at the switch depth: depth d always lives in P[d & 1]
        std::vector<double> rows(size_t(g->n) * kCols);
        SABA_CUDA_CHECK(cudaMemcpyAsync(rows.data(), E.st->P[tt[0] & 1].p, sizeof(double) * rows.size(),
                                        cudaMemcpyDeviceToHost, E.s));
        SABA_CUDA_CHECK(cudaStreamSynchronize(E.s));
        for (uint32_t v = 0; v < g->n; ++v) prob_out[v] = rows[size_t(v) * kCols];
        *depth_out = tt[0];
        E.clear_batch(1);
        SABA_CUDA_CHECK(cudaStreamSynchronize(E.s));
    });
}

int saba_cu_estimate_edge(saba_cu_graph* g, uint32_t v_i, uint32_t v_j, const double* prob,
                          uint32_t tau_eff, uint64_t n_req, int mode, uint64_t edge_seed,
                          uint32_t lanes, uint64_t mult, double* out) {
    return guard([&] {
        check_arg(tau_eff >= 1, "estimate_edge: tau_eff must be >= 1");  // aesc.hpp:537-538
        check_arg(n_req >= 1, "estimate_edge: n_req must be >= 1");
        check_arg(g && prob && out, "null argument");
        check_arg(v_i < g->n && v_j < g->n, "vertex out of range");
        check_arg(g->h_off[v_i + 1] > g->h_off[v_i] && g->h_off[v_j + 1] > g->h_off[v_j],
                  "cannot walk from an isolated vertex");
        check_arg(mode == SABA_MODE_HASH || mode == SABA_MODE_SABA, "mode not supported on GPU");
        check_arg(lanes >= 1 && lanes <= 64, "lanes must be in [1, 64]");
        std::lock_guard<std::recursive_mutex> lock(g->mu);
        DeviceScope scope(g->device);
        Engine E(g);
        // dense rho = p / degree (aesc.hpp:541-548 uses the division form here)
        std::vector<double> rho(g->n);
        for (uint32_t v = 0; v < g->n; ++v) rho[v] = prob[v] != 0.0 ? prob[v] / double(E.deg(v)) : 0.0;
        double* d_rho = static_cast<double*>(E.st->rho1.ensure(sizeof(double) * g->n));
        SABA_CUDA_CHECK(cudaMemcpyAsync(d_rho, rho.data(), sizeof(double) * g->n, cudaMemcpyHostToDevice, E.s));
        double* d_out = static_cast<double*>(E.st->s_hat.ensure(sizeof(double) * std::max<uint64_t>(g->m, 1)));
        SABA_CUDA_CHECK(cudaMemsetAsync(d_out, 0, sizeof(double), E.s));
        TileBuilder tb;
        tb.add(0, v_i, v_j, tau_eff + 1, n_req, edge_seed, 0);
        uint32_t launches = 0;
        run_tiles(g, E.st, E.s, tb, d_rho, nullptr, mult, d_out, &launches);
        SABA_CUDA_CHECK(cudaMemcpyAsync(out, d_out, sizeof(double), cudaMemcpyDeviceToHost, E.s));
        SABA_CUDA_CHECK(cudaStreamSynchronize(E.s));
    });
}

}  // extern "C"
