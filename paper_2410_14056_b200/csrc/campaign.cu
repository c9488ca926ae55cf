// Bouquets walk campaigns on sm_100a.
//
//   K1a start_hist_kernel       uniform-random starts: K_v histogram
//   K1b CUB scan                K_v -> walk-list offsets
//   K1c gen_sorted_keys_kernel  per-vertex walk seeds counter_hash(vseed,k)>>32
//                               (walker.hpp:437-438) as keys (v<<32 | seed),
//                               sorted within each start vertex by the warp
//                               that generates them (SABA, walker.hpp:439: a
//                               warp is a 32-lane bouquet), plus the step-0
//                               visit of every walk (walker.hpp:216-220);
//                               gen_keys_kernel + CUB segmented sort for large
//                               per-vertex campaigns
//   K2  L-1 lockstep hashed steps per lane (walker.hpp:221-235) + the
//       VisitCountSink epilogue (walker.hpp:355); launch_walk picks
//       walk_count_rank_kernel      default up to 2^21 vertices: degree-ranked
//                                   records, the top records and 16-bit visit
//                                   counters in shared memory, the rest as
//                                   warp-aggregated L2 reductions
//       walk_count_fat_priv_kernel  L2-resident graphs of <= 80K vertices: one
//                                   fat gather per step, every counter in
//                                   shared memory
//       walk_count_fat_kernel       other L2-resident graphs
//       walk_count_hot_kernel       beyond 2^21 vertices: 32-bit hub counters
//                                   in shared memory (one 1024-thread block
//                                   per SM), visits counted at departure
//       walk_count_kernel           generic fallback (and uint32 counters)
//
// A GPU bouquet is a warp: lanes hold consecutive entries of the sorted key
// array, so they share their start vertex and hold adjacent seeds — the
// reference's lane-batched bouquet (walker.hpp:207-236) at width 32. Each
// thread advances WPT independent bouquet lanes so that several dependent
// gather chains are in flight per thread (the walk is a pure random-gather
// workload: no tensor cores).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>
#include <cub/iterator/transform_input_iterator.cuh>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <exception>

#include "device_graph.cuh"
#include "saba_hash.cuh"
#include "walk_common.cuh"

namespace saba_cu {

namespace {

constexpr int kWalkThreads = 256;

__global__ void start_hist_kernel(uint64_t W, uint64_t start_stream, uint32_t n,
                                  uint32_t* __restrict__ kv) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t w = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; w < W; w += stride) {
        const uint32_t v = scaled_index(uint32_t(counter_hash(start_stream, w) >> 32), n);
        atomicAdd(kv + v, 1u);
    }
}

struct U32ToU64 {
    __host__ __device__ uint64_t operator()(uint32_t x) const { return x; }
};

// Warp per start vertex. The walk list of this call is [r0, r1) of the
// flattened (vertex, k) list; keys land at [0, r1 - r0).
__global__ void gen_keys_kernel(uint32_t n, const uint32_t* __restrict__ kv, uint64_t k_uniform,
                                const uint64_t* __restrict__ off, uint64_t r0, uint64_t r1,
                                uint64_t master, uint64_t* __restrict__ keys,
                                int* __restrict__ seg, unsigned long long* __restrict__ counts) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t v = warp; v < n; v += nwarps) {
        const uint64_t K = kv ? kv[v] : k_uniform;
        const uint64_t o = kv ? off[v] : uint64_t(v) * k_uniform;
        const uint64_t lo = o > r0 ? o : r0;
        const uint64_t hi = (o + K) < r1 ? (o + K) : r1;
        if (lane == 0) {
            const uint64_t b = lo < r1 ? lo : r1;
            seg[v] = int(b - r0);
            if (v == n - 1) seg[n] = int(r1 - r0);
            if (hi > lo) counts[v] += hi - lo;  // step-0 visits; this warp owns v
        }
        if (hi <= lo) continue;
        const uint64_t vseed = substream(master, v);
        for (uint64_t k = lo - o + lane; k < hi - o; k += 32)
            keys[o + k - r0] = (uint64_t(v) << 32) | walk_seed(vseed, k);
    }
}

// K1 fused (SABA mode): the same keys as gen_keys_kernel, sorted by seed
// within each start vertex's share of the range by the warp that generates
// them — a bitonic network over <= kSortCap seeds in the warp's slice of
// shared memory — so no separate segmented sort pass (and no second key
// buffer) is needed. A vertex holding more than kSortCap walks of the range
// is sorted in runs of kSortCap (walk order is a performance device only:
// counts are order-independent sums); the host picks this kernel when the
// expected K_v is far below the cap.
constexpr uint32_t kSortCap = 256;
__global__ void __launch_bounds__(256)
    gen_sorted_keys_kernel(uint32_t n, const uint32_t* __restrict__ kv, uint64_t k_uniform,
                           const uint64_t* __restrict__ off, uint64_t r0, uint64_t r1, uint64_t master,
                           uint64_t* __restrict__ keys, unsigned long long* __restrict__ counts) {
    __shared__ uint32_t buf[8][kSortCap];
    const uint32_t lane = threadIdx.x & 31;
    uint32_t* sb = buf[threadIdx.x >> 5];
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t v = warp; v < n; v += nwarps) {
        const uint64_t K = kv ? kv[v] : k_uniform;
        const uint64_t o = kv ? off[v] : uint64_t(v) * k_uniform;
        const uint64_t lo = o > r0 ? o : r0;
        const uint64_t hi = (o + K) < r1 ? (o + K) : r1;
        if (hi <= lo) continue;
        if (lane == 0) counts[v] += hi - lo;  // step-0 visits; this warp owns v
        const uint64_t vseed = substream(master, v);
        for (uint64_t c0 = lo; c0 < hi; c0 += kSortCap) {
            const uint32_t m = uint32_t(min(uint64_t(kSortCap), hi - c0));
            if (m <= 32) {  // one seed per lane: the bitonic network over shuffles
                uint32_t x = lane < m ? walk_seed(vseed, c0 - o + lane) : 0xffffffffu;
                for (uint32_t size = 2; size <= 32; size <<= 1)
                    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
                        const uint32_t y = __shfl_xor_sync(0xffffffffu, x, stride);
                        const bool keep_min = ((lane & stride) == 0) == ((lane & size) == 0);
                        x = keep_min ? min(x, y) : max(x, y);
                    }
                if (lane < m) keys[c0 - r0 + lane] = (uint64_t(v) << 32) | x;
                continue;
            }
            uint32_t P = 64;
            while (P < m) P <<= 1;
            for (uint32_t i = lane; i < P; i += 32)
                sb[i] = i < m ? walk_seed(vseed, c0 - o + i) : 0xffffffffu;  // padding sorts last
            __syncwarp();
            for (uint32_t size = 2; size <= P; size <<= 1)
                for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
                    for (uint32_t i = lane; i < P; i += 32) {
                        const uint32_t j = i ^ stride;
                        if (j > i) {
                            const uint32_t a = sb[i], b = sb[j];
                            if ((a > b) == ((i & size) == 0)) {
                                sb[i] = b;
                                sb[j] = a;
                            }
                        }
                    }
                    __syncwarp();
                }
            for (uint32_t i = lane; i < m; i += 32) keys[c0 - r0 + i] = (uint64_t(v) << 32) | sb[i];
            __syncwarp();
        }
    }
}

// CT = counter type: uint32 per-launch counters (half the L2 footprint of
// uint64) whenever a launch cannot overflow them, flushed into the uint64
// sink by add_counts_kernel. PACKED = 21-bit packed adjacency.
template <int WPT, bool PACKED, class CT, bool AGG>
__global__ void __launch_bounds__(kWalkThreads)
    walk_count_kernel(const uint2* __restrict__ csr, const uint32_t* __restrict__ adj,
                      const uint64_t* __restrict__ adjp, const uint64_t* __restrict__ keys,
                      uint64_t nwalks, uint32_t L, uint64_t mult, CT* __restrict__ counts) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t base = warp * 32 * WPT; base < nwalks; base += nwarps * 32 * WPT) {
        uint32_t cur[WPT], seed[WPT];
        bool act[WPT];
#pragma unroll
        for (int r = 0; r < WPT; ++r) {
            const uint64_t i = base + uint64_t(r) * 32 + lane;
            act[r] = i < nwalks;
            const uint64_t k = act[r] ? __ldcs(reinterpret_cast<const unsigned long long*>(keys) + i) : 0;
            cur[r] = uint32_t(k >> 32);
            seed[r] = uint32_t(k);
        }
        for (uint32_t l = 1; l < L; ++l) {
            const StepHash shs = step_hash(mult, l);
            uint2 rec[WPT];
#pragma unroll
            for (int r = 0; r < WPT; ++r) rec[r] = act[r] ? ldg_csr(csr + cur[r]) : make_uint2(0, 0);
            uint32_t nxt[WPT];
#pragma unroll
            for (int r = 0; r < WPT; ++r) {
                const uint32_t raw = seed[r] ^ hash_state_fast(shs, cur[r]);
                nxt[r] = act[r] ? adj_at<PACKED>(adj, adjp, rec[r].x + scaled_index(raw, rec[r].y)) : 0u;
            }
#pragma unroll
            for (int r = 0; r < WPT; ++r) {
                cur[r] = nxt[r];
                if constexpr (AGG)
                    warp_count_visit(counts, nxt[r], act[r], lane);
                else
                    count_visit(counts, nxt[r], act[r]);
            }
        }
    }
}

// K2 over the fat adjacency: the {base, degree} of the next vertex arrives
// with its id, so each step is ONE dependent gather + the visit reduction.
template <int WPT, bool AGG>
__global__ void __launch_bounds__(kWalkThreads)
    walk_count_fat_kernel(const uint2* __restrict__ csr, const uint64_t* __restrict__ fat,
                          uint32_t idb, uint32_t sh, const uint64_t* __restrict__ keys,
                          uint64_t nwalks, uint32_t L, uint64_t mult,
                          unsigned long long* __restrict__ counts) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    const uint64_t idmask = (uint64_t(1) << idb) - 1, bmask = (uint64_t(1) << (sh - idb)) - 1;
    for (uint64_t base = warp * 32 * WPT; base < nwalks; base += nwarps * 32 * WPT) {
        uint32_t cur[WPT], seed[WPT], sbase[WPT], deg[WPT];
        bool act[WPT];
#pragma unroll
        for (int r = 0; r < WPT; ++r) {
            const uint64_t i = base + uint64_t(r) * 32 + lane;
            act[r] = i < nwalks;
            const uint64_t k = act[r] ? __ldcs(reinterpret_cast<const unsigned long long*>(keys) + i) : 0;
            cur[r] = uint32_t(k >> 32);
            seed[r] = uint32_t(k);
            const uint2 rec = act[r] ? ldg_csr(csr + cur[r]) : make_uint2(0, 1);
            sbase[r] = rec.x;
            deg[r] = rec.y;
        }
        for (uint32_t l = 1; l < L; ++l) {
            const StepHash shs = step_hash(mult, l);
#pragma unroll
            for (int r = 0; r < WPT; ++r) {
                const uint32_t raw = seed[r] ^ hash_state_fast(shs, cur[r]);
                const uint64_t f = act[r] ? __ldg(reinterpret_cast<const unsigned long long*>(fat) +
                                                  sbase[r] + scaled_index(raw, deg[r]))
                                          : 0ull;
                cur[r] = uint32_t(f & idmask);
                sbase[r] = uint32_t((f >> idb) & bmask);
                deg[r] = uint32_t(f >> sh);
            }
#pragma unroll
            for (int r = 0; r < WPT; ++r) {
                if constexpr (AGG)
                    warp_count_visit(counts, cur[r], act[r], lane);
                else
                    count_visit(counts, cur[r], act[r]);
            }
        }
    }
}

// K2 over the fat adjacency with EVERY vertex's counter in shared memory
// (graphs of up to ~80K vertices: 16-bit fields, smem_count16): a step is one
// dependent gather and one shared-memory atomic, and no L2 reduction is left
// on the step path. One block per SM; the block passes a barrier every
// count16_steps() steps so that the 16-bit fields cannot carry (all warps of
// a block run the same number of rounds and steps).
template <int WPT, int THREADS>
__global__ void __launch_bounds__(THREADS)
    walk_count_fat_priv_kernel(const uint2* __restrict__ csr, const uint64_t* __restrict__ fat,
                               uint32_t idb, uint32_t sh, const uint64_t* __restrict__ keys,
                               uint64_t nwalks, uint32_t L, uint64_t mult, uint32_t n,
                               unsigned long long* __restrict__ counts) {
    extern __shared__ uint32_t cnt16[];
    const uint32_t words = (n + 1) / 2;
    for (uint32_t i = threadIdx.x; i < words; i += THREADS) cnt16[i] = 0;
    __syncthreads();
    constexpr uint32_t kSync = count16_steps(THREADS, WPT);
    static_assert(kSync >= 1, "block too large for 16-bit counters");
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (uint64_t(blockIdx.x) * THREADS + threadIdx.x) >> 5;
    const uint64_t nwarps = (uint64_t(gridDim.x) * THREADS) >> 5;
    const uint64_t per_round = nwarps * 32 * WPT;
    const uint64_t rounds = (nwalks + per_round - 1) / per_round;
    const uint64_t idmask = (uint64_t(1) << idb) - 1, bmask = (uint64_t(1) << (sh - idb)) - 1;
    for (uint64_t round = 0; round < rounds; ++round) {
        const uint64_t base = round * per_round + warp * 32 * WPT;
        uint32_t cur[WPT], seed[WPT], sbase[WPT], deg[WPT];
        bool act[WPT];
#pragma unroll
        for (int r = 0; r < WPT; ++r) {
            const uint64_t i = base + uint64_t(r) * 32 + lane;
            act[r] = i < nwalks;
            const uint64_t k = act[r] ? __ldcs(reinterpret_cast<const unsigned long long*>(keys) + i) : 0;
            cur[r] = uint32_t(k >> 32);
            seed[r] = uint32_t(k);
            const uint2 rec = act[r] ? ldg_csr(csr + cur[r]) : make_uint2(0, 1);
            sbase[r] = rec.x;
            deg[r] = rec.y;
        }
        for (uint32_t l = 1; l < L; ++l) {
            const StepHash shs = step_hash(mult, l);
#pragma unroll
            for (int r = 0; r < WPT; ++r) {
                const uint32_t raw = seed[r] ^ hash_state_fast(shs, cur[r]);
                const uint64_t f = act[r] ? __ldg(reinterpret_cast<const unsigned long long*>(fat) +
                                                  sbase[r] + scaled_index(raw, deg[r]))
                                          : 0ull;
                cur[r] = uint32_t(f & idmask);
                sbase[r] = uint32_t((f >> idb) & bmask);
                deg[r] = uint32_t(f >> sh);
            }
#pragma unroll
            for (int r = 0; r < WPT; ++r) {
                SABA_DCHECK(!act[r] || cur[r] < n);
                if (act[r]) smem_count16(cnt16, cur[r], counts, cur[r]);
            }
#ifndef SABA_COUNT16_NOSYNC  // measurement builds only: without the barrier the 16-bit fields may carry
            if (l % kSync == 0) __syncthreads();
#endif
        }
        __syncthreads();
    }
    for (uint32_t i = threadIdx.x; i < words; i += THREADS) {
        const uint32_t w = cnt16[i];
        if (w & 0xFFFFu) atomicAdd(counts + 2 * i, (unsigned long long)(w & 0xFFFFu));
        if (w >> 16) atomicAdd(counts + 2 * i + 1, (unsigned long long)(w >> 16));
    }
}

// K2 with hub-privatised counters. Visits are counted at DEPARTURE: the
// record of x_{l-1} loaded at step l already says whether x_{l-1} is one of
// the highest-degree vertices (field y >> shift), whose counters live in
// shared memory for the whole launch; every other visit is an L2 reduction.
// Large blocks (1024 threads) share one big table: at the register-limited
// occupancy a block per SM holds up to ~56K hub counters instead of 3 x 16K.
// x_0 is counted by gen_keys_kernel and x_{L-1} after the loop, so the
// multiset of counted vertices equals the reference's (walker.hpp:216-232).
template <int WPT, bool PACKED, bool AGG, int THREADS>
__global__ void __launch_bounds__(THREADS)
    walk_count_hot_kernel(const uint2* __restrict__ csr_hot, const uint32_t* __restrict__ adj,
                          const uint64_t* __restrict__ adjp, const uint32_t* __restrict__ hot_vertex,
                          uint32_t nhot, uint32_t shift, const uint64_t* __restrict__ keys,
                          uint64_t nwalks, uint32_t L, uint64_t mult,
                          unsigned long long* __restrict__ counts) {
    extern __shared__ uint32_t hot_cnt[];
    for (uint32_t i = threadIdx.x; i < nhot; i += blockDim.x) hot_cnt[i] = 0;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t base = warp * 32 * WPT; base < nwalks; base += nwarps * 32 * WPT) {
        uint32_t cur[WPT], seed[WPT];
        bool act[WPT];
#pragma unroll
        for (int r = 0; r < WPT; ++r) {
            const uint64_t i = base + uint64_t(r) * 32 + lane;
            act[r] = i < nwalks;
            const uint64_t k = act[r] ? __ldcs(reinterpret_cast<const unsigned long long*>(keys) + i) : 0;
            cur[r] = uint32_t(k >> 32);
            seed[r] = uint32_t(k);
        }
        for (uint32_t l = 1; l < L; ++l) {
            const StepHash shs = step_hash(mult, l);
            uint2 rec[WPT];
#pragma unroll
            for (int r = 0; r < WPT; ++r) rec[r] = act[r] ? ldg_csr(csr_hot + cur[r]) : make_uint2(0, 0);
            // the neighbour gathers of all WPT walks are issued before any
            // of them is consumed; the visit of the departing vertex is
            // counted while they are in flight
            AdjWord<PACKED> nxt[WPT];
#pragma unroll
            for (int r = 0; r < WPT; ++r) {
                const uint32_t deg = rec[r].y & ((1u << shift) - 1);
                const uint32_t raw = seed[r] ^ hash_state_fast(shs, cur[r]);
                nxt[r] = adj_load<PACKED>(adj, adjp, act[r] ? rec[r].x + scaled_index(raw, deg) : 0u);
            }
            if (l >= 2) {  // count the departing vertex x_{l-1}
#pragma unroll
                for (int r = 0; r < WPT; ++r) {
                    const uint32_t slot = rec[r].y >> shift;
                    const bool hot = act[r] && slot != 0;
                    SABA_DCHECK(!hot || slot - 1 < nhot);
                    if (hot) atomicAdd(hot_cnt + (slot - 1), 1u);
                    if constexpr (AGG)
                        warp_count_visit(counts, cur[r], act[r] && !hot, lane);
                    else
                        count_visit(counts, cur[r], act[r] && !hot);
                }
            }
#pragma unroll
            for (int r = 0; r < WPT; ++r) cur[r] = act[r] ? adj_id<PACKED>(nxt[r]) : 0u;
        }
#pragma unroll
        for (int r = 0; r < WPT; ++r) {  // the last vertex x_{L-1}
            if constexpr (AGG)
                warp_count_visit(counts, cur[r], act[r] && L > 1, lane);
            else
                count_visit(counts, cur[r], act[r] && L > 1);
        }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < nhot; i += blockDim.x)
        if (hot_cnt[i]) atomicAdd(counts + hot_vertex[i], (unsigned long long)hot_cnt[i]);
}

// K2 over degree-ranked records (see saba_cu_graph::d_rec). A walk carries
// the RANK r of its vertex (descending degree): rec[r] = {id, base, degree} in
// one uint64 and the neighbour slots hold ranks. A walk sits on v with
// probability ~ deg(v) / 2m, so what the step path needs of the most visited
// vertices is kept in shared memory for the whole launch:
//   r < nrec: the record itself (no L2 request for the {base, degree} gather)
//   r < ncnt: the visit counter, a 16-bit field (smem_count16; no L2 reduction)
// K2 is bound by the SM's L1-miss request rate (~1 request per clock: one
// each for the record, the neighbour slot and the visit reduction of a step),
// so every request kept in shared memory is throughput. Walks, selections and
// the counted multiset are exactly those of walk_count_hot_kernel: visits are
// counted at departure, x_0 by the key generator, x_{L-1} after the loop.
// One block per SM; all warps run the same rounds and steps and pass a
// barrier every count16_steps() steps (see smem_count16).
template <int WPT, int THREADS, class CT>
__global__ void __launch_bounds__(THREADS)
    walk_count_rank_kernel(const uint64_t* __restrict__ rec, const uint32_t* __restrict__ rank,
                           const uint64_t* __restrict__ adj_rank, uint32_t nb, uint32_t db, uint32_t nrec,
                           uint32_t ncnt, const uint64_t* __restrict__ keys, uint64_t nwalks, uint32_t L,
                           uint64_t mult, CT* __restrict__ counts) {
    extern __shared__ uint64_t rank_smem[];
    uint64_t* rec_s = rank_smem;
    uint32_t* cnt16 = reinterpret_cast<uint32_t*>(rank_smem + nrec);
    const uint32_t cwords = (ncnt + 1) / 2;
    for (uint32_t i = threadIdx.x; i < nrec; i += THREADS) rec_s[i] = rec[i];
    for (uint32_t i = threadIdx.x; i < cwords; i += THREADS) cnt16[i] = 0;
    __syncthreads();
    constexpr uint32_t kSync = count16_steps(THREADS, WPT);
    static_assert(kSync >= 1, "block too large for 16-bit counters");
    const uint64_t idmask = (uint64_t(1) << nb) - 1, bmask = (uint64_t(1) << (db - nb)) - 1;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (uint64_t(blockIdx.x) * THREADS + threadIdx.x) >> 5;
    const uint64_t nwarps = (uint64_t(gridDim.x) * THREADS) >> 5;
    const uint64_t per_round = nwarps * 32 * WPT;
    const uint64_t rounds = (nwalks + per_round - 1) / per_round;
    auto record = [&](uint32_t r) {
        return r < nrec ? rec_s[r] : __ldg(reinterpret_cast<const unsigned long long*>(rec) + r);
    };
    for (uint64_t round = 0; round < rounds; ++round) {
        const uint64_t base = round * per_round + warp * 32 * WPT;
        uint32_t cur[WPT], seed[WPT];  // cur = rank of the walk's vertex
        bool act[WPT];
#pragma unroll
        for (int r = 0; r < WPT; ++r) {
            const uint64_t i = base + uint64_t(r) * 32 + lane;
            act[r] = i < nwalks;
            const uint64_t k = act[r] ? __ldcs(reinterpret_cast<const unsigned long long*>(keys) + i) : 0;
            cur[r] = act[r] ? __ldg(rank + uint32_t(k >> 32)) : 0u;
            seed[r] = uint32_t(k);
        }
        for (uint32_t l = 1; l < L; ++l) {
            const StepHash shs = step_hash(mult, l);
            uint64_t q[WPT];
#pragma unroll
            for (int r = 0; r < WPT; ++r) q[r] = act[r] ? record(cur[r]) : 0ull;
            AdjWord<true> nxt[WPT];
#pragma unroll
            for (int r = 0; r < WPT; ++r) {
                const uint32_t id = uint32_t(q[r] & idmask);
                const uint32_t sbase = uint32_t((q[r] >> nb) & bmask);
                const uint32_t deg = uint32_t(q[r] >> db);
                SABA_DCHECK(!act[r] || deg > 0);
                const uint32_t raw = seed[r] ^ hash_state_fast(shs, id);
                nxt[r] = adj_load<true>(nullptr, adj_rank, act[r] ? sbase + scaled_index(raw, deg) : 0u);
            }
            if (l >= 2) {  // count the departing vertex x_{l-1} while the gathers are in flight
#pragma unroll
                for (int r = 0; r < WPT; ++r) {
                    const uint32_t id = uint32_t(q[r] & idmask);
                    const bool hot = act[r] && cur[r] < ncnt;
                    if (hot) smem_count16(cnt16, cur[r], counts, id);
                    warp_count_visit(counts, id, act[r] && !hot, lane);
                }
            }
#pragma unroll
            for (int r = 0; r < WPT; ++r) cur[r] = act[r] ? adj_id<true>(nxt[r]) : 0u;
#ifndef SABA_COUNT16_NOSYNC  // measurement builds only: without the barrier the 16-bit fields may carry
            if (l % kSync == 0) __syncthreads();
#endif
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < WPT; ++r) {  // the last vertex x_{L-1}
            const bool last = act[r] && L > 1;
            const uint32_t id = last ? uint32_t(record(cur[r]) & idmask) : 0u;
            const bool hot = last && cur[r] < ncnt;
            if (hot) smem_count16(cnt16, cur[r], counts, id);
            warp_count_visit(counts, id, last && !hot, lane);
        }
        __syncthreads();
    }
    for (uint32_t i = threadIdx.x; i < cwords; i += THREADS) {
        const uint32_t w = cnt16[i];
        if (w & 0xFFFFu) atomicAdd(counts + uint32_t(rec[2 * i] & idmask), CT(w & 0xFFFFu));
        if (w >> 16) atomicAdd(counts + uint32_t(rec[2 * i + 1] & idmask), CT(w >> 16));
    }
}

// Kernel variant (tuning knob; SABA_WALK_VARIANT="wpt=4,packed=1,c32=1,agg=1").
struct WalkVariant {
    int wpt = 4;
    bool packed = true;
    bool c32 = false;
    bool agg = true;
    int blocks_per_sm = 0;  // 0 = occupancy maximum
    int fat = -1;           // one-gather steps over the fat adjacency: 1 on, 0 off, -1 auto
    int hot = -1;           // hub counters in shared memory: 1 on, 0 off, -1 auto
    int hot_threads = 1024; // block size of the hub-counter kernel (256, 512, 1024)
    int hot_count = 0;      // hub table entries (0 = as many as shared memory holds)
    int sort = -1;          // K1 SABA sort: 1 fused warp sort, 0 CUB segmented sort, -1 auto
    int rec = -1;           // degree-ranked records (walk_count_rank_kernel): 1 on, 0 off, -1 auto
    int hrec = -1;          // rank kernel: records kept in shared memory (-1 = auto)
    int hcnt = -1;          // rank kernel: 16-bit counters kept in shared memory (-1 = auto)
    int priv = -1;          // fat kernel with all counters in shared memory (small graphs): 1/-1 on, 0 off
};

WalkVariant walk_variant() {
    static WalkVariant v = [] {
        WalkVariant w;
        if (const char* e = getenv("SABA_WALK_VARIANT")) {
            std::string s(e);
            auto get = [&](const char* k, int def) {  // whole keys only: "rec=" must not match "hrec="
                for (auto p = s.find(k); p != std::string::npos; p = s.find(k, p + 1))
                    if (p == 0 || s[p - 1] == ',') return atoi(s.c_str() + p + strlen(k));
                return def;
            };
            w.wpt = get("wpt=", w.wpt);
            w.packed = get("packed=", w.packed) != 0;
            w.c32 = get("c32=", w.c32) != 0;
            w.agg = get("agg=", w.agg) != 0;
            w.blocks_per_sm = get("bps=", 0);
            w.fat = get("fat=", w.fat);
            w.hot = get("hot=", w.hot);
            w.hot_threads = get("hthreads=", w.hot_threads);
            w.hot_count = get("hcount=", w.hot_count);
            w.sort = get("sort=", w.sort);
            w.rec = get("rec=", w.rec);
            w.hrec = get("hrec=", w.hrec);
            w.hcnt = get("hcnt=", w.hcnt);
            w.priv = get("priv=", w.priv);
        }
        return w;
    }();
    return v;
}

// The top vertices by degree get a shared-memory counter slot, packed into
// the spare high bits of the degree field (hot_shift = bits of max degree).
__global__ void hot_keys_kernel(const uint2* __restrict__ csr, uint32_t n, uint32_t dmax,
                                uint32_t* __restrict__ key, uint32_t* __restrict__ id) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        key[v] = dmax - csr[v].y;  // ascending sort = descending degree; keys fit bits(dmax)
        id[v] = v;
    }
}

__global__ void hot_mark_kernel(const uint32_t* __restrict__ sorted_id, uint32_t h, uint32_t shift,
                                uint2* __restrict__ csr_hot, uint32_t* __restrict__ hot_vertex) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < h; i += gridDim.x * blockDim.x) {
        const uint32_t v = sorted_id[i];
        hot_vertex[i] = v;
        csr_hot[v].y |= (i + 1) << shift;
    }
}

// Built on the device (it sits on the end-to-end path of every new graph):
// a stable radix sort by descending degree keeps ties in ascending id.
bool ensure_hot(saba_cu_graph* g) {
    if (g->hot_tried) return g->d_csr_hot != nullptr;
    g->hot_tried = true;
    if (g->n == 0) return false;
    uint32_t shift = 1;
    while (shift < 31 && (g->max_degree >> shift) != 0) ++shift;
    const WalkVariant v = walk_variant();
    g->hot_threads = v.hot_threads;
    // shared table: 128 KB per SM. Shared memory and L1 share one SRAM and
    // the L1 holds the in-flight gathers' lines; tables above ~160 KB starve
    // it (cfg2: 23.2 ms at 128 KB, 31.3 ms at 176 KB, 66 ms at 226 KB;
    // profiles/r01_walk_variant_sweep5_hot1024.txt)
    const uint32_t cap = v.hot_count > 0
                             ? uint32_t(v.hot_count)
                             : uint32_t(std::min<size_t>((size_t(128) << 10) / sizeof(uint32_t) - 1,
                                                         (g->smem_optin - 1024) / sizeof(uint32_t)) *
                                        std::max(256, std::min(1024, g->hot_threads)) / 1024);
    const uint32_t n = g->n;
    const uint32_t h = std::min({n, (1u << (32 - shift)) - 1, cap});
    if (h == 0) return false;
    g->hot_shift = shift;
    DevBuf k0, k1, i0, i1, tmp;
    cub::DoubleBuffer<uint32_t> keys(static_cast<uint32_t*>(k0.ensure(4 * size_t(n))),
                                     static_cast<uint32_t*>(k1.ensure(4 * size_t(n))));
    cub::DoubleBuffer<uint32_t> ids(static_cast<uint32_t*>(i0.ensure(4 * size_t(n))),
                                    static_cast<uint32_t*>(i1.ensure(4 * size_t(n))));
    const int blocks = int(std::min<uint32_t>((n + 255) / 256, uint32_t(g->sm_count) * 8));
    hot_keys_kernel<<<blocks, 256>>>(g->d_csr, n, g->max_degree, keys.Current(), ids.Current());
    SABA_CUDA_CHECK(cudaGetLastError());
    size_t tb = 0;
    int key_bits = 1;  // radix passes only over the bits a degree can set
    while (key_bits < 32 && (g->max_degree >> key_bits) != 0) ++key_bits;
    SABA_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, ids, int(n), 0, key_bits));
    SABA_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(tmp.ensure(tb), tb, keys, ids, int(n), 0, key_bits));
    g->d_csr_hot = static_cast<uint2*>(pool_alloc(sizeof(uint2) * n));
    g->d_hot_vertex = static_cast<uint32_t*>(pool_alloc(sizeof(uint32_t) * h));
    SABA_CUDA_CHECK(cudaMemcpy(g->d_csr_hot, g->d_csr, sizeof(uint2) * n, cudaMemcpyDeviceToDevice));
    hot_mark_kernel<<<(h + 255) / 256, 256>>>(ids.Current(), h, shift, g->d_csr_hot, g->d_hot_vertex);
    SABA_CUDA_CHECK(cudaGetLastError());
    SABA_CUDA_CHECK(cudaDeviceSynchronize());
    g->hot_count = h;
    return true;
}


__global__ void rec_build_kernel(const uint32_t* __restrict__ sorted_id, const uint2* __restrict__ csr, uint32_t n,
                                 uint32_t nb, uint32_t db, uint64_t* __restrict__ rec, uint32_t* __restrict__ rank) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t v = sorted_id[i];
        const uint2 r = csr[v];
        rec[i] = uint64_t(v) | (uint64_t(r.x) << nb) | (uint64_t(r.y) << db);
        rank[v] = i;
    }
}

__global__ void rank_adj_kernel(const uint32_t* __restrict__ adj, const uint32_t* __restrict__ rank, uint64_t two_m,
                                uint64_t* __restrict__ packed) {
    const uint64_t words = (two_m + 2) / 3;
    for (uint64_t w = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; w < words;
         w += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t x = 0;
        for (uint32_t q = 0; q < 3; ++q) {
            const uint64_t s = 3 * w + q;
            if (s < two_m) x |= uint64_t(rank[adj[s]]) << (kPackBits * q);
        }
        packed[w] = x;
    }
}

// Degree-ranked records (walk_count_rank_kernel), built on the device once per
// graph: a stable descending-degree order (ties by ascending id). Needs ranks
// that pack into 21 bits and {id, base, degree} in 64 bits.
bool ensure_rec(saba_cu_graph* g) {
    if (g->rec_tried) return g->d_rec != nullptr;
    g->rec_tried = true;
    if (g->n == 0 || g->n > kPackMax || g->m == 0) return false;
    g->hot_threads = walk_variant().hot_threads;
    auto bits = [](uint64_t x) {
        uint32_t b = 1;
        while (b < 64 && (uint64_t(1) << b) <= x) ++b;
        return b;
    };
    const uint32_t nb = bits(g->n - 1), bb = bits(2 * g->m), dbits = bits(g->max_degree);
    if (nb + bb + dbits > 64) return false;
    const uint32_t n = g->n;
    DevBuf k0, k1, i0, i1, tmp;
    cub::DoubleBuffer<uint32_t> keys(static_cast<uint32_t*>(k0.ensure(4 * size_t(n))),
                                     static_cast<uint32_t*>(k1.ensure(4 * size_t(n))));
    cub::DoubleBuffer<uint32_t> ids(static_cast<uint32_t*>(i0.ensure(4 * size_t(n))),
                                    static_cast<uint32_t*>(i1.ensure(4 * size_t(n))));
    const int blocks = int(std::min<uint32_t>((n + 255) / 256, uint32_t(g->sm_count) * 8));
    hot_keys_kernel<<<blocks, 256>>>(g->d_csr, n, g->max_degree, keys.Current(), ids.Current());
    SABA_CUDA_CHECK(cudaGetLastError());
    size_t tb = 0;
    int key_bits = 1;  // radix passes only over the bits a degree can set
    while (key_bits < 32 && (g->max_degree >> key_bits) != 0) ++key_bits;
    SABA_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, ids, int(n), 0, key_bits));
    SABA_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(tmp.ensure(tb), tb, keys, ids, int(n), 0, key_bits));
    g->rec_nb = nb;
    g->rec_db = nb + bb;
    g->d_rec = static_cast<uint64_t*>(pool_alloc(sizeof(uint64_t) * n));
    g->d_rank = static_cast<uint32_t*>(pool_alloc(sizeof(uint32_t) * n));
    rec_build_kernel<<<blocks, 256>>>(ids.Current(), g->d_csr, n, nb, g->rec_db, g->d_rec, g->d_rank);
    SABA_CUDA_CHECK(cudaGetLastError());
    const uint64_t words = (2 * g->m + 2) / 3;
    g->d_adj_rank = static_cast<uint64_t*>(pool_alloc(sizeof(uint64_t) * (words ? words : 1)));
    rank_adj_kernel<<<g->sm_count * 8, 256>>>(g->d_adj, g->d_rank, 2 * g->m, g->d_adj_rank);
    SABA_CUDA_CHECK(cudaGetLastError());
    SABA_CUDA_CHECK(cudaDeviceSynchronize());
    return true;
}

template <int WPT, int T, class CT>
bool launch_rank_t(saba_cu_graph* g, const uint64_t* keys, uint64_t nw, uint32_t L, uint64_t mult, void* counts,
                   cudaStream_t st) {
    const WalkVariant v = walk_variant();
    // 63 KB of shared memory (the 64 KB carve-out; the rest of the SM's SRAM
    // stays L1, which holds the lines of the gathers in flight): 20 KB of
    // records, 43 KB of 16-bit counters. Counters come first: without them
    // the reductions on the hottest vertices serialise in L2 (2,560 records +
    // 22,016 counters: 17.3 ms on cfg2; 7,936 records and no counters: 45 ms;
    // 128 KB split 6,144 / 40,960: 18.7 ms; profiles/r02_k2_rank_sweep.txt).
    const size_t budget = std::min<size_t>(size_t(63) << 10, g->smem_optin - 1024);
    const uint32_t nrec = std::min<uint32_t>(g->n, v.hrec >= 0 ? uint32_t(v.hrec) : uint32_t(budget * 20 / 63 / 8));
    const uint32_t ncnt = std::min<uint32_t>(g->n, v.hcnt >= 0 ? uint32_t(v.hcnt) : uint32_t(budget * 43 / 63 / 2));
    const size_t smem = sizeof(uint64_t) * nrec + sizeof(uint32_t) * ((size_t(ncnt) + 1) / 2);
    if (smem > g->smem_optin - 1024) return false;
    auto k = walk_count_rank_kernel<WPT, T, CT>;
    SABA_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int occ = 0;
    SABA_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, T, smem));
    if (occ < 1) return false;
    k<<<uint32_t(g->sm_count) * occ, T, smem, st>>>(g->d_rec, g->d_rank, g->d_adj_rank, g->rec_nb, g->rec_db, nrec,
                                                    ncnt, keys, nw, L, mult, static_cast<CT*>(counts));
    SABA_CUDA_CHECK(cudaGetLastError());
    g->last_nrec = nrec;
    g->last_ncnt = ncnt;
    return true;
}

__global__ void add_counts_kernel(const uint32_t* __restrict__ c32, uint32_t n,
                                  unsigned long long* __restrict__ counts) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        const uint32_t c = c32[v];
        if (c) counts[v] += c;
    }
}


template <int WPT, bool P, class CT, bool A>
void launch_walk_t(const saba_cu_graph* g, int bps, const uint64_t* keys, uint64_t nw, uint32_t L,
                   uint64_t mult, void* counts, cudaStream_t st) {
    auto k = walk_count_kernel<WPT, P, CT, A>;
    int occ = 0;
    SABA_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kWalkThreads, 0));
    if (bps <= 0 || bps > occ) bps = occ > 0 ? occ : 1;
    k<<<g->sm_count * bps, kWalkThreads, 0, st>>>(g->d_csr, g->d_adj, g->d_adj_packed, keys, nw, L,
                                                  mult, static_cast<CT*>(counts));
    SABA_CUDA_CHECK(cudaGetLastError());
}

template <int WPT>
void launch_walk_w(const saba_cu_graph* g, const WalkVariant& v, bool packed, bool c32,
                   const uint64_t* keys, uint64_t nw, uint32_t L, uint64_t mult, void* counts,
                   cudaStream_t st) {
    using U64 = unsigned long long;
#define SABA_LW(P, CT, A) launch_walk_t<WPT, P, CT, A>(g, v.blocks_per_sm, keys, nw, L, mult, counts, st)
    if (packed) {
        if (c32) { if (v.agg) SABA_LW(true, uint32_t, true); else SABA_LW(true, uint32_t, false); }
        else { if (v.agg) SABA_LW(true, U64, true); else SABA_LW(true, U64, false); }
    } else {
        if (c32) { if (v.agg) SABA_LW(false, uint32_t, true); else SABA_LW(false, uint32_t, false); }
        else { if (v.agg) SABA_LW(false, U64, true); else SABA_LW(false, U64, false); }
    }
#undef SABA_LW
}

template <int WPT, bool A>
void launch_fat_t(saba_cu_graph* g, int bps, const uint64_t* keys, uint64_t nw, uint32_t L,
                  uint64_t mult, void* counts, cudaStream_t st) {
    auto k = walk_count_fat_kernel<WPT, A>;
    int occ = 0;
    SABA_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kWalkThreads, 0));
    if (bps <= 0 || bps > occ) bps = occ > 0 ? occ : 1;
    k<<<g->sm_count * bps, kWalkThreads, 0, st>>>(g->d_csr, g->d_adj_fat, g->fat_idb, g->fat_sh, keys,
                                                  nw, L, mult, static_cast<unsigned long long*>(counts));
    SABA_CUDA_CHECK(cudaGetLastError());
}

// all-vertex 16-bit counters: at most 160 KB of shared memory (see ensure_hot
// on why the table must leave L1 room for the gathers in flight)
constexpr uint32_t kPrivMaxVertices = (160u << 10) / 2;
bool launch_fat_priv(saba_cu_graph* g, const uint64_t* keys, uint64_t nw, uint32_t L, uint64_t mult,
                     void* counts, cudaStream_t st) {
    constexpr int T = 1024, WPT = 4;
    auto k = walk_count_fat_priv_kernel<WPT, T>;
    const size_t smem = sizeof(uint32_t) * ((size_t(g->n) + 1) / 2);
    SABA_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int occ = 0;
    SABA_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, T, smem));
    if (occ < 1) return false;
    k<<<uint32_t(g->sm_count) * occ, T, smem, st>>>(g->d_csr, g->d_adj_fat, g->fat_idb, g->fat_sh, keys, nw, L,
                                                    mult, g->n, static_cast<unsigned long long*>(counts));
    SABA_CUDA_CHECK(cudaGetLastError());
    g->last_nrec = 0;
    g->last_ncnt = g->n;
    return true;
}

template <int WPT, bool P, bool A, int T>
bool launch_hot_t(saba_cu_graph* g, const uint64_t* keys, uint64_t nw, uint32_t L, uint64_t mult,
                  void* counts, cudaStream_t st) {
    auto k = walk_count_hot_kernel<WPT, P, A, T>;
    const size_t smem = sizeof(uint32_t) * g->hot_count;
    SABA_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int occ = 0;
    SABA_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, T, smem));
    if (occ < 1) return false;
    const uint64_t blocks = uint64_t(g->sm_count) * occ;
    // shared uint32 counters: a block can see at most ceil(nw / walks per
    // round) * walks per block-round walks of L visits each
    const uint64_t per_round = blocks * T * WPT;
    const uint64_t per_block = (nw + per_round - 1) / per_round * T * WPT;
    if (per_block * L >= (uint64_t(1) << 32)) return false;
    k<<<uint32_t(blocks), T, smem, st>>>(g->d_csr_hot, g->d_adj, g->d_adj_packed, g->d_hot_vertex,
                                         g->hot_count, g->hot_shift, keys, nw, L, mult,
                                         static_cast<unsigned long long*>(counts));
    SABA_CUDA_CHECK(cudaGetLastError());
    g->last_nrec = 0;
    g->last_ncnt = g->hot_count;
    return true;
}

template <bool P, bool A>
bool launch_hot_p(saba_cu_graph* g, const uint64_t* keys, uint64_t nw, uint32_t L, uint64_t mult,
                  void* counts, cudaStream_t st) {
    switch (g->hot_threads) {
        case 256: return launch_hot_t<4, P, A, 256>(g, keys, nw, L, mult, counts, st);
        case 512: return launch_hot_t<4, P, A, 512>(g, keys, nw, L, mult, counts, st);
        default: return launch_hot_t<4, P, A, 1024>(g, keys, nw, L, mult, counts, st);
    }
}

void launch_walk(saba_cu_graph* g, bool c32, const uint64_t* keys, uint64_t nw, uint32_t L,
                 uint64_t mult, void* counts, cudaStream_t st) {
    const WalkVariant v = walk_variant();
    g->last_nrec = g->last_ncnt = 0;
    // auto: the fat array (8 B/slot) pays off while it stays L2-resident;
    // beyond that the packed 2.67 B/slot adjacency moves fewer DRAM bytes
    // (cfg1: 24% faster fat, cfg2: 21% slower; profiles/r01_walk_variant_sweep2.txt)
    const bool want_fat = v.fat == 1 || (v.fat == -1 && 16 * g->m <= (uint64_t(48) << 20));
    if (want_fat && !c32 && ensure_fat(g)) {
        g->last_k2 = SABA_K2_FAT_PRIV;
        if (v.priv != 0 && g->n <= kPrivMaxVertices && launch_fat_priv(g, keys, nw, L, mult, counts, st)) return;
        g->last_k2 = SABA_K2_FAT;
        switch (v.wpt) {
            case 2: v.agg ? launch_fat_t<2, true>(g, v.blocks_per_sm, keys, nw, L, mult, counts, st)
                          : launch_fat_t<2, false>(g, v.blocks_per_sm, keys, nw, L, mult, counts, st); break;
            case 8: v.agg ? launch_fat_t<8, true>(g, v.blocks_per_sm, keys, nw, L, mult, counts, st)
                          : launch_fat_t<8, false>(g, v.blocks_per_sm, keys, nw, L, mult, counts, st); break;
            default: v.agg ? launch_fat_t<4, true>(g, v.blocks_per_sm, keys, nw, L, mult, counts, st)
                           : launch_fat_t<4, false>(g, v.blocks_per_sm, keys, nw, L, mult, counts, st); break;
        }
        return;
    }
    const bool packed = v.packed && g->d_adj_packed != nullptr;
    if (v.rec != 0 && v.hot != 0 && v.packed && ensure_rec(g)) {
        using U64 = unsigned long long;
        const bool ok = c32 ? launch_rank_t<4, 1024, uint32_t>(g, keys, nw, L, mult, counts, st)
                        : g->hot_threads == 512 ? launch_rank_t<4, 512, U64>(g, keys, nw, L, mult, counts, st)
                                                : launch_rank_t<4, 1024, U64>(g, keys, nw, L, mult, counts, st);
        g->last_k2 = SABA_K2_RANK;
        if (ok) return;
    }
    if (v.hot != 0 && !c32 && ensure_hot(g)) {
        const bool ok = packed ? (v.agg ? launch_hot_p<true, true>(g, keys, nw, L, mult, counts, st)
                                        : launch_hot_p<true, false>(g, keys, nw, L, mult, counts, st))
                               : (v.agg ? launch_hot_p<false, true>(g, keys, nw, L, mult, counts, st)
                                        : launch_hot_p<false, false>(g, keys, nw, L, mult, counts, st));
        g->last_k2 = SABA_K2_HOT;
        if (ok) return;
    }
    g->last_k2 = SABA_K2_GENERIC;
    switch (v.wpt) {
        case 1: launch_walk_w<1>(g, v, packed, c32, keys, nw, L, mult, counts, st); break;
        case 2: launch_walk_w<2>(g, v, packed, c32, keys, nw, L, mult, counts, st); break;
        case 8: launch_walk_w<8>(g, v, packed, c32, keys, nw, L, mult, counts, st); break;
        default: launch_walk_w<4>(g, v, packed, c32, keys, nw, L, mult, counts, st); break;
    }
}

// Branching statistics (BranchCollector, walker.hpp:64-109, 234, 430-449):
// block per start vertex. The vertex's K_v seeds are generated and (Saba)
// sorted in shared memory, so the reference's bouquets — `lanes` consecutive
// entries of the vertex's sorted seed list — are rebuilt exactly; each thread
// replays whole bouquets and records, per step, the number of distinct lane
// vertices and the degree sum at selection time. Integer sums: order-free.
// smem: K_v seeds (u32, padded to a power of two) | hist[lanes+1] | per_step[L-1]
__global__ void branch_stats_kernel(const uint2* __restrict__ csr, const uint32_t* __restrict__ adj,
                                    const uint64_t* __restrict__ adjp_unused, uint32_t n,
                                    const uint32_t* __restrict__ kv, uint64_t k_uniform,
                                    uint32_t kpad, uint32_t L, uint32_t lanes, int sorted,
                                    uint64_t master, uint64_t mult, uint32_t shard_index,
                                    uint32_t shard_count,
                                    unsigned long long* __restrict__ hist,
                                    unsigned long long* __restrict__ per_step,
                                    unsigned long long* __restrict__ totals) {
    extern __shared__ unsigned long long smem_u64[];
    unsigned long long* s_hist = smem_u64;
    unsigned long long* s_step = s_hist + (lanes + 1);
    uint32_t* seeds = reinterpret_cast<uint32_t*>(s_step + (L - 1));
    for (uint32_t i = threadIdx.x; i < lanes + 1 + (L - 1); i += blockDim.x) smem_u64[i] = 0;
    unsigned long long t_distinct = 0, t_samples = 0, t_lane_steps = 0, t_degsum = 0;
    // Shards take start vertices in stripes (v mod shard_count): every bouquet
    // belongs to one start vertex, so the shards' integer sums add up to the
    // unsharded statistics exactly.
    for (uint64_t vv = uint64_t(blockIdx.x) * shard_count + shard_index; vv < n;
         vv += uint64_t(gridDim.x) * shard_count) {
        const uint32_t v = uint32_t(vv);
        const uint32_t K = kv ? kv[v] : uint32_t(k_uniform);
        if (K == 0) continue;
        const uint64_t vseed = substream(master, v);
        __syncthreads();
        const uint32_t P = sorted ? kpad : K;
        for (uint32_t k = threadIdx.x; k < P; k += blockDim.x)
            seeds[k] = k < K ? walk_seed(vseed, k) : 0xffffffffu;  // padding sorts last
        __syncthreads();
        if (sorted) {  // bitonic sort of the padded seed list (walker.hpp:439)
            for (uint32_t size = 2; size <= P; size <<= 1)
                for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
                    for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
                        const uint32_t j = i ^ stride;
                        if (j > i) {
                            const bool up = (i & size) == 0;
                            const uint32_t a = seeds[i], b = seeds[j];
                            if ((a > b) == up) {
                                seeds[i] = b;
                                seeds[j] = a;
                            }
                        }
                    }
                    __syncthreads();
                }
        }
        const uint32_t nb = (K + lanes - 1) / lanes;
        for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) {
            const uint32_t act = min(lanes, K - b * lanes);
            uint32_t cur[64], tmp[64];
            for (uint32_t i = 0; i < act; ++i) cur[i] = v;
            for (uint32_t l = 1; l < L; ++l) {
                unsigned long long degsum = 0;
                for (uint32_t i = 0; i < act; ++i) {
                    const uint2 rec = ldg_csr(csr + cur[i]);
                    degsum += rec.y;
                    const uint32_t raw = seeds[b * lanes + i] ^ hash_state(mult, cur[i], l);
                    cur[i] = ldg_u32(adj + rec.x + scaled_index(raw, rec.y));
                }
                // distinct lane vertices (insertion sort, walker.hpp:77-90)
                for (uint32_t i = 0; i < act; ++i) {
                    const uint32_t x = cur[i];
                    uint32_t j = i;
                    while (j > 0 && tmp[j - 1] > x) {
                        tmp[j] = tmp[j - 1];
                        --j;
                    }
                    tmp[j] = x;
                }
                uint32_t distinct = 1;
                for (uint32_t i = 1; i < act; ++i) distinct += tmp[i] != tmp[i - 1];
                atomicAdd(s_hist + distinct, 1ull);
                atomicAdd(s_step + (l - 1), (unsigned long long)distinct);
                t_distinct += distinct;
                t_samples += 1;
                t_lane_steps += act;
                t_degsum += degsum;
            }
        }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < lanes + 1; i += blockDim.x)
        if (s_hist[i]) atomicAdd(hist + i, s_hist[i]);
    for (uint32_t i = threadIdx.x; i < L - 1; i += blockDim.x)
        if (s_step[i]) atomicAdd(per_step + i, s_step[i]);
    if (t_samples) {
        atomicAdd(totals + 0, t_distinct);
        atomicAdd(totals + 1, t_samples);
        atomicAdd(totals + 2, t_lane_steps);
        atomicAdd(totals + 3, t_degsum);
    }
}

// rng_stream (stream.hpp:29-83): the raw pre-selection word seed ^ h(cur, l)
// of every step, merged step-major per start (word (l-1)*K + k of the start's
// block). Thread per (start, k) walk. xor_mod = 1 selects raw % degree.
__global__ void rng_stream_kernel(const uint2* __restrict__ csr, const uint32_t* __restrict__ adj,
                                  const uint32_t* __restrict__ starts, uint64_t total, uint64_t K,
                                  uint32_t L, uint64_t master, uint64_t mult, int xor_mod,
                                  uint32_t* __restrict__ words) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
        const uint64_t si = i / K, k = i - si * K;
        uint32_t cur = starts[si];
        const uint32_t seed = walk_seed(substream(master, cur), k);  // stream.hpp:45, 58
        uint32_t* out = words + si * K * (L - 1) + k;
        for (uint32_t l = 1; l < L; ++l) {
            const uint2 rec = ldg_csr(csr + cur);
            const uint32_t raw = seed ^ hash_state(mult, cur, l);
            out[uint64_t(l - 1) * K] = raw;
            cur = ldg_u32(adj + rec.x + (xor_mod ? raw % rec.y : scaled_index(raw, rec.y)));
        }
    }
}

// One thread per walk; materialises the path (random_walk, walker.hpp:283-302).
__global__ void walk_paths_kernel(const uint2* __restrict__ csr, const uint32_t* __restrict__ adj,
                                  const uint32_t* __restrict__ starts,
                                  const uint32_t* __restrict__ seeds, uint64_t count, uint32_t L,
                                  uint64_t mult, uint32_t* __restrict__ paths) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
        uint32_t cur = starts[i];
        const uint32_t seed = seeds[i];
        uint32_t* out = paths + i * L;
        out[0] = cur;
        for (uint32_t l = 1; l < L; ++l) {
            const uint2 rec = ldg_csr(csr + cur);
            cur = ldg_u32(adj + rec.x + scaled_index(seed ^ hash_state(mult, cur, l), rec.y));
            out[l] = cur;
        }
    }
}

constexpr uint64_t kChunkWalks = uint64_t(1) << 27;  // keys per pass (1 GiB x2)

void validate_campaign(const saba_cu_graph* g, const saba_cu_campaign_config& c) {
    // walker.hpp:461-468, same order and messages
    if (c.total_walks == 0) check_arg(c.walks_per_vertex >= 1, "walks_per_vertex must be >= 1");
    check_arg(c.length >= 1, "length must be >= 1");
    check_arg(c.lanes >= 1 && c.lanes <= 64 && (c.lanes & (c.lanes - 1)) == 0,
              "lanes must be a power of two in [1, 64]");
    if (c.length > 1)
        check_arg(g->min_degree >= 1, "campaign requires degree >= 1 at every vertex when L > 1");
    check_arg(c.mode == SABA_MODE_HASH || c.mode == SABA_MODE_SABA,
              "mode not supported on GPU (naive/vector-mod are CPU LCG baselines)");
    check_arg(c.shard_count >= 1 && c.shard_index < c.shard_count, "bad shard index/count");
}


// Enqueue the whole campaign shard on `st`. Returns walks executed.
uint64_t enqueue_campaign(saba_cu_graph* g, const saba_cu_campaign_config& c,
                          unsigned long long* counts, cudaStream_t st, bool timing,
                          float* walk_ms, uint32_t* launches) {
    const uint32_t n = g->n;
    const bool uniform_starts = c.total_walks > 0;
    const uint64_t total = uniform_starts ? c.total_walks : uint64_t(n) * c.walks_per_vertex;
    check_arg(uniform_starts || c.walks_per_vertex <= (uint64_t(1) << 40) / (n ? n : 1),
              "walks_per_vertex too large");
    const uint64_t r0 = total * c.shard_index / c.shard_count;
    const uint64_t r1 = total * (uint64_t(c.shard_index) + 1) / c.shard_count;
    uint32_t* kv = nullptr;
    uint64_t* off = nullptr;
    if (uniform_starts) {
        kv = static_cast<uint32_t*>(g->kv.ensure(sizeof(uint32_t) * n, st));
        off = static_cast<uint64_t*>(g->off.ensure(sizeof(uint64_t) * (size_t(n) + 1), st));
        SABA_CUDA_CHECK(cudaMemsetAsync(kv, 0, sizeof(uint32_t) * n, st));
        const uint64_t sstream = substream(c.master_seed, kStartTag);
        const int hb = int(std::min<uint64_t>((c.total_walks + 255) / 256, uint64_t(g->sm_count) * 16));
        start_hist_kernel<<<hb, 256, 0, st>>>(c.total_walks, sstream, n, kv);
        SABA_CUDA_CHECK(cudaGetLastError());
        ++*launches;
        size_t tmp = 0;
        cub::TransformInputIterator<uint64_t, U32ToU64, const uint32_t*> it(kv, U32ToU64());
        SABA_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, it, off, int(n), st));
        void* t = g->cub_tmp.ensure(tmp, st);
        SABA_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(t, tmp, it, off, int(n), st));
        ++*launches;
    }
    const uint64_t chunk_cap = std::min<uint64_t>(kChunkWalks, r1 - r0 ? r1 - r0 : 1);
    // SABA sort fused into key generation when the walks per start vertex are
    // well below the warp sort's cap (uniform starts: K_v ~ Poisson(W/n));
    // large per-vertex campaigns keep the full segmented sort.
    // SABA_WALK_VARIANT sort=0 forces the CUB segmented sort, sort=1 the fused one.
    const double mean_k = uniform_starts ? double(c.total_walks) / double(n ? n : 1) : double(c.walks_per_vertex);
    const int sort_knob = walk_variant().sort;
    const bool fused_sort = c.mode == SABA_MODE_SABA && (sort_knob == 1 || (sort_knob < 0 && mean_k <= 64.0));
    uint64_t* keys = static_cast<uint64_t*>(g->keys.ensure(sizeof(uint64_t) * chunk_cap, st));
    uint64_t* keys_alt = c.mode == SABA_MODE_SABA && !fused_sort
                             ? static_cast<uint64_t*>(g->keys_alt.ensure(sizeof(uint64_t) * chunk_cap, st))
                             : nullptr;
    int* seg = static_cast<int*>(g->seg.ensure(sizeof(int) * (size_t(n) + 1), st));
    // uint32 counters are exact when this launch's visits cannot reach 2^32
    const bool c32 = walk_variant().c32 && chunk_cap * c.length < (uint64_t(1) << 32);
    uint32_t* counts32 = c32 ? static_cast<uint32_t*>(g->counts32.ensure(sizeof(uint32_t) * n, st)) : nullptr;
    float total_walk_ms = 0.f;
    for (uint64_t a = r0; a < r1; a += chunk_cap) {
        const uint64_t b = std::min(r1, a + chunk_cap);
        const uint64_t nw = b - a;
        const int gb = int(std::min<uint64_t>((uint64_t(n) * 32 + 255) / 256, uint64_t(g->sm_count) * 32));
        const uint64_t* walk_keys = keys;
        if (fused_sort) {  // K1 generate + per-vertex seed sort in one pass
            gen_sorted_keys_kernel<<<gb, 256, 0, st>>>(n, kv, c.walks_per_vertex, off, a, b, c.master_seed, keys,
                                                       counts);
            SABA_CUDA_CHECK(cudaGetLastError());
            ++*launches;
        } else {
            gen_keys_kernel<<<gb, 256, 0, st>>>(n, kv, c.walks_per_vertex, off, a, b, c.master_seed, keys,
                                                seg, counts);
            SABA_CUDA_CHECK(cudaGetLastError());
            ++*launches;
        }
        if (c.mode == SABA_MODE_SABA && !fused_sort) {
            size_t tmp = 0;
            SABA_CUDA_CHECK(cub::DeviceSegmentedSort::SortKeys(nullptr, tmp, keys, keys_alt, int(nw),
                                                               int(n), seg, seg + 1, st));
            void* t = g->cub_tmp.ensure(tmp, st);
            SABA_CUDA_CHECK(cub::DeviceSegmentedSort::SortKeys(t, tmp, keys, keys_alt, int(nw), int(n),
                                                               seg, seg + 1, st));
            ++*launches;
            walk_keys = keys_alt;
        }
        if (c.length > 1) {
            if (c32) SABA_CUDA_CHECK(cudaMemsetAsync(counts32, 0, sizeof(uint32_t) * n, st));
            if (timing) SABA_CUDA_CHECK(cudaEventRecord(g->ev1, st));
            launch_walk(g, c32, walk_keys, nw, c.length, c.hash_multiplier,
                        c32 ? static_cast<void*>(counts32) : static_cast<void*>(counts), st);
            ++*launches;
            if (timing) SABA_CUDA_CHECK(cudaEventRecord(g->ev2, st));
            if (c32) {
                add_counts_kernel<<<g->sm_count * 4, 256, 0, st>>>(counts32, n, counts);
                SABA_CUDA_CHECK(cudaGetLastError());
                ++*launches;
            }
            if (timing) {
                SABA_CUDA_CHECK(cudaEventSynchronize(g->ev2));
                float ms = 0.f;
                SABA_CUDA_CHECK(cudaEventElapsedTime(&ms, g->ev1, g->ev2));
                total_walk_ms += ms;
            }
        }
    }
    if (walk_ms) *walk_ms = total_walk_ms;
    return r1 - r0;
}

void fill_report(const saba_cu_graph* g, const saba_cu_campaign_config& c, uint64_t shard_walks,
                 saba_cu_campaign_report* rep) {
    const uint64_t total = c.total_walks > 0 ? c.total_walks : uint64_t(g->n) * c.walks_per_vertex;
    rep->total_steps = total * (c.length - 1);
    rep->total_events = total * c.length;
    rep->shard_walks = shard_walks;
    rep->shard_steps = shard_walks * (c.length - 1);
    rep->kernel = c.length > 1 ? g->last_k2 : SABA_K2_NONE;
}

}  // namespace
}  // namespace saba_cu

using namespace saba_cu;

extern "C" {

int saba_cu_rng_stream(saba_cu_graph* g, const uint32_t* starts, uint32_t nstarts,
                       uint64_t walks_per_vertex, uint32_t length, int selector, uint64_t master,
                       uint64_t mult, uint32_t* words_out, uint64_t* nwords) {
    return guard([&] {
        check_arg(g && nwords, "null argument");
        // stream.hpp:32-36, same order and messages
        check_arg(walks_per_vertex >= 1, "rng_stream: walks_per_vertex must be >= 1");
        check_arg(length >= 1, "rng_stream: length must be >= 1");
        check_arg(nstarts > 0 && starts, "rng_stream: no start vertices");
        for (uint32_t i = 0; i < nstarts; ++i) {
            check_arg(starts[i] < g->n, "start vertex out of range");
            check_arg(length == 1 || g->h_off[starts[i] + 1] > g->h_off[starts[i]],
                      "cannot walk from an isolated vertex");
        }
        check_arg(selector == 1 || selector == 2,
                  "rng_stream: only the hashed selectors (xor, scaled) run on GPU");
        check_arg(length == 1 || walks_per_vertex <= UINT64_MAX / (uint64_t(length) - 1) / nstarts,
                  "rng_stream: nstarts * walks_per_vertex * (length - 1) overflows");
        *nwords = uint64_t(nstarts) * walks_per_vertex * (length - 1);
        if (length == 1) return;
        check_arg(words_out != nullptr, "null output");
        std::lock_guard<std::recursive_mutex> lock(g->mu);
        DeviceScope scope(g->device);
        // The stream feeds statistical test dumps that can be gigabytes long
        // (stream.hpp:39-80 emits one start at a time): generate it in chunks
        // of whole starts, at most ~256 MB of words per chunk (at least one
        // start), each copied out before the next is generated.
        const uint64_t per_start = walks_per_vertex * (length - 1);
        const uint64_t chunk = std::max<uint64_t>(1, std::min<uint64_t>(nstarts, (uint64_t(64) << 20) / per_start));
        DevBuf d_st, d_w;
        d_st.ensure(sizeof(uint32_t) * nstarts);
        d_w.ensure(sizeof(uint32_t) * chunk * per_start);
        SABA_CUDA_CHECK(cudaMemcpy(d_st.p, starts, sizeof(uint32_t) * nstarts, cudaMemcpyHostToDevice));
        for (uint64_t s0 = 0; s0 < nstarts; s0 += chunk) {
            const uint64_t ns = std::min<uint64_t>(chunk, nstarts - s0);
            const uint64_t total = ns * walks_per_vertex;
            const int blocks = int(std::min<uint64_t>((total + 255) / 256, uint64_t(g->sm_count) * 8));
            rng_stream_kernel<<<blocks, 256>>>(g->d_csr, g->d_adj, d_st.as<uint32_t>() + s0, total,
                                               walks_per_vertex, length, master, mult, selector == 1,
                                               d_w.as<uint32_t>());
            SABA_CUDA_CHECK(cudaGetLastError());
            copy_d2h(words_out + s0 * per_start, d_w.p, sizeof(uint32_t) * ns * per_start, 0);
        }
    });
}

int saba_cu_walk_paths(saba_cu_graph* g, const uint32_t* starts, const uint32_t* seeds,
                       uint64_t count, uint32_t length, uint64_t mult, uint32_t* paths_out) {
    return guard([&] {
        check_arg(g && (count == 0 || (starts && seeds && paths_out)), "null argument");
        check_arg(length >= 1, "walk length must be >= 1");  // walker.hpp:271
        for (uint64_t i = 0; i < count; ++i) {
            check_arg(starts[i] < g->n, "start vertex out of range");
            check_arg(length == 1 || g->h_off[starts[i] + 1] > g->h_off[starts[i]],
                      "cannot walk from an isolated vertex");
        }
        if (count == 0) return;
        std::lock_guard<std::recursive_mutex> lock(g->mu);
        DeviceScope scope(g->device);
        DevBuf d_st, d_sd, d_p;
        d_st.ensure(sizeof(uint32_t) * count);
        d_sd.ensure(sizeof(uint32_t) * count);
        d_p.ensure(sizeof(uint32_t) * count * length);
        SABA_CUDA_CHECK(cudaMemcpy(d_st.p, starts, sizeof(uint32_t) * count, cudaMemcpyHostToDevice));
        SABA_CUDA_CHECK(cudaMemcpy(d_sd.p, seeds, sizeof(uint32_t) * count, cudaMemcpyHostToDevice));
        const int blocks = int(std::min<uint64_t>((count + 255) / 256, uint64_t(g->sm_count) * 8));
        walk_paths_kernel<<<blocks, 256>>>(g->d_csr, g->d_adj, d_st.as<uint32_t>(), d_sd.as<uint32_t>(),
                                           count, length, mult, d_p.as<uint32_t>());
        SABA_CUDA_CHECK(cudaGetLastError());
        SABA_CUDA_CHECK(cudaMemcpy(paths_out, d_p.p, sizeof(uint32_t) * count * length,
                                   cudaMemcpyDeviceToHost));
    });
}

int saba_cu_campaign_tables(const saba_cu_graph* g, uint32_t* records, uint32_t* counters) {
    return guard([&] {
        check_arg(g && records && counters, "null argument");
        *records = g->last_nrec;
        *counters = g->last_ncnt;
    });
}

int saba_cu_walk_campaign_device(saba_cu_graph* g, const saba_cu_campaign_config* cfg,
                                 uint64_t* counts_dev, void* stream, int timing,
                                 saba_cu_campaign_report* rep) {
    return guard([&] {
        check_arg(g && cfg && counts_dev, "null argument");
        validate_campaign(g, *cfg);
        std::lock_guard<std::recursive_mutex> lock(g->mu);
        DeviceScope scope(g->device);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        saba_cu_campaign_report r{};
        float walk_ms = 0.f;
        g->enter(st);
        if (timing) SABA_CUDA_CHECK(cudaEventRecord(g->ev0, st));
        const uint64_t w = enqueue_campaign(g, *cfg, reinterpret_cast<unsigned long long*>(counts_dev),
                                            st, timing != 0, &walk_ms, &r.launches);
        g->leave(st);
        if (timing) {
            SABA_CUDA_CHECK(cudaEventRecord(g->ev1, st));
            SABA_CUDA_CHECK(cudaEventSynchronize(g->ev1));
            float ms = 0.f;
            SABA_CUDA_CHECK(cudaEventElapsedTime(&ms, g->ev0, g->ev1));
            r.seconds = ms * 1e-3;
            r.walk_kernel_ms = walk_ms;
        }
        fill_report(g, *cfg, w, &r);
        if (rep) *rep = r;
    });
}

int saba_cu_branching_stats(saba_cu_graph* g, const saba_cu_campaign_config* cfg,
                            uint64_t* histogram_out, uint64_t* per_step_out, uint64_t* totals_out) {
    return guard([&] {
        check_arg(g && cfg && histogram_out && per_step_out && totals_out, "null argument");
        validate_campaign(g, *cfg);
        check_arg(cfg->length > 1, "branching statistics need walks of length > 1");
        std::lock_guard<std::recursive_mutex> lock(g->mu);
        DeviceScope scope(g->device);
        const uint32_t n = g->n, L = cfg->length, lanes = cfg->lanes;
        uint32_t* kv = nullptr;
        uint64_t kmax = cfg->walks_per_vertex;
        DevBuf d_kv;
        if (cfg->total_walks > 0) {
            kv = static_cast<uint32_t*>(d_kv.ensure(sizeof(uint32_t) * n));
            SABA_CUDA_CHECK(cudaMemset(kv, 0, sizeof(uint32_t) * n));
            const int hb = int(std::min<uint64_t>((cfg->total_walks + 255) / 256, uint64_t(g->sm_count) * 16));
            start_hist_kernel<<<hb, 256>>>(cfg->total_walks, substream(cfg->master_seed, kStartTag), n, kv);
            SABA_CUDA_CHECK(cudaGetLastError());
            std::vector<uint32_t> h(n);
            SABA_CUDA_CHECK(cudaMemcpy(h.data(), kv, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost));
            kmax = *std::max_element(h.begin(), h.end());
        }
        uint32_t kpad = 1;
        while (kpad < kmax) kpad <<= 1;
        const size_t smem = sizeof(uint64_t) * (lanes + L) + sizeof(uint32_t) * kpad;
        check_arg(smem <= 220 * 1024, "branching statistics: too many walks per vertex or steps for one block");
        SABA_CUDA_CHECK(cudaFuncSetAttribute(branch_stats_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(smem)));
        DevBuf d_hist, d_step, d_tot;
        auto* hist = static_cast<unsigned long long*>(d_hist.ensure(sizeof(uint64_t) * (lanes + 1)));
        auto* step = static_cast<unsigned long long*>(d_step.ensure(sizeof(uint64_t) * (L - 1)));
        auto* tot = static_cast<unsigned long long*>(d_tot.ensure(sizeof(uint64_t) * 4));
        SABA_CUDA_CHECK(cudaMemset(hist, 0, sizeof(uint64_t) * (lanes + 1)));
        SABA_CUDA_CHECK(cudaMemset(step, 0, sizeof(uint64_t) * (L - 1)));
        SABA_CUDA_CHECK(cudaMemset(tot, 0, sizeof(uint64_t) * 4));
        const uint64_t nv = (uint64_t(n) + cfg->shard_count - 1) / cfg->shard_count;
        const int blocks = int(std::max<uint64_t>(1, std::min<uint64_t>(nv, uint64_t(g->sm_count) * 8)));
        branch_stats_kernel<<<blocks, 256, smem>>>(g->d_csr, g->d_adj, g->d_adj_packed, n, kv,
                                                   cfg->walks_per_vertex, kpad, L, lanes,
                                                   cfg->mode == SABA_MODE_SABA, cfg->master_seed,
                                                   cfg->hash_multiplier, cfg->shard_index, cfg->shard_count,
                                                   hist, step, tot);
        SABA_CUDA_CHECK(cudaGetLastError());
        SABA_CUDA_CHECK(cudaMemcpy(histogram_out, hist, sizeof(uint64_t) * (lanes + 1), cudaMemcpyDeviceToHost));
        SABA_CUDA_CHECK(cudaMemcpy(per_step_out, step, sizeof(uint64_t) * (L - 1), cudaMemcpyDeviceToHost));
        SABA_CUDA_CHECK(cudaMemcpy(totals_out, tot, sizeof(uint64_t) * 4, cudaMemcpyDeviceToHost));
    });
}

int saba_cu_walk_campaign(saba_cu_graph* g, const saba_cu_campaign_config* cfg,
                          uint64_t* counts_out, saba_cu_campaign_report* rep) {
    return guard([&] {
        check_arg(g && cfg && counts_out, "null argument");
        validate_campaign(g, *cfg);
        std::lock_guard<std::recursive_mutex> lock(g->mu);
        // One shard per replica (a multi-device handle): replica r
        // of R runs walk range shard_index * R + r of shard_count * R, which
        // tile this call's range exactly; one host thread per replica, then
        // one combine of the integer counts on the first replica.
        const std::vector<saba_cu_graph*> reps = replicas_of(g);
        const uint32_t R = uint32_t(reps.size());
        const bool trace = getenv("SABA_TRACE") != nullptr;
        auto T0 = std::chrono::steady_clock::now();
        auto lap = [&](const char* what) {
            if (!trace) return;
            const auto T1 = std::chrono::steady_clock::now();
            fprintf(stderr, "[saba] campaign %-16s %8.3f ms\n", what,
                    std::chrono::duration<double, std::milli>(T1 - T0).count());
            T0 = T1;
        };
        std::vector<DevBuf> bufs(R);
        std::vector<uint64_t> walks(R, 0);
        std::vector<float> walk_ms(R, 0.f), span_ms(R, 0.f);
        std::vector<uint32_t> launches(R, 0);
        std::vector<std::exception_ptr> err(R);
        const auto t0 = std::chrono::steady_clock::now();
        auto run = [&](uint32_t r) {
            try {
                saba_cu_graph* h = reps[r];
                std::unique_lock<std::recursive_mutex> lk(h->mu, std::defer_lock);
                if (r) lk.lock();  // replica 0 is g, already held by this thread
                DeviceScope scope(h->device);
                saba_cu_campaign_config c = *cfg;
                c.shard_index = cfg->shard_index * R + r;
                c.shard_count = cfg->shard_count * R;
                bufs[r].ensure(sizeof(uint64_t) * h->n, 0);
                SABA_CUDA_CHECK(cudaMemsetAsync(bufs[r].p, 0, sizeof(uint64_t) * h->n, 0));
                h->enter(0);
                SABA_CUDA_CHECK(cudaEventRecord(h->ev0, 0));
                walks[r] = enqueue_campaign(h, c, bufs[r].as<unsigned long long>(), 0, true, &walk_ms[r],
                                            &launches[r]);
                h->leave(0);
                SABA_CUDA_CHECK(cudaEventRecord(h->ev1, 0));
                SABA_CUDA_CHECK(cudaEventSynchronize(h->ev1));
                SABA_CUDA_CHECK(cudaEventElapsedTime(&span_ms[r], h->ev0, h->ev1));
            } catch (...) {
                err[r] = std::current_exception();
            }
        };
        std::vector<std::thread> threads;
        for (uint32_t r = 1; r < R; ++r) threads.emplace_back(run, r);
        run(0);
        for (auto& t : threads) t.join();
        for (auto& e : err)
            if (e) std::rethrow_exception(e);
        lap("enqueue + wait");
        std::vector<void*> ptrs;
        for (auto& b : bufs) ptrs.push_back(b.p);
        reduce_to_root(reps, ptrs, g->n, ReduceType::U64, std::vector<cudaStream_t>(R, nullptr));
        DeviceScope scope(g->device);
        lap("combine");
        copy_d2h(counts_out, bufs[0].p, sizeof(uint64_t) * g->n, 0);  // staged through pinned buffers when large
        lap("counts d2h");
        saba_cu_campaign_report r{};
        if (R == 1) {
            r.seconds = span_ms[0] * 1e-3;  // device events around the campaign
        } else {
            r.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        }
        uint64_t w = 0;
        for (uint32_t i = 0; i < R; ++i) {
            w += walks[i];
            r.walk_kernel_ms = std::max(r.walk_kernel_ms, double(walk_ms[i]));
            r.launches += launches[i];
        }
        fill_report(g, *cfg, w, &r);
        if (rep) *rep = r;
    });
}

}  // extern "C"
