// Device helpers shared by the campaign (K2) and AESC walk-phase (K4) kernels.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

// Checked builds (tools/build_variant.sh checked "-DSABA_CHECKED"): device
// asserts on the indices the cross-block protocols produce (frontier appends,
// work-list hand-out, bucket scatters, hub-counter slots, walk vertices). The
// compute-sanitizer is not available on the GPU pool, so these plus small
// cases compared with the CPU reference stand in for memcheck.
#ifdef SABA_CHECKED
#include <cstdio>
#define SABA_DCHECK(c)                                                                   \
    do {                                                                                 \
        if (!(c)) {                                                                      \
            printf("SABA_DCHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c);           \
            __trap();                                                                    \
        }                                                                                \
    } while (0)
#else
#define SABA_DCHECK(c) \
    do {               \
    } while (0)
#endif

namespace saba_cu {

// One 8-byte read-only gather of {base, degree} (LDG.E.64.CONSTANT).
__device__ __forceinline__ uint2 ldg_csr(const uint2* p) { return __ldg(p); }
__device__ __forceinline__ uint32_t ldg_u32(const uint32_t* p) { return __ldg(p); }
__device__ __forceinline__ double ldg_f64(const double* p) { return __ldg(p); }

// Read-only gathers that do not allocate in L1: adjacency slots are touched
// uniformly at random, so caching them in L1 only evicts the hot {base, deg}
// records of hub vertices that L1 can actually keep.
// SABA_ADJ_LD (experiment builds, tools/build_variant.sh) picks the cache
// operator of these gathers: 0 nc.L1::no_allocate, 1 plain nc (L1-allocating),
// 2 .cg (L2 only), 3 nc.L1::evict_first, 4 .cs, 5 .lu, 6/7/8 nc with an L2
// prefetch size of 128 / 256 / 64 bytes.
#ifndef SABA_ADJ_LD
#define SABA_ADJ_LD 1
#endif
#if SABA_ADJ_LD == 0
#define SABA_ADJ_LD_OP "ld.global.nc.L1::no_allocate"
#elif SABA_ADJ_LD == 1
#define SABA_ADJ_LD_OP "ld.global.nc"
#elif SABA_ADJ_LD == 2
#define SABA_ADJ_LD_OP "ld.global.cg"
#elif SABA_ADJ_LD == 3
#define SABA_ADJ_LD_OP "ld.global.nc.L1::evict_first"
#elif SABA_ADJ_LD == 4
#define SABA_ADJ_LD_OP "ld.global.cs"
#elif SABA_ADJ_LD == 5
#define SABA_ADJ_LD_OP "ld.global.lu"
#elif SABA_ADJ_LD == 6
#define SABA_ADJ_LD_OP "ld.global.nc.L2::128B"
#elif SABA_ADJ_LD == 7
#define SABA_ADJ_LD_OP "ld.global.nc.L2::256B"
#else
#define SABA_ADJ_LD_OP "ld.global.nc.L2::64B"
#endif
__device__ __forceinline__ uint64_t ldg_na_u64(const uint64_t* p) {
    uint64_t v;
    asm(SABA_ADJ_LD_OP ".u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint32_t ldg_na_u32(const uint32_t* p) {
    uint32_t v;
    asm(SABA_ADJ_LD_OP ".u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

// Neighbour id at directed slot s. Packed: 3 x 21-bit fields per uint64.
// The gather and the field extraction are separate calls so that a thread can
// issue the gathers of all its walks before it consumes the first one.
template <bool PACKED>
struct AdjWord {
    uint64_t word;
    uint32_t shift;
};
template <bool PACKED>
__device__ __forceinline__ AdjWord<PACKED> adj_load(const uint32_t* __restrict__ adj,
                                                    const uint64_t* __restrict__ packed, uint32_t s) {
    AdjWord<PACKED> a;
    if constexpr (PACKED) {
        const uint32_t w = __umulhi(s, 0xAAAAAAABu) >> 1;  // s / 3 for s < 2^32
        a.shift = 21 * (s - 3 * w);
        a.word = ldg_na_u64(packed + w);
    } else {
        a.shift = 0;
        a.word = ldg_na_u32(adj + s);
    }
    return a;
}
template <bool PACKED>
__device__ __forceinline__ uint32_t adj_id(const AdjWord<PACKED>& a) {
    if constexpr (PACKED)
        return uint32_t(a.word >> a.shift) & 0x1FFFFFu;
    else
        return uint32_t(a.word);
}
template <bool PACKED>
__device__ __forceinline__ uint32_t adj_at(const uint32_t* __restrict__ adj,
                                           const uint64_t* __restrict__ packed, uint32_t s) {
    return adj_id<PACKED>(adj_load<PACKED>(adj, packed, s));
}

// VisitCountSink epilogue (walker.hpp:355) with warp aggregation: lanes of a
// SABA bouquet sit on the same vertex in runs of adjacent lanes, so the head
// of every run of equal `v` (found with one shuffle + ballot) issues a single
// L2 reduction for the whole run. Divergent lanes degrade to one reduction
// each. Inactive lanes end a run (any active mask); all 32 lanes must call.
template <class CT>
__device__ __forceinline__ void warp_count_visit(CT* __restrict__ counts, uint32_t v, bool act,
                                                 uint32_t lane) {
    const uint32_t prev = __shfl_up_sync(0xffffffffu, v, 1);
    const uint32_t amask = __ballot_sync(0xffffffffu, act);
    const bool prev_act = lane > 0 && ((amask >> (lane - 1)) & 1u);
    const bool head = act && (!prev_act || prev != v);
    const uint32_t heads = __ballot_sync(0xffffffffu, head);
    if (head) {
        // the run ends at the next head or the next inactive lane above this one
        const uint32_t stops = (heads | ~amask) & ~((2u << lane) - 1u);
        const uint32_t end = stops ? uint32_t(__ffs(stops) - 1) : 32u;
        atomicAdd(counts + v, static_cast<CT>(end - lane));
    }
}

// Shared-memory visit counters, two 16-bit fields per 32-bit word: bits 0-14
// of a field count, bit 15 is a guard. The increment that sets the guard
// (old field value 0x7FFF) moves 2^15 visits to the vertex's global counter
// and clears the guard again. A field never carries into its neighbour as
// long as a block makes fewer than 2^15 increments between two of its
// barriers: every guard set before a barrier is cleared before it, so each
// field is below 0x8000 at a barrier and below 0x8000 + 2^15 before the next
// (kCount16Steps below bounds the steps between barriers accordingly).
template <class CT>
__device__ __forceinline__ void smem_count16(uint32_t* __restrict__ tab, uint32_t slot,
                                             CT* __restrict__ counts, uint32_t vertex) {
    const uint32_t sh = (slot & 1u) << 4;
    const uint32_t old = atomicAdd(tab + (slot >> 1), 1u << sh);
    if (((old >> sh) & 0xFFFFu) == 0x7FFFu) {
        atomicSub(tab + (slot >> 1), 0x8000u << sh);
        atomicAdd(counts + vertex, CT(32768));
    }
}
// steps between block barriers so that THREADS * WPT * steps < 2^15
__host__ __device__ constexpr uint32_t count16_steps(uint32_t threads, uint32_t wpt) {
    return (32768u - 1u) / (threads * wpt);
}

}  // namespace saba_cu

namespace saba_cu {
template <class CT>
__device__ __forceinline__ void count_visit(CT* __restrict__ counts, uint32_t v, bool act) {
    if (act) atomicAdd(counts + v, CT(1));
}
}  // namespace saba_cu
