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
__device__ __forceinline__ uint64_t ldg_na_u64(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint32_t ldg_na_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

// Neighbour id at directed slot s. Packed: 3 x 21-bit fields per uint64.
template <bool PACKED>
__device__ __forceinline__ uint32_t adj_at(const uint32_t* __restrict__ adj,
                                           const uint64_t* __restrict__ packed, uint32_t s) {
    if constexpr (PACKED) {
        const uint32_t w = __umulhi(s, 0xAAAAAAABu) >> 1;  // s / 3 for s < 2^32
        const uint32_t r = s - 3 * w;
        return uint32_t(ldg_na_u64(packed + w) >> (21 * r)) & 0x1FFFFFu;
    } else {
        return ldg_na_u32(adj + s);
    }
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

}  // namespace saba_cu

namespace saba_cu {
template <class CT>
__device__ __forceinline__ void count_visit(CT* __restrict__ counts, uint32_t v, bool act) {
    if (act) atomicAdd(counts + v, CT(1));
}
}  // namespace saba_cu
