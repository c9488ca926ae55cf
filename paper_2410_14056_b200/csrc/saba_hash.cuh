// Stateless selection primitives shared by host and device code.
// These are the integer definitions the whole path is bit-exact against:
//   mix64 / counter_hash / substream   common.hpp:24-41
//   HashSpec::state h(cur, l)          rng.hpp:20-31
//   scaled_index (Eq. 5, h_max=2^32)   rng.hpp:61-63
#pragma once
#include <cstdint>

#if defined(__CUDACC__)
#define SABA_HD __host__ __device__ __forceinline__
#else
#define SABA_HD inline
#endif

namespace saba_cu {

SABA_HD uint64_t mix64(uint64_t x) {
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

SABA_HD uint64_t counter_hash(uint64_t master, uint64_t index) {
    return mix64(master + (index + 1) * 0x9e3779b97f4a7c15ull);
}

SABA_HD uint64_t substream(uint64_t master, uint64_t tag) {
    return mix64(master ^ mix64(tag + 0x632be59bd9b4e019ull));
}

// h(cur, l) = high word of two multiply/xor-shift rounds over (cur << 32 | l).
SABA_HD uint32_t hash_state(uint64_t mult, uint32_t vertex, uint32_t step) {
    uint64_t x = (static_cast<uint64_t>(vertex) << 32) | step;
    x *= mult;
    x ^= x >> 47;
    x *= mult;
    x ^= x >> 47;
    return static_cast<uint32_t>(x >> 32);
}

SABA_HD uint32_t scaled_index(uint32_t raw, uint32_t degree) {
#if defined(__CUDA_ARCH__)
    return __umulhi(raw, degree);
#else
    return static_cast<uint32_t>((static_cast<uint64_t>(raw) * degree) >> 32);
#endif
}

// Walk seed of a campaign walk: counter_hash(vseed, k) >> 32 (walker.hpp:438).
SABA_HD uint32_t walk_seed(uint64_t stream, uint64_t k) {
    return static_cast<uint32_t>(counter_hash(stream, k) >> 32);
}

constexpr uint64_t kStartTag = 0x5354415254ull;  // "START": uniform-start stream
constexpr uint64_t kAescTag = 0x41455343ull;     // "AESC" (aesc.hpp:603)

}  // namespace saba_cu
