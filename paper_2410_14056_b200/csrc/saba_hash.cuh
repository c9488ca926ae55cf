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

// hash_state split for the walk kernels, where every lane of a step shares
// l. With M = mult = (m_hi, m_lo) and x = cur << 32 | l:
//   x * M       = ((cur * m_lo) << 32) + l * M        (mod 2^64), so
//   x1_hi       = cur * m_lo + hi32(l * M),  x1_lo = lo32(l * M)
//   y = x1 ^ (x1 >> 47): only the low word changes: y_lo = x1_lo ^ (x1_hi >> 15)
//   the final x ^= x >> 47 never reaches the returned high word, so
//   h = hi32(y * M) = umulhi(y_lo, m_lo) + y_lo * m_hi + x1_hi * m_lo (mod 2^32).
// Six 32-bit operations per lane instead of two full 64-bit products; equal
// to hash_state bit for bit (tests/test_host.py checks the identity).
struct StepHash {
    uint32_t lm_lo, lm_hi, m_lo, m_hi;
};
SABA_HD StepHash step_hash(uint64_t mult, uint32_t step) {
    const uint64_t lm = static_cast<uint64_t>(step) * mult;
    return {static_cast<uint32_t>(lm), static_cast<uint32_t>(lm >> 32), static_cast<uint32_t>(mult),
            static_cast<uint32_t>(mult >> 32)};
}
SABA_HD uint32_t mulhi32(uint32_t a, uint32_t b) {
#if defined(__CUDA_ARCH__)
    return __umulhi(a, b);
#else
    return static_cast<uint32_t>((static_cast<uint64_t>(a) * b) >> 32);
#endif
}
SABA_HD uint32_t hash_state_fast(const StepHash& s, uint32_t vertex) {
    const uint32_t x1_hi = vertex * s.m_lo + s.lm_hi;
    const uint32_t y_lo = s.lm_lo ^ (x1_hi >> 15);
    return mulhi32(y_lo, s.m_lo) + y_lo * s.m_hi + x1_hi * s.m_lo;
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
