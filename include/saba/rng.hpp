// saba drop-in (B200 / sm_100a) — stateless selection primitives and seeds.
// API of the reference's saba/rng.hpp (HashSpec, selectors, Lcg64, SeedSet).
// The walk kernels on the GPU evaluate exactly these integer functions.
#pragma once

#include <algorithm>
#include <vector>

#include "saba/common.hpp"

namespace saba {

/// h(cur, l): two multiply / xor-shift-47 rounds over (cur << 32 | l), high word.
struct HashSpec {
    uint64_t multiplier = SABA_DEFAULT_HASH_MULTIPLIER;

    [[nodiscard]] uint32_t state(uint32_t vertex, uint32_t step) const noexcept {
        uint64_t h = ((uint64_t)vertex << 32) | step;
        for (int round = 0; round < 2; ++round) {
            h *= multiplier;
            h ^= h >> 47;
        }
        return uint32_t(h >> 32);
    }
};

inline constexpr uint64_t kHashRange = uint64_t(1) << 32;

/// Division-free Eq. (5): floor(raw * degree / 2^32).
inline constexpr uint32_t scaled_index(uint32_t raw, uint32_t degree) noexcept {
    return uint32_t((uint64_t(raw) * degree) >> 32);
}

inline uint32_t select_mod(uint32_t raw, uint32_t degree) {
    check_arg(degree != 0, "select_mod: degree must be >= 1");
    return raw % degree;
}
inline uint32_t select_xor_mod(uint32_t seed, uint32_t state, uint32_t degree) {
    check_arg(degree != 0, "select_xor_mod: degree must be >= 1");
    return (seed ^ state) % degree;
}
inline uint32_t select_scaled(uint32_t seed, uint32_t state, uint32_t degree) {
    check_arg(degree != 0, "select_scaled: degree must be >= 1");
    return scaled_index(seed ^ state, degree);
}

enum class SelectorKind { NaiveMod, XorMod, Scaled };

inline const char* to_string(SelectorKind k) noexcept {
    return k == SelectorKind::Scaled ? "scaled" : k == SelectorKind::XorMod ? "xor" : "naive";
}

/// 64-bit LCG baseline stream (high word per step). CPU-only: the GPU engine
/// implements the Bouquets hash path, not the LCG baselines.
struct Lcg64 {
    uint64_t state;
    explicit constexpr Lcg64(uint64_t seed) noexcept : state(mix64(seed)) {}
    constexpr uint32_t next() noexcept {
        state = 0x5851f42d4c957f2dull * state + 0x14057b7ef767814full;
        return uint32_t(state >> 32);
    }
};

enum class SeedOrdering { AsGenerated, Sorted };

struct SeedSet {
    std::vector<uint32_t> seeds;
    SeedOrdering ordering = SeedOrdering::AsGenerated;
    uint64_t master_seed = 0;
};

/// seed_i = counter_hash(master, i) >> 32; Sorted = the bouquet arrangement.
inline SeedSet gen_seeds(size_t count, uint64_t master_seed, SeedOrdering ordering) {
    check_arg(count > 0, "gen_seeds: count must be >= 1");
    SeedSet out{std::vector<uint32_t>(count), ordering, master_seed};
    uint64_t i = 0;
    for (uint32_t& s : out.seeds) s = uint32_t(counter_hash(master_seed, i++) >> 32);
    if (ordering == SeedOrdering::Sorted) std::sort(out.seeds.begin(), out.seeds.end());
    return out;
}

inline SeedSet gen_sorted_seeds(size_t count, uint64_t master_seed) {
    return gen_seeds(count, master_seed, SeedOrdering::Sorted);
}

}  // namespace saba
