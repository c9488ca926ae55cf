// saba drop-in (B200 / sm_100a) — raw selector-word export (Dieharder).
// API of the reference's saba/stream.hpp; the words are produced on the GPU
// (saba_cu_rng_stream). The NaiveMod (LCG) selector has no GPU path.
#pragma once

#include <ostream>
#include <vector>

#include "saba/walker.hpp"

namespace saba {

struct StreamSpec {
    std::vector<uint32_t> starts;
    uint64_t walks_per_vertex = 1;
    uint32_t length = 2;
    SelectorKind selector = SelectorKind::Scaled;
    uint64_t master_seed = 42;
    HashSpec hash{};
};

/// Little-endian 32-bit words seed ^ h(cur, l) of every step, K walks per
/// start, step-major within a start's block. Returns the number of words.
inline uint64_t rng_stream(const Graph& g, const StreamSpec& spec, std::ostream& out) {
    uint64_t nwords = 0;
    std::vector<uint32_t> words(spec.starts.size() * spec.walks_per_vertex *
                                (spec.length > 1 ? spec.length - 1 : 0));
    detail::raise_on(saba_cu_rng_stream(g.device_handle(), spec.starts.data(),
                                        uint32_t(spec.starts.size()), spec.walks_per_vertex,
                                        spec.length, int(spec.selector), spec.master_seed,
                                        spec.hash.multiplier, words.empty() ? nullptr : words.data(),
                                        &nwords),
                     "rng_stream");
    for (uint64_t i = 0; i < nwords; ++i) {
        const uint32_t w = words[i];
        const char b[4] = {char(w & 0xff), char((w >> 8) & 0xff), char((w >> 16) & 0xff), char(w >> 24)};
        out.write(b, 4);
    }
    check_data(out.good(), "rng_stream: sink write failure");
    return nwords;
}

}  // namespace saba
