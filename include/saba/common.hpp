// saba drop-in (B200 / sm_100a) — shared definitions.
//
// Header-compatible replacement for the reference's saba/common.hpp: the same
// names in namespace saba, with the compute entry points of the other headers
// routed to libsaba_cuda.so through the C ABI in saba_cuda.h. Link with
// -lsaba_cuda (paper_2410_14056_b200/libsaba_cuda.so).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <algorithm>
#include <vector>
#include <cstdlib>

#include "saba_cuda.h"

namespace saba {

using std::size_t;
using std::uint32_t;
using std::uint64_t;

/// Argument / precondition failures surface as std::invalid_argument and
/// data / runtime failures as std::runtime_error, exactly as the reference's
/// check_arg / check_data split (reference common.hpp:13-21).
inline void check_arg(bool ok, const char* msg) {
    if (!ok) throw std::invalid_argument(msg);
}
inline void check_data(bool ok, const std::string& msg) {
    if (!ok) throw std::runtime_error(msg);
}

namespace detail {
/// Convert a C-ABI status into the reference's exception types.
inline void raise_on(int status, const char* what) {
    if (status == SABA_OK) return;
    std::string msg = saba_cu_last_error();
    if (msg.empty()) msg = what;
    if (status == SABA_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

/// The devices behind a config's `threads` (walker.hpp:372, aesc.hpp:47): the
/// reference's thread count becomes a GPU count, 0 = every visible device, as
/// 0 = every hardware thread there. SABA_DEVICES="0,0,1" overrides the list
/// (repeats are logical shards on one GPU). Results do not depend on it.
inline std::vector<int> devices_for(int threads) {
    std::vector<int> d;
    if (const char* e = std::getenv("SABA_DEVICES"); e && *e) {
        for (const char* p = e; *p;) {
            char* end = nullptr;
            const long v = std::strtol(p, &end, 10);
            if (end == p) break;
            d.push_back(int(v));
            p = *end == ',' ? end + 1 : end;
        }
        if (!d.empty()) return d;
    }
    const int count = std::max(1, saba_cu_device_count());
    const int k = threads <= 0 ? count : std::min(threads, count);
    for (int i = 0; i < k; ++i) d.push_back(i);
    return d;
}
}  // namespace detail

// The stream-word primitives every walk seed is derived from (splitmix64
// finalizer, counter stream, child stream). Pure integer functions shared with
// the device code (paper_2410_14056_b200/csrc/saba_hash.cuh).
inline constexpr uint64_t mix64(uint64_t z) noexcept {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
inline constexpr uint64_t counter_hash(uint64_t master, uint64_t index) noexcept {
    return mix64(master + 0x9e3779b97f4a7c15ull * (index + 1));
}
inline constexpr uint64_t substream(uint64_t master, uint64_t tag) noexcept {
    return mix64(master ^ mix64(0x632be59bd9b4e019ull + tag));
}

}  // namespace saba
