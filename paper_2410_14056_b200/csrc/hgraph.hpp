// Host CSR graph behind the saba_hgraph C handle (graph_host.cpp builds it on
// the CPU, graph_build.cu on the device) and the generator tables both share.
#pragma once
#include <cstdint>
#include <memory>
#include <utility>
#include <vector>

#include "saba_hash.cuh"

namespace saba_cu {
// resize() without value-initialisation: the CSR arrays are always fully
// written after sizing, and zero-filling ~1 GB on one thread (plus its page
// faults) cost more than building the whole graph on the device.
template <class T>
struct UninitAlloc : std::allocator<T> {
    template <class U>
    struct rebind {
        using other = UninitAlloc<U>;
    };
    UninitAlloc() = default;
    template <class U>
    UninitAlloc(const UninitAlloc<U>&) noexcept {}
    template <class U>
    void construct(U* p) noexcept {
        ::new (static_cast<void*>(p)) U;
    }
    template <class U, class... A>
    void construct(U* p, A&&... a) {
        ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
    }
};
using IdVec = std::vector<uint32_t, UninitAlloc<uint32_t>>;
}  // namespace saba_cu

struct saba_hgraph {
    uint32_t n = 0;
    uint64_t m = 0;
    saba_cu::IdVec off;  // n + 1 offsets (graph.hpp:242 layout)
    saba_cu::IdVec adj;  // 2m neighbour ids, ascending per slice
};

namespace saba_cu {

struct ChungLuTables {
    std::vector<double> prob;     // Vose alias table over the capped weights
    std::vector<uint32_t> alias;
    uint64_t samples = 0;         // edge samples = round(sum w / 2)
};
void chung_lu_tables(uint32_t n, double gamma, double mean_degree, double max_degree, uint64_t seed,
                     ChungLuTables& t);

// R-MAT quadrant thresholds on a 32-bit uniform (a, a+b, a+b+c)
struct RmatThresholds {
    uint64_t ta, tb, tc;
};
inline RmatThresholds rmat_thresholds(double a, double b, double c) {
    const double two32 = 4294967296.0;
    return {uint64_t(a * two32), uint64_t((a + b) * two32), uint64_t((a + b + c) * two32)};
}

constexpr uint64_t kRmatTag = 0x524d4154ull;    // "RMAT"
constexpr uint64_t kChungLuTag = 0x43484c32ull;  // endpoint stream

// Endpoints (u, v) of R-MAT sample i of stream s: one counter_hash per two
// levels, quadrant by 32-bit threshold, high bit first.
SABA_HD void rmat_sample(uint64_t s, uint64_t i, uint32_t scale, const RmatThresholds& t, uint32_t& u,
                         uint32_t& v) {
    u = 0;
    v = 0;
    const uint64_t si = counter_hash(s, i);
    for (uint32_t lvl = 0; lvl < scale; lvl += 2) {
        const uint64_t h = counter_hash(si, lvl);
        for (uint32_t q = 0; q < 2 && lvl + q < scale; ++q) {
            const uint64_t r = q ? (h & 0xffffffffu) : (h >> 32);
            const uint32_t bit = 1u << (scale - 1 - (lvl + q));
            if (r < t.ta) {
            } else if (r < t.tb) {
                v |= bit;
            } else if (r < t.tc) {
                u |= bit;
            } else {
                u |= bit;
                v |= bit;
            }
        }
    }
}

// Endpoint e (0/1) of Chung–Lu sample i of stream s through the alias table.
SABA_HD uint32_t chung_lu_end(uint64_t s, uint64_t i, int e, uint32_t n, const double* prob,
                              const uint32_t* alias) {
    const uint64_t h = counter_hash(s, 2 * i + uint64_t(e));
    const uint32_t col = scaled_index(uint32_t(h >> 32), n);
    const double coin = double(uint32_t(h)) * 0x1.0p-32;
    return coin < prob[col] ? col : alias[col];
}

}  // namespace saba_cu
