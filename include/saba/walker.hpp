// saba drop-in (B200 / sm_100a) — Bouquets walk engine.
// API of the reference's saba/walker.hpp. random_walk / random_bouquet and
// run_walk_campaign execute on the GPU (saba_cu_walk_paths,
// saba_cu_walk_campaign). Saba and Hash produce identical walks and share the
// kernels; the Naive / VectorMod LCG baselines have no GPU path and throw
// std::invalid_argument (there is no CPU fallback).
#pragma once

#include <bit>
#include <cmath>
#include <span>
#include <string>
#include <type_traits>
#include <vector>

#include "saba/graph.hpp"
#include "saba/rng.hpp"

namespace saba {

enum class WalkMode { Naive, VectorMod, Hash, Saba };

inline const char* to_string(WalkMode m) noexcept {
    static const char* const names[] = {"naive", "vector-mod", "hash", "saba"};
    return names[int(m)];
}

inline WalkMode parse_walk_mode(const std::string& s) {
    for (WalkMode m : {WalkMode::Naive, WalkMode::VectorMod, WalkMode::Hash, WalkMode::Saba})
        if (s == to_string(m)) return m;
    throw std::invalid_argument("unknown walk mode: " + s);
}

inline constexpr bool is_lane_mode(WalkMode m) noexcept { return m != WalkMode::Naive; }
inline constexpr uint32_t kMaxLanes = 64;

struct Walk {
    std::vector<uint32_t> vertices;
    uint64_t walk_id = 0;
    uint32_t seed = 0;
};

struct BranchingStats {
    uint32_t lanes = 0;
    std::vector<uint64_t> histogram;
    uint64_t samples = 0;
    double mean = 0.0;
    uint32_t p1 = 0, p10 = 0, p25 = 0;
    double mean_candidate_degree = 0.0;
};

/// Percentiles (ceil(q * total)-th smallest, 1-based) and mean of a
/// distinct-lanes histogram.
inline BranchingStats branching_stats(std::span<const uint64_t> histogram) {
    BranchingStats st;
    double weighted = 0.0;
    for (size_t c = 0; c < histogram.size(); ++c) {
        st.samples += histogram[c];
        weighted += double(c) * double(histogram[c]);
    }
    check_arg(st.samples > 0, "branching_stats: empty trace");
    auto pct = [&](double q) {
        const uint64_t want = std::max<uint64_t>(1, uint64_t(std::ceil(q * double(st.samples))));
        uint64_t seen = 0;
        for (size_t c = 0; c < histogram.size(); ++c)
            if ((seen += histogram[c]) >= want) return uint32_t(c);
        return uint32_t(histogram.size() - 1);
    };
    st.lanes = histogram.empty() ? 0 : uint32_t(histogram.size() - 1);
    st.histogram.assign(histogram.begin(), histogram.end());
    st.mean = weighted / double(st.samples);
    st.p1 = pct(0.01);
    st.p10 = pct(0.10);
    st.p25 = pct(0.25);
    return st;
}

inline BranchingStats branching_stats(std::span<const uint32_t> trace, uint32_t lanes) {
    check_arg(!trace.empty(), "branching_stats: empty trace");
    std::vector<uint64_t> h(size_t(lanes) + 1, 0);
    for (uint32_t c : trace) {
        check_arg(c >= 1 && c <= lanes, "branching_stats: count out of range");
        ++h[c];
    }
    return branching_stats(std::span<const uint64_t>(h));
}

namespace detail {
inline void require_walkable(const Graph& g, uint32_t start, uint32_t length) {
    check_arg(length >= 1, "walk length must be >= 1");
    check_arg(start < g.vertex_count(), "start vertex out of range");
    check_arg(length == 1 || g.degree(start) >= 1, "cannot walk from an isolated vertex");
}
inline void require_scaled(SelectorKind s) {
    check_arg(s == SelectorKind::Scaled,
              "selector not supported on GPU (the Bouquets engine implements the scaled hash)");
}
}  // namespace detail

/// One walk of `length` vertices from `start` (GPU).
inline Walk random_walk(const Graph& g, uint32_t start, uint32_t length, SelectorKind selector,
                        uint32_t seed, const HashSpec& hash = {}) {
    detail::require_walkable(g, start, length);
    detail::require_scaled(selector);
    Walk w;
    w.seed = seed;
    w.vertices.resize(length);
    detail::raise_on(saba_cu_walk_paths(g.device_handle(), &start, &seed, 1, length, hash.multiplier,
                                        w.vertices.data()),
                     "random_walk");
    return w;
}

/// `width` lockstep lanes from `start`, one per seed (GPU); each lane equals
/// random_walk with its seed.
inline std::vector<Walk> random_bouquet(const Graph& g, uint32_t start, uint32_t length,
                                        uint32_t width, const SeedSet& seeds, SelectorKind selector,
                                        const HashSpec& hash = {}) {
    check_arg(width >= 1 && width <= kMaxLanes, "bouquet width must be in [1, 64]");
    check_arg(seeds.seeds.size() >= width, "seed set smaller than bouquet width");
    detail::require_walkable(g, start, length);
    detail::require_scaled(selector);
    std::vector<uint32_t> starts(width, start), paths(size_t(width) * length);
    detail::raise_on(saba_cu_walk_paths(g.device_handle(), starts.data(), seeds.seeds.data(), width,
                                        length, hash.multiplier, paths.data()),
                     "random_bouquet");
    std::vector<Walk> out(width);
    for (uint32_t b = 0; b < width; ++b) {
        out[b].walk_id = b;
        out[b].seed = seeds.seeds[b];
        out[b].vertices.assign(paths.begin() + size_t(b) * length, paths.begin() + size_t(b + 1) * length);
    }
    return out;
}

/// Per-vertex visit counter (the campaign sink of the benchmarks).
struct VisitCountSink {
    struct Shard {
        std::vector<uint64_t> counts;
        void visit(uint64_t, uint32_t, uint32_t v) noexcept { ++counts[v]; }
    };
    std::vector<uint64_t> counts;
    explicit VisitCountSink(uint32_t n) : counts(n, 0) {}
    [[nodiscard]] Shard make_shard() const { return Shard{std::vector<uint64_t>(counts.size(), 0)}; }
    void absorb(Shard& sh) {
        for (size_t i = 0; i < counts.size(); ++i) counts[i] += sh.counts[i];
    }
};

template <class S>
concept CampaignSink = requires(S s, typename S::Shard sh, uint64_t id, uint32_t step, uint32_t v) {
    { s.make_shard() } -> std::convertible_to<typename S::Shard>;
    sh.visit(id, step, v);
    s.absorb(sh);
};

struct CampaignConfig {
    uint64_t walks_per_vertex = 2048;
    uint32_t length = 10;
    WalkMode mode = WalkMode::Saba;
    uint32_t lanes = 8;
    int threads = 0;  // GPUs (0 = all visible; detail::devices_for)
    uint64_t master_seed = 42;
    bool collect_stats = false;
    HashSpec hash{};
};

struct DistinctProxy {
    std::vector<uint64_t> per_step;
    uint64_t total = 0;
};

struct CampaignReport {
    double seconds = 0.0;
    uint64_t total_steps = 0;
    uint64_t total_events = 0;
    int threads_used = 1;
    bool has_stats = false;
    BranchingStats branching;
    DistinctProxy proxy;
};

namespace detail {
inline CampaignReport campaign_on_gpu(const Graph& g, const CampaignConfig& cfg, uint64_t total_walks,
                                      std::vector<uint64_t>& counts) {
    saba_cu_campaign_config c{};
    c.walks_per_vertex = cfg.walks_per_vertex;
    c.total_walks = total_walks;
    c.length = cfg.length;
    c.lanes = cfg.lanes;
    c.mode = int32_t(cfg.mode);
    c.threads = cfg.threads;
    c.master_seed = cfg.master_seed;
    c.hash_multiplier = cfg.hash.multiplier;
    c.shard_index = 0;
    c.shard_count = 1;
    std::vector<uint64_t> add(g.vertex_count());
    saba_cu_campaign_report r{};
    const std::vector<int> devices = detail::devices_for(cfg.threads);
    detail::raise_on(saba_cu_walk_campaign(g.device_group(devices), &c, add.data(), &r), "run_walk_campaign");
    for (size_t i = 0; i < add.size(); ++i) counts[i] += add[i];
    CampaignReport rep;
    rep.seconds = r.seconds;
    rep.total_steps = r.total_steps;
    rep.total_events = r.total_events;
    rep.threads_used = int(devices.size());
    if (cfg.collect_stats && cfg.length > 1) {  // the untimed stats pass (walker.hpp:471, 526-536)
        std::vector<uint64_t> hist(size_t(cfg.lanes) + 1), per_step(cfg.length - 1), tot(4);
        detail::raise_on(saba_cu_branching_stats(g.device_handle(), &c, hist.data(), per_step.data(),
                                                 tot.data()),
                         "branching statistics");
        rep.has_stats = true;
        rep.branching = branching_stats(std::span<const uint64_t>(hist));
        rep.branching.mean_candidate_degree = tot[2] ? double(tot[3]) / double(tot[2]) : 0.0;
        rep.proxy.per_step = std::move(per_step);
        rep.proxy.total = tot[0];
    }
    return rep;
}
}  // namespace detail

/// Exactly K walks of L vertices from every vertex, visit counts into the
/// sink. The GPU engine supports VisitCountSink.
template <CampaignSink Sink>
CampaignReport run_walk_campaign(const Graph& g, const CampaignConfig& cfg, Sink& sink) {
    static_assert(std::is_same_v<Sink, VisitCountSink>,
                  "the GPU campaign accumulates per-vertex visit counts (VisitCountSink)");
    return detail::campaign_on_gpu(g, cfg, 0, sink.counts);
}

/// Extension: `total_walks` walks from uniform-random starts.
inline CampaignReport run_walk_campaign_uniform(const Graph& g, const CampaignConfig& cfg,
                                                uint64_t total_walks, VisitCountSink& sink) {
    check_arg(total_walks >= 1, "total_walks must be >= 1");
    return detail::campaign_on_gpu(g, cfg, total_walks, sink.counts);
}

}  // namespace saba
