// saba drop-in (B200 / sm_100a) — TGT+ all-edges spanning centrality.
// API of the reference's saba/aesc.hpp. The truncation plan is computed by the
// library's exact host restatement; propagation, the two-way walk estimator
// and symmetrisation run on the GPU (saba_cu_aesc and friends).
#pragma once

#include <algorithm>
#include <cstdio>
#include <ostream>
#include <span>
#include <vector>

#include "saba/graph.hpp"
#include "saba/walker.hpp"

namespace saba {

struct AescConfig {
    double epsilon = 0.05;
    double delta = 0.05;
    uint32_t power_iterations = 30;
    uint32_t candidate_nodes = 0;  // accepted, unused (as in the reference)
    WalkMode mode = WalkMode::Saba;
    uint64_t master_seed = 42;
    int threads = 0;               // GPUs (0 = all visible; detail::devices_for)
    uint32_t lanes = 8;
    uint32_t max_truncation = 128;
    bool per_edge_tau = false;
    int64_t switch_depth_cap = -1;
    HashSpec hash{};
};

struct TruncationPlan {
    std::vector<uint32_t> tau;        // per edge id
    std::vector<uint32_t> tau_tilde;  // per source
    double lambda_hat = 0.0;
    bool clamped = false;
    uint32_t max_tau = 0;
};

struct LandingProbs {
    uint32_t source = 0;
    uint32_t depth = 0;
    std::vector<uint32_t> support;  // ascending
    std::vector<double> prob;

    [[nodiscard]] double prob_of(uint32_t v) const {
        const auto it = std::lower_bound(support.begin(), support.end(), v);
        return (it != support.end() && *it == v) ? prob[size_t(it - support.begin())] : 0.0;
    }
    [[nodiscard]] double sum() const {
        double s = 0.0;
        for (double p : prob) s += p;
        return s;
    }
};

struct WalkBudget {
    uint64_t n_walks = 0;
    uint64_t n_req = 0;
};

struct CentralityEstimate {
    std::vector<double> s_hat;  // per edge id
    std::vector<double> g_hat;  // per directed slot
    AescConfig config;
    TruncationPlan plan;
    bool bipartite = false;
    uint64_t total_walk_pairs = 0;
    uint64_t total_walk_steps = 0;
    double seconds = 0.0;
};

inline uint64_t walk_budget(uint32_t tau_effective, double epsilon, double delta, uint32_t degree,
                            uint64_t edge_count) {
    uint64_t out = 0;
    detail::raise_on(saba_cu_walk_budget(tau_effective, epsilon, delta, degree, edge_count, &out),
                     "walk_budget");
    return out;
}

inline TruncationPlan truncated_lengths(const Graph& g, double epsilon, uint32_t power_iterations,
                                        uint32_t max_truncation = 128, bool per_edge = false) {
    TruncationPlan p;
    p.tau.resize(g.edge_count());
    int clamped = 0;
    detail::raise_on(saba_cu_truncated_lengths(g.device_handle(), epsilon, power_iterations,
                                               max_truncation, per_edge ? 1 : 0, p.tau.data(),
                                               &p.lambda_hat, &clamped),
                     "truncated_lengths");
    p.clamped = clamped != 0;
    p.max_tau = p.tau.empty() ? 0 : *std::max_element(p.tau.begin(), p.tau.end());
    return p;
}

inline std::pair<LandingProbs, uint32_t> propagate_landing_probabilities(
    const Graph& g, uint32_t source, const TruncationPlan& plan, double epsilon, double delta,
    int64_t switch_depth_cap = -1) {
    std::vector<double> dense(g.vertex_count());
    uint32_t depth = 0;
    detail::raise_on(saba_cu_propagate(g.device_handle(), source, plan.tau.data(), epsilon, delta,
                                       switch_depth_cap, dense.data(), &depth),
                     "propagate_landing_probabilities");
    LandingProbs lp;
    lp.source = source;
    lp.depth = depth;
    for (uint32_t v = 0; v < g.vertex_count(); ++v)
        if (dense[v] != 0.0) {
            lp.support.push_back(v);
            lp.prob.push_back(dense[v]);
        }
    return {std::move(lp), depth};
}

inline double estimate_edge(const Graph& g, uint32_t v_i, uint32_t v_j, const LandingProbs& landing,
                            uint32_t tau_eff, uint64_t n_req, WalkMode mode, uint64_t edge_seed,
                            uint32_t lanes = 8, const HashSpec& hash = {}) {
    check_arg(tau_eff >= 1, "estimate_edge: tau_eff must be >= 1");
    check_arg(n_req >= 1, "estimate_edge: n_req must be >= 1");
    std::vector<double> dense(g.vertex_count(), 0.0);
    for (size_t i = 0; i < landing.support.size(); ++i) dense[landing.support[i]] = landing.prob[i];
    double out = 0.0;
    detail::raise_on(saba_cu_estimate_edge(g.device_handle(), v_i, v_j, dense.data(), tau_eff, n_req,
                                           int(mode), edge_seed, lanes, hash.multiplier, &out),
                     "estimate_edge");
    return out;
}

namespace detail {
inline CentralityEstimate run_aesc(const Graph& g, const AescConfig& cfg,
                                   const std::vector<uint32_t>* sources) {
    saba_cu_aesc_config c{};
    c.epsilon = cfg.epsilon;
    c.delta = cfg.delta;
    c.power_iterations = cfg.power_iterations;
    c.candidate_nodes = cfg.candidate_nodes;
    c.mode = int32_t(cfg.mode);
    c.threads = cfg.threads;
    c.master_seed = cfg.master_seed;
    c.lanes = cfg.lanes;
    c.max_truncation = cfg.max_truncation;
    c.per_edge_tau = cfg.per_edge_tau ? 1 : 0;
    c.switch_depth_cap = cfg.switch_depth_cap;
    c.hash_multiplier = cfg.hash.multiplier;
    CentralityEstimate est;
    est.config = cfg;
    est.g_hat.resize(2 * g.edge_count());
    if (!sources) est.s_hat.resize(g.edge_count());
    est.plan.tau.resize(g.edge_count());
    est.plan.tau_tilde.resize(g.vertex_count());
    saba_cu_aesc_report r{};
    detail::raise_on(saba_cu_aesc(g.device_group(detail::devices_for(cfg.threads)), &c, sources ? sources->data() : nullptr,
                                  sources ? sources->size() : 0, 0, 1, est.g_hat.data(),
                                  sources ? nullptr : est.s_hat.data(), est.plan.tau.data(),
                                  est.plan.tau_tilde.data(), &r),
                     "aesc");
    est.plan.lambda_hat = r.lambda_hat;
    est.plan.clamped = r.clamped != 0;
    est.plan.max_tau = r.max_tau;
    est.bipartite = r.bipartite != 0;
    est.total_walk_pairs = r.total_walk_pairs;
    est.total_walk_steps = r.total_walk_steps;
    est.seconds = r.seconds;
    return est;
}
}  // namespace detail

/// All-edges spanning centrality with |s - SC| <= epsilon w.p. >= 1 - delta;
/// deterministic for a fixed configuration (and identical for any GPU count).
inline CentralityEstimate aesc(const Graph& g, const AescConfig& cfg) {
    return detail::run_aesc(g, cfg, nullptr);
}

/// Extension: the estimator restricted to `sources` (SURVEY §8d subset protocol).
inline CentralityEstimate aesc_sources(const Graph& g, const AescConfig& cfg,
                                       const std::vector<uint32_t>& sources) {
    return detail::run_aesc(g, cfg, &sources);
}

/// `u<TAB>v<TAB>%.6g` per edge, original labels with u < v, ascending.
inline void write_centrality_tsv(std::ostream& out, const Graph& g, std::span<const double> values) {
    check_arg(values.size() == g.edge_count(), "write_centrality_tsv: value count != edge count");
    struct Row {
        uint64_t u, v;
        double x;
    };
    std::vector<Row> rows;
    rows.reserve(values.size());
    for (uint32_t e = 0; e < values.size(); ++e) {
        const auto [a, b] = g.edge(e);
        const uint64_t x = g.original_id(a), y = g.original_id(b);
        rows.push_back({std::min(x, y), std::max(x, y), values[e]});
    }
    std::sort(rows.begin(), rows.end(), [](const Row& p, const Row& q) {
        return p.u != q.u ? p.u < q.u : p.v < q.v;
    });
    char text[64];
    for (const Row& r : rows) {
        std::snprintf(text, sizeof(text), "%.6g", r.x);
        out << r.u << '\t' << r.v << '\t' << text << '\n';
    }
}

}  // namespace saba
