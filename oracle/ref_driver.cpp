// TEST INFRASTRUCTURE ONLY — thin extern "C" shim over the UNMODIFIED
// reference headers (/root/reference/proj/include/saba/*.hpp, compiled in
// place by oracle/Makefile into oracle/_ref/libsaba_ref.so). It is the golden
// source that pins oracle/saba_oracle.c and the CPU baseline ("kind":
// "reference") of bench.py. Nothing here is product code; no reference source
// is copied — every computation below is a call into the reference.
#include "saba/aesc.hpp"
#include "saba/gen.hpp"
#include "saba/stream.hpp"

#include <sstream>
#include "saba/graph.hpp"
#include "saba/walker.hpp"

#include <chrono>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#define REF_API extern "C" __attribute__((visibility("default")))

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

saba::Graph* as_graph(void* h) { return static_cast<saba::Graph*>(h); }
}  // namespace

REF_API const char* ref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- graphs

// Graph::from_edges (graph.hpp:86-105) on explicit pairs.
REF_API int ref_graph_from_edges(uint32_t n_hint, const uint32_t* pairs, uint64_t count, void** out) {
    return guarded([&] {
        std::vector<std::pair<uint32_t, uint32_t>> p(count);
        for (uint64_t i = 0; i < count; ++i) p[i] = {pairs[2 * i], pairs[2 * i + 1]};
        *out = new saba::Graph(saba::Graph::from_edges(n_hint, std::move(p)));
    });
}

// Rebuild a reference Graph from a CSR by feeding its (u<v) edges back
// through Graph::from_edges.
REF_API int ref_graph_from_csr(uint32_t n, const uint32_t* off, const uint32_t* adj, void** out) {
    return guarded([&] {
        std::vector<std::pair<uint32_t, uint32_t>> p;
        for (uint32_t u = 0; u < n; ++u)
            for (uint32_t s = off[u]; s < off[u + 1]; ++s)
                if (adj[s] > u) p.emplace_back(u, adj[s]);
        *out = new saba::Graph(saba::Graph::from_edges(n, std::move(p)));
    });
}

REF_API int ref_gen_scale_free(uint32_t n, uint32_t attach, uint64_t seed, void** out) {
    return guarded([&] { *out = new saba::Graph(saba::make_scale_free(n, attach, seed)); });
}

REF_API int ref_gen_random_connected(uint32_t n, uint32_t extra, uint64_t seed, void** out) {
    return guarded([&] { *out = new saba::Graph(saba::make_random_connected(n, extra, seed)); });
}

REF_API void ref_graph_free(void* g) { delete as_graph(g); }
REF_API uint32_t ref_graph_n(void* g) { return as_graph(g)->vertex_count(); }
REF_API uint64_t ref_graph_m(void* g) { return as_graph(g)->edge_count(); }

REF_API void ref_graph_csr(void* h, uint32_t* off, uint32_t* adj, uint32_t* slot_edge) {
    const saba::Graph& g = *as_graph(h);
    std::memcpy(off, g.offsets_data(), sizeof(uint32_t) * (g.vertex_count() + 1));
    std::memcpy(adj, g.adjacency_data(), sizeof(uint32_t) * 2 * g.edge_count());
    if (slot_edge)
        for (uint64_t s = 0; s < 2 * g.edge_count(); ++s) slot_edge[s] = g.slot_edge(uint32_t(s));
}

REF_API void ref_graph_edges(void* h, uint32_t* uv) {
    const saba::Graph& g = *as_graph(h);
    for (uint32_t e = 0; e < g.edge_count(); ++e) {
        auto [u, v] = g.edge(e);
        uv[2 * e] = u;
        uv[2 * e + 1] = v;
    }
}

// ----------------------------------------------------------------- walks

// random_walk (walker.hpp:283-302), Scaled selector.
REF_API int ref_random_walk(void* h, uint32_t start, uint32_t length, uint32_t seed, uint64_t mult,
                            uint32_t* path) {
    return guarded([&] {
        saba::HashSpec hs{mult};
        const saba::Walk w =
            saba::random_walk(*as_graph(h), start, length, saba::SelectorKind::Scaled, seed, hs);
        std::memcpy(path, w.vertices.data(), sizeof(uint32_t) * w.vertices.size());
    });
}

// random_bouquet (walker.hpp:306-338), Scaled selector, sorted seeds from
// gen_sorted_seeds(width, master) (rng.hpp:119-123).
REF_API int ref_random_bouquet(void* h, uint32_t start, uint32_t length, uint32_t width,
                               uint64_t master, uint64_t mult, uint32_t* seeds_out,
                               uint32_t* paths) {
    return guarded([&] {
        saba::HashSpec hs{mult};
        const saba::SeedSet seeds = saba::gen_sorted_seeds(width, master);
        const auto walks = saba::random_bouquet(*as_graph(h), start, length, width, seeds,
                                                saba::SelectorKind::Scaled, hs);
        for (uint32_t b = 0; b < width; ++b) {
            seeds_out[b] = walks[b].seed;
            std::memcpy(paths + uint64_t(b) * length, walks[b].vertices.data(),
                        sizeof(uint32_t) * length);
        }
    });
}

// run_walk_campaign (walker.hpp:456-538) with the VisitCountSink.
// mode: 0 naive, 1 vector-mod, 2 hash, 3 saba.
REF_API int ref_campaign(void* h, uint64_t K, uint32_t L, int mode, uint32_t lanes, int threads,
                         uint64_t master, uint64_t mult, uint64_t* counts, double* seconds,
                         uint64_t* total_steps) {
    return guarded([&] {
        const saba::Graph& g = *as_graph(h);
        saba::CampaignConfig cfg;
        cfg.walks_per_vertex = K;
        cfg.length = L;
        cfg.mode = static_cast<saba::WalkMode>(mode);
        cfg.lanes = lanes;
        cfg.threads = threads;
        cfg.master_seed = master;
        cfg.hash = saba::HashSpec{mult};
        saba::VisitCountSink sink(g.vertex_count());
        const saba::CampaignReport rep = saba::run_walk_campaign(g, cfg, sink);
        std::memcpy(counts, sink.counts.data(), sizeof(uint64_t) * g.vertex_count());
        if (seconds) *seconds = rep.seconds;
        if (total_steps) *total_steps = rep.total_steps;
    });
}

// run_walk_campaign with collect_stats = true (walker.hpp:470-536): the
// reference's BranchCollector output. hist[lanes+1], per_step[L-1],
// out4 = {proxy.total, branching.samples, 0, 0}, mean_deg = mean_candidate_degree.
REF_API int ref_campaign_stats(void* h, uint64_t K, uint32_t L, int mode, uint32_t lanes,
                               int threads, uint64_t master, uint64_t mult, uint64_t* hist,
                               uint64_t* per_step, uint64_t* out4, double* mean_deg,
                               double* mean) {
    return guarded([&] {
        const saba::Graph& g = *as_graph(h);
        saba::CampaignConfig cfg;
        cfg.walks_per_vertex = K;
        cfg.length = L;
        cfg.mode = static_cast<saba::WalkMode>(mode);
        cfg.lanes = lanes;
        cfg.threads = threads;
        cfg.master_seed = master;
        cfg.collect_stats = true;
        cfg.hash = saba::HashSpec{mult};
        saba::VisitCountSink sink(g.vertex_count());
        const saba::CampaignReport rep = saba::run_walk_campaign(g, cfg, sink);
        saba::check_data(rep.has_stats, "no stats collected");
        std::memcpy(hist, rep.branching.histogram.data(), sizeof(uint64_t) * (lanes + 1));
        std::memcpy(per_step, rep.proxy.per_step.data(), sizeof(uint64_t) * (L - 1));
        out4[0] = rep.proxy.total;
        out4[1] = rep.branching.samples;
        out4[2] = out4[3] = 0;
        *mean_deg = rep.branching.mean_candidate_degree;
        *mean = rep.branching.mean;
    });
}

// Uniform-random-start campaign: K_v walks of v are the
// reference's own campaign_vertex_scaled<Sorted>(g, v, K_v, ...) with
// vseed = substream(master, v), driven by the same OpenMP schedule and
// shard merge as run_walk_campaign (walker.hpp:473-519). If k_per_vertex is
// NULL the K_v are derived from (W, master). `vertex_stride`/`vertex_phase`
// restrict the run to v ≡ phase (mod stride) — a bounded CPU sample.
REF_API int ref_campaign_kv(void* h, const uint64_t* k_per_vertex, uint64_t W, uint32_t L,
                            int sorted, uint32_t lanes, int threads, uint64_t master, uint64_t mult,
                            uint32_t vertex_stride, uint32_t vertex_phase, uint64_t* counts,
                            double* seconds, uint64_t* total_steps) {
    return guarded([&] {
        const saba::Graph& g = *as_graph(h);
        const uint32_t n = g.vertex_count();
        std::vector<uint64_t> kv(n, 0);
        if (k_per_vertex) {
            std::memcpy(kv.data(), k_per_vertex, sizeof(uint64_t) * n);
        } else {
            const uint64_t s = saba::substream(master, 0x5354415254ull);
            for (uint64_t w = 0; w < W; ++w)
                ++kv[saba::scaled_index(uint32_t(saba::counter_hash(s, w) >> 32), n)];
        }
        const int nt = saba::resolve_threads(threads);
        saba::VisitCountSink sink(n);
        std::vector<saba::VisitCountSink::Shard> shards;
        for (int t = 0; t < nt; ++t) shards.push_back(sink.make_shard());
        const saba::HashSpec hs{mult};
        if (vertex_stride == 0) vertex_stride = 1;
        uint64_t steps = 0;
        const auto t0 = std::chrono::steady_clock::now();
#pragma omp parallel num_threads(nt) reduction(+ : steps)
        {
#ifdef _OPENMP
            const int rank = omp_get_thread_num();
#else
            const int rank = 0;
#endif
            std::vector<uint64_t> keys;
#pragma omp for schedule(dynamic, 4)
            for (int64_t vi = vertex_phase; vi < int64_t(n); vi += vertex_stride) {
                const uint32_t v = uint32_t(vi);
                if (kv[v] == 0) continue;
                const uint64_t vseed = saba::substream(master, v);
                if (sorted)
                    saba::detail::campaign_vertex_scaled<true>(g, v, kv[v], L, lanes, vseed, hs,
                                                               keys, shards[rank], nullptr);
                else
                    saba::detail::campaign_vertex_scaled<false>(g, v, kv[v], L, lanes, vseed, hs,
                                                                keys, shards[rank], nullptr);
                steps += kv[v] * uint64_t(L - 1);
            }
        }
        const auto t1 = std::chrono::steady_clock::now();
        for (int t = 0; t < nt; ++t) sink.absorb(shards[t]);
        std::memcpy(counts, sink.counts.data(), sizeof(uint64_t) * n);
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        if (total_steps) *total_steps = steps;
    });
}

REF_API int ref_max_threads() { return saba::resolve_threads(0); }

// ------------------------------------------------------------------ AESC

REF_API int ref_walk_budget(uint32_t tau_eff, double eps, double delta, uint32_t degree,
                            uint64_t m, uint64_t* out) {
    return guarded([&] { *out = saba::walk_budget(tau_eff, eps, delta, degree, m); });
}

// truncated_lengths (aesc.hpp:210-248)
REF_API int ref_truncated_lengths(void* h, double eps, uint32_t omega, uint32_t tau_max,
                                  int per_edge, uint32_t* tau, double* lambda_hat, int* clamped) {
    return guarded([&] {
        const saba::TruncationPlan p =
            saba::truncated_lengths(*as_graph(h), eps, omega, tau_max, per_edge != 0);
        std::memcpy(tau, p.tau.data(), sizeof(uint32_t) * p.tau.size());
        *lambda_hat = p.lambda_hat;
        *clamped = p.clamped ? 1 : 0;
    });
}

// propagate_landing_probabilities (aesc.hpp:406-422) -> dense prob[n].
REF_API int ref_propagate(void* h, uint32_t source, const uint32_t* tau, double eps, double delta,
                          int64_t cap, double* prob, uint32_t* depth) {
    return guarded([&] {
        const saba::Graph& g = *as_graph(h);
        saba::TruncationPlan plan;
        plan.tau.assign(tau, tau + g.edge_count());
        auto [lp, tt] = saba::propagate_landing_probabilities(g, source, plan, eps, delta, cap);
        std::memset(prob, 0, sizeof(double) * g.vertex_count());
        for (size_t i = 0; i < lp.support.size(); ++i) prob[lp.support[i]] = lp.prob[i];
        *depth = tt;
    });
}

// estimate_edge (aesc.hpp:533-553) with a dense landing vector.
REF_API int ref_estimate_edge(void* h, uint32_t vi, uint32_t vj, const double* prob_dense,
                              uint32_t depth, uint32_t tau_eff, uint64_t n_req, int mode,
                              uint64_t edge_seed, uint32_t lanes, uint64_t mult, double* out) {
    return guarded([&] {
        const saba::Graph& g = *as_graph(h);
        saba::LandingProbs lp;
        lp.source = vi;
        lp.depth = depth;
        for (uint32_t v = 0; v < g.vertex_count(); ++v)
            if (prob_dense[v] != 0.0) {
                lp.support.push_back(v);
                lp.prob.push_back(prob_dense[v]);
            }
        *out = saba::estimate_edge(g, vi, vj, lp, tau_eff, n_req, static_cast<saba::WalkMode>(mode),
                                   edge_seed, lanes, saba::HashSpec{mult});
    });
}

struct RefAescConfig {
    double epsilon, delta;
    uint32_t power_iterations;
    uint64_t master_seed;
    uint32_t max_truncation;
    int per_edge_tau;
    int64_t switch_depth_cap;
    uint64_t hash_multiplier;
    int threads;
    int mode;
    uint32_t lanes;
};

static saba::AescConfig to_cfg(const RefAescConfig* c) {
    saba::AescConfig cfg;
    cfg.epsilon = c->epsilon;
    cfg.delta = c->delta;
    cfg.power_iterations = c->power_iterations;
    cfg.master_seed = c->master_seed;
    cfg.max_truncation = c->max_truncation;
    cfg.per_edge_tau = c->per_edge_tau != 0;
    cfg.switch_depth_cap = c->switch_depth_cap;
    cfg.hash = saba::HashSpec{c->hash_multiplier};
    cfg.threads = c->threads;
    cfg.mode = static_cast<saba::WalkMode>(c->mode);
    cfg.lanes = c->lanes;
    return cfg;
}

// Full aesc() (aesc.hpp:636-708).
REF_API int ref_aesc(void* h, const RefAescConfig* c, double* g_hat, double* s_hat, uint32_t* tau,
                     uint32_t* tau_tilde, double* lambda_hat, uint64_t* pairs, uint64_t* steps,
                     double* seconds) {
    return guarded([&] {
        const saba::Graph& g = *as_graph(h);
        const auto t0 = std::chrono::steady_clock::now();
        const saba::CentralityEstimate est = saba::aesc(g, to_cfg(c));
        const auto t1 = std::chrono::steady_clock::now();
        std::memcpy(g_hat, est.g_hat.data(), sizeof(double) * est.g_hat.size());
        if (s_hat) std::memcpy(s_hat, est.s_hat.data(), sizeof(double) * est.s_hat.size());
        std::memcpy(tau, est.plan.tau.data(), sizeof(uint32_t) * est.plan.tau.size());
        std::memcpy(tau_tilde, est.plan.tau_tilde.data(), sizeof(uint32_t) * g.vertex_count());
        *lambda_hat = est.plan.lambda_hat;
        *pairs = est.total_walk_pairs;
        *steps = est.total_walk_steps;
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    });
}

// aesc() restricted to a source subset: the same setup as aesc.hpp:644-657,
// then the reference's detail::aesc_source over `sources` under OpenMP
// dynamic,1 (SURVEY §8d subset protocol). Slots of other sources stay 0.
// *seconds covers the per-source loop only; *plan_seconds the setup.
REF_API int ref_aesc_sources(void* h, const RefAescConfig* c, const uint32_t* sources,
                             uint64_t count, double* g_hat, uint32_t* tau, uint32_t* tau_tilde,
                             double* lambda_hat, uint64_t* pairs, uint64_t* steps, double* seconds,
                             double* plan_seconds) {
    return guarded([&] {
        const saba::Graph& g = *as_graph(h);
        const saba::AescConfig cfg = to_cfg(c);
        const uint32_t n = g.vertex_count();
        const auto m = static_cast<uint32_t>(g.edge_count());
        const auto p0 = std::chrono::steady_clock::now();
        saba::TruncationPlan plan = saba::truncated_lengths(
            g, cfg.epsilon / 2.0, cfg.power_iterations, cfg.max_truncation, cfg.per_edge_tau);
        plan.tau_tilde.assign(n, 0);
        const bool bip = saba::bipartition(g).first;
        std::vector<double> gh(2 * size_t(m), 0.0);
        std::vector<double> inv_deg(n);
        for (uint32_t v = 0; v < n; ++v) inv_deg[v] = 1.0 / double(g.degree(v));
        const double bip_init = bip ? 1.0 / (2.0 * double(m)) : 0.0;
        const int nt = saba::resolve_threads(cfg.threads);
        std::vector<uint64_t> pt(nt, 0), st(nt, 0);
        std::exception_ptr failure;
        const auto t0 = std::chrono::steady_clock::now();
#pragma omp parallel num_threads(nt)
        {
#ifdef _OPENMP
            const int rank = omp_get_thread_num();
#else
            const int rank = 0;
#endif
            saba::detail::AescWorkspace ws;
#pragma omp for schedule(dynamic, 1)
            for (int64_t i = 0; i < int64_t(count); ++i) {
                if (failure) continue;
                try {
                    saba::detail::aesc_source(g, cfg, plan, inv_deg, bip_init, sources[i], ws,
                                              gh.data(), plan.tau_tilde.data(), pt[rank], st[rank]);
                } catch (...) {
#pragma omp critical(ref_aesc_failure)
                    if (!failure) failure = std::current_exception();
                }
            }
        }
        const auto t1 = std::chrono::steady_clock::now();
        if (failure) std::rethrow_exception(failure);
        std::memcpy(g_hat, gh.data(), sizeof(double) * gh.size());
        std::memcpy(tau, plan.tau.data(), sizeof(uint32_t) * m);
        std::memcpy(tau_tilde, plan.tau_tilde.data(), sizeof(uint32_t) * n);
        *lambda_hat = plan.lambda_hat;
        *pairs = 0;
        *steps = 0;
        for (int t = 0; t < nt; ++t) {
            *pairs += pt[t];
            *steps += st[t];
        }
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        if (plan_seconds) *plan_seconds = std::chrono::duration<double>(t0 - p0).count();
    });
}

// rng_stream (stream.hpp:29-83): raw little-endian pre-selection words.
// selector: 0 naive, 1 xor, 2 scaled. Returns the number of words in *nwords.
REF_API int ref_rng_stream(void* h, const uint32_t* starts, uint32_t nstarts, uint64_t K, uint32_t L,
                           int selector, uint64_t master, uint64_t mult, uint32_t* words_out,
                           uint64_t* nwords) {
    return guarded([&] {
        saba::StreamSpec spec;
        spec.starts.assign(starts, starts + nstarts);
        spec.walks_per_vertex = K;
        spec.length = L;
        spec.selector = static_cast<saba::SelectorKind>(selector);
        spec.master_seed = master;
        spec.hash = saba::HashSpec{mult};
        std::ostringstream out;
        *nwords = saba::rng_stream(*as_graph(h), spec, out);
        const std::string bytes = out.str();
        std::memcpy(words_out, bytes.data(), bytes.size());
    });
}
