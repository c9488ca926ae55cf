// Drop-in check of the C++ surface (include/saba/*.hpp) against the
// reference's own test expectations (proj/tests/test_*.cpp). Host-only
// checks always run; GPU checks run when a CUDA device is present.
//   g++ -std=c++20 -I include tests/cpp/dropin_test.cpp -L paper_2410_14056_b200 -lsaba_cuda
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <sstream>
#include <stdexcept>

#include "saba/aesc.hpp"
#include "saba/walker.hpp"

static int failures = 0;
#define CHECK(cond)                                                          \
    do {                                                                     \
        if (!(cond)) {                                                       \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            ++failures;                                                      \
        }                                                                    \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                 \
    do {                                            \
        bool thrown_ = false;                       \
        try {                                       \
            (void)(expr);                           \
        } catch (const type&) {                     \
            thrown_ = true;                         \
        } catch (...) {                             \
        }                                           \
        CHECK(thrown_ && #type);                    \
    } while (0)

using namespace saba;

static Graph fig1() { return Graph::from_edges(4, {{0, 1}, {0, 2}, {1, 2}, {1, 3}, {2, 3}}); }
static Graph path(uint32_t n) {
    std::vector<std::pair<uint32_t, uint32_t>> e;
    for (uint32_t v = 0; v + 1 < n; ++v) e.emplace_back(v, v + 1);
    return Graph::from_edges(n, e);
}
static Graph complete(uint32_t n) {
    std::vector<std::pair<uint32_t, uint32_t>> e;
    for (uint32_t u = 0; u < n; ++u)
        for (uint32_t v = u + 1; v < n; ++v) e.emplace_back(u, v);
    return Graph::from_edges(n, e);
}

static void host_checks() {
    // test_aesc.cpp:27
    CHECK(walk_budget(5, 0.05, 0.05, 4, 100) == 44936);
    CHECK_THROWS_AS(walk_budget(0, 0.05, 0.05, 1, 10), std::invalid_argument);
    // test_graph.cpp:18-62
    std::istringstream a("# comment\n\n  30\t7 \n7 9\n");
    const Graph g = Graph::load_edge_list(a);
    CHECK(g.vertex_count() == 3 && g.edge_count() == 2);
    CHECK(g.original_id(0) == 30 && g.original_id(1) == 7 && g.original_id(2) == 9);
    std::istringstream bad("0 x\n");
    CHECK_THROWS_AS(Graph::load_edge_list(bad), std::runtime_error);
    std::istringstream loop("0 0\n");
    CHECK_THROWS_AS(Graph::load_edge_list(loop), std::runtime_error);
    const Graph f = fig1();
    const auto nb = f.neighbors(1);
    CHECK(nb.size() == 3 && nb[0] == 0 && nb[1] == 2 && nb[2] == 3);
    CHECK(f.edge_index(2, 1) == f.edge_index(1, 2));
    std::ostringstream out;
    f.write_edge_list(out);
    std::istringstream back(out.str());
    const Graph f2 = Graph::load_edge_list(back);
    CHECK(f2.offsets() == f.offsets() && f2.adjacency() == f.adjacency());
    CHECK(is_connected(f) && !bipartition(f).first && bipartition(path(5)).first);
    // test_walker.cpp:213-226
    std::vector<uint64_t> hist(9, 0);
    hist[1] = 2, hist[2] = 10, hist[4] = 30, hist[8] = 58;
    const BranchingStats st = branching_stats(std::span<const uint64_t>(hist));
    CHECK(st.p1 == 1 && st.p10 == 2 && st.p25 == 4 && std::abs(st.mean - 6.06) < 1e-12);
    // test_rng.cpp
    CHECK(select_scaled(0xffffffffu, 0, 5) == 4 && select_mod(10, 3) == 1);
    const SeedSet s = gen_sorted_seeds(1000, 77);
    CHECK(std::is_sorted(s.seeds.begin(), s.seeds.end()));
}

static void gpu_checks() {
    const Graph f = fig1();
    // device canonicalisation == host canonicalisation (graph.hpp:86-105):
    // loops, reversed and repeated pairs, an isolated tail vertex
    {
        const std::vector<std::pair<uint32_t, uint32_t>> messy = {
            {3, 1}, {1, 3}, {2, 2}, {0, 4}, {4, 0}, {4, 0}, {1, 4}, {5, 5}, {2, 1}};
        const Graph h = Graph::from_edges(7, messy), d = Graph::from_edges(7, messy, 0);
        CHECK(d.vertex_count() == 7 && d.edge_count() == h.edge_count());
        CHECK(d.offsets() == h.offsets() && d.adjacency() == h.adjacency());
    }
    // test_walker.cpp:49-75
    CHECK(random_walk(f, 2, 1, SelectorKind::Scaled, 77).vertices == std::vector<uint32_t>{2});
    CHECK(random_walk(path(2), 0, 3, SelectorKind::Scaled, 123).vertices ==
          (std::vector<uint32_t>{0, 1, 0}));
    CHECK_THROWS_AS(random_walk(f, 0, 0, SelectorKind::Scaled, 1), std::invalid_argument);
    // test_walker.cpp:78-88
    const SeedSet seeds = gen_sorted_seeds(8, 99);
    const auto lanes = random_bouquet(f, 0, 12, 8, seeds, SelectorKind::Scaled);
    for (uint32_t b = 0; b < 8; ++b)
        CHECK(lanes[b].vertices == random_walk(f, 0, 12, SelectorKind::Scaled, seeds.seeds[b]).vertices);
    // test_walker.cpp:103-163
    CampaignConfig cfg;
    cfg.walks_per_vertex = 13;
    cfg.length = 4;
    VisitCountSink sink(4);
    const CampaignReport rep = run_walk_campaign(f, cfg, sink);
    uint64_t total = 0;
    for (uint64_t c : sink.counts) total += c;
    CHECK(rep.total_steps == 4 * 13 * 3 && total == 4 * 13 * 4);
    cfg.mode = WalkMode::Hash;
    VisitCountSink hs(4);
    run_walk_campaign(f, cfg, hs);
    CHECK(hs.counts == sink.counts);
    cfg.lanes = 7;
    CHECK_THROWS_AS(run_walk_campaign(f, cfg, hs), std::invalid_argument);
    // test_aesc.cpp:49-86
    const TruncationPlan k20 = truncated_lengths(complete(20), 0.05, 30);
    CHECK(std::abs(k20.lambda_hat - 1.0 / 19.0) < 1e-6 && k20.tau[0] <= 9);
    const TruncationPlan p100 = truncated_lengths(path(100), 0.05, 60, 128);
    CHECK(p100.clamped && p100.tau[0] == 127);
    // test_aesc.cpp:102-117 (depth 2 from A)
    TruncationPlan plan;
    plan.tau.assign(f.edge_count(), 3);
    const auto [lp, d] = propagate_landing_probabilities(f, 0, plan, 0.05, 0.05, 2);
    CHECK(d == 2 && std::abs(lp.prob_of(0) - 1.0 / 3) < 1e-14 && std::abs(lp.prob_of(1) - 1.0 / 6) < 1e-14);
    // test_aesc.cpp:183-198, 310-330
    AescConfig ac;
    ac.epsilon = 0.05;
    const CentralityEstimate tri = aesc(complete(3), ac);
    for (double x : tri.s_hat) CHECK(std::abs(x - 2.0 / 3.0) <= 0.05);
    const CentralityEstimate est = aesc(f, AescConfig{});
    for (uint32_t e = 0; e < f.edge_count(); ++e) {
        const auto [u, v] = f.edge(e);
        CHECK(est.s_hat[e] == est.g_hat[f.slot_of(u, v)] + est.g_hat[f.slot_of(v, u)]);
    }
    ac.epsilon = 0.0;
    CHECK_THROWS_AS(aesc(f, ac), std::invalid_argument);
    ac.epsilon = 0.05;
    CHECK_THROWS_AS(aesc(Graph::from_edges(4, {{0, 1}, {2, 3}}), ac), std::runtime_error);
    // GPU-count invariance (test_aesc.cpp:292-308, test_walker.cpp:152-158):
    // `threads` is a device count; SABA_DEVICES lists logical shards on one GPU
    {
        std::vector<std::pair<uint32_t, uint32_t>> e;
        for (uint32_t i = 0; i < 400; ++i) {
            e.push_back({i, (i + 1) % 400});
            e.push_back({i, (i * 7 + 3) % 400});
        }
        const Graph g = Graph::from_edges(400, e);
        AescConfig c1;
        c1.epsilon = 0.2;
        c1.threads = 1;
        CampaignConfig cc;
        cc.walks_per_vertex = 64;
        cc.length = 16;
        cc.threads = 1;
        unsetenv("SABA_DEVICES");
        const CentralityEstimate one = aesc(g, c1);
        VisitCountSink s1(400);
        run_walk_campaign(g, cc, s1);
        for (const char* devs : {"0,0", "0,0,0"}) {
            setenv("SABA_DEVICES", devs, 1);
            const CentralityEstimate many = aesc(g, c1);
            CHECK(many.g_hat == one.g_hat && many.s_hat == one.s_hat);
            CHECK(many.plan.tau_tilde == one.plan.tau_tilde && many.total_walk_pairs == one.total_walk_pairs);
            VisitCountSink sn(400);
            const CampaignReport rn = run_walk_campaign(g, cc, sn);
            CHECK(sn.counts == s1.counts && rn.threads_used == int(std::strlen(devs) + 1) / 2);
        }
        unsetenv("SABA_DEVICES");
    }
    std::ostringstream tsv;
    const std::vector<double> third(3, 2.0 / 3.0);
    write_centrality_tsv(tsv, complete(3), third);
    CHECK(tsv.str() == "0\t1\t0.666667\n0\t2\t0.666667\n1\t2\t0.666667\n");  // acceptance.cpp:129
}

int main() {
    host_checks();
    const bool gpu = saba_cu_device_count() > 0;
    if (gpu) gpu_checks();
    std::printf("dropin_test: %s checks %s (%d failures)\n", gpu ? "host+gpu" : "host",
                failures ? "FAILED" : "passed", failures);
    return failures ? 1 : 0;
}
