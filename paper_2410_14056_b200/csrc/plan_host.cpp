// TGT+ truncation plan and walk budget (host).
//
// These integer decisions (tau, n_req, and the tau~ crossover budget) are
// computed from float64 arithmetic, so the product restates them with the
// reference's exact operation order: lambda_hat must be bitwise equal for tau
// to match, and every walk length and budget follows from tau.
//   estimate_decay      aesc.hpp:137-190
//   make_odd_clamped    aesc.hpp:192-203
//   truncated_lengths   aesc.hpp:210-248
//   walks_needed_raw    aesc.hpp:103-110
//   walk_budget         aesc.hpp:117-126
// Built without FMA contraction (-ffp-contract=off), like the reference.
#include "plan_host.hpp"

#include <algorithm>
#include <cmath>
#include <limits>

#include "capi_util.hpp"
#include "saba_hash.cuh"

namespace saba_cu {

// Level-synchronous parallel BFS from vertex 0: returns the number of
// reached vertices and the level parity of each (0xff = unreached).
uint32_t host_bfs_parity(const HostCsr& g, std::vector<uint8_t>& parity) {
    parity.assign(g.n, 0xff);
    if (g.n == 0) return 0;
    std::vector<uint32_t> frontier{0}, next;
    parity[0] = 0;
    uint32_t reached = 1;
    uint8_t level = 0;
    while (!frontier.empty()) {
        ++level;
        next.clear();
        const int64_t F = int64_t(frontier.size());
#pragma omp parallel
        {
            std::vector<uint32_t> local;
#pragma omp for schedule(dynamic, 64) nowait
            for (int64_t i = 0; i < F; ++i) {
                const uint32_t u = frontier[size_t(i)];
                for (uint32_t s = g.off[u]; s < g.off[u + 1]; ++s) {
                    const uint32_t v = g.adj[s];
                    if (__atomic_load_n(&parity[v], __ATOMIC_RELAXED) != 0xff) continue;
                    uint8_t expect = 0xff;
                    if (__atomic_compare_exchange_n(&parity[v], &expect, uint8_t(level & 1), false,
                                                    __ATOMIC_RELAXED, __ATOMIC_RELAXED))
                        local.push_back(v);
                }
            }
#pragma omp critical(saba_bfs_merge)
            next.insert(next.end(), local.begin(), local.end());
        }
        reached += uint32_t(next.size());
        frontier.swap(next);
    }
    return reached;
}

bool host_is_connected(const HostCsr& g) {
    std::vector<uint8_t> parity;
    return g.n > 0 && host_bfs_parity(g, parity) == g.n;
}

// Connected graphs only: the reference's BFS 2-colouring (graph.hpp:271-292)
// has its root on side 0, so side = BFS level parity whenever the graph is
// bipartite, which holds iff no edge joins two vertices of equal parity.
bool bipartition_connected(const HostCsr& g, const std::vector<uint8_t>& parity,
                           std::vector<char>& side) {
    bool bip = true;
    const int64_t N = g.n;
#pragma omp parallel for schedule(dynamic, 1024) reduction(&& : bip)
    for (int64_t u = 0; u < N; ++u)
        for (uint32_t s = g.off[u]; s < g.off[u + 1]; ++s)
            if (parity[size_t(u)] == parity[g.adj[s]]) bip = false;
    side.clear();
    if (bip) side.assign(parity.begin(), parity.end());
    return bip;
}

bool host_bipartition(const HostCsr& g, std::vector<char>& side) {
    side.assign(g.n, -1);
    std::vector<uint32_t> q;
    for (uint32_t r = 0; r < g.n; ++r) {
        if (side[r] != -1) continue;
        side[r] = 0;
        q.assign(1, r);
        for (size_t h = 0; h < q.size(); ++h) {
            const uint32_t u = q[h];
            for (uint32_t s = g.off[u]; s < g.off[u + 1]; ++s) {
                const uint32_t v = g.adj[s];
                if (side[v] == -1) {
                    side[v] = char(1 - side[u]);
                    q.push_back(v);
                } else if (side[v] == side[u]) {
                    side.clear();
                    return false;
                }
            }
        }
    }
    return true;
}

double host_estimate_decay(const HostCsr& g, uint32_t iters, bool bip, const std::vector<char>& side,
                           const SpmvFn* spmv) {
    const uint32_t n = g.n;
    const double two_m = 2.0 * double(g.m);
    std::vector<double> phi(n), isd(n), x(n), y(n), z(n), sgn(n, 1.0);
    for (uint32_t v = 0; v < n; ++v) {
        const double d = double(g.off[v + 1] - g.off[v]);
        phi[v] = std::sqrt(d / two_m);
        isd[v] = d > 0 ? 1.0 / std::sqrt(d) : 0.0;
        if (bip && side[v]) sgn[v] = -1.0;
        x[v] = double(counter_hash(0x0ddc0ffeeull, v) >> 11) * 0x1.0p-53 - 0.5;
    }
    auto project = [&](std::vector<double>& w) {
        double dphi = 0.0, dpsi = 0.0;
        for (uint32_t v = 0; v < n; ++v) {
            dphi += w[v] * phi[v];
            if (bip) dpsi += w[v] * sgn[v] * phi[v];
        }
        for (uint32_t v = 0; v < n; ++v) {
            w[v] -= dphi * phi[v];
            if (bip) w[v] -= dpsi * sgn[v] * phi[v];
        }
    };
    auto norm = [&](const std::vector<double>& w) {
        double s = 0.0;
        for (double t : w) s += t * t;
        return std::sqrt(s);
    };
    project(x);
    const double nx = norm(x);
    if (nx < 1e-12) return 0.0;
    for (double& t : x) t /= nx;
    double lambda = 0.0;
    // Element-wise passes and the SpMV rows are independent, so they run in
    // parallel with each element computed exactly as the reference does
    // (row sums in neighbour order); the three reductions (two projections,
    // the norm) stay sequential, so lambda_hat is bit-identical.
    const int64_t N = n;
    for (uint32_t it = 0; it < iters; ++it) {
        if (spmv) {
            (*spmv)(x, isd, y);
        } else {
#pragma omp parallel for schedule(static)
            for (int64_t v = 0; v < N; ++v) z[v] = x[v] * isd[v];
#pragma omp parallel for schedule(dynamic, 1024)
            for (int64_t u = 0; u < N; ++u) {
                double acc = 0.0;
                for (uint32_t s = g.off[u]; s < g.off[u + 1]; ++s) acc += z[g.adj[s]];
                y[u] = acc * isd[u];
            }
        }
        project(y);
        const double ny = norm(y);
        if (ny < 1e-15) return 0.0;
        lambda = ny;
#pragma omp parallel for schedule(static)
        for (int64_t v = 0; v < N; ++v) x[v] = y[v] / ny;
    }
    return std::min(lambda, 1.0);
}

namespace {
uint32_t make_odd_clamped(double raw, uint32_t max_truncation, bool& clamped) {
    uint32_t t = raw < 1.0 ? 1u
                           : uint32_t(std::min(raw, double(std::numeric_limits<uint32_t>::max() - 1)));
    t |= 1u;
    if (t > max_truncation) {
        t = max_truncation;
        if ((t & 1u) == 0) t -= 1;
        clamped = true;
    }
    return std::max(t, 1u);
}
}  // namespace

Plan host_truncated_lengths(const HostCsr& g, const uint32_t* slot_edge, double eps,
                            uint32_t omega, uint32_t max_truncation, bool per_edge, const SpmvFn* spmv) {
    check_arg(eps > 0.0 && eps < 1.0, "truncated_lengths: epsilon must be in (0,1)");
    check_arg(omega >= 1, "truncated_lengths: omega must be >= 1");
    check_arg(max_truncation >= 1, "truncated_lengths: tau_max must be >= 1");
    std::vector<uint8_t> parity;
    check_data(g.n > 0 && host_bfs_parity(g, parity) == g.n,
               "truncated_lengths: graph must be connected");
    std::vector<char> side;
    const bool bip = bipartition_connected(g, parity, side);
    Plan p;
    p.bipartite = bip;
    p.lambda_hat = host_estimate_decay(g, omega, bip, side, spmv);
    auto tau_for = [&](double dmax) -> uint32_t {
        if (p.lambda_hat >= 1.0 - 1e-6) {
            p.clamped = true;
            uint32_t t = max_truncation;
            if (t > 1 && (t & 1u) == 0) t -= 1;
            return t;
        }
        if (p.lambda_hat <= 1e-9) return 1;
        const double raw = std::ceil(std::log(4.0 * dmax / (eps * (1.0 - p.lambda_hat))) /
                                     std::log(1.0 / p.lambda_hat));
        return make_odd_clamped(raw, max_truncation, p.clamped);
    };
    p.tau.resize(g.m);
    if (per_edge) {
        for (uint32_t u = 0; u < g.n; ++u)
            for (uint32_t s = g.off[u]; s < g.off[u + 1]; ++s) {
                const uint32_t v = g.adj[s];
                if (v <= u) continue;
                const uint32_t du = g.off[u + 1] - g.off[u], dv = g.off[v + 1] - g.off[v];
                p.tau[slot_edge[s]] = tau_for(double(std::max(du, dv)));
            }
    } else {
        uint32_t dmax = 0;
        for (uint32_t v = 0; v < g.n; ++v) dmax = std::max(dmax, g.off[v + 1] - g.off[v]);
        std::fill(p.tau.begin(), p.tau.end(), tau_for(double(dmax)));
    }
    p.max_tau = p.tau.empty() ? 0 : *std::max_element(p.tau.begin(), p.tau.end());
    p.uniform = !per_edge;
    return p;
}

double walks_needed_raw(int64_t tau_eff, double eps, double delta, uint32_t degree, uint64_t m) {
    if (tau_eff <= 0) return 0.0;
    const double scale = 0.5 * eps * double(degree);
    const double t = double(tau_eff);
    return std::ceil((2.0 * t * t / (scale * scale)) * std::log(4.0 * double(m) / delta));
}

uint64_t walk_budget(uint32_t tau_eff, double eps, double delta, uint32_t degree, uint64_t m) {
    check_arg(tau_eff >= 1, "walk_budget: tau_effective must be >= 1");
    check_arg(degree >= 1, "walk_budget: degree must be >= 1");
    check_arg(eps > 0.0 && eps < 1.0, "walk_budget: epsilon must be in (0,1)");
    check_arg(delta > 0.0 && delta < 1.0, "walk_budget: delta must be in (0,1)");
    const double v = walks_needed_raw(tau_eff, eps, delta, degree, m);
    check_arg(v < 9.0e18, "walk_budget: budget overflows");
    return uint64_t(v);
}

}  // namespace saba_cu

extern "C" int saba_cu_walk_budget(uint32_t tau_effective, double epsilon, double delta,
                                   uint32_t degree, uint64_t edge_count, uint64_t* out) {
    return saba_cu::guard([&] {
        saba_cu::check_arg(out != nullptr, "null output");
        *out = saba_cu::walk_budget(tau_effective, epsilon, delta, degree, edge_count);
    });
}
