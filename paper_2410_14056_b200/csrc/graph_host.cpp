// Host-side graph construction: canonicalisation into the reference's CSR
// (Graph::from_edges + build_csr, graph.hpp:86-105, 199-237), largest
// connected component extraction, and the seeded generators the BASELINE
// configs need (ER, R-MAT, Chung–Lu — none exist in the reference, SURVEY
// §0.2) plus the reference's own test generators (gen.hpp:17-69).
//
// Canonicalisation is a parallel LSD radix sort over packed (min<<32 | max)
// keys; because edges are then visited in sorted (u, v) order, one fill pass
// already yields ascending neighbour slices (every neighbour < u arrives
// before every neighbour > u), so no per-slice sort is needed.
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <unordered_set>
#include <vector>

#include "capi_util.hpp"
#include "saba_hash.cuh"

#include "hgraph.hpp"

namespace saba_cu {

namespace {

// Parallel LSD radix sort of 64-bit keys restricted to their low `bits` bits.
void radix_sort_u64(std::vector<uint64_t>& keys, int bits) {
    const size_t N = keys.size();
    if (N < (1u << 16)) {
        std::sort(keys.begin(), keys.end());
        return;
    }
    constexpr int D = 11;
    constexpr int R = 1 << D;
    std::vector<uint64_t> tmp(N);
    const int T = std::max(1, omp_get_max_threads());
    std::vector<size_t> hist(size_t(T) * R);
    for (int shift = 0; shift < bits; shift += D) {
        std::fill(hist.begin(), hist.end(), 0);
#pragma omp parallel num_threads(T)
        {
            const int t = omp_get_thread_num();
            const size_t lo = N * t / T, hi = N * (t + 1) / T;
            size_t* h = &hist[size_t(t) * R];
            for (size_t i = lo; i < hi; ++i) ++h[(keys[i] >> shift) & (R - 1)];
#pragma omp barrier
#pragma omp single
            {
                size_t run = 0;
                for (int d = 0; d < R; ++d)
                    for (int tt = 0; tt < T; ++tt) {
                        size_t c = hist[size_t(tt) * R + d];
                        hist[size_t(tt) * R + d] = run;
                        run += c;
                    }
            }
            for (size_t i = lo; i < hi; ++i) tmp[h[(keys[i] >> shift) & (R - 1)]++] = keys[i];
        }
        keys.swap(tmp);
    }
}

int bits_for(uint64_t x) {
    int b = 1;
    while (b < 64 && (uint64_t(1) << b) <= x) ++b;
    return b;
}

// keys: sorted, unique, (u<<32 | v) with u < v < n.
saba_hgraph* csr_from_sorted_keys(uint32_t n, const std::vector<uint64_t>& keys) {
    check_data(n > 0, "empty graph");
    check_data(2 * keys.size() <= 0xffffffffull, "graph too large: 2m must fit in 32 bits");
    auto* g = new saba_hgraph;
    g->n = n;
    g->m = keys.size();
    g->off.assign(size_t(n) + 1, 0);
    for (uint64_t k : keys) {
        ++g->off[(k >> 32) + 1];
        ++g->off[(k & 0xffffffffu) + 1];
    }
    for (uint32_t u = 0; u < n; ++u) g->off[u + 1] += g->off[u];
    g->adj.resize(2 * keys.size());
    std::vector<uint32_t> cur(g->off.begin(), g->off.end() - 1);
    for (uint64_t k : keys) {
        const uint32_t u = uint32_t(k >> 32), v = uint32_t(k);
        g->adj[cur[u]++] = v;
        g->adj[cur[v]++] = u;
    }
    return g;
}

saba_hgraph* from_pairs(uint32_t n_hint, std::vector<uint64_t>& keys) {
    // keys already packed as (min<<32 | max); loops still present
    uint32_t n = n_hint;
    for (uint64_t k : keys) n = std::max(n, uint32_t(k & 0xffffffffu) + 1);
    keys.erase(std::remove_if(keys.begin(), keys.end(),
                              [](uint64_t k) { return (k >> 32) == (k & 0xffffffffu); }),
               keys.end());
    radix_sort_u64(keys, 32 + bits_for(n));
    keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
    return csr_from_sorted_keys(n, keys);
}

// Large copies out of a graph land in fresh caller pages: fault them in on
// every core, not one.
void par_copy(uint32_t* dst, const uint32_t* src, size_t count) {
    constexpr size_t kPiece = size_t(1) << 18;
    const int64_t pieces = int64_t((count + kPiece - 1) / kPiece);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < pieces; ++i) {
        const size_t o = size_t(i) * kPiece;
        std::memcpy(dst + o, src + o, sizeof(uint32_t) * std::min(kPiece, count - o));
    }
}

inline uint64_t pack(uint32_t a, uint32_t b) {
    if (a > b) std::swap(a, b);
    return (uint64_t(a) << 32) | b;
}

saba_hgraph* largest_component(const saba_hgraph& g) {
    const uint32_t n = g.n;
    std::vector<uint32_t> comp(n, UINT32_MAX), queue;
    queue.reserve(n);
    uint32_t best = 0, best_size = 0, ncomp = 0;
    for (uint32_t r = 0; r < n; ++r) {
        if (comp[r] != UINT32_MAX) continue;
        queue.clear();
        queue.push_back(r);
        comp[r] = ncomp;
        for (size_t h = 0; h < queue.size(); ++h) {
            const uint32_t u = queue[h];
            for (uint32_t s = g.off[u]; s < g.off[u + 1]; ++s)
                if (comp[g.adj[s]] == UINT32_MAX) {
                    comp[g.adj[s]] = ncomp;
                    queue.push_back(g.adj[s]);
                }
        }
        if (queue.size() > best_size) {
            best_size = uint32_t(queue.size());
            best = ncomp;
        }
        ++ncomp;
    }
    std::vector<uint32_t> id(n, UINT32_MAX);
    uint32_t k = 0;
    for (uint32_t v = 0; v < n; ++v)
        if (comp[v] == best) id[v] = k++;
    // relabelling is monotone, so the (u<v) edges stay sorted
    std::vector<uint64_t> keys;
    keys.reserve(g.m);
    for (uint32_t u = 0; u < n; ++u) {
        if (comp[u] != best) continue;
        for (uint32_t s = g.off[u]; s < g.off[u + 1]; ++s)
            if (g.adj[s] > u) keys.push_back((uint64_t(id[u]) << 32) | id[g.adj[s]]);
    }
    return csr_from_sorted_keys(k, keys);
}

saba_hgraph* maybe_lcc(saba_hgraph* g, int keep_lcc) {
    if (!keep_lcc) return g;
    saba_hgraph* l = largest_component(*g);
    delete g;
    return l;
}

inline double unit53(uint64_t h) { return double(h >> 11) * 0x1.0p-53; }

// Lcg64 (rng.hpp:82-91), used only by the reference's own test generators.
struct Lcg {
    uint64_t s;
    explicit Lcg(uint64_t seed) : s(mix64(seed)) {}
    uint32_t next() {
        s = s * 0x5851f42d4c957f2dull + 0x14057b7ef767814full;
        return uint32_t(s >> 32);
    }
};

}  // namespace

// Chung–Lu weights and the Vose alias table of the endpoint distribution;
// shared by the host and device generators so both sample the same graph.
void chung_lu_tables(uint32_t n, double gamma, double mean_degree, double max_degree, uint64_t seed,
                     ChungLuTables& t) {
    check_arg(n >= 2, "chung_lu: need n >= 2");
    check_arg(gamma > 1.0, "chung_lu: gamma must be > 1");
    check_arg(mean_degree > 0 && max_degree >= 1, "chung_lu: bad degree parameters");
    const uint64_t s = substream(seed, 0x43484c55ull /*"CHLU"*/);
    // weights: Pareto draws w = U^(-1/(gamma-1)), U in (0, 1]
    std::vector<double> w(n);
    const double ex = -1.0 / (gamma - 1.0);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < int64_t(n); ++i)
        w[size_t(i)] = std::pow(1.0 - unit53(counter_hash(s, uint64_t(i))), ex);
    // scale c such that the mean of the CAPPED weights min(c w, cap) is
    // mean_degree (capping removes tail mass; bisection, deterministic)
    auto capped_mean = [&](double c) {
        double s = 0.0;
        for (double x : w) s += std::min(x * c, max_degree);
        return s / double(n);
    };
    double lo = 0.0, hi = 1.0;
    while (capped_mean(hi) < mean_degree && hi < 1e30) hi *= 2.0;
    check_arg(capped_mean(hi) >= mean_degree, "chung_lu: mean_degree unreachable under the cap");
    for (int it = 0; it < 100; ++it) {
        const double mid = 0.5 * (lo + hi);
        (capped_mean(mid) < mean_degree ? lo : hi) = mid;
    }
    const double scalef = hi;
    double total = 0.0;
    for (double& x : w) {
        x = std::min(x * scalef, max_degree);
        total += x;
    }
    // Vose alias table over w / total
    std::vector<double> prob(n);
    std::vector<uint32_t> alias(n, 0), small, large;
    for (uint32_t i = 0; i < n; ++i) {
        prob[i] = w[i] * double(n) / total;
        (prob[i] < 1.0 ? small : large).push_back(i);
    }
    while (!small.empty() && !large.empty()) {
        const uint32_t l = small.back(), g = large.back();
        small.pop_back();
        alias[l] = g;
        prob[g] = (prob[g] + prob[l]) - 1.0;
        if (prob[g] < 1.0) {
            large.pop_back();
            small.push_back(g);
        }
    }
    for (uint32_t i : large) prob[i] = 1.0;
    for (uint32_t i : small) prob[i] = 1.0;
    t.prob = std::move(prob);
    t.alias = std::move(alias);
    t.samples = uint64_t(std::llround(total / 2.0));
}

}  // namespace saba_cu

using namespace saba_cu;

extern "C" {

int saba_hgraph_from_edges(uint32_t n_hint, const uint32_t* pairs, uint64_t count,
                           saba_hgraph** out) {
    return guard([&] {
        check_arg(out != nullptr, "null output");
        check_arg(count == 0 || pairs != nullptr, "null pairs");
        std::vector<uint64_t> keys(count);
        for (uint64_t i = 0; i < count; ++i) keys[i] = pack(pairs[2 * i], pairs[2 * i + 1]);
        *out = from_pairs(n_hint, keys);
    });
}

int saba_hgraph_from_csr(uint32_t n, const uint32_t* off, const uint32_t* adj, saba_hgraph** out) {
    return guard([&] {
        check_arg(out && off && (off[n] == 0 || adj), "null argument");
        check_data(n > 0, "empty graph");
        check_data(off[0] == 0 && off[n] % 2 == 0, "malformed CSR offsets");
        auto* g = new saba_hgraph;
        g->n = n;
        g->m = off[n] / 2;
        g->off.assign(off, off + n + 1);
        g->adj.assign(adj, adj + off[n]);
        for (uint32_t u = 0; u < n; ++u) {
            check_data(off[u] <= off[u + 1], "malformed CSR offsets");
            for (uint32_t s = off[u]; s < off[u + 1]; ++s) {
                check_data(adj[s] < n && adj[s] != u, "CSR has a self-loop or bad id");
                check_data(s == off[u] || adj[s - 1] < adj[s], "CSR slices must be sorted and unique");
            }
        }
        *out = g;
    });
}

int saba_gen_erdos_renyi(uint32_t n, uint64_t m, uint64_t seed, saba_hgraph** out) {
    return guard([&] {
        check_arg(out != nullptr, "null output");
        check_arg(n >= 2, "erdos_renyi: need n >= 2");
        check_arg(m <= uint64_t(n) * (n - 1) / 2, "erdos_renyi: too many edges");
        const uint64_t s = substream(seed, 0x45524452ull /*"ERDR"*/);
        std::unordered_set<uint64_t> seen;
        seen.reserve(size_t(m * 2));
        std::vector<uint64_t> keys;
        keys.reserve(m);
        for (uint64_t i = 0; keys.size() < m; ++i) {
            const uint64_t h = counter_hash(s, i);
            const uint32_t a = scaled_index(uint32_t(h >> 32), n);
            const uint32_t b = scaled_index(uint32_t(h), n);
            if (a == b) continue;
            const uint64_t k = pack(a, b);
            if (seen.insert(k).second) keys.push_back(k);
        }
        *out = from_pairs(n, keys);
    });
}

int saba_gen_rmat(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                  uint64_t seed, int keep_lcc, saba_hgraph** out) {
    return guard([&] {
        check_arg(out != nullptr, "null output");
        check_arg(scale >= 1 && scale <= 31, "rmat: scale must be in [1, 31]");
        check_arg(edge_factor >= 1, "rmat: edge_factor must be >= 1");
        check_arg(a > 0 && b >= 0 && c >= 0 && a + b + c < 1.0, "rmat: bad quadrant probabilities");
        const uint64_t samples = uint64_t(edge_factor) << scale;
        const uint64_t s = substream(seed, kRmatTag);
        const RmatThresholds thr = rmat_thresholds(a, b, c);
        std::vector<uint64_t> keys(samples);
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < int64_t(samples); ++i) {
            uint32_t u, v;
            rmat_sample(s, uint64_t(i), scale, thr, u, v);
            keys[size_t(i)] = pack(u, v);
        }
        *out = maybe_lcc(from_pairs(uint32_t(1u << scale), keys), keep_lcc);
    });
}

int saba_gen_chung_lu(uint32_t n, double gamma, double mean_degree, double max_degree,
                      uint64_t seed, int keep_lcc, saba_hgraph** out) {
    return guard([&] {
        check_arg(out != nullptr, "null output");
        ChungLuTables t;
        chung_lu_tables(n, gamma, mean_degree, max_degree, seed, t);
        const std::vector<double>& prob = t.prob;
        const std::vector<uint32_t>& alias = t.alias;
        const uint64_t samples = t.samples;
        const uint64_t s2 = substream(seed, kChungLuTag);
        std::vector<uint64_t> keys(samples);
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < int64_t(samples); ++i)
            keys[size_t(i)] = pack(chung_lu_end(s2, uint64_t(i), 0, n, prob.data(), alias.data()),
                                   chung_lu_end(s2, uint64_t(i), 1, n, prob.data(), alias.data()));
        *out = maybe_lcc(from_pairs(n, keys), keep_lcc);
    });
}

// gen.hpp:17-44
int saba_gen_scale_free(uint32_t n, uint32_t attach, uint64_t seed, saba_hgraph** out) {
    return guard([&] {
        check_arg(attach >= 1 && n >= attach + 1, "make_scale_free: need n >= attach + 1");
        Lcg rng(substream(seed, 0x5caefee));
        std::vector<uint64_t> keys;
        std::vector<uint32_t> pool, picked;
        for (uint32_t u = 0; u <= attach; ++u)
            for (uint32_t v = u + 1; v <= attach; ++v) {
                keys.push_back(pack(u, v));
                pool.push_back(u);
                pool.push_back(v);
            }
        for (uint32_t v = attach + 1; v < n; ++v) {
            picked.clear();
            while (picked.size() < attach) {
                const uint32_t u = pool[scaled_index(rng.next(), uint32_t(pool.size()))];
                if (std::find(picked.begin(), picked.end(), u) == picked.end()) picked.push_back(u);
            }
            for (uint32_t u : picked) {
                keys.push_back(pack(u, v));
                pool.push_back(u);
                pool.push_back(v);
            }
        }
        *out = from_pairs(n, keys);
    });
}

// gen.hpp:48-69
int saba_gen_random_connected(uint32_t n, uint32_t extra, uint64_t seed, saba_hgraph** out) {
    return guard([&] {
        check_arg(n >= 2, "make_random_connected: need n >= 2");
        Lcg rng(substream(seed, 0xc0113c7));
        std::vector<uint64_t> keys;
        std::unordered_set<uint64_t> seen;
        for (uint32_t v = 1; v < n; ++v) {
            const uint64_t k = pack(scaled_index(rng.next(), v), v);
            keys.push_back(k);
            seen.insert(k);
        }
        const uint64_t max_edges = uint64_t(n) * (n - 1) / 2;
        const uint32_t budget = uint32_t(std::min<uint64_t>(extra, max_edges - (n - 1)));
        for (uint32_t added = 0; added < budget;) {
            const uint32_t a = scaled_index(rng.next(), n);
            const uint32_t b = scaled_index(rng.next(), n);
            if (a == b) continue;
            const uint64_t k = pack(a, b);
            if (!seen.insert(k).second) continue;
            keys.push_back(k);
            ++added;
        }
        *out = from_pairs(n, keys);
    });
}

int saba_hgraph_largest_component(const saba_hgraph* in, saba_hgraph** out) {
    return guard([&] {
        check_arg(in && out, "null argument");
        *out = largest_component(*in);
    });
}

int saba_hgraph_data(const saba_hgraph* g, const uint32_t** offsets, const uint32_t** adjacency) {
    return guard([&] {
        check_arg(g && offsets && adjacency, "null argument");
        *offsets = g->off.data();
        *adjacency = g->adj.data();
    });
}

uint32_t saba_hgraph_vertex_count(const saba_hgraph* g) { return g ? g->n : 0; }
uint64_t saba_hgraph_edge_count(const saba_hgraph* g) { return g ? g->m : 0; }

int saba_hgraph_csr(const saba_hgraph* g, uint32_t* offsets, uint32_t* adjacency) {
    return guard([&] {
        check_arg(g && offsets && adjacency, "null argument");
        par_copy(offsets, g->off.data(), g->off.size());
        par_copy(adjacency, g->adj.data(), g->adj.size());
    });
}

void saba_hgraph_free(saba_hgraph* g) { delete g; }

}  // extern "C"
