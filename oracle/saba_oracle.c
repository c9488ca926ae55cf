/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference hot path
 * (Bouquets walks + TGT+ AESC), the parity checker for the sm_100a product.
 * See saba_oracle.h for the contract; every function cites the reference
 * file:line it restates (paths relative to /root/reference/proj/include/saba).
 *
 * Floating point: compiled with -O2 -ffp-contract=off and no -march, like the
 * reference (-O3 -DNDEBUG, no -march => no FMA contraction on x86-64), so the
 * float64 sequences below round exactly as the reference's do.
 */
#include "saba_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ hashes */

/* common.hpp:24-31 splitmix64 finalizer */
uint64_t oracle_mix64(uint64_t x) {
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

/* common.hpp:34-36 */
uint64_t oracle_counter_hash(uint64_t master, uint64_t index) {
    return oracle_mix64(master + (index + 1) * 0x9e3779b97f4a7c15ull);
}

/* common.hpp:39-41 */
uint64_t oracle_substream(uint64_t master, uint64_t tag) {
    return oracle_mix64(master ^ oracle_mix64(tag + 0x632be59bd9b4e019ull));
}

/* rng.hpp:23-30  h(cur, l) */
uint32_t oracle_hash_state(uint64_t mult, uint32_t vertex, uint32_t step) {
    uint64_t x = ((uint64_t)vertex << 32) | (uint64_t)step;
    x *= mult;
    x ^= x >> 47;
    x *= mult;
    x ^= x >> 47;
    return (uint32_t)(x >> 32);
}

/* rng.hpp:61-63  Eq. (5) with h_max = 2^32 */
uint32_t oracle_scaled_index(uint32_t raw, uint32_t degree) {
    return (uint32_t)(((uint64_t)raw * (uint64_t)degree) >> 32);
}

/* one hashed selection step: walker.hpp:196-200 / 224-230 */
static inline uint32_t step_once(const uint32_t* off, const uint32_t* adj, uint32_t cur,
                                 uint32_t l, uint32_t seed, uint64_t mult) {
    const uint32_t base = off[cur];
    const uint32_t deg = off[cur + 1] - base;
    const uint32_t raw = seed ^ oracle_hash_state(mult, cur, l);
    return adj[base + oracle_scaled_index(raw, deg)];
}

/* ------------------------------------------------------------------- walks */

/* walker.hpp:188-203, 283-302 */
void oracle_random_walk(const uint32_t* off, const uint32_t* adj, uint32_t start,
                        uint32_t length, uint32_t seed, uint64_t mult, uint32_t* path) {
    uint32_t cur = start;
    if (length == 0) return;
    path[0] = cur;
    for (uint32_t l = 1; l < length; ++l) {
        cur = step_once(off, adj, cur, l, seed, mult);
        path[l] = cur;
    }
}

/* walker.hpp:430-449 (campaign_vertex_scaled) driven as in run_walk_campaign
 * walker.hpp:481-519; per-thread shards merged in thread order. */
void oracle_campaign_counts(const uint32_t* off, const uint32_t* adj, uint32_t n,
                            const uint64_t* kpv, uint64_t K, uint32_t length, uint64_t master,
                            uint64_t mult, int threads, uint64_t* counts) {
    memset(counts, 0, sizeof(uint64_t) * n);
#ifdef _OPENMP
    if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel num_threads(threads)
#endif
    {
        uint64_t* shard = (uint64_t*)calloc(n, sizeof(uint64_t));
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 64)
#endif
        for (int64_t vi = 0; vi < (int64_t)n; ++vi) {
            const uint32_t v = (uint32_t)vi;
            const uint64_t kv = kpv ? kpv[v] : K;
            const uint64_t vseed = oracle_substream(master, v);
            for (uint64_t k = 0; k < kv; ++k) {
                const uint32_t seed = (uint32_t)(oracle_counter_hash(vseed, k) >> 32);
                uint32_t cur = v;
                ++shard[cur];
                for (uint32_t l = 1; l < length; ++l) {
                    cur = step_once(off, adj, cur, l, seed, mult);
                    ++shard[cur];
                }
            }
        }
#ifdef _OPENMP
#pragma omp critical(oracle_merge)
#endif
        for (uint32_t v = 0; v < n; ++v) counts[v] += shard[v];
        free(shard);
    }
}

/* SURVEY §8(d) uniform-start mapping (not a reference API; the per-vertex
 * walks then follow walker.hpp:430-449 with K_v). */
void oracle_uniform_start_counts(uint32_t n, uint64_t W, uint64_t master, uint64_t* k_out) {
    const uint64_t s = oracle_substream(master, 0x5354415254ull);
    memset(k_out, 0, sizeof(uint64_t) * n);
    for (uint64_t w = 0; w < W; ++w)
        ++k_out[oracle_scaled_index((uint32_t)(oracle_counter_hash(s, w) >> 32), n)];
}

/* ------------------------------------------------------------- graph utils */

/* graph.hpp:250-267 */
int oracle_is_connected(const uint32_t* off, const uint32_t* adj, uint32_t n) {
    if (n == 0) return 0;
    char* seen = (char*)calloc(n, 1);
    uint32_t* q = (uint32_t*)malloc(sizeof(uint32_t) * n);
    uint32_t head = 0, tail = 0, reached = 1;
    q[tail++] = 0;
    seen[0] = 1;
    while (head < tail) {
        const uint32_t u = q[head++];
        for (uint32_t s = off[u]; s < off[u + 1]; ++s) {
            const uint32_t v = adj[s];
            if (!seen[v]) { seen[v] = 1; ++reached; q[tail++] = v; }
        }
    }
    free(seen);
    free(q);
    return reached == n;
}

/* graph.hpp:271-292: BFS 2-colouring per component, roots on side 0 */
int oracle_bipartition(const uint32_t* off, const uint32_t* adj, uint32_t n, signed char* side) {
    uint32_t* q = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
    for (uint32_t v = 0; v < n; ++v) side[v] = -1;
    for (uint32_t root = 0; root < n; ++root) {
        if (side[root] != -1) continue;
        side[root] = 0;
        uint32_t head = 0, tail = 0;
        q[tail++] = root;
        while (head < tail) {
            const uint32_t u = q[head++];
            for (uint32_t s = off[u]; s < off[u + 1]; ++s) {
                const uint32_t v = adj[s];
                if (side[v] == -1) { side[v] = (signed char)(1 - side[u]); q[tail++] = v; }
                else if (side[v] == side[u]) { free(q); return 0; }
            }
        }
    }
    free(q);
    return 1;
}

static uint32_t find_slot(const uint32_t* off, const uint32_t* adj, uint32_t u, uint32_t v) {
    uint32_t lo = off[u], hi = off[u + 1];
    while (lo < hi) {
        const uint32_t mid = lo + (hi - lo) / 2;
        if (adj[mid] < v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

/* Edge ids are ranks of (u<v) pairs in sorted order (graph.hpp:92-100); the
 * sorted CSR visits them in exactly that order when u ascends and only
 * v > u is taken. */
void oracle_slot_edges(const uint32_t* off, const uint32_t* adj, uint32_t n, uint32_t* slot_edge) {
    uint32_t e = 0;
    for (uint32_t u = 0; u < n; ++u)
        for (uint32_t s = off[u]; s < off[u + 1]; ++s)
            if (adj[s] > u) slot_edge[s] = e++;
    for (uint32_t u = 0; u < n; ++u)
        for (uint32_t s = off[u]; s < off[u + 1]; ++s)
            if (adj[s] < u) slot_edge[s] = slot_edge[find_slot(off, adj, adj[s], u)];
}

/* --------------------------------------------------------- truncation plan */

/* aesc.hpp:137-190: deflated power iteration on D^-1/2 A D^-1/2 */
double oracle_estimate_decay(const uint32_t* off, const uint32_t* adj, uint32_t n, uint64_t m,
                             uint32_t iterations, int bip, const signed char* side) {
    const double two_m = 2.0 * (double)m;
    double* phi = (double*)malloc(sizeof(double) * n);
    double* isd = (double*)malloc(sizeof(double) * n);
    double* x = (double*)malloc(sizeof(double) * n);
    double* y = (double*)malloc(sizeof(double) * n);
    double* z = (double*)malloc(sizeof(double) * n);
    double lambda = 0.0, result;
    for (uint32_t v = 0; v < n; ++v) {
        const double d = (double)(off[v + 1] - off[v]);
        phi[v] = sqrt(d / two_m);
        isd[v] = d > 0 ? 1.0 / sqrt(d) : 0.0;
        x[v] = (double)(oracle_counter_hash(0x0ddc0ffeeull, v) >> 11) * 0x1.0p-53 - 0.5;
    }
#define SGN(v) ((bip && side[v]) ? -1.0 : 1.0)
#define PROJECT(w)                                                        \
    do {                                                                  \
        double dphi = 0.0, dpsi = 0.0;                                    \
        for (uint32_t v = 0; v < n; ++v) {                                \
            dphi += (w)[v] * phi[v];                                      \
            if (bip) dpsi += (w)[v] * SGN(v) * phi[v];                    \
        }                                                                 \
        for (uint32_t v = 0; v < n; ++v) {                                \
            (w)[v] -= dphi * phi[v];                                      \
            if (bip) (w)[v] -= dpsi * SGN(v) * phi[v];                    \
        }                                                                 \
    } while (0)
#define NORM(w, out)                                                      \
    do {                                                                  \
        double s_ = 0.0;                                                  \
        for (uint32_t v = 0; v < n; ++v) s_ += (w)[v] * (w)[v];           \
        out = sqrt(s_);                                                   \
    } while (0)

    PROJECT(x);
    double nx;
    NORM(x, nx);
    if (nx < 1e-12) { result = 0.0; goto done; }
    for (uint32_t v = 0; v < n; ++v) x[v] /= nx;
    for (uint32_t it = 0; it < iterations; ++it) {
        for (uint32_t v = 0; v < n; ++v) z[v] = x[v] * isd[v];
        for (uint32_t u = 0; u < n; ++u) {
            double acc = 0.0;
            for (uint32_t s = off[u]; s < off[u + 1]; ++s) acc += z[adj[s]];
            y[u] = acc * isd[u];
        }
        PROJECT(y);
        double ny;
        NORM(y, ny);
        if (ny < 1e-15) { result = 0.0; goto done; }
        lambda = ny;
        for (uint32_t v = 0; v < n; ++v) x[v] = y[v] / ny;
    }
    result = lambda < 1.0 ? lambda : 1.0;
done:
#undef SGN
#undef PROJECT
#undef NORM
    free(phi); free(isd); free(x); free(y); free(z);
    return result;
}

/* aesc.hpp:192-203 */
static uint32_t make_odd_clamped(double raw, uint32_t max_truncation, int* clamped) {
    uint32_t t;
    if (raw < 1.0) t = 1u;
    else t = (uint32_t)(raw < 4294967294.0 ? raw : 4294967294.0);
    t |= 1u;
    if (t > max_truncation) {
        t = max_truncation;
        if ((t & 1u) == 0) t -= 1;
        *clamped = 1;
    }
    return t > 1u ? t : 1u;
}

/* aesc.hpp:223-235 (tau_for) */
static uint32_t tau_for(double lambda, double dmax, double eps, uint32_t max_trunc, int* clamped) {
    if (lambda >= 1.0 - 1e-6) {
        *clamped = 1;
        uint32_t t = max_trunc;
        if (t > 1 && (t & 1u) == 0) t -= 1;
        return t;
    }
    if (lambda <= 1e-9) return 1;
    const double raw = ceil(log(4.0 * dmax / (eps * (1.0 - lambda))) / log(1.0 / lambda));
    return make_odd_clamped(raw, max_trunc, clamped);
}

/* aesc.hpp:210-248 */
int oracle_truncated_lengths(const uint32_t* off, const uint32_t* adj, uint32_t n, uint64_t m,
                             double epsilon, uint32_t omega, uint32_t max_truncation,
                             int per_edge, uint32_t* tau, double* lambda_hat, int* clamped) {
    if (!(epsilon > 0.0 && epsilon < 1.0) || omega < 1 || max_truncation < 1) return 1;
    if (!oracle_is_connected(off, adj, n)) return 2;
    signed char* side = (signed char*)malloc(n ? n : 1);
    const int bip = oracle_bipartition(off, adj, n, side);
    const double lambda = oracle_estimate_decay(off, adj, n, m, omega, bip, side);
    free(side);
    *lambda_hat = lambda;
    *clamped = 0;
    if (per_edge) {
        /* edge ids in sorted (u<v) order; see oracle_slot_edges */
        uint32_t e = 0;
        for (uint32_t u = 0; u < n; ++u)
            for (uint32_t s = off[u]; s < off[u + 1]; ++s) {
                const uint32_t v = adj[s];
                if (v <= u) continue;
                const uint32_t du = off[u + 1] - off[u], dv = off[v + 1] - off[v];
                tau[e++] = tau_for(lambda, (double)(du > dv ? du : dv), epsilon, max_truncation,
                                   clamped);
            }
    } else {
        uint32_t dmax = 0;
        for (uint32_t v = 0; v < n; ++v)
            if (off[v + 1] - off[v] > dmax) dmax = off[v + 1] - off[v];
        const uint32_t t = tau_for(lambda, (double)dmax, epsilon, max_truncation, clamped);
        for (uint64_t e = 0; e < m; ++e) tau[e] = t;
    }
    return 0;
}

/* aesc.hpp:103-110 */
double oracle_walks_needed_raw(int64_t tau_eff, double epsilon, double delta, uint32_t degree,
                               uint64_t m) {
    if (tau_eff <= 0) return 0.0;
    const double scale = 0.5 * epsilon * (double)degree;
    const double t = (double)tau_eff;
    return ceil((2.0 * t * t / (scale * scale)) * log(4.0 * (double)m / delta));
}

/* aesc.hpp:117-126 */
int oracle_walk_budget(uint32_t tau_eff, double epsilon, double delta, uint32_t degree,
                       uint64_t m, uint64_t* out) {
    if (tau_eff < 1 || degree < 1 || !(epsilon > 0.0 && epsilon < 1.0) ||
        !(delta > 0.0 && delta < 1.0))
        return 1;
    const double v = oracle_walks_needed_raw(tau_eff, epsilon, delta, degree, m);
    if (!(v < 9.0e18)) return 1;
    *out = (uint64_t)v;
    return 0;
}

/* aesc.hpp:362-374 */
static double source_budget_sum(const uint32_t* off, uint32_t src, const uint32_t* tau,
                                const uint32_t* slot_edge, double eps, double delta, uint64_t m,
                                uint32_t l) {
    const uint32_t deg = off[src + 1] - off[src];
    double total = 0.0;
    for (uint32_t s = off[src]; s < off[src] + deg; ++s)
        total += oracle_walks_needed_raw((int64_t)tau[slot_edge[s]] - (int64_t)l, eps, delta, deg,
                                         m);
    return total;
}

/* --------------------------------------------------------------- propagation
 * LandingPropagator (aesc.hpp:288-355): push in support discovery order,
 * support(l+1) = touched set, support degree sum exact. Dense zeroed arrays
 * replace the reference's epoch stamps (same values: aesc.hpp:338-340). */
typedef struct {
    double* val[2];
    char* in[2];
    uint32_t* sup[2];
    uint32_t nsup[2];
    int cur;
    uint64_t degsum;
} prop_ws;

static void prop_init(prop_ws* p, uint32_t n) {
    for (int s = 0; s < 2; ++s) {
        p->val[s] = (double*)calloc(n, sizeof(double));
        p->in[s] = (char*)calloc(n, 1);
        p->sup[s] = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
        p->nsup[s] = 0;
    }
}

static void prop_free(prop_ws* p) {
    for (int s = 0; s < 2; ++s) { free(p->val[s]); free(p->in[s]); free(p->sup[s]); }
}

static void prop_clear(prop_ws* p, int s) {
    for (uint32_t i = 0; i < p->nsup[s]; ++i) {
        p->val[s][p->sup[s][i]] = 0.0;
        p->in[s][p->sup[s][i]] = 0;
    }
    p->nsup[s] = 0;
}

/* aesc.hpp:290-301 */
static void prop_start(prop_ws* p, const uint32_t* off, uint32_t src) {
    prop_clear(p, 0);
    prop_clear(p, 1);
    p->cur = 0;
    p->sup[0][0] = src;
    p->nsup[0] = 1;
    p->val[0][src] = 1.0;
    p->in[0][src] = 1;
    p->degsum = off[src + 1] - off[src];
}

/* aesc.hpp:303-330 */
static void prop_step(prop_ws* p, const uint32_t* off, const uint32_t* adj) {
    const int c = p->cur, nx = 1 - c;
    prop_clear(p, nx);
    uint64_t degsum = 0;
    for (uint32_t i = 0; i < p->nsup[c]; ++i) {
        const uint32_t v = p->sup[c][i];
        const double share = p->val[c][v] / (double)(off[v + 1] - off[v]);
        for (uint32_t s = off[v]; s < off[v + 1]; ++s) {
            const uint32_t x = adj[s];
            if (!p->in[nx][x]) {
                p->in[nx][x] = 1;
                p->val[nx][x] = share;
                p->sup[nx][p->nsup[nx]++] = x;
                degsum += off[x + 1] - off[x];
            } else {
                p->val[nx][x] += share;
            }
        }
    }
    p->cur = nx;
    p->degsum = degsum;
}

#define PROB(p, v) ((p)->val[(p)->cur][v])

/* aesc.hpp:380-400 with the aesc_source hook (aesc.hpp:580-588) when g_hat != NULL */
static uint32_t advance_to_switch(prop_ws* p, const uint32_t* off, const uint32_t* adj,
                                  uint64_t m, uint32_t src, const uint32_t* tau,
                                  const uint32_t* slot_edge, double eps, double delta,
                                  int64_t cap, const double* inv_deg, double* g_hat) {
    uint32_t tau_src = 0;
    for (uint32_t s = off[src]; s < off[src + 1]; ++s)
        if (tau[slot_edge[s]] > tau_src) tau_src = tau[slot_edge[s]];
    uint32_t l = 0;
    while (l < tau_src && (cap < 0 || (int64_t)l < cap)) {
        if ((double)p->degsum >= source_budget_sum(off, src, tau, slot_edge, eps, delta, m, l))
            break;
        prop_step(p, off, adj);
        ++l;
        if (g_hat) {
            const double pi = PROB(p, src) * inv_deg[src];
            for (uint32_t s = off[src]; s < off[src + 1]; ++s) {
                if (l > tau[slot_edge[s]]) continue;
                const uint32_t j = adj[s];
                g_hat[s] += pi - PROB(p, j) * inv_deg[j];
            }
        }
    }
    return l;
}

void oracle_propagate(const uint32_t* off, const uint32_t* adj, uint32_t n, uint64_t m,
                      uint32_t source, const uint32_t* tau, const uint32_t* slot_edge,
                      double epsilon, double delta, int64_t cap, double* prob, uint32_t* depth) {
    prop_ws p;
    prop_init(&p, n);
    prop_start(&p, off, source);
    *depth = advance_to_switch(&p, off, adj, m, source, tau, slot_edge, epsilon, delta, cap, NULL,
                               NULL);
    memset(prob, 0, sizeof(double) * n);
    for (uint32_t i = 0; i < p.nsup[p.cur]; ++i) {
        const uint32_t v = p.sup[p.cur][i];
        prob[v] = PROB(&p, v);
    }
    prop_free(&p);
}

/* ------------------------------------------------------------- walk phase */

/* run_estimation_side + run_two_way_pairs (aesc.hpp:448-525), Saba/Hash
 * modes. Per-walk scores are order-free (aesc.hpp:439-441), so walks are
 * taken in k order; the (a_k - b_k)/n fold keeps the reference's k order,
 * which the 2^20 blocking (aesc.hpp:514-523) does not change. */
static double two_way_pairs(const uint32_t* off, const uint32_t* adj, uint64_t mult,
                            uint32_t vi, uint32_t vj, uint32_t len, uint64_t n_req,
                            uint64_t edge_seed, const double* rho) {
    const double inv_n = 1.0 / (double)n_req;
    double acc = 0.0;
    for (uint64_t k = 0; k < n_req; ++k) {
        double sc[2];
        for (uint32_t side = 0; side < 2; ++side) {
            const uint32_t seed = (uint32_t)(oracle_counter_hash(edge_seed, 2 * k + side) >> 32);
            uint32_t cur = side ? vj : vi;
            double a = 0.0;
            for (uint32_t l = 1; l < len; ++l) {
                cur = step_once(off, adj, cur, l, seed, mult);
                a += rho[cur];
            }
            sc[side] = a;
        }
        acc += (sc[0] - sc[1]) * inv_n;
    }
    return acc;
}

/* aesc.hpp:566-629 */
static int aesc_source(const uint32_t* off, const uint32_t* adj, uint32_t n, uint64_t m,
                       const oracle_aesc_config* cfg, const uint32_t* tau,
                       const uint32_t* slot_edge, const double* inv_deg, double bip_init,
                       uint32_t src, prop_ws* p, double* rho, double* g_hat,
                       uint32_t* tau_tilde, uint64_t* pairs, uint64_t* steps) {
    const uint32_t lo = off[src], hi = off[src + 1], deg_i = hi - lo;
    for (uint32_t s = lo; s < hi; ++s) g_hat[s] = inv_deg[src] + bip_init;
    prop_start(p, off, src);
    const uint32_t tt = advance_to_switch(p, off, adj, m, src, tau, slot_edge, cfg->epsilon,
                                          cfg->delta, cfg->switch_depth_cap, inv_deg, g_hat);
    tau_tilde[src] = tt;
    int any = 0;
    for (uint32_t s = lo; s < hi && !any; ++s) any = tau[slot_edge[s]] > tt;
    if (!any) return 0;

    for (uint32_t i = 0; i < p->nsup[p->cur]; ++i) {
        const uint32_t v = p->sup[p->cur][i];
        rho[v] = PROB(p, v) * inv_deg[v];
    }
    const uint64_t src_seed = oracle_substream(oracle_substream(cfg->master_seed, 0x41455343ull), src);
    int rc = 0;
    for (uint32_t s = lo; s < hi; ++s) {
        const int64_t tau_eff = (int64_t)tau[slot_edge[s]] - (int64_t)tt;
        if (tau_eff <= 0) continue;
        uint64_t n_req;
        if (oracle_walk_budget((uint32_t)tau_eff, cfg->epsilon, cfg->delta, deg_i, m, &n_req)) {
            rc = 1;
            break;
        }
        if (!(cfg->switch_depth_cap < 0 || n_req * (uint64_t)tau_eff <= (1ull << 26))) {
            rc = 1;
            break;
        }
        const uint64_t edge_seed = oracle_substream(src_seed, s);
        g_hat[s] += two_way_pairs(off, adj, cfg->hash_multiplier, src, adj[s],
                                  (uint32_t)(tau_eff + 1), n_req, edge_seed, rho);
        *pairs += n_req;
        *steps += 2 * n_req * (uint64_t)tau_eff;
    }
    for (uint32_t i = 0; i < p->nsup[p->cur]; ++i) rho[p->sup[p->cur][i]] = 0.0;
    return rc;
}

static uint32_t slot_of(const uint32_t* off, const uint32_t* adj, uint32_t u, uint32_t v) {
    return find_slot(off, adj, u, v);
}

/* aesc.hpp:636-708 */
int oracle_aesc(const uint32_t* off, const uint32_t* adj, uint32_t n, uint64_t m,
                const oracle_aesc_config* cfg, const uint32_t* sources, uint64_t nsources,
                double* g_hat, double* s_hat, uint32_t* tau, uint32_t* tau_tilde,
                double* lambda_hat, uint64_t* pairs_out, uint64_t* steps_out) {
    if (!(cfg->epsilon > 0.0 && cfg->epsilon < 1.0)) return 1;
    if (!(cfg->delta > 0.0 && cfg->delta < 1.0)) return 1;
    if (cfg->power_iterations < 1) return 1;
    if (!oracle_is_connected(off, adj, n)) return 2;

    int clamped = 0;
    int rc = oracle_truncated_lengths(off, adj, n, m, cfg->epsilon / 2.0, cfg->power_iterations,
                                      cfg->max_truncation, cfg->per_edge_tau, tau, lambda_hat,
                                      &clamped);
    if (rc) return rc;
    signed char* side = (signed char*)malloc(n);
    const int bip = oracle_bipartition(off, adj, n, side);
    free(side);
    uint32_t* slot_edge = (uint32_t*)malloc(sizeof(uint32_t) * 2 * m);
    oracle_slot_edges(off, adj, n, slot_edge);
    double* inv_deg = (double*)malloc(sizeof(double) * n);
    for (uint32_t v = 0; v < n; ++v) inv_deg[v] = 1.0 / (double)(off[v + 1] - off[v]);
    const double bip_init = bip ? 1.0 / (2.0 * (double)m) : 0.0;
    memset(g_hat, 0, sizeof(double) * 2 * m);
    memset(tau_tilde, 0, sizeof(uint32_t) * n);

    const uint64_t count = sources ? nsources : n;
    uint64_t pairs = 0, steps = 0;
    int fail = 0;
    int threads = cfg->threads;
#ifdef _OPENMP
    if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel num_threads(threads) reduction(+ : pairs, steps)
#endif
    {
        prop_ws p;
        prop_init(&p, n);
        double* rho = (double*)calloc(n, sizeof(double));
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
        for (int64_t i = 0; i < (int64_t)count; ++i) {
            const uint32_t src = sources ? sources[i] : (uint32_t)i;
            if (aesc_source(off, adj, n, m, cfg, tau, slot_edge, inv_deg, bip_init, src, &p,
                            rho, g_hat, tau_tilde, &pairs, &steps)) {
#ifdef _OPENMP
#pragma omp atomic write
#endif
                fail = 1;
            }
        }
        prop_free(&p);
        free(rho);
    }
    *pairs_out = pairs;
    *steps_out = steps;
    if (!fail && s_hat) {
        uint32_t e = 0;
        for (uint32_t u = 0; u < n; ++u)
            for (uint32_t s = off[u]; s < off[u + 1]; ++s) {
                const uint32_t v = adj[s];
                if (v <= u) continue;
                s_hat[e++] = g_hat[s] + g_hat[slot_of(off, adj, v, u)];
            }
    }
    free(slot_edge);
    free(inv_deg);
    return fail ? 1 : 0;
}

/* Walk-list range [r0, r1) of the flattened (vertex, k) list with K_v walks
 * per vertex (kpv == NULL: uniform K): the unit of the multi-GPU sharding
 * (SURVEY §8e). Counts of all ranges sum to oracle_campaign_counts. */
void oracle_campaign_range(const uint32_t* off, const uint32_t* adj, uint32_t n,
                           const uint64_t* kpv, uint64_t K, uint32_t length, uint64_t master,
                           uint64_t mult, uint64_t r0, uint64_t r1, uint64_t* counts) {
    memset(counts, 0, sizeof(uint64_t) * n);
    uint64_t base = 0;
    for (uint32_t v = 0; v < n; ++v) {
        const uint64_t kv = kpv ? kpv[v] : K;
        const uint64_t lo = base > r0 ? base : r0;
        const uint64_t hi = base + kv < r1 ? base + kv : r1;
        const uint64_t vseed = oracle_substream(master, v);
        for (uint64_t i = lo; i < hi; ++i) {
            const uint32_t seed = (uint32_t)(oracle_counter_hash(vseed, i - base) >> 32);
            uint32_t cur = v;
            ++counts[cur];
            for (uint32_t l = 1; l < length; ++l) {
                cur = step_once(off, adj, cur, l, seed, mult);
                ++counts[cur];
            }
        }
        base += kv;
    }
}
