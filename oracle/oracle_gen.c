/*
 * TEST INFRASTRUCTURE ONLY — plain-C restatement of the BASELINE graph
 * generators (Erdős–Rényi G(n,m), R-MAT, Chung–Lu) and of the reference's
 * canonicalisation Graph::from_edges / build_csr (graph.hpp:86-105, 199-237)
 * plus the largest-connected-component reduction.
 *
 * The reference has no generator for these graphs; the product
 * builds them in paper_2410_14056_b200/csrc/graph_host.cpp (host) and
 * graph_build.cu (device). This file exists so that the reference arm of
 * bench.py (`--impl reference`) and the CPU checkers can build the identical
 * CSR without loading the product library: tests/test_oracle_golden.py pins
 * it against the product's generators bit for bit.
 *
 * Seeded streams: counter_hash / substream (common.hpp:24-41), restated in
 * saba_oracle.c. The float64 Chung–Lu weights use the same libm pow and the
 * same operation order as the product (no FMA: -ffp-contract=off).
 */
#include "saba_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static uint64_t pack_pair(uint32_t a, uint32_t b) {
    if (a > b) {
        uint32_t t = a;
        a = b;
        b = t;
    }
    return ((uint64_t)a << 32) | b;
}

/* LSD radix sort of the low `bits` bits, 11 bits per pass (OpenMP histogram). */
static void radix_sort(uint64_t* keys, uint64_t N, int bits) {
    enum { D = 11, R = 1 << D };
    uint64_t* const tmp = (uint64_t*)malloc(sizeof(uint64_t) * (N ? N : 1));
    int T = 1;
#ifdef _OPENMP
    T = omp_get_max_threads();
#endif
    uint64_t* hist = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)T * R);
    uint64_t *src = keys, *dst = tmp;
    for (int shift = 0; shift < bits; shift += D) {
        memset(hist, 0, sizeof(uint64_t) * (size_t)T * R);
#pragma omp parallel num_threads(T)
        {
            int t = 0;
#ifdef _OPENMP
            t = omp_get_thread_num();
#endif
            const uint64_t lo = N * (uint64_t)t / (uint64_t)T, hi = N * (uint64_t)(t + 1) / (uint64_t)T;
            uint64_t* h = hist + (size_t)t * R;
            for (uint64_t i = lo; i < hi; ++i) ++h[(src[i] >> shift) & (R - 1)];
#pragma omp barrier
#pragma omp single
            {
                uint64_t run = 0;
                for (int d = 0; d < R; ++d)
                    for (int tt = 0; tt < T; ++tt) {
                        const uint64_t c = hist[(size_t)tt * R + d];
                        hist[(size_t)tt * R + d] = run;
                        run += c;
                    }
            }
            for (uint64_t i = lo; i < hi; ++i) dst[h[(src[i] >> shift) & (R - 1)]++] = src[i];
        }
        uint64_t* sw = src;
        src = dst;
        dst = sw;
    }
    if (src != keys) memcpy(keys, src, sizeof(uint64_t) * N);
    free(tmp);
    free(hist);
}

static int bits_for(uint64_t x) {
    int b = 1;
    while (b < 64 && ((uint64_t)1 << b) <= x) ++b;
    return b;
}

/* CSR of sorted unique (u<<32 | v), u < v < n: graph.hpp:199-237 fills the
 * slices in edge order, which for sorted edges is already ascending. */
static void csr_from_keys(uint32_t n, const uint64_t* keys, uint64_t m, oracle_csr* out) {
    out->n = n;
    out->m = m;
    out->off = (uint32_t*)calloc((size_t)n + 1, sizeof(uint32_t));
    out->adj = (uint32_t*)malloc(sizeof(uint32_t) * (2 * m ? 2 * m : 1));
    for (uint64_t i = 0; i < m; ++i) {
        ++out->off[(keys[i] >> 32) + 1];
        ++out->off[(keys[i] & 0xffffffffu) + 1];
    }
    for (uint32_t u = 0; u < n; ++u) out->off[u + 1] += out->off[u];
    uint32_t* cur = (uint32_t*)malloc(sizeof(uint32_t) * ((size_t)n + 1));
    memcpy(cur, out->off, sizeof(uint32_t) * n);
    for (uint64_t i = 0; i < m; ++i) {
        const uint32_t u = (uint32_t)(keys[i] >> 32), v = (uint32_t)keys[i];
        out->adj[cur[u]++] = v;
        out->adj[cur[v]++] = u;
    }
    free(cur);
}

/* Graph::from_edges (graph.hpp:86-105): loops dropped, pairs canonicalised
 * (min, max), sorted, deduplicated. keys: packed pairs (consumed). */
static void from_pairs(uint32_t n_hint, uint64_t* keys, uint64_t count, oracle_csr* out) {
    uint32_t n = n_hint;
    uint64_t w = 0;
    for (uint64_t i = 0; i < count; ++i) {
        const uint32_t a = (uint32_t)(keys[i] >> 32), b = (uint32_t)keys[i];
        if (b + 1 > n) n = b + 1;
        if (a != b) keys[w++] = keys[i];
    }
    radix_sort(keys, w, 32 + bits_for(n));
    uint64_t u = 0;
    for (uint64_t i = 0; i < w; ++i)
        if (u == 0 || keys[i] != keys[u - 1]) keys[u++] = keys[i];
    csr_from_keys(n, keys, u, out);
}

/* Largest connected component (BFS in ascending root order, first largest
 * wins), relabelled in ascending original id (monotone: edge order kept). */
static void largest_component(const oracle_csr* g, oracle_csr* out) {
    const uint32_t n = g->n;
    uint32_t* comp = (uint32_t*)malloc(sizeof(uint32_t) * n);
    uint32_t* queue = (uint32_t*)malloc(sizeof(uint32_t) * n);
    memset(comp, 0xff, sizeof(uint32_t) * n);
    uint32_t best = 0, best_size = 0, ncomp = 0;
    for (uint32_t r = 0; r < n; ++r) {
        if (comp[r] != 0xffffffffu) continue;
        uint32_t qn = 0;
        queue[qn++] = r;
        comp[r] = ncomp;
        for (uint32_t h = 0; h < qn; ++h) {
            const uint32_t x = queue[h];
            for (uint32_t s = g->off[x]; s < g->off[x + 1]; ++s)
                if (comp[g->adj[s]] == 0xffffffffu) {
                    comp[g->adj[s]] = ncomp;
                    queue[qn++] = g->adj[s];
                }
        }
        if (qn > best_size) {
            best_size = qn;
            best = ncomp;
        }
        ++ncomp;
    }
    uint32_t* id = queue; /* reuse */
    uint32_t k = 0;
    for (uint32_t v = 0; v < n; ++v) id[v] = comp[v] == best ? k++ : 0xffffffffu;
    uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (g->m ? g->m : 1));
    uint64_t m = 0;
    for (uint32_t x = 0; x < n; ++x) {
        if (comp[x] != best) continue;
        for (uint32_t s = g->off[x]; s < g->off[x + 1]; ++s)
            if (g->adj[s] > x) keys[m++] = ((uint64_t)id[x] << 32) | id[g->adj[s]];
    }
    csr_from_keys(k, keys, m, out);
    free(keys);
    free(comp);
    free(queue);
}

static void finish(oracle_csr* g, int keep_lcc) {
    if (!keep_lcc) return;
    oracle_csr l;
    largest_component(g, &l);
    oracle_csr_free(g);
    *g = l;
}

void oracle_csr_free(oracle_csr* g) {
    free(g->off);
    free(g->adj);
    g->off = NULL;
    g->adj = NULL;
}

/* G(n, m): pairs (scaled_index(h>>32, n), scaled_index(h, n)) of
 * counter_hash(substream(seed, "ERDR"), i), loops skipped, the first m
 * distinct unordered pairs kept (open-addressing set). */
int oracle_gen_erdos_renyi(uint32_t n, uint64_t m, uint64_t seed, oracle_csr* out) {
    if (n < 2 || m > (uint64_t)n * (n - 1) / 2) return 1;
    const uint64_t s = oracle_substream(seed, 0x45524452ull);
    uint64_t cap = 16;
    while (cap < 4 * m) cap <<= 1;
    uint64_t* set = (uint64_t*)malloc(sizeof(uint64_t) * cap);
    memset(set, 0xff, sizeof(uint64_t) * cap);
    uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (m ? m : 1));
    uint64_t got = 0;
    for (uint64_t i = 0; got < m; ++i) {
        const uint64_t h = oracle_counter_hash(s, i);
        const uint32_t a = oracle_scaled_index((uint32_t)(h >> 32), n);
        const uint32_t b = oracle_scaled_index((uint32_t)h, n);
        if (a == b) continue;
        const uint64_t k = pack_pair(a, b);
        uint64_t slot = oracle_mix64(k) & (cap - 1);
        int fresh = 1;
        while (set[slot] != ~0ull) {
            if (set[slot] == k) {
                fresh = 0;
                break;
            }
            slot = (slot + 1) & (cap - 1);
        }
        if (!fresh) continue;
        set[slot] = k;
        keys[got++] = k;
    }
    free(set);
    from_pairs(n, keys, m, out);
    free(keys);
    return 0;
}

/* R-MAT: sample i's endpoints from counter_hash(counter_hash(s, i), lvl)
 * words, two levels per hash (high word first), quadrant by 32-bit
 * thresholds (a, a+b, a+b+c) * 2^32, high bit first. */
int oracle_gen_rmat(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                    uint64_t seed, int keep_lcc, oracle_csr* out) {
    if (scale < 1 || scale > 31 || edge_factor < 1) return 1;
    const uint64_t samples = (uint64_t)edge_factor << scale;
    const uint64_t s = oracle_substream(seed, 0x524d4154ull);
    const double two32 = 4294967296.0;
    const uint64_t ta = (uint64_t)(a * two32), tb = (uint64_t)((a + b) * two32),
                   tc = (uint64_t)((a + b + c) * two32);
    uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * samples);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)samples; ++i) {
        uint32_t u = 0, v = 0;
        const uint64_t si = oracle_counter_hash(s, (uint64_t)i);
        for (uint32_t lvl = 0; lvl < scale; lvl += 2) {
            const uint64_t h = oracle_counter_hash(si, lvl);
            for (uint32_t q = 0; q < 2 && lvl + q < scale; ++q) {
                const uint64_t r = q ? (h & 0xffffffffu) : (h >> 32);
                const uint32_t bit = 1u << (scale - 1 - (lvl + q));
                if (r < ta) {
                } else if (r < tb) {
                    v |= bit;
                } else if (r < tc) {
                    u |= bit;
                } else {
                    u |= bit;
                    v |= bit;
                }
            }
        }
        keys[i] = pack_pair(u, v);
    }
    from_pairs(1u << scale, keys, samples, out);
    free(keys);
    finish(out, keep_lcc);
    return 0;
}

static double unit53(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }

static double capped_mean(const double* w, uint32_t n, double c, double cap) {
    double s = 0.0;
    for (uint32_t i = 0; i < n; ++i) {
        const double x = w[i] * c;
        s += cap < x ? cap : x;
    }
    return s / (double)n;
}

/* Chung–Lu: Pareto weights U^(-1/(gamma-1)), scaled by bisection so the mean
 * of the capped weights is mean_degree, a Vose alias table over them, and
 * round(sum w / 2) samples whose endpoints are drawn through the table. */
int oracle_gen_chung_lu(uint32_t n, double gamma, double mean_degree, double max_degree,
                        uint64_t seed, int keep_lcc, oracle_csr* out) {
    if (n < 2 || !(gamma > 1.0) || !(mean_degree > 0) || !(max_degree >= 1)) return 1;
    const uint64_t s = oracle_substream(seed, 0x43484c55ull);
    double* w = (double*)malloc(sizeof(double) * n);
    const double ex = -1.0 / (gamma - 1.0);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; ++i) w[i] = pow(1.0 - unit53(oracle_counter_hash(s, (uint64_t)i)), ex);
    double lo = 0.0, hi = 1.0;
    while (capped_mean(w, n, hi, max_degree) < mean_degree && hi < 1e30) hi *= 2.0;
    if (capped_mean(w, n, hi, max_degree) < mean_degree) {
        free(w);
        return 1;
    }
    for (int it = 0; it < 100; ++it) {
        const double mid = 0.5 * (lo + hi);
        if (capped_mean(w, n, mid, max_degree) < mean_degree) lo = mid; else hi = mid;
    }
    double total = 0.0;
    for (uint32_t i = 0; i < n; ++i) {
        const double x = w[i] * hi;
        w[i] = max_degree < x ? max_degree : x;
        total += w[i];
    }
    double* prob = (double*)malloc(sizeof(double) * n);
    uint32_t* alias = (uint32_t*)calloc(n, sizeof(uint32_t));
    uint32_t* small = (uint32_t*)malloc(sizeof(uint32_t) * n);
    uint32_t* large = (uint32_t*)malloc(sizeof(uint32_t) * n);
    uint32_t ns = 0, nl = 0;
    for (uint32_t i = 0; i < n; ++i) {
        prob[i] = w[i] * (double)n / total;
        if (prob[i] < 1.0) small[ns++] = i; else large[nl++] = i;
    }
    while (ns && nl) {
        const uint32_t l = small[--ns], g = large[nl - 1];
        alias[l] = g;
        prob[g] = (prob[g] + prob[l]) - 1.0;
        if (prob[g] < 1.0) {
            --nl;
            small[ns++] = g;
        }
    }
    for (uint32_t i = 0; i < nl; ++i) prob[large[i]] = 1.0;
    for (uint32_t i = 0; i < ns; ++i) prob[small[i]] = 1.0;
    const uint64_t samples = (uint64_t)llround(total / 2.0);
    const uint64_t s2 = oracle_substream(seed, 0x43484c32ull);
    uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (samples ? samples : 1));
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)samples; ++i) {
        uint32_t e[2];
        for (int k = 0; k < 2; ++k) {
            const uint64_t h = oracle_counter_hash(s2, 2 * (uint64_t)i + (uint64_t)k);
            const uint32_t col = oracle_scaled_index((uint32_t)(h >> 32), n);
            const double coin = (double)(uint32_t)h * 0x1.0p-32;
            e[k] = coin < prob[col] ? col : alias[col];
        }
        keys[i] = pack_pair(e[0], e[1]);
    }
    from_pairs(n, keys, samples, out);
    free(keys);
    free(w);
    free(prob);
    free(alias);
    free(small);
    free(large);
    finish(out, keep_lcc);
    return 0;
}
