/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference's Bouquets /
 * TGT+ AESC hot path, used as the parity checker for the sm_100a product.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load it. The product never links or calls it.
 *
 * Parity is pinned: tests/test_oracle_golden.py checks every function below
 * against golden vectors produced by the reference itself, compiled unchanged
 * from /root/reference/proj/include (oracle/ref_driver.cpp -> oracle/_ref/).
 *
 * Graphs are raw CSR: offsets[n+1], adjacency[2m] with sorted neighbour slices
 * (graph.hpp:199-237 layout).
 */
#ifndef SABA_ORACLE_H
#define SABA_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* common.hpp:24-41, rng.hpp:20-31, rng.hpp:61-63 */
uint64_t oracle_mix64(uint64_t x);
uint64_t oracle_counter_hash(uint64_t master, uint64_t index);
uint64_t oracle_substream(uint64_t master, uint64_t tag);
uint32_t oracle_hash_state(uint64_t multiplier, uint32_t vertex, uint32_t step);
uint32_t oracle_scaled_index(uint32_t raw, uint32_t degree);

/* walker.hpp:188-203 (walk_stream_hashed<Scaled>) as used by random_walk
 * (walker.hpp:283-302). Writes `length` vertices. */
void oracle_random_walk(const uint32_t* off, const uint32_t* adj, uint32_t start,
                        uint32_t length, uint32_t seed, uint64_t mult, uint32_t* path);

/* Visit counts of the Saba/Hash campaign (walker.hpp:430-449, 456-538):
 * walks k = 0..K_v-1 from every v with seed counter_hash(substream(master,v),k)>>32.
 * k_per_vertex == NULL means uniform K.  counts[n] is overwritten.
 * Sorting is omitted: counts are order-invariant (walker.hpp:25-26,
 * test_walker.cpp:147-151). threads <= 0 -> all. */
void oracle_campaign_counts(const uint32_t* off, const uint32_t* adj, uint32_t n,
                            const uint64_t* k_per_vertex, uint64_t K, uint32_t length,
                            uint64_t master, uint64_t mult, int threads, uint64_t* counts);

/* Range [r0, r1) of the flattened (vertex, k) walk list (sharding unit). */
void oracle_campaign_range(const uint32_t* off, const uint32_t* adj, uint32_t n,
                           const uint64_t* k_per_vertex, uint64_t K, uint32_t length,
                           uint64_t master, uint64_t mult, uint64_t r0, uint64_t r1,
                           uint64_t* counts);

/* Uniform-random starts: K_v = #{w < W : scaled_index(
 * counter_hash(substream(master,0x5354415254), w)>>32, n) == v}. */
void oracle_uniform_start_counts(uint32_t n, uint64_t W, uint64_t master, uint64_t* k_out);

/* ---- AESC (aesc.hpp) ---- */
int oracle_is_connected(const uint32_t* off, const uint32_t* adj, uint32_t n);
/* returns 1 if bipartite and fills side[n] (graph.hpp:271-292) */
int oracle_bipartition(const uint32_t* off, const uint32_t* adj, uint32_t n, signed char* side);
/* slot -> undirected edge id, ids in sorted (u<v) order (graph.hpp:86-105, 199-237) */
void oracle_slot_edges(const uint32_t* off, const uint32_t* adj, uint32_t n, uint32_t* slot_edge);

double oracle_estimate_decay(const uint32_t* off, const uint32_t* adj, uint32_t n, uint64_t m,
                             uint32_t iterations, int bipartite, const signed char* side);
/* truncated_lengths (aesc.hpp:210-248). tau[m]. returns 0 ok, 1 bad arg, 2 data */
int oracle_truncated_lengths(const uint32_t* off, const uint32_t* adj, uint32_t n, uint64_t m,
                             double epsilon, uint32_t omega, uint32_t max_truncation,
                             int per_edge, uint32_t* tau, double* lambda_hat, int* clamped);
double oracle_walks_needed_raw(int64_t tau_eff, double epsilon, double delta, uint32_t degree,
                               uint64_t m);
/* returns 0 ok / 1 invalid argument; aesc.hpp:117-126 */
int oracle_walk_budget(uint32_t tau_eff, double epsilon, double delta, uint32_t degree,
                       uint64_t m, uint64_t* out);

typedef struct {
    double epsilon, delta;
    uint32_t power_iterations;
    uint64_t master_seed;
    uint32_t max_truncation;
    int per_edge_tau;
    int64_t switch_depth_cap;
    uint64_t hash_multiplier;
    int threads;
} oracle_aesc_config;

/* Landing probabilities after advance_to_switch (aesc.hpp:406-422): prob[n]
 * dense (0 outside support), returns tau~ in *depth. */
void oracle_propagate(const uint32_t* off, const uint32_t* adj, uint32_t n, uint64_t m,
                      uint32_t source, const uint32_t* tau, const uint32_t* slot_edge,
                      double epsilon, double delta, int64_t cap, double* prob,
                      uint32_t* depth);

/* Full aesc() (aesc.hpp:636-708) or, with sources != NULL, aesc_source()
 * over the listed sources only (other slots of g_hat left 0).  s_hat may be
 * NULL. Returns 0 ok, 1 invalid argument, 2 data error. */
int oracle_aesc(const uint32_t* off, const uint32_t* adj, uint32_t n, uint64_t m,
                const oracle_aesc_config* cfg, const uint32_t* sources, uint64_t nsources,
                double* g_hat, double* s_hat, uint32_t* tau, uint32_t* tau_tilde,
                double* lambda_hat, uint64_t* pairs, uint64_t* steps);

/* BASELINE generators (oracle_gen.c): CSR identical to the product's
 * saba_gen_* / saba_cu_gen_*; release with oracle_csr_free. Return 0 ok,
 * 1 invalid argument. */
typedef struct {
    uint32_t n;
    uint64_t m;
    uint32_t* off;
    uint32_t* adj;
} oracle_csr;
void oracle_csr_free(oracle_csr* g);
int oracle_gen_erdos_renyi(uint32_t n, uint64_t m, uint64_t seed, oracle_csr* out);
int oracle_gen_rmat(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                    uint64_t seed, int keep_lcc, oracle_csr* out);
int oracle_gen_chung_lu(uint32_t n, double gamma, double mean_degree, double max_degree,
                        uint64_t seed, int keep_lcc, oracle_csr* out);

#ifdef __cplusplus
}
#endif
#endif
