/*
 * saba_cuda.h — C ABI of libsaba_cuda.so, the sm_100a (B200) implementation
 * of the Bouquets (SABA) walk engine and the TGT+ all-edges spanning
 * centrality (AESC) estimator of arXiv 2410.14056.
 *
 * The reference is a header-only C++ library with no plugin or FFI layer
 * (SURVEY §8b): its callers use the C++ API directly. This ABI is what that
 * API lands on; the headers under include/saba are the drop-in C++ surface built on it and
 * every entry point below names the reference interface it replaces
 * (paths relative to /root/reference/proj/include/saba).
 *
 * Conventions
 *   - plain pointers + sizes; no C++ or torch types;
 *   - host buffers are owned by the caller, read-only inputs / preallocated
 *     outputs; `*_device` variants take device pointers and a cudaStream_t
 *     passed as void*;
 *   - every function returns a status: SABA_OK, SABA_EINVAL (the reference
 *     throws std::invalid_argument: check_arg, common.hpp:14-16), SABA_EDATA
 *     (std::runtime_error: check_data, common.hpp:19-21), SABA_ECUDA;
 *     saba_cu_last_error() returns the (thread-local) message;
 *   - there is no CPU fallback: without a usable sm_100 device every compute
 *     entry point fails with SABA_ECUDA.
 */
#ifndef SABA_CUDA_H
#define SABA_CUDA_H

#include <stdint.h>

#if defined(__GNUC__)
#define SABA_API __attribute__((visibility("default")))
#else
#define SABA_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define SABA_OK 0
#define SABA_EINVAL 1
#define SABA_EDATA 2
#define SABA_ECUDA 3

#define SABA_MODE_NAIVE 0      /* WalkMode::Naive      (walker.hpp:30) — rejected on GPU */
#define SABA_MODE_VECTOR_MOD 1 /* WalkMode::VectorMod  — rejected on GPU */
#define SABA_MODE_HASH 2       /* WalkMode::Hash: unsorted seeds */
#define SABA_MODE_SABA 3       /* WalkMode::Saba: seed-sorted bouquets */

#define SABA_DEFAULT_HASH_MULTIPLIER 0xc6a4a7935bd1e995ull /* HashSpec, rng.hpp:20 */

SABA_API const char* saba_cu_last_error(void);
/* library / build identification, e.g. "saba_cuda sm_100a" */
SABA_API const char* saba_cu_version(void);
/* number of CUDA devices visible (0 on a CPU-only host) */
SABA_API int saba_cu_device_count(void);
/* Page-locked host memory for result buffers (counts, g_hat): copies into such
 * a buffer are direct DMA instead of a staged copy. No reference counterpart
 * (the reference has no device); free with saba_cu_pinned_free. */
SABA_API int saba_cu_pinned_alloc(uint64_t bytes, void** out);
SABA_API int saba_cu_pinned_free(void* p);

/* ======================================================================
 * Host graphs (graph.hpp:28-247, gen.hpp; BASELINE generators)
 * Canonicalisation follows Graph::from_edges (graph.hpp:86-105): self-loops
 * dropped, duplicates/reversals merged, slices sorted ascending.
 * ==================================================================== */
typedef struct saba_hgraph saba_hgraph;

/* Graph::from_edges. pairs = count (u,v) pairs, interleaved. */
SABA_API int saba_hgraph_from_edges(uint32_t n_hint, const uint32_t* pairs, uint64_t count,
                           saba_hgraph** out);
/* Adopt an existing sorted, symmetric, loop-free CSR (validated). */
SABA_API int saba_hgraph_from_csr(uint32_t n, const uint32_t* offsets, const uint32_t* adjacency,
                         saba_hgraph** out);
/* Erdős–Rényi G(n, m): m distinct non-loop pairs from a counter_hash stream. */
SABA_API int saba_gen_erdos_renyi(uint32_t n, uint64_t m, uint64_t seed, saba_hgraph** out);
/* R-MAT (a, b, c, d = 1-a-b-c), 2^scale vertices, edge_factor*2^scale samples;
 * symmetrised, deduplicated, loops removed; keep_lcc keeps the largest
 * connected component relabelled in ascending original id. */
SABA_API int saba_gen_rmat(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                  uint64_t seed, int keep_lcc, saba_hgraph** out);
/* Chung–Lu: n expected degrees drawn from a power law (pdf exponent gamma),
 * scaled to mean_degree, capped at max_degree after scaling; sum(w)/2 edge
 * samples with endpoints drawn proportional to w. */
SABA_API int saba_gen_chung_lu(uint32_t n, double gamma, double mean_degree, double max_degree,
                      uint64_t seed, int keep_lcc, saba_hgraph** out);
/* make_scale_free / make_random_connected (gen.hpp:17-69) — test graphs. */
SABA_API int saba_gen_scale_free(uint32_t n, uint32_t attach, uint64_t seed, saba_hgraph** out);
SABA_API int saba_gen_random_connected(uint32_t n, uint32_t extra, uint64_t seed, saba_hgraph** out);
SABA_API int saba_hgraph_largest_component(const saba_hgraph* in, saba_hgraph** out);
/* The same constructions on a device, bit-identical CSR:
 * Graph::from_edges (graph.hpp:86-105) as a device radix sort + unique of the
 * directed pairs, optionally reduced to the largest connected component
 * (device union-find); the R-MAT / Chung–Lu samplers above with their edge
 * samples drawn on the device. */
SABA_API int saba_cu_graph_from_edges(uint32_t n_hint, const uint32_t* pairs, uint64_t count, int keep_lcc,
                                      int device, saba_hgraph** out);
SABA_API int saba_cu_gen_rmat(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                              uint64_t seed, int keep_lcc, int device, saba_hgraph** out);
SABA_API int saba_cu_gen_chung_lu(uint32_t n, double gamma, double mean_degree, double max_degree,
                                  uint64_t seed, int keep_lcc, int device, saba_hgraph** out);
SABA_API uint32_t saba_hgraph_vertex_count(const saba_hgraph* g);
SABA_API uint64_t saba_hgraph_edge_count(const saba_hgraph* g);
/* borrow the handle's offsets[n+1] / adjacency[2m] (valid until saba_hgraph_free) */
SABA_API int saba_hgraph_data(const saba_hgraph* g, const uint32_t** offsets, const uint32_t** adjacency);
/* copy out offsets[n+1] and adjacency[2m] */
SABA_API int saba_hgraph_csr(const saba_hgraph* g, uint32_t* offsets, uint32_t* adjacency);
SABA_API void saba_hgraph_free(saba_hgraph* g);

/* ======================================================================
 * Device graphs (K0). The handle owns one replica of the CSR on `device`,
 * laid out as packed (base, degree) uint2 per vertex + uint32 adjacency,
 * plus host copies used by the truncation plan. Immutable, like Graph
 * (graph.hpp:24-27); not re-entrant.
 * ==================================================================== */
typedef struct saba_cu_graph saba_cu_graph;

SABA_API int saba_cu_graph_create(const uint32_t* offsets, const uint32_t* adjacency, uint32_t n,
                         uint64_t two_m, int device, saba_cu_graph** out);
/* Multi-device handle: one replica of the CSR on each of
 * devices[0..ndev) — repeats allowed (logical shards sharing one GPU, each
 * with its own replica and workspaces). The handle is the replica on
 * devices[0]. saba_cu_walk_campaign and saba_cu_aesc given such a handle run
 * one shard per replica, one host thread each, and combine once on
 * devices[0] (an NCCL reduce over NVLink when the devices are distinct and
 * libnccl.so.2 can be opened; peer copies + an add kernel otherwise). The
 * results are bit-identical to a one-device run: counts are integer sums and
 * every g_hat slot has a single writer. The C++ drop-in maps
 * CampaignConfig/AescConfig::threads to the device count (walker.hpp:372,
 * aesc.hpp:47: 0 = all). */
SABA_API int saba_cu_graph_create_multi(const uint32_t* offsets, const uint32_t* adjacency, uint32_t n,
                                        uint64_t two_m, const int* devices, int ndev, saba_cu_graph** out);
SABA_API int saba_cu_graph_replica_count(const saba_cu_graph* g);
SABA_API int saba_cu_graph_destroy(saba_cu_graph* g);
SABA_API uint32_t saba_cu_graph_vertex_count(const saba_cu_graph* g);
SABA_API uint64_t saba_cu_graph_edge_count(const saba_cu_graph* g);

/* ======================================================================
 * Walks (walker.hpp:188-203, 207-236, 283-338)
 * ==================================================================== */

/* random_walk / random_bouquet lanes: count walks; walk i starts at
 * starts[i] with seed seeds[i]; paths_out[i*length + l] = vertex at step l.
 * Validation mirrors require_walkable (walker.hpp:270-274). */
SABA_API int saba_cu_walk_paths(saba_cu_graph* g, const uint32_t* starts, const uint32_t* seeds,
                       uint64_t count, uint32_t length, uint64_t hash_multiplier,
                       uint32_t* paths_out);

/* CampaignConfig (walker.hpp:367-376) plus the two campaign shapes:
 *   total_walks == 0 : exactly walks_per_vertex walks from every vertex
 *                      (run_walk_campaign, walker.hpp:456-538);
 *   total_walks  > 0 : uniform-random starts: K_v walks of v,
 *                      walk k of v seeded counter_hash(substream(master,v),k)>>32.
 * Sharding: the flattened (vertex, k) walk list is cut into shard_count equal
 * contiguous ranges; this call runs range shard_index. Summing the counts of
 * all shards gives exactly the unsharded counts (any shard_count). */
typedef struct {
    uint64_t walks_per_vertex;
    uint64_t total_walks;
    uint32_t length;
    uint32_t lanes;
    int32_t mode;
    int32_t threads; /* accepted for parity; the GPU ignores it */
    uint64_t master_seed;
    uint64_t hash_multiplier;
    uint32_t shard_index;
    uint32_t shard_count;
} saba_cu_campaign_config;

/* CampaignReport (walker.hpp:383-391) + device-side detail. */
typedef struct {
    double seconds;        /* wall time of the device work (events) */
    uint64_t total_steps;  /* walks * (L-1) over the whole campaign */
    uint64_t total_events; /* walks * L */
    uint64_t shard_walks;  /* walks executed by this call */
    uint64_t shard_steps;  /* their steps */
    double walk_kernel_ms; /* K2 alone */
    uint32_t launches;     /* kernels launched by this call */
    uint32_t kernel;       /* K2 variant that ran: SABA_K2_* */
} saba_cu_campaign_report;
#define SABA_K2_NONE 0     /* length 1: no steps */
#define SABA_K2_GENERIC 1  /* walk_count_kernel: csr + neighbour gathers, L2 reductions */
#define SABA_K2_FAT 2      /* walk_count_fat_kernel: one gather per step (L2-resident graphs) */
#define SABA_K2_HOT 3      /* walk_count_hot_kernel: 32-bit hub counters in shared memory */
#define SABA_K2_RANK 4     /* walk_count_rank_kernel: hub records + 16-bit hub counters in shared memory */
#define SABA_K2_FAT_PRIV 5 /* walk_count_fat_priv_kernel: every counter in shared memory (small graphs) */

/* Visit counts (VisitCountSink, walker.hpp:352-365) copied to host counts[n]. */
SABA_API int saba_cu_walk_campaign(saba_cu_graph* g, const saba_cu_campaign_config* cfg,
                          uint64_t* counts_out, saba_cu_campaign_report* report);
/* Device-resident variant: counts_dev (n uint64 on the graph's device) is
 * ACCUMULATED into (callers zero it), all work is enqueued on `stream`
 * (cudaStream_t; NULL = legacy default stream) and the call returns without
 * synchronising; report->seconds / walk_kernel_ms are 0 unless timing != 0
 * (which synchronises). */
SABA_API int saba_cu_walk_campaign_device(saba_cu_graph* g, const saba_cu_campaign_config* cfg,
                                 uint64_t* counts_dev, void* stream, int timing,
                                 saba_cu_campaign_report* report);

/* Shared-memory tables of the handle's last campaign launch: how many of the
 * highest-degree vertices had their {base, degree} record (records) and their
 * visit counter (counters) on the SM. 0 / 0 for the kernels without tables.
 * Diagnostic for bench lines (walker.hpp:352-365 has no counterpart). */
SABA_API int saba_cu_campaign_tables(const saba_cu_graph* g, uint32_t* records, uint32_t* counters);

/* rng_stream (stream.hpp:29-83): the raw 32-bit pre-selection words
 * seed ^ h(cur, l) of walks_per_vertex walks from each start, step-major per
 * start (walk k's word of step l at index (l-1)*K + k of its start's block).
 * selector: 1 = xor-mod, 2 = scaled (0 = the LCG baseline is rejected).
 * *nwords = nstarts*K*(length-1); words_out may be NULL when length == 1. */
SABA_API int saba_cu_rng_stream(saba_cu_graph* g, const uint32_t* starts, uint32_t nstarts,
                                uint64_t walks_per_vertex, uint32_t length, int selector,
                                uint64_t master_seed, uint64_t hash_multiplier,
                                uint32_t* words_out, uint64_t* nwords);

/* Branching statistics of the campaign's bouquets (BranchCollector,
 * walker.hpp:64-109 as driven by campaign_vertex_scaled, 430-449): bouquets
 * are `lanes` consecutive entries of each start vertex's (Saba: sorted) seed
 * list; per bouquet step the distinct lane vertices are counted.
 * histogram_out[lanes+1], per_step_out[length-1] (distinct-access proxy,
 * bench.hpp:45-50), totals_out[4] = {total_distinct, samples, lane_steps,
 * degree_sum}. length > 1. A shard (shard_index of shard_count) covers the
 * start vertices v with v % shard_count == shard_index; the shards' outputs
 * add up to the unsharded statistics exactly (integer sums). */
SABA_API int saba_cu_branching_stats(saba_cu_graph* g, const saba_cu_campaign_config* cfg,
                                     uint64_t* histogram_out, uint64_t* per_step_out,
                                     uint64_t* totals_out);

/* ======================================================================
 * TGT+ AESC (aesc.hpp)
 * ==================================================================== */

/* AescConfig (aesc.hpp:40-53). */
typedef struct {
    double epsilon;
    double delta;
    uint32_t power_iterations;
    uint32_t candidate_nodes; /* accepted, unused (aesc.hpp:44) */
    int32_t mode;
    int32_t threads;          /* accepted; GPU ignores */
    uint64_t master_seed;
    uint32_t lanes;
    uint32_t max_truncation;
    int32_t per_edge_tau;
    int32_t workers;          /* extension: batch workers per device (0 = auto; results unchanged) */
    int64_t switch_depth_cap;
    uint64_t hash_multiplier;
} saba_cu_aesc_config;

typedef struct {
    double seconds;            /* device work of the estimator (all phases) */
    double plan_seconds;       /* host truncation plan */
    double propagation_ms;     /* K3 */
    double walk_ms;            /* K4 (+ reduction) */
    uint64_t total_walk_pairs; /* CentralityEstimate counters (aesc.hpp:92-93) */
    uint64_t total_walk_steps;
    uint64_t edge_visits;      /* propagation edge-visits actually executed */
    uint64_t sources;          /* sources processed */
    double lambda_hat;
    int32_t bipartite;
    int32_t clamped;
    uint32_t max_tau;
    uint32_t launches;
    uint32_t replicas;         /* device replicas that ran shards of this call */
    uint32_t workers;          /* batch workers per replica */
    double walk_kernel_ms;     /* K4 walk kernels alone (events around each launch), summed */
    double setup_seconds;      /* per-call setup between the plan and the first batch (slot records,
                                  workspaces, tau upload): like the plan, not per-source work */
} saba_cu_aesc_report;

/* walk_budget (aesc.hpp:117-126). */
SABA_API int saba_cu_walk_budget(uint32_t tau_effective, double epsilon, double delta, uint32_t degree,
                        uint64_t edge_count, uint64_t* out);
/* truncated_lengths (aesc.hpp:210-248): tau_out[m] per edge id. */
SABA_API int saba_cu_truncated_lengths(saba_cu_graph* g, double epsilon, uint32_t power_iterations,
                              uint32_t max_truncation, int per_edge, uint32_t* tau_out,
                              double* lambda_hat, int* clamped);

/* aesc (aesc.hpp:636-708). sources == NULL: every vertex (the full
 * estimator); otherwise only the listed sources (deduplicated: a repeated
 * source is idempotent, as in the reference's per-source loop; their g_hat
 * slots and tau_tilde entries; others left 0, s_hat not formed). Outputs
 * (host): g_hat[2m] per directed slot, s_hat[m] per edge id (may be NULL),
 * tau[m], tau_tilde[n]. Sharding: shard shard_index of shard_count runs the
 * sources saba_cu_aesc_shard_sources returns; every source runs on exactly one
 * shard, so summing the shards' g_hat is exact (single writer per slot). */
SABA_API int saba_cu_aesc(saba_cu_graph* g, const saba_cu_aesc_config* cfg, const uint32_t* sources,
                 uint64_t source_count, uint32_t shard_index, uint32_t shard_count,
                 double* g_hat_out, double* s_hat_out, uint32_t* tau_out,
                 uint32_t* tau_tilde_out, saba_cu_aesc_report* report);

/* aesc with the estimate left on the device, for callers that combine
 * shards themselves (one process per GPU: an NCCL all-reduce of g_hat_dev is
 * exact, each slot having one writer) and then form s_hat with
 * saba_cu_symmetrise. g_hat_dev: 2m doubles on g's device, fully written
 * (0 outside this shard's sources' slots), ordered on `stream`; tau_out[m]
 * and tau_tilde_out[n] are host outputs and may be NULL. */
SABA_API int saba_cu_aesc_device(saba_cu_graph* g, const saba_cu_aesc_config* cfg, const uint32_t* sources,
                                 uint64_t source_count, uint32_t shard_index, uint32_t shard_count,
                                 double* g_hat_dev, uint32_t* tau_out, uint32_t* tau_tilde_out, void* stream,
                                 saba_cu_aesc_report* report);
/* K5 (aesc.hpp:702-706) on device buffers: s_hat_dev[e] = g_hat_dev[u->v] +
 * g_hat_dev[v->u] for every edge id e = {u, v}; enqueued on `stream`. */
SABA_API int saba_cu_symmetrise(saba_cu_graph* g, const double* g_hat_dev, double* s_hat_dev, void* stream);

/* The distinct sources shard shard_index of shard_count runs (sources ==
 * NULL: all vertices; host-only, needs no device): cost-stratified — ascending degree (the walk work of
 * a source is ~tau^3/d at a uniform tau, aesc.hpp:103-110), dealt to the
 * shards in snake order. out may be NULL to query *out_count. */
SABA_API int saba_aesc_shard_sources(const uint32_t* offsets, uint32_t n, const uint32_t* sources,
                                     uint64_t source_count, uint32_t shard_index, uint32_t shard_count,
                                     uint32_t* out, uint64_t* out_count);

/* propagate_landing_probabilities (aesc.hpp:406-422): dense prob_out[n] at
 * the switch depth; *depth_out = tau~. tau[m] per edge id. */
SABA_API int saba_cu_propagate(saba_cu_graph* g, uint32_t source, const uint32_t* tau, double epsilon,
                      double delta, int64_t switch_depth_cap, double* prob_out,
                      uint32_t* depth_out);

/* estimate_edge (aesc.hpp:533-553) with a dense landing vector prob[n]. */
SABA_API int saba_cu_estimate_edge(saba_cu_graph* g, uint32_t v_i, uint32_t v_j, const double* prob,
                          uint32_t tau_eff, uint64_t n_req, int mode, uint64_t edge_seed,
                          uint32_t lanes, uint64_t hash_multiplier, double* out);

#ifdef __cplusplus
}
#endif
#endif /* SABA_CUDA_H */
