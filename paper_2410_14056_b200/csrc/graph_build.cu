// Graph ingest on the device: Graph::from_edges
// canonicalisation (graph.hpp:86-105, build_csr 199-237), the largest
// connected component, and the BASELINE R-MAT / Chung–Lu samplers, producing
// the same CSR, bit for bit, as the host path in graph_host.cpp.
//
//   G1 gb_directed      sample i -> directed keys (a<<32|b), (b<<32|a); self
//                       loops become a sentinel that sorts after every vertex
//   G2 CUB radix sort   of the 2·samples u64 keys over 32 + bits(n) bits
//   G3 CUB unique       duplicates / reversals merge (both directions present)
//   G4 gb_offsets       CSR offsets from the sorted run boundaries; slot s of
//                       the adjacency is the low word of key s, so every
//                       neighbour slice comes out ascending
//   G5 gb_hook/gb_components  connected components by lock-free union-find
//                       (larger root hooked under smaller, CAS), so each root
//                       is its component's minimum vertex
//   G6 gb_sizes + max   component sizes; the largest wins, ties to the
//                       smallest root — the host BFS's first-found maximum
//   G7 gb_relabel       ids in ascending original order inside the LCC
//                       (monotone, so the key order survives) and compaction
//
// Everything between the input upload and the CSR download is device
// resident; the host copy of the result is what Graph (graph.hpp) holds.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <vector>

#include "capi_util.hpp"
#include "device_graph.cuh"
#include "hgraph.hpp"
#include "saba_hash.cuh"
#include "walk_common.cuh"

namespace saba_cu {
namespace {

int id_bits(uint64_t n) {  // smallest b with 2^b > n (n itself is the sentinel row)
    int b = 1;
    while (b < 63 && (uint64_t(1) << b) <= n) ++b;
    return b;
}

__device__ __forceinline__ void emit_pair(uint64_t* __restrict__ dir, uint64_t i, uint32_t a, uint32_t b,
                                          uint64_t sentinel) {
    if (a == b) {
        dir[2 * i] = sentinel;
        dir[2 * i + 1] = sentinel;
    } else {
        dir[2 * i] = (uint64_t(a) << 32) | b;
        dir[2 * i + 1] = (uint64_t(b) << 32) | a;
    }
}

__global__ void gb_directed_pairs(const uint32_t* __restrict__ pairs, uint64_t count, uint64_t sentinel,
                                  uint64_t* __restrict__ dir) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint2 p = reinterpret_cast<const uint2*>(pairs)[i];
        emit_pair(dir, i, p.x, p.y, sentinel);
    }
}

__global__ void gb_directed_rmat(uint64_t s, uint64_t samples, uint32_t scale, RmatThresholds t,
                                 uint64_t sentinel, uint64_t* __restrict__ dir) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < samples;
         i += uint64_t(gridDim.x) * blockDim.x) {
        uint32_t u, v;
        rmat_sample(s, i, scale, t, u, v);
        emit_pair(dir, i, u, v, sentinel);
    }
}

__global__ void gb_directed_chung_lu(uint64_t s, uint64_t samples, uint32_t n, const double* __restrict__ prob,
                                     const uint32_t* __restrict__ alias, uint64_t sentinel,
                                     uint64_t* __restrict__ dir) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < samples;
         i += uint64_t(gridDim.x) * blockDim.x)
        emit_pair(dir, i, chung_lu_end(s, i, 0, n, prob, alias), chung_lu_end(s, i, 1, n, prob, alias),
                  sentinel);
}

// off[v] = first slot of row v: for every boundary between rows u0 < u1 of
// the sorted keys, rows (u0, u1] start there (rows without edges included).
__global__ void gb_offsets(const uint64_t* __restrict__ keys, uint64_t two_m, uint32_t n,
                           uint32_t* __restrict__ off, uint32_t* __restrict__ adj) {
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p <= two_m;
         p += uint64_t(gridDim.x) * blockDim.x) {
        const int64_t prev = p == 0 ? -1 : int64_t(keys[p - 1] >> 32);
        const int64_t cur = p == two_m ? int64_t(n) : int64_t(keys[p] >> 32);
        for (int64_t v = prev + 1; v <= cur; ++v) off[v] = uint32_t(p);
        if (p < two_m) adj[p] = uint32_t(keys[p]);
    }
}

__device__ __forceinline__ uint32_t find_root(uint32_t* parent, uint32_t v) {
    uint32_t p = parent[v];
    while (p != v) {  // path halving; parents only ever decrease
        const uint32_t gp = parent[p];
        if (gp != p) parent[v] = gp;
        v = p;
        p = gp;
    }
    return v;
}

// union by (root id): the larger root is hooked under the smaller one, so
// every root is the minimum vertex of its tree
__global__ void gb_hook(const uint64_t* __restrict__ keys, uint64_t two_m, uint32_t* parent) {
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < two_m;
         p += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t k = keys[p];
        const uint32_t u = uint32_t(k >> 32), v = uint32_t(k);
        if (u > v) continue;  // each undirected edge once
        uint32_t ru = find_root(parent, u), rv = find_root(parent, v);
        while (ru != rv) {
            const uint32_t hi = max(ru, rv), lo = min(ru, rv);
            const uint32_t old = atomicCAS(parent + hi, hi, lo);
            if (old == hi) break;
            SABA_DCHECK(old < hi);  // parents only ever point to smaller ids: no cycles
            ru = find_root(parent, old);
            rv = lo;
        }
    }
}

// Component of every vertex into a separate array: the forest is final, and
// a read-only walk cannot be undone by another thread's path halving (which
// may still write an intermediate ancestor into parent[v]).
__global__ void gb_components(const uint32_t* __restrict__ parent, uint32_t n, uint32_t* __restrict__ comp,
                              uint32_t* __restrict__ size) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        uint32_t r = v;
        while (parent[r] != r) r = parent[r];
        comp[v] = r;
        atomicAdd(size + r, 1u);
    }
}

// (size << 32 | ~root): the maximum is the largest component, ties to the
// smallest root (the first component the host's ascending BFS finds)
__global__ void gb_size_keys(const uint32_t* __restrict__ size, uint32_t n, uint64_t* __restrict__ out) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
        out[r] = (uint64_t(size[r]) << 32) | uint32_t(~r);
}

__global__ void gb_keep(const uint32_t* __restrict__ comp, uint32_t n, const uint64_t* __restrict__ best,
                        uint32_t* __restrict__ keep) {
    const uint32_t root = ~uint32_t(*best);
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
        keep[v] = comp[v] == root ? 1u : 0u;
}

// keys of kept rows, relabelled through the exclusive scan of keep
__global__ void gb_relabel(const uint64_t* __restrict__ in, uint64_t two_m, const uint32_t* __restrict__ keep,
                           const uint32_t* __restrict__ id, uint64_t* __restrict__ out,
                           const uint32_t* __restrict__ out_pos) {
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < two_m;
         p += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t k = in[p];
        const uint32_t u = uint32_t(k >> 32), v = uint32_t(k);
        if (!keep[u]) continue;
        out[out_pos[p]] = (uint64_t(id[u]) << 32) | id[v];
    }
}

__global__ void gb_row_kept(const uint64_t* __restrict__ keys, uint64_t two_m, const uint32_t* __restrict__ keep,
                            uint32_t* __restrict__ flag) {
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < two_m;
         p += uint64_t(gridDim.x) * blockDim.x)
        flag[p] = keep[uint32_t(keys[p] >> 32)];
}

__global__ void gb_iota(uint32_t* p, uint32_t n) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) p[v] = v;
}

__global__ void gb_max_id(const uint32_t* __restrict__ pairs, uint64_t count, unsigned int* __restrict__ max_id) {
    uint32_t mx = 0;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < 2 * count;
         i += uint64_t(gridDim.x) * blockDim.x)
        mx = max(mx, pairs[i]);
    mx = __reduce_max_sync(0xffffffffu, mx);
    if ((threadIdx.x & 31) == 0) atomicMax(max_id, mx);
}

struct Timer {
    bool on = getenv("SABA_TRACE") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void lap(const char* what, cudaStream_t s) {
        if (!on) return;
        cudaStreamSynchronize(s);
        const auto t1 = std::chrono::steady_clock::now();
        fprintf(stderr, "[saba] graph_build %-22s %9.2f ms\n", what,
                std::chrono::duration<double, std::milli>(t1 - t).count());
        t = t1;
    }
};

// Device pipeline state: directed keys (double buffer) and one buffer per
// purpose, all from the stream-ordered pool. Buffers are never resized
// mid-pipeline (the pool frees on the legacy stream, not on `s`).
struct Builder {
    DeviceScope scope;  // the caller's current device is restored on return
    cudaStream_t s = nullptr;
    int grid = 148 * 8;
    DevBuf k0, k1, tmp, num, in_pairs, in_max, parent, comp, size, skey, flag, relab, off, gen_a, gen_b;
    Timer T;
    uint64_t samples = 0;
    uint64_t* dir() { return scratch<uint64_t>(k0, 2 * samples); }

    explicit Builder(int device) : scope(device) {
        ensure_pool(device);
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        grid = sms * 8;
        SABA_CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    }
    ~Builder() {
        if (s) {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    }

    template <class T>
    T* scratch(DevBuf& b, size_t count) {
        return static_cast<T*>(b.ensure(sizeof(T) * (count ? count : 1)));
    }
    void* temp(size_t bytes) {  // CUB temporaries: grow between synchronised uses only
        if (bytes > tmp.bytes) SABA_CUDA_CHECK(cudaStreamSynchronize(s));
        return tmp.ensure(bytes);
    }
    template <class T>
    T fetch(const T* d) {
        T h{};
        SABA_CUDA_CHECK(cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, s));
        SABA_CUDA_CHECK(cudaStreamSynchronize(s));
        return h;
    }

    // sort + unique the 2·samples directed keys of an n-vertex graph
    // (loops = sentinel) -> CSR, optionally reduced to its largest component
    saba_hgraph* finish(uint32_t n, bool keep_lcc) {
        check_data(n > 0, "empty graph");
        const int bits = std::min(64, 32 + id_bits(n));
        const uint64_t nk = 2 * samples;
        cub::DoubleBuffer<uint64_t> kb(scratch<uint64_t>(k0, nk), scratch<uint64_t>(k1, nk));
        size_t tb = 0;
        if (nk) {
            SABA_CUDA_CHECK(cub::DeviceRadixSort::SortKeys(nullptr, tb, kb, int64_t(nk), 0, bits, s));
            SABA_CUDA_CHECK(cub::DeviceRadixSort::SortKeys(temp(tb), tb, kb, int64_t(nk), 0, bits, s));
        }
        T.lap("sort", s);
        uint64_t* sorted = kb.Current();
        uint64_t* keys = kb.Alternate();  // unique keys
        uint64_t* d_num = scratch<uint64_t>(num, 2);
        uint64_t two_m = 0;
        if (nk) {
            size_t tu = 0;
            SABA_CUDA_CHECK(cub::DeviceSelect::Unique(nullptr, tu, sorted, keys, d_num, int64_t(nk), s));
            SABA_CUDA_CHECK(cub::DeviceSelect::Unique(temp(tu), tu, sorted, keys, d_num, int64_t(nk), s));
            two_m = fetch(d_num);
            if (two_m && (fetch(keys + two_m - 1) >> 32) >= n) --two_m;  // the loop sentinel sorts last
        }
        T.lap("unique", s);
        check_data(two_m <= 0xffffffffull, "graph too large: 2m must fit in 32 bits");
        uint32_t n_out = n;
        if (keep_lcc) {
            uint32_t* par = scratch<uint32_t>(parent, n);
            uint32_t* sz = scratch<uint32_t>(size, n);
            gb_iota<<<grid, 256, 0, s>>>(par, n);
            SABA_CUDA_CHECK(cudaMemsetAsync(sz, 0, sizeof(uint32_t) * n, s));
            if (two_m) gb_hook<<<grid, 256, 0, s>>>(keys, two_m, par);
            uint32_t* cmp = scratch<uint32_t>(comp, n);
            gb_components<<<grid, 256, 0, s>>>(par, n, cmp, sz);
            uint64_t* sk = scratch<uint64_t>(skey, n);
            uint64_t* best = d_num + 1;
            gb_size_keys<<<grid, 256, 0, s>>>(sz, n, sk);
            size_t tr = 0;
            SABA_CUDA_CHECK(cub::DeviceReduce::Max(nullptr, tr, sk, best, int(n), s));
            SABA_CUDA_CHECK(cub::DeviceReduce::Max(temp(tr), tr, sk, best, int(n), s));
            uint32_t* keep = sz;  // sizes are consumed
            gb_keep<<<grid, 256, 0, s>>>(cmp, n, best, keep);
            uint32_t* id = par;  // roots are consumed
            size_t ts = 0;
            SABA_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, ts, keep, id, int(n), s));
            SABA_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(temp(ts), ts, keep, id, int(n), s));
            n_out = uint32_t(fetch(best) >> 32);
            T.lap("components", s);
            if (two_m) {
                // output positions of the kept keys (rows of the component)
                uint32_t* fl = scratch<uint32_t>(flag, two_m);
                gb_row_kept<<<grid, 256, 0, s>>>(keys, two_m, keep, fl);
                uint32_t* pos = reinterpret_cast<uint32_t*>(sorted);  // sorted keys are consumed
                size_t tp = 0;
                SABA_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, tp, fl, pos, int64_t(two_m), s));
                SABA_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(temp(tp), tp, fl, pos, int64_t(two_m), s));
                uint64_t* out = scratch<uint64_t>(relab, two_m);
                gb_relabel<<<grid, 256, 0, s>>>(keys, two_m, keep, id, out, pos);
                two_m = uint64_t(fetch(pos + two_m - 1)) + fetch(fl + two_m - 1);
                keys = out;
            }
            T.lap("relabel", s);
        }
        auto* g = new saba_hgraph;
        g->n = n_out;
        g->m = two_m / 2;
        g->off.resize(size_t(n_out) + 1);
        g->adj.resize(two_m);
        uint32_t* d_off = scratch<uint32_t>(off, size_t(n_out) + 1);
        uint32_t* d_adj = reinterpret_cast<uint32_t*>(sorted);  // free again (2m u32 <= nk u64)
        gb_offsets<<<grid, 256, 0, s>>>(keys, two_m, n_out, d_off, d_adj);
        SABA_CUDA_CHECK(cudaGetLastError());
        copy_d2h(g->off.data(), d_off, sizeof(uint32_t) * (size_t(n_out) + 1), s);
        if (two_m) copy_d2h(g->adj.data(), d_adj, sizeof(uint32_t) * two_m, s);
        T.lap("csr + download", s);
        return g;
    }
};

}  // namespace
}  // namespace saba_cu

using namespace saba_cu;

extern "C" {

int saba_cu_graph_from_edges(uint32_t n_hint, const uint32_t* pairs, uint64_t count, int keep_lcc, int device,
                             saba_hgraph** out) {
    return guard([&] {
        check_arg(out != nullptr, "null output");
        check_arg(count == 0 || pairs != nullptr, "null pairs");
        check_arg(count < (uint64_t(1) << 30), "graph_build: at most 2^30 pairs");
        Builder B(device);
        B.samples = count;
        uint32_t* d_pairs = B.scratch<uint32_t>(B.in_pairs, 2 * count);
        unsigned int* d_max = B.scratch<unsigned int>(B.in_max, 1);
        SABA_CUDA_CHECK(cudaMemsetAsync(d_max, 0, sizeof(unsigned int), B.s));
        if (count) {
            copy_h2d(d_pairs, pairs, sizeof(uint32_t) * 2 * count, B.s);
            gb_max_id<<<B.grid, 256, 0, B.s>>>(d_pairs, count, d_max);
        }
        // n = max(n_hint, largest id + 1) over every pair, loops included
        // (graph.hpp:87-91)
        const uint64_t n = std::max<uint64_t>(n_hint, count ? uint64_t(B.fetch(d_max)) + 1 : 0);
        check_arg(n <= 0xffffffffull, "vertex id out of range");
        B.T.lap("upload + max id", B.s);
        // loops become a row id >= n that sorts after every real row
        const uint64_t sent = id_bits(n) >= 32 ? ~uint64_t(0) : (uint64_t(1) << (32 + id_bits(n))) - 1;
        if (count) gb_directed_pairs<<<B.grid, 256, 0, B.s>>>(d_pairs, count, sent, B.dir());
        SABA_CUDA_CHECK(cudaGetLastError());
        B.T.lap("directed keys", B.s);
        *out = B.finish(uint32_t(n), keep_lcc != 0);
    });
}

int saba_cu_gen_rmat(uint32_t scale, uint32_t edge_factor, double a, double b, double c, uint64_t seed,
                     int keep_lcc, int device, saba_hgraph** out) {
    return guard([&] {
        check_arg(out != nullptr, "null output");
        check_arg(scale >= 1 && scale <= 31, "rmat: scale must be in [1, 31]");
        check_arg(edge_factor >= 1, "rmat: edge_factor must be >= 1");
        check_arg(a > 0 && b >= 0 && c >= 0 && a + b + c < 1.0, "rmat: bad quadrant probabilities");
        check_arg((uint64_t(edge_factor) << scale) < (uint64_t(1) << 30), "graph_build: at most 2^30 samples");
        Builder B(device);
        B.samples = uint64_t(edge_factor) << scale;
        const uint32_t n = 1u << scale;
        const uint64_t sent = id_bits(n) >= 32 ? ~uint64_t(0) : (uint64_t(1) << (32 + id_bits(n))) - 1;
        gb_directed_rmat<<<B.grid, 256, 0, B.s>>>(substream(seed, kRmatTag), B.samples, scale,
                                                  rmat_thresholds(a, b, c), sent, B.dir());
        SABA_CUDA_CHECK(cudaGetLastError());
        B.T.lap("samples", B.s);
        *out = B.finish(n, keep_lcc != 0);
    });
}

int saba_cu_gen_chung_lu(uint32_t n, double gamma, double mean_degree, double max_degree, uint64_t seed,
                         int keep_lcc, int device, saba_hgraph** out) {
    return guard([&] {
        check_arg(out != nullptr, "null output");
        ChungLuTables t;
        chung_lu_tables(n, gamma, mean_degree, max_degree, seed, t);
        Builder B(device);
        B.T.lap("alias table (host)", B.s);
        B.samples = t.samples;
        check_arg(t.samples < (uint64_t(1) << 30), "graph_build: at most 2^30 samples");
        double* prob = B.scratch<double>(B.gen_a, n);
        uint32_t* alias = B.scratch<uint32_t>(B.gen_b, n);
        copy_h2d(prob, t.prob.data(), sizeof(double) * n, B.s);
        copy_h2d(alias, t.alias.data(), sizeof(uint32_t) * n, B.s);
        const uint64_t sent = (uint64_t(1) << (32 + id_bits(n))) - 1;
        gb_directed_chung_lu<<<B.grid, 256, 0, B.s>>>(substream(seed, kChungLuTag), B.samples, n, prob, alias,
                                                      sent, B.dir());
        SABA_CUDA_CHECK(cudaGetLastError());
        B.T.lap("samples", B.s);
        *out = B.finish(n, keep_lcc != 0);
    });
}

}  // extern "C"
