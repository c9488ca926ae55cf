// K0: device CSR upload and the handle lifecycle; library identification.
#include <algorithm>
#include <chrono>
#include <mutex>
#include <omp.h>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "device_graph.cuh"
#include "saba_hash.cuh"

namespace saba_cu {

namespace {
thread_local std::string t_last_error;

// off[v], off[v+1] -> packed {base, degree}: the two values every step reads
// together (walker.hpp:225-226) become one 8-byte gather.
__global__ void pack_csr_kernel(const uint32_t* __restrict__ off, uint32_t n, uint2* __restrict__ csr) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        const uint32_t b = off[v];
        csr[v] = make_uint2(b, off[v + 1] - b);
    }
}
// slot s -> word s/3, field s%3 (21 bits each)
__global__ void pack_adj_kernel(const uint32_t* __restrict__ adj, uint64_t two_m,
                                uint64_t* __restrict__ packed) {
    const uint64_t words = (two_m + 2) / 3;
    for (uint64_t w = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; w < words;
         w += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t x = 0;
        for (uint32_t r = 0; r < 3; ++r) {
            const uint64_t s = 3 * w + r;
            if (s < two_m) x |= uint64_t(adj[s]) << (kPackBits * r);
        }
        packed[w] = x;
    }
}
__global__ void check_ids_kernel(const uint32_t* __restrict__ adj, uint64_t two_m, uint32_t n,
                                 unsigned int* __restrict__ bad) {
    uint32_t b = 0;
    for (uint64_t s = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; s < two_m;
         s += uint64_t(gridDim.x) * blockDim.x)
        b |= adj[s] >= n;
    if (__any_sync(0xffffffffu, b) && (threadIdx.x & 31) == 0) atomicOr(bad, 1u);
}
// Fat adjacency: slot s -> adj[s] | base(adj[s]) << idb | degree(adj[s]) << sh.
__global__ void build_fat_kernel(const uint2* __restrict__ csr, const uint32_t* __restrict__ adj,
                                 uint64_t two_m, uint32_t idb, uint32_t sh, uint64_t* __restrict__ fat) {
    for (uint64_t s = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; s < two_m;
         s += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t v = adj[s];
        const uint2 r = csr[v];
        fat[s] = uint64_t(v) | (uint64_t(r.x) << idb) | (uint64_t(r.y) << sh);
    }
}
__global__ void build_fat16_kernel(const uint2* __restrict__ csr, const uint32_t* __restrict__ adj,
                                   uint64_t two_m, uint4* __restrict__ fat16) {
    for (uint64_t s = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; s < two_m;
         s += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t v = adj[s];
        const uint2 r = csr[v];
        fat16[s] = make_uint4(v, r.x, r.y, 0u);
    }
}
}  // namespace

bool ensure_fat16(saba_cu_graph* g) {
    if (g->fat16_tried) return g->d_adj_fat16 != nullptr;
    g->fat16_tried = true;
    if (g->m == 0) return false;
    g->d_adj_fat16 = static_cast<uint4*>(pool_alloc(sizeof(uint4) * 2 * g->m));
    build_fat16_kernel<<<g->sm_count * 8, 256>>>(g->d_csr, g->d_adj, 2 * g->m, g->d_adj_fat16);
    SABA_CUDA_CHECK(cudaGetLastError());
    SABA_CUDA_CHECK(cudaDeviceSynchronize());
    return true;
}

// Fat adjacency + hub slot: slot s -> fat[s] | (hub slot of adj[s] + 1) << shift
// (0 = not a hub). Hubs are the highest-degree vertices, ties by ascending id;
// the order is computed on the host (the fat form exists only for small,
// L2-resident graphs).
namespace {
__global__ void build_fat_hub_kernel(const uint64_t* __restrict__ fat, const uint32_t* __restrict__ adj,
                                     const uint32_t* __restrict__ slot_of, uint64_t two_m, uint32_t shift,
                                     uint64_t* __restrict__ out) {
    for (uint64_t s = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; s < two_m;
         s += uint64_t(gridDim.x) * blockDim.x)
        out[s] = fat[s] | (uint64_t(slot_of[adj[s]]) << shift);
}
}  // namespace

bool ensure_fat_hub(saba_cu_graph* g, uint32_t max_hubs) {
    if (g->fat_hub_tried) return g->d_adj_fat_hub != nullptr;
    g->fat_hub_tried = true;
    if (!ensure_fat(g) || max_hubs == 0) return false;
    uint32_t db = 1;
    while (db < 32 && (g->max_degree >> db) != 0) ++db;
    const uint32_t shift = g->fat_sh + db;
    if (shift + 8 > 64) return false;  // fewer than 255 hubs are not worth a table
    const uint32_t spare = 64 - shift;
    const uint32_t h = uint32_t(std::min<uint64_t>({uint64_t(g->n), (spare >= 32 ? UINT32_MAX : (1u << spare) - 1u),
                                                    uint64_t(max_hubs)}));
    const uint32_t n = g->n;
    std::vector<uint32_t> order(n), slot_of(n, 0u);
    for (uint32_t v = 0; v < n; ++v) order[v] = v;
    const auto& off = g->h_off;
    std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
        return off[a + 1] - off[a] > off[b + 1] - off[b];
    });
    for (uint32_t i = 0; i < h; ++i) slot_of[order[i]] = i + 1;
    DevBuf d_slot;
    uint32_t* ds = static_cast<uint32_t*>(d_slot.ensure(sizeof(uint32_t) * n));
    g->d_fat_hub_vertex = static_cast<uint32_t*>(pool_alloc(sizeof(uint32_t) * h));
    g->d_adj_fat_hub = static_cast<uint64_t*>(pool_alloc(sizeof(uint64_t) * 2 * g->m));
    SABA_CUDA_CHECK(cudaMemcpy(ds, slot_of.data(), sizeof(uint32_t) * n, cudaMemcpyHostToDevice));
    SABA_CUDA_CHECK(cudaMemcpy(g->d_fat_hub_vertex, order.data(), sizeof(uint32_t) * h, cudaMemcpyHostToDevice));
    build_fat_hub_kernel<<<g->sm_count * 8, 256>>>(g->d_adj_fat, g->d_adj, ds, 2 * g->m, shift, g->d_adj_fat_hub);
    SABA_CUDA_CHECK(cudaGetLastError());
    SABA_CUDA_CHECK(cudaDeviceSynchronize());
    g->fat_hub_count = h;
    g->fat_hub_shift = shift;
    return true;
}

bool ensure_fat(saba_cu_graph* g) {
    if (g->fat_tried) return g->d_adj_fat != nullptr;
    g->fat_tried = true;
    auto bits = [](uint64_t x) {  // bits to represent values in [0, x]
        uint32_t b = 1;
        while (b < 64 && (uint64_t(1) << b) <= x) ++b;
        return b;
    };
    const uint32_t idb = bits(g->n ? g->n - 1 : 0), bb = bits(2 * g->m), db = bits(g->max_degree);
    if (idb + bb + db > 64 || g->m == 0) return false;
    g->fat_idb = idb;
    g->fat_sh = idb + bb;
    g->d_adj_fat = static_cast<uint64_t*>(pool_alloc(sizeof(uint64_t) * 2 * g->m));
    build_fat_kernel<<<g->sm_count * 8, 256>>>(g->d_csr, g->d_adj, 2 * g->m, g->fat_idb, g->fat_sh,
                                               g->d_adj_fat);
    SABA_CUDA_CHECK(cudaGetLastError());
    SABA_CUDA_CHECK(cudaDeviceSynchronize());
    return true;
}

void ensure_pool(int device) {
    static bool done[64] = {};
    if (device < 0 || device >= 64 || done[device]) return;
    cudaMemPool_t pool;
    SABA_CUDA_CHECK(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t keep = UINT64_MAX;
    SABA_CUDA_CHECK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    // SABA_L2_FETCH=32|64|128: DRAM -> L2 fetch granularity (tuning switch)
    if (const char* e = getenv("SABA_L2_FETCH"))
        SABA_CUDA_CHECK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, size_t(atoi(e))));
    done[device] = true;
}

void* pool_alloc_on(size_t bytes, cudaStream_t s) {
    int dev = 0;
    cudaGetDevice(&dev);
    ensure_pool(dev);
    void* p = nullptr;
    SABA_CUDA_CHECK(cudaMallocAsync(&p, bytes, s));
    return p;
}

void pool_free_on(void* p, cudaStream_t s) { cudaFreeAsync(p, s); }

void* pool_alloc(size_t bytes) {
    int dev = 0;
    cudaGetDevice(&dev);
    ensure_pool(dev);
    void* p = nullptr;
    SABA_CUDA_CHECK(cudaMallocAsync(&p, bytes, 0));
    SABA_CUDA_CHECK(cudaStreamSynchronize(0));
    return p;
}

namespace {
constexpr size_t kStageBytes = size_t(32) << 20;  // per staging buffer
struct Staging {
    std::mutex mu;
    void* buf[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    int device = -1;
    void ensure(int dev) {
        if (buf[0] && device == dev) return;
        for (int i = 0; i < 2; ++i) {
            if (!buf[i]) SABA_CUDA_CHECK(cudaMallocHost(&buf[i], kStageBytes));
            if (ev[i]) cudaEventDestroy(ev[i]);
            SABA_CUDA_CHECK(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
        }
        device = dev;
    }
};
Staging g_staging;

bool is_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

void par_memcpy(void* dst, const void* src, size_t bytes) {
    constexpr size_t kPiece = size_t(1) << 20;  // 256 KB pieces were slower (thread wake-ups outweigh the fault spread)
    const int64_t pieces = int64_t((bytes + kPiece - 1) / kPiece);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < pieces; ++i) {
        const size_t o = size_t(i) * kPiece;
        std::memcpy(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o,
                    std::min(kPiece, bytes - o));
    }
}

__global__ void fill_u32_kernel(uint32_t* __restrict__ d, uint32_t v, size_t n) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        d[i] = v;
}
}  // namespace

void copy_h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (bytes == 0) return;
    if (bytes <= (size_t(4) << 20) || is_pinned(src)) {
        SABA_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
        SABA_CUDA_CHECK(cudaStreamSynchronize(s));
        return;
    }
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(g_staging.mu);
    g_staging.ensure(dev);
    size_t i = 0;
    for (size_t o = 0; o < bytes; o += kStageBytes, ++i) {
        const int b = int(i & 1);
        const size_t len = std::min(kStageBytes, bytes - o);
        if (i >= 2) SABA_CUDA_CHECK(cudaEventSynchronize(g_staging.ev[b]));  // buffer free again
        par_memcpy(g_staging.buf[b], static_cast<const char*>(src) + o, len);
        SABA_CUDA_CHECK(cudaMemcpyAsync(static_cast<char*>(dst) + o, g_staging.buf[b], len,
                                        cudaMemcpyHostToDevice, s));
        SABA_CUDA_CHECK(cudaEventRecord(g_staging.ev[b], s));
    }
    SABA_CUDA_CHECK(cudaStreamSynchronize(s));
}

void copy_d2h(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (bytes == 0) return;
    if (bytes <= (size_t(4) << 20) || is_pinned(dst)) {
        SABA_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
        SABA_CUDA_CHECK(cudaStreamSynchronize(s));
        return;
    }
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(g_staging.mu);
    g_staging.ensure(dev);
    const size_t chunks = (bytes + kStageBytes - 1) / kStageBytes;
    auto issue = [&](size_t i) {
        const int b = int(i & 1);
        const size_t o = i * kStageBytes, len = std::min(kStageBytes, bytes - o);
        SABA_CUDA_CHECK(cudaMemcpyAsync(g_staging.buf[b], static_cast<const char*>(src) + o, len,
                                        cudaMemcpyDeviceToHost, s));
        SABA_CUDA_CHECK(cudaEventRecord(g_staging.ev[b], s));
    };
    issue(0);
    if (chunks > 1) issue(1);
    for (size_t i = 0; i < chunks; ++i) {
        const int b = int(i & 1);
        const size_t o = i * kStageBytes, len = std::min(kStageBytes, bytes - o);
        SABA_CUDA_CHECK(cudaEventSynchronize(g_staging.ev[b]));
        par_memcpy(static_cast<char*>(dst) + o, g_staging.buf[b], len);
        if (i + 2 < chunks) issue(i + 2);
    }
}

void fill_u32(uint32_t* dst, uint32_t value, size_t count, cudaStream_t s) {
    if (count == 0) return;
    fill_u32_kernel<<<1184, 256, 0, s>>>(dst, value, count);
    SABA_CUDA_CHECK(cudaGetLastError());
}

void pool_free(void* p) {
    cudaFreeAsync(p, 0);
}

const IdVec& host_adj(saba_cu_graph* g) {
    if (g->h_adj.size() != 2 * g->m) {
        DeviceScope scope(g->device);
        g->h_adj.resize(2 * g->m);  // not zero-filled: copy_d2h writes every slot
        if (g->m) copy_d2h(g->h_adj.data(), g->d_adj, sizeof(uint32_t) * 2 * g->m, 0);
    }
    return g->h_adj;
}

void set_last_error(const std::string& msg) { t_last_error = msg; }

void release_aesc_state(saba_cu_graph* g);  // aesc.cu

const IdVec& slot_edges(saba_cu_graph* g) {
    if (!g->h_slot_edge.empty() || g->m == 0) return g->h_slot_edge;
    // edge ids are ranks of the (u<v) pairs in sorted order (graph.hpp:92-100)
    const auto& off = g->h_off;
    const auto& adj = host_adj(g);
    IdVec se(2 * g->m);  // every slot is written below
    // forward slots (u -> v, v > u) are numbered in CSR order: per-vertex
    // counts, a prefix sum, then independent numbering and reverse lookups
    const int64_t N = g->n;
    std::vector<uint32_t> first(size_t(N) + 1, 0);
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t u = 0; u < N; ++u) {
        uint32_t c = 0;
        for (uint32_t s = off[u]; s < off[u + 1]; ++s) c += adj[s] > uint32_t(u);
        first[size_t(u) + 1] = c;
    }
    for (int64_t u = 0; u < N; ++u) first[size_t(u) + 1] += first[size_t(u)];
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t u = 0; u < N; ++u) {
        uint32_t e = first[size_t(u)];
        for (uint32_t s = off[u]; s < off[u + 1]; ++s)
            if (adj[s] > uint32_t(u)) se[s] = e++;
    }
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t ui = 0; ui < N; ++ui) {
        const uint32_t u = uint32_t(ui);
        for (uint32_t s = off[u]; s < off[u + 1]; ++s)
            if (adj[s] < u) {
                const uint32_t v = adj[s];
                uint32_t lo = off[v], hi = off[v + 1];
                while (lo < hi) {
                    const uint32_t mid = lo + (hi - lo) / 2;
                    if (adj[mid] < u) lo = mid + 1; else hi = mid;
                }
                se[s] = se[lo];
            }
    }
    g->h_slot_edge.swap(se);
    return g->h_slot_edge;
}

}  // namespace saba_cu

void saba_cu_graph::enter(cudaStream_t s) {
    if (ev_use_recorded && last_stream != s) SABA_CUDA_CHECK(cudaStreamWaitEvent(s, ev_use, 0));
}

void saba_cu_graph::leave(cudaStream_t s) {
    if (!ev_use) SABA_CUDA_CHECK(cudaEventCreateWithFlags(&ev_use, cudaEventDisableTiming));
    SABA_CUDA_CHECK(cudaEventRecord(ev_use, s));
    ev_use_recorded = true;
    last_stream = s;
}

saba_cu_graph::~saba_cu_graph() {
    for (saba_cu_graph* p : peers) {
        saba_cu::DeviceScope scope(p->device);
        delete p;
    }
    saba_cu::release_nccl(this);
    cudaDeviceSynchronize();  // no kernel of an earlier asynchronous call may still read the replica
    if (ev_use) cudaEventDestroy(ev_use);
    saba_cu::release_aesc_state(this);
    if (d_csr) saba_cu::pool_free(d_csr);
    if (d_adj) saba_cu::pool_free(d_adj);
    if (d_adj_packed) saba_cu::pool_free(d_adj_packed);
    if (d_adj_fat) saba_cu::pool_free(d_adj_fat);
    if (d_adj_fat16) saba_cu::pool_free(d_adj_fat16);
    if (d_adj_fat_hub) saba_cu::pool_free(d_adj_fat_hub);
    if (d_fat_hub_vertex) saba_cu::pool_free(d_fat_hub_vertex);
    if (d_csr_hot) saba_cu::pool_free(d_csr_hot);
    if (d_hot_vertex) saba_cu::pool_free(d_hot_vertex);
    if (d_rec) saba_cu::pool_free(d_rec);
    if (d_rank) saba_cu::pool_free(d_rank);
    if (d_adj_rank) saba_cu::pool_free(d_adj_rank);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (ev2) cudaEventDestroy(ev2);
}

using namespace saba_cu;

extern "C" {

const char* saba_cu_last_error(void) { return t_last_error.c_str(); }

const char* saba_cu_version(void) { return "saba_cuda 0.1 sm_100a"; }

int saba_cu_pinned_alloc(uint64_t bytes, void** out) {
    return guard([&] {
        check_arg(out != nullptr && bytes > 0, "null argument");
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
            cudaGetLastError();
            throw CudaError("no CUDA device available (libsaba_cuda has no CPU fallback)");
        }
        SABA_CUDA_CHECK(cudaHostAlloc(out, size_t(bytes), cudaHostAllocPortable));
    });
}

int saba_cu_pinned_free(void* p) {
    return guard([&] {
        if (p) SABA_CUDA_CHECK(cudaFreeHost(p));
    });
}

int saba_cu_device_count(void) {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return c;
}

}  // extern "C"

namespace {
saba_cu_graph* create_replica(const uint32_t* offsets, const uint32_t* adjacency, uint32_t n, uint64_t two_m,
                              int device) {
    saba_cu_graph* result = nullptr;
    {
        check_arg(offsets != nullptr, "null argument");
        check_arg(two_m == 0 || adjacency != nullptr, "null adjacency");
        check_data(n > 0, "empty graph");
        check_data(offsets[0] == 0 && offsets[n] == two_m && two_m % 2 == 0,
                   "offsets do not describe a 2m-slot adjacency");
        check_data(two_m <= 0xffffffffull, "graph too large: 2m must fit in 32 bits");
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
            cudaGetLastError();
            throw CudaError("no CUDA device available (libsaba_cuda has no CPU fallback)");
        }
        check_arg(device >= 0 && device < ndev, "device index out of range");
        DeviceScope scope(device);
        static cudaDeviceProp props[64];  // queried once per device (slow call)
        static bool have_props[64] = {};
        check_arg(device < 64, "device index out of range");
        if (!have_props[device]) {
            SABA_CUDA_CHECK(cudaGetDeviceProperties(&props[device], device));
            have_props[device] = true;
        }
        const cudaDeviceProp& prop = props[device];
        check_data(prop.major >= 10, "libsaba_cuda is built for sm_100a (B200)");

        const bool trace = getenv("SABA_TRACE") != nullptr;
        auto T0 = std::chrono::steady_clock::now();
        auto lap = [&](const char* what) {
            if (!trace) return;
            cudaDeviceSynchronize();
            const auto T1 = std::chrono::steady_clock::now();
            fprintf(stderr, "[saba] graph_create %-12s %8.3f ms\n", what,
                    std::chrono::duration<double, std::milli>(T1 - T0).count());
            T0 = T1;
        };
        auto g = std::make_unique<saba_cu_graph>();
        g->device = device;
        g->sm_count = prop.multiProcessorCount;
        g->smem_optin = prop.sharedMemPerBlockOptin;
        g->n = n;
        g->m = two_m / 2;
        lap("start");
        // The uploads are enqueued first (asynchronous from pinned host
        // memory); the host-side copy of the offsets and the degree scan run
        // while they are in flight.
        ensure_pool(device);
        DevBuf d_offb, d_bad;
        uint32_t* d_off = static_cast<uint32_t*>(d_offb.ensure(sizeof(uint32_t) * (size_t(n) + 1)));
        unsigned int* bad = static_cast<unsigned int*>(d_bad.ensure(sizeof(unsigned int)));
        g->d_csr = static_cast<uint2*>(pool_alloc_on(sizeof(uint2) * size_t(n), 0));
        g->d_adj = static_cast<uint32_t*>(pool_alloc_on(sizeof(uint32_t) * (two_m ? two_m : 1), 0));
        if (n <= kPackMax && two_m)
            g->d_adj_packed = static_cast<uint64_t*>(pool_alloc_on(sizeof(uint64_t) * ((two_m + 2) / 3), 0));
        SABA_CUDA_CHECK(cudaMemcpyAsync(d_off, offsets, sizeof(uint32_t) * (size_t(n) + 1),
                                        cudaMemcpyHostToDevice, 0));
        if (two_m)
            SABA_CUDA_CHECK(cudaMemcpyAsync(g->d_adj, adjacency, sizeof(uint32_t) * two_m,
                                            cudaMemcpyHostToDevice, 0));
        pack_csr_kernel<<<(n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096, 256>>>(d_off, n, g->d_csr);
        SABA_CUDA_CHECK(cudaGetLastError());
        SABA_CUDA_CHECK(cudaMemsetAsync(bad, 0, sizeof(unsigned int), 0));
        check_ids_kernel<<<g->sm_count * 8, 256>>>(g->d_adj, two_m, n, bad);
        SABA_CUDA_CHECK(cudaGetLastError());
        if (g->d_adj_packed) {
            pack_adj_kernel<<<g->sm_count * 8, 256>>>(g->d_adj, two_m, g->d_adj_packed);
            SABA_CUDA_CHECK(cudaGetLastError());
        }
        if (trace) {
            const auto T1 = std::chrono::steady_clock::now();
            fprintf(stderr, "[saba] graph_create %-12s %8.3f ms\n", "enqueue",
                    std::chrono::duration<double, std::milli>(T1 - T0).count());
            T0 = T1;
        }
        g->h_off.assign(offsets, offsets + n + 1);
        uint32_t dmin = UINT32_MAX, dmax = 0;
        bool monotone = true;
        for (uint32_t v = 0; v < n; ++v) {
            monotone &= offsets[v] <= offsets[v + 1];
            const uint32_t d = offsets[v + 1] - offsets[v];
            dmin = d < dmin ? d : dmin;
            dmax = d > dmax ? d : dmax;
        }
        g->min_degree = dmin;
        g->max_degree = dmax;
        if (trace) {
            const auto T1 = std::chrono::steady_clock::now();
            fprintf(stderr, "[saba] graph_create %-12s %8.3f ms\n", "host scan",
                    std::chrono::duration<double, std::milli>(T1 - T0).count());
            T0 = T1;
        }
        unsigned int h_bad = 0;
        SABA_CUDA_CHECK(cudaMemcpy(&h_bad, bad, sizeof(h_bad), cudaMemcpyDeviceToHost));
        SABA_CUDA_CHECK(cudaDeviceSynchronize());
        lap("h2d + pack");
        // the replica (and its unique_ptr) is released only after the device is idle
        check_data(monotone, "offsets must be nondecreasing");
        check_data(h_bad == 0, "adjacency id out of range");
        SABA_CUDA_CHECK(cudaEventCreate(&g->ev0));
        SABA_CUDA_CHECK(cudaEventCreate(&g->ev1));
        SABA_CUDA_CHECK(cudaEventCreate(&g->ev2));
        lap("events");
        result = g.release();
    }
    return result;
}
}  // namespace

extern "C" {

int saba_cu_graph_create(const uint32_t* offsets, const uint32_t* adjacency, uint32_t n,
                         uint64_t two_m, int device, saba_cu_graph** out) {
    return guard([&] {
        check_arg(out != nullptr, "null argument");
        *out = create_replica(offsets, adjacency, n, two_m, device);
    });
}

int saba_cu_graph_create_multi(const uint32_t* offsets, const uint32_t* adjacency, uint32_t n,
                               uint64_t two_m, const int* devices, int ndev, saba_cu_graph** out) {
    return guard([&] {
        check_arg(out != nullptr && devices != nullptr, "null argument");
        check_arg(ndev >= 1, "need at least one device");
        std::unique_ptr<saba_cu_graph> g(create_replica(offsets, adjacency, n, two_m, devices[0]));
        for (int i = 1; i < ndev; ++i)
            g->peers.push_back(create_replica(offsets, adjacency, n, two_m, devices[i]));
        *out = g.release();
    });
}

int saba_cu_graph_replica_count(const saba_cu_graph* g) { return g ? 1 + int(g->peers.size()) : 0; }

int saba_cu_graph_destroy(saba_cu_graph* g) {
    return guard([&] {
        if (!g) return;
        DeviceScope scope(g->device);
        delete g;
    });
}

uint32_t saba_cu_graph_vertex_count(const saba_cu_graph* g) { return g ? g->n : 0; }
uint64_t saba_cu_graph_edge_count(const saba_cu_graph* g) { return g ? g->m : 0; }

}  // extern "C"
