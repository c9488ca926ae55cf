// Device graph handle (K0): one CSR replica per handle, packed for the walk
// kernels, plus host copies for validation and the AESC truncation plan.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <mutex>
#include <vector>

#include "capi_util.hpp"
#include "hgraph.hpp"

namespace saba_cu {

// Stream-ordered allocations from the device's default memory pool, which is
// configured (ensure_pool) to keep freed memory cached: workspaces of a new
// graph handle reuse the previous handle's memory instead of paying
// cudaMalloc/cudaFree again (this is on the end-to-end path of every call).
void ensure_pool(int device);
void* pool_alloc(size_t bytes);                      // ready for any stream on return
void* pool_alloc_on(size_t bytes, cudaStream_t s);  // stream-ordered: usable by work on s
void pool_free(void* p);                             // ordered on the legacy stream
void pool_free_on(void* p, cudaStream_t s);

// Grow-only device buffer. Growth is stream-ordered on the stream that will
// use the buffer (ensure(b, s)): the old block is released after every
// earlier operation on s and the new one is valid for work enqueued on s
// afterwards. A handle's workspaces are only ever touched from one stream at
// a time; entry points taking a caller stream first order that stream after
// the handle's previous user (saba_cu_graph::enter), so a grow can never free
// memory a kernel of an earlier call is still reading.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    int dev = -1;  // device the block belongs to (freed there)
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes), dev(o.dev) { o.p = nullptr; o.bytes = 0; }
    ~DevBuf() { release(); }
    void release() {
        if (!p) return;
        int cur = -1;
        cudaGetDevice(&cur);
        if (dev >= 0 && cur != dev) cudaSetDevice(dev);
        pool_free(p);
        if (dev >= 0 && cur != dev) cudaSetDevice(cur);
        p = nullptr;
        bytes = 0;
    }
    void* ensure(size_t b) {
        if (b <= bytes && p) return p;
        release();
        p = pool_alloc(b ? b : 1);
        cudaGetDevice(&dev);
        bytes = b;
        return p;
    }
    void* ensure(size_t b, cudaStream_t s) {
        if (b <= bytes && p) return p;
        if (p) pool_free_on(p, s);
        p = nullptr;
        bytes = 0;
        p = pool_alloc_on(b ? b : 1, s);
        cudaGetDevice(&dev);
        bytes = b;
        return p;
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// RAII device switch.
struct DeviceScope {
    int prev = -1;
    explicit DeviceScope(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) SABA_CUDA_CHECK(cudaSetDevice(dev));
    }
    ~DeviceScope() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

struct AescState;  // aesc.cu

}  // namespace saba_cu

struct saba_cu_graph {
    int device = 0;
    int sm_count = 148;
    size_t smem_optin = 232448;  // sharedMemPerBlockOptin
    uint32_t n = 0;
    uint64_t m = 0;
    uint32_t max_degree = 0;
    uint32_t min_degree = 0;
    std::vector<uint32_t> h_off;         // host offsets (graph.hpp:242 layout)
    saba_cu::IdVec h_adj;                // host adjacency, fetched lazily (host_adj)
    saba_cu::IdVec h_slot_edge;          // directed slot -> edge id (lazy)
    uint2* d_csr = nullptr;              // {base, degree} per vertex
    uint32_t* d_adj = nullptr;           // 2m neighbour ids, sorted per slice
    // 3 x 21-bit ids per uint64 when n <= 2^21 (2.67 B/slot instead of 4):
    // shrinks the random-gather working set so more of it stays in L2
    uint64_t* d_adj_packed = nullptr;
    // "fat" adjacency for the campaign: slot s holds its neighbour's
    // {id, base, degree} in one uint64 (id | base << fat_idb | deg << fat_sh),
    // so a walk step is one dependent gather instead of two. Built on first
    // use when the three fields fit in 64 bits.
    uint64_t* d_adj_fat = nullptr;
    // 16-byte records {id, base, degree, 0} per slot (AESC walks on graphs
    // too large for the 8-byte fat form): one dependent gather per step
    uint4* d_adj_fat16 = nullptr;
    bool fat16_tried = false;
    uint32_t fat_idb = 0, fat_sh = 0;
    bool fat_tried = false;
    // fat adjacency with a hub slot in its spare high bits (AESC long walks on
    // L2-resident graphs): the rho values of the highest-degree vertices of
    // the column a block is walking live in shared memory, indexed by slot-1
    uint64_t* d_adj_fat_hub = nullptr;
    uint32_t* d_fat_hub_vertex = nullptr;  // slot -> vertex
    uint32_t fat_hub_count = 0, fat_hub_shift = 0;
    bool fat_hub_tried = false;
    // Hub-privatised counting: {base, degree | (hot slot + 1) << hot_shift};
    // the top-degree vertices count their visits in shared memory.
    uint2* d_csr_hot = nullptr;
    uint32_t* d_hot_vertex = nullptr;  // slot -> vertex
    uint32_t hot_count = 0;
    // Degree-ranked walk records (walk_count_rank_kernel): vertex of rank r
    // (descending degree, ties by id) has rec[r] = id | base << rec_nb |
    // degree << rec_db in one uint64, and the adjacency is restated in rank
    // space (same slot order). The kernel keeps the first records and the
    // visit counters of the first ranks in shared memory: hub tests are
    // plain comparisons of the rank.
    uint64_t* d_rec = nullptr;
    uint32_t* d_rank = nullptr;      // vertex id -> rank
    uint64_t* d_adj_rank = nullptr;  // 3 x 21-bit ranks per uint64 (n <= 2^21)
    uint32_t rec_nb = 0, rec_db = 0;
    bool rec_tried = false;
    uint32_t last_k2 = 0;  // SABA_K2_* of the last campaign launch (reported)
    uint32_t last_nrec = 0, last_ncnt = 0;  // its shared-memory tables (saba_cu_campaign_tables)
    uint32_t hot_shift = 18;  // degree bits below the slot field (fits max_degree)
    int hot_threads = 1024;   // block size the hot table was sized for
    bool hot_tried = false;
    // campaign workspace (grow-only, reused across calls)
    saba_cu::DevBuf kv, off, keys, keys_alt, seg, cub_tmp, counts32;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr;
    saba_cu::AescState* aesc = nullptr;  // owned; freed by release_aesc_state (aesc.cu)
    // Every entry point holds `mu` for its whole call: the lazy builders
    // (host adjacency, slot edges, fat / hot tables) and the workspaces above
    // are shared state, and the reference's Graph allows unrestricted
    // concurrent use (graph.hpp:24-27), so concurrent calls on one handle are
    // serialised here instead of racing.
    std::recursive_mutex mu;
    // Stream chain of the asynchronous entry points: the stream of the last
    // call and an event recorded at its end (see DevBuf).
    cudaStream_t last_stream = nullptr;
    cudaEvent_t ev_use = nullptr;
    bool ev_use_recorded = false;
    void enter(cudaStream_t s);  // order s after the previous user of the handle
    void leave(cudaStream_t s);  // record this call's end on s
    // Multi-device handle (saba_cu_graph_create_multi): the replicas on
    // devices[1..ndev) (owned); this handle is the replica on devices[0].
    // Entry points given such a handle run one shard per replica, one host
    // thread each, and combine on this replica (multi_device.cu).
    std::vector<saba_cu_graph*> peers;
    void* nccl = nullptr;  // saba_cu::NcclGroup (multi_device.cu), created on first combine
    ~saba_cu_graph();
};

namespace saba_cu {
const IdVec& slot_edges(saba_cu_graph* g);
const IdVec& host_adj(saba_cu_graph* g);  // D2H once, then cached
// Build the fat adjacency once (false if {id, base, degree} exceed 64 bits).
bool ensure_fat(saba_cu_graph* g);
bool ensure_fat16(saba_cu_graph* g);
bool ensure_fat_hub(saba_cu_graph* g, uint32_t max_hubs);
bool ensure_fat_hub(saba_cu_graph* g, uint32_t max_hubs);
// Fat adjacency is worth it while it stays comfortably L2-resident.
inline bool fat_fits_l2(const saba_cu_graph* g) { return 16 * g->m <= (uint64_t(48) << 20); }
constexpr uint32_t kPackBits = 21;
constexpr uint32_t kPackMax = 1u << kPackBits;  // ids must be < 2^21 to pack

// Multi-device combine (multi_device.cu). replicas[0] is the root; bufs[r]
// lives on replicas[r]'s device, `count` elements each, all zero outside the
// slots that replica wrote. On return bufs[0] holds the element-wise sum
// (exact: every element has at most one non-zero contributor for g_hat, and
// integer sums for visit counts). An NCCL reduce over NVLink when the devices
// are distinct and libnccl is loadable; otherwise (logical shards sharing a
// device, or no NCCL) peer copies into the root plus an add kernel.
enum class ReduceType { U64, F64 };
void reduce_to_root(const std::vector<saba_cu_graph*>& replicas, const std::vector<void*>& bufs,
                    size_t count, ReduceType type, const std::vector<cudaStream_t>& streams);
// The replicas of a handle in shard order: {g, g->peers...}.
std::vector<saba_cu_graph*> replicas_of(saba_cu_graph* g);
// Name of the combine reduce_to_root used last ("nccl" / "peer"), for reports.
const char* last_combine_kind();
void release_nccl(saba_cu_graph* g);

// Host <-> device copies of large caller-owned (pageable) buffers at PCIe
// speed: through a pinned double-buffered staging ring with a parallel host
// memcpy; already-pinned buffers go direct. Both return when the copy is
// complete (the caller's buffer may be reused).
void copy_h2d(void* dst, const void* src, size_t bytes, cudaStream_t s);
void copy_d2h(void* dst, const void* src, size_t bytes, cudaStream_t s);
void fill_u32(uint32_t* dst, uint32_t value, size_t count, cudaStream_t s);
}
