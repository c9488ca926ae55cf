// Device graph handle (K0): one CSR replica per handle, packed for the walk
// kernels, plus host copies for validation and the AESC truncation plan.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <vector>

#include "capi_util.hpp"
#include "hgraph.hpp"

namespace saba_cu {

// Stream-ordered allocations from the device's default memory pool, which is
// configured (ensure_pool) to keep freed memory cached: workspaces of a new
// graph handle reuse the previous handle's memory instead of paying
// cudaMalloc/cudaFree again (this is on the end-to-end path of every call).
void ensure_pool(int device);
void* pool_alloc(size_t bytes);
void pool_free(void* p);

// Grow-only device buffer.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() {
        if (p) pool_free(p);
    }
    void* ensure(size_t b) {
        if (b <= bytes && p) return p;
        if (p) pool_free(p);
        p = nullptr;
        bytes = 0;
        p = pool_alloc(b ? b : 1);
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
    // Hub-privatised counting: {base, degree | (hot slot + 1) << hot_shift};
    // the top-degree vertices count their visits in shared memory.
    uint2* d_csr_hot = nullptr;
    uint32_t* d_hot_vertex = nullptr;  // slot -> vertex
    uint32_t hot_count = 0;
    uint32_t hot_shift = 18;  // degree bits below the slot field (fits max_degree)
    int hot_threads = 1024;   // block size the hot table was sized for
    bool hot_tried = false;
    // campaign workspace (grow-only, reused across calls)
    saba_cu::DevBuf kv, off, keys, keys_alt, seg, cub_tmp, counts32;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr;
    saba_cu::AescState* aesc = nullptr;  // owned; freed by release_aesc_state (aesc.cu)
    ~saba_cu_graph();
};

namespace saba_cu {
const IdVec& slot_edges(saba_cu_graph* g);
const IdVec& host_adj(saba_cu_graph* g);  // D2H once, then cached
// Build the fat adjacency once (false if {id, base, degree} exceed 64 bits).
bool ensure_fat(saba_cu_graph* g);
bool ensure_fat16(saba_cu_graph* g);
// Fat adjacency is worth it while it stays comfortably L2-resident.
inline bool fat_fits_l2(const saba_cu_graph* g) { return 16 * g->m <= (uint64_t(48) << 20); }
constexpr uint32_t kPackBits = 21;
constexpr uint32_t kPackMax = 1u << kPackBits;  // ids must be < 2^21 to pack

// Host <-> device copies of large caller-owned (pageable) buffers at PCIe
// speed: through a pinned double-buffered staging ring with a parallel host
// memcpy; already-pinned buffers go direct. Both return when the copy is
// complete (the caller's buffer may be reused).
void copy_h2d(void* dst, const void* src, size_t bytes, cudaStream_t s);
void copy_d2h(void* dst, const void* src, size_t bytes, cudaStream_t s);
void fill_u32(uint32_t* dst, uint32_t value, size_t count, cudaStream_t s);
}
