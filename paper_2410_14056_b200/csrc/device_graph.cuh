// Device graph handle (K0): one CSR replica per handle, packed for the walk
// kernels, plus host copies for validation and the AESC truncation plan.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <vector>

#include "capi_util.hpp"

namespace saba_cu {

// Grow-only device buffer.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    void* ensure(size_t b) {
        if (b <= bytes && p) return p;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        SABA_CUDA_CHECK(cudaMalloc(&p, b ? b : 1));
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
    uint32_t n = 0;
    uint64_t m = 0;
    uint32_t max_degree = 0;
    uint32_t min_degree = 0;
    std::vector<uint32_t> h_off, h_adj;  // host CSR (graph.hpp:242-243 layout)
    std::vector<uint32_t> h_slot_edge;   // directed slot -> edge id (lazy)
    uint2* d_csr = nullptr;              // {base, degree} per vertex
    uint32_t* d_adj = nullptr;           // 2m neighbour ids, sorted per slice
    // campaign workspace (grow-only, reused across calls)
    saba_cu::DevBuf kv, off, keys, keys_alt, seg, cub_tmp;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr;
    saba_cu::AescState* aesc = nullptr;  // owned; freed by release_aesc_state (aesc.cu)
    ~saba_cu_graph();
};

namespace saba_cu {
const std::vector<uint32_t>& slot_edges(saba_cu_graph* g);
}
