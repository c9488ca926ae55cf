// Multi-device handles and the one combine step of a sharded run.
//
// A multi-device handle holds one CSR replica per entry of a device list
// (repeats allowed: logical shards sharing a GPU, each with its own replica
// and workspaces, which is how the 1/2/N-device invariance is tested on one
// GPU). Walk campaigns and AESC shard their work over the replicas — one host
// thread per replica — and combine once at the end:
//   * visit counts: integer sums, so any reduction order is exact;
//   * g_hat: every directed slot is written by exactly one source, i.e. by
//     one replica, and the others hold +0.0 there, so the sum is exact too.
// With distinct devices the combine is an NCCL reduce to the first replica
// over NVLink/NVSwitch (libnccl.so.2 is opened at run time, reusing the copy
// torch already loaded if any, so the library has no link-time NCCL
// dependency); with repeated devices (or no NCCL) it is peer copies into the
// root plus an add kernel. Either way the result equals a one-device run bit
// for bit.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <mutex>
#include <set>
#include <string>

#include "device_graph.cuh"

namespace saba_cu {

namespace {

struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                           cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl_api() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        if (const char* e = getenv("SABA_NCCL"); e && atoi(e) == 0) {
            api.why = "disabled (SABA_NCCL=0)";
            return;
        }
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // torch's copy, if loaded
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) {
            api.why = "libnccl.so.2 not found";
            return;
        }
        auto sym = [&](const char* n) { return dlsym(h, n); };
        api.CommInitAll = reinterpret_cast<decltype(api.CommInitAll)>(sym("ncclCommInitAll"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
        api.Reduce = reinterpret_cast<decltype(api.Reduce)>(sym("ncclReduce"));
        api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
        api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
        api.ok = api.CommInitAll && api.CommDestroy && api.Reduce && api.GroupStart && api.GroupEnd &&
                 api.GetErrorString;
        if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
    });
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw CudaError(std::string("NCCL ") + what + ": " + nccl_api().GetErrorString(r));
}

struct NcclGroup {
    std::vector<ncclComm_t> comms;
    ~NcclGroup() {
        for (ncclComm_t c : comms)
            if (c) nccl_api().CommDestroy(c);
    }
};

thread_local const char* t_combine = "none";

__global__ void add_u64_kernel(unsigned long long* __restrict__ dst, const unsigned long long* __restrict__ src,
                               size_t n) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        dst[i] += src[i];
}
__global__ void add_f64_kernel(double* __restrict__ dst, const double* __restrict__ src, size_t n) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        dst[i] += src[i];
}

}  // namespace

std::vector<saba_cu_graph*> replicas_of(saba_cu_graph* g) {
    std::vector<saba_cu_graph*> r{g};
    r.insert(r.end(), g->peers.begin(), g->peers.end());
    return r;
}

const char* last_combine_kind() { return t_combine; }

void release_nccl(saba_cu_graph* g) {
    delete static_cast<NcclGroup*>(g->nccl);
    g->nccl = nullptr;
}

void reduce_to_root(const std::vector<saba_cu_graph*>& reps, const std::vector<void*>& bufs, size_t count,
                    ReduceType type, const std::vector<cudaStream_t>& streams) {
    const size_t R = reps.size();
    if (R <= 1 || count == 0) {
        t_combine = "none";
        return;
    }
    std::set<int> devs;
    for (auto* r : reps) devs.insert(r->device);
    const size_t esz = 8;
    saba_cu_graph* root = reps[0];
    if (devs.size() == R && nccl_api().ok) {
        if (!root->nccl) {
            std::vector<int> list;
            for (auto* r : reps) list.push_back(r->device);
            auto* grp = new NcclGroup;
            grp->comms.assign(R, nullptr);
            try {
                nccl_check(nccl_api().CommInitAll(grp->comms.data(), int(R), list.data()), "ncclCommInitAll");
            } catch (...) {
                delete grp;
                throw;
            }
            root->nccl = grp;
        }
        auto* grp = static_cast<NcclGroup*>(root->nccl);
        const ncclDataType_t dt = type == ReduceType::U64 ? ncclUint64 : ncclFloat64;
        nccl_check(nccl_api().GroupStart(), "ncclGroupStart");
        for (size_t r = 0; r < R; ++r) {
            DeviceScope scope(reps[r]->device);
            nccl_check(nccl_api().Reduce(bufs[r], r == 0 ? bufs[0] : nullptr, count, dt, ncclSum, 0, grp->comms[r],
                                         streams[r]),
                       "ncclReduce");
        }
        nccl_check(nccl_api().GroupEnd(), "ncclGroupEnd");
        for (size_t r = 0; r < R; ++r) {
            DeviceScope scope(reps[r]->device);
            SABA_CUDA_CHECK(cudaStreamSynchronize(streams[r]));
        }
        t_combine = "nccl";
        return;
    }
    // peer copies into the root, then an add kernel per replica
    DeviceScope scope(root->device);
    cudaStream_t s = streams[0];
    DevBuf stage;
    void* st = stage.ensure(esz * count, s);
    for (size_t r = 1; r < R; ++r) {
        {
            DeviceScope sr(reps[r]->device);
            SABA_CUDA_CHECK(cudaStreamSynchronize(streams[r]));
        }
        if (reps[r]->device == root->device)
            SABA_CUDA_CHECK(cudaMemcpyAsync(st, bufs[r], esz * count, cudaMemcpyDeviceToDevice, s));
        else
            SABA_CUDA_CHECK(cudaMemcpyPeerAsync(st, root->device, bufs[r], reps[r]->device, esz * count, s));
        const int grid = root->sm_count * 4;
        if (type == ReduceType::U64)
            add_u64_kernel<<<grid, 256, 0, s>>>(static_cast<unsigned long long*>(bufs[0]),
                                                static_cast<const unsigned long long*>(st), count);
        else
            add_f64_kernel<<<grid, 256, 0, s>>>(static_cast<double*>(bufs[0]), static_cast<const double*>(st), count);
        SABA_CUDA_CHECK(cudaGetLastError());
    }
    SABA_CUDA_CHECK(cudaStreamSynchronize(s));
    t_combine = "peer";
}

}  // namespace saba_cu
