// Random-gather ceiling microbenchmark (SURVEY §7 hard part 3): many
// independent dependent-load chains over a uint32 array of S bytes, each hop
// a 4-byte gather at a hashed index — the memory behaviour of one walk step
// without the graph. Reports hops/s and 32 B-sector GB/s per working-set size,
// with and without an extra RED.ADD per hop (the visit counter).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_ceiling tools/gather_ceiling.cu
//   tools/gather_ceiling [l2_fetch_granularity_bytes]
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mixh(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x;
}

__global__ void fill(uint32_t* a, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        a[i] = mixh(uint32_t(i) * 2654435761u + 12345u);
}

template <int WPT, bool RED>
__global__ void __launch_bounds__(256) chase(const uint32_t* __restrict__ a, uint32_t n, int hops,
                                             uint32_t* __restrict__ cnt, uint32_t ncnt, uint32_t* sink) {
    uint32_t idx[WPT];
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
    for (int r = 0; r < WPT; ++r) idx[r] = __umulhi(mixh(t * WPT + r), n);
    for (int h = 0; h < hops; ++h) {
        uint32_t v[WPT];
#pragma unroll
        for (int r = 0; r < WPT; ++r) v[r] = __ldg(a + idx[r]);
#pragma unroll
        for (int r = 0; r < WPT; ++r) {
            idx[r] = __umulhi(mixh(v[r] ^ h), n);
            if (RED) atomicAdd(cnt + __umulhi(v[r], ncnt), 1u);
        }
    }
    uint32_t acc = 0;
#pragma unroll
    for (int r = 0; r < WPT; ++r) acc ^= idx[r];
    if (acc == 0x12345678u) sink[0] = acc;
}

template <int WPT, bool RED>
double run(const uint32_t* a, uint32_t n, uint32_t* cnt, uint32_t ncnt, uint32_t* sink, int sms) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, chase<WPT, RED>, 256, 0);
    const int blocks = sms * occ;
    const int hops = 64;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    chase<WPT, RED><<<blocks, 256>>>(a, n, hops, cnt, ncnt, sink);
    cudaEventRecord(e0);
    chase<WPT, RED><<<blocks, 256>>>(a, n, hops, cnt, ncnt, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    return double(blocks) * 256 * WPT * hops / (ms * 1e-3);
}

int main(int argc, char** argv) {
    cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
    // optional argv[1]: cudaLimitMaxL2FetchGranularity in bytes (0..128)
    if (argc > 1) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, size_t(atoi(argv[1])));
    size_t gran = 0;
    cudaDeviceGetLimit(&gran, cudaLimitMaxL2FetchGranularity);
    printf("# %s SMs=%d L2=%d MB  L2 fetch granularity %zu B\n", p.name, p.multiProcessorCount,
           p.l2CacheSize >> 20, gran);
    uint32_t *a, *cnt, *sink;
    const uint64_t maxn = (1ull << 30) / 4 * 2;  // 2 GiB
    cudaMalloc(&a, maxn * 4); cudaMalloc(&cnt, 64 << 20); cudaMalloc(&sink, 4);
    fill<<<4096, 256>>>(a, maxn);
    cudaMemset(cnt, 0, 64 << 20);
    printf("# MB  hops/s(wpt4)  GB/s@32B  hops/s(+RED 2.6MB cnt)  hops/s(wpt1)\n");
    for (double mb : {4.0, 16.0, 32.0, 48.0, 64.0, 80.0, 96.0, 112.0, 128.0, 192.0, 256.0, 512.0, 2048.0}) {
        const uint32_t n = uint32_t(mb * (1 << 20) / 4);
        const double r4 = run<4, false>(a, n, cnt, 1, sink, p.multiProcessorCount);
        const double rr = run<4, true>(a, n, cnt, 646264, sink, p.multiProcessorCount);
        const double r1 = run<1, false>(a, n, cnt, 1, sink, p.multiProcessorCount);
        printf("%6.0f  %.3e  %8.1f  %.3e  %.3e\n", mb, r4, r4 * 32 / 1e9, rr, r1);
    }
    cudaError_t e = cudaGetLastError();
    printf("# %s\n", cudaGetErrorString(e));
    return 0;
}
