// Sectors per L2 request of random gathers by load width (4 / 8 / 16 bytes) and cache
// operator, over an S-MB array: run under ncu --metrics lts__t_sectors_srcunit_tex_op_read.sum,
// lts__t_requests_srcunit_tex_op_read.sum,dram__bytes_read.sum (one launch per variant).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_width tools/gather_width.cu
//   tools/gather_width [MB=84]
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
// W = bytes per gather; NA = ld.global.nc.L1::no_allocate instead of plain nc
template <int W, bool NA>
__global__ void __launch_bounds__(256) chase(const uint32_t* __restrict__ a, uint32_t nelem, int hops, uint32_t* sink) {
    constexpr int WPT = 4;
    uint32_t idx[WPT];
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
    for (int r = 0; r < WPT; ++r) idx[r] = __umulhi(mixh(t * WPT + r), nelem);
    for (int h = 0; h < hops; ++h) {
        uint32_t v[WPT];
#pragma unroll
        for (int r = 0; r < WPT; ++r) {
            const char* p = reinterpret_cast<const char*>(a) + size_t(idx[r]) * W;
            if (W == 4) {
                if (NA) asm("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v[r]) : "l"(p));
                else asm("ld.global.nc.u32 %0, [%1];" : "=r"(v[r]) : "l"(p));
            } else if (W == 8) {
                uint64_t x;
                if (NA) asm("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(x) : "l"(p));
                else asm("ld.global.nc.u64 %0, [%1];" : "=l"(x) : "l"(p));
                v[r] = uint32_t(x) ^ uint32_t(x >> 32);
            } else {
                uint32_t x0, x1, x2, x3;
                if (NA) asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3) : "l"(p));
                else asm("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3) : "l"(p));
                v[r] = x0 ^ x1 ^ x2 ^ x3;
            }
        }
#pragma unroll
        for (int r = 0; r < WPT; ++r) idx[r] = __umulhi(mixh(v[r] ^ h), nelem);
    }
    uint32_t acc = 0;
#pragma unroll
    for (int r = 0; r < WPT; ++r) acc ^= idx[r];
    if (acc == 0x12345678u) sink[0] = acc;
}
template <int W, bool NA>
void run(const uint32_t* a, size_t bytes, uint32_t* sink, int sms) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, chase<W, NA>, 256, 0);
    const int blocks = sms * occ, hops = 64;
    const uint32_t nelem = uint32_t(bytes / W);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    chase<W, NA><<<blocks, 256>>>(a, nelem, hops, sink);
    cudaEventRecord(e0);
    chase<W, NA><<<blocks, 256>>>(a, nelem, hops, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("width %2d %s  %.3e gathers/s\n", W, NA ? "no_allocate" : "plain nc   ", double(blocks) * 256 * 4 * hops / (ms * 1e-3));
}
int main(int argc, char** argv) {
    cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
    const size_t bytes = size_t(argc > 1 ? atoi(argv[1]) : 84) << 20;
    uint32_t *a, *sink;
    cudaMalloc(&a, bytes); cudaMalloc(&sink, 4);
    fill<<<4096, 256>>>(a, bytes / 4);
    printf("# %s, %zu MB array, random gathers (2 launches per variant; ncu: the second)\n", p.name, bytes >> 20);
    run<4, false>(a, bytes, sink, p.multiProcessorCount);
    run<4, true>(a, bytes, sink, p.multiProcessorCount);
    run<8, false>(a, bytes, sink, p.multiProcessorCount);
    run<8, true>(a, bytes, sink, p.multiProcessorCount);
    run<16, false>(a, bytes, sink, p.multiProcessorCount);
    run<16, true>(a, bytes, sink, p.multiProcessorCount);
    printf("# %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
