// Random 16-byte gather microbenchmark: which load flavour fetches the
// fewest DRAM sectors per request on B200? (profiling aid, not product)
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

template <int V>
__device__ __forceinline__ uint4 ld(const uint4* p, uint64_t pol) {
    uint4 v;
    if (V == 0) asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
    if (V == 1) asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    if (V == 2) asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    if (V == 3) asm volatile("ld.global.cv.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    if (V == 4) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    if (V == 5) asm volatile("ld.global.cg.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
    if (V == 6) asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

template <int V, int MLP>
__global__ void gather(const uint4* __restrict__ a, uint64_t n, uint64_t iters, uint32_t* out) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    uint64_t st = mix(t + 12345);
    for (uint64_t k = 0; k < iters; ++k) {
        uint4 v[MLP];
#pragma unroll
        for (int m = 0; m < MLP; ++m) {
            st += 0x9E3779B97F4A7C15ULL;
            v[m] = ld<V>(a + __umul64hi(mix(st), n), pol);
        }
#pragma unroll
        for (int m = 0; m < MLP; ++m) acc ^= v[m].x ^ v[m].w;
    }
    if (acc == 0x12345678) out[0] = acc;
}

int main(int argc, char** argv) {
    const uint64_t n = 87114705ULL;  // config-2 step records
    uint4* a;
    uint32_t* out;
    cudaMalloc(&a, n * 16);
    cudaMemset(a, 1, n * 16);
    cudaMalloc(&out, 4);
    int gran = argc > 1 ? atoi(argv[1]) : 0;
    if (gran) {
        cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran);
        size_t g = 0;
        cudaDeviceGetLimit(&g, cudaLimitMaxL2FetchGranularity);
        printf("set granularity %d -> %s, now %zu\n", gran, cudaGetErrorString(e), g);
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = 148 * 8, threads = 256;
    const uint64_t iters = 64;
    auto run = [&](const char* name, void (*k)(const uint4*, uint64_t, uint64_t, uint32_t*), int mlp) {
        k<<<blocks, threads>>>(a, n, iters / mlp * 0 + 8, out);
        cudaEventRecord(e0);
        k<<<blocks, threads>>>(a, n, iters / mlp, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double loads = (double)blocks * threads * (iters / mlp) * mlp;
        printf("%-28s %8.3f ms  %7.2f Gload/s  %7.1f GB/s(32B/load)\n", name, ms, loads / ms / 1e6, loads * 32 / ms / 1e6);
    };
    run("nc.noalloc+evict_first MLP4", gather<0, 4>, 4);
    run("nc (ldg) MLP4", gather<1, 4>, 4);
    run("cg MLP4", gather<2, 4>, 4);
    run("cv MLP4", gather<3, 4>, 4);
    run("nc.noalloc MLP4", gather<4, 4>, 4);
    run("cg+evict_first MLP4", gather<5, 4>, 4);
    run("relaxed.gpu MLP4", gather<6, 4>, 4);
    run("cg MLP8", gather<2, 8>, 8);
    run("cg MLP1", gather<2, 1>, 1);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
