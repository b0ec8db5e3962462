// pgl_sgd.cu — the PG-SGD iteration kernels for sm_100a.
//
// k_sgd_hogwild: one launch per iteration over a persistent grid. Each warp
// is one reference worker (engine.cpp:103-172): it owns an exact share of the
// iteration's step budget (floor(N/W), +1 for the first N mod W warps) and
// runs it 32 steps per round, lane l taking step 32*round + l. A batch's
// cooling coin is drawn by the lane owning the batch's first step and
// broadcast with __shfl_sync, so for batch_size % 32 == 0 the cooling branch
// is warp-uniform (the paper's warp merging) and lanes of
// one warp never diverge on it. Lane t's xoshiro256+ stream is exactly the
// reference's seed_worker(seed, t) stream; states live in registers for the
// whole launch and in SoA arrays (coalesced) between launches.
//
// k_sgd_replay: one lane runs the reference's threads=1 loop verbatim on
// FP64 coordinates with seed_worker(seed, 0): bit-identical to
// pglayout::run_layout(threads = 1).
#include <cuda_runtime.h>

#include "pgl_device.cuh"

namespace pgl {

namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;

__global__ void k_seed_rng(DevRng rng, uint64_t n, uint64_t seed) {
    const uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (t >= n) return;
    uint64_t s[4];
    seed_worker(seed, t, s);
    rng.s0[t] = s[0];
    rng.s1[t] = s[1];
    rng.s2[t] = s[2];
    rng.s3[t] = s[3];
}

__device__ __forceinline__ void flush_stats(DevStats* st, int idx, uint32_t v) {
    const uint32_t sum = __reduce_add_sync(kFull, v);
    if ((threadIdx.x & 31) == 0 && sum) atomicAdd(&st->v[idx], static_cast<unsigned long long>(sum));
}

template <typename T>
__global__ void __launch_bounds__(256) k_sgd_hogwild(DevGraph g, void* __restrict__ coords, DevRng rng,
                                                     DevStats* stats, IterArgs a) {
    const uint64_t tid = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    const uint32_t warp = static_cast<uint32_t>(tid >> 5);
    const uint32_t lane = threadIdx.x & 31;
    if (warp >= a.n_warps) return;  // whole warps only: the grid is warp-exact

    Xo r{rng.s0[tid], rng.s1[tid], rng.s2[tid], rng.s3[tid]};
    const uint64_t share = a.steps / a.n_warps;
    const uint64_t count = share + (warp < a.steps % a.n_warps ? 1 : 0);

    uint32_t applied = 0, b_first = 0, b_first_cool = 0, b_second = 0;
    bool carry = false;  // cooling flag of the batch still open at the round boundary
    for (uint64_t base = 0; base < count; base += 32) {
        const uint64_t s = base + lane;
        const bool active = s < count;
        const uint64_t in_batch = s % a.batch;
        bool mine = false;
        if (active && in_batch == 0) {  // this lane opens a batch (engine.cpp:115-124)
            if (a.force_cooling) {
                mine = true;
                ++b_second;
            } else {
                mine = r.coin();
                ++b_first;
                b_first_cool += mine;
            }
        }
        const int opener = in_batch <= lane ? static_cast<int>(lane - in_batch) : -1;
        const bool opened = __shfl_sync(kFull, mine, opener < 0 ? 0 : opener);
        const bool cooling = a.force_cooling ? true : (opener >= 0 ? opened : carry);
        carry = __shfl_sync(kFull, cooling, 31);
        if (active) applied += pgsgd_step<T>(g, coords, r, cooling, a.eta, a.theta, a.drf);
    }

    rng.s0[tid] = r.a;
    rng.s1[tid] = r.b;
    rng.s2[tid] = r.c;
    rng.s3[tid] = r.d;
    flush_stats(stats, 2, applied);
    flush_stats(stats, 4, b_first);
    flush_stats(stats, 5, b_first_cool);
    flush_stats(stats, 6, b_second);
    flush_stats(stats, 7, b_second);
}

__global__ void k_sgd_replay(DevGraph g, double* __restrict__ coords, uint64_t* rng4, DevStats* stats,
                             IterArgs a) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    Xo r{rng4[0], rng4[1], rng4[2], rng4[3]};
    unsigned long long applied = 0, bf = 0, bfc = 0, bs = 0;
    bool cooling = false;
    for (uint64_t s = 0; s < a.steps; ++s) {
        if (s % a.batch == 0) {
            cooling = a.force_cooling || r.coin();
            if (a.force_cooling)
                ++bs;
            else {
                ++bf;
                bfc += cooling;
            }
        }
        applied += pgsgd_step<double>(g, coords, r, cooling, a.eta, a.theta, a.drf);
    }
    rng4[0] = r.a;
    rng4[1] = r.b;
    rng4[2] = r.c;
    rng4[3] = r.d;
    stats->v[2] += applied;
    stats->v[4] += bf;
    stats->v[5] += bfc;
    stats->v[6] += bs;
    stats->v[7] += bs;
}

__global__ void k_f64_to_f32(const double* __restrict__ s, float* __restrict__ d, uint64_t n) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        d[i] = static_cast<float>(s[i]);
}

__global__ void k_f32_to_f64(const float* __restrict__ s, double* __restrict__ d, uint64_t n) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        d[i] = static_cast<double>(s[i]);
}

}  // namespace

LaunchShape sgd_shape(int device, int coord_f64, uint32_t max_warps, int block_threads) {
    LaunchShape sh;
    sh.threads = block_threads > 0 ? block_threads : 256;
    int sms = 0, occ = 0;
    PGL_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    if (coord_f64)
        PGL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sgd_hogwild<double>, sh.threads, 0));
    else
        PGL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sgd_hogwild<float>, sh.threads, 0));
    if (occ < 1) occ = 1;
    uint64_t warps = static_cast<uint64_t>(sms) * occ * (sh.threads / 32);
    if (max_warps && warps > max_warps) warps = max_warps;
    if (warps < 1) warps = 1;
    sh.blocks = static_cast<int>((warps * 32 + sh.threads - 1) / sh.threads);
    return sh;
}

void launch_seed_rng(DevRng rng, uint64_t n_lanes, uint64_t seed, void* stream) {
    const int tpb = 256;
    k_seed_rng<<<static_cast<unsigned>((n_lanes + tpb - 1) / tpb), tpb, 0,
                 static_cast<cudaStream_t>(stream)>>>(rng, n_lanes, seed);
    PGL_CUDA(cudaGetLastError());
}

void launch_sgd_hogwild(const DevGraph& g, void* coords, int coord_f64, DevRng rng, DevStats* stats,
                        const IterArgs& a, LaunchShape shape, void* stream) {
    auto s = static_cast<cudaStream_t>(stream);
    if (coord_f64)
        k_sgd_hogwild<double><<<shape.blocks, shape.threads, 0, s>>>(g, coords, rng, stats, a);
    else
        k_sgd_hogwild<float><<<shape.blocks, shape.threads, 0, s>>>(g, coords, rng, stats, a);
    PGL_CUDA(cudaGetLastError());
}

void launch_sgd_replay(const DevGraph& g, double* coords, uint64_t* rng4, DevStats* stats,
                       const IterArgs& a, void* stream) {
    k_sgd_replay<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(g, coords, rng4, stats, a);
    PGL_CUDA(cudaGetLastError());
}

void launch_f64_to_f32(const double* src, float* dst, uint64_t n, void* stream) {
    k_f64_to_f32<<<592, 256, 0, static_cast<cudaStream_t>(stream)>>>(src, dst, n);
    PGL_CUDA(cudaGetLastError());
}

void launch_f32_to_f64(const float* src, double* dst, uint64_t n, void* stream) {
    k_f32_to_f64<<<592, 256, 0, static_cast<cudaStream_t>(stream)>>>(src, dst, n);
    PGL_CUDA(cudaGetLastError());
}

}  // namespace pgl
