// pgl_sps.cu — sampled path stress as a deterministic GPU reduction.
//
// Estimator of metrics.cpp:108-159: per path p with >= 2 steps,
// samples_per_node * |p| samples of (distinct uniform step pair, coin-flipped
// endpoints, up to 9 coin attempts for a nonzero d_ref), term
// ((|v_i - v_j| - d_ref) / d_ref)^2 (pair_stress, metrics.cpp:52-57), mean,
// second-pass sigma (n - 1), CI mean +- 1.96 sigma / sqrt(n).
//
// PGL_SPS_COUNTER: every sample owns a counter-based stream (splitmix64 at
// counter sample*64 + t, keyed per path), so the two passes regenerate the
// same terms without storing them (the reference stores all terms: 70 GB at
// config 2). Fixed chunks of 4096 samples are reduced in a fixed tree order
// and the chunk partials folded in a fixed order, so the result is
// bit-reproducible for any grid size and equals the C
// restatement orc_sps_counter bit for bit.
#include <cuda_runtime.h>

#include <chrono>

#include "pgl_device.cuh"

namespace pgl {

namespace {

constexpr int kLanes = 256;
constexpr int kChunk = 4096;
constexpr int kFinal = 1024;
constexpr uint64_t kStreamSps = 1ULL << 61;  // rng.hpp:77

__device__ __forceinline__ uint64_t ctr_draw(uint64_t key, uint64_t ctr) {
    uint64_t z = key + (ctr + 1) * kPhi;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

template <typename T>
__device__ __forceinline__ int sps_sample(const DevGraph& g, const void* coords, uint64_t seed,
                                          uint32_t spn, uint64_t q, double& term) {
    uint32_t lo = 0, hi = g.n_paths;
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (static_cast<uint64_t>(spn) * __ldg(g.cum + mid) <= q)
            lo = mid;
        else
            hi = mid;
    }
    const uint64_t base = __ldg(g.cum + lo);
    const uint64_t ns = __ldg(g.cum + lo + 1) - base;
    if (ns < 2) return -1;
    const uint64_t s = q - static_cast<uint64_t>(spn) * base;
    uint64_t key = seed ^ (kPhi * (kStreamSps + lo + 1));
    key = splitmix_next(key);
    const uint64_t i = __umul64hi(ctr_draw(key, s * 64), ns);
    uint64_t j = i;
    for (uint64_t t = 1; t < 48 && j == i; ++t) j = __umul64hi(ctr_draw(key, s * 64 + t), ns);
    if (j == i) return 0;
    const StepRec ri = load_step(g.step + base + i);
    const StepRec rj = load_step(g.step + base + j);
    for (uint64_t att = 0; att < 9; ++att) {
        const uint64_t rr = ctr_draw(key, s * 64 + 48 + att);
        const int ei = (rr >> 63) ? 0 : 1;
        const int ej = ((rr >> 62) & 1) ? 0 : 1;
        const uint64_t pi = step_pos(ri, ei), pj = step_pos(rj, ej);
        if (pi == pj) continue;
        const double d = abs_diff(pi, pj);
        double vix, viy, vjx, vjy;
        Coord<T>::get(coords, ri.node, ei, vix, viy);
        Coord<T>::get(coords, rj.node, ej, vjx, vjy);
        const double dx = vix - vjx, dy = viy - vjy;
        const double err = (sqrt(dx * dx + dy * dy) - d) / d;
        term = err * err;
        return 1;
    }
    return 0;
}

template <typename T>
__global__ void __launch_bounds__(kLanes) k_sps_chunks(DevGraph g, const void* __restrict__ coords,
                                                       uint64_t seed, uint32_t spn, uint64_t Q,
                                                       uint64_t n_chunks, int pass,
                                                       const double* __restrict__ scal,
                                                       double* __restrict__ part,
                                                       unsigned long long* cnt) {
    __shared__ double red[kLanes];
    const double mean = pass ? scal[1] : 0.0;
    uint32_t nt = 0, nsk = 0;
    for (uint64_t ch = blockIdx.x; ch < n_chunks; ch += gridDim.x) {
        double acc = 0.0;
        const uint64_t end = (ch + 1) * kChunk < Q ? (ch + 1) * kChunk : Q;
        for (uint64_t q = ch * kChunk + threadIdx.x; q < end; q += kLanes) {
            double t;
            const int k = sps_sample<T>(g, coords, seed, spn, q, t);
            if (k == 1) {
                if (pass == 0) {
                    acc += t;
                    ++nt;
                } else {
                    acc += (t - mean) * (t - mean);
                }
            } else if (k == 0) {
                ++nsk;
            }
        }
        red[threadIdx.x] = acc;
        __syncthreads();
        for (int stride = kLanes / 2; stride >= 1; stride >>= 1) {
            if (threadIdx.x < stride) red[threadIdx.x] += red[threadIdx.x + stride];
            __syncthreads();
        }
        if (threadIdx.x == 0) part[ch] = red[0];
        __syncthreads();
    }
    if (pass == 0) {
        const uint32_t a = __reduce_add_sync(0xFFFFFFFFu, nt);
        const uint32_t b = __reduce_add_sync(0xFFFFFFFFu, nsk);
        if ((threadIdx.x & 31) == 0) {
            if (a) atomicAdd(cnt + 0, static_cast<unsigned long long>(a));
            if (b) atomicAdd(cnt + 1, static_cast<unsigned long long>(b));
        }
    }
}

__global__ void __launch_bounds__(kFinal) k_sps_fold(const double* __restrict__ part, uint64_t n_chunks,
                                                    int pass, const unsigned long long* cnt,
                                                    double* scal) {
    __shared__ double red[kFinal];
    double acc = 0.0;
    for (uint64_t c = threadIdx.x; c < n_chunks; c += kFinal) acc += part[c];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int stride = kFinal / 2; stride >= 1; stride >>= 1) {
        if (threadIdx.x < stride) red[threadIdx.x] += red[threadIdx.x + stride];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        if (pass == 0) {
            scal[0] = red[0];
            scal[1] = cnt[0] > 0 ? red[0] / static_cast<double>(cnt[0]) : 0.0;
        } else {
            scal[2] = red[0];
        }
    }
}

}  // namespace

void run_sps_counter(const DevGraph& g, const void* coords, int coord_f64 /* pgl_coord_precision */, uint64_t seed, uint32_t spn,
                     SpsScratch& sc, pgl_stress_report* out, double* kernel_ms, void* stream) {
    auto s = static_cast<cudaStream_t>(stream);
    const uint64_t Q = static_cast<uint64_t>(spn) * g.total_steps;
    const uint64_t n_chunks = (Q + kChunk - 1) / kChunk;
    if (n_chunks > sc.n_chunks_cap) {
        if (sc.part) PGL_CUDA(cudaFree(sc.part));
        PGL_CUDA(cudaMalloc(&sc.part, (n_chunks + 1) * sizeof(double)));
        sc.n_chunks_cap = n_chunks;
    }
    if (!sc.cnt) PGL_CUDA(cudaMalloc(&sc.cnt, 2 * sizeof(unsigned long long)));
    if (!sc.scal) PGL_CUDA(cudaMalloc(&sc.scal, 4 * sizeof(double)));
    PGL_CUDA(cudaMemsetAsync(sc.cnt, 0, 2 * sizeof(unsigned long long), s));
    PGL_CUDA(cudaMemsetAsync(sc.scal, 0, 4 * sizeof(double), s));

    int dev = 0, sms = 0, occ = 0;
    PGL_CUDA(cudaGetDevice(&dev));
    PGL_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    PGL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sps_chunks<double>, kLanes, 0));
    uint64_t blocks = static_cast<uint64_t>(sms) * (occ > 0 ? occ : 1);
    if (blocks > n_chunks) blocks = n_chunks ? n_chunks : 1;

    cudaEvent_t e0, e1;
    PGL_CUDA(cudaEventCreate(&e0));
    PGL_CUDA(cudaEventCreate(&e1));
    PGL_CUDA(cudaEventRecord(e0, s));
    for (int pass = 0; pass < 2; ++pass) {
        if (n_chunks) {
            if (coord_f64 == PGL_COORD_F64)
                k_sps_chunks<double><<<static_cast<unsigned>(blocks), kLanes, 0, s>>>(
                    g, coords, seed, spn, Q, n_chunks, pass, sc.scal, sc.part, sc.cnt);
            else if (coord_f64 == PGL_COORD_F32)
                k_sps_chunks<float><<<static_cast<unsigned>(blocks), kLanes, 0, s>>>(
                    g, coords, seed, spn, Q, n_chunks, pass, sc.scal, sc.part, sc.cnt);
            else
                k_sps_chunks<AnchF32><<<static_cast<unsigned>(blocks), kLanes, 0, s>>>(
                    g, coords, seed, spn, Q, n_chunks, pass, sc.scal, sc.part, sc.cnt);
            PGL_CUDA(cudaGetLastError());
        }
        k_sps_fold<<<1, kFinal, 0, s>>>(sc.part, n_chunks, pass, sc.cnt, sc.scal);
        PGL_CUDA(cudaGetLastError());
    }
    PGL_CUDA(cudaEventRecord(e1, s));
    unsigned long long cnt[2];
    double scal[4];
    PGL_CUDA(copy_async(cnt, sc.cnt, sizeof cnt, cudaMemcpyDeviceToHost, s));
    PGL_CUDA(copy_async(scal, sc.scal, sizeof scal, cudaMemcpyDeviceToHost, s));
    PGL_CUDA(cudaStreamSynchronize(s));
    float ms = 0.f;
    PGL_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (kernel_ms) *kernel_ms = ms;
    out->n = cnt[0];
    out->skipped = cnt[1];
    out->mean = scal[1];
    finish_report(out, scal[2]);
}

}  // namespace pgl
