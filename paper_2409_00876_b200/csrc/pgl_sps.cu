// pgl_sps.cu — sampled path stress as a deterministic GPU reduction.
//
// Estimator of metrics.cpp:108-159: per path p with >= 2 steps,
// samples_per_node * |p| samples of (distinct step pair, coin-flipped
// endpoints, up to 9 coin attempts for a nonzero d_ref), term
// ((|v_i - v_j| - d_ref) / d_ref)^2 (pair_stress, metrics.cpp:52-57), mean,
// sigma with n - 1, CI mean +- 1.96 sigma / sqrt(n).
//
// PGL_SPS_COUNTER: every sample owns a counter-based stream (splitmix64 at
// counter sample*16 + t, keyed per path), so nothing is stored (the
// reference stores all terms: 70 GB at config 2, spn 100). The primary step
// is stratified -- sample s of path p takes i = s mod |p|, every step exactly
// spn times, consecutive samples on consecutive steps (coalesced i-side
// records and endpoints) -- and j is uniform over the other steps, so every
// term has the reference's distribution given i and the mean is unbiased for
// the same quantity. One pass: (count, mean, M2) per lane by Welford, merged
// pairwise (Chan et al.) in a fixed tree within each path-major chunk of
// 16384 samples and in a fixed fold across chunks -- bit-reproducible for any
// grid size and equal to the C restatement orc_sps_counter bit
// for bit.
#include <cuda_runtime.h>

#include <chrono>
#include <vector>

#include "pgl_device.cuh"

namespace pgl {

namespace {

constexpr int kLanes = 256;
constexpr uint64_t kChunk = 16384;  // samples per chunk: 64 per lane
constexpr int kFinal = 1024;
constexpr uint64_t kStreamSps = 1ULL << 61;  // rng.hpp:77

__device__ __forceinline__ uint64_t ctr_draw(uint64_t key, uint64_t ctr) {
    uint64_t z = key + (ctr + 1) * kPhi;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// Running (count, mean, M2) of a set of terms: Welford per lane, Chan et
// al.'s pairwise merge between lanes and chunks. Every operation is IEEE
// double (-fmad=false), in a fixed order, so the C restatement
// (orc_sps_counter) reproduces it bit for bit.
struct Moments {
    double n, mean, m2;
};

__device__ __forceinline__ void push(Moments& a, double t) {
    a.n += 1.0;
    const double d = t - a.mean;
    a.mean += d / a.n;
    a.m2 += d * (t - a.mean);
}

__device__ __forceinline__ Moments merge(const Moments& a, const Moments& b) {
    if (b.n == 0.0) return a;
    if (a.n == 0.0) return b;
    const double n = a.n + b.n;
    const double d = b.mean - a.mean;
    return Moments{n, a.mean + d * (b.n / n), a.m2 + b.m2 + d * d * (a.n * b.n / n)};
}

// Sample s of path p (|p| = ns >= 2 steps, s < spn * ns): primary step
// i = s mod ns -- each step exactly spn times, consecutive samples on
// consecutive steps -- and j uniform over the other ns - 1 steps; then up to
// 9 coin attempts for a nonzero d_ref (metrics.cpp:116-148). Draw t of sample
// s is the splitmix64 output at counter s*16 + t of the path's key.
#ifndef PGL_SPS_GROUP
#define PGL_SPS_GROUP 2
#endif
#ifndef PGL_SPS_MINB
#define PGL_SPS_MINB 1
#endif
constexpr int kGroup = PGL_SPS_GROUP;  // samples per lane in flight

// One block per chunk (grid-stride): chunks are path-major -- chunk c of
// path p covers samples [c*kChunk, min((c+1)*kChunk, spn*|p|)) of p -- so the
// path is found once per chunk (chunk_cum: prefix of chunks per path), not
// once per sample. Lane l takes samples l, l+256, ...; lane moments are
// merged by a halving tree; one Moments per chunk.
template <typename T>
__global__ void __launch_bounds__(kLanes, PGL_SPS_MINB) k_sps_chunks(DevGraph g, const void* __restrict__ coords, uint64_t seed,
                                                       uint32_t spn, const uint64_t* __restrict__ chunk_cum,
                                                       uint64_t n_chunks, Moments* __restrict__ part,
                                                       unsigned long long* skipped) {
    __shared__ Moments red[kLanes];
    uint32_t nsk = 0;
    for (uint64_t ch = blockIdx.x; ch < n_chunks; ch += gridDim.x) {
        uint32_t lo = 0, hi = g.n_paths;  // largest p with chunk_cum[p] <= ch
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (__ldg(chunk_cum + mid) <= ch)
                lo = mid;
            else
                hi = mid;
        }
        const uint64_t base = __ldg(g.cum + lo);
        const uint64_t ns = __ldg(g.cum + lo + 1) - base;
        const uint64_t s0 = (ch - __ldg(chunk_cum + lo)) * kChunk;
        const uint64_t s_end = static_cast<uint64_t>(spn) * ns < s0 + kChunk ? static_cast<uint64_t>(spn) * ns
                                                                             : s0 + kChunk;
        uint64_t key = seed ^ (kPhi * (kStreamSps + lo + 1));
        key = splitmix_next(key);
        const uint64_t i0 = s0 % ns;
        Moments m{0.0, 0.0, 0.0};
        // kGroup samples per lane in flight: their record loads, then their
        // coordinate loads, are issued together (memory-level parallelism);
        // the terms are pushed in sample order, as the C restatement does
        for (uint64_t g0 = threadIdx.x; s0 + g0 < s_end; g0 += kGroup * kLanes) {
            StepRec ri[kGroup], rj[kGroup];
            int ok[kGroup];
            uint64_t pos[kGroup][2];
#pragma unroll
            for (int q = 0; q < kGroup; ++q) {
                const uint64_t off = g0 + static_cast<uint64_t>(q) * kLanes;
                ok[q] = s0 + off < s_end;
                if (!ok[q]) continue;
                uint64_t i = i0 + off;
                if (ns >= kChunk) {
                    if (i >= ns) i -= ns;
                } else {
                    i = static_cast<uint32_t>(i) % static_cast<uint32_t>(ns);
                }
                uint64_t j = __umul64hi(ctr_draw(key, (s0 + off) * 16), ns - 1);
                j += j >= i ? 1 : 0;
                ri[q] = load_step(g.step + base + i);
                rj[q] = load_step(g.step + base + j);
            }
            int ends[kGroup];
#pragma unroll
            for (int q = 0; q < kGroup; ++q) {
                if (!ok[q]) continue;
                ok[q] = 0;
                const uint64_t s = s0 + g0 + static_cast<uint64_t>(q) * kLanes;
                for (uint64_t att = 0; att < 9; ++att) {  // metrics.cpp:116-148: up to 9 coin attempts
                    const uint64_t rr = ctr_draw(key, s * 16 + 1 + att);
                    const int ei = (rr >> 63) ? 0 : 1;
                    const int ej = ((rr >> 62) & 1) ? 0 : 1;
                    const uint64_t pi = step_pos(ri[q], ei), pj = step_pos(rj[q], ej);
                    if (pi == pj) continue;
                    pos[q][0] = pi;
                    pos[q][1] = pj;
                    ends[q] = ei | (ej << 1);
                    ok[q] = 1;
                    break;
                }
            }
            double vix[kGroup], viy[kGroup], vjx[kGroup], vjy[kGroup];
#pragma unroll
            for (int q = 0; q < kGroup; ++q) {
                if (!ok[q]) continue;
                Coord<T>::get(coords, ri[q].node, ends[q] & 1, vix[q], viy[q]);
                Coord<T>::get(coords, rj[q].node, ends[q] >> 1, vjx[q], vjy[q]);
            }
#pragma unroll
            for (int q = 0; q < kGroup; ++q) {
                if (s0 + g0 + static_cast<uint64_t>(q) * kLanes >= s_end) continue;
                if (!ok[q]) {
                    ++nsk;
                    continue;
                }
                const double d = abs_diff(pos[q][0], pos[q][1]);
                const double dx = vix[q] - vjx[q], dy = viy[q] - vjy[q];
                const double err = (sqrt(dx * dx + dy * dy) - d) / d;
                push(m, err * err);
            }
        }
        red[threadIdx.x] = m;
        __syncthreads();
        for (int stride = kLanes / 2; stride >= 1; stride >>= 1) {
            if (threadIdx.x < stride) red[threadIdx.x] = merge(red[threadIdx.x], red[threadIdx.x + stride]);
            __syncthreads();
        }
        if (threadIdx.x == 0) part[ch] = red[0];
        __syncthreads();
    }
    const uint32_t b = __reduce_add_sync(0xFFFFFFFFu, nsk);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(skipped, static_cast<unsigned long long>(b));
}

// Fold the chunk moments in a fixed order: lane l merges chunks l, l+1024,
// ... in sequence, then a halving tree.
__global__ void __launch_bounds__(kFinal) k_sps_fold(const Moments* __restrict__ part, uint64_t n_chunks,
                                                    Moments* out) {
    __shared__ Moments red[kFinal];
    Moments acc{0.0, 0.0, 0.0};
    for (uint64_t c = threadIdx.x; c < n_chunks; c += kFinal) acc = merge(acc, part[c]);
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int stride = kFinal / 2; stride >= 1; stride >>= 1) {
        if (threadIdx.x < stride) red[threadIdx.x] = merge(red[threadIdx.x], red[threadIdx.x + stride]);
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = red[0];
}

}  // namespace

// Counter-based sampled path stress (PGL_SPS_COUNTER), one pass over
// spn * sum|p| samples; deterministic for any grid.
void run_sps_counter(const DevGraph& g, const void* coords, int coord_kind, const uint64_t* path_n_steps,
                     uint64_t seed, uint32_t spn, SpsScratch& sc, pgl_stress_report* out, double* kernel_ms,
                     void* stream) {
    auto s = static_cast<cudaStream_t>(stream);
    const uint32_t P = g.n_paths;
    std::vector<uint64_t> chunk_cum(P + 1, 0);
    for (uint32_t p = 0; p < P; ++p) {
        const uint64_t ns = path_n_steps[p];
        const uint64_t q = ns >= 2 ? static_cast<uint64_t>(spn) * ns : 0;
        chunk_cum[p + 1] = chunk_cum[p] + (q + kChunk - 1) / kChunk;
    }
    const uint64_t n_chunks = chunk_cum[P];
    const size_t need = (n_chunks + 1) * sizeof(Moments) + (P + 1) * sizeof(uint64_t);
    if (need > sc.part_bytes) {
        if (sc.part) PGL_CUDA(cudaFree(sc.part));
        PGL_CUDA(cudaMalloc(&sc.part, need));
        sc.part_bytes = need;
    }
    Moments* part = static_cast<Moments*>(sc.part);
    uint64_t* d_chunk_cum = reinterpret_cast<uint64_t*>(part + n_chunks + 1);
    if (!sc.cnt) PGL_CUDA(cudaMalloc(&sc.cnt, 2 * sizeof(unsigned long long)));
    if (!sc.scal) PGL_CUDA(cudaMalloc(&sc.scal, 4 * sizeof(double)));
    PGL_CUDA(cudaMemsetAsync(sc.cnt, 0, 2 * sizeof(unsigned long long), s));
    PGL_CUDA(cudaMemsetAsync(sc.scal, 0, 4 * sizeof(double), s));
    PGL_CUDA(copy_async(d_chunk_cum, chunk_cum.data(), (P + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, s));

    int dev = 0, sms = 0, occ = 0;
    PGL_CUDA(cudaGetDevice(&dev));
    PGL_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    PGL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sps_chunks<double>, kLanes, 0));
    uint64_t blocks = static_cast<uint64_t>(sms) * (occ > 0 ? occ : 1) * 4;
    if (blocks > n_chunks) blocks = n_chunks ? n_chunks : 1;

    cudaEvent_t e0, e1;
    PGL_CUDA(cudaEventCreate(&e0));
    PGL_CUDA(cudaEventCreate(&e1));
    PGL_CUDA(cudaEventRecord(e0, s));
    Moments* tot = reinterpret_cast<Moments*>(sc.scal);
    if (n_chunks) {
        if (coord_kind == PGL_COORD_F64)
            k_sps_chunks<double><<<static_cast<unsigned>(blocks), kLanes, 0, s>>>(g, coords, seed, spn, d_chunk_cum,
                                                                               n_chunks, part, sc.cnt + 1);
        else if (coord_kind == PGL_COORD_F32)
            k_sps_chunks<float><<<static_cast<unsigned>(blocks), kLanes, 0, s>>>(g, coords, seed, spn, d_chunk_cum,
                                                                              n_chunks, part, sc.cnt + 1);
        else
            k_sps_chunks<AnchF32><<<static_cast<unsigned>(blocks), kLanes, 0, s>>>(g, coords, seed, spn, d_chunk_cum,
                                                                                n_chunks, part, sc.cnt + 1);
        PGL_CUDA(cudaGetLastError());
    }
    k_sps_fold<<<1, kFinal, 0, s>>>(part, n_chunks, tot);
    PGL_CUDA(cudaGetLastError());
    PGL_CUDA(cudaEventRecord(e1, s));
    unsigned long long cnt[2];
    Moments m;
    PGL_CUDA(copy_async(cnt, sc.cnt, sizeof cnt, cudaMemcpyDeviceToHost, s));
    PGL_CUDA(copy_async(&m, tot, sizeof m, cudaMemcpyDeviceToHost, s));
    PGL_CUDA(cudaStreamSynchronize(s));
    float ms = 0.f;
    PGL_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (kernel_ms) *kernel_ms = ms;
    out->n = static_cast<uint64_t>(m.n);
    out->skipped = cnt[1];
    out->mean = m.mean;
    finish_report(out, m.m2);
}

}  // namespace pgl
