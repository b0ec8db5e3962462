// pgl_sps_stream.cu — PGL_SPS_STREAM: the reference's sampled path stress
// (metrics.cpp:108-159) with ITS OWN random stream, replayed in parallel.
//
// Per path p the reference draws from one xoshiro256+ stream
// seed_worker(seed, 2^61 + p) (rng.hpp:63-77), sample after sample: i =
// next_below(n); j = next_below(n) until j != i; then up to 9 coin pairs
// (e_i, e_j) until path_position differs; term ((|v_i - v_j| - d)/d)^2. The
// number of draws per sample is data dependent (collisions, degenerate
// endpoint pairs), so the stream cannot be split by sample index. Instead:
//   1. the stream is cut into chunks of D = 4096 draws; the xoshiro state
//      transition is linear over GF(2)^256, so the state at draw c*D is the
//      path's seed state times T^(c*D), applied as a product of precomputed
//      T^(2^k) (k >= 12) jump matrices (one matrix-vector product per set bit);
//   2. every chunk parses its draws from each of the four regular entry
//      phases (at a sample start; after i; after i, j; after i, j and the first
//      coin) and records the exit phase and the number of samples started;
//   3. one thread per path composes these chunk maps in order ("phase scan"),
//      parsing the rare irregular entries (after a collision redraw or a
//      degenerate coin pair) on the spot, which fixes every chunk's true entry
//      state and first sample index;
//   4. two passes over the chunks evaluate the terms of the samples that start
//      in each chunk (a sample may run past the chunk end), the sum and then
//      the squared deviations, folded in a fixed order.
// The terms, n and skipped are the reference's exactly; mean and sigma differ
// from its serial sums only by summation order (~1e-16 relative).
#include <cuda_runtime.h>

#include <vector>

#include "pgl_device.cuh"

namespace pgl {

namespace {

constexpr int kLog2D = 12;
constexpr uint64_t kD = 1ULL << kLog2D;
constexpr int kJumps = 44;  // T^(2^k), k = 12 .. 55
constexpr uint64_t kStreamSps = 1ULL << 61;  // rng.hpp:77
constexpr int kFold = 1024;

// ---- parse state ----------------------------------------------------------
// stage 0: next draw is i; 1: next is j (have i); 2: next is coin e_i of
// attempt `att` (have i, j); 3: next is coin e_j (have the e_i coin in c1).
// "Regular" = att == 0 and no collision redraw: then the state is fully
// given by the stage and the last `stage` draws before the boundary.
struct PState {
    uint64_t i, j;
    uint8_t stage, att, c1, regular;
    uint32_t _pad;
};

struct ChunkMap {        // per chunk: exit of the parse from each regular entry
    uint8_t exit_stage[4];  // 0..3 regular exit, 255 = irregular exit
    uint32_t started[4];    // samples started inside the chunk
};

struct ChunkEntry {      // per chunk: the true entry (after the phase scan)
    PState st;
    uint64_t first_sample;  // index of the first sample that starts in the chunk
    uint32_t active;        // the chunk starts at least one counted sample
    uint32_t _pad;
};

struct PathInfo {
    uint64_t base;           // cum_steps[p]
    uint64_t n;              // |p|
    uint64_t samples;        // spn * |p| (0 if |p| < 2)
    uint64_t chunk0;         // first global chunk index of the path
    uint64_t n_chunks;
};

// stream state of path p at draw index c * D
__device__ Xo chunk_state(uint64_t seed, uint32_t p, uint64_t c, const uint64_t* __restrict__ jumps) {
    uint64_t s[4];
    seed_worker(seed, kStreamSps + p, s);
    for (int k = 0; c; ++k, c >>= 1)
        if (c & 1) gf2_apply(s, jumps + static_cast<uint64_t>(k) * 256 * 4);
    return Xo{s[0], s[1], s[2], s[3]};
}

// One draw through the sampler's state machine. Returns 1 when a sample
// completes with a term (e_i, e_j in *ei/*ej), 2 when it completes skipped,
// 0 otherwise. `start` is set when the draw starts a sample.
__device__ __forceinline__ int step_draw(PState& s, uint64_t x, const DevGraph& g, uint64_t base, uint64_t n,
                                         bool& start, int& ei, int& ej) {
    start = false;
    switch (s.stage) {
        case 0:
            s.i = __umul64hi(x, n);
            s.stage = 1;
            s.att = 0;
            s.regular = 1;
            start = true;
            return 0;
        case 1:
            s.j = __umul64hi(x, n);
            if (s.j == s.i) {
                s.regular = 0;  // collision: redraw j (metrics.cpp:121-124)
                return 0;
            }
            s.stage = 2;
            return 0;
        case 2:
            s.c1 = static_cast<uint8_t>(x >> 63);
            s.stage = 3;
            return 0;
        default: {
            ei = s.c1 ? 0 : 1;               // flip_coin() ? start : end
            ej = (x >> 63) ? 0 : 1;
            const uint64_t d = s.i > s.j ? s.i - s.j : s.j - s.i;
            bool degenerate = false;
            if (d == 1) {  // only abutting steps can share a position
                const StepRec ri = load_step(g.step + base + s.i);
                const StepRec rj = load_step(g.step + base + s.j);
                degenerate = step_pos(ri, ei) == step_pos(rj, ej);
            }
            if (!degenerate) {
                s.stage = 0;
                return 1;
            }
            s.regular = 0;
            if (++s.att == 9) {  // nine degenerate coin pairs: skipped (metrics.cpp:129-147)
                s.stage = 0;
                return 2;
            }
            s.stage = 2;
            return 0;
        }
    }
}

// Regular entry state of phase `ph` from the draws just before the boundary
// (last[k] = draw at boundary - 1 - k).
__device__ __forceinline__ PState regular_entry(int ph, const uint64_t last[3], uint64_t n) {
    PState s{};
    s.stage = static_cast<uint8_t>(ph);
    s.regular = 1;
    if (ph >= 1) s.i = __umul64hi(last[ph - 1], n);
    if (ph >= 2) s.j = __umul64hi(last[ph - 2], n);
    if (ph == 3) s.c1 = static_cast<uint8_t>(last[0] >> 63);
    return s;
}

__device__ __forceinline__ uint32_t path_of_chunk(const PathInfo* __restrict__ pi, uint32_t P, uint64_t c) {
    uint32_t lo = 0, hi = P;
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (pi[mid].chunk0 <= c)
            lo = mid;
        else
            hi = mid;
    }
    return lo;
}

// Parse chunk draws [0, D) from `s`; returns the exit state, counts starts.
__device__ PState parse_chunk(PState s, Xo r, const DevGraph& g, uint64_t base, uint64_t n, uint32_t& started) {
    started = 0;
    for (uint64_t k = 0; k < kD; ++k) {
        bool st;
        int ei, ej;
        step_draw(s, r.next(), g, base, n, st, ei, ej);
        started += st;
    }
    return s;
}

// ---- 2. chunk maps ------------------------------------------------------------
__global__ void k_stream_maps(DevGraph g, uint64_t seed, const PathInfo* __restrict__ pinfo, uint32_t P,
                              uint64_t n_chunks, const uint64_t* __restrict__ jumps, ChunkMap* __restrict__ maps,
                              uint64_t* __restrict__ prev3) {
    const uint64_t c = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (c >= n_chunks) return;
    const uint32_t p = path_of_chunk(pinfo, P, c);
    const PathInfo pi = pinfo[p];
    const uint64_t lc = c - pi.chunk0;
    // the 3 draws before the chunk (regular entries need them)
    uint64_t last[3] = {0, 0, 0};
    Xo r;
    if (lc == 0) {
        r = chunk_state(seed, p, 0, jumps);
    } else {
        Xo q = chunk_state(seed, p, lc - 1, jumps);
        for (uint64_t k = 0; k < kD - 3; ++k) q.next();
        last[2] = q.next();
        last[1] = q.next();
        last[0] = q.next();
        r = q;
    }
    prev3[3 * c] = last[0];
    prev3[3 * c + 1] = last[1];
    prev3[3 * c + 2] = last[2];
    ChunkMap m;
    for (int ph = 0; ph < 4; ++ph) {
        if (lc == 0 && ph > 0) {
            m.exit_stage[ph] = 255;
            m.started[ph] = 0;
            continue;
        }
        uint32_t st = 0;
        const PState e = parse_chunk(regular_entry(ph, last, pi.n), r, g, pi.base, pi.n, st);
        m.exit_stage[ph] = e.regular && e.att == 0 ? e.stage : 255;
        m.started[ph] = st;
    }
    maps[c] = m;
}

// ---- 3. phase scan: one thread per path --------------------------------------------
// Regular entries carry only their stage (the values are the 3 draws before
// the chunk, prev3); irregular ones (rare) are found by parsing the chunk here
// and carry the full state.
__global__ void k_stream_scan(DevGraph g, uint64_t seed, const PathInfo* __restrict__ pinfo, uint32_t P,
                              const uint64_t* __restrict__ jumps, const ChunkMap* __restrict__ maps,
                              const uint64_t* __restrict__ prev3, ChunkEntry* __restrict__ entries,
                              unsigned* incomplete) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    const PathInfo pi = pinfo[p];
    PState s{};
    s.regular = 1;
    uint64_t done = 0;  // samples started so far
    for (uint64_t lc = 0; lc < pi.n_chunks; ++lc) {
        const uint64_t c = pi.chunk0 + lc;
        ChunkEntry ce;
        ce.st = s;
        ce.first_sample = done;
        ce.active = done < pi.samples ? 1u : 0u;
        ce._pad = 0;
        entries[c] = ce;
        if (done >= pi.samples) continue;
        uint32_t started;
        const bool reg = s.regular && s.att == 0;
        if (reg && maps[c].exit_stage[s.stage] != 255) {
            started = maps[c].started[s.stage];
            const uint8_t st = maps[c].exit_stage[s.stage];
            s = PState{};
            s.stage = st;
            s.regular = 1;
        } else {
            if (reg) {  // rebuild the regular entry's values
                const uint64_t last[3] = {prev3[3 * c], prev3[3 * c + 1], prev3[3 * c + 2]};
                s = regular_entry(s.stage, last, pi.n);
            }
            s = parse_chunk(s, chunk_state(seed, p, lc, jumps), g, pi.base, pi.n, started);
        }
        done += started;
    }
    if (done < pi.samples) atomicAdd(incomplete, 1u);
}

// ---- 4. terms ------------------------------------------------------------------------
template <typename T>
__global__ void k_stream_terms(DevGraph g, const void* __restrict__ coords, uint64_t seed,
                               const PathInfo* __restrict__ pinfo, uint32_t P, uint64_t n_chunks,
                               const uint64_t* __restrict__ jumps, const ChunkEntry* __restrict__ entries,
                               const uint64_t* __restrict__ prev3, int pass, const double* __restrict__ scal, double* __restrict__ part,
                               unsigned long long* __restrict__ cnt) {
    const uint64_t c = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (c >= n_chunks) return;
    double acc = 0.0;
    uint32_t nt = 0, nsk = 0;
    const ChunkEntry ce = entries[c];
    if (ce.active) {
        const uint32_t p = path_of_chunk(pinfo, P, c);
        const PathInfo pi = pinfo[p];
        const double mean = pass ? scal[1] : 0.0;
        Xo r = chunk_state(seed, p, c - pi.chunk0, jumps);
        PState s = ce.st;
        if (s.regular && s.att == 0 && s.stage > 0) {
            const uint64_t last[3] = {prev3[3 * c], prev3[3 * c + 1], prev3[3 * c + 2]};
            s = regular_entry(s.stage, last, pi.n);
        }
        uint64_t sample = ce.first_sample;
        bool mine = false;  // the sample in progress started in this chunk
        for (uint64_t k = 0;; ++k) {
            if (k >= kD && (s.stage == 0 || !mine)) break;   // past the chunk: finish only our own sample
            if (s.stage == 0 && sample >= pi.samples) break;  // all the path's samples are done
            bool st;
            int ei, ej;
            const int res = step_draw(s, r.next(), g, pi.base, pi.n, st, ei, ej);
            if (st) {
                mine = k < kD;
                ++sample;
            }
            if (res && mine) {
                if (res == 2) {
                    ++nsk;
                } else {
                    const StepRec ri = load_step(g.step + pi.base + s.i);
                    const StepRec rj = load_step(g.step + pi.base + s.j);
                    const double d = abs_diff(step_pos(ri, ei), step_pos(rj, ej));
                    double vix, viy, vjx, vjy;
                    Coord<T>::get(coords, ri.node, ei, vix, viy);
                    Coord<T>::get(coords, rj.node, ej, vjx, vjy);
                    const double dx = vix - vjx, dy = viy - vjy;
                    const double e = (sqrt(dx * dx + dy * dy) - d) / d;  // pair_stress, metrics.cpp:52-57
                    const double t = e * e;
                    if (pass == 0) {
                        acc += t;
                        ++nt;
                    } else {
                        acc += (t - mean) * (t - mean);
                    }
                }
            }
        }
    }
    part[c] = acc;
    if (pass == 0 && (nt || nsk)) {
        atomicAdd(cnt + 0, static_cast<unsigned long long>(nt));
        atomicAdd(cnt + 1, static_cast<unsigned long long>(nsk));
    }
}

__global__ void __launch_bounds__(kFold) k_stream_fold(const double* __restrict__ part, uint64_t n, int pass,
                                                       const unsigned long long* cnt, double* scal) {
    __shared__ double red[kFold];
    double acc = 0.0;
    for (uint64_t c = threadIdx.x; c < n; c += kFold) acc += part[c];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int w = kFold / 2; w >= 1; w >>= 1) {
        if (static_cast<int>(threadIdx.x) < w) red[threadIdx.x] += red[threadIdx.x + w];
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

// ---- host: jump matrices ----------------------------------------------------------
void xo_step(uint64_t s[4]) {  // RngState::next's state update (rng.hpp:21-31)
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = (s[3] << 45) | (s[3] >> 19);
}

void matvec(const uint64_t* M, const uint64_t in[4], uint64_t out[4]) {
    out[0] = out[1] = out[2] = out[3] = 0;
    for (int b = 0; b < 256; ++b)
        if ((in[b >> 6] >> (b & 63)) & 1)
            for (int w = 0; w < 4; ++w) out[w] ^= M[b * 4 + w];
}

// T^(2^k) for k = kLog2D .. kLog2D + kJumps - 1, column-major [256][4] each
std::vector<uint64_t> jump_tables() {
    std::vector<uint64_t> M(256 * 4), Q(256 * 4);
    for (int b = 0; b < 256; ++b) {
        uint64_t s[4] = {0, 0, 0, 0};
        s[b >> 6] = 1ULL << (b & 63);
        xo_step(s);
        for (int w = 0; w < 4; ++w) M[b * 4 + w] = s[w];
    }
    std::vector<uint64_t> out;
    for (int k = 0; k < kLog2D + kJumps; ++k) {
        if (k >= kLog2D) out.insert(out.end(), M.begin(), M.end());
        for (int b = 0; b < 256; ++b) matvec(M.data(), &M[b * 4], &Q[b * 4]);  // M := M * M
        M.swap(Q);
    }
    return out;
}

}  // namespace

void run_sps_stream(const DevGraph& g, const void* coords, int coord_f64, uint64_t seed, uint32_t spn,
                    pgl_stress_report* out, double* kernel_ms, void* stream_) {
    cudaStream_t s = static_cast<cudaStream_t>(stream_);
    const uint32_t P = g.n_paths;
    std::vector<uint64_t> cum(P + 1);
    PGL_CUDA(copy_async(cum.data(), g.cum, (P + 1) * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    PGL_CUDA(cudaStreamSynchronize(s));
    static const std::vector<uint64_t> J = jump_tables();
    uint64_t* dj = nullptr;
    PGL_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dj), J.size() * sizeof(uint64_t), s));
    PGL_CUDA(copy_async(dj, J.data(), J.size() * sizeof(uint64_t), cudaMemcpyHostToDevice, s));

    cudaEvent_t e0, e1;
    PGL_CUDA(cudaEventCreate(&e0));
    PGL_CUDA(cudaEventCreate(&e1));
    PGL_CUDA(cudaEventRecord(e0, s));
    double margin = 1.0;
    unsigned long long cnt_h[2] = {0, 0};
    double scal_h[4] = {0, 0, 0, 0};
    for (int attempt = 0;; ++attempt) {
        // chunks per path: expected draws per sample <= 4 + 2/(n-1) + 4/n (collision
        // redraws, degenerate coin pairs of abutting steps), with margin
        std::vector<PathInfo> pinfo(P);
        uint64_t total = 0;
        for (uint32_t p = 0; p < P; ++p) {
            const uint64_t n = cum[p + 1] - cum[p];
            PathInfo& pi = pinfo[p];
            pi.base = cum[p];
            pi.n = n;
            pi.samples = n >= 2 ? static_cast<uint64_t>(spn) * n : 0;
            const double per = n >= 2 ? 4.0 + 2.0 / static_cast<double>(n - 1) + 4.0 / static_cast<double>(n) : 0.0;
            const double draws = margin * (static_cast<double>(pi.samples) * per * 1.01 + 64.0) + (pi.samples ? kD : 0);
            pi.n_chunks = pi.samples ? static_cast<uint64_t>(draws / static_cast<double>(kD)) + 1 : 0;
            pi.chunk0 = total;
            total += pi.n_chunks;
        }
        if (P == 0 || total == 0) break;
        PathInfo* dpi = nullptr;
        ChunkMap* maps = nullptr;
        ChunkEntry* ent = nullptr;
        double* part = nullptr;
        double* scal = nullptr;
        unsigned long long* cnt = nullptr;
        unsigned* incomplete = nullptr;
        uint64_t* prev3 = nullptr;
        PGL_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&prev3), 3 * total * sizeof(uint64_t), s));
        PGL_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dpi), P * sizeof(PathInfo), s));
        PGL_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&maps), total * sizeof(ChunkMap), s));
        PGL_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ent), total * sizeof(ChunkEntry), s));
        PGL_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&part), total * sizeof(double), s));
        PGL_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&scal), 4 * sizeof(double), s));
        PGL_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&cnt), 2 * sizeof(unsigned long long), s));
        PGL_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&incomplete), sizeof(unsigned), s));
        PGL_CUDA(copy_async(dpi, pinfo.data(), P * sizeof(PathInfo), cudaMemcpyHostToDevice, s));
        PGL_CUDA(cudaMemsetAsync(cnt, 0, 2 * sizeof(unsigned long long), s));
        PGL_CUDA(cudaMemsetAsync(scal, 0, 4 * sizeof(double), s));
        PGL_CUDA(cudaMemsetAsync(incomplete, 0, sizeof(unsigned), s));
        const unsigned blocks = static_cast<unsigned>((total + 127) / 128);
        k_stream_maps<<<blocks, 128, 0, s>>>(g, seed, dpi, P, total, dj, maps, prev3);
        PGL_CUDA(cudaGetLastError());
        k_stream_scan<<<(P + 63) / 64, 64, 0, s>>>(g, seed, dpi, P, dj, maps, prev3, ent, incomplete);
        PGL_CUDA(cudaGetLastError());
        unsigned inc = 0;
        PGL_CUDA(copy_async(&inc, incomplete, sizeof inc, cudaMemcpyDeviceToHost, s));
        PGL_CUDA(cudaStreamSynchronize(s));
        if (inc == 0) {
            for (int pass = 0; pass < 2; ++pass) {
                if (coord_f64 == PGL_COORD_F64)
                    k_stream_terms<double><<<blocks, 128, 0, s>>>(g, coords, seed, dpi, P, total, dj, ent, prev3, pass,
                                                                  scal, part, cnt);
                else if (coord_f64 == PGL_COORD_F32)
                    k_stream_terms<float><<<blocks, 128, 0, s>>>(g, coords, seed, dpi, P, total, dj, ent, prev3, pass,
                                                                 scal, part, cnt);
                else
                    k_stream_terms<AnchF32><<<blocks, 128, 0, s>>>(g, coords, seed, dpi, P, total, dj, ent, prev3,
                                                                   pass, scal, part, cnt);
                PGL_CUDA(cudaGetLastError());
                k_stream_fold<<<1, kFold, 0, s>>>(part, total, pass, cnt, scal);
                PGL_CUDA(cudaGetLastError());
            }
            PGL_CUDA(copy_async(cnt_h, cnt, sizeof cnt_h, cudaMemcpyDeviceToHost, s));
            PGL_CUDA(copy_async(scal_h, scal, sizeof scal_h, cudaMemcpyDeviceToHost, s));
        }
        PGL_CUDA(cudaStreamSynchronize(s));
        for (void* ptr : {static_cast<void*>(prev3), static_cast<void*>(dpi), static_cast<void*>(maps), static_cast<void*>(ent),
                          static_cast<void*>(part), static_cast<void*>(scal), static_cast<void*>(cnt),
                          static_cast<void*>(incomplete)})
            PGL_CUDA(cudaFreeAsync(ptr, s));
        if (inc == 0) break;
        if (attempt > 8) raise(PGL_ERR_INDEX_OUT_OF_RANGE, "sampled stress stream replay did not converge");
        margin *= 2.0;  // some path needed more draws than budgeted: redo with more chunks
    }
    PGL_CUDA(cudaEventRecord(e1, s));
    PGL_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    PGL_CUDA(cudaFreeAsync(dj, s));
    PGL_CUDA(cudaStreamSynchronize(s));
    if (kernel_ms) *kernel_ms = ms;
    out->n = cnt_h[0];
    out->skipped = cnt_h[1];
    out->mean = scal_h[1];
    finish_report(out, scal_h[2]);
}

}  // namespace pgl
