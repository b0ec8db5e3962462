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
// (PGL_MODE_REPLAY lives in pgl_replay.cu.)
#include <cuda_runtime.h>

#include <algorithm>

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

// One selected step pair in flight between the two pipeline stages.
struct Sel {
    StepRec ri, rj;
    uint32_t flags;  // bit0 valid, bit1 e_i is end, bit2 e_j is end, bit4 active primary step, bit5 cooling
};

// Stage A (warp-uniform call): the batch decision of engine.cpp:115-124 for
// this round, then select_step_pair (:52-80) and the two endpoint coins, and
// issue the two step-record gathers. Nothing waits on the gathers here.
// `bpos` is base % batch, advanced here by one round (no 64-bit modulo per
// lane and round).
template <bool kActiveCheck>
__device__ __forceinline__ Sel stage_select(const DevGraph& g, Xo& r, const IterArgs& a, uint64_t base,
                                            uint64_t count, uint32_t lane, bool& carry, uint32_t& b_first,
                                            uint32_t& b_first_cool, uint32_t& b_second, uint64_t pol_stream,
                                            uint32_t& bpos) {
    const uint64_t s = base + lane;
    const bool active = s < count;
    uint32_t in_batch = bpos + lane;
    if (a.batch >= 32) {
        if (in_batch >= a.batch) in_batch -= a.batch;
        bpos += 32;
        if (bpos >= a.batch) bpos -= a.batch;
    } else {
        in_batch %= a.batch;
        bpos = (bpos + 32) % a.batch;
    }
    bool mine = false;
    if (active && in_batch == 0) {
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

    Sel out;
    out.flags = 0;
    out.ri = out.rj = StepRec{0, 0, 0, 0};
    if (!active) return out;
    out.flags = 16u | (cooling ? 32u : 0u);
    const uint64_t x = r.next();
    const uint64_t pick = __umul64hi(x, g.total_steps);
    const uint32_t p = select_path(g, x, pick);
    const uint64_t pbase = __ldg(g.cum + p);
    const int64_t n = static_cast<int64_t>(__ldg(g.cum + p + 1) - pbase);
    if (a.visits != nullptr) atomicAdd(a.visits + pick, 1u);  // diagnostics only
    if (n < 2) return out;
    const int64_t i = static_cast<int64_t>(pick - pbase);
    int64_t j;
    uint64_t bits;
    if (cooling) {
        const uint32_t zn = static_cast<uint32_t>(__ldg(&g.pc[p].zn));
        const uint64_t zt = __ldg(&g.pc[p].ztab);
        const int64_t k = static_cast<int64_t>(zipf_alias(g.zalias + zt, zn, r.next()));
        diag_zipf(a, static_cast<uint64_t>(k));
        bits = r.next();
        const int64_t sign = (bits >> 61) & 1 ? 1 : -1;
        j = i + sign * k;
        if (j < 0 || j >= n) {
            j = i - sign * k;
            if (j < 0 || j >= n) {
                j = i + sign * k;
                j = j < 0 ? 0 : (j > n - 1 ? n - 1 : j);
            }
        }
        if (j == i) return out;
    } else {
        j = static_cast<int64_t>(r.below(static_cast<uint64_t>(n)));
        if (j == i) {
            j = static_cast<int64_t>(r.below(static_cast<uint64_t>(n)));
            if (j == i) return out;
        }
        bits = r.next();
    }
    out.ri = load_step_stream(g.step + pbase + i, pol_stream);
    out.rj = load_step_stream(g.step + pbase + j, pol_stream);
    // coin true -> Endpoint::start (engine.cpp:89-91): a set bit means start
    out.flags = 17u | (cooling ? 32u : 0u) | ((bits >> 63) ? 0u : 2u) | (((bits >> 62) & 1) ? 0u : 4u);
    return out;
}

// Stage B: the update(s) of one selected pair (engine.cpp:133-170).
template <typename T>
__device__ __forceinline__ uint32_t stage_update(const Sel& sel, void* coords, Xo& r, const IterArgs& a,
                                                 uint64_t pol, uint32_t& primary, uint32_t& skipped) {
    if (sel.flags & 16u) ++primary;
    if (!(sel.flags & 1u)) {
        if (sel.flags & 16u) {
            skipped += a.drf;  // an invalid selection skips all drf updates
            diag_outcome(a, sel.flags & 32u, false);
        }
        return 0;
    }
    const int ei = (sel.flags >> 1) & 1, ej = (sel.flags >> 2) & 1;
    uint32_t applied = hog_update_t<T>(coords, sel.ri.node, ei, sel.rj.node, ej,
                                     abs_diff(step_pos(sel.ri, ei), step_pos(sel.rj, ej)), a.eta, r, pol);
    skipped += 1u - applied;
    diag_outcome(a, sel.flags & 32u, applied != 0);
    if (a.drf > 1) {
        unsigned used = 1u << ((ei ? 2 : 0) | (ej ? 1 : 0));
        for (uint32_t extra = 1; extra < a.drf; ++extra) {
            int ea, eb;
            do {
                const uint64_t bits = r.next();
                ea = (bits >> 63) ? 0 : 1;
                eb = ((bits >> 62) & 1) ? 0 : 1;
            } while (used & (1u << ((ea ? 2 : 0) | (eb ? 1 : 0))));
            used |= 1u << ((ea ? 2 : 0) | (eb ? 1 : 0));
            const uint32_t ok = hog_update_t<T>(coords, sel.ri.node, ea, sel.rj.node, eb,
                                                abs_diff(step_pos(sel.ri, ea), step_pos(sel.rj, eb)), a.eta, r, pol);
            applied += ok;
            skipped += 1u - ok;
        }
    }
    return applied;
}

// kDepth: rounds in flight per warp. Round r's step records are gathered
// while rounds r-kDepth+1 .. r-1 update; the records are read-only, so a
// deeper record pipeline adds memory-level parallelism without widening any
// coordinate's read-to-write window (each update still reads its endpoints
// and writes them back in one stage, as apply_endpoint_update does).
// kPrefetch: while round r updates, the endpoint lines of round r+1 (whose
// records arrived a round earlier) are pulled into L2 -- no registers, no
// read of the values, so no update sees an older coordinate than without.
template <typename T, int kMinBlocks, int kDepth, bool kPrefetch = false>
__global__ void __launch_bounds__(256, kMinBlocks) k_sgd_hogwild(DevGraph g, void* __restrict__ coords, DevRng rng,
                                                     DevStats* stats, IterArgs a) {
    static_assert(kDepth >= 2 && kDepth <= 4, "pipeline depth");
    const uint64_t tid = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    const uint32_t warp = static_cast<uint32_t>(tid >> 5);
    const uint32_t lane = threadIdx.x & 31;
    if (warp >= a.n_warps) return;  // whole warps only: the grid is warp-exact

    Xo r{rng.s0[tid], rng.s1[tid], rng.s2[tid], rng.s3[tid]};
    const uint64_t share = a.steps / a.n_warps;
    const uint64_t count = share + (warp < a.steps % a.n_warps ? 1 : 0);
    const uint64_t pol_keep = policy_evict_last();
    const uint64_t pol_stream = policy_evict_first();

    uint32_t applied = 0, b_first = 0, b_first_cool = 0, b_second = 0, primary = 0, skipped = 0;
    bool carry = false;
    uint32_t bpos = 0;
    // Software pipeline over rounds: the step records of the next kDepth-1
    // rounds are in flight while this round gathers and updates coordinates.
    Sel q[kDepth - 1];
#pragma unroll
    for (int d = 0; d < kDepth - 1; ++d) {
        q[d].flags = 0;
        if (static_cast<uint64_t>(d) * 32 < count)
            q[d] = stage_select<true>(g, r, a, static_cast<uint64_t>(d) * 32, count, lane, carry, b_first,
                                      b_first_cool, b_second, pol_stream, bpos);
    }
    for (uint64_t base = 0; base < count; base += 32) {
        Sel nxt;
        nxt.flags = 0;
        const uint64_t ahead = base + static_cast<uint64_t>(kDepth - 1) * 32;
        if (ahead < count)
            nxt = stage_select<true>(g, r, a, ahead, count, lane, carry, b_first, b_first_cool, b_second,
                                     pol_stream, bpos);
        if constexpr (kPrefetch && kDepth >= 3) {
            if (q[1].flags & 1u) {
                prefetch_l2(Coord<T>::copy_src(coords, q[1].ri.node, (q[1].flags >> 1) & 1));
                prefetch_l2(Coord<T>::copy_src(coords, q[1].rj.node, (q[1].flags >> 2) & 1));
            }
        }
        applied += stage_update<T>(q[0], coords, r, a, pol_keep, primary, skipped);
#pragma unroll
        for (int d = 0; d + 1 < kDepth - 1; ++d) q[d] = q[d + 1];
        q[kDepth - 2] = nxt;
    }

    rng.s0[tid] = r.a;
    rng.s1[tid] = r.b;
    rng.s2[tid] = r.c;
    rng.s3[tid] = r.d;
    flush_stats(stats, 0, primary);
    flush_stats(stats, 1, primary * a.drf);  // attempted: drf per primary step (engine.cpp:126)
    flush_stats(stats, 2, applied);
    flush_stats(stats, 3, skipped);
    flush_stats(stats, 4, b_first);
    flush_stats(stats, 5, b_first_cool);
    flush_stats(stats, 6, b_second);
    flush_stats(stats, 7, b_second);
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

// Kernel variants (pgl_layout_ext.kernel_variant with PGL_SAMPLING_IID; 0 =
// the host's auto choice): 8 = depth 2, 2 blocks/SM (the round-1 kernel);
// 1-5: bit 0 = occupancy target 3 blocks/SM (80 registers, spills) instead
// of 2, variant >> 1 = extra rounds of step records in flight (depth 2, 3
// or 4); 6 / 7 = depth 3 / 4 with the next round's endpoints prefetched
// into L2.
template <typename T>
const void* hogwild_fn(int variant) {
    switch (variant) {
        case 1: return reinterpret_cast<const void*>(k_sgd_hogwild<T, 3, 2>);
        case 2: return reinterpret_cast<const void*>(k_sgd_hogwild<T, 1, 3>);
        case 3: return reinterpret_cast<const void*>(k_sgd_hogwild<T, 3, 3>);
        case 4: return reinterpret_cast<const void*>(k_sgd_hogwild<T, 1, 4>);
        case 5: return reinterpret_cast<const void*>(k_sgd_hogwild<T, 3, 4>);
        case 6: return reinterpret_cast<const void*>(k_sgd_hogwild<T, 1, 3, true>);
        case 7: return reinterpret_cast<const void*>(k_sgd_hogwild<T, 1, 4, true>);
        default: return reinterpret_cast<const void*>(k_sgd_hogwild<T, 1, 2>);
    }
}

const void* hogwild_fn_kind(int coord_kind, int variant) {
    return coord_kind == PGL_COORD_F64   ? hogwild_fn<double>(variant)
           : coord_kind == PGL_COORD_F32 ? hogwild_fn<float>(variant)
                                         : hogwild_fn<AnchF32>(variant);
}

LaunchShape sgd_shape(int device, int coord_kind, uint32_t max_warps, int block_threads, int variant) {
    LaunchShape sh;
    sh.threads = block_threads > 0 ? block_threads : 256;
    sh.variant = variant;
    int sms = 0, occ = 0;
    PGL_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    PGL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &occ, hogwild_fn_kind(coord_kind, variant), sh.threads, 0));
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

void launch_sgd_hogwild(const DevGraph& g, void* coords, int coord_kind, DevRng rng, DevStats* stats,
                        const IterArgs& a, LaunchShape shape, void* stream) {
    auto s = static_cast<cudaStream_t>(stream);
    void* args[] = {const_cast<DevGraph*>(&g), &coords, &rng, &stats, const_cast<IterArgs*>(&a)};
    PGL_CUDA(cudaLaunchKernel(hogwild_fn_kind(coord_kind, shape.variant),
                              dim3(shape.blocks), dim3(shape.threads), args, 0, s));
    PGL_CUDA(cudaGetLastError());
}

// FP64 layout <-> anchored FP32 store (one thread per node); `dst`/`src`
// is the store's base (anch_base): node n at base + 16 n, block b's anchor
// at base - 8 (b + 1)
__global__ void k_f64_to_anch(const double* __restrict__ src, char* __restrict__ dst, uint64_t V) {
    for (uint64_t n = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; n < V;
         n += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const double anchor = src[4 * (n & ~static_cast<uint64_t>(31))];  // the block's first start x
        if ((n & 31) == 0) *(reinterpret_cast<double*>(dst) - 1 - (n >> 5)) = anchor;
        float4 f;
        f.x = static_cast<float>(src[4 * n] - anchor);
        f.y = static_cast<float>(src[4 * n + 1]);
        f.z = static_cast<float>(src[4 * n + 2] - anchor);
        f.w = static_cast<float>(src[4 * n + 3]);
        *reinterpret_cast<float4*>(dst + 16 * n) = f;
    }
}

__global__ void k_anch_to_f64(const char* __restrict__ src, double* __restrict__ dst, uint64_t V) {
    for (uint64_t n = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; n < V;
         n += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const double anchor = *(reinterpret_cast<const double*>(src) - 1 - (n >> 5));
        const float4 f = *reinterpret_cast<const float4*>(src + 16 * n);
        dst[4 * n] = anchor + static_cast<double>(f.x);
        dst[4 * n + 1] = f.y;
        dst[4 * n + 2] = anchor + static_cast<double>(f.z);
        dst[4 * n + 3] = f.w;
    }
}

// Re-anchor between iterations: a block's anchor moves to its first node's
// current start x, so the f32 offsets stay small as the layout drifts from
// the initial one (one warp per block; the anchor update is exact in FP64,
// each offset is rounded once).
__global__ void k_reanchor(char* __restrict__ store, uint64_t V) {
    const uint64_t warp = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nblocks = (V + 31) / 32;
    for (uint64_t b = warp; b < nblocks; b += (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5) {
        double* anc = reinterpret_cast<double*>(store) - 1 - b;
        char* blk = store + b * 512;
        const double a_old = *anc;
        const float dx0 = *reinterpret_cast<const float*>(blk);  // node 0's start x offset
        const double a_new = a_old + static_cast<double>(dx0);
        if (b * 32 + lane < V) {
            float4* f = reinterpret_cast<float4*>(blk + lane * 16);
            float4 v = *f;
            v.x = static_cast<float>(a_old + static_cast<double>(v.x) - a_new);
            v.z = static_cast<float>(a_old + static_cast<double>(v.z) - a_new);
            *f = v;
        }
        __syncwarp();
        if (lane == 0) *anc = a_new;
    }
}

// Id locality of the graph, for the anchored store's auto choice: for each
// block of 32 consecutive node ids, the range of the path positions
// (256-nt units) of the steps that visit its nodes; lanes of a warp that hit
// the same block combine first (__match_any_sync). A block whose nodes lie
// far apart along the paths would hold f32 offsets far from its anchor.
__global__ void k_block_span(const StepRec* __restrict__ step, uint64_t S, unsigned int* __restrict__ lo,
                             unsigned int* __restrict__ hi) {
    for (uint64_t k0 = blockIdx.x * static_cast<uint64_t>(blockDim.x); k0 < S;
         k0 += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t k = k0 + threadIdx.x;
        const bool ok = k < S;
        uint32_t blk = 0xFFFFFFFFu, pos = 0;
        if (ok) {
            const StepRec r = step[k];
            blk = r.node >> 5;
            const uint64_t p = static_cast<uint64_t>(r.ps_lo) | (static_cast<uint64_t>(r.hi & 0xFFFFu) << 32);
            pos = static_cast<uint32_t>(p >> 8);
        }
        const unsigned peers = __match_any_sync(0xFFFFFFFFu, blk);
        const uint32_t mn = __reduce_min_sync(peers, pos), mx = __reduce_max_sync(peers, pos);
        if (ok && (threadIdx.x & 31) == static_cast<unsigned>(__ffs(peers) - 1)) {
            atomicMin(lo + blk, mn);
            atomicMax(hi + blk, mx);
        }
    }
}

__global__ void k_count_wide_blocks(const unsigned int* __restrict__ lo, const unsigned int* __restrict__ hi,
                                    uint64_t n_blocks, uint32_t max_span, unsigned long long* out) {
    uint32_t wide = 0, seen = 0;
    for (uint64_t b = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; b < n_blocks;
         b += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        if (lo[b] <= hi[b]) {
            ++seen;
            wide += hi[b] - lo[b] > max_span;
        }
    }
    const uint32_t w = __reduce_add_sync(0xFFFFFFFFu, wide), s = __reduce_add_sync(0xFFFFFFFFu, seen);
    if ((threadIdx.x & 31) == 0) {
        if (w) atomicAdd(out, static_cast<unsigned long long>(w));
        if (s) atomicAdd(out + 1, static_cast<unsigned long long>(s));
    }
}

void block_span_stats(const StepRec* step, uint64_t S, uint64_t n_nodes, uint32_t max_span_256nt,
                      unsigned long long* out, void* stream) {
    auto s = static_cast<cudaStream_t>(stream);
    const uint64_t nb = (n_nodes + 31) / 32;
    unsigned int* buf = nullptr;
    PGL_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&buf), 2 * std::max<uint64_t>(nb, 1) * sizeof(unsigned int), s));
    PGL_CUDA(cudaMemsetAsync(buf, 0xFF, nb * sizeof(unsigned int), s));
    PGL_CUDA(cudaMemsetAsync(buf + nb, 0, nb * sizeof(unsigned int), s));
    PGL_CUDA(cudaMemsetAsync(out, 0, 2 * sizeof(unsigned long long), s));
    if (S) k_block_span<<<1184, 256, 0, s>>>(step, S, buf, buf + nb);
    k_count_wide_blocks<<<592, 256, 0, s>>>(buf, buf + nb, nb, max_span_256nt, out);
    PGL_CUDA(cudaGetLastError());
    PGL_CUDA(cudaFreeAsync(buf, s));
}

// Layout::all_finite (layout.cpp:9-18) on the device: count the nodes with
// a non-finite coordinate and the smallest such node id (out[0], out[1];
// out[1] starts at ~0).
template <typename T>
__global__ void k_count_nonfinite(const void* __restrict__ coords, uint64_t V, unsigned long long* out) {
    uint32_t bad = 0;
    for (uint64_t n = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; n < V;
         n += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        double sx, sy, ex, ey;
        Coord<T>::get(coords, static_cast<uint32_t>(n), 0, sx, sy);
        Coord<T>::get(coords, static_cast<uint32_t>(n), 1, ex, ey);
        if (!(isfinite(sx) && isfinite(sy) && isfinite(ex) && isfinite(ey))) {
            ++bad;
            atomicMin(out + 1, static_cast<unsigned long long>(n));
        }
    }
    const uint32_t b = __reduce_add_sync(0xFFFFFFFFu, bad);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(out, static_cast<unsigned long long>(b));
}

void launch_count_nonfinite(const void* coords, int coord_kind, uint64_t n_nodes, unsigned long long* out,
                            void* stream) {
    auto s = static_cast<cudaStream_t>(stream);
    PGL_CUDA(cudaMemsetAsync(out, 0, sizeof(unsigned long long), s));
    PGL_CUDA(cudaMemsetAsync(out + 1, 0xFF, sizeof(unsigned long long), s));
    if (coord_kind == PGL_COORD_F64)
        k_count_nonfinite<double><<<592, 256, 0, s>>>(coords, n_nodes, out);
    else if (coord_kind == PGL_COORD_F32)
        k_count_nonfinite<float><<<592, 256, 0, s>>>(coords, n_nodes, out);
    else
        k_count_nonfinite<AnchF32><<<592, 256, 0, s>>>(coords, n_nodes, out);
    PGL_CUDA(cudaGetLastError());
}

void launch_reanchor(void* store, uint64_t n_nodes, void* stream) {
    k_reanchor<<<592, 256, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<char*>(store), n_nodes);
    PGL_CUDA(cudaGetLastError());
}

void launch_f64_to_anch(const double* src, void* dst, uint64_t n_nodes, void* stream) {
    k_f64_to_anch<<<592, 256, 0, static_cast<cudaStream_t>(stream)>>>(src, static_cast<char*>(dst), n_nodes);
    PGL_CUDA(cudaGetLastError());
}

void launch_anch_to_f64(const void* src, double* dst, uint64_t n_nodes, void* stream) {
    k_anch_to_f64<<<592, 256, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<const char*>(src), dst, n_nodes);
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
