// pgl_replay.cu — PGL_MODE_REPLAY: the reference's threads = 1 run on one
// device lane, bit for bit (engine.cpp:103-172 with seed_worker(seed, 0)).
//
// A single lane is latency-bound, so the loop is software-pipelined with an
// exact speculation: the random draws of a step depend only on the RNG
// stream and the graph index, except the jitter draw of a coincident pair
// (engine.cpp:292-296), which depends on coordinates. While step s updates
// coordinates, step s+1 is already planned from the RNG state step s would
// leave without a jitter, and its two step records are in flight. If step s
// does draw a jitter, the plan of s+1 is discarded and redone from the true
// state. Coordinates live in shared memory when 32 B x nodes fits.
// k_sgd_replay_pc (below, the one launched) splits planning and updating
// across two warps instead.
#include <cuda_runtime.h>

#include <mutex>
#include <type_traits>
#include <vector>

#include "pgl_device.cuh"

namespace pgl {

namespace {

struct Plan {
    StepRec ri, rj;
    uint64_t gi, gj;  // global step indices of i and j
    Xo r_mid;      // stream right after the two endpoint coins
    Xo r_end;      // stream after this step's draws, assuming no jitter
    int ei, ej;
    bool valid;
    bool opened;   // this step opened a batch
    bool cooling;  // cooling flag in force for this step
};

// select_step_pair (engine.cpp:52-80), the two coins (:137-138) and the
// coins of the drf extra combinations (:155-161) under a known cooling flag.
// R is Xo, or XoCount when the caller needs the number of draws.
template <typename R>
__device__ __forceinline__ Plan plan_known(const DevGraph& g, const IterArgs& a, R& r, bool cooling,
                                           bool load_records) {
    Plan P;
    P.opened = false;
    P.cooling = cooling;
    P.valid = false;
    P.ei = P.ej = 0;
    P.ri = P.rj = StepRec{0, 0, 0, 0};
    P.gi = P.gj = 0;
    const uint64_t x = r.next();
    const uint64_t pick = __umul64hi(x, g.total_steps);
    const uint32_t p = select_path(g, x, pick);
    const PathConst pc = g.pc[p];
    const int64_t n = static_cast<int64_t>(pc.n);
    if (n >= 2) {
        const int64_t i = static_cast<int64_t>(pick - pc.base);
        int64_t j = i;
        bool ok = true;
        if (cooling) {
            const int64_t k = static_cast<int64_t>(zipf_sample(pc, a.theta, r));
            const int64_t sign = r.coin() ? 1 : -1;
            j = i + sign * k;
            if (j < 0 || j >= n) {
                j = i - sign * k;
                if (j < 0 || j >= n) {
                    j = i + sign * k;
                    j = j < 0 ? 0 : (j > n - 1 ? n - 1 : j);
                }
            }
            ok = j != i;
        } else {
            j = static_cast<int64_t>(r.below(pc.n));
            if (j == i) {
                j = static_cast<int64_t>(r.below(pc.n));
                ok = j != i;
            }
        }
        if (ok) {
            P.valid = true;
            P.gi = pc.base + i;
            P.gj = pc.base + j;
            if (load_records) {
                P.ri = load_step(g.step + P.gi);
                P.rj = load_step(g.step + P.gj);
            }
            P.ei = r.coin() ? 0 : 1;
            P.ej = r.coin() ? 0 : 1;
        }
    }
    if constexpr (std::is_same_v<R, Xo>)
        P.r_mid = r;
    else
        P.r_mid = r.r;
    if (P.valid && a.drf > 1) {
        unsigned used = 1u << ((P.ei ? 2 : 0) | (P.ej ? 1 : 0));
        for (uint32_t extra = 1; extra < a.drf; ++extra) {
            int ea, eb;
            do {
                ea = r.coin() ? 0 : 1;
                eb = r.coin() ? 0 : 1;
            } while (used & (1u << ((ea ? 2 : 0) | (eb ? 1 : 0))));
            used |= 1u << ((ea ? 2 : 0) | (eb ? 1 : 0));
        }
    }
    if constexpr (std::is_same_v<R, Xo>)
        P.r_end = r;
    else
        P.r_end = r.r;
    return P;
}

// Batch decision (engine.cpp:115-124) then plan_known.
__device__ __forceinline__ Plan plan_step(const DevGraph& g, const IterArgs& a, uint64_t s, Xo r, bool& cooling,
                                          bool load_records = true) {
    const bool opened = (s % a.batch) == 0;
    if (opened) cooling = a.force_cooling || r.coin();
    Plan P = plan_known(g, a, r, cooling, load_records);
    P.opened = opened;
    return P;
}

// apply_endpoint_update (engine.cpp:276-306), IEEE FP64 (-fmad=false), on a
// generic pointer (shared or global). Sets `jitter` when it drew one.
__device__ __forceinline__ bool apply_exact(double* c, uint32_t ni, int ei, uint32_t nj, int ej, double d_ref,
                                            double eta, Xo& r, bool& jitter) {
    if (!(d_ref > 0.0)) return false;
    const double w = 1.0 / (d_ref * d_ref);
    double mu = eta * w;
    if (mu > 1.0) mu = 1.0;
    double* pi = c + 4 * static_cast<uint64_t>(ni) + 2 * ei;
    double* pj = c + 4 * static_cast<uint64_t>(nj) + 2 * ej;
    const double vix = pi[0], viy = pi[1], vjx = pj[0], vjy = pj[1];
    const double dx = vix - vjx;
    const double dy = viy - vjy;
    const double mag = sqrt(dx * dx + dy * dy);
    double ux, uy;
    if (mag < 1e-9) {
        const double angle = 2.0 * 3.14159265358979323846 * r.uniform();
        ux = cos(angle);
        uy = sin(angle);
        jitter = true;
    } else {
        ux = dx / mag;
        uy = dy / mag;
    }
    const double delta = mu * (mag - d_ref) / 2.0;
    pi[0] = vix - delta * ux;
    pi[1] = viy - delta * uy;
    pj[0] = vjx + delta * ux;
    pj[1] = vjy + delta * uy;
    return true;
}

// ---- producer / consumer replay ----------------------------------------------
// Two warps, one active lane each. The PRODUCER (warp 0) walks the RNG stream
// and the graph index: batch decision, pick, partner, coins (plan_step), then
// has the TMA engine copy the two step records into a ring slot (bulk copy,
// mbarrier completion). The CONSUMER (warp 1) owns the coordinates: endpoint
// loads, apply_exact, write-back, drf extras, RunStats. Nothing the producer
// computes depends on coordinates except through a jitter draw
// (engine.cpp:292-296); when the consumer draws one, it posts the true
// stream state and the producer restarts planning from the next step under a
// new epoch while the consumer discards the stale slots. The consumer's
// sequence of operations is exactly the reference's, so results stay bit
// for bit; the producer's latency (Zipf transcendentals, index loads, record
// gathers) runs concurrently on the other warp.

constexpr uint32_t kRing = 128;

struct alignas(16) Slot {
    StepRec ri, rj;   // TMA destination (valid steps only)
    Xo r_mid;         // stream after the two endpoint coins
    Xo r_end;         // stream after this step, assuming no jitter
    uint64_t step;
    uint32_t flags;   // bit0 valid, bit1 opened, bit2 cooling, bit3 e_i end, bit4 e_j end
    uint32_t epoch;
};

struct ReplayCtl {
    unsigned long long tail;      // slots consumed (consumer -> producer)
    Xo req_state;                 // restart stream state
    unsigned long long req_step;  // restart step
    uint32_t req_cool;            // batch cooling flag in force after the jittered step
    uint32_t req_epoch;           // restart request epoch (consumer -> producer)
    uint32_t done;                // consumer finished
    uint32_t _pad;
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;"
                 :: "r"(smem_addr(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" :: "r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred P;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P, [%0], %1;\n"
        " @!P bra WAIT_%=;\n}\n" :: "r"(smem_addr(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(b)) : "memory");
}

__global__ void __launch_bounds__(64) k_sgd_replay_pc(DevGraph g, double* __restrict__ gcoords, uint64_t* rng4,
                                                      DevStats* stats, IterArgs a, int use_smem,
                                                      const uint64_t* __restrict__ jumps) {
    extern __shared__ __align__(16) unsigned char smem[];
    Slot* ring = reinterpret_cast<Slot*>(smem);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kRing * sizeof(Slot));
    ReplayCtl* ctl = reinterpret_cast<ReplayCtl*>(smem + kRing * (sizeof(Slot) + 8));
    double* scoords = reinterpret_cast<double*>(smem + kRing * (sizeof(Slot) + 8) + sizeof(ReplayCtl));
    const uint64_t n4 = 4 * g.n_nodes;
    double* coords = gcoords;
    if (use_smem) {
        for (uint64_t k = threadIdx.x; k < n4; k += blockDim.x) scoords[k] = gcoords[k];
        coords = scoords;
    }
    if (threadIdx.x == 0) {
        for (uint32_t k = 0; k < kRing; ++k) mbar_init(bar + k, 1);
        ctl->tail = 0;
        ctl->req_epoch = 0;
        ctl->done = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    volatile ReplayCtl* vc = ctl;

    if (threadIdx.x < 32) {  // ---------------- producer (warp 0) ----------------
        // Speculative lane-parallel planning. A round covers up to 32 steps of
        // one batch (the batch coin, if any, is drawn first). A regular step
        // consumes c = 5 draws when cooling (pick, Zipf accepted at the first
        // try, sign, two coins) or 4 when not (pick, partner, two coins), so
        // lane t plans step s0 + t from the stream jumped ahead by t*c draws
        // (jumps[c - 4][t] = T^(t*c), T = xoshiro's GF(2) transition). Every
        // plan up to and including the first irregular one (a Zipf
        // rejection, a collision redraw, a skipped step) started from the
        // right stream position and is kept; the next round starts after it.
        // drf > 1 (coin pairs until an unused combination) plans one step
        // per round.
        const uint32_t lane = threadIdx.x;
        Xo r{rng4[0], rng4[1], rng4[2], rng4[3]};
        bool cool_state = false;  // engine.cpp:113
        uint32_t epoch = 0;
        uint64_t s0 = 0, q = 0;
        for (;;) {
            const uint32_t req = __shfl_sync(0xFFFFFFFFu, lane == 0 ? vc->req_epoch : 0u, 0);
            if (req != epoch) {  // consumer drew a jitter: replan from its state
                __threadfence_block();
                epoch = req;
                r = Xo{vc->req_state.a, vc->req_state.b, vc->req_state.c, vc->req_state.d};
                s0 = vc->req_step;
                cool_state = vc->req_cool != 0;
            }
            if (s0 >= a.steps) {
                if (__shfl_sync(0xFFFFFFFFu, lane == 0 ? vc->done : 0u, 0)) break;
                continue;
            }
            const unsigned long long tail = __shfl_sync(0xFFFFFFFFull, lane == 0 ? vc->tail : 0ull, 0);
            if (q + 32 - tail > kRing) continue;  // ring full (re-checks the restart request)
            // the round: steps s0 .. s0 + m - 1, one batch
            Xo rb = r;
            bool cool = cool_state;
            const uint64_t in_b = s0 % a.batch;
            const bool opened = in_b == 0;
            if (opened) cool = a.force_cooling || rb.coin();
            uint64_t m = a.batch - in_b;
            if (m > 32) m = 32;
            if (m > a.steps - s0) m = a.steps - s0;
            if (a.drf > 1) m = 1;
            const uint32_t c = cool ? 5u : 4u;
            Plan P{};
            bool regular = true;
            if (lane < m) {
                uint64_t st[4] = {rb.a, rb.b, rb.c, rb.d};
                if (lane) gf2_apply(st, jumps + (static_cast<uint64_t>(c - 4) * 32 + lane) * 256 * 4);
                XoCount rc{Xo{st[0], st[1], st[2], st[3]}, 0};
                P = plan_known(g, a, rc, cool, /*load_records=*/false);
                regular = rc.n == c;
            }
            const unsigned irr = __ballot_sync(0xFFFFFFFFu, lane < m && !regular);
            const uint32_t keep = irr ? static_cast<uint32_t>(__ffs(irr)) : static_cast<uint32_t>(m);  // lanes kept
            if (lane < keep) {
                Slot& sl = ring[(q + lane) % kRing];
                sl.r_mid = P.r_mid;
                sl.r_end = P.r_end;
                sl.step = s0 + lane;
                sl.epoch = epoch;
                sl.flags = (P.valid ? 1u : 0u) | ((opened && lane == 0) ? 2u : 0u) | (cool ? 4u : 0u) |
                           (P.ei ? 8u : 0u) | (P.ej ? 16u : 0u);
                uint64_t* b = bar + ((q + lane) % kRing);
                if (P.valid) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    mbar_arrive_tx(b, 2 * sizeof(StepRec));
                    tma_load(&sl.ri, g.step + P.gi, sizeof(StepRec), b);
                    tma_load(&sl.rj, g.step + P.gj, sizeof(StepRec), b);
                } else {
                    mbar_arrive(b);
                }
            }
            // the stream continues after the last kept plan
            r.a = __shfl_sync(0xFFFFFFFFu, P.r_end.a, keep - 1);
            r.b = __shfl_sync(0xFFFFFFFFu, P.r_end.b, keep - 1);
            r.c = __shfl_sync(0xFFFFFFFFu, P.r_end.c, keep - 1);
            r.d = __shfl_sync(0xFFFFFFFFu, P.r_end.d, keep - 1);
            cool_state = cool;
            s0 += keep;
            q += keep;
        }
    } else if (threadIdx.x == 32) {  // ---------------- consumer ----------------
        unsigned long long applied = 0, bf = 0, bfc = 0, bs = 0;
        uint32_t epoch = 0;
        Xo r{rng4[0], rng4[1], rng4[2], rng4[3]};
        uint64_t q = 0, next_step = 0;
        while (next_step < a.steps) {
            Slot& sl = ring[q % kRing];
            mbar_wait(bar + (q % kRing), static_cast<uint32_t>((q / kRing) & 1));
            const uint32_t fl = sl.flags;
            const bool mine = sl.epoch == epoch && sl.step == next_step;
            if (mine) {
                if (fl & 2u) {
                    if (a.force_cooling)
                        ++bs;
                    else {
                        ++bf;
                        bfc += (fl >> 2) & 1u;
                    }
                }
                Xo live = sl.r_mid;
                bool jitter = false;
                if (fl & 1u) {
                    const StepRec ri = sl.ri, rj = sl.rj;
                    const int ei = (fl >> 3) & 1, ej = (fl >> 4) & 1;
                    applied += apply_exact(coords, ri.node, ei, rj.node, ej,
                                           abs_diff(step_pos(ri, ei), step_pos(rj, ej)), a.eta, live, jitter);
                    if (a.drf > 1) {
                        unsigned used = 1u << ((ei ? 2 : 0) | (ej ? 1 : 0));
                        for (uint32_t extra = 1; extra < a.drf; ++extra) {
                            int ea, eb;
                            do {
                                ea = live.coin() ? 0 : 1;
                                eb = live.coin() ? 0 : 1;
                            } while (used & (1u << ((ea ? 2 : 0) | (eb ? 1 : 0))));
                            used |= 1u << ((ea ? 2 : 0) | (eb ? 1 : 0));
                            applied += apply_exact(coords, ri.node, ea, rj.node, eb,
                                                   abs_diff(step_pos(ri, ea), step_pos(rj, eb)), a.eta, live, jitter);
                        }
                    }
                }
                ++next_step;
                if (jitter) {
                    r = live;
                    if (next_step < a.steps) {  // restart the producer at next_step from the true stream
                        ++epoch;
                        vc->req_state.a = live.a;
                        vc->req_state.b = live.b;
                        vc->req_state.c = live.c;
                        vc->req_state.d = live.d;
                        vc->req_step = next_step;
                        vc->req_cool = (fl >> 2) & 1u;
                        __threadfence_block();
                        vc->req_epoch = epoch;
                    }
                } else {
                    r = sl.r_end;
                }
            }
            ++q;
            __threadfence_block();
            vc->tail = q;
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
        __threadfence_block();
        vc->done = 1;
    }
    __syncthreads();
    if (use_smem)
        for (uint64_t k = threadIdx.x; k < n4; k += blockDim.x) gcoords[k] = scoords[k];
}

constexpr size_t kSmemCap = 220 * 1024;
constexpr size_t kRingBytes = kRing * (sizeof(Slot) + 8) + sizeof(ReplayCtl);

}  // namespace

namespace {

// jumps[c - 4][t] = T^(t * c), c in {4, 5}, t in [0, 32): T = xoshiro256's
// state transition over GF(2)^256 (column-major [256][4] u64 per matrix).
std::vector<uint64_t> replay_jump_tables() {
    auto step = [](uint64_t s[4]) {  // RngState::next's state update (rng.hpp:21-31)
        const uint64_t t = s[1] << 17;
        s[2] ^= s[0];
        s[3] ^= s[1];
        s[1] ^= s[2];
        s[0] ^= s[3];
        s[2] ^= t;
        s[3] = (s[3] << 45) | (s[3] >> 19);
    };
    auto matvec = [](const uint64_t* M, const uint64_t in[4], uint64_t out[4]) {
        out[0] = out[1] = out[2] = out[3] = 0;
        for (int b = 0; b < 256; ++b)
            if ((in[b >> 6] >> (b & 63)) & 1)
                for (int w = 0; w < 4; ++w) out[w] ^= M[b * 4 + w];
    };
    auto mul = [&](const std::vector<uint64_t>& A, const std::vector<uint64_t>& B) {  // A * B
        std::vector<uint64_t> C(256 * 4);
        for (int b = 0; b < 256; ++b) matvec(A.data(), &B[b * 4], &C[b * 4]);
        return C;
    };
    std::vector<uint64_t> T(256 * 4), I(256 * 4, 0);
    for (int b = 0; b < 256; ++b) {
        uint64_t s[4] = {0, 0, 0, 0};
        s[b >> 6] = 1ULL << (b & 63);
        I[b * 4 + (b >> 6)] = 1ULL << (b & 63);
        step(s);
        for (int w = 0; w < 4; ++w) T[b * 4 + w] = s[w];
    }
    std::vector<uint64_t> out;
    for (int c = 4; c <= 5; ++c) {
        std::vector<uint64_t> Tc = I;
        for (int k = 0; k < c; ++k) Tc = mul(T, Tc);
        std::vector<uint64_t> P = I;
        for (int t = 0; t < 32; ++t) {
            out.insert(out.end(), P.begin(), P.end());
            P = mul(Tc, P);
        }
    }
    return out;
}

const uint64_t* device_jump_tables(int device) {
    static std::mutex mu;
    static std::vector<std::pair<int, uint64_t*>> tabs;
    std::lock_guard<std::mutex> lock(mu);
    for (auto& t : tabs)
        if (t.first == device) return t.second;
    static const std::vector<uint64_t> host = replay_jump_tables();
    uint64_t* d = nullptr;
    PGL_CUDA(cudaMalloc(&d, host.size() * sizeof(uint64_t)));
    PGL_CUDA(cudaMemcpy(d, host.data(), host.size() * sizeof(uint64_t), cudaMemcpyHostToDevice));
    tabs.emplace_back(device, d);
    return d;
}

}  // namespace

void launch_sgd_replay(const DevGraph& g, double* coords, uint64_t* rng4, DevStats* stats, const IterArgs& a,
                       void* stream) {
    int dev = 0;
    PGL_CUDA(cudaGetDevice(&dev));
    const uint64_t* jumps = device_jump_tables(dev);
    const size_t cbytes = 32 * g.n_nodes;
    const int use_smem = kRingBytes + cbytes <= kSmemCap ? 1 : 0;
    const size_t bytes = kRingBytes + (use_smem ? cbytes : 0);
    PGL_CUDA(cudaFuncSetAttribute(k_sgd_replay_pc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kSmemCap)));
    k_sgd_replay_pc<<<1, 64, bytes, static_cast<cudaStream_t>(stream)>>>(g, coords, rng4, stats, a, use_smem, jumps);
    PGL_CUDA(cudaGetLastError());
}

}  // namespace pgl
