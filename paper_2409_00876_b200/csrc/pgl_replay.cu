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

// Batch decision (engine.cpp:115-124), select_step_pair (:52-80), the two
// coins (:137-138) and the coins of the drf extra combinations (:155-161).
__device__ __forceinline__ Plan plan_step(const DevGraph& g, const IterArgs& a, uint64_t s, Xo r, bool& cooling,
                                          bool load_records = true) {
    Plan P;
    P.opened = (s % a.batch) == 0;
    if (P.opened) cooling = a.force_cooling || r.coin();
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
    P.r_mid = r;
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
    P.r_end = r;
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

__global__ void __launch_bounds__(64) k_sgd_replay_pc(DevGraph g, double* __restrict__ gcoords, uint64_t* rng4,
                                                      DevStats* stats, IterArgs a, int use_smem) {
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

    if (threadIdx.x == 0) {  // ---------------- producer ----------------
        Xo r{rng4[0], rng4[1], rng4[2], rng4[3]};
        bool cool_state = false;  // engine.cpp:113
        uint32_t epoch = 0;
        uint64_t s = 0, q = 0;
        for (;;) {
            if (vc->req_epoch != epoch) {  // consumer drew a jitter: replan from its state
                __threadfence_block();
                epoch = vc->req_epoch;
                r = Xo{vc->req_state.a, vc->req_state.b, vc->req_state.c, vc->req_state.d};
                s = vc->req_step;
                cool_state = vc->req_cool != 0;
            }
            if (s >= a.steps) {
                if (vc->done) break;
                continue;
            }
            while (q - vc->tail >= kRing) {  // ring full
                if (vc->req_epoch != epoch) break;
            }
            if (q - vc->tail >= kRing) continue;
            const Plan P = plan_step(g, a, s, r, cool_state, /*load_records=*/false);
            Slot& sl = ring[q % kRing];
            sl.r_mid = P.r_mid;
            sl.r_end = P.r_end;
            sl.step = s;
            sl.epoch = epoch;
            sl.flags = (P.valid ? 1u : 0u) | (P.opened ? 2u : 0u) | (P.cooling ? 4u : 0u) | (P.ei ? 8u : 0u) |
                       (P.ej ? 16u : 0u);
            uint64_t* b = bar + (q % kRing);
            if (P.valid) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_arrive_tx(b, 2 * sizeof(StepRec));
                tma_load(&sl.ri, g.step + P.gi, sizeof(StepRec), b);
                tma_load(&sl.rj, g.step + P.gj, sizeof(StepRec), b);
            } else {
                mbar_arrive(b);
            }
            r = P.r_end;
            ++s;
            ++q;
        }
    } else if (threadIdx.x == 32) {  // ---------------- consumer ----------------
        unsigned long long applied = 0, bf = 0, bfc = 0, bs = 0, primary = 0, skipped = 0;
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
                ++primary;
                if (!(fl & 1u)) skipped += a.drf;  // engine.cpp:128-131
                if (fl & 1u) {
                    const StepRec ri = sl.ri, rj = sl.rj;
                    const int ei = (fl >> 3) & 1, ej = (fl >> 4) & 1;
                    const uint32_t ok0 = apply_exact(coords, ri.node, ei, rj.node, ej,
                                                     abs_diff(step_pos(ri, ei), step_pos(rj, ej)), a.eta, live, jitter);
                    applied += ok0;
                    skipped += 1u - ok0;
                    if (a.drf > 1) {
                        unsigned used = 1u << ((ei ? 2 : 0) | (ej ? 1 : 0));
                        for (uint32_t extra = 1; extra < a.drf; ++extra) {
                            int ea, eb;
                            do {
                                ea = live.coin() ? 0 : 1;
                                eb = live.coin() ? 0 : 1;
                            } while (used & (1u << ((ea ? 2 : 0) | (eb ? 1 : 0))));
                            used |= 1u << ((ea ? 2 : 0) | (eb ? 1 : 0));
                            const uint32_t ok = apply_exact(coords, ri.node, ea, rj.node, eb,
                                                            abs_diff(step_pos(ri, ea), step_pos(rj, eb)), a.eta, live,
                                                            jitter);
                            applied += ok;
                            skipped += 1u - ok;
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
        stats->v[0] += primary;
        stats->v[1] += primary * a.drf;
        stats->v[2] += applied;
        stats->v[3] += skipped;
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

void launch_sgd_replay(const DevGraph& g, double* coords, uint64_t* rng4, DevStats* stats, const IterArgs& a,
                       void* stream) {
    const size_t cbytes = 32 * g.n_nodes;
    const int use_smem = kRingBytes + cbytes <= kSmemCap ? 1 : 0;
    const size_t bytes = kRingBytes + (use_smem ? cbytes : 0);
    PGL_CUDA(cudaFuncSetAttribute(k_sgd_replay_pc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kSmemCap)));
    k_sgd_replay_pc<<<1, 64, bytes, static_cast<cudaStream_t>(stream)>>>(g, coords, rng4, stats, a, use_smem);
    PGL_CUDA(cudaGetLastError());
}

}  // namespace pgl
