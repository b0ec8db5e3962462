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
#include <cuda_runtime.h>

#include "pgl_device.cuh"

namespace pgl {

namespace {

struct Plan {
    StepRec ri, rj;
    Xo r_mid;      // stream right after the two endpoint coins
    Xo r_end;      // stream after this step's draws, assuming no jitter
    int ei, ej;
    bool valid;
    bool opened;   // this step opened a batch
    bool cooling;  // cooling flag in force for this step
};

// Batch decision (engine.cpp:115-124), select_step_pair (:52-80), the two
// coins (:137-138) and the coins of the drf extra combinations (:155-161).
__device__ __forceinline__ Plan plan_step(const DevGraph& g, const IterArgs& a, uint64_t s, Xo r, bool& cooling) {
    Plan P;
    P.opened = (s % a.batch) == 0;
    if (P.opened) cooling = a.force_cooling || r.coin();
    P.cooling = cooling;
    P.valid = false;
    P.ei = P.ej = 0;
    P.ri = P.rj = StepRec{0, 0, 0, 0};
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
            P.ri = load_step(g.step + pc.base + i);
            P.rj = load_step(g.step + pc.base + j);
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

__global__ void __launch_bounds__(32) k_sgd_replay2(DevGraph g, double* __restrict__ gcoords, uint64_t* rng4,
                                                    DevStats* stats, IterArgs a, int use_smem) {
    extern __shared__ double smem_coords[];
    const uint64_t n4 = 4 * g.n_nodes;
    double* coords = gcoords;
    if (use_smem) {
        for (uint64_t k = threadIdx.x; k < n4; k += blockDim.x) smem_coords[k] = gcoords[k];
        __syncwarp();
        coords = smem_coords;
    }
    if (threadIdx.x == 0) {
        Xo r{rng4[0], rng4[1], rng4[2], rng4[3]};
        unsigned long long applied = 0, bf = 0, bfc = 0, bs = 0;
        bool cool_state = false;  // planner's batch state (engine.cpp:113)
        Plan cur = plan_step(g, a, 0, r, cool_state);
        for (uint64_t s = 0; s < a.steps; ++s) {
            const bool cool_after_cur = cool_state;
            Plan nxt;
            const bool more = s + 1 < a.steps;
            if (more) nxt = plan_step(g, a, s + 1, cur.r_end, cool_state);  // speculative
            // ---- execute step s (engine.cpp:115-170) ----
            if (cur.opened) {
                if (a.force_cooling)
                    ++bs;
                else {
                    ++bf;
                    bfc += cur.cooling;
                }
            }
            Xo live = cur.r_mid;
            bool jitter = false;
            if (cur.valid) {
                applied += apply_exact(coords, cur.ri.node, cur.ei, cur.rj.node, cur.ej,
                                       abs_diff(step_pos(cur.ri, cur.ei), step_pos(cur.rj, cur.ej)), a.eta, live,
                                       jitter);
                if (a.drf > 1) {
                    unsigned used = 1u << ((cur.ei ? 2 : 0) | (cur.ej ? 1 : 0));
                    for (uint32_t extra = 1; extra < a.drf; ++extra) {
                        int ea, eb;
                        do {
                            ea = live.coin() ? 0 : 1;
                            eb = live.coin() ? 0 : 1;
                        } while (used & (1u << ((ea ? 2 : 0) | (eb ? 1 : 0))));
                        used |= 1u << ((ea ? 2 : 0) | (eb ? 1 : 0));
                        applied += apply_exact(coords, cur.ri.node, ea, cur.rj.node, eb,
                                               abs_diff(step_pos(cur.ri, ea), step_pos(cur.rj, eb)), a.eta, live,
                                               jitter);
                    }
                }
            }
            if (jitter) {  // the speculation of s+1 started from the wrong stream position
                r = live;
                if (more) {
                    cool_state = cool_after_cur;
                    nxt = plan_step(g, a, s + 1, r, cool_state);
                }
            } else {
                r = cur.r_end;
            }
            if (more) cur = nxt;
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
    if (use_smem) {
        __syncwarp();
        for (uint64_t k = threadIdx.x; k < n4; k += blockDim.x) gcoords[k] = smem_coords[k];
    }
}

constexpr size_t kSmemCap = 200 * 1024;

}  // namespace

void launch_sgd_replay(const DevGraph& g, double* coords, uint64_t* rng4, DevStats* stats, const IterArgs& a,
                       void* stream) {
    const size_t bytes = 32 * g.n_nodes;
    const int use_smem = bytes <= kSmemCap ? 1 : 0;
    if (use_smem)
        PGL_CUDA(cudaFuncSetAttribute(k_sgd_replay2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(kSmemCap)));
    k_sgd_replay2<<<1, 32, use_smem ? bytes : 0, static_cast<cudaStream_t>(stream)>>>(g, coords, rng4, stats, a,
                                                                                       use_smem);
    PGL_CUDA(cudaGetLastError());
}

}  // namespace pgl
