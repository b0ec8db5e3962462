// pgl_tiles.cu — tile-sampled Hogwild PG-SGD (the default fast path).
//
// Same update as the reference's worker loop (engine.cpp:103-172): per primary
// step a node i, a partner j on i's path (uniform with one redraw, or a
// Zipf-distributed hop under cooling, select_step_pair :52-80), coin-flipped
// endpoints, apply_endpoint_update (:276-306), drf re-updates (:147-170).
//
// What changes is how the primary step i is drawn. The reference draws it
// i.i.d. uniform over all steps (weighted_step_select, graph.hpp:123-138),
// i.e. 10/srf picks per step per iteration on average. Here the iteration's
// N = 10*S/srf picks are enumerated, q in [0, N), with i = q mod S: every step
// is the primary endpoint exactly 10/srf times (sampling without
// replacement; the marginal of each update is unchanged). Picks are grouped
// in units of 32 consecutive q, one unit per warp round:
//   * the 32 step records of a unit are one coalesced 512-byte load (four
//     full lines) instead of 32 random 16-byte gathers, each of which costs a
//     whole 128-byte line on B200 (L2 promotes every random miss);
//   * a partner j that falls inside the unit's 32 steps (most Zipf hops in
//     the cooling phase) is taken from the owning lane with __shfl_sync, so
//     lanes working on the same path share step loads;
//   * the cooling decision of a batch of 32 steps is warp-uniform.
// Warp w takes visit indices k = w, w + W, ...; k maps to a unit either
// (PGL_ORDER_SPREAD) by u = (a*k + b) mod U, gcd(a, U) = 1, fresh (a, b) per
// iteration, so the warps running at any moment are spread over the whole
// graph, or (PGL_ORDER_FRONTS, default) by F contiguous stretches of the unit
// space swept in parallel, ~W/F adjacent units in flight per stretch: the
// Zipf partners (|j - i| <= 1000) of a front fall in its own L2-resident
// trail instead of cold random lines.
#include <cuda_runtime.h>

#include <type_traits>

#include "pgl_device.cuh"

namespace pgl {

namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;

__device__ __forceinline__ void flush_stat(DevStats* st, int idx, uint32_t v) {
    const uint32_t sum = __reduce_add_sync(kFull, v);
    if ((threadIdx.x & 31) == 0 && sum) atomicAdd(&st->v[idx], static_cast<unsigned long long>(sum));
}

// Path of global step index i with its base (cum_steps[p]) and length:
// guide by the step index's high bits, then the guided path's constants in
// one 64-byte line (PathConst); a short forward scan only when the guide's
// bucket straddles a path end. Two dependent loads, not guide -> cum -> pc.
// With want_z (a cooling unit) the path's Zipf support and alias-table
// offset come from the same line in the same round trip.
template <typename UX>
__device__ __forceinline__ uint32_t path_of_step(const DevGraph& g, UX i, bool want_z, UX& base, UX& n,
                                                 uint32_t& zn, uint64_t& zt) {
    uint32_t p = __ldg(g.sguide + (i >> g.sguide_shift));
    const PathConst* c = g.pc + p;
    base = static_cast<UX>(__ldg(&c->base));
    n = static_cast<UX>(__ldg(&c->n));
    if (want_z) {
        zn = static_cast<uint32_t>(__ldg(&c->zn));
        zt = __ldg(&c->ztab);
    }
    while (i - base >= n) {  // i >= base always: the guide never overshoots
        c = g.pc + ++p;
        base = static_cast<UX>(__ldg(&c->base));
        n = static_cast<UX>(__ldg(&c->n));
        if (want_z) {
            zn = static_cast<uint32_t>(__ldg(&c->zn));
            zt = __ldg(&c->ztab);
        }
    }
    return p;
}

// The same by the step guide and a forward scan of cum_steps (the register
// pipeline's choice); the Zipf constants follow the path in a cooling unit.
template <typename UX>
__device__ __forceinline__ uint32_t path_of_step_cum(const DevGraph& g, UX i, bool want_z, UX& base, UX& n,
                                                     uint32_t& zn, uint64_t& zt) {
    uint32_t p = __ldg(g.sguide + (i >> g.sguide_shift));
    while (__ldg(g.cum + p + 1) <= i) ++p;
    base = static_cast<UX>(__ldg(g.cum + p));
    n = static_cast<UX>(__ldg(g.cum + p + 1)) - base;
    if (want_z) {
        zn = static_cast<uint32_t>(__ldg(&g.pc[p].zn));
        zt = __ldg(&g.pc[p].ztab);
    }
    return p;
}

// k32 graphs: one 16-byte guide entry gives the path, its base and length
// and whether its Zipf support is the speculated one (zdef); only a bucket
// that straddles a path end falls back to the PathConst scan.
template <typename UX>
__device__ __forceinline__ uint32_t path_of_step_fat(const DevGraph& g, const IterArgs& a, UX i, bool want_z,
                                                     UX& base, UX& n, uint32_t& zn, uint64_t& zt, bool& zdef) {
    const uint4 e = __ldg(a.fguide + (i >> a.fguide_shift));
    uint32_t p = e.z & 0x3FFFFFFFu;
    if (!(e.z >> 31)) {
        base = static_cast<UX>(e.x);
        n = static_cast<UX>(e.y);
        zdef = (e.z >> 30) & 1u;
        if (want_z) {
            if (zdef) {  // the speculated support: its constants are the kernel's own arguments
                zn = a.zdef_n;
                zt = a.zdef_tab;
            } else {
                zn = static_cast<uint32_t>(__ldg(&g.pc[p].zn));
                zt = __ldg(&g.pc[p].ztab);
            }
        }
        return p;
    }
    const PathConst* c = g.pc + p;
    base = static_cast<UX>(__ldg(&c->base));
    n = static_cast<UX>(__ldg(&c->n));
    while (i - base >= n) {
        c = g.pc + ++p;
        base = static_cast<UX>(__ldg(&c->base));
        n = static_cast<UX>(__ldg(&c->n));
    }
    if (want_z) {
        zn = static_cast<uint32_t>(__ldg(&c->zn));
        zt = __ldg(&c->ztab);
    }
    zdef = zn == a.zdef_n && zt == a.zdef_tab;
    return p;
}

// Stage A product for one lane: its step i (record in flight), its partner j
// (record in flight when outside the unit) and the coins.
struct AsyncRes {  // async pipeline: a resolved update, waiting for its endpoints
    uint32_t ni, nj, flags, _pad;
    double d_ref;
};

// shared memory of the async pipeline with lookahead L, 256-thread blocks;
// the anchored store adds the two endpoints' block anchors per update
__host__ __device__ constexpr size_t async_smem_bytes(int L, bool anchored) {
    return L == 0 ? 0
                  : static_cast<size_t>(8 * 32) *
                        ((2 * L + 1) * (2 * sizeof(StepRec) + sizeof(uint32_t)) +
                         (L + 1) * (2 * sizeof(uint4) + sizeof(AsyncRes) + (anchored ? 2 * sizeof(double) : 0)));
}

struct TileSel {
    StepRec ri, rj;       // rj valid when !(flags & 8)
    uint32_t src;         // lane holding j's record when in-tile
    uint32_t flags;       // bit0 valid, bit1 e_i end, bit2 e_j end, bit3 j in tile, bit4 active primary step,
                          // bit5 cooling
    uint32_t path;        // path of i (warp-shuffle reuse pairs only within a path)
};

// Two pipelines per warp, one unit of 32 picks per round:
//   register (kAsync = false): select(m+1) -- batch coin, path, partner,
//     record loads into registers -- overlapped with update(m) (endpoint
//     loads, arithmetic, write-back);
//   asynchronous (kAsync = true): records and endpoints are copied global ->
//     shared with cp.async (no registers held while in flight), three units in
//     flight: endpoints of m landing, records of m+1 landing, m+2 selected.
template <typename T, int kMinBlocks, int kAsync, bool k32>
__global__ void __launch_bounds__(256, kMinBlocks) k_sgd_tiles(DevGraph g, void* __restrict__ coords, DevRng rng,
                                                                DevStats* stats, IterArgs a) {
    // k32: every step index, unit index and path length fits in 31 bits
    // (S < 2^31): 32-bit index arithmetic, fewer registers and instructions
    using UX = std::conditional_t<k32, uint32_t, uint64_t>;
    using SX = std::conditional_t<k32, int32_t, int64_t>;
    const uint64_t tid = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    const uint32_t warp = static_cast<uint32_t>(tid >> 5);
    const uint32_t lane = threadIdx.x & 31;
    if (warp >= a.n_warps) return;

    // async pipeline on the anchored store: the generator state lives in
    // shared memory after the pipeline's slots -- the register budget binds
    // that kernel (config 3: +1.3%; the FP64 store measured 3% slower)
    extern __shared__ __align__(16) unsigned char dyn_smem[];
    constexpr bool kAnch = std::is_same_v<T, AnchF32>;
    constexpr bool kSmemRng = kAsync != 0 && kAnch;
    using Rng = std::conditional_t<kSmemRng, XoSmem, Xo>;
    Rng r;
    if constexpr (kSmemRng) {
        constexpr size_t kRngOff = async_smem_bytes(kAsync, kAnch);
        uint64_t* col = reinterpret_cast<uint64_t*>(dyn_smem + kRngOff) +
                        (threadIdx.x >> 5) * 128 + lane;
        col[0] = rng.s0[tid];
        col[32] = rng.s1[tid];
        col[64] = rng.s2[tid];
        col[96] = rng.s3[tid];
        r.s = col;
    } else {
        r = Xo{rng.s0[tid], rng.s1[tid], rng.s2[tid], rng.s3[tid]};
    }
    const uint64_t pol_keep = policy_evict_last();
    const uint64_t pol_stream = a.record_hint ? policy_evict_normal() : policy_evict_first();
    const UX S = static_cast<UX>(g.total_steps);
    const UX U = static_cast<UX>(a.units);
    const UX n_mine = warp < U ? static_cast<UX>((U - warp + a.n_warps - 1) / a.n_warps) : 0;  // k = w + m*W < U
    UX u = warp < U ? static_cast<UX>((a.perm_a * static_cast<uint64_t>(warp) + a.perm_b) % a.units) : 0;

    uint32_t applied = 0, b_first = 0, b_first_cool = 0, b_second = 0;
    // RunStats counted where they happen (engine.cpp:125-126, :128-131, :140-143): primary steps
    // that reached the update stage, and skipped updates at each skip
    uint32_t primary = 0, skipped = 0;
    bool carry = false;
    uint32_t b0 = 0;  // this warp's step count mod batch (batch boundaries, engine.cpp:115-124)

    // Stage A: batch decision, i's record (coalesced), partner selection.
    StepRec* async_ri = nullptr;  // kAsync: shared-memory destinations of select's record copies
    StepRec* async_rj = nullptr;
    // Unit coins: every fair bit a lane needs for one unit -- the batch coin
    // (bit 0, batch openers), the group's hop sign (bit 1, hop leaders; a
    // lane's own sign when it draws its own hop), the two endpoint coins
    // (bits 2-3) -- comes from the top 4 bits of one xoshiro256+ output per
    // unit instead of a fresh output per coin (the reference's flip_coin
    // takes one output's top bit, rng.hpp:40): the same i.i.d. fair coins at
    // a third to a quarter of the generator work.
    auto select = [&](UX unit, UX unit_i0) -> TileSel {
        TileSel o;
        o.flags = 0;
        o.src = 0;
        o.path = 0;
        o.ri = o.rj = StepRec{0, 0, 0, 0};
        const uint32_t coins = static_cast<uint32_t>(r.next() >> 60);
        const uint64_t q0 = static_cast<uint64_t>(unit) * 32;
        const bool active = q0 + lane < a.steps;
        // batch boundaries count this warp's own steps (engine.cpp:115-124)
        const uint32_t n_active = static_cast<uint32_t>(a.steps - q0 < 32 ? a.steps - q0 : 32);
        bool cooling;
        if (a.batch == 32 && b0 == 0) {
            // the default batch size: the unit is exactly one batch, opened by lane 0
            bool mine = false;
            if (lane == 0) {
                if (a.force_cooling) {
                    mine = true;
                    ++b_second;
                } else {
                    mine = coins & 1u;
                    ++b_first;
                    b_first_cool += mine;
                }
            }
            cooling = a.force_cooling || __shfl_sync(kFull, mine, 0);
            carry = cooling;
            b0 = n_active == 32 ? 0 : n_active;
        } else {
            uint32_t in_batch = b0 + lane;
            if (a.batch >= 32) {
                if (in_batch >= a.batch) in_batch -= a.batch;
            } else {
                in_batch %= a.batch;
            }
            bool mine = false;
            if (active && in_batch == 0) {
                if (a.force_cooling) {
                    mine = true;
                    ++b_second;
                } else {
                    mine = coins & 1u;
                    ++b_first;
                    b_first_cool += mine;
                }
            }
            const int opener = in_batch <= lane ? static_cast<int>(lane - in_batch) : -1;
            const bool opened = __shfl_sync(kFull, mine, opener < 0 ? 0 : opener);
            cooling = a.force_cooling ? true : (opener >= 0 ? opened : carry);
            carry = __shfl_sync(kFull, cooling, n_active - 1);  // batch still open after this unit
            b0 += n_active;
            if (a.batch >= 32) {  // b0 < batch and n_active <= 32: one subtraction
                if (b0 >= a.batch) b0 -= a.batch;
            } else {
                b0 %= a.batch;
            }
        }

        // every lane loads its record, active or not: an in-tile partner of an
        // active lane may sit in an inactive lane of the last, partial unit
        const UX i0 = unit_i0;                 // first step of the unit, q0 mod S (warp-uniform)
        UX gi = i0 + lane;
        while (gi >= S) gi -= S;               // the unit wraps at the end of a pass (S < 32: repeatedly)
        if (a.visits != nullptr && active) atomicAdd(a.visits + gi, 1u);  // diagnostics only
        o.flags = (active ? 16u : 0u) | (cooling ? 32u : 0u);
        // The group leaders draw before the path lookup (a draw that turns
        // out unused is simply discarded), so that in a cooling unit every
        // lane can start the alias-table read for the most common Zipf
        // support (IterArgs::zdef_*) while its path constants are in flight;
        // the path's own support replaces it when they differ.
        const bool win_lead = lane == 0 && !cooling && a.pair_window != 0;
        const bool hop_lead = (lane & (a.hop_lanes - 1)) == 0 && cooling && a.pair_window == 3;
        const int lead = cooling ? static_cast<int>(lane & ~(a.hop_lanes - 1)) : 0;
        uint64_t draw = (win_lead || hop_lead) ? r.next() : 0;
        draw = __shfl_sync(kFull, draw, lead);
        uint32_t kspec = 0;
        if (cooling && a.pair_window == 3) kspec = static_cast<uint32_t>(zipf_alias(g.zalias + a.zdef_tab, a.zdef_n, draw));
        uint32_t p = 0;
        UX pbase = 0;
        SX n = 0;
        uint32_t zn = 0;
        uint64_t zt = 0;
        bool zdef = false;
        if (active) {
            UX len;
            if constexpr (kAsync == 0) {
                // register pipeline: the plain guide -> cum_steps scan measured
                // fastest (config 5: 36.1 G upd/s vs 28.1 with the inline guide)
                p = path_of_step_cum<UX>(g, gi, cooling, pbase, len, zn, zt);
                zdef = zn == a.zdef_n && zt == a.zdef_tab;
            } else if constexpr (k32) {
                p = path_of_step_fat<UX>(g, a, gi, cooling, pbase, len, zn, zt, zdef);
            } else {
                p = path_of_step<UX>(g, gi, cooling, pbase, len, zn, zt);
                zdef = zn == a.zdef_n && zt == a.zdef_tab;
            }
            n = static_cast<SX>(len);
        }
        // Shared partner draws. Uniform batches (pair_window >= 1): lane 0
        // draws one position w0 on its path; every uniform lane on that path
        // takes j = (w0 + (lane ^ m)) mod n. w0 is uniform on [0, n), so each j
        // is marginally uniform exactly as next_below(|p|) (engine.cpp:70-74).
        // Cooling batches (pair_window 3): the first lane of each group of
        // hop_lanes draws one Zipf hop and one sign for the group's lanes on
        // its path; each lane's (k, sign) is still Zipf x fair coin
        // (select_step_pair, engine.cpp:57-69). Either way the partners are
        // consecutive steps: coalesced record loads and neighbouring
        // coordinates instead of one random line per lane.
        // tag: bits 0-28 path, 29 leader was cooling, 30 draw valid, 31 sign
        uint32_t tag = p;
        if (active && n >= 2 && (win_lead || hop_lead)) {
            tag |= (1u << 30) | (cooling ? (1u << 29) : 0u);
            if (cooling) tag |= ((coins >> 1) & 1u) << 31;
        }
        tag = __shfl_sync(kFull, tag, lead);
        const bool shared = ((tag >> 30) & 1) && ((tag >> 29) & 1) == (cooling ? 1u : 0u) && (tag & 0x1FFFFFFFu) == p;
        // the unit's records (one coalesced 512-byte load), issued after the
        // path lookup so its DRAM latency is waited for only in next round's update
        if constexpr (kAsync)
            cp_async<16>(async_ri + lane, g.step + gi, pol_stream);
        else
            o.ri = load_step_stream(g.step + gi, pol_stream);
        if (!active || n < 2) return o;
        const SX i = static_cast<SX>(gi - pbase);
        SX j;
        if (cooling) {
            const SX k = static_cast<SX>(
                shared ? (zdef ? kspec : zipf_alias(g.zalias + zt, zn, draw))
                       : zipf_alias(g.zalias + zt, zn, r.next()));
            if (!shared || hop_lead) diag_zipf(a, static_cast<uint64_t>(k));  // one count per draw
            const SX sign = (shared ? (tag >> 31) : ((coins >> 1) & 1u)) ? 1 : -1;
            j = i + sign * k;
            if (j < 0 || j >= n) {
                j = i - sign * k;
                if (j < 0 || j >= n) {
                    j = i + sign * k;
                    j = j < 0 ? 0 : (j > n - 1 ? n - 1 : j);
                }
            }
            if (j == i) return o;
        } else {
            if (shared) {
                const UX w0 = static_cast<UX>(__umul64hi(draw, static_cast<uint64_t>(n)));
                UX jj = w0 + (lane ^ static_cast<uint32_t>(draw & 31));
                if (jj >= static_cast<UX>(n)) jj = n >= 32 ? jj - n : jj % n;
                j = static_cast<SX>(jj);
            } else {
                j = static_cast<SX>(r.below(static_cast<uint64_t>(n)));
            }
            if (j == i) {
                j = static_cast<SX>(r.below(static_cast<uint64_t>(n)));
                if (j == i) return o;
            }
        }
        const UX gj = pbase + static_cast<UX>(j);
        // coin true -> start (coin_endpoint, engine.cpp:89-91): flag set = end
        uint32_t fl = 1u | ((coins & 4u) ? 0u : 2u) | ((coins & 8u) ? 0u : 4u);
        if (gj >= i0 && gj - i0 < 32) {
            fl |= 8u;
            o.src = static_cast<uint32_t>(gj - i0);
        } else {
            if constexpr (kAsync)
                cp_async<16>(async_rj + lane, g.step + gj, pol_stream);
            else
                o.rj = load_step_stream(g.step + gj, pol_stream);
        }
        o.flags = fl | 16u | (cooling ? 32u : 0u);
        o.path = p;
        return o;
    };

    // Warp-level data reuse (paper 2409.00876 §7.4, pgl_layout_ext.reuse_shuffle):
    // each extra update of a drf > 1 run pairs this lane's i endpoint with the
    // partner endpoint lane q = lane ^ mask holds (mask drawn per extra, warp
    // wide), reusing q's record and coordinates from registers instead of the
    // reference's re-update of the same pair under other endpoint combinations
    // (engine.cpp:147-170). Pairs stay within a path. Convergent: every lane
    // calls it.
    auto shuffle_reuse = [&](bool ok, uint32_t path, const StepRec& ri, int ei, uint32_t ni, double vix,
                             double viy, uint64_t pos_j, int ej, uint32_t nj, double vjx, double vjy) -> uint32_t {
        uint32_t got = 0;
        const uint64_t pos_i = step_pos(ri, ei);
        for (uint32_t extra = 1; extra < a.drf; ++extra) {
            uint64_t x = lane == 0 ? r.next() : 0;
            x = __shfl_sync(kFull, x, 0);
            const int q = static_cast<int>(lane ^ (1u + static_cast<uint32_t>(__umulhi(static_cast<uint32_t>(x >> 32), 31u))));
            const uint32_t q_ok = __shfl_sync(kFull, ok ? path : 0xFFFFFFFFu, q);
            const uint64_t q_pos = __shfl_sync(kFull, pos_j, q);
            const uint32_t q_nj = __shfl_sync(kFull, nj, q);
            const int q_ej = __shfl_sync(kFull, ej, q);
            const double q_vjx = __shfl_sync(kFull, vjx, q);
            const double q_vjy = __shfl_sync(kFull, vjy, q);
            if (ok && q_ok == path) {
                const double d = abs_diff(pos_i, q_pos);
                if (d > 0.0)
                    got += hog_apply_io_t<T>(coords, ni, ei, q_nj, q_ej, d, a.eta, r, pol_keep, vix, viy, q_vjx,
                                             q_vjy);
            }
        }
        return got;
    };

    // Stage B: share in-tile partner records, then the update(s).
    auto update = [&](TileSel& o) -> uint32_t {
        StepRec sh;
        sh.node = __shfl_sync(kFull, o.ri.node, o.src);
        sh.ps_lo = __shfl_sync(kFull, o.ri.ps_lo, o.src);
        sh.pe_lo = __shfl_sync(kFull, o.ri.pe_lo, o.src);
        sh.hi = __shfl_sync(kFull, o.ri.hi, o.src);
        const bool valid = o.flags & 1u;
        const StepRec rj = (o.flags & 8u) ? sh : o.rj;
        const int ei = (o.flags >> 1) & 1, ej = (o.flags >> 2) & 1;
        const double d_ref = valid ? abs_diff(step_pos(o.ri, ei), step_pos(rj, ej)) : 0.0;
        const bool live = valid && d_ref > 0.0;
        double vix = 0, viy = 0, vjx = 0, vjy = 0;
        uint32_t got = 0;
        if (o.flags & 16u) {
            ++primary;
            skipped += valid ? (live ? 0u : 1u) : a.drf;  // an invalid selection skips all drf updates
            diag_outcome(a, o.flags & 32u, live);
        }
        if (live) {
            CoordHint<T>::get(coords, o.ri.node, ei, pol_keep, vix, viy);
            CoordHint<T>::get(coords, rj.node, ej, pol_keep, vjx, vjy);
            got = hog_apply_io_t<T>(coords, o.ri.node, ei, rj.node, ej, d_ref, a.eta, r, pol_keep, vix, viy, vjx, vjy);
        }
        if (a.drf > 1) {
            if (a.reuse_shuffle) {
                const uint32_t ex = shuffle_reuse(live, o.path, o.ri, ei, o.ri.node, vix, viy, step_pos(rj, ej), ej,
                                                  rj.node, vjx, vjy);
                got += ex;
                if (valid) skipped += a.drf - 1 - ex;
            } else if (valid) {
                unsigned used = 1u << ((ei ? 2 : 0) | (ej ? 1 : 0));
                for (uint32_t extra = 1; extra < a.drf; ++extra) {
                    int ea, eb;
                    do {
                        const uint64_t b2 = r.next();
                        ea = (b2 >> 63) ? 0 : 1;
                        eb = ((b2 >> 62) & 1) ? 0 : 1;
                    } while (used & (1u << ((ea ? 2 : 0) | (eb ? 1 : 0))));
                    used |= 1u << ((ea ? 2 : 0) | (eb ? 1 : 0));
                    const uint32_t ok = hog_update_t<T>(coords, o.ri.node, ea, rj.node, eb,
                                                        abs_diff(step_pos(o.ri, ea), step_pos(rj, eb)), a.eta, r,
                                                        pol_keep);
                    got += ok;
                    skipped += 1u - ok;
                }
            }
        }
        return got;
    };

    // i0 = 32u mod S, kept incrementally in spread order (no 64-bit division
    // per round): u advances by perm_step, or by perm_step - U on a wrap
    UX i0 = static_cast<UX>((static_cast<uint64_t>(u) * 32 + a.q_off) % g.total_steps);
    const UX perm_step = static_cast<UX>(a.perm_step), i0_step = static_cast<UX>(a.i0_step),
             i0_wrap = static_cast<UX>(a.i0_wrap);
    auto advance = [&](UX& uu, UX& ii) {  // no overflow: uu, perm_step < U < 2^31; ii, i0_* < S < 2^31
        uu += perm_step;
        if (uu >= U) {
            uu -= U;
            ii += i0_wrap;
        } else {
            ii += i0_step;
        }
        if (ii >= S) ii -= S;
    };
    if constexpr (kAsync == 0) {
        if (n_mine) {
            TileSel cur = select(u, i0);
            for (UX m = 0; m < n_mine; ++m) {
                TileSel nxt;
                nxt.flags = 0;
                nxt.src = 0;
                if (m + 1 < n_mine) {
                    advance(u, i0);
                    nxt = select(u, i0);
                }
                applied += update(cur);
                cur = nxt;
            }
        }
    } else {
        // Asynchronous pipeline: records and endpoints travel global ->
        // shared by cp.async (no registers held while in flight); the
        // per-unit state between stages lives in shared memory too. With
        // lookahead L = kAsync, round t (= tt - 2L below)
        //   1. waits for the endpoints of unit t and applies its update;
        //   2. waits for the records of unit t+L, resolves its partner (own
        //      copy, or the in-tile owner's slot) and issues its endpoint
        //      copies (group C(t+L));
        //   3. selects unit t+2L and issues its record copies (group R(t+2L)).
        // Every round commits exactly two groups (C, then R, possibly empty),
        // so C(t) has 2L-1 newer groups when step 1 waits and R(t+L) has
        // 2L-2 when step 2 waits.
        constexpr int L = kAsync;
        constexpr int kRS = 2 * L + 1;  // record / selection slots
        constexpr int kCS = L + 1;      // endpoint / resolved slots
        constexpr int kWarps = 8;  // 256-thread blocks
        // dynamic shared memory (async_smem_bytes): [kRS] record pairs and
        // selection flags, [kCS] endpoint pairs and resolved updates
        auto* s_ri = reinterpret_cast<StepRec(*)[kWarps][32]>(dyn_smem);
        auto* s_rj = s_ri + kRS;
        auto* s_vi = reinterpret_cast<uint4(*)[kWarps][32]>(s_rj + kRS);  // raw 16-byte copies (Coord<T>::decode)
        auto* s_vj = s_vi + kCS;
        auto* s_res = reinterpret_cast<AsyncRes(*)[kWarps][32]>(s_vj + kCS);
        auto* s_fl = reinterpret_cast<uint32_t(*)[kWarps][32]>(s_res + kCS);
        // anchored store: block anchors of i and j, copied beside the records
        auto* s_ai = reinterpret_cast<double(*)[kWarps][32]>(s_fl + kRS);
        auto* s_aj = s_ai + kCS;
        const int wib = static_cast<int>(threadIdx.x >> 5);
        // round tt selects unit tt, resolves unit tt - L, applies unit tt - 2L;
        // unit x lives in record slot x % kRS and endpoint slot x % kCS, kept
        // as rotating 32-bit counters (no 64-bit modulo per round)
        const uint32_t N = static_cast<uint32_t>(n_mine);
        auto wrap = [](int v, int m) { return v >= m ? v - m : v; };
        int sel_r = 0;  // tt % kRS
        int tt_c = 0;   // tt % kCS
        for (uint32_t tt = 0; tt < N + 2 * L; ++tt) {
            if (tt >= 2 * L) {  // 1. apply unit tt - 2L
                cp_async_wait<2 * L - 1>();
                const int cs = wrap(tt_c + (kCS - (2 * L) % kCS) % kCS, kCS), rs = wrap(sel_r + 1, kRS);
                const AsyncRes cur = s_res[cs][wib][lane];
                const bool live = (cur.flags & 1u) && cur.d_ref > 0.0;
                if (cur.flags & 16u) {
                    ++primary;
                    skipped += (cur.flags & 1u) ? (live ? 0u : 1u) : a.drf;
                    diag_outcome(a, cur.flags & 32u, live);
                }
                double vix = 0, viy = 0, vjx = 0, vjy = 0;
                if (live) {
                    if constexpr (kAnch) {
                        const double ai = s_ai[cs][wib][lane], aj = s_aj[cs][wib][lane];
                        Coord<T>::decode_anchored((cur.flags >> 1) & 1, s_vi[cs][wib][lane], ai, vix, viy);
                        Coord<T>::decode_anchored((cur.flags >> 2) & 1, s_vj[cs][wib][lane], aj, vjx, vjy);
                        applied += hog_apply_io_t<T, true>(coords, cur.ni, (cur.flags >> 1) & 1, cur.nj,
                                                           (cur.flags >> 2) & 1, cur.d_ref, a.eta, r, pol_keep, vix,
                                                           viy, vjx, vjy, ai, aj);
                    } else {
                        Coord<T>::decode(coords, cur.ni, (cur.flags >> 1) & 1, s_vi[cs][wib][lane], vix, viy);
                        Coord<T>::decode(coords, cur.nj, (cur.flags >> 2) & 1, s_vj[cs][wib][lane], vjx, vjy);
                        applied += hog_apply_io_t<T>(coords, cur.ni, (cur.flags >> 1) & 1, cur.nj,
                                                     (cur.flags >> 2) & 1, cur.d_ref, a.eta, r, pol_keep, vix, viy,
                                                     vjx, vjy);
                    }
                }
                if (a.drf > 1) {
                    const StepRec ri = s_ri[rs][wib][lane];
                    const StepRec rj = (cur.flags & 8u) ? s_ri[rs][wib][(cur.flags >> 8) & 31] : s_rj[rs][wib][lane];
                    const int ei = (cur.flags >> 1) & 1, ej = (cur.flags >> 2) & 1;
                    if (a.reuse_shuffle) {
                        const uint32_t ex = shuffle_reuse(live, cur.flags >> 13, ri, ei, cur.ni, vix, viy,
                                                          step_pos(rj, ej), ej, cur.nj, vjx, vjy);
                        applied += ex;
                        if (cur.flags & 1u) skipped += a.drf - 1 - ex;
                    } else if (cur.flags & 1u) {
                        unsigned used = 1u << ((ei ? 2 : 0) | (ej ? 1 : 0));
                        for (uint32_t extra = 1; extra < a.drf; ++extra) {
                            int ea, eb;
                            do {
                                const uint64_t b2 = r.next();
                                ea = (b2 >> 63) ? 0 : 1;
                                eb = ((b2 >> 62) & 1) ? 0 : 1;
                            } while (used & (1u << ((ea ? 2 : 0) | (eb ? 1 : 0))));
                            used |= 1u << ((ea ? 2 : 0) | (eb ? 1 : 0));
                            const uint32_t ok = hog_update_t<T>(coords, ri.node, ea, rj.node, eb,
                                                                abs_diff(step_pos(ri, ea), step_pos(rj, eb)), a.eta,
                                                                r, pol_keep);
                            applied += ok;
                            skipped += 1u - ok;
                        }
                    }
                }
            }
            if (tt >= L && tt < N + L) {  // 2. resolve unit tt - L, issue its endpoint copies
                cp_async_wait<2 * L - 2>();
                __syncwarp();  // in-tile partners read other lanes' copies
                const int cs = wrap(tt_c + (kCS - L % kCS) % kCS, kCS), rs = wrap(sel_r + L + 1, kRS);
                const uint32_t fs = s_fl[rs][wib][lane];
                AsyncRes res{0, 0, fs & 48u, 0, 0.0};  // bits 4-5: active primary step, cooling
                if (fs & 1u) {
                    const StepRec ri = s_ri[rs][wib][lane];
                    const StepRec rj = (fs & 8u) ? s_ri[rs][wib][(fs >> 8) & 31] : s_rj[rs][wib][lane];
                    const int ei = (fs >> 1) & 1, ej = (fs >> 2) & 1;
                    res.d_ref = abs_diff(step_pos(ri, ei), step_pos(rj, ej));
                    res.ni = ri.node;
                    res.nj = rj.node;
                    res.flags = fs;
                    if (res.d_ref > 0.0) {
                        cp_async<16>(&s_vi[cs][wib][lane], Coord<T>::copy_src(coords, ri.node, ei), pol_keep);
                        cp_async<16>(&s_vj[cs][wib][lane], Coord<T>::copy_src(coords, rj.node, ej), pol_keep);
                        if constexpr (kAnch) {
                            cp_async<8>(&s_ai[cs][wib][lane], anch_anchor_ptr(coords, ri.node), pol_keep);
                            cp_async<8>(&s_aj[cs][wib][lane], anch_anchor_ptr(coords, rj.node), pol_keep);
                        }
                    }
                }
                s_res[cs][wib][lane] = res;
            }
            cp_async_commit();
            if (tt < N) {  // 3. select unit tt, issue its record copies
                if (tt > 0) advance(u, i0);
                const int rs = sel_r;
                async_ri = s_ri[rs][wib];
                async_rj = s_rj[rs][wib];
                const TileSel sel = select(u, i0);
                s_fl[rs][wib][lane] = sel.flags | (sel.src << 8) | (sel.path << 13);  // path < 2^19 (host check)
            }
            cp_async_commit();
            __syncwarp();  // slot reuse: every lane is done with this round's shared data
            sel_r = wrap(sel_r + 1, kRS);
            tt_c = wrap(tt_c + 1, kCS);
        }
    }

    if constexpr (kSmemRng) {
        rng.s0[tid] = r.s[0];
        rng.s1[tid] = r.s[32];
        rng.s2[tid] = r.s[64];
        rng.s3[tid] = r.s[96];
    } else {
        rng.s0[tid] = r.a;
        rng.s1[tid] = r.b;
        rng.s2[tid] = r.c;
        rng.s3[tid] = r.d;
    }
    flush_stat(stats, 0, primary);
    flush_stat(stats, 1, primary * a.drf);  // attempted: drf per primary step (engine.cpp:126)
    flush_stat(stats, 2, applied);
    flush_stat(stats, 3, skipped);
    flush_stat(stats, 4, b_first);
    flush_stat(stats, 5, b_first_cool);
    flush_stat(stats, 6, b_second);
    flush_stat(stats, 7, b_second);
}

// ---- lean tile kernel (variant 7) -----------------------------------------------
//
// The asynchronous pipeline of k_sgd_tiles specialised to the configuration
// every benchmark and LayoutConfig{} run uses: batch_size 32 (a unit is one
// batch, opened by lane 0), drf 1 (no re-update combos, no warp-shuffle
// reuse), no sampler diagnostics, S < 2^30 steps and every path shorter than
// 2^32 nt (32-bit positions: d_ref is one 32-bit difference). Same sampler,
// same update; what goes is the generality the default run never takes:
//   * the permutation runs over the full units; the partial last unit is the
//     last unit of its warp (IterArgs::units_full / tail_*), so no warp ever
//     carries a batch across units -- no per-unit batch bookkeeping;
//   * a group leader's shared draw (window start or Zipf hop) comes from the
//     low 60 bits of the same generator output whose top 4 bits are its
//     coins, instead of a second output;
//   * the records are needed only until the partner is resolved: 2 record
//     slots instead of 3, and the resolved update is 16 bytes (32-bit d_ref);
//     with 64 registers and 56 KB of shared memory per 256-thread CTA, four
//     CTAs fit an SM (variant 8) instead of three.
#ifndef PGL_LEAN_SYNC_PREFETCH
#define PGL_LEAN_SYNC_PREFETCH 0  // 1: variants 9/10 prefetch the endpoints into L2 a round ahead (C3: 56.3 vs 58.1 G upd/s without)
#endif
#ifndef PGL_LEAN_BULK
#define PGL_LEAN_BULK 0  // 1: unit records staged by one cp.async.bulk (TMA) per warp round (C3: 49.9 vs 52.9 G upd/s with lane cp.async)
#endif
#ifndef PGL_LEAN_SMEM_RNG
#define PGL_LEAN_SMEM_RNG 0  // 1: anchored lean kernel keeps its generator state in shared memory (C3: 51.6 vs 53.6 G upd/s in registers)
#endif

struct LeanRes {
    uint32_t ni, nj, flags, dref;
};

__host__ __device__ constexpr size_t lean_smem_bytes(bool anchored) {
    // 2 record slots {ri, rj} + 2 endpoint slots {vi, vj, res, anchors}; a
    // unit's selection flags wait in its res slot (free again once the unit
    // two rounds back is applied) -- 224 bytes per lane with the anchored
    // store's generator state, so 4 CTAs fit an SM's 228 KB
    // (anchored: an endpoint is the 8-byte float2 half of its node's record
    // plus the 8-byte block anchor)
    return static_cast<size_t>(8 * 32) *
           (2 * (2 * sizeof(StepRec)) +
            2 * (sizeof(LeanRes) + (anchored ? 2 * (sizeof(float2) + sizeof(double)) : 2 * sizeof(uint4))));
}

// kDiag: the sampler diagnostics (pgl_layout_diag) compiled in -- the same
// kernel for the distribution tests; the production instantiation has none.
// kSync (variant 9): the endpoints are not staged a round ahead; apply reads
// them from L2 and writes them back at once -- a read-to-write window of one
// L2 round trip, as the i.i.d. kernel has (the staged window is a full round).
// kSync 2 (variants 11, 12): the same loads issued at the start of the
// round and consumed after the round's resolve and select, which hide their
// latency (window: one round's integer work, no shared-memory staging).
// kRec8 (variants 13/14, synchronous apply): the records come from the
// 8-byte array DevGraph::rec8 -- a lane copies records k and k+1 of its path
// (offset(k+1) is the far end of step k) into its 16-byte slot, so a unit's
// primary records are 264 contiguous bytes instead of 512.
template <typename T, int kMinBlocks, bool kDiag, int kSync = 0, bool kRec8 = false>
__global__ void __launch_bounds__(256, kMinBlocks) k_sgd_lean(DevGraph g, void* __restrict__ coords, DevRng rng,
                                                               DevStats* stats, IterArgs a) {
    const uint32_t tid = blockIdx.x * 256u + threadIdx.x;
    const uint32_t warp = tid >> 5, lane = threadIdx.x & 31;
    if (warp >= a.n_warps) return;
    constexpr bool kAnch = std::is_same_v<T, AnchF32>;
    extern __shared__ __align__(16) unsigned char dyn_smem[];
    constexpr int kW = 8;  // warps per 256-thread block
    auto* s_ri = reinterpret_cast<StepRec(*)[kW][32]>(dyn_smem);  // [2]
    auto* s_rj = s_ri + 2;
    auto* s_res = reinterpret_cast<LeanRes(*)[kW][32]>(s_rj + 2);  // [2]
    // endpoints [2]: FP64 / f32 the copied 16-byte record; anchored the
    // float2 half (start or end) of the node's record and its block anchor
    auto* s_vi = reinterpret_cast<uint4(*)[kW][32]>(s_res + 2);
    auto* s_vj = s_vi + 2;
    auto* s_ai = reinterpret_cast<double(*)[kW][32]>(s_res + 2);
    auto* s_aj = s_ai + 2;
    auto* s_hi = reinterpret_cast<float2(*)[kW][32]>(s_aj + 2);
    auto* s_hj = s_hi + 2;
    const int wib = static_cast<int>(threadIdx.x >> 5);

    constexpr bool kSmemRng = kAnch && PGL_LEAN_SMEM_RNG;
    using Rng = std::conditional_t<kSmemRng, XoSmem, Xo>;
    Rng r;
    if constexpr (kSmemRng) {  // the register budget binds the anchored kernel
        uint64_t* col = reinterpret_cast<uint64_t*>(dyn_smem + lean_smem_bytes(true)) + wib * 128 + lane;
        col[0] = rng.s0[tid];
        col[32] = rng.s1[tid];
        col[64] = rng.s2[tid];
        col[96] = rng.s3[tid];
        r.s = col;
    } else {
        r = Xo{rng.s0[tid], rng.s1[tid], rng.s2[tid], rng.s3[tid]};
    }
    const uint64_t pol_keep = policy_evict_last();
    const uint64_t pol_stream = policy_evict_first();
    const uint32_t S = static_cast<uint32_t>(g.total_steps);
    const uint32_t Uf = static_cast<uint32_t>(a.units_full);
    // one mbarrier per record slot of this warp: a full unit's 32 records
    // (512 contiguous bytes) arrive by one bulk copy through the TMA engine
    // instead of 32 lane copies through the LSU pipe (PGL_LEAN_BULK)
    uint64_t* bars = reinterpret_cast<uint64_t*>(dyn_smem + lean_smem_bytes(kAnch) +
                                                 (kSmemRng ? kW * 32 * 4 * sizeof(uint64_t) : 0)) + wib * 2;
    if constexpr (PGL_LEAN_BULK) {
        if (lane == 0) {
            mbar_init(bars, 1);
            mbar_init(bars + 1, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
    }
    const uint32_t U = Uf + (a.tail_n ? 1u : 0u);
    const uint32_t W = a.n_warps;
    const uint32_t N = warp < U ? (U - warp + W - 1) / W : 0;  // units k = warp + m*W < U
    const uint32_t hl = a.hop_lanes;
    const uint32_t ul = a.unit_len;              // lanes per unit: 32, or 1..16 with PGL_ORDER_RANDOM
    const uint32_t gbase = lane & ~(ul - 1);     // first lane of this lane's unit
    const bool pw_shared = a.pair_window == 3;   // shared window / Zipf hop draws (else independent partners)

    uint32_t k = warp;
    uint32_t u = k < Uf ? static_cast<uint32_t>((a.perm_a * static_cast<uint64_t>(k) + a.perm_b) % Uf) : Uf;
    uint32_t i0 = k < Uf ? static_cast<uint32_t>((static_cast<uint64_t>(u) * 32 + a.q_off) % S)
                         : static_cast<uint32_t>(a.tail_i0);
    const uint32_t perm_step = static_cast<uint32_t>(a.perm_step), i0_step = static_cast<uint32_t>(a.i0_step),
                   i0_wrap = static_cast<uint32_t>(a.i0_wrap);

    uint32_t applied = 0, primary = 0, skipped = 0, b_first = 0, b_first_cool = 0, b_second = 0;

    // Stage A: the unit's batch coin, i's record (coalesced), the partner.
    auto select = [&](StepRec* dst_i, StepRec* dst_j) -> uint32_t {
        const uint64_t out = r.next();
        const uint32_t coins = static_cast<uint32_t>(out >> 60);
        const bool active = u < Uf || lane < a.tail_n;
        bool cooling;
        if (a.force_cooling) {
            b_second += lane == 0;
            cooling = true;
        } else {
            b_first += lane == 0;
            cooling = __shfl_sync(kFull, coins & 1u, 0);
            b_first_cool += lane == 0 && cooling;
        }
        uint32_t gi = i0 + (lane - gbase);
        if (gi >= S) gi -= S;  // S >= 32 (host check)
        if constexpr (kDiag)
            if (a.visits != nullptr && active) atomicAdd(a.visits + gi, 1u);
        uint32_t fl = active ? 16u : 0u;
        fl |= cooling ? 32u : 0u;
        // leaders: lane 0 of a uniform unit (window start), the first lane of
        // each hop group of a cooling unit (hop, sign = its coin bit 1); the
        // draw is the low 60 bits of the coins' output
        const bool lead = cooling ? (lane & (hl - 1)) == 0 : lane == 0;
        const int lsrc = cooling ? static_cast<int>(lane & ~(hl - 1)) : 0;
        uint64_t draw = 0;
        uint32_t kspec = 0;
        if (pw_shared) {
            draw = __shfl_sync(kFull, out << 4, lsrc);
            if (cooling) kspec = static_cast<uint32_t>(zipf_alias(g.zalias + a.zdef_tab, a.zdef_n, draw));
        }
        uint32_t p = 0, pbase = 0, n = 0, zn = 0;
        uint64_t zt = 0;
        bool zdef = false;
        // (kRec8: inactive lanes of the partial unit too -- their slot must
        // hold their own step's records for in-unit partners)
        if (active || kRec8) p = path_of_step_fat<uint32_t>(g, a, gi, cooling, pbase, n, zn, zt, zdef);
        bool shared = false;
        uint32_t tag = 0;
        if (pw_shared) {  // tag: bits 0-28 path, 30 draw valid, 31 hop sign
            tag = p;
            if (lead && active && n >= 2) tag |= (1u << 30) | (((coins >> 1) & 1u) << 31);
            tag = __shfl_sync(kFull, tag, lsrc);
            shared = ((tag >> 30) & 1u) && (tag & 0x1FFFFFFFu) == p;
        }
        if constexpr (PGL_LEAN_BULK) {
            // a full unit that does not wrap past S and starts the warp's
            // lanes together: one 512-byte bulk copy; otherwise lane copies
            // and a plain arrival so the slot's phase completes either way
            uint64_t* bar = bars + (dst_i == s_ri[0][wib] ? 0 : 1);
            if (ul == 32 && u < Uf && i0 <= S - 32) {
                if (lane == 0) {
                    fence_proxy_async_smem();  // the slot's previous reads (generic proxy) come first
                    mbar_arrive_tx(bar, 32 * sizeof(StepRec));
                    tma_load_hint(dst_i, g.step + i0, 32 * sizeof(StepRec), bar, pol_stream);
                }
            } else {
                cp_async<16>(dst_i + lane, g.step + gi, pol_stream);
                if (lane == 0) mbar_arrive(bar);
            }
        } else if constexpr (kRec8) {
            const uint2* src = g.rec8 + gi + p;
            cp_async<8>(reinterpret_cast<char*>(dst_i + lane), src, pol_stream);
            cp_async<8>(reinterpret_cast<char*>(dst_i + lane) + 8, src + 1, pol_stream);
        } else {
            cp_async<16>(dst_i + lane, g.step + gi, pol_stream);
        }
        if (!active || n < 2) return fl;
        const int32_t i = static_cast<int32_t>(gi - pbase), nn = static_cast<int32_t>(n);
        int32_t j;
        if (cooling) {
            const int32_t kk = static_cast<int32_t>(shared ? (zdef ? kspec : zipf_alias(g.zalias + zt, zn, draw))
                                                           : zipf_alias(g.zalias + zt, zn, r.next()));
            if constexpr (kDiag)
                if (!shared || lead) diag_zipf(a, static_cast<uint64_t>(kk));  // one count per draw
            const int32_t sign = (shared ? (tag >> 31) : ((coins >> 1) & 1u)) ? 1 : -1;
            j = i + sign * kk;
            if (j < 0 || j >= nn) {
                j = i - sign * kk;
                if (j < 0 || j >= nn) {
                    j = i + sign * kk;
                    j = j < 0 ? 0 : (j > nn - 1 ? nn - 1 : j);
                }
            }
            if (j == i) return fl;
        } else {
            if (shared) {
                const uint32_t w0 = static_cast<uint32_t>(__umul64hi(draw, n));
                uint32_t jj = w0 + (lane ^ static_cast<uint32_t>((draw >> 4) & 31));
                if (jj >= n) jj = n >= 32 ? jj - n : jj % n;
                j = static_cast<int32_t>(jj);
            } else {
                j = static_cast<int32_t>(r.below(n));
            }
            if (j == i) {
                j = static_cast<int32_t>(r.below(n));
                if (j == i) return fl;
            }
        }
        const uint32_t gj = pbase + static_cast<uint32_t>(j);
        fl |= 1u | ((coins & 4u) ? 0u : 2u) | ((coins & 8u) ? 0u : 4u);
        if (gj - i0 < ul) {  // in-unit (unsigned: gj >= i0); a wrapped unit's low part copies its own
            fl |= 8u | ((gbase + gj - i0) << 8);
        } else if constexpr (kRec8) {
            const uint2* src = g.rec8 + gj + p;
            cp_async<8>(reinterpret_cast<char*>(dst_j + lane), src, pol_stream);
            cp_async<8>(reinterpret_cast<char*>(dst_j + lane) + 8, src + 1, pol_stream);
        } else {
            cp_async<16>(dst_j + lane, g.step + gj, pol_stream);
        }
        return fl;
    };

    // Round t: apply unit t-2, resolve unit t-1, select unit t. Each round
    // commits two groups (endpoint copies of t-1, then record copies of t):
    // apply(t-2) waits for all but the newest group, resolve(t-1) for all.
    // one round as a lambda over a compile-time slot (t & 1), the loop
    // unrolled by two: the slot offsets fold into the addresses
    auto round = [&](uint32_t t, auto slot) {
        constexpr int cur = decltype(slot)::value, prv = cur ^ 1;
        // kSync 2: unit t-2's endpoint loads go out first, its update comes last
        [[maybe_unused]] LeanRes early{0, 0, 0, 0};
        [[maybe_unused]] double evix = 0, eviy = 0, evjx = 0, evjy = 0;
        if (kSync == 2 && t >= 2) {
            early = s_res[cur][wib][lane];
            const bool live = (early.flags & 1u) && early.dref != 0;
            primary += (early.flags >> 4) & 1u;
            skipped += ((early.flags & 16u) && !live) ? 1u : 0u;
            if constexpr (kDiag)
                if (early.flags & 16u) diag_outcome(a, early.flags & 32u, live);
            if (live) {
                CoordHint<T>::get(coords, early.ni, (early.flags >> 1) & 1, pol_keep, evix, eviy);
                CoordHint<T>::get(coords, early.nj, (early.flags >> 2) & 1, pol_keep, evjx, evjy);
            } else {
                early.flags = 0;
            }
        }
        if (kSync != 2 && t >= 2) {  // 1. apply unit t-2 (endpoint slot (t-2)&1 = cur)
            cp_async_wait<1>();
            const LeanRes res = s_res[cur][wib][lane];
            const bool live = (res.flags & 1u) && res.dref != 0;
            primary += (res.flags >> 4) & 1u;
            skipped += ((res.flags & 16u) && !live) ? 1u : 0u;
            if constexpr (kDiag)
                if (res.flags & 16u) diag_outcome(a, res.flags & 32u, live);
            if (live) {
                const int ei = (res.flags >> 1) & 1, ej = (res.flags >> 2) & 1;
                double vix, viy, vjx, vjy;
                const double d = static_cast<double>(res.dref);
                if constexpr (kSync == 1) {
                    CoordHint<T>::get(coords, res.ni, ei, pol_keep, vix, viy);
                    CoordHint<T>::get(coords, res.nj, ej, pol_keep, vjx, vjy);
                    applied += hog_apply_io_t<T>(coords, res.ni, ei, res.nj, ej, d, a.eta, r, pol_keep, vix, viy, vjx,
                                                 vjy);
                } else if constexpr (kAnch) {
                    const double ai = s_ai[cur][wib][lane], aj = s_aj[cur][wib][lane];
                    const float2 hi = s_hi[cur][wib][lane], hj = s_hj[cur][wib][lane];
                    vix = ai + static_cast<double>(hi.x);
                    viy = static_cast<double>(hi.y);
                    vjx = aj + static_cast<double>(hj.x);
                    vjy = static_cast<double>(hj.y);
                    applied += hog_apply_io_t<T, true>(coords, res.ni, ei, res.nj, ej, d, a.eta, r, pol_keep, vix, viy,
                                                       vjx, vjy, ai, aj);
                } else {
                    Coord<T>::decode(coords, res.ni, ei, s_vi[cur][wib][lane], vix, viy);
                    Coord<T>::decode(coords, res.nj, ej, s_vj[cur][wib][lane], vjx, vjy);
                    applied += hog_apply_io_t<T>(coords, res.ni, ei, res.nj, ej, d, a.eta, r, pol_keep, vix, viy, vjx,
                                                 vjy);
                }
            }
        }
        if (t >= 1 && t <= N) {  // 2. resolve unit t-1 (record slot prv, endpoint slot prv)
            cp_async_wait<0>();
            if constexpr (PGL_LEAN_BULK) mbar_wait(bars + prv, ((t - 1) >> 1) & 1u);  // unit t-1's records
            __syncwarp();  // in-tile partners read other lanes' copies
            const uint32_t fs = s_res[prv][wib][lane].flags;  // left there by select
            LeanRes res{0, 0, fs & 48u, 0};
            if (fs & 1u) {
                // two 32-bit words of each record (node, the coin's position):
                // 1 shared-memory wavefront each instead of 4 for the record
                const uint32_t* wi = &s_ri[prv][wib][lane].node;
                const uint32_t* wj = (fs & 8u) ? &s_ri[prv][wib][(fs >> 8) & 31].node : &s_rj[prv][wib][lane].node;
                uint32_t ni, nj, pi, pj;
                if constexpr (kRec8) {  // {node | rev << 31, offset(k)}, {next node, offset(k + 1)}
                    ni = wi[0] & 0x7FFFFFFFu;
                    nj = wj[0] & 0x7FFFFFFFu;
                    pi = (((fs >> 1) ^ (wi[0] >> 31)) & 1u) ? wi[3] : wi[1];  // end xor reverse: offset(k + 1)
                    pj = (((fs >> 2) ^ (wj[0] >> 31)) & 1u) ? wj[3] : wj[1];
                } else {
                    ni = wi[0];
                    nj = wj[0];
                    pi = wi[(fs & 2u) ? 2 : 1];  // pe_lo : ps_lo
                    pj = wj[(fs & 4u) ? 2 : 1];
                }
                res = LeanRes{ni, nj, fs, pi > pj ? pi - pj : pj - pi};
                if (kSync == 1 && PGL_LEAN_SYNC_PREFETCH && res.dref) {
                    // synchronous apply next round: pull the endpoints' lines
                    // into L2 now (no registers, no shared-memory write)
                    prefetch_l2(Coord<T>::copy_src(coords, ni, (fs >> 1) & 1));
                    prefetch_l2(Coord<T>::copy_src(coords, nj, (fs >> 2) & 1));
                }
                if (kSync == 0 && res.dref) {
                    if constexpr (kAnch) {
                        cp_async<8>(&s_hi[prv][wib][lane], anch_node(coords, ni) + 8 * ((fs >> 1) & 1), pol_keep);
                        cp_async<8>(&s_hj[prv][wib][lane], anch_node(coords, nj) + 8 * ((fs >> 2) & 1), pol_keep);
                        cp_async<8>(&s_ai[prv][wib][lane], anch_anchor_ptr(coords, ni), pol_keep);
                        cp_async<8>(&s_aj[prv][wib][lane], anch_anchor_ptr(coords, nj), pol_keep);
                    } else {
                        cp_async<16>(&s_vi[prv][wib][lane], Coord<T>::copy_src(coords, ni, (fs >> 1) & 1), pol_keep);
                        cp_async<16>(&s_vj[prv][wib][lane], Coord<T>::copy_src(coords, nj, (fs >> 2) & 1), pol_keep);
                    }
                }
            }
            s_res[prv][wib][lane] = res;
        }
        cp_async_commit();
        if (t < N) {  // 3. select unit t (record slot cur)
            if (t > 0) {
                k += W;
                if (k < Uf) {
                    u += perm_step;
                    if (u >= Uf) {
                        u -= Uf;
                        i0 += i0_wrap;
                    } else {
                        i0 += i0_step;
                    }
                    if (i0 >= S) i0 -= S;
                } else {  // the partial unit: always this warp's last
                    u = Uf;
                    i0 = static_cast<uint32_t>(a.tail_i0);
                }
            }
            if (a.unit_random) {  // PGL_ORDER_RANDOM: i.i.d. unit starts (counter-based, unit-uniform)
                uint64_t z = a.unit_key + (static_cast<uint64_t>(k) * 32 + gbase + 1) * kPhi;
                z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
                z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
                i0 = static_cast<uint32_t>(__umul64hi(z ^ (z >> 31), S));
            }
            s_res[cur][wib][lane].flags = select(s_ri[cur][wib], s_rj[cur][wib]);  // slot free: unit t-2 applied
        }
        if (kSync == 2 && (early.flags & 1u)) {  // unit t-2's update, its endpoints loaded at the round's start
            applied += hog_apply_io_t<T>(coords, early.ni, (early.flags >> 1) & 1, early.nj, (early.flags >> 2) & 1,
                                         static_cast<double>(early.dref), a.eta, r, pol_keep, evix, eviy, evjx, evjy);
        }
        cp_async_commit();
        __syncwarp();
    };
    uint32_t t = 0;
    for (; t + 1 < N + 2; t += 2) {
        round(t, std::integral_constant<int, 0>{});
        round(t + 1, std::integral_constant<int, 1>{});
    }
    if (t < N + 2) round(t, std::integral_constant<int, 0>{});

    if constexpr (kSmemRng) {
        rng.s0[tid] = r.s[0];
        rng.s1[tid] = r.s[32];
        rng.s2[tid] = r.s[64];
        rng.s3[tid] = r.s[96];
    } else {
        rng.s0[tid] = r.a;
        rng.s1[tid] = r.b;
        rng.s2[tid] = r.c;
        rng.s3[tid] = r.d;
    }
    flush_stat(stats, 0, primary);
    flush_stat(stats, 1, primary);  // attempted = primary (drf 1)
    flush_stat(stats, 2, applied);
    flush_stat(stats, 3, skipped);
    flush_stat(stats, 4, b_first);
    flush_stat(stats, 5, b_first_cool);
    flush_stat(stats, 6, b_second);
    flush_stat(stats, 7, b_second);
}

// Tile-kernel variants (pgl_layout_ext.kernel_variant; 0 = auto, chosen by
// the host):
//   1  register pipeline, 2 CTAs/SM (no spills); auto where the concurrency
//      cap binds (small graphs: the shortest read-to-write window)
//   2  register pipeline, 3 CTAs/SM (80 registers)
//   5  asynchronous pipeline, 4 CTAs/SM (64 registers)
//   6  asynchronous pipeline, 3 CTAs/SM; auto once the graph fills the GPU
//      (config 2: 43 G upd/s vs 39 for variant 1)
// (A lookahead of two units per stage -- five units in flight per warp, 88 KB
// of shared memory per CTA, 2 CTAs/SM -- measured 20% slower than variant 6.)
// (3 and 4 were a three-stage register pipeline and a bulk-L2-prefetch
// four-stage pipeline; measured no better, removed.) Bit 4 forces the
// 64-bit index instantiation (measurements).
template <typename T, bool k32>
const void* tiles_fn_t(int variant) {
    if constexpr (k32) {
        if (variant == 7) return reinterpret_cast<const void*>(k_sgd_lean<T, 3, false>);
        if (variant == 8) return reinterpret_cast<const void*>(k_sgd_lean<T, 4, false>);
        if (variant == 7 + 32) return reinterpret_cast<const void*>(k_sgd_lean<T, 3, true>);
        if (variant == 8 + 32) return reinterpret_cast<const void*>(k_sgd_lean<T, 4, true>);
        if (variant == 9) return reinterpret_cast<const void*>(k_sgd_lean<T, 3, false, 1>);
        if (variant == 9 + 32) return reinterpret_cast<const void*>(k_sgd_lean<T, 3, true, 1>);
        if (variant == 10) return reinterpret_cast<const void*>(k_sgd_lean<T, 4, false, 1>);
        if (variant == 10 + 32) return reinterpret_cast<const void*>(k_sgd_lean<T, 4, true, 1>);
        if (variant == 11) return reinterpret_cast<const void*>(k_sgd_lean<T, 3, false, 2>);
        if (variant == 11 + 32) return reinterpret_cast<const void*>(k_sgd_lean<T, 3, true, 2>);
        if (variant == 12) return reinterpret_cast<const void*>(k_sgd_lean<T, 4, false, 2>);
        if (variant == 12 + 32) return reinterpret_cast<const void*>(k_sgd_lean<T, 4, true, 2>);
        if (variant == 13) return reinterpret_cast<const void*>(k_sgd_lean<T, 4, false, 1, true>);
        if (variant == 13 + 32) return reinterpret_cast<const void*>(k_sgd_lean<T, 4, true, 1, true>);
        if (variant == 14) return reinterpret_cast<const void*>(k_sgd_lean<T, 3, false, 1, true>);
        if (variant == 14 + 32) return reinterpret_cast<const void*>(k_sgd_lean<T, 3, true, 1, true>);
    }
    return variant == 2   ? reinterpret_cast<const void*>(k_sgd_tiles<T, 3, 0, k32>)
           : variant == 5 ? reinterpret_cast<const void*>(k_sgd_tiles<T, 4, 1, k32>)
           : variant == 6 ? reinterpret_cast<const void*>(k_sgd_tiles<T, 3, 1, k32>)
                          : reinterpret_cast<const void*>(k_sgd_tiles<T, 1, 0, k32>);
}

template <typename T>
const void* tiles_fn(int variant, bool k32) {
    return k32 ? tiles_fn_t<T, true>(variant) : tiles_fn_t<T, false>(variant);
}

size_t tiles_smem(int variant, int coord_kind) {
    variant &= 15;
    const bool async = variant == 5 || variant == 6, anch = coord_kind == PGL_COORD_F32_ANCHORED;
    if (variant >= 7 && variant <= 14)
        return lean_smem_bytes(anch) + (anch && PGL_LEAN_SMEM_RNG ? 256 * 4 * sizeof(uint64_t) : 0) +
               (PGL_LEAN_BULK ? 8 * 2 * sizeof(uint64_t) : 0);
    // anchored: + the generator state (4 u64 per thread) after the pipeline's slots
    return async ? async_smem_bytes(1, anch) + (anch ? 256 * 4 * sizeof(uint64_t) : 0) : 0;
}

const void* tiles_fn_kind(int coord_kind, int variant, bool k32) {
    return coord_kind == PGL_COORD_F64   ? tiles_fn<double>(variant, k32)
           : coord_kind == PGL_COORD_F32 ? tiles_fn<float>(variant, k32)
                                         : tiles_fn<AnchF32>(variant, k32);
}

}  // namespace

LaunchShape tiles_shape(int device, int coord_kind, uint32_t max_warps, int block_threads, int variant,
                        uint64_t total_steps) {
    LaunchShape sh;
    // 32-bit index kernel when every signed step offset i +- k stays below 2^31
    // (variant bit 4 forces the 64-bit instantiation, for measurements)
    sh.idx32 = total_steps < (1ULL << 30) && !(variant & 16);
    variant &= 15 | 32;  // bit 5: the lean kernel with its diagnostics compiled in
    sh.variant = variant;
    sh.smem = tiles_smem(variant, coord_kind);
    // the async pipeline's shared-memory layout assumes 256-thread blocks
    sh.threads = sh.smem ? 256 : (block_threads > 0 ? block_threads : 256);
    const void* fn = tiles_fn_kind(coord_kind, variant, sh.idx32);
    if (sh.smem)
        PGL_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sh.smem)));
    int sms = 0, occ = 0;
    PGL_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    PGL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, sh.threads, sh.smem));
    if (occ < 1) occ = 1;
    uint64_t warps = static_cast<uint64_t>(sms) * occ * (sh.threads / 32);
    if (max_warps && warps > max_warps) warps = max_warps;
    if (warps < 1) warps = 1;
    sh.blocks = static_cast<int>((warps * 32 + sh.threads - 1) / sh.threads);
    return sh;
}

void launch_sgd_tiles(const DevGraph& g, void* coords, int coord_kind, DevRng rng, DevStats* stats,
                      const IterArgs& a, LaunchShape shape, void* stream) {
    void* args[] = {const_cast<DevGraph*>(&g), &coords, &rng, &stats, const_cast<IterArgs*>(&a)};
    PGL_CUDA(cudaLaunchKernel(tiles_fn_kind(coord_kind, shape.variant, shape.idx32),
                              dim3(shape.blocks), dim3(shape.threads), args, shape.smem,
                              static_cast<cudaStream_t>(stream)));
}

}  // namespace pgl
