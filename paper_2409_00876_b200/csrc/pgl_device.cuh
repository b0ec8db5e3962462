// pgl_device.cuh — device building blocks of the PG-SGD step on sm_100a.
//
// Every function restates one piece of the reference hot loop and keeps its
// exact arithmetic: the translation unit is compiled with -fmad=false so no
// double expression is contracted into an FMA, matching the reference's
// default x86-64 (no-FMA) build bit for bit.
#pragma once

#include <cstdint>

#include "pgl_internal.hpp"

namespace pgl {

constexpr uint64_t kPhi = 0x9E3779B97F4A7C15ULL;

// diagnostics helpers (uniform branch on a kernel argument: free when off)
__device__ __forceinline__ void diag_zipf(const IterArgs& a, uint64_t k) {
    if (a.zhist != nullptr) atomicAdd(a.zhist + (k < a.zhist_len ? k : a.zhist_len - 1), 1ULL);
}
__device__ __forceinline__ void diag_outcome(const IterArgs& a, bool cooling, bool applied) {
    if (a.outcomes != nullptr) {
        atomicAdd(a.outcomes + (cooling ? 2 : 0), 1ULL);
        if (applied) atomicAdd(a.outcomes + (cooling ? 3 : 1), 1ULL);
    }
}

// ---- xoshiro256+ held in registers (rng.hpp:21-47) ------------------------

struct Xo {
    uint64_t a, b, c, d;

    __device__ __forceinline__ uint64_t next() {
        const uint64_t out = a + d;
        const uint64_t t = b << 17;
        c ^= a;
        d ^= b;
        b ^= c;
        a ^= d;
        c ^= t;
        d = (d << 45) | (d >> 19);
        return out;
    }
    // next_uniform: 53 high bits scaled by 2^-53 (rng.hpp:35-37)
    __device__ __forceinline__ double uniform() {
        return static_cast<double>(next() >> 11) * 0x1.0p-53;
    }
    // flip_coin: top bit (rng.hpp:40)
    __device__ __forceinline__ bool coin() { return (next() >> 63) != 0; }
    // next_below: high word of the 128-bit product (rng.hpp:44-47)
    __device__ __forceinline__ uint64_t below(uint64_t n) { return __umul64hi(next(), n); }
};

// The same generator with its state in shared memory (four 32-lane
// columns per warp, one u64 per lane each: conflict-free 8-byte accesses),
// for kernels whose register budget is the binding limit: the state costs
// one 32-bit address instead of eight registers held across the loop.
struct XoSmem {
    uint64_t* s;  // lane's word of column 0; column w at s + 32 * w

    __device__ __forceinline__ uint64_t next() {
        uint64_t a = s[0], b = s[32], c = s[64], d = s[96];
        const uint64_t out = a + d;
        const uint64_t t = b << 17;
        c ^= a;
        d ^= b;
        b ^= c;
        a ^= d;
        c ^= t;
        d = (d << 45) | (d >> 19);
        s[0] = a;
        s[32] = b;
        s[64] = c;
        s[96] = d;
        return out;
    }
    __device__ __forceinline__ double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    __device__ __forceinline__ bool coin() { return (next() >> 63) != 0; }
    __device__ __forceinline__ uint64_t below(uint64_t n) { return __umul64hi(next(), n); }
};

__host__ __device__ __forceinline__ uint64_t splitmix_next(uint64_t& st) {
    uint64_t z = (st += kPhi);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// seed_worker (rng.hpp:63-71): GPU lane t draws the reference worker-t stream.
__host__ __device__ __forceinline__ void seed_worker(uint64_t seed, uint64_t worker, uint64_t s[4]) {
    uint64_t key = seed ^ (kPhi * (worker + 1));
    for (int w = 0; w < 4; ++w) s[w] = splitmix_next(key);
    if ((s[0] | s[1] | s[2] | s[3]) == 0) s[0] = kPhi;
}

// s := M s over GF(2)^256; M column-major, [256][4] u64 (xoshiro's state
// transition is linear, so a power of it jumps the stream ahead).
__device__ __forceinline__ void gf2_apply(uint64_t s[4], const uint64_t* __restrict__ M) {
    uint64_t y0 = 0, y1 = 0, y2 = 0, y3 = 0;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
        uint64_t x = s[w];
        while (x) {
            const int b = __ffsll(static_cast<long long>(x)) - 1;
            x &= x - 1;
            const uint64_t* c = M + (static_cast<uint64_t>(w) * 64 + b) * 4;
            y0 ^= __ldg(c);
            y1 ^= __ldg(c + 1);
            y2 ^= __ldg(c + 2);
            y3 ^= __ldg(c + 3);
        }
    }
    s[0] = y0;
    s[1] = y1;
    s[2] = y2;
    s[3] = y3;
}

// ---- Zipf by rejection inversion (rng.hpp:103-144) ------------------------

__device__ __forceinline__ double zipf_helper1(double x) {
    if (fabs(x) > 1e-8) return log1p(x) / x;
    return 1.0 - x * (0.5 - x * (1.0 / 3.0 - 0.25 * x));
}
__device__ __forceinline__ double zipf_helper2(double x) {
    if (fabs(x) > 1e-8) return expm1(x) / x;
    return 1.0 + x * 0.5 * (1.0 + x * (1.0 / 3.0) * (1.0 + 0.25 * x));
}
__device__ __forceinline__ double zipf_H(double theta, double x) {
    const double lx = log(x);
    return zipf_helper2((1.0 - theta) * lx) * lx;
}
__device__ __forceinline__ double zipf_h(double theta, double x) { return exp(-theta * log(x)); }
__device__ __forceinline__ double zipf_Hinv(double theta, double x) {
    double t = x * (1.0 - theta);
    if (t < -1.0) t = -1.0;
    return exp(zipf_helper1(t) * x);
}

template <typename R>
__device__ __forceinline__ uint64_t zipf_sample(const PathConst& pc, double theta, R& r) {
    if (pc.zn == 1) return 1;
    for (;;) {
        const double u = pc.hxn + r.uniform() * (pc.hx1 - pc.hxn);
        const double x = zipf_Hinv(theta, u);
        uint64_t k = static_cast<uint64_t>(x + 0.5);
        if (k < 1)
            k = 1;
        else if (k > pc.zn)
            k = pc.zn;
        const double kd = static_cast<double>(k);
        if (kd - x <= pc.s || u >= zipf_H(theta, kd + 0.5) - zipf_h(theta, kd)) return k;
    }
}

// ---- graph index reads ------------------------------------------------------

__device__ __forceinline__ StepRec load_step(const StepRec* p) {
    // Read-only, random, no reuse: non-coherent path, skip L1 allocation.
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return StepRec{v.x, v.y, v.z, v.w};
}

// path_position (graph.hpp:98-109): `end` selects Endpoint::end.
__device__ __forceinline__ uint64_t step_pos(const StepRec& r, int end) {
    return end ? (static_cast<uint64_t>(r.pe_lo) | (static_cast<uint64_t>(r.hi >> 16) << 32))
               : (static_cast<uint64_t>(r.ps_lo) | (static_cast<uint64_t>(r.hi & 0xFFFFu) << 32));
}

// weighted_step_select (graph.hpp:123-138): the reference binary-searches
// cum_steps; a guide table indexed by the draw's top bits lands on the
// answer's path or just before it, so the search becomes 1-2 compares.
__device__ __forceinline__ uint32_t select_path(const DevGraph& g, uint64_t x, uint64_t pick) {
    uint32_t p = __ldg(g.guide + (x >> (64 - g.guide_bits)));
    while (__ldg(g.cum + p + 1) <= pick) ++p;
    return p;
}

// ---- coordinate store ---------------------------------------------------------
// F32: one float4 {sx,sy,ex,ey} per node (16 B). F64: two double2 per node
// (32 B, one sector). Hogwild contract (layout.hpp:12-15): an
// endpoint is read and written as one 8/16-byte access (no torn scalar),
// through L2 (.cg) so a lane never re-reads a stale L1 line.

template <typename T> struct Coord;

// Anchored FP32 (PGL_COORD_F32_ANCHORED): nodes in blocks of 32, x kept as
// an f32 offset from the block's f64 anchor (the block's first start x,
// re-anchored between iterations). `base` is the first node's float4
// {sx, sy, ex, ey}; the anchors sit below it in reverse block order
// (pgl_internal.hpp anch_bytes). Half the bytes of FP64 per endpoint, with
// f32 error relative to a node's displacement from its anchor, not to its
// absolute x (which reaches 2e8 at chromosome scale, where plain f32 loses
// local detail).
struct AnchF32 {};
__device__ __forceinline__ const char* anch_node(const void* base, uint32_t node) {
    return reinterpret_cast<const char*>(base) + static_cast<uint64_t>(node) * 16;
}
__device__ __forceinline__ const double* anch_anchor_ptr(const void* base, uint32_t node) {
    return reinterpret_cast<const double*>(base) - 1 - (node >> 5);
}
__device__ __forceinline__ double anch_anchor(const void* base, uint32_t node) {
    // read-only during a layout: the L1 path is safe for the anchor word
    return __ldg(anch_anchor_ptr(base, node));
}

template <> struct Coord<AnchF32> {
    __device__ __forceinline__ static void get(const void* base, uint32_t node, int end, double& x, double& y) {
        const float2 v = __ldcg(reinterpret_cast<const float2*>(anch_node(base, node)) + end);
        x = anch_anchor(base, node) + static_cast<double>(v.x);
        y = static_cast<double>(v.y);
    }
    __device__ __forceinline__ static void set(void* base, uint32_t node, int end, double x, double y) {
        __stcg(const_cast<float2*>(reinterpret_cast<const float2*>(anch_node(base, node))) + end,
               make_float2(static_cast<float>(x - anch_anchor(base, node)), static_cast<float>(y)));
    }
    // the async pipeline copies a node's whole 16-byte record, then decodes
    __device__ __forceinline__ static const void* copy_src(const void* base, uint32_t node, int) {
        return anch_node(base, node);
    }
    __device__ __forceinline__ static void decode(const void* base, uint32_t node, int end, const uint4& raw,
                                                  double& x, double& y) {
        const float4 f = reinterpret_cast<const float4&>(raw);
        x = anch_anchor(base, node) + static_cast<double>(end ? f.z : f.x);
        y = static_cast<double>(end ? f.w : f.y);
    }
    // the same with the block anchor already at hand (the async pipeline
    // copies it to shared memory beside the node record)
    __device__ __forceinline__ static void decode_anchored(int end, const uint4& raw, double anchor, double& x,
                                                           double& y) {
        const float4 f = reinterpret_cast<const float4&>(raw);
        x = anchor + static_cast<double>(end ? f.z : f.x);
        y = static_cast<double>(end ? f.w : f.y);
    }
};

template <> struct Coord<float> {
    __device__ __forceinline__ static void get(const void* base, uint32_t node, int end,
                                               double& x, double& y) {
        const float2 v = __ldcg(reinterpret_cast<const float2*>(base) + 2 * static_cast<uint64_t>(node) + end);
        x = static_cast<double>(v.x);
        y = static_cast<double>(v.y);
    }
    __device__ __forceinline__ static void set(void* base, uint32_t node, int end, double x, double y) {
        __stcg(reinterpret_cast<float2*>(base) + 2 * static_cast<uint64_t>(node) + end,
               make_float2(static_cast<float>(x), static_cast<float>(y)));
    }
    __device__ __forceinline__ static const void* copy_src(const void* base, uint32_t node, int) {
        return reinterpret_cast<const float4*>(base) + node;
    }
    __device__ __forceinline__ static void decode(const void*, uint32_t, int end, const uint4& raw, double& x,
                                                  double& y) {
        const float4 f = reinterpret_cast<const float4&>(raw);
        x = static_cast<double>(end ? f.z : f.x);
        y = static_cast<double>(end ? f.w : f.y);
    }
};

template <> struct Coord<double> {
    __device__ __forceinline__ static void get(const void* base, uint32_t node, int end,
                                               double& x, double& y) {
        const double2 v = __ldcg(reinterpret_cast<const double2*>(base) + 2 * static_cast<uint64_t>(node) + end);
        x = v.x;
        y = v.y;
    }
    __device__ __forceinline__ static void set(void* base, uint32_t node, int end, double x, double y) {
        __stcg(reinterpret_cast<double2*>(base) + 2 * static_cast<uint64_t>(node) + end, make_double2(x, y));
    }
    __device__ __forceinline__ static const void* copy_src(const void* base, uint32_t node, int end) {
        return reinterpret_cast<const double2*>(base) + 2 * static_cast<uint64_t>(node) + end;
    }
    __device__ __forceinline__ static void decode(const void*, uint32_t, int, const uint4& raw, double& x,
                                                  double& y) {
        const double2 d = reinterpret_cast<const double2&>(raw);
        x = d.x;
        y = d.y;
    }
};

__device__ __forceinline__ double abs_diff(uint64_t a, uint64_t b) {
    return static_cast<double>(a > b ? a - b : b - a);
}

// ---- Hogwild fast path helpers -------------------------------------------------
// The Hogwild kernel does not need to reproduce the reference's rounding (its
// races already make it nondeterministic), so it avoids every call into the
// IEEE division/sqrt slow paths: those CALLs force the loop state through the
// stack. Reciprocal and reciprocal square root start from the MUFU 64-bit
// approximations and are refined by Newton steps to ~1 ulp.

#ifndef PGL_HOG_NR
#define PGL_HOG_NR 2  // Newton steps after the MUFU approximation: 2 = ~1 ulp, 1 = ~2^-40 relative
#endif

__device__ __forceinline__ double rcp_nr(double b) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(b));
    double e = fma(-b, y, 1.0);
    y = fma(y, e, y);
    if constexpr (PGL_HOG_NR >= 2) {
        e = fma(-b, y, 1.0);
        y = fma(y, e, y);
    }
    return y;
}

__device__ __forceinline__ double rsqrt_nr(double s) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(s));
    const double h = 0.5 * s;
    y = y * fma(-h * y, y, 1.5);
    y = y * fma(-h * y, y, 1.5);
    if constexpr (PGL_HOG_NR >= 2) y = y * fma(-h * y, y, 1.5);
    return y;
}

__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// Step record gather, streaming: read-only path, no L1 allocation, L2
// evict-first so the one-touch records do not push the coordinates out.
__device__ __forceinline__ StepRec load_step_stream(const StepRec* p, uint64_t pol) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(pol));
    return StepRec{v.x, v.y, v.z, v.w};
}

// Coordinate endpoint access through L2 (.cg) with an evict-last policy: the
// coordinate array is the reused working set (1.7k touches per node per
// iteration at config 2) and should stay L2-resident.
template <typename T> struct CoordHint;

template <> struct CoordHint<float> {
    __device__ __forceinline__ static void get(const void* base, uint32_t node, int end, uint64_t pol,
                                               double& x, double& y) {
        const float2* a = reinterpret_cast<const float2*>(base) + 2 * static_cast<uint64_t>(node) + end;
        float fx, fy;
        asm volatile("ld.global.cg.L2::cache_hint.v2.f32 {%0,%1}, [%2], %3;"
                     : "=f"(fx), "=f"(fy) : "l"(a), "l"(pol));
        x = fx;
        y = fy;
    }
    __device__ __forceinline__ static void set(void* base, uint32_t node, int end, uint64_t pol, double x,
                                               double y) {
        float2* a = reinterpret_cast<float2*>(base) + 2 * static_cast<uint64_t>(node) + end;
        asm volatile("st.global.cg.L2::cache_hint.v2.f32 [%0], {%1,%2}, %3;"
                     :: "l"(a), "f"(static_cast<float>(x)), "f"(static_cast<float>(y)), "l"(pol) : "memory");
    }
};

template <> struct CoordHint<double> {
    __device__ __forceinline__ static void get(const void* base, uint32_t node, int end, uint64_t pol,
                                               double& x, double& y) {
        const double2* a = reinterpret_cast<const double2*>(base) + 2 * static_cast<uint64_t>(node) + end;
        asm volatile("ld.global.cg.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                     : "=d"(x), "=d"(y) : "l"(a), "l"(pol));
    }
    __device__ __forceinline__ static void set(void* base, uint32_t node, int end, uint64_t pol, double x,
                                               double y) {
        double2* a = reinterpret_cast<double2*>(base) + 2 * static_cast<uint64_t>(node) + end;
        asm volatile("st.global.cg.L2::cache_hint.v2.f64 [%0], {%1,%2}, %3;" :: "l"(a), "d"(x), "d"(y), "l"(pol)
                     : "memory");
    }
};

template <> struct CoordHint<AnchF32> {
    __device__ __forceinline__ static void get(const void* base, uint32_t node, int end, uint64_t pol,
                                               double& x, double& y) {
        const float2* a = reinterpret_cast<const float2*>(anch_node(base, node)) + end;
        float fx, fy;
        asm volatile("ld.global.cg.L2::cache_hint.v2.f32 {%0,%1}, [%2], %3;"
                     : "=f"(fx), "=f"(fy) : "l"(a), "l"(pol));
        x = anch_anchor(base, node) + static_cast<double>(fx);
        y = fy;
    }
    __device__ __forceinline__ static void set(void* base, uint32_t node, int end, uint64_t pol, double x,
                                               double y) {
        set_anchored(base, node, end, pol, x, y, anch_anchor(base, node));
    }
    __device__ __forceinline__ static void set_anchored(void* base, uint32_t node, int end, uint64_t pol, double x,
                                                        double y, double anchor) {
        const float2* a = reinterpret_cast<const float2*>(anch_node(base, node)) + end;
        const float fx = static_cast<float>(x - anchor);
        asm volatile("st.global.cg.L2::cache_hint.v2.f32 [%0], {%1,%2}, %3;"
                     :: "l"(a), "f"(fx), "f"(static_cast<float>(y)), "l"(pol) : "memory");
    }
};

// Zipf(zn, theta) on [1, zn] by Walker's alias method: one 64-bit draw, the
// column from its high word, the keep/alias test on its low word. The table
// is built on the host from the exact pmf k^-theta / H(zn, theta), so the
// distribution is the one ZipfSampler (rng.hpp:103-117) samples.
__device__ __forceinline__ uint64_t zipf_alias(const ZipfAlias* tab, uint32_t zn, uint64_t x) {
    const uint32_t col = __umulhi(static_cast<uint32_t>(x >> 32), zn);
    const uint2 e = __ldg(reinterpret_cast<const uint2*>(tab) + col);
    return 1 + (static_cast<uint32_t>(x) < e.x ? col : e.y);
}

// Asynchronous global -> shared copies (LDGSTS), completion tracked per
// thread by commit/wait groups: the loads hold no registers while in flight.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
template <int kBytes>
__device__ __forceinline__ void cp_async(void* smem_dst, const void* gsrc, uint64_t pol) {
    if constexpr (kBytes == 16)
        asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;"
                     :: "r"(smem_u32(smem_dst)), "l"(gsrc), "l"(pol) : "memory");
    else
        asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], %2, %3;"
                     :: "r"(smem_u32(smem_dst)), "l"(gsrc), "n"(kBytes), "l"(pol) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" :: "n"(N) : "memory"); }


// mbarrier + bulk (TMA-engine) copies global -> shared: completion is
// counted in bytes on the barrier (complete_tx), the copy goes through the
// async proxy rather than the LSU pipe.
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
__device__ __forceinline__ void tma_load_hint(void* dst, const void* src, uint32_t bytes, uint64_t* b, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        :: "r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(b)), "l"(pol) : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2::evict_last [%0];" :: "l"(p));
}

// generic-proxy accesses of shared memory before a later async-proxy write
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// apply_endpoint_update (engine.cpp:276-306) on the Hogwild store, without
// calls into IEEE slow paths. Returns 1 if applied.
template <typename T, typename R>
__device__ __forceinline__ uint32_t hog_apply_t(void* coords, uint32_t ni, int ei, uint32_t nj, int ej,
                                              double d_ref, double eta, R& r, uint64_t pol, double vix,
                                              double viy, double vjx, double vjy);

template <typename T, typename R>
__device__ __forceinline__ uint32_t hog_update_t(void* coords, uint32_t ni, int ei, uint32_t nj, int ej,
                                               double d_ref, double eta, R& r, uint64_t pol) {
    if (!(d_ref > 0.0)) return 0;
    double vix, viy, vjx, vjy;
    CoordHint<T>::get(coords, ni, ei, pol, vix, viy);
    CoordHint<T>::get(coords, nj, ej, pol, vjx, vjy);
    return hog_apply_t<T>(coords, ni, ei, nj, ej, d_ref, eta, r, pol, vix, viy, vjx, vjy);
}

// hog_apply_t that also returns the new v_i (warp-shuffle reuse keeps
// updating the same i endpoint).
template <typename T, bool kGivenAnchors = false, typename R>
__device__ __forceinline__ uint32_t hog_apply_io_t(void* coords, uint32_t ni, int ei, uint32_t nj, int ej,
                                                 double d_ref, double eta, R& r, uint64_t pol, double& vix,
                                                 double& viy, double vjx, double vjy, double anc_i = 0.0,
                                                 double anc_j = 0.0);

// The arithmetic and write-back half of hog_update_t, on endpoint values the
// caller loaded (d_ref > 0).
template <typename T, typename R>
__device__ __forceinline__ uint32_t hog_apply_t(void* coords, uint32_t ni, int ei, uint32_t nj, int ej,
                                              double d_ref, double eta, R& r, uint64_t pol, double vix,
                                              double viy, double vjx, double vjy) {
    return hog_apply_io_t<T>(coords, ni, ei, nj, ej, d_ref, eta, r, pol, vix, viy, vjx, vjy);
}

// kGivenAnchors (anchored store only): the caller holds both nodes' block
// anchors, so the write-back does not re-read them.
template <typename T, bool kGivenAnchors, typename R>
__device__ __forceinline__ uint32_t hog_apply_io_t(void* coords, uint32_t ni, int ei, uint32_t nj, int ej,
                                                 double d_ref, double eta, R& r, uint64_t pol, double& vix,
                                                 double& viy, double vjx, double vjy, double anc_i,
                                                 double anc_j) {
    double mu = eta * rcp_nr(d_ref * d_ref);
    if (mu > 1.0) mu = 1.0;
    const double dx = vix - vjx;
    const double dy = viy - vjy;
    const double s2 = dx * dx + dy * dy;
    double ux, uy, mag;
    if (s2 < 1e-18) {  // |v_i - v_j| < 1e-9: random unit direction
        float sn, cs;
        sincospif(2.0f * static_cast<float>(r.uniform()), &sn, &cs);
        ux = cs;
        uy = sn;
        mag = sqrt(s2);
    } else {
        const double rs = rsqrt_nr(s2);
        mag = s2 * rs;
        ux = dx * rs;
        uy = dy * rs;
    }
    const double delta = mu * (mag - d_ref) * 0.5;
    vix -= delta * ux;
    viy -= delta * uy;
    if constexpr (kGivenAnchors) {
        CoordHint<T>::set_anchored(coords, ni, ei, pol, vix, viy, anc_i);
        CoordHint<T>::set_anchored(coords, nj, ej, pol, vjx + delta * ux, vjy + delta * uy, anc_j);
    } else {
        CoordHint<T>::set(coords, ni, ei, pol, vix, viy);
        CoordHint<T>::set(coords, nj, ej, pol, vjx + delta * ux, vjy + delta * uy);
    }
    return 1;
}


}  // namespace pgl
