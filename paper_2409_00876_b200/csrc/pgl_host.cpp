// pgl_host.cpp — host driver and C-ABI of libpgl_b200.so.
//
// Host side of the drop-in for pglayout::run_layout / run_layout_reuse /
// sampled_path_stress (engine.cpp:174-247, metrics.cpp:108-159):
//   validate_config (engine.cpp:15-28) -> make_schedule (:251-274) ->
//   init_layout (layout.cpp:20-34, bit-exact, FP64) -> pack the graph into
//   16-byte step records + guide table -> H2D -> n_iters kernel launches on
//   one stream -> D2H of the coordinates in Layout::snapshot order.
// Everything here is plain C++ (g++, -ffp-contract=off); the device code is
// in pgl_sgd.cu / pgl_sps.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "pgl_internal.hpp"

namespace pgl {

namespace {

const char* const kTypeNames[] = {
    "",           "InvalidParameter", "UnknownNode",   "EmptyPath",      "IndexOutOfRange",
    "EmptyGraph", "DegenerateGraph",  "MalformedLine", "UnknownSegment", "NoPaths",
    "NonFiniteCoordinate", "MalformedRow", "CountMismatch", "ZeroReference", "CorpusTooLarge"};

// ErrorKind of each exception class (errors.hpp:31-44) -> status.
int status_of(int type) {
    switch (type) {
        case PGL_ERR_INVALID_PARAMETER: return PGL_E_USAGE;
        case PGL_ERR_INDEX_OUT_OF_RANGE: return PGL_E_INTERNAL;
        case PGL_ERR_CUDA: return PGL_E_INTERNAL;
        case PGL_ERR_CALLBACK: return PGL_E_CALLBACK;
        case PGL_ERR_NONE: return PGL_OK;
        default: return type <= PGL_ERR_CORPUS_TOO_LARGE ? PGL_E_INPUT : PGL_E_INTERNAL;
    }
}

thread_local std::string t_err;
thread_local int t_err_type = 0;

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        t_err.clear();
        t_err_type = 0;
        return PGL_OK;
    } catch (const Failure& f) {
        t_err = f.what();
        t_err_type = f.type;
        return status_of(f.type);
    } catch (const std::bad_alloc&) {
        t_err = "host allocation failed";
        t_err_type = PGL_ERR_CUDA;
        return PGL_E_INTERNAL;
    } catch (const std::exception& e) {
        t_err = e.what();
        t_err_type = PGL_ERR_CUDA;
        return PGL_E_INTERNAL;
    }
}

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

unsigned host_threads() {
    const unsigned h = std::thread::hardware_concurrency();
    return std::max(1u, std::min(h ? h : 1u, 64u));
}

template <typename F>
void parallel_for(uint64_t n, F&& f) {  // f(begin, end)
    const unsigned T = static_cast<unsigned>(std::min<uint64_t>(host_threads(), std::max<uint64_t>(1, n / 65536)));
    if (T <= 1) {
        f(uint64_t{0}, n);
        return;
    }
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < T; ++t)
        pool.emplace_back([&, t] { f(n * t / T, n * (t + 1) / T); });
    for (auto& th : pool) th.join();
}

// ---- reference host math, restated --------------------------------------

constexpr uint64_t kPhi = 0x9E3779B97F4A7C15ULL;

struct HostRng {  // xoshiro256+ (rng.hpp:13-48)
    uint64_t s[4];
    HostRng(uint64_t seed, uint64_t worker) {
        uint64_t key = seed ^ (kPhi * (worker + 1));
        for (auto& w : s) {
            uint64_t z = (key += kPhi);
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
            w = z ^ (z >> 31);
        }
        if ((s[0] | s[1] | s[2] | s[3]) == 0) s[0] = kPhi;
    }
    uint64_t next() {
        const uint64_t out = s[0] + s[3], t = s[1] << 17;
        s[2] ^= s[0];
        s[3] ^= s[1];
        s[1] ^= s[2];
        s[0] ^= s[3];
        s[2] ^= t;
        s[3] = (s[3] << 45) | (s[3] >> 19);
        return out;
    }
    double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    bool coin() { return (next() >> 63) != 0; }
    uint64_t below(uint64_t n) { return static_cast<uint64_t>((static_cast<unsigned __int128>(next()) * n) >> 64); }
};

constexpr uint64_t kStreamInit = 1ULL << 62;   // rng.hpp:76
constexpr uint64_t kStreamSynth = 1ULL << 60;  // rng.hpp:78

void validate_config(const pgl_layout_config& c) {  // engine.cpp:15-28
    if (c.n_iters < 1) raise(PGL_ERR_INVALID_PARAMETER, "n_iters must be >= 1");
    if (c.threads < 1) raise(PGL_ERR_INVALID_PARAMETER, "threads must be >= 1");
    if (c.batch_size < 1) raise(PGL_ERR_INVALID_PARAMETER, "batch_size must be >= 1");
    if (!(c.zipf_theta > 0.0) || !std::isfinite(c.zipf_theta))
        raise(PGL_ERR_INVALID_PARAMETER, "zipf_theta must be positive");
    if (c.zipf_space_max < 1) raise(PGL_ERR_INVALID_PARAMETER, "zipf_space_max must be >= 1");
    if (!(c.eta_min_eps > 0.0)) raise(PGL_ERR_INVALID_PARAMETER, "eta_min_eps must be positive");
    if (c.drf != 1 && c.drf != 2 && c.drf != 4) raise(PGL_ERR_INVALID_PARAMETER, "drf must be 1, 2 or 4");
    if (c.srf < 1) raise(PGL_ERR_INVALID_PARAMETER, "srf must be >= 1");
}

void eta_schedule(double eta_max, double eta_min, uint32_t n, double* etas) {  // engine.cpp:251-264
    if (n < 1) raise(PGL_ERR_INVALID_PARAMETER, "schedule needs n_iters >= 1");
    if (!(eta_max > 0.0) || !(eta_min > 0.0) || !(eta_min <= eta_max))
        raise(PGL_ERR_INVALID_PARAMETER, "schedule needs 0 < eta_min <= eta_max");
    const double lambda = n > 1 ? std::log(eta_max / eta_min) / (n - 1) : 0.0;
    for (uint32_t t = 0; t < n; ++t) etas[t] = eta_max * std::exp(-lambda * t);
}

// Summary of a graph view, computed once.
struct ViewSummary {
    uint64_t total_steps = 0, total_nt = 0, max_path_len = 0;
    bool usable = false;
};

ViewSummary summarize(const pgl_graph_view* v) {
    if (!v) raise(PGL_ERR_INVALID_PARAMETER, "graph view is null");
    if (v->n_paths && (!v->path_steps || !v->path_n_steps || !v->path_total_len))
        raise(PGL_ERR_INVALID_PARAMETER, "graph view has paths but null path arrays");
    if (v->n_nodes && !v->node_len) raise(PGL_ERR_INVALID_PARAMETER, "graph view has nodes but no node_len");
    ViewSummary s;
    for (uint64_t n = 0; n < v->n_nodes; ++n) s.total_nt += v->node_len[n];
    for (uint32_t p = 0; p < v->n_paths; ++p) {
        if (v->path_n_steps[p] == 0) raise(PGL_ERR_EMPTY_PATH, "path " + std::to_string(p) + " has no steps");
        s.total_steps += v->path_n_steps[p];
        s.max_path_len = std::max(s.max_path_len, v->path_total_len[p]);
        if (v->path_n_steps[p] >= 2) s.usable = true;
    }
    return s;
}

void schedule_for(const pgl_graph_view* v, const ViewSummary& s, const pgl_layout_config& c, double* etas) {
    if (v->n_paths == 0 || !s.usable) raise(PGL_ERR_DEGENERATE_GRAPH, "schedule needs a path pair with d_ref > 0");
    const uint64_t dmax = std::max<uint64_t>(1, s.max_path_len);  // engine.cpp:269-270
    eta_schedule(static_cast<double>(dmax) * static_cast<double>(dmax), c.eta_min_eps, c.n_iters, etas);
}

// init_layout (layout.cpp:20-34): x = running offset in node-id order, y
// uniform in +-sqrt(total nt) from stream seed_worker(seed, 2^62), start
// then end per node. Sequential by construction (one stream).
void init_layout(const pgl_graph_view* v, uint64_t total_nt, uint64_t seed, double* out) {
    HostRng r(seed, kStreamInit);
    const double amp = std::sqrt(static_cast<double>(total_nt));
    uint64_t off = 0;
    for (uint64_t n = 0; n < v->n_nodes; ++n) {
        out[4 * n + 0] = static_cast<double>(off);
        out[4 * n + 1] = (2.0 * r.uniform() - 1.0) * amp;
        out[4 * n + 2] = static_cast<double>(off + v->node_len[n]);
        out[4 * n + 3] = (2.0 * r.uniform() - 1.0) * amp;
        off += v->node_len[n];
    }
}

// Device buffers come from the device's stream-ordered memory pool on the
// owning graph's stream; the pool keeps up to kPoolKeep bytes reserved after
// a graph is destroyed, so repeated layouts (pgl_layout_run per call) do not
// pay cudaMalloc/cudaFree of their 1-15 GB index every time.
constexpr uint64_t kPoolKeep = 48ULL << 30;

void keep_pool(int device) {
    static std::mutex mu;
    static std::vector<int> done;
    std::lock_guard<std::mutex> lock(mu);
    if (std::find(done.begin(), done.end(), device) != done.end()) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t keep = kPoolKeep;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    done.push_back(device);
}

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    cudaStream_t s = nullptr;  // allocation / free stream (the owning graph's)
    void alloc(size_t count) {
        if (count <= n && p) return;
        release();
        PGL_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), std::max<size_t>(1, count) * sizeof(T), s));
        n = count;
    }
    void release() {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        n = 0;
    }
    ~DevBuf() { release(); }
};

// Pinned staging blocks are recycled through a small process-wide pool
// (cudaHostAlloc/cudaFreeHost of 128 MiB cost tens of milliseconds).
struct PinnedPool {
    std::mutex mu;
    std::vector<std::pair<void*, size_t>> free;
    size_t held = 0;
    static constexpr size_t kCap = 1ULL << 30;
    void* get(size_t b, size_t* got) {
        {
            std::lock_guard<std::mutex> lock(mu);
            for (size_t k = 0; k < free.size(); ++k)
                if (free[k].second >= b) {
                    void* p = free[k].first;
                    *got = free[k].second;
                    held -= *got;
                    free.erase(free.begin() + static_cast<long>(k));
                    return p;
                }
        }
        void* p = nullptr;
        PGL_CUDA(cudaHostAlloc(&p, b, cudaHostAllocDefault));
        *got = b;
        return p;
    }
    void put(void* p, size_t b) {
        {
            std::lock_guard<std::mutex> lock(mu);
            if (held + b <= kCap) {
                free.emplace_back(p, b);
                held += b;
                return;
            }
        }
        cudaFreeHost(p);
    }
};
PinnedPool& pinned_pool() {
    static PinnedPool* pool = new PinnedPool;  // leaked: outlives static destructors
    return *pool;
}

struct PinnedBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void alloc(size_t b) {
        if (b <= bytes && p) return;
        release();
        p = pinned_pool().get(b, &bytes);
    }
    void release() {
        if (p) pinned_pool().put(p, bytes);
        p = nullptr;
        bytes = 0;
    }
    ~PinnedBuf() { release(); }
};

struct DeviceGuard {  // restores the caller's current device
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        PGL_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

}  // namespace

[[noreturn]] void raise(int type, const std::string& detail) {
    const char* name = (type >= 0 && type <= PGL_ERR_CORPUS_TOO_LARGE) ? kTypeNames[type] : "CudaError";
    throw Failure(type, std::string(name) + ": " + detail);
}

[[noreturn]] void raise_cuda(int err, const char* what, const char* file, int line) {
    throw Failure(PGL_ERR_CUDA, std::string("CudaError: ") + cudaGetErrorString(static_cast<cudaError_t>(err)) +
                                    " in " + what + " (" + file + ":" + std::to_string(line) + ")");
}

void zipf_constants(uint64_t n, double theta, double* hx1, double* hxn, double* s) {
    // ZipfSampler ctor (rng.hpp:91-98) with its helpers (:122-144).
    auto helper1 = [](double x) { return std::abs(x) > 1e-8 ? std::log1p(x) / x : 1.0 - x * (0.5 - x * (1.0 / 3.0 - 0.25 * x)); };
    auto helper2 = [](double x) {
        return std::abs(x) > 1e-8 ? std::expm1(x) / x : 1.0 + x * 0.5 * (1.0 + x * (1.0 / 3.0) * (1.0 + 0.25 * x));
    };
    auto H = [&](double x) {
        const double lx = std::log(x);
        return helper2((1.0 - theta) * lx) * lx;
    };
    auto h = [&](double x) { return std::exp(-theta * std::log(x)); };
    auto Hinv = [&](double x) {
        double t = x * (1.0 - theta);
        if (t < -1.0) t = -1.0;
        return std::exp(helper1(t) * x);
    };
    *hx1 = H(1.5) - 1.0;
    *hxn = H(static_cast<double>(n) + 0.5);
    *s = 2.0 - Hinv(H(2.5) - h(2.0));
}

void finish_report(pgl_stress_report* r, double ssd) {  // metrics.cpp:14-23
    r->std_dev = r->n >= 2 ? std::sqrt(ssd / static_cast<double>(r->n - 1)) : 0.0;
    const double half = r->n > 0 ? 1.96 * r->std_dev / std::sqrt(static_cast<double>(r->n)) : 0.0;
    r->ci_low = r->mean - half;
    r->ci_high = r->mean + half;
}

// Walker/Vose alias table for Zipf(zn, theta) on [1, zn] with the exact pmf
// k^-theta / H(zn, theta) that the rejection-inversion sampler targets
// (rng.hpp:83-151). Appended to `out`; thresholds are P(keep) * 2^32.
void append_zipf_alias(uint64_t zn, double theta, std::vector<ZipfAlias>& out) {
    if (zn > (1ULL << 24)) raise(PGL_ERR_INVALID_PARAMETER, "zipf support above 2^24 is not supported by the GPU sampler");
    const size_t n = static_cast<size_t>(zn), off = out.size();
    std::vector<double> q(n);
    double h = 0.0, comp = 0.0;  // Kahan sum of k^-theta, smallest terms first
    for (size_t k = n; k >= 1; --k) {
        const double t = std::pow(static_cast<double>(k), -theta) - comp;
        const double s2 = h + t;
        comp = (s2 - h) - t;
        h = s2;
    }
    for (size_t k = 0; k < n; ++k) q[k] = std::pow(static_cast<double>(k + 1), -theta) / h * static_cast<double>(n);
    out.resize(off + n);
    std::vector<uint32_t> small, large;
    for (size_t k = 0; k < n; ++k) (q[k] < 1.0 ? small : large).push_back(static_cast<uint32_t>(k));
    while (!small.empty() && !large.empty()) {
        const uint32_t sm = small.back(), lg = large.back();
        small.pop_back();
        large.pop_back();
        const double t = q[sm] * 4294967296.0;
        out[off + sm] = ZipfAlias{static_cast<uint32_t>(std::min(t, 4294967295.0)), lg};
        q[lg] = (q[lg] + q[sm]) - 1.0;
        (q[lg] < 1.0 ? small : large).push_back(lg);
    }
    for (uint32_t k : large) out[off + k] = ZipfAlias{0xFFFFFFFFu, k};
    for (uint32_t k : small) out[off + k] = ZipfAlias{0xFFFFFFFFu, k};  // rounding leftovers
}

}  // namespace pgl

using namespace pgl;

// ---- the resident graph ------------------------------------------------------

struct pgl_graph {
    int device = 0;
    cudaStream_t stream = nullptr;
    uint64_t n_nodes = 0;
    uint32_t n_paths = 0;
    ViewSummary sum;
    std::vector<uint64_t> node_len;      // host copy (init_layout)
    std::vector<uint64_t> path_n_steps;  // host copy (zipf supports)
    DevBuf<StepRec> step;
    DevBuf<uint2> rec8;                  // 8-byte records, built on first use (lean variants 13/14)
    DevBuf<uint64_t> cum;
    DevBuf<uint32_t> guide;
    DevBuf<uint32_t> sguide;
    uint32_t sguide_bits = 0, sguide_shift = 0;
    DevBuf<PathConst> pc;
    DevBuf<uint4> fguide;                // per-layout path guide with inline constants (k_sgd_tiles)
    uint32_t fguide_shift = 0;
    DevBuf<ZipfAlias> zalias;
    uint32_t guide_bits = 8;
    DevBuf<double> coords64;             // [4V] FP64 layout / staging
    DevBuf<float> coords32;              // [4V] FP32 layout
    int layout_f64 = -1;                 // precision of the resident layout (-1: none)
    int ids_local = -1;                  // node ids follow path order (anchored store usable); -1 unknown
    DevBuf<uint64_t> rng;                // SoA xoshiro states
    DevBuf<unsigned long long> stats;    // [8]
    SpsScratch sps{};
    pgl_timing timing{};
    PinnedBuf pin;

    void set_stream(cudaStream_t st) {
        stream = st;
        step.s = cum.s = stream;
        rec8.s = stream;
        guide.s = sguide.s = stream;
        pc.s = fguide.s = stream;
        zalias.s = stream;
        coords64.s = stream;
        coords32.s = stream;
        rng.s = stream;
        stats.s = stream;
    }
    ~pgl_graph() {
        if (sps.part) cudaFree(sps.part);
        if (sps.cnt) cudaFree(sps.cnt);
        if (sps.scal) cudaFree(sps.scal);
        step.release();
        rec8.release();
        cum.release();
        guide.release();
        sguide.release();
        pc.release();
        fguide.release();
        zalias.release();
        coords64.release();
        coords32.release();
        rng.release();
        stats.release();
        if (stream) {
            cudaStreamSynchronize(stream);
            cudaStreamDestroy(stream);
        }
    }

    DevGraph dev() const {
        DevGraph d;
        d.step = step.p;
        d.rec8 = rec8.p;
        d.cum = cum.p;
        d.guide = guide.p;
        d.pc = pc.p;
        d.zalias = zalias.p;
        d.sguide = sguide.p;
        d.sguide_bits = sguide_bits;
        d.sguide_shift = sguide_shift;
        d.total_steps = sum.total_steps;
        d.n_paths = n_paths;
        d.guide_bits = guide_bits;
        d.n_nodes = n_nodes;
        return d;
    }
};

namespace {

// Pack the borrowed reference-format view into 16-byte step records,
// multithreaded on the host, streamed through two pinned chunks so packing
// overlaps the H2D copy.
// cum_steps, the selection guide and the step-index guide (shared by both
// ways of building the step records).
void upload_tables(pgl_graph* G, const std::vector<uint64_t>& cum) {
    const uint64_t S = G->sum.total_steps;
    const uint32_t P = G->n_paths;
    G->step.alloc(S);
    G->cum.alloc(P + 1);
    PGL_CUDA(copy_async(G->cum.p, cum.data(), (P + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, G->stream));

    // guide table: bucket b of the top guide_bits of the selection draw
    // starts at pick floor(b * S / 2^bits); store the path containing it.
    uint32_t bits = 8;
    while ((1u << bits) < 8u * std::max<uint32_t>(P, 1) && bits < 16) ++bits;
    G->guide_bits = bits;
    std::vector<uint32_t> guide(1u << bits, 0);
    for (uint64_t b = 0; b < guide.size(); ++b) {
        const uint64_t first = static_cast<uint64_t>((static_cast<unsigned __int128>(b) * S) >> bits);
        guide[b] = static_cast<uint32_t>(std::upper_bound(cum.begin(), cum.end(), first) - cum.begin() - 1);
        if (guide[b] >= P) guide[b] = P ? P - 1 : 0;
    }
    {   // step-index guide: path containing step b << shift (path_of_step)
        uint32_t L = 1;
        while ((1ULL << L) < std::max<uint64_t>(S, 2)) ++L;
        // ~16 buckets per path keeps the forward scan at ~1 step while the
        // table stays small enough to live in L1 next to the async
        // pipeline's shared memory (2^10 entries = 4 KB at 90 paths)
        uint32_t want = 10;
        while ((1u << want) < 16u * std::max<uint32_t>(P, 1) && want < 14) ++want;
        const uint32_t sb = std::min<uint32_t>(L, want);
        G->sguide_bits = sb;
        G->sguide_shift = L - sb;
        std::vector<uint32_t> sg(1u << sb, 0);
        for (uint64_t b = 0; b < sg.size(); ++b) {
            const uint64_t first = b << G->sguide_shift;
            const uint64_t pth = static_cast<uint64_t>(std::upper_bound(cum.begin(), cum.end(), first) - cum.begin() - 1);
            sg[b] = static_cast<uint32_t>(std::min<uint64_t>(pth, P ? P - 1 : 0));
        }
        G->sguide.alloc(sg.size());
        PGL_CUDA(copy_async(G->sguide.p, sg.data(), sg.size() * sizeof(uint32_t), cudaMemcpyHostToDevice,
                                 G->stream));
        PGL_CUDA(cudaStreamSynchronize(G->stream));
    }
    G->guide.alloc(guide.size());
    PGL_CUDA(copy_async(G->guide.p, guide.data(), guide.size() * sizeof(uint32_t), cudaMemcpyHostToDevice,
                             G->stream));
    PGL_CUDA(cudaStreamSynchronize(G->stream));
}

// Compact upload: one u32 word per step (node | reverse << 31, 4 bytes
// instead of a 16-byte record) plus u32 node lengths; the device rebuilds
// the offsets and records exactly as for a GFA (build_records_device).
// Valid when the view is what build_graph makes (graph.cpp:38-50): every
// step's seq_len is its node's length and offsets are the running sums.
// Checked step by step while packing; returns false (nothing built) when a
// view is not of that form, and pack_graph then uploads full records.
bool pack_graph_compact(pgl_graph* G, const pgl_graph_view* v, const std::vector<uint64_t>& cum) {
    const uint64_t S = G->sum.total_steps, V = v->n_nodes;
    if (V >= (1ULL << 31) || S == 0) return false;
    std::vector<uint32_t> len32(V);
    for (uint64_t n = 0; n < V; ++n) {
        if (v->node_len[n] > 0xFFFFFFFFull) return false;
        len32[n] = static_cast<uint32_t>(v->node_len[n]);
    }
    DevBuf<uint32_t> dlen, dsteps;
    dlen.s = dsteps.s = G->stream;
    dlen.alloc(std::max<uint64_t>(V, 1));
    dsteps.alloc(S);
    PGL_CUDA(copy_async(dlen.p, len32.data(), V * sizeof(uint32_t), cudaMemcpyHostToDevice, G->stream));
    const uint64_t kChunk = std::min<uint64_t>(1ULL << 25, S);  // <= 32 Mi steps = 128 MiB
    G->pin.alloc(2 * kChunk * sizeof(uint32_t));
    uint32_t* bufs[2] = {static_cast<uint32_t*>(G->pin.p), static_cast<uint32_t*>(G->pin.p) + kChunk};
    cudaEvent_t done[2];
    PGL_CUDA(cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming));
    PGL_CUDA(cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming));
    std::atomic<int> bad_node{0}, irregular{0};
    const uint64_t n_chunks = (S + kChunk - 1) / kChunk;
    for (uint64_t c = 0; c < n_chunks && !bad_node.load() && !irregular.load(); ++c) {
        uint32_t* buf = bufs[c & 1];
        if (c >= 2) PGL_CUDA(cudaEventSynchronize(done[c & 1]));
        const uint64_t k0 = c * kChunk, k1 = std::min(S, k0 + kChunk);
        parallel_for(k1 - k0, [&](uint64_t b, uint64_t e) {
            uint64_t k = k0 + b;
            uint32_t p = static_cast<uint32_t>(std::upper_bound(cum.begin(), cum.end(), k) - cum.begin() - 1);
            bool odd = false, bad = false;
            for (; k < k0 + e; ++k) {
                while (k >= cum[p + 1]) ++p;
                const pgl_path_step* ps = v->path_steps[p];
                const uint64_t i = k - cum[p];
                const pgl_path_step& st = ps[i];
                if (st.node_id >= V) {
                    bad = true;
                    break;
                }
                const uint64_t want = i ? ps[i - 1].offset + ps[i - 1].seq_len : 0;
                odd |= st.seq_len != len32[st.node_id] || st.offset != want || st.node_id >= (1u << 31);
                buf[k - k0] = st.node_id | (st.orient ? 1u << 31 : 0u);
            }
            if (bad) bad_node.store(1, std::memory_order_relaxed);
            if (odd) irregular.store(1, std::memory_order_relaxed);
        });
        PGL_CUDA(copy_async(dsteps.p + k0, buf, (k1 - k0) * sizeof(uint32_t), cudaMemcpyHostToDevice,
                                 G->stream));
        PGL_CUDA(cudaEventRecord(done[c & 1], G->stream));
    }
    PGL_CUDA(cudaStreamSynchronize(G->stream));
    cudaEventDestroy(done[0]);
    cudaEventDestroy(done[1]);
    if (bad_node.load()) raise(PGL_ERR_UNKNOWN_NODE, "path references a node outside the graph");
    if (irregular.load()) return false;
    build_records_device(dsteps.p, dlen.p, G->cum.p, G->n_paths, S, G->step.p, G->stream);
    PGL_CUDA(cudaStreamSynchronize(G->stream));
    return true;
}

void pack_graph(pgl_graph* G, const pgl_graph_view* v) {
    const uint64_t S = G->sum.total_steps;
    const uint32_t P = v->n_paths;
    std::vector<uint64_t> cum(P + 1, 0);
    for (uint32_t p = 0; p < P; ++p) cum[p + 1] = cum[p] + v->path_n_steps[p];
    for (uint32_t p = 0; p < P; ++p)
        if (v->path_total_len[p] >= (1ULL << 48))
            raise(PGL_ERR_INVALID_PARAMETER, "path longer than 2^48 nucleotides");
    upload_tables(G, cum);
    if (pack_graph_compact(G, v, cum)) return;

    const uint64_t kChunk = std::min<uint64_t>(1ULL << 22, std::max<uint64_t>(S, 1));  // <= 4 Mi steps = 64 MiB
    G->pin.alloc(2 * kChunk * sizeof(StepRec));
    StepRec* bufs[2] = {static_cast<StepRec*>(G->pin.p), static_cast<StepRec*>(G->pin.p) + kChunk};
    cudaEvent_t done[2];
    PGL_CUDA(cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming));
    PGL_CUDA(cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming));
    std::atomic<int> bad_node{0};
    const uint64_t n_chunks = (S + kChunk - 1) / kChunk;
    for (uint64_t c = 0; c < n_chunks; ++c) {
        StepRec* buf = bufs[c & 1];
        if (c >= 2) PGL_CUDA(cudaEventSynchronize(done[c & 1]));
        const uint64_t k0 = c * kChunk, k1 = std::min(S, k0 + kChunk);
        parallel_for(k1 - k0, [&](uint64_t b, uint64_t e) {
            uint64_t k = k0 + b;
            uint32_t p = static_cast<uint32_t>(std::upper_bound(cum.begin(), cum.end(), k) - cum.begin() - 1);
            for (; k < k0 + e; ++k) {
                while (k >= cum[p + 1]) ++p;
                const pgl_path_step& st = v->path_steps[p][k - cum[p]];
                if (st.node_id >= v->n_nodes) bad_node.store(1, std::memory_order_relaxed);
                // path_position (graph.hpp:98-109): the far side of a
                // forward visit is its end, of a reverse visit its start.
                const uint64_t near = st.offset, far = st.offset + st.seq_len;
                const uint64_t ps = st.orient ? far : near, pe = st.orient ? near : far;
                buf[k - k0] = StepRec{st.node_id, static_cast<uint32_t>(ps), static_cast<uint32_t>(pe),
                                      static_cast<uint32_t>((ps >> 32) | ((pe >> 32) << 16))};
            }
        });
        PGL_CUDA(copy_async(G->step.p + k0, buf, (k1 - k0) * sizeof(StepRec), cudaMemcpyHostToDevice,
                                 G->stream));
        PGL_CUDA(cudaEventRecord(done[c & 1], G->stream));
    }
    PGL_CUDA(cudaStreamSynchronize(G->stream));
    cudaEventDestroy(done[0]);
    cudaEventDestroy(done[1]);
    if (bad_node.load()) raise(PGL_ERR_UNKNOWN_NODE, "path references a node outside the graph");
}

pgl_graph* create_graph(int device, const pgl_graph_view* v) {
    const ViewSummary s = summarize(v);
    DeviceGuard dg(device);
    auto G = std::make_unique<pgl_graph>();
    G->device = device;
    keep_pool(device);
    cudaStream_t st;
    PGL_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    G->set_stream(st);
    G->n_nodes = v->n_nodes;
    G->n_paths = v->n_paths;
    G->sum = s;
    if (v->n_nodes >= (1ULL << 32)) raise(PGL_ERR_INVALID_PARAMETER, "more than 2^32 nodes");
    G->node_len.assign(v->node_len, v->node_len + v->n_nodes);
    G->path_n_steps.assign(v->path_n_steps, v->path_n_steps + v->n_paths);
    pack_graph(G.get(), v);
    G->stats.alloc(10);
    return G.release();
}

// The resident layout's store as the kernels address it (anchored: the base
// above the block anchors, anch_base).
const void* resident_coords(pgl_graph* G, int kind) {
    if (kind == PGL_COORD_F64) return G->coords64.p;
    if (kind == PGL_COORD_F32) return G->coords32.p;
    return anch_base(G->coords32.p, G->n_nodes);
}

// The resident layout as FP64 in G->coords64 (a no-op for an FP64 layout).
void to_f64(pgl_graph* G, int kind) {
    const uint64_t V = G->n_nodes;
    if (kind == PGL_COORD_F32)
        launch_f32_to_f64(G->coords32.p, G->coords64.p, 4 * V, G->stream);
    else if (kind == PGL_COORD_F32_ANCHORED)
        launch_anch_to_f64(anch_base(G->coords32.p, V), G->coords64.p, V, G->stream);
}

// pgl_graph_create_gfa: GFA -> compact steps on the host -> step records on
// the device (pgl_pack.cu). The 24-byte PathStep arrays are never built.
pgl_graph* create_graph_gfa(int device, GfaGraph* gf) {
    const CompactGraph c = gfa_compact(gf);
    DeviceGuard dg(device);
    keep_pool(device);
    auto G = std::make_unique<pgl_graph>();
    G->device = device;
    cudaStream_t st;
    PGL_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    G->set_stream(st);
    G->n_nodes = c.n_nodes;
    G->n_paths = c.n_paths;
    if (c.n_nodes >= (1ULL << 31)) raise(PGL_ERR_INVALID_PARAMETER, "more than 2^31 nodes");
    G->node_len.assign(c.node_len, c.node_len + c.n_nodes);
    G->path_n_steps.resize(c.n_paths);
    ViewSummary sm;
    for (uint64_t n = 0; n < c.n_nodes; ++n) sm.total_nt += c.node_len[n];
    for (uint32_t p = 0; p < c.n_paths; ++p) {
        G->path_n_steps[p] = c.path_begin[p + 1] - c.path_begin[p];
        sm.max_path_len = std::max(sm.max_path_len, c.path_total[p]);
        if (G->path_n_steps[p] >= 2) sm.usable = true;
        if (c.path_total[p] >= (1ULL << 48)) raise(PGL_ERR_INVALID_PARAMETER, "path longer than 2^48 nucleotides");
    }
    sm.total_steps = c.path_begin[c.n_paths];
    G->sum = sm;
    std::vector<uint64_t> cum(c.path_begin, c.path_begin + c.n_paths + 1);
    upload_tables(G.get(), cum);
    // node lengths as u32 (path nodes are checked <= 2^32-1 by the parser)
    std::vector<uint32_t> len32(c.n_nodes);
    for (uint64_t n = 0; n < c.n_nodes; ++n)
        len32[n] = static_cast<uint32_t>(std::min<uint64_t>(c.node_len[n], 0xFFFFFFFFull));
    DevBuf<uint32_t> dlen, dsteps;
    dlen.s = dsteps.s = G->stream;
    dlen.alloc(std::max<uint64_t>(c.n_nodes, 1));
    dsteps.alloc(std::max<uint64_t>(sm.total_steps, 1));
    PGL_CUDA(copy_async(dlen.p, len32.data(), c.n_nodes * sizeof(uint32_t), cudaMemcpyHostToDevice, G->stream));
    PGL_CUDA(copy_async(dsteps.p, c.steps, sm.total_steps * sizeof(uint32_t), cudaMemcpyHostToDevice, G->stream));
    build_records_device(dsteps.p, dlen.p, G->cum.p, c.n_paths, sm.total_steps, G->step.p, G->stream);
    PGL_CUDA(cudaStreamSynchronize(G->stream));
    G->stats.alloc(10);
    return G.release();
}

// Resident view-like accessors for the schedule/init helpers.
pgl_graph_view view_of(const pgl_graph* G) {
    pgl_graph_view v{};
    v.n_nodes = G->n_nodes;
    v.node_len = G->node_len.data();
    v.n_paths = G->n_paths;
    return v;
}

constexpr uint32_t kHopLanes = 8;  // default lanes per shared Zipf hop

// Tile-kernel variant (pgl_tiles.cu): auto = the asynchronous cp.async
// pipeline at 3 CTAs/SM once the concurrency cap allows 8 warps per SM,
// else the register pipeline, whose shorter read-to-write window keeps
// small graphs' layouts closest to the reference.
// lean_ok: the run is one the lean async kernel (variants 7, 8) covers --
// batch 32, drf 1, no warp-shuffle reuse, the shared window + Zipf-hop
// sampler, 32 <= S < 2^30 steps, paths shorter than 2^32 nt.
int tile_variant(int device, const pgl_layout_ext& ext, uint32_t cap, bool lean_ok, bool rec8_ok) {
    int v = static_cast<int>(ext.kernel_variant & 15);
    const int force64 = static_cast<int>(ext.kernel_variant & 16);
    if (v == 0) {
        int sms = 0;
        PGL_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        // the async pipeline once the cap allows a CTA's worth of warps per
        // SM (config 5, cap 2988 warps: 38.7 vs 36.1 G upd/s for variant 1,
        // at lower SPS) -- its lean specialisation where the run allows, with
        // synchronous apply at 4 CTAs/SM (variant 10: C3 58.0 vs 53.6 G upd/s
        // for the staged variant 7, profiles/r02_ab_sync_early.jsonl);
        // the register pipeline's shorter read-to-write window where the
        // cap binds hard (config 1). The lean default reads the 8-byte
        // records (variant 13: C3 61.2 vs 58.6, C2 63.9 vs 59.9 G upd/s for
        // variant 10, profiles/r02_ab_rec8_c{3,2}.jsonl)
        v = cap >= static_cast<uint32_t>(sms) * 8 ? (lean_ok && !force64 ? (rec8_ok ? 13 : 10) : 6) : 1;
    }
    if (v != 1 && v != 2 && v != 5 && v != 6 && !(v >= 7 && v <= 14))
        raise(PGL_ERR_INVALID_PARAMETER, "pgl_layout_ext.kernel_variant: tile kernel variants are 0, 1, 2, 5-14");
    if (v >= 7 && v <= 14 && (!lean_ok || force64))
        raise(PGL_ERR_INVALID_PARAMETER,
              "pgl_layout_ext.kernel_variant 7-14 (lean) needs batch_size 32, drf 1, no reuse_shuffle, "
              "pair_window 1 or 3, 32 <= steps < 2^30 and paths shorter than 2^32 nt");
    if ((v == 13 || v == 14) && !rec8_ok)
        raise(PGL_ERR_INVALID_PARAMETER, "pgl_layout_ext.kernel_variant 13/14 (8-byte records) needs fewer than 2^31 nodes");
    return v | force64 | (v >= 7 && v <= 14 && ext.diag ? 32 : 0);
}

// The i.i.d. kernel's variant when pgl_layout_ext.kernel_variant is 0
// (pgl_sgd.cu hogwild_fn).
constexpr int kIidAutoVariant = 8;

uint32_t auto_max_warps(uint64_t n_nodes) {
    // Hogwild concurrency cap: keep the number of in-flight updates well
    // below the number of endpoints so concurrent read-modify-writes on one
    // endpoint stay rare (SURVEY.md §7 hard part 1). One warp (32 lanes) per
    // 80 nodes, at least 4 warps: config 1 (10k nodes) runs 124 warps; the
    // cap sweep there put the median SPS within 0.7% of the reference up to
    // 128 warps and 4% above it at 512. From ~200k nodes up the occupancy
    // limit binds first.
    const uint64_t w = n_nodes / 80;
    return static_cast<uint32_t>(std::max<uint64_t>(4, std::min<uint64_t>(w, 1u << 24)));
}

// Device -> pageable host copy of a large result through two recycled
// pinned chunks: the DMA of chunk c+1 overlaps the host threads' copy of
// chunk c out of pinned memory (and the page faults of a fresh destination
// are taken by all host threads instead of the driver's single staging
// thread).
void copy_out_staged(void* dst, const void* src, uint64_t bytes, cudaStream_t stream) {
    constexpr uint64_t kChunk = 32ULL << 20;
    if (bytes <= 2 * kChunk) {
        PGL_CUDA(copy_async(dst, src, bytes, cudaMemcpyDeviceToHost, stream));
        PGL_CUDA(cudaStreamSynchronize(stream));
        return;
    }
    PinnedBuf pin;
    pin.alloc(2 * kChunk);
    char* bufs[2] = {static_cast<char*>(pin.p), static_cast<char*>(pin.p) + kChunk};
    cudaEvent_t done[2];
    PGL_CUDA(cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming));
    PGL_CUDA(cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming));
    const uint64_t n = (bytes + kChunk - 1) / kChunk;
    auto issue = [&](uint64_t c) {
        const uint64_t o = c * kChunk, b = std::min(kChunk, bytes - o);
        PGL_CUDA(copy_async(bufs[c & 1], static_cast<const char*>(src) + o, b, cudaMemcpyDeviceToHost, stream));
        PGL_CUDA(cudaEventRecord(done[c & 1], stream));
    };
    issue(0);
    for (uint64_t c = 0; c < n; ++c) {
        if (c + 1 < n) issue(c + 1);
        PGL_CUDA(cudaEventSynchronize(done[c & 1]));
        const uint64_t o = c * kChunk, b = std::min(kChunk, bytes - o);
        const char* from = bufs[c & 1];
        char* to = static_cast<char*>(dst) + o;
        parallel_for(b, [&](uint64_t lo, uint64_t hi) { std::memcpy(to + lo, from + lo, hi - lo); });
    }
    cudaEventDestroy(done[0]);
    cudaEventDestroy(done[1]);
}

void graph_layout(pgl_graph* G, const pgl_layout_config* cfgp, const pgl_layout_ext* extp, int reuse,
                  pgl_iteration_cb cb, int cb_wants_coords, void* user, double* out_coords,
                  pgl_run_stats* stats_out, const double* pre_init) {
    const double t_call = now_s();
    if (!cfgp) raise(PGL_ERR_INVALID_PARAMETER, "config is null");
    const pgl_layout_config cfg = *cfgp;
    pgl_layout_ext ext;
    pgl_layout_ext_default(&ext);
    if (extp) {
        if (extp->struct_size < 16 || extp->struct_size > sizeof(pgl_layout_ext))
            raise(PGL_ERR_INVALID_PARAMETER, "pgl_layout_ext.struct_size mismatch");
        std::memcpy(&ext, extp, extp->struct_size);
    }
    if (ext.sampling == PGL_SAMPLING_AUTO) {
        // the tile sampler once the concurrency cap allows the lean tile
        // kernel's full residency (3 CTAs x 8 warps per SM), the i.i.d. kernel
        // where the cap binds (pgl_b200.h PGL_SAMPLING_AUTO;
        // profiles/r02_quality_*.jsonl); warp-shuffle reuse needs the tiles
        int sms = 0;
        PGL_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, G->device));
        const uint32_t cap = ext.max_warps ? ext.max_warps : auto_max_warps(G->n_nodes);
        // (a tile-kernel knob -- variant, unit order or length, partner
        // window, hop lanes, warp-shuffle reuse -- asks for the tiles)
        const bool tile_knobs = ext.kernel_variant || ext.unit_order || ext.unit_len || ext.pair_window ||
                                ext.hop_lanes || ext.reuse_shuffle;
        ext.sampling = tile_knobs || cap >= static_cast<uint32_t>(sms) * 24 ? PGL_SAMPLING_TILES : PGL_SAMPLING_IID;
    }
    if (ext.mode == PGL_MODE_HOGWILD && ext.sampling == PGL_SAMPLING_IID && ext.kernel_variant > 8)
        raise(PGL_ERR_INVALID_PARAMETER, "pgl_layout_ext.kernel_variant: i.i.d. kernel variants are 0-8");
    if (ext.reuse_shuffle && (ext.mode != PGL_MODE_HOGWILD || ext.sampling != PGL_SAMPLING_TILES))
        raise(PGL_ERR_INVALID_PARAMETER, "pgl_layout_ext.reuse_shuffle needs the Hogwild tile sampler");
    if (ext.reuse_shuffle && G->n_paths >= (1u << 19))
        raise(PGL_ERR_INVALID_PARAMETER, "pgl_layout_ext.reuse_shuffle supports fewer than 2^19 paths");
    if (ext.unit_order == PGL_ORDER_FRONTS)
        raise(PGL_ERR_INVALID_PARAMETER, "pgl_layout_ext.unit_order: the fronts order is not available in this build");
    if (ext.unit_order > PGL_ORDER_RANDOM)
        raise(PGL_ERR_INVALID_PARAMETER, "pgl_layout_ext.unit_order: unknown order");
    if (ext.unit_len & (ext.unit_len - 1) || ext.unit_len > 32)
        raise(PGL_ERR_INVALID_PARAMETER, "pgl_layout_ext.unit_len must be 0 or a power of two <= 32");
    if (ext.unit_len && ext.unit_len < 32 && ext.unit_order != PGL_ORDER_RANDOM)
        raise(PGL_ERR_INVALID_PARAMETER, "pgl_layout_ext.unit_len below 32 needs unit_order PGL_ORDER_RANDOM");
    if (ext.coord_precision > PGL_COORD_AUTO)
        raise(PGL_ERR_INVALID_PARAMETER, "pgl_layout_ext.coord_precision: unknown coordinate store");
    if (ext.hop_lanes & (ext.hop_lanes - 1) || ext.hop_lanes > 32)
        raise(PGL_ERR_INVALID_PARAMETER, "pgl_layout_ext.hop_lanes must be 0 or a power of two <= 32");
    if (reuse) {  // run_layout_reuse, engine.cpp:328-334
        if (cfg.drf != 2 && cfg.drf != 4) raise(PGL_ERR_INVALID_PARAMETER, "update reuse needs drf of 2 or 4");
        if (cfg.srf < 1) raise(PGL_ERR_INVALID_PARAMETER, "srf must be >= 1");
    }
    validate_config(cfg);
    if (G->n_paths == 0 || !G->sum.usable)
        raise(PGL_ERR_DEGENERATE_GRAPH, "layout needs at least one path with two or more steps");
    if (ext.mode != PGL_MODE_HOGWILD && ext.mode != PGL_MODE_REPLAY) raise(PGL_ERR_INVALID_PARAMETER, "unknown mode");
    if (ext.sampling > PGL_SAMPLING_AUTO) raise(PGL_ERR_INVALID_PARAMETER, "unknown sampling");

    DeviceGuard dg(G->device);
    const pgl_graph_view hv = view_of(G);
    std::vector<double> etas(cfg.n_iters);
    {  // make_schedule (engine.cpp:266-274): eta_max = (longest path)^2
        const uint64_t dmax = std::max<uint64_t>(1, G->sum.max_path_len);
        eta_schedule(static_cast<double>(dmax) * static_cast<double>(dmax), cfg.eta_min_eps, cfg.n_iters,
                     etas.data());
    }

    const int replay = ext.mode == PGL_MODE_REPLAY;
    // coordinate store: pgl_coord_precision (replay is FP64)
    int kind = replay ? PGL_COORD_F64 : static_cast<int>(ext.coord_precision);
    if (kind == PGL_COORD_AUTO) {
        // FP64 while the array fits comfortably in L2; beyond that the
        // anchored FP32 store -- which needs blocks of 32 consecutive node ids
        // to lie close together along the paths (true for build_graph /
        // write_gfa numbering, not for an arbitrary GFA id order): checked on
        // the device once per graph, >= 99% of the blocks within 2^20 nt
        if (32 * G->n_nodes <= (64ULL << 20)) {
            kind = PGL_COORD_F64;
        } else {
            if (G->ids_local < 0) {
                unsigned long long r[2];
                block_span_stats(G->step.p, G->sum.total_steps, G->n_nodes, (1u << 20) / 256, G->stats.p + 8,
                                 G->stream);
                PGL_CUDA(copy_async(r, G->stats.p + 8, sizeof r, cudaMemcpyDeviceToHost, G->stream));
                PGL_CUDA(cudaStreamSynchronize(G->stream));
                G->ids_local = r[0] * 100 <= r[1] ? 1 : 0;
            }
            kind = G->ids_local ? PGL_COORD_F32_ANCHORED : PGL_COORD_F64;
        }
    }
    const uint64_t V = G->n_nodes;

    // init_layout on the host (bit-exact), upload, narrow to FP32 on device.
    const double t_init = now_s();
    const double* hinit = pre_init;  // pgl_layout_run computes it beside the graph upload
    if (!hinit) {
        G->pin.alloc(std::max<size_t>(G->pin.bytes, 4 * V * sizeof(double)));
        init_layout(&hv, G->sum.total_nt, cfg.global_seed, static_cast<double*>(G->pin.p));
        hinit = static_cast<const double*>(G->pin.p);
    }
    G->coords64.alloc(4 * V);
    cudaEvent_t ev_begin, ev_end;
    PGL_CUDA(cudaEventCreate(&ev_begin));
    PGL_CUDA(cudaEventCreate(&ev_end));
    PGL_CUDA(cudaEventRecord(ev_begin, G->stream));
    PGL_CUDA(copy_async(G->coords64.p, hinit, 4 * V * sizeof(double), cudaMemcpyHostToDevice, G->stream));
    void* coords = G->coords64.p;
    if (kind == PGL_COORD_F32) {
        G->coords32.alloc(4 * V);
        launch_f64_to_f32(G->coords64.p, G->coords32.p, 4 * V, G->stream);
        coords = G->coords32.p;
    } else if (kind == PGL_COORD_F32_ANCHORED) {
        G->coords32.alloc(anch_bytes(V) / sizeof(float));
        coords = anch_base(G->coords32.p, V);
        launch_f64_to_anch(G->coords64.p, coords, V, G->stream);
    }

    // per-path constants for this config (zipf_params_for, engine.cpp:36-39)
    // plus one alias table per distinct Zipf support for the Hogwild kernel.
    std::vector<PathConst> pcs(G->n_paths);
    std::vector<ZipfAlias> tables;
    uint32_t zdef_n = 1;
    uint64_t zdef_tab = 0;
    {
        uint64_t base = 0;
        struct Memo {
            uint64_t zn;
            double k[3];
            uint64_t off;
        };
        std::vector<Memo> memo;
        for (uint32_t p = 0; p < G->n_paths; ++p) {
            const uint64_t n = G->path_n_steps[p];
            const uint64_t span = n < 2 ? 1 : n - 1;
            const uint64_t zn = std::min<uint64_t>(span, cfg.zipf_space_max);
            auto it = std::find_if(memo.begin(), memo.end(), [&](const Memo& m) { return m.zn == zn; });
            if (it == memo.end()) {
                Memo m{zn, {0, 0, 0}, tables.size()};
                zipf_constants(zn, cfg.zipf_theta, &m.k[0], &m.k[1], &m.k[2]);
                if (!replay) append_zipf_alias(zn, cfg.zipf_theta, tables);
                memo.push_back(m);
                it = memo.end() - 1;
            }
            pcs[p] = PathConst{base, n, zn, it->k[0], it->k[1], it->k[2], it->off};
            base += n;
        }
        // the support (and alias table) carrying the most steps
        uint64_t best = 0;
        for (const Memo& m : memo) {
            uint64_t steps = 0;
            for (uint32_t p = 0; p < G->n_paths; ++p)
                if (pcs[p].zn == m.zn) steps += pcs[p].n;
            if (steps > best) {
                best = steps;
                zdef_n = static_cast<uint32_t>(m.zn);
                zdef_tab = m.off;
            }
        }
    }
    G->pc.alloc(pcs.size());
    PGL_CUDA(copy_async(G->pc.p, pcs.data(), pcs.size() * sizeof(PathConst), cudaMemcpyHostToDevice,
                             G->stream));
    // Path guide with the constants inline, for k_sgd_tiles on graphs with
    // S < 2^30: bucket b of the step index's top bits -> {base, |p|, p | flags}
    // where flag 31 = the bucket straddles a path end (scan PathConst as
    // usual) and flag 30 = the path's Zipf support is zdef: one load resolves
    // the path, its base and length, and whether the speculative alias read
    // applies. ~8 buckets per path, 2^10-2^13 entries of 16 bytes.
    std::vector<uint4> fg;
    {
        const uint64_t S = G->sum.total_steps;
        uint32_t L = 1;
        while ((1ULL << L) < std::max<uint64_t>(S, 2)) ++L;
        uint32_t fb = 10;
        while ((1u << fb) < 8u * std::max<uint32_t>(G->n_paths, 1) && fb < 13) ++fb;
        fb = std::min(fb, L);
        G->fguide_shift = L - fb;
        fg.assign(1u << fb, uint4{0, 0, 1u << 31, 0});
        if (S < (1ULL << 30) && G->n_paths) {
            uint32_t p = 0;
            for (uint64_t b = 0; b < fg.size(); ++b) {
                const uint64_t first = b << G->fguide_shift;
                if (first >= S) break;
                const uint64_t last = std::min<uint64_t>(((b + 1) << G->fguide_shift) - 1, S - 1);
                while (pcs[p].base + pcs[p].n <= first) ++p;
                const bool straddle = pcs[p].base + pcs[p].n <= last;
                const bool zd = pcs[p].zn == zdef_n && pcs[p].ztab == zdef_tab;
                fg[b] = uint4{static_cast<uint32_t>(pcs[p].base), static_cast<uint32_t>(pcs[p].n),
                              p | (straddle ? 1u << 31 : 0u) | (zd ? 1u << 30 : 0u), 0};
            }
        }
        G->fguide.alloc(fg.size());
        PGL_CUDA(copy_async(G->fguide.p, fg.data(), fg.size() * sizeof(uint4), cudaMemcpyHostToDevice,
                                 G->stream));
    }
    G->zalias.alloc(std::max<size_t>(tables.size(), 1));
    if (!tables.empty())
        PGL_CUDA(copy_async(G->zalias.p, tables.data(), tables.size() * sizeof(ZipfAlias),
                                 cudaMemcpyHostToDevice, G->stream));
    PGL_CUDA(cudaMemsetAsync(G->stats.p, 0, 10 * sizeof(unsigned long long), G->stream));

    // RNG states: lane t <- seed_worker(seed, t) (rng.hpp:63-71)
    LaunchShape shape;
    uint32_t n_warps = 1;
    uint64_t lanes = 1;
    const bool lean_ok = cfg.batch_size == 32 && cfg.drf == 1 && !ext.reuse_shuffle &&
                         (ext.pair_window == 0 || ext.pair_window == 1 || ext.pair_window == 3) &&
                         G->sum.total_steps >= 32 &&
                         G->sum.total_steps < (1ULL << 30) && G->sum.max_path_len < (1ULL << 32);
    if (!replay) {
        const uint32_t cap = ext.max_warps ? ext.max_warps : auto_max_warps(V);
        shape = ext.sampling == PGL_SAMPLING_IID
                    ? sgd_shape(G->device, kind, cap, static_cast<int>(ext.block_threads),
                                ext.kernel_variant ? static_cast<int>(ext.kernel_variant) : kIidAutoVariant)
                    : tiles_shape(G->device, kind, cap, static_cast<int>(ext.block_threads),
                                  tile_variant(G->device, ext, cap, lean_ok, V < (1ULL << 31)), G->sum.total_steps);
        const uint64_t grid_warps = static_cast<uint64_t>(shape.blocks) * shape.threads / 32;
        n_warps = static_cast<uint32_t>(std::min<uint64_t>(grid_warps, cap));
        if (ext.unit_order == PGL_ORDER_RANDOM &&
            (ext.sampling != PGL_SAMPLING_TILES || (shape.variant & 15) < 7 || (shape.variant & 15) > 14))
            raise(PGL_ERR_INVALID_PARAMETER, "pgl_layout_ext.unit_order: the random order needs the lean tile kernel "
                                             "(kernel_variant 7 or 8)");
        lanes = static_cast<uint64_t>(shape.blocks) * shape.threads;
    } else {
        lanes = 1;
    }
    G->rng.alloc(4 * std::max<uint64_t>(lanes, 1));
    DevRng rng{G->rng.p, G->rng.p + lanes, G->rng.p + 2 * lanes, G->rng.p + 3 * lanes};
    launch_seed_rng(rng, lanes, cfg.global_seed, G->stream);

    // L2 persistence window on the coordinate array (fits: C1/C2 sizes).
    const size_t coord_bytes = kind == PGL_COORD_F64 ? 4 * V * sizeof(double)
                               : kind == PGL_COORD_F32 ? 4 * V * sizeof(float)
                                                       : anch_bytes(V);
    if (ext.l2_persist && !replay) {
        int max_persist = 0, max_window = 0;
        cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, G->device);
        cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, G->device);
        if (max_persist > 0 && max_window > 0) {
            cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min<size_t>(coord_bytes, max_persist));
            cudaStreamAttrValue attr{};
            attr.accessPolicyWindow.base_ptr = coords;
            attr.accessPolicyWindow.num_bytes = std::min<size_t>(coord_bytes, max_window);
            attr.accessPolicyWindow.hitRatio =
                std::min(1.0f, static_cast<float>(max_persist) / static_cast<float>(std::max<size_t>(coord_bytes, 1)));
            attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
            attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
            cudaStreamSetAttribute(G->stream, cudaStreamAttributeAccessPolicyWindow, &attr);
        }
    }
    PGL_CUDA(cudaStreamSynchronize(G->stream));
    const double init_ms = (now_s() - t_init) * 1e3;

    // Random 16-byte record gathers: fetch exactly one 32-byte sector per L2
    // miss instead of the default promoted line (restored below).
    size_t prev_gran = 0;
    cudaDeviceGetLimit(&prev_gran, cudaLimitMaxL2FetchGranularity);
    if (!replay) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, ext.l2_fetch_bytes ? ext.l2_fetch_bytes : 32);
    const uint64_t spi = 10 * G->sum.total_steps / cfg.srf;  // engine.cpp:197
    if (!replay && ext.sampling == PGL_SAMPLING_TILES && ((shape.variant & 15) == 13 || (shape.variant & 15) == 14) &&
        !G->rec8.p) {
        G->rec8.alloc(G->sum.total_steps + G->n_paths);
        build_rec8_device(G->step.p, G->cum.p, G->n_paths, G->sum.total_steps, G->rec8.p, G->stream);
    }
    const DevGraph dg_ = G->dev();
    // sampler diagnostics of the Hogwild kernels (pgl_layout_diag)
    DevBuf<unsigned int> visits;
    DevBuf<unsigned long long> zhist, outc;
    visits.s = zhist.s = outc.s = G->stream;
    if (ext.diag && !replay) {
        if (ext.diag->primary_visits) {
            visits.alloc(std::max<uint64_t>(G->sum.total_steps, 1));
            PGL_CUDA(cudaMemsetAsync(visits.p, 0, G->sum.total_steps * sizeof(unsigned int), G->stream));
        }
        if (ext.diag->zipf_draws && ext.diag->zipf_draws_len) {
            zhist.alloc(ext.diag->zipf_draws_len);
            PGL_CUDA(cudaMemsetAsync(zhist.p, 0, ext.diag->zipf_draws_len * sizeof(unsigned long long), G->stream));
        }
        outc.alloc(4);
        PGL_CUDA(cudaMemsetAsync(outc.p, 0, 4 * sizeof(unsigned long long), G->stream));
    }
    DevStats* dstats = reinterpret_cast<DevStats*>(G->stats.p);
    std::vector<cudaEvent_t> ev(2 * cfg.n_iters);
    for (auto& e : ev) PGL_CUDA(cudaEventCreate(&e));
    std::vector<double> host_coords;
    bool aborted = false;
    uint32_t iters_run = 0;
    for (uint32_t it = 0; it < cfg.n_iters && !aborted; ++it) {
        ++iters_run;
        const double t_it = now_s();
        IterArgs a;
        a.eta = etas[it];
        a.theta = cfg.zipf_theta;
        a.steps = spi;
        a.force_cooling = 2ULL * it >= static_cast<uint64_t>(cfg.n_iters) ? 1 : 0;  // engine.cpp:202-203
        a.batch = cfg.batch_size;
        a.drf = cfg.drf;
        a.n_warps = n_warps;
        a.units = (spi + 31) / 32;
        const bool lean = !replay && ext.sampling == PGL_SAMPLING_TILES &&
                          ((shape.variant & 15) >= 7 && (shape.variant & 15) <= 14);
        a.units_full = spi / 32;
        a.tail_n = static_cast<uint32_t>(spi % 32);
        {   // unit order of k_sgd_tiles: u = (a*k + b) mod U, gcd(a, U) = 1,
            // a near U/phi (low-discrepancy), jittered per iteration (the lean
            // kernel permutes the full units only)
            HostRng pr(cfg.global_seed, (1ULL << 59) + it);
            const uint64_t U = std::max<uint64_t>(lean ? a.units_full : a.units, 1);
            uint64_t m = static_cast<uint64_t>(static_cast<double>(U) * 0.6180339887498949) + pr.below(U / 16 + 1);
            m %= U;
            if (m == 0) m = 1;
            while (std::gcd(m, U) != 1) m = (m + 1) % U == 0 ? 1 : m + 1;
            a.perm_a = m;
            a.perm_b = pr.below(U);
            a.perm_step = static_cast<uint64_t>((static_cast<unsigned __int128>(m) * n_warps) % U);
            {
                const uint64_t S = G->sum.total_steps;
                a.i0_step = static_cast<uint64_t>((static_cast<unsigned __int128>(a.perm_step) * 32) % S);
                const uint64_t uw = static_cast<uint64_t>((static_cast<unsigned __int128>(U) * 32) % S);
                a.i0_wrap = (a.i0_step + S - uw) % S;
            }
            a.pair_window = ext.pair_window == 1 ? 0 : (ext.pair_window == 2 ? 1 : 3);
            a.record_hint = ext.record_hint;
            // lanes per shared Zipf hop: 8 on the async pipelines; 1 (independent
            // hops) on the register pipeline, which runs small graphs where the
            // cap binds (config 1: SPS ratio 1.008 vs 1.017 with 8,
            // profiles/r02_quality_c1.jsonl)
            const int sv = shape.variant & 15;
            a.hop_lanes = ext.hop_lanes ? ext.hop_lanes : (sv == 1 || sv == 2 ? 1u : kHopLanes);
            a.reuse_shuffle = ext.reuse_shuffle ? 1 : 0;
            a.zdef_n = zdef_n;
            a.zdef_tab = zdef_tab;
            a.fguide = G->fguide.p;
            a.fguide_shift = G->fguide_shift;
            // rotate the enumeration's start every iteration: with srf not
            // dividing 10, N mod S steps get one extra visit per pass
            a.q_off = pr.below(std::max<uint64_t>(G->sum.total_steps, 1));
            a.tail_i0 = (a.units_full * 32 + a.q_off) % std::max<uint64_t>(G->sum.total_steps, 1);
            a.unit_random = ext.unit_order == PGL_ORDER_RANDOM ? 1 : 0;
            a.unit_len = ext.unit_len ? ext.unit_len : 32;
            a.unit_key = pr.next();
            a.visits = visits.p;
            a.zhist = zhist.p;
            a.zhist_len = zhist.p ? ext.diag->zipf_draws_len : 0;
            a.outcomes = outc.p;
        }
        if (kind == PGL_COORD_F32_ANCHORED && it > 0) launch_reanchor(coords, V, G->stream);
        PGL_CUDA(cudaEventRecord(ev[2 * it], G->stream));
        if (replay)
            launch_sgd_replay(dg_, G->coords64.p, G->rng.p, dstats, a, G->stream);
        else if (ext.sampling == PGL_SAMPLING_IID)
            launch_sgd_hogwild(dg_, coords, kind, rng, dstats, a, shape, G->stream);
        else
            launch_sgd_tiles(dg_, coords, kind, rng, dstats, a, shape, G->stream);
        PGL_CUDA(cudaEventRecord(ev[2 * it + 1], G->stream));
        if (cb) {  // IterationCallback at the boundary (engine.cpp:223-229)
            const double* cptr = nullptr;
            if (cb_wants_coords) {
                host_coords.resize(4 * V);
                to_f64(G, kind);
                PGL_CUDA(copy_async(host_coords.data(), G->coords64.p, 4 * V * sizeof(double),
                                         cudaMemcpyDeviceToHost, G->stream));
                cptr = host_coords.data();
            }
            PGL_CUDA(cudaStreamSynchronize(G->stream));
            if (cb(it, cptr, a.eta, now_s() - t_it, user) != 0) aborted = true;
        }
    }
    PGL_CUDA(cudaEventRecord(ev_end, G->stream));
    // Layout::all_finite (layout.cpp:9-18) of the result, on the device:
    // stats[8] = nodes with a non-finite coordinate, stats[9] = the first one
    launch_count_nonfinite(coords, kind, V, G->stats.p + 8, G->stream);
    PGL_CUDA(cudaStreamSynchronize(G->stream));
    G->layout_f64 = kind;
    {
        float dms = 0.f;
        cudaEventElapsedTime(&dms, ev_begin, ev_end);
        G->timing.device_ms = dms;
        cudaEventDestroy(ev_begin);
        cudaEventDestroy(ev_end);
    }
    double kms = 0.0;
    uint32_t launches = 0;
    for (uint32_t it = 0; it < iters_run; ++it) {
        float ms = 0.f;
        PGL_CUDA(cudaEventElapsedTime(&ms, ev[2 * it], ev[2 * it + 1]));
        kms += ms;
        ++launches;
    }
    for (auto& e : ev) cudaEventDestroy(e);
    if (!replay && prev_gran) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, prev_gran);
    if (aborted) raise(PGL_ERR_CALLBACK, "iteration callback requested abort");

    unsigned long long dst[10];
    PGL_CUDA(copy_sync(dst, G->stats.p, sizeof dst, cudaMemcpyDeviceToHost));
    G->timing.coord_kind = static_cast<uint32_t>(kind);
    G->timing.nonfinite_nodes = static_cast<uint32_t>(std::min<unsigned long long>(dst[8], 0xFFFFFFFFull));
    if (dst[8])
        raise(PGL_ERR_NON_FINITE_COORDINATE, "node " + std::to_string(dst[9]) +
                                                 " has a non-finite coordinate after the layout (" +
                                                 std::to_string(dst[8]) + " nodes; device all_finite check)");
    if (stats_out) {
        // every field is a device count (DevStats); tests hold them to the
        // reference's identities (test_engine.cpp:257-278)
        pgl_run_stats st{};
        st.primary_steps = dst[0];
        st.updates_attempted = dst[1];
        st.updates_applied = dst[2];
        st.updates_skipped = dst[3];
        st.batches_first_half = dst[4];
        st.batches_first_half_cooling = dst[5];
        st.batches_second_half = dst[6];
        st.batches_second_half_cooling = dst[7];
        *stats_out = st;
    }
    if (ext.diag && !replay) {
        if (visits.p)
            PGL_CUDA(copy_async(ext.diag->primary_visits, visits.p, G->sum.total_steps * sizeof(unsigned int),
                                     cudaMemcpyDeviceToHost, G->stream));
        if (zhist.p)
            PGL_CUDA(copy_async(ext.diag->zipf_draws, zhist.p,
                                     ext.diag->zipf_draws_len * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                     G->stream));
        PGL_CUDA(copy_async(ext.diag->outcomes, outc.p, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                 G->stream));
        PGL_CUDA(cudaStreamSynchronize(G->stream));
    }
    if (out_coords) {
        to_f64(G, kind);
        copy_out_staged(out_coords, G->coords64.p, 4 * V * sizeof(double), G->stream);
    }
    if (ext.l2_persist && !replay) {
        cudaStreamAttrValue attr{};
        attr.accessPolicyWindow.num_bytes = 0;
        cudaStreamSetAttribute(G->stream, cudaStreamAttributeAccessPolicyWindow, &attr);
        cudaCtxResetPersistingL2Cache();
    }
    G->timing.kernel_ms = kms;
    G->timing.launches = launches;
    G->timing.init_ms = init_ms;
    G->timing.grid_blocks = replay ? 1 : static_cast<uint32_t>(shape.blocks);
    G->timing.block_threads = replay ? 1 : static_cast<uint32_t>(shape.threads);
    G->timing.device_threads = replay ? 1 : static_cast<uint64_t>(n_warps) * 32;
    G->timing.kernel_variant = replay || ext.sampling != PGL_SAMPLING_TILES ? 0u : static_cast<uint32_t>(shape.variant & 15);
    G->timing.total_ms = (now_s() - t_call) * 1e3;
}

void graph_stress(pgl_graph* G, const double* coords, uint64_t seed, uint32_t spn, uint32_t method,
                  pgl_stress_report* out, double* kernel_ms) {
    if (spn < 1) raise(PGL_ERR_INVALID_PARAMETER, "samples_per_node must be >= 1");
    if (!out) raise(PGL_ERR_INVALID_PARAMETER, "report is null");
    DeviceGuard dg(G->device);
    const uint64_t V = G->n_nodes;
    const void* dc;
    int f64;
    if (coords) {
        G->coords64.alloc(4 * V);
        PGL_CUDA(copy_async(G->coords64.p, coords, 4 * V * sizeof(double), cudaMemcpyHostToDevice, G->stream));
        dc = G->coords64.p;
        f64 = PGL_COORD_F64;
        G->layout_f64 = -1;  // the resident layout is overwritten
    } else {
        if (G->layout_f64 < 0) raise(PGL_ERR_INVALID_PARAMETER, "no resident layout: run pgl_graph_layout first");
        f64 = G->layout_f64;  // pgl_coord_precision of the resident layout
        dc = resident_coords(G, f64);
    }
    std::memset(out, 0, sizeof *out);
    if (method == PGL_SPS_COUNTER)
        run_sps_counter(G->dev(), dc, f64, G->path_n_steps.data(), seed, spn, G->sps, out, kernel_ms, G->stream);
    else if (method == PGL_SPS_STREAM)
        run_sps_stream(G->dev(), dc, f64, seed, spn, out, kernel_ms, G->stream);
    else
        raise(PGL_ERR_INVALID_PARAMETER, "unknown sampled stress method");
}

void graph_exact_stress(pgl_graph* G, const double* coords, pgl_stress_report* out, double* kernel_ms) {
    if (!out) raise(PGL_ERR_INVALID_PARAMETER, "report is null");
    DeviceGuard dg(G->device);
    const uint64_t V = G->n_nodes;
    if (coords) {
        G->coords64.alloc(4 * V);
        PGL_CUDA(copy_async(G->coords64.p, coords, 4 * V * sizeof(double), cudaMemcpyHostToDevice, G->stream));
        G->layout_f64 = -1;  // the resident layout is overwritten
    } else {
        if (G->layout_f64 < 0) raise(PGL_ERR_INVALID_PARAMETER, "no resident layout: run pgl_graph_layout first");
        to_f64(G, G->layout_f64);
    }
    std::memset(out, 0, sizeof *out);
    double ssd = 0.0;
    run_exact_stress(G->dev(), G->coords64.p, out, &ssd, kernel_ms, G->stream);
    finish_report(out, ssd);  // metrics.cpp:14-23
}

// ---- synthetic fixture (synthetic.cpp:24-120, walks only) ----------------------

struct Synthetic {
    std::vector<uint64_t> node_len;
    std::vector<std::vector<pgl_path_step>> paths;
    std::vector<const pgl_path_step*> ptrs;
    std::vector<uint64_t> n_steps, totals;
};

Synthetic* generate(uint64_t seed, uint64_t B, uint32_t n_paths, double rate) {
    if (B < 2) raise(PGL_ERR_INVALID_PARAMETER, "backbone needs at least 2 nodes");
    if (n_paths < 1) raise(PGL_ERR_INVALID_PARAMETER, "need at least one path");
    if (!(rate >= 0.0 && rate <= 1.0)) raise(PGL_ERR_INVALID_PARAMETER, "variant_rate must lie in [0, 1]");
    enum : uint8_t { SNV = 0, INS = 1, DEL = 2, NONE = 3 };
    HostRng r(seed, kStreamSynth);
    std::vector<uint8_t> bb_len(B), kind(B, NONE), alt_len(B, 0);
    for (uint64_t b = 0; b < B; ++b) bb_len[b] = static_cast<uint8_t>(8 + r.below(25));
    for (uint64_t b = 0; b < B; ++b) {
        if (r.uniform() >= rate) continue;
        uint8_t feas[3];
        uint64_t nf = 0;
        if (b + 3 <= B) feas[nf++] = SNV;
        if (b + 2 <= B) feas[nf++] = INS;
        if (b + 3 <= B) feas[nf++] = DEL;
        if (nf == 0) continue;
        kind[b] = feas[r.below(nf)];
        if (kind[b] != DEL) alt_len[b] = static_cast<uint8_t>(8 + r.below(25));
    }
    auto S = std::make_unique<Synthetic>();
    std::vector<uint32_t> bb_id(B), alt_id(B, 0);
    S->node_len.reserve(B + B / 8);
    for (uint64_t b = 0; b < B; ++b) {
        bb_id[b] = static_cast<uint32_t>(S->node_len.size());
        S->node_len.push_back(bb_len[b]);
        if (kind[b] == INS) {
            alt_id[b] = static_cast<uint32_t>(S->node_len.size());
            S->node_len.push_back(alt_len[b]);
        }
        if (b >= 1 && kind[b - 1] == SNV) {
            alt_id[b - 1] = static_cast<uint32_t>(S->node_len.size());
            S->node_len.push_back(alt_len[b - 1]);
        }
    }
    if (S->node_len.size() >= (1ULL << 32)) raise(PGL_ERR_INVALID_PARAMETER, "too many nodes");
    S->paths.resize(n_paths);
    for (uint32_t p = 0; p < n_paths; ++p) {
        auto& steps = S->paths[p];
        steps.reserve(B + B / 16);
        uint64_t off = 0;
        auto push = [&](uint32_t id) {
            const uint32_t len = static_cast<uint32_t>(S->node_len[id]);
            steps.push_back(pgl_path_step{off, id, len, 0, {}});
            off += len;
        };
        uint64_t b = 0;
        while (b < B) {
            push(bb_id[b]);
            if (kind[b] != NONE && r.coin()) {
                if (kind[b] == SNV) {
                    push(alt_id[b]);
                    b += 2;
                } else if (kind[b] == INS) {
                    push(alt_id[b]);
                    b += 1;
                } else {
                    b += 2;
                }
                continue;
            }
            b += 1;
        }
        S->totals.push_back(off);
        S->n_steps.push_back(steps.size());
        S->ptrs.push_back(steps.data());
    }
    return S.release();
}

// ---- config 5 fixture: nested bubbles, inversions, duplications ----------------
// A deterministic high-complexity generator (not in the
// reference, whose generator only makes SNV/indel bubbles). A backbone of B
// nodes (lengths U[8, 32]) carries site records; each site spans [a, b) and
// is one of
//   substitution: an alternative branch of fresh nodes that is itself a
//                 backbone with its own sites (nesting up to `depth` levels);
//   inversion:    the span's nodes visited in reverse order and orientation;
//   deletion:     the span skipped;
//   duplication:  the span visited twice (node revisits within a path).
// Every path walks the top backbone; at each site it takes the alternative
// with the site's allele frequency (per path, per site draw). The result is
// plain build_graph input (node lengths + oriented walks), so the reference
// and the oracle can be handed the identical graph.
struct NestedSite {
    uint64_t a, b;        // span [a, b) on the level's backbone
    uint8_t kind;         // 0 sub, 1 inv, 2 del, 3 dup
    double freq;
    int32_t child = -1;   // substitution: index of the alternative level
};
struct NestedLevel {
    std::vector<uint32_t> nodes;   // the level's backbone node ids
    std::vector<int32_t> site_at;  // site starting at backbone position, -1 none
    std::vector<NestedSite> sites;
};

Synthetic* generate_nested(uint64_t seed, uint64_t B, uint32_t n_paths, uint32_t depth, double rate) {
    if (B < 2) raise(PGL_ERR_INVALID_PARAMETER, "backbone needs at least 2 nodes");
    if (n_paths < 1) raise(PGL_ERR_INVALID_PARAMETER, "need at least one path");
    if (!(rate >= 0.0 && rate <= 0.5)) raise(PGL_ERR_INVALID_PARAMETER, "site rate must lie in [0, 0.5]");
    auto S = std::make_unique<Synthetic>();
    HostRng r(seed, kStreamSynth + 5);
    std::vector<NestedLevel> levels;
    auto new_node = [&]() {
        S->node_len.push_back(8 + r.below(25));
        return static_cast<uint32_t>(S->node_len.size() - 1);
    };
    // build a level of length L at nesting depth d; returns its index
    std::function<int32_t(uint64_t, uint32_t)> build = [&](uint64_t L, uint32_t d) -> int32_t {
        const int32_t id = static_cast<int32_t>(levels.size());
        levels.emplace_back();
        std::vector<uint32_t> nodes(L);
        for (auto& n : nodes) n = new_node();
        std::vector<int32_t> site_at(L, -1);
        std::vector<NestedSite> sites;
        for (uint64_t x = 0; x + 1 < L;) {
            if (r.uniform() >= rate) {
                ++x;
                continue;
            }
            const uint64_t span = 1 + r.below(std::min<uint64_t>(L - x, d == 0 ? 64 : 16));
            NestedSite st;
            st.a = x;
            st.b = x + span;
            const uint64_t k = r.below(d + 1 < depth ? 4 : 3);  // deepest level: no substitutions
            st.kind = static_cast<uint8_t>(k == 3 ? 0 : k + 1);
            st.freq = 0.05 + 0.9 * r.uniform();
            site_at[x] = static_cast<int32_t>(sites.size());
            sites.push_back(st);
            x = st.b;
        }
        for (auto& st : sites)
            if (st.kind == 0) st.child = build(std::max<uint64_t>(1, (st.b - st.a) + r.below(8)), d + 1);
        levels[id].nodes = std::move(nodes);
        levels[id].site_at = std::move(site_at);
        levels[id].sites = std::move(sites);
        return id;
    };
    build(B, 0);
    if (S->node_len.size() >= (1ULL << 32)) raise(PGL_ERR_INVALID_PARAMETER, "too many nodes");
    S->paths.resize(n_paths);
    for (uint32_t p = 0; p < n_paths; ++p) {
        auto& steps = S->paths[p];
        steps.reserve(B + B / 8);
        uint64_t off = 0;
        HostRng pr(seed ^ 0x5EED5EEDULL, kStreamSynth + 6 + p);
        auto push = [&](uint32_t id, uint8_t rev) {
            const uint32_t len = static_cast<uint32_t>(S->node_len[id]);
            steps.push_back(pgl_path_step{off, id, len, rev, {}});
            off += len;
        };
        std::function<void(int32_t)> walk = [&](int32_t lv) {
            const NestedLevel& L = levels[lv];
            uint64_t x = 0;
            while (x < L.nodes.size()) {
                const int32_t si = L.site_at[x];
                if (si >= 0 && pr.uniform() < L.sites[si].freq) {
                    const NestedSite& st = L.sites[si];
                    switch (st.kind) {
                        case 0: walk(st.child); break;
                        case 1:
                            for (uint64_t y = st.b; y-- > st.a;) push(L.nodes[y], 1);
                            break;
                        case 2: break;
                        default:
                            for (int rep = 0; rep < 2; ++rep)
                                for (uint64_t y = st.a; y < st.b; ++y) push(L.nodes[y], 0);
                    }
                    x = st.b;
                    continue;
                }
                push(L.nodes[x], 0);
                ++x;
            }
        };
        walk(0);
        if (steps.empty()) push(levels[0].nodes[0], 0);
        S->totals.push_back(off);
        S->n_steps.push_back(steps.size());
        S->ptrs.push_back(steps.data());
    }
    return S.release();
}

}  // namespace

struct pgl_synthetic : Synthetic {};

namespace pgl {
std::atomic<uint64_t> g_h2d_bytes{0}, g_d2h_bytes{0};
void count_copy(cudaMemcpyKind kind, size_t bytes) {
    if (kind == cudaMemcpyHostToDevice)
        g_h2d_bytes.fetch_add(bytes, std::memory_order_relaxed);
    else if (kind == cudaMemcpyDeviceToHost)
        g_d2h_bytes.fetch_add(bytes, std::memory_order_relaxed);
}
}  // namespace pgl

// ---- C ABI -----------------------------------------------------------------------

extern "C" {

const char* pgl_last_error(void) { return t_err.c_str(); }
int pgl_last_error_type(void) { return t_err_type; }
int pgl_abi_version(void) { return PGL_ABI_VERSION; }

int pgl_transfer_bytes(uint64_t* h2d, uint64_t* d2h) {
    if (h2d) *h2d = g_h2d_bytes.load(std::memory_order_relaxed);
    if (d2h) *d2h = g_d2h_bytes.load(std::memory_order_relaxed);
    return PGL_OK;
}

int pgl_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

void pgl_layout_config_default(pgl_layout_config* c) {  // engine.hpp:13-23
    std::memset(c, 0, sizeof *c);
    c->global_seed = 42;
    c->n_iters = 30;
    c->threads = 1;
    c->batch_size = 32;
    c->zipf_theta = 0.99;
    c->zipf_space_max = 1000;
    c->eta_min_eps = 0.01;
    c->drf = 1;
    c->srf = 1;
}

void pgl_layout_ext_default(pgl_layout_ext* e) {
    std::memset(e, 0, sizeof *e);
    e->struct_size = sizeof(pgl_layout_ext);
    e->mode = PGL_MODE_HOGWILD;
    e->coord_precision = PGL_COORD_AUTO;
    e->sampling = PGL_SAMPLING_AUTO;
}

int pgl_graph_create(int device, const pgl_graph_view* v, pgl_graph** out) {
    return guarded([&] {
        if (!out) raise(PGL_ERR_INVALID_PARAMETER, "out is null");
        *out = create_graph(device, v);
    });
}

int pgl_graph_destroy(pgl_graph* g) {
    return guarded([&] {
        if (!g) return;
        DeviceGuard dg(g->device);
        delete g;
    });
}

int pgl_graph_info_get(const pgl_graph* g, pgl_graph_info* out) {
    return guarded([&] {
        if (!g || !out) raise(PGL_ERR_INVALID_PARAMETER, "null argument");
        std::memset(out, 0, sizeof *out);
        out->n_nodes = g->n_nodes;
        out->n_paths = g->n_paths;
        out->device = static_cast<uint32_t>(g->device);
        out->total_steps = g->sum.total_steps;
        out->total_nucleotides = g->sum.total_nt;
        out->max_path_len = g->sum.max_path_len;
        out->device_bytes = g->step.n * sizeof(StepRec) + g->cum.n * 8 + g->guide.n * 4 + g->pc.n * sizeof(PathConst) +
                            g->coords64.n * 8 + g->coords32.n * 4 + g->rng.n * 8;
        out->usable = g->sum.usable ? 1 : 0;
    });
}

int pgl_graph_export_index(const pgl_graph* g, uint64_t* positions, uint32_t* nodes, uint64_t* cum) {
    return guarded([&] {
        if (!g) raise(PGL_ERR_INVALID_PARAMETER, "graph is null");
        DeviceGuard dg(g->device);
        const uint64_t S = g->sum.total_steps;
        std::vector<StepRec> recs(S);
        if (S) PGL_CUDA(copy_sync(recs.data(), g->step.p, S * sizeof(StepRec), cudaMemcpyDeviceToHost));
        for (uint64_t k = 0; k < S; ++k) {
            const StepRec& r = recs[k];
            if (positions) {
                positions[2 * k] = static_cast<uint64_t>(r.ps_lo) | (static_cast<uint64_t>(r.hi & 0xFFFFu) << 32);
                positions[2 * k + 1] = static_cast<uint64_t>(r.pe_lo) | (static_cast<uint64_t>(r.hi >> 16) << 32);
            }
            if (nodes) nodes[k] = r.node;
        }
        if (cum) PGL_CUDA(copy_sync(cum, g->cum.p, (g->n_paths + 1) * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    });
}

int pgl_graph_layout(pgl_graph* g, const pgl_layout_config* cfg, const pgl_layout_ext* ext, int reuse,
                     pgl_iteration_cb cb, int cb_wants_coords, void* user, double* out_coords,
                     pgl_run_stats* stats) {
    return guarded([&] {
        if (!g) raise(PGL_ERR_INVALID_PARAMETER, "graph is null");
        graph_layout(g, cfg, ext, reuse, cb, cb_wants_coords, user, out_coords, stats, nullptr);
    });
}

int pgl_graph_last_timing(const pgl_graph* g, pgl_timing* out) {
    return guarded([&] {
        if (!g || !out) raise(PGL_ERR_INVALID_PARAMETER, "null argument");
        *out = g->timing;
    });
}

int pgl_layout_run(int device, const pgl_graph_view* v, const pgl_layout_config* cfg, const pgl_layout_ext* ext,
                   int reuse, pgl_iteration_cb cb, int cb_wants_coords, void* user, double* out_coords,
                   pgl_run_stats* stats) {
    return guarded([&] {
        // Validate before touching the device, in the reference's order
        // (engine.cpp:176-179; reuse checks first, engine.cpp:330-332).
        if (!cfg) raise(PGL_ERR_INVALID_PARAMETER, "config is null");
        if (reuse) {
            if (cfg->drf != 2 && cfg->drf != 4) raise(PGL_ERR_INVALID_PARAMETER, "update reuse needs drf of 2 or 4");
            if (cfg->srf < 1) raise(PGL_ERR_INVALID_PARAMETER, "srf must be >= 1");
        }
        validate_config(*cfg);
        const ViewSummary s = summarize(v);
        if (v->n_paths == 0 || !s.usable)
            raise(PGL_ERR_DEGENERATE_GRAPH, "layout needs at least one path with two or more steps");
        // init_layout (host, sequential RNG, bit-exact) runs on its own
        // thread while the graph is packed and uploaded; it needs only the
        // node lengths and the seed
        PinnedBuf init;
        init.alloc(std::max<uint64_t>(4 * v->n_nodes, 1) * sizeof(double));
        std::thread init_thread(
            [&] { init_layout(v, s.total_nt, cfg->global_seed, static_cast<double*>(init.p)); });
        std::unique_ptr<pgl_graph> G;
        try {
            G.reset(create_graph(device, v));
        } catch (...) {
            init_thread.join();
            throw;
        }
        init_thread.join();
        graph_layout(G.get(), cfg, ext, reuse, cb, cb_wants_coords, user, out_coords, stats,
                     static_cast<const double*>(init.p));
        DeviceGuard dg(device);
        G.reset();
    });
}

int pgl_graph_stress(pgl_graph* g, const double* coords, uint64_t seed, uint32_t spn, uint32_t method,
                     pgl_stress_report* out, double* kernel_ms) {
    return guarded([&] {
        if (!g) raise(PGL_ERR_INVALID_PARAMETER, "graph is null");
        graph_stress(g, coords, seed, spn, method, out, kernel_ms);
    });
}

int pgl_graph_all_finite(pgl_graph* g, const double* coords, uint64_t* bad_nodes, uint64_t* first_bad) {
    return guarded([&] {
        if (!g) raise(PGL_ERR_INVALID_PARAMETER, "graph is null");
        DeviceGuard dg(g->device);
        const uint64_t V = g->n_nodes;
        const void* dc;
        int kind;
        if (coords) {
            g->coords64.alloc(4 * V);
            PGL_CUDA(copy_async(g->coords64.p, coords, 4 * V * sizeof(double), cudaMemcpyHostToDevice, g->stream));
            dc = g->coords64.p;
            kind = PGL_COORD_F64;
            g->layout_f64 = -1;  // the resident layout is overwritten
        } else {
            if (g->layout_f64 < 0) raise(PGL_ERR_INVALID_PARAMETER, "no resident layout: run pgl_graph_layout first");
            kind = g->layout_f64;
            dc = resident_coords(g, kind);
        }
        launch_count_nonfinite(dc, kind, V, g->stats.p + 8, g->stream);
        unsigned long long r[2];
        PGL_CUDA(copy_async(r, g->stats.p + 8, sizeof r, cudaMemcpyDeviceToHost, g->stream));
        PGL_CUDA(cudaStreamSynchronize(g->stream));
        if (bad_nodes) *bad_nodes = r[0];
        if (first_bad) *first_bad = r[0] ? r[1] : 0;
    });
}

int pgl_sampled_path_stress(int device, const pgl_graph_view* v, const double* coords, uint64_t seed, uint32_t spn,
                            uint32_t method, pgl_stress_report* out) {
    return guarded([&] {
        if (spn < 1) raise(PGL_ERR_INVALID_PARAMETER, "samples_per_node must be >= 1");
        if (!coords) raise(PGL_ERR_INVALID_PARAMETER, "coords is null");
        std::unique_ptr<pgl_graph> G(create_graph(device, v));
        graph_stress(G.get(), coords, seed, spn, method, out, nullptr);
        DeviceGuard dg(device);
        G.reset();
    });
}

int pgl_graph_exact_stress(pgl_graph* g, const double* coords, pgl_stress_report* out, double* kernel_ms) {
    return guarded([&] {
        if (!g) raise(PGL_ERR_INVALID_PARAMETER, "graph is null");
        graph_exact_stress(g, coords, out, kernel_ms);
    });
}

int pgl_exact_path_stress(int device, const pgl_graph_view* v, const double* coords, pgl_stress_report* out) {
    return guarded([&] {
        if (!coords) raise(PGL_ERR_INVALID_PARAMETER, "coords is null");
        std::unique_ptr<pgl_graph> G(create_graph(device, v));
        graph_exact_stress(G.get(), coords, out, nullptr);
        DeviceGuard dg(device);
        G.reset();
    });
}

struct pgl_gfa {
    pgl::GfaGraph* g;
};

int pgl_graph_create_gfa(int device, const char* path, uint32_t threads, pgl_graph** out) {
    return guarded([&] {
        if (!path || !out) raise(PGL_ERR_INVALID_PARAMETER, "null argument");
        *out = nullptr;
        std::unique_ptr<GfaGraph, void (*)(GfaGraph*)> gf(gfa_parse_file(path, threads, /*compact=*/true), gfa_free);
        *out = create_graph_gfa(device, gf.get());
    });
}

int pgl_gfa_parse_file(const char* path, uint32_t threads, pgl_gfa** out) {
    return guarded([&] {
        if (!path || !out) raise(PGL_ERR_INVALID_PARAMETER, "null argument");
        *out = nullptr;
        GfaGraph* g = gfa_parse_file(path, threads);
        *out = new pgl_gfa{g};
    });
}

int pgl_gfa_parse_buffer(const char* data, uint64_t size, uint32_t threads, pgl_gfa** out) {
    return guarded([&] {
        if ((!data && size) || !out) raise(PGL_ERR_INVALID_PARAMETER, "null argument");
        *out = nullptr;
        GfaGraph* g = gfa_parse_buffer(data ? data : "", size, threads);
        *out = new pgl_gfa{g};
    });
}

int pgl_gfa_info_get(const pgl_gfa* g, pgl_gfa_info* out) {
    return guarded([&] {
        if (!g || !out) raise(PGL_ERR_INVALID_PARAMETER, "null argument");
        gfa_info(g->g, out);
    });
}

int pgl_gfa_view(const pgl_gfa* g, pgl_graph_view* out) {
    return guarded([&] {
        if (!g || !out) raise(PGL_ERR_INVALID_PARAMETER, "null argument");
        gfa_view(g->g, out);
    });
}

int pgl_gfa_edges(const pgl_gfa* g, pgl_edge* out) {
    return guarded([&] {
        if (!g || !out) raise(PGL_ERR_INVALID_PARAMETER, "null argument");
        pgl_gfa_info i;
        gfa_info(g->g, &i);
        std::memcpy(out, gfa_edges(g->g), i.n_edges * sizeof(pgl_edge));
    });
}

const char* pgl_gfa_path_name(const pgl_gfa* g, uint32_t path) { return g ? gfa_path_name(g->g, path) : nullptr; }

int pgl_gfa_free(pgl_gfa* g) {
    if (g) {
        gfa_free(g->g);
        delete g;
    }
    return PGL_OK;
}

int pgl_layout_write_tsv(const char* path, const double* coords, uint64_t n_nodes, uint32_t threads) {
    return guarded([&] {
        if (!path || (!coords && n_nodes)) raise(PGL_ERR_INVALID_PARAMETER, "null argument");
        layout_write_tsv(path, coords, n_nodes, threads);
    });
}

int pgl_layout_read_tsv(const char* path, uint32_t threads, uint64_t* n_nodes, double** coords) {
    return guarded([&] {
        if (!path || !n_nodes || !coords) raise(PGL_ERR_INVALID_PARAMETER, "null argument");
        *coords = nullptr;
        *n_nodes = 0;
        std::vector<double> v = layout_read_tsv(path, threads);
        double* m = static_cast<double*>(std::malloc(std::max<size_t>(v.size(), 1) * sizeof(double)));
        if (!m) throw std::bad_alloc();
        std::memcpy(m, v.data(), v.size() * sizeof(double));
        *coords = m;
        *n_nodes = v.size() / 4;
    });
}

int pgl_layout_format_tsv(const double* coords, uint64_t n_nodes, uint32_t threads, char** text, uint64_t* size) {
    return guarded([&] {
        if ((!coords && n_nodes) || !text || !size) raise(PGL_ERR_INVALID_PARAMETER, "null argument");
        *text = nullptr;
        *size = 0;
        const std::string t = layout_format_tsv(coords, n_nodes, threads);
        char* m = static_cast<char*>(std::malloc(t.size() + 1));
        if (!m) throw std::bad_alloc();
        std::memcpy(m, t.data(), t.size());
        m[t.size()] = 0;
        *text = m;
        *size = t.size();
    });
}

int pgl_layout_parse_tsv(const char* data, uint64_t size, uint32_t threads, uint64_t* n_nodes, double** coords) {
    return guarded([&] {
        if ((!data && size) || !n_nodes || !coords) raise(PGL_ERR_INVALID_PARAMETER, "null argument");
        *coords = nullptr;
        *n_nodes = 0;
        std::vector<double> v = layout_read_tsv_buffer(data ? data : "", size, threads);
        double* m = static_cast<double*>(std::malloc(std::max<size_t>(v.size(), 1) * sizeof(double)));
        if (!m) throw std::bad_alloc();
        std::memcpy(m, v.data(), v.size() * sizeof(double));
        *coords = m;
        *n_nodes = v.size() / 4;
    });
}

void pgl_free(void* p) { std::free(p); }

int pgl_make_schedule(const pgl_graph_view* v, const pgl_layout_config* cfg, double* etas) {
    return guarded([&] {
        if (!cfg || !etas) raise(PGL_ERR_INVALID_PARAMETER, "null argument");
        const ViewSummary s = summarize(v);
        schedule_for(v, s, *cfg, etas);
    });
}

int pgl_init_layout(const pgl_graph_view* v, uint64_t seed, double* out) {
    return guarded([&] {
        if (!v || !out) raise(PGL_ERR_INVALID_PARAMETER, "null argument");
        uint64_t nt = 0;
        for (uint64_t n = 0; n < v->n_nodes; ++n) nt += v->node_len[n];
        init_layout(v, nt, seed, out);
    });
}

int pgl_synthetic_generate(uint64_t seed, uint64_t backbone, uint32_t n_paths, double rate, pgl_synthetic** out) {
    return guarded([&] {
        if (!out) raise(PGL_ERR_INVALID_PARAMETER, "out is null");
        *out = static_cast<pgl_synthetic*>(generate(seed, backbone, n_paths, rate));
    });
}

int pgl_synthetic_generate_nested(uint64_t seed, uint64_t backbone, uint32_t n_paths, uint32_t depth,
                                  double site_rate, pgl_synthetic** out) {
    return guarded([&] {
        if (!out) raise(PGL_ERR_INVALID_PARAMETER, "out is null");
        if (depth < 1 || depth > 8) raise(PGL_ERR_INVALID_PARAMETER, "nesting depth must lie in [1, 8]");
        *out = static_cast<pgl_synthetic*>(generate_nested(seed, backbone, n_paths, depth, site_rate));
    });
}

int pgl_synthetic_view(const pgl_synthetic* s, pgl_graph_view* v) {
    return guarded([&] {
        if (!s || !v) raise(PGL_ERR_INVALID_PARAMETER, "null argument");
        std::memset(v, 0, sizeof *v);
        v->n_nodes = s->node_len.size();
        v->node_len = s->node_len.data();
        v->n_paths = static_cast<uint32_t>(s->paths.size());
        v->path_steps = s->ptrs.data();
        v->path_n_steps = s->n_steps.data();
        v->path_total_len = s->totals.data();
    });
}

int pgl_synthetic_free(pgl_synthetic* s) {
    delete static_cast<Synthetic*>(s);
    return PGL_OK;
}

int pgl_shard_plan(int n_devices, int n_graphs, const pgl_graph_view* const* graphs,
                   const pgl_layout_config* cfgs, int* assignment, double* work, double* device_load) {
    return guarded([&] {
        if (n_devices < 1) raise(PGL_ERR_INVALID_PARAMETER, "need at least one device");
        if (n_graphs < 0 || (n_graphs && (!graphs || !cfgs || !assignment)))
            raise(PGL_ERR_INVALID_PARAMETER, "null graph list");
        // LPT: heaviest graph first onto the least-loaded device;
        // a graph's work is its update count, total_steps * n_iters * drf / srf.
        std::vector<double> w(n_graphs);
        for (int k = 0; k < n_graphs; ++k) {
            const ViewSummary s = summarize(graphs[k]);
            validate_config(cfgs[k]);
            w[k] = static_cast<double>(s.total_steps) * cfgs[k].n_iters * cfgs[k].drf / cfgs[k].srf;
            if (work) work[k] = w[k];
        }
        std::vector<int> order(n_graphs);
        std::iota(order.begin(), order.end(), 0);
        std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return w[a] > w[b]; });
        std::vector<double> load(n_devices, 0.0);
        for (int k : order) {
            const int d = static_cast<int>(std::min_element(load.begin(), load.end()) - load.begin());
            load[d] += w[k];
            assignment[k] = d;
        }
        if (device_load) std::copy(load.begin(), load.end(), device_load);
    });
}

int pgl_layout_shards(int n_devices, const int* devices, int n_graphs, const pgl_graph_view* const* graphs,
                      const pgl_layout_config* cfgs, const pgl_layout_ext* ext, double* const* out_coords,
                      pgl_run_stats* stats, double* seconds, int* assignment) {
    return guarded([&] {
        if (n_devices < 1 || !devices) raise(PGL_ERR_INVALID_PARAMETER, "need at least one device");
        std::vector<int> plan(std::max(n_graphs, 1));
        const int rc = pgl_shard_plan(n_devices, n_graphs, graphs, cfgs, plan.data(), nullptr, nullptr);
        if (rc != PGL_OK) throw Failure(rc, pgl_last_error());
        std::vector<std::vector<int>> queue(n_devices);
        for (int k = 0; k < n_graphs; ++k) {
            queue[plan[k]].push_back(k);
            if (assignment) assignment[k] = plan[k];
        }
        std::vector<std::thread> pool;
        std::vector<std::string> errs(n_devices);
        std::vector<int> err_types(n_devices, 0);
        for (int d = 0; d < n_devices; ++d)
            pool.emplace_back([&, d] {
                try {
                    for (int k : queue[d]) {
                        const double t0 = now_s();
                        std::unique_ptr<pgl_graph> G(create_graph(devices[d], graphs[k]));
                        graph_layout(G.get(), &cfgs[k], ext, 0, nullptr, 0, nullptr,
                                     out_coords ? out_coords[k] : nullptr, stats ? &stats[k] : nullptr, nullptr);
                        {
                            DeviceGuard dg(devices[d]);
                            G.reset();
                        }
                        if (seconds) seconds[k] = now_s() - t0;
                    }
                } catch (const Failure& f) {
                    errs[d] = f.what();
                    err_types[d] = f.type;
                } catch (const std::exception& e) {
                    errs[d] = e.what();
                    err_types[d] = PGL_ERR_CUDA;
                }
            });
        for (auto& t : pool) t.join();
        for (int d = 0; d < n_devices; ++d)
            if (err_types[d]) throw Failure(err_types[d], errs[d]);
    });
}

}  // extern "C"
