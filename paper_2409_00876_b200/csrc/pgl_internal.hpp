// pgl_internal.hpp — declarations shared by the host driver (pgl_host.cpp)
// and the sm_100a kernels (pgl_sgd.cu, pgl_sps.cu). Not part of the ABI.
#pragma once

#include <cstdint>
#include <cuda_runtime_api.h>
#include <vector_types.h>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/pgl_b200.h"

namespace pgl {

// Typed failure carrying the reference exception class (errors.hpp:31-44).
struct Failure : std::runtime_error {
    int type;
    Failure(int t, const std::string& m) : std::runtime_error(m), type(t) {}
};

[[noreturn]] void raise(int type, const std::string& detail);
[[noreturn]] void raise_cuda(int err, const char* what, const char* file, int line);

// Host <-> device copies go through these so the library can report the
// bytes it moved (pgl_transfer_bytes: the e2e bench counts them, it does not
// estimate them).
void count_copy(cudaMemcpyKind kind, size_t bytes);
inline cudaError_t copy_async(void* dst, const void* src, size_t n, cudaMemcpyKind kind, cudaStream_t s) {
    count_copy(kind, n);
    return cudaMemcpyAsync(dst, src, n, kind, s);
}
inline cudaError_t copy_sync(void* dst, const void* src, size_t n, cudaMemcpyKind kind) {
    count_copy(kind, n);
    return cudaMemcpy(dst, src, n, kind);
}

#define PGL_CUDA(call)                                                         \
    do {                                                                       \
        const int pgl_e_ = static_cast<int>(call);                             \
        if (pgl_e_ != 0) ::pgl::raise_cuda(pgl_e_, #call, __FILE__, __LINE__); \
    } while (0)

// ---- device-side data layout --------

// One path step, 16 bytes = half a 32-byte sector, 16-byte aligned so a
// random gather touches exactly one sector. The orientation is folded into
// the two endpoint positions (path_position, graph.hpp:98-109):
//   x = node id
//   y = low 32 bits of pos(start endpoint)   z = low 32 bits of pos(end endpoint)
//   w = (pos_start >> 32) | (pos_end >> 32) << 16     (positions < 2^48)
struct alignas(16) StepRec {
    uint32_t node, ps_lo, pe_lo, hi;
};

// Per-path constants, 48 bytes: step range, Zipf support and the rejection-
// inversion constants of ZipfSampler (rng.hpp:95-97) computed on the host
// with the same libm as the reference.
struct alignas(16) PathConst {
    uint64_t base;    // cum_steps[p]
    uint64_t n;       // |p|
    uint64_t zn;      // Zipf support n = min(max(|p|-1,1), zipf_space_max)
    double hx1, hxn, s;
    uint64_t ztab;    // offset of this support's alias table in DevGraph::zalias
};

// Walker/Vose alias table entry for Zipf(zn, theta) on [1, zn]: column c is
// kept when the 32-bit threshold test passes, else replaced by alias.
struct ZipfAlias {
    uint32_t thresh;  // P(keep column) * 2^32 (saturating)
    uint32_t alias;   // 0-based alternative column
};

// Anchored FP32 coordinate store (PGL_COORD_F32_ANCHORED): nodes in blocks
// of 32, one f64 anchor per block. The allocation is [anchors of blocks
// nb-1 .. 0, 8 B each, padded to 256 B][32*nb float4 {sx,sy,ex,ey}]; kernels
// get the base = the first node: node n at base + 16 n (one IMAD.WIDE),
// the anchor of block b at base - 8 (b + 1).
inline uint64_t anch_anchor_bytes(uint64_t n_nodes) { return (((n_nodes + 31) / 32) * 8 + 255) & ~uint64_t{255}; }
inline uint64_t anch_bytes(uint64_t n_nodes) { return anch_anchor_bytes(n_nodes) + ((n_nodes + 31) / 32) * 512; }
inline void* anch_base(void* alloc, uint64_t n_nodes) { return static_cast<char*>(alloc) + anch_anchor_bytes(n_nodes); }

// Everything a kernel needs to read the resident graph.
struct DevGraph {
    const StepRec* step;      // [S]
    const uint64_t* cum;      // [P+1]
    const uint32_t* guide;    // [1 << guide_bits] path of the bucket's first pick
    const PathConst* pc;      // [P]
    const ZipfAlias* zalias;  // alias tables, one per distinct Zipf support
    uint64_t total_steps;
    uint32_t n_paths;
    uint32_t guide_bits;
    uint64_t n_nodes;
    const uint32_t* sguide;   // [1 << sguide_bits] path of step (b << sguide_shift)
    uint32_t sguide_shift;
    uint32_t sguide_bits;
    // [S + P] 8-byte step records {node | reverse << 31, offset} with one
    // sentinel {0, total_len} after each path, so step k's two endpoint
    // positions are offset(k) and offset(k + 1) (lean variants 13/14; built
    // on first use, paths < 2^32 nt)
    const uint2* rec8;
};

struct IterArgs {
    double eta;
    double theta;
    uint64_t steps;       // primary steps this iteration (all warps)
    uint32_t force_cooling;
    uint32_t batch;
    uint32_t drf;
    uint32_t n_warps;     // Hogwild workers = resident warps
    // tile sampling (k_sgd_tiles): units of 32 consecutive picks q, step
    // i = q mod S, visited in the order u = (a*k + b) mod U.
    uint64_t units;       // U = ceil(steps / 32)
    uint64_t perm_a;      // multiplier, gcd(a, U) = 1, a < U
    uint64_t perm_b;      // offset < U
    uint64_t perm_step;   // (a * n_warps) mod U
    uint64_t i0_step;     // (32 * perm_step) mod S: first-step advance of a round
    uint64_t i0_wrap;     // (32 * (perm_step - U)) mod S: the same when u wraps
    uint32_t pair_window; // 0 independent partners, 1 shared uniform window, 3 window + shared Zipf hop
    uint32_t record_hint; // 0 = records evict_first in L2, 1 = evict_normal
    uint32_t hop_lanes;   // lanes sharing one Zipf hop (pair_window 3): 1..32, power of two
    uint32_t reuse_shuffle;  // drf > 1 extras by warp-shuffle reuse (paper §7.4) instead of endpoint combos
    uint32_t zdef_n;      // the Zipf support covering the most steps, and its alias-table
    uint64_t zdef_tab;    //   offset: read speculatively by k_sgd_tiles' cooling units
    const uint4* fguide;  // path guide with inline constants (S < 2^30), see graph_layout
    uint32_t fguide_shift;
    uint64_t q_off;       // per-iteration start offset of the enumeration: step i = (q + q_off) mod S,
                          //   so the N mod S extra visits of a pass rotate over the steps
    // sampler diagnostics (pgl_layout_diag), null when off
    unsigned int* visits;            // [S] primary visit counts
    unsigned long long* zhist;       // [zhist_len] Zipf hops drawn
    unsigned long long* outcomes;    // [4] {uniform attempted, applied, cooling attempted, applied}
    uint32_t zhist_len;
    // lean tile kernel (k_sgd_lean): the permutation runs over the full
    // units only, u = (perm_a*k + perm_b) mod units_full; the partial last
    // unit (tail_n picks, first step tail_i0) is k = units_full, the last
    // unit of its warp, so every warp's batches stay aligned to its units
    uint64_t units_full;
    uint32_t tail_n;
    uint64_t tail_i0;
    // PGL_ORDER_RANDOM (lean kernel): unit k starts at step
    // mulhi(splitmix(unit_key, k), S) instead of the permutation's
    uint32_t unit_random;
    uint64_t unit_key;
    uint32_t unit_len;    // lean kernel: consecutive picks per unit (32; 1..16 with unit_random)
};


// Device RNG states, structure of arrays (coalesced): s[k][lane].
struct DevRng {
    uint64_t* s0;
    uint64_t* s1;
    uint64_t* s2;
    uint64_t* s3;
};

// Accumulated on device with warp-aggregated atomics; RunStats order:
// [0] primary steps that reached the update stage, [1] attempted (drf per
// primary step, engine.cpp:125-126), [2] applied, [3] skipped (counted where
// each skip happens: an invalid selection skips drf, a d_ref <= 0 update 1),
// [4..7] batch counters.
struct DevStats {
    unsigned long long v[8];
};

// ---- kernel launchers (pgl_sgd.cu / pgl_sps.cu) ---------------------------

struct LaunchShape {
    int blocks = 0;
    int threads = 256;
    int variant = 0;
    bool idx32 = false;  // tile kernel: 32-bit index instantiation
    size_t smem = 0;     // dynamic shared memory per CTA
};

// Occupancy-derived persistent grid for the Hogwild kernel.
LaunchShape sgd_shape(int device, int coord_f64, uint32_t max_warps, int block_threads, int variant);

void launch_seed_rng(DevRng rng, uint64_t n_lanes, uint64_t seed, void* stream);
void launch_sgd_hogwild(const DevGraph& g, void* coords, int coord_f64, DevRng rng,
                        DevStats* stats, const IterArgs& a, LaunchShape shape,
                        void* stream);
void launch_sgd_tiles(const DevGraph& g, void* coords, int coord_f64, DevRng rng,
                      DevStats* stats, const IterArgs& a, LaunchShape shape, void* stream);
LaunchShape tiles_shape(int device, int coord_f64, uint32_t max_warps, int block_threads, int variant,
                        uint64_t total_steps);
void launch_sgd_replay(const DevGraph& g, double* coords, uint64_t* rng4,
                       DevStats* stats, const IterArgs& a, void* stream);

struct SpsScratch {
    void* part;              // per-chunk moments + chunk prefix per path
    unsigned long long* cnt; // [2]: spare, skipped
    double* scal;            // [4]: total moments (n, mean, M2), spare
    size_t part_bytes;
};
// Counter-based sampled path stress on a resident graph (metrics.cpp:108-159
// estimator). Fills out (mean, n, sd, ci) deterministically.
void run_sps_counter(const DevGraph& g, const void* coords, int coord_kind, const uint64_t* path_n_steps,
                     uint64_t seed, uint32_t spn, SpsScratch& scratch,
                     pgl_stress_report* out, double* kernel_ms, void* stream);
void run_sps_stream(const DevGraph& g, const void* coords, int coord_f64,
                    uint64_t seed, uint32_t spn, pgl_stress_report* out,
                    double* kernel_ms, void* stream);

// Exact path stress (pgl_exact.cu): mean, n, skipped into out; the
// squared-deviation sum into sum_sq_dev (finish_report does the rest).
void run_exact_stress(const DevGraph& g, const double* coords, pgl_stress_report* out, double* sum_sq_dev,
                      double* kernel_ms, void* stream);

// GFA ingest (pgl_gfa.cpp).
struct GfaGraph;
// compact = true keeps only u32 step words (node | reverse << 31) and
// cum_steps (the device builds the step records: pgl_graph_create_gfa)
GfaGraph* gfa_parse_buffer(const char* data, uint64_t size, unsigned threads, bool compact = false);
GfaGraph* gfa_parse_file(const char* path, unsigned threads, bool compact = false);
struct CompactGraph {
    uint64_t n_nodes;
    const uint64_t* node_len;
    uint32_t n_paths;
    const uint64_t* path_begin;  // [P+1]
    const uint64_t* path_total;  // [P]
    const uint32_t* steps;       // [S] node | reverse << 31
};
CompactGraph gfa_compact(const GfaGraph* g);
void gfa_free(GfaGraph* g);
void gfa_view(const GfaGraph* g, pgl_graph_view* v);
void gfa_info(const GfaGraph* g, pgl_gfa_info* out);
const pgl_edge* gfa_edges(const GfaGraph* g);
const char* gfa_path_name(const GfaGraph* g, uint32_t p);

// Layout table IO (pgl_tsv.cpp).
void layout_write_tsv(const char* path, const double* coords, uint64_t n_nodes, uint32_t threads);
std::string layout_format_tsv(const double* coords, uint64_t n_nodes, uint32_t threads);
std::vector<double> layout_read_tsv(const char* path, uint32_t threads);
std::vector<double> layout_read_tsv_buffer(const char* data, uint64_t size, uint32_t threads);

// Step records from compact steps on the device (pgl_pack.cu).
void build_records_device(const uint32_t* d_steps, const uint32_t* d_node_len, const uint64_t* d_cum, uint32_t P,
                          uint64_t S, StepRec* d_out, void* stream);

// Small device helpers used by the host driver.
void launch_f64_to_f32(const double* src, float* dst, uint64_t n, void* stream);
void launch_f64_to_anch(const double* src, void* dst, uint64_t n_nodes, void* stream);
void launch_anch_to_f64(const void* src, double* dst, uint64_t n_nodes, void* stream);
void launch_reanchor(void* store, uint64_t n_nodes, void* stream);
// out[0] = blocks of 32 node ids whose path positions span more than
// max_span_256nt * 256 nt, out[1] = blocks visited by some step
void build_rec8_device(const StepRec* step, const uint64_t* cum, uint32_t P, uint64_t S, uint2* out,
                       cudaStream_t stream);
void block_span_stats(const StepRec* step, uint64_t S, uint64_t n_nodes, uint32_t max_span_256nt,
                      unsigned long long* out, void* stream);
void launch_count_nonfinite(const void* coords, int coord_kind, uint64_t n_nodes, unsigned long long* out,
                            void* stream);
void launch_f32_to_f64(const float* src, double* dst, uint64_t n, void* stream);

// ---- host helpers (pgl_host.cpp) -----------------------------------------

void zipf_constants(uint64_t n, double theta, double* hx1, double* hxn, double* s);
void finish_report(pgl_stress_report* r, double sum_sq_dev);
void append_zipf_alias(uint64_t zn, double theta, std::vector<ZipfAlias>& out);

}  // namespace pgl
