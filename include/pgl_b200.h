/*
 * pgl_b200.h — C-ABI of the B200-native PG-SGD layout hot path.
 *
 * This is the drop-in boundary between the reference's C++ layout API
 * (namespace pglayout, /root/reference/proj/include/pglayout/engine.hpp and
 * metrics.hpp) and libpgl_b200.so (sm_100a CUDA kernels + C++ host driver).
 * No C++ or torch type crosses it: plain structs, pointers and sizes only.
 *
 * Reference interfaces replaced (file:line under /root/reference/proj):
 *   pgl_layout_run              <- pglayout::run_layout        include/pglayout/engine.hpp:80-82, src/engine.cpp:323-326
 *                                  pglayout::run_layout_reuse  include/pglayout/engine.hpp:86-88, src/engine.cpp:328-334
 *   pgl_sampled_path_stress     <- pglayout::sampled_path_stress include/pglayout/metrics.hpp:49-51, src/metrics.cpp:108-159
 *   pgl_exact_path_stress       <- pglayout::exact_path_stress  include/pglayout/metrics.hpp:39, src/metrics.cpp:75-106
 *   pgl_graph_create/_layout/.. <- same two calls, split so the packed graph stays resident in HBM
 *                                  across calls (the reference rebuilds nothing either: PangenomeGraph
 *                                  is immutable, graph.hpp:61-88)
 *   pgl_gfa_parse_file/_buffer  <- pglayout::parse_gfa + build_graph include/pglayout/gfa.hpp:22, src/gfa.cpp:57-153,
 *                                  src/graph.cpp:7-59 (multithreaded; same ids, offsets, errors)
 *   pgl_layout_write_tsv        <- pglayout::write_layout_tsv include/pglayout/layout_io.hpp:13, src/layout_io.cpp:31-46
 *   pgl_layout_read_tsv         <- pglayout::read_layout_tsv  include/pglayout/layout_io.hpp:15, src/layout_io.cpp:48-110
 *   pgl_make_schedule           <- pglayout::make_schedule     include/pglayout/engine.hpp:44, src/engine.cpp:266-274
 *   pgl_init_layout             <- pglayout::init_layout       include/pglayout/layout.hpp:91, src/layout.cpp:20-34
 *   pgl_last_error/_type        <- the typed exceptions of include/pglayout/errors.hpp:10-42
 *
 * Error convention: every function returns a pgl_status equal to the
 * reference ErrorKind + 1 (usage -> 1, input -> 2, internal -> 3; the CLI's
 * exit codes, tools/pglayout_main.cpp:34-41), plus PGL_E_CALLBACK when the
 * caller's iteration callback asked to abort. pgl_last_error() gives the
 * message (thread-local, "TypeName: detail" exactly like errors.hpp:22-27) and
 * pgl_last_error_type() the concrete exception class so a C++ facade can
 * rethrow the identical type.
 *
 * Threading: calls on different devices from different host threads are
 * independent (one CUDA stream per call/graph). This is the multi-GPU
 * scheduler's contract: independent chromosome graphs, no collective.
 */
#ifndef PGL_B200_H
#define PGL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PGL_ABI_VERSION 1

/* ---- status / error types ---------------------------------------------- */

typedef enum pgl_status {
    PGL_OK = 0,
    PGL_E_USAGE = 1,    /* ErrorKind::usage    (errors.hpp:12) */
    PGL_E_INPUT = 2,    /* ErrorKind::input */
    PGL_E_INTERNAL = 3, /* ErrorKind::internal, also every CUDA failure */
    PGL_E_CALLBACK = 4  /* the iteration callback returned nonzero */
} pgl_status;

/* One value per exception class of errors.hpp:31-44, same order. */
typedef enum pgl_error_type {
    PGL_ERR_NONE = 0,
    PGL_ERR_INVALID_PARAMETER = 1,
    PGL_ERR_UNKNOWN_NODE = 2,
    PGL_ERR_EMPTY_PATH = 3,
    PGL_ERR_INDEX_OUT_OF_RANGE = 4,
    PGL_ERR_EMPTY_GRAPH = 5,
    PGL_ERR_DEGENERATE_GRAPH = 6,
    PGL_ERR_MALFORMED_LINE = 7,
    PGL_ERR_UNKNOWN_SEGMENT = 8,
    PGL_ERR_NO_PATHS = 9,
    PGL_ERR_NON_FINITE_COORDINATE = 10,
    PGL_ERR_MALFORMED_ROW = 11,
    PGL_ERR_COUNT_MISMATCH = 12,
    PGL_ERR_ZERO_REFERENCE = 13,
    PGL_ERR_CORPUS_TOO_LARGE = 14,
    PGL_ERR_CUDA = 100,
    PGL_ERR_CALLBACK = 101
} pgl_error_type;

const char* pgl_last_error(void);
int pgl_last_error_type(void);
int pgl_abi_version(void);
/* Number of visible CUDA devices (0 when no GPU / no driver). Never fails. */
int pgl_device_count(void);

/* Bytes the library has copied host -> device and device -> host since it
 * was loaded (every cudaMemcpy it issues, all devices): the e2e bench reads
 * it around its timed calls. */
int pgl_transfer_bytes(uint64_t* h2d, uint64_t* d2h);

/* ---- configuration ------------------------------------------------------ */

/* Field-for-field LayoutConfig (engine.hpp:13-23), same order and defaults.
 * Layout-identical to the C++ struct on LP64 (size 56). */
typedef struct pgl_layout_config {
    uint64_t global_seed;    /* 42 */
    uint32_t n_iters;        /* 30 */
    uint32_t threads;        /* 1; validated >= 1, ignored by the GPU kernel */
    uint32_t batch_size;     /* 32: steps sharing one cooling decision */
    uint32_t _pad0;
    double zipf_theta;       /* 0.99 */
    uint64_t zipf_space_max; /* 1000 */
    double eta_min_eps;      /* 0.01 */
    uint32_t drf;            /* 1, 2 or 4 */
    uint32_t srf;            /* >= 1 */
} pgl_layout_config;

void pgl_layout_config_default(pgl_layout_config* cfg);

/* Execution modes of the device engine. */
typedef enum pgl_mode {
    /* Hogwild PG-SGD over a persistent grid: every warp is one reference
     * worker, lanes run consecutive steps of the warp's share, cooling is
     * decided per batch and is warp-uniform for batch_size % 32 == 0. */
    PGL_MODE_HOGWILD = 0,
    /* One device lane replays the reference's threads=1 run exactly: stream
     * seed_worker(seed, 0), the draw order of engine.cpp:103-172, FP64
     * coordinates. Bit-identical to pglayout::run_layout(threads=1). */
    PGL_MODE_REPLAY = 1
} pgl_mode;

/* How the Hogwild kernel draws the primary step of each update. */
typedef enum pgl_sampling {
    /* The iteration's N = 10*S/srf picks are enumerated, q in [0, N), step
     * q mod S: every step is the primary endpoint exactly N/S times (without
     * replacement); 32 consecutive picks form one warp round whose step
     * records are one coalesced load and whose in-tile partners are shared
     * by __shfl_sync. Partner, coins and update as the reference. */
    PGL_SAMPLING_TILES = 0,
    /* weighted_step_select per pick, i.i.d. (graph.hpp:123-138). */
    PGL_SAMPLING_IID = 1,
    /* default: the tile sampler where the graph fills the GPU (the Hogwild
     * concurrency cap -- one warp per 80 nodes -- allows the lean tile
     * kernel's full residency, 24 warps per SM: >= ~284k nodes on a B200),
     * the i.i.d. kernel where the cap binds (small or dense graphs, e.g.
     * configs 1 and 5: there the tile kernels' correlated updates and longer
     * read-to-write window move the sampled path stress 2-4% off the
     * reference's, the i.i.d. kernel stays within 1%). */
    PGL_SAMPLING_AUTO = 2
} pgl_sampling;

/* Order in which the tile sampler visits its units of 32 picks. */
typedef enum pgl_unit_order {
    PGL_ORDER_AUTO = 0,   /* = PGL_ORDER_SPREAD */
    /* u = (a*k + b) mod U, a ~ U/phi: concurrent warps spread over the whole graph */
    PGL_ORDER_SPREAD = 1,
    /* contiguous sweep fronts: measured no faster once partners are windowed;
     * rejected (InvalidParameter) by this build, the value stays reserved */
    PGL_ORDER_FRONTS = 2,
    /* unit starts drawn i.i.d. uniform over the steps (with replacement), so
     * a step's primary-visit count per iteration spreads like the
     * reference's i.i.d. picks (Poisson-like around 10/srf) instead of being
     * exactly N/S; lean kernel (variants 7/8) only */
    PGL_ORDER_RANDOM = 3
} pgl_unit_order;

typedef enum pgl_coord_precision {
    PGL_COORD_F32 = 0, /* one float4 {sx,sy,ex,ey} per node (16 B); loses
                          local precision once coordinates exceed ~1e7 */
    PGL_COORD_F64 = 1, /* two double2 per node (32 B = one sector); default */
    /* f32 offsets from an FP64 anchor per block of 32 nodes (the block's first
     * start x of the initial layout): 16.5 B per node, with the f32 error
     * relative to a node's displacement from its anchor rather than to its
     * absolute x, which reaches 2e8 at chromosome scale */
    PGL_COORD_F32_ANCHORED = 2,
    /* default: FP64 while the FP64 array (32 B/node) fits comfortably in L2
     * (<= 64 MiB), the anchored store beyond (measured at config 3: +15%
     * updates/s at equal sampled path stress) */
    PGL_COORD_AUTO = 3
} pgl_coord_precision;

/* B200-specific knobs kept out of pgl_layout_config so that struct stays
 * ABI-identical to LayoutConfig. Zero-initialise and set struct_size. */
typedef struct pgl_layout_ext {
    uint32_t struct_size;     /* sizeof(pgl_layout_ext) */
    uint32_t mode;            /* pgl_mode */
    uint32_t coord_precision; /* pgl_coord_precision (default PGL_COORD_AUTO) */
    uint32_t max_warps;       /* 0 = auto concurrency cap (scales with node count) */
    uint32_t block_threads;   /* 0 = default (256) */
    uint32_t l2_persist;      /* 1 = L2 persistence window on the coordinate array */
    uint32_t kernel_variant;  /* tile kernel: 0 = auto (10 for LayoutConfig{}-shaped runs once
                                 the concurrency cap allows full residency, 6 for the general
                                 case, 1 where the cap binds); 1/2 = register pipeline, 2/3
                                 CTAs/SM; 5/6 = cp.async pipeline via shared memory, 4/3
                                 CTAs/SM; 7-12 = the lean kernel (pgl_tiles.cu).
                                 i.i.d. kernel (PGL_SAMPLING_IID): 0 = auto; 8 = two-stage,
                                 2 CTAs/SM; 1-5: bit 0 = 3 CTAs/SM, variant >> 1 = rounds of
                                 step records in flight beyond the current one (depth 2-4);
                                 6/7 = depth 3/4 + next round's endpoints prefetched to L2 */
    uint32_t l2_fetch_bytes;  /* cudaLimitMaxL2FetchGranularity during the layout; 0 = 32 */
    uint32_t sampling;        /* pgl_sampling (Hogwild mode only; default PGL_SAMPLING_AUTO) */
    uint32_t unit_order;      /* pgl_unit_order (tile sampling only) */
    uint32_t front_warps;     /* reserved (was: warps per sweep front) */
    uint32_t pair_window;     /* 0 = auto (= 3), 1 = independent partner draws,
                                 2 = one shared random window per unit (see pgl_tiles.cu),
                                 3 = 2 + one shared Zipf hop per unit in cooling batches */
    uint32_t record_hint;     /* L2 policy of step-record loads: 0 = evict_first, 1 = evict_normal */
    uint32_t hop_lanes;       /* lanes sharing one Zipf hop (pair_window 3); 0 = auto (8) */
    uint32_t reuse_shuffle;   /* drf > 1: 0 = the reference's re-update of the same step pair
                                 under unused endpoint combinations (engine.cpp:147-170);
                                 1 = warp-level data reuse (paper §7.4): extra updates pair
                                 this lane's i with another lane's partner, from registers */
    uint32_t unit_len;        /* lean tile kernel (variants 7/8): consecutive picks per unit, a
                                 power of two; 0 = auto (32). Below 32 needs PGL_ORDER_RANDOM:
                                 each group of unit_len lanes takes its own i.i.d. start, and
                                 unit_len 1 with pair_window 1 draws every primary step i.i.d.
                                 uniform and every partner independently -- the reference's
                                 selection distribution (weighted_step_select,
                                 select_step_pair) on the lean pipeline */
    struct pgl_layout_diag* diag; /* sampler diagnostics (Hogwild modes), NULL = off */
} pgl_layout_ext;

/* Sampler diagnostics, counted inside the Hogwild kernels while they run
 * (they cost a few atomics per update, so measurements leave them off).
 * Every member is optional. */
typedef struct pgl_layout_diag {
    uint32_t* primary_visits; /* host [total_steps]: how often each step was the primary step i,
                                 summed over the run (the reference draws i i.i.d.,
                                 graph.hpp:123-138; the tile sampler enumerates) */
    uint64_t* zipf_draws;     /* host [zipf_draws_len]: histogram of the Zipf hops k drawn by
                                 cooling selections (one count per draw, k >= len in the last
                                 cell; ZipfSampler, rng.hpp:103-117) */
    uint32_t zipf_draws_len;
    uint32_t _pad;
    uint64_t outcomes[4];     /* out: primary updates {uniform attempted, uniform applied,
                                 cooling attempted, cooling applied} (the selection rules of
                                 select_step_pair + apply_endpoint_update, test_engine.cpp:210-240) */
} pgl_layout_diag;

void pgl_layout_ext_default(pgl_layout_ext* ext);

/* ---- graph view (host memory, borrowed) --------------------------------- */

/* Layout-identical to pglayout::PathStep (graph.hpp:35-41): 24 bytes,
 * offset @0, node_id @8, seq_len @12, orient @16 (0 = forward, 1 = reverse). */
typedef struct pgl_path_step {
    uint64_t offset;
    uint32_t node_id;
    uint32_t seq_len;
    uint8_t orient;
    uint8_t _pad[7];
} pgl_path_step;

/* A borrowed view of a built PangenomeGraph (graph.hpp:61-88). The facade
 * fills path_steps[k] = g.paths[k].steps.data() — zero copy. */
typedef struct pgl_graph_view {
    uint64_t n_nodes;
    const uint64_t* node_len;               /* [n_nodes] NodeRecord::seq_len */
    uint32_t n_paths;
    uint32_t _pad0;
    const pgl_path_step* const* path_steps; /* [n_paths] */
    const uint64_t* path_n_steps;           /* [n_paths] Path::steps.size() */
    const uint64_t* path_total_len;         /* [n_paths] Path::total_len */
} pgl_graph_view;

/* RunStats (engine.hpp:61-70), same field order. */
typedef struct pgl_run_stats {
    uint64_t primary_steps;
    uint64_t updates_attempted;
    uint64_t updates_applied;
    uint64_t updates_skipped;
    uint64_t batches_first_half;
    uint64_t batches_first_half_cooling;
    uint64_t batches_second_half;
    uint64_t batches_second_half_cooling;
} pgl_run_stats;

/* StressReport (metrics.hpp:13-20), same field order. */
typedef struct pgl_stress_report {
    double mean;
    uint64_t n;
    double std_dev;
    double ci_low;
    double ci_high;
    uint64_t skipped;
} pgl_stress_report;

/* IterationCallback (engine.hpp:72-74). `coords` is [4*n_nodes] doubles in
 * Layout::snapshot order (sx,sy,ex,ey per node, layout.hpp:58-68) when the
 * caller asked for them, else NULL. Valid only during the call. Return 0 to
 * continue; nonzero aborts the run with PGL_E_CALLBACK. */
typedef int (*pgl_iteration_cb)(uint32_t iter, const double* coords, double eta,
                                double seconds, void* user);

/* ---- one-shot layout: the drop-in for run_layout / run_layout_reuse ----- */

/* reuse = 0: run_layout semantics; reuse = 1: run_layout_reuse (drf in {2,4}).
 * out_coords: [4*n_nodes] doubles (snapshot order). stats may be NULL. ext may be NULL. */
int pgl_layout_run(int device, const pgl_graph_view* graph,
                   const pgl_layout_config* cfg, const pgl_layout_ext* ext,
                   int reuse, pgl_iteration_cb cb, int cb_wants_coords,
                   void* user, double* out_coords, pgl_run_stats* stats);

/* ---- resident graph session ---------------------------------------------- */

typedef struct pgl_graph pgl_graph;

typedef struct pgl_graph_info {
    uint64_t n_nodes;
    uint32_t n_paths;
    uint32_t device;
    uint64_t total_steps;
    uint64_t total_nucleotides;
    uint64_t max_path_len;       /* d_max of make_schedule, engine.cpp:269-270 */
    uint64_t device_bytes;       /* HBM held by the packed graph + layout */
    uint32_t usable;             /* some path has >= 2 steps (engine.cpp:30-34) */
    uint32_t _pad0;
} pgl_graph_info;

/* Pack the graph (step records, cum_steps, guide table) and upload it. */
int pgl_graph_create(int device, const pgl_graph_view* graph, pgl_graph** out);
int pgl_graph_destroy(pgl_graph* g);
int pgl_graph_info_get(const pgl_graph* g, pgl_graph_info* out);

/* GFA straight into HBM: the file is parsed on `threads` host threads
 * (pgl_gfa_parse_file semantics and errors) into node lengths and one 4-byte
 * word per step; the device builds the step records (build_graph offsets
 * and path_position by a scan). The 24-byte PathStep arrays are never
 * materialised on the host. */
int pgl_graph_create_gfa(int device, const char* path, uint32_t threads, pgl_graph** out);

/* Parity hook: copy the packed device index back to the host, decoded.
 * positions[2*S] = path_position(start), path_position(end) of every step
 * in path order (graph.hpp:98-109); nodes[S] = PathStep::node_id;
 * cum[P+1] = cum_steps (graph.hpp:75-76). Any pointer may be NULL. */
int pgl_graph_export_index(const pgl_graph* g, uint64_t* positions,
                           uint32_t* nodes, uint64_t* cum);

/* Same semantics as pgl_layout_run on an already-resident graph. The final
 * layout also stays resident on the device (for pgl_graph_stress).
 * out_coords may be NULL (no device-to-host copy). */
int pgl_graph_layout(pgl_graph* g, const pgl_layout_config* cfg,
                     const pgl_layout_ext* ext, int reuse, pgl_iteration_cb cb,
                     int cb_wants_coords, void* user, double* out_coords,
                     pgl_run_stats* stats);

/* Device timing of the last pgl_graph_layout: CUDA events on the launching
 * stream around the SGD kernels only, summed over iterations. */
typedef struct pgl_timing {
    double kernel_ms;      /* sum over SGD launches */
    double init_ms;        /* host init_layout + upload of the initial layout */
    double total_ms;       /* whole call, host wall */
    double device_ms;      /* CUDA events on the graph's stream: from the upload of
                              the initial layout to the end of the last SGD kernel */
    uint32_t launches;     /* SGD kernel launches (one per iteration) */
    uint32_t grid_blocks;
    uint32_t block_threads;
    uint32_t nonfinite_nodes; /* Layout::all_finite on the device after the layout (layout.cpp:9-18):
                                 nodes with a non-finite coordinate; nonzero raises
                                 NonFiniteCoordinate */
    uint64_t device_threads; /* resident lanes = concurrent Hogwild workers*32 */
    uint32_t coord_kind;      /* pgl_coord_precision the layout ran with (PGL_COORD_AUTO resolved) */
    uint32_t kernel_variant;  /* the Hogwild kernel that ran: tile variant 1/2/5/6/7/8 (auto resolved),
                                 0 for the i.i.d. kernel and replay */
} pgl_timing;

int pgl_graph_last_timing(const pgl_graph* g, pgl_timing* out);

/* Layout::all_finite (layout.cpp:9-18) on the device: how many nodes have a
 * non-finite coordinate, and the first such node id (0 if none), for the
 * resident layout (coords NULL) or a host layout [4*n_nodes]. Every layout
 * call runs the same check on its result and raises NonFiniteCoordinate
 * when it fails. */
int pgl_graph_all_finite(pgl_graph* g, const double* coords, uint64_t* bad_nodes, uint64_t* first_bad);

/* ---- sampled path stress: the drop-in for sampled_path_stress ----------- */

typedef enum pgl_sps_method {
    /* Counter-based per-sample streams, deterministic fixed-order two-pass
     * reduction; same estimator as metrics.cpp:108-159, different draws. */
    PGL_SPS_COUNTER = 0,
    /* The reference's own per-path xoshiro stream seed_worker(seed, 2^61+pi)
     * replayed in parallel (jump-ahead + phase scan): the same terms as the
     * reference, so n and skipped are identical and mean/sd agree to ~1e-15. */
    PGL_SPS_STREAM = 1
} pgl_sps_method;

/* coords: host [4*n_nodes] doubles in snapshot order. */
int pgl_sampled_path_stress(int device, const pgl_graph_view* graph,
                            const double* coords, uint64_t seed,
                            uint32_t samples_per_node, uint32_t method,
                            pgl_stress_report* out);

/* On a resident graph. coords NULL = the layout left on the device by the
 * last pgl_graph_layout (no host round trip). */
int pgl_graph_stress(pgl_graph* g, const double* coords, uint64_t seed,
                     uint32_t samples_per_node, uint32_t method,
                     pgl_stress_report* out, double* kernel_ms);

/* ---- exact path stress: the drop-in for exact_path_stress --------------- */

/* Every step pair i < j of every path, the reference's per-pair term
 * (step_pair_stress, metrics.cpp:59-73; IEEE, bit-identical terms), two
 * passes (mean, then squared deviations), n/skipped exact; sums in
 * double-double with a fixed fold order (deterministic, within a few ulps of
 * the exact sum of the terms). O(sum |p|^2): meant for small graphs. */
int pgl_exact_path_stress(int device, const pgl_graph_view* graph,
                          const double* coords, pgl_stress_report* out);

/* On a resident graph; coords NULL = the resident layout. */
int pgl_graph_exact_stress(pgl_graph* g, const double* coords,
                           pgl_stress_report* out, double* kernel_ms);

/* ---- GFA ingest: the drop-in for parse_gfa + build_graph ----------------- */

/* Edge (graph.hpp:24-30); *_end: 0 = Endpoint::start, 1 = Endpoint::end. */
typedef struct pgl_edge {
    uint32_t from;
    uint32_t to;
    uint8_t from_end;
    uint8_t to_end;
    uint8_t _pad[6];
} pgl_edge;

typedef struct pgl_gfa_info {
    uint64_t n_nodes;
    uint64_t n_edges;
    uint64_t total_steps;
    uint64_t skipped_records;  /* GfaParseStats::skipped_records (gfa.hpp:10-12) */
    uint32_t n_paths;
    uint32_t _pad0;
} pgl_gfa_info;

/* A parsed, built graph (owns its PathStep arrays). Same node ids (order of
 * S declaration), edges (L order), paths (P order), offsets and exception
 * classes/messages as parse_gfa followed by build_graph; the file is mmap'd
 * and parsed on `threads` host threads (0 = all). */
typedef struct pgl_gfa pgl_gfa;
int pgl_gfa_parse_file(const char* path, uint32_t threads, pgl_gfa** out);
int pgl_gfa_parse_buffer(const char* data, uint64_t size, uint32_t threads, pgl_gfa** out);
int pgl_gfa_info_get(const pgl_gfa* g, pgl_gfa_info* out);
/* The borrowed view for pgl_layout_run / pgl_graph_create (valid until free). */
int pgl_gfa_view(const pgl_gfa* g, pgl_graph_view* out);
/* Copies the n_edges edges into out. */
int pgl_gfa_edges(const pgl_gfa* g, pgl_edge* out);
/* Path name (P record column 2); NULL when out of range. */
const char* pgl_gfa_path_name(const pgl_gfa* g, uint32_t path);
int pgl_gfa_free(pgl_gfa* g);

/* ---- layout table IO: the drop-in for write/read_layout_tsv -------------- */

/* Byte-identical to write_layout_tsv ("%zu\t%.17g\t%.17g\t%.17g\t%.17g\n"
 * rows under the reference header), formatted on `threads` host threads
 * (0 = all). coords: [4*n_nodes] snapshot order. NonFiniteCoordinate names
 * the lowest offending node, as the serial writer does. */
int pgl_layout_write_tsv(const char* path, const double* coords, uint64_t n_nodes, uint32_t threads);
/* read_layout_tsv: *coords receives a malloc'd [4 * *n_nodes] array (free
 * with pgl_free); same exception classes/messages, first failure in line
 * order. */
int pgl_layout_read_tsv(const char* path, uint32_t threads, uint64_t* n_nodes, double** coords);
/* In-memory forms (the reference's ostream/istream signatures): *text is a
 * malloc'd, NUL-terminated buffer of *size bytes; free both with pgl_free. */
int pgl_layout_format_tsv(const double* coords, uint64_t n_nodes, uint32_t threads, char** text, uint64_t* size);
int pgl_layout_parse_tsv(const char* data, uint64_t size, uint32_t threads, uint64_t* n_nodes, double** coords);
void pgl_free(void* p);

/* ---- host-side helpers of the path (bit-exact with the reference) -------- */

/* etas[n_iters] of make_schedule (engine.cpp:251-274). */
int pgl_make_schedule(const pgl_graph_view* graph, const pgl_layout_config* cfg,
                      double* etas);
/* init_layout (layout.cpp:20-34) into out[4*n_nodes]. */
int pgl_init_layout(const pgl_graph_view* graph, uint64_t seed, double* out);

/* ---- multi-GPU shard scheduler ------------------------------------------ */

/* Lays out n_graphs independent graphs on n_devices GPUs: longest-processing-
 * time-first assignment by sum|p| * n_iters, one host thread + stream per
 * device, no collective. out_coords[k] receives graph k's layout (may be
 * NULL to skip the copy); seconds[k] the per-graph wall time; assignment[k]
 * the device index used. */
/* The scheduler's plan alone (host only, no device touched): LPT over the
 * graphs' update counts (total_steps * n_iters * drf / srf), heaviest first
 * onto the least-loaded of n_devices, ties to the lowest index.
 * assignment[k] gets graph k's device index; work[k] (optional) its update
 * count; device_load[d] (optional) the summed work per device.
 * pgl_layout_shards runs exactly this plan. */
int pgl_shard_plan(int n_devices, int n_graphs, const pgl_graph_view* const* graphs,
                   const pgl_layout_config* cfgs, int* assignment, double* work,
                   double* device_load);

int pgl_layout_shards(int n_devices, const int* devices, int n_graphs,
                      const pgl_graph_view* const* graphs,
                      const pgl_layout_config* cfgs, const pgl_layout_ext* ext,
                      double* const* out_coords, pgl_run_stats* stats,
                      double* seconds, int* assignment);

/* ---- synthetic input fixture (host only) --------------------------------- */

/* generate_synthetic_pangenome (synthetic.cpp:24-120): same nodes, walks,
 * offsets for the same arguments. Edges are not materialised (the layout
 * path never reads them); n_edges reports their count when requested. */
typedef struct pgl_synthetic pgl_synthetic;
int pgl_synthetic_generate(uint64_t seed, uint64_t backbone_nodes,
                           uint32_t n_paths, double variant_rate,
                           pgl_synthetic** out);
/* Config 5 fixture (not in the reference): nested bubbles up to `depth`
 * levels (substitution branches with their own sites), inversions (reverse
 * steps), deletions and duplications (node revisits), `site_rate` sites per
 * backbone node, per-path allele choices. Deterministic in its arguments;
 * its walks are plain build_graph input. */
int pgl_synthetic_generate_nested(uint64_t seed, uint64_t backbone_nodes, uint32_t n_paths,
                                  uint32_t depth, double site_rate, pgl_synthetic** out);
int pgl_synthetic_view(const pgl_synthetic* s, pgl_graph_view* view);
int pgl_synthetic_free(pgl_synthetic* s);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* PGL_B200_H */
