/*
 * oracle/pgl_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference PG-SGD path (/root/reference/proj),
 * used as the parity checker for the CUDA path. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it; the
 * product (libpgl_b200.so) never links or calls it.
 *
 * Parity pinned: every function is checked against the reference library
 * itself (oracle/_ref/libpglref.so, built from the reference sources by
 * oracle/Makefile) and against the known answers of the reference's tests
 * (tests/test_oracle.py, tests/golden/).
 */
#ifndef PGL_ORACLE_H
#define PGL_ORACLE_H

#include <stdint.h>

#include "../include/pgl_b200.h"

typedef struct orc_graph {
    uint64_t n_nodes;
    uint64_t* node_len;     /* [n_nodes] */
    uint32_t n_paths;
    uint64_t* cum;          /* [n_paths+1] cum_steps (graph.hpp:75-76) */
    uint64_t* path_total;   /* [n_paths] total_len */
    uint32_t* step_node;    /* [S] */
    uint8_t* step_rev;      /* [S] 1 = reverse */
    uint64_t* step_off;     /* [S] PathStep::offset */
    uint32_t* step_len;     /* [S] PathStep::seq_len */
    uint64_t total_steps;
    uint64_t total_nt;
} orc_graph;

/* rng.hpp:13-71 */
void orc_rng_seed(uint64_t seed, uint64_t worker, uint64_t s[4]);
uint64_t orc_rng_next(uint64_t s[4]);
void orc_rng_draws(uint64_t seed, uint64_t worker, uint64_t count, uint64_t* out);

/* graph.cpp:7-59 from flat walks; returns error type (0 ok) */
int orc_build(uint64_t n_nodes, const uint64_t* node_len, uint32_t n_paths,
              const uint64_t* path_n_steps, const uint32_t* step_node,
              const uint8_t* step_rev, orc_graph** out);
/* synthetic.cpp:24-120 (walks only; edges are not materialised) */
int orc_generate(uint64_t seed, uint64_t backbone, uint32_t n_paths, double rate,
                 orc_graph** out);
void orc_free(orc_graph* g);
void orc_counts(const orc_graph* g, uint64_t* counts4); /* nodes, paths, steps, nt */
void orc_export(const orc_graph* g, uint64_t* node_len, uint64_t* cum,
                uint64_t* path_total, uint32_t* step_node, uint8_t* step_rev,
                uint64_t* step_off, uint32_t* step_len);
void orc_positions(const orc_graph* g, uint64_t* out2);

/* rng.hpp:89-151 */
int orc_zipf_samples(uint64_t n, double theta, uint64_t seed, uint64_t worker,
                     uint64_t count, uint64_t* out);
/* hx1, hxn, s constants of ZipfSampler (rng.hpp:95-97) */
void orc_zipf_constants(uint64_t n, double theta, double out3[3]);
/* graph.hpp:123-138 */
int orc_weighted_select(const orc_graph* g, uint64_t seed, uint64_t worker,
                        uint64_t count, uint32_t* path, uint64_t* step);

/* layout.cpp:20-34 */
void orc_init_layout(const orc_graph* g, uint64_t seed, double* out);
/* engine.cpp:251-274; returns error type */
int orc_make_schedule(const orc_graph* g, const pgl_layout_config* cfg, double* etas);

/* engine.cpp:276-306 */
int orc_apply_update(double* coords, uint32_t ni, int ei_end, uint32_t nj,
                     int ej_end, double d_ref, double eta, uint64_t s[4]);

typedef void (*orc_iter_cb)(uint32_t iter, const double* coords, double eta,
                            void* user);
/* engine.cpp:174-247 with one worker (threads = 1 semantics; cfg->threads
 * is validated but the run is always the reproducible single stream).
 * Returns an error type (pgl_error_type), 0 ok. */
int orc_run_layout(const orc_graph* g, const pgl_layout_config* cfg, int reuse,
                   double* out_coords, pgl_run_stats* stats, orc_iter_cb cb,
                   void* user);

/* metrics.cpp:108-159, streaming two-pass (stream replayed for sigma). */
int orc_sampled_path_stress(const orc_graph* g, const double* coords,
                            uint64_t seed, uint32_t spn, pgl_stress_report* out);
/* metrics.cpp:75-106 */
void orc_exact_path_stress(const orc_graph* g, const double* coords,
                           pgl_stress_report* out);

/* CPU restatement of the product's PGL_SPS_COUNTER estimator (same sample
 * space and term as metrics.cpp:108-159, counter-based draws, fixed-order
 * chunked reduction) — pins the GPU kernel bit-for-bit. */
int orc_sps_counter(const orc_graph* g, const double* coords, uint64_t seed,
                    uint32_t spn, pgl_stress_report* out);

const char* orc_last_error(void);

#endif
