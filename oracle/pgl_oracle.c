/*
 * oracle/pgl_oracle.c — TEST INFRASTRUCTURE ONLY: the parity checker.
 *
 * A plain-C restatement of the reference's PG-SGD layout path
 * (/root/reference/proj, C++20). Each function cites the reference lines it
 * follows. Compiled with -ffp-contract=off so every double expression is
 * evaluated exactly as the reference's default (no-FMA) x86-64 build does.
 *
 * Pinned against the reference library itself (oracle/_ref/libpglref.so) and
 * the reference tests' known answers by tests/test_oracle.py. Never linked
 * into or called by the product.
 */
#include "pgl_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static char g_err[512];
const char* orc_last_error(void) { return g_err; }

static int fail(int type, const char* name, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s: %s", name, msg);
    return type;
}

/* ---- RNG: rng.hpp:13-71 ------------------------------------------------- */

static const uint64_t kPhi = 0x9E3779B97F4A7C15ULL;
static const uint64_t kStreamInit = 1ULL << 62;   /* rng.hpp:76 */
static const uint64_t kStreamSps = 1ULL << 61;    /* rng.hpp:77 */
static const uint64_t kStreamSynth = 1ULL << 60;  /* rng.hpp:78 */

static inline uint64_t rotl64(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }

/* xoshiro256+ step, rng.hpp:21-31 */
uint64_t orc_rng_next(uint64_t s[4]) {
    const uint64_t out = s[0] + s[3];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return out;
}

static inline uint64_t splitmix_step(uint64_t* st) { /* rng.hpp:52-57 */
    uint64_t z = (*st += kPhi);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

void orc_rng_seed(uint64_t seed, uint64_t worker, uint64_t s[4]) { /* rng.hpp:63-71 */
    uint64_t key = seed ^ (kPhi * (worker + 1));
    for (int w = 0; w < 4; ++w) s[w] = splitmix_step(&key);
    if ((s[0] | s[1] | s[2] | s[3]) == 0) s[0] = kPhi;
}

void orc_rng_draws(uint64_t seed, uint64_t worker, uint64_t count, uint64_t* out) {
    uint64_t s[4];
    orc_rng_seed(seed, worker, s);
    for (uint64_t k = 0; k < count; ++k) out[k] = orc_rng_next(s);
}

static inline double uniform01(uint64_t s[4]) { /* rng.hpp:35-37 */
    return (double)(orc_rng_next(s) >> 11) * 0x1.0p-53;
}
static inline int coin(uint64_t s[4]) { return (orc_rng_next(s) >> 63) != 0; } /* :40 */
static inline uint64_t below(uint64_t s[4], uint64_t n) { /* :44-47 */
    return (uint64_t)(((unsigned __int128)orc_rng_next(s) * n) >> 64);
}

/* ---- Zipf by rejection inversion: rng.hpp:89-151 ----------------------- */

typedef struct { uint64_t n; double theta, hx1, hxn, s; } zipf_t;

static double zh1(double x) { /* helper1, rng.hpp:136-139 */
    if (fabs(x) > 1e-8) return log1p(x) / x;
    return 1.0 - x * (0.5 - x * (1.0 / 3.0 - 0.25 * x));
}
static double zh2(double x) { /* helper2, rng.hpp:141-144 */
    if (fabs(x) > 1e-8) return expm1(x) / x;
    return 1.0 + x * 0.5 * (1.0 + x * (1.0 / 3.0) * (1.0 + 0.25 * x));
}
static double zH(const zipf_t* z, double x) { /* h_integral, :122-125 */
    const double lx = log(x);
    return zh2((1.0 - z->theta) * lx) * lx;
}
static double zh(const zipf_t* z, double x) { return exp(-z->theta * log(x)); } /* :127 */
static double zHinv(const zipf_t* z, double x) { /* :129-133 */
    double t = x * (1.0 - z->theta);
    if (t < -1.0) t = -1.0;
    return exp(zh1(t) * x);
}
static void zipf_init(zipf_t* z, uint64_t n, double theta) { /* ctor :91-98 */
    z->n = n;
    z->theta = theta;
    z->hx1 = zH(z, 1.5) - 1.0;
    z->hxn = zH(z, (double)n + 0.5);
    z->s = 2.0 - zHinv(z, zH(z, 2.5) - zh(z, 2.0));
}
static uint64_t zipf_draw(const zipf_t* z, uint64_t s[4]) { /* sample, :103-117 */
    if (z->n == 1) return 1;
    for (;;) {
        const double u = z->hxn + uniform01(s) * (z->hx1 - z->hxn);
        const double x = zHinv(z, u);
        uint64_t k = (uint64_t)(x + 0.5);
        if (k < 1) k = 1;
        else if (k > z->n) k = z->n;
        const double kd = (double)k;
        if (kd - x <= z->s || u >= zH(z, kd + 0.5) - zh(z, kd)) return k;
    }
}

void orc_zipf_constants(uint64_t n, double theta, double out3[3]) {
    zipf_t z;
    zipf_init(&z, n, theta);
    out3[0] = z.hx1;
    out3[1] = z.hxn;
    out3[2] = z.s;
}

int orc_zipf_samples(uint64_t n, double theta, uint64_t seed, uint64_t worker,
                     uint64_t count, uint64_t* out) {
    if (n < 1) return fail(PGL_ERR_INVALID_PARAMETER, "InvalidParameter", "zipf support must be non-empty");
    if (!(theta > 0.0) || !isfinite(theta))
        return fail(PGL_ERR_INVALID_PARAMETER, "InvalidParameter", "zipf exponent must be positive and finite");
    zipf_t z;
    zipf_init(&z, n, theta);
    uint64_t s[4];
    orc_rng_seed(seed, worker, s);
    for (uint64_t k = 0; k < count; ++k) out[k] = zipf_draw(&z, s);
    return 0;
}

/* ---- graph: graph.cpp:7-59, graph.hpp:98-138 ---------------------------- */

static orc_graph* graph_alloc(uint64_t n_nodes, uint32_t n_paths, uint64_t n_steps) {
    orc_graph* g = (orc_graph*)calloc(1, sizeof *g);
    g->n_nodes = n_nodes;
    g->n_paths = n_paths;
    g->node_len = (uint64_t*)malloc((n_nodes + 1) * sizeof(uint64_t));
    g->cum = (uint64_t*)calloc(n_paths + 1, sizeof(uint64_t));
    g->path_total = (uint64_t*)calloc(n_paths + 1, sizeof(uint64_t));
    g->step_node = (uint32_t*)malloc((n_steps + 1) * sizeof(uint32_t));
    g->step_rev = (uint8_t*)malloc(n_steps + 1);
    g->step_off = (uint64_t*)malloc((n_steps + 1) * sizeof(uint64_t));
    g->step_len = (uint32_t*)malloc((n_steps + 1) * sizeof(uint32_t));
    return g;
}

void orc_free(orc_graph* g) {
    if (!g) return;
    free(g->node_len);
    free(g->cum);
    free(g->path_total);
    free(g->step_node);
    free(g->step_rev);
    free(g->step_off);
    free(g->step_len);
    free(g);
}

/* Offsets, totals, cum_steps exactly as build_graph (graph.cpp:7-59). */
int orc_build(uint64_t n_nodes, const uint64_t* node_len, uint32_t n_paths,
              const uint64_t* path_n_steps, const uint32_t* step_node,
              const uint8_t* step_rev, orc_graph** out) {
    uint64_t S = 0;
    for (uint32_t p = 0; p < n_paths; ++p) S += path_n_steps[p];
    orc_graph* g = graph_alloc(n_nodes, n_paths, S);
    for (uint64_t n = 0; n < n_nodes; ++n) {
        if (node_len[n] == 0) { orc_free(g); return fail(PGL_ERR_INVALID_PARAMETER, "InvalidParameter", "zero sequence length"); }
        g->node_len[n] = node_len[n];
        g->total_nt += node_len[n];
    }
    uint64_t k = 0;
    g->cum[0] = 0;
    for (uint32_t p = 0; p < n_paths; ++p) {
        if (path_n_steps[p] == 0) { orc_free(g); return fail(PGL_ERR_EMPTY_PATH, "EmptyPath", "path has no steps"); }
        uint64_t off = 0;
        for (uint64_t s = 0; s < path_n_steps[p]; ++s, ++k) {
            const uint32_t v = step_node[k];
            if (v >= n_nodes) { orc_free(g); return fail(PGL_ERR_UNKNOWN_NODE, "UnknownNode", "path references unknown node"); }
            const uint64_t len = g->node_len[v];
            if (len > 0xFFFFFFFFULL) { orc_free(g); return fail(PGL_ERR_INVALID_PARAMETER, "InvalidParameter", "node too long"); }
            g->step_node[k] = v;
            g->step_rev[k] = step_rev[k] ? 1 : 0;
            g->step_off[k] = off;
            g->step_len[k] = (uint32_t)len;
            off += len;
        }
        g->path_total[p] = off;
        g->cum[p + 1] = k;
    }
    g->total_steps = k;
    *out = g;
    return 0;
}

/* generate_synthetic_pangenome, synthetic.cpp:24-120 (walk part). */
enum { B_SNV = 0, B_INS = 1, B_DEL = 2, B_NONE = 3 };

int orc_generate(uint64_t seed, uint64_t B, uint32_t n_paths, double rate, orc_graph** out) {
    if (B < 2) return fail(PGL_ERR_INVALID_PARAMETER, "InvalidParameter", "backbone needs at least 2 nodes");
    if (n_paths < 1) return fail(PGL_ERR_INVALID_PARAMETER, "InvalidParameter", "need at least one path");
    if (!(rate >= 0.0 && rate <= 1.0)) return fail(PGL_ERR_INVALID_PARAMETER, "InvalidParameter", "variant_rate must lie in [0, 1]");
    uint64_t s[4];
    orc_rng_seed(seed, kStreamSynth, s);
    uint64_t* bb_len = (uint64_t*)malloc(B * sizeof(uint64_t));
    uint8_t* type = (uint8_t*)malloc(B);
    uint64_t* alt_len = (uint64_t*)calloc(B, sizeof(uint64_t));
    uint32_t* alt_id = (uint32_t*)calloc(B, sizeof(uint32_t));
    for (uint64_t b = 0; b < B; ++b) bb_len[b] = 8 + below(s, 25);           /* :40-41 */
    for (uint64_t b = 0; b < B; ++b) {                                       /* :44-57 */
        type[b] = B_NONE;
        if (uniform01(s) >= rate) continue;
        uint8_t feas[3];
        uint64_t nf = 0;
        if (b + 3 <= B) feas[nf++] = B_SNV;
        if (b + 2 <= B) feas[nf++] = B_INS;
        if (b + 3 <= B) feas[nf++] = B_DEL;
        if (nf == 0) continue;
        type[b] = feas[below(s, nf)];
        if (type[b] != B_DEL) alt_len[b] = 8 + below(s, 25);
    }
    /* ids in positional order, :62-75 */
    uint64_t n_nodes = 0;
    uint64_t* lens = (uint64_t*)malloc(3 * B * sizeof(uint64_t));
    uint32_t* bb_id = (uint32_t*)malloc(B * sizeof(uint32_t));
    for (uint64_t b = 0; b < B; ++b) {
        bb_id[b] = (uint32_t)n_nodes;
        lens[n_nodes++] = bb_len[b];
        if (type[b] == B_INS) { alt_id[b] = (uint32_t)n_nodes; lens[n_nodes++] = alt_len[b]; }
        if (b >= 1 && type[b - 1] == B_SNV) { alt_id[b - 1] = (uint32_t)n_nodes; lens[n_nodes++] = alt_len[b - 1]; }
    }
    /* walks, :77-104 */
    uint64_t cap = (uint64_t)n_paths * (B + B / 4 + 16);
    uint32_t* steps = (uint32_t*)malloc(cap * sizeof(uint32_t));
    uint64_t* pn = (uint64_t*)calloc(n_paths, sizeof(uint64_t));
    uint64_t k = 0;
    for (uint32_t p = 0; p < n_paths; ++p) {
        const uint64_t k0 = k;
        uint64_t b = 0;
        while (b < B) {
            if (k + 2 >= cap) { cap *= 2; steps = (uint32_t*)realloc(steps, cap * sizeof(uint32_t)); }
            steps[k++] = bb_id[b];
            if (type[b] != B_NONE && coin(s)) {
                if (type[b] == B_SNV) { steps[k++] = alt_id[b]; b += 2; continue; }
                if (type[b] == B_INS) { steps[k++] = alt_id[b]; b += 1; continue; }
                b += 2; /* deletion */
                continue;
            }
            b += 1;
        }
        pn[p] = k - k0;
    }
    uint8_t* rev = (uint8_t*)calloc(k + 1, 1);
    const int rc = orc_build(n_nodes, lens, n_paths, pn, steps, rev, out);
    free(bb_len); free(type); free(alt_len); free(alt_id); free(lens); free(bb_id);
    free(steps); free(pn); free(rev);
    return rc;
}

void orc_counts(const orc_graph* g, uint64_t* c) {
    c[0] = g->n_nodes;
    c[1] = g->n_paths;
    c[2] = g->total_steps;
    c[3] = g->total_nt;
}

void orc_export(const orc_graph* g, uint64_t* node_len, uint64_t* cum, uint64_t* path_total,
                uint32_t* step_node, uint8_t* step_rev, uint64_t* step_off, uint32_t* step_len) {
    memcpy(node_len, g->node_len, g->n_nodes * sizeof(uint64_t));
    memcpy(cum, g->cum, (g->n_paths + 1) * sizeof(uint64_t));
    memcpy(path_total, g->path_total, g->n_paths * sizeof(uint64_t));
    memcpy(step_node, g->step_node, g->total_steps * sizeof(uint32_t));
    memcpy(step_rev, g->step_rev, g->total_steps);
    memcpy(step_off, g->step_off, g->total_steps * sizeof(uint64_t));
    memcpy(step_len, g->step_len, g->total_steps * sizeof(uint32_t));
}

/* path_position, graph.hpp:98-109 (k = global step index, end = Endpoint::end) */
static inline uint64_t position(const orc_graph* g, uint64_t k, int end) {
    const int far = g->step_rev[k] ? !end : end;
    return g->step_off[k] + (far ? g->step_len[k] : 0);
}

void orc_positions(const orc_graph* g, uint64_t* out) {
    for (uint64_t k = 0; k < g->total_steps; ++k) {
        out[2 * k] = position(g, k, 0);
        out[2 * k + 1] = position(g, k, 1);
    }
}

/* weighted_step_select, graph.hpp:123-138 */
static void wselect(const orc_graph* g, uint64_t s[4], uint32_t* path, uint64_t* step) {
    const uint64_t pick = below(s, g->total_steps);
    uint64_t lo = 0, hi = g->n_paths; /* cum.size() - 1 */
    while (hi - lo > 1) {
        const uint64_t mid = (lo + hi) / 2;
        if (g->cum[mid] <= pick) lo = mid;
        else hi = mid;
    }
    *path = (uint32_t)lo;
    *step = pick - g->cum[lo];
}

int orc_weighted_select(const orc_graph* g, uint64_t seed, uint64_t worker, uint64_t count,
                        uint32_t* path, uint64_t* step) {
    if (g->total_steps == 0) return fail(PGL_ERR_EMPTY_GRAPH, "EmptyGraph", "weighted_step_select on a graph without path steps");
    uint64_t s[4];
    orc_rng_seed(seed, worker, s);
    for (uint64_t k = 0; k < count; ++k) wselect(g, s, &path[k], &step[k]);
    return 0;
}

/* ---- layout init + schedule: layout.cpp:20-34, engine.cpp:251-274 ------- */

void orc_init_layout(const orc_graph* g, uint64_t seed, double* out) {
    uint64_t s[4];
    orc_rng_seed(seed, kStreamInit, s);
    const double amp = sqrt((double)g->total_nt);
    uint64_t off = 0;
    for (uint64_t n = 0; n < g->n_nodes; ++n) {
        out[4 * n + 0] = (double)off;
        out[4 * n + 1] = (2.0 * uniform01(s) - 1.0) * amp;
        out[4 * n + 2] = (double)(off + g->node_len[n]);
        out[4 * n + 3] = (2.0 * uniform01(s) - 1.0) * amp;
        off += g->node_len[n];
    }
}

static int usable(const orc_graph* g) { /* engine.cpp:30-34 */
    for (uint32_t p = 0; p < g->n_paths; ++p)
        if (g->cum[p + 1] - g->cum[p] >= 2) return 1;
    return 0;
}

static int validate(const pgl_layout_config* c) { /* engine.cpp:15-28 */
    const char* IP = "InvalidParameter";
    if (c->n_iters < 1) return fail(PGL_ERR_INVALID_PARAMETER, IP, "n_iters must be >= 1");
    if (c->threads < 1) return fail(PGL_ERR_INVALID_PARAMETER, IP, "threads must be >= 1");
    if (c->batch_size < 1) return fail(PGL_ERR_INVALID_PARAMETER, IP, "batch_size must be >= 1");
    if (!(c->zipf_theta > 0.0) || !isfinite(c->zipf_theta)) return fail(PGL_ERR_INVALID_PARAMETER, IP, "zipf_theta must be positive");
    if (c->zipf_space_max < 1) return fail(PGL_ERR_INVALID_PARAMETER, IP, "zipf_space_max must be >= 1");
    if (!(c->eta_min_eps > 0.0)) return fail(PGL_ERR_INVALID_PARAMETER, IP, "eta_min_eps must be positive");
    if (c->drf != 1 && c->drf != 2 && c->drf != 4) return fail(PGL_ERR_INVALID_PARAMETER, IP, "drf must be 1, 2 or 4");
    if (c->srf < 1) return fail(PGL_ERR_INVALID_PARAMETER, IP, "srf must be >= 1");
    return 0;
}

int orc_make_schedule(const orc_graph* g, const pgl_layout_config* cfg, double* etas) {
    if (g->n_paths == 0 || !usable(g)) return fail(PGL_ERR_DEGENERATE_GRAPH, "DegenerateGraph", "schedule needs a path pair with d_ref > 0");
    uint64_t dmax = 1;
    for (uint32_t p = 0; p < g->n_paths; ++p) if (g->path_total[p] > dmax) dmax = g->path_total[p];
    const double emax = (double)dmax * (double)dmax, emin = cfg->eta_min_eps;
    const uint32_t n = cfg->n_iters;
    if (n < 1) return fail(PGL_ERR_INVALID_PARAMETER, "InvalidParameter", "schedule needs n_iters >= 1");
    if (!(emax > 0.0) || !(emin > 0.0) || !(emin <= emax)) return fail(PGL_ERR_INVALID_PARAMETER, "InvalidParameter", "schedule needs 0 < eta_min <= eta_max");
    const double lambda = n > 1 ? log(emax / emin) / (n - 1) : 0.0;
    for (uint32_t t = 0; t < n; ++t) etas[t] = emax * exp(-lambda * t);
    return 0;
}

/* ---- update + hot loop: engine.cpp:52-172, :276-306 --------------------- */

int orc_apply_update(double* c, uint32_t ni, int ei, uint32_t nj, int ej, double d_ref,
                     double eta, uint64_t s[4]) {
    if (!(d_ref > 0.0)) return 0;
    const double w = 1.0 / (d_ref * d_ref);
    double mu = eta * w;
    if (mu > 1.0) mu = 1.0;
    double* pi = c + 4 * (uint64_t)ni + 2 * ei;
    double* pj = c + 4 * (uint64_t)nj + 2 * ej;
    const double vix = pi[0], viy = pi[1], vjx = pj[0], vjy = pj[1];
    const double dx = vix - vjx, dy = viy - vjy;
    const double mag = sqrt(dx * dx + dy * dy);
    double ux, uy;
    if (mag < 1e-9) {
        const double angle = 2.0 * 3.14159265358979323846 * uniform01(s);
        ux = cos(angle);
        uy = sin(angle);
    } else {
        ux = dx / mag;
        uy = dy / mag;
    }
    const double delta = mu * (mag - d_ref) / 2.0;
    pi[0] = vix - delta * ux;
    pi[1] = viy - delta * uy;
    pj[0] = vjx + delta * ux;
    pj[1] = vjy + delta * uy;
    return 1;
}

typedef struct { uint32_t p; uint64_t i, j; int ok; } pair_t;

static pair_t select_pair(const orc_graph* g, uint64_t s[4], int cooling, const zipf_t* zs) {
    pair_t r = {0, 0, 0, 0};
    uint64_t step;
    wselect(g, s, &r.p, &step);
    const int64_t n = (int64_t)(g->cum[r.p + 1] - g->cum[r.p]);
    if (n < 2) return r;
    const int64_t i = (int64_t)step;
    int64_t j;
    if (cooling) {
        const int64_t k = (int64_t)zipf_draw(&zs[r.p], s);
        const int64_t sign = coin(s) ? 1 : -1;
        j = i + sign * k;
        if (j < 0 || j >= n) {
            j = i - sign * k;
            if (j < 0 || j >= n) {
                j = i + sign * k;
                j = j < 0 ? 0 : (j > n - 1 ? n - 1 : j);
            }
        }
        if (j == i) return r;
    } else {
        j = (int64_t)below(s, (uint64_t)n);
        if (j == i) {
            j = (int64_t)below(s, (uint64_t)n);
            if (j == i) return r;
        }
    }
    r.i = (uint64_t)i;
    r.j = (uint64_t)j;
    r.ok = 1;
    return r;
}

static double ref_dist(const orc_graph* g, uint64_t base, uint64_t i, int ei, uint64_t j, int ej) {
    const uint64_t a = position(g, base + i, ei), b = position(g, base + j, ej);
    return (double)(a > b ? a - b : b - a);
}

int orc_run_layout(const orc_graph* g, const pgl_layout_config* cfg, int reuse, double* out,
                   pgl_run_stats* stats, orc_iter_cb cb, void* user) {
    if (reuse) { /* engine.cpp:328-334 */
        if (cfg->drf != 2 && cfg->drf != 4) return fail(PGL_ERR_INVALID_PARAMETER, "InvalidParameter", "update reuse needs drf of 2 or 4");
        if (cfg->srf < 1) return fail(PGL_ERR_INVALID_PARAMETER, "InvalidParameter", "srf must be >= 1");
    }
    int rc = validate(cfg);
    if (rc) return rc;
    if (g->n_paths == 0 || !usable(g))
        return fail(PGL_ERR_DEGENERATE_GRAPH, "DegenerateGraph", "layout needs at least one path with two or more steps");
    double* etas = (double*)malloc(cfg->n_iters * sizeof(double));
    rc = orc_make_schedule(g, cfg, etas);
    if (rc) { free(etas); return rc; }
    orc_init_layout(g, cfg->global_seed, out);
    zipf_t* zs = (zipf_t*)malloc((g->n_paths + 1) * sizeof(zipf_t));
    for (uint32_t p = 0; p < g->n_paths; ++p) { /* zipf_params_for, engine.cpp:36-39 */
        const uint64_t n = g->cum[p + 1] - g->cum[p];
        const uint64_t span = n < 2 ? 1 : n - 1;
        zipf_init(&zs[p], span < cfg->zipf_space_max ? span : cfg->zipf_space_max, cfg->zipf_theta);
    }
    uint64_t s[4];
    orc_rng_seed(cfg->global_seed, 0, s);
    pgl_run_stats st;
    memset(&st, 0, sizeof st);
    const uint64_t spi = 10 * g->total_steps / cfg->srf; /* engine.cpp:197 */
    for (uint32_t it = 0; it < cfg->n_iters; ++it) {
        const double eta = etas[it];
        const int force = 2ULL * it >= (uint64_t)cfg->n_iters;
        int cooling = 0;
        for (uint64_t k = 0; k < spi; ++k) { /* run_worker_steps, :114-171 */
            if (k % cfg->batch_size == 0) {
                cooling = force || coin(s);
                if (force) { ++st.batches_second_half; ++st.batches_second_half_cooling; }
                else { ++st.batches_first_half; if (cooling) ++st.batches_first_half_cooling; }
            }
            ++st.primary_steps;
            st.updates_attempted += cfg->drf;
            const pair_t sel = select_pair(g, s, cooling, zs);
            if (!sel.ok) { st.updates_skipped += cfg->drf; continue; }
            const uint64_t base = g->cum[sel.p];
            const uint32_t ni = g->step_node[base + sel.i], nj = g->step_node[base + sel.j];
            const int ei = coin(s) ? 0 : 1; /* coin true -> start (engine.cpp:89-91) */
            const int ej = coin(s) ? 0 : 1;
            if (orc_apply_update(out, ni, ei, nj, ej, ref_dist(g, base, sel.i, ei, sel.j, ej), eta, s)) ++st.updates_applied;
            else ++st.updates_skipped;
            if (cfg->drf > 1) {
                unsigned used = 1u << ((ei ? 2 : 0) | (ej ? 1 : 0));
                for (uint32_t x = 1; x < cfg->drf; ++x) {
                    int a, b;
                    do {
                        a = coin(s) ? 0 : 1;
                        b = coin(s) ? 0 : 1;
                    } while (used & (1u << ((a ? 2 : 0) | (b ? 1 : 0))));
                    used |= 1u << ((a ? 2 : 0) | (b ? 1 : 0));
                    if (orc_apply_update(out, ni, a, nj, b, ref_dist(g, base, sel.i, a, sel.j, b), eta, s)) ++st.updates_applied;
                    else ++st.updates_skipped;
                }
            }
        }
        if (cb) cb(it, out, eta, user);
    }
    if (stats) *stats = st;
    free(etas);
    free(zs);
    return 0;
}

/* ---- metrics: metrics.cpp:14-23, :52-57, :75-159 ------------------------ */

static void finish(pgl_stress_report* r, double ssd) { /* finish_report, metrics.cpp:14-23 */
    r->std_dev = r->n >= 2 ? sqrt(ssd / (double)(r->n - 1)) : 0.0;
    const double half = r->n > 0 ? 1.96 * r->std_dev / sqrt((double)r->n) : 0.0;
    r->ci_low = r->mean - half;
    r->ci_high = r->mean + half;
}

static inline double pstress(const double* vi, const double* vj, double d) { /* :52-57 */
    const double dx = vi[0] - vj[0], dy = vi[1] - vj[1];
    const double err = (sqrt(dx * dx + dy * dy) - d) / d;
    return err * err;
}

/* One pass over the reference's per-path streams (metrics.cpp:116-148).
 * pass 0 accumulates sum/n/skipped, pass 1 the squared deviations. */
static void sps_pass(const orc_graph* g, const double* c, uint64_t seed, uint32_t spn, int pass,
                     double mean, double* acc, uint64_t* n, uint64_t* skipped) {
    for (uint32_t p = 0; p < g->n_paths; ++p) {
        const uint64_t ns = g->cum[p + 1] - g->cum[p], base = g->cum[p];
        if (ns < 2) continue;
        uint64_t s[4];
        orc_rng_seed(seed, kStreamSps + p, s);
        const uint64_t total = (uint64_t)spn * ns;
        for (uint64_t k = 0; k < total; ++k) {
            const uint64_t i = below(s, ns);
            uint64_t j;
            do { j = below(s, ns); } while (j == i);
            int kept = 0;
            for (int a = 0; a < 9 && !kept; ++a) {
                const int ei = coin(s) ? 0 : 1, ej = coin(s) ? 0 : 1;
                const uint64_t pi = position(g, base + i, ei), pj = position(g, base + j, ej);
                if (pi == pj) continue;
                const double d = (double)(pi > pj ? pi - pj : pj - pi);
                const double t = pstress(c + 4 * (uint64_t)g->step_node[base + i] + 2 * ei,
                                         c + 4 * (uint64_t)g->step_node[base + j] + 2 * ej, d);
                if (pass == 0) { *acc += t; ++*n; }
                else *acc += (t - mean) * (t - mean);
                kept = 1;
            }
            if (!kept && pass == 0) ++*skipped;
        }
    }
}

int orc_sampled_path_stress(const orc_graph* g, const double* c, uint64_t seed, uint32_t spn,
                            pgl_stress_report* r) {
    if (spn < 1) return fail(PGL_ERR_INVALID_PARAMETER, "InvalidParameter", "samples_per_node must be >= 1");
    memset(r, 0, sizeof *r);
    double sum = 0.0, ssd = 0.0;
    sps_pass(g, c, seed, spn, 0, 0.0, &sum, &r->n, &r->skipped);
    r->mean = r->n > 0 ? sum / (double)r->n : 0.0;
    sps_pass(g, c, seed, spn, 1, r->mean, &ssd, NULL, NULL);
    finish(r, ssd);
    return 0;
}

static int step_pair_term(const orc_graph* g, const double* c, uint64_t base, uint64_t i, uint64_t j,
                          double* out) { /* step_pair_stress + for_each_pair_term, :25-39, :59-73 */
    double sum = 0.0;
    int cnt = 0;
    for (int ei = 0; ei < 2; ++ei) {
        const uint64_t pi = position(g, base + i, ei);
        for (int ej = 0; ej < 2; ++ej) {
            const uint64_t pj = position(g, base + j, ej);
            if (pi == pj) continue;
            const double d = (double)(pi > pj ? pi - pj : pj - pi);
            sum += pstress(c + 4 * (uint64_t)g->step_node[base + i] + 2 * ei,
                           c + 4 * (uint64_t)g->step_node[base + j] + 2 * ej, d);
            ++cnt;
        }
    }
    if (!cnt) return 0;
    *out = sum / cnt;
    return 1;
}

void orc_exact_path_stress(const orc_graph* g, const double* c, pgl_stress_report* r) {
    memset(r, 0, sizeof *r);
    double sum = 0.0, ssd = 0.0, t;
    for (uint32_t p = 0; p < g->n_paths; ++p) {
        const uint64_t ns = g->cum[p + 1] - g->cum[p], base = g->cum[p];
        for (uint64_t i = 0; i + 1 < ns; ++i)
            for (uint64_t j = i + 1; j < ns; ++j) {
                if (step_pair_term(g, c, base, i, j, &t)) { sum += t; ++r->n; }
                else ++r->skipped;
            }
    }
    r->mean = r->n > 0 ? sum / (double)r->n : 0.0;
    if (r->n >= 2)
        for (uint32_t p = 0; p < g->n_paths; ++p) {
            const uint64_t ns = g->cum[p + 1] - g->cum[p], base = g->cum[p];
            for (uint64_t i = 0; i + 1 < ns; ++i)
                for (uint64_t j = i + 1; j < ns; ++j)
                    if (step_pair_term(g, c, base, i, j, &t)) ssd += (t - r->mean) * (t - r->mean);
        }
    finish(r, ssd);
}

/* ---- the product's counter-based SPS estimator, restated ---------------- */
/* (pgl_sps.cu, PGL_SPS_COUNTER.) Path p with ns = |p| >= 2 steps has
 * spn*ns samples; sample s takes the primary step i = s mod ns (each step
 * exactly spn times) and j uniform over the other ns-1 steps:
 * j = hi64(draw(s*16) * (ns-1)), +1 when j >= i. Draw t of sample s is the
 * splitmix64 output at counter s*16 + t of the stream keyed by
 * splitmix64(seed ^ phi*(2^61 + p + 1)); up to 9 coin attempts at counters
 * s*16+1 .. s*16+9 (top bit -> e_i, next bit -> e_j, set -> start) for a
 * nonzero d_ref (metrics.cpp:116-148). Reduction, in this exact order:
 * path-major chunks of SPS_CHUNK samples; in a chunk lane l (of SPS_LANES)
 * runs Welford over samples l, l+SPS_LANES, ...; lane moments are merged by
 * a halving tree (Chan et al. pairwise merge); chunk moments are folded by
 * SPS_FINAL lanes with stride SPS_FINAL, then a halving tree. */
#define SPS_LANES 256
#define SPS_CHUNK 16384
#define SPS_FINAL 1024

static inline uint64_t ctr_draw(uint64_t key, uint64_t ctr) {
    uint64_t z = key + (ctr + 1) * kPhi;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static inline uint64_t ctr_key(uint64_t seed, uint32_t p) {
    uint64_t key = seed ^ (kPhi * (kStreamSps + p + 1));
    return splitmix_step(&key);
}

/* returns 1 with a term, 0 skipped (9 degenerate coin pairs) */
static int ctr_sample(const orc_graph* g, const double* c, uint64_t key, uint64_t base, uint64_t ns, uint64_t s,
                      uint64_t i, double* term) {
    uint64_t j = (uint64_t)(((unsigned __int128)ctr_draw(key, s * 16) * (ns - 1)) >> 64);
    if (j >= i) ++j;
    for (uint64_t a = 0; a < 9; ++a) {
        const uint64_t r = ctr_draw(key, s * 16 + 1 + a);
        const int ei = (r >> 63) ? 0 : 1, ej = ((r >> 62) & 1) ? 0 : 1;
        const uint64_t pi = position(g, base + i, ei), pj = position(g, base + j, ej);
        if (pi == pj) continue;
        const double d = (double)(pi > pj ? pi - pj : pj - pi);
        *term = pstress(c + 4 * (uint64_t)g->step_node[base + i] + 2 * ei,
                        c + 4 * (uint64_t)g->step_node[base + j] + 2 * ej, d);
        return 1;
    }
    return 0;
}

typedef struct { double n, mean, m2; } moments;

static inline void mpush(moments* a, double t) {
    a->n += 1.0;
    const double d = t - a->mean;
    a->mean += d / a->n;
    a->m2 += d * (t - a->mean);
}

static inline moments mmerge(moments a, moments b) {
    if (b.n == 0.0) return a;
    if (a.n == 0.0) return b;
    const double n = a.n + b.n;
    const double d = b.mean - a.mean;
    moments r = {n, a.mean + d * (b.n / n), a.m2 + b.m2 + d * d * (a.n * b.n / n)};
    return r;
}

static moments mtree(moments* v, int n) {
    for (int stride = n / 2; stride >= 1; stride /= 2)
        for (int k = 0; k < stride; ++k) v[k] = mmerge(v[k], v[k + stride]);
    return v[0];
}

int orc_sps_counter(const orc_graph* g, const double* c, uint64_t seed, uint32_t spn,
                    pgl_stress_report* r) {
    if (spn < 1) return fail(PGL_ERR_INVALID_PARAMETER, "InvalidParameter", "samples_per_node must be >= 1");
    memset(r, 0, sizeof *r);
    uint64_t n_chunks = 0;
    for (uint32_t p = 0; p < g->n_paths; ++p) {
        const uint64_t ns = g->cum[p + 1] - g->cum[p];
        if (ns >= 2) n_chunks += ((uint64_t)spn * ns + SPS_CHUNK - 1) / SPS_CHUNK;
    }
    moments* part = (moments*)calloc(n_chunks + 1, sizeof(moments));
    moments lane[SPS_LANES], fin[SPS_FINAL];
    uint64_t ch = 0;
    for (uint32_t p = 0; p < g->n_paths; ++p) {
        const uint64_t base = g->cum[p], ns = g->cum[p + 1] - base;
        if (ns < 2) continue;
        const uint64_t key = ctr_key(seed, p), q = (uint64_t)spn * ns;
        for (uint64_t s0 = 0; s0 < q; s0 += SPS_CHUNK, ++ch) {
            for (int l = 0; l < SPS_LANES; ++l) {
                moments m = {0.0, 0.0, 0.0};
                for (uint64_t s = s0 + (uint64_t)l; s < s0 + SPS_CHUNK && s < q; s += SPS_LANES) {
                    double t;
                    if (ctr_sample(g, c, key, base, ns, s, s % ns, &t))
                        mpush(&m, t);
                    else
                        ++r->skipped;
                }
                lane[l] = m;
            }
            part[ch] = mtree(lane, SPS_LANES);
        }
    }
    for (int l = 0; l < SPS_FINAL; ++l) {
        moments acc = {0.0, 0.0, 0.0};
        for (uint64_t k = (uint64_t)l; k < n_chunks; k += SPS_FINAL) acc = mmerge(acc, part[k]);
        fin[l] = acc;
    }
    const moments tot = mtree(fin, SPS_FINAL);
    r->n = (uint64_t)tot.n;
    r->mean = tot.mean;
    finish(r, tot.m2);
    free(part);
    return 0;
}
