// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY (checker, never shipped).
//
// extern "C" wrapper around the UNMODIFIED reference library, compiled from
// the sources under /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libpglref.so. The reference namespace is renamed to `pglref`
// on the command line (-Dpglayout=pglref) so nothing collides with the
// product. Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may
// load it.
//
// Every entry point returns 0 on success or (ErrorKind + 1) when the
// reference threw (errors.hpp:10-42); pglref_last_error() has the message.

#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "pglayout/engine.hpp"
#include "pglayout/gfa.hpp"
#include "pglayout/layout_io.hpp"
#include "pglayout/graph.hpp"
#include "pglayout/layout.hpp"
#include "pglayout/metrics.hpp"
#include "pglayout/rng.hpp"
#include "pglayout/synthetic.hpp"

#include <chrono>
#include <fstream>
#include <sstream>

#include "../include/pgl_b200.h"

using namespace pglayout;  // == pglref after the -D rename

namespace {

thread_local std::string g_err;

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        g_err.clear();
        return 0;
    } catch (const Error& e) {
        g_err = e.what();
        return static_cast<int>(e.kind()) + 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

LayoutConfig to_cfg(const pgl_layout_config* c) {
    LayoutConfig cfg;
    cfg.global_seed = c->global_seed;
    cfg.n_iters = c->n_iters;
    cfg.threads = c->threads;
    cfg.batch_size = c->batch_size;
    cfg.zipf_theta = c->zipf_theta;
    cfg.zipf_space_max = c->zipf_space_max;
    cfg.eta_min_eps = c->eta_min_eps;
    cfg.drf = c->drf;
    cfg.srf = c->srf;
    return cfg;
}

Layout layout_from(const PangenomeGraph& g, const double* coords) {
    Layout l(g);
    for (std::size_t n = 0; n < g.node_count(); ++n) {
        l.set(static_cast<NodeId>(n), Endpoint::start, {coords[4 * n], coords[4 * n + 1]});
        l.set(static_cast<NodeId>(n), Endpoint::end, {coords[4 * n + 2], coords[4 * n + 3]});
    }
    return l;
}

void snapshot_into(const Layout& l, double* out) {
    const std::vector<double> s = l.snapshot();
    std::memcpy(out, s.data(), s.size() * sizeof(double));
}

void report_into(const StressReport& r, pgl_stress_report* out) {
    out->mean = r.mean;
    out->n = r.n;
    out->std_dev = r.std_dev;
    out->ci_low = r.ci_low;
    out->ci_high = r.ci_high;
    out->skipped = r.skipped;
}

} // namespace

extern "C" {

typedef void (*pglref_cb)(uint32_t iter, const double* coords, double eta,
                          double secs, void* user);

const char* pglref_last_error(void) { return g_err.c_str(); }

// generate_synthetic_pangenome (synthetic.cpp:24); gfa_roundtrip = 1 writes
// it with write_gfa and parses it back with parse_gfa (config C1).
int pglref_generate(uint64_t seed, uint64_t backbone, uint32_t paths,
                    double rate, int gfa_roundtrip, void** out) {
    return guarded([&] {
        auto* g = new PangenomeGraph(
            generate_synthetic_pangenome(seed, backbone, paths, rate));
        if (gfa_roundtrip) {
            std::stringstream ss;
            write_gfa(*g, ss);
            auto* h = new PangenomeGraph(parse_gfa(ss));
            delete g;
            g = h;
        }
        *out = g;
    });
}

// parse_gfa (gfa.cpp:57-153) of an in-memory GFA text.
int pglref_parse_gfa(const char* data, uint64_t size, void** out, uint64_t* skipped) {
    return guarded([&] {
        std::stringstream ss(std::string(data, size));
        GfaParseStats st;
        *out = new PangenomeGraph(parse_gfa(ss, &st));
        if (skipped) *skipped = st.skipped_records;
    });
}

// parse_gfa from a file through std::ifstream, as the CLI does
// (tools/pglayout_main.cpp); secs = wall time of the parse.
int pglref_parse_gfa_file(const char* path, void** out, uint64_t* skipped, double* secs) {
    return guarded([&] {
        const auto t0 = std::chrono::steady_clock::now();
        std::ifstream in(path);
        if (!in) throw InvalidParameter(std::string("cannot open ") + path);
        GfaParseStats st;
        *out = new PangenomeGraph(parse_gfa(in, &st));
        if (skipped) *skipped = st.skipped_records;
        if (secs) *secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

// write_layout_tsv / read_layout_tsv (layout_io.cpp:31-110) through files.
int pglref_write_layout_tsv(const char* path, const double* coords, uint64_t n_nodes) {
    return guarded([&] {
        Layout l(n_nodes);
        for (uint64_t n = 0; n < n_nodes; ++n) {
            l.set(static_cast<NodeId>(n), Endpoint::start, {coords[4 * n], coords[4 * n + 1]});
            l.set(static_cast<NodeId>(n), Endpoint::end, {coords[4 * n + 2], coords[4 * n + 3]});
        }
        std::ofstream out(path);
        write_layout_tsv(l, out);
    });
}

int pglref_read_layout_tsv(const char* path, uint64_t* n_nodes, double* coords, uint64_t cap) {
    return guarded([&] {
        std::ifstream in(path);
        const Layout l = read_layout_tsv(in);
        *n_nodes = l.node_count();
        if (coords && 4 * l.node_count() <= cap) snapshot_into(l, coords);
    });
}

// write_gfa (gfa.cpp:155-178) to a file.
int pglref_write_gfa(void* gp, const char* path) {
    return guarded([&] {
        std::ofstream out(path);
        write_gfa(*static_cast<PangenomeGraph*>(gp), out);
        if (!out) throw InvalidParameter(std::string("cannot write ") + path);
    });
}

void pglref_edges(void* gp, uint32_t* from, uint8_t* from_end, uint32_t* to, uint8_t* to_end) {
    const auto& g = *static_cast<PangenomeGraph*>(gp);
    for (std::size_t k = 0; k < g.edges.size(); ++k) {
        from[k] = g.edges[k].from;
        to[k] = g.edges[k].to;
        from_end[k] = g.edges[k].from_end == Endpoint::end ? 1 : 0;
        to_end[k] = g.edges[k].to_end == Endpoint::end ? 1 : 0;
    }
}

const char* pglref_path_name(void* gp, uint32_t p) {
    return static_cast<PangenomeGraph*>(gp)->paths.at(p).name.c_str();
}

// build_graph (graph.cpp:7) from flat walks: step_rev[k] != 0 = reverse.
int pglref_build(uint64_t n_nodes, const uint64_t* node_len, uint32_t n_paths,
                 const uint64_t* path_n_steps, const uint32_t* step_node,
                 const uint8_t* step_rev, void** out) {
    return guarded([&] {
        std::vector<std::uint64_t> lens(node_len, node_len + n_nodes);
        std::vector<NamedWalk> walks(n_paths);
        std::uint64_t k = 0;
        for (uint32_t p = 0; p < n_paths; ++p) {
            walks[p].name = "p" + std::to_string(p);
            for (uint64_t s = 0; s < path_n_steps[p]; ++s, ++k)
                walks[p].steps.push_back(
                    {step_node[k], step_rev[k] ? Orientation::reverse : Orientation::forward});
        }
        *out = new PangenomeGraph(build_graph(std::move(lens), {}, std::move(walks)));
    });
}

void pglref_free(void* g) { delete static_cast<PangenomeGraph*>(g); }

// counts[0..4] = n_nodes, n_paths, total_steps, total_nucleotides, n_edges
void pglref_counts(void* gp, uint64_t* counts) {
    const auto& g = *static_cast<PangenomeGraph*>(gp);
    counts[0] = g.node_count();
    counts[1] = g.paths.size();
    counts[2] = g.total_steps();
    counts[3] = g.total_nucleotides();
    counts[4] = g.edges.size();
}

// Flat export of the index (graph.hpp:35-48, cum_steps graph.hpp:75-76).
void pglref_export(void* gp, uint64_t* node_len, uint64_t* cum_steps,
                   uint64_t* path_total_len, uint32_t* step_node,
                   uint8_t* step_rev, uint64_t* step_offset, uint32_t* step_len) {
    const auto& g = *static_cast<PangenomeGraph*>(gp);
    for (std::size_t n = 0; n < g.node_count(); ++n) node_len[n] = g.nodes[n].seq_len;
    const auto& cum = g.cum_steps();
    for (std::size_t p = 0; p < cum.size(); ++p) cum_steps[p] = cum[p];
    std::uint64_t k = 0;
    for (std::size_t p = 0; p < g.paths.size(); ++p) {
        path_total_len[p] = g.paths[p].total_len;
        for (const PathStep& st : g.paths[p].steps) {
            step_node[k] = st.node_id;
            step_rev[k] = st.orient == Orientation::reverse ? 1 : 0;
            step_offset[k] = st.offset;
            step_len[k] = st.seq_len;
            ++k;
        }
    }
}

// path_position (graph.hpp:98-109) for every (step, endpoint): out[2k] start, out[2k+1] end.
void pglref_positions(void* gp, uint64_t* out) {
    const auto& g = *static_cast<PangenomeGraph*>(gp);
    std::uint64_t k = 0;
    for (const Path& p : g.paths)
        for (std::size_t s = 0; s < p.steps.size(); ++s, ++k) {
            out[2 * k] = path_position(p, s, Endpoint::start);
            out[2 * k + 1] = path_position(p, s, Endpoint::end);
        }
}

int pglref_run_layout(void* gp, const pgl_layout_config* c, int reuse,
                      double* out_coords, uint64_t* stats8, pglref_cb cb,
                      void* user, double* iter_secs) {
    return guarded([&] {
        const auto& g = *static_cast<PangenomeGraph*>(gp);
        const LayoutConfig cfg = to_cfg(c);
        RunStats st;
        IterationCallback on_iter;
        if (cb || iter_secs) {
            on_iter = [&](std::uint32_t iter, const Layout& l, double eta, double secs) {
                if (iter_secs) iter_secs[iter] = secs;
                if (cb) {
                    const std::vector<double> s = l.snapshot();
                    cb(iter, s.data(), eta, secs, user);
                }
            };
        }
        const Layout out = reuse ? run_layout_reuse(g, cfg, on_iter, &st)
                                 : run_layout(g, cfg, on_iter, &st);
        if (out_coords) snapshot_into(out, out_coords);
        if (stats8) {
            const std::uint64_t v[8] = {st.primary_steps, st.updates_attempted,
                                        st.updates_applied, st.updates_skipped,
                                        st.batches_first_half, st.batches_first_half_cooling,
                                        st.batches_second_half, st.batches_second_half_cooling};
            std::memcpy(stats8, v, sizeof v);
        }
    });
}

int pglref_init_layout(void* gp, uint64_t seed, double* out) {
    return guarded([&] { snapshot_into(init_layout(*static_cast<PangenomeGraph*>(gp), seed), out); });
}

int pglref_make_schedule(void* gp, const pgl_layout_config* c, double* etas,
                         double* eta_max_min_lambda) {
    return guarded([&] {
        const SgdSchedule s = make_schedule(*static_cast<PangenomeGraph*>(gp), to_cfg(c));
        for (std::size_t t = 0; t < s.etas.size(); ++t) etas[t] = s.etas[t];
        if (eta_max_min_lambda) {
            eta_max_min_lambda[0] = s.eta_max;
            eta_max_min_lambda[1] = s.eta_min;
            eta_max_min_lambda[2] = s.lambda;
        }
    });
}

int pglref_make_eta_schedule(double eta_max, double eta_min, uint32_t n, double* etas) {
    return guarded([&] {
        const SgdSchedule s = make_eta_schedule(eta_max, eta_min, n);
        for (std::size_t t = 0; t < s.etas.size(); ++t) etas[t] = s.etas[t];
    });
}

int pglref_sampled_path_stress(void* gp, const double* coords, uint64_t seed,
                               uint32_t spn, pgl_stress_report* out) {
    return guarded([&] {
        const auto& g = *static_cast<PangenomeGraph*>(gp);
        report_into(sampled_path_stress(g, layout_from(g, coords), seed, spn), out);
    });
}

int pglref_exact_path_stress(void* gp, const double* coords, pgl_stress_report* out) {
    return guarded([&] {
        const auto& g = *static_cast<PangenomeGraph*>(gp);
        report_into(exact_path_stress(g, layout_from(g, coords)), out);
    });
}

// Raw xoshiro256+ outputs of seed_worker(seed, worker) (rng.hpp:21-71).
void pglref_rng_draws(uint64_t seed, uint64_t worker, uint64_t count, uint64_t* out) {
    RngState r = seed_worker(seed, worker);
    for (uint64_t i = 0; i < count; ++i) out[i] = r.next();
}

void pglref_rng_state(uint64_t seed, uint64_t worker, uint64_t* s4) {
    const RngState r = seed_worker(seed, worker);
    for (int i = 0; i < 4; ++i) s4[i] = r.s[i];
}

int pglref_zipf_samples(uint64_t n, double theta, uint64_t seed, uint64_t worker,
                        uint64_t count, uint64_t* out) {
    return guarded([&] {
        ZipfSampler z({n, theta});
        RngState r = seed_worker(seed, worker);
        for (uint64_t i = 0; i < count; ++i) out[i] = z.sample(r);
    });
}

int pglref_weighted_select(void* gp, uint64_t seed, uint64_t worker, uint64_t count,
                           uint32_t* path, uint64_t* step) {
    return guarded([&] {
        const auto& g = *static_cast<PangenomeGraph*>(gp);
        RngState r = seed_worker(seed, worker);
        for (uint64_t i = 0; i < count; ++i) {
            const StepSelection s = weighted_step_select(r, g);
            path[i] = s.path_index;
            step[i] = s.step_index;
        }
    });
}

// apply_endpoint_update (engine.cpp:276-306) on a 4*n coordinate array;
// rng state s4 is read and written back. Returns outcome in *applied.
int pglref_apply_update(double* coords, uint64_t n_nodes, uint32_t ni, int ei_end,
                        uint32_t nj, int ej_end, double d_ref, double eta,
                        uint64_t* s4, int* applied) {
    return guarded([&] {
        Layout l(n_nodes);
        for (std::size_t n = 0; n < n_nodes; ++n) {
            l.set(static_cast<NodeId>(n), Endpoint::start, {coords[4 * n], coords[4 * n + 1]});
            l.set(static_cast<NodeId>(n), Endpoint::end, {coords[4 * n + 2], coords[4 * n + 3]});
        }
        RngState r;
        for (int i = 0; i < 4; ++i) r.s[i] = s4[i];
        const StepOutcome o = apply_endpoint_update(
            l, ni, ei_end ? Endpoint::end : Endpoint::start, nj,
            ej_end ? Endpoint::end : Endpoint::start, d_ref, eta, r);
        for (int i = 0; i < 4; ++i) s4[i] = r.s[i];
        snapshot_into(l, coords);
        *applied = o == StepOutcome::applied;
    });
}

// layout_step (engine.cpp:308-321) repeated `count` times from a seeded stream;
// applied[k] receives each outcome. coords in/out.
int pglref_layout_steps(void* gp, double* coords, uint64_t seed, uint64_t worker,
                        double eta, int cooling, const pgl_layout_config* c,
                        uint64_t count, uint8_t* applied) {
    return guarded([&] {
        const auto& g = *static_cast<PangenomeGraph*>(gp);
        Layout l = layout_from(g, coords);
        RngState r = seed_worker(seed, worker);
        const LayoutConfig cfg = to_cfg(c);
        for (uint64_t k = 0; k < count; ++k)
            applied[k] = layout_step(g, l, r, eta, cooling != 0, cfg) == StepOutcome::applied;
        snapshot_into(l, coords);
    });
}

} // extern "C"
