// integration/pglayout_b200_metrics.cpp — drop-in replacement for the
// reference's src/metrics.cpp (include/pglayout/metrics.hpp) on the GPU:
//   sampled_path_stress   -> pgl_sampled_path_stress(PGL_SPS_STREAM): the
//                            documented per-path stream (seed_worker(seed,
//                            2^61 + path)) replayed in parallel on the device,
//                            i.e. the reference's own terms; n and skipped
//                            identical, mean/sd to ~1e-15
//   exact_path_stress     -> pgl_exact_path_stress: every step pair on the
//                            device, bit-identical terms, double-double sums
//   report_tsv, pair_stress, step_pair_stress, correlation_harness: host
//                            (metrics.hpp:22-66 contracts; the harness calls
//                            the two device metrics above)
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "pglayout/metrics.hpp"
#include "pgl_facade_errors.hpp"

namespace pglayout {

namespace {

static_assert(sizeof(PathStep) == sizeof(pgl_path_step), "PathStep ABI");

struct View {  // zero-copy pgl_graph_view of a PangenomeGraph
    std::vector<uint64_t> node_len, n_steps, totals;
    std::vector<const pgl_path_step*> steps;
    pgl_graph_view v{};
    explicit View(const PangenomeGraph& g) {
        for (const NodeRecord& n : g.nodes) node_len.push_back(n.seq_len);
        for (const Path& p : g.paths) {
            steps.push_back(reinterpret_cast<const pgl_path_step*>(p.steps.data()));
            n_steps.push_back(p.steps.size());
            totals.push_back(p.total_len);
        }
        v.n_nodes = g.node_count();
        v.node_len = node_len.data();
        v.n_paths = static_cast<uint32_t>(g.paths.size());
        v.path_steps = steps.data();
        v.path_n_steps = n_steps.data();
        v.path_total_len = totals.data();
    }
};

StressReport from_c(const pgl_stress_report& r) {
    StressReport s;
    s.mean = r.mean;
    s.n = r.n;
    s.std_dev = r.std_dev;
    s.ci_low = r.ci_low;
    s.ci_high = r.ci_high;
    s.skipped = r.skipped;
    return s;
}

int device() {
    const char* d = std::getenv("PGLAYOUT_B200_DEVICE");
    return d ? std::atoi(d) : 0;
}

uint64_t path_pos(const PathStep& s, Endpoint e) {  // path_position, graph.hpp:98-109
    const bool far = (s.orient == Orientation::forward) == (e == Endpoint::end);
    return far ? s.offset + s.seq_len : s.offset;
}

}  // namespace

std::string report_tsv(const StressReport& r) {
    char buf[256];
    std::snprintf(buf, sizeof buf, "%.9g\t%llu\t%.9g\t%.9g\t%.9g\t%llu", r.mean,
                  static_cast<unsigned long long>(r.n), r.std_dev, r.ci_low, r.ci_high,
                  static_cast<unsigned long long>(r.skipped));
    return buf;
}

double pair_stress(Vec2 v_i, Vec2 v_j, double d_ref) {
    if (!(d_ref > 0.0)) throw ZeroReference("pair_stress needs a positive reference distance");
    const double e = ((v_i - v_j).norm() - d_ref) / d_ref;
    return e * e;
}

std::optional<double> step_pair_stress(const Path& path, std::uint64_t i, std::uint64_t j, const Layout& layout) {
    if (i >= path.steps.size() || j >= path.steps.size())
        throw IndexOutOfRange("step pair (" + std::to_string(i) + ", " + std::to_string(j) + ") in path '" +
                              path.name + "'");
    double sum = 0.0;
    int count = 0;
    for (Endpoint ei : {Endpoint::start, Endpoint::end})
        for (Endpoint ej : {Endpoint::start, Endpoint::end}) {
            const uint64_t a = path_pos(path.steps[i], ei), b = path_pos(path.steps[j], ej);
            if (a == b) continue;
            sum += pair_stress(layout.get(path.steps[i].node_id, ei), layout.get(path.steps[j].node_id, ej),
                               static_cast<double>(a > b ? a - b : b - a));
            ++count;
        }
    if (!count) return std::nullopt;
    return sum / count;
}

StressReport exact_path_stress(const PangenomeGraph& g, const Layout& layout) {
    const View view(g);
    const std::vector<double> c = layout.snapshot();
    pgl_stress_report r;
    b200::check(pgl_exact_path_stress(device(), &view.v, c.data(), &r));
    return from_c(r);
}

StressReport sampled_path_stress(const PangenomeGraph& g, const Layout& layout, std::uint64_t seed,
                                 std::uint32_t samples_per_node) {
    if (samples_per_node < 1) throw InvalidParameter("samples_per_node must be >= 1");
    const View view(g);
    const std::vector<double> c = layout.snapshot();
    pgl_stress_report r;
    b200::check(pgl_sampled_path_stress(device(), &view.v, c.data(), seed, samples_per_node, PGL_SPS_STREAM, &r));
    return from_c(r);
}

CorrelationReport correlation_harness(const std::vector<const PangenomeGraph*>& graphs,
                                      const std::vector<const Layout*>& layouts, std::uint64_t seed,
                                      std::uint32_t samples_per_node) {
    if (graphs.size() != layouts.size())
        throw CountMismatch("harness got " + std::to_string(graphs.size()) + " graphs but " +
                            std::to_string(layouts.size()) + " layouts");
    constexpr std::uint64_t kExactLimit = 10000;  // metrics.hpp:59-61
    CorrelationReport rep;
    for (std::size_t k = 0; k < graphs.size(); ++k) {
        if (graphs[k]->total_steps() > kExactLimit)
            throw CorpusTooLarge("graph " + std::to_string(k) + " has " + std::to_string(graphs[k]->total_steps()) +
                                 " steps; the exact metric is quadratic and capped at " + std::to_string(kExactLimit));
        const double exact = exact_path_stress(*graphs[k], *layouts[k]).mean;
        const double sampled = sampled_path_stress(*graphs[k], *layouts[k], seed + k, samples_per_node).mean;
        rep.points.emplace_back(exact, sampled);
        rep.max_relative_deviation =
            std::max(rep.max_relative_deviation, std::abs(sampled - exact) / std::max(std::abs(exact), 1e-12));
    }
    const std::size_t n = rep.points.size();
    if (n >= 2) {  // Pearson r of (exact, sampled)
        double mx = 0.0, my = 0.0;
        for (const auto& pt : rep.points) {
            mx += pt.first;
            my += pt.second;
        }
        mx /= static_cast<double>(n);
        my /= static_cast<double>(n);
        double sxx = 0.0, syy = 0.0, sxy = 0.0;
        for (const auto& pt : rep.points) {
            sxx += (pt.first - mx) * (pt.first - mx);
            syy += (pt.second - my) * (pt.second - my);
            sxy += (pt.first - mx) * (pt.second - my);
        }
        if (sxx > 0.0 && syy > 0.0) rep.pearson_r = sxy / std::sqrt(sxx * syy);
    }
    return rep;
}

}  // namespace pglayout
