// integration/pglayout_b200_io.cpp — drop-in replacement for the
// reference's src/gfa.cpp and src/layout_io.cpp (include/pglayout/gfa.hpp,
// layout_io.hpp), on libpgl_b200.so's multithreaded host IO:
//   parse_gfa          -> pgl_gfa_parse_buffer (mmap-free: the stream is read
//                         once into memory), then the reference's own
//                         build_graph on the parsed walks (same graph, same
//                         exception classes and messages)
//   write_gfa          -> written here from the model (gfa.hpp:24-27 contract:
//                         star sequences + LN tags, 0M overlaps, 1-based names)
//   write_layout_tsv   -> pgl_layout_format_tsv (byte-identical rows)
//   read_layout_tsv    -> pgl_layout_parse_tsv
#include <iterator>
#include <istream>
#include <ostream>
#include <string>
#include <vector>

#include "pglayout/gfa.hpp"
#include "pglayout/layout_io.hpp"
#include "pgl_facade_errors.hpp"

namespace pglayout {

namespace {

std::string slurp(std::istream& in) {
    return std::string(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
}

struct GfaHandle {
    pgl_gfa* g = nullptr;
    ~GfaHandle() { pgl_gfa_free(g); }
};

}  // namespace

PangenomeGraph parse_gfa(std::istream& in, GfaParseStats* stats) {
    const std::string text = slurp(in);
    GfaHandle h;
    b200::check(pgl_gfa_parse_buffer(text.data(), text.size(), 0, &h.g));
    pgl_gfa_info info;
    b200::check(pgl_gfa_info_get(h.g, &info));
    pgl_graph_view v;
    b200::check(pgl_gfa_view(h.g, &v));
    std::vector<std::uint64_t> lengths(v.node_len, v.node_len + v.n_nodes);
    std::vector<pgl_edge> ce(info.n_edges);
    if (info.n_edges) b200::check(pgl_gfa_edges(h.g, ce.data()));
    std::vector<Edge> edges(info.n_edges);
    for (std::size_t k = 0; k < ce.size(); ++k)
        edges[k] = Edge{ce[k].from, ce[k].from_end ? Endpoint::end : Endpoint::start, ce[k].to,
                        ce[k].to_end ? Endpoint::end : Endpoint::start};
    std::vector<NamedWalk> walks(v.n_paths);
    for (uint32_t p = 0; p < v.n_paths; ++p) {
        walks[p].name = pgl_gfa_path_name(h.g, p);
        walks[p].steps.resize(v.path_n_steps[p]);
        const pgl_path_step* s = v.path_steps[p];
        for (std::uint64_t k = 0; k < v.path_n_steps[p]; ++k)
            walks[p].steps[k] = WalkStep{s[k].node_id, s[k].orient ? Orientation::reverse : Orientation::forward};
    }
    if (stats) stats->skipped_records = info.skipped_records;
    return build_graph(std::move(lengths), std::move(edges), std::move(walks));
}

void write_gfa(const PangenomeGraph& g, std::ostream& out) {
    std::string s = "H\tVN:Z:1.0\n";
    for (std::size_t i = 0; i < g.node_count(); ++i)
        s += "S\t" + std::to_string(i + 1) + "\t*\tLN:i:" + std::to_string(g.nodes[i].seq_len) + "\n";
    for (const Edge& e : g.edges) {
        s += "L\t" + std::to_string(e.from + 1) + (e.from_end == Endpoint::end ? "\t+\t" : "\t-\t") +
             std::to_string(e.to + 1) + (e.to_end == Endpoint::start ? "\t+\t0M\n" : "\t-\t0M\n");
    }
    for (const Path& p : g.paths) {
        s += "P\t" + p.name + '\t';
        for (std::size_t k = 0; k < p.steps.size(); ++k) {
            if (k) s += ',';
            s += std::to_string(p.steps[k].node_id + 1);
            s += p.steps[k].orient == Orientation::forward ? '+' : '-';
        }
        s += "\t*\n";
    }
    out << s;
}

void write_layout_tsv(const Layout& layout, std::ostream& out) {
    const std::vector<double> c = layout.snapshot();
    char* text = nullptr;
    std::uint64_t size = 0;
    b200::check(pgl_layout_format_tsv(c.data(), layout.node_count(), 0, &text, &size));
    out.write(text, static_cast<std::streamsize>(size));
    pgl_free(text);
}

Layout read_layout_tsv(std::istream& in) {
    const std::string text = slurp(in);
    std::uint64_t n = 0;
    double* c = nullptr;
    b200::check(pgl_layout_parse_tsv(text.data(), text.size(), 0, &n, &c));
    Layout layout(n);
    for (std::uint64_t i = 0; i < n; ++i) {
        layout.set(static_cast<NodeId>(i), Endpoint::start, {c[4 * i], c[4 * i + 1]});
        layout.set(static_cast<NodeId>(i), Endpoint::end, {c[4 * i + 2], c[4 * i + 3]});
    }
    pgl_free(c);
    return layout;
}

}  // namespace pglayout
