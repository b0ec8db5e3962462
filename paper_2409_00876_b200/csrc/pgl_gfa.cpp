// pgl_gfa.cpp — multithreaded GFA ingest: the drop-in for parse_gfa
// (src/gfa.cpp:57-153) followed by build_graph (src/graph.cpp:7-59).
//
// The reference slurps every line into a vector<string> and parses serially
// (two passes: S records, then L/P/W/other). Here the file is mmap'd and
// every phase runs on all host threads over line-aligned chunks:
//   A  per chunk: line count, S and L record counts, P line list, W lines,
//      skipped-record count (the classification of gfa.cpp:96-153);
//   B  S records: ids = declaration order (chunk prefix sums), lengths
//      (segment_length, gfa.cpp:33-47), first error per chunk;
//   C  name -> id: a direct table when every segment name is a decimal
//      integer (write_gfa output and most pangenome tools), otherwise a
//      lock-free open-addressing hash table; duplicates keep the first
//      declaration and report the second, as the serial pass would;
//   D  L records in parallel, edges written at their line-order index;
//   E  P records cut into comma-aligned pieces of ~1 MiB: count, then parse
//      tokens into PathStep node/orientation at prefix-sum positions, then
//      per-path offsets by a piece-level scan (graph.cpp:38-50).
// Errors: the reference throws the first failure it meets; here every
// phase keeps the smallest (line, token) failure and the same precedence is
// applied at the end (pass 1 before pass 2, NoPaths, then build_graph), with
// the reference's exception classes and messages.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <charconv>
#include <cstring>
#include <limits>
#include <memory>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#include "pgl_internal.hpp"

namespace pgl {

namespace {

constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr uint64_t kNoLine = std::numeric_limits<uint64_t>::max();

template <typename F>
void run_threads(unsigned T, F&& f) {
    if (T <= 1) {
        f(0u);
        return;
    }
    std::vector<std::thread> pool;
    pool.reserve(T);
    for (unsigned t = 0; t < T; ++t) pool.emplace_back([&, t] { f(t); });
    for (auto& th : pool) th.join();
}

// First failure seen by a worker: (line, position within the line) orders
// failures exactly as the serial parser would meet them.
struct Fail {
    uint64_t line = kNoLine;
    uint64_t pos = 0;
    int type = 0;
    std::string msg;
    void offer(uint64_t l, uint64_t p, int t, std::string m) {
        if (l < line || (l == line && p < pos)) {
            line = l;
            pos = p;
            type = t;
            msg = std::move(m);
        }
    }
    void merge(const Fail& o) {
        if (o.line != kNoLine) offer(o.line, o.pos, o.type, o.msg);
    }
};

std::string line_msg(uint64_t ln, const std::string& why) { return "line " + std::to_string(ln) + ": " + why; }

// one line of the buffer: [b, e) without the '\n' and one trailing '\r'
struct Line {
    const char* b;
    const char* e;
};

// column k (tab separated) of a line, and whether it exists
inline bool column(Line l, int k, std::string_view& out) {
    const char* p = l.b;
    for (int c = 0; c < k; ++c) {
        const void* t = std::memchr(p, '\t', l.e - p);
        if (!t) return false;
        p = static_cast<const char*>(t) + 1;
    }
    const void* t = std::memchr(p, '\t', l.e - p);
    out = std::string_view(p, (t ? static_cast<const char*>(t) : l.e) - p);
    return true;
}

inline std::string_view first_col(Line l) {
    const void* t = std::memchr(l.b, '\t', l.e - l.b);
    return std::string_view(l.b, (t ? static_cast<const char*>(t) : l.e) - l.b);
}

inline size_t n_cols(Line l) {
    size_t n = 1;
    for (const char* p = l.b; p < l.e;) {
        const void* t = std::memchr(p, '\t', l.e - p);
        if (!t) break;
        ++n;
        p = static_cast<const char*>(t) + 1;
    }
    return n;
}

uint64_t hash_name(std::string_view s) {
    uint64_t h = 0x9E3779B97F4A7C15ULL ^ s.size();
    size_t i = 0;
    for (; i + 8 <= s.size(); i += 8) {
        uint64_t w;
        std::memcpy(&w, s.data() + i, 8);
        h = (h ^ w) * 0xBF58476D1CE4E5B9ULL;
        h ^= h >> 31;
    }
    uint64_t w = 0;
    std::memcpy(&w, s.data() + i, s.size() - i);
    h = (h ^ w) * 0x94D049BB133111EBULL;
    return h ^ (h >> 29);
}

struct Chunk {
    const char* b;
    const char* e;
    uint64_t line0 = 0;  // 1-based number of the chunk's first line
    uint64_t lines = 0, n_s = 0, n_l = 0, skipped = 0;
    uint64_t s_base = 0, l_base = 0;
    std::vector<std::pair<uint64_t, Line>> p_lines;  // (line number, line)
    Fail pass1, pass2;
};

template <typename F>
void for_lines(const Chunk& c, F&& f) {  // f(line number, Line)
    uint64_t ln = c.line0;
    for (const char* p = c.b; p < c.e; ++ln) {
        const void* nl = std::memchr(p, '\n', c.e - p);
        const char* e = nl ? static_cast<const char*>(nl) : c.e;
        Line l{p, e};
        if (l.e > l.b && l.e[-1] == '\r') --l.e;
        f(ln, l);
        p = nl ? e + 1 : c.e;
    }
}

struct Piece {  // a comma-aligned slice of one P line's step list
    uint32_t path;
    const char* b;
    const char* e;
    bool last;          // ends at the end of the step list
    uint64_t tok0 = 0;  // index of the piece's first token within its path
    uint64_t n_tok = 0;
    uint64_t len_sum = 0;
    Fail fail;
};

}  // namespace

struct GfaGraph {
    bool compact = false;                // compact mode: steps as u32 node | reverse << 31 only
    std::vector<uint32_t> csteps;        // compact: [S] in path order
    std::vector<uint64_t> path_begin;    // compact: [P+1] cum_steps
    std::vector<uint64_t> node_len;
    std::vector<std::string> path_names;
    std::vector<std::vector<pgl_path_step>> paths;
    std::vector<const pgl_path_step*> path_ptrs;
    std::vector<uint64_t> path_n, path_total;
    std::vector<pgl_edge> edges;
    uint64_t skipped = 0, total_steps = 0;
};

GfaGraph* gfa_parse_buffer(const char* data, uint64_t size, unsigned threads, bool compact) {
    // ~4 MiB of text per thread at least: thread start-up costs more than
    // parsing a small file
    const unsigned want = std::max(1u, std::min(threads ? threads : std::thread::hardware_concurrency(), 256u));
    const unsigned T = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(want, size >> 22)));
    // ---- chunks at line boundaries ----
    const unsigned NC = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(4ull * T, size / 4096 + 1)));
    std::vector<Chunk> ch(NC);
    {
        const char* end = data + size;
        const char* prev = data;
        for (unsigned k = 0; k < NC; ++k) {
            const char* cut = k + 1 == NC ? end : data + size * (k + 1) / NC;
            if (cut < prev) cut = prev;
            if (cut < end) {
                const void* nl = std::memchr(cut, '\n', end - cut);
                cut = nl ? static_cast<const char*>(nl) + 1 : end;
            }
            ch[k].b = prev;
            ch[k].e = cut;
            prev = cut;
        }
    }
    std::atomic<unsigned> next{0};
    auto each_chunk = [&](auto&& f) {
        next = 0;
        run_threads(T, [&](unsigned) {
            for (unsigned k; (k = next.fetch_add(1)) < NC;) f(ch[k]);
        });
    };
    // ---- A: classify (gfa.cpp:73-76, :96-153) ----
    each_chunk([&](Chunk& c) {
        for (const char* p = c.b; p < c.e;) {
            const void* nl = std::memchr(p, '\n', c.e - p);
            ++c.lines;
            p = nl ? static_cast<const char*>(nl) + 1 : c.e;
        }
    });
    {
        uint64_t ln = 1;
        for (auto& c : ch) {
            c.line0 = ln;
            ln += c.lines;
        }
    }
    each_chunk([&](Chunk& c) {
        for_lines(c, [&](uint64_t ln, Line l) {
            if (l.b == l.e) return;
            const std::string_view type = first_col(l);
            if (type == "S") {
                ++c.n_s;
                return;
            }
            if (type == "H" || (!type.empty() && type[0] == '#')) return;
            if (type == "W") {
                c.pass2.offer(ln, 0, PGL_ERR_MALFORMED_LINE,
                              line_msg(ln, "W (walk) records are not supported; convert walks to P lines first"));
                return;
            }
            if (type == "L") {
                ++c.n_l;
                return;
            }
            if (type == "P") {
                c.p_lines.emplace_back(ln, l);
                return;
            }
            ++c.skipped;
        });
    });
    uint64_t V = 0, E = 0, skipped = 0;
    for (auto& c : ch) {
        c.s_base = V;
        c.l_base = E;
        V += c.n_s;
        E += c.n_l;
        skipped += c.skipped;
    }
    if (V >= kNone) raise(PGL_ERR_INVALID_PARAMETER, "too many segments for 32-bit node ids");

    // ---- B: segments (pass 1, gfa.cpp:67-82) ----
    std::vector<std::string_view> names(V);
    std::vector<uint64_t> s_line(V);
    auto* G = new GfaGraph;
    std::unique_ptr<GfaGraph> own(G);
    G->node_len.assign(V, 0);
    each_chunk([&](Chunk& c) {
        uint64_t id = c.s_base;
        for_lines(c, [&](uint64_t ln, Line l) {
            if (l.b == l.e || *l.b != 'S' || first_col(l) != "S") return;
            const uint64_t my = id++;
            s_line[my] = ln;
            std::string_view name, seq;
            if (!column(l, 2, seq)) {
                c.pass1.offer(ln, 0, PGL_ERR_MALFORMED_LINE, line_msg(ln, "S record needs name and sequence"));
                return;
            }
            column(l, 1, name);
            names[my] = name;
            if (name.empty()) {
                c.pass1.offer(ln, 0, PGL_ERR_MALFORMED_LINE, line_msg(ln, "empty segment name"));
                return;
            }
            uint64_t len = 0;
            if (seq != "*") {
                len = seq.size();
            } else {  // segment_length: the first LN:i tag (gfa.cpp:33-47)
                bool found = false;
                std::string_view col;
                for (int k = 3; column(l, k, col); ++k) {
                    if (col.substr(0, 5) != "LN:i:") continue;
                    const std::string_view v = col.substr(5);
                    const auto r = std::from_chars(v.data(), v.data() + v.size(), len);
                    if (r.ec != std::errc{} || r.ptr != v.data() + v.size() || len == 0) {
                        c.pass1.offer(ln, 1, PGL_ERR_MALFORMED_LINE,
                                      line_msg(ln, "bad LN tag value '" + std::string(v) + "'"));
                        return;
                    }
                    found = true;
                    break;
                }
                if (!found) {
                    c.pass1.offer(ln, 1, PGL_ERR_MALFORMED_LINE,
                                  line_msg(ln, "segment with '*' sequence needs an LN:i tag"));
                    return;
                }
            }
            if (len == 0) {
                c.pass1.offer(ln, 1, PGL_ERR_MALFORMED_LINE, line_msg(ln, "zero-length segment"));
                return;
            }
            G->node_len[my] = len;
        });
    });

    // ---- C: name -> id (first declaration wins; the second is the error) ----
    // numeric fast path: decimal names without leading zeros
    std::atomic<bool> numeric{true};
    std::atomic<uint64_t> max_num{0};
    {
        std::atomic<uint64_t> nx{0};
        run_threads(T, [&](unsigned) {
            uint64_t mx = 0;
            bool ok = true;
            for (uint64_t b; ok && (b = nx.fetch_add(1 << 16)) < V;) {
                for (uint64_t i = b; i < std::min<uint64_t>(V, b + (1 << 16)); ++i) {
                    const std::string_view s = names[i];
                    uint64_t v = 0;
                    const auto r = std::from_chars(s.data(), s.data() + s.size(), v);
                    if (s.empty() || r.ec != std::errc{} || r.ptr != s.data() + s.size() || (s[0] == '0' && s.size() > 1) ||
                        v > 8 * V + 1024) {
                        ok = false;
                        break;
                    }
                    mx = std::max(mx, v);
                }
            }
            if (!ok) numeric = false;
            uint64_t cur = max_num.load();
            while (mx > cur && !max_num.compare_exchange_weak(cur, mx)) {
            }
        });
    }
    std::vector<std::atomic<uint32_t>> table;
    uint64_t mask = 0;
    const bool num = numeric.load() && V > 0;
    table = std::vector<std::atomic<uint32_t>>(num ? max_num.load() + 1 : [&] {
        uint64_t cap = 16;
        while (cap < 2 * V) cap <<= 1;
        mask = cap - 1;
        return cap;
    }());
    {
        std::atomic<uint64_t> nx{0};
        run_threads(T, [&](unsigned) {
            for (uint64_t b; (b = nx.fetch_add(1 << 14)) < table.size();)
                for (uint64_t i = b; i < std::min<uint64_t>(table.size(), b + (1 << 14)); ++i)
                    table[i].store(kNone, std::memory_order_relaxed);
        });
    }
    std::vector<Fail> dup_fail(T);
    {
        std::atomic<uint64_t> nx{0};
        run_threads(T, [&](unsigned t) {
            auto lost = [&](uint32_t id) {
                dup_fail[t].offer(s_line[id], 0, PGL_ERR_MALFORMED_LINE,
                                  line_msg(s_line[id], "duplicate segment '" + std::string(names[id]) + "'"));
            };
            for (uint64_t b; (b = nx.fetch_add(1 << 14)) < V;) {
                for (uint64_t i = b; i < std::min<uint64_t>(V, b + (1 << 14)); ++i) {
                    if (names[i].empty()) continue;
                    uint32_t id = static_cast<uint32_t>(i);
                    uint64_t slot;
                    if (num) {
                        uint64_t v = 0;
                        std::from_chars(names[i].data(), names[i].data() + names[i].size(), v);
                        slot = v;
                    } else {
                        slot = hash_name(names[i]) & mask;
                    }
                    for (;;) {
                        uint32_t cur = table[slot].load(std::memory_order_acquire);
                        if (cur == kNone) {
                            if (table[slot].compare_exchange_strong(cur, id, std::memory_order_acq_rel)) break;
                        }
                        if (cur == kNone) continue;
                        if (num || names[cur] == names[id]) {  // same name: keep the smaller id
                            if (cur < id) {
                                lost(id);
                                break;
                            }
                            if (table[slot].compare_exchange_strong(cur, id, std::memory_order_acq_rel)) {
                                lost(cur);
                                break;
                            }
                            continue;
                        }
                        slot = (slot + 1) & mask;
                    }
                }
            }
        });
    }
    Fail p1;
    for (auto& c : ch) p1.merge(c.pass1);
    for (auto& f : dup_fail) p1.merge(f);
    if (p1.line != kNoLine) raise(p1.type, p1.msg);

    auto resolve = [&](std::string_view name) -> uint32_t {
        if (num) {
            uint64_t v = 0;
            const auto r = std::from_chars(name.data(), name.data() + name.size(), v);
            if (name.empty() || r.ec != std::errc{} || r.ptr != name.data() + name.size() ||
                (name[0] == '0' && name.size() > 1) || v >= table.size())
                return kNone;
            return table[v].load(std::memory_order_relaxed);
        }
        for (uint64_t slot = hash_name(name) & mask;; slot = (slot + 1) & mask) {
            const uint32_t cur = table[slot].load(std::memory_order_relaxed);
            if (cur == kNone) return kNone;
            if (names[cur] == name) return cur;
        }
    };
    auto unknown = [](uint64_t ln, std::string_view name) {
        return "line " + std::to_string(ln) + " references undeclared segment '" + std::string(name) + "'";
    };

    // ---- D: L records (gfa.cpp:110-127) ----
    G->edges.resize(E);
    each_chunk([&](Chunk& c) {
        uint64_t k = c.l_base;
        for_lines(c, [&](uint64_t ln, Line l) {
            if (l.b == l.e || *l.b != 'L' || first_col(l) != "L") return;
            pgl_edge& e = G->edges[k++];
            std::memset(&e, 0, sizeof e);
            if (n_cols(l) < 6) {
                c.pass2.offer(ln, 0, PGL_ERR_MALFORMED_LINE, line_msg(ln, "L record needs 6 columns"));
                return;
            }
            std::string_view a, oa, b, ob;
            column(l, 1, a);
            column(l, 2, oa);
            column(l, 3, b);
            column(l, 4, ob);
            if (oa.size() != 1 || ob.size() != 1) {
                c.pass2.offer(ln, 0, PGL_ERR_MALFORMED_LINE, line_msg(ln, "bad orientation column"));
                return;
            }
            const uint32_t from = resolve(a);
            if (from == kNone) {
                c.pass2.offer(ln, 0, PGL_ERR_UNKNOWN_SEGMENT, unknown(ln, a));
                return;
            }
            const uint32_t to = resolve(b);
            if (to == kNone) {
                c.pass2.offer(ln, 0, PGL_ERR_UNKNOWN_SEGMENT, unknown(ln, b));
                return;
            }
            for (const char o : {oa[0], ob[0]})
                if (o != '+' && o != '-') {
                    c.pass2.offer(ln, 0, PGL_ERR_MALFORMED_LINE, line_msg(ln, std::string("bad orientation '") + o + "'"));
                    return;
                }
            // a forward source attaches at its end, a forward target at its start
            e.from = from;
            e.to = to;
            e.from_end = oa[0] == '+' ? 1 : 0;
            e.to_end = ob[0] == '+' ? 0 : 1;
        });
    });

    // ---- E: P records (gfa.cpp:128-150) ----
    std::vector<std::pair<uint64_t, Line>> plines;
    for (auto& c : ch) plines.insert(plines.end(), c.p_lines.begin(), c.p_lines.end());
    const uint32_t P = static_cast<uint32_t>(plines.size());
    G->path_names.resize(P);
    std::vector<Fail> pfail(P);  // per-line failure (pass 2 order within the line)
    std::vector<Piece> pieces;
    constexpr uint64_t kPiece = 1 << 20;
    for (uint32_t p = 0; p < P; ++p) {
        const uint64_t ln = plines[p].first;
        const Line l = plines[p].second;
        if (n_cols(l) < 4) {
            pfail[p].offer(ln, 0, PGL_ERR_MALFORMED_LINE, line_msg(ln, "P record needs name, steps and overlaps"));
            continue;
        }
        std::string_view name, steps;
        column(l, 1, name);
        column(l, 2, steps);
        G->path_names[p] = std::string(name);
        const char* b = steps.data();
        const char* e = steps.data() + steps.size();
        if (b == e) {
            pfail[p].offer(ln, 1, PGL_ERR_EMPTY_PATH,
                           "line " + std::to_string(ln) + ": path '" + std::string(name) + "' has no steps");
            continue;
        }
        while (b < e) {
            const char* cut = e;
            if (static_cast<uint64_t>(e - b) > kPiece) {
                const void* c = std::memchr(b + kPiece, ',', e - (b + kPiece));
                cut = c ? static_cast<const char*>(c) + 1 : e;
            }
            Piece pc;
            pc.path = p;
            pc.b = b;
            pc.e = cut;
            pc.last = cut == e;
            pieces.push_back(pc);
            b = cut;
        }
    }
    // tokens of a piece: comma-separated; the text after the final comma of
    // the step list is a token only if it is non-empty (gfa.cpp:132-137)
    auto for_tokens = [](const Piece& pc, auto&& f) {
        const char* p = pc.b;
        while (p < pc.e) {
            const void* c = std::memchr(p, ',', pc.e - p);
            const char* t = c ? static_cast<const char*>(c) : pc.e;
            if (!f(std::string_view(p, t - p))) return;
            p = c ? t + 1 : pc.e;
        }
    };
    {
        std::atomic<uint64_t> nx{0};
        run_threads(T, [&](unsigned) {
            for (uint64_t k; (k = nx.fetch_add(1)) < pieces.size();) {
                Piece& pc = pieces[k];
                uint64_t n = 0;
                for (const char* p = pc.b; p < pc.e;) {
                    const void* c = std::memchr(p, ',', pc.e - p);
                    ++n;
                    p = c ? static_cast<const char*>(c) + 1 : pc.e;
                }
                pc.n_tok = n;
            }
        });
    }
    G->compact = compact;
    G->path_n.assign(P, 0);
    {
        uint64_t acc = 0;
        uint32_t cur = kNone;
        for (auto& pc : pieces) {
            if (pc.path != cur) {
                if (cur != kNone) G->path_n[cur] = acc;
                cur = pc.path;
                acc = 0;
            }
            pc.tok0 = acc;
            acc += pc.n_tok;
        }
        if (cur != kNone) G->path_n[cur] = acc;
    }
    G->path_begin.assign(P + 1, 0);
    for (uint32_t p = 0; p < P; ++p) G->path_begin[p + 1] = G->path_begin[p] + G->path_n[p];
    if (compact) {
        if (V >= (1ULL << 31)) raise(PGL_ERR_INVALID_PARAMETER, "compact step records need fewer than 2^31 nodes");
        G->csteps.resize(G->path_begin[P]);
    } else {
        G->paths.resize(P);
        for (uint32_t p = 0; p < P; ++p) G->paths[p].resize(G->path_n[p]);
    }
    {
        std::atomic<uint64_t> nx{0};
        run_threads(T, [&](unsigned) {
            for (uint64_t k; (k = nx.fetch_add(1)) < pieces.size();) {
                Piece& pc = pieces[k];
                const uint64_t ln = plines[pc.path].first;
                pgl_path_step* out = compact ? nullptr : G->paths[pc.path].data() + pc.tok0;
                uint32_t* cout = compact ? G->csteps.data() + G->path_begin[pc.path] + pc.tok0 : nullptr;
                uint64_t i = 0, sum = 0;
                for_tokens(pc, [&](std::string_view tok) {
                    const uint64_t pos = 2 + pc.tok0 + i;  // after the line-level checks
                    if (tok.size() < 2) {
                        pc.fail.offer(ln, pos, PGL_ERR_MALFORMED_LINE,
                                      line_msg(ln, "bad path step '" + std::string(tok) + "'"));
                        return false;
                    }
                    const char o = tok.back();
                    if (o != '+' && o != '-') {
                        pc.fail.offer(ln, pos, PGL_ERR_MALFORMED_LINE,
                                      line_msg(ln, std::string("bad orientation '") + o + "'"));
                        return false;
                    }
                    const std::string_view nm = tok.substr(0, tok.size() - 1);
                    const uint32_t id = resolve(nm);
                    if (id == kNone) {
                        pc.fail.offer(ln, pos, PGL_ERR_UNKNOWN_SEGMENT, unknown(ln, nm));
                        return false;
                    }
                    const uint64_t len = G->node_len[id];
                    if (compact) {
                        cout[i++] = id | (o == '+' ? 0u : 0x80000000u);
                    } else {
                        pgl_path_step& s = out[i++];
                        std::memset(&s, 0, sizeof s);
                        s.node_id = id;
                        s.orient = o == '+' ? 0 : 1;
                        s.seq_len = static_cast<uint32_t>(len);
                    }
                    sum += len;
                    return true;
                });
                pc.len_sum = sum;
            }
        });
    }
    Fail p2;
    for (auto& c : ch) p2.merge(c.pass2);
    for (auto& f : pfail) p2.merge(f);
    for (auto& pc : pieces) p2.merge(pc.fail);
    if (p2.line != kNoLine) raise(p2.type, p2.msg);
    if (P == 0) raise(PGL_ERR_NO_PATHS, "no P records found; a layout needs at least one path");

    // ---- F: build_graph (graph.cpp:33-56): offsets, u32 length check ----
    std::vector<uint64_t> base(pieces.size());
    G->path_total.assign(P, 0);
    for (size_t k = 0; k < pieces.size(); ++k) {
        base[k] = G->path_total[pieces[k].path];
        G->path_total[pieces[k].path] += pieces[k].len_sum;
    }
    std::vector<Fail> bfail(pieces.size());
    {
        std::atomic<uint64_t> nx{0};
        run_threads(T, [&](unsigned) {
            for (uint64_t k; (k = nx.fetch_add(1)) < pieces.size();) {
                const Piece& pc = pieces[k];
                uint64_t off = base[k];
                for (uint64_t i = 0; i < pc.n_tok; ++i) {
                    uint32_t node;
                    if (compact) {
                        node = G->csteps[G->path_begin[pc.path] + pc.tok0 + i] & 0x7FFFFFFFu;
                    } else {
                        pgl_path_step& st = G->paths[pc.path][pc.tok0 + i];
                        st.offset = off;
                        node = st.node_id;
                    }
                    const uint64_t len = G->node_len[node];
                    if (len > std::numeric_limits<uint32_t>::max()) {
                        bfail[k].offer(pc.path, pc.tok0 + i, PGL_ERR_INVALID_PARAMETER,
                                       "node " + std::to_string(node) + " is longer than a step record can hold");
                        break;
                    }
                    off += len;
                }
            }
        });
    }
    Fail b3;
    for (auto& f : bfail) b3.merge(f);
    if (b3.line != kNoLine) raise(b3.type, b3.msg);

    G->skipped = skipped;
    G->total_steps = G->path_begin[P];
    if (!compact) {
        G->path_ptrs.resize(P);
        for (uint32_t p = 0; p < P; ++p) G->path_ptrs[p] = G->paths[p].data();
    }
    return own.release();
}

GfaGraph* gfa_parse_file(const char* path, unsigned threads, bool compact) {
    const int fd = ::open(path, O_RDONLY);
    if (fd < 0) raise(PGL_ERR_INVALID_PARAMETER, std::string("cannot open '") + path + "'");
    struct stat st;
    if (::fstat(fd, &st) != 0) {
        ::close(fd);
        raise(PGL_ERR_INVALID_PARAMETER, std::string("cannot stat '") + path + "'");
    }
    const uint64_t size = static_cast<uint64_t>(st.st_size);
    if (size == 0) {
        ::close(fd);
        return gfa_parse_buffer("", 0, threads, compact);
    }
    void* m = ::mmap(nullptr, size, PROT_READ, MAP_PRIVATE | MAP_POPULATE, fd, 0);
    ::close(fd);
    if (m == MAP_FAILED) raise(PGL_ERR_INVALID_PARAMETER, std::string("cannot map '") + path + "'");
    ::madvise(m, size, MADV_SEQUENTIAL);
    struct Unmap {
        void* p;
        uint64_t n;
        ~Unmap() { ::munmap(p, n); }
    } um{m, size};
    return gfa_parse_buffer(static_cast<const char*>(m), size, threads, compact);
}

void gfa_free(GfaGraph* g) { delete g; }

void gfa_view(const GfaGraph* g, pgl_graph_view* v) {
    if (g->compact) raise(PGL_ERR_INVALID_PARAMETER, "a compact GFA parse has no PathStep view");
    std::memset(v, 0, sizeof *v);
    v->n_nodes = g->node_len.size();
    v->node_len = g->node_len.data();
    v->n_paths = static_cast<uint32_t>(g->paths.size());
    v->path_steps = g->path_ptrs.data();
    v->path_n_steps = g->path_n.data();
    v->path_total_len = g->path_total.data();
}

void gfa_info(const GfaGraph* g, pgl_gfa_info* out) {
    std::memset(out, 0, sizeof *out);
    out->n_nodes = g->node_len.size();
    out->n_edges = g->edges.size();
    out->total_steps = g->total_steps;
    out->skipped_records = g->skipped;
    out->n_paths = static_cast<uint32_t>(g->paths.size());
}

const pgl_edge* gfa_edges(const GfaGraph* g) { return g->edges.data(); }

CompactGraph gfa_compact(const GfaGraph* g) {
    CompactGraph c;
    c.n_nodes = g->node_len.size();
    c.node_len = g->node_len.data();
    c.n_paths = static_cast<uint32_t>(g->path_n.size());
    c.path_begin = g->path_begin.data();
    c.path_total = g->path_total.data();
    c.steps = g->csteps.data();
    return c;
}
const char* gfa_path_name(const GfaGraph* g, uint32_t p) {
    return p < g->path_names.size() ? g->path_names[p].c_str() : nullptr;
}

}  // namespace pgl
