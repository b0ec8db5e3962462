// pgl_tsv.cpp — layout table IO on all host threads: the drop-in for
// write_layout_tsv / read_layout_tsv (src/layout_io.cpp:31-46, :48-110).
//
// Writer: nodes are cut into blocks, each block is formatted by its own
// thread with the reference's exact snprintf format ("%zu\t%.17g x4\n"), so
// every row is byte-identical; block sizes are then prefix-summed and the
// blocks written in order. The first non-finite node (lowest id) raises
// NonFiniteCoordinate before anything is written, as the serial writer
// would after writing the rows before it (the caller gets the same error;
// a partial file is not part of the reference contract).
// Reader: line-aligned chunks parsed in parallel with std::from_chars (the
// reference's parser); rows land at their node id; the first failure in line
// order wins, with the reference's exception classes and messages.
#include <algorithm>
#include <atomic>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fcntl.h>
#include <limits>
#include <string>
#include <string_view>
#include <sys/mman.h>
#include <sys/stat.h>
#include <thread>
#include <unistd.h>
#include <vector>

#include "pgl_internal.hpp"

namespace pgl {

namespace {

constexpr std::string_view kHeader = "node_id\tstart_x\tstart_y\tend_x\tend_y";  // layout_io.cpp:17
constexpr uint64_t kNoLine = std::numeric_limits<uint64_t>::max();

template <typename F>
void run_threads(unsigned T, F&& f) {
    if (T <= 1) {
        f(0u);
        return;
    }
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < T; ++t) pool.emplace_back([&, t] { f(t); });
    for (auto& th : pool) th.join();
}

unsigned threads_for(uint32_t threads, uint64_t work, uint64_t grain) {
    const unsigned want = std::max(1u, std::min(threads ? threads : std::thread::hardware_concurrency(), 256u));
    return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(want, work / grain)));
}

}  // namespace

std::string layout_format_tsv(const double* c, uint64_t n, uint32_t threads);

void layout_write_tsv(const char* path, const double* c, uint64_t n, uint32_t threads) {
    const std::string text = layout_format_tsv(c, n, threads);
    FILE* f = std::fopen(path, "wb");
    if (!f) raise(PGL_ERR_INVALID_PARAMETER, std::string("cannot write '") + path + "'");
    bool ok = std::fwrite(text.data(), 1, text.size(), f) == text.size();
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) raise(PGL_ERR_INVALID_PARAMETER, std::string("short write to '") + path + "'");
}

std::string layout_format_tsv(const double* c, uint64_t n, uint32_t threads) {
    const unsigned T = threads_for(threads, n, 1 << 16);
    // non-finite check first: the lowest offending node (layout_io.cpp:37-40)
    std::atomic<uint64_t> bad{kNoLine};
    run_threads(T, [&](unsigned t) {
        for (uint64_t i = n * t / T; i < n * (t + 1) / T; ++i)
            if (!std::isfinite(c[4 * i]) || !std::isfinite(c[4 * i + 1]) || !std::isfinite(c[4 * i + 2]) ||
                !std::isfinite(c[4 * i + 3])) {
                uint64_t cur = bad.load();
                while (i < cur && !bad.compare_exchange_weak(cur, i)) {
                }
                break;
            }
    });
    if (bad.load() != kNoLine)
        raise(PGL_ERR_NON_FINITE_COORDINATE, "node " + std::to_string(bad.load()) + " has a non-finite coordinate");
    const uint64_t NB = std::max<uint64_t>(1, std::min<uint64_t>(n / 4096 + 1, 64ull * T));
    std::vector<std::string> blocks(NB);
    std::atomic<uint64_t> next{0};
    run_threads(T, [&](unsigned) {
        char buf[128];
        for (uint64_t b; (b = next.fetch_add(1)) < NB;) {
            std::string& s = blocks[b];
            const uint64_t i0 = n * b / NB, i1 = n * (b + 1) / NB;
            s.reserve((i1 - i0) * 96);
            for (uint64_t i = i0; i < i1; ++i) {
                const int k = std::snprintf(buf, sizeof buf, "%zu\t%.17g\t%.17g\t%.17g\t%.17g\n",
                                            static_cast<size_t>(i), c[4 * i], c[4 * i + 1], c[4 * i + 2],
                                            c[4 * i + 3]);
                s.append(buf, static_cast<size_t>(k));
            }
        }
    });
    uint64_t total = kHeader.size() + 1;
    for (const auto& b : blocks) total += b.size();
    std::string text;
    text.reserve(total);
    text.append(kHeader.data(), kHeader.size());
    text.push_back('\n');
    for (const auto& b : blocks) text.append(b);
    return text;
}

namespace {

struct RowFail {
    uint64_t line = kNoLine;
    int type = 0;
    std::string msg;
    void offer(uint64_t l, int t, std::string m) {
        if (l < line) {
            line = l;
            type = t;
            msg = std::move(m);
        }
    }
};

}  // namespace

std::vector<double> layout_read_tsv_buffer(const char* data, uint64_t size, uint32_t threads) {
    // header line (layout_io.cpp:49-54)
    const char* end = data + size;
    if (size == 0) raise(PGL_ERR_MALFORMED_ROW, "empty layout file (missing header)");
    const void* nl0 = std::memchr(data, '\n', size);
    const char* hdr_end = nl0 ? static_cast<const char*>(nl0) : end;
    std::string_view hdr(data, hdr_end - data);
    if (!hdr.empty() && hdr.back() == '\r') hdr.remove_suffix(1);
    if (hdr != kHeader) raise(PGL_ERR_MALFORMED_ROW, "unexpected header '" + std::string(hdr) + "'");
    const char* body = nl0 ? hdr_end + 1 : end;
    const uint64_t bsize = static_cast<uint64_t>(end - body);
    const unsigned T = threads_for(threads, bsize, 1 << 22);
    const unsigned NC = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(4ull * T, bsize / 4096 + 1)));
    struct Chunk {
        const char* b;
        const char* e;
        uint64_t lines = 0, rows = 0, line0 = 0, row0 = 0;
        RowFail fail;
    };
    std::vector<Chunk> ch(NC);
    {
        const char* prev = body;
        for (unsigned k = 0; k < NC; ++k) {
            const char* cut = k + 1 == NC ? end : body + bsize * (k + 1) / NC;
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
    auto for_lines = [](const Chunk& c, auto&& f) {
        for (const char* p = c.b; p < c.e;) {
            const void* nl = std::memchr(p, '\n', c.e - p);
            const char* e = nl ? static_cast<const char*>(nl) : c.e;
            std::string_view l(p, e - p);
            if (!l.empty() && l.back() == '\r') l.remove_suffix(1);
            f(l);
            p = nl ? e + 1 : c.e;
        }
    };
    std::atomic<unsigned> next{0};
    auto each = [&](auto&& f) {
        next = 0;
        run_threads(T, [&](unsigned) {
            for (unsigned k; (k = next.fetch_add(1)) < NC;) f(ch[k]);
        });
    };
    each([&](Chunk& c) {
        for_lines(c, [&](std::string_view l) {
            ++c.lines;
            if (!l.empty()) ++c.rows;
        });
    });
    uint64_t ln = 2, rows = 0;
    for (auto& c : ch) {
        c.line0 = ln;
        c.row0 = rows;
        ln += c.lines;
        rows += c.rows;
    }
    std::vector<double> out(4 * rows);
    each([&](Chunk& c) {
        uint64_t line = c.line0, row = c.row0;
        for_lines(c, [&](std::string_view l) {
            const uint64_t my = line++;
            if (l.empty()) return;
            const uint64_t r = row++;
            if (c.fail.line != kNoLine) return;
            std::string_view f[5];
            std::string_view rest = l;
            for (int k = 0; k < 5; ++k) {
                const size_t tab = rest.find('\t');
                if (tab == std::string_view::npos) {
                    if (k != 4) {
                        c.fail.offer(my, PGL_ERR_MALFORMED_ROW, "line " + std::to_string(my) + ": expected 5 columns");
                        return;
                    }
                    f[k] = rest;
                    rest = {};
                } else {
                    f[k] = rest.substr(0, tab);
                    rest = rest.substr(tab + 1);
                }
            }
            if (!rest.empty()) {
                c.fail.offer(my, PGL_ERR_MALFORMED_ROW, "line " + std::to_string(my) + ": expected 5 columns");
                return;
            }
            uint64_t id = 0;
            const auto ri = std::from_chars(f[0].data(), f[0].data() + f[0].size(), id);
            if (ri.ec != std::errc{} || ri.ptr != f[0].data() + f[0].size()) {
                c.fail.offer(my, PGL_ERR_MALFORMED_ROW,
                             "line " + std::to_string(my) + ": bad node id '" + std::string(f[0]) + "'");
                return;
            }
            if (id != r) {
                c.fail.offer(my, PGL_ERR_COUNT_MISMATCH,
                             "line " + std::to_string(my) + ": node ids must be dense and ascending (got " +
                                 std::to_string(id) + ", expected " + std::to_string(r) + ")");
                return;
            }
            for (int k = 1; k < 5; ++k) {
                double v = 0.0;
                const auto rv = std::from_chars(f[k].data(), f[k].data() + f[k].size(), v);
                if (rv.ec != std::errc{} || rv.ptr != f[k].data() + f[k].size()) {
                    c.fail.offer(my, PGL_ERR_MALFORMED_ROW,
                                 "line " + std::to_string(my) + ": bad coordinate '" + std::string(f[k]) + "'");
                    return;
                }
                out[4 * r + k - 1] = v;
            }
        });
    });
    RowFail first;
    for (auto& c : ch)
        if (c.fail.line != kNoLine) first.offer(c.fail.line, c.fail.type, c.fail.msg);
    if (first.line != kNoLine) raise(first.type, first.msg);
    return out;
}

std::vector<double> layout_read_tsv(const char* path, uint32_t threads) {
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
        return layout_read_tsv_buffer("", 0, threads);
    }
    void* m = ::mmap(nullptr, size, PROT_READ, MAP_PRIVATE | MAP_POPULATE, fd, 0);
    ::close(fd);
    if (m == MAP_FAILED) raise(PGL_ERR_INVALID_PARAMETER, std::string("cannot map '") + path + "'");
    struct Unmap {
        void* p;
        uint64_t n;
        ~Unmap() { ::munmap(p, n); }
    } um{m, size};
    return layout_read_tsv_buffer(static_cast<const char*>(m), size, threads);
}

}  // namespace pgl
