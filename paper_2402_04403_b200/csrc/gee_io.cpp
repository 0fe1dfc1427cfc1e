// gee_io.cpp -- multithreaded host IO for the GEE path's data formats
// (libgee_io.so; C ABI in include/gee_io.h).
//
// Replaces the reference's per-line Python ingestion and whole-file binary
// readers (files under /root/reference/pkg/src/gee):
//   load_edge_list      graph.py:94-145     gee_io_edges_parse / _copy_*
//   write_edge_list     graph.py:148-156    gee_io_edges_write
//   load_labels         labeling.py:33-73   gee_io_labels_parse / _copy
//   write_labels        labeling.py:81-84   gee_io_labels_write
//   write/read_binary_cache graph.py:204-235  gee_io_csr_write / _header / _read
//   write/read_embedding    encoder.py:209-237 gee_io_emb_write / _header / _read
//
// Text is memory-mapped and cut into byte chunks at '\n' boundaries; each
// worker parses its chunk independently (fields, Python int()/float()
// grammar, the reference's per-line check order) and records the first bad
// line of its chunk.  The reported error is the one in the earliest chunk,
// with its line number rebased by the line counts of the chunks before it,
// which is exactly the line the reference's sequential loop stops at.
// Binary files are read and written with positioned I/O from all workers;
// f64<->f32 conversion happens in per-worker bounce buffers.
#include "../../include/gee_io.h"

#include <errno.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <charconv>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <immintrin.h>
#include <functional>
#include <string>
#include <thread>
#include <vector>

namespace {

thread_local std::string g_err;
thread_local int g_errno = 0;

int fail(int code, const char *fmt, ...)
{
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

int fail_os(const char *path)
{
    g_errno = errno;
    g_err = std::string(strerror(g_errno)) + ": '" + path + "'";
    return GEE_IO_ERR_OS;
}

void clear_error()
{
    g_err.clear();
    g_errno = 0;
}

int nthreads(int threads)
{
    if (threads > 0) return threads;
    unsigned h = std::thread::hardware_concurrency();
    return h ? (int)h : 1;
}

// Run fn(i) for i in [0, count) on `threads` workers (dynamic assignment).
void parallel_for(int64_t count, int threads, const std::function<void(int64_t)> &fn)
{
    if (count <= 0) return;
    int t = (int)std::min<int64_t>(nthreads(threads), count);
    if (t <= 1) {
        for (int64_t i = 0; i < count; i++) fn(i);
        return;
    }
    std::atomic<int64_t> next{0};
    std::vector<std::thread> pool;
    pool.reserve(t);
    for (int w = 0; w < t; w++)
        pool.emplace_back([&] {
            for (int64_t i; (i = next.fetch_add(1)) < count;) fn(i);
        });
    for (auto &th : pool) th.join();
}

// ------------------------------------------------------------ file helpers
struct Mapped {
    const char *p = nullptr;
    size_t n = 0;
    int fd = -1;
    ~Mapped()
    {
        if (p && n) munmap((void *)p, n);
        if (fd >= 0) close(fd);
    }
};

int map_file(const char *path, Mapped &m)
{
    m.fd = open(path, O_RDONLY | O_CLOEXEC);
    if (m.fd < 0) return fail_os(path);
    struct stat st;
    if (fstat(m.fd, &st) != 0) return fail_os(path);
    if (S_ISDIR(st.st_mode)) {
        errno = EISDIR;
        return fail_os(path);
    }
    m.n = (size_t)st.st_size;
    if (m.n == 0) return GEE_IO_OK;
    void *p = mmap(nullptr, m.n, PROT_READ, MAP_PRIVATE, m.fd, 0);
    if (p == MAP_FAILED) {
        m.n = 0;
        return fail_os(path);
    }
    madvise(p, m.n, MADV_WILLNEED);
    m.p = (const char *)p;
    return GEE_IO_OK;
}

// pread/pwrite the whole range (short transfers retried).
bool pread_all(int fd, void *dst, size_t bytes, off_t off)
{
    char *d = (char *)dst;
    while (bytes) {
        ssize_t r = pread(fd, d, bytes, off);
        if (r < 0 && errno == EINTR) continue;
        if (r <= 0) return false;
        d += r, bytes -= (size_t)r, off += r;
    }
    return true;
}

bool pwrite_all(int fd, const void *src, size_t bytes, off_t off)
{
    const char *s = (const char *)src;
    while (bytes) {
        ssize_t r = pwrite(fd, s, bytes, off);
        if (r < 0 && errno == EINTR) continue;
        if (r <= 0) return false;
        s += r, bytes -= (size_t)r, off += r;
    }
    return true;
}

// Chunk [0, n) of a text buffer at line starts: every chunk but the last
// ends just after a '\n' (so a "\r\n" pair is never split).
std::vector<size_t> text_chunks(const char *p, size_t n, int threads)
{
    std::vector<size_t> cuts{0};
    if (n == 0) return cuts;
    const size_t target = std::max<size_t>(1 << 20, n / ((size_t)nthreads(threads) * 8));
    for (size_t pos = target; pos < n; pos += target) {
        const char *nl = (const char *)memchr(p + pos, '\n', n - pos);
        if (!nl) break;
        size_t c = (size_t)(nl - p) + 1;
        if (c >= n) break;
        if (c > cuts.back()) cuts.push_back(c);
        pos = c;
    }
    cuts.push_back(n);
    return cuts;
}

// ---------------------------------------------------- lexical (Python rules)
// str.split() whitespace inside a line (ASCII); \n and \r end lines.
inline bool is_ws(unsigned char c) { return c == ' ' || c == '\t' || c == '\v' || c == '\f' || (c >= 0x1c && c <= 0x1f); }
inline bool is_digit(char c) { return c >= '0' && c <= '9'; }

struct Tok {
    const char *p;
    size_t n;
};

// One line [b, e) (terminator excluded) split on whitespace; returns the
// field count (all of them) and the first `cap` tokens.
inline int split_fields(const char *b, const char *e, Tok *tok, int cap)
{
    int nf = 0;
    const char *q = b;
    while (true) {
        while (q < e && is_ws((unsigned char)*q)) q++;
        if (q >= e) break;
        const char *s = q;
        while (q < e && !is_ws((unsigned char)*q)) q++;
        if (nf < cap) tok[nf] = Tok{s, (size_t)(q - s)};
        nf++;
    }
    return nf;
}

// Python int(): [+-]? digit ('_'? digit)*.  Returns false on bad syntax;
// *sat = true when |value| exceeds int64 (value saturated).
inline bool parse_int(Tok t, int64_t *out, bool *sat)
{
    const char *p = t.p, *e = t.p + t.n;
    bool neg = false;
    if (p < e && (*p == '+' || *p == '-')) neg = *p++ == '-';
    if (p >= e || !is_digit(*p)) return false;
    unsigned __int128 v = 0;
    bool big = false;
    bool prev_us = false;
    for (; p < e; p++) {
        if (*p == '_') {
            if (prev_us) return false;
            prev_us = true;
            continue;
        }
        if (!is_digit(*p)) return false;
        prev_us = false;
        if (!big) {
            v = v * 10 + (unsigned)(*p - '0');
            if (v > (unsigned __int128)INT64_MAX + 1) big = true;
        }
    }
    if (prev_us) return false;
    if (neg) {
        if (big || v > (unsigned __int128)INT64_MAX + 1) {
            *out = INT64_MIN, *sat = true;
        } else {
            *out = v == (unsigned __int128)INT64_MAX + 1 ? INT64_MIN : -(int64_t)v;
            *sat = false;
        }
    } else {
        if (big || v > (unsigned __int128)INT64_MAX) {
            *out = INT64_MAX, *sat = true;
        } else {
            *out = (int64_t)v, *sat = false;
        }
    }
    return true;
}

inline bool ieq(const char *p, size_t n, const char *word)
{
    size_t m = strlen(word);
    if (n != m) return false;
    for (size_t i = 0; i < n; i++)
        if ((p[i] | 0x20) != word[i]) return false;
    return true;
}

const double kPow10[] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,  1e8,  1e9,  1e10, 1e11,
                         1e12, 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};

// Python float(): [+-]? (inf | infinity | nan | number), case-insensitive
// words; number = (digits ['.' [digits]] | '.' digits) [(e|E) [+-] digits],
// digits = digit ('_'? digit)*.  Correctly rounded (Clinger's exact fast
// path, else glibc strtod on the underscore-free copy).
bool parse_float(Tok t, double *out)
{
    const char *p = t.p, *e = t.p + t.n;
    bool neg = false;
    if (p < e && (*p == '+' || *p == '-')) neg = *p++ == '-';
    if (p >= e) return false;
    if (!is_digit(*p) && *p != '.') {
        size_t r = (size_t)(e - p);
        if (ieq(p, r, "inf") || ieq(p, r, "infinity")) {
            *out = neg ? -HUGE_VAL : HUGE_VAL;
            return true;
        }
        if (ieq(p, r, "nan")) {
            *out = neg ? -NAN : NAN;
            return true;
        }
        return false;
    }
    char buf[128];
    std::string big;
    char *w = buf;
    const size_t cap = t.n + 1;
    if (cap > sizeof buf) {
        big.resize(cap);
        w = &big[0];
    }
    char *w0 = w;
    if (neg) *w++ = '-';
    // mantissa digits for the fast path
    uint64_t mant = 0;
    int mdig = 0, frac_digits = 0;
    bool exact = true;
    auto digits = [&](bool frac) -> int {  // returns digit count, -1 on bad '_'
        int cnt = 0;
        bool prev_us = false;
        while (p < e && (is_digit(*p) || *p == '_')) {
            if (*p == '_') {
                if (cnt == 0 || prev_us) return -1;
                prev_us = true;
                p++;
                continue;
            }
            prev_us = false;
            *w++ = *p;
            if (mant == 0 && *p == '0') {
                if (frac) frac_digits++;
            } else if (mdig < 19) {
                mant = mant * 10 + (uint64_t)(*p - '0');
                mdig++;
                if (frac) frac_digits++;
            } else {
                exact = false;
                if (frac) frac_digits++;
            }
            cnt++;
            p++;
        }
        if (prev_us) return -1;
        return cnt;
    };
    int ip = digits(false);
    if (ip < 0) return false;
    int fp = 0;
    if (p < e && *p == '.') {
        *w++ = *p++;
        fp = digits(true);
        if (fp < 0) return false;
    }
    if (ip + fp == 0) return false;
    int64_t exp10 = 0;
    if (p < e && (*p == 'e' || *p == 'E')) {
        *w++ = *p++;
        bool eneg = false;
        if (p < e && (*p == '+' || *p == '-')) {
            eneg = *p == '-';
            *w++ = *p++;
        }
        if (p >= e || !is_digit(*p)) return false;
        bool prev_us = false;
        int cnt = 0;
        while (p < e && (is_digit(*p) || *p == '_')) {
            if (*p == '_') {
                if (prev_us || cnt == 0) return false;
                prev_us = true;
                p++;
                continue;
            }
            prev_us = false;
            *w++ = *p;
            if (exp10 < 100000000) exp10 = exp10 * 10 + (*p - '0');
            cnt++;
            p++;
        }
        if (prev_us) return false;
        if (eneg) exp10 = -exp10;
    }
    if (p != e) return false;
    *w = 0;
    const int64_t scale = exp10 - frac_digits;
    if (exact && mant <= (1ull << 53) && scale >= -22 && scale <= 22) {
        double v = (double)mant;
        v = scale < 0 ? v / kPow10[-scale] : v * kPow10[scale];
        *out = neg ? -v : v;
        return true;
    }
    *out = strtod(w0, nullptr);
    return true;
}

// ------------------------------------------------------ line iteration
// Calls fn(b, e) for every line of [p, p+n) (terminator excluded); fn
// returns false to stop.  Returns the number of lines visited.
template <class F>
int64_t for_lines(const char *p, size_t n, F &&fn)
{
    const char *q = p, *end = p + n;
    int64_t lines = 0;
    while (q < end) {
        const char *s = q;
        while (q < end && *q != '\n' && *q != '\r') q++;
        const char *le = q;
        if (q < end) {
            if (*q == '\r' && q + 1 < end && q[1] == '\n') q++;
            q++;
        }
        lines++;
        if (!fn(s, le, lines)) return lines;
    }
    return lines;
}

struct ChunkErr {
    int64_t line = 0;  // 1-based line within the chunk; 0 = none
    int code = 0;
    std::string msg;   // reason (after "line L: ")
};

}  // namespace

// =================================================================== edges
struct gee_io_edges {
    struct Part {
        std::vector<int64_t> src, dst;
        std::vector<double> w;
        int64_t max_id = -1;
        int64_t lines = 0;
        ChunkErr err;
    };
    std::vector<Part> parts;
    std::vector<int64_t> base;  // first edge index of each part
    int64_t s = 0;
    int64_t max_id = -1;
    bool weighted = false;
};

extern "C" int gee_io_version(void) { return 1; }
extern "C" const char *gee_io_last_error(void) { return g_err.c_str(); }
extern "C" int gee_io_last_errno(void) { return g_errno; }

extern "C" int gee_io_edges_parse(const char *path, int weighted, int threads, gee_io_edges **out)
{
    clear_error();
    if (!path || !out) return fail(GEE_IO_ERR_INVALID, "NULL argument");
    *out = nullptr;
    Mapped m;
    if (int rc = map_file(path, m)) return rc;
    auto cuts = text_chunks(m.p, m.n, threads);
    auto *h = new gee_io_edges;
    h->weighted = weighted != 0;
    const size_t nparts = cuts.size() - 1;
    h->parts.resize(nparts);
    parallel_for((int64_t)nparts, threads, [&](int64_t ci) {
        auto &pt = h->parts[ci];
        const char *b = m.p + cuts[ci];
        const size_t len = cuts[ci + 1] - cuts[ci];
        pt.src.reserve(len / 8);
        pt.dst.reserve(len / 8);
        if (weighted) pt.w.reserve(len / 8);
        int64_t mx = -1;
        pt.lines = for_lines(b, len, [&](const char *s, const char *e, int64_t ln) {
            if (s < e && *s == '#') return true;
            Tok f[3];
            const int nf = split_fields(s, e, f, 3);
            if (nf == 0) return true;
            auto bad = [&](int code, std::string msg) {
                pt.err.line = ln, pt.err.code = code, pt.err.msg = std::move(msg);
                return false;
            };
            if (nf != 2 && nf != 3) return bad(GEE_IO_ERR_PARSE, "expected 2 or 3 fields, got " + std::to_string(nf));
            int64_t u, v;
            bool su, sv;
            if (!parse_int(f[0], &u, &su) || !parse_int(f[1], &v, &sv))
                return bad(GEE_IO_ERR_PARSE, "node ids must be integers");
            if (u < 0 || v < 0) return bad(GEE_IO_ERR_PARSE, "negative node id");
            if (su || sv) return bad(GEE_IO_ERR_VALUE, "node id exceeds int64");
            if (weighted) {
                if (nf < 3) return bad(GEE_IO_ERR_PARSE, "missing weight field");
                double w;
                if (!parse_float(f[2], &w)) return bad(GEE_IO_ERR_PARSE, "weight is not a number");
                if (!std::isfinite(w)) return bad(GEE_IO_ERR_PARSE, "weight is not finite");
                pt.w.push_back(w);
            }
            pt.src.push_back(u);
            pt.dst.push_back(v);
            mx = std::max(mx, std::max(u, v));
            return true;
        });
        pt.max_id = mx;
    });
    int64_t line0 = 0;
    for (size_t ci = 0; ci < nparts; ci++) {
        auto &pt = h->parts[ci];
        if (pt.err.line) {
            int code = pt.err.code;
            fail(code, "%s: line %lld: %s", path, (long long)(line0 + pt.err.line), pt.err.msg.c_str());
            delete h;
            return code;
        }
        line0 += pt.lines;
    }
    h->base.resize(nparts + 1, 0);
    for (size_t ci = 0; ci < nparts; ci++) {
        h->base[ci + 1] = h->base[ci] + (int64_t)h->parts[ci].src.size();
        h->max_id = std::max(h->max_id, h->parts[ci].max_id);
    }
    h->s = h->base[nparts];
    *out = h;
    return GEE_IO_OK;
}

extern "C" int64_t gee_io_edges_count(const gee_io_edges *h) { return h ? h->s : -1; }
extern "C" int64_t gee_io_edges_max_id(const gee_io_edges *h) { return h ? h->max_id : -1; }
extern "C" void gee_io_edges_free(gee_io_edges *h) { delete h; }

extern "C" int gee_io_edges_copy_i32(const gee_io_edges *h, int32_t *src, int32_t *dst, float *w, int threads)
{
    clear_error();
    if (!h) return fail(GEE_IO_ERR_INVALID, "NULL handle");
    if (h->s && (!src || !dst)) return fail(GEE_IO_ERR_INVALID, "NULL array argument");
    if (h->max_id > INT32_MAX)
        return fail(GEE_IO_ERR_VALUE, "node count %lld exceeds CSR limit %d", (long long)h->max_id + 1, INT32_MAX);
    parallel_for((int64_t)h->parts.size(), threads, [&](int64_t ci) {
        const auto &pt = h->parts[ci];
        const int64_t o = h->base[ci];
        const size_t m = pt.src.size();
        for (size_t i = 0; i < m; i++) src[o + i] = (int32_t)pt.src[i], dst[o + i] = (int32_t)pt.dst[i];
        if (w) {
            if (h->weighted)
                for (size_t i = 0; i < m; i++) w[o + i] = (float)pt.w[i];
            else
                for (size_t i = 0; i < m; i++) w[o + i] = 1.0f;
        }
    });
    return GEE_IO_OK;
}

extern "C" int gee_io_edges_copy_i64(const gee_io_edges *h, int64_t *src, int64_t *dst, double *w, int threads)
{
    clear_error();
    if (!h) return fail(GEE_IO_ERR_INVALID, "NULL handle");
    if (h->s && (!src || !dst)) return fail(GEE_IO_ERR_INVALID, "NULL array argument");
    parallel_for((int64_t)h->parts.size(), threads, [&](int64_t ci) {
        const auto &pt = h->parts[ci];
        const int64_t o = h->base[ci];
        const size_t m = pt.src.size();
        if (m) {
            memcpy(src + o, pt.src.data(), m * 8);
            memcpy(dst + o, pt.dst.data(), m * 8);
        }
        if (w) {
            if (h->weighted) {
                if (m) memcpy(w + o, pt.w.data(), m * 8);
            } else {
                for (size_t i = 0; i < m; i++) w[o + i] = 1.0;
            }
        }
    });
    return GEE_IO_OK;
}

// ------------------------------------------------------- Python float repr
namespace {

// repr(float(x)) (float_repr_style 'short'): shortest digits that round-trip,
// fixed notation when the decimal exponent lies in [-4, 16), else d.ddde+XX.
int py_repr(double x, char *out)
{
    if (std::isnan(x)) return sprintf(out, "nan");
    if (std::isinf(x)) return sprintf(out, x < 0 ? "-inf" : "inf");
    char *o = out;
    if (std::signbit(x)) *o++ = '-', x = -x;
    if (x == 0) return (int)(o - out) + sprintf(o, "0.0");
    char buf[40];
    // shortest round-trip digits (libstdc++'s Ryu-based to_chars)
    auto r = std::to_chars(buf, buf + sizeof buf - 1, x, std::chars_format::scientific);
    *r.ptr = 0;
    // buf = d[.ddd]e[+-]XX
    char digs[24];
    int nd = 0;
    const char *q = buf;
    for (; *q && *q != 'e'; q++)
        if (is_digit(*q)) digs[nd++] = *q;
    while (nd > 1 && digs[nd - 1] == '0') nd--;
    const int e10 = atoi(q + 1);  // value = d.ddd * 10^e10
    const int decpt = e10 + 1;     // value = 0.ddd * 10^decpt
    if (decpt > -4 && decpt <= 16) {
        if (decpt <= 0) {
            *o++ = '0', *o++ = '.';
            for (int i = 0; i < -decpt; i++) *o++ = '0';
            for (int i = 0; i < nd; i++) *o++ = digs[i];
        } else if (decpt < nd) {
            for (int i = 0; i < decpt; i++) *o++ = digs[i];
            *o++ = '.';
            for (int i = decpt; i < nd; i++) *o++ = digs[i];
        } else {
            for (int i = 0; i < nd; i++) *o++ = digs[i];
            for (int i = nd; i < decpt; i++) *o++ = '0';
            *o++ = '.', *o++ = '0';
        }
        *o = 0;
        return (int)(o - out);
    }
    *o++ = digs[0];
    if (nd > 1) {
        *o++ = '.';
        for (int i = 1; i < nd; i++) *o++ = digs[i];
    }
    o += sprintf(o, "e%c%02d", e10 < 0 ? '-' : '+', e10 < 0 ? -e10 : e10);
    return (int)(o - out);
}

inline char *put_i64(char *o, int64_t v)
{
    char t[24];
    int n = 0;
    uint64_t u = v < 0 ? (uint64_t)0 - (uint64_t)v : (uint64_t)v;
    do t[n++] = (char)('0' + u % 10), u /= 10;
    while (u);
    if (v < 0) *o++ = '-';
    while (n) *o++ = t[--n];
    return o;
}

// Write rows [0, count) formatted by fmt(i, out_ptr) -> end_ptr, in
// rounds: each worker formats a block into its own buffer, then the round
// is written in order.  `row_max` bounds one row's bytes.
int write_text_rows(const char *path, int64_t count, size_t row_max, int threads,
                    const std::function<char *(int64_t, char *)> &fmt)
{
    int fd = open(path, O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0666);
    if (fd < 0) return fail_os(path);
    const int t = nthreads(threads);
    const int64_t per_block = std::max<int64_t>(1, (int64_t)((8u << 20) / std::max<size_t>(row_max, 1)));
    std::vector<std::vector<char>> bufs(t);
    std::vector<size_t> used(t);
    off_t off = 0;
    bool ok = true;
    for (int64_t r0 = 0; r0 < count && ok; r0 += per_block * t) {
        parallel_for(t, t, [&](int64_t b) {
            const int64_t lo = r0 + b * per_block, hi = std::min(count, lo + per_block);
            used[b] = 0;
            if (lo >= hi) return;
            auto &buf = bufs[b];
            buf.resize((size_t)(hi - lo) * row_max);
            char *o = buf.data();
            for (int64_t i = lo; i < hi; i++) o = fmt(i, o);
            used[b] = (size_t)(o - buf.data());
        });
        for (int b = 0; b < t && ok; b++) {
            if (!used[b]) continue;
            ok = pwrite_all(fd, bufs[b].data(), used[b], off);
            off += (off_t)used[b];
        }
    }
    if (!ok) {
        int rc = fail_os(path);
        close(fd);
        return rc;
    }
    if (close(fd) != 0) return fail_os(path);
    return GEE_IO_OK;
}

}  // namespace

extern "C" int gee_io_edges_write(const char *path, const int32_t *src, const int32_t *dst, const float *w,
                                  int64_t s, int threads)
{
    clear_error();
    if (!path || (s > 0 && (!src || !dst))) return fail(GEE_IO_ERR_INVALID, "NULL argument");
    return write_text_rows(path, s, 64, threads, [&](int64_t i, char *o) {
        o = put_i64(o, src[i]);
        *o++ = ' ';
        o = put_i64(o, dst[i]);
        if (w) {
            *o++ = ' ';
            o += py_repr((double)w[i], o);
        }
        *o++ = '\n';
        return o;
    });
}

// ================================================================== labels
struct gee_io_labels {
    struct Part {
        std::vector<int64_t> c0, c1;
        int64_t lines = 0;
        ChunkErr err;
    };
    std::vector<Part> parts;
    std::vector<int64_t> base;
    int width = 0;
    int64_t rows = 0;
};

extern "C" int gee_io_labels_parse(const char *path, int threads, gee_io_labels **out)
{
    clear_error();
    if (!path || !out) return fail(GEE_IO_ERR_INVALID, "NULL argument");
    *out = nullptr;
    Mapped m;
    if (int rc = map_file(path, m)) return rc;
    // the first data line fixes the width (labeling.py:53-56)
    int width = 0;
    for_lines(m.p, m.n, [&](const char *s, const char *e, int64_t) {
        if (s < e && *s == '#') return true;
        Tok f[2];
        const int nf = split_fields(s, e, f, 2);
        if (nf == 0) return true;
        width = nf;
        return false;
    });
    auto cuts = text_chunks(m.p, m.n, threads);
    auto *h = new gee_io_labels;
    h->width = (width == 1 || width == 2) ? width : 0;
    const size_t nparts = cuts.size() - 1;
    h->parts.resize(nparts);
    parallel_for((int64_t)nparts, threads, [&](int64_t ci) {
        auto &pt = h->parts[ci];
        const char *b = m.p + cuts[ci];
        const size_t len = cuts[ci + 1] - cuts[ci];
        pt.lines = for_lines(b, len, [&](const char *s, const char *e, int64_t ln) {
            if (s < e && *s == '#') return true;
            Tok f[2];
            const int nf = split_fields(s, e, f, 2);
            if (nf == 0) return true;
            auto bad = [&](const char *msg) {
                pt.err.line = ln, pt.err.code = GEE_IO_ERR_PARSE, pt.err.msg = msg;
                return false;
            };
            if (nf != 1 && nf != 2) return bad("expected 1 or 2 fields");
            if (nf != width) return bad("mixed label formats");
            int64_t a, c = 0;
            bool sat;
            if (!parse_int(f[0], &a, &sat) || (nf == 2 && !parse_int(f[1], &c, &sat)))
                return bad("fields must be integers");
            pt.c0.push_back(a);
            if (nf == 2) pt.c1.push_back(c);
            return true;
        });
    });
    int64_t line0 = 0;
    for (size_t ci = 0; ci < nparts; ci++) {
        auto &pt = h->parts[ci];
        if (pt.err.line) {
            fail(GEE_IO_ERR_PARSE, "%s: line %lld: %s", path, (long long)(line0 + pt.err.line), pt.err.msg.c_str());
            delete h;
            return GEE_IO_ERR_PARSE;
        }
        line0 += pt.lines;
    }
    h->base.resize(nparts + 1, 0);
    for (size_t ci = 0; ci < nparts; ci++) h->base[ci + 1] = h->base[ci] + (int64_t)h->parts[ci].c0.size();
    h->rows = h->base[nparts];
    *out = h;
    return GEE_IO_OK;
}

extern "C" int gee_io_labels_width(const gee_io_labels *h) { return h ? h->width : -1; }
extern "C" int64_t gee_io_labels_rows(const gee_io_labels *h) { return h ? h->rows : -1; }
extern "C" void gee_io_labels_free(gee_io_labels *h) { delete h; }

extern "C" int gee_io_labels_copy(const gee_io_labels *h, int64_t *col0, int64_t *col1)
{
    clear_error();
    if (!h) return fail(GEE_IO_ERR_INVALID, "NULL handle");
    if (h->rows && (!col0 || (h->width == 2 && !col1))) return fail(GEE_IO_ERR_INVALID, "NULL array argument");
    for (size_t ci = 0; ci < h->parts.size(); ci++) {
        const auto &pt = h->parts[ci];
        if (pt.c0.empty()) continue;
        memcpy(col0 + h->base[ci], pt.c0.data(), pt.c0.size() * 8);
        if (h->width == 2) memcpy(col1 + h->base[ci], pt.c1.data(), pt.c1.size() * 8);
    }
    return GEE_IO_OK;
}

extern "C" int gee_io_labels_write(const char *path, const int32_t *labels, int64_t n, int threads)
{
    clear_error();
    if (!path || (n > 0 && !labels)) return fail(GEE_IO_ERR_INVALID, "NULL argument");
    return write_text_rows(path, n, 16, threads, [&](int64_t i, char *o) {
        o = put_i64(o, labels[i]);
        *o++ = '\n';
        return o;
    });
}

// ============================================================ binary files
namespace {

const char kCsrMagic[8] = {'G', 'E', 'E', 'C', 'S', 'R', '1', 0};
const char kEmbMagic[8] = {'G', 'E', 'E', 'E', 'M', 'B', '1', 0};
constexpr size_t kCsrHead = 26;  // struct "<8sBBQQ"
constexpr size_t kEmbHead = 24;  // struct "<8sQQ"
constexpr size_t kPiece = 32u << 20;

std::string u128_str(unsigned __int128 v)
{
    char t[48];
    int n = 0;
    do t[n++] = (char)('0' + (int)(v % 10)), v /= 10;
    while (v);
    std::string s;
    while (n) s.push_back(t[--n]);
    return s;
}

inline uint64_t rd_u64(const unsigned char *p)
{
    uint64_t v;
    memcpy(&v, p, 8);
    return v;  // little-endian host (x86-64 / aarch64)
}

struct Fd {
    int fd = -1;
    ~Fd()
    {
        if (fd >= 0) close(fd);
    }
};

// Open + size + header bytes; FormatError "truncated header" if short.
int open_with_header(const char *path, Fd &f, off_t &size, unsigned char *head, size_t head_len)
{
    f.fd = open(path, O_RDONLY | O_CLOEXEC);
    if (f.fd < 0) return fail_os(path);
    struct stat st;
    if (fstat(f.fd, &st) != 0) return fail_os(path);
    if (S_ISDIR(st.st_mode)) {
        errno = EISDIR;
        return fail_os(path);
    }
    size = st.st_size;
    if ((size_t)size < head_len) return fail(GEE_IO_ERR_FORMAT, "%s: truncated header", path);
    if (!pread_all(f.fd, head, head_len, 0)) return fail_os(path);
    return GEE_IO_OK;
}

// Read `count` elements of `esz` bytes at file offset `off` into dst,
// converting with conv(src_bytes, dst_index, m) when given.
int par_read(int fd, const char *path, off_t off, int64_t count, size_t esz, void *dst, int threads,
             const std::function<void(const char *, int64_t, int64_t)> &conv)
{
    if (count <= 0) return GEE_IO_OK;
    const int64_t per = (int64_t)(kPiece / esz);
    const int64_t pieces = (count + per - 1) / per;
    std::atomic<int> bad{0};
    std::atomic<int> bad_errno{0};
    parallel_for(pieces, threads, [&](int64_t pi) {
        if (bad.load()) return;
        const int64_t lo = pi * per, m = std::min(count - lo, per);
        if (!conv) {
            if (!pread_all(fd, (char *)dst + lo * esz, (size_t)m * esz, off + (off_t)(lo * esz))) {
                bad_errno = errno ? errno : EIO;
                bad = 1;
            }
            return;
        }
        std::vector<char> tmp((size_t)m * esz);
        if (!pread_all(fd, tmp.data(), tmp.size(), off + (off_t)(lo * esz))) {
            bad_errno = errno ? errno : EIO;
            bad = 1;
            return;
        }
        conv(tmp.data(), lo, m);
    });
    if (bad) {
        errno = bad_errno;
        return fail_os(path);
    }
    return GEE_IO_OK;
}

// Write `count` elements of `esz` bytes at `off`, produced by
// gen(tmp, index, m) into a bounce buffer (or straight from src).
int par_write(int fd, const char *path, off_t off, int64_t count, size_t esz, const void *src, int threads,
              const std::function<void(char *, int64_t, int64_t)> &gen)
{
    if (count <= 0) return GEE_IO_OK;
    const int64_t per = (int64_t)(kPiece / esz);
    const int64_t pieces = (count + per - 1) / per;
    std::atomic<int> bad{0};
    std::atomic<int> bad_errno{0};
    parallel_for(pieces, threads, [&](int64_t pi) {
        if (bad.load()) return;
        const int64_t lo = pi * per, m = std::min(count - lo, per);
        bool ok;
        if (!gen) {
            ok = pwrite_all(fd, (const char *)src + lo * esz, (size_t)m * esz, off + (off_t)(lo * esz));
        } else {
            std::vector<char> tmp((size_t)m * esz);
            gen(tmp.data(), lo, m);
            ok = pwrite_all(fd, tmp.data(), tmp.size(), off + (off_t)(lo * esz));
        }
        if (!ok) {
            bad_errno = errno ? errno : EIO;
            bad = 1;
        }
    });
    if (bad) {
        errno = bad_errno;
        return fail_os(path);
    }
    return GEE_IO_OK;
}

}  // namespace

extern "C" int gee_io_csr_header(const char *path, int *directed, int64_t *n, int64_t *s)
{
    clear_error();
    if (!path) return fail(GEE_IO_ERR_INVALID, "NULL argument");
    Fd f;
    off_t size;
    unsigned char h[kCsrHead];
    if (int rc = open_with_header(path, f, size, h, kCsrHead)) return rc;
    if (memcmp(h, kCsrMagic, 8) != 0) return fail(GEE_IO_ERR_FORMAT, "%s: not a graph cache (bad magic)", path);
    if (h[8] != 1) return fail(GEE_IO_ERR_FORMAT, "%s: unsupported cache version %d", path, (int)h[8]);
    const uint64_t nn = rd_u64(h + 10), ss = rd_u64(h + 18);
    const unsigned __int128 expected =
        (unsigned __int128)kCsrHead + (unsigned __int128)8 * ((unsigned __int128)nn + 1) + (unsigned __int128)12 * ss;
    if (expected != (unsigned __int128)size)
        return fail(GEE_IO_ERR_FORMAT, "%s: expected %s bytes, found %lld", path, u128_str(expected).c_str(),
                    (long long)size);
    if (directed) *directed = h[9];
    if (n) *n = (int64_t)nn;
    if (s) *s = (int64_t)ss;
    return GEE_IO_OK;
}

extern "C" int gee_io_csr_read(const char *path, int64_t n, int64_t s, int64_t *offsets, int32_t *targets,
                               float *w32, double *w64, int threads)
{
    int directed;
    int64_t hn, hs;
    if (int rc = gee_io_csr_header(path, &directed, &hn, &hs)) return rc;
    if (hn != n || hs != s) return fail(GEE_IO_ERR_INVALID, "n/s do not match the file header");
    if ((w32 && w64) || !offsets || (s > 0 && !targets)) return fail(GEE_IO_ERR_INVALID, "bad array arguments");
    Fd f;
    f.fd = open(path, O_RDONLY | O_CLOEXEC);
    if (f.fd < 0) return fail_os(path);
    off_t off = kCsrHead;
    if (int rc = par_read(f.fd, path, off, n + 1, 8, offsets, threads, nullptr)) return rc;
    off += (off_t)(8 * (n + 1));
    if (int rc = par_read(f.fd, path, off, s, 4, targets, threads, nullptr)) return rc;
    off += (off_t)(4 * s);
    if (w64) return par_read(f.fd, path, off, s, 8, w64, threads, nullptr);
    if (w32)
        return par_read(f.fd, path, off, s, 8, nullptr, threads, [&](const char *b, int64_t lo, int64_t m) {
            const double *d = (const double *)b;
            for (int64_t i = 0; i < m; i++) w32[lo + i] = (float)d[i];
        });
    return GEE_IO_OK;
}

extern "C" int gee_io_csr_write(const char *path, int directed, int64_t n, int64_t s, const int64_t *offsets,
                                const int32_t *targets, const float *w, int threads)
{
    clear_error();
    if (!path || n < 0 || s < 0 || !offsets || (s > 0 && !targets)) return fail(GEE_IO_ERR_INVALID, "bad arguments");
    Fd f;
    f.fd = open(path, O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0666);
    if (f.fd < 0) return fail_os(path);
    unsigned char h[kCsrHead];
    memcpy(h, kCsrMagic, 8);
    h[8] = 1;
    h[9] = directed ? 1 : 0;
    const uint64_t nn = (uint64_t)n, ss = (uint64_t)s;
    memcpy(h + 10, &nn, 8);
    memcpy(h + 18, &ss, 8);
    if (!pwrite_all(f.fd, h, kCsrHead, 0)) return fail_os(path);
    off_t off = kCsrHead;
    if (int rc = par_write(f.fd, path, off, n + 1, 8, offsets, threads, nullptr)) return rc;
    off += (off_t)(8 * (n + 1));
    if (int rc = par_write(f.fd, path, off, s, 4, targets, threads, nullptr)) return rc;
    off += (off_t)(4 * s);
    if (int rc = par_write(f.fd, path, off, s, 8, nullptr, threads, [&](char *b, int64_t lo, int64_t m) {
            double *d = (double *)b;
            if (w)
                for (int64_t i = 0; i < m; i++) d[i] = (double)w[lo + i];
            else
                for (int64_t i = 0; i < m; i++) d[i] = 1.0;
        }))
        return rc;
    int fd = f.fd;
    f.fd = -1;
    if (close(fd) != 0) return fail_os(path);
    return GEE_IO_OK;
}

extern "C" int gee_io_emb_header(const char *path, int64_t *n, int64_t *k)
{
    clear_error();
    if (!path) return fail(GEE_IO_ERR_INVALID, "NULL argument");
    Fd f;
    off_t size;
    unsigned char h[kEmbHead];
    if (int rc = open_with_header(path, f, size, h, kEmbHead)) return rc;
    if (memcmp(h, kEmbMagic, 8) != 0) return fail(GEE_IO_ERR_FORMAT, "%s: not an embedding file (bad magic)", path);
    const uint64_t nn = rd_u64(h + 8), kk = rd_u64(h + 16);
    const unsigned __int128 expected = (unsigned __int128)kEmbHead + (unsigned __int128)8 * nn * kk;
    if (expected != (unsigned __int128)size)
        return fail(GEE_IO_ERR_FORMAT, "%s: expected %s bytes, found %lld", path, u128_str(expected).c_str(),
                    (long long)size);
    if (n) *n = (int64_t)nn;
    if (k) *k = (int64_t)kk;
    return GEE_IO_OK;
}

extern "C" int gee_io_emb_read(const char *path, int64_t n, int64_t k, double *z, int threads)
{
    int64_t hn, hk;
    if (int rc = gee_io_emb_header(path, &hn, &hk)) return rc;
    if (hn != n || hk != k) return fail(GEE_IO_ERR_INVALID, "n/k do not match the file header");
    if (n * k > 0 && !z) return fail(GEE_IO_ERR_INVALID, "NULL array argument");
    Fd f;
    f.fd = open(path, O_RDONLY | O_CLOEXEC);
    if (f.fd < 0) return fail_os(path);
    return par_read(f.fd, path, kEmbHead, n * k, 8, z, threads, nullptr);
}

namespace {

// numpy savetxt "%.17g" of one value (zeros short-circuited: most of a
// sparse embedding is 0).
inline char *put_g17(char *o, double v)
{
    if (v == 0) {
        if (std::signbit(v)) *o++ = '-';
        *o++ = '0';
        return o;
    }
    if (std::isnan(v)) {
        memcpy(o, "nan", 3);
        return o + 3;
    }
    return o + sprintf(o, "%.17g", v);
}

}  // namespace

extern "C" int gee_io_emb_write(const char *path, const void *z, int z_is_f64, int64_t n, int64_t k, int fmt,
                                int threads)
{
    clear_error();
    if (!path || n < 0 || k < 0 || (n * k > 0 && !z) || (fmt != 0 && fmt != 1))
        return fail(GEE_IO_ERR_INVALID, "bad arguments");
    const float *zf = (const float *)z;
    const double *zd = (const double *)z;
    if (fmt == 0)
        return write_text_rows(path, n, (size_t)k * 26 + 2, threads, [&](int64_t i, char *o) {
            for (int64_t j = 0; j < k; j++) {
                if (j) *o++ = ',';
                o = put_g17(o, z_is_f64 ? zd[i * k + j] : (double)zf[i * k + j]);
            }
            *o++ = '\n';
            return o;
        });
    Fd f;
    f.fd = open(path, O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0666);
    if (f.fd < 0) return fail_os(path);
    unsigned char h[kEmbHead];
    memcpy(h, kEmbMagic, 8);
    const uint64_t nn = (uint64_t)n, kk = (uint64_t)k;
    memcpy(h + 8, &nn, 8);
    memcpy(h + 16, &kk, 8);
    if (!pwrite_all(f.fd, h, kEmbHead, 0)) return fail_os(path);
    int rc;
    if (z_is_f64)
        rc = par_write(f.fd, path, kEmbHead, n * k, 8, z, threads, nullptr);
    else
        rc = par_write(f.fd, path, kEmbHead, n * k, 8, nullptr, threads, [&](char *b, int64_t lo, int64_t m) {
            double *d = (double *)b;
            for (int64_t i = 0; i < m; i++) d[i] = (double)zf[lo + i];
        });
    if (rc) return rc;
    int fd = f.fd;
    f.fd = -1;
    if (close(fd) != 0) return fail_os(path);
    return GEE_IO_OK;
}

// ===================================================== row-sparse Z expand
namespace {

// dst <- src (bytes), 32-byte non-temporal stores (AVX2) where dst is
// 32-byte aligned: host memory measured 196 GB/s with 32-byte streaming
// stores on the GPU box against ~87 GB/s for ordinary stores
__attribute__((target("avx2"))) inline void stream_copy32(char *dst, const char *src, size_t bytes)
{
    size_t head = (32 - ((uintptr_t)dst & 31)) & 31;
    if (head > bytes) head = bytes;
    memcpy(dst, src, head);
    dst += head, src += head, bytes -= head;
    const size_t body = bytes & ~(size_t)31;
    for (size_t i = 0; i < body; i += 32)
        _mm256_stream_si256(reinterpret_cast<__m256i *>(dst + i),
                            _mm256_loadu_si256(reinterpret_cast<const __m256i *>(src + i)));
    memcpy(dst + body, src + body, bytes - body);
}

static bool have_avx2()
{
    static const bool v = __builtin_cpu_supports("avx2");
    return v;
}

// dst <- src (bytes), 16-byte non-temporal stores where dst is aligned
inline void stream_copy(char *dst, const char *src, size_t bytes)
{
    if (have_avx2()) {
        stream_copy32(dst, src, bytes);
        return;
    }
    size_t head = (16 - ((uintptr_t)dst & 15)) & 15;
    if (head > bytes) head = bytes;
    memcpy(dst, src, head);
    dst += head, src += head, bytes -= head;
    size_t body = bytes & ~(size_t)15;
    for (size_t i = 0; i < body; i += 16)
        _mm_stream_si128(reinterpret_cast<__m128i *>(dst + i), _mm_loadu_si128(reinterpret_cast<const __m128i *>(src + i)));
    memcpy(dst + body, src + body, bytes - body);
}

// AVX-512 rebuild of rows [s0, s1) into stage (row-major, k floats per row):
// each 16-class piece of a row is one masked expand-load of the row's next
// packed values (zeros where the mask is clear) and one masked store, so no
// zero fill and no per-value scatter; returns the advanced value position.
// The masked stores never write past a row's k floats.
__attribute__((target("avx512f,avx512vl,popcnt"))) int64_t expand_rows_avx512(const uint64_t *mask, const float *vals,
                                                                               int64_t pos, int64_t s0, int64_t s1,
                                                                               int k, int mw, float *stage)
{
    for (int64_t r = s0; r < s1; r++) {
        float *row = stage + (r - s0) * k;
        for (int j = 0; j < mw; j++) {
            const uint64_t m = mask[r * mw + j];
            for (int q = 0; q < 4; q++) {
                const int c0 = 64 * j + 16 * q;
                if (c0 >= k) break;
                const __mmask16 mm = (__mmask16)(m >> (16 * q));
                const __m512 v = _mm512_maskz_expandloadu_ps(mm, vals + pos);
                pos += _mm_popcnt_u32((unsigned)mm);
                const int valid = k - c0 < 16 ? k - c0 : 16;
                _mm512_mask_storeu_ps(row + c0, (__mmask16)(valid == 16 ? 0xffffu : (1u << valid) - 1u), v);
            }
        }
    }
    return pos;
}

// dst <- src (bytes), 64-byte non-temporal stores where dst is aligned
__attribute__((target("avx512f"))) void stream_copy64(char *dst, const char *src, size_t bytes)
{
    size_t head = (64 - ((uintptr_t)dst & 63)) & 63;
    if (head > bytes) head = bytes;
    memcpy(dst, src, head);
    dst += head, src += head, bytes -= head;
    const size_t body = bytes & ~(size_t)63;
    for (size_t i = 0; i < body; i += 64)
        _mm512_stream_si512(reinterpret_cast<__m512i *>(dst + i),
                            _mm512_loadu_si512(reinterpret_cast<const void *>(src + i)));
    memcpy(dst + body, src + body, bytes - body);
}

// AVX-512 path unless the CPU lacks it or GEE_IO_SCALAR is set (tests
// compare both paths)
bool use_avx512()
{
    static const bool cpu = __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512vl");
    if (!cpu) return false;
    const char *e = getenv("GEE_IO_SCALAR");
    return !(e && *e && *e != '0');
}

}  // namespace

extern "C" int gee_io_expand_rows(const uint64_t *mask, const float *vals, const int64_t *block_off, int64_t rows,
                                  int32_t k, float *z, int threads)
{
    clear_error();
    if (rows <= 0) return GEE_IO_OK;
    if (k < 1 || !mask || !block_off || !z) return fail(GEE_IO_ERR_INVALID, "bad arguments");
    const int mw = (k + 63) / 64;
    const int64_t nb = (rows + GEE_ZC_BLOCK_ROWS - 1) / GEE_ZC_BLOCK_ROWS;
    if (block_off[nb] > 0 && !vals) return fail(GEE_IO_ERR_INVALID, "NULL vals");
    constexpr int SUB = 32;  // rows staged per streaming copy
    const bool simd = use_avx512();
    parallel_for(nb, threads, [&](int64_t b) {
        thread_local std::vector<float> stage;
        if (stage.size() < (size_t)SUB * k) stage.resize((size_t)SUB * k);
        int64_t pos = block_off[b];
        const int64_t r0 = b * GEE_ZC_BLOCK_ROWS;
        const int64_t r1 = std::min(rows, r0 + GEE_ZC_BLOCK_ROWS);
        if (simd) {
            for (int64_t s0 = r0; s0 < r1; s0 += SUB) {
                const int64_t s1 = std::min(r1, s0 + SUB);
                pos = expand_rows_avx512(mask, vals, pos, s0, s1, k, mw, stage.data());
                stream_copy64(reinterpret_cast<char *>(z + s0 * k), reinterpret_cast<const char *>(stage.data()),
                              (size_t)(s1 - s0) * k * sizeof(float));
            }
            return;
        }
        for (int64_t s0 = r0; s0 < r1; s0 += SUB) {
            const int64_t s1 = std::min(r1, s0 + SUB);
            std::fill(stage.begin(), stage.begin() + (s1 - s0) * k, 0.0f);
            for (int64_t r = s0; r < s1; r++) {
                float *row = stage.data() + (r - s0) * k;
                for (int j = 0; j < mw; j++) {
                    uint64_t m = mask[r * mw + j];
                    while (m) {
                        row[64 * j + __builtin_ctzll(m)] = vals[pos++];
                        m &= m - 1;
                    }
                }
            }
            stream_copy(reinterpret_cast<char *>(z + s0 * k), reinterpret_cast<const char *>(stage.data()),
                        (size_t)(s1 - s0) * k * sizeof(float));
        }
    });
    _mm_sfence();
    return GEE_IO_OK;
}
