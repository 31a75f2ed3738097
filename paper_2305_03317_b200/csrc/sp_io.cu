// sp_io.cu -- native edge-list loader (trident/graph.py:119-151).
//
// Parses the whitespace-separated `u v [w]` text of load_edge_list from a
// memory buffer with all host threads into one [u | v | w] block (host code,
// no device needed; the caller then builds the graph with
// sp_graph_from_edges).  Semantics follow the reference line for line:
//   * lines end at "\n", "\r\n" or "\r" (Python universal newlines), numbered
//     from 1; the last line needs no terminator;
//   * a line is skipped when it is blank or starts with '#' after stripping
//     Python whitespace (ASCII: space \t \n \r \v \f \x1c-\x1f);
//   * 2 or 3 fields (str.split()) -> else kind 1 ("expected 2 or 3 fields");
//   * every field parses like int(): optional sign, decimal digits with
//     single '_' between digits -> else kind 2 ("non-integer field");
//   * u < 0 or v < 0 -> kind 3 ("negative vertex id");
//   * the first failing line (smallest number) is reported, exactly the line
//     the reference raises FormatError on.  The host layer rebuilds the
//     reference's message from that line's text (its own repr()).
//   * any byte >= 0x80 -> SP_ERR_UNSUPPORTED: the caller parses with Python
//     (the reference decodes UTF-8 and Unicode whitespace/digits apply).
// Values beyond int32 (ids or weights) -> SP_ERR_UNSUPPORTED with the int64
// min/max, reported by the host layer as the backend's range ArgError.
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <thread>
#include <vector>

#include "sp_common.cuh"

using namespace sp;

namespace {

inline bool py_space(unsigned char c) {
    return c == ' ' || (c >= '\t' && c <= '\r') || (c >= 0x1c && c <= 0x1f);
}

enum { kOk = 0, kFields = 1, kNonInt = 2, kNegative = 3 };

// Python int() of an ASCII field: sign, digits, single '_' between digits.
// Saturates to +-2^62 (only the int32 range matters to the caller).
inline bool py_int(const char *s, const char *e, int64_t *out) {
    bool neg = false;
    if (s < e && (*s == '+' || *s == '-')) neg = *s++ == '-';
    if (s == e) return false;
    int64_t v = 0;
    bool prev_digit = false;
    for (; s < e; s++) {
        const char c = *s;
        if (c >= '0' && c <= '9') {
            if (v < ((int64_t)1 << 58)) v = v * 10 + (c - '0');
            prev_digit = true;
        } else if (c == '_') {
            if (!prev_digit || s + 1 == e || !(s[1] >= '0' && s[1] <= '9')) return false;
            prev_digit = false;
        } else {
            return false;
        }
    }
    *out = neg ? -v : v;
    return true;
}

struct Part {
    const char *b, *e;            // [b, e) holds whole lines
    int64_t lines = 0;            // lines in the part
    int64_t err_line = -1;        // first failing line (local, 1-based)
    int err_kind = kOk;
    bool non_ascii = false;
    std::vector<int32_t> u, v, w;
    int64_t lo = INT64_MAX, hi = INT64_MIN, wlo = INT64_MAX, whi = INT64_MIN;
};

// Next line start after p (handles \r\n as one terminator).
inline const char *next_line(const char *p, const char *e) {
    while (p < e && *p != '\n' && *p != '\r') p++;
    if (p < e && *p == '\r') {
        p++;
        if (p < e && *p == '\n') p++;
    } else if (p < e) {
        p++;
    }
    return p;
}

void scan_non_ascii(Part &pt, const char *from) {
    for (const char *q = from; q < pt.e; q++)
        if ((unsigned char)*q >= 0x80) {
            pt.non_ascii = true;
            return;
        }
}

void parse_lines(Part &pt, int64_t dw);

void parse_part(Part &pt, int64_t dw) {
    parse_lines(pt, dw);
    if (pt.err_kind != kOk && !pt.non_ascii) scan_non_ascii(pt, pt.b);
}

void parse_lines(Part &pt, int64_t dw) {
    const char *p = pt.b;
    while (p < pt.e) {
        const char *ls = p;
        const char *le = p;
        while (le < pt.e && *le != '\n' && *le != '\r') le++;
        p = next_line(ls, pt.e);
        pt.lines++;
        for (const char *q = ls; q < le; q++)
            if ((unsigned char)*q >= 0x80) {
                pt.non_ascii = true;
                return;
            }
        const char *s = ls, *t = le;  // strip
        while (s < t && py_space(*s)) s++;
        while (t > s && py_space(t[-1])) t--;
        if (s == t || *s == '#') continue;
        const char *fb[4], *fe[4];
        int nf = 0;
        for (const char *q = s; q < t;) {
            while (q < t && py_space(*q)) q++;
            if (q >= t) break;
            const char *f0 = q;
            while (q < t && !py_space(*q)) q++;
            if (nf < 4) {
                fb[nf] = f0;
                fe[nf] = q;
            }
            nf++;
        }
        if (nf != 2 && nf != 3) {
            pt.err_line = pt.lines;
            pt.err_kind = kFields;
            return;
        }
        int64_t a, b, c = dw;
        if (!py_int(fb[0], fe[0], &a) || !py_int(fb[1], fe[1], &b) ||
            (nf == 3 && !py_int(fb[2], fe[2], &c))) {
            pt.err_line = pt.lines;
            pt.err_kind = kNonInt;
            return;
        }
        if (a < 0 || b < 0) {
            pt.err_line = pt.lines;
            pt.err_kind = kNegative;
            return;
        }
        pt.lo = std::min(pt.lo, std::min(a, b));
        pt.hi = std::max(pt.hi, std::max(a, b));
        pt.wlo = std::min(pt.wlo, c);
        pt.whi = std::max(pt.whi, c);
        pt.u.push_back((int32_t)a);
        pt.v.push_back((int32_t)b);
        pt.w.push_back((int32_t)c);
    }
}

}  // namespace

extern "C" void sp_free_host(void *p) { free(p); }

extern "C" int sp_parse_edge_text(const char *buf, int64_t len, int64_t default_weight,
                                  int nthreads, int32_t **out, int64_t *info) {
    // info[0] = error kind (0 ok), info[1] = error line, info[2..3] = id
    // min/max, info[4..5] = weight min/max, info[6] = edges, info[7] = the
    // stride of the [u | v | w] block in *out
    SP_CHECK(out && info && (buf || len == 0) && len >= 0, SP_ERR_ARG,
             "sp_parse_edge_text: bad arguments");
    *out = nullptr;
    for (int i = 0; i < 8; i++) info[i] = 0;
    int T = nthreads > 0 ? nthreads : (int)std::thread::hardware_concurrency();
    T = std::max(1, std::min(T, 64));
    if (len < (int64_t)1 << 20) T = 1;
    std::vector<Part> parts(T);
    const char *e = buf + len;
    const char *cur = buf;
    for (int i = 0; i < T; i++) {
        parts[i].b = cur;
        const char *target = i + 1 == T ? e : buf + (len * (i + 1)) / T;
        if (target < cur) target = cur;
        // move to a line start (never split "\r\n")
        const char *q = target;
        if (q < e && q > buf) {
            if (q[-1] == '\r' && *q == '\n') q++;
            else if (q[-1] != '\n' && q[-1] != '\r') q = next_line(q, e);
        }
        parts[i].e = i + 1 == T ? e : q;
        cur = parts[i].e;
    }
    std::vector<std::thread> th;
    for (int i = 1; i < T; i++) th.emplace_back(parse_part, std::ref(parts[i]), default_weight);
    parse_part(parts[0], default_weight);
    for (auto &t : th) t.join();
    int64_t line0 = 0, ne = 0;
    int64_t lo = INT64_MAX, hi = INT64_MIN, wlo = INT64_MAX, whi = INT64_MIN;
    for (int i = 0; i < T; i++)
        if (parts[i].non_ascii) {
            set_error("non-ASCII edge-list text: parsed by the host layer");
            return SP_ERR_UNSUPPORTED;
        }
    for (int i = 0; i < T; i++) {
        Part &pt = parts[i];
        if (pt.err_kind != kOk) {  // the earliest part with an error holds the first one
            info[0] = pt.err_kind;
            info[1] = line0 + pt.err_line;
            set_error("line %lld: malformed edge-list line", (long long)info[1]);
            return SP_ERR_ARG;
        }
        line0 += pt.lines;
        ne += (int64_t)pt.u.size();
        lo = std::min(lo, pt.lo);
        hi = std::max(hi, pt.hi);
        wlo = std::min(wlo, pt.wlo);
        whi = std::max(whi, pt.whi);
    }
    info[2] = lo;
    info[3] = hi;
    info[4] = wlo;
    info[5] = whi;
    info[6] = ne;
    if (ne && (hi > 2147483647 || wlo < -2147483647 - 1LL || whi > 2147483647)) {
        set_error("edge-list values outside the int32 range");
        return SP_ERR_UNSUPPORTED;
    }
    // one host block [u | v | w] for the caller (sp_free_host)
    const int64_t cap = std::max<int64_t>(1, ne);
    int32_t *blk = (int32_t *)malloc((size_t)cap * 3 * sizeof(int32_t));
    SP_CHECK(blk, SP_ERR_OOM, "host allocation of %lld edges failed", (long long)ne);
    int64_t at = 0;
    std::vector<std::thread> cp;
    for (int i = 0; i < T; i++) {
        const int64_t off = at;
        at += (int64_t)parts[i].u.size();
        cp.emplace_back([&, i, off]() {
            const Part &pt = parts[i];
            if (pt.u.empty()) return;
            memcpy(blk + off, pt.u.data(), pt.u.size() * 4);
            memcpy(blk + cap + off, pt.v.data(), pt.v.size() * 4);
            memcpy(blk + 2 * cap + off, pt.w.data(), pt.w.size() * 4);
        });
    }
    for (auto &t : cp) t.join();
    *out = blk;
    info[7] = cap;
    return SP_OK;
}
