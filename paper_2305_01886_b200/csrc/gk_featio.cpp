// gk_featio.cpp -- feature-CSV writer / parser (include/gk_featio.h).
//
// Host-only C++ in libgkhost.so.  The writer reproduces the reference's
// features_to_csv (features.py:250-261: csv.writer with the excel dialect,
// lineterminator "\n", values format(v, ".17g")); the parser reproduces
// features_from_csv (features.py:264-272: csv.DictReader + float()) on the
// plain dialect and declines everything else (see the header).  Rows are
// formatted / parsed in parallel over row chunks.

#include "gk_featio.h"

#include <locale.h>

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

namespace {

int n_workers(int n_threads, int64_t work) {
    int th = n_threads > 0 ? n_threads : (int)std::thread::hardware_concurrency();
    if (th < 1) th = 1;
    return (int)std::min<int64_t>(th, std::max<int64_t>(1, work));
}

template <class F>
void run_parallel(int th, F &&body) {
    if (th == 1) {
        body(0);
        return;
    }
    std::vector<std::thread> pool;
    pool.reserve(th);
    for (int t = 0; t < th; t++) pool.emplace_back(body, t);
    for (auto &p : pool) p.join();
}

// ---------------------------------------------------------------- writer

// csv QUOTE_MINIMAL (CPython _csv.c join_append_data): quote when the field
// holds the delimiter, the quote char, '\r' or '\n'; double embedded quotes.
void put_field(std::string &s, std::string_view f) {
    if (f.find_first_of(",\"\r\n") == std::string_view::npos) {
        s.append(f);
        return;
    }
    s.push_back('"');
    for (char c : f) {
        if (c == '"') s.push_back('"');
        s.push_back(c);
    }
    s.push_back('"');
}

// %.17g by exact 128-bit integer arithmetic for 1e-5 <= |v| < 1.7e38 (the
// range feature values live in): N = v * 10^(16-k) rounded half-even to an
// integer of 17 digits, then printf's %g layout.  Returns the length, or 0
// outside the range (the caller takes std::to_chars' exact general path).
// Cross-checked against CPython's format(v, ".17g") in tests/test_featio.py.
using u128 = unsigned __int128;

struct Pow10 {
    u128 p[24];
    Pow10() {
        p[0] = 1;
        for (int i = 1; i < 24; i++) p[i] = p[i - 1] * 10;
    }
};
const Pow10 kPow10;

const char kDigits2[] =
    "00010203040506070809101112131415161718192021222324252627282930313233343536373839"
    "40414243444546474849505152535455565758596061626364656667686970717273747576777879"
    "8081828384858687888990919293949596979899";

int g17_fast(double v, char *out) {
    const double a = std::fabs(v);
    if (!(a >= 1e-5) || !(a < 1.7e38)) return 0;
    uint64_t bits;
    memcpy(&bits, &a, sizeof bits);                       // normal here: a = m * 2^e exactly
    const uint64_t m = (bits & ((1ull << 52) - 1)) | (1ull << 52);
    const int e = (int)(bits >> 52) - 1075;
    int k = ((e + 52) * 78913) >> 18;                     // floor(log10 2^(e+52)): k or k - 1
    uint64_t N = 0;
    for (int pass = 0; pass < 4; pass++) {
        const int s = 16 - k;
        if (s > 22) return 0;
        u128 q, r, half;
        bool exact_half_possible = true;
        if (s >= 0) {
            const u128 num = (u128)m * kPow10.p[s];     // < 2^53 * 10^22 < 2^127
            if (e >= 0) {
                q = num << e;                              // v >= 2^52: s <= 1
                r = 0;
                half = 1;
                exact_half_possible = false;
            } else {
                const int sh = -e;
                if (sh >= 127) return 0;
                q = num >> sh;
                r = num & (((u128)1 << sh) - 1);
                half = (u128)1 << (sh - 1);
            }
        } else {
            const u128 num = (u128)m << e;                // e >= 4 here, v < 2^127
            const u128 d = kPow10.p[-s];
            q = num / d;
            r = num % d;
            half = d / 2;                                  // d even: exact half
        }
        if (q < (u128)10000000000000000ULL) {     // v < 10^k (before rounding): k too high
            k -= 1;
            continue;
        }
        if (exact_half_possible && (r > half || (r == half && (q & 1)))) q += 1;
        if (q >= (u128)100000000000000000ULL) {  // k underestimated, or a carry to 10^17:
            k += 1;                               // redo one digit higher
            continue;
        }
        N = (uint64_t)q;
        break;
    }
    if (N == 0) return 0;
    char d[18];
    for (int i = 15; i >= 1; i -= 2) {                    // two digits per step
        const unsigned t = (unsigned)(N % 100);
        N /= 100;
        d[i + 1] = kDigits2[2 * t + 1];
        d[i] = kDigits2[2 * t];
    }
    d[0] = (char)('0' + N);
    int nd = 17;
    char *w = out;
    if (v < 0) *w++ = '-';
    if (k >= -4 && k < 17) {
        if (k >= 0) {
            memcpy(w, d, (size_t)k + 1);
            w += k + 1;
            int last = 16;
            while (last > k && d[last] == '0') last--;
            if (last > k) {
                *w++ = '.';
                memcpy(w, d + k + 1, (size_t)(last - k));
                w += last - k;
            }
        } else {
            while (nd > 1 && d[nd - 1] == '0') nd--;
            *w++ = '0';
            *w++ = '.';
            for (int i = 0; i < -k - 1; i++) *w++ = '0';
            memcpy(w, d, (size_t)nd);
            w += nd;
        }
    } else {
        while (nd > 1 && d[nd - 1] == '0') nd--;
        *w++ = d[0];
        if (nd > 1) {
            *w++ = '.';
            memcpy(w, d + 1, (size_t)nd - 1);
            w += nd - 1;
        }
        *w++ = 'e';
        int x = k;
        *w++ = x < 0 ? '-' : '+';
        if (x < 0) x = -x;
        if (x >= 100) *w++ = (char)('0' + x / 100);
        *w++ = (char)('0' + (x / 10) % 10);
        *w++ = (char)('0' + x % 10);
    }
    return (int)(w - out);
}

// format(v, ".17g"): NaN prints "nan" whatever its sign; everything else is
// printf's %.17g, which std::to_chars(general, 17) is specified to match.
void put_value(std::string &s, double v) {
    if (std::isnan(v)) {
        s.append("nan");
        return;
    }
    if (std::isinf(v)) {
        s.append(v < 0 ? "-inf" : "inf");
        return;
    }
    char b[40];
    const int n = g17_fast(v, b);
    if (n) {
        s.append(b, (size_t)n);
        return;
    }
    const auto r = std::to_chars(b, b + sizeof b, v, std::chars_format::general, 17);
    s.append(b, r.ptr);
}

// ---------------------------------------------------------------- parser

struct Field {
    const char *p;
    size_t n;
    bool quoted;
    bool has_dq;  // quoted with "" escapes
};

struct Parsed {
    int64_t n_rows = 0;
    int32_t n_cols = 0;
    int32_t kernel_col = -1;
    std::string names;
    std::vector<int64_t> names_off;
    std::string kernels;
    std::vector<int64_t> kernels_off;
    std::vector<double> values;
};

locale_t c_locale() {
    static locale_t loc = newlocale(LC_NUMERIC_MASK, "C", (locale_t)0);
    return loc;
}

bool ieq(const char *p, size_t n, const char *lit) {
    if (strlen(lit) != n) return false;
    for (size_t i = 0; i < n; i++) {
        char c = p[i];
        if (c >= 'A' && c <= 'Z') c = (char)(c - 'A' + 'a');
        if (c != lit[i]) return false;
    }
    return true;
}

// float(field) for the strict grammar; false = not in the grammar.
bool parse_number(const char *p, size_t n, double *out) {
    if (n == 0 || n > 400) return false;
    size_t i = 0;
    const bool neg = p[0] == '-';
    if (p[0] == '+' || p[0] == '-') i = 1;
    const char *q = p + i;
    const size_t m = n - i;
    if (ieq(q, m, "nan")) {
        *out = neg ? -std::nan("") : std::nan("");
        return true;
    }
    if (ieq(q, m, "inf") || ieq(q, m, "infinity")) {
        *out = neg ? -HUGE_VAL : HUGE_VAL;
        return true;
    }
    size_t dig = 0;
    while (i < n && p[i] >= '0' && p[i] <= '9') i++, dig++;
    if (i < n && p[i] == '.') {
        i++;
        while (i < n && p[i] >= '0' && p[i] <= '9') i++, dig++;
    }
    if (dig == 0) return false;
    if (i < n && (p[i] == 'e' || p[i] == 'E')) {
        i++;
        if (i < n && (p[i] == '+' || p[i] == '-')) i++;
        size_t ed = 0;
        while (i < n && p[i] >= '0' && p[i] <= '9') i++, ed++;
        if (ed == 0) return false;
    }
    if (i != n) return false;
    const char *f = p[0] == '+' ? p + 1 : p;      // from_chars takes no '+'
    const auto r = std::from_chars(f, p + n, *out);
    if (r.ec == std::errc() && r.ptr == p + n) return true;
    char buf[408];                                  // out of range: strtod's +-inf / +-0
    memcpy(buf, p, n);
    buf[n] = 0;
    *out = strtod_l(buf, nullptr, c_locale());  // correctly rounded, +-inf / +-0 at the ends
    return true;
}

// One record starting at p (< end).  Fills fields; returns the start of the
// next record, or nullptr when the record is outside the accepted dialect.
const char *read_record(const char *p, const char *end, std::vector<Field> &fields) {
    fields.clear();
    for (;;) {
        Field f{p, 0, false, false};
        if (p < end && *p == '"') {
            f.quoted = true;
            const char *s = ++p;
            for (;;) {
                const char *q = (const char *)memchr(p, '"', (size_t)(end - p));
                if (!q) return nullptr;              // unterminated quote
                if (q + 1 < end && q[1] == '"') {
                    f.has_dq = true;
                    p = q + 2;
                    continue;
                }
                f.p = s;
                f.n = (size_t)(q - s);
                p = q + 1;
                break;
            }
        } else {
            const char *s = p;
            while (p < end && *p != ',' && *p != '\n' && *p != '\r') {
                if (*p == '"') return nullptr;       // quote inside an unquoted field
                p++;
            }
            f.p = s;
            f.n = (size_t)(p - s);
        }
        fields.push_back(f);
        if (p == end) return end;
        if (*p == ',') {
            p++;
            continue;
        }
        if (*p == '\r') {
            if (p + 1 < end && p[1] == '\n') return p + 2;
            return nullptr;                          // bare '\r'
        }
        if (*p == '\n') return p + 1;
        return nullptr;                              // text after a closing quote
    }
}

std::string unquote(const Field &f) {
    if (!f.has_dq) return std::string(f.p, f.n);
    std::string s;
    s.reserve(f.n);
    for (size_t i = 0; i < f.n; i++) {
        s.push_back(f.p[i]);
        if (f.p[i] == '"') i++;  // "" -> "
    }
    return s;
}

struct Chunk {
    std::string kernels;
    std::vector<int64_t> klen;
    std::vector<double> values;
    int64_t rows = 0;
    bool ok = true;
    std::string why;
};

}  // namespace

extern "C" {

int gk_featcsv_write(const char *names, const int64_t *names_off, int32_t n_cols,
                     const char *kernels, const int64_t *kernels_off, const double *feat,
                     int64_t n_rows, int64_t ld, const int32_t *cols, int n_threads, char **out,
                     size_t *len) {
    *out = nullptr;
    *len = 0;
    std::string head;
    head.append("kernel");
    for (int32_t j = 0; j < n_cols; j++) {
        head.push_back(',');
        put_field(head, std::string_view(names + names_off[j],
                                         (size_t)(names_off[j + 1] - names_off[j])));
    }
    head.push_back('\n');
    const int th = n_workers(n_threads, n_rows / 2048);
    std::vector<std::string> parts((size_t)th);
    run_parallel(th, [&](int t) {
        const int64_t r0 = n_rows * t / th, r1 = n_rows * (t + 1) / th;
        std::string &s = parts[(size_t)t];
        s.reserve((size_t)(r1 - r0) * (size_t)(24 + 20 * n_cols));
        for (int64_t r = r0; r < r1; r++) {
            put_field(s, std::string_view(kernels + kernels_off[r],
                                          (size_t)(kernels_off[r + 1] - kernels_off[r])));
            const double *row = feat + r * ld;
            for (int32_t j = 0; j < n_cols; j++) {
                s.push_back(',');
                put_value(s, row[cols[j]]);
            }
            s.push_back('\n');
        }
    });
    size_t total = head.size();
    for (auto &s : parts) total += s.size();
    char *buf = (char *)malloc(total + 1);
    if (!buf) return -1;
    char *w = buf;
    memcpy(w, head.data(), head.size());
    w += head.size();
    for (auto &s : parts) {
        memcpy(w, s.data(), s.size());
        w += s.size();
    }
    *w = 0;
    *out = buf;
    *len = total;
    return 0;
}

void gk_featcsv_buf_free(char *buf) { free(buf); }

void *gk_featcsv_parse(const char *text, size_t len, int n_threads, int *status, char *why,
                       size_t cap) {
    Parsed *P = new (std::nothrow) Parsed();
    if (!P) return nullptr;
    auto decline = [&](const std::string &w) {
        *status = GK_FEATCSV_NEEDS_REFERENCE_PATH;
        if (why && cap) snprintf(why, cap, "%s", w.c_str());
        return (void *)P;
    };
    *status = GK_FEATCSV_OK;
    if (why && cap) why[0] = 0;
    P->names_off.push_back(0);
    P->kernels_off.push_back(0);
    const char *p = text, *end = text + len;
    if (p == end) return P;                       // DictReader over "" -> no rows
    std::vector<Field> fields;
    const char *body = read_record(p, end, fields);
    if (!body) return decline("header outside the plain dialect");
    if (fields.size() == 1 && fields[0].n == 0 && !fields[0].quoted)
        return decline("blank header line");
    P->n_cols = (int32_t)fields.size();
    std::vector<std::string> hdr;
    for (size_t j = 0; j < fields.size(); j++) {
        hdr.push_back(unquote(fields[j]));
        for (size_t i = 0; i < j; i++)
            if (hdr[i] == hdr[j]) return decline("duplicate column '" + hdr[j] + "'");
        if (hdr[j] == "kernel") P->kernel_col = (int32_t)j;
        P->names += hdr[j];
        P->names_off.push_back((int64_t)P->names.size());
    }

    // chunk boundaries on record starts: without quotes in the body every
    // '\n' ends a record; with quotes, one serial scan tracks quote state
    const size_t body_len = (size_t)(end - body);
    const bool quotes = body_len && memchr(body, '"', body_len) != nullptr;
    const int th = n_workers(n_threads, (int64_t)(body_len >> 16));
    std::vector<const char *> cut((size_t)th + 1, end);
    cut[0] = body;
    if (!quotes) {
        for (int t = 1; t < th; t++) {
            const char *target = body + body_len * (size_t)t / (size_t)th;
            if (target < cut[(size_t)t - 1]) target = cut[(size_t)t - 1];
            const char *nl = (const char *)memchr(target, '\n', (size_t)(end - target));
            cut[(size_t)t] = nl ? nl + 1 : end;
        }
    } else {
        bool inq = false;
        int t = 1;
        const char *target = body + body_len / (size_t)th;
        for (const char *q = body; q < end && t < th; q++) {
            if (*q == '"') inq = !inq;
            else if (*q == '\n' && !inq && q + 1 > target) {
                cut[(size_t)t++] = q + 1;
                target = body + body_len * (size_t)t / (size_t)th;
            }
        }
    }

    std::vector<Chunk> chunks((size_t)th);
    const int32_t nc = P->n_cols, kc = P->kernel_col;
    run_parallel(th, [&](int t) {
        Chunk &C = chunks[(size_t)t];
        std::vector<Field> f;
        const char *q = cut[(size_t)t], *e = cut[(size_t)t + 1];
        while (q < e) {
            const char *nx = read_record(q, e, f);
            if (!nx) {
                C.ok = false;
                C.why = "record outside the plain dialect";
                return;
            }
            if (f.size() == 1 && f[0].n == 0 && !f[0].quoted) {
                C.ok = false;
                C.why = "blank line";
                return;
            }
            if ((int32_t)f.size() != nc) {
                C.ok = false;
                C.why = "ragged row";
                return;
            }
            for (int32_t j = 0; j < nc; j++) {
                if (j == kc) {
                    const std::string k = unquote(f[(size_t)j]);
                    C.kernels += k;
                    C.klen.push_back((int64_t)k.size());
                    C.values.push_back(0.0);
                    continue;
                }
                double v;
                if (f[(size_t)j].quoted || !parse_number(f[(size_t)j].p, f[(size_t)j].n, &v)) {
                    C.ok = false;
                    C.why = "field outside the numeric grammar";
                    return;
                }
                C.values.push_back(v);
            }
            C.rows++;
            q = nx;
        }
    });
    for (auto &C : chunks)
        if (!C.ok) return decline(C.why);
    for (auto &C : chunks) {
        P->n_rows += C.rows;
        P->values.insert(P->values.end(), C.values.begin(), C.values.end());
        P->kernels += C.kernels;
        for (int64_t l : C.klen) P->kernels_off.push_back(P->kernels_off.back() + l);
    }
    return P;
}

void gk_featcsv_sizes_of(const void *h, gk_featcsv_sizes *out) {
    const Parsed *P = (const Parsed *)h;
    out->n_rows = P->n_rows;
    out->n_cols = P->n_cols;
    out->kernel_col = P->kernel_col;
    out->names_bytes = (int64_t)P->names.size();
    out->kernel_bytes = (int64_t)P->kernels.size();
}

int gk_featcsv_copy(const void *h, char *names, int64_t *names_off, char *kernels,
                    int64_t *kernels_off, double *values) {
    const Parsed *P = (const Parsed *)h;
    if (names) memcpy(names, P->names.data(), P->names.size());
    if (names_off) memcpy(names_off, P->names_off.data(), P->names_off.size() * sizeof(int64_t));
    if (kernels && P->kernel_col >= 0) {
        memcpy(kernels, P->kernels.data(), P->kernels.size());
        memcpy(kernels_off, P->kernels_off.data(), P->kernels_off.size() * sizeof(int64_t));
    }
    if (values) memcpy(values, P->values.data(), P->values.size() * sizeof(double));
    return 0;
}

void gk_featcsv_free(void *h) { delete (Parsed *)h; }

}  // extern "C"
