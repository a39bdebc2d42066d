// gk_ensio.cpp -- native ensemble JSON loader (host C++, no CUDA).  SURVEY §8(f)#3.
//
// Parses the portable ensemble document (reference power.py:73-125) straight
// into the flat breadth-first node layout of gk.h, trees in parallel.  The
// accepted language is the reference's: json.loads (duplicate keys -> last
// wins, NaN / Infinity literals, int vs float tokens) followed by
// load_ensemble's checks and _validate_tree (power.py:36-70).  Whenever the
// outcome would be an exception -- or the document uses something this loader
// does not model -- it reports GK_ENS_NEEDS_REFERENCE_PATH and the Python loader
// produces the reference's exact behaviour.
#include "gk_ensio.h"

#include <algorithm>
#include <charconv>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

namespace {

struct Bail {
    const char *why;
};

struct Cursor {
    const char *p, *end;
};

inline void ws(Cursor &c) {
    while (c.p < c.end && (*c.p == ' ' || *c.p == '\t' || *c.p == '\n' || *c.p == '\r')) c.p++;
}
inline bool eat(Cursor &c, char ch) {
    ws(c);
    if (c.p < c.end && *c.p == ch) {
        c.p++;
        return true;
    }
    return false;
}
inline void expect(Cursor &c, char ch, const char *why) {
    if (!eat(c, ch)) throw Bail{why};
}

void put_utf8(std::string &o, uint32_t cp) {
    if (cp < 0x80) {
        o.push_back((char)cp);
    } else if (cp < 0x800) {
        o.push_back((char)(0xC0 | (cp >> 6)));
        o.push_back((char)(0x80 | (cp & 0x3F)));
    } else if (cp < 0x10000) {
        o.push_back((char)(0xE0 | (cp >> 12)));
        o.push_back((char)(0x80 | ((cp >> 6) & 0x3F)));
        o.push_back((char)(0x80 | (cp & 0x3F)));
    } else {
        o.push_back((char)(0xF0 | (cp >> 18)));
        o.push_back((char)(0x80 | ((cp >> 12) & 0x3F)));
        o.push_back((char)(0x80 | ((cp >> 6) & 0x3F)));
        o.push_back((char)(0x80 | (cp & 0x3F)));
    }
}

uint32_t hex4(Cursor &c) {
    if (c.end - c.p < 4) throw Bail{"bad \\u escape"};
    uint32_t v = 0;
    for (int k = 0; k < 4; k++) {
        const char h = *c.p++;
        v <<= 4;
        if (h >= '0' && h <= '9') v |= (uint32_t)(h - '0');
        else if (h >= 'a' && h <= 'f') v |= (uint32_t)(h - 'a' + 10);
        else if (h >= 'A' && h <= 'F') v |= (uint32_t)(h - 'A' + 10);
        else throw Bail{"bad \\u escape"};
    }
    return v;
}

// a JSON string (cursor at the opening quote); lone surrogates -> reference path
void string(Cursor &c, std::string &o) {
    ws(c);
    if (c.p >= c.end || *c.p != '"') throw Bail{"expected a string"};
    c.p++;
    o.clear();
    while (true) {
        if (c.p >= c.end) throw Bail{"unterminated string"};
        const unsigned char ch = (unsigned char)*c.p++;
        if (ch == '"') return;
        if (ch < 0x20) throw Bail{"control character in string"};
        if (ch != '\\') {
            o.push_back((char)ch);
            continue;
        }
        if (c.p >= c.end) throw Bail{"bad escape"};
        const char e = *c.p++;
        switch (e) {
            case '"': o.push_back('"'); break;
            case '\\': o.push_back('\\'); break;
            case '/': o.push_back('/'); break;
            case 'b': o.push_back('\b'); break;
            case 'f': o.push_back('\f'); break;
            case 'n': o.push_back('\n'); break;
            case 'r': o.push_back('\r'); break;
            case 't': o.push_back('\t'); break;
            case 'u': {
                uint32_t cp = hex4(c);
                if (cp >= 0xD800 && cp < 0xDC00) {
                    if (c.end - c.p < 6 || c.p[0] != '\\' || c.p[1] != 'u') throw Bail{"lone surrogate"};
                    c.p += 2;
                    const uint32_t lo = hex4(c);
                    if (lo < 0xDC00 || lo >= 0xE000) throw Bail{"lone surrogate"};
                    cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                } else if (cp >= 0xDC00 && cp < 0xE000) {
                    throw Bail{"lone surrogate"};
                }
                put_utf8(o, cp);
                break;
            }
            default: throw Bail{"bad escape"};
        }
    }
}

struct Num {
    double v = 0.0;
    bool is_int = false;   // a JSON integer token
    bool exact = true;     // the integer is exactly representable (|n| <= 2^53)
    int64_t i = 0;
};

// a JSON number (Python json grammar) or NaN / Infinity / -Infinity
bool number(Cursor &c, Num &n) {
    ws(c);
    const char *s = c.p;
    auto lit = [&](const char *w, double v) {
        const size_t L = std::strlen(w);
        if ((size_t)(c.end - c.p) >= L && std::memcmp(c.p, w, L) == 0) {
            c.p += L;
            n.v = v;
            n.is_int = false;
            return true;
        }
        return false;
    };
    if (lit("NaN", NAN) || lit("Infinity", INFINITY) || lit("-Infinity", -INFINITY)) return true;
    const char *q = c.p;
    if (q < c.end && *q == '-') q++;
    if (q >= c.end || !(*q >= '0' && *q <= '9')) return false;
    if (*q == '0') q++;
    else
        while (q < c.end && *q >= '0' && *q <= '9') q++;
    bool is_int = true;
    if (q < c.end && *q == '.') {
        const char *d = ++q;
        while (q < c.end && *q >= '0' && *q <= '9') q++;
        if (q == d) return false;
        is_int = false;
    }
    if (q < c.end && (*q == 'e' || *q == 'E')) {
        q++;
        if (q < c.end && (*q == '+' || *q == '-')) q++;
        const char *d = q;
        while (q < c.end && *q >= '0' && *q <= '9') q++;
        if (q == d) return false;
        is_int = false;
    }
    c.p = q;
    n.is_int = is_int;
    const size_t L = (size_t)(q - s);
    if (is_int) {
        const size_t digits = L - (*s == '-');
        n.exact = digits <= 15;
        if (n.exact) {
            int64_t v = 0;
            for (const char *d = s + (*s == '-'); d < q; d++) v = v * 10 + (*d - '0');
            n.i = *s == '-' ? -v : v;
            n.v = (double)n.i;  // exact: |i| < 10^15 < 2^53 (and -0 -> 0, like float(-0))
            return true;
        }
    }
    char buf[80];
    if (L < sizeof buf) {
        std::memcpy(buf, s, L);
        buf[L] = 0;
        n.v = std::strtod(buf, nullptr);  // correctly rounded, like float()
    } else {
        n.v = std::strtod(std::string(s, q).c_str(), nullptr);
    }
    return true;
}

void value_skip(Cursor &c, int depth = 0);

void array_skip(Cursor &c, int depth) {
    expect(c, '[', "expected [");
    if (eat(c, ']')) return;
    do value_skip(c, depth + 1);
    while (eat(c, ','));
    expect(c, ']', "expected ]");
}

void object_skip(Cursor &c, int depth) {
    std::string k;
    expect(c, '{', "expected {");
    if (eat(c, '}')) return;
    do {
        string(c, k);
        expect(c, ':', "expected :");
        value_skip(c, depth + 1);
    } while (eat(c, ','));
    expect(c, '}', "expected }");
}

void value_skip(Cursor &c, int depth) {
    if (depth > 500) throw Bail{"nesting too deep"};
    ws(c);
    if (c.p >= c.end) throw Bail{"unexpected end"};
    const char ch = *c.p;
    if (ch == '{') return object_skip(c, depth);
    if (ch == '[') return array_skip(c, depth);
    if (ch == '"') {
        std::string s;
        return string(c, s);
    }
    for (const char *w : {"true", "false", "null"}) {
        const size_t L = std::strlen(w);
        if ((size_t)(c.end - c.p) >= L && std::memcmp(c.p, w, L) == 0) {
            c.p += L;
            return;
        }
    }
    Num n;
    if (!number(c, n)) throw Bail{"bad value"};
}

// the extent of one JSON value (objects / arrays by bracket depth, strings with
// escapes), without validating it: tree elements are re-parsed in full by
// parse_tree (in parallel), which must consume exactly this span
void value_span(Cursor &c) {
    ws(c);
    if (c.p >= c.end) throw Bail{"unexpected end"};
    if (*c.p != '{' && *c.p != '[') return value_skip(c);
    int depth = 0;
    while (c.p < c.end) {
        const char ch = *c.p++;
        if (ch == '"') {
            while (true) {
                const char *q = static_cast<const char *>(std::memchr(c.p, '"', (size_t)(c.end - c.p)));
                if (!q) throw Bail{"unterminated string"};
                const char *b = q;
                while (b > c.p && b[-1] == '\\') b--;
                c.p = q + 1;
                if (((q - b) & 1) == 0) break;  // an even run of backslashes: closing quote
            }
        } else if (ch == '{' || ch == '[') {
            depth++;
        } else if (ch == '}' || ch == ']') {
            if (--depth == 0) return;
        }
    }
    throw Bail{"unbalanced value"};
}

Num need_number(Cursor &c, const char *why) {
    Num n;
    if (!number(c, n)) throw Bail{why};
    if (n.is_int && !n.exact) throw Bail{"integer beyond 2^53"};
    return n;
}

void number_array(Cursor &c, std::vector<double> &out, const char *why) {
    out.clear();
    expect(c, '[', why);
    if (eat(c, ']')) return;
    do out.push_back(need_number(c, why).v);
    while (eat(c, ','));
    expect(c, ']', why);
}

// ----------------------------------------------------------------- trees

struct Tree {
    // original order
    std::vector<int32_t> feat, left, right;
    std::vector<double> val;
    std::vector<uint8_t> kind;
    // flat (BFS) order
    std::vector<double> fv;
    std::vector<int32_t> ff, fl;
    int32_t depth = 0;
    const char *bail = nullptr;
};

void parse_tree(const char *b, const char *e, int n_feat, Tree &T) {
    Cursor c{b, e};
    std::string key;
    const char *nodes_at = nullptr;
    expect(c, '{', "tree must be an object");
    if (!eat(c, '}')) {
        do {
            string(c, key);
            expect(c, ':', "expected :");
            ws(c);
            if (key == "nodes") nodes_at = c.p;  // last occurrence wins
            value_skip(c);
        } while (eat(c, ','));
        expect(c, '}', "expected }");
    }
    ws(c);
    if (c.p != e) throw Bail{"tree span"};
    if (!nodes_at) throw Bail{"tree without nodes"};
    c.p = nodes_at;
    expect(c, '[', "nodes must be a list");
    if (!eat(c, ']')) {
        do {
            // one node object; unknown keys or non-number fields -> reference path
            bool has_v = false, has_f = false, has_t = false, has_l = false, has_r = false;
            Num v, f, t, l, r;
            expect(c, '{', "node must be an object");
            if (!eat(c, '}')) {
                do {
                    string(c, key);
                    expect(c, ':', "expected :");
                    if (key == "value") {
                        v = need_number(c, "leaf value");
                        has_v = true;
                    } else if (key == "threshold") {
                        t = need_number(c, "threshold");
                        has_t = true;
                    } else if (key == "feature" || key == "left" || key == "right") {
                        Num x = need_number(c, "index");
                        if (!x.is_int) throw Bail{"non-integer index"};
                        if (key == "feature") f = x, has_f = true;
                        else if (key == "left") l = x, has_l = true;
                        else r = x, has_r = true;
                    } else {
                        throw Bail{"unknown node key"};
                    }
                } while (eat(c, ','));
                expect(c, '}', "expected }");
            }
            if (has_v) {
                if (has_f || has_t || has_l || has_r) throw Bail{"leaf with split keys"};
                T.feat.push_back(-1);
                T.left.push_back(-1);
                T.right.push_back(-1);
                T.val.push_back(v.v);
                T.kind.push_back((uint8_t)(GK_ENS_LEAF | (v.is_int ? GK_ENS_VALUE_INT : 0)));
            } else {
                if (!(has_f && has_t && has_l && has_r)) throw Bail{"split missing a key"};
                if (f.i < 0 || f.i >= n_feat) throw Bail{"feature out of range"};
                T.feat.push_back((int32_t)f.i);
                T.left.push_back(l.i < 0 || l.i > INT32_MAX ? -1 : (int32_t)l.i);
                T.right.push_back(r.i < 0 || r.i > INT32_MAX ? -1 : (int32_t)r.i);
                if (l.i < 0 || r.i < 0) throw Bail{"child out of range"};
                T.val.push_back(t.v);
                T.kind.push_back((uint8_t)(t.is_int ? GK_ENS_VALUE_INT : 0));
            }
        } while (eat(c, ','));
        expect(c, ']', "expected ]");
    }
    const int64_t n = (int64_t)T.feat.size();
    if (n == 0) throw Bail{"tree has no nodes"};
    for (int64_t i = 0; i < n; i++)
        if (!(T.kind[i] & GK_ENS_LEAF) && (T.left[i] >= n || T.right[i] >= n))
            throw Bail{"child out of range"};
    // reached exactly once from the root (power.py:56-70)
    std::vector<uint8_t> seen((size_t)n, 0);
    std::vector<int32_t> stack{0};
    while (!stack.empty()) {
        const int32_t i = stack.back();
        stack.pop_back();
        if (seen[i]) throw Bail{"node reached twice"};
        seen[i] = 1;
        if (!(T.kind[i] & GK_ENS_LEAF)) {
            stack.push_back(T.left[i]);
            stack.push_back(T.right[i]);
        }
    }
    for (int64_t i = 0; i < n; i++)
        if (!seen[i]) throw Bail{"unreachable node"};
    // breadth-first renumbering, children adjacent (ensemble._flatten_tree)
    std::vector<int32_t> order{0}, dep{0};
    order.reserve((size_t)n);
    dep.reserve((size_t)n);
    T.fv.resize((size_t)n);
    T.ff.resize((size_t)n);
    T.fl.resize((size_t)n);
    for (size_t k = 0; k < order.size(); k++) {
        const int32_t o = order[k];
        if (T.kind[o] & GK_ENS_LEAF) {
            T.fv[k] = T.val[o];
            T.ff[k] = -1;
            T.fl[k] = (int32_t)k - 1;
        } else {
            const int32_t lft = (int32_t)order.size();
            order.push_back(T.left[o]);
            order.push_back(T.right[o]);
            dep.push_back(dep[k] + 1);
            dep.push_back(dep[k] + 1);
            T.depth = std::max(T.depth, dep[k] + 1);
            T.fv[k] = T.val[o];
            T.ff[k] = T.feat[o];
            T.fl[k] = lft;
        }
    }
}

struct Handle {
    std::vector<Tree> trees;
    std::vector<int64_t> off;
    std::vector<double> lo, hi, gains;
    std::vector<std::string> manifest;
    double base = 0.0;
    uint64_t n_nodes = 0;
    uint32_t max_depth = 0;
};

void parse_doc(const char *text, size_t len, int n_threads, Handle &H) {
    Cursor c{text, text + len};
    std::string key;
    bool have_ver = false, have_man = false, have_sc = false, have_trees = false, have_gains = false;
    Num ver;
    std::vector<std::pair<const char *, const char *>> spans;
    std::vector<double> smin, smax;
    bool have_min = false, have_max = false;
    expect(c, '{', "document must be an object");
    if (!eat(c, '}')) {
        do {
            string(c, key);
            expect(c, ':', "expected :");
            if (key == "schema_version") {
                ws(c);
                if (!number(c, ver)) {  // true == 1 in Python, strings -> error: reference path
                    throw Bail{"schema_version"};
                }
                have_ver = true;
            } else if (key == "base_score") {
                H.base = need_number(c, "base_score").v;
            } else if (key == "feature_manifest") {
                H.manifest.clear();
                expect(c, '[', "feature_manifest must be a list");
                if (!eat(c, ']')) {
                    std::string s;
                    do {
                        string(c, s);
                        H.manifest.push_back(s);
                    } while (eat(c, ','));
                    expect(c, ']', "expected ]");
                }
                have_man = true;
            } else if (key == "scaling") {
                have_min = have_max = false;
                expect(c, '{', "scaling must be an object");
                if (!eat(c, '}')) {
                    std::string k2;
                    do {
                        string(c, k2);
                        expect(c, ':', "expected :");
                        if (k2 == "min") number_array(c, smin, "scaling.min"), have_min = true;
                        else if (k2 == "max") number_array(c, smax, "scaling.max"), have_max = true;
                        else value_skip(c);
                    } while (eat(c, ','));
                    expect(c, '}', "expected }");
                }
                have_sc = true;
            } else if (key == "trees") {
                spans.clear();
                expect(c, '[', "trees must be a list");
                if (!eat(c, ']')) {
                    do {
                        ws(c);
                        const char *b = c.p;
                        value_span(c);
                        spans.emplace_back(b, c.p);
                    } while (eat(c, ','));
                    expect(c, ']', "expected ]");
                }
                have_trees = true;
            } else if (key == "gains") {
                number_array(c, H.gains, "gains");
                have_gains = true;
            } else {
                value_skip(c);
            }
        } while (eat(c, ','));
        expect(c, '}', "expected }");
    }
    ws(c);
    if (c.p != c.end) throw Bail{"extra data"};
    // load_ensemble's checks (power.py:86-113), in its order
    const bool ver_ok = have_ver && (ver.is_int ? (ver.exact && ver.i == 1) : ver.v == 1.0);
    if (!ver_ok) throw Bail{"schema_version"};
    if (!have_man || H.manifest.empty()) throw Bail{"feature_manifest"};
    {
        std::vector<std::string> s(H.manifest);
        std::sort(s.begin(), s.end());
        if (std::adjacent_find(s.begin(), s.end()) != s.end()) throw Bail{"duplicate manifest"};
    }
    const size_t k = H.manifest.size();
    if (!have_sc || !have_min || !have_max) throw Bail{"scaling"};
    if (smin.size() != k || smax.size() != k) throw Bail{"scaling length"};
    for (size_t i = 0; i < k; i++)
        if (smax[i] < smin[i]) throw Bail{"scaling max < min"};
    H.lo = smin;
    H.hi = smax;
    if (!have_trees) throw Bail{"trees"};
    if (!have_gains) H.gains.assign(k, 0.0);
    if (H.gains.size() != k) throw Bail{"gains length"};
    for (double g : H.gains)
        if (g < 0) throw Bail{"negative gain"};
    // trees in parallel
    const size_t nt = spans.size();
    H.trees.resize(nt);
    std::atomic<size_t> next{0};
    std::atomic<bool> failed{false};
    const char *why = nullptr;
    std::atomic<const char *> why_a{nullptr};
    auto worker = [&]() {
        while (!failed.load(std::memory_order_relaxed)) {
            const size_t t = next.fetch_add(1);
            if (t >= nt) break;
            try {
                parse_tree(spans[t].first, spans[t].second, (int)k, H.trees[t]);
            } catch (const Bail &b) {
                why_a.store(b.why);
                failed.store(true);
            }
        }
    };
    int th = n_threads > 0 ? n_threads : (int)std::thread::hardware_concurrency();
    th = std::max(1, std::min<int>(th, (int)std::max<size_t>(nt, 1)));
    std::vector<std::thread> pool;
    for (int i = 1; i < th; i++) pool.emplace_back(worker);
    worker();
    for (auto &p : pool) p.join();
    why = why_a.load();
    if (failed.load()) throw Bail{why ? why : "tree"};
    H.off.resize(nt);
    uint64_t o = 0;
    for (size_t t = 0; t < nt; t++) {
        H.off[t] = (int64_t)o;
        o += H.trees[t].fv.size();
        H.max_depth = std::max<uint32_t>(H.max_depth, (uint32_t)H.trees[t].depth);
    }
    H.n_nodes = o;
}

#pragma pack(push, 1)
struct NodeRec {
    double v;
    int32_t feature, left;
};
#pragma pack(pop)
static_assert(sizeof(NodeRec) == 16, "gk_node");

// ------------------------------------------------------------------ writer

// CPython float.__repr__: the shortest digit string that round-trips, fixed
// notation when -4 < decpt <= 16 else exponent (Python/pystrtod.c
// format_float_short, 'r' mode, Py_DTSF_ADD_DOT_0); json's NaN / Infinity.
void put_double(std::string &o, double x) {
    if (std::isnan(x)) {
        o += "NaN";
        return;
    }
    if (std::isinf(x)) {
        o += x > 0 ? "Infinity" : "-Infinity";
        return;
    }
    if (x == 0.0) {
        o += std::signbit(x) ? "-0.0" : "0.0";
        return;
    }
    // shortest round-trip digits (std::to_chars, Ryu: the shortest digit string
    // that parses back to x, the closest one to x among several) -- the same
    // digits CPython's dtoa mode 0 produces
    const bool neg = std::signbit(x);
    const double ax = std::fabs(x);
    char digits[24];
    int nd = 0, e10 = 0;
    {
        char b[64];
        const auto r = std::to_chars(b, b + sizeof b - 1, ax, std::chars_format::scientific);
        *r.ptr = 0;
        const char *q = b;
        while (q < r.ptr && *q != 'e') {
            if (*q != '.') digits[nd++] = *q;
            q++;
        }
        e10 = std::atoi(q + 1);
    }
    while (nd > 1 && digits[nd - 1] == '0') nd--;  // %.*e pads with zeros
    const int decpt = e10 + 1;
    if (neg) o.push_back('-');
    if (decpt <= -4 || decpt > 16) {
        o.push_back(digits[0]);
        if (nd > 1) {
            o.push_back('.');
            o.append(digits + 1, (size_t)(nd - 1));
        }
        char eb[8];
        std::snprintf(eb, sizeof eb, "e%c%02d", e10 < 0 ? '-' : '+', e10 < 0 ? -e10 : e10);
        o += eb;
    } else if (decpt <= 0) {
        o += "0.";
        o.append((size_t)(-decpt), '0');
        o.append(digits, (size_t)nd);
    } else if (decpt < nd) {
        o.append(digits, (size_t)decpt);
        o.push_back('.');
        o.append(digits + decpt, (size_t)(nd - decpt));
    } else {
        o.append(digits, (size_t)nd);
        o.append((size_t)(decpt - nd), '0');
        o += ".0";
    }
}

// json.dumps(str) with ensure_ascii=True (input UTF-8)
void put_string(std::string &o, const char *s, size_t n) {
    static const char *hex = "0123456789abcdef";
    auto u4 = [&](uint32_t v) {
        o += "\\u";
        o.push_back(hex[(v >> 12) & 15]);
        o.push_back(hex[(v >> 8) & 15]);
        o.push_back(hex[(v >> 4) & 15]);
        o.push_back(hex[v & 15]);
    };
    o.push_back('"');
    for (size_t i = 0; i < n;) {
        const unsigned char c = (unsigned char)s[i];
        uint32_t cp;
        int len;
        if (c < 0x80) cp = c, len = 1;
        else if ((c >> 5) == 6) cp = c & 0x1F, len = 2;
        else if ((c >> 4) == 14) cp = c & 0x0F, len = 3;
        else cp = c & 0x07, len = 4;
        for (int k = 1; k < len && i + k < n; k++) cp = (cp << 6) | ((unsigned char)s[i + k] & 0x3F);
        i += (size_t)len;
        switch (cp) {
            case '"': o += "\\\""; continue;
            case '\\': o += "\\\\"; continue;
            case '\n': o += "\\n"; continue;
            case '\r': o += "\\r"; continue;
            case '\t': o += "\\t"; continue;
            case '\b': o += "\\b"; continue;
            case '\f': o += "\\f"; continue;
            default: break;
        }
        if (cp < 0x20 || (cp > 0x7E && cp < 0x10000)) {  // json ESCAPE_ASCII: [^\ -~]
            u4(cp);
        } else if (cp >= 0x10000) {
            const uint32_t v = cp - 0x10000;
            u4(0xD800 + (v >> 10));
            u4(0xDC00 + (v & 0x3FF));
        } else {
            o.push_back((char)cp);
        }
    }
    o.push_back('"');
}

struct Fmt {
    int indent;
    void nl(std::string &o, int level) const {
        if (indent < 0) return;
        o.push_back('\n');
        o.append((size_t)(indent * level), ' ');
    }
    const char *item_sep() const { return indent < 0 ? ", " : ","; }
};

void put_doubles(std::string &o, const Fmt &F, int level, const double *v, size_t n) {
    if (n == 0) {
        o += "[]";
        return;
    }
    o.push_back('[');
    for (size_t i = 0; i < n; i++) {
        if (i) o += F.item_sep();
        F.nl(o, level + 1);
        put_double(o, v[i]);
    }
    F.nl(o, level);
    o.push_back(']');
}

}  // namespace

extern "C" {

int gk_ens_float_repr(const double *x, uint64_t n, char **out, size_t *len) {
    std::string o;
    for (uint64_t i = 0; i < n; i++) {
        if (i) o.push_back(' ');
        put_double(o, x[i]);
    }
    *out = static_cast<char *>(std::malloc(o.size() + 1));
    if (!*out) return -1;
    std::memcpy(*out, o.data(), o.size());
    (*out)[o.size()] = 0;
    *len = o.size();
    return 0;
}

int gk_ens_write(int64_t schema_version, double base_score, const char *manifest,
                 const int64_t *manifest_off, uint64_t n_feat, const double *scale_lo,
                 const double *scale_hi, const double *gains, uint64_t n_trees,
                 const int64_t *node_off, const uint8_t *is_leaf, const int32_t *feature,
                 const double *val, const int32_t *left, const int32_t *right, int indent,
                 int n_threads, char **out, size_t *len) {
    try {
        const Fmt F{indent};
        // trees formatted in parallel (level 2: inside "trees": [ ... ])
        std::vector<std::string> parts(n_trees);
        std::atomic<uint64_t> next{0};
        auto worker = [&]() {
            std::string key;
            while (true) {
                const uint64_t t = next.fetch_add(1);
                if (t >= n_trees) break;
                std::string &o = parts[t];
                o.reserve((size_t)(node_off[t + 1] - node_off[t]) * (indent < 0 ? 60 : 110));
                F.nl(o, 2);
                o.push_back('{');
                F.nl(o, 3);
                o += "\"nodes\": ";
                const int64_t a = node_off[t], b = node_off[t + 1];
                if (a == b) {
                    o += "[]";
                } else {
                    o.push_back('[');
                    for (int64_t i = a; i < b; i++) {
                        if (i > a) o += F.item_sep();
                        F.nl(o, 4);
                        o.push_back('{');
                        if (is_leaf[i]) {
                            F.nl(o, 5);
                            o += "\"value\": ";
                            put_double(o, val[i]);
                        } else {
                            char ib[16];
                            F.nl(o, 5);
                            std::snprintf(ib, sizeof ib, "%d", feature[i]);
                            o += "\"feature\": ";
                            o += ib;
                            o += F.item_sep();
                            F.nl(o, 5);
                            o += "\"threshold\": ";
                            put_double(o, val[i]);
                            o += F.item_sep();
                            F.nl(o, 5);
                            std::snprintf(ib, sizeof ib, "%d", left[i]);
                            o += "\"left\": ";
                            o += ib;
                            o += F.item_sep();
                            F.nl(o, 5);
                            std::snprintf(ib, sizeof ib, "%d", right[i]);
                            o += "\"right\": ";
                            o += ib;
                        }
                        F.nl(o, 4);
                        o.push_back('}');
                    }
                    F.nl(o, 3);
                    o.push_back(']');
                }
                F.nl(o, 2);
                o.push_back('}');
            }
        };
        int th = n_threads > 0 ? n_threads : (int)std::thread::hardware_concurrency();
        th = std::max(1, std::min<int>(th, (int)std::max<uint64_t>(n_trees, 1)));
        std::vector<std::thread> pool;
        for (int i = 1; i < th; i++) pool.emplace_back(worker);
        worker();
        for (auto &p : pool) p.join();

        std::string o;
        size_t total = 4096;
        for (auto &p : parts) total += p.size() + 2;
        o.reserve(total + n_feat * 64);
        char ib[32];
        o.push_back('{');
        F.nl(o, 1);
        std::snprintf(ib, sizeof ib, "%lld", (long long)schema_version);
        o += "\"schema_version\": ";
        o += ib;
        o += F.item_sep();
        F.nl(o, 1);
        o += "\"base_score\": ";
        put_double(o, base_score);
        o += F.item_sep();
        F.nl(o, 1);
        o += "\"feature_manifest\": ";
        if (n_feat == 0) {
            o += "[]";
        } else {
            o.push_back('[');
            for (uint64_t i = 0; i < n_feat; i++) {
                if (i) o += F.item_sep();
                F.nl(o, 2);
                put_string(o, manifest + manifest_off[i], (size_t)(manifest_off[i + 1] - manifest_off[i]));
            }
            F.nl(o, 1);
            o.push_back(']');
        }
        o += F.item_sep();
        F.nl(o, 1);
        o += "\"scaling\": {";
        F.nl(o, 2);
        o += "\"min\": ";
        put_doubles(o, F, 2, scale_lo, n_feat);
        o += F.item_sep();
        F.nl(o, 2);
        o += "\"max\": ";
        put_doubles(o, F, 2, scale_hi, n_feat);
        F.nl(o, 1);
        o.push_back('}');
        o += F.item_sep();
        F.nl(o, 1);
        o += "\"trees\": ";
        if (n_trees == 0) {
            o += "[]";
        } else {
            o.push_back('[');
            for (uint64_t t = 0; t < n_trees; t++) {
                if (t) o += F.item_sep();
                o += parts[t];
                std::string().swap(parts[t]);
            }
            F.nl(o, 1);
            o.push_back(']');
        }
        o += F.item_sep();
        F.nl(o, 1);
        o += "\"gains\": ";
        put_doubles(o, F, 1, gains, n_feat);
        F.nl(o, 0);
        o.push_back('}');
        *out = static_cast<char *>(std::malloc(o.size() + 1));
        if (!*out) return -1;
        std::memcpy(*out, o.data(), o.size());
        (*out)[o.size()] = 0;
        *len = o.size();
        return 0;
    } catch (const std::bad_alloc &) {
        return -1;
    }
}

void gk_ens_buf_free(char *buf) { std::free(buf); }

void *gk_ens_parse(const char *text, size_t len, int n_threads, int *status, char *why,
                   size_t cap) {
    Handle *H = new (std::nothrow) Handle();
    if (!H) return nullptr;
    *status = GK_ENS_OK;
    try {
        parse_doc(text, len, n_threads, *H);
    } catch (const Bail &b) {
        *status = GK_ENS_NEEDS_REFERENCE_PATH;
        if (why && cap) {
            std::strncpy(why, b.why, cap - 1);
            why[cap - 1] = 0;
        }
    } catch (const std::bad_alloc &) {
        delete H;
        return nullptr;
    }
    return H;
}

void gk_ens_sizes_of(const void *h, gk_ens_sizes *out) {
    const Handle *H = static_cast<const Handle *>(h);
    std::memset(out, 0, sizeof *out);
    if (!H) return;
    out->n_trees = H->trees.size();
    out->n_nodes = H->n_nodes;
    out->n_feat = H->manifest.size();
    for (const auto &m : H->manifest) out->manifest_bytes += m.size();
    out->max_depth = H->max_depth;
    out->base_score = H->base;
}

int gk_ens_copy(const void *h, void *nodes, int64_t *tree_off, int32_t *tree_depth,
                double *scale_lo, double *scale_hi, double *gains, char *manifest,
                int64_t *manifest_off, int32_t *orig_feature, double *orig_value,
                int32_t *orig_left, int32_t *orig_right, uint8_t *orig_kind) {
    const Handle *H = static_cast<const Handle *>(h);
    if (!H) return -1;
    NodeRec *nd = static_cast<NodeRec *>(nodes);
    for (size_t t = 0; t < H->trees.size(); t++) {
        const Tree &T = H->trees[t];
        const size_t o = (size_t)H->off[t], n = T.fv.size();
        if (tree_off) tree_off[t] = H->off[t];
        if (tree_depth) tree_depth[t] = T.depth;
        for (size_t i = 0; i < n; i++) {
            if (nd) nd[o + i] = NodeRec{T.fv[i], T.ff[i], T.fl[i]};
            if (orig_feature) orig_feature[o + i] = T.feat[i];
            if (orig_value) orig_value[o + i] = T.val[i];
            if (orig_left) orig_left[o + i] = T.left[i];
            if (orig_right) orig_right[o + i] = T.right[i];
            if (orig_kind) orig_kind[o + i] = T.kind[i];
        }
    }
    const size_t k = H->manifest.size();
    if (scale_lo) std::memcpy(scale_lo, H->lo.data(), k * sizeof(double));
    if (scale_hi) std::memcpy(scale_hi, H->hi.data(), k * sizeof(double));
    if (gains) std::memcpy(gains, H->gains.data(), k * sizeof(double));
    if (manifest && manifest_off) {
        int64_t at = 0;
        for (size_t i = 0; i < k; i++) {
            manifest_off[i] = at;
            std::memcpy(manifest + at, H->manifest[i].data(), H->manifest[i].size());
            at += (int64_t)H->manifest[i].size();
        }
        manifest_off[k] = at;
    }
    return 0;
}

void gk_ens_free(void *h) { delete static_cast<Handle *>(h); }

}  // extern "C"
