// gk_ptx.cpp -- native PTX front-end (host C++, no CUDA): PTX text -> the
// packed device records of gk.h, in parallel over kernels.  SURVEY §8(f)#1.
//
// Behaviour restates the reference parser and classifier statement by statement
// (file:line in each function) and this package's host packer (pack.py
// CorpusBuilder.add), so the output is byte-identical to
// pack_corpus([parse_ptx(text, name, loop_counts=...) ...]).
//
// Text handling follows CPython's str semantics for ASCII input: str.strip()
// and the regex `\s` treat \t \n \v \f \r \x1c-\x1f and ' ' as whitespace, `\w`
// is [A-Za-z0-9_].  Non-ASCII input is reported as GK_PTX_UNSUPPORTED (the
// Python parser then handles the batch).
#include "gk_ptx.h"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <cstring>
#include <deque>
#include <functional>
#include <queue>
#include <string>
#include <string_view>
#include <thread>
#include <unordered_map>
#include <unordered_set>
#include <vector>

namespace {

using SV = std::string_view;

// ------------------------------------------------------------ characters

inline bool py_space(unsigned char c) {
    return c == ' ' || (c >= 9 && c <= 13) || (c >= 0x1c && c <= 0x1f);
}
inline bool alpha(unsigned char c) { return (c >= 'A' && c <= 'Z') || (c >= 'a' && c <= 'z'); }
inline bool digit(unsigned char c) { return c >= '0' && c <= '9'; }
inline bool word(unsigned char c) { return alpha(c) || digit(c) || c == '_'; }
inline bool ident_start(unsigned char c) { return alpha(c) || c == '_' || c == '$'; }
inline bool ident_char(unsigned char c) { return word(c) || c == '$'; }

SV strip(SV s) {
    size_t a = 0, b = s.size();
    while (a < b && py_space((unsigned char)s[a])) a++;
    while (b > a && py_space((unsigned char)s[b - 1])) b--;
    return s.substr(a, b - a);
}

// ------------------------------------------------------------ opcode table

enum { C_COMPUTE = 0, C_GLOBAL = 1, C_SHARED = 2, C_MISC = 3 };
enum { R_SP = 0, R_SFU = 1, R_DPU = 2, R_LSU = 3, R_WS = 4 };
constexpr uint8_t F_BRANCH = 0x04, F_GLOAD = 0x08, F_GSTORE = 0x10;

struct Pair {
    uint8_t cls = C_MISC, res = R_WS;
};

// classify.py:26-44 (rules), in the line format of ptx_native.opcode_table_text:
//   F cls res | M roots.. | S name|- cls res | D res | X roots.. | B roots.. | R root cls res
struct Table {
    Pair fallback;
    std::deque<std::string> store;  // owns the names the views below point at
    std::unordered_set<SV> memory_roots, double_exempt, branch_roots;
    std::unordered_map<SV, Pair> spaces, roots;
    SV keep(const std::string &x) {
        store.push_back(x);
        return store.back();
    }
    void add_all(std::unordered_set<SV> &set, const std::vector<std::string> &f) {
        for (size_t q = 1; q < f.size(); q++) set.insert(keep(f[q]));
    }
    bool has_generic = false;
    uint8_t double_res = R_DPU;

    bool parse(const char *text) {
        std::string_view all(text ? text : "");
        size_t pos = 0;
        while (pos < all.size()) {
            size_t e = all.find('\n', pos);
            if (e == SV::npos) e = all.size();
            SV line = all.substr(pos, e - pos);
            pos = e + 1;
            std::vector<std::string> f;
            size_t i = 0;
            while (i < line.size()) {
                while (i < line.size() && line[i] == ' ') i++;
                size_t j = i;
                while (j < line.size() && line[j] != ' ') j++;
                if (j > i) f.emplace_back(line.substr(i, j - i));
                i = j;
            }
            if (f.empty()) continue;
            const std::string &k = f[0];
            auto num = [&](size_t q) { return (uint8_t)std::atoi(f[q].c_str()); };
            if (k == "F" && f.size() == 3) {
                fallback = {num(1), num(2)};
            } else if (k == "M") {
                add_all(memory_roots, f);
            } else if (k == "S" && f.size() == 4) {
                std::string name = f[1] == "-" ? std::string() : f[1];
                if (name.empty()) has_generic = true;
                spaces[keep(name)] = {num(2), num(3)};
            } else if (k == "D" && f.size() == 2) {
                double_res = num(1);
            } else if (k == "X") {
                add_all(double_exempt, f);
            } else if (k == "B") {
                add_all(branch_roots, f);
            } else if (k == "R" && f.size() == 4) {
                roots[keep(f[1])] = {num(2), num(3)};
            } else {
                return false;
            }
        }
        return true;
    }
};

// parser.py:22-31
const std::unordered_set<SV> &special_regs() {
    static const std::unordered_set<SV> s = {
        "%tid", "%ntid", "%ctaid", "%nctaid", "%laneid", "%warpid", "%nwarpid",
        "%smid", "%nsmid", "%gridid", "%clock", "%clock64", "%clock_hi",
        "%lanemask_eq", "%lanemask_le", "%lanemask_lt", "%lanemask_ge",
        "%lanemask_gt", "%WARP_SZ"};
    return s;
}
const std::unordered_set<SV> &no_dest_roots() {
    static const std::unordered_set<SV> s = {
        "st", "bra", "bar", "ret", "call", "exit", "red", "membar", "fence", "trap", "nop",
        "prefetch"};
    return s;
}
// profiles.py FLOAT_KINDS / INT_KINDS (latency kind of the first typed suffix)
char kind_of(SV piece) {
    static const std::unordered_set<SV> fk = {"f16", "f16x2", "f32", "f64", "bf16"};
    static const std::unordered_set<SV> ik = {
        "s8", "s16", "s32", "s64", "u8", "u16", "u32", "u64", "b8", "b16", "b32", "b64", "pred"};
    if (fk.count(piece)) return 'f';
    if (ik.count(piece)) return 's';
    return 0;
}

// ------------------------------------------------------------ per kernel

struct Error {
    int kind = GK_PTX_OK;
    int64_t line = -1;
    std::string msg;
};

struct Inst {
    SV root, target;       // target = operands[0] (branch label)
    uint8_t cls, res;
    char kind;             // latency kind of the suffixes
    bool branch, pred, ret_exit, gload, gstore;
    uint32_t use0, n_use, def0, n_def;  // into the kernel's register pool
    int64_t line;
};

struct Block {
    SV label;
    bool labelled = false;
    uint32_t i0 = 0, n = 0;  // instruction range
};

struct Packed {
    Error err;
    std::vector<std::pair<uint64_t, std::string>> warnings;  // (kernel, opcode)
    // tokens: res, flags, local sig, lst_row, lst_len, n_pred
    struct Tok {
        uint8_t res, flags;
        uint32_t sig;
        uint16_t row, len;
        uint32_t npred;
    };
    std::vector<Tok> tok;
    std::vector<uint16_t> preds;
    struct Blk {
        int64_t mult;
        uint32_t tok0, n, fpred0, n_fpred;
        uint16_t n_glob;
        uint16_t res_cnt[5];
        uint8_t is_exit;
    };
    std::vector<Blk> blk;
    std::vector<uint32_t> fpreds, topo;
    uint32_t max_n = 0;
    std::vector<std::string> sigs;  // local signature keys: cls, kind, root
};

struct Item {
    SV text, name;
    std::vector<std::pair<SV, int64_t>> loops;
};

// parser.py:34-42 -- block comments first (newlines kept), then line comments
std::string strip_comments(SV t) {
    std::string a;
    a.reserve(t.size());
    size_t i = 0;
    while (i < t.size()) {
        size_t p = t.find("/*", i);
        if (p == SV::npos) break;
        size_t q = t.find("*/", p + 2);
        if (q == SV::npos) break;  // an unclosed /* does not match the regex
        a.append(t.substr(i, p - i));
        for (size_t k = p; k < q + 2; k++)
            if (t[k] == '\n') a.push_back('\n');
        i = q + 2;
    }
    a.append(t.substr(i));
    std::string b;
    b.reserve(a.size());
    i = 0;
    while (i < a.size()) {
        size_t p = a.find("//", i);
        if (p == std::string::npos) {
            b.append(a, i, std::string::npos);
            break;
        }
        b.append(a, i, p - i);
        size_t e = a.find('\n', p);
        if (e == std::string::npos) break;
        i = e;
    }
    return b;
}

// parser.py:45-62 (`\.entry\s+([A-Za-z_$][\w$]*)`, first '{' after, brace depth)
bool extract_body(SV text, SV name, SV &body, int64_t &first_line, Error &err) {
    std::vector<SV> seen;
    size_t pos = 0;
    while (true) {
        size_t p = text.find(".entry", pos);
        if (p == SV::npos) break;
        size_t j = p + 6;
        size_t ws = j;
        while (j < text.size() && py_space((unsigned char)text[j])) j++;
        if (j == ws || j >= text.size() || !ident_start((unsigned char)text[j])) {
            pos = p + 1;
            continue;
        }
        size_t s = j;
        while (j < text.size() && ident_char((unsigned char)text[j])) j++;
        SV got = text.substr(s, j - s);
        seen.push_back(got);
        pos = j;
        if (got != name) continue;
        size_t open = text.find('{', j);
        if (open == SV::npos) {
            err = {GK_PTX_VALUE_ERROR, -1, "substring not found"};
            return false;
        }
        int depth = 0;
        for (size_t k = open; k < text.size(); k++) {
            if (text[k] == '{') {
                depth++;
            } else if (text[k] == '}') {
                if (--depth == 0) {
                    body = text.substr(open + 1, k - open - 1);
                    first_line = 1 + (int64_t)std::count(text.begin(), text.begin() + open, '\n');
                    return true;
                }
            }
        }
        err = {GK_PTX_PARSE_ERROR, -1, "unbalanced braces in kernel '" + std::string(name) + "'"};
        return false;
    }
    std::string list;
    for (size_t k = 0; k < seen.size(); k++) {
        if (k) list += ", ";
        list += seen[k];
    }
    err = {GK_PTX_PARSE_ERROR, -1,
           "kernel '" + std::string(name) + "' not found (entries: " + (list.empty() ? "none" : list) +
               ")"};
    return false;
}

class KernelParser {
   public:
    KernelParser(const Table &t, bool strict) : T(t), strict(strict) {}

    void run(const Item &it, uint64_t kidx, Packed &out) {
        out = Packed();
        kidx_ = kidx;
        out_ = &out;
        std::string text = strip_comments(it.text);
        SV body;
        int64_t first_line = 0;
        if (!extract_body(text, it.name, body, first_line, out.err)) return;
        insts.clear();
        blocks.clear();
        pool.clear();
        reg_id.clear();
        if (!split(body, first_line)) return;
        if (blocks.empty()) {
            fail(GK_PTX_PARSE_ERROR, -1, "kernel '" + std::string(it.name) + "' has an empty body");
            return;
        }
        if (!cfg(it)) return;
        pack();
    }

   private:
    const Table &T;
    bool strict;
    uint64_t kidx_ = 0;
    Packed *out_ = nullptr;
    std::vector<Inst> insts;
    std::vector<Block> blocks;
    std::vector<uint32_t> pool;
    std::unordered_map<SV, uint32_t> reg_id;
    std::deque<std::string> own;  // synthesized labels
    std::vector<std::pair<int, int>> edges;
    std::vector<std::pair<std::pair<int, int>, std::pair<bool, int64_t>>> back;  // (src,dst)->trips
    std::vector<SV> pieces_, ops_;
    std::vector<uint32_t> defs_, uses_;

    void fail(int kind, int64_t line, std::string msg) {
        out_->err.kind = kind;
        out_->err.line = line;
        out_->err.msg = std::move(msg);
    }

    uint32_t reg(SV r) {
        auto it = reg_id.find(r);
        if (it != reg_id.end()) return it->second;
        uint32_t id = (uint32_t)reg_id.size();
        reg_id.emplace(r, id);
        return id;
    }

    // classify.py:68-99
    bool classify(SV root, const std::vector<SV> &pieces, Pair &out) {
        const SV r = root;
        if (T.memory_roots.count(r)) {
            for (SV p : pieces) {
                auto it = T.spaces.find(p);
                if (it != T.spaces.end()) {
                    out = it->second;
                    return true;
                }
            }
            auto it = T.spaces.find(SV());
            if (it == T.spaces.end()) {
                fail(GK_PTX_PARSE_ERROR, -1, "opcode table has no generic memory space");
                return false;
            }
            out = it->second;
            return true;
        }
        auto it = T.roots.find(r);
        if (it != T.roots.end()) {
            out = it->second;
            if (out.cls == C_COMPUTE && !T.double_exempt.count(r))
                for (SV p : pieces)
                    if (p == "f64") {
                        out.res = T.double_res;
                        break;
                    }
            return true;
        }
        if (strict) {
            fail(GK_PTX_PARSE_ERROR, -1, "unknown opcode '" + std::string(r) + "'");
            return false;
        }
        out_->warnings.emplace_back(kidx_, std::string(r));
        out = T.fallback;
        return true;
    }

    // parser.py:86-139
    bool parse_instruction(SV stmt, int64_t line) {
        stmt = strip(stmt);
        bool has_pred = false;
        SV pred_reg;
        // ^@(!?)(%[A-Za-z_$][\w$]*)\s+
        if (stmt.size() >= 3 && stmt[0] == '@') {
            size_t j = 1;
            if (j < stmt.size() && stmt[j] == '!') j++;
            if (j + 1 < stmt.size() && stmt[j] == '%' && ident_start((unsigned char)stmt[j + 1])) {
                size_t s = j;
                j += 2;
                while (j < stmt.size() && ident_char((unsigned char)stmt[j])) j++;
                size_t e = j;
                while (j < stmt.size() && py_space((unsigned char)stmt[j])) j++;
                if (j > e) {
                    has_pred = true;
                    pred_reg = stmt.substr(s, e - s);
                    stmt = strip(stmt.substr(j));
                }
            }
        }
        if (stmt.empty()) {
            fail(GK_PTX_PARSE_ERROR, line, "empty statement after predicate");
            return false;
        }
        size_t h = 0;
        while (h < stmt.size() && !py_space((unsigned char)stmt[h])) h++;
        SV head = stmt.substr(0, h);
        size_t r0 = h;
        while (r0 < stmt.size() && py_space((unsigned char)stmt[r0])) r0++;
        SV rest = stmt.substr(r0);
        // [A-Za-z][\w.]* (fullmatch)
        bool ok = !head.empty() && alpha((unsigned char)head[0]);
        for (size_t k = 1; ok && k < head.size(); k++)
            ok = word((unsigned char)head[k]) || head[k] == '.';
        if (!ok) {
            fail(GK_PTX_PARSE_ERROR, line, "unparseable instruction '" + std::string(stmt) + "'");
            return false;
        }
        std::vector<SV> &pieces = pieces_;  // suffixes without their leading '.'
        pieces.clear();
        size_t dot = head.find('.');
        SV root = head.substr(0, dot);
        while (dot != SV::npos) {
            size_t nx = head.find('.', dot + 1);
            pieces.push_back(head.substr(dot + 1, (nx == SV::npos ? head.size() : nx) - dot - 1));
            dot = nx;
        }
        Pair cr;
        if (!classify(root, pieces, cr)) return false;

        // operands: top-level comma split (parser.py:65-83)
        std::vector<SV> &ops = ops_;
        ops.clear();
        {
            int depth = 0;
            size_t start = 0;
            for (size_t k = 0; k < rest.size(); k++) {
                char c = rest[k];
                if (c == '[' || c == '{' || c == '(') depth++;
                else if (c == ']' || c == '}' || c == ')') depth--;
                else if (c == ',' && depth == 0) {
                    ops.push_back(strip(rest.substr(start, k - start)));
                    start = k + 1;
                }
            }
            SV last = strip(rest.substr(std::min(start, rest.size())));
            if (!last.empty()) ops.push_back(last);
        }
        Inst in;
        in.root = root;
        in.target = ops.empty() ? SV() : ops[0];
        in.cls = cr.cls;
        in.res = cr.res;
        in.kind = 0;
        for (SV p : pieces) {
            char k = kind_of(p);
            if (k) {
                in.kind = k;
                break;
            }
        }
        const SV rs = root;
        in.branch = T.branch_roots.count(rs) > 0;
        in.pred = has_pred;
        in.ret_exit = rs == "ret" || rs == "exit";
        in.gload = cr.cls == C_GLOBAL && (rs == "ld" || rs == "ldu");
        in.gstore = cr.cls == C_GLOBAL && rs == "st";
        in.line = line;
        // def / use registers (%[A-Za-z_$][\w$]*(?:\.[xyzw])?)
        std::vector<uint32_t> &defs = defs_, &uses = uses_;
        defs.clear();
        uses.clear();
        const bool dest = !no_dest_roots().count(rs);
        for (size_t k = 0; k < ops.size(); k++) {
            SV op = ops[k];
            const bool as_def = k == 0 && dest && !(op.size() && op[0] == '[');
            size_t q = 0;
            while (q < op.size()) {
                if (op[q] != '%' || q + 1 >= op.size() || !ident_start((unsigned char)op[q + 1])) {
                    q++;
                    continue;
                }
                size_t s = q;
                q += 2;
                while (q < op.size() && ident_char((unsigned char)op[q])) q++;
                size_t stem_end = q;
                if (q + 1 < op.size() && op[q] == '.' &&
                    (op[q + 1] == 'x' || op[q + 1] == 'y' || op[q + 1] == 'z' || op[q + 1] == 'w'))
                    q += 2;
                SV r = op.substr(s, q - s);
                if (as_def && !special_regs().count(op.substr(s, stem_end - s)))
                    defs.push_back(reg(r));
                else
                    uses.push_back(reg(r));
            }
        }
        if (has_pred) uses.push_back(reg(pred_reg));
        in.use0 = (uint32_t)pool.size();
        in.n_use = (uint32_t)uses.size();
        pool.insert(pool.end(), uses.begin(), uses.end());
        in.def0 = (uint32_t)pool.size();
        in.n_def = (uint32_t)defs.size();
        pool.insert(pool.end(), defs.begin(), defs.end());
        insts.push_back(in);
        return true;
    }

    // parser.py:156-213 -- statements, labels, block splitting
    bool split(SV body, int64_t first_line) {
        Block cur;
        cur.i0 = 0;
        auto flush = [&]() {
            if (cur.n || cur.labelled) blocks.push_back(cur);
            cur = Block();
            cur.i0 = (uint32_t)insts.size();
        };
        size_t pos = 0;
        int64_t off = 0;
        while (true) {
            size_t e = body.find('\n', pos);
            SV raw = body.substr(pos, (e == SV::npos ? body.size() : e) - pos);
            const int64_t lineno = first_line + off;
            SV rest = strip(raw);
            while (!rest.empty()) {
                // ^([A-Za-z_$][\w$]*):
                if (ident_start((unsigned char)rest[0])) {
                    size_t j = 1;
                    while (j < rest.size() && ident_char((unsigned char)rest[j])) j++;
                    if (j < rest.size() && rest[j] == ':') {
                        if (cur.n || cur.labelled) flush();
                        cur.label = rest.substr(0, j);
                        cur.labelled = true;
                        rest = strip(rest.substr(j + 1));
                        continue;
                    }
                }
                if (rest[0] == '.' || rest[0] == '{' || rest[0] == '}') break;
                size_t sc = rest.find(';');
                SV stmt = strip(rest.substr(0, sc));
                rest = sc == SV::npos ? SV() : strip(rest.substr(sc + 1));
                if (stmt.empty()) continue;
                if (sc == SV::npos) {
                    fail(GK_PTX_PARSE_ERROR, lineno, "missing ';' after '" + std::string(stmt) + "'");
                    return false;
                }
                if (!parse_instruction(stmt, lineno)) return false;
                cur.n++;
                const Inst &in = insts.back();
                if (in.branch || in.ret_exit) flush();
            }
            if (e == SV::npos) break;
            pos = e + 1;
            off++;
        }
        flush();
        return true;
    }

    // parser.py:214-257 + types.py:79-124 + pack.py CorpusBuilder.add checks
    bool cfg(const Item &it) {
        const int nb = (int)blocks.size();
        std::unordered_map<SV, int> index;
        own.clear();
        for (int i = 0; i < nb; i++) {
            if (blocks[i].label.empty()) {
                own.push_back("bb" + std::to_string(i));
                blocks[i].label = own.back();
            }
            if (index.count(blocks[i].label)) {
                fail(GK_PTX_PARSE_ERROR, -1, "duplicate label '" + std::string(blocks[i].label) + "'");
                return false;
            }
            index.emplace(blocks[i].label, i);
        }
        edges.clear();
        back.clear();
        for (int i = 0; i < nb; i++) {
            const Block &b = blocks[i];
            const Inst *last = b.n ? &insts[b.i0 + b.n - 1] : nullptr;
            if (last && last->branch) {
                auto f = index.find(last->target);
                if (f == index.end()) {
                    fail(GK_PTX_PARSE_ERROR, last->line,
                         "branch to unknown label '" + std::string(last->target) + "'");
                    return false;
                }
                const int j = f->second;
                if (j <= i) back.push_back({{i, j}, {false, 0}});
                else edges.push_back({i, j});
                if (last->pred && i + 1 < nb) edges.push_back({i, i + 1});
            } else if (last && last->ret_exit && !last->pred) {
                continue;
            } else if (i + 1 < nb) {
                edges.push_back({i, i + 1});
            }
        }
        // loop counts: the first back edge into a labelled head takes its count
        std::vector<std::pair<SV, int64_t>> pending(it.loops);
        std::vector<bool> used(pending.size(), false);
        for (auto &be : back) {
            SV head = blocks[be.first.second].label;
            for (size_t q = 0; q < pending.size(); q++)
                if (!used[q] && pending[q].first == head) {
                    used[q] = true;
                    be.second = {true, pending[q].second};
                    break;
                }
        }
        std::vector<std::string> left;
        for (size_t q = 0; q < pending.size(); q++)
            if (!used[q]) left.emplace_back(pending[q].first);
        if (!left.empty()) {
            std::sort(left.begin(), left.end());
            std::string m = "loop counts for labels that head no loop: ";
            for (size_t q = 0; q < left.size(); q++) m += (q ? ", " : "") + left[q];
            fail(GK_PTX_PARSE_ERROR, -1, m);
            return false;
        }
        return true;
    }

    uint32_t sig_id(uint8_t cls, char kind, SV root) {
        std::string key;
        key.push_back((char)('0' + cls));
        if (cls == C_GLOBAL || cls == C_SHARED) {
            key.push_back('-');
        } else {
            key.push_back(kind ? kind : '-');
            key.append(root);
        }
        auto &sigs = out_->sigs;
        auto it = sig_local.find(key);
        if (it != sig_local.end()) return it->second;
        uint32_t id = (uint32_t)sigs.size();
        sig_local.emplace(key, id);
        sigs.push_back(std::move(key));
        return id;
    }
    std::unordered_map<std::string, uint32_t> sig_local;

    void pack() {
        Packed &P = *out_;
        sig_local.clear();
        const int nb = (int)blocks.size();
        // Kahn order, lowest index first (types.py:87-107)
        std::vector<int> indeg(nb, 0);
        std::vector<std::vector<int>> succ(nb);
        std::vector<std::vector<int>> preds_of(nb);
        std::vector<char> has_succ(nb, 0);
        for (auto &e : edges) {
            indeg[e.second]++;
            succ[e.first].push_back(e.second);
            preds_of[e.second].push_back(e.first);
            has_succ[e.first] = 1;
        }
        std::priority_queue<int, std::vector<int>, std::greater<int>> heap;
        for (int i = 0; i < nb; i++)
            if (!indeg[i]) heap.push(i);
        while (!heap.empty()) {
            int u = heap.top();
            heap.pop();
            P.topo.push_back((uint32_t)u);
            for (int v : succ[u])
                if (--indeg[v] == 0) heap.push(v);
        }
        if ((int)P.topo.size() != nb) {
            fail(GK_PTX_SCHEDULE_ERROR, -1, "control-flow graph is cyclic after removing back edges");
            return;
        }
        // loop multipliers (types.py:109-124): exact products, int64 range check
        struct M {
            __int128 v = 1;
            bool zero = false, big = false;
        };
        std::vector<M> mult(nb);
        for (auto &be : back) {
            const int src = be.first.first, dst = be.first.second;
            if (!be.second.first) {
                fail(GK_PTX_SCHEDULE_ERROR, -1,
                     "back edge into block '" + std::string(blocks[dst].label) +
                         "' has no iteration count; supply one per loop");
                return;
            }
            const int64_t f = be.second.second;
            for (int b = dst; b <= src; b++) {
                M &m = mult[b];
                if (f == 0) {
                    m.zero = true;
                } else if (!m.big) {
                    m.v *= f;
                    const __int128 lim = (__int128)1 << 64;
                    if (m.v > lim || m.v < -lim) m.big = true;
                }
            }
        }
        // blocks and tokens (pack.py CorpusBuilder.add)
        std::vector<int32_t> writer;   // last writer per register, this block
        std::vector<uint32_t> wblk;    // block stamp of writer
        writer.assign(reg_id.size(), -1);
        wblk.assign(reg_id.size(), UINT32_MAX);
        std::vector<uint32_t> ps;
        for (int b = 0; b < nb; b++) {
            const Block &B = blocks[b];
            const uint32_t n = B.n;
            if (n > P.max_n) P.max_n = n;
            if (n > 65535) {
                fail(GK_PTX_SCHEDULE_ERROR, -1, "basic block longer than 65535 instructions");
                return;
            }
            uint16_t res_cnt[5] = {0, 0, 0, 0, 0};
            for (uint32_t i = 0; i < n; i++) res_cnt[insts[B.i0 + i].res % 5]++;
            uint16_t res_row[5], seen[5] = {0, 0, 0, 0, 0};
            uint32_t acc = 0;
            for (int r = 0; r < 5; r++) {
                res_row[r] = (uint16_t)acc;
                acc += res_cnt[r];
            }
            uint16_t n_glob = 0;
            const uint32_t t0 = (uint32_t)P.tok.size();
            for (uint32_t i = 0; i < n; i++) {
                const Inst &in = insts[B.i0 + i];
                uint8_t flags = in.cls;
                if (in.branch) flags |= F_BRANCH;
                if (in.cls == C_GLOBAL) {
                    n_glob++;
                    if (in.gload) flags |= F_GLOAD;
                    else if (in.gstore) flags |= F_GSTORE;
                }
                const uint8_t rc = in.res % 5;
                // def-use DAG, last writer wins (parser.py:142-153)
                ps.clear();
                for (uint32_t u = 0; u < in.n_use; u++) {
                    const uint32_t r = pool[in.use0 + u];
                    if (wblk[r] == (uint32_t)b) ps.push_back((uint32_t)writer[r]);
                }
                for (uint32_t d = 0; d < in.n_def; d++) {
                    const uint32_t r = pool[in.def0 + d];
                    writer[r] = (int32_t)i;
                    wblk[r] = (uint32_t)b;
                }
                std::sort(ps.begin(), ps.end());
                ps.erase(std::unique(ps.begin(), ps.end()), ps.end());
                Packed::Tok t;
                t.res = rc;
                t.flags = flags;
                t.sig = sig_id(in.cls, in.kind, in.root);
                t.row = res_row[rc];
                t.len = seen[rc];
                t.npred = (uint32_t)ps.size();
                seen[rc]++;
                for (uint32_t p : ps) P.preds.push_back((uint16_t)p);
                P.tok.push_back(t);
            }
            Packed::Blk rec;
            const M &m = mult[b];
            if (!m.zero && (m.big || m.v >= ((__int128)1 << 63) || m.v < -((__int128)1 << 63))) {
                fail(GK_PTX_SCHEDULE_ERROR, -1, "loop multiplier exceeds int64");
                return;
            }
            rec.mult = m.zero ? 0 : (int64_t)m.v;
            rec.tok0 = t0;
            rec.n = n;
            rec.fpred0 = (uint32_t)P.fpreds.size();
            rec.n_fpred = (uint32_t)preds_of[b].size();
            for (int u : preds_of[b]) P.fpreds.push_back((uint32_t)u);
            rec.n_glob = n_glob;
            for (int r = 0; r < 5; r++) rec.res_cnt[r] = res_cnt[r];
            rec.is_exit = has_succ[b] ? 0 : 1;
            P.blk.push_back(rec);
        }
    }
};

// ------------------------------------------------------------ the handle

#pragma pack(push, 1)
struct TokRec {
    uint8_t res, cls;
    uint16_t sig;
    uint32_t pred0;
    uint16_t lst_row, lst_len;
    uint32_t pad_;
};
#pragma pack(pop)
struct BlkRec {
    int64_t mult;
    uint32_t tok0, n, fpred0;
    uint16_t n_fpred, n_glob;
    uint16_t res_cnt[5];
    uint8_t is_exit, pad_;
};
struct KerRec {
    uint32_t blk0, n_blk, topo0, max_n, tok0, n_tok, pad_[2];
};
static_assert(sizeof(TokRec) == 16, "gk_token");
static_assert(sizeof(BlkRec) == 40, "gk_block");
static_assert(sizeof(KerRec) == 32, "gk_kernel");

struct Handle {
    Error err;
    uint64_t bad = 0;
    std::vector<TokRec> tok;
    std::vector<uint16_t> preds;
    std::vector<BlkRec> blk;
    std::vector<uint32_t> fpreds, topo;
    std::vector<KerRec> ker;
    std::vector<std::string> sigs;
    std::vector<std::pair<uint64_t, std::string>> warnings;
};

}  // namespace

extern "C" {

int gk_ptx_abi_version(void) { return GK_PTX_ABI_VERSION; }

void *gk_ptx_pack(const char *blob, const int64_t *text_begin, const int64_t *text_end,
                  const char *names, const int64_t *name_off, const int64_t *loop_off,
                  const char *labels, const int64_t *label_off, const int64_t *loop_count,
                  uint64_t n, const char *table, int strict, int n_threads) {
    Table T;
    if (!T.parse(table)) return nullptr;
    Handle *H = new (std::nothrow) Handle();
    if (!H) return nullptr;
    std::vector<Item> items(n);
    std::vector<char> ascii(n, 1);
    for (uint64_t i = 0; i < n; i++) {
        Item &it = items[i];
        it.text = SV(blob + text_begin[i], (size_t)(text_end[i] - text_begin[i]));
        it.name = SV(names + name_off[i], (size_t)(name_off[i + 1] - name_off[i]));
        for (int64_t j = loop_off[i]; j < loop_off[i + 1]; j++)
            it.loops.push_back({SV(labels + label_off[j], (size_t)(label_off[j + 1] - label_off[j])),
                                loop_count[j]});
    }
    const bool timing = std::getenv("GK_PTX_TIMING") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto t_start = now();
    std::vector<Packed> outs(n);
    std::atomic<uint64_t> next{0};
    std::atomic<uint64_t> first_bad{UINT64_MAX};
    auto worker = [&]() {
        KernelParser kp(T, strict != 0);
        while (true) {
            const uint64_t i = next.fetch_add(1);
            if (i >= n) break;
            if (i > first_bad.load(std::memory_order_relaxed)) continue;  // past the first error
            const Item &it = items[i];
            bool ok = true;
            for (unsigned char c : it.text) ok &= c < 0x80;
            for (unsigned char c : it.name) ok &= c < 0x80;
            if (!ok) {
                outs[i].err = {GK_PTX_UNSUPPORTED, -1, "non-ASCII PTX text"};
            } else {
                kp.run(it, i, outs[i]);
            }
            if (outs[i].err.kind != GK_PTX_OK) {
                uint64_t cur = first_bad.load();
                while (i < cur && !first_bad.compare_exchange_weak(cur, i)) {
                }
            }
        }
    };
    int nt = n_threads > 0 ? n_threads : (int)std::thread::hardware_concurrency();
    if (nt < 1) nt = 1;
    if ((uint64_t)nt > n) nt = (int)std::max<uint64_t>(n, 1);
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; t++) pool.emplace_back(worker);
    worker();
    for (auto &th : pool) th.join();

    auto t_parsed = now();
    // sequential merge in kernel order (signature ids in first-seen order)
    const uint64_t stop = first_bad.load();
    for (uint64_t i = 0; i < n && i <= stop; i++)
        for (auto &w : outs[i].warnings) H->warnings.push_back(w);
    if (stop != UINT64_MAX) {
        H->err = outs[stop].err;
        H->bad = stop;
        return H;
    }
    std::unordered_map<std::string, uint32_t> gsig;
    uint64_t nt_tok = 0, np = 0, nbk = 0, nfp = 0;
    for (auto &o : outs) {
        nt_tok += o.tok.size();
        np += o.preds.size();
        nbk += o.blk.size();
        nfp += o.fpreds.size();
    }
    H->tok.resize(nt_tok + 1);
    H->preds.reserve(np);
    H->blk.reserve(nbk);
    H->fpreds.reserve(nfp);
    H->topo.reserve(nbk);
    H->ker.reserve(n);
    uint32_t pred0 = 0;
    uint64_t tk = 0;
    std::vector<uint32_t> remap;
    for (uint64_t i = 0; i < n; i++) {
        Packed &o = outs[i];
        remap.resize(o.sigs.size());
        for (size_t s = 0; s < o.sigs.size(); s++) {
            auto it = gsig.find(o.sigs[s]);
            if (it == gsig.end()) {
                it = gsig.emplace(o.sigs[s], (uint32_t)H->sigs.size()).first;
                H->sigs.push_back(o.sigs[s]);
            }
            remap[s] = it->second;
        }
        KerRec k{};
        k.blk0 = (uint32_t)H->blk.size();
        k.n_blk = (uint32_t)o.blk.size();
        k.topo0 = (uint32_t)H->topo.size();
        k.max_n = o.max_n;
        k.tok0 = (uint32_t)tk;
        k.n_tok = (uint32_t)o.tok.size();
        const uint32_t tbase = (uint32_t)tk, fbase = (uint32_t)H->fpreds.size();
        for (auto &t : o.tok) {
            TokRec &r = H->tok[tk++];
            r.res = t.res;
            r.cls = t.flags;
            r.sig = (uint16_t)remap[t.sig];
            r.pred0 = pred0;
            r.lst_row = t.row;
            r.lst_len = t.len;
            r.pad_ = 0;
            pred0 += t.npred;
        }
        H->preds.insert(H->preds.end(), o.preds.begin(), o.preds.end());
        for (auto &b : o.blk) {
            BlkRec r{};
            r.mult = b.mult;
            r.tok0 = b.tok0 + tbase;
            r.n = b.n;
            r.fpred0 = b.fpred0 + fbase;
            r.n_fpred = (uint16_t)b.n_fpred;
            r.n_glob = b.n_glob;
            for (int q = 0; q < 5; q++) r.res_cnt[q] = b.res_cnt[q];
            r.is_exit = b.is_exit;
            H->blk.push_back(r);
        }
        H->fpreds.insert(H->fpreds.end(), o.fpreds.begin(), o.fpreds.end());
        H->topo.insert(H->topo.end(), o.topo.begin(), o.topo.end());
        H->ker.push_back(k);
        o = Packed();
    }
    TokRec &s = H->tok[nt_tok];
    std::memset(&s, 0, sizeof s);
    s.pred0 = pred0;
    outs.clear();
    outs.shrink_to_fit();
    if (timing) {
        auto t_end = now();
        std::fprintf(stderr, "gk_ptx_pack: %d threads, parse %.3f s, merge %.3f s\n", nt,
                     std::chrono::duration<double>(t_parsed - t_start).count(),
                     std::chrono::duration<double>(t_end - t_parsed).count());
    }
    return H;
}

int gk_ptx_error(const void *h, uint64_t *kernel, int64_t *line, char *msg, size_t cap) {
    const Handle *H = static_cast<const Handle *>(h);
    if (!H) return GK_PTX_PARSE_ERROR;
    if (kernel) *kernel = H->bad;
    if (line) *line = H->err.line;
    if (msg && cap) {
        size_t k = std::min(cap - 1, H->err.msg.size());
        std::memcpy(msg, H->err.msg.data(), k);
        msg[k] = 0;
    }
    return H->err.kind;
}

void gk_ptx_sizes_of(const void *h, gk_ptx_sizes *out) {
    const Handle *H = static_cast<const Handle *>(h);
    std::memset(out, 0, sizeof *out);
    if (!H) return;
    out->n_tok = H->tok.empty() ? 0 : H->tok.size() - 1;
    out->n_preds = H->preds.size();
    out->n_blk = H->blk.size();
    out->n_fpreds = H->fpreds.size();
    out->n_topo = H->topo.size();
    out->n_ker = H->ker.size();
    out->n_sig = H->sigs.size();
    out->n_warn = H->warnings.size();
}

int gk_ptx_copy(const void *h, void *tok, uint16_t *preds, void *blk, uint32_t *fpreds,
                uint32_t *topo, void *ker) {
    const Handle *H = static_cast<const Handle *>(h);
    if (!H || H->err.kind != GK_PTX_OK) return -1;
    if (tok) std::memcpy(tok, H->tok.data(), H->tok.size() * sizeof(TokRec));
    if (preds && !H->preds.empty()) std::memcpy(preds, H->preds.data(), H->preds.size() * 2);
    if (blk && !H->blk.empty()) std::memcpy(blk, H->blk.data(), H->blk.size() * sizeof(BlkRec));
    if (fpreds && !H->fpreds.empty()) std::memcpy(fpreds, H->fpreds.data(), H->fpreds.size() * 4);
    if (topo && !H->topo.empty()) std::memcpy(topo, H->topo.data(), H->topo.size() * 4);
    if (ker && !H->ker.empty()) std::memcpy(ker, H->ker.data(), H->ker.size() * sizeof(KerRec));
    return 0;
}

int gk_ptx_sig(const void *h, uint64_t i, int *cls, char *root_buf, size_t cap, int *kind) {
    const Handle *H = static_cast<const Handle *>(h);
    if (!H || i >= H->sigs.size()) return -1;
    const std::string &k = H->sigs[i];
    *cls = k[0] - '0';
    *kind = k[1] == '-' ? 0 : k[1];
    const size_t len = k.size() - 2;
    if (root_buf && cap) {
        size_t m = std::min(cap - 1, len);
        std::memcpy(root_buf, k.data() + 2, m);
        root_buf[m] = 0;
    }
    return (int)len;
}

int gk_ptx_warning(const void *h, uint64_t w, uint64_t *kernel, char *buf, size_t cap) {
    const Handle *H = static_cast<const Handle *>(h);
    if (!H || w >= H->warnings.size()) return -1;
    *kernel = H->warnings[w].first;
    const std::string &s = H->warnings[w].second;
    if (buf && cap) {
        size_t m = std::min(cap - 1, s.size());
        std::memcpy(buf, s.data(), m);
        buf[m] = 0;
    }
    return (int)s.size();
}

void gk_ptx_free(void *h) { delete static_cast<Handle *>(h); }

}  // extern "C"
