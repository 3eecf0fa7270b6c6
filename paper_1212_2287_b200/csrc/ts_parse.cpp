// ts_parse.cpp -- native parser for the reference's text model format
// (grammar: SPEC.md "External Interfaces"; behaviour: ref model.py:390-602).
//
//   ensemble <num_features:int> <num_trees:int>
//   tree <weight:float>
//   node <id:int> <fid:int> <theta:float> <left:int> <right:int>
//   leaf <id:int> <value:float>
//   end
//
// Produces the flat model the packer consumes (nodes in file-id order, ids
// dense per tree) without building any per-node objects, so 20,000-tree
// models (BASELINE config 4b, ~41M lines) load in seconds.  Error classes,
// messages and line/column positions follow the reference parser: syntax
// errors (TS_ERR_SYNTAX, 1-based line/col) and semantic errors
// (TS_ERR_INVALID, message names tree and id).
#include <errno.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <type_traits>
#include <vector>

#include "ts_internal.h"

namespace ts {
namespace {

// Node ids index a dense per-tree table; larger ids are refused (the
// reference would reject them later as non-dense unless 16M nodes follow).
constexpr long long kMaxNodeId = 1ll << 24;

struct Tok {
    const char *p;
    int len;
    int col;  // 1-based
};

struct Parser {
    const char *s, *end;
    int line = 0;
    int err_line = 0, err_col = 0;
    std::vector<Tok> toks;

    // Next non-blank, non-comment line; false at EOF.
    bool next_line() {
        while (s < end) {
            const char *ls = s;
            const char *le = (const char *)memchr(s, '\n', end - s);
            if (!le) le = end;
            s = le < end ? le + 1 : end;
            line++;
            const char *q = le;
            if (q > ls && q[-1] == '\r') q--;  // splitlines() treats \r\n as one break
            toks.clear();
            const char *c = ls;
            while (c < q) {
                while (c < q && (*c == ' ' || *c == '\t' || *c == '\f' || *c == '\v')) c++;
                if (c >= q) break;
                const char *t0 = c;
                while (c < q && !(*c == ' ' || *c == '\t' || *c == '\f' || *c == '\v')) c++;
                toks.push_back(Tok{t0, (int)(c - t0), (int)(t0 - ls) + 1});
            }
            if (toks.empty() || toks[0].p[0] == '#') continue;
            return true;
        }
        return false;
    }

    int syntax(const std::string &msg, int ln, int col) {
        err_line = ln;
        err_col = col;
        char buf[64];
        snprintf(buf, sizeof buf, "line %d, col %d: ", ln, col);
        return fail(TS_ERR_SYNTAX, buf + msg);
    }
};

bool word(const Tok &t, const char *w) {
    return (int)strlen(w) == t.len && memcmp(t.p, w, t.len) == 0;
}

std::string repr(const Tok &t) { return "'" + std::string(t.p, t.len) + "'"; }

// Python int()/float() accept '_' between digits (PEP 515); drop those and
// reject any other underscore.
bool strip_underscores(std::string *s) {
    if (s->find('_') == std::string::npos) return true;
    std::string o;
    for (size_t i = 0; i < s->size(); i++) {
        char c = (*s)[i];
        if (c == '_') {
            if (i == 0 || i + 1 >= s->size()) return false;
            char a = (*s)[i - 1], b = (*s)[i + 1];
            if (!(a >= '0' && a <= '9' && b >= '0' && b <= '9')) return false;
            continue;
        }
        o.push_back(c);
    }
    *s = o;
    return true;
}

bool parse_int(const Tok &t, long long *v) {
    std::string s(t.p, t.len);
    if (!strip_underscores(&s)) return false;
    if (s.empty()) return false;
    size_t i = (s[0] == '+' || s[0] == '-') ? 1 : 0;
    if (i >= s.size()) return false;
    for (size_t k = i; k < s.size(); k++)
        if (s[k] < '0' || s[k] > '9') return false;
    errno = 0;
    *v = strtoll(s.c_str(), nullptr, 10);
    return errno == 0;
}

bool parse_float(const Tok &t, double *v) {
    std::string s(t.p, t.len);
    if (s.empty() || !strip_underscores(&s)) return false;
    // strtod also takes hex floats and "nan(...)", which Python's float()
    // rejects; accept decimal, inf/infinity and nan forms only.
    if (s.find_first_of("xX(") != std::string::npos) return false;
    char *e = nullptr;
    *v = strtod(s.c_str(), &e);
    return e && *e == '\0';
}

}  // namespace
}  // namespace ts

using namespace ts;

extern "C" int ts_parse_model(const char *text, int64_t len, ts_flat_model **out) {
    if (!out) return fail(TS_ERR_INVALID, "out is NULL");
    *out = nullptr;
    Parser P;
    P.s = text;
    P.end = text + (len < 0 ? 0 : len);
    auto *m = new ts_flat_model();
    memset(m, 0, sizeof *m);
    auto bail = [&](int rc) {
        m->err_line = P.err_line;
        m->err_col = P.err_col;
        *out = m;  // carries the error position; free with ts_flat_free
        return rc;
    };
    if (!P.next_line()) return bail(P.syntax("empty document, expected 'ensemble' header", 1, 1));
    if (!word(P.toks[0], "ensemble") || P.toks.size() != 3)
        return bail(P.syntax("expected header 'ensemble <num_features> <num_trees>'", P.line,
                             P.toks[0].col));
    long long nf, nt;
    if (!parse_int(P.toks[1], &nf))
        return bail(P.syntax("expected integer num_features, got " + repr(P.toks[1]), P.line,
                             P.toks[1].col));
    if (!parse_int(P.toks[2], &nt))
        return bail(P.syntax("expected integer num_trees, got " + repr(P.toks[2]), P.line,
                             P.toks[2].col));
    if (nf < 1) return bail(fail(TS_ERR_INVALID, "num_features must be positive, got " +
                                                     std::to_string(nf)));
    if (nt < 1) return bail(fail(TS_ERR_INVALID, "num_trees must be positive, got " +
                                                     std::to_string(nt)));
    if (nf > INT32_MAX || nt > INT32_MAX) return bail(fail(TS_ERR_UNSUPPORTED, "model too large"));

    std::vector<int64_t> off(1, 0);
    std::vector<double> weights;
    std::vector<int32_t> fid, left, right;
    std::vector<float> value;
    std::vector<int32_t> tfid, tl, tr;
    std::vector<float> tv;
    std::vector<uint8_t> defined;
    int last = P.line;
    for (long long t = 0; t < nt; t++) {
        if (!P.next_line())
            return bail(P.syntax("expected " + std::to_string(nt) + " tree blocks, found " +
                                     std::to_string(t), last, 1));
        last = P.line;
        if (!word(P.toks[0], "tree") || P.toks.size() != 2)
            return bail(P.syntax("expected 'tree <weight>'", P.line, P.toks[0].col));
        double w;
        if (!parse_float(P.toks[1], &w))
            return bail(P.syntax("expected float weight, got " + repr(P.toks[1]), P.line,
                                 P.toks[1].col));
        tfid.clear();
        tl.clear();
        tr.clear();
        tv.clear();
        defined.clear();
        auto ensure = [&](long long id) {
            if ((size_t)id >= defined.size()) {
                size_t n = (size_t)id + 1;
                tfid.resize(n, 0);
                tl.resize(n, -1);
                tr.resize(n, -1);
                tv.resize(n, 0.f);
                defined.resize(n, 0);
            }
        };
        const std::string tmsg = "tree " + std::to_string(t);
        while (true) {
            if (!P.next_line()) return bail(P.syntax(tmsg + ": missing 'end'", last, 1));
            last = P.line;
            const Tok &w0 = P.toks[0];
            if (word(w0, "end")) {
                if (P.toks.size() != 1)
                    return bail(P.syntax("unexpected tokens after 'end'", P.line, P.toks[1].col));
                break;
            }
            long long nid;
            if (word(w0, "node")) {
                if (P.toks.size() != 6)
                    return bail(P.syntax("expected 'node <id> <fid> <theta> <left> <right>'",
                                         P.line, w0.col));
                long long f, lc, rc;
                double th;
                if (!parse_int(P.toks[1], &nid))
                    return bail(P.syntax("expected integer node id, got " + repr(P.toks[1]),
                                         P.line, P.toks[1].col));
                if (!parse_int(P.toks[2], &f))
                    return bail(P.syntax("expected integer feature id, got " + repr(P.toks[2]),
                                         P.line, P.toks[2].col));
                if (!parse_float(P.toks[3], &th))
                    return bail(P.syntax("expected float threshold, got " + repr(P.toks[3]),
                                         P.line, P.toks[3].col));
                if (!parse_int(P.toks[4], &lc))
                    return bail(P.syntax("expected integer left child id, got " +
                                             repr(P.toks[4]), P.line, P.toks[4].col));
                if (!parse_int(P.toks[5], &rc))
                    return bail(P.syntax("expected integer right child id, got " +
                                             repr(P.toks[5]), P.line, P.toks[5].col));
                if (f < 0)
                    return bail(P.syntax("feature id must be non-negative", P.line,
                                         P.toks[2].col));
                if (f >= nf)
                    return bail(fail(TS_ERR_INVALID,
                                     tmsg + ", line " + std::to_string(P.line) + ": feature id " +
                                         std::to_string(f) + " out of range (num_features=" +
                                         std::to_string(nf) + ")"));
                if (!isfinite((float)th))
                    return bail(fail(TS_ERR_INVALID, tmsg + ", line " + std::to_string(P.line) +
                                                         ": threshold must be finite"));
                if (nid < 0)
                    return bail(P.syntax("node id must be non-negative", P.line, P.toks[1].col));
                if (nid >= kMaxNodeId || lc > INT32_MAX || rc > INT32_MAX || lc < INT32_MIN ||
                    rc < INT32_MIN)
                    return bail(fail(TS_ERR_UNSUPPORTED, tmsg + ": node id too large"));
                ensure(nid);
                if (defined[nid])
                    return bail(fail(TS_ERR_INVALID,
                                     tmsg + ": duplicate node id " + std::to_string(nid)));
                defined[nid] = 1;
                tfid[nid] = (int32_t)f;
                tv[nid] = (float)th;
                tl[nid] = (int32_t)lc;
                tr[nid] = (int32_t)rc;
            } else if (word(w0, "leaf")) {
                if (P.toks.size() != 3)
                    return bail(P.syntax("expected 'leaf <id> <value>'", P.line, w0.col));
                double v;
                if (!parse_int(P.toks[1], &nid))
                    return bail(P.syntax("expected integer node id, got " + repr(P.toks[1]),
                                         P.line, P.toks[1].col));
                if (!parse_float(P.toks[2], &v))
                    return bail(P.syntax("expected float leaf value, got " + repr(P.toks[2]),
                                         P.line, P.toks[2].col));
                if (!isfinite((float)v))
                    return bail(fail(TS_ERR_INVALID, tmsg + ", line " + std::to_string(P.line) +
                                                         ": leaf value must be finite"));
                if (nid < 0)
                    return bail(P.syntax("node id must be non-negative", P.line, P.toks[1].col));
                if (nid >= kMaxNodeId)
                    return bail(fail(TS_ERR_UNSUPPORTED, tmsg + ": node id too large"));
                ensure(nid);
                if (defined[nid])
                    return bail(fail(TS_ERR_INVALID,
                                     tmsg + ": duplicate node id " + std::to_string(nid)));
                defined[nid] = 1;
                tfid[nid] = -1;
                tv[nid] = (float)v;
                tl[nid] = tr[nid] = -1;
            } else {
                return bail(P.syntax("expected 'node', 'leaf' or 'end', got " + repr(w0), P.line,
                                     w0.col));
            }
        }
        // graph checks (ref model.py:538-602)
        const size_t n = defined.size();
        size_t count = 0;
        for (uint8_t d : defined) count += d;
        if (count == 0) return bail(fail(TS_ERR_INVALID, tmsg + ": empty tree block"));
        if (count != n) {
            size_t missing = 0;
            while (defined[missing]) missing++;
            return bail(fail(TS_ERR_INVALID, tmsg + ": node ids must be dense in [0, " +
                                                 std::to_string(count) + "), id " +
                                                 std::to_string(missing) + " is missing"));
        }
        std::vector<int32_t> refs(n, 0);
        for (size_t i = 0; i < n; i++) {
            if (tfid[i] < 0) continue;
            for (int32_t c : {tl[i], tr[i]}) {
                if (c < 0 || (size_t)c >= n)
                    return bail(fail(TS_ERR_INVALID, tmsg + ": node " + std::to_string(i) +
                                                         " references dangling child id " +
                                                         std::to_string(c)));
                refs[c]++;
            }
        }
        if (refs[0])
            return bail(fail(TS_ERR_INVALID, tmsg + ": root (id 0) must not appear as a child"));
        for (size_t i = 1; i < n; i++)
            if (refs[i] > 1)
                return bail(fail(TS_ERR_INVALID, tmsg + ": node " + std::to_string(i) +
                                                     " has multiple parents"));
        std::vector<uint8_t> seen(n, 0);
        std::vector<int32_t> q(1, 0);
        seen[0] = 1;
        for (size_t h = 0; h < q.size(); h++) {
            int32_t i = q[h];
            if (tfid[i] < 0) continue;
            for (int32_t c : {tl[i], tr[i]})
                if (!seen[c]) {
                    seen[c] = 1;
                    q.push_back(c);
                }
        }
        if (q.size() != n) {
            size_t orphan = 0;
            while (seen[orphan]) orphan++;
            return bail(fail(TS_ERR_INVALID,
                             tmsg + ": node " + std::to_string(orphan) +
                                 " is unreachable from the root (disconnected or cyclic block)"));
        }
        weights.push_back(w);
        fid.insert(fid.end(), tfid.begin(), tfid.end());
        value.insert(value.end(), tv.begin(), tv.end());
        left.insert(left.end(), tl.begin(), tl.end());
        right.insert(right.end(), tr.begin(), tr.end());
        off.push_back((int64_t)fid.size());
    }
    if (P.next_line())
        return bail(P.syntax("unexpected content after final tree", P.line, P.toks[0].col));
    for (double w : weights)  // Ensemble() checks weights after parsing (ref model.py:209-211)
        if (!isfinite(w)) {
            char buf[96];
            snprintf(buf, sizeof buf, "tree weight must be finite, got %g", w);
            return bail(fail(TS_ERR_INVALID, buf));
        }

    m->num_features = (int32_t)nf;
    m->num_trees = (int32_t)nt;
    m->num_nodes = (int64_t)fid.size();
    auto dup = [](const auto &v) {
        using T = typename std::decay_t<decltype(v)>::value_type;
        T *p = (T *)malloc(std::max<size_t>(1, v.size()) * sizeof(T));
        if (p && !v.empty()) memcpy(p, v.data(), v.size() * sizeof(T));
        return p;
    };
    m->tree_node_offset = dup(off);
    m->tree_weight = dup(weights);
    m->node_fid = dup(fid);
    m->node_value = dup(value);
    m->node_left = dup(left);
    m->node_right = dup(right);
    *out = m;
    if (!m->tree_node_offset || !m->tree_weight || !m->node_fid || !m->node_value ||
        !m->node_left || !m->node_right)
        return fail(TS_ERR_NOMEM, "out of host memory");
    return TS_OK;
}

extern "C" void ts_flat_free(ts_flat_model *m) {
    if (!m) return;
    free(m->tree_node_offset);
    free(m->tree_weight);
    free(m->node_fid);
    free(m->node_value);
    free(m->node_left);
    free(m->node_right);
    delete m;
}
