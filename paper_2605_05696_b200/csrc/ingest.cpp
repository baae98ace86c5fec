// Trace ingest: JSONL request records -> flattened token CSR in caller memory.
//
// Replaces model.parse_trace / _parse_request / flatten (reference
// model.py:116-170 and :80-98) on the host side of the serve path, so a trace
// reaches K0/K1 as u32 token buffers (pinned host memory, one H2D) without a
// Python object per token. Two passes over the same text:
//   irm_trace_scan  validates every line exactly as the reference does (same
//                   error precedence, line number and field) and counts sizes;
//   irm_trace_fill  writes tokens, per-request / per-segment offsets, kinds,
//                   turns and the session / shared_id strings.
// Lines follow Python's text-file iteration: universal newlines (\n, \r\n, \r)
// for files, '\n' only for in-memory streams (io.StringIO); whitespace-only lines
// are skipped (model.py:162-165). The JSON grammar is Python's json
// module's: NaN / Infinity literals parse (as non-integers), duplicate keys keep
// the last value, control characters inside strings are invalid. Lines are
// parsed in parallel on host threads (IRM_INGEST_THREADS, default all cores);
// the reported error is the first one in line order, as the sequential reference.
#include <algorithm>
#include <atomic>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/irminsul_b200.h"

namespace irm {
void set_error(const char *fmt, ...);
}

namespace {

enum JType : uint8_t { J_NULL, J_TRUE, J_FALSE, J_INT, J_FLOAT, J_STR, J_ARR, J_OBJ };

struct JNode {
    JType type;
    bool neg = false;       // J_INT: negative
    bool big = false;       // J_INT: magnitude >= 2^64
    bool packed = false;    // J_ARR of u32 integers only: values in Parser::ints[first, first + count)
    uint64_t mag = 0;       // J_INT magnitude
    uint32_t str = 0, len = 0;  // J_STR: decoded bytes in Parser::strbuf
    uint32_t first = 0, count = 0;  // J_ARR / J_OBJ: children in Parser::kids (objects: key, value pairs)
    const char *src = nullptr;
    uint32_t src_len = 0;   // raw text of the value (for repr in messages)
};

struct Parser {
    const char *p, *end;
    std::vector<JNode> nodes;
    std::vector<uint32_t> kids;
    std::string strbuf;
    std::vector<uint32_t> stk;
    std::vector<uint32_t> ints;  // packed token arrays
    const char *err = nullptr;

    void ws() {
        while (p < end && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) ++p;
    }
    bool lit(const char *s) {
        const size_t n = strlen(s);
        if ((size_t)(end - p) >= n && memcmp(p, s, n) == 0) {
            p += n;
            return true;
        }
        return false;
    }
    static int hexv(char c) {
        if (c >= '0' && c <= '9') return c - '0';
        if (c >= 'a' && c <= 'f') return c - 'a' + 10;
        if (c >= 'A' && c <= 'F') return c - 'A' + 10;
        return -1;
    }
    void put_utf8(uint32_t cp) {
        if (cp < 0x80) {
            strbuf.push_back((char)cp);
        } else if (cp < 0x800) {
            strbuf.push_back((char)(0xC0 | (cp >> 6)));
            strbuf.push_back((char)(0x80 | (cp & 0x3F)));
        } else if (cp < 0x10000) {  // lone surrogates pass through (Python's 'surrogatepass')
            strbuf.push_back((char)(0xE0 | (cp >> 12)));
            strbuf.push_back((char)(0x80 | ((cp >> 6) & 0x3F)));
            strbuf.push_back((char)(0x80 | (cp & 0x3F)));
        } else {
            strbuf.push_back((char)(0xF0 | (cp >> 18)));
            strbuf.push_back((char)(0x80 | ((cp >> 12) & 0x3F)));
            strbuf.push_back((char)(0x80 | ((cp >> 6) & 0x3F)));
            strbuf.push_back((char)(0x80 | (cp & 0x3F)));
        }
    }
    bool string(JNode &n) {  // p at the opening quote
        ++p;
        n.type = J_STR;
        n.str = (uint32_t)strbuf.size();
        while (true) {
            if (p >= end) return fail("unterminated string");
            const unsigned char c = (unsigned char)*p;
            if (c == '"') {
                ++p;
                break;
            }
            if (c < 0x20) return fail("invalid control character in string");
            if (c != '\\') {
                strbuf.push_back((char)c);
                ++p;
                continue;
            }
            if (++p >= end) return fail("unterminated escape");
            const char e = *p++;
            switch (e) {
                case '"': strbuf.push_back('"'); break;
                case '\\': strbuf.push_back('\\'); break;
                case '/': strbuf.push_back('/'); break;
                case 'b': strbuf.push_back('\b'); break;
                case 'f': strbuf.push_back('\f'); break;
                case 'n': strbuf.push_back('\n'); break;
                case 'r': strbuf.push_back('\r'); break;
                case 't': strbuf.push_back('\t'); break;
                case 'u': {
                    auto hex4 = [&](uint32_t &v) {
                        if (end - p < 4) return false;
                        v = 0;
                        for (int i = 0; i < 4; ++i) {
                            const int h = hexv(p[i]);
                            if (h < 0) return false;
                            v = v * 16 + (uint32_t)h;
                        }
                        p += 4;
                        return true;
                    };
                    uint32_t cp;
                    if (!hex4(cp)) return fail("invalid \\uXXXX escape");
                    if (cp >= 0xD800 && cp < 0xDC00 && end - p >= 6 && p[0] == '\\' && p[1] == 'u') {
                        const char *save = p;
                        p += 2;
                        uint32_t lo;
                        if (hex4(lo) && lo >= 0xDC00 && lo < 0xE000) cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                        else p = save;
                    }
                    put_utf8(cp);
                    break;
                }
                default: return fail("invalid escape");
            }
        }
        n.len = (uint32_t)(strbuf.size() - n.str);
        return true;
    }
    bool number(JNode &n) {
        const char *s = p;
        if (p < end && *p == '-') {
            ++p;
            if (lit("Infinity")) {
                n.type = J_FLOAT;
                return true;
            }
        }
        if (p >= end || !(*p >= '0' && *p <= '9')) return fail("invalid number");
        uint64_t mag = 0;
        bool big = false;
        if (*p == '0') {
            ++p;
        } else {
            while (p < end && *p >= '0' && *p <= '9') {
                uint64_t m10;
                if (__builtin_mul_overflow(mag, (uint64_t)10, &m10) ||
                    __builtin_add_overflow(m10, (uint64_t)(*p - '0'), &mag))
                    big = true;
                ++p;
            }
        }
        bool flt = false;
        if (p < end && *p == '.') {
            ++p;
            if (p >= end || !(*p >= '0' && *p <= '9')) return fail("invalid number");
            while (p < end && *p >= '0' && *p <= '9') ++p;
            flt = true;
        }
        if (p < end && (*p == 'e' || *p == 'E')) {
            ++p;
            if (p < end && (*p == '+' || *p == '-')) ++p;
            if (p >= end || !(*p >= '0' && *p <= '9')) return fail("invalid number");
            while (p < end && *p >= '0' && *p <= '9') ++p;
            flt = true;
        }
        n.type = flt ? J_FLOAT : J_INT;
        n.neg = *s == '-';
        n.mag = mag;
        n.big = big;
        return true;
    }
    // '[' u32 (',' u32)* ']' with no signs, fractions, exponents or leading zeros;
    // anything else rewinds and takes the general path (which reports errors)
    bool packed_array(JNode &n) {
        const char *save = p;
        const size_t i0 = ints.size();
        ++p;
        ws();
        if (p < end && *p == ']') {
            ++p;
        } else {
            while (true) {
                ws();
                if (p >= end || *p < '0' || *p > '9') goto slow;
                uint64_t v = (uint64_t)(*p++ - '0');
                if (v == 0 && p < end && *p >= '0' && *p <= '9') goto slow;
                int nd = 1;
                while (p < end && *p >= '0' && *p <= '9' && nd < 11) {
                    v = v * 10 + (uint64_t)(*p++ - '0');
                    ++nd;
                }
                if (v > 0xFFFFFFFFull || (p < end && (*p == '.' || *p == 'e' || *p == 'E' || (*p >= '0' && *p <= '9'))))
                    goto slow;
                ints.push_back((uint32_t)v);
                ws();
                if (p < end && *p == ',') {
                    ++p;
                    continue;
                }
                if (p < end && *p == ']') {
                    ++p;
                    break;
                }
                goto slow;
            }
        }
        n.type = J_ARR;
        n.packed = true;
        n.first = (uint32_t)i0;
        n.count = (uint32_t)(ints.size() - i0);
        return true;
    slow:
        p = save;
        ints.resize(i0);
        return false;
    }
    bool fail(const char *m) {
        if (!err) err = m;
        return false;
    }
    // iterative value parser: children are appended after their parent is complete, so
    // each container records its children in kids[first, first + count)
    bool value(uint32_t &out, int depth = 0) {
        if (depth > 1000) return fail("nesting too deep");
        ws();
        if (p >= end) return fail("expecting value");
        JNode n;
        n.src = p;
        const char c = *p;
        if (c == '[' && packed_array(n)) {
            // fast path: an array of plain u32 integers (every token list of a valid trace)
        } else if (c == '{' || c == '[') {
            const bool obj = c == '{';
            ++p;
            const size_t base = stk.size();  // children collect on a shared stack
            ws();
            if (p < end && *p == (obj ? '}' : ']')) {
                ++p;
            } else {
                while (true) {
                    if (obj) {
                        ws();
                        if (p >= end || *p != '"') return fail("expecting property name in double quotes");
                        JNode k;
                        k.src = p;
                        if (!string(k)) return false;
                        k.src_len = (uint32_t)(p - k.src);
                        nodes.push_back(k);
                        stk.push_back((uint32_t)nodes.size() - 1);
                        ws();
                        if (p >= end || *p != ':') return fail("expecting ':' delimiter");
                        ++p;
                    }
                    uint32_t v;
                    if (!value(v, depth + 1)) return false;
                    stk.push_back(v);
                    ws();
                    if (p < end && *p == ',') {
                        ++p;
                        continue;
                    }
                    if (p < end && *p == (obj ? '}' : ']')) {
                        ++p;
                        break;
                    }
                    return fail("expecting ',' delimiter");
                }
            }
            n.type = obj ? J_OBJ : J_ARR;
            n.first = (uint32_t)kids.size();
            const size_t cnt = stk.size() - base;
            n.count = (uint32_t)(obj ? cnt / 2 : cnt);
            kids.insert(kids.end(), stk.begin() + (ptrdiff_t)base, stk.end());
            stk.resize(base);
        } else if (c == '"') {
            if (!string(n)) return false;
        } else if (c == '-' || (c >= '0' && c <= '9')) {
            if (!number(n)) return false;
        } else if (c == 'n' && lit("null")) {
            n.type = J_NULL;
        } else if (c == 't' && lit("true")) {
            n.type = J_TRUE;
        } else if (c == 'f' && lit("false")) {
            n.type = J_FALSE;
        } else if ((c == 'N' && lit("NaN")) || (c == 'I' && lit("Infinity"))) {
            n.type = J_FLOAT;
        } else {
            return fail("expecting value");
        }
        n.src_len = (uint32_t)(p - n.src);
        nodes.push_back(n);
        out = (uint32_t)nodes.size() - 1;
        return true;
    }
    bool parse_line(const char *b, const char *e, uint32_t &root) {
        p = b;
        end = e;
        nodes.clear();
        kids.clear();
        strbuf.clear();
        stk.clear();
        ints.clear();
        const size_t guess = (size_t)(e - b) / 4 + 16;  // ~one value per 4+ bytes of JSON
        if (nodes.capacity() < guess) nodes.reserve(guess);
        if (kids.capacity() < guess) kids.reserve(guess);
        if (stk.capacity() < guess) stk.reserve(guess);
        if (ints.capacity() < guess) ints.reserve(guess);
        err = nullptr;
        if (!value(root)) return false;
        ws();
        if (p != end) return fail("extra data");
        return true;
    }
    std::string sv(const JNode &n) const { return std::string(strbuf.data() + n.str, n.len); }
    // last value of key (duplicate keys: the last one wins, as in Python)
    int find(const JNode &obj, const char *key) const {
        int found = -1;
        const size_t kl = strlen(key);
        for (uint32_t i = 0; i < obj.count; ++i) {
            const JNode &k = nodes[kids[obj.first + 2 * i]];
            if (k.len == kl && memcmp(strbuf.data() + k.str, key, kl) == 0) found = (int)kids[obj.first + 2 * i + 1];
        }
        return found;
    }
};

const char *const KINDS[] = {"system", "header", "history", "tool", "doc", "marker", "body", "other"};
constexpr int N_KINDS = 8, MARKER_KIND = 5, MARKER_LEN = 64;

struct Err {
    int64_t line = 0;
    std::string field, msg;
};

std::string repr_raw(const JNode &n) { return std::string(n.src, n.src_len); }

// Python's repr of a float (the shortest round-trip digits, scientific when the decimal
// point position is <= -4 or > 16, "inf" / "nan"), for messages that quote a JSON number
std::string py_float_repr(const JNode &n) {
    const std::string raw = repr_raw(n);
    const double v = strtod(raw.c_str(), nullptr);
    if (std::isnan(v)) return "nan";
    if (std::isinf(v)) return v < 0 ? "-inf" : "inf";
    char buf[64];
    const auto r = std::to_chars(buf, buf + sizeof buf, std::fabs(v), std::chars_format::scientific);
    const std::string sci(buf, r.ptr);
    const size_t epos = sci.find('e');
    std::string digits = sci.substr(0, epos);
    digits.erase(std::remove(digits.begin(), digits.end(), '.'), digits.end());
    const int exp10 = atoi(sci.c_str() + epos + 1);
    const int decpt = exp10 + 1, nd = (int)digits.size();
    std::string out = std::signbit(v) ? "-" : "";
    if (decpt > -4 && decpt <= 16) {
        if (decpt <= 0) out += "0." + std::string(-decpt, '0') + digits;
        else if (decpt >= nd) out += digits + std::string(decpt - nd, '0') + ".0";
        else out += digits.substr(0, decpt) + "." + digits.substr(decpt);
    } else {
        out += digits.substr(0, 1);
        if (nd > 1) out += "." + digits.substr(1);
        char e[16];
        snprintf(e, sizeof e, "e%c%02d", exp10 < 0 ? '-' : '+', std::abs(exp10));
        out += e;
    }
    return out;
}

// Python repr of a JSON value as the reference's f-strings print it (strings quoted)
std::string py_repr(const Parser &P, const JNode &n) {
    switch (n.type) {
        case J_NULL: return "None";
        case J_TRUE: return "True";
        case J_FALSE: return "False";
        case J_FLOAT: return py_float_repr(n);
        case J_STR: {
            const std::string s = P.sv(n);
            const bool dq = s.find('\'') != std::string::npos && s.find('"') == std::string::npos;
            return (dq ? "\"" : "'") + s + (dq ? "\"" : "'");
        }
        case J_ARR: {
            std::string o = "[";
            for (uint32_t i = 0; i < n.count; ++i) {
                if (i) o += ", ";
                o += n.packed ? std::to_string(P.ints[n.first + i]) : py_repr(P, P.nodes[P.kids[n.first + i]]);
            }
            return o + "]";
        }
        case J_OBJ: {
            std::string o = "{";
            for (uint32_t i = 0; i < n.count; ++i) {  // (duplicate keys: Python keeps the last; rare here)
                if (i) o += ", ";
                o += py_repr(P, P.nodes[P.kids[n.first + 2 * i]]) + ": " + py_repr(P, P.nodes[P.kids[n.first + 2 * i + 1]]);
            }
            return o + "}";
        }
        default: return repr_raw(n);  // integers: their digits
    }
}

struct Sizes {
    int64_t n_req = 0, n_tok = 0, n_seg = 0, n_str = 0;
};

struct Out {
    uint32_t *tok;
    int64_t *req_tok_off, *req_seg_off, *req_turn, *req_sess_off, *seg_tok_off, *seg_shared_off;
    uint8_t *seg_kind;
    char *strings;
};

// validate one parsed record (model.py:116-156); on success optionally write it
bool record(const Parser &P, uint32_t root, int64_t line, Err &e, Sizes &sz, const Out *o) {
    auto bad = [&](const char *f, const std::string &m) {
        e.line = line;
        e.field = f;
        e.msg = m;
        return false;
    };
    const JNode &obj = P.nodes[root];
    if (obj.type != J_OBJ) return bad("<line>", "expected a JSON object");
    auto extra_of = [&](const JNode &o_, std::initializer_list<const char *> allowed, std::string &first) {
        bool any = false;
        for (uint32_t i = 0; i < o_.count; ++i) {
            const std::string k = P.sv(P.nodes[P.kids[o_.first + 2 * i]]);
            bool ok = false;
            for (const char *a : allowed) ok |= k == a;
            if (!ok && (!any || k < first)) {
                first = k;
                any = true;
            }
        }
        return any;
    };
    std::string ex;
    if (extra_of(obj, {"session_id", "turn", "segments"}, ex)) {
        e.line = line;
        e.field = ex;
        e.msg = "unknown field";
        return false;
    }
    const int s_i = P.find(obj, "session_id"), t_i = P.find(obj, "turn"), g_i = P.find(obj, "segments");
    if (s_i < 0) return bad("session_id", "missing field");
    if (t_i < 0) return bad("turn", "missing field");
    if (g_i < 0) return bad("segments", "missing field");
    const JNode &sid = P.nodes[s_i], &turn = P.nodes[t_i], &segs = P.nodes[g_i];
    if (sid.type != J_STR) return bad("session_id", "expected a string");
    if (turn.type != J_INT || (turn.neg && (turn.mag != 0 || turn.big)))
        return bad("turn", "expected a non-negative integer");
    if (turn.big || turn.mag > (uint64_t)INT64_MAX) return bad("turn", "turn beyond int64 (unsupported)");
    if (segs.type != J_ARR) return bad("segments", "expected a list");
    const int64_t tok0 = sz.n_tok, seg0 = sz.n_seg, str0 = sz.n_str;
    for (uint32_t si = 0; si < segs.count; ++si) {
        const JNode &seg = P.nodes[P.kids[segs.first + si]];
        if (seg.type != J_OBJ) return bad("segments", "segment must be an object");
        if (extra_of(seg, {"kind", "tokens", "shared_id"}, ex)) {
            e.line = line;
            e.field = ex;
            e.msg = "unknown field";
            return false;
        }
        const int k_i = P.find(seg, "kind"), x_i = P.find(seg, "tokens"), h_i = P.find(seg, "shared_id");
        int kind = -1;
        if (k_i >= 0 && P.nodes[k_i].type == J_STR) {
            const std::string k = P.sv(P.nodes[k_i]);
            for (int q = 0; q < N_KINDS; ++q)
                if (k == KINDS[q]) kind = q;
        }
        if (kind < 0)
            return bad("kind", "unknown segment kind " + (k_i >= 0 ? py_repr(P, P.nodes[k_i]) : std::string("None")));
        if (x_i < 0 || P.nodes[x_i].type != J_ARR) return bad("tokens", "expected a list");
        const JNode &toks = P.nodes[x_i];
        for (uint32_t ti = 0; ti < toks.count && !toks.packed; ++ti) {
            const JNode &t = P.nodes[P.kids[toks.first + ti]];
            if (t.type != J_INT) return bad("tokens", "non-integer token " + py_repr(P, t));
            if ((t.neg && (t.mag != 0 || t.big)) || t.big || t.mag > 0xFFFFFFFFull)
                return bad("tokens", "token " + repr_raw(t) + " outside unsigned 32-bit range");
        }
        if (h_i >= 0 && P.nodes[h_i].type != J_NULL && P.nodes[h_i].type != J_STR)
            return bad("shared_id", "expected string or null");
        if (kind == MARKER_KIND && toks.count != MARKER_LEN)
            return bad("tokens", "marker segment must hold exactly 64 tokens");
        if (o) {
            o->seg_kind[sz.n_seg] = (uint8_t)kind;
            o->seg_tok_off[sz.n_seg] = sz.n_tok - tok0;
            if (toks.packed) {
                memcpy(o->tok + sz.n_tok, P.ints.data() + toks.first, (size_t)toks.count * 4);
            } else {
                for (uint32_t ti = 0; ti < toks.count; ++ti) o->tok[sz.n_tok + ti] = (uint32_t)P.nodes[P.kids[toks.first + ti]].mag;
            }
            if (h_i >= 0 && P.nodes[h_i].type == J_STR) {
                const JNode &h = P.nodes[h_i];
                o->seg_shared_off[2 * sz.n_seg] = sz.n_str;
                o->seg_shared_off[2 * sz.n_seg + 1] = h.len;
                memcpy(o->strings + sz.n_str, P.strbuf.data() + h.str, h.len);
            } else {
                o->seg_shared_off[2 * sz.n_seg] = -1;
                o->seg_shared_off[2 * sz.n_seg + 1] = 0;
            }
        }
        if (h_i >= 0 && P.nodes[h_i].type == J_STR) sz.n_str += P.nodes[h_i].len;
        sz.n_tok += toks.count;
        sz.n_seg += 1;
    }
    if (o) {
        o->req_tok_off[sz.n_req] = tok0;
        o->req_seg_off[sz.n_req] = seg0;
        o->req_turn[sz.n_req] = (int64_t)turn.mag;
        o->req_sess_off[2 * sz.n_req] = sz.n_str;
        o->req_sess_off[2 * sz.n_req + 1] = sid.len;
        memcpy(o->strings + sz.n_str, P.strbuf.data() + sid.str, sid.len);
    }
    (void)str0;
    sz.n_str += sid.len;
    sz.n_req += 1;
    return true;
}

bool blank(const char *b, const char *e) {  // str.strip() == "" for ASCII whitespace
    for (; b < e; ++b)
        if (!(*b == ' ' || *b == '\t' || *b == '\v' || *b == '\f' || (*b >= 0x1c && *b <= 0x1f))) return false;
    return true;
}

struct Line {
    const char *b, *e;
    int64_t no;  // 1-based line number in the text
};
struct LineSz {
    int64_t tok, seg, str;
};

// non-blank lines of the text (universal newlines or '\n' only)
void split(const char *text, int64_t len, bool universal, std::vector<Line> &lines) {
    lines.clear();
    const char *p = text, *end = text + len;
    int64_t no = 0;
    universal = universal && memchr(text, '\r', (size_t)len) != nullptr;  // no CR: same as '\n' only
    while (p < end) {
        const char *b = p;
        const void *q = memchr(p, '\n', (size_t)(end - p));
        p = q ? (const char *)q : end;
        if (universal) {  // a CR before the LF ends the line there (CRLF or a lone CR)
            const void *r = memchr(b, '\r', (size_t)(p - b));
            if (r) p = (const char *)r;
        }
        const char *le = p;
        if (p < end) {
            if (*p == '\r' && p + 1 < end && p[1] == '\n') p += 2;
            else ++p;
        }
        ++no;
        if (!blank(b, le)) lines.push_back({b, le, no});
    }
}

int n_threads(size_t n_lines) {
    static const int hw = [] {
        const char *env = getenv("IRM_INGEST_THREADS");
        const int v = env ? atoi(env) : (int)std::thread::hardware_concurrency();
        return v > 0 ? v : 1;
    }();
    const int want = (int)((n_lines + 3) / 4);
    return std::max(1, std::min(hw, std::min(want, 64)));
}

// parse lines [i0, i1) of `lines`: sizes (o == nullptr) or outputs at the offsets in `at`
bool parse_range(const std::vector<Line> &lines, size_t i0, size_t i1, std::vector<LineSz> &ls,
                 const std::vector<Sizes> *at, const Out *o, Err &e, std::atomic<int64_t> &stop_line) {
    Parser P;
    for (size_t i = i0; i < i1; ++i) {
        const Line &L = lines[i];
        if (L.no > stop_line.load(std::memory_order_relaxed)) return true;  // an earlier line already failed
        uint32_t root;
        Sizes sz = at ? (*at)[i] : Sizes{};
        const Sizes s0 = sz;
        bool ok = P.parse_line(L.b, L.e, root);
        if (!ok) {
            e.line = L.no;
            e.field = "<line>";
            e.msg = std::string("invalid JSON: ") + (P.err ? P.err : "parse error");
        } else {
            ok = record(P, root, L.no, e, sz, o);
        }
        if (!ok) {
            int64_t cur = stop_line.load();
            while (L.no < cur && !stop_line.compare_exchange_weak(cur, L.no)) {
            }
            return false;
        }
        if (!at) ls[i] = {sz.n_tok - s0.n_tok, sz.n_seg - s0.n_seg, sz.n_str - s0.n_str};
    }
    return true;
}

// run fn(t, i0, i1) over contiguous slices of n items on the worker threads
template <class F>
void parallel(size_t n, F fn) {
    const int T = n_threads(n);
    if (T == 1) {
        fn(0, (size_t)0, n);
        return;
    }
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t) {
        const size_t i0 = n * (size_t)t / (size_t)T, i1 = n * (size_t)(t + 1) / (size_t)T;
        th.emplace_back([=, &fn] { fn(t, i0, i1); });
    }
    for (auto &x : th) x.join();
}

// the first error in line order among the workers' errors
int first_error(std::vector<Err> &errs, std::vector<char> &failed, Err &e) {
    int64_t best = INT64_MAX;
    for (size_t t = 0; t < errs.size(); ++t)
        if (failed[t] && errs[t].line < best) {
            best = errs[t].line;
            e = errs[t];
        }
    return best == INT64_MAX ? IRM_OK : IRM_EINVAL;
}

// scan results of the last irm_trace_scan on this thread, reused by irm_trace_fill
struct ScanCache {
    const char *text = nullptr;
    int64_t len = -1;
    bool universal = false;
    std::vector<Line> lines;
    std::vector<LineSz> ls;
};
thread_local ScanCache cache;

int scan(const char *text, int64_t len, bool universal, Sizes &tot, Err &e) {
    ScanCache &c = cache;
    c.text = nullptr;
    split(text, len, universal, c.lines);
    c.ls.assign(c.lines.size(), LineSz{0, 0, 0});
    const int T = n_threads(c.lines.size());
    std::vector<Err> errs((size_t)T);
    std::vector<char> failed((size_t)T, 0);
    std::atomic<int64_t> stop{INT64_MAX};
    parallel(c.lines.size(), [&](int t, size_t i0, size_t i1) {
        failed[(size_t)t] = !parse_range(c.lines, i0, i1, c.ls, nullptr, nullptr, errs[(size_t)t], stop);
    });
    if (first_error(errs, failed, e) != IRM_OK) return IRM_EINVAL;
    tot = Sizes{};
    for (const LineSz &l : c.ls) {
        tot.n_req += 1;
        tot.n_tok += l.tok;
        tot.n_seg += l.seg;
        tot.n_str += l.str;
    }
    c.text = text;
    c.len = len;
    c.universal = universal;
    return IRM_OK;
}

int fill(const char *text, int64_t len, bool universal, Err &e, const Out &o) {
    ScanCache &c = cache;
    if (c.text != text || c.len != len || c.universal != universal) {
        Sizes tot;
        const int rc = scan(text, len, universal, tot, e);
        if (rc != IRM_OK) return rc;
    }
    const size_t n = c.lines.size();
    std::vector<Sizes> at(n);
    Sizes run_{};
    for (size_t i = 0; i < n; ++i) {
        at[i] = run_;
        run_.n_req += 1;
        run_.n_tok += c.ls[i].tok;
        run_.n_seg += c.ls[i].seg;
        run_.n_str += c.ls[i].str;
    }
    const int T = n_threads(n);
    std::vector<Err> errs((size_t)T);
    std::vector<char> failed((size_t)T, 0);
    std::atomic<int64_t> stop{INT64_MAX};
    std::vector<LineSz> unused;
    parallel(n, [&](int t, size_t i0, size_t i1) {
        failed[(size_t)t] = !parse_range(c.lines, i0, i1, unused, &at, &o, errs[(size_t)t], stop);
    });
    c.text = nullptr;
    if (first_error(errs, failed, e) != IRM_OK) return IRM_EINVAL;
    o.req_tok_off[run_.n_req] = run_.n_tok;
    o.req_seg_off[run_.n_req] = run_.n_seg;
    return IRM_OK;
}

void report(const Err &e, int64_t *err_line, char *err_field, int32_t field_cap) {
    if (err_line) *err_line = e.line;
    if (err_field && field_cap > 0) {
        const size_t n = e.field.size() < (size_t)(field_cap - 1) ? e.field.size() : (size_t)(field_cap - 1);
        memcpy(err_field, e.field.data(), n);
        err_field[n] = 0;
    }
    irm::set_error("%s", e.msg.c_str());
}

}  // namespace

extern "C" int irm_trace_scan(const char *text, int64_t len, int32_t universal, int64_t *sizes, int64_t *err_line,
                              char *err_field, int32_t field_cap) {
    if ((!text && len > 0) || len < 0 || !sizes) {
        irm::set_error("null pointer or negative length");
        return IRM_EINVAL;
    }
    Sizes sz;
    Err e;
    const int rc = scan(text, len, universal != 0, sz, e);
    if (rc != IRM_OK) {
        report(e, err_line, err_field, field_cap);
        return rc;
    }
    sizes[0] = sz.n_req;
    sizes[1] = sz.n_tok;
    sizes[2] = sz.n_seg;
    sizes[3] = sz.n_str;
    return IRM_OK;
}

extern "C" int irm_trace_fill(const char *text, int64_t len, int32_t universal, uint32_t *tokens, int64_t *req_tok_off,
                              int64_t *req_seg_off, int64_t *req_turn, int64_t *req_session, uint8_t *seg_kind,
                              int64_t *seg_tok_off, int64_t *seg_shared, char *strings) {
    if ((!text && len > 0) || !req_tok_off || !req_seg_off || !req_turn || !req_session) {
        irm::set_error("null pointer");
        return IRM_EINVAL;
    }
    Out o{tokens, req_tok_off, req_seg_off, req_turn, req_session, seg_tok_off, seg_shared, seg_kind, strings};
    Err e;
    const int rc = fill(text, len, universal != 0, e, o);
    if (rc != IRM_OK) report(e, nullptr, nullptr, 0);
    return rc;
}
