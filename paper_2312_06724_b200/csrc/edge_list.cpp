// edge_list.cpp -- native text edge-list parser (host code), the fast path of
// load_edge_list (reference bigraph.py:272-350, a per-line Python loop).
//
// Semantics restated for ASCII input: lines end at '\n', "\r\n" or '\r'
// (Python text-mode universal newlines); each line is stripped of ASCII
// whitespace (' ', \t \n \v \f \r, \x1c-\x1f: what str.strip() removes from
// ASCII text); blank lines and lines starting with '#' are skipped; columns
// split on runs of whitespace (delimiter absent) or on an exact delimiter
// string (empty fields kept, like str.split(sep)); 2 columns take the default
// weight, 3 columns parse the weight; U labels are numbered in order of first
// appearance as a U label, V labels likewise; repeated (u, v) pairs sum their
// weights in line order (from_edges, bigraph.py:115-130).
//
// Anything this restatement does not cover exactly returns PARSE_FALLBACK so
// the caller runs the reference-semantics Python loop instead: non-ASCII
// bytes (unicode whitespace and labels), weight tokens other than plain
// decimal numbers (Python float() also takes "inf", "nan", "1_000", ...), and
// every error (the Python loop raises the reference's exact message).
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <string_view>
#include <vector>

#include "common.cuh"

namespace bh {

namespace {

inline bool is_ws(unsigned char c) { return c == ' ' || (c >= 0x09 && c <= 0x0d) || (c >= 0x1c && c <= 0x1f); }

// Plain decimal float: [+-] digits [. digits] [(e|E) [+-] digits], at least one digit.
bool parse_plain_float(std::string_view tok, double &out) {
    size_t i = 0, n = tok.size();
    if (n == 0) return false;
    if (tok[i] == '+' || tok[i] == '-') i++;
    size_t dig = 0;
    while (i < n && tok[i] >= '0' && tok[i] <= '9') i++, dig++;
    if (i < n && tok[i] == '.') {
        i++;
        while (i < n && tok[i] >= '0' && tok[i] <= '9') i++, dig++;
    }
    if (dig == 0) return false;
    if (i < n && (tok[i] == 'e' || tok[i] == 'E')) {
        i++;
        if (i < n && (tok[i] == '+' || tok[i] == '-')) i++;
        size_t ed = 0;
        while (i < n && tok[i] >= '0' && tok[i] <= '9') i++, ed++;
        if (ed == 0) return false;
    }
    if (i != n) return false;
    // strtod needs a terminator; glibc strtod rounds correctly, as float() does
    char small[64];
    std::string big;
    const char *z;
    if (n < sizeof(small)) {
        std::memcpy(small, tok.data(), n);
        small[n] = 0;
        z = small;
    } else {
        big.assign(tok);
        z = big.c_str();
    }
    char *end = nullptr;
    out = std::strtod(z, &end);
    return end == z + n;
}

inline uint64_t mix64(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    return x ^ (x >> 33);
}

inline uint64_t hash_bytes(std::string_view s) {  // FNV-1a, then mixed
    uint64_t h = 1469598103934665603ull;
    for (unsigned char c : s) h = (h ^ c) * 1099511628211ull;
    return mix64(h);
}

// Open-addressing tables (linear probing, power-of-two capacity, load <= 1/2):
// the per-line work is a few probes into flat arrays instead of node allocations.
struct LabelTable {  // label -> first-seen id
    std::vector<int64_t> slot;  // id + 1, 0 = empty
    std::vector<uint64_t> hv;
    std::vector<std::string_view> labels;
    LabelTable() : slot(1024, 0), hv(1024, 0) {}
    int64_t find(std::string_view s, uint64_t h) const {
        const size_t m = slot.size() - 1;
        for (size_t i = h & m;; i = (i + 1) & m) {
            const int64_t id = slot[i] - 1;
            if (id < 0) return -1;
            if (hv[i] == h && labels[id] == s) return id;
        }
    }
    int64_t insert(std::string_view s, uint64_t h) {  // id of s, adding it if new
        if (2 * (labels.size() + 1) > slot.size()) grow();
        const size_t m = slot.size() - 1;
        for (size_t i = h & m;; i = (i + 1) & m) {
            const int64_t id = slot[i] - 1;
            if (id < 0) {
                slot[i] = (int64_t)labels.size() + 1;
                hv[i] = h;
                labels.push_back(s);
                return (int64_t)labels.size() - 1;
            }
            if (hv[i] == h && labels[id] == s) return id;
        }
    }
    void grow() {
        std::vector<int64_t> os = std::move(slot);
        std::vector<uint64_t> oh = std::move(hv);
        slot.assign(os.size() * 2, 0);
        hv.assign(os.size() * 2, 0);
        const size_t m = slot.size() - 1;
        for (size_t j = 0; j < os.size(); j++) {
            if (!os[j]) continue;
            size_t i = oh[j] & m;
            while (slot[i]) i = (i + 1) & m;
            slot[i] = os[j];
            hv[i] = oh[j];
        }
    }
};

struct PairTable {  // (u, v) -> merged edge index
    std::vector<uint64_t> key;   // (u << 32 | v) + 1, 0 = empty
    std::vector<int64_t> val;
    size_t n = 0;
    PairTable() : key(1024, 0), val(1024, 0) {}
    int64_t &at(uint64_t k, bool &fresh) {
        if (2 * (n + 1) > key.size()) grow();
        const size_t m = key.size() - 1;
        for (size_t i = mix64(k) & m;; i = (i + 1) & m) {
            if (key[i] == k + 1) {
                fresh = false;
                return val[i];
            }
            if (!key[i]) {
                key[i] = k + 1;
                n++;
                fresh = true;
                return val[i];
            }
        }
    }
    void grow() {
        std::vector<uint64_t> ok = std::move(key);
        std::vector<int64_t> ov = std::move(val);
        key.assign(ok.size() * 2, 0);
        val.assign(ok.size() * 2, 0);
        const size_t m = key.size() - 1;
        for (size_t j = 0; j < ok.size(); j++) {
            if (!ok[j]) continue;
            size_t i = mix64(ok[j] - 1) & m;
            while (key[i]) i = (i + 1) & m;
            key[i] = ok[j];
            val[i] = ov[j];
        }
    }
};

}  // namespace

EdgeListResult parse_edge_list(const char *buf, int64_t len, const char *delim, int64_t delim_len,
                               bool has_default, double default_weight) {
    EdgeListResult r;
    for (int64_t i = 0; i < len; i++)
        if ((unsigned char)buf[i] >= 0x80) {
            r.status = PARSE_FALLBACK;
            return r;
        }
    LabelTable u_index, v_index;
    PairTable pair_index;
    std::vector<std::string_view> cols;
    int64_t lineno = 0, pos = 0;
    while (pos < len) {
        // one physical line (universal newlines)
        int64_t end = pos;
        while (end < len && buf[end] != '\n' && buf[end] != '\r') end++;
        int64_t next = end;
        if (next < len) next += (buf[next] == '\r' && next + 1 < len && buf[next + 1] == '\n') ? 2 : 1;
        lineno++;
        int64_t a = pos, b = end;
        pos = next;
        while (a < b && is_ws((unsigned char)buf[a])) a++;
        while (b > a && is_ws((unsigned char)buf[b - 1])) b--;
        if (a == b || buf[a] == '#') continue;
        cols.clear();
        if (!delim) {
            int64_t i = a;
            while (i < b) {
                while (i < b && is_ws((unsigned char)buf[i])) i++;
                int64_t j = i;
                while (j < b && !is_ws((unsigned char)buf[j])) j++;
                if (j > i) cols.emplace_back(buf + i, (size_t)(j - i));
                i = j;
            }
        } else {
            const std::string_view line(buf + a, (size_t)(b - a)), sep(delim, (size_t)delim_len);
            size_t i = 0;
            while (true) {
                const size_t j = line.find(sep, i);
                if (j == std::string_view::npos) {
                    cols.push_back(line.substr(i));
                    break;
                }
                cols.push_back(line.substr(i, j - i));
                i = j + sep.size();
            }
        }
        double w;
        if (cols.size() == 2) {
            if (!has_default) {
                r.status = PARSE_ERROR;
                r.err_line = lineno;
                return r;
            }
            w = default_weight;
        } else if (cols.size() == 3) {
            std::string_view t = cols[2];  // float() ignores surrounding whitespace
            while (!t.empty() && is_ws((unsigned char)t.front())) t.remove_prefix(1);
            while (!t.empty() && is_ws((unsigned char)t.back())) t.remove_suffix(1);
            if (!parse_plain_float(t, w)) {
                r.status = PARSE_FALLBACK;  // "inf", "1_0", "abc", ...: Python decides (value or error)
                return r;
            }
        } else {
            r.status = PARSE_ERROR;
            r.err_line = lineno;
            return r;
        }
        if (!std::isfinite(w) || w <= 0) {
            r.status = PARSE_ERROR;
            r.err_line = lineno;
            return r;
        }
        const std::string_view ul = cols[0], vl = cols[1];
        const uint64_t hu = hash_bytes(ul), hvl = hash_bytes(vl);
        if (v_index.find(ul, hu) >= 0 || u_index.find(vl, hvl) >= 0) {
            r.status = PARSE_ERROR;
            r.err_line = lineno;
            return r;
        }
        const int64_t ui = u_index.insert(ul, hu), vi = v_index.insert(vl, hvl);
        if (u_index.labels.size() >= (1ull << 31) || v_index.labels.size() >= (1ull << 31)) {
            r.status = PARSE_FALLBACK;
            return r;
        }
        bool fresh;
        int64_t &slot = pair_index.at(((uint64_t)ui << 32) | (uint64_t)vi, fresh);
        if (fresh) {
            slot = (int64_t)r.ew.size();
            r.eu.push_back(ui);
            r.ev.push_back(vi);
            r.ew.push_back(0.0 + w);
        } else {
            r.ew[slot] += w;  // merged in line order
        }
    }
    if (r.ew.empty()) {
        r.status = PARSE_ERROR;  // "empty graph: no data lines found"
        r.err_line = 0;
        return r;
    }
    r.u_labels.reserve(u_index.labels.size());
    for (auto s : u_index.labels) r.u_labels.emplace_back(s);
    r.v_labels.reserve(v_index.labels.size());
    for (auto s : v_index.labels) r.v_labels.emplace_back(s);
    return r;
}

}  // namespace bh
