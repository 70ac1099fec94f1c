// formats.cpp -- host readers for the offline engine's artefacts, written
// fresh and format-compatible with the reference:
//   MPEX  expert weights   inc/io.hpp:210-251  ("MPEX", u32 version 1,
//         u32 d_model, u32 d_ff, then w_gate, w_up, w_down f32 LE row-major)
//   NDJSON partition map   inc/serde.hpp:100-151 (one document per expert:
//         expert_id, n_subexperts, assignment, cost, config) plus the gates
//         stage fields r / gates (inc/serde.hpp:156-168).
// Error behaviour mirrors the reference (ValidationError -> 1, IoError -> 2).
#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <utility>

#include "mp_layer_impl.h"
#include "moeprism/moe_layer.h"

namespace mp {

namespace {

[[noreturn]] void fail(int code, const std::string& msg) { throw Failure{code, msg}; }

uint32_t le_u32(const unsigned char* b) {
    return uint32_t(b[0]) | uint32_t(b[1]) << 8 | uint32_t(b[2]) << 16 | uint32_t(b[3]) << 24;
}

// ------------------------------------------------------------ tiny JSON
struct JVal {
    enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
    bool b = false;
    double num = 0.0;
    bool is_int = false;
    bool neg = false;
    uint64_t u = 0;
    std::string s;
    std::vector<JVal> arr;
    std::vector<std::pair<std::string, JVal>> obj;

    const JVal* get(const char* key) const {
        for (const auto& kv : obj)
            if (kv.first == key) return &kv.second;
        return nullptr;
    }
};

struct Parser {
    const std::string& t;
    size_t i = 0;
    explicit Parser(const std::string& text) : t(text) {}

    [[noreturn]] void err(const std::string& what) {
        fail(MP_ERR_VALIDATION, "parse error at byte " + std::to_string(i) + ": " + what);
    }
    void ws() {
        while (i < t.size() && std::isspace(static_cast<unsigned char>(t[i]))) ++i;
    }
    bool lit(const char* w) {
        size_t n = std::strlen(w);
        if (t.compare(i, n, w) == 0) {
            i += n;
            return true;
        }
        return false;
    }
    JVal value(int depth = 0) {
        if (depth > 64) err("nesting too deep");
        ws();
        if (i >= t.size()) err("unexpected end of input");
        JVal v;
        const char c = t[i];
        if (c == '{') {
            v.kind = JVal::Obj;
            ++i;
            ws();
            if (i < t.size() && t[i] == '}') {
                ++i;
                return v;
            }
            for (;;) {
                ws();
                if (i >= t.size() || t[i] != '"') err("expected object key");
                std::string key = str();
                ws();
                if (i >= t.size() || t[i] != ':') err("expected ':'");
                ++i;
                v.obj.emplace_back(std::move(key), value(depth + 1));
                ws();
                if (i < t.size() && t[i] == ',') {
                    ++i;
                    continue;
                }
                if (i < t.size() && t[i] == '}') {
                    ++i;
                    return v;
                }
                err("expected ',' or '}'");
            }
        }
        if (c == '[') {
            v.kind = JVal::Arr;
            ++i;
            ws();
            if (i < t.size() && t[i] == ']') {
                ++i;
                return v;
            }
            for (;;) {
                v.arr.push_back(value(depth + 1));
                ws();
                if (i < t.size() && t[i] == ',') {
                    ++i;
                    continue;
                }
                if (i < t.size() && t[i] == ']') {
                    ++i;
                    return v;
                }
                err("expected ',' or ']'");
            }
        }
        if (c == '"') {
            v.kind = JVal::Str;
            v.s = str();
            return v;
        }
        if (lit("true")) {
            v.kind = JVal::Bool;
            v.b = true;
            return v;
        }
        if (lit("false")) {
            v.kind = JVal::Bool;
            return v;
        }
        if (lit("null")) return v;
        return number();
    }
    std::string str() {
        ++i;  // opening quote
        std::string out;
        while (i < t.size() && t[i] != '"') {
            if (t[i] == '\\') {
                ++i;
                if (i >= t.size()) err("bad escape");
                const char e = t[i];
                if (e == 'u') {
                    if (i + 4 >= t.size()) err("bad \\u escape");
                    out += '?';
                    i += 4;
                } else {
                    out += e == 'n' ? '\n' : e == 't' ? '\t' : e == 'r' ? '\r' : e == 'b' ? '\b' : e == 'f' ? '\f' : e;
                }
                ++i;
            } else {
                out += t[i++];
            }
        }
        if (i >= t.size()) err("unterminated string");
        ++i;
        return out;
    }
    JVal number() {
        JVal v;
        v.kind = JVal::Num;
        const size_t st = i;
        if (i < t.size() && t[i] == '-') ++i;
        bool digits = false, frac = false;
        while (i < t.size() && std::isdigit(static_cast<unsigned char>(t[i]))) ++i, digits = true;
        if (i < t.size() && t[i] == '.') {
            frac = true;
            ++i;
            while (i < t.size() && std::isdigit(static_cast<unsigned char>(t[i]))) ++i;
        }
        if (i < t.size() && (t[i] == 'e' || t[i] == 'E')) {
            frac = true;
            ++i;
            if (i < t.size() && (t[i] == '+' || t[i] == '-')) ++i;
            while (i < t.size() && std::isdigit(static_cast<unsigned char>(t[i]))) ++i;
        }
        if (!digits) err("invalid literal");
        const std::string tok = t.substr(st, i - st);
        v.num = std::strtod(tok.c_str(), nullptr);
        v.neg = tok[0] == '-';
        if (!frac) {
            v.is_int = true;
            v.u = std::strtoull(tok.c_str() + (v.neg ? 1 : 0), nullptr, 10);
        }
        return v;
    }
};

// detail::require (inc/serde.hpp:42-51): missing field or wrong type -> ValidationError
const JVal& require(const JVal& j, const char* key, const std::string& what) {
    const JVal* v = j.kind == JVal::Obj ? j.get(key) : nullptr;
    if (!v) fail(MP_ERR_VALIDATION, what + " is missing the '" + key + "' field");
    return *v;
}
uint64_t as_uint(const JVal& v, const char* key, const std::string& what) {
    if (v.kind != JVal::Num || v.neg) fail(MP_ERR_VALIDATION, what + " field '" + key + "': not an unsigned number");
    return v.is_int ? v.u : static_cast<uint64_t>(v.num);
}
std::vector<uint32_t> as_u32_array(const JVal& v, const char* key, const std::string& what) {
    if (v.kind != JVal::Arr) fail(MP_ERR_VALIDATION, what + " field '" + key + "': not an array");
    std::vector<uint32_t> out;
    out.reserve(v.arr.size());
    for (const auto& e : v.arr) out.push_back(static_cast<uint32_t>(as_uint(e, key, what)));
    return out;
}

}  // namespace

void validate_partition(uint32_t n_sub, const uint32_t* a, size_t n) {
    if (n_sub < 1) fail(MP_ERR_VALIDATION, "partition needs at least one sub-expert");
    if (n < n_sub) fail(MP_ERR_VALIDATION, "partition needs at least as many neurons as sub-experts");
    std::vector<size_t> sizes(n_sub, 0);
    for (size_t c = 0; c < n; ++c) {
        if (a[c] >= n_sub)
            fail(MP_ERR_VALIDATION,
                 "partition label " + std::to_string(a[c]) + " out of range for N=" + std::to_string(n_sub));
        ++sizes[a[c]];
    }
    size_t lo = sizes[0], hi = sizes[0];
    for (size_t s : sizes) lo = s < lo ? s : lo, hi = s > hi ? s : hi;
    if (lo == 0) fail(MP_ERR_VALIDATION, "every sub-expert must be non-empty");
    if (hi - lo > 1)
        fail(MP_ERR_VALIDATION, "partition is not balanced: sizes range from " + std::to_string(lo) + " to " +
                                    std::to_string(hi));
}

// MPAM activation matrix (inc/io.hpp:147-158 save_activation_matrix,
// :162-200 load_activation_matrix binary branch): "MPAM", u32 version 1,
// u32 rows, u32 cols, rows*cols little-endian f32 row-major.  The reader
// rejects trailing bytes and non-finite values and rectifies (|v|) like the
// reference's loader.
void write_mpam(const std::string& path, uint32_t rows, uint32_t cols, const float* data) {
    if (rows < 1 || cols < 1) fail(MP_ERR_VALIDATION, "activation matrix must have at least one row and one column");
    for (size_t i = 0; i < (size_t)rows * cols; ++i)
        if (!std::isfinite(data[i]) || data[i] < 0.0f)
            fail(MP_ERR_VALIDATION, "activation matrix entries must be finite and non-negative");
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) fail(MP_ERR_IO, "cannot open " + path + " for writing");
    unsigned char hdr[16] = {'M', 'P', 'A', 'M'};
    const uint32_t v[3] = {1u, rows, cols};
    for (int i = 0; i < 3; ++i)
        for (int b = 0; b < 4; ++b) hdr[4 + 4 * i + b] = static_cast<unsigned char>(v[i] >> (8 * b));
    out.write(reinterpret_cast<const char*>(hdr), 16);
    out.write(reinterpret_cast<const char*>(data), static_cast<std::streamsize>((size_t)rows * cols * 4));
    if (!out) fail(MP_ERR_IO, "failed while writing " + path);
}

std::vector<float> read_mpam(const std::string& path, uint32_t& rows, uint32_t& cols) {
    std::ifstream in(path, std::ios::binary);
    if (!in) fail(MP_ERR_IO, "cannot open " + path);
    unsigned char hdr[16];
    if (!in.read(reinterpret_cast<char*>(hdr), 4) || std::memcmp(hdr, "MPAM", 4) != 0)
        fail(MP_ERR_VALIDATION, path + " does not start with the 'MPAM' magic");
    if (!in.read(reinterpret_cast<char*>(hdr + 4), 12)) fail(MP_ERR_VALIDATION, "truncated file while reading header");
    if (le_u32(hdr + 4) != 1) fail(MP_ERR_VALIDATION, path + " has unsupported version " + std::to_string(le_u32(hdr + 4)));
    rows = le_u32(hdr + 8);
    cols = le_u32(hdr + 12);
    if (rows < 1 || cols < 1) fail(MP_ERR_VALIDATION, path + " declares an empty matrix");
    std::vector<float> d((size_t)rows * cols);
    if (!in.read(reinterpret_cast<char*>(d.data()), static_cast<std::streamsize>(d.size() * 4)))
        fail(MP_ERR_VALIDATION, "truncated file while reading matrix data");
    char extra;
    if (in.read(&extra, 1)) fail(MP_ERR_VALIDATION, path + " holds more data than its header declares");
    for (size_t i = 0; i < d.size(); ++i) {
        if (!std::isfinite(d[i]))
            fail(MP_ERR_VALIDATION, path + ": non-finite value at row " + std::to_string(i / cols) + ", col " +
                                        std::to_string(i % cols));
        d[i] = std::fabs(d[i]);
    }
    return d;
}

MpexData read_mpex(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) fail(MP_ERR_IO, "cannot open " + path);
    unsigned char hdr[16];
    if (!in.read(reinterpret_cast<char*>(hdr), 4) || std::memcmp(hdr, "MPEX", 4) != 0)
        fail(MP_ERR_VALIDATION, path + " does not start with the 'MPEX' magic");
    if (!in.read(reinterpret_cast<char*>(hdr + 4), 4)) fail(MP_ERR_VALIDATION, "truncated file while reading version");
    const uint32_t version = le_u32(hdr + 4);
    if (version != 1) fail(MP_ERR_VALIDATION, path + " has unsupported version " + std::to_string(version));
    if (!in.read(reinterpret_cast<char*>(hdr + 8), 4)) fail(MP_ERR_VALIDATION, "truncated file while reading d_model");
    if (!in.read(reinterpret_cast<char*>(hdr + 12), 4)) fail(MP_ERR_VALIDATION, "truncated file while reading d_ff");
    MpexData m;
    m.d_model = le_u32(hdr + 8);
    m.d_ff = le_u32(hdr + 12);
    if (m.d_model < 1 || m.d_ff < 1) fail(MP_ERR_VALIDATION, path + " declares empty expert dimensions");
    const size_t n = static_cast<size_t>(m.d_model) * m.d_ff;
    for (auto* w : {&m.w_gate, &m.w_up, &m.w_down}) {
        w->resize(n);
        if (!in.read(reinterpret_cast<char*>(w->data()), static_cast<std::streamsize>(n * 4)))
            fail(MP_ERR_VALIDATION, "truncated file while reading expert weights");
        // file is little-endian f32; this host is little-endian (x86-64 / aarch64)
    }
    char extra;
    if (in.read(&extra, 1)) fail(MP_ERR_VALIDATION, path + " holds more data than its header declares");
    for (const auto* w : {&m.w_gate, &m.w_up, &m.w_down})
        for (float v : *w)
            if (!std::isfinite(v)) fail(MP_ERR_VALIDATION, "toy expert weight is not finite");
    return m;
}

std::vector<PartitionDocHost> read_partition_map(const std::string& path) {
    std::ifstream in(path);
    if (!in) fail(MP_ERR_IO, "cannot open " + path);
    std::vector<PartitionDocHost> docs;
    std::string line;
    size_t lineno = 0;
    while (std::getline(in, line)) {
        ++lineno;
        if (line.empty()) continue;
        JVal j;
        try {
            Parser p(line);
            j = p.value();
            p.ws();
            if (p.i != line.size()) p.err("trailing characters");
        } catch (const Failure& f) {
            fail(MP_ERR_VALIDATION, path + ":" + std::to_string(lineno) + ": " + f.msg);
        }
        const std::string what = "partition map";
        PartitionDocHost d;
        d.expert_id = as_uint(require(j, "expert_id", what), "expert_id", what);
        d.n_subexperts = static_cast<uint32_t>(as_uint(require(j, "n_subexperts", what), "n_subexperts", what));
        d.assignment = as_u32_array(require(j, "assignment", what), "assignment", what);
        const JVal& cost = require(j, "cost", what);
        if (cost.kind != JVal::Num) fail(MP_ERR_VALIDATION, what + " field 'cost': not a number");
        const JVal& cfg = require(j, "config", what);
        const std::string cw = "solver config";
        for (const char* key : {"n_subexperts", "k_deact", "t0", "alpha", "iterations", "seed"})
            if (require(cfg, key, cw).kind != JVal::Num)
                fail(MP_ERR_VALIDATION, cw + " field '" + std::string(key) + "': not a number");
        validate_partition(d.n_subexperts, d.assignment.data(), d.assignment.size());
        if (j.get("gates") || j.get("r")) {
            const std::string gw = "gate set";
            d.has_gates = true;
            d.r = static_cast<uint32_t>(as_uint(require(j, "r", gw), "r", gw));
            const JVal& g = require(j, "gates", gw);
            if (g.kind != JVal::Arr) fail(MP_ERR_VALIDATION, gw + " field 'gates': not an array");
            for (const auto& row : g.arr) d.gates.push_back(as_u32_array(row, "gates", gw));
            // validate(GateSet), inc/gating.hpp:33-43
            if (d.n_subexperts < 1 || d.gates.size() != d.n_subexperts || d.r < 1)
                fail(MP_ERR_VALIDATION, "gate set shape is inconsistent");
            for (const auto& l : d.gates) {
                if (l.empty()) fail(MP_ERR_VALIDATION, "every sub-expert needs at least one gate neuron");
                for (size_t q = 1; q < l.size(); ++q)
                    if (l[q] < l[q - 1]) fail(MP_ERR_VALIDATION, "gate neuron lists must be ascending");
            }
        }
        docs.push_back(std::move(d));
    }
    if (docs.empty()) fail(MP_ERR_VALIDATION, path + " holds no documents");
    return docs;
}

}  // namespace mp
