// GRAPHSNAP1 load straight into a device graph.
//
// Replaces, for the k-hop path, snapshot_from_string / snapshot_load
// (proj/core/src/snapshot.cpp:162-259) followed by relation_matrix: the text
// is copied to the GPU once, every line is split and parsed by its own thread
// (node and edge lines are independent), the edge keys of the requested
// relation (or ANY) are compacted, sorted, de-duplicated and assembled into
// CSR + CSC on the device. Labels and properties are validated but not kept
// (the k-hop path never reads them).
//
// Error behaviour is the reference's, message for message: the GPU pass only
// classifies lines as "certainly valid" or "suspect" (a conservative subset of
// the grammar: plain decimal ids, identifier keys/labels/relations, simple
// numerals); suspect lines -- real errors and the rare exotic literal like
// "inf" or ".5" -- are re-checked in file order on the host by an exact
// restatement of the reference's rules (std::from_chars like encoding.cpp,
// the same split / field / argument-evaluation order), and the first failing
// line yields "snapshot parse error at line N: ...".
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <charconv>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <optional>
#include <string>
#include <string_view>
#include <vector>

#include "mgk_internal.cuh"

namespace mgk {
namespace snap {

// ---- host: exact restatement of the reference's snapshot grammar ----------------
namespace {

std::vector<std::string_view> split(std::string_view s, char sep) {  // snapshot.cpp:18-30
    std::vector<std::string_view> parts;
    size_t start = 0;
    for (;;) {
        const size_t pos = s.find(sep, start);
        if (pos == std::string_view::npos) {
            parts.push_back(s.substr(start));
            return parts;
        }
        parts.push_back(s.substr(start, pos - start));
        start = pos + 1;
    }
}

bool ident(std::string_view s) {  // encoding.cpp:118-127
    if (s.empty()) return false;
    auto head = [](char c) { return (c >= 'A' && c <= 'Z') || (c >= 'a' && c <= 'z') || c == '_'; };
    if (!head(s[0])) return false;
    for (char c : s.substr(1))
        if (!head(c) && !(c >= '0' && c <= '9')) return false;
    return true;
}

template <typename T>
bool whole(std::string_view t, T& v) {  // parse_uint / parse_int / parse_double (encoding.cpp:91-116)
    auto [ptr, ec] = std::from_chars(t.data(), t.data() + t.size(), v);
    return ec == std::errc{} && ptr == t.data() + t.size();
}

std::string q(std::string_view s) { return "'" + std::string(s) + "'"; }

int hexv(char c) {
    if (c >= '0' && c <= '9') return c - '0';
    if (c >= 'a' && c <= 'f') return c - 'a' + 10;
    if (c >= 'A' && c <= 'F') return c - 'A' + 10;
    return -1;
}

// decode_value (snapshot.cpp:37-48) + percent_decode (encoding.cpp:44-62)
std::optional<std::string> check_value(char type, std::string_view text) {
    switch (type) {
        case 'i': {
            int64_t v;
            if (!whole(text, v)) return "not a 64-bit integer: " + q(text);
            return std::nullopt;
        }
        case 'f': {
            double v;
            if (!whole(text, v)) return "not a floating-point number: " + q(text);
            return std::nullopt;
        }
        case 'b':
            if (text == "true" || text == "false") return std::nullopt;
            return "bad boolean " + q(text);
        case 's':
            for (size_t i = 0; i < text.size(); ++i) {
                if (text[i] != '%') continue;
                if (i + 2 >= text.size()) return "truncated percent escape at position " + std::to_string(i);
                if (hexv(text[i + 1]) < 0 || hexv(text[i + 2]) < 0)
                    return std::string("malformed percent escape '%") + text[i + 1] + text[i + 2] + "'";
                i += 2;
            }
            return std::nullopt;
        default:
            return std::string("unknown property type '") + type + "'";
    }
}

// decode_props (snapshot.cpp:110-125). An item needs "key:t:" -- the reference
// peeks one byte past a 3-byte item, which is never ':' (the next byte ends
// the item or the field), so a too-short item is malformed.
std::optional<std::string> check_props(std::string_view field) {
    if (field.empty()) return std::nullopt;
    for (std::string_view item : split(field, ';')) {
        const size_t first = item.find(':');
        if (first == std::string_view::npos || first + 2 >= item.size() || item[first + 2] != ':')
            return "malformed property item " + q(item);
        const std::string_view key = item.substr(0, first);
        if (!ident(key)) return "bad property key " + q(key);
        if (auto e = check_value(item[first + 1], item.substr(first + 3))) return e;
    }
    return std::nullopt;
}

}  // namespace

// node line i (snapshot.cpp:185-205 + create_node, graph.cpp:31-43)
std::optional<std::string> check_node_line(std::string_view line, uint64_t i) {
    const auto f = split(line, '\t');
    if (f.size() != 3) return std::string("node line must have 3 tab-separated fields");
    uint64_t id = 0;
    if (!whole(f[0], id)) return std::string("bad node id");
    if (id != i) return "node id " + std::to_string(id) + " out of order (expected " + std::to_string(i) + ")";
    std::vector<std::string_view> labels;
    if (!f[1].empty()) labels = split(f[1], ',');
    if (auto e = check_props(f[2])) return e;  // decode_props runs before create_node
    for (auto l : labels)
        if (!ident(l)) return "label " + q(l) + " is not a valid identifier";
    return std::nullopt;
}

// edge line (snapshot.cpp:216-225 + create_edge, graph.cpp:54-68). The call
// create_edge(parse_uint(f0), string(f1), parse_uint(f2), decode_props(f3))
// evaluates its arguments right to left in the reference build (g++), so the
// props are checked first, then dst, then src.
std::optional<std::string> check_edge_line(std::string_view line, uint64_t node_count, uint64_t* src_out,
                                           uint64_t* dst_out, std::string_view* rel_out) {
    const auto f = split(line, '\t');
    if (f.size() != 4) return std::string("edge line must have 4 tab-separated fields");
    if (auto e = check_props(f[3])) return e;
    uint64_t src = 0, dst = 0;
    if (!whole(f[2], dst)) return "not an unsigned 64-bit integer: " + q(f[2]);
    if (!whole(f[0], src)) return "not an unsigned 64-bit integer: " + q(f[0]);
    if (src >= node_count || dst >= node_count)
        return "unknown node id " + std::to_string(src >= node_count ? src : dst) + " in edge (" +
               std::to_string(src) + ")-[:" + std::string(f[1]) + "]->(" + std::to_string(dst) + ")";
    if (!ident(f[1])) return "relation type " + q(f[1]) + " is not a valid identifier";
    if (src_out) *src_out = src;
    if (dst_out) *dst_out = dst;
    if (rel_out) *rel_out = f[1];
    return std::nullopt;
}

std::string at_line(uint64_t line, const std::string& what) {
    return "snapshot parse error at line " + std::to_string(line) + ": " + what;
}

// LineReader (snapshot.cpp:52-80): lines split on '\n'; a final '\n' does not
// start another line.
struct Lines {
    std::string_view text;
    size_t pos = 0;
    bool pending = false;
    uint64_t no = 0;
    bool next(std::string_view& line) {
        if (pos >= text.size() && !pending) return false;
        ++no;
        const size_t nl = text.find('\n', pos);
        if (nl == std::string_view::npos) {
            line = text.substr(pos);
            pos = text.size();
            pending = false;
        } else {
            line = text.substr(pos, nl - pos);
            pos = nl + 1;
            pending = pos < text.size();
        }
        return true;
    }
};

// Header: "GRAPHSNAP1", "NODES <n>" (snapshot.cpp:165-177). Returns the byte
// offset just past the NODES line.
std::optional<std::string> parse_header(std::string_view text, uint64_t* n, size_t* body) {
    Lines r{text};
    std::string_view line;
    if (!r.next(line) || line != "GRAPHSNAP1") return at_line(1, "missing GRAPHSNAP1 header");
    if (!r.next(line)) return at_line(r.no + 1, "expected NODES <count>");
    if (line.substr(0, 6) != "NODES ") return at_line(r.no, "expected NODES <count>");
    if (!whole(line.substr(6), *n)) return at_line(r.no, "bad NODES count");
    *body = r.pos;
    return std::nullopt;
}

// The whole grammar, sequentially (the host-only checker behind
// mgk_snapshot_check, and the reference semantics the GPU path must match).
std::optional<std::string> check_all(std::string_view text, uint64_t* n_out, uint64_t* m_out) {
    uint64_t n = 0;
    size_t body = 0;
    if (auto e = parse_header(text, &n, &body)) return e;
    Lines r{text};
    std::string_view line;
    r.next(line);
    r.next(line);
    for (uint64_t i = 0; i < n; ++i) {
        if (!r.next(line)) return at_line(r.no + 1, "unexpected end of file in node section");
        if (auto e = check_node_line(line, i)) return at_line(r.no, *e);
    }
    if (!r.next(line)) return at_line(r.no + 1, "expected EDGES <count>");
    if (line.substr(0, 6) != "EDGES ") return at_line(r.no, "expected EDGES <count>");
    uint64_t m = 0;
    if (!whole(line.substr(6), m)) return at_line(r.no, "bad EDGES count");
    for (uint64_t i = 0; i < m; ++i) {
        if (!r.next(line)) return at_line(r.no + 1, "unexpected end of file in edge section");
        if (auto e = check_edge_line(line, n, nullptr, nullptr, nullptr)) return at_line(r.no, *e);
    }
    while (r.next(line))
        if (!line.empty()) return at_line(r.no, "trailing content after edge section");
    *n_out = n;
    *m_out = m;
    return std::nullopt;
}

// ---- device: line split + conservative per-line validation ------------------------
namespace {

struct IsNewline {
    const char* t;
    __host__ __device__ bool operator()(uint64_t i) const { return t[i] == '\n'; }
};

struct LineTab {
    const uint64_t* nl;  // sorted '\n' positions
    uint64_t nnl, len;
    __device__ void bounds(uint64_t idx, uint64_t& b, uint64_t& e) const {
        b = idx == 0 ? 0 : nl[idx - 1] + 1;
        e = idx < nnl ? nl[idx] : len;
    }
};

__device__ bool d_digit(char c) { return c >= '0' && c <= '9'; }
__device__ bool d_head(char c) { return (c >= 'A' && c <= 'Z') || (c >= 'a' && c <= 'z') || c == '_'; }
__device__ bool d_hex(char c) { return d_digit(c) || (c >= 'a' && c <= 'f') || (c >= 'A' && c <= 'F'); }

__device__ bool d_ident(const char* s, uint64_t n) {
    if (n == 0 || !d_head(s[0])) return false;
    for (uint64_t i = 1; i < n; ++i)
        if (!d_head(s[i]) && !d_digit(s[i])) return false;
    return true;
}

// plain decimal, 1..19 digits (no overflow possible)
__device__ bool d_uint(const char* s, uint64_t n, uint64_t& v) {
    if (n == 0 || n > 19) return false;
    v = 0;
    for (uint64_t i = 0; i < n; ++i) {
        if (!d_digit(s[i])) return false;
        v = v * 10 + (uint64_t)(s[i] - '0');
    }
    return true;
}

// certainly-valid property values; anything else is left to the host
__device__ bool d_value(char type, const char* s, uint64_t n) {
    switch (type) {
        case 'i': {
            uint64_t i = (n && s[0] == '-') ? 1 : 0, v;
            return n - i <= 18 && d_uint(s + i, n - i, v);
        }
        case 'b':
            return (n == 4 && s[0] == 't' && s[1] == 'r' && s[2] == 'u' && s[3] == 'e') ||
                   (n == 5 && s[0] == 'f' && s[1] == 'a' && s[2] == 'l' && s[3] == 's' && s[4] == 'e');
        case 's':
            for (uint64_t i = 0; i < n; ++i)
                if (s[i] == '%') {
                    if (i + 2 >= n || !d_hex(s[i + 1]) || !d_hex(s[i + 2])) return false;
                    i += 2;
                }
            return true;
        case 'f': {  // -?D{1,20}(.D{0,20})?([eE][-+]?D{1,3})?, |exponent| <= 280
            uint64_t i = (n && s[0] == '-') ? 1 : 0, d = 0;
            while (i < n && d_digit(s[i])) ++i, ++d;
            if (d == 0 || d > 20) return false;
            if (i < n && s[i] == '.') {
                ++i;
                uint64_t fd = 0;
                while (i < n && d_digit(s[i])) ++i, ++fd;
                if (fd > 20) return false;
            }
            if (i < n && (s[i] == 'e' || s[i] == 'E')) {
                ++i;
                if (i < n && (s[i] == '-' || s[i] == '+')) ++i;
                uint64_t ed = 0, ev = 0;
                while (i < n && d_digit(s[i])) ev = ev * 10 + (uint64_t)(s[i] - '0'), ++i, ++ed;
                if (ed == 0 || ed > 3 || ev > 280) return false;
            }
            return i == n;
        }
        default:
            return false;
    }
}

__device__ bool d_props(const char* s, uint64_t n) {
    if (n == 0) return true;
    uint64_t a = 0;
    for (;;) {
        uint64_t b = a;
        while (b < n && s[b] != ';') ++b;
        const char* it = s + a;
        const uint64_t len = b - a;
        uint64_t first = 0;
        while (first < len && it[first] != ':') ++first;
        if (first + 2 >= len || it[first + 2] != ':') return false;
        if (!d_ident(it, first)) return false;
        if (!d_value(it[first + 1], it + first + 3, len - first - 3)) return false;
        if (b >= n) return true;
        a = b + 1;
    }
}

__global__ void node_lines(const char* t, LineTab L, uint64_t first_line, uint64_t count, uint8_t* suspect) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < count;
         j += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t b, e;
        L.bounds(first_line + j, b, e);
        const char* s = t + b;
        const uint64_t n = e - b;
        uint64_t t1 = 0;
        while (t1 < n && s[t1] != '\t') ++t1;
        uint64_t t2 = t1 + 1;
        while (t2 < n && s[t2] != '\t') ++t2;
        bool ok = t1 < n && t2 < n;
        if (ok)
            for (uint64_t i = t2 + 1; i < n; ++i)
                if (s[i] == '\t') ok = false;
        uint64_t id = 0;
        ok = ok && d_uint(s, t1, id) && id == j;
        if (ok && t2 > t1 + 1) {  // labels: comma-separated identifiers
            uint64_t a = t1 + 1;
            for (;;) {
                uint64_t c = a;
                while (c < t2 && s[c] != ',') ++c;
                if (!d_ident(s + a, c - a)) {
                    ok = false;
                    break;
                }
                if (c >= t2) break;
                a = c + 1;
            }
        }
        ok = ok && d_props(s + t2 + 1, n - t2 - 1);
        suspect[first_line + j] = ok ? 0 : 1;
    }
}

// edge lines: validate, and emit (src << 32 | dst) for the wanted relation
__global__ void edge_lines(const char* t, LineTab L, uint64_t first_line, uint64_t count, uint64_t nodes,
                           const char* rel, uint32_t rel_len, int any, uint8_t* suspect,
                           unsigned long long* keys, uint8_t* keep) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < count;
         j += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t b, e;
        L.bounds(first_line + j, b, e);
        const char* s = t + b;
        const uint64_t n = e - b;
        uint64_t tb[3], nt = 0;
        for (uint64_t i = 0; i < n; ++i)
            if (s[i] == '\t') {
                if (nt < 3) tb[nt] = i;
                ++nt;
            }
        bool ok = nt == 3;
        uint64_t src = 0, dst = 0;
        ok = ok && d_uint(s, tb[0], src) && d_uint(s + tb[1] + 1, tb[2] - tb[1] - 1, dst) && src < nodes &&
             dst < nodes && d_ident(s + tb[0] + 1, tb[1] - tb[0] - 1) &&
             d_props(s + tb[2] + 1, n - tb[2] - 1);
        bool match = false;
        if (ok) {
            match = any != 0;
            if (!match && tb[1] - tb[0] - 1 == rel_len) {
                match = true;
                for (uint32_t i = 0; i < rel_len; ++i)
                    if (s[tb[0] + 1 + i] != rel[i]) match = false;
            }
        }
        suspect[first_line + j] = ok ? 0 : 1;
        keep[j] = match ? 1 : 0;
        keys[j] = ((unsigned long long)src << 32) | dst;
    }
}

__global__ void trailing_lines(const LineTab L, uint64_t first_line, uint64_t count, uint8_t* suspect) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < count;
         j += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t b, e;
        L.bounds(first_line + j, b, e);
        suspect[first_line + j] = e > b ? 1 : 0;
    }
}

constexpr int kTB = 256;
unsigned blocks_for(uint64_t n) { return (unsigned)std::min<uint64_t>((n + kTB - 1) / kTB, 148ull * 64); }

#define SNAP_TRY(x)                        \
    do {                                   \
        if ((e = (x)) != cudaSuccess) goto done; \
    } while (0)

}  // namespace

// Returns cudaSuccess with *err empty on success; *err set on a parse error.
cudaError_t load_to_graph(Graph* g, const char* text, uint64_t len, const char* relation, uint64_t* node_count,
                          std::string* err) {
    err->clear();
    uint64_t n = 0;
    size_t body = 0;
    if (auto pe = parse_header(std::string_view(text, len), &n, &body)) {
        *err = *pe;
        return cudaSuccess;
    }
    if (n >= 0xFFFFFFFFull) return cudaErrorInvalidValue;
    cudaError_t e = cudaSuccess;
    cudaStream_t s = nullptr;
    char *d_text = nullptr, *d_rel = nullptr;
    uint64_t *d_nl = nullptr, *d_cnt = nullptr, *d_sus = nullptr;
    uint8_t *suspect = nullptr, *keep = nullptr;
    unsigned long long *keys = nullptr, *alt = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    uint64_t nnl = 0, L = 0, m = 0, m_have = 0, nsus = 0;
    std::vector<uint64_t> nl_host;
    std::string first_err;
    uint64_t err_line = ~0ull;
    const uint64_t edges_idx = 2 + n;  // 0-based index of the EDGES line
    auto host_line = [&](uint64_t idx, uint64_t* b, uint64_t* en) -> cudaError_t {
        uint64_t pr[2] = {0, 0};
        if (idx > 0) {
            cudaError_t r = cudaMemcpy(pr, d_nl + idx - 1, idx < nnl ? 16 : 8, cudaMemcpyDeviceToHost);
            if (r) return r;
            *b = pr[0] + 1;
            *en = idx < nnl ? pr[1] : len;
        } else {
            cudaError_t r = nnl ? cudaMemcpy(pr, d_nl, 8, cudaMemcpyDeviceToHost) : cudaSuccess;
            if (r) return r;
            *b = 0;
            *en = nnl ? pr[0] : len;
        }
        return cudaSuccess;
    };
    SNAP_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    SNAP_TRY(cudaMalloc(&d_text, std::max<uint64_t>(len, 1)));
    SNAP_TRY(cudaMemcpyAsync(d_text, text, len, cudaMemcpyHostToDevice, s));
    {
        // '\n' positions: count them first (one pass) to size the array exactly
        SNAP_TRY(cudaMalloc(&d_cnt, 8));
        IsNewline pred{d_text};
        cub::CountingInputIterator<uint64_t> it(0);
        auto flag_it = cub::TransformInputIterator<uint64_t, IsNewline, cub::CountingInputIterator<uint64_t>>(it, pred);
        SNAP_TRY(cub::DeviceReduce::Sum(nullptr, tmp_bytes, flag_it, d_cnt, (int64_t)len, s));
        SNAP_TRY(cudaMallocAsync(&tmp, tmp_bytes, s));
        SNAP_TRY(cub::DeviceReduce::Sum(tmp, tmp_bytes, flag_it, d_cnt, (int64_t)len, s));
        SNAP_TRY(cudaMemcpyAsync(&nnl, d_cnt, 8, cudaMemcpyDeviceToHost, s));
        SNAP_TRY(cudaStreamSynchronize(s));
        cudaFreeAsync(tmp, s);
        tmp = nullptr;
        SNAP_TRY(cudaMalloc(&d_nl, std::max<uint64_t>(nnl, 1) * 8));
        size_t tb2 = 0;
        SNAP_TRY(cub::DeviceSelect::If(nullptr, tb2, it, d_nl, d_cnt, (int64_t)len, pred, s));
        SNAP_TRY(cudaMallocAsync(&tmp, tb2, s));
        SNAP_TRY(cub::DeviceSelect::If(tmp, tb2, it, d_nl, d_cnt, (int64_t)len, pred, s));
        cudaFreeAsync(tmp, s);
        tmp = nullptr;
        // host_line below reads d_nl with plain (legacy-stream) copies
        SNAP_TRY(cudaStreamSynchronize(s));
    }
    L = nnl + ((len > 0 && text[len - 1] != '\n') ? 1 : 0);
    SNAP_TRY(cudaMalloc(&suspect, std::max<uint64_t>(L, 1)));
    SNAP_TRY(cudaMemsetAsync(suspect, 0, std::max<uint64_t>(L, 1), s));
    {
        const uint64_t nodes_have = std::min<uint64_t>(n, L > 2 ? L - 2 : 0);
        LineTab lt{d_nl, nnl, len};
        if (nodes_have) node_lines<<<blocks_for(nodes_have), kTB, 0, s>>>(d_text, lt, 2, nodes_have, suspect);
        SNAP_TRY(cudaGetLastError());
        if (nodes_have < n) {  // EOF inside the node section
            err_line = L + 1;
            first_err = "unexpected end of file in node section";
        } else if (L <= edges_idx) {
            err_line = L + 1;
            first_err = "expected EDGES <count>";
        } else {
            uint64_t b = 0, en = 0;
            SNAP_TRY(host_line(edges_idx, &b, &en));
            const std::string_view line(text + b, en - b);
            if (line.substr(0, 6) != "EDGES ") {
                err_line = edges_idx + 1;
                first_err = "expected EDGES <count>";
            } else if (!whole(line.substr(6), m)) {
                err_line = edges_idx + 1;
                first_err = "bad EDGES count";
            } else {
                const uint64_t first = edges_idx + 1;
                m_have = std::min<uint64_t>(m, L - first);
                SNAP_TRY(cudaMalloc(&keys, std::max<uint64_t>(m_have, 1) * 8));
                SNAP_TRY(cudaMalloc(&alt, std::max<uint64_t>(m_have, 1) * 8));
                SNAP_TRY(cudaMalloc(&keep, std::max<uint64_t>(m_have, 1)));
                const size_t rl = relation ? std::strlen(relation) : 0;
                SNAP_TRY(cudaMalloc(&d_rel, std::max<size_t>(rl, 1)));
                if (rl) SNAP_TRY(cudaMemcpyAsync(d_rel, relation, rl, cudaMemcpyHostToDevice, s));
                if (m_have)
                    edge_lines<<<blocks_for(m_have), kTB, 0, s>>>(d_text, lt, first, m_have, n, d_rel,
                                                                 (uint32_t)rl, relation ? 0 : 1, suspect,
                                                                 keys, keep);
                SNAP_TRY(cudaGetLastError());
                if (m_have < m) {
                    err_line = L + 1;
                    first_err = "unexpected end of file in edge section";
                } else if (L > first + m) {
                    trailing_lines<<<blocks_for(L - first - m), kTB, 0, s>>>(lt, first + m, L - first - m, suspect);
                    SNAP_TRY(cudaGetLastError());
                }
            }
        }
    }
    // suspect lines, ascending: the host decides with the exact rules
    SNAP_TRY(cudaMalloc(&d_sus, std::max<uint64_t>(L, 1) * 8));
    {
        cub::CountingInputIterator<uint64_t> it(0);
        size_t tb2 = 0;
        SNAP_TRY(cub::DeviceSelect::Flagged(nullptr, tb2, it, suspect, d_sus, d_cnt, (int64_t)L, s));
        SNAP_TRY(cudaMallocAsync(&tmp, tb2, s));
        SNAP_TRY(cub::DeviceSelect::Flagged(tmp, tb2, it, suspect, d_sus, d_cnt, (int64_t)L, s));
        cudaFreeAsync(tmp, s);
        tmp = nullptr;
        SNAP_TRY(cudaMemcpyAsync(&nsus, d_cnt, 8, cudaMemcpyDeviceToHost, s));
        SNAP_TRY(cudaStreamSynchronize(s));
    }
    if (nsus) {
        std::vector<uint64_t> sus(nsus);
        SNAP_TRY(cudaMemcpy(sus.data(), d_sus, nsus * 8, cudaMemcpyDeviceToHost));
        for (uint64_t idx : sus) {
            if (idx + 1 >= err_line) break;
            uint64_t b = 0, en = 0;
            SNAP_TRY(host_line(idx, &b, &en));
            const std::string_view line(text + b, en - b);
            std::optional<std::string> le;
            if (idx < edges_idx) le = check_node_line(line, idx - 2);
            else if (idx <= edges_idx + m) le = check_edge_line(line, n, nullptr, nullptr, nullptr);
            else if (!line.empty()) le = std::string("trailing content after edge section");
            if (le) {
                err_line = idx + 1;
                first_err = *le;
                break;
            }
            // a valid exotic line: recover its key for the edge list
            if (idx > edges_idx && idx <= edges_idx + m) {
                uint64_t src = 0, dst = 0;
                std::string_view rel;
                check_edge_line(line, n, &src, &dst, &rel);
                const unsigned long long key = ((unsigned long long)src << 32) | dst;
                const uint8_t kp = (!relation || rel == relation) ? 1 : 0;
                const uint64_t j = idx - edges_idx - 1;
                // on s: ordered before the compaction below
                SNAP_TRY(cudaMemcpyAsync(keys + j, &key, 8, cudaMemcpyHostToDevice, s));
                SNAP_TRY(cudaMemcpyAsync(keep + j, &kp, 1, cudaMemcpyHostToDevice, s));
                SNAP_TRY(cudaStreamSynchronize(s));  // key / kp live on this stack frame
            }
        }
    }
    if (err_line != ~0ull) {
        *err = at_line(err_line, first_err);
        goto done;
    }
    *node_count = n;
    {
        // compact the wanted relation's keys, then sort / unique / CSR + CSC
        uint64_t mk = 0;
        if (m) {
            size_t tb2 = 0;
            SNAP_TRY(cub::DeviceSelect::Flagged(nullptr, tb2, keys, keep, alt, d_cnt, (int64_t)m, s));
            SNAP_TRY(cudaMallocAsync(&tmp, tb2, s));
            SNAP_TRY(cub::DeviceSelect::Flagged(tmp, tb2, keys, keep, alt, d_cnt, (int64_t)m, s));
            cudaFreeAsync(tmp, s);
            tmp = nullptr;
            SNAP_TRY(cudaMemcpyAsync(&mk, d_cnt, 8, cudaMemcpyDeviceToHost, s));
            SNAP_TRY(cudaStreamSynchronize(s));
            std::swap(keys, alt);
        }
        cudaFree(d_text);
        d_text = nullptr;
        g->dg.n = (uint32_t)std::max<uint64_t>(n, 16);  // the store's capacity (graph.cpp:15-30)
        SNAP_TRY(graph_from_keys(g, keys, alt, mk, s));
        SNAP_TRY(locality_relabel(g, s));
    }
done:
    if (tmp) cudaFreeAsync(tmp, s);
    if (s) cudaStreamSynchronize(s);
    cudaFree(d_text);
    cudaFree(d_rel);
    cudaFree(d_nl);
    cudaFree(d_cnt);
    cudaFree(d_sus);
    cudaFree(suspect);
    cudaFree(keep);
    cudaFree(keys);
    cudaFree(alt);
    if (s) cudaStreamDestroy(s);
    return e;
}

}  // namespace snap
}  // namespace mgk
