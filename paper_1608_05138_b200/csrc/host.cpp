// host.cpp -- host-side pieces of the path that are not device work:
//   * edge-list parsing  (load_edge_list, /root/reference/proj/src/graph.cpp:47-91)
//   * synthetic generators (RMAT / G(n,m) / Barabasi-Albert, SPEC "cli" module)
//   * the 128-bit count algebra (global_from_unrestricted, counts.cpp:86-111)
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <mutex>
#include <unordered_set>
#include <vector>

#include "graph.cuh"

namespace gl {

// ------------------------------------------------------------------ device memory pool

namespace {
struct Pool {
    std::mutex mu;
    std::multimap<size_t, std::pair<int, void*>> cached; // size -> (device, ptr)
    size_t cached_bytes = 0;
};
Pool& pool() {
    static Pool* p = new Pool; // never destroyed: blocks may be freed during static teardown
    return *p;
}
constexpr size_t kPoolMaxCached = 96ull << 30;
} // namespace

void* pool_alloc(size_t bytes, int device, size_t* got) {
    bytes = (bytes + 255) & ~size_t(255);
    Pool& P = pool();
    {
        std::lock_guard<std::mutex> lk(P.mu);
        for (auto it = P.cached.lower_bound(bytes); it != P.cached.end() && it->first <= 2 * bytes; ++it) {
            if (it->second.first != device) continue;
            void* p = it->second.second;
            *got = it->first;
            P.cached_bytes -= it->first;
            P.cached.erase(it);
            return p;
        }
    }
    void* p = nullptr;
    static const bool dbg = std::getenv("GL_DEBUG_POOL") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    cudaError_t e = cudaMalloc(&p, bytes);
    if (dbg)
        std::fprintf(stderr, "[gl pool] cudaMalloc %zu B: %.3f ms\n", bytes,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    if (e == cudaErrorMemoryAllocation) { // give the cache back and retry once
        cudaGetLastError();
        pool_trim();
        e = cudaMalloc(&p, bytes);
    }
    cuda_check(e, "cudaMalloc", __FILE__, __LINE__);
    *got = bytes;
    return p;
}

void pool_free(void* p, size_t bytes, int device) {
    Pool& P = pool();
    {
        std::lock_guard<std::mutex> lk(P.mu);
        if (P.cached_bytes + bytes <= kPoolMaxCached) {
            P.cached.emplace(bytes, std::make_pair(device, p));
            P.cached_bytes += bytes;
            return;
        }
    }
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(device);
    cudaFree(p);
    cudaSetDevice(cur);
}

void pool_trim() {
    Pool& P = pool();
    std::lock_guard<std::mutex> lk(P.mu);
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto& kv : P.cached) {
        cudaSetDevice(kv.second.first);
        cudaFree(kv.second.second);
    }
    cudaSetDevice(cur);
    P.cached.clear();
    P.cached_bytes = 0;
}

// ------------------------------------------------------------------ parser

namespace {

inline bool is_sep(char c) { return c == ' ' || c == '\t' || c == '\r'; }

// std::from_chars semantics for an unsigned 64-bit token: digits only,
// no sign, overflow is an error.
bool parse_u64(const char* b, const char* e, u64& out) {
    if (b == e) return false;
    u64 v = 0;
    for (const char* p = b; p < e; ++p) {
        if (*p < '0' || *p > '9') return false;
        u64 d = (u64)(*p - '0');
        if (v > (~0ull - d) / 10) return false;
        v = v * 10 + d;
    }
    out = v;
    return true;
}

} // namespace

// Line-oriented like std::getline: '\n' ends a line, ' ', '\t', '\r'
// separate tokens, '#' and '%' lines are comments, "%%MatrixMarket" arms a
// skip of the next non-comment line (the dimension line).
std::vector<u64> parse_edge_list(const char* text, size_t len) {
    std::vector<u64> out;
    u64 line_no = 0;
    bool skip_dim = false;
    size_t pos = 0;
    while (pos < len) {
        size_t eol = pos;
        while (eol < len && text[eol] != '\n') ++eol;
        ++line_no;
        const char* b = text + pos;
        const char* e = text + eol;
        pos = eol + 1;
        while (b < e && is_sep(*b)) ++b;
        if (b == e) continue;
        if (*b == '#') continue;
        if (*b == '%') {
            static const char kMM[] = "%%MatrixMarket";
            if ((size_t)(e - b) >= sizeof(kMM) - 1 && std::memcmp(b, kMM, sizeof(kMM) - 1) == 0)
                skip_dim = true;
            continue;
        }
        if (skip_dim) {
            skip_dim = false;
            continue;
        }
        const char* tok[3][2];
        int nt = 0;
        const char* p = b;
        while (p < e) {
            while (p < e && is_sep(*p)) ++p;
            if (p >= e) break;
            const char* q = p;
            while (q < e && !is_sep(*q)) ++q;
            if (nt < 3) {
                tok[nt][0] = p;
                tok[nt][1] = q;
            }
            ++nt;
            p = q;
        }
        if (nt != 2)
            throw parse_error(line_no, "expected two integer tokens, got " + std::to_string(nt));
        u64 x, y;
        if (!parse_u64(tok[0][0], tok[0][1], x))
            throw parse_error(line_no, "malformed token '" + std::string(tok[0][0], tok[0][1]) + "'");
        if (!parse_u64(tok[1][0], tok[1][1], y))
            throw parse_error(line_no, "malformed token '" + std::string(tok[1][0], tok[1][1]) + "'");
        out.push_back(x);
        out.push_back(y);
    }
    return out;
}

// The reference's error for one data line (its own text, no '\n'), numbered
// line_no: the device parser (parse.cu) locates the first bad line, this
// formats exactly the message the scanner above would have thrown there.
void throw_line_error(const char* line, size_t len, u64 line_no) {
    const char* b = line;
    const char* e = line + len;
    const char* tok[2][2] = {};
    int nt = 0;
    const char* p = b;
    while (p < e) {
        while (p < e && is_sep(*p)) ++p;
        if (p >= e) break;
        const char* q = p;
        while (q < e && !is_sep(*q)) ++q;
        if (nt < 2) {
            tok[nt][0] = p;
            tok[nt][1] = q;
        }
        ++nt;
        p = q;
    }
    if (nt != 2) throw parse_error(line_no, "expected two integer tokens, got " + std::to_string(nt));
    u64 x;
    if (!parse_u64(tok[0][0], tok[0][1], x))
        throw parse_error(line_no, "malformed token '" + std::string(tok[0][0], tok[0][1]) + "'");
    if (!parse_u64(tok[1][0], tok[1][1], x))
        throw parse_error(line_no, "malformed token '" + std::string(tok[1][0], tok[1][1]) + "'");
    throw parse_error(line_no, "malformed line");
}

std::vector<u64> parse_edge_list_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw io_error("cannot open '" + path + "'");
    std::vector<char> buf((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    return parse_edge_list(buf.data(), buf.size());
}

// ------------------------------------------------------------------ generators

RmatParams make_rmat_params(u32 scale, double a, double b, double c, u64 seed) {
    if (scale == 0 || scale > 40) throw invalid_argument("rmat scale must be in [1, 40]");
    if (a < 0 || b < 0 || c < 0 || a + b + c > 1.0) throw invalid_argument("rmat probabilities invalid");
    RmatParams p;
    p.scale = scale;
    auto th = [](double x) -> u32 {
        double v = x * 4294967296.0;
        if (v >= 4294967295.0) return 0xffffffffu;
        return (u32)v;
    };
    p.ta = th(a);
    p.tb = th(a + b);
    p.tc = th(a + b + c);
    p.seed = seed;
    return p;
}

std::vector<u64> generate_rmat_host(const RmatParams& p, u64 count) {
    std::vector<u64> out(2 * count);
    for (u64 i = 0; i < count; ++i) rmat_edge(p, i, out[2 * i], out[2 * i + 1]);
    return out;
}

namespace {
inline u64 bounded(u64 h, u64 n) { return (u64)(((u128)h * n) >> 64); }
} // namespace

std::vector<u64> generate_gnm(u64 n, u64 m, u64 seed) {
    if (n < 2 && m > 0) throw invalid_argument("G(n,m) needs n >= 2 for m > 0");
    u128 maxm = (u128)n * (n - (n ? 1 : 0)) / 2;
    if ((u128)m > maxm) throw invalid_argument("G(n,m): m exceeds C(n,2)");
    std::vector<u64> out;
    out.reserve(2 * m);
    std::unordered_set<u64> seen;
    seen.reserve(2 * m + 1);
    for (u64 i = 0; out.size() < 2 * m; ++i) {
        u64 a = bounded(hash2(seed, 2 * i), n), b = bounded(hash2(seed, 2 * i + 1), n);
        if (a == b) continue;
        u64 x = a < b ? a : b, y = a < b ? b : a;
        u64 key = n < (1ull << 32) ? (x << 32 | y) : (u64)((u128)x * n + y);
        if (!seen.insert(key).second) continue;
        out.push_back(a);
        out.push_back(b);
    }
    return out;
}

// Barabasi-Albert preferential attachment: vertices 0..k form a clique, every
// later vertex v attaches k distinct targets drawn uniformly from the
// endpoint list (i.e. proportional to degree).
std::vector<u64> generate_ba(u64 n, u32 k, u64 seed) {
    if (k == 0) throw invalid_argument("BA attach must be >= 1");
    std::vector<u64> out;
    if (n == 0) return out;
    u64 n0 = std::min<u64>(n, (u64)k + 1);
    std::vector<u64> ends;
    ends.reserve(2 * ((u64)k * n + n0 * n0));
    out.reserve(2 * ((u64)k * n + n0 * n0 / 2));
    for (u64 a = 0; a < n0; ++a)
        for (u64 b = a + 1; b < n0; ++b) {
            out.push_back(b);
            out.push_back(a);
            ends.push_back(a);
            ends.push_back(b);
        }
    std::vector<u64> picked;
    u64 ctr = 0;
    for (u64 v = n0; v < n; ++v) {
        picked.clear();
        while (picked.size() < k) {
            u64 w = ends[bounded(hash2(seed, ctr++), ends.size())];
            bool dup = false;
            for (u64 p : picked) dup |= (p == w);
            if (!dup) picked.push_back(w);
        }
        for (u64 w : picked) {
            out.push_back(v);
            out.push_back(w);
            ends.push_back(v);
            ends.push_back(w);
        }
    }
    return out;
}

// ------------------------------------------------------------------ algebra

namespace {
u128 choose2(u64 x) { return x < 2 ? 0 : (u128)x * (x - 1) / 2; }
u128 choose3(u64 x) { return x < 3 ? 0 : (u128)x * (x - 1) / 2 * (x - 2) / 3; }
u128 choose4(u64 x) { return x < 4 ? 0 : (u128)x * (x - 1) / 2 * (x - 2) / 3 * (x - 3) / 4; }

u128 exact_div(u128 num, unsigned den, const char* what) {
    if (num % den != 0)
        throw consistency_error(std::string(what) + ": inexact division by " + std::to_string(den));
    return num / den;
}
u128 exact_sub(u128 a, u128 b, const char* what) {
    if (a < b) throw consistency_error(std::string(what) + ": negative intermediate");
    return a - b;
}
} // namespace

// X_1..X_17 from the unrestricted sums; same closed forms and the same
// exactness checks as counts.cpp:86-111 (errata 1-3 of SPEC.md applied there).
void global_from_unrestricted(const u128 c[17], u64 n, u64 m, u128 X[18]) {
    for (int i = 0; i < 18; ++i) X[i] = 0;
    X[1] = m;
    X[2] = exact_sub(choose2(n), m, "X2");
    X[3] = exact_div(c[3], 3, "X3");
    X[4] = exact_div(c[4], 2, "X4");
    X[5] = c[5];
    X[6] = exact_sub(choose3(n), X[3] + X[4] + X[5], "X6");
    X[7] = exact_div(c[7], 6, "X7");
    X[8] = exact_sub(c[8], c[7], "X8");
    X[9] = exact_div(exact_sub(c[9], 4 * X[8], "X9"), 2, "X9");
    X[10] = exact_div(c[10], 4, "X10");
    X[11] = exact_div(exact_sub(c[11], X[9], "X11"), 3, "X11");
    X[12] = exact_sub(c[12], c[10], "X12");
    X[13] = exact_div(exact_sub(c[13], X[9], "X13"), 3, "X13");
    X[14] = exact_div(exact_sub(c[14], 6 * X[7] + 4 * X[8] + 2 * X[9] + 4 * X[10] + 2 * X[12], "X14"), 2,
                      "X14");
    X[15] = exact_div(exact_sub(c[15], 2 * X[12], "X15"), 2, "X15");
    X[16] = exact_sub(c[16], 2 * X[14], "X16");
    u128 conn = 0;
    for (int i = 7; i <= 16; ++i) conn += X[i];
    X[17] = exact_sub(choose4(n), conn, "X17");
}

} // namespace gl
