// parse.cu -- load_edge_list (/root/reference/proj/src/graph.cpp:47-85) on the
// device: the edge-list text is copied to HBM once and cut into lines, classed,
// checked and parsed by one thread per line, so a text input feeds
// gl_graph_build_device without a host parse.
//
// Reference rules (same as the host scanner in host.cpp, pinned by
// tests/golden/parser.json): '\n' ends a line (std::getline); ' ', '\t', '\r'
// separate tokens; a line whose first non-separator is '#' or '%' is a
// comment; "%%MatrixMarket" arms a skip of the next line that is neither blank
// nor a comment (the dimension line); every other line must hold exactly two
// tokens that std::from_chars reads completely as u64 (digits only, no sign,
// no overflow), else parse_error(line, ...) at the FIRST such line.
//
// Passes (L = number of lines):
//   1. newline positions (cub::DeviceSelect::If over the byte indices)
//   2. k_line_class: class of every line (blank/comment, data, MatrixMarket
//      header), its error kind, and an "event" key (i+1)<<1 | is_header for the
//      data and header lines
//   3. inclusive max-scan of the events: a data line is the skipped dimension
//      line iff the closest earlier event is a header
//   4. k_line_keep: keep flags; the lowest kept line with an error is the
//      reference's throw site (atomicMin)
//   5. exclusive sum of the keep flags -> output slots; k_line_emit parses the
//      kept lines a second time straight into their slots (no per-line u64
//      staging: the text is re-read instead, 2 x text bytes of traffic)
#include <cub/cub.cuh>

#include <cstring>
#include <string>
#include <vector>

#include "graph.cuh"

namespace gl {

namespace {

constexpr unsigned char kBlank = 0, kData = 1, kHeader = 2;
constexpr unsigned char kErrNone = 0, kErrTokens = 1, kErrTok0 = 2, kErrTok1 = 3;

__device__ __forceinline__ bool is_sep_d(char c) { return c == ' ' || c == '\t' || c == '\r'; }

struct IsNewline {
    const char* text;
    __device__ __forceinline__ bool operator()(const u64 i) const { return text[i] == '\n'; }
};

struct MaxU64 {
    __device__ __forceinline__ u64 operator()(u64 a, u64 b) const { return a > b ? a : b; }
};

__device__ __forceinline__ void line_bounds(const u64* __restrict__ nl, u64 nnl, u64 len, u64 i, u64& s, u64& e) {
    s = i ? nl[i - 1] + 1 : 0;
    e = i < nnl ? nl[i] : len;
}

// digits only, no sign, no overflow (std::from_chars on the whole token)
__device__ __forceinline__ bool parse_u64_d(const char* b, const char* e, u64& out) {
    if (b == e) return false;
    u64 v = 0;
    for (const char* p = b; p < e; ++p) {
        const char c = *p;
        if (c < '0' || c > '9') return false;
        const u64 d = (u64)(c - '0');
        if (v > (~0ull - d) / 10) return false;
        v = v * 10 + d;
    }
    out = v;
    return true;
}

// tokens of a data line [b, e): count (capped at 3) and the first two
__device__ __forceinline__ int tokens(const char* b, const char* e, const char* tk[2][2]) {
    int nt = 0;
    const char* p = b;
    while (p < e) {
        while (p < e && is_sep_d(*p)) ++p;
        if (p >= e) break;
        const char* q = p;
        while (q < e && !is_sep_d(*q)) ++q;
        if (nt < 2) {
            tk[nt][0] = p;
            tk[nt][1] = q;
        }
        if (++nt > 2) break;
        p = q;
    }
    return nt;
}

__global__ void k_line_class(const char* __restrict__ text, u64 len, const u64* __restrict__ nl, u64 nnl, u64 L,
                             unsigned char* __restrict__ cls, unsigned char* __restrict__ err,
                             u64* __restrict__ ev) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < L; i += (u64)gridDim.x * blockDim.x) {
        u64 s, e;
        line_bounds(nl, nnl, len, i, s, e);
        const char* b = text + s;
        const char* end = text + e;
        while (b < end && is_sep_d(*b)) ++b;
        unsigned char c = kBlank, er = kErrNone;
        if (b < end && *b != '#') {
            if (*b == '%') {
                const char kMM[] = "%%MatrixMarket";
                bool mm = end - b >= 14;
                for (int k = 0; mm && k < 14; ++k) mm = b[k] == kMM[k];
                c = mm ? kHeader : kBlank;
            } else {
                c = kData;
                const char* tk[2][2];
                const int nt = tokens(b, end, tk);
                u64 x;
                if (nt != 2)
                    er = kErrTokens;
                else if (!parse_u64_d(tk[0][0], tk[0][1], x))
                    er = kErrTok0;
                else if (!parse_u64_d(tk[1][0], tk[1][1], x))
                    er = kErrTok1;
            }
        }
        cls[i] = c;
        err[i] = er;
        ev[i] = c == kBlank ? 0ull : ((i + 1) << 1) | (c == kHeader ? 1ull : 0ull);
    }
}

__global__ void k_line_keep(const unsigned char* __restrict__ cls, const unsigned char* __restrict__ err,
                            const u64* __restrict__ evmax, u64 L, u32* __restrict__ keep,
                            unsigned long long* __restrict__ first_err) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < L; i += (u64)gridDim.x * blockDim.x) {
        u32 k = 0;
        if (cls[i] == kData) {
            const bool skipped = i > 0 && (evmax[i - 1] & 1ull); // the dimension line after a header
            if (!skipped) {
                if (err[i] != kErrNone)
                    atomicMin(first_err, (unsigned long long)i);
                else
                    k = 1;
            }
        }
        keep[i] = k;
    }
}

__global__ void k_line_emit(const char* __restrict__ text, u64 len, const u64* __restrict__ nl, u64 nnl, u64 L,
                            const u32* __restrict__ keep, const u32* __restrict__ pos, u64* __restrict__ pairs) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < L; i += (u64)gridDim.x * blockDim.x) {
        if (!keep[i]) continue;
        u64 s, e;
        line_bounds(nl, nnl, len, i, s, e);
        const char* tk[2][2];
        tokens(text + s, text + e, tk);
        u64 x = 0, y = 0;
        parse_u64_d(tk[0][0], tk[0][1], x);
        parse_u64_d(tk[1][0], tk[1][1], y);
        const u64 p = pos[i];
        pairs[2 * p] = x;
        pairs[2 * p + 1] = y;
    }
}

inline unsigned grid_of(u64 n, int sms) {
    u64 g = (n + 255) / 256;
    const u64 cap = (u64)sms * 16;
    return (unsigned)(g < 1 ? 1 : (g > cap ? cap : g));
}

} // namespace

// host.cpp: the reference's message for one bad line (the host scanner on
// that line alone, numbered line_no)
void throw_line_error(const char* line, size_t len, u64 line_no);

// Parse host text on `device`; the pairs stay in *d_pairs (2 x u64 each,
// DevBuf owned by the caller).  Throws parse_error like the reference.
u64 parse_edge_list_device(const char* host_text, u64 len, int device, DevBuf& d_pairs, cudaStream_t s) {
    GL_CUDA(cudaSetDevice(device));
    int sms = 0;
    GL_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    if (len == 0) return 0;
    DevBuf text, nl, nsel, tmp;
    text.alloc(len);
    GL_CUDA(cudaMemcpyAsync(text.p, host_text, len, cudaMemcpyHostToDevice, s));
    const char* dt = text.as<const char>();
    // 1. newline positions
    nsel.alloc(sizeof(u64));
    size_t bytes = 0;
    cub::CountingInputIterator<u64> idx(0);
    // upper bound of the newline count is len; size the output by a first count
    {
        // count newlines first (one DeviceReduce over a transform) to size the list
        auto isnl = cub::TransformInputIterator<u64, IsNewline, cub::CountingInputIterator<u64>>(idx, IsNewline{dt});
        GL_CUDA(cub::DeviceReduce::Sum(nullptr, bytes, isnl, nsel.as<u64>(), (int64_t)len, s));
        tmp.alloc(bytes);
        GL_CUDA(cub::DeviceReduce::Sum(tmp.p, bytes, isnl, nsel.as<u64>(), (int64_t)len, s));
    }
    u64 nnl = 0;
    GL_CUDA(cudaMemcpyAsync(&nnl, nsel.p, sizeof(u64), cudaMemcpyDeviceToHost, s));
    GL_CUDA(cudaStreamSynchronize(s));
    nl.alloc((nnl + 1) * sizeof(u64));
    if (nnl) {
        bytes = 0;
        GL_CUDA(cub::DeviceSelect::If(nullptr, bytes, idx, nl.as<u64>(), nsel.as<u64>(), (int64_t)len, IsNewline{dt}, s));
        tmp.alloc(bytes);
        GL_CUDA(cub::DeviceSelect::If(tmp.p, bytes, idx, nl.as<u64>(), nsel.as<u64>(), (int64_t)len, IsNewline{dt}, s));
    }
    char lastc = 0;
    GL_CUDA(cudaMemcpyAsync(&lastc, dt + len - 1, 1, cudaMemcpyDeviceToHost, s));
    GL_CUDA(cudaStreamSynchronize(s));
    const u64 L = nnl + (lastc != '\n' ? 1 : 0); // getline: no empty line after a final '\n'
    if (L >= (1ull << 32)) throw invalid_argument("edge list has >= 2^32 lines");
    // 2. classes, errors, events
    DevBuf cls, err, ev, keep, pos, ferr;
    cls.alloc(L);
    err.alloc(L);
    ev.alloc(L * sizeof(u64));
    k_line_class<<<grid_of(L, sms), 256, 0, s>>>(dt, len, nl.as<u64>(), nnl, L, cls.as<unsigned char>(),
                                                 err.as<unsigned char>(), ev.as<u64>());
    GL_LAUNCH_CHECK();
    // 3. closest earlier event (in place)
    bytes = 0;
    GL_CUDA(cub::DeviceScan::InclusiveScan(nullptr, bytes, ev.as<u64>(), ev.as<u64>(), MaxU64{}, (int64_t)L, s));
    tmp.alloc(bytes);
    GL_CUDA(cub::DeviceScan::InclusiveScan(tmp.p, bytes, ev.as<u64>(), ev.as<u64>(), MaxU64{}, (int64_t)L, s));
    // 4. keep flags, first error
    keep.alloc((L + 1) * sizeof(u32));
    pos.alloc((L + 1) * sizeof(u32));
    ferr.alloc(sizeof(u64));
    GL_CUDA(cudaMemsetAsync(ferr.p, 0xff, sizeof(u64), s));
    k_line_keep<<<grid_of(L, sms), 256, 0, s>>>(cls.as<unsigned char>(), err.as<unsigned char>(), ev.as<u64>(), L,
                                                keep.as<u32>(), ferr.as<unsigned long long>());
    GL_LAUNCH_CHECK();
    GL_CUDA(cudaMemsetAsync(keep.as<u32>() + L, 0, sizeof(u32), s));
    u64 first_err = 0;
    GL_CUDA(cudaMemcpyAsync(&first_err, ferr.p, sizeof(u64), cudaMemcpyDeviceToHost, s));
    GL_CUDA(cudaStreamSynchronize(s));
    if (first_err != ~0ull) {
        u64 b = 0, e = len;
        if (first_err > 0) GL_CUDA(cudaMemcpy(&b, nl.as<u64>() + first_err - 1, sizeof(u64), cudaMemcpyDeviceToHost));
        if (first_err > 0) ++b;
        if (first_err < nnl) GL_CUDA(cudaMemcpy(&e, nl.as<u64>() + first_err, sizeof(u64), cudaMemcpyDeviceToHost));
        throw_line_error(host_text + b, (size_t)(e - b), first_err + 1);
        throw parse_error(first_err + 1, "malformed line"); // not reached
    }
    // 5. slots, emit
    bytes = 0;
    GL_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, keep.as<u32>(), pos.as<u32>(), (int64_t)(L + 1), s));
    tmp.alloc(bytes);
    GL_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, keep.as<u32>(), pos.as<u32>(), (int64_t)(L + 1), s));
    u32 count = 0;
    GL_CUDA(cudaMemcpyAsync(&count, pos.as<u32>() + L, sizeof(u32), cudaMemcpyDeviceToHost, s));
    GL_CUDA(cudaStreamSynchronize(s));
    d_pairs.alloc(((u64)count + 1) * 2 * sizeof(u64));
    if (count)
        k_line_emit<<<grid_of(L, sms), 256, 0, s>>>(dt, len, nl.as<u64>(), nnl, L, keep.as<u32>(), pos.as<u32>(),
                                                    d_pairs.as<u64>());
    GL_LAUNCH_CHECK();
    GL_CUDA(cudaStreamSynchronize(s)); // the temporaries go back to the (stream-unaware) pool
    return count;
}

} // namespace gl
