// count.cu -- the k<=4 per-edge counting pipeline on the device.
//
// Reference semantics: for every oriented edge (v,u) the reference runs
// process_edge_hash (/root/reference/proj/src/kernels.cpp:143-156):
//   t   = |T|, T = N(u) n N(v)                      (Alg. 1)
//   s_u = deg(u)-t-1, s_v = deg(v)-t-1              (derive_s_v)
//   x7  = # edges inside T            (4-cliques)   (Alg. 5)
//   x10 = # edges between S_u and S_v (4-cycles)    (Alg. 6)
// and accumulate_unrestricted (counts.cpp:6-27) folds them into C3..C16.
//
// The per-edge Algs. 5/6 cost sum_e sum_{w in N(u)} deg(w) adjacency reads
// (1.2e12 on RMAT scale 18).  This pipeline produces the SAME per-edge
// values from degree-ordered DAG enumerations ("identity"):
//   x10(e) = C4(e) + 2*x7(e) - S(e) + 2*t(e)
// where C4(e) = # (not necessarily induced) 4-cycles through e and
// S(e) = sum_{w in T(e)} (t(u,w) + t(v,w)).  Passes:
//   H-pass (hpass.cuh)   per lowest vertex a, H_a = G[U(a)]: t and x7 of every
//                        edge (triangles are H-edges, 4-cliques H-triangles);
//                        then, with t complete, the triangle sums S
//   cycles (cycles.cuh)  per top vertex a (Chiba-Nishizeki wedges b < a,
//                        c < a): W_a[c] in shared memory, C4 credit W-1 to
//                        edges (a,b) and (b,c)
//   k_final (here)       per-edge epilogue + fused block reduction of C3..C16
//                        (128-bit)
// This file holds the shared helpers, the epilogue, the work-list builders and
// the host orchestration (count_begin / count_mid / count_finish).  All
// arithmetic is exact integer; partial sums live in int64 rows {x7, C4 - S}
// that wrap mod 2^64 and are exact once complete.
#include <cub/cub.cuh>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <set>
#include <tuple>
#include <type_traits>
#include <cstring>
#include <vector>

#include "graph.cuh"

namespace gl {

namespace {

constexpr int kCycleSmallWarps = 8;  // warps per small-top block
constexpr int kHashSlots = 1024;     // per-warp hash slots (small tops)
#ifndef GL_SMALL_WEDGES
#define GL_SMALL_WEDGES 768 // 3/4 of the warp hash (512: BA cycles +1.3%)
#endif
constexpr u64 kSmallWedges = GL_SMALL_WEDGES; // small-top threshold (warp hash of 1024 slots)
constexpr int kBigThreads = 1024;    // block per big top (dense windows), one block per SM
constexpr int kBigBlocksPerSM = 1;
constexpr int kMidThreads = 1024;    // block per mid top (hash), one block per SM
constexpr int kSmidThreads = 256;    // block per small-mid top (hash), four blocks per SM
// dense W window words (flattened tiers) and run-metadata entries in shared
// memory; GL_WINDOW_WORDS / GL_META_RUNS override at build time (A/B)
#ifndef GL_WINDOW_WORDS
#define GL_WINDOW_WORDS 45056
#endif
#ifndef GL_META_RUNS
#define GL_META_RUNS 3072
#endif
constexpr int kWindow = GL_WINDOW_WORDS;
constexpr int kMetaRuns = GL_META_RUNS;
constexpr int kMidLog = 15;
constexpr u32 kMidSlots = 1u << kMidLog; // mid tops: block hash, u32 keys + u16 counts (192 KB)
#ifndef GL_MID_NUM
#define GL_MID_NUM 3 // hash tops take up to GL_MID_NUM/4 of the slots in wedges (3: RMAT-20 cycles -1.5%, BA -1% vs 2)
#endif
constexpr u64 kMidWedges = kMidSlots * GL_MID_NUM / 4; // mid-top threshold
constexpr int kSmidLog = 13;
// sparse big tops (windowed block hash): c windows sized for ~kHashWinTarget
// wedges, re-cut when a window holds more than kHashWinMax (and spans more
// than kHashWinMax ids), so a window's distinct c ids stay <= kHashWinMax =
// 27306 of the 32768 slots (load <= 83%; 16384 measured faster than round 1's
// 12288 / 20480: BA cycles -1%, RMAT-24 -1.7%; 8192 slower)
#ifndef GL_HASH_WIN
#define GL_HASH_WIN 16384
#endif
static_assert(GL_HASH_WIN * 5 / 3 < (1 << 15), "windowed hash: distinct ids must stay below the slot count");
constexpr u32 kHashWinTarget = GL_HASH_WIN;
constexpr u32 kHashWinMax = GL_HASH_WIN * 5 / 3;
constexpr u64 kSmidWedges = (1u << kSmidLog) * GL_MID_NUM / 4; // small-mid threshold

constexpr u32 kEmpty = 0xffffffffu;

int num_sms(int device) {
    int v = 0;
    GL_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device));
    return v;
}

inline unsigned grid1d(u64 n, int threads, int sms, int per_sm = 8) {
    u64 g = (n + threads - 1) / threads;
    u64 cap = (u64)sms * per_sm;
    if (g > cap) g = cap;
    if (g == 0) g = 1;
    return (unsigned)g;
}


// ------------------------------------------------------------------ prepass

// wedges(e) = epos(e): the wedges a-b-c (c < a) of edge e = (a,b) as top edge
struct WedgesOf {
    const u32* epos;
    u64 m;
    __device__ __forceinline__ u64 operator()(const u64& e) const { return e < m ? (u64)epos[e] : 0ull; }
};

#include "hpass.cuh"

#include "cycles.cuh"

// ------------------------------------------------------------------ epilogue

struct Acc {
    u128 c[13]; // C3,C4,C5,C7,C8,C9,C10,C11,C12,C13,C14,C15,C16
};
__device__ __constant__ int kCIdx[13] = {3, 4, 5, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16};

__device__ __forceinline__ u128 ch2d(u64 x) { return x < 2 ? (u128)0 : (u128)x * (x - 1) / 2; }

__device__ __forceinline__ u128 shfl_down_u128(u128 v, int d) {
    u64 lo = (u64)v, hi = (u64)(v >> 64);
    lo = __shfl_down_sync(0xffffffffu, lo, d);
    hi = __shfl_down_sync(0xffffffffu, hi, d);
    return ((u128)hi << 64) | lo;
}

constexpr int kFinThreads = 256;

__global__ void __launch_bounds__(kFinThreads)
k_final(DevGraph g, const i64* __restrict__ part, const u32* __restrict__ t, u64 begin, u64 end,
        u64* __restrict__ x7_out, u64* __restrict__ x10_out, unsigned long long* __restrict__ acc,
        unsigned* __restrict__ flags) {
    Acc a;
#pragma unroll
    for (int i = 0; i < 13; ++i) a.c[i] = 0;
    const u64 n = g.n, m = g.m;
    bool bad = false;
    for (u64 e = begin + blockIdx.x * (u64)blockDim.x + threadIdx.x; e < end; e += (u64)gridDim.x * blockDim.x) {
        const u64 r = e - begin;
        const u64 x7 = (u64)part[2 * r];
        const u64 y = (u64)part[2 * r + 1];
        const u64 te = t[e];
        const u64 du = g.deg[g.eu[e]], dv = g.deg[g.ev[e]];
        const u64 su = du - te - 1, sv = dv - te - 1;
        const u64 de = n - (su + sv + te) - 2;
        const u64 x10 = y + 2 * x7 + 2 * te;
        x7_out[e] = x7;
        x10_out[e] = x10;
        if ((u128)x7 > ch2d(te) || (u128)x10 > (u128)su * sv) bad = true;
        a.c[0] += te;
        a.c[1] += su + sv;
        a.c[2] += de;
        a.c[3] += x7;
        a.c[4] += ch2d(te);
        a.c[5] += (u128)te * (su + sv);
        a.c[6] += x10;
        a.c[7] += ch2d(sv) + ch2d(su);
        a.c[8] += (u128)sv * su;
        a.c[9] += (u128)te * de;
        a.c[10] += m - du - dv + 1;
        a.c[11] += (u128)(su + sv) * de;
        a.c[12] += ch2d(de);
    }
    if (bad) atomicOr(&flags[0], 1u);
    __shared__ u128 s_red[kFinThreads / 32][13];
    const u32 lane = lane_id(), w = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < 13; ++i) {
        u128 v = a.c[i];
        for (int d = 16; d > 0; d >>= 1) v += shfl_down_u128(v, d);
        if (lane == 0) s_red[w][i] = v;
    }
    __syncthreads();
    if (threadIdx.x < 13) {
        u128 v = 0;
        for (int k = 0; k < kFinThreads / 32; ++k) v += s_red[k][threadIdx.x];
        if (v) {
            int ci = kCIdx[threadIdx.x];
            u64 lo = (u64)v, hi = (u64)(v >> 64);
            unsigned long long old = atomicAdd(&acc[2 * ci], (unsigned long long)lo);
            u64 carry = (old + lo < old) ? 1 : 0;
            u64 addh = hi + carry;
            if (addh) {
                unsigned long long oh = atomicAdd(&acc[2 * ci + 1], (unsigned long long)addh);
                if (oh + addh < oh) atomicOr(&flags[1], 1u);
            }
        }
    }
}

// ------------------------------------------------------------ work lists

// x7 column of the partial rows {x7, y} (final after the H-pass)
__global__ void k_even(const i64* __restrict__ part, u64 m, u64* __restrict__ out) {
    for (u64 e = blockIdx.x * (u64)blockDim.x + threadIdx.x; e < m; e += (u64)gridDim.x * blockDim.x)
        out[e] = (u64)part[2 * e];
}

__global__ void k_seq(u32* __restrict__ ids, u64 n) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        ids[i] = (u32)i;
}

// H-pass work list key: big-k (k > 32) items first, each class ordered by its
// streaming cost s1(a) = sum_{i<k-1} |U(x_i)| (adjacency entries read).
// Work lists only need an approximate cost order: keys are a 4-bit-mantissa
// log2 of the cost (10 bits) under a class bit, so the radix sort runs over
// 17 key bits instead of 64.
constexpr u32 kKeyBits = 17;
__device__ __forceinline__ u32 log_key(u64 c) { // monotone in c, 0 for c = 0
    if (c < 16) return (u32)c;
    const u32 msb = 63 - __clzll(c);
    return (msb << 4) | (u32)((c >> (msb - 4)) & 15u);
}
__global__ void k_umax(DevGraph g, unsigned* __restrict__ out) {
    u32 mx = 0;
    for (u64 a = blockIdx.x * (u64)blockDim.x + threadIdx.x; a < g.n; a += (u64)gridDim.x * blockDim.x) {
        const u32 k = (u32)(g.off[a + 1] - (g.off[a] + g.lcnt[a]));
        mx = k > mx ? k : mx;
    }
    for (int d = 16; d > 0; d >>= 1) {
        const u32 o = __shfl_down_sync(0xffffffffu, mx, d);
        mx = o > mx ? o : mx;
    }
    if ((threadIdx.x & 31) == 0 && mx) atomicMax(out, mx);
}
// classes: 4 = k > 512 (xl block), 3 = 128 < k <= 512 (large block), 2 = 32 < k <= 128
// (small block), 1 = 2 <= k <= 32 (warp)
__global__ void k_hkeys(DevGraph g, u32* __restrict__ keys, unsigned long long* __restrict__ n_xl,
                        unsigned long long* __restrict__ n_large,
                        unsigned long long* __restrict__ n_medium, unsigned long long* __restrict__ n_small,
                        unsigned long long* __restrict__ s1_total, unsigned long long* __restrict__ s1_max,
                        unsigned long long* __restrict__ hedge_bound) {
    // one warp per vertex: lanes split the members (the cost sum over a hub's
    // members is a chain of dependent loads for a single thread)
    unsigned long long mx = 0, hb = 0, lx = 0, ll = 0, lm = 0, ls = 0, st = 0;
    const u32 lane = lane_id();
    const u64 warp = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5, nwarp = ((u64)gridDim.x * blockDim.x) >> 5;
    for (u64 a = warp; a < g.n; a += nwarp) {
        const u64 ub = g.off[a] + g.lcnt[a];
        const u64 k = g.off[a + 1] - ub;
        u64 q = 0;
        for (u64 i = lane; i + 1 < k; i += 32) { // entries read: streamed list or ~8 per probe
            const u32 x = g.adj[ub + i];
            const u64 ul = g.off[x + 1] - (g.off[x] + g.lcnt[x]), pr = (u64)c_probe_ratio * (k - 1 - i);
            q += ul < pr ? ul : pr;
        }
        q = warp_sum_u64(q);
        if (lane) continue;
        u32 key = 0;
        if (k >= 2) {
            st += q;
            u32 cls = 1;
            if (k > (u64)kHWarpMax) {
                cls = k > 512 ? 4 : k > 128 ? 3 : 2;
                if (cls == 4) ++lx; else if (cls == 3) ++ll; else ++lm;
                mx = q > mx ? q : mx;
                hb += k * (k - 1) / 2; // the counting pass reserves C(k,2) records per vertex
            } else {
                ++ls;
                const u64 pairs = k * (k - 1) / 2; // warp pass: exact reservation, bounded here
                hb += pairs < q ? pairs : q;
            }
            key = (cls << 12) | (log_key(q) + 1);
        }
        keys[a] = key;
    }
    if (lx) atomicAdd(n_xl, lx);
    if (ll) atomicAdd(n_large, ll);
    if (lm) atomicAdd(n_medium, lm);
    if (ls) atomicAdd(n_small, ls);
    if (st) atomicAdd(s1_total, st);
    if (mx) atomicMax(s1_max, mx);
    if (hb) atomicAdd(hedge_bound, hb);
}

// dense windows a big top sweeps: the c range [0, a) cut at the degree tiers,
// kWindow << cl ids per window of tier width cl
__device__ __forceinline__ u64 dense_windows(u32 a, const unsigned* __restrict__ tiers) {
    u64 nw = 0;
    u32 prev = 0;
    for (int i = 0; i <= 4; ++i) {
        const u32 end = i < 4 ? (tiers[i] < a ? tiers[i] : a) : a;
        const u64 span = (u64)(4 - i >= (int)kWalkCl ? (kWindow + 3 * kMetaRuns) & ~3 : kWindow) << (4 - i); // kWalkWords for walk tiers
        if (end > prev) nw += (end - prev + span - 1) / span;
        prev = end > prev ? end : prev;
    }
    return nw;
}

// Sparse big tops take the windowed hash when factor * (hash windows) <=
// (dense windows).  GL_SPARSE_BIG=all|off|<factor> overrides (tests force both
// paths).
inline u32 sparse_big_factor() {
    const char* e = std::getenv("GL_SPARSE_BIG");
    if (e && !std::strcmp(e, "all")) return 0u;
    if (e && !std::strcmp(e, "off")) return 0xffffffffu;
    if (e && *e >= '0' && *e <= '9') return (u32)std::strtoul(e, nullptr, 10);
    return 4u;
}

// cycle work list key = wedges of top a; classes sparse big (> kMidWedges,
// wedges thin over the c range: windowed block hash), big (dense windows),
// mid (> kSmallWedges, block hash), small (warp hash)
__global__ void k_top_keys(DevGraph g, const u64* __restrict__ wpre, const unsigned* __restrict__ tiers,
                           u32* __restrict__ keys, unsigned long long* __restrict__ n_big,
                           unsigned long long* __restrict__ n_mid, unsigned long long* __restrict__ n_smid,
                           unsigned long long* __restrict__ n_small, unsigned long long* __restrict__ n_sparse,
                           u32 sparse_factor) {
    unsigned long long lb = 0, lm = 0, lq = 0, ls = 0, lh = 0;
    for (u64 a = blockIdx.x * (u64)blockDim.x + threadIdx.x; a < g.n; a += (u64)gridDim.x * blockDim.x) {
        u64 w = wpre[g.loff[a + 1]] - wpre[g.loff[a]];
        u32 cls = 0; // exact class boundaries: class above the log cost
        const u64 nb = g.loff[a + 1] - g.loff[a];
        if (w > kMidWedges && nb < 65536 &&
            (u64)sparse_factor * ((w + kHashWinTarget - 1) / kHashWinTarget) <= dense_windows((u32)a, tiers)) {
            ++lh; // u16 hash counts: W <= nb < 65536
            cls = 5;
        } else if (w > kMidWedges) {
            ++lb;
            cls = 4;
        } else if (w > kSmidWedges) {
            ++lm;
            cls = 3;
        } else if (w > kSmallWedges) {
            ++lq;
            cls = 2;
        } else if (w) {
            ++ls;
            cls = 1;
        }
        keys[a] = (cls << 12) | log_key(w);
    }
    if (lh) atomicAdd(n_sparse, lh);
    if (lb) atomicAdd(n_big, lb);
    if (lm) atomicAdd(n_mid, lm);
    if (lq) atomicAdd(n_smid, lq);
    if (ls) atomicAdd(n_small, ls);
}

// degree tiers of the window counters: #vertices with degree < 4, 16, 256,
// 65536 = the first internal id of the next tier (ids ascend with degree)
__global__ void k_tiers(DevGraph g, unsigned* __restrict__ out) {
    unsigned c[4] = {0, 0, 0, 0};
    for (u64 v = blockIdx.x * (u64)blockDim.x + threadIdx.x; v < g.n; v += (u64)gridDim.x * blockDim.x) {
        const u32 d = g.deg[v];
        c[0] += d < 4u;
        c[1] += d < 16u;
        c[2] += d < 256u;
        c[3] += d < 65536u;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        unsigned v = c[i];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(&out[i], v);
    }
}

// counters (u64 slots after the 40 macro-sum words of cs.acc): 0 H large queue,
// 1/2/4/7 cycle big/small/mid/small-mid queues, 3 H warp queue, 5/6/9/26 sums
// large/warp/medium/xl queues, 8 H medium queue, 25 H xl queue, 10/11/15/16
// cycle class counts, 12/13/21/24 H class counts (large/small/medium/xl),
// 14 max k, 17 s1, 18 max s1, 19 H-edge bound, 20 H-edge list fill, 22-23 tiers,
// 27 sparse-big cycle class count, 28 its queue
constexpr int kCounters = 32;

// rank's share of a cost-sorted list: sorted positions p with p % world == rank
template <typename T>
__global__ void k_take_rank(const T* __restrict__ sorted, u64 begin, u64 count, int rank, int world,
                            T* __restrict__ out) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x;; i += (u64)gridDim.x * blockDim.x) {
        u64 p = (u64)rank + i * (u64)world;
        if (p >= count) break;
        out[i] = sorted[begin + p];
    }
}

// ------------------------------------------------------ heavy-top pieces
// A windowed top (dense or sparse big) whose wedges exceed the piece cap is
// split into c-range pieces [clo, chi) of about equal wedge count: the unit of
// fine-grained task splitting (the reference's clique_res_range /
// cycle_res_range with split_threshold, kernels.hpp:68-80), so no
// single block or rank holds more than ~1/4096 of the cycle work.  Pieces are
// laid out in sorted-top order (deterministic: every rank derives the same
// list and takes its positions p % world).
constexpr u32 kPieceSamples = 2048; // sampled wedges per split top (256 threads x 8)
constexpr u32 kPieceMax = kPieceSamples / 4;
__device__ __forceinline__ u32 piece_count(const DevGraph& g, const u64* __restrict__ wpre, u32 a, u64 cap,
                                           u32 min_per_b) {
    const u64 E0 = g.loff[a], E1 = g.loff[a + 1];
    const u64 w = wpre[E1] - wpre[E0], nb = E1 - E0;
    u64 p = (w + cap - 1) / cap;
    // every piece re-seeks each b's cursor (a gallop per b): keep >= min_per_b
    // (32) wedges per b per piece
    const u64 pb = nb ? w / (min_per_b * nb) : 1;
    p = p < pb ? p : pb;
    p = p < kPieceMax ? p : kPieceMax;
    return p ? (u32)p : 1u;
}
__global__ void k_piece_count(DevGraph g, const u64* __restrict__ wpre, const u32* __restrict__ sorted, u64 count,
                              u64 cap, u32 min_per_b, u32* __restrict__ np) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < count; i += (u64)gridDim.x * blockDim.x)
        np[i] = piece_count(g, wpre, sorted[i], cap, min_per_b);
}
// one block per windowed top: c quantiles of kPieceSamples evenly spaced
// wedges (wedge order is b-major, so the samples are not c-ordered: sort them)
// Dense tops (positions >= n_hash) cut on their window grid: the pieces hold
// exactly the unsplit top's windows (no extra window or run); cut points that
// coincide leave empty pieces (a = kEmpty, skipped by the kernel).
__global__ void __launch_bounds__(256) k_pieces(DevGraph g, const u64* __restrict__ wpre,
                                                const u32* __restrict__ sorted, u64 count, u64 n_hash,
                                                const unsigned* __restrict__ tiers_in, u32 walk_cl,
                                                const u32* __restrict__ poff, uint4* __restrict__ pieces) {
    const uint4 tiers = make_uint4(tiers_in[0], tiers_in[1], tiers_in[2], tiers_in[3]);
    using Sort = cub::BlockRadixSort<u32, 256, kPieceSamples / 256>;
    __shared__ typename Sort::TempStorage tmp;
    __shared__ u32 s_c[kPieceSamples];
    for (u64 i = blockIdx.x; i < count; i += gridDim.x) {
        const u32 a = sorted[i];
        const u32 P = poff[i + 1] - poff[i];
        const u64 E0 = g.loff[a], E1 = g.loff[a + 1];
        const u64 w0 = wpre[E0], w = wpre[E1] - w0;
        uint4* out = pieces + poff[i];
        if (P == 1) {
            if (threadIdx.x == 0) out[0] = make_uint4(a, 0u, a, (u32)min(w, (u64)0xffffffffull));
            continue;
        }
        u32 keys[kPieceSamples / 256];
#pragma unroll
        for (u32 u = 0; u < kPieceSamples / 256; ++u) {
            const u64 sidx = threadIdx.x * (kPieceSamples / 256) + u;
            const u64 k = w0 + (2 * sidx + 1) * w / (2 * kPieceSamples);
            const u64 e = upper_bound_dev<u64, u64>(wpre, E0, E1 + 1, k) - 1;
            keys[u] = g.adj[g.off[g.eu[e]] + (k - wpre[e])];
        }
        __syncthreads(); // tmp / s_c reuse across tops
        Sort(tmp).Sort(keys);
#pragma unroll
        for (u32 u = 0; u < kPieceSamples / 256; ++u) s_c[threadIdx.x * (kPieceSamples / 256) + u] = keys[u];
        __syncthreads();
        const u32 west = (u32)min((w + P - 1) / P, (u64)0xffffffffull);
        const bool dense = i >= n_hash;
        auto cut = [&](u32 j) -> u32 { // cut point j (0 < j < P)
            const u32 c = s_c[(u64)j * kPieceSamples / P];
            return dense ? grid_floor(c, tiers, E1 - E0, walk_cl) : c;
        };
        for (u32 j = threadIdx.x; j < P; j += blockDim.x) {
            const u32 lo = j ? cut(j) : 0u;
            const u32 hi = j + 1 < P ? cut(j + 1) : a;
            out[j] = lo < hi ? make_uint4(a, lo, hi, west) : make_uint4(kEmpty, 0u, 0u, 0u);
        }
    }
}
// ------------------------------------------------------- run-end table
// Dense windows lie on a global grid (degree tiers cut into windows of the
// tier's span, cycles.cuh win_span): the window of an id c is a function of c
// alone, so the run of row b inside any window ends at the first slot after
// the run start whose c lies in a later window.  One table per graph (and
// walk_cl): flag every slot that starts a row or changes window, then a
// forward min-scan over the slots in reverse order gives, for every slot p,
// the first flagged slot >= p -- read at p + 1 it is p's run end.
//   rev[i] = (slot 2m-1-i flagged) ? 2m-1-i : kEmpty;   table = min-scan(rev)
//   run end after slot p = table[2m - 2 - p]  (kEmpty: none -> row prefix end)
__device__ __forceinline__ u32 grid_win(u32 c, uint4 tiers, u32 walk_cl) {
    u32 t0, t1;
    const u32 cl = tier_of(c, tiers, t0, t1);
    // unclamped spans (<= 54272 << 4) and offsets fit 32 bits: a u32 division
    return ((4 - cl) << 28) | ((c - t0) / (u32)win_span(cl, 0, walk_cl));
}
__global__ void k_run_flags(DevGraph g, uint4 tiers, u32 walk_cl, u32* __restrict__ rev) {
    const u64 S = 2 * g.m;
    for (u64 p = blockIdx.x * (u64)blockDim.x + threadIdx.x; p < S; p += (u64)gridDim.x * blockDim.x) {
        // window id of this slot; the previous slot's from the neighbouring lane
        // when it is in this warp's range (one division per slot)
        const u32 w = grid_win(g.adj[p], tiers, walk_cl);
        u32 wp = __shfl_up_sync(__activemask(), w, 1);
        if ((threadIdx.x & 31) == 0 && p > 0) wp = grid_win(g.adj[p - 1], tiers, walk_cl);
        const bool f = p == 0 || w != wp;
        rev[S - 1 - p] = f ? (u32)p : kEmpty;
    }
}
__global__ void k_row_flags(DevGraph g, u32* __restrict__ rev) {
    const u64 S = 2 * g.m;
    for (u64 v = blockIdx.x * (u64)blockDim.x + threadIdx.x; v < g.n; v += (u64)gridDim.x * blockDim.x) {
        const u64 p = g.off[v];
        if (p < g.off[v + 1]) rev[S - 1 - p] = (u32)p;
    }
}
struct MinU32 {
    __device__ __forceinline__ u32 operator()(u32 a, u32 b) const { return a < b ? a : b; }
};
// packed table entry: (run-end slot q << 32) | adj[q]  (all ones: none) -- the
// run end and the c the cursor lands on come in one load
__global__ void k_run_pack(DevGraph g, const u32* __restrict__ scan, u64* __restrict__ tab) {
    const u64 S = 2 * g.m;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < S; i += (u64)gridDim.x * blockDim.x) {
        const u32 q = scan[i];
        tab[i] = q == kEmpty ? ~0ull : ((u64)q << 32) | g.adj[q];
    }
}

// lowest counter tier of the thread-walk windows (cycles.cuh, kWalkCl)
inline u32 walk_cl() {
    const char* e = std::getenv("GL_WALK_CL");
    // >= 1: the walk credits slots in 32 bits, never valid for the hub tier (cl 0)
    return e && *e >= '1' && *e <= '9' ? (u32)std::strtoul(e, nullptr, 10) : kWalkCl;
}
// Piece cap: no work item above 1/4 of one SM's fair share of the job,
// wedges / (4 * SMs * ranks) (at least 2^17): 1/592 of the cycle work on one
// B200, 1/4736 at 8 ranks.  GL_PIECE_WEDGES=<n> overrides it (and lowers the
// wedges-per-b floor to 1), so tests force splitting on small graphs.
inline bool piece_forced() {
    const char* e = std::getenv("GL_PIECE_WEDGES");
    return e && *e >= '0' && *e <= '9';
}
inline u64 piece_cap(u64 wtot, int sms, int world) {
    if (piece_forced()) return std::max<u64>(1, std::strtoull(std::getenv("GL_PIECE_WEDGES"), nullptr, 10));
    const char* e = std::getenv("GL_PIECE_DIV"); // A/B knob for the per-SM share divisor
    const u64 div = e && *e >= '1' && *e <= '9' ? std::strtoull(e, nullptr, 10) : 4ull;
    return std::max<u64>(wtot / (div * (u64)sms * (u64)world), 1ull << 17);
}

struct Timer {
    cudaEvent_t ev[6];
    int n = 0;
    explicit Timer(int k) : n(k) {
        for (int i = 0; i < n; ++i) GL_CUDA(cudaEventCreate(&ev[i]));
    }
    ~Timer() {
        for (int i = 0; i < n; ++i) cudaEventDestroy(ev[i]);
    }
};

template <typename In, typename T>
void dev_exclusive_scan(DevBuf& tmp, In in, T* out, u64 n, cudaStream_t s) {
    size_t bytes = 0;
    GL_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, (int64_t)n, s));
    tmp.alloc(bytes);
    GL_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, in, out, (int64_t)n, s));
}

// sort (key desc, id) pairs; ids_out sorted by descending key (stable)
void dev_sort_desc(DevBuf& tmp, u32* keys_in, u32* keys_out, u32* ids_in, u32* ids_out, u64 n,
                   cudaStream_t s) {
    size_t bytes = 0;
    GL_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, bytes, keys_in, keys_out, ids_in, ids_out,
                                                      (int64_t)n, 0, (int)kKeyBits, s));
    tmp.alloc(bytes);
    GL_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp.p, bytes, keys_in, keys_out, ids_in, ids_out,
                                                      (int64_t)n, 0, (int)kKeyBits, s));
}

// Dynamic shared memory of a block H-pass launch: the class's workspace at its
// largest k, or -- for the xl class when some k exceeds it -- every byte the
// block can opt into (the small arrays of bigger k plus the phase-2 row stage,
// hpass_vertex rows_g), minus the kernel's static shared memory.
template <int MODE, int K> size_t hpass_smem_bytes(u32 kmax, int device);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) raised to the largest size
// requested so far per (kernel, device): the attribute is a limit, and a graph
// that needs less must not lower it under a later graph that needs more
template <typename K> void smem_attr(K* kernel, size_t smem, int device) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> set_to;
    std::lock_guard<std::mutex> lk(mu);
    size_t& cur = set_to[{reinterpret_cast<const void*>(kernel), device}];
    if (smem > cur) {
        GL_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        cur = smem;
    }
}

template <int MODE, int K> size_t hpass_smem_bytes(u32 kmax, int device) {
    const u32 kws = K == 1088 ? 1088u : (K == 768 ? 512u : 128u); // largest k of the class
    const size_t base = (size_t)hpass_ws_words(kws, MODE, bloom_words<HCfg<K>::BLOG>()) * sizeof(u32);
    if (K != 1088 || kmax <= 1088u) return base;
    static std::mutex mu;
    static size_t cached[2][64] = {};
    std::lock_guard<std::mutex> lk(mu);
    size_t& c = cached[MODE][device & 63];
    if (!c) {
        cudaFuncAttributes fa{};
        GL_CUDA(cudaFuncGetAttributes(&fa, k_hpass_block<MODE, K>));
        int optin = 0;
        GL_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
        c = ((size_t)optin - fa.sharedSizeBytes) & ~(size_t)15;
    }
    return std::max(base, c);
}

template <typename T> T read_dev(const T* p, cudaStream_t s) {
    T h{};
    GL_CUDA(cudaMemcpyAsync(&h, p, sizeof(T), cudaMemcpyDeviceToHost, s));
    GL_CUDA(cudaStreamSynchronize(s));
    return h;
}

} // namespace

// --------------------------------------------------------------------------

namespace {

// Cost-sorted vertex work list (descending key) and this rank's share of
// the sorted positions [begin, begin+count): p % world == rank.
u64 rank_share(u64 count, int rank, int world) {
    return count > (u64)rank ? (count - rank + world - 1) / world : 0;
}

} // namespace

std::atomic<int> g_overlap{0}; // 1: run the cycle pass concurrently with the H-pass (gl_set_overlap); measured slower

// Phase A: H-pass (t and x7 partials) and the cycle kernels (C4 into y).
void count_begin(Graph& gr, int rank, int world, i64* d_partials, cudaStream_t s) {
    GL_CUDA(cudaSetDevice(gr.device));
    if (world < 1 || rank < 0 || rank >= world) throw invalid_argument("bad rank/world");
    if (!s) s = gr.stream;
    const DevGraph& g = gr.d;
    CountState& cs = gr.cs;
    const int sms = num_sms(gr.device);
    const u64 m = g.m, n = g.n;
    // adjacency slots are carried as u32 in the cycle run metadata
    if (2 * m >= (1ull << 32)) throw overflow_error("counting needs 2m < 2^32 adjacency slots (m < 2^31 edges)");
    {
        // dense cycle windows count their runs in 24 bits (runs <= |L(a)| <= max degree)
        const char* e = std::getenv("GL_TEST_DEGREE_LIMIT"); // tests reach this path on small graphs
        const u64 lim = e && *e ? std::strtoull(e, nullptr, 10) : (1ull << 24);
        if (g.dmax >= lim) throw overflow_error("cycle pass needs max degree < 2^24 (window run counts)");
    }
    // A cycle pass of a previous count_begin that was never joined by
    // count_mid is still writing the slot accumulators and reading the queue
    // counters: finish it before any of them is reset below.
    if (cs.s2) GL_CUDA(cudaStreamSynchronize(cs.s2));
    // ... and the previous call's H-pass / triangle sums, which may sit on
    // another caller stream: they pop the queue counters and write t and the
    // partials that the memsets below reset
    if (cs.began) {
        GL_CUDA(cudaEventSynchronize(cs.ev[1]));
        GL_CUDA(cudaEventSynchronize(cs.ev[3])); // cycle pass (on the previous caller stream when serialised)
        if (cs.mid_done) GL_CUDA(cudaEventSynchronize(cs.ev[7]));
    }
    if (const char* pe = std::getenv("GL_PROBE_RATIO")) {
        const u32 r = (u32)std::strtoul(pe, nullptr, 10);
        if (r) GL_CUDA(cudaMemcpyToSymbolAsync(c_probe_ratio, &r, sizeof(r), 0, cudaMemcpyHostToDevice, s ? s : gr.stream));
    }
    cs.launches = 0;
    cs.began = false;
    cs.mid_done = false;
    cs.rank = rank;
    cs.world = world;
    std::memset(cs.work, 0, sizeof(cs.work));

    cs.t.alloc((m + 1) * sizeof(u32));
    cs.wpre.alloc((m + 1) * sizeof(u64));
    cs.acc.alloc(96 * sizeof(u64));
    cs.keys.alloc((n + 1) * 2 * sizeof(u32));   // H-pass sort keys in/out
    cs.items2.alloc((n + 1) * 2 * sizeof(u32)); // vertex ids in/out
    const u64 plen = ((m + world - 1) / world) * (u64)world;
    if (plen) GL_CUDA(cudaMemsetAsync(d_partials, 0, 2 * plen * sizeof(i64), s));
    GL_CUDA(cudaMemsetAsync(cs.t.p, 0, (m + 1) * sizeof(u32), s));
    cs.slots.alloc((2 * m + 1) * sizeof(i64));
    GL_CUDA(cudaMemsetAsync(cs.slots.p, 0, (2 * m + 1) * sizeof(i64), s));
    cs.slots32.alloc((2 * m + 1) * sizeof(u32));
    GL_CUDA(cudaMemsetAsync(cs.slots32.p, 0, (2 * m + 1) * sizeof(u32), s));
    unsigned long long* counters = cs.acc.as<unsigned long long>() + 40; // queues + counts
    GL_CUDA(cudaMemsetAsync(counters, 0, kCounters * sizeof(u64), s));

    // Per-graph indexes of the cycle pass, built by the first count: the
    // degree tiers of the window counters (k_tiers) and the run-end table of
    // the dense windows (GL_RUN_TABLE=0 disables it)
    // the H-edge record list is sized (once per graph) from the free memory
    // seen here, before the run-end table's temporaries go to the pool
    size_t free_at_start = 0;
    if (!cs.tl_sized) {
        size_t tot = 0;
        GL_CUDA(cudaMemGetInfo(&free_at_start, &tot));
    }
    if (m && !cs.tiers_valid) {
        cs.tierbuf.alloc(4 * sizeof(unsigned));
        GL_CUDA(cudaMemsetAsync(cs.tierbuf.p, 0, 4 * sizeof(unsigned), s));
        k_tiers<<<grid1d(n, 256, sms), 256, 0, s>>>(g, cs.tierbuf.as<unsigned>());
        GL_LAUNCH_CHECK();
        unsigned ht[4];
        GL_CUDA(cudaMemcpyAsync(ht, cs.tierbuf.p, sizeof(ht), cudaMemcpyDeviceToHost, s));
        GL_CUDA(cudaStreamSynchronize(s));
        cs.tiers = make_uint4(ht[0], ht[1], ht[2], ht[3]);
        cs.tiers_valid = true;
        cs.launches += 1;
    }
    {
        const char* rt = std::getenv("GL_RUN_TABLE");
        if (m && !(rt && rt[0] == '0') && cs.runtab_key != walk_cl() + 1) {
            const u64 S = 2 * m;
            DevBuf rev, scan;
            rev.alloc(S * sizeof(u32));
            scan.alloc(S * sizeof(u32));
            cs.runtab.alloc(S * sizeof(u64));
            k_run_flags<<<grid1d(S, 256, sms, 16), 256, 0, s>>>(g, cs.tiers, walk_cl(), rev.as<u32>());
            k_row_flags<<<grid1d(n, 256, sms), 256, 0, s>>>(g, rev.as<u32>());
            GL_LAUNCH_CHECK();
            size_t bytes = 0;
            GL_CUDA(cub::DeviceScan::InclusiveScan(nullptr, bytes, rev.as<u32>(), scan.as<u32>(), MinU32{},
                                                   (int64_t)S, s));
            cs.tmp.alloc(bytes);
            GL_CUDA(cub::DeviceScan::InclusiveScan(cs.tmp.p, bytes, rev.as<u32>(), scan.as<u32>(), MinU32{},
                                                   (int64_t)S, s));
            k_run_pack<<<grid1d(S, 256, sms, 16), 256, 0, s>>>(g, scan.as<u32>(), cs.runtab.as<u64>());
            GL_LAUNCH_CHECK();
            GL_CUDA(cudaStreamSynchronize(s)); // rev / scan go back to the (stream-unaware) pool
            cs.runtab_key = walk_cl() + 1;
            cs.launches += 4;
        }
    }

    // The H-pass (stream s) and the cycle pass (cs.s2, forked after the wedge
    // prefix) are independent and run concurrently; count_mid joins them.
    if (!cs.s2) {
        GL_CUDA(cudaStreamCreateWithFlags(&cs.s2, cudaStreamNonBlocking));
        for (int i = 0; i < 8; ++i) GL_CUDA(cudaEventCreate(&cs.ev[i]));
    }
    cudaStream_t s2 = g_overlap.load() ? cs.s2 : s; // serial mode: everything on s
    cs.keys_c.alloc((n + 1) * 2 * sizeof(u32));
    cs.items_c.alloc((n + 1) * 3 * sizeof(u32)); // id in/out, piece offsets
    GL_CUDA(cudaEventRecord(cs.ev[0], s));
    if (m == 0) {
        for (int i = 1; i < 4; ++i) GL_CUDA(cudaEventRecord(cs.ev[i], s));
        GL_CUDA(cudaEventRecord(cs.ev[6], s)); // fork/join point of the (empty) cycle pass
    } else {
        // wedge prefix straight from epos (wedges(e) = epos(e), 0 past the end):
        // no m-sized scratch
        {
            const WedgesOf op{g.epos, m};
            cub::TransformInputIterator<u64, WedgesOf, cub::CountingInputIterator<u64>> it(
                cub::CountingInputIterator<u64>(0), op);
            dev_exclusive_scan(cs.tmp, it, cs.wpre.as<u64>(), m + 1, s);
        }
        cs.launches += 2;
        GL_CUDA(cudaEventRecord(cs.ev[6], s)); // fork: the cycle pass needs the wedge prefix only
        GL_CUDA(cudaStreamWaitEvent(s2, cs.ev[6], 0));

        // H-pass: vertices by streaming cost descending; k > 32 block kernel, else warp kernel.
        // The rank's lists stay in items3b / items3s for the triangle-sum pass (count_mid).
        {
            u32* kin = cs.keys.as<u32>();
            u32* kout = kin + (n + 1);
            u32* iin = cs.items2.as<u32>();
            u32* iout = iin + (n + 1);
            k_hkeys<<<grid1d(n, 256, sms), 256, 0, s>>>(g, kin, counters + 24, counters + 12, counters + 21,
                                                        counters + 13, counters + 17, counters + 18, counters + 19);
            k_umax<<<grid1d(n, 256, sms), 256, 0, s>>>(g, (unsigned*)(counters + 14));
            k_seq<<<grid1d(n, 256, sms), 256, 0, s>>>(iin, n);
            GL_LAUNCH_CHECK();
            dev_sort_desc(cs.tmp, kin, kout, iin, iout, n, s);
            cs.launches += 3 + 10;
            u64 hc[kCounters]; // one host round trip for all class counts and bounds
            GL_CUDA(cudaMemcpyAsync(hc, counters, sizeof(hc), cudaMemcpyDeviceToHost, s));
            GL_CUDA(cudaStreamSynchronize(s));
            const u64 nxl = hc[24], nbig = hc[12], nmedk = hc[21], nsmall = hc[13];
            if (std::getenv("GL_DEBUG"))
                std::fprintf(stderr, "[gl] H-pass classes xl %llu large %llu medium %llu small %llu, kmax %llu, s1 %llu\n",
                             (unsigned long long)nxl, (unsigned long long)nbig, (unsigned long long)nmedk,
                             (unsigned long long)nsmall, (unsigned long long)(hc[14] & 0xffffffffu),
                             (unsigned long long)hc[17]);
            cs.s1 = hc[17];
            cs.work[0] = 4 * cs.s1 / (u64)world; // adjacency bytes streamed by the intersections
            const u64 myxl = rank_share(nxl, rank, world);
            const u64 mybig = rank_share(nbig, rank, world);
            const u64 mymedk = rank_share(nmedk, rank, world);
            const u64 mysmall = rank_share(nsmall, rank, world);
            cs.n_items3x = myxl;
            cs.n_items3b = mybig;
            cs.n_items3m = mymedk;
            cs.n_items3s = mysmall;
            cs.items3x.alloc((myxl + 1) * sizeof(u32));
            cs.items3b.alloc((mybig + 1) * sizeof(u32));
            cs.items3m.alloc((mymedk + 1) * sizeof(u32));
            cs.items3s.alloc((mysmall + 1) * sizeof(u32));
            // persistent H-edge records for the sums pass (every class): sized once
            // per graph from the reservation bound (C(k,2) per block vertex,
            // min(C(k,2), s1) per warp vertex), at most ~40% of the free memory;
            // headers in list order xl, large, medium, small
            if (!cs.tl_sized) {
                const size_t fr = free_at_start;
                cs.tl_cap = std::min<u64>(hc[19] / (u64)world + 1, (u64)(0.4 * (double)fr) / sizeof(uint2));
                // GL_TL_EXACT=1: reserve exactly after phase 2 instead of C(k,2) up front
                // (fills the list with more real records on large graphs, but the copy
                // costs more than the re-derivations it saves: RMAT-24 +0.8%, RMAT-26
                // +0.2% -- off by default)
                const char* ex = std::getenv("GL_TL_EXACT");
                cs.tl_exact = ex && ex[0] == '1' ? 1u : 0u;
                cs.tl_sized = true;
            }
            cs.tlist.alloc((cs.tl_cap + 1) * sizeof(uint2));
            cs.tl_base.alloc((myxl + mybig + mymedk + mysmall + 1) * sizeof(u64));
            cs.tl_n.alloc((myxl + mybig + mymedk + mysmall + 1) * sizeof(u32));
            if (myxl || mybig || mymedk) {
                const u64 s1max = hc[18];
                const u32 kmax = (u32)(hc[14] & 0xffffffffu);
                if (kmax >= 65536u) throw overflow_error("|U(a)| >= 65536: H-edge packing needs 16-bit member ids");
                cs.h_gstride = 0;
                cs.h_kmax = kmax;
                if (kmax > 1088u) { // beyond the xl shared-memory workspace: per-block global scratch
                    cs.h_gstride = (hpass_ws_words(kmax, kHPassCount, bloom_words<HCfg<1088>::BLOG>()) + 1) & ~1ull;
                    cs.scratch.alloc((u64)sms * HCfg<1088>::MINB * cs.h_gstride * sizeof(u32));
                }
                const u64 hcap_x = std::min<u64>(s1max, (u64)kmax * (kmax - 1) / 2) + 1;
                const u64 hcap_l = std::min<u64>(s1max, 512ull * 511 / 2) + 1;
                const u64 hcap_m = std::min<u64>(s1max, 128ull * 127 / 2) + 1;
                cs.hlist.alloc(std::max<u64>(std::max<u64>((u64)sms * HCfg<1088>::MINB * hcap_x,
                                                           (u64)sms * HCfg<768>::MINB * hcap_l),
                                             (u64)sms * HCfg<128>::MINB * hcap_m) *
                               sizeof(uint2));
                auto launch = [&](auto kc, u64 count, u64 offset, u64 total, u32* list, u64 hbase, u64 hcap,
                                  unsigned long long* queue) {
                    constexpr int K = decltype(kc)::value;
                    k_take_rank<u32><<<grid1d(count, 256, sms), 256, 0, s>>>(iout, offset, total, rank, world, list);
                    GL_LAUNCH_CHECK();
                    const size_t smem = hpass_smem_bytes<kHPassCount, K>(kmax, gr.device);
                    smem_attr(k_hpass_block<kHPassCount, K>, smem, gr.device);
                    const TriList TL{cs.tlist.as<uint2>(), cs.tl_cap, counters + 20, cs.tl_base.as<u64>() + hbase,
                                     cs.tl_n.as<u32>() + hbase, cs.tl_exact};
                    const bool glob = K == 1088 && cs.h_gstride;
                    k_hpass_block<kHPassCount, K><<<(unsigned)sms * HCfg<K>::MINB, HCfg<K>::THREADS, smem, s>>>(
                        g, list, count, queue, cs.t.as<u32>(), d_partials, glob ? cs.scratch.as<u32>() : nullptr,
                        glob ? cs.h_gstride : 0, cs.hlist.as<uint2>(), hcap, TL, (u32)(smem / sizeof(u32)));
                    GL_LAUNCH_CHECK();
                    cs.launches += 2;
                };
                if (myxl)
                    launch(std::integral_constant<int, 1088>{}, myxl, 0, nxl, cs.items3x.as<u32>(), 0, hcap_x,
                           counters + 25);
                if (mybig)
                    launch(std::integral_constant<int, 768>{}, mybig, nxl, nbig, cs.items3b.as<u32>(), myxl, hcap_l,
                           counters + 0);
                if (mymedk)
                    launch(std::integral_constant<int, 128>{}, mymedk, nxl + nbig, nmedk, cs.items3m.as<u32>(),
                           myxl + mybig, hcap_m, counters + 8);
            }
            if (mysmall) {
                k_take_rank<u32><<<grid1d(mysmall, 256, sms), 256, 0, s>>>(iout, nxl + nbig + nmedk, nsmall, rank, world,
                                                                      cs.items3s.as<u32>());
                GL_LAUNCH_CHECK();
                const TriList TL{cs.tlist.as<uint2>(), cs.tl_cap, counters + 20,
                                 cs.tl_base.as<u64>() + myxl + mybig + mymedk, cs.tl_n.as<u32>() + myxl + mybig + mymedk,
                                 cs.tl_exact};
                k_hpass_warp<kHPassCount><<<(unsigned)sms * 8, kHWarpsPerBlock * 32, 0, s>>>(
                    g, cs.items3s.as<u32>(), mysmall, counters + 3, cs.t.as<u32>(), d_partials, TL);
                GL_LAUNCH_CHECK();
                cs.launches += 2;
            }
        }
        GL_CUDA(cudaEventRecord(cs.ev[1], s));
        if (world == 1 && (cs.out_t || cs.out_x7)) {
            // t and x7 are final now (only the H-pass writes them): copy them out
            // on s3 while the cycle pass runs (gl_count_edges)
            if (!cs.s3) {
                GL_CUDA(cudaStreamCreateWithFlags(&cs.s3, cudaStreamNonBlocking));
                GL_CUDA(cudaEventCreateWithFlags(&cs.ev_out, cudaEventDisableTiming));
            }
            GL_CUDA(cudaStreamWaitEvent(cs.s3, cs.ev[1], 0));
            if (cs.out_t) GL_CUDA(cudaMemcpyAsync(cs.out_t, cs.t.p, m * sizeof(u32), cudaMemcpyDeviceToHost, cs.s3));
            if (cs.out_x7) {
                // staged in the x7 output array itself: k_final later writes the
                // same values there (x7_out[e] = part[2e])
                cs.x7.alloc((m + 1) * sizeof(u64));
                k_even<<<grid1d(m, 256, sms), 256, 0, cs.s3>>>(d_partials, m, cs.x7.as<u64>());
                GL_LAUNCH_CHECK();
                GL_CUDA(cudaMemcpyAsync(cs.out_x7, cs.x7.p, m * sizeof(u64), cudaMemcpyDeviceToHost, cs.s3));
                cs.launches += 1;
            }
            GL_CUDA(cudaEventRecord(cs.ev_out, cs.s3));
        }

        // cycles: top vertices, split small (warp hash) / big (block windows)
        GL_CUDA(cudaEventRecord(cs.ev[2], s2));
        {
            u32* kin = cs.keys_c.as<u32>();
            u32* kout = kin + (n + 1);
            u32* iin = cs.items_c.as<u32>();
            u32* iout = iin + (n + 1);
            k_top_keys<<<grid1d(n, 256, sms), 256, 0, s2>>>(g, cs.wpre.as<u64>(), cs.tierbuf.as<const unsigned>(),
                                                           kin, counters + 10, counters + 15, counters + 16,
                                                           counters + 11, counters + 27, sparse_big_factor());
            k_seq<<<grid1d(n, 256, sms), 256, 0, s2>>>(iin, n);
            GL_LAUNCH_CHECK();
            dev_sort_desc(cs.tmp_c, kin, kout, iin, iout, n, s2);
            u64 cc[kCounters];
            GL_CUDA(cudaMemcpyAsync(cc, counters, sizeof(cc), cudaMemcpyDeviceToHost, s2));
            const u64 wtot = read_dev(cs.wpre.as<u64>() + m, s2);
            const u64 nsparse = cc[27], nbig = cc[10], nmid = cc[15], nsmid = cc[16], nsmall = cc[11];
            if (std::getenv("GL_DEBUG"))
                std::fprintf(stderr, "[gl] cycle classes sparse-big %llu big %llu mid %llu small-mid %llu small %llu\n",
                             (unsigned long long)nsparse, (unsigned long long)nbig, (unsigned long long)nmid,
                             (unsigned long long)nsmid, (unsigned long long)nsmall);
            const uint4 tiers = cs.tiers;
            // slot credits: u32 unless c is a hub (degree >= 65536 = ids >= tiers.w), see Credits
            const Credits credits{cs.slots.as<i64>(), cs.slots32.as<u32>(), tiers.w};
            cs.work[2] = 12 * wtot / (u64)world; // 4 B c id + 8 B slot credit per wedge
            cs.launches += 2 + 10;
            const u64 mysparse = rank_share(nsparse, rank, world);
            const u64 mybig = rank_share(nbig, rank, world);
            const u64 mymid = rank_share(nmid, rank, world);
            const u64 mysmid = rank_share(nsmid, rank, world);
            const u64 mysmall = rank_share(nsmall, rank, world);
            // windowed tops -> pieces (positions [0, nsparse + nbig) of the sorted list)
            const u64 nwin = nsparse + nbig;
            u64 psparse = 0, pbig = 0;
            if (nwin) {
                u32* np = kin; // scratch: keys are sorted into kout already
                k_piece_count<<<grid1d(nwin, 256, sms), 256, 0, s2>>>(
                    g, cs.wpre.as<u64>(), iout, nwin, piece_cap(wtot, sms, world), piece_forced() ? 1u : 32u, np);
                GL_CUDA(cudaMemsetAsync(np + nwin, 0, sizeof(u32), s2));
                u32* poff = cs.items_c.as<u32>() + 2 * (n + 1); // see the allocation above
                dev_exclusive_scan(cs.tmp_c, (const u32*)np, poff, nwin + 1, s2);
                u32 hp[2];
                GL_CUDA(cudaMemcpyAsync(&hp[0], poff + nsparse, sizeof(u32), cudaMemcpyDeviceToHost, s2));
                GL_CUDA(cudaMemcpyAsync(&hp[1], poff + nwin, sizeof(u32), cudaMemcpyDeviceToHost, s2));
                GL_CUDA(cudaStreamSynchronize(s2));
                psparse = hp[0];
                pbig = hp[1] - hp[0];
                cs.pieces.alloc(((u64)hp[1] * 2 + 2) * sizeof(uint4)); // all pieces, then this rank's share
                k_pieces<<<(unsigned)std::min<u64>(nwin, (u64)sms * 8), 256, 0, s2>>>(
                    g, cs.wpre.as<u64>(), iout, nwin, nsparse, cs.tierbuf.as<const unsigned>(), walk_cl(), poff,
                    cs.pieces.as<uint4>());
                GL_LAUNCH_CHECK();
                cs.launches += 4;
                if (std::getenv("GL_DEBUG"))
                    std::fprintf(stderr, "[gl] cycle pieces: %llu sparse-big, %llu big (from %llu windowed tops, cap %llu)\n",
                                 (unsigned long long)psparse, (unsigned long long)pbig, (unsigned long long)nwin,
                                 (unsigned long long)piece_cap(wtot, sms, world));
            }
            const u64 mysparse_p = rank_share(psparse, rank, world), mybig_p = rank_share(pbig, rank, world);
            uint4* pall = cs.pieces.as<uint4>();
            uint4* psp = pall + psparse + pbig;
            uint4* pbg = psp + mysparse_p;
            cs.cycle_pieces = psparse + pbig;
            u32* lsparse = iin;
            u32* lbig = lsparse + mysparse;
            u32* lmid = lbig + mybig;
            u32* lsmid = lmid + mymid;
            u32* lsmall = lsmid + mysmid;
            if (mysparse_p || mybig_p || mymid || mysmid) {
                if (2 * m >= (1ull << 32)) throw overflow_error("cycle pass needs 2m < 2^32 adjacency slots");
                // per-block scratch: big tops need dmax + 2 entries, hash tops at most
                // their wedge bound (nb <= wedges)
                const u32 cap_big = (g.dmax + 3) & ~1u;
                const u32 cap_hash = std::min<u32>(cap_big, (u32)kMidWedges + 2);
                const u64 w_big = (big_scratch_words(cap_big) + 1) & ~1ull;
                const u64 w_hash = (big_scratch_words(cap_hash) + 1) & ~1ull;
                if (mybig_p || mysparse_p) cs.cursor.alloc((u64)sms * kBigBlocksPerSM * w_big * sizeof(u32));
                // run-end table of the dense windows (once per graph and walk_cl; GL_RUN_TABLE=0 disables)
                const char* rt = std::getenv("GL_RUN_TABLE");
                const bool use_runs = mybig_p && !(rt && rt[0] == '0') && cs.runtab_key == walk_cl() + 1;
                if (mymid || mysmid) cs.cursor2.alloc((u64)sms * 4 * w_hash * sizeof(u32));
                auto launch = [&](auto kind, u32* list, u64 count, u64 offset, u64 total, unsigned long long* queue) {
                    constexpr int K = decltype(kind)::value;
                    constexpr bool WIN = Cyc<K>::WIN;
                    const u32 cap = K == 0 || K == 3 ? cap_big : cap_hash;
                    u32* scratch = K == 0 || K == 3 ? cs.cursor.as<u32>() : cs.cursor2.as<u32>();
                    uint4* plist = K == 3 ? psp : pbg;
                    if (WIN)
                        k_take_rank<uint4><<<grid1d(count, 256, sms), 256, 0, s2>>>(pall, offset, total, rank, world,
                                                                                    plist);
                    else
                        k_take_rank<u32><<<grid1d(count, 256, sms), 256, 0, s2>>>(iout, offset, total, rank, world, list);
                    GL_LAUNCH_CHECK();
                    const size_t smem = (size_t)cyc_smem_words<K>() * sizeof(u32);
                    smem_attr(k_cycle_block<K>, smem, gr.device);
                    k_cycle_block<K><<<(unsigned)sms * Cyc<K>::MINB, Cyc<K>::THREADS, smem, s2>>>(
                        g, list, plist, count, queue, credits, scratch, cap, tiers, walk_cl(),
                        K == 0 && use_runs ? cs.runtab.as<u64>() : nullptr);
                    GL_LAUNCH_CHECK();
                    cs.launches += 2;
                };
                // sorted list: [sparse big | big | mid | small-mid | small]; the
                // windowed classes go as pieces [sparse big pieces | big pieces]
                if (mysparse_p)
                    launch(std::integral_constant<int, 3>{}, nullptr, mysparse_p, 0, psparse, counters + 28);
                if (mybig_p) launch(std::integral_constant<int, 0>{}, nullptr, mybig_p, psparse, pbig, counters + 1);
                if (mymid) launch(std::integral_constant<int, 1>{}, lmid, mymid, nsparse + nbig, nmid, counters + 4);
                if (mysmid)
                    launch(std::integral_constant<int, 2>{}, lsmid, mysmid, nsparse + nbig + nmid, nsmid, counters + 7);
            }
            if (mysmall) {
                k_take_rank<u32><<<grid1d(mysmall, 256, sms), 256, 0, s2>>>(iout, nsparse + nbig + nmid + nsmid, nsmall, rank,
                                                                       world, lsmall);
                GL_LAUNCH_CHECK();
                const size_t smem = (size_t)kCycleSmallWarps * kSmallWarpWords * sizeof(u32);
                smem_attr(k_cycle_small, smem, gr.device);
                k_cycle_small<<<(unsigned)sms * 3, kCycleSmallWarps * 32, smem, s2>>>(
                    g, cs.wpre.as<u64>(), lsmall, mysmall, counters + 2, credits);
                GL_LAUNCH_CHECK();
                cs.launches += 2;
            }
        }
    }
    if (m) GL_CUDA(cudaEventRecord(cs.ev[3], s2)); // cycle pass done
    cs.ms[1] = 0;
    cs.began = true;
}

// Phase B: triangle sums S (needs the complete t on this rank).
void count_mid(Graph& gr, i64* d_partials, cudaStream_t s) {
    GL_CUDA(cudaSetDevice(gr.device));
    if (!s) s = gr.stream;
    CountState& cs = gr.cs;
    if (!cs.began) throw state_error("gl_count_mid before gl_count_begin");
    // a second fold would add the slot credits to y twice
    if (cs.mid_done) throw state_error("gl_count_mid called twice for one gl_count_begin");
    const DevGraph& g = gr.d;
    const int sms = num_sms(gr.device);
    GL_CUDA(cudaEventRecord(cs.ev[4], s));
    // triangle sums over the same vertex shares as this rank's H-pass
    unsigned long long* counters = cs.acc.as<unsigned long long>() + 40;
    auto sums = [&](auto kc, u64 count, const u32* list, u64 hbase, unsigned long long* queue) {
        constexpr int K = decltype(kc)::value;
        const size_t smem = hpass_smem_bytes<kHPassSums, K>(cs.h_kmax, gr.device);
        smem_attr(k_hpass_block<kHPassSums, K>, smem, gr.device);
        const TriList TL{cs.tlist.as<uint2>(), cs.tl_cap, counters + 20, cs.tl_base.as<u64>() + hbase,
                         cs.tl_n.as<u32>() + hbase, cs.tl_exact};
        const bool glob = K == 1088 && cs.h_gstride;
        k_hpass_block<kHPassSums, K><<<(unsigned)sms * HCfg<K>::MINB, HCfg<K>::THREADS, smem, s>>>(
            g, list, count, queue, cs.t.as<u32>(), d_partials, glob ? cs.scratch.as<u32>() : nullptr,
            glob ? cs.h_gstride : 0, nullptr, 0, TL, (u32)(smem / sizeof(u32)));
        GL_LAUNCH_CHECK();
        cs.launches += 1;
    };
    if (g.m && cs.n_items3x) sums(std::integral_constant<int, 1088>{}, cs.n_items3x, cs.items3x.as<u32>(), 0, counters + 26);
    if (g.m && cs.n_items3b)
        sums(std::integral_constant<int, 768>{}, cs.n_items3b, cs.items3b.as<u32>(), cs.n_items3x, counters + 5);
    if (g.m && cs.n_items3m)
        sums(std::integral_constant<int, 128>{}, cs.n_items3m, cs.items3m.as<u32>(), cs.n_items3x + cs.n_items3b,
             counters + 9);
    if (g.m && cs.n_items3s) {
        const u64 hb = cs.n_items3x + cs.n_items3b + cs.n_items3m;
        const TriList TL{cs.tlist.as<uint2>(), cs.tl_cap, counters + 20, cs.tl_base.as<u64>() + hb,
                         cs.tl_n.as<u32>() + hb, cs.tl_exact};
        k_hpass_warp<kHPassSums><<<(unsigned)sms * 8, kHWarpsPerBlock * 32, 0, s>>>(
            g, cs.items3s.as<u32>(), cs.n_items3s, counters + 6, cs.t.as<u32>(), d_partials, TL);
        GL_LAUNCH_CHECK();
        cs.launches += 1;
    }
    GL_CUDA(cudaEventRecord(cs.ev[5], s));
    // join the cycle pass, then fold its per-slot C4 credits into the y rows
    // (after the sums: both update y, the fold non-atomically)
    GL_CUDA(cudaStreamWaitEvent(s, cs.ev[3], 0));
    if (g.m) {
        k_fold_slots<<<grid1d(g.m, 256, sms), 256, 0, s>>>(g, Credits{cs.slots.as<i64>(), cs.slots32.as<u32>(), 0u},
                                                           d_partials);
        GL_LAUNCH_CHECK();
        cs.launches += 1;
    }
    GL_CUDA(cudaEventRecord(cs.ev[7], s)); // end of count_mid (re-entry fence of count_begin)
    cs.mid_done = true;
}

void count_finish(Graph& gr, const i64* d_part_shard, u64 begin, u64 end, u128 C[17], cudaStream_t s) {
    GL_CUDA(cudaSetDevice(gr.device));
    if (!s) s = gr.stream;
    CountState& cs = gr.cs;
    if (!cs.began || !cs.mid_done) throw state_error("gl_count_finish before gl_count_begin/gl_count_mid");
    const DevGraph& g = gr.d;
    if (end > g.m) end = g.m;
    if (begin > end) throw invalid_argument("edge_begin > edge_end");
    const int sms = num_sms(gr.device);
    cs.x7.alloc((g.m + 1) * sizeof(u64));
    cs.x10.alloc((g.m + 1) * sizeof(u64));
    unsigned long long* acc = cs.acc.as<unsigned long long>();
    GL_CUDA(cudaMemsetAsync(acc, 0, 40 * sizeof(u64), s));
    Timer tm(2);
    GL_CUDA(cudaEventRecord(tm.ev[0], s));
    if (end > begin) {
        k_final<<<grid1d(end - begin, kFinThreads, sms, 4), kFinThreads, 0, s>>>(
            g, d_part_shard, cs.t.as<u32>(), begin, end, cs.x7.as<u64>(), cs.x10.as<u64>(), acc,
            (unsigned*)(acc + 36));
        GL_LAUNCH_CHECK();
        cs.launches += 1;
    }
    GL_CUDA(cudaEventRecord(tm.ev[1], s));
    u64 h[40];
    GL_CUDA(cudaMemcpyAsync(h, acc, sizeof(h), cudaMemcpyDeviceToHost, s));
    GL_CUDA(cudaStreamSynchronize(s));
    GL_CUDA(cudaEventElapsedTime(&cs.ms[3], tm.ev[0], tm.ev[1]));
    // phase times of begin/mid (their events completed before this sync):
    // H-pass, triangle sums, cycle pass (concurrent with the other two)
    GL_CUDA(cudaEventElapsedTime(&cs.ms[0], cs.ev[0], cs.ev[1]));
    GL_CUDA(cudaEventElapsedTime(&cs.ms[1], cs.ev[4], cs.ev[5]));
    GL_CUDA(cudaEventElapsedTime(&cs.ms[2], cs.ev[2], cs.ev[3]));
    cs.ms[4] = cs.ms[0] + cs.ms[1] + cs.ms[2] + cs.ms[3];
    cs.work[3] = 52 * (end - begin); // t,x7,y,eu,ev,2 degrees in; x7,x10 out
    const unsigned* flags = reinterpret_cast<const unsigned*>(h + 36);
    if (flags[0]) throw consistency_error("per-edge bound violated (x7 > C(t,2) or x10 > s_u*s_v)");
    if (flags[1]) throw overflow_error("128-bit count accumulator overflow");
    for (int i = 0; i < 17; ++i) C[i] = ((u128)h[2 * i + 1] << 64) | h[2 * i];
    // triangle sums: one H-edge record per triangle (C3 = sum t = 3 * triangles
    // of this shard), each an 8 B record read + 4 B t gather + 8 B RED
    cs.work[1] = (u64)(20 * (C[3] / 3));
    cs.shard_begin = begin;
    cs.shard_end = end;
    cs.have_micro = true;
}

namespace {
__global__ void k_micro(DevGraph g, const u32* __restrict__ t, const u64* __restrict__ x7,
                        const u64* __restrict__ x10, u64 first, u64 count, u64* __restrict__ out) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < count; i += (u64)gridDim.x * blockDim.x) {
        u64 e = first + i;
        u64 te = t[e];
        u64 du = g.deg[g.eu[e]], dv = g.deg[g.ev[e]];
        u64 su = du - te - 1, sv = dv - te - 1;
        u64 de = g.n - (su + sv + te) - 2;
        u64* o = out + 10 * i; // counts.cpp:122-136 field order
        o[0] = e;
        o[1] = te;
        o[2] = su + sv;
        o[3] = de;
        o[4] = x7[e];
        o[5] = x10[e];
        o[6] = te;
        o[7] = su;
        o[8] = sv;
        o[9] = de;
    }
}

// sum of neighbour degrees per vertex (one warp per vertex)
__global__ void k_nbr_degree_sum(DevGraph g, u64* __restrict__ out) {
    const u64 warp = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5, nwarp = ((u64)gridDim.x * blockDim.x) >> 5;
    for (u64 v = warp; v < g.n; v += nwarp) {
        u64 s = 0;
        for (u64 p = g.off[v] + lane_id(); p < g.off[v + 1]; p += 32) s += g.deg[g.adj[p]];
        s = warp_sum_u64(s);
        if (lane_id() == 0) out[v] = s;
    }
}
// EdgeMotifRecord rows {edge_id | t << 32, s_u | s_v << 32, x7, x10, work_units}
__global__ void k_motif(DevGraph g, const u32* __restrict__ t, const u64* __restrict__ x7,
                        const u64* __restrict__ x10, const u64* __restrict__ nbrsum, u64 first, u64 count,
                        u64* __restrict__ out) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < count; i += (u64)gridDim.x * blockDim.x) {
        const u64 e = first + i;
        const u32 u = g.eu[e], v = g.ev[e];
        const u64 te = t[e], du = g.deg[u], dv = g.deg[v];
        u64* o = out + 5 * i;
        o[0] = e | (te << 32);
        o[1] = (du - te - 1) | ((dv - te - 1) << 32);
        o[2] = x7[e];
        o[3] = x10[e];
        o[4] = du + dv + nbrsum[u];
    }
}
} // namespace

void edge_motif_records(const Graph& gr, u64 first, u64 count, u64* host_out) {
    GL_CUDA(cudaSetDevice(gr.device));
    const CountState& cs = gr.cs;
    if (!cs.have_micro) throw state_error("no counts computed yet");
    if (first < cs.shard_begin || first > cs.shard_end || count > cs.shard_end - first)
        throw invalid_argument("edge range outside the computed shard");
    if (count == 0) return;
    cudaStream_t s = gr.stream;
    const int sms = num_sms(gr.device);
    DevBuf nbr, tmp;
    nbr.alloc((gr.d.n + 1) * sizeof(u64));
    k_nbr_degree_sum<<<grid1d(gr.d.n * 32, 256, sms), 256, 0, s>>>(gr.d, nbr.as<u64>());
    GL_LAUNCH_CHECK();
    const u64 chunk = 1ull << 22;
    tmp.alloc(std::min(count, chunk) * 5 * sizeof(u64));
    for (u64 off = 0; off < count; off += chunk) {
        const u64 c = std::min(chunk, count - off);
        k_motif<<<grid1d(c, 256, sms), 256, 0, s>>>(gr.d, cs.t.as<u32>(), cs.x7.as<u64>(), cs.x10.as<u64>(),
                                                    nbr.as<u64>(), first + off, c, tmp.as<u64>());
        GL_LAUNCH_CHECK();
        GL_CUDA(cudaMemcpyAsync(host_out + 5 * off, tmp.p, c * 5 * sizeof(u64), cudaMemcpyDeviceToHost, s));
        GL_CUDA(cudaStreamSynchronize(s)); // tmp is reused by the next chunk
    }
}

void micro_records(const Graph& gr, u64 first, u64 count, u64* host_out) {
    GL_CUDA(cudaSetDevice(gr.device));
    const CountState& cs = gr.cs;
    if (!cs.have_micro) throw state_error("no counts computed yet");
    if (first < cs.shard_begin || first > cs.shard_end || count > cs.shard_end - first)
        throw invalid_argument("edge range outside the computed shard");
    if (count == 0) return;
    cudaStream_t s = gr.stream;
    const u64 chunk = 1ull << 22;
    DevBuf tmp;
    tmp.alloc(std::min(count, chunk) * 10 * sizeof(u64));
    const int sms = num_sms(gr.device);
    for (u64 off = 0; off < count; off += chunk) {
        u64 c = std::min(chunk, count - off);
        k_micro<<<grid1d(c, 256, sms), 256, 0, s>>>(gr.d, cs.t.as<u32>(), cs.x7.as<u64>(), cs.x10.as<u64>(),
                                                    first + off, c, tmp.as<u64>());
        GL_LAUNCH_CHECK();
        GL_CUDA(cudaMemcpyAsync(host_out + 10 * off, tmp.p, c * 10 * sizeof(u64), cudaMemcpyDeviceToHost, s));
    }
    GL_CUDA(cudaStreamSynchronize(s));
}

} // namespace gl

#ifdef GL_CYCLE_PROF
extern "C" int gl_debug_cycle_profile(unsigned long long* out, int reset) {
    if (cudaMemcpyFromSymbol(out, gl::g_cycle_prof, sizeof(unsigned long long) * 64) != cudaSuccess) return -4;
    if (reset) {
        unsigned long long z[64] = {0};
        if (cudaMemcpyToSymbol(gl::g_cycle_prof, z, sizeof(z)) != cudaSuccess) return -4;
    }
    return 0;
}
#endif
