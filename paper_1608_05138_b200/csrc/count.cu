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
// S(e) = sum_{w in T(e)} (t(u,w) + t(v,w)).  Kernels:
//   k_tri<0>   t(e) for all edges: one probe per element of the shorter of
//              U(u)\{..v}, U(v); each triangle found once at its lowest pair
//   k_tri<1>   S(e) contributions, same probe space, reads t
//   k_clique   per lowest pair (a,b): T+ = U(a) n U(b) staged in shared
//              memory; edges inside T+ give x7 to all six clique edges
//   k_cycle_s/ per top vertex a (Chiba-Nishizeki wedges b<a, c<a): W[c] in a
//   k_cycle_b  warp hash (small) or block-dense shared-memory windows (big);
//              C4 credit W[c]-1 to edges (a,b) and (b,c)
//   k_final    per-edge epilogue + fused block reduction of C3..C16 (128-bit)
// All arithmetic is exact integer; partial sums live in int64 rows
// {x7, C4 - S} that wrap mod 2^64 and are exact once complete.
#include <cub/cub.cuh>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
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
constexpr u64 kSmallWedges = 512;    // small-top threshold (<= half the slots)
constexpr int kBigThreads = 1024;    // block per big top (dense windows), one block per SM
constexpr int kBigBlocksPerSM = 1;
constexpr int kMidThreads = 1024;    // block per mid top (hash), one block per SM
constexpr int kSmidThreads = 256;    // block per small-mid top (hash), four blocks per SM
constexpr int kWindow = 32768;       // dense W window words (u32, or 2 x u16) in shared memory
constexpr int kMidLog = 15;
constexpr u32 kMidSlots = 1u << kMidLog; // mid tops: block hash, u32 keys + u16 counts (192 KB)
constexpr u64 kMidWedges = kMidSlots / 2; // mid-top threshold (<= half the hash slots)
constexpr int kSmidLog = 13;
constexpr u64 kSmidWedges = (1u << kSmidLog) / 2; // small-mid threshold

constexpr u32 kEmpty = 0xffffffffu;

int g_num_sms = 0;
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
__global__ void k_prepass(DevGraph g, u64* __restrict__ wedges) {
    for (u64 e = blockIdx.x * (u64)blockDim.x + threadIdx.x; e < g.m; e += (u64)gridDim.x * blockDim.x)
        wedges[e] = g.epos[e];
}

// ------------------------------------------------------------------ H-pass
//
// Per lowest vertex a, the out-neighbourhood H_a = G[U(a)] (k = |U(a)|
// members x_0 < ... < x_{k-1}, ascending id).  Every triangle (a < x < y) is
// an edge (x,y) of H_a and every 4-clique (a < x < y < z) a triangle of H_a.
//
// MODE kHPassCount (t and x7 partials), one pass over all a yields, each once:
//   t(x,y)  += 1                       t(a,x)  += deg_H(x)
//   x7(x,y) += |N_H(x) n N_H(y)|       x7(a,x) += #triangles of H_a at x
// with H_a staged as a bitmap adjacency matrix (ceil(k/32) u32 words per row):
// global atomics are per triangle, never per 4-clique (a 4-clique is only
// ever a popcount of an AND of two shared-memory rows).
//
// MODE kHPassSums (S partials, t complete): every triangle tau = (a,x,y)
// credits y(e) -= t of the other two edges to each of its three edges
// (y = C4 - S, S(e) = sum over triangles at e of the other two t's); the
// (a,x) credits are summed per member in shared memory.
//
// H-edges are found by streaming: member x_i's upper list U(x_i) is read
// coalesced by one warp and every entry is looked up in a shared-memory hash
// of U(a) (4k slots, u32 keys, u16 member index).  Cost: sum_i |U(x_i)|
// coalesced adjacency reads + one smem probe each, no global binary search.

constexpr int kHPassCount = 0, kHPassSums = 1;
constexpr int kHWarpMax = 32;       // 2 <= k <= 32: one warp, one u32 row per lane
constexpr int kHWarpsPerBlock = 8;
constexpr int kHBlockThreads = 512; // k > 32: one block per vertex
constexpr int kHSmemMax = 768;      // k <= 768: workspace in shared memory
constexpr int kHUnroll = 8;         // streamed rounds in flight per warp
constexpr u32 kHProbeRatio = 8;     // probe instead of stream when |U(x_i)| > 8 * candidates

__device__ __forceinline__ u64 warp_sum_u64(u64 v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    return v;
}

__device__ __forceinline__ u64 u_begin(const DevGraph& g, u32 x) { return g.off[x] + g.lcnt[x]; }

// member filter of the block H-pass: 2^BLOG bits (8 KB for large k, 1 KB for k <= 128)
template <int BLOG> __device__ __forceinline__ u32 bloom_bit(u32 y) { return (y * 0x2545F491u) >> (32 - BLOG); }
template <int BLOG> __host__ __device__ constexpr u32 bloom_words() { return (1u << BLOG) / 32; }
// block H-pass configurations: k > 512 (1024 threads, one block per SM, the
// workspace in shared memory up to k = 1088), 128 < k <= 512 (512 threads, two
// blocks per SM) and 32 < k <= 128 (128 threads, eight blocks per SM: the
// fixed per-vertex latency of the many small vertices overlaps across blocks)
template <int KMAX> struct HCfg;
template <> struct HCfg<1088> { static constexpr int THREADS = 1024, MINB = 1, BLOG = 16; };
template <> struct HCfg<768> { static constexpr int THREADS = 512, MINB = 2, BLOG = 16; };
template <> struct HCfg<128> { static constexpr int THREADS = 128, MINB = 8, BLOG = 13; };

__device__ __forceinline__ u32 hp_log(u32 k) { // hash slots 2^log >= 2k, >= 64 (Bloom filters the misses)
    u32 l = 32 - __clz(2 * k - 1);
    return l < 6 ? 6 : l;
}
__host__ __device__ inline u64 hpass_ws_words(u32 k, int mode, u32 bloom_w) {
    u32 l = 6;
    while ((1u << l) < 2 * k) ++l;
    const u64 H = 1ull << l;
    const u64 W = (k + 31) / 32;
    const u64 body = mode == 0 ? 2ull * k + (u64)k * (W | 1)  // xs, tri, rows (odd stride)
                               : 4ull * k + 2;          // xs, ta, acc (u64, aligned)
    return body + 2 + H + H / 2 + bloom_w + 2ull * k; // + member list bounds
}

__device__ __forceinline__ void atomic_add_i64(i64* p, i64 v) {
    atomicAdd(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v);
}

// Guided chunked grabs from a work-list queue for warp-per-item kernels: one
// atomic per chunk of about remaining / (4 * warps in the grid) items (1..32),
// so millions of light items do not serialise on the queue counter.
struct WarpGrab {
    unsigned long long next = 0, end = 0;
    __device__ __forceinline__ bool pop(unsigned long long* queue, u64 n_items, unsigned long long* idx) {
        if (next == end) {
            unsigned long long b = 0, c = 0;
            if (lane_id() == 0) {
                const unsigned long long seen = *(volatile unsigned long long*)queue;
                const unsigned long long warps = (unsigned long long)gridDim.x * (blockDim.x >> 5);
                c = seen < n_items ? (n_items - seen) / (4 * warps) : 1;
                c = c < 1 ? 1 : (c > 32 ? 32 : c);
                b = atomicAdd(queue, c);
            }
            next = __shfl_sync(0xffffffffu, b, 0);
            end = next + __shfl_sync(0xffffffffu, c, 0);
        }
        if (next >= n_items) return false;
        *idx = next++;
        return true;
    }
};

// Persistent H-edge records of the block H-pass: the counting pass appends
// every H-edge (i | j << 16, e_xy) of vertex a to one device-wide list and
// records (base, count) per work item; the triangle-sum pass then streams the
// records instead of re-deriving them (base = kNoList: list full, re-derive).
struct TriList {
    uint2* rec;
    u64 cap;
    unsigned long long* count;
    u64* base;   // per work item
    u32* n;      // per work item
};
constexpr u64 kNoList = ~0ull;

// 2 <= k <= 32: one warp per vertex a.  Phase 1 streams every member's upper
// list U(x_i) with the whole warp (coalesced) and looks each entry up in
// U(a) (32 sorted ids in shared memory, 5-step search); a hit sets bit j of
// row i and records the edge id of (x_i, x_j) in a 32 x 32 shared table, so
// phase 2 needs no global search.  kHPassCount: t and x7 credits as in the
// block kernel; kHPassSums: the three S credits of every triangle.
template <int MODE>
__global__ void __launch_bounds__(kHWarpsPerBlock * 32)
k_hpass_warp(DevGraph g, const u32* __restrict__ items, u64 n_items, unsigned long long* __restrict__ queue,
             u32* __restrict__ t, i64* __restrict__ part, TriList TL) {
    __shared__ u32 s_x[kHWarpsPerBlock][32];
    __shared__ u32 s_row[kHWarpsPerBlock][32];
    __shared__ u32 s_ta[kHWarpsPerBlock][32];
    __shared__ u32 s_e[kHWarpsPerBlock][32][33]; // edge id of (x_i, x_j), j > i (padded)
    __shared__ unsigned long long s_acc[kHWarpsPerBlock][32];
    __shared__ u32 s_pre[kHWarpsPerBlock][32], s_ppre[kHWarpsPerBlock][32];
    __shared__ u64 s_xb[kHWarpsPerBlock][32], s_xe[kHWarpsPerBlock][32];
    const u32 lane = lane_id(), wib = threadIdx.x >> 5;
    u32* xs = s_x[wib];
    u32* rows = s_row[wib];
    u32* ta = s_ta[wib];
    unsigned long long* acc = s_acc[wib];
    WarpGrab grab;
    unsigned long long idx = 0;
    while (grab.pop(queue, n_items, &idx)) {
        const u32 a = items[idx];
        const u64 ub = u_begin(g, a);
        const u32 k = (u32)(g.off[a + 1] - ub);
        if (MODE == kHPassSums && TL.rec && TL.base[idx] != kNoList) {
            // stream the records the counting pass kept for this vertex
            const u32 nrec = TL.n[idx];
            if (nrec == 0) continue;
            const uint2* rec = TL.rec + TL.base[idx];
            if (lane < k) ta[lane] = t[g.eid[ub + lane]];
            acc[lane] = 0;
            __syncwarp();
            for (u32 r = lane; r < nrec; r += 32) {
                const uint2 rv = rec[r];
                const u32 i = rv.x & 0xffffu, j = rv.x >> 16;
                const u64 ti = ta[i], tj = ta[j], txy = t[rv.y];
                atomic_add_i64(&part[2 * (u64)rv.y + 1], -(i64)(ti + tj));
                atomicAdd(&acc[i], (unsigned long long)(tj + txy));
                atomicAdd(&acc[j], (unsigned long long)(ti + txy));
            }
            __syncwarp();
            if (lane < k && acc[lane]) atomic_add_i64(&part[2 * (u64)g.eid[ub + lane] + 1], -(i64)acc[lane]);
            __syncwarp();
            continue;
        }
        u64 xb = 0, xe = 0;
        if (lane < k) {
            const u32 x = g.adj[ub + lane];
            xs[lane] = x;
            xb = u_begin(g, x);
            xe = g.off[x + 1];
            if (MODE == kHPassSums) ta[lane] = t[g.eid[ub + lane]];
        } else {
            xs[lane] = kEmpty; // sorts after every id: searches stay inside [0, k)
        }
        rows[lane] = 0;
        acc[lane] = 0;
        __syncwarp();
        const u32 xmax = xs[k - 1];
        // phase 1: member i's H-row by streaming U(x_i) when it is short
        // (|U(x_i)| <= 8 * rem_i, rem_i = k-1-i) or else by probing the rem_i
        // candidates x_j (j > i) into U(x_i) with binary searches.  Both work
        // lists are flattened over the warp (prefix sums in shared memory, a
        // 5-step search maps a lane to its member), 4 rounds in flight.
        const u32 rem = lane + 1 < k ? k - 1 - lane : 0u;
        const u32 ul = (u32)(xe - xb);
        const bool probe = rem && ul > 8u * rem;
        const u32 slen = rem && !probe ? ul : 0u, plen = probe ? rem : 0u;
        u32 sin = slen, pin = plen;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const u32 o1 = __shfl_up_sync(0xffffffffu, sin, d);
            const u32 o2 = __shfl_up_sync(0xffffffffu, pin, d);
            if (lane >= (u32)d) {
                sin += o1;
                pin += o2;
            }
        }
        const u32 stot = __shfl_sync(0xffffffffu, sin, 31), ptot = __shfl_sync(0xffffffffu, pin, 31);
        s_pre[wib][lane] = sin - slen;
        s_ppre[wib][lane] = pin - plen;
        s_xb[wib][lane] = xb;
        s_xe[wib][lane] = xe;
        __syncwarp();
        for (u32 r0 = 0; r0 < stot; r0 += 128) {
            u32 yv[4], iv[4];
            u64 pv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const u32 r = r0 + 32u * u + lane;
                iv[u] = 0;
                yv[u] = kEmpty;
                if (r < stot) {
                    u32 mi = 0; // last member whose prefix <= r (empty lists share prefixes)
#pragma unroll
                    for (int step = 16; step > 0; step >>= 1)
                        if (mi + step < 32 && s_pre[wib][mi + step] <= r) mi += step;
                    iv[u] = mi;
                    pv[u] = s_xb[wib][mi] + (r - s_pre[wib][mi]);
                    yv[u] = g.adj[pv[u]];
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const u32 y = yv[u];
                if (y <= xmax) {
                    u32 lo = 0;
#pragma unroll
                    for (int step = 16; step > 0; step >>= 1)
                        if (xs[lo + step - 1] < y) lo += step;
                    if (xs[lo] == y) { // lo > i: y is above x_i
                        atomicOr(&rows[iv[u]], 1u << lo);
                        s_e[wib][iv[u]][lo] = g.eid[pv[u]];
                    }
                }
            }
        }
        for (u32 r0 = 0; r0 < ptot; r0 += 32) {
            const u32 r = r0 + lane;
            if (r < ptot) {
                u32 mi = 0;
#pragma unroll
                for (int step = 16; step > 0; step >>= 1)
                    if (mi + step < 32 && s_ppre[wib][mi + step] <= r) mi += step;
                const u32 j = mi + 1 + (r - s_ppre[wib][mi]);
                const u32 y = xs[j];
                const u64 b1 = s_xe[wib][mi];
                const u64 pp = lower_bound_dev<u32, u64>(g.adj, s_xb[wib][mi], b1, y);
                if (pp < b1 && g.adj[pp] == y) {
                    atomicOr(&rows[mi], 1u << j);
                    s_e[wib][mi][j] = g.eid[pp];
                }
            }
        }
        __syncwarp();
        // symmetrise: lane j collects the members whose upper row names j
        const u32 row = rows[lane];
        u32 col = 0;
#pragma unroll 8
        for (int j = 0; j < 32; ++j) {
            const u32 bb = __ballot_sync(0xffffffffu, (row >> j) & 1u);
            if (lane == (u32)j) col = bb;
        }
        const u32 full = row | col;
        __syncwarp();
        rows[lane] = full;
        if (MODE == kHPassCount && TL.rec) {
            // keep this vertex's H-edges (i | j << 16, e) for the sums pass: exact
            // reservation, vertices without triangles record an empty list
            const u32 mine = __popc(row);
            u32 pos = mine;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const u32 o = __shfl_up_sync(0xffffffffu, pos, d);
                if (lane >= (u32)d) pos += o;
            }
            const u32 nh = __shfl_sync(0xffffffffu, pos, 31);
            unsigned long long base = 0;
            if (lane == 0) {
                if (nh) {
                    base = atomicAdd(TL.count, (unsigned long long)nh);
                    if (base + nh > TL.cap) base = kNoList;
                }
                TL.base[idx] = base;
                TL.n[idx] = nh;
            }
            base = __shfl_sync(0xffffffffu, base, 0);
            if (base != kNoList) {
                uint2* out = TL.rec + base + (pos - mine);
                u32 bits = row;
                while (bits) {
                    const u32 j = __ffs(bits) - 1;
                    bits &= bits - 1;
                    *out++ = make_uint2((j << 16) | lane, s_e[wib][lane][j]);
                }
            }
        }
        __syncwarp();
        // phase 2: per H-edge (lane, j > lane)
        u32 tri = 0;
        u32 bits = MODE == kHPassCount ? full : row;
        while (bits) {
            const int j = __ffs(bits) - 1;
            bits &= bits - 1;
            if (MODE == kHPassCount) {
                const u32 c = __popc(full & rows[j]);
                tri += c;
                if ((u32)j > lane) {
                    const u32 e = s_e[wib][lane][j];
                    atomicAdd(&t[e], 1u);
                    if (c) atomic_add_i64(&part[2 * (u64)e], (i64)c);
                }
            } else {
                const u32 e = s_e[wib][lane][j];
                const u64 txy = t[e];
                atomic_add_i64(&part[2 * (u64)e + 1], -(i64)((u64)ta[lane] + ta[j]));
                atomicAdd(&acc[lane], (unsigned long long)(ta[j] + txy));
                atomicAdd(&acc[j], (unsigned long long)(ta[lane] + txy));
            }
        }
        __syncwarp();
        if (lane < k) {
            const u32 e = g.eid[ub + lane];
            if (MODE == kHPassCount) {
                const u32 deg = __popc(full);
                if (deg) atomicAdd(&t[e], deg);
                if (tri) atomic_add_i64(&part[2 * (u64)e], (i64)(tri >> 1));
            } else {
                if (acc[lane]) atomic_add_i64(&part[2 * (u64)e + 1], -(i64)acc[lane]);
            }
        }
        __syncwarp();
    }
}

// In-place exclusive scan of n u32 (generic pointer) by the whole block;
// returns the total.  Chunks of 2*blockDim with a running carry.
template <int THREADS>
__device__ u32 block_exclusive_scan(u32* a, u32 n) {
    using BlockScan = cub::BlockScan<u32, THREADS>;
    __shared__ typename BlockScan::TempStorage tmp;
    __shared__ u32 s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (u32 base = 0; base < n; base += 2 * THREADS) {
        u32 v[2];
        const u32 i0 = base + 2 * threadIdx.x;
        v[0] = i0 < n ? a[i0] : 0;
        v[1] = i0 + 1 < n ? a[i0 + 1] : 0;
        u32 total;
        BlockScan(tmp).ExclusiveSum(v, v, total);
        const u32 carry = s_carry;
        if (i0 < n) a[i0] = v[0] + carry;
        if (i0 + 1 < n) a[i0 + 1] = v[1] + carry;
        __syncthreads();
        if (threadIdx.x == 0) s_carry = carry + total;
        __syncthreads();
    }
    return s_carry;
}

// In-place exclusive scan of n u64 by the whole block; returns the total.
template <int THREADS>
__device__ u64 block_exclusive_scan64(u64* a, u32 n) {
    using BlockScan = cub::BlockScan<u64, THREADS>;
    __shared__ typename BlockScan::TempStorage tmp;
    __shared__ u64 s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (u32 base = 0; base < n; base += 2 * THREADS) {
        u64 v[2];
        const u32 i0 = base + 2 * threadIdx.x;
        v[0] = i0 < n ? a[i0] : 0;
        v[1] = i0 + 1 < n ? a[i0 + 1] : 0;
        u64 total;
        BlockScan(tmp).ExclusiveSum(v, v, total);
        const u64 carry = s_carry;
        if (i0 < n) a[i0] = v[0] + carry;
        if (i0 + 1 < n) a[i0 + 1] = v[1] + carry;
        __syncthreads();
        if (threadIdx.x == 0) s_carry = carry + total;
        __syncthreads();
    }
    return s_carry;
}

// k > 32: one block per vertex a.  Setup stages U(a) (xs) and its hash;
// phase 1 streams the members' upper lists (warps grab members), phase 2
// (kHPassCount) streams the H-edge list: popcount of the two rows, one t and
// one x7 credit per H-edge; phase 3 credits the edges (a, x_i).
// One vertex a of the block H-pass.  Inlined twice, with ws = the dynamic
// shared memory (k <= kHSmemMax: every workspace access compiles to LDS/STS/
// ATOMS) or the block's global scratch (larger k).

template <int MODE, int BLOG, typename Cand>
__device__ __forceinline__ void hpass_vertex(const DevGraph& g, u32* __restrict__ t, i64* __restrict__ part, u32* ws,
                                             Cand* cbuf, uint2* hlist, u32& s_nh, u32& s_mi, u32 a, u64 ub, u32 k,
                                             u32 W, u32 hl, u32 H, const TriList& TL, u64 idx, u64& s_base) {
    const u32 lane = lane_id();
    if (MODE == kHPassSums && TL.rec && TL.base[idx] != kNoList) {
        // stream this vertex's H-edge records: t of (x_i, x_j) gathered, the
        // (a, x) credits summed per member in shared memory
        u32* ta = ws;
        unsigned long long* acc = reinterpret_cast<unsigned long long*>(ws + ((k + 1) & ~1u));
        for (u32 i = threadIdx.x; i < k; i += blockDim.x) {
            ta[i] = t[g.eid[ub + i]];
            acc[i] = 0;
        }
        __syncthreads();
        const uint2* rec = TL.rec + TL.base[idx];
        const u32 nrec = TL.n[idx];
        constexpr int U = 4;
        for (u32 r0 = threadIdx.x; r0 < nrec; r0 += U * blockDim.x) {
            uint2 rv[U];
            u32 tv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const u32 r = r0 + u * blockDim.x;
                rv[u] = r < nrec ? rec[r] : make_uint2(0, kEmpty);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) tv[u] = rv[u].y != kEmpty ? t[rv[u].y] : 0u;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (rv[u].y == kEmpty) continue;
                const u32 i = rv[u].x & 0xffffu, j = rv[u].x >> 16;
                const u64 ti = ta[i], tj = ta[j], txy = tv[u];
                atomic_add_i64(&part[2 * (u64)rv[u].y + 1], -(i64)(ti + tj));
                atomicAdd(&acc[i], (unsigned long long)(tj + txy));
                atomicAdd(&acc[j], (unsigned long long)(ti + txy));
            }
        }
        __syncthreads();
        for (u32 i = threadIdx.x; i < k; i += blockDim.x)
            if (acc[i]) atomic_add_i64(&part[2 * (u64)g.eid[ub + i] + 1], -(i64)acc[i]);
        return;
    }
    u32* xs = ws;
    u32* tri = xs + k;                      // kHPassCount
    u32* rows = tri + k;                    // kHPassCount
    u32* ta = xs + k;                       // kHPassSums
    unsigned long long* acc = reinterpret_cast<unsigned long long*>(ws + ((2ull * k + 1) & ~1ull)); // kHPassSums
    // bitmap rows use an odd word stride RS so that the rows of different
    // members fall in different banks (phase 2 reads two arbitrary rows)
    const u32 RS = W | 1u;
    const u64 body = MODE == kHPassCount ? 2ull * k + (u64)k * RS : ((2ull * k + 1) & ~1ull) + 2ull * k;
    u32* bloom = ws + body;
    u32* hkey = bloom + bloom_words<BLOG>();
    unsigned short* hval = reinterpret_cast<unsigned short*>(hkey + H);
    u32* mb = hkey + H + H / 2; // member list bounds U(x_i) = [mb, me): loaded once,
    u32* me = mb + k;           // in parallel, instead of per member in phase 1
    for (u32 i = threadIdx.x; i < k; i += blockDim.x) {
        const u32 x = g.adj[ub + i];
        xs[i] = x;
        mb[i] = (u32)u_begin(g, x);
        me[i] = (u32)g.off[x + 1];
        if (MODE == kHPassCount) {
            tri[i] = 0;
        } else {
            ta[i] = t[g.eid[ub + i]];
            acc[i] = 0;
        }
    }
    if (MODE == kHPassCount)
        for (u64 w = threadIdx.x; w < (u64)k * RS; w += blockDim.x) rows[w] = 0;
    for (u32 h = threadIdx.x; h < H; h += blockDim.x) hkey[h] = kEmpty;
    for (u32 w = threadIdx.x; w < bloom_words<BLOG>(); w += blockDim.x) bloom[w] = 0;
    __syncthreads();
    for (u32 i = threadIdx.x; i < k; i += blockDim.x) {
        const u32 x = xs[i];
        u32 h = (x * 0x9E3779B1u) >> (32 - hl);
        while (atomicCAS(&hkey[h], kEmpty, x) != kEmpty) h = (h + 1) & (H - 1);
        hval[h] = (unsigned short)i;
        const u32 bb = bloom_bit<BLOG>(x);
        atomicOr(&bloom[bb >> 5], 1u << (bb & 31));
    }
    if (MODE == kHPassCount && threadIdx.x == 0) {
        // reserve C(k,2) records of the device-wide list up front, so phase 1
        // appends the H-edges straight into it (no per-block copy)
        u64 b = kNoList;
        if (TL.rec) {
            const u64 need = (u64)k * (k - 1) / 2;
            b = atomicAdd(TL.count, (unsigned long long)need);
            if (b + need > TL.cap) b = kNoList;
            TL.base[idx] = b;
        }
        s_base = b;
    }
    __syncthreads();
    uint2* const hout = (MODE == kHPassCount && s_base != kNoList) ? TL.rec + s_base : hlist;
    const u32 xmax = xs[k - 1];
    // phase 1: warps grab members i < k-1 and stream U(x_i)
    for (;;) {
        u32 i = 0;
        if (lane == 0) i = atomicAdd(&s_mi, 1u);
        i = __shfl_sync(0xffffffffu, i, 0);
        if (i + 1 >= k) break;
        const u64 xb = mb[i], xe = me[i];
        u64 acc_i = 0; // kHPassSums: credit of (a, x_i), summed over the member
        const u64 ti = MODE == kHPassSums ? (u64)ta[i] : 0;
        // one round of (hit, j = member index, e = edge id of (x_i, x_j)) with all lanes
        auto on_hits = [&](bool hit, u32 j, u32 e) {
            if (MODE == kHPassCount) {
                if (hit) {
                    atomicOr(&rows[(u64)i * RS + (j >> 5)], 1u << (j & 31));
                    atomicOr(&rows[(u64)j * RS + (i >> 5)], 1u << (i & 31));
                }
                const unsigned bal = __ballot_sync(0xffffffffu, hit);
                if (bal) {
                    u32 base = 0;
                    if (lane == 0) base = atomicAdd(&s_nh, (u32)__popc(bal));
                    base = __shfl_sync(0xffffffffu, base, 0);
                    if (hit) hout[base + __popc(bal & ((1u << lane) - 1u))] = make_uint2((j << 16) | i, e);
                }
            } else if (hit) {
                const u64 txy = t[e];
                const u64 tj = ta[j];
                atomic_add_i64(&part[2 * (u64)e + 1], -(i64)(ti + tj));
                acc_i += tj + txy;
                atomicAdd(&acc[j], (unsigned long long)(ti + txy));
            }
        };
        const u32 rem = k - 1 - i;
        if (xe - xb > (u64)kHProbeRatio * rem) {
            // U(x_i) much longer than the candidates x_j (j > i): probe each
            // candidate with a binary search instead of streaming the list
            for (u32 j0 = i + 1; j0 < k; j0 += 32) {
                const u32 j = j0 + lane;
                bool hit = false;
                u32 e = 0;
                if (j < k) {
                    const u32 y = xs[j];
                    const u64 pp = lower_bound_dev<u32, u64>(g.adj, xb, xe, y);
                    if (pp < xe && g.adj[pp] == y) {
                        hit = true;
                        e = g.eid[pp];
                    }
                }
                on_hits(hit, j, e);
            }
        } else
        for (u64 p0 = xb; p0 < xe; p0 += 32u * kHUnroll) {
            // kHUnroll coalesced rounds in flight; Bloom-filter them, then
            // compact the candidates into the warp's buffer so that the
            // exact lookups and the hit work run with full lanes
            u32 yv[kHUnroll];
#pragma unroll
            for (int u = 0; u < kHUnroll; ++u) {
                const u64 p = p0 + 32u * u + lane;
                yv[u] = p < xe ? __ldg(g.adj + p) : kEmpty;
            }
            u32 cand = 0;
#pragma unroll
            for (int u = 0; u < kHUnroll; ++u) {
                const u32 bb = bloom_bit<BLOG>(yv[u]);
                if (yv[u] <= xmax && ((bloom[bb >> 5] >> (bb & 31)) & 1u)) cand |= 1u << u; // kEmpty > xmax
            }
            const u32 c = __popc(cand);
            u32 pos = c;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const u32 o = __shfl_up_sync(0xffffffffu, pos, d);
                if (lane >= (u32)d) pos += o;
            }
            const u32 tot = __shfl_sync(0xffffffffu, pos, 31);
            if (tot == 0) continue;
            pos -= c;
#pragma unroll
            for (int u = 0; u < kHUnroll; ++u) {
                if ((cand >> u) & 1u) {
                    if constexpr (sizeof(Cand) == sizeof(uint2))
                        cbuf[pos] = make_uint2(yv[u], 32u * u + lane);
                    else
                        cbuf[pos] = (unsigned short)(32u * u + lane);
                    ++pos;
                }
            }
            __syncwarp();
            for (u32 q0 = 0; q0 < tot; q0 += 32) {
                const u32 q = q0 + lane;
                bool hit = false;
                u32 j = 0, e = 0;
                if (q < tot) {
                    u32 off, y;
                    if constexpr (sizeof(Cand) == sizeof(uint2)) {
                        off = cbuf[q].y;
                        y = cbuf[q].x;
                    } else {
                        off = cbuf[q];
                        y = __ldg(g.adj + p0 + off); // L1-hot: this warp just read it
                    }
                    u32 h = (y * 0x9E3779B1u) >> (32 - hl);
                    for (;;) {
                        const u32 kk = hkey[h];
                        if (kk == y) {
                            hit = true;
                            j = hval[h];
                            break;
                        }
                        if (kk == kEmpty) break;
                        h = (h + 1) & (H - 1);
                    }
                    if (hit) e = g.eid[p0 + off];
                }
                on_hits(hit, j, e);
            }
            __syncwarp();
        }
        if (MODE == kHPassSums) {
            acc_i = warp_sum_u64(acc_i);
            if (lane == 0 && acc_i) atomicAdd(&acc[i], (unsigned long long)acc_i);
        }
    }
    __syncthreads();
    if (MODE == kHPassCount) {
        // phase 2: stream the H-edges (kept in the device-wide list when it had room)
        const u32 nh = s_nh;
        if (TL.rec && threadIdx.x == 0) TL.n[idx] = nh;
        for (u32 h = threadIdx.x; h < nh; h += blockDim.x) {
            const uint2 he = hout[h];
            const u32 i = he.x & 0xffffu, j = he.x >> 16;
            const u32* ri = rows + (u64)i * RS;
            const u32* rj = rows + (u64)j * RS;
            u32 c = 0;
            for (u32 v = 0; v < W; ++v) c += __popc(ri[v] & rj[v]);
            atomicAdd(&t[he.y], 1u);
            if (c) {
                atomicAdd(&tri[i], c);
                atomicAdd(&tri[j], c);
                atomic_add_i64(&part[2 * (u64)he.y], (i64)c);
            }
        }
        __syncthreads();
        // phase 3: edges (a, x_i)
        for (u32 i = threadIdx.x; i < k; i += blockDim.x) {
            u32 deg = 0;
            const u32* ri = rows + (u64)i * RS;
            for (u32 v = 0; v < W; ++v) deg += __popc(ri[v]);
            const u32 e = g.eid[ub + i];
            if (deg) atomicAdd(&t[e], deg);
            if (tri[i]) atomic_add_i64(&part[2 * (u64)e], (i64)(tri[i] >> 1));
        }
    } else {
        for (u32 i = threadIdx.x; i < k; i += blockDim.x)
            if (acc[i]) atomic_add_i64(&part[2 * (u64)g.eid[ub + i] + 1], -(i64)acc[i]);
    }
}

template <int MODE, int KMAX>
__global__ void __launch_bounds__(HCfg<KMAX>::THREADS, HCfg<KMAX>::MINB)
k_hpass_block(DevGraph g, const u32* __restrict__ items, u64 n_items, unsigned long long* __restrict__ queue,
              u32* __restrict__ t, i64* __restrict__ part, u32* __restrict__ gscratch, u64 gstride,
              uint2* __restrict__ hlist_all, u64 hcap, TriList TL) {
    constexpr int BLOG = HCfg<KMAX>::BLOG;
    extern __shared__ u32 smem[];
    __shared__ unsigned long long s_idx;
    __shared__ u64 s_base;
    __shared__ u32 s_nh, s_mi;
    // per-warp candidate buffer: (y, offset) for the sums pass; the counting
    // pass keeps offsets only (its bitmap rows need the shared memory) and
    // re-reads y from L1
    // (the 1024-thread xl configuration keeps offsets in both modes: 48 KB static limit)
    using Cand = typename std::conditional<MODE == kHPassSums && HCfg<KMAX>::THREADS <= 512, uint2,
                                           unsigned short>::type;
    __shared__ Cand s_cbuf[HCfg<KMAX>::THREADS / 32][32 * kHUnroll];
    const u32 lane = lane_id();
    Cand* cbuf = s_cbuf[threadIdx.x >> 5];
    uint2* hlist = MODE == kHPassCount ? hlist_all + (u64)blockIdx.x * hcap : nullptr;
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) {
            s_idx = atomicAdd(queue, 1ull);
            s_nh = 0;
            s_mi = 0;
        }
        __syncthreads();
        const unsigned long long idx = s_idx;
        if (idx >= n_items) break;
        const u32 a = items[idx];
        const u64 ub = u_begin(g, a);
        const u32 k = (u32)(g.off[a + 1] - ub);
        const u32 W = (k + 31) >> 5;
        const u32 hl = hp_log(k), H = 1u << hl;
        if (MODE == kHPassSums) // one generic-pointer copy measured faster for the lighter sums pass
            hpass_vertex<MODE, BLOG>(g, t, part, k <= (u32)KMAX ? smem : gscratch + (u64)blockIdx.x * gstride,
                                     cbuf, hlist, s_nh, s_mi, a, ub, k, W, hl, H, TL, idx, s_base);
        else if (k <= (u32)KMAX)
            hpass_vertex<MODE, BLOG>(g, t, part, smem, cbuf, hlist, s_nh, s_mi, a, ub, k, W, hl, H, TL, idx, s_base);
        else
            hpass_vertex<MODE, BLOG>(g, t, part, gscratch + (u64)blockIdx.x * gstride, cbuf, hlist, s_nh, s_mi, a,
                                     ub, k, W, hl, H, TL, idx, s_base);
    }
}

// ------------------------------------------------------------------ cycles

__device__ __forceinline__ u32 hslot(u32 key) { return (key * 0x9E3779B1u) >> (32 - 10); }
static_assert(kHashSlots == 1024, "hslot assumes 1024 slots");

// Small tops: one warp per top vertex a, W[c] in a warp-private hash.
__global__ void __launch_bounds__(kCycleSmallWarps * 32)
k_cycle_small(DevGraph g, const u64* __restrict__ wpre, const u32* __restrict__ items, u64 n_items,
              unsigned long long* __restrict__ queue, i64* __restrict__ slot_acc) {
    extern __shared__ u32 smem[];
    const u32 lane = lane_id();
    const u32 wib = threadIdx.x >> 5;
    u32* keys = smem + wib * 2 * kHashSlots;
    u32* cnt = keys + kHashSlots;
    for (u32 i = lane; i < kHashSlots; i += 32) {
        keys[i] = kEmpty;
        cnt[i] = 0;
    }
    __syncwarp();
    for (;;) {
        unsigned long long idx = 0;
        if (lane == 0) idx = atomicAdd(queue, 1ull);
        idx = __shfl_sync(0xffffffffu, idx, 0);
        if (idx >= n_items) break;
        const u32 a = items[idx];
        const u64 E0 = g.loff[a], E1 = g.loff[a + 1];
        const u64 w0 = wpre[E0], w1 = wpre[E1];
        const u32 nw = (u32)(w1 - w0);
        // pass 1: W[c]++
        for (u32 base = 0; base < nw; base += 32) {
            u32 k = base + lane;
            if (k < nw) {
                u64 gi = w0 + k;
                u64 e = upper_bound_dev<u64, u64>(wpre, E0, E1 + 1, gi) - 1;
                u32 b = g.eu[e];
                u32 cv = g.adj[g.off[b] + (gi - wpre[e])];
                u32 h = hslot(cv);
                for (;;) {
                    u32 prev = atomicCAS(&keys[h], kEmpty, cv);
                    if (prev == kEmpty || prev == cv) break;
                    h = (h + 1) & (kHashSlots - 1);
                }
                atomicAdd(&cnt[h], 1u);
            }
        }
        __syncwarp();
        // pass 2: credit W[c]-1 to (b,c) and, summed per b, to (a,b)
        for (u32 base = 0; base < nw; base += 32) {
            u32 k = base + lane;
            u64 e = ~0ull, val = 0;
            if (k < nw) {
                u64 gi = w0 + k;
                e = upper_bound_dev<u64, u64>(wpre, E0, E1 + 1, gi) - 1;
                u32 b = g.eu[e];
                u64 slot = g.off[b] + (gi - wpre[e]);
                u32 cv = g.adj[slot];
                u32 h = hslot(cv);
                while (keys[h] != cv) h = (h + 1) & (kHashSlots - 1);
                val = cnt[h] - 1;
                if (val) atomic_add_i64(&slot_acc[slot], (i64)val);
            }
            u64 sum;
            bool tail = seg_tail_sum(e, val, &sum);
            if (k < nw && tail && sum) atomic_add_i64(&slot_acc[g.off[a] + (e - E0)], (i64)sum);
        }
        __syncwarp();
        for (u32 i = lane; i < kHashSlots; i += 32) {
            keys[i] = kEmpty;
            cnt[i] = 0;
        }
        __syncwarp();
    }
}

// Big tops: one block per top vertex a, dense W windows over c in shared
// memory (16-bit packed counters when |L(a)| < 65536: 64K c-values per
// window, else 32-bit: 32K).  Per window the non-empty runs
// N(b) n [lo,hi) of the lower neighbours b are compacted (flag scan) and
// prefix-summed in per-block global scratch; the wedges are then flattened
// block-wide: each warp takes rounds of 32 consecutive wedges, finds the
// round's first run with one warp-uniform binary search and each lane's run
// among the next 32 (all non-empty) with a 5-step shuffle search.  Credits go
// to per-adjacency-slot accumulators (consecutive wedges of a run are
// consecutive slots), folded into edge rows by k_fold_slots.

// Shared-space access with a 32-bit address computed once per kernel (the
// generic-pointer form re-derives the shared window base per access).
__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void red_shared_add(u32 addr, u32 v) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ u32 ld_shared(u32 addr) {
    u32 v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
// RED.ADD.U64 to global issued under a predicate (no branch around it)
__device__ __forceinline__ void red_add_u64_if(i64* p, u64 v) {
    asm volatile("{ .reg .pred q; setp.ne.u64 q, %1, 0; @q red.global.add.u64 [%0], %1; }" ::"l"(p), "l"(v)
                 : "memory");
}

// Packed window counters: 2^cl counters of (32 >> cl) bits per word.  The
// width follows the degree tier of the window's c ids (internal ids ascend
// with degree): W_a[c] <= deg(c), so ids with degree < 4 take 2-bit counters,
// < 16 4-bit, < 256 8-bit, < 65536 16-bit, the rest 32-bit -- the window over
// low-degree ids is up to 16x wider than a 32-bit one.
__device__ __forceinline__ void w_inc(u32* W, u32 i, u32 cl) {
    atomicAdd(&W[i >> cl], 1u << ((i & ((1u << cl) - 1u)) << (5 - cl)));
}
__device__ __forceinline__ u32 w_get(const u32* W, u32 i, u32 cl) {
    const u32 v = W[i >> cl] >> ((i & ((1u << cl) - 1u)) << (5 - cl));
    return cl == 0 ? v : v & ((1u << (32u >> cl)) - 1u);
}

// first index in [lo, hi) with a[idx] >= x, galloping from lo: runs inside a
// window are usually a handful of entries, so this costs ~log2(run) loads.
__device__ __forceinline__ u64 gallop_lower_bound(const u32* __restrict__ a, u64 lo, u64 hi, u32 x) {
    if (lo >= hi || a[lo] >= x) return lo;
    u64 step = 1, base = lo;
    for (;;) {
        const u64 probe = base + step;
        if (probe >= hi) return lower_bound_dev<u32, u64>(a, base + 1, hi, x);
        if (a[probe] >= x) return lower_bound_dev<u32, u64>(a, base + 1, probe, x);
        base = probe;
        step <<= 1;
    }
}

constexpr int kNcBatch = 8; // b's whose window test loads are issued together

#ifdef GL_CYCLE_PROF
__device__ unsigned long long g_cycle_prof[32]; // [0..10] dense windows, [16..26] mid hash,
                                                // [12] uniform rounds, [13] mixed rounds (dense)
#endif

// First index in [lo, hi) with a[idx] >= x, searching outward from a hint
// (the previous window's run end of the same row): a doubling probe towards
// the answer from the hint, then a binary search -- ~2 log2 |error| loads.
__device__ __forceinline__ u64 gallop_from(const u32* __restrict__ a, u64 lo, u64 hi, u64 hint, u32 x) {
    if (hint <= lo || hint >= hi) return gallop_lower_bound(a, lo, hi, x);
    if (a[hint] < x) return gallop_lower_bound(a, hint + 1, hi, x);
    // answer in [lo, hint]: double backwards
    u64 r = hint, step = 1;
    for (;;) {
        if (r < lo + step) return lower_bound_dev<u32, u64>(a, lo, r, x);
        const u64 p = r - step;
        if (a[p] < x) return lower_bound_dev<u32, u64>(a, p + 1, r, x);
        r = p;
        step <<= 1;
    }
}

// per-block scratch layout (cap = dmax + 2 entries each, cap even)
struct BigScratch {
    u32 *cur, *hpos, *rend, *pre, *rj, *rs, *nextc, *rwin, *plen;
    u64* rb;
};
// compacted runs of one window: wedge prefix pre[nnz+1], first adjacency slot
// rs[q] (u32: 2m < 2^32 is checked on the host), lower-neighbour index rj[q];
// in shared memory when nnz fits, else in the block's global scratch
struct RunMeta {
    u32 *pre, *rs, *rj;
};
__device__ __forceinline__ BigScratch big_scratch(u32* base, u32 cap) {
    BigScratch s;
    s.cur = base;
    s.hpos = base + cap;
    s.rend = base + 2 * (u64)cap;
    s.pre = base + 3 * (u64)cap;              // cap + 1 entries
    s.rj = base + 4 * (u64)cap + 1;
    s.rs = base + 5 * (u64)cap + 1;
    s.rb = reinterpret_cast<u64*>(base + ((6 * (u64)cap + 2) & ~1ull)); // 8B aligned (base is)
    s.nextc = reinterpret_cast<u32*>(s.rb + cap); // c at the cursor (kEmpty: row done)
    s.rwin = s.nextc + cap;                        // window of b's last recorded run
    s.plen = s.rwin + cap;                         // length of b's last run (search hint)
    return s;
}
__host__ __device__ inline u64 big_scratch_words(u32 cap) { return 11ull * cap + 8; }


// W[c] table of one block: dense window over c in [lo, lo+span) (big tops)
// or an open-addressing hash over all c < a (mid tops, HASH).  Hash keys are
// u32 (kEmpty = free), counts u16 packed two per word.
// cycle block kernel kinds: 0 dense windows (big tops), 1 block hash with
// 2^15 slots (mid tops), 2 block hash with 2^13 slots and four 256-thread
// blocks per SM (small-mid tops: their fixed per-top latency overlaps)
template <int KIND> struct Cyc;
template <> struct Cyc<0> {
    static constexpr bool HASH = false;
    static constexpr int THREADS = kBigThreads, MINB = kBigBlocksPerSM;
    static constexpr u32 LOG = 0, WORDS = kWindow, META = 7168;
};
template <> struct Cyc<1> {
    static constexpr bool HASH = true;
    static constexpr int THREADS = kMidThreads, MINB = 1;
    static constexpr u32 LOG = kMidLog, WORDS = (1u << kMidLog) * 3 / 2, META = 2048;
};
template <> struct Cyc<2> {
    static constexpr bool HASH = true;
    static constexpr int THREADS = kSmidThreads, MINB = 4;
    static constexpr u32 LOG = kSmidLog, WORDS = (1u << kSmidLog) * 3 / 2, META = 256;
};
template <int KIND> __host__ __device__ constexpr u32 cyc_smem_words() {
    return Cyc<KIND>::WORDS + 3 * Cyc<KIND>::META + 1;
}


template <int KIND>
__device__ __forceinline__ void tab_inc(u32* W, u32 c, u32 lo, u32 cl) {
    constexpr u32 NS = 1u << Cyc<KIND>::LOG;
    if (Cyc<KIND>::HASH) {
        u32* keys = W;
        u32 h = (c * 0x9E3779B1u) >> (32 - Cyc<KIND>::LOG);
        for (;;) {
            const u32 k = keys[h];
            if (k == c) break;
            if (k == kEmpty) {
                const u32 prev = atomicCAS(&keys[h], kEmpty, c);
                if (prev == kEmpty || prev == c) break;
            }
            h = (h + 1) & (NS - 1);
        }
        atomicAdd(&W[NS + (h >> 1)], 1u << ((h & 1) << 4));
    } else {
        w_inc(W, c - lo, cl);
    }
}
template <int KIND>
__device__ __forceinline__ u32 tab_get(const u32* W, u32 c, u32 lo, u32 cl) {
    constexpr u32 NS = 1u << Cyc<KIND>::LOG;
    if (Cyc<KIND>::HASH) {
        u32 h = (c * 0x9E3779B1u) >> (32 - Cyc<KIND>::LOG);
        while (W[h] != c) h = (h + 1) & (NS - 1);
        return (W[NS + (h >> 1)] >> ((h & 1) << 4)) & 0xffffu;
    } else {
        return w_get(W, c - lo, cl);
    }
}
// dense windows only: the hash is always bulk-cleared (a deleted key would
// break the probe chains of the clears still to come)
__device__ __forceinline__ void tab_clear_one(u32* W, u32 c, u32 lo, u32 cl) { W[(c - lo) >> cl] = 0; }

template <int KIND, int PASS>
__device__ __forceinline__ void wedge_op(u32* W, u32 cv, u32 lo, u32 cl, i64* __restrict__ slot_acc, u64 slot,
                                         u64& val) {
    if (!Cyc<KIND>::HASH) { // dense window: 32-bit shared addresses, predicated RED
        const u32 ci = cv - lo;
        const u32 addr = smem_u32(W) + ((ci >> cl) << 2);
        const u32 sh = (ci & ((1u << cl) - 1u)) << (5 - cl);
        if (PASS == 0) {
            red_shared_add(addr, 1u << sh);
        } else if (PASS == 1) {
            const u32 w = ld_shared(addr) >> sh;
            const u32 v = (cl == 0 ? w : w & ((1u << (32u >> cl)) - 1u)) - 1u;
            red_add_u64_if(&slot_acc[slot], (u64)v);
            val = v;
        } else {
            W[ci >> cl] = 0;
        }
        return;
    }
    if (PASS == 0) {
        tab_inc<KIND>(W, cv, lo, cl);
    } else if (PASS == 1) {
        const u32 v = tab_get<KIND>(W, cv, lo, cl) - 1u;
        if (v) atomic_add_i64(&slot_acc[slot], (i64)v);
        val = v;
    } else {
        tab_clear_one(W, cv, lo, cl);
    }
}

// Last index in [0, n) with a[idx] <= x (a non-decreasing, a[0] <= x), by the
// whole warp: 32 probes per step, so log32(n) dependent loads instead of log2(n).
__device__ __forceinline__ u32 warp_upper_bound(const u32* a, u32 n, u32 x) {
    const u32 lane = lane_id();
    u32 lo = 0, hi = n;
    while (hi - lo > 32u) {
        const u32 step = (hi - lo + 31u) >> 5;
        const u32 idx = lo + lane * step;
        const bool ok = idx < hi && a[idx] <= x;
        const unsigned bal = __ballot_sync(0xffffffffu, ok);
        lo += (31u - __clz(bal)) * step;
        hi = lo + step < hi ? lo + step : hi;
    }
    const u32 idx = lo + lane;
    const unsigned bal = __ballot_sync(0xffffffffu, idx < hi && a[idx] <= x);
    return lo + 31u - __clz(bal);
}

// One pass over a warp's range [kb, ke) of a window's flattened wedge list
// (compacted runs q, S.pre = wedge prefix, run q = adjacency slots
// [S.rs[q], S.rs[q] + len)).  Stretches of full 32-wedge rounds inside one
// run take the uniform path: slot = base + lane, four rounds of loads in
// flight, the (a,b) credit kept per lane and warp-reduced once per stretch.
// Rounds that straddle runs take the mixed path: each lane finds its run
// among the next 32 starts by a 5-step shuffle search and the (a,b) credit is
// a segmented shuffle sum whose tail lanes issue the RED.
//   PASS 0: W[c]++     PASS 1: credit W[c]-1 to (b,c) and, summed, to (a,b)
//   PASS 2: W[c] = 0 (sparse clear of a dense window)
constexpr int kUnroll = 8; // uniform-path rounds with loads in flight per lane

template <int KIND, int PASS>
__device__ __forceinline__ void window_pass(const DevGraph& g, const RunMeta& S, u32 nnz, u32 kb, u32 ke, u32* W,
                                            u32 lo, u32 cl, u64 abase, i64* __restrict__ slot_acc) {
    const u32 lane = lane_id();
    if (kb >= ke) return;
    u32 bs = warp_upper_bound(S.pre, nnz + 1, kb);
    u32 k0 = kb;
    while (k0 < ke) {
        u32 e1 = S.pre[bs + 1];
        while (e1 <= k0) e1 = S.pre[++bs + 1];
        const u32 stop = e1 < ke ? e1 : ke;
        if (stop - k0 >= 32u) {
            // uniform stretch of full rounds inside run bs
            const u32 nfull = (stop - k0) >> 5;
#ifdef GL_CYCLE_PROF_ROUNDS
            if (KIND == 0 && PASS == 1 && lane_id() == 0) atomicAdd(&g_cycle_prof[12], (unsigned long long)nfull);
#endif
            const u64 sbase = (u64)S.rs[bs] + (k0 - S.pre[bs]) + lane;
            u64 acc = 0;
            // software pipeline: the next kHalf rounds' loads are in flight
            // while the current kHalf rounds update the window
            constexpr int kHalf = kUnroll / 2;
            u32 cv[kHalf];
#pragma unroll
            for (int u = 0; u < kHalf; ++u) cv[u] = (u32)u < nfull ? __ldg(g.adj + sbase + 32u * u) : kEmpty;
            for (u32 r = 0; r < nfull; r += kHalf) {
                u32 nx[kHalf];
#pragma unroll
                for (int u = 0; u < kHalf; ++u)
                    nx[u] = r + kHalf + u < nfull ? __ldg(g.adj + sbase + 32u * (r + kHalf + u)) : kEmpty;
#pragma unroll
                for (int u = 0; u < kHalf; ++u) {
                    if (cv[u] != kEmpty) {
                        u64 v = 0;
                        wedge_op<KIND, PASS>(W, cv[u], lo, cl, slot_acc, sbase + 32u * (r + u), v);
                        acc += v;
                    }
                }
#pragma unroll
                for (int u = 0; u < kHalf; ++u) cv[u] = nx[u];
            }
            if (PASS == 1) {
                acc = warp_sum_u64(acc);
                if (lane == 0 && acc) atomic_add_i64(&slot_acc[abase + S.rj[bs]], (i64)acc);
            }
            k0 += nfull << 5;
        } else {
            // mixed round [k0, k0 + 32): runs bs, bs+1, ... start at pre[bs+j];
            // one OR-reduction gives the bitmask of run starts inside the round,
            // from which every lane reads its run (popcount), its offset and
            // its segment (highest start at or below it)
#ifdef GL_CYCLE_PROF_ROUNDS
            if (KIND == 0 && PASS == 1 && lane_id() == 0) atomicAdd(&g_cycle_prof[13], 1ull);
#endif
            const u32 k = k0 + lane;
            const bool valid = k < ke;
            const u32 pi = bs + lane <= nnz ? S.pre[bs + lane] : 0xffffffffu;
            const u32 rel = pi - k0; // >= 1 for lanes >= 1 (pre strictly increasing)
            const u32 starts = __reduce_or_sync(0xffffffffu, (lane > 0 && rel < 32u) ? 1u << rel : 0u);
            const u32 le = starts & (0xffffffffu >> (31 - lane)); // starts at or below this lane
            const u32 owner = __popc(le);
            const u32 q = bs + owner;
            const u32 seg0 = owner ? 31u - __clz(le) : 0u;
            const u32 pi0 = __shfl_sync(0xffffffffu, pi, 0); // all lanes: full-mask shuffle
            const u32 off = owner ? lane - seg0 : k - pi0;
            u64 v = 0;
            if (valid) {
                const u64 slot = (u64)S.rs[q] + off;
                wedge_op<KIND, PASS>(W, __ldg(g.adj + slot), lo, cl, slot_acc, slot, v);
            }
            if (PASS == 1) {
                const bool tail = valid && (lane == 31 || k + 1 == ke || ((starts >> (lane + 1)) & 1u));
                if (cl) {
                    // counters of <= 16 bits: the segment sum fits u32
                    u32 v32 = (u32)v;
#pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {
                        const u32 t = __shfl_up_sync(0xffffffffu, v32, d);
                        if (lane >= seg0 + (u32)d) v32 += t;
                    }
                    if (tail && v32) atomic_add_i64(&slot_acc[abase + S.rj[q]], (i64)v32);
                } else {
#pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {
                        const u64 t = __shfl_up_sync(0xffffffffu, v, d);
                        if (lane >= seg0 + (u32)d) v += t;
                    }
                    if (tail && v) atomic_add_i64(&slot_acc[abase + S.rj[q]], (i64)v);
                }
            }
            k0 += 32;
            bs = __shfl_sync(0xffffffffu, q, 31);
        }
    }
}

// Guided self-scheduling of a window pass: a warp grabs about 1/(2*nwarps) of
// the wedges still unclaimed (at most 8192, at least 64), so the grabs shrink
// towards the end of the pass and the block's barrier waits for a short tail.
__device__ __forceinline__ u32 grab_size(u32 remaining, u32 nwarps) {
    u32 g = remaining / (2u * nwarps);
    g = g < 8192u ? g : 8192u;
    g = (g + 31u) & ~31u;
    return g > 64u ? g : 64u;
}

// Mid and big tops: one block per top a (persistent blocks, atomic queue over
// the cost-sorted list).  Big tops (!HASH) sweep c in dense shared-memory
// windows (16-bit packed counters while |L(a)| < 65536: 2*kWindow c-values
// per window, else 32-bit: kWindow); per window the non-empty runs
// N(b) n [lo,hi) of the lower neighbours b are found by galloping from each
// b's cursor, compacted (flag scan) and prefix-summed -- in shared memory when
// they fit (RunMeta) -- and walked by window_pass, warps grabbing kGrab-wedge
// ranges from a shared counter so that the cost differences between long-run
// and short-run ranges do not stall the block at the pass barriers.  Mid tops
// (HASH, <= kMidWedges wedges) take all c < a at once in a block hash: runs
// are the full row prefixes N(b) n [0,a), one "window", no cursors.  Credits
// go to per-adjacency-slot accumulators (consecutive wedges of a run are
// consecutive slots), folded into edge rows by k_fold_slots.
template <int KIND, int PASS>
__device__ __forceinline__ void grab_pass(const DevGraph& g, const RunMeta& M, u32 nnz, u32 T, u32* counter, u32* W,
                                          u32 lo, u32 cl, u64 abase, i64* __restrict__ slot_acc) {
    const u32 nwarps = blockDim.x >> 5;
    for (;;) {
        u32 k0 = 0, grab = 0;
        if (lane_id() == 0) {
            const u32 seen = *(volatile u32*)counter;
            grab = grab_size(seen < T ? T - seen : 0u, nwarps);
            k0 = atomicAdd(counter, grab);
        }
        k0 = __shfl_sync(0xffffffffu, k0, 0);
        grab = __shfl_sync(0xffffffffu, grab, 0);
        if (k0 >= T) break;
        window_pass<KIND, PASS>(g, M, nnz, k0, k0 + grab < T ? k0 + grab : T, W, lo, cl, abase, slot_acc);
    }
}

template <int KIND>
__global__ void __launch_bounds__(Cyc<KIND>::THREADS, Cyc<KIND>::MINB)
k_cycle_block(DevGraph g, const u32* __restrict__ items, u64 n_items, unsigned long long* __restrict__ queue,
              i64* __restrict__ slot_acc, u32* __restrict__ gscratch, u32 cap, uint4 tiers) {
    constexpr bool HASH = Cyc<KIND>::HASH;
    constexpr int THREADS = Cyc<KIND>::THREADS;
    constexpr u32 kWords = Cyc<KIND>::WORDS, kMeta = Cyc<KIND>::META, kSlots = 1u << Cyc<KIND>::LOG;
    extern __shared__ u32 W[]; // kWords table words, then the run metadata
    __shared__ unsigned long long s_idx;
    __shared__ u32 s_next, s_work[3];
    BigScratch S = big_scratch(gscratch + (u64)blockIdx.x * ((big_scratch_words(cap) + 1) & ~1ull), cap);
    const RunMeta Msm{W + kWords, W + kWords + kMeta + 1, W + kWords + 2 * kMeta + 1};
    const RunMeta Mgl{S.pre, S.rs, S.rj};
    for (u32 i = threadIdx.x; i < kWords; i += THREADS) W[i] = (HASH && i < kSlots) ? kEmpty : 0u;
#ifdef GL_CYCLE_PROF
    // make prof: per-phase clock64 totals (thread 0, between barriers): 0 setup,
    // 6 gallop, 1 scan, 2 compaction, 3 pass 0, 4 pass 1, 7 clear, 5 grab;
    // 8 windows, 9 wedges, 10 tops (scripts/cycle_phases.py)
    unsigned long long pf[11] = {0};
    unsigned long long pt = clock64();
#define GL_PROF_MARK(k)                                   \
    if (threadIdx.x == 0) {                               \
        const unsigned long long now_ = clock64();        \
        pf[k] += now_ - pt;                               \
        pt = now_;                                        \
    }
#define GL_PROF_SYNC_MARK(k) \
    __syncthreads();         \
    GL_PROF_MARK(k)
#define GL_PROF_ADD(k, v) \
    if (threadIdx.x == 0) pf[k] += (v);
#else
#define GL_PROF_MARK(k)
#define GL_PROF_SYNC_MARK(k)
#define GL_PROF_ADD(k, v)
#endif
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) s_idx = atomicAdd(queue, 1ull);
        __syncthreads();
        const unsigned long long idx = s_idx;
        if (idx >= n_items) break;
        GL_PROF_MARK(5);
        const u32 a = items[idx];
        const u64 E0 = g.loff[a];
        const u32 nb = (u32)(g.loff[a + 1] - E0);
        const u64 abase = g.off[a]; // slot of (a, b_j) is abase + j: L(a) is the row prefix

        if (threadIdx.x == 0) s_next = HASH ? 0u : kEmpty;
        __syncthreads();
        // per-b row base and run end (|N(b) n [0,a)| = epos), cursors at 0
        for (u32 j = threadIdx.x; j < nb; j += THREADS) {
            const u64 e = E0 + j;
            const u64 rb = g.off[g.eu[e]];
            const u32 re = g.epos[e];
            S.rb[j] = rb;
            S.rend[j] = re;
            S.cur[j] = 0;
            const u32 c = re > 0 ? g.adj[rb] : kEmpty;
            S.nextc[j] = c;
            S.rwin[j] = kEmpty;
            S.plen[j] = 0;
            if (!HASH && c != kEmpty) atomicMin(&s_next, c);
        }
        __syncthreads();
        GL_PROF_MARK(0);
        GL_PROF_ADD(10, 1);
        // Windows from the smallest c on.  Each b keeps its cursor and the c
        // value under it (nextc), so a window only gallops the b's whose next c
        // falls inside it; for the others one coalesced nextc load suffices.
        u32 win = 0;
        for (u32 lo = s_next, hi = 0; lo < a; lo = hi, ++win) {
            // window [lo, hi): inside one degree tier, counters of that tier's width
            u32 cl = 1, tend = a;
            if (!HASH) {
                cl = lo < tiers.x ? 4u : lo < tiers.y ? 3u : lo < tiers.z ? 2u : lo < tiers.w ? 1u : 0u;
                tend = lo < tiers.x ? tiers.x : lo < tiers.y ? tiers.y : lo < tiers.z ? tiers.z : lo < tiers.w ? tiers.w : a;
            }
            u64 span = (u64)kWindow << cl;
            // keep nb * span < 2^31: window wedge counts and indices are u32
            if ((u64)nb * span >= (1ull << 31)) span = ((1ull << 31) / nb) & ~31ull;
            hi = HASH ? a : (u32)std::min<u64>(std::min<u64>((u64)lo + span, (u64)tend), (u64)a);

            // run ends of the b's with a c in [lo, hi); runs are ordered
            // thread-major (thread t owns b = t + i*THREADS), so one block scan
            // of per-thread (runs, wedges) places them
            u32 my_runs = 0, my_wedges = 0;
            for (u32 j0 = threadIdx.x; j0 < nb; j0 += kNcBatch * THREADS) {
                u32 nc[kNcBatch];
#pragma unroll
                for (int u = 0; u < kNcBatch; ++u) {
                    const u32 j = j0 + u * THREADS;
                    nc[u] = j < nb ? S.nextc[j] : kEmpty;
                }
#pragma unroll
                for (int u = 0; u < kNcBatch; ++u) {
                    if (nc[u] >= hi) continue; // no c of b in this window (kEmpty >= hi)
                    const u32 j = j0 + u * THREADS;
                    const u32 c0 = S.cur[j], re = S.rend[j];
                    const u64 rb = S.rb[j];
                    u32 h = re;
                    if (!HASH) {
                        const u32 pl = S.plen[j];
                        h = (u32)(gallop_from(g.adj, rb + c0, rb + re, rb + c0 + (pl ? pl - 1 : 0), hi) - rb);
                        S.plen[j] = h - c0;
                    }
                    S.hpos[j] = c0; // run start
                    S.rwin[j] = win;
                    S.cur[j] = h;
                    S.nextc[j] = h < re ? g.adj[rb + h] : kEmpty;
                    ++my_runs;
                    my_wedges += h - c0;
                }
            }
            GL_PROF_SYNC_MARK(6);
            u64 tot;
            u64 mine = ((u64)my_runs << 32) | my_wedges;
            {
                using BlockScan = cub::BlockScan<u64, THREADS>;
                __shared__ typename BlockScan::TempStorage tmp;
                BlockScan(tmp).ExclusiveSum(mine, mine, tot);
            }
            const u32 nnz = (u32)(tot >> 32), T = (u32)tot;
            GL_PROF_MARK(1);
            GL_PROF_ADD(8, 1);
            GL_PROF_ADD(9, T);
            const RunMeta M = nnz <= kMeta ? Msm : Mgl;
            if (my_runs) {
                u32 q = (u32)(mine >> 32), w = (u32)mine;
                for (u32 j0 = threadIdx.x; j0 < nb && q < (u32)(mine >> 32) + my_runs; j0 += kNcBatch * THREADS) {
                    u32 rw[kNcBatch];
#pragma unroll
                    for (int u = 0; u < kNcBatch; ++u) {
                        const u32 j = j0 + u * THREADS;
                        rw[u] = j < nb ? S.rwin[j] : kEmpty;
                    }
#pragma unroll
                    for (int u = 0; u < kNcBatch; ++u) {
                        if (rw[u] != win) continue;
                        const u32 j = j0 + u * THREADS;
                        const u32 c0 = S.hpos[j], h = S.cur[j];
                        M.rj[q] = j;
                        M.rs[q] = (u32)(S.rb[j] + c0);
                        M.pre[q] = w;
                        ++q;
                        w += h - c0;
                    }
                }
            }
            if (threadIdx.x == 0) M.pre[nnz] = T;
            if (threadIdx.x < 3) s_work[threadIdx.x] = 0;
            __syncthreads();
            GL_PROF_MARK(2);
            if (T) {
                const bool bulk_clear = HASH || T > kWords / 8;
                {
                    if (nnz <= kMeta) // shared-memory metadata: LDS in the walk
                        grab_pass<KIND, 0>(g, Msm, nnz, T, &s_work[0], W, lo, cl, abase, slot_acc);
                    else
                        grab_pass<KIND, 0>(g, Mgl, nnz, T, &s_work[0], W, lo, cl, abase, slot_acc);
                }
                __syncthreads();
                GL_PROF_MARK(3);
                {
                    if (nnz <= kMeta)
                        grab_pass<KIND, 1>(g, Msm, nnz, T, &s_work[1], W, lo, cl, abase, slot_acc);
                    else
                        grab_pass<KIND, 1>(g, Mgl, nnz, T, &s_work[1], W, lo, cl, abase, slot_acc);
                }
                __syncthreads();
                GL_PROF_MARK(4);
                if (bulk_clear) {
                    const u32 words = HASH ? kWords : (hi - lo + (1u << cl) - 1u) >> cl;
                    for (u32 i = threadIdx.x; i < words; i += THREADS) W[i] = (HASH && i < kSlots) ? kEmpty : 0u;
                } else if (!HASH) {
                    if (nnz <= kMeta)
                        grab_pass<KIND, 2>(g, Msm, nnz, T, &s_work[2], W, lo, cl, abase, slot_acc);
                    else
                        grab_pass<KIND, 2>(g, Mgl, nnz, T, &s_work[2], W, lo, cl, abase, slot_acc);
                }
            }
            GL_PROF_SYNC_MARK(7);
            __syncthreads();
            GL_PROF_MARK(5);
        }
    }
#ifdef GL_CYCLE_PROF
    if (threadIdx.x == 0)
        for (int k = 0; k < 11; ++k) atomicAdd(&g_cycle_prof[k + (KIND ? 16 : 0)], pf[k]);
#endif
}

// y(e) += the two adjacency-slot accumulators of edge e (v's row, u's row).
__global__ void k_fold_slots(DevGraph g, const i64* __restrict__ slot_acc, i64* __restrict__ part) {
    for (u64 e = blockIdx.x * (u64)blockDim.x + threadIdx.x; e < g.m; e += (u64)gridDim.x * blockDim.x) {
        const u32 v = g.ev[e], u = g.eu[e];
        const i64 s = slot_acc[g.off[v] + (e - g.loff[v])] + slot_acc[g.off[u] + g.epos[e]];
        if (s) part[2 * e + 1] += s;
    }
}

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

__global__ void k_seq(u32* __restrict__ ids, u64 n) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        ids[i] = (u32)i;
}

// H-pass work list key: big-k (k > 32) items first, each class ordered by its
// streaming cost s1(a) = sum_{i<k-1} |U(x_i)| (adjacency entries read).
// Work lists only need an approximate cost order: keys are a 4-bit-mantissa
// log2 of the cost (10 bits) under a class bit, so the radix sort runs over
// 17 key bits instead of 64.
constexpr u32 kKeyBits = 17, kClassBit = 1u << 16;
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
            const u64 ul = g.off[x + 1] - (g.off[x] + g.lcnt[x]), pr = (u64)kHProbeRatio * (k - 1 - i);
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

// cycle work list key = wedges of top a; classes big (> kMidWedges, dense
// windows), mid (> kSmallWedges, block hash), small (warp hash)
__global__ void k_top_keys(DevGraph g, const u64* __restrict__ wpre, u32* __restrict__ keys,
                           unsigned long long* __restrict__ n_big, unsigned long long* __restrict__ n_mid,
                           unsigned long long* __restrict__ n_smid, unsigned long long* __restrict__ n_small) {
    unsigned long long lb = 0, lm = 0, lq = 0, ls = 0;
    for (u64 a = blockIdx.x * (u64)blockDim.x + threadIdx.x; a < g.n; a += (u64)gridDim.x * blockDim.x) {
        u64 w = wpre[g.loff[a + 1]] - wpre[g.loff[a]];
        u32 cls = 0; // exact class boundaries: class above the log cost
        if (w > kMidWedges) {
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
// 14 max k, 17 s1, 18 max s1, 19 H-edge bound, 20 H-edge list fill, 22-23 tiers
constexpr int kCounters = 32;

// rank's share of a cost-sorted list: sorted positions p with p % world == rank
__global__ void k_take_rank(const u32* __restrict__ sorted, u64 begin, u64 count, int rank, int world,
                            u32* __restrict__ out) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x;; i += (u64)gridDim.x * blockDim.x) {
        u64 p = (u64)rank + i * (u64)world;
        if (p >= count) break;
        out[i] = sorted[begin + p];
    }
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

template <typename T>
void dev_exclusive_scan(DevBuf& tmp, const T* in, T* out, u64 n, cudaStream_t s) {
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

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device, size)
template <typename K> void smem_attr(K* kernel, size_t smem, int device) {
    static std::mutex mu;
    static std::set<std::tuple<const void*, int, size_t>> done;
    std::lock_guard<std::mutex> lk(mu);
    if (done.insert({reinterpret_cast<const void*>(kernel), device, smem}).second)
        GL_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
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

std::atomic<int> g_overlap{1}; // run the cycle pass concurrently with the H-pass (gl_set_overlap)

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
    cs.launches = 0;
    cs.began = false;
    cs.mid_done = false;
    cs.rank = rank;
    cs.world = world;
    std::memset(cs.work, 0, sizeof(cs.work));

    cs.t.alloc((m + 1) * sizeof(u32));
    cs.wpre.alloc((m + 1) * sizeof(u64));
    cs.acc.alloc(96 * sizeof(u64));
    cs.keys.alloc((std::max(m, n) + 1) * 2 * sizeof(u64)); // key in/out
    cs.items2.alloc((std::max(m, n) + 1) * 2 * sizeof(u32)); // id in/out
    const u64 plen = ((m + world - 1) / world) * (u64)world;
    if (plen) GL_CUDA(cudaMemsetAsync(d_partials, 0, 2 * plen * sizeof(i64), s));
    GL_CUDA(cudaMemsetAsync(cs.t.p, 0, (m + 1) * sizeof(u32), s));
    cs.slots.alloc((2 * m + 1) * sizeof(i64));
    GL_CUDA(cudaMemsetAsync(cs.slots.p, 0, (2 * m + 1) * sizeof(i64), s));
    unsigned long long* counters = cs.acc.as<unsigned long long>() + 40; // queues + counts
    GL_CUDA(cudaMemsetAsync(counters, 0, kCounters * sizeof(u64), s));

    // The H-pass (stream s) and the cycle pass (cs.s2, forked after the wedge
    // prefix) are independent and run concurrently; count_mid joins them.
    if (cs.s2) GL_CUDA(cudaStreamSynchronize(cs.s2)); // a previous, un-joined cycle pass
    if (!cs.s2) {
        GL_CUDA(cudaStreamCreateWithFlags(&cs.s2, cudaStreamNonBlocking));
        for (int i = 0; i < 8; ++i) GL_CUDA(cudaEventCreate(&cs.ev[i]));
    }
    cudaStream_t s2 = g_overlap.load() ? cs.s2 : s; // serial mode: everything on s
    cs.keys_c.alloc((n + 1) * 2 * sizeof(u32));
    cs.items_c.alloc((n + 1) * 2 * sizeof(u32));
    GL_CUDA(cudaEventRecord(cs.ev[0], s));
    if (m == 0) {
        for (int i = 1; i < 4; ++i) GL_CUDA(cudaEventRecord(cs.ev[i], s));
        GL_CUDA(cudaEventRecord(cs.ev[6], s)); // fork/join point of the (empty) cycle pass
    } else {
        u64* wedges = cs.keys.as<u64>(); // scratch reuse before the sorts
        k_prepass<<<grid1d(m, 256, sms), 256, 0, s>>>(g, wedges);
        GL_LAUNCH_CHECK();
        GL_CUDA(cudaMemsetAsync(wedges + m, 0, sizeof(u64), s));
        dev_exclusive_scan<u64>(cs.tmp, wedges, cs.wpre.as<u64>(), m + 1, s);
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
                size_t fr = 0, tot = 0;
                GL_CUDA(cudaMemGetInfo(&fr, &tot));
                cs.tl_cap = std::min<u64>(hc[19] / (u64)world + 1, (u64)(0.4 * (double)fr) / sizeof(uint2));
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
                    k_take_rank<<<grid1d(count, 256, sms), 256, 0, s>>>(iout, offset, total, rank, world, list);
                    GL_LAUNCH_CHECK();
                    const u32 kws = K == 1088 ? 1088u : (K == 768 ? 512u : 128u); // largest k of the class
                    const size_t smem =
                        (size_t)hpass_ws_words(kws, kHPassCount, bloom_words<HCfg<K>::BLOG>()) * sizeof(u32);
                    smem_attr(k_hpass_block<kHPassCount, K>, smem, gr.device);
                    const TriList TL{cs.tlist.as<uint2>(), cs.tl_cap, counters + 20, cs.tl_base.as<u64>() + hbase,
                                     cs.tl_n.as<u32>() + hbase};
                    const bool glob = K == 1088 && cs.h_gstride;
                    k_hpass_block<kHPassCount, K><<<(unsigned)sms * HCfg<K>::MINB, HCfg<K>::THREADS, smem, s>>>(
                        g, list, count, queue, cs.t.as<u32>(), d_partials, glob ? cs.scratch.as<u32>() : nullptr,
                        glob ? cs.h_gstride : 0, cs.hlist.as<uint2>(), hcap, TL);
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
                k_take_rank<<<grid1d(mysmall, 256, sms), 256, 0, s>>>(iout, nxl + nbig + nmedk, nsmall, rank, world,
                                                                      cs.items3s.as<u32>());
                GL_LAUNCH_CHECK();
                const TriList TL{cs.tlist.as<uint2>(), cs.tl_cap, counters + 20,
                                 cs.tl_base.as<u64>() + myxl + mybig + mymedk, cs.tl_n.as<u32>() + myxl + mybig + mymedk};
                k_hpass_warp<kHPassCount><<<(unsigned)sms * 8, kHWarpsPerBlock * 32, 0, s>>>(
                    g, cs.items3s.as<u32>(), mysmall, counters + 3, cs.t.as<u32>(), d_partials, TL);
                GL_LAUNCH_CHECK();
                cs.launches += 2;
            }
        }
        GL_CUDA(cudaEventRecord(cs.ev[1], s));

        // cycles: top vertices, split small (warp hash) / big (block windows)
        GL_CUDA(cudaEventRecord(cs.ev[2], s2));
        {
            u32* kin = cs.keys_c.as<u32>();
            u32* kout = kin + (n + 1);
            u32* iin = cs.items_c.as<u32>();
            u32* iout = iin + (n + 1);
            k_top_keys<<<grid1d(n, 256, sms), 256, 0, s2>>>(g, cs.wpre.as<u64>(), kin, counters + 10, counters + 15,
                                                           counters + 16, counters + 11);
            k_tiers<<<grid1d(n, 256, sms), 256, 0, s2>>>(g, (unsigned*)(counters + 22));
            k_seq<<<grid1d(n, 256, sms), 256, 0, s2>>>(iin, n);
            GL_LAUNCH_CHECK();
            dev_sort_desc(cs.tmp_c, kin, kout, iin, iout, n, s2);
            u64 cc[kCounters];
            GL_CUDA(cudaMemcpyAsync(cc, counters, sizeof(cc), cudaMemcpyDeviceToHost, s2));
            const u64 wtot = read_dev(cs.wpre.as<u64>() + m, s2);
            const u64 nbig = cc[10], nmid = cc[15], nsmid = cc[16], nsmall = cc[11];
            const uint4 tiers = make_uint4((u32)cc[22], (u32)(cc[22] >> 32), (u32)cc[23], (u32)(cc[23] >> 32));
            cs.work[2] = 12 * wtot / (u64)world; // 4 B c id + 8 B slot credit per wedge
            cs.launches += 2 + 10;
            const u64 mybig = rank_share(nbig, rank, world);
            const u64 mymid = rank_share(nmid, rank, world);
            const u64 mysmid = rank_share(nsmid, rank, world);
            const u64 mysmall = rank_share(nsmall, rank, world);
            u32* lbig = iin;
            u32* lmid = lbig + mybig;
            u32* lsmid = lmid + mymid;
            u32* lsmall = lsmid + mysmid;
            if (mybig || mymid || mysmid) {
                if (2 * m >= (1ull << 32)) throw overflow_error("cycle pass needs 2m < 2^32 adjacency slots");
                // per-block scratch: big tops need dmax + 2 entries, hash tops at most
                // their wedge bound (nb <= wedges)
                const u32 cap_big = (g.dmax + 3) & ~1u;
                const u32 cap_hash = std::min<u32>(cap_big, (u32)kMidWedges + 2);
                const u64 w_big = (big_scratch_words(cap_big) + 1) & ~1ull;
                const u64 w_hash = (big_scratch_words(cap_hash) + 1) & ~1ull;
                if (mybig) cs.cursor.alloc((u64)sms * kBigBlocksPerSM * w_big * sizeof(u32));
                if (mymid || mysmid) cs.cursor2.alloc((u64)sms * 4 * w_hash * sizeof(u32));
                auto launch = [&](auto kind, u32* list, u64 count, u64 offset, u64 total, unsigned long long* queue) {
                    constexpr int K = decltype(kind)::value;
                    const u32 cap = K == 0 ? cap_big : cap_hash;
                    u32* scratch = K == 0 ? cs.cursor.as<u32>() : cs.cursor2.as<u32>();
                    k_take_rank<<<grid1d(count, 256, sms), 256, 0, s2>>>(iout, offset, total, rank, world, list);
                    GL_LAUNCH_CHECK();
                    const size_t smem = (size_t)cyc_smem_words<K>() * sizeof(u32);
                    smem_attr(k_cycle_block<K>, smem, gr.device);
                    k_cycle_block<K><<<(unsigned)sms * Cyc<K>::MINB, Cyc<K>::THREADS, smem, s2>>>(
                        g, list, count, queue, cs.slots.as<i64>(), scratch, cap, tiers);
                    GL_LAUNCH_CHECK();
                    cs.launches += 2;
                };
                if (mybig) launch(std::integral_constant<int, 0>{}, lbig, mybig, 0, nbig, counters + 1);
                if (mymid) launch(std::integral_constant<int, 1>{}, lmid, mymid, nbig, nmid, counters + 4);
                if (mysmid) launch(std::integral_constant<int, 2>{}, lsmid, mysmid, nbig + nmid, nsmid, counters + 7);
            }
            if (mysmall) {
                k_take_rank<<<grid1d(mysmall, 256, sms), 256, 0, s2>>>(iout, nbig + nmid + nsmid, nsmall, rank, world, lsmall);
                GL_LAUNCH_CHECK();
                const size_t smem = (size_t)kCycleSmallWarps * 2 * kHashSlots * sizeof(u32);
                smem_attr(k_cycle_small, smem, gr.device);
                k_cycle_small<<<(unsigned)sms * 3, kCycleSmallWarps * 32, smem, s2>>>(
                    g, cs.wpre.as<u64>(), lsmall, mysmall, counters + 2, cs.slots.as<i64>());
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
    const DevGraph& g = gr.d;
    const int sms = num_sms(gr.device);
    GL_CUDA(cudaEventRecord(cs.ev[4], s));
    // triangle sums over the same vertex shares as this rank's H-pass
    unsigned long long* counters = cs.acc.as<unsigned long long>() + 40;
    auto sums = [&](auto kc, u64 count, const u32* list, u64 hbase, unsigned long long* queue) {
        constexpr int K = decltype(kc)::value;
        const u32 kws = K == 1088 ? 1088u : (K == 768 ? 512u : 128u);
        const size_t smem = (size_t)hpass_ws_words(kws, kHPassSums, bloom_words<HCfg<K>::BLOG>()) * sizeof(u32);
        smem_attr(k_hpass_block<kHPassSums, K>, smem, gr.device);
        const TriList TL{cs.tlist.as<uint2>(), cs.tl_cap, counters + 20, cs.tl_base.as<u64>() + hbase,
                         cs.tl_n.as<u32>() + hbase};
        const bool glob = K == 1088 && cs.h_gstride;
        k_hpass_block<kHPassSums, K><<<(unsigned)sms * HCfg<K>::MINB, HCfg<K>::THREADS, smem, s>>>(
            g, list, count, queue, cs.t.as<u32>(), d_partials, glob ? cs.scratch.as<u32>() : nullptr,
            glob ? cs.h_gstride : 0, nullptr, 0, TL);
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
                         cs.tl_n.as<u32>() + hb};
        k_hpass_warp<kHPassSums><<<(unsigned)sms * 8, kHWarpsPerBlock * 32, 0, s>>>(
            g, cs.items3s.as<u32>(), cs.n_items3s, counters + 6, cs.t.as<u32>(), d_partials, TL);
        GL_LAUNCH_CHECK();
        cs.launches += 1;
    }
    cs.work[1] = cs.work[0];
    GL_CUDA(cudaEventRecord(cs.ev[5], s));
    // join the cycle pass, then fold its per-slot C4 credits into the y rows
    // (after the sums: both update y, the fold non-atomically)
    GL_CUDA(cudaStreamWaitEvent(s, cs.ev[3], 0));
    if (g.m) {
        k_fold_slots<<<grid1d(g.m, 256, sms), 256, 0, s>>>(g, cs.slots.as<i64>(), d_partials);
        GL_LAUNCH_CHECK();
        cs.launches += 1;
    }
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
} // namespace

void micro_records(const Graph& gr, u64 first, u64 count, u64* host_out) {
    GL_CUDA(cudaSetDevice(gr.device));
    const CountState& cs = gr.cs;
    if (!cs.have_micro) throw state_error("no counts computed yet");
    if (first < cs.shard_begin || first + count > cs.shard_end)
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
    if (cudaMemcpyFromSymbol(out, gl::g_cycle_prof, sizeof(unsigned long long) * 32) != cudaSuccess) return -4;
    if (reset) {
        unsigned long long z[32] = {0};
        if (cudaMemcpyToSymbol(gl::g_cycle_prof, z, sizeof(z)) != cudaSuccess) return -4;
    }
    return 0;
}
#endif
