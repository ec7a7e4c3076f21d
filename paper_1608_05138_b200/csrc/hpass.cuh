// hpass.cuh -- the clique / triangle pass (H-pass) kernels: per lowest vertex a,
// H_a = G[U(a)] by streaming + hashing, 4-clique popcounts, persisted H-edge
// records, triangle sums.  Included by count.cu inside gl::<anonymous> (one
// translation unit with the host orchestration).
#pragma once

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
#ifndef GL_HUNROLL
#define GL_HUNROLL 8
#endif
constexpr int kHUnroll = GL_HUNROLL; // streamed rounds in flight per warp
constexpr u32 kHProbeRatio = 16;    // probe instead of stream when |U(x_i)| > 16 * candidates (8: RMAT-24 H-pass +2.5%)
__constant__ u32 c_probe_ratio = kHProbeRatio; // GL_PROBE_RATIO overrides (tuning experiments)

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
#ifndef GL_BLOG768
#define GL_BLOG768 16
#endif
template <> struct HCfg<768> { static constexpr int THREADS = 512, MINB = 2, BLOG = GL_BLOG768; };
#ifndef GL_H128_THREADS
#define GL_H128_THREADS 128
#endif
template <> struct HCfg<128> { static constexpr int THREADS = GL_H128_THREADS, MINB = 1024 / GL_H128_THREADS, BLOG = 13; };

__device__ __forceinline__ u32 hp_log(u32 k) { // hash slots 2^log >= 2k, >= 64 (Bloom filters the misses)
    u32 l = 32 - __clz(2 * k - 1);
    return l < 6 ? 6 : l;
}
// bitmap row stride of H_a in u32 words: rows are read as u64 words with an
// odd u64 stride, so the rows of different members fall in different banks
// (phase 2 reads two arbitrary rows) and each popcount step covers 64 members
__host__ __device__ inline u32 hrow_stride(u32 k) { return 2u * (((k + 63u) >> 6) | 1u); }

__host__ __device__ inline u64 hpass_ws_words(u32 k, int mode, u32 bloom_w) {
    u32 l = 6;
    while ((1u << l) < 2 * k) ++l;
    const u64 H = 1ull << l;
    const u64 body = mode == 0 ? 2ull * k + (u64)k * hrow_stride(k)  // xs, tri, rows (8-byte aligned: 2k even)
                               : 4ull * k + 2;          // xs, ta, acc (u64, aligned)
    return body + 2 + H + H / 2 + bloom_w + 2ull * k; // + member list bounds
}

// the counting workspace without the bitmap rows (xs, tri, hash, Bloom, member
// bounds): kept in shared memory for k beyond the class KMAX while the rows go
// to the block's global scratch (hpass_vertex rows_g)
__host__ __device__ inline u64 hpass_small_words(u32 k, u32 bloom_w) {
    u32 l = 6;
    while ((1u << l) < 2 * k) ++l;
    const u64 H = 1ull << l;
    return 2ull * k + 2 + H + H / 2 + bloom_w + 2ull * k;
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
    // exact (GL_TL_EXACT=1, off by default): block vertices write their records
    // to the block's own list and copy them in with an exact reservation after
    // phase 2 instead of reserving C(k,2) up front
    u32 exact;
};
constexpr u64 kNoList = ~0ull;
// TriList::n flags: the low 31 bits count the records; kRecSoA marks the
// structure-of-arrays layout of a big-k vertex (pairs, then edge ids)
constexpr u32 kRecSoA = 0x80000000u, kRecCountMask = 0x7fffffffu;

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
        const bool probe = rem && ul > c_probe_ratio * rem;
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
// shared memory (k <= the class KMAX: every workspace access compiles to LDS/STS/
// ATOMS) or the block's global scratch (larger k).

// big (kHPassCount, k beyond the shared workspace): no bitmap is built in
// phase 1 (only the H-edge records); phase 2 rebuilds H_a's rows one column
// chunk at a time in the stage_words of shared memory left after the small
// arrays -- every record sets its two bits of the chunk -- and adds each
// chunk's popcounts (t once, x7 and the member degrees per chunk).
template <int MODE, int BLOG, typename Cand>
__device__ __forceinline__ void hpass_vertex(const DevGraph& g, u32* __restrict__ t, i64* __restrict__ part, u32* ws,
                                             Cand* cbuf, uint2* hlist, u32& s_nh, u32& s_mi, u32 a, u64 ub, u32 k,
                                             u32 W, u32 hl, u32 H, const TriList& TL, u64 idx, u64& s_base,
                                             u64 hcap = 0, bool big = false, u32 stage_words = 0) {
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
        const u32 nrec = TL.n[idx] & kRecCountMask;
        // kRecSoA: a big-k vertex kept its records as two u32 arrays in its
        // C(k,2)-record reservation (member pairs, then edge ids)
        const bool soa = TL.n[idx] & kRecSoA;
        const u32* rij = reinterpret_cast<const u32*>(rec);
        const u32* re_ = rij + (TL.exact ? (u64)nrec : (u64)k * (k - 1) / 2);
#ifndef GL_SUMS_U
#define GL_SUMS_U 4
#endif
        constexpr int U = GL_SUMS_U; // records in flight per thread
        for (u32 r0 = threadIdx.x; r0 < nrec; r0 += U * blockDim.x) {
            uint2 rv[U];
            u32 tv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const u32 r = r0 + u * blockDim.x;
                rv[u] = r >= nrec ? make_uint2(0, kEmpty) : soa ? make_uint2(rij[r], re_[r]) : rec[r];
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
    u32* rows = tri + k;                    // kHPassCount (not used when big)
    u32* ta = xs + k;                       // kHPassSums
    unsigned long long* acc = reinterpret_cast<unsigned long long*>(ws + ((2ull * k + 1) & ~1ull)); // kHPassSums
    const u32 RS = hrow_stride(k), W2 = (k + 63u) >> 6; // u32 stride, u64 words per row
    const u64 body = MODE == kHPassCount ? 2ull * k + (big ? 0ull : (u64)k * RS) : ((2ull * k + 1) & ~1ull) + 2ull * k;
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
    if (MODE == kHPassCount && !big)
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
        if (TL.rec && !TL.exact) {
            const u64 need = (u64)k * (k - 1) / 2;
            b = atomicAdd(TL.count, (unsigned long long)need);
            if (b + need > TL.cap) b = kNoList;
            TL.base[idx] = b;
        }
        s_base = b;
    }
    __syncthreads();
    uint2* const hout = (MODE == kHPassCount && s_base != kNoList) ? TL.rec + s_base : hlist;
    // big k: records as SoA over the same region (capacity C(k,2) in the
    // device-wide list, hcap in the block's own list)
    u32* const hij = reinterpret_cast<u32*>(hout);
    u32* const hee = hij + ((MODE == kHPassCount && s_base != kNoList) ? (u64)k * (k - 1) / 2 : hcap);
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
                if (hit && !big) {
                    atomicOr(&rows[(u64)i * RS + (j >> 5)], 1u << (j & 31));
                    atomicOr(&rows[(u64)j * RS + (i >> 5)], 1u << (i & 31));
                }
                const unsigned bal = __ballot_sync(0xffffffffu, hit);
                if (bal) {
                    u32 base = 0;
                    if (lane == 0) base = atomicAdd(&s_nh, (u32)__popc(bal));
                    base = __shfl_sync(0xffffffffu, base, 0);
                    if (hit) {
                        const u32 at = base + __popc(bal & ((1u << lane) - 1u));
                        if (big) { // SoA: the chunk sweeps of phase 2 read the pairs alone
                            hij[at] = (j << 16) | i;
                            hee[at] = e;
                        } else {
                            hout[at] = make_uint2((j << 16) | i, e);
                        }
                    }
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
        if (xe - xb > (u64)c_probe_ratio * rem) {
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
    if (MODE == kHPassCount && big) {
        // phase 2 for big k: per column chunk [64 c0, 64 (c0 + nw)), rebuild
        // the chunk of every row from the H-edge records (shared 64-bit
        // atomicOr), then one popcount sweep over the records; member degrees
        // accumulate per chunk (phase 3)
        const u32 nh = s_nh;
        if (TL.rec && threadIdx.x == 0) TL.n[idx] = nh | kRecSoA;
        // phase 1's hash, Bloom filter, member ids and list bounds are dead
        // now: the member degrees take xs' place and the stage everything
        // after tri (stage_words = the workspace words beyond xs and tri)
        u32* degs = xs; // u32[k]: member degree in H_a
        u32* st0 = tri + k;
        unsigned long long* st = reinterpret_cast<unsigned long long*>(st0 + ((uintptr_t)st0 & 4u ? 1 : 0));
        const u32 avail = stage_words > 2 ? stage_words - 2 : 0u;          // u32 words for the stage
        u32 cw = avail / (2u * k) - 1u;                                    // u64 words per row per chunk
        cw = cw < 1u ? 1u : (cw > W2 ? W2 : cw);
        const u32 sst = cw | 1u;                                           // odd stride: conflict-free rows
        for (u32 i = threadIdx.x; i < k; i += blockDim.x) degs[i] = 0;
        for (u32 c0 = 0; c0 < W2; c0 += cw) {
            const u32 nw = W2 - c0 < cw ? W2 - c0 : cw;
            const u32 lo = c0 * 64u, hi = (c0 + nw) * 64u;
            for (u32 q = threadIdx.x; q < k * sst; q += blockDim.x) st[q] = 0ull;
            __syncthreads();
            for (u32 h = threadIdx.x; h < nh; h += blockDim.x) {
                const u32 ij = hij[h];
                const u32 i = ij & 0xffffu, j = ij >> 16;
                if (j >= lo && j < hi) atomicOr(&st[(u64)i * sst + ((j - lo) >> 6)], 1ull << (j & 63));
                if (i >= lo && i < hi) atomicOr(&st[(u64)j * sst + ((i - lo) >> 6)], 1ull << (i & 63));
            }
            __syncthreads();
            for (u32 h = threadIdx.x; h < nh; h += blockDim.x) {
                const uint2 he = make_uint2(hij[h], hee[h]);
                const u32 i = he.x & 0xffffu, j = he.x >> 16;
                const unsigned long long* ri = st + (u64)i * sst;
                const unsigned long long* rj = st + (u64)j * sst;
                u32 c = 0;
                for (u32 v = 0; v < nw; ++v) c += __popcll(ri[v] & rj[v]);
                if (c0 == 0) atomicAdd(&t[he.y], 1u);
                if (c) {
                    atomicAdd(&tri[i], c);
                    atomicAdd(&tri[j], c);
                    atomic_add_i64(&part[2 * (u64)he.y], (i64)c);
                }
            }
            for (u32 i = threadIdx.x; i < k; i += blockDim.x) {
                u32 d = 0;
                for (u32 v = 0; v < nw; ++v) d += __popcll(st[(u64)i * sst + v]);
                degs[i] += d;
            }
            __syncthreads();
        }
        // phase 3: edges (a, x_i)
        for (u32 i = threadIdx.x; i < k; i += blockDim.x) {
            const u32 e = g.eid[ub + i];
            if (degs[i]) atomicAdd(&t[e], degs[i]);
            if (tri[i]) atomic_add_i64(&part[2 * (u64)e], (i64)(tri[i] >> 1));
        }
    } else if (MODE == kHPassCount) {
        // phase 2: stream the H-edges (kept in the device-wide list when it had room)
        const u32 nh = s_nh;
        if (TL.rec && threadIdx.x == 0) TL.n[idx] = nh;
        // the next record's load is in flight during this record's popcounts
        uint2 nx = threadIdx.x < nh ? hout[threadIdx.x] : make_uint2(0u, 0u);
        for (u32 h = threadIdx.x; h < nh; h += blockDim.x) {
            const uint2 he = nx;
            if (h + blockDim.x < nh) nx = hout[h + blockDim.x];
            const u32 i = he.x & 0xffffu, j = he.x >> 16;
            const unsigned long long* ri = reinterpret_cast<const unsigned long long*>(rows + (u64)i * RS);
            const unsigned long long* rj = reinterpret_cast<const unsigned long long*>(rows + (u64)j * RS);
            u32 c = 0;
            for (u32 v = 0; v < W2; ++v) c += __popcll(ri[v] & rj[v]);
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
            const unsigned long long* ri = reinterpret_cast<const unsigned long long*>(rows + (u64)i * RS);
            for (u32 v = 0; v < W2; ++v) deg += __popcll(ri[v]);
            const u32 e = g.eid[ub + i];
            if (deg) atomicAdd(&t[e], deg);
            if (tri[i]) atomic_add_i64(&part[2 * (u64)e], (i64)(tri[i] >> 1));
        }
    } else {
        for (u32 i = threadIdx.x; i < k; i += blockDim.x)
            if (acc[i]) atomic_add_i64(&part[2 * (u64)g.eid[ub + i] + 1], -(i64)acc[i]);
    }
    if (MODE == kHPassCount && TL.rec && TL.exact) {
        // exact reservation: copy this vertex's records from the block's list
        // (pairs then edge ids when big, with the edge ids at offset nh)
        __shared__ u64 s_cp;
        const u32 nh = s_nh;
        if (threadIdx.x == 0) {
            u64 b = kNoList;
            if (nh) {
                b = atomicAdd(TL.count, (unsigned long long)nh);
                if (b + nh > TL.cap) b = kNoList;
            }
            TL.base[idx] = nh ? b : 0;
            TL.n[idx] = nh | (big ? kRecSoA : 0u);
            s_cp = b;
        }
        __syncthreads();
        const u64 b = s_cp;
        if (nh && b != kNoList) {
            if (big) {
                u32* dij = reinterpret_cast<u32*>(TL.rec + b);
                for (u32 h = threadIdx.x; h < nh; h += blockDim.x) {
                    dij[h] = hij[h];
                    dij[nh + h] = hee[h];
                }
            } else {
                uint2* d = TL.rec + b;
                for (u32 h = threadIdx.x; h < nh; h += blockDim.x) d[h] = hout[h];
            }
        }
    }
}

template <int MODE, int KMAX>
__global__ void __launch_bounds__(HCfg<KMAX>::THREADS, HCfg<KMAX>::MINB)
k_hpass_block(DevGraph g, const u32* __restrict__ items, u64 n_items, unsigned long long* __restrict__ queue,
              u32* __restrict__ t, i64* __restrict__ part, u32* __restrict__ gscratch, u64 gstride,
              uint2* __restrict__ hlist_all, u64 hcap, TriList TL, u32 smem_words) {
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
        if (MODE == kHPassSums) { // one generic-pointer copy measured faster for the lighter sums pass
            const bool sm = hpass_ws_words(k, kHPassSums, bloom_words<BLOG>()) <= smem_words;
            hpass_vertex<MODE, BLOG>(g, t, part, sm ? smem : gscratch + (u64)blockIdx.x * gstride, cbuf, hlist,
                                     s_nh, s_mi, a, ub, k, W, hl, H, TL, idx, s_base);
        } else if (k <= (u32)KMAX) {
            hpass_vertex<MODE, BLOG>(g, t, part, smem, cbuf, hlist, s_nh, s_mi, a, ub, k, W, hl, H, TL, idx, s_base);
        } else if (hpass_small_words(k, bloom_words<BLOG>()) + 8ull * k <= smem_words) {
            // H_a's rows rebuilt per column chunk in shared memory from the
            // H-edge records (the small arrays, degrees and stage all shared)
            hpass_vertex<MODE, BLOG>(g, t, part, smem, cbuf, hlist, s_nh, s_mi, a, ub, k, W, hl, H, TL, idx, s_base,
                                     hcap, true, smem_words - 2 * k);
        } else {
            hpass_vertex<MODE, BLOG>(g, t, part, gscratch + (u64)blockIdx.x * gstride, cbuf, hlist, s_nh, s_mi, a,
                                     ub, k, W, hl, H, TL, idx, s_base);
        }
    }
}

