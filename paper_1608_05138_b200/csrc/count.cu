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
#include <cstring>
#include <vector>

#include "graph.cuh"

namespace gl {

namespace {

constexpr int kTriThreads = 256;
constexpr int kTriTile = 2048;       // probes per block tile
constexpr int kCliqueWarps = 8;      // warps per clique block
constexpr int kCliqueCap = 512;      // T+ entries per warp in shared memory
constexpr int kCycleSmallWarps = 8;  // warps per small-top block
constexpr int kHashSlots = 1024;     // per-warp hash slots (small tops)
constexpr u64 kSmallWedges = 512;    // small-top threshold (<= half the slots)
constexpr int kBigThreads = 1024;    // block per big top
constexpr int kWindow = 32768;       // dense W window (u32) in shared memory
constexpr int kChunk = 2048;         // b-chunk per flattened pass

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

__device__ __forceinline__ void atomic_add_i64(i64* p, i64 v) {
    atomicAdd(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v);
}

// ------------------------------------------------------------------ prepass

// probes(e) = min(|U(u) after v|, |U(v)|), wedges(e) = epos(e)
// lsum (optional): sum of |A|+|B| over edges with probes, i.e. the adjacency
// entries a merge-based intersection would read (the algorithmic bytes / 4).
__global__ void k_prepass(DevGraph g, u64* __restrict__ probes, u64* __restrict__ wedges,
                          unsigned long long* __restrict__ lsum) {
    u64 acc = 0;
    for (u64 e = blockIdx.x * (u64)blockDim.x + threadIdx.x; e < g.m; e += (u64)gridDim.x * blockDim.x) {
        u32 v = g.ev[e], u = g.eu[e];
        u64 la = g.off[u + 1] - (g.off[u] + g.epos[e] + 1);
        u64 lb = g.off[v + 1] - (g.off[v] + g.lcnt[v]);
        bool any = la && lb;
        probes[e] = any ? (la < lb ? la : lb) : 0;
        wedges[e] = g.epos[e];
        acc += any ? la + lb : 0;
    }
    if (lsum) {
        for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
        if ((threadIdx.x & 31) == 0 && acc) atomicAdd(lsum, (unsigned long long)acc);
    }
}

// ------------------------------------------------------------------ triangles

struct TriCtx {
    u32 v, u;
    u64 a_begin, a_end, b_begin, b_end;
};

__device__ __forceinline__ TriCtx tri_ctx(const DevGraph& g, u64 e) {
    TriCtx c;
    c.v = g.ev[e];
    c.u = g.eu[e];
    c.a_begin = g.off[c.u] + g.epos[e] + 1;
    c.a_end = g.off[c.u + 1];
    c.b_begin = g.off[c.v] + g.lcnt[c.v];
    c.b_end = g.off[c.v + 1];
    return c;
}

// Probe r of edge e: returns found, and the A-side (u row) / B-side (v row) slots.
__device__ __forceinline__ bool tri_probe(const DevGraph& g, const TriCtx& c, u64 r, u64* sa, u64* sb) {
    const u64 la = c.a_end - c.a_begin, lb = c.b_end - c.b_begin;
    if (la <= lb) {
        u64 s = c.a_begin + r;
        u32 x = g.adj[s];
        u64 p = lower_bound_dev<u32, u64>(g.adj, c.b_begin, c.b_end, x);
        *sa = s;
        *sb = p;
        return p < c.b_end && g.adj[p] == x;
    } else {
        u64 s = c.b_begin + r;
        u32 x = g.adj[s];
        u64 p = lower_bound_dev<u32, u64>(g.adj, c.a_begin, c.a_end, x);
        *sa = p;
        *sb = s;
        return p < c.a_end && g.adj[p] == x;
    }
}

// MODE 0: t(e) and tplus(e).  MODE 1: S(e) contributions into y rows.
template <int MODE>
__global__ void __launch_bounds__(kTriThreads)
k_tri(DevGraph g, const u64* __restrict__ pre, u64 item_begin, u64 item_end, u32* __restrict__ t,
      u32* __restrict__ tplus, i64* __restrict__ part) {
    __shared__ u64 s_e[2];
    for (u64 tile = item_begin + (u64)blockIdx.x * kTriTile; tile < item_end;
         tile += (u64)gridDim.x * kTriTile) {
        const u64 tile_end = tile + kTriTile < item_end ? tile + kTriTile : item_end;
        __syncthreads();
        if (threadIdx.x < 2) {
            u64 x = threadIdx.x == 0 ? tile : tile_end - 1;
            s_e[threadIdx.x] = upper_bound_dev<u64, u64>(pre, 0, g.m + 1, x) - 1;
        }
        __syncthreads();
        const u64 e_lo = s_e[0], e_hi = s_e[1] + 1;
        for (u64 base = tile; base < tile_end; base += kTriThreads) {
            const u64 i = base + threadIdx.x;
            const bool valid = i < tile_end;
            u64 e = ~0ull;
            bool found = false;
            u64 sa = 0, sb = 0;
            if (valid) {
                e = upper_bound_dev<u64, u64>(pre, e_lo, e_hi + 1 > g.m + 1 ? g.m + 1 : e_hi + 1, i) - 1;
                TriCtx c = tri_ctx(g, e);
                found = tri_probe(g, c, i - pre[e], &sa, &sb);
            }
            if (MODE == 0) {
                if (found) {
                    atomicAdd(&t[g.eid[sa]], 1u);
                    atomicAdd(&t[g.eid[sb]], 1u);
                }
                u64 sum;
                bool tail = seg_tail_sum(e, found ? 1ull : 0ull, &sum);
                if (valid && tail && sum) {
                    atomicAdd(&t[e], (u32)sum);
                    atomicAdd(&tplus[e], (u32)sum);
                }
            } else {
                u64 contrib = 0;
                if (found) {
                    u32 ea = g.eid[sa], eb = g.eid[sb];
                    u64 te = t[e], ta = t[ea], tb = t[eb];
                    atomic_add_i64(&part[2 * (u64)ea + 1], -(i64)(te + tb));
                    atomic_add_i64(&part[2 * (u64)eb + 1], -(i64)(te + ta));
                    contrib = ta + tb;
                }
                u64 sum;
                bool tail = seg_tail_sum(e, contrib, &sum);
                if (valid && tail && sum) atomic_add_i64(&part[2 * e + 1], -(i64)sum);
            }
        }
    }
}

// ------------------------------------------------------------------ cliques

// Warp-local T+ staging: c, deg (clique degree inside T+), eid(u,c), eid(v,c),
// flattened work prefix.
struct TBuf {
    u32 *c, *deg, *eu, *ev, *pre;
};

__device__ __forceinline__ TBuf tbuf_at(u32* base, u32 cap) {
    TBuf b;
    b.c = base;
    b.deg = base + cap;
    b.eu = base + 2 * cap;
    b.ev = base + 3 * cap;
    b.pre = base + 4 * cap;
    return b;
}

__device__ __forceinline__ u64 warp_sum_u64(u64 v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    return v;
}

__global__ void __launch_bounds__(kCliqueWarps * 32)
k_clique(DevGraph g, const u32* __restrict__ items, u64 n_items, unsigned long long* __restrict__ queue,
         i64* __restrict__ part, u32* __restrict__ gscratch, u32 gcap, unsigned long long* __restrict__ work) {
    extern __shared__ u32 smem[];
    const u32 lane = lane_id();
    const u32 wib = threadIdx.x >> 5;
    const u64 gwarp = (u64)blockIdx.x * kCliqueWarps + wib;
    u64 my_work = 0;
    for (;;) {
        unsigned long long idx = 0;
        if (lane == 0) idx = atomicAdd(queue, 1ull);
        idx = __shfl_sync(0xffffffffu, idx, 0);
        if (idx >= n_items) break;
        const u64 e = items[idx];
        TriCtx c = tri_ctx(g, e);
        const u64 la = c.a_end - c.a_begin, lb = c.b_end - c.b_begin;
        const u64 ls = la < lb ? la : lb;
        const bool big = ls > (u64)kCliqueCap;
        TBuf tb = big ? tbuf_at(gscratch + gwarp * 5ull * gcap, gcap)
                      : tbuf_at(smem + wib * 5u * kCliqueCap, kCliqueCap);
        // 1. T+ = U(u) after v  n  U(v), in ascending id order
        u32 T = 0;
        for (u64 base = 0; base < ls; base += 32) {
            u64 r = base + lane;
            u64 sa = 0, sb = 0;
            bool found = r < ls && tri_probe(g, c, r, &sa, &sb);
            unsigned bal = __ballot_sync(0xffffffffu, found);
            if (found) {
                u32 pos = T + __popc(bal & ((1u << lane) - 1u));
                tb.c[pos] = g.adj[sa];
                tb.eu[pos] = g.eid[sa];
                tb.ev[pos] = g.eid[sb];
                tb.deg[pos] = 0;
            }
            T += __popc(bal);
        }
        my_work += ls;
        __syncwarp();
        // 2. per-member work = min(|U(c)|, members after c); exclusive prefix
        u32 carry = 0;
        for (u32 base = 0; base < T; base += 32) {
            u32 i = base + lane;
            u32 w = 0;
            if (i < T) {
                u32 x = tb.c[i];
                u64 lu = g.off[x + 1] - (g.off[x] + g.lcnt[x]);
                u64 rem = T - 1 - i;
                w = (u32)(lu < rem ? lu : rem);
            }
            u32 incl = w;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                u32 o = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= (u32)d) incl += o;
            }
            if (i < T) tb.pre[i] = carry + incl - w;
            carry += __shfl_sync(0xffffffffu, incl, 31);
        }
        const u32 W2 = carry;
        __syncwarp();
        // 3. flattened intersections: edges (c, d) inside T+
        u64 K = 0;
        for (u32 base = 0; base < W2; base += 32) {
            u32 k = base + lane;
            if (k < W2) {
                u32 i = upper_bound_dev<u32, u32>(tb.pre, 0, T, k) - 1;
                u32 r = k - tb.pre[i];
                u32 x = tb.c[i];
                u64 ub = g.off[x] + g.lcnt[x], ue = g.off[x + 1];
                u64 lu = ue - ub;
                u32 rem = T - 1 - i;
                bool found;
                u32 j;
                u64 slot;
                if (lu <= rem) {
                    slot = ub + r;
                    u32 d = g.adj[slot];
                    j = lower_bound_dev<u32, u32>(tb.c, i + 1, T, d);
                    found = j < T && tb.c[j] == d;
                } else {
                    j = i + 1 + r;
                    u32 d = tb.c[j];
                    slot = lower_bound_dev<u32, u64>(g.adj, ub, ue, d);
                    found = slot < ue && g.adj[slot] == d;
                }
                if (found) {
                    atomicAdd(&tb.deg[i], 1u);
                    atomicAdd(&tb.deg[j], 1u);
                    ++K;
                    atomic_add_i64(&part[2 * (u64)g.eid[slot]], 1); // top edge (c, d)
                }
            }
        }
        my_work += W2;
        __syncwarp();
        K = warp_sum_u64(K);
        if (lane == 0 && K) atomic_add_i64(&part[2 * e], (i64)K);
        for (u32 i = lane; i < T; i += 32) {
            u32 d = tb.deg[i];
            if (d) {
                atomic_add_i64(&part[2 * (u64)tb.eu[i]], (i64)d);
                atomic_add_i64(&part[2 * (u64)tb.ev[i]], (i64)d);
            }
        }
        __syncwarp();
    }
    if (lane == 0 && my_work) atomicAdd(work, (unsigned long long)my_work);
}

// ------------------------------------------------------------------ cycles

__device__ __forceinline__ u32 hslot(u32 key) { return (key * 0x9E3779B1u) >> (32 - 10); }
static_assert(kHashSlots == 1024, "hslot assumes 1024 slots");

// Small tops: one warp per top vertex a, W[c] in a warp-private hash.
__global__ void __launch_bounds__(kCycleSmallWarps * 32)
k_cycle_small(DevGraph g, const u64* __restrict__ wpre, const u32* __restrict__ items, u64 n_items,
              unsigned long long* __restrict__ queue, i64* __restrict__ part) {
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
                if (val) atomic_add_i64(&part[2 * (u64)g.eid[slot] + 1], (i64)val);
            }
            u64 sum;
            bool tail = seg_tail_sum(e, val, &sum);
            if (k < nw && tail && sum) atomic_add_i64(&part[2 * e + 1], (i64)sum);
        }
        __syncwarp();
        for (u32 i = lane; i < kHashSlots; i += 32) {
            keys[i] = kEmpty;
            cnt[i] = 0;
        }
        __syncwarp();
    }
}

// Block-wide exclusive scan of up to kChunk u32 values (kBigThreads threads,
// 2 values per thread).  Returns the total.
__device__ __forceinline__ u32 block_scan_chunk(u32* s_vals, u32 n, u32* s_warp) {
    using BlockScan = cub::BlockScan<u32, kBigThreads>;
    __shared__ typename BlockScan::TempStorage tmp;
    (void)s_warp;
    u32 v[2];
    const u32 t = threadIdx.x;
    v[0] = (2 * t < n) ? s_vals[2 * t] : 0;
    v[1] = (2 * t + 1 < n) ? s_vals[2 * t + 1] : 0;
    u32 total;
    BlockScan(tmp).ExclusiveSum(v, v, total);
    __syncthreads();
    if (2 * t < n) s_vals[2 * t] = v[0];
    if (2 * t + 1 < n) s_vals[2 * t + 1] = v[1];
    __syncthreads();
    return total;
}
static_assert(kChunk == 2 * kBigThreads, "chunk = 2 items per thread");

// Big tops: one block per top vertex a, dense W windows in shared memory.
__global__ void __launch_bounds__(kBigThreads, 1)
k_cycle_big(DevGraph g, const u32* __restrict__ items, u64 n_items, unsigned long long* __restrict__ queue,
            i64* __restrict__ part, u32* __restrict__ gcur, u32 gcur_cap) {
    extern __shared__ u32 smem[];
    u32* W = smem;                    // kWindow
    u32* s_pre = smem + kWindow;      // kChunk + 1
    __shared__ unsigned long long s_idx;
    __shared__ u32 s_next;
    u32* cur = gcur + (u64)blockIdx.x * 2 * gcur_cap;
    u32* hpos = cur + gcur_cap;
    for (u32 i = threadIdx.x; i < kWindow; i += blockDim.x) W[i] = 0;
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) s_idx = atomicAdd(queue, 1ull);
        __syncthreads();
        const unsigned long long idx = s_idx;
        if (idx >= n_items) break;
        const u32 a = items[idx];
        const u64 E0 = g.loff[a];
        const u32 nb = (u32)(g.loff[a + 1] - E0);
        if (threadIdx.x == 0) s_next = kEmpty;
        __syncthreads();
        for (u32 j = threadIdx.x; j < nb; j += blockDim.x) {
            cur[j] = 0;
            u64 e = E0 + j;
            if (g.epos[e] > 0) atomicMin(&s_next, g.adj[g.off[g.eu[e]]]);
        }
        __syncthreads();
        u32 lo = s_next;
        while (lo != kEmpty && lo < a) {
            const u32 hi = (u64)lo + kWindow < (u64)a ? lo + kWindow : a;
            // run ends for this window
            for (u32 j = threadIdx.x; j < nb; j += blockDim.x) {
                u64 e = E0 + j;
                u64 rb = g.off[g.eu[e]];
                u64 p = lower_bound_dev<u32, u64>(g.adj, rb + cur[j], rb + g.epos[e], hi);
                hpos[j] = (u32)(p - rb);
            }
            __syncthreads();
            // three flattened passes: count, credit, clear
            for (int pass = 0; pass < 3; ++pass) {
                for (u32 cb = 0; cb < nb; cb += kChunk) {
                    const u32 cn = nb - cb < (u32)kChunk ? nb - cb : (u32)kChunk;
                    for (u32 j = threadIdx.x; j < cn; j += blockDim.x) s_pre[j] = hpos[cb + j] - cur[cb + j];
                    __syncthreads();
                    const u32 total = block_scan_chunk(s_pre, cn, nullptr);
                    if (threadIdx.x == 0) s_pre[cn] = total;
                    __syncthreads();
                    for (u32 base = 0; base < total; base += blockDim.x) {
                        const u32 k = base + threadIdx.x;
                        u64 key = ~0ull, val = 0;
                        if (k < total) {
                            u32 jj = upper_bound_dev<u32, u32>(s_pre, 0, cn + 1, k) - 1;
                            // skip empty runs (equal prefixes): upper_bound lands on the last equal
                            u32 j = cb + jj;
                            u64 e = E0 + j;
                            u64 slot = g.off[g.eu[e]] + cur[j] + (k - s_pre[jj]);
                            u32 cv = g.adj[slot];
                            if (pass == 0) {
                                atomicAdd(&W[cv - lo], 1u);
                            } else if (pass == 1) {
                                val = W[cv - lo] - 1;
                                key = e;
                                if (val) atomic_add_i64(&part[2 * (u64)g.eid[slot] + 1], (i64)val);
                            } else {
                                W[cv - lo] = 0;
                            }
                        }
                        if (pass == 1) {
                            u64 sum;
                            bool tail = seg_tail_sum(key, val, &sum);
                            if (k < total && tail && sum) atomic_add_i64(&part[2 * key + 1], (i64)sum);
                        }
                    }
                    __syncthreads();
                }
            }
            // advance cursors, find next non-empty window start
            if (threadIdx.x == 0) s_next = kEmpty;
            __syncthreads();
            for (u32 j = threadIdx.x; j < nb; j += blockDim.x) {
                cur[j] = hpos[j];
                u64 e = E0 + j;
                if (cur[j] < g.epos[e]) atomicMin(&s_next, g.adj[g.off[g.eu[e]] + cur[j]]);
            }
            __syncthreads();
            lo = s_next;
        }
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

__global__ void k_clique_keys(const u32* __restrict__ tplus, const u64* __restrict__ probes, u64 m,
                              u64* __restrict__ keys, unsigned long long* __restrict__ cnt) {
    u32 local = 0;
    for (u64 e = blockIdx.x * (u64)blockDim.x + threadIdx.x; e < m; e += (u64)gridDim.x * blockDim.x) {
        u64 tp = tplus[e];
        u64 k = tp >= 2 ? tp * (tp + 8) + probes[e] : 0;
        keys[e] = k;
        local += k ? 1 : 0;
    }
    if (local) atomicAdd(cnt, (unsigned long long)local);
}

__global__ void k_top_keys(DevGraph g, const u64* __restrict__ wpre, u64* __restrict__ keys,
                           unsigned long long* __restrict__ cnt) {
    unsigned long long lb = 0, ls = 0;
    for (u64 a = blockIdx.x * (u64)blockDim.x + threadIdx.x; a < g.n; a += (u64)gridDim.x * blockDim.x) {
        u64 w = wpre[g.loff[a + 1]] - wpre[g.loff[a]];
        keys[a] = w;
        if (w > kSmallWedges)
            ++lb;
        else if (w)
            ++ls;
    }
    if (lb) atomicAdd(&cnt[0], lb);
    if (ls) atomicAdd(&cnt[1], ls);
}

// rank's share of a cost-sorted list: sorted positions p with p % world == rank
__global__ void k_take_rank(const u32* __restrict__ sorted, u64 begin, u64 count, int rank, int world,
                            u32* __restrict__ out) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x;; i += (u64)gridDim.x * blockDim.x) {
        u64 p = (u64)rank + i * (u64)world;
        if (p >= count) break;
        out[i] = sorted[begin + p];
    }
}

__global__ void k_max_u32(const u32* __restrict__ a, const u32* __restrict__ ids, u64 n,
                          const DevGraph g, unsigned* __restrict__ out) {
    u32 mx = 0;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        u64 e = ids[i];
        TriCtx c = tri_ctx(g, e);
        u64 la = c.a_end - c.a_begin, lb = c.b_end - c.b_begin;
        u32 v = (u32)(la < lb ? la : lb);
        mx = v > mx ? v : mx;
    }
    (void)a;
    for (int d = 16; d > 0; d >>= 1) {
        u32 o = __shfl_down_sync(0xffffffffu, mx, d);
        mx = o > mx ? o : mx;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(out, mx);
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
void dev_sort_desc(DevBuf& tmp, u64* keys_in, u64* keys_out, u32* ids_in, u32* ids_out, u64 n,
                   cudaStream_t s) {
    size_t bytes = 0;
    GL_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, bytes, keys_in, keys_out, ids_in, ids_out,
                                                      (int64_t)n, 0, 64, s));
    tmp.alloc(bytes);
    GL_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp.p, bytes, keys_in, keys_out, ids_in, ids_out,
                                                      (int64_t)n, 0, 64, s));
}

template <typename T> T read_dev(const T* p, cudaStream_t s) {
    T h{};
    GL_CUDA(cudaMemcpyAsync(&h, p, sizeof(T), cudaMemcpyDeviceToHost, s));
    GL_CUDA(cudaStreamSynchronize(s));
    return h;
}

} // namespace

// --------------------------------------------------------------------------

void count_begin(Graph& gr, int rank, int world, i64* d_partials, cudaStream_t s) {
    GL_CUDA(cudaSetDevice(gr.device));
    if (world < 1 || rank < 0 || rank >= world) throw invalid_argument("bad rank/world");
    if (!s) s = gr.stream;
    const DevGraph& g = gr.d;
    CountState& cs = gr.cs;
    const int sms = num_sms(gr.device);
    const u64 m = g.m, n = g.n;
    cs.launches = 0;
    cs.began = false;
    std::memset(cs.work, 0, sizeof(cs.work));

    cs.t.alloc((m + 1) * sizeof(u32));
    cs.tplus.alloc((m + 1) * sizeof(u32));
    cs.pre1.alloc((m + 1) * sizeof(u64));
    cs.wpre.alloc((m + 1) * sizeof(u64));
    cs.acc.alloc(64 * sizeof(u64));
    cs.keys.alloc((std::max(m, n) + 1) * 2 * sizeof(u64)); // key in/out
    cs.items2.alloc((std::max(m, n) + 1) * 2 * sizeof(u32)); // id in/out
    const u64 plen = ((m + world - 1) / world) * (u64)world;
    if (plen) GL_CUDA(cudaMemsetAsync(d_partials, 0, 2 * plen * sizeof(i64), s));
    GL_CUDA(cudaMemsetAsync(cs.t.p, 0, (m + 1) * sizeof(u32), s));
    GL_CUDA(cudaMemsetAsync(cs.tplus.p, 0, (m + 1) * sizeof(u32), s));
    unsigned long long* counters = cs.acc.as<unsigned long long>() + 40; // queues + counts
    GL_CUDA(cudaMemsetAsync(counters, 0, 24 * sizeof(u64), s));

    Timer tm(4);
    GL_CUDA(cudaEventRecord(tm.ev[0], s));
    if (m == 0) {
        for (int i = 1; i < 4; ++i) GL_CUDA(cudaEventRecord(tm.ev[i], s));
    } else {
        u64* probes = cs.keys.as<u64>();     // scratch reuse before the sorts
        u64* wedges = probes + (m + 1);
        k_prepass<<<grid1d(m, 256, sms), 256, 0, s>>>(g, probes, wedges, counters + 17);
        GL_LAUNCH_CHECK();
        GL_CUDA(cudaMemsetAsync(probes + m, 0, sizeof(u64), s));
        GL_CUDA(cudaMemsetAsync(wedges + m, 0, sizeof(u64), s));
        dev_exclusive_scan<u64>(cs.tmp, probes, cs.pre1.as<u64>(), m + 1, s);
        dev_exclusive_scan<u64>(cs.tmp, wedges, cs.wpre.as<u64>(), m + 1, s);
        cs.launches += 3;
        const u64 P = read_dev(cs.pre1.as<u64>() + m, s);
        const u64 L = read_dev<unsigned long long>(counters + 17, s);
        cs.work[0] = 4 * L; // t pass; the S pass adds this rank's slice below

        // triangles (replicated on every rank: every rank needs all of t)
        if (P) {
            unsigned gt = (unsigned)std::min<u64>((P + kTriTile - 1) / kTriTile, (u64)sms * 8);
            k_tri<0><<<gt, kTriThreads, 0, s>>>(g, cs.pre1.as<u64>(), 0, P, cs.t.as<u32>(),
                                                  cs.tplus.as<u32>(), d_partials);
            GL_LAUNCH_CHECK();
            // triangle sums S, this rank's slice of the probe space
            u64 b = P * (u64)rank / world, en = P * (u64)(rank + 1) / world;
            if (en > b) {
                unsigned gs = (unsigned)std::min<u64>((en - b + kTriTile - 1) / kTriTile, (u64)sms * 8);
                k_tri<1><<<gs, kTriThreads, 0, s>>>(g, cs.pre1.as<u64>(), b, en, cs.t.as<u32>(),
                                                      cs.tplus.as<u32>(), d_partials);
                GL_LAUNCH_CHECK();
                cs.work[0] += (u64)((double)(4 * L) * (double)(en - b) / (double)P);
            }
            cs.launches += 2;
        }
        GL_CUDA(cudaEventRecord(tm.ev[1], s));

        // cliques: lowest pairs with |T+| >= 2, cost-sorted, rank share
        {
            u64* kin = cs.keys.as<u64>();
            u64* kout = kin + (m + 1);
            u32* iin = cs.items2.as<u32>();
            u32* iout = iin + (m + 1);
            // probes still needed for the key: recompute into kout first
            k_prepass<<<grid1d(m, 256, sms), 256, 0, s>>>(g, kout, kin, nullptr); // kout=probes, kin=wedges(unused)
            k_clique_keys<<<grid1d(m, 256, sms), 256, 0, s>>>(cs.tplus.as<u32>(), kout, m, kin, counters + 8);
            k_seq<<<grid1d(m, 256, sms), 256, 0, s>>>(iin, m);
            GL_LAUNCH_CHECK();
            dev_sort_desc(cs.tmp, kin, kout, iin, iout, m, s);
            const u64 cnt = read_dev<unsigned long long>(counters + 8, s);
            const u64 mine = cnt > (u64)rank ? (cnt - rank + world - 1) / world : 0;
            cs.n_items2 = mine;
            cs.launches += 5;
            if (mine) {
                // T+ upper bound for the global-scratch fallback
                k_max_u32<<<grid1d(cnt, 256, sms), 256, 0, s>>>(nullptr, iout, cnt, g, (unsigned*)(counters + 9));
                u32 maxls = (u32)read_dev<unsigned long long>(counters + 9, s);
                u32* mylist = iin; // reuse
                k_take_rank<<<grid1d(mine, 256, sms), 256, 0, s>>>(iout, 0, cnt, rank, world, mylist);
                GL_LAUNCH_CHECK();
                const unsigned blocks = (unsigned)sms * 2;
                u32 gcap = 0;
                if (maxls > (u32)kCliqueCap) {
                    gcap = maxls;
                    cs.scratch.alloc((u64)blocks * kCliqueWarps * 5ull * gcap * sizeof(u32));
                }
                const size_t smem = (size_t)kCliqueWarps * 5 * kCliqueCap * sizeof(u32);
                GL_CUDA(cudaFuncSetAttribute(k_clique, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                k_clique<<<blocks, kCliqueWarps * 32, smem, s>>>(g, mylist, mine, counters + 0, d_partials,
                                                                  gcap ? cs.scratch.as<u32>() : nullptr, gcap,
                                                                  counters + 16);
                GL_LAUNCH_CHECK();
                cs.launches += 3;
            }
        }
        GL_CUDA(cudaEventRecord(tm.ev[2], s));

        // cycles: top vertices, split small (warp hash) / big (block windows)
        {
            u64* kin = cs.keys.as<u64>();
            u64* kout = kin + (n + 1);
            u32* iin = cs.items2.as<u32>();
            u32* iout = iin + (n + 1);
            k_top_keys<<<grid1d(n, 256, sms), 256, 0, s>>>(g, cs.wpre.as<u64>(), kin, counters + 10);
            k_seq<<<grid1d(n, 256, sms), 256, 0, s>>>(iin, n);
            GL_LAUNCH_CHECK();
            dev_sort_desc(cs.tmp, kin, kout, iin, iout, n, s);
            const u64 nbig = read_dev<unsigned long long>(counters + 10, s);
            const u64 nsmall = read_dev<unsigned long long>(counters + 11, s);
            cs.work[2] = 8 * read_dev(cs.wpre.as<u64>() + m, s) / (u64)world; // c id + eid per wedge
            cs.launches += 3;
            const u64 mybig = nbig > (u64)rank ? (nbig - rank + world - 1) / world : 0;
            const u64 mysmall = nsmall > (u64)rank ? (nsmall - rank + world - 1) / world : 0;
            cs.n_items3b = mybig;
            cs.n_items3s = mysmall;
            u32* lbig = iin;
            u32* lsmall = iin + mybig;
            if (mybig) {
                k_take_rank<<<grid1d(mybig, 256, sms), 256, 0, s>>>(iout, 0, nbig, rank, world, lbig);
                GL_LAUNCH_CHECK();
                u32 cap = g.dmax + 1;
                const unsigned blocks = (unsigned)sms;
                cs.cursor.alloc((u64)blocks * 2 * cap * sizeof(u32));
                const size_t smem = (size_t)(kWindow + kChunk + 1) * sizeof(u32);
                GL_CUDA(cudaFuncSetAttribute(k_cycle_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                k_cycle_big<<<blocks, kBigThreads, smem, s>>>(g, lbig, mybig, counters + 1, d_partials,
                                                              cs.cursor.as<u32>(), cap);
                GL_LAUNCH_CHECK();
                cs.launches += 2;
            }
            if (mysmall) {
                k_take_rank<<<grid1d(mysmall, 256, sms), 256, 0, s>>>(iout, nbig, nsmall, rank, world, lsmall);
                GL_LAUNCH_CHECK();
                const size_t smem = (size_t)kCycleSmallWarps * 2 * kHashSlots * sizeof(u32);
                GL_CUDA(cudaFuncSetAttribute(k_cycle_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                k_cycle_small<<<(unsigned)sms * 3, kCycleSmallWarps * 32, smem, s>>>(
                    g, cs.wpre.as<u64>(), lsmall, mysmall, counters + 2, d_partials);
                GL_LAUNCH_CHECK();
                cs.launches += 2;
            }
        }
    }
    GL_CUDA(cudaEventRecord(tm.ev[3], s));
    GL_CUDA(cudaEventSynchronize(tm.ev[3]));
    GL_CUDA(cudaEventElapsedTime(&cs.ms[0], tm.ev[0], tm.ev[1]));
    GL_CUDA(cudaEventElapsedTime(&cs.ms[1], tm.ev[1], tm.ev[2]));
    GL_CUDA(cudaEventElapsedTime(&cs.ms[2], tm.ev[2], tm.ev[3]));
    if (m) cs.work[1] = 4 * read_dev<unsigned long long>(counters + 16, s);
    cs.began = true;
}

void count_finish(Graph& gr, const i64* d_part_shard, u64 begin, u64 end, u128 C[17], cudaStream_t s) {
    GL_CUDA(cudaSetDevice(gr.device));
    if (!s) s = gr.stream;
    CountState& cs = gr.cs;
    if (!cs.began) throw state_error("gl_count_finish before gl_count_begin");
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
