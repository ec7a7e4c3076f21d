// cycles.cuh -- the 4-cycle pass kernels: per top vertex a (Chiba-Nishizeki
// wedges a-b-c, b < a, c < a), W_a[c] in degree-tiered dense shared-memory
// windows (big tops) or block / warp hashes (smaller tops), C4 credits to
// adjacency-slot accumulators.  Included by count.cu inside gl::<anonymous>.
#pragma once

// ------------------------------------------------------------------ cycles

__device__ __forceinline__ u32 hslot(u32 key) { return (key * 0x9E3779B1u) >> (32 - 10); }
static_assert(kHashSlots == 1024, "hslot assumes 1024 slots");

// The slot credits stream through a 2m x 8 B array with no reuse inside a
// window (every (b,c) slot gets one credit per top): they are issued with an
// L2 evict-first policy so they do not push out the window's adjacency slices
// (re-read by pass 1), the run metadata and the block scratch.  GL_NO_L2_HINT
// drops the hints (A/B).
__device__ __forceinline__ void red_add_u64_if(i64* p, u64 v) {
#ifdef GL_NO_L2_HINT
    asm volatile("{ .reg .pred q; setp.ne.u64 q, %1, 0; @q red.global.add.u64 [%0], %1; }" ::"l"(p), "l"(v)
                 : "memory");
#else
    asm volatile("{ .reg .pred q; .reg .b64 pol; createpolicy.fractional.L2::evict_first.b64 pol, 1.0;"
                 " setp.ne.u64 q, %1, 0; @q red.global.add.L2::cache_hint.u64 [%0], %1, pol; }" ::"l"(p),
                 "l"(v)
                 : "memory");
#endif
}
// 32-bit form of the slot credit (same evict-first policy)
__device__ __forceinline__ void red_add_u32_if(u32* p, u32 v) {
#ifdef GL_NO_L2_HINT
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %1, 0; @q red.global.add.u32 [%0], %1; }" ::"l"(p), "r"(v)
                 : "memory");
#else
    asm volatile("{ .reg .pred q; .reg .b64 pol; createpolicy.fractional.L2::evict_first.b64 pol, 1.0;"
                 " setp.ne.u32 q, %1, 0; @q red.global.add.L2::cache_hint.u32 [%0], %1, pol; }" ::"l"(p),
                 "r"(v)
                 : "memory");
#endif
}
// C4 credit accumulators.  The credit of slot (b,c) from top a is W_a[c]-1 <=
// deg(c)-1 and b's tops are its upper neighbours U(b), so a slot's total is
// <= |U(b)| (deg(c)-1); under degree order |U(b)|^2 <= 2m < 2^32, hence for
// every c of degree < 65536 the total fits 32 bits: those slots take a u32
// RED (half the read-modify-write bytes of the slot array, the largest DRAM
// stream at scale).  Slots whose c is a hub (degree >= 65536: ids >= hub, the
// 32-bit counter tier) and the per-run (a,b) sums stay 64-bit.
struct Credits {
    i64* s64;
    u32* s32;
    u32 hub;
};
__device__ __forceinline__ void credit_slot(const Credits& cr, u64 slot, u32 c, u32 v) {
    if (c >= cr.hub)
        red_add_u64_if(&cr.s64[slot], (u64)v);
    else
        red_add_u32_if(&cr.s32[slot], v);
}
// dense windows: every c of a window lies in one counter tier, and the hub ids
// are exactly the 32-bit tier (cl == 0) -- a loop-invariant choice
__device__ __forceinline__ void credit_slot_tier(const Credits& cr, u64 slot, u32 cl, u32 v) {
    if (cl == 0)
        red_add_u64_if(&cr.s64[slot], (u64)v);
    else
        red_add_u32_if(&cr.s32[slot], v);
}

// one-use 8-byte load (run-end table) with the same evict-first policy
__device__ __forceinline__ u64 ld_u64_stream(const u64* p) {
    u64 v;
#ifdef GL_NO_L2_HINT
    v = __ldg(p);
#else
    asm volatile("{ .reg .b64 pol; createpolicy.fractional.L2::evict_first.b64 pol, 1.0;"
                 " ld.global.nc.L2::cache_hint.u64 %0, [%1], pol; }" : "=l"(v) : "l"(p));
#endif
    return v;
}

// Small tops: one warp per top vertex a, W[c] in a warp-private hash.
// per-warp shared words of k_cycle_small: keys u32[kHashSlots], counts u16
// packed in kHashSlots/2 words, the touched-slot list u16[kSmallWedges],
// the list length, and for tops with nb <= kSmallLocalB the run table
// pre u32[nb+1] (wedge prefix) and rbase u32[nb] (row base of b)
constexpr u32 kSmallLocalB = 128;
constexpr u32 kSmallWarpWords =
    kHashSlots + kHashSlots / 2 + (u32)kSmallWedges / 2 + 1 + (kSmallLocalB + 1) + kSmallLocalB;

__global__ void __launch_bounds__(kCycleSmallWarps * 32)
k_cycle_small(DevGraph g, const u64* __restrict__ wpre, const u32* __restrict__ items, u64 n_items,
              unsigned long long* __restrict__ queue, Credits cr) {
    extern __shared__ u32 smem[];
    const u32 lane = lane_id();
    const u32 wib = threadIdx.x >> 5;
    u32* keys = smem + wib * kSmallWarpWords;
    u32* cnt = keys + kHashSlots; // two u16 counts per word
    unsigned short* list = reinterpret_cast<unsigned short*>(cnt + kHashSlots / 2);
    u32* nlist = cnt + kHashSlots / 2 + (u32)kSmallWedges / 2;
    u32* pre = nlist + 1;
    u32* rbase = pre + kSmallLocalB + 1;
    for (u32 i = lane; i < kHashSlots; i += 32) keys[i] = kEmpty;
    for (u32 i = lane; i < kHashSlots / 2; i += 32) cnt[i] = 0;
    __syncwarp();
    for (;;) {
        unsigned long long idx = 0;
        if (lane == 0) idx = atomicAdd(queue, 1ull);
        idx = __shfl_sync(0xffffffffu, idx, 0);
        if (idx >= n_items) break;
        const u32 a = items[idx];
        const u64 E0 = g.loff[a], E1 = g.loff[a + 1];
        const u32 nb = (u32)(E1 - E0);
        const u64 w0 = wpre[E0];
        const u32 nw = (u32)(wpre[E1] - w0);
        // run table of the top in shared memory when small (the per-wedge run
        // search is then LDS), else searched in wpre
        const bool loc = nb <= kSmallLocalB;
        if (loc) {
            for (u32 j = lane; j < nb; j += 32) {
                pre[j] = (u32)(wpre[E0 + j] - w0);
                rbase[j] = (u32)g.off[g.eu[E0 + j]];
            }
            if (lane == 0) pre[nb] = nw;
        }
        if (lane == 0) *nlist = 0;
        __syncwarp();
        // wedge k -> (run j, adjacency slot)
        auto locate = [&](u32 k, u32& j, u64& slot) {
            if (loc) {
                j = upper_bound_dev<u32, u32>(pre, 0, nb + 1, k) - 1;
                slot = (u64)rbase[j] + (k - pre[j]);
            } else {
                const u64 gi = w0 + k;
                const u64 e = upper_bound_dev<u64, u64>(wpre, E0, E1 + 1, gi) - 1;
                j = (u32)(e - E0);
                slot = g.off[g.eu[e]] + (gi - wpre[e]);
            }
        };
        // pass 1: W[c]++; first inserts record their slot for the sparse clear
        for (u32 base = 0; base < nw; base += 32) {
            const u32 k = base + lane;
            bool fresh = false;
            u32 h = 0;
            if (k < nw) {
                u32 j;
                u64 slot;
                locate(k, j, slot);
                const u32 cv = g.adj[slot];
                h = hslot(cv);
                for (;;) {
                    const u32 prev = atomicCAS(&keys[h], kEmpty, cv);
                    if (prev == kEmpty) {
                        fresh = true;
                        break;
                    }
                    if (prev == cv) break;
                    h = (h + 1) & (kHashSlots - 1);
                }
                atomicAdd(&cnt[h >> 1], 1u << ((h & 1) << 4));
            }
            const unsigned bal = __ballot_sync(0xffffffffu, fresh);
            const u32 at = *nlist; // every lane reads before lane 0 advances it
            __syncwarp();
            if (fresh) list[at + __popc(bal & ((1u << lane) - 1u))] = (unsigned short)h;
            if (lane == 0) *nlist = at + __popc(bal);
            __syncwarp();
        }
        // pass 2: credit W[c]-1 to (b,c) and, summed per b, to (a,b)
        for (u32 base = 0; base < nw; base += 32) {
            const u32 k = base + lane;
            u32 j = 0xffffffffu;
            u64 val = 0;
            if (k < nw) {
                u64 slot;
                locate(k, j, slot);
                const u32 cv = g.adj[slot];
                u32 h = hslot(cv);
                while (keys[h] != cv) h = (h + 1) & (kHashSlots - 1);
                val = ((cnt[h >> 1] >> ((h & 1) << 4)) & 0xffffu) - 1u;
                if (val) credit_slot(cr, slot, cv, (u32)val);
            }
            u64 sum;
            const bool tail = seg_tail_sum(j, val, &sum);
            if (k < nw && tail && sum) atomic_add_i64(&cr.s64[g.off[a] + j], (i64)sum);
        }
        __syncwarp();
        // sparse clear: only the slots this top filled (a count word is shared
        // by slots h and h^1; both are either listed or already zero)
        const u32 nl = *nlist;
        for (u32 i = lane; i < nl; i += 32) {
            const u32 h = list[i];
            keys[h] = kEmpty;
            cnt[h >> 1] = 0;
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
__device__ __forceinline__ void st_shared(u32 addr, u32 v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ u32 ld_shared(u32 addr) {
    u32 v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
// RED.ADD.U64 to global issued under a predicate (no branch around it)

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
__device__ unsigned long long g_cycle_prof[64]; // [0..10] dense windows, [16..26] mid hash,
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

// Dense-window grid of a top with nb lower neighbours: windows never cross a
// degree tier; inside tier [t0, t1) (counter width 32 >> cl bits) they start at
// t0 + i * span.  span keeps nb * span < 2^31 (window wedge counts and indices
// are u32).  A fixed grid lets a top's c-range pieces cut on window boundaries
// (the pieces then hold exactly the windows of the unsplit top).
// Windows over the lowest-degree tier (cl >= kWalkCl = 4: 2-bit counters,
// degree < 4) hold short runs (RMAT-24: 6.4 wedges per run, 24% of the windows
// for 1.6% of the wedges): there each thread walks its b's runs itself (no run
// search, no scan, no flattening) and the window spans the whole dynamic
// shared memory (the run metadata is not needed).  The 4-bit tier walked too
// until the flattened mixed rounds went two at a time (measured: RMAT-20
// cycles -3% flattened, RMAT-24 +0.8%).  walk_cl = the lowest counter tier that
// walks (default kWalkCl; 5 = never, GL_WALK_CL overrides).
constexpr u32 kWalkCl = 4;
constexpr u32 kWalkWords = (kWindow + 3 * kMetaRuns) & ~3u; // Cyc<0>: WORDS + 3 * META (+1 unused)
__host__ __device__ __forceinline__ u64 win_span(u32 cl, u64 nb, u32 walk_cl) {
    if (cl >= walk_cl) return (u64)kWalkWords << cl;
    u64 span = (u64)kWindow << cl;
    // window wedges are scanned in 40 bits (nb * span bounds them); a window
    // that comes out above 2^31 wedges (u32 walk indices) is re-cut at run time
    if (nb * span >= (1ull << 40)) span = ((1ull << 40) / nb) & ~31ull;
    return span;
}
__device__ __forceinline__ u32 tier_of(u32 c, uint4 tiers, u32& t0, u32& t1) {
    if (c < tiers.x) { t0 = 0; t1 = tiers.x; return 4; }
    if (c < tiers.y) { t0 = tiers.x; t1 = tiers.y; return 3; }
    if (c < tiers.z) { t0 = tiers.y; t1 = tiers.z; return 2; }
    if (c < tiers.w) { t0 = tiers.z; t1 = tiers.w; return 1; }
    t0 = tiers.w;
    t1 = 0xffffffffu;
    return 0;
}
__device__ __forceinline__ u32 grid_floor(u32 c, uint4 tiers, u64 nb, u32 walk_cl) {
    u32 t0, t1;
    const u64 span = win_span(tier_of(c, tiers, t0, t1), nb, walk_cl);
    return t0 + (u32)(((u64)(c - t0) / span) * span);
}

// per-block scratch layout (cap = dmax + 2 entries each, cap even)
struct BigScratch {
    u32 *cur, *hpos, *rend, *pre, *rj, *rs, *nextc, *rwin, *plen, *lastc;
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
    s.lastc = s.plen + cap;                        // last c of b's row prefix N(b) n [0, a)
    return s;
}
__host__ __device__ inline u64 big_scratch_words(u32 cap) { return 12ull * cap + 8; }


// W[c] table of one block: dense window over c in [lo, lo+span) (big tops)
// or an open-addressing hash over all c < a (mid tops, HASH).  Hash keys are
// u32 (kEmpty = free), counts u16 packed two per word.
// cycle block kernel kinds: 0 dense windows (big tops), 1 block hash with
// 2^15 slots (mid tops), 2 block hash with 2^13 slots and four 256-thread
// blocks per SM (small-mid tops: their fixed per-top latency overlaps),
// 3 windowed block hash (sparse big tops: c windows cut by wedge count, not by
// the shared-memory span, so a top whose wedges are thin over a wide c range
// takes a few hash windows instead of many near-empty dense ones).  WIN: the
// c range is swept in windows with per-b cursors.
template <int KIND> struct Cyc;
template <> struct Cyc<0> {
    static constexpr bool HASH = false, WIN = true;
    static constexpr int THREADS = kBigThreads, MINB = kBigBlocksPerSM;
    static constexpr u32 LOG = 0, WORDS = kWindow, META = kMetaRuns;
};
template <> struct Cyc<1> {
    static constexpr bool HASH = true, WIN = false;
    static constexpr int THREADS = kMidThreads, MINB = 1;
    static constexpr u32 LOG = kMidLog, WORDS = (1u << kMidLog) * 3 / 2, META = 2048;
};
template <> struct Cyc<2> {
    static constexpr bool HASH = true, WIN = false;
    static constexpr int THREADS = kSmidThreads, MINB = 4;
    static constexpr u32 LOG = kSmidLog, WORDS = (1u << kSmidLog) * 3 / 2, META = 256;
};
template <> struct Cyc<3> {
    static constexpr bool HASH = true, WIN = true;
    static constexpr int THREADS = kMidThreads, MINB = 1;
    static constexpr u32 LOG = kMidLog, WORDS = (1u << kMidLog) * 3 / 2, META = 2048;
};
template <int KIND> __host__ __device__ constexpr u32 cyc_smem_words() {
    return Cyc<KIND>::WORDS + 3 * Cyc<KIND>::META + 1;
}


template <int KIND>
__device__ __forceinline__ void tab_inc(u32* W, u32 c, u32 lo, u32 cl) {
    constexpr u32 NS = 1u << Cyc<KIND>::LOG;
    if (Cyc<KIND>::HASH) {
        u32* keys = W;
        u32 h = (c * 0x9E3779B1u) >> ((32 - Cyc<KIND>::LOG) & 31);
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
        u32 h = (c * 0x9E3779B1u) >> ((32 - Cyc<KIND>::LOG) & 31);
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
__device__ __forceinline__ void wedge_op(u32* W, u32 wb, u32 cv, u32 lo, u32 cl, Credits cr, u64 slot,
                                         u64& val) {
    if (!Cyc<KIND>::HASH) { // dense window: 32-bit shared addresses (wb = W's), predicated RED
        const u32 ci = cv - lo;
        const u32 addr = wb + ((ci >> cl) << 2);
        const u32 sh = (ci & ((1u << cl) - 1u)) << (5 - cl);
        if (PASS == 0) {
            red_shared_add(addr, 1u << sh);
        } else if (PASS == 1) {
            const u32 w = ld_shared(addr) >> sh;
            const u32 v = (cl == 0 ? w : w & ((1u << (32u >> cl)) - 1u)) - 1u;
            credit_slot_tier(cr, slot, cl, v);
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
        if (v) credit_slot(cr, slot, cv, v);
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
// run take the uniform path: slot = base + lane, kUnroll/2 rounds of loads in
// flight, the (a,b) credit kept per lane and warp-reduced once per stretch.
// Rounds that straddle runs take the mixed path, two rounds per step: each
// lane finds its run from one OR-reduction of the run starts in its round,
// both rounds' adjacency loads are issued before either round's ops, and the
// (a,b) credit is a segmented shuffle sum whose tail lanes issue the RED.
//   PASS 0: W[c]++     PASS 1: credit W[c]-1 to (b,c) and, summed, to (a,b)
//   PASS 2: W[c] = 0 (sparse clear of a dense window)
#ifndef GL_KUNROLL
#define GL_KUNROLL 12
#endif
constexpr int kUnroll = GL_KUNROLL; // uniform-path rounds with loads in flight per lane (12: -1..2% vs 8 or 16)

template <bool B> struct HubTag { static constexpr bool v = B; };

template <int KIND, int PASS>
__device__ __forceinline__ void window_pass(const DevGraph& g, const RunMeta& S, u32 nnz, u32 kb, u32 ke, u32* W,
                                            u32 lo, u32 cl, u64 abase, Credits cr) {
    const u32 lane = lane_id();
    if (kb >= ke) return;
    const u32 wb = smem_u32(W);
    u32 bs = warp_upper_bound(S.pre, nnz + 1, kb);
    u32 k0 = kb;
    while (k0 < ke) {
        u32 e1 = S.pre[bs + 1];
        // bs holds wedge k0 - 1 or k0: runs are non-empty, so one step
        if (e1 <= k0) e1 = S.pre[++bs + 1];
        const u32 stop = e1 < ke ? e1 : ke;
        if (stop - k0 >= 32u) {
            // uniform stretch of full rounds inside run bs
            const u32 nfull = (stop - k0) >> 5;
#ifdef GL_CYCLE_PROF_ROUNDS
            if (KIND == 0 && PASS == 1 && lane_id() == 0) atomicAdd(&g_cycle_prof[12], (unsigned long long)nfull);
#endif
            // dense windows: the counter tier's hub/non-hub credit choice is
            // taken once per stretch, not per wedge
            auto stretch = [&](auto hubc) {
                constexpr bool HUB = decltype(hubc)::v;
                const u64 sbase = (u64)S.rs[bs] + (k0 - S.pre[bs]) + lane;
                u64 acc = 0;
                // every round of the stretch is full: branch-free wedge ops on a
                // hoisted shared base (dense windows), groups of kHalf rounds with
                // the next group's loads in flight; the last group overlaps the
                // (predicated) loads of the < kHalf tail rounds
                constexpr int kHalf = kUnroll / 2;
                const u32* __restrict__ src = g.adj + sbase;
                auto op = [&](u32 cv, u32 r) {
                    if constexpr (!Cyc<KIND>::HASH && HUB) {
                        const u32 addr = wb + ((cv - lo) << 2);
                        if (PASS == 0) {
                            red_shared_add(addr, 1u);
                        } else if (PASS == 1) {
                            const u32 v = ld_shared(addr) - 1u;
                            red_add_u64_if(&cr.s64[sbase + 32u * r], (u64)v);
                            acc += v;
                        } else {
                            st_shared(addr, 0u);
                        }
                    } else if constexpr (!Cyc<KIND>::HASH) {
                        const u32 ci = cv - lo;
                        const u32 addr = wb + ((ci >> cl) << 2);
                        const u32 sh = (ci & ((1u << cl) - 1u)) << (5 - cl);
                        if (PASS == 0) {
                            red_shared_add(addr, 1u << sh);
                        } else if (PASS == 1) {
                            const u32 w = ld_shared(addr) >> sh;
                            const u32 v = (w & ((1u << (32u >> cl)) - 1u)) - 1u; // cl >= 1 here
                            red_add_u32_if(&cr.s32[sbase + 32u * r], v);
                            acc += v;
                        } else {
                            st_shared(addr, 0u);
                        }
                    } else {
                        u64 v = 0;
                        wedge_op<KIND, PASS>(W, wb, cv, lo, cl, cr, sbase + 32u * r, v);
                        acc += v;
                    }
                };
                u32 r = 0;
                if (nfull >= (u32)kHalf) {
                    u32 cv[kHalf];
#pragma unroll
                    for (int u = 0; u < kHalf; ++u) cv[u] = __ldg(src + 32u * u);
                    for (; r + 2 * kHalf <= nfull; r += kHalf) {
                        u32 nx[kHalf];
#pragma unroll
                        for (int u = 0; u < kHalf; ++u) nx[u] = __ldg(src + 32u * (r + kHalf + u));
#pragma unroll
                        for (int u = 0; u < kHalf; ++u) op(cv[u], r + u);
#pragma unroll
                        for (int u = 0; u < kHalf; ++u) cv[u] = nx[u];
                    }
                    // the final group with the < kHalf tail rounds' loads in flight
                    u32 tl[kHalf];
#pragma unroll
                    for (int u = 0; u < kHalf; ++u) tl[u] = r + kHalf + u < nfull ? __ldg(src + 32u * (r + kHalf + u)) : 0u;
#pragma unroll
                    for (int u = 0; u < kHalf; ++u) op(cv[u], r + u);
                    r += kHalf;
#pragma unroll
                    for (int u = 0; u < kHalf; ++u)
                        if (r + u < nfull) op(tl[u], r + u);
                    r = nfull;
                }
                // the < kHalf remaining rounds: all loads in flight, then the ops
                if (r < nfull) {
                    u32 cv[kHalf];
#pragma unroll
                    for (int u = 0; u < kHalf; ++u) cv[u] = r + u < nfull ? __ldg(src + 32u * (r + u)) : 0u;
#pragma unroll
                    for (int u = 0; u < kHalf; ++u)
                        if (r + u < nfull) op(cv[u], r + u);
                }
                if (PASS == 1) {
                    acc = warp_sum_u64(acc);
                    if (lane == 0 && acc) atomic_add_i64(&cr.s64[abase + S.rj[bs]], (i64)acc);
                }
                k0 += nfull << 5;
            };
            if constexpr (Cyc<KIND>::HASH) {
                stretch(HubTag<false>{});
            } else {
                if (cl == 0)
                    stretch(HubTag<true>{});
                else
                    stretch(HubTag<false>{});
            }
        } else {
            // mixed round [k0, k0 + 32): runs bs, bs+1, ... start at pre[bs+j];
            // one OR-reduction gives the bitmask of run starts inside the round,
            // from which every lane reads its run (popcount), its offset and
            // its segment (highest start at or below it)
#ifdef GL_CYCLE_PROF_ROUNDS
            if (KIND == 0 && PASS == 1 && lane_id() == 0) atomicAdd(&g_cycle_prof[13], 1ull);
#endif
            // two rounds per step when the warp's range allows: both rounds'
            // lanes mapped to (run, slot) and both adjacency loads in flight
            // before either round's wedge ops.
            auto map = [&](u32 r0, u32 b0, u32& starts, u32& seg0, u32& q, u32& off) {
                const u32 pi = b0 + lane <= nnz ? S.pre[b0 + lane] : 0xffffffffu;
                const u32 rel = pi - r0; // >= 1 for lanes >= 1 (b0 holds wedge r0)
                starts = __reduce_or_sync(0xffffffffu, (lane > 0 && rel < 32u) ? 1u << rel : 0u);
                const u32 le = starts & (0xffffffffu >> (31 - lane));
                const u32 owner = __popc(le);
                q = b0 + owner;
                seg0 = owner ? 31u - __clz(le) : 0u;
                const u32 pi0 = __shfl_sync(0xffffffffu, pi, 0);
                off = owner ? lane - seg0 : r0 + lane - pi0;
            };
            auto finish = [&](u32 r0, u32 starts, u32 seg0, u32 q, u64 slot, u32 cv) {
                const u32 k = r0 + lane;
                const bool valid = k < ke;
                u64 v = 0;
                if (valid) wedge_op<KIND, PASS>(W, wb, cv, lo, cl, cr, slot, v);
                if (PASS == 1) {
                    const bool tail = valid && (lane == 31 || k + 1 == ke || ((starts >> (lane + 1)) & 1u));
                    if (cl) {
                        u32 v32 = (u32)v;
#pragma unroll
                        for (int d = 1; d < 32; d <<= 1) {
                            const u32 t = __shfl_up_sync(0xffffffffu, v32, d);
                            if (lane >= seg0 + (u32)d) v32 += t;
                        }
                        if (tail && v32) atomic_add_i64(&cr.s64[abase + S.rj[q]], (i64)v32);
                    } else {
#pragma unroll
                        for (int d = 1; d < 32; d <<= 1) {
                            const u64 t = __shfl_up_sync(0xffffffffu, v, d);
                            if (lane >= seg0 + (u32)d) v += t;
                        }
                        if (tail && v) atomic_add_i64(&cr.s64[abase + S.rj[q]], (i64)v);
                    }
                }
            };
            u32 st1, sg1, q1, of1;
            map(k0, bs, st1, sg1, q1, of1);
            const bool v1 = k0 + lane < ke;
            const u64 sl1 = v1 ? (u64)S.rs[q1] + of1 : 0ull;
            const u32 c1 = v1 ? __ldg(g.adj + sl1) : 0u;
            u32 bs2 = __shfl_sync(0xffffffffu, q1, 31);
            if (k0 + 32u < ke) {
                // the run holding wedge k0 + 32: the last round's, or the next
                // when that one ends at the boundary (a round sees 31 starts)
                bs2 += S.pre[bs2 + 1] <= k0 + 32u ? 1u : 0u;
                u32 st2, sg2, q2, of2;
                map(k0 + 32u, bs2, st2, sg2, q2, of2);
                const bool v2 = k0 + 32u + lane < ke;
                const u64 sl2 = v2 ? (u64)S.rs[q2] + of2 : 0ull;
                const u32 c2 = v2 ? __ldg(g.adj + sl2) : 0u;
                finish(k0, st1, sg1, q1, sl1, c1);
                finish(k0 + 32u, st2, sg2, q2, sl2, c2);
                k0 += 64;
                bs = __shfl_sync(0xffffffffu, q2, 31);
            } else {
                finish(k0, st1, sg1, q1, sl1, c1);
                k0 += 32;
                bs = bs2;
            }
        }
    }
}

// Guided self-scheduling of a window pass: a warp grabs about 1/(2*nwarps) of
// the wedges still unclaimed (at most 8192, at least 64), so the grabs shrink
// towards the end of the pass and the block's barrier waits for a short tail.
#ifndef GL_GRAB_DIV
#define GL_GRAB_DIV 2
#endif
#ifndef GL_GRAB_MAX
#define GL_GRAB_MAX 8192
#endif
__device__ __forceinline__ u32 grab_size(u32 remaining, u32 nwarps) {
    u32 g = remaining / (GL_GRAB_DIV * nwarps);
    g = g < (u32)GL_GRAB_MAX ? g : (u32)GL_GRAB_MAX;
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
                                          u32 lo, u32 cl, u64 abase, Credits cr) {
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
        window_pass<KIND, PASS>(g, M, nnz, k0, k0 + grab < T ? k0 + grab : T, W, lo, cl, abase, cr);
    }
}

// Bulk reset of the first `words` table words (a multiple of 4) with 16-byte
// stores: hash key words (< kslots) to kEmpty, counter words to 0.
__device__ __forceinline__ void table_clear(u32* W, u32 words, u32 kslots, u32 threads) {
    uint4* W4 = reinterpret_cast<uint4*>(W);
    const uint4 e = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty), z = make_uint4(0, 0, 0, 0);
    for (u32 i = threadIdx.x; i < words / 4; i += threads) W4[i] = 4 * i < kslots ? e : z;
}

// One pass over a window's runs.  Run metadata that did not fit in shared
// memory (nnz > kMeta, written to the block's global scratch by the
// compaction) is staged back through shared memory kMeta runs at a time, so
// the walk's run lookups stay LDS instead of dependent L2 round trips; the
// W window is complete before the pass starts, so chunking changes nothing.
template <int KIND, int PASS>
__device__ __forceinline__ void meta_pass(const DevGraph& g, const RunMeta& Msm, const RunMeta& Mgl, u32 nnz, u32 T,
                                          u32* counter, u32* W, u32 lo, u32 cl, u64 abase,
                                          Credits cr) {
    constexpr u32 kMeta = Cyc<KIND>::META;
    if (nnz <= kMeta) {
        grab_pass<KIND, PASS>(g, Msm, nnz, T, counter, W, lo, cl, abase, cr);
        return;
    }
    for (u32 q0 = 0; q0 < nnz; q0 += kMeta) {
        const u32 nq = nnz - q0 < kMeta ? nnz - q0 : kMeta;
        const u32 base = Mgl.pre[q0], end = Mgl.pre[q0 + nq];
        __syncthreads(); // the previous chunk's walkers are done with Msm
        for (u32 i = threadIdx.x; i <= nq; i += blockDim.x) {
            Msm.pre[i] = Mgl.pre[q0 + i] - base;
            if (i < nq) {
                Msm.rs[i] = Mgl.rs[q0 + i];
                Msm.rj[i] = Mgl.rj[q0 + i];
            }
        }
        if (threadIdx.x == 0) *counter = 0;
        __syncthreads();
        grab_pass<KIND, PASS>(g, Msm, nq, end - base, counter, W, lo, cl, abase, cr);
    }
}

// Thread-walk window [lo, hi) of a dense top (low-degree tiers): each thread
// walks the runs of its b's (b = thread + i * THREADS) from the cursor while
// c < hi -- pass 0 increments W and finds the run end as it goes, pass 1
// re-walks the run crediting W-1 to (b,c) and the run's sum to (a,b); then the
// used window words are bulk-cleared.  Four entries of a row are loaded per
// step (one sector, independent loads).
constexpr int kWalkStep = 4;
__device__ __noinline__ void walk_window(const DevGraph& g, const BigScratch& S, u32 nb, u32* W, u32 lo, u32 hi,
                                            u32 cl, u32 win, u64 abase, Credits cr) {
    const u32 wb = smem_u32(W);
    const u32 T = blockDim.x;
#ifdef GL_CYCLE_PROF
    u32 pr = 0, pw = 0;
#endif
    // pass 0: kNcBatch cursor-c loads in flight, then walk the active b's
    for (u32 j0 = threadIdx.x; j0 < nb; j0 += kNcBatch * T) {
        u32 nc[kNcBatch];
#pragma unroll
        for (int u = 0; u < kNcBatch; ++u) nc[u] = j0 + u * T < nb ? S.nextc[j0 + u * T] : kEmpty;
#pragma unroll 1
        for (int u = 0; u < kNcBatch; ++u) {
            u32 c = nc[u];
            if (c >= hi) continue; // kEmpty >= hi
            const u32 j = j0 + u * T;
            const u64 rb = S.rb[j];
            const u32 re = S.rend[j], h0 = S.cur[j];
            u32 h = h0;
            for (;;) {
                u32 nx[kWalkStep];
#pragma unroll
                for (int v = 0; v < kWalkStep; ++v) nx[v] = h + 1 + v < re ? __ldg(g.adj + rb + h + 1 + v) : kEmpty;
                bool stop = false;
#pragma unroll
                for (int v = 0; v < kWalkStep; ++v) {
                    if (!stop) {
                        const u32 ci = c - lo;
                        red_shared_add(wb + ((ci >> cl) << 2), 1u << ((ci & ((1u << cl) - 1u)) << (5 - cl)));
                        ++h;
                        c = nx[v];
                        stop = c >= hi;
                    }
                }
                if (stop) break;
            }
#ifdef GL_CYCLE_PROF
            ++pr;
            pw += h - h0;
#endif
            S.hpos[j] = h0;
            S.cur[j] = h;
            S.nextc[j] = c; // >= hi or kEmpty
            S.rwin[j] = win;
        }
    }
#ifdef GL_CYCLE_PROF
    pr = __reduce_add_sync(0xffffffffu, pr);
    pw = __reduce_add_sync(0xffffffffu, pw);
    if (lane_id() == 0) {
        atomicAdd(&g_cycle_prof[33 + 4 * cl], (unsigned long long)pr);
        atomicAdd(&g_cycle_prof[34 + 4 * cl], (unsigned long long)pw);
    }
    if (threadIdx.x == 0) atomicAdd(&g_cycle_prof[32 + 4 * cl], 1ull);
#endif
    __syncthreads();
    // pass 1: re-walk the runs of this window, W-1 to (b,c), the run's sum to (a,b)
    for (u32 j0 = threadIdx.x; j0 < nb; j0 += kNcBatch * T) {
        u32 rw[kNcBatch];
#pragma unroll
        for (int u = 0; u < kNcBatch; ++u) rw[u] = j0 + u * T < nb ? S.rwin[j0 + u * T] : kEmpty;
#pragma unroll 1
        for (int u = 0; u < kNcBatch; ++u) {
            if (rw[u] != win) continue;
            const u32 j = j0 + u * T;
            const u64 rb = S.rb[j];
            const u32 h1 = S.cur[j];
            u64 sum = 0;
            for (u32 p = S.hpos[j]; p < h1; p += kWalkStep) {
                u32 cv[kWalkStep];
#pragma unroll
                for (int v = 0; v < kWalkStep; ++v) cv[v] = p + v < h1 ? __ldg(g.adj + rb + p + v) : kEmpty;
#pragma unroll
                for (int v = 0; v < kWalkStep; ++v) {
                    if (cv[v] != kEmpty) {
                        const u32 ci = cv[v] - lo;
                        const u32 w = ld_shared(wb + ((ci >> cl) << 2)) >> ((ci & ((1u << cl) - 1u)) << (5 - cl));
                        const u32 val = (w & ((1u << (32u >> cl)) - 1u)) - 1u;
                        red_add_u32_if(&cr.s32[rb + p + v], val); // walk tiers: cl >= 1, never the hub tier
                        sum += val;
                    }
                }
            }
            if (sum) atomic_add_i64(&cr.s64[abase + j], (i64)sum);
        }
    }
    __syncthreads();
    const u32 words = (hi - lo + (1u << cl) - 1u) >> cl;
    table_clear(W, (words + 3u) & ~3u, 0u, T);
    __syncthreads();
}

template <int KIND>
__global__ void __launch_bounds__(Cyc<KIND>::THREADS, Cyc<KIND>::MINB)
k_cycle_block(DevGraph g, const u32* __restrict__ items, const uint4* __restrict__ pieces, u64 n_items,
              unsigned long long* __restrict__ queue, Credits cr, u32* __restrict__ gscratch, u32 cap,
              uint4 tiers, u32 walk_cl, const u64* __restrict__ nxt_rev) {
    constexpr bool HASH = Cyc<KIND>::HASH, WIN = Cyc<KIND>::WIN;
    constexpr int THREADS = Cyc<KIND>::THREADS;
    constexpr u32 kWords = Cyc<KIND>::WORDS, kMeta = Cyc<KIND>::META, kSlots = 1u << Cyc<KIND>::LOG;
    extern __shared__ u32 W[]; // kWords table words, then the run metadata
    __shared__ unsigned long long s_idx;
    __shared__ u32 s_next, s_work[3];
    BigScratch S = big_scratch(gscratch + (u64)blockIdx.x * ((big_scratch_words(cap) + 1) & ~1ull), cap);
    const RunMeta Msm{W + kWords, W + kWords + kMeta + 1, W + kWords + 2 * kMeta + 1};
    const RunMeta Mgl{S.pre, S.rs, S.rj};
    table_clear(W, kWords, HASH ? kSlots : 0u, THREADS);
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
        // windowed kinds take pieces (a, clo, chi, wedge estimate): the wedges
        // of top a whose c lies in [clo, chi) -- a heavy top is split into
        // c-range pieces that different blocks (and ranks) take; every credit is
        // an atomic add, so the pieces of a top sum exactly
        uint4 pc = make_uint4(0, 0, 0, 0);
        if constexpr (WIN) {
            pc = pieces[idx];
            if (pc.x == kEmpty) continue; // empty piece (its cut points coincided)
        }
        const u32 a = WIN ? pc.x : items[idx];
        const u32 clo = pc.y, chi = WIN ? pc.z : a;
        const u64 E0 = g.loff[a];
        const u32 nb = (u32)(g.loff[a + 1] - E0);
        const u64 abase = g.off[a]; // slot of (a, b_j) is abase + j: L(a) is the row prefix

        if constexpr (!WIN) {
            // Hash tops take all c < a in one window: b's run is its whole row
            // prefix N(b) n [0, a) (|.| = epos), so the runs are placed straight
            // from (eu, epos) -- no cursors, no scratch round trips.
            u32 my_runs = 0, my_wedges = 0;
            for (u32 j = threadIdx.x; j < nb; j += THREADS) {
                const u32 re = g.epos[E0 + j];
                my_runs += re > 0;
                my_wedges += re;
            }
            u64 tot, mine = ((u64)my_runs << 32) | my_wedges;
            {
                using BlockScan = cub::BlockScan<u64, THREADS>;
                __shared__ typename BlockScan::TempStorage tmp;
                BlockScan(tmp).ExclusiveSum(mine, mine, tot);
            }
            const u32 nnz = (u32)(tot >> 32), T = (u32)tot;
            const RunMeta M = nnz <= kMeta ? Msm : Mgl;
            u32 q = (u32)(mine >> 32), w = (u32)mine;
            for (u32 j = threadIdx.x; j < nb && my_runs; j += THREADS) {
                const u64 e = E0 + j;
                const u32 re = g.epos[e];
                if (!re) continue;
                M.rj[q] = j;
                M.rs[q] = (u32)g.off[g.eu[e]];
                M.pre[q] = w;
                ++q;
                w += re;
            }
            if (threadIdx.x == 0) M.pre[nnz] = T;
            if (threadIdx.x < 3) s_work[threadIdx.x] = 0;
            __syncthreads();
            GL_PROF_MARK(2);
            GL_PROF_ADD(8, 1);
            GL_PROF_ADD(9, T);
            GL_PROF_ADD(10, 1);
            if (T) {
                meta_pass<KIND, 0>(g, Msm, Mgl, nnz, T, &s_work[0], W, 0, 1, abase, cr);
                __syncthreads();
                GL_PROF_MARK(3);
                meta_pass<KIND, 1>(g, Msm, Mgl, nnz, T, &s_work[1], W, 0, 1, abase, cr);
                __syncthreads();
                GL_PROF_MARK(4);
                table_clear(W, kWords, kSlots, THREADS);
            }
            GL_PROF_SYNC_MARK(7);
            continue;
        }
        if (threadIdx.x == 0) s_next = WIN ? kEmpty : 0u;
        __syncthreads();
        // per-b row base and run end (|N(b) n [0,a)| = epos), cursors at the
        // piece's first c (0 for an unsplit top or a first piece); the piece's
        // upper end chi is a window boundary, found by the window loop's run search
        for (u32 j = threadIdx.x; j < nb; j += THREADS) {
            const u64 e = E0 + j;
            const u64 rb = g.off[g.eu[e]];
            const u32 re = g.epos[e];
            S.rb[j] = rb;
            S.rend[j] = re;
            u32 c0 = 0;
            const u32 lc = re > 0 ? g.adj[rb + re - 1] : 0u;
            if (clo && re) {
                // seek the piece's first c: gallop from an interpolated position
                const u32 fc = g.adj[rb];
                if (lc < clo) {
                    c0 = re;
                } else if (fc < clo) {
                    const u64 hint = (u64)(re - 1) * (clo - fc) / (lc - fc);
                    c0 = (u32)(gallop_from(g.adj, rb, rb + re, rb + hint, clo) - rb);
                }
            }
            S.cur[j] = c0;
            const u32 c = c0 < re ? g.adj[rb + c0] : kEmpty;
            if (WIN) S.lastc[j] = lc;
            S.nextc[j] = c < chi ? c : kEmpty;
            S.rwin[j] = kEmpty;
            S.plen[j] = 0;
            if (WIN && c < chi) atomicMin(&s_next, c);
        }
        __syncthreads();
        u64 rem = pc.w; // wedges of this piece not yet in a window (KIND 3 window sizing; estimate for a split top)
        GL_PROF_MARK(0);
        GL_PROF_ADD(10, 1);
        // Windows from the smallest c on.  Each b keeps its cursor and the c
        // value under it (nextc), so a window only gallops the b's whose next c
        // falls inside it; for the others one coalesced nextc load suffices.
        u32 win = 0;
        bool meta_dirty = true; // block-uniform: run metadata may sit in the walk windows' words
        // dense windows start on the top's window grid (so pieces cut on grid
        // points reproduce the unsplit top's windows); hash windows at s_next
        u32 lo0 = s_next;
        if (!HASH && lo0 < chi) {
            lo0 = grid_floor(lo0, tiers, nb, walk_cl);
            lo0 = lo0 > clo ? lo0 : clo;
        }
        for (u32 lo = lo0, hi = 0; lo < chi; lo = hi, ++win) {
            // window [lo, hi): inside one degree tier, counters of that tier's width
            u32 cl = 1, tend = chi;
            if (!HASH) {
                cl = lo < tiers.x ? 4u : lo < tiers.y ? 3u : lo < tiers.z ? 2u : lo < tiers.w ? 1u : 0u;
                tend = lo < tiers.x ? tiers.x : lo < tiers.y ? tiers.y : lo < tiers.z ? tiers.z : lo < tiers.w ? tiers.w : chi;
                tend = tend < chi ? tend : chi;
            }
            u64 span = win_span(cl, nb, walk_cl);
            if (KIND == 3) { // about kHashWinTarget wedges if they were uniform over [lo, chi)
                span = rem ? (u64)(chi - lo) * kHashWinTarget / rem : (u64)(chi - lo);
                span = span ? span : 1;
                // keep nb * span < 2^31: window wedge counts and indices are u32
                if ((u64)nb * span >= (1ull << 31)) span = ((1ull << 31) / nb) & ~31ull;
            }
            hi = !WIN ? a : (u32)std::min<u64>(std::min<u64>((u64)lo + span, (u64)tend), (u64)chi);

            if constexpr (!HASH) {
                if (cl >= walk_cl) {
                    // short runs: thread-walk window (see kWalkCl).  The window
                    // words reach into the run-metadata area: clear it first if a
                    // flattened window of the previous top used it.
                    if (meta_dirty) {
                        table_clear(W + kWords, kWalkWords - kWords, 0u, THREADS);
                        __syncthreads();
                        meta_dirty = false;
                    }
                    walk_window(g, S, nb, W, lo, hi, cl, win, abase, cr);
                    GL_PROF_MARK(3);
                    continue;
                }
            }
            u32 my_runs, nnz, T;
            u64 my_wedges, mine;
            constexpr u32 kRunShift = 40; // (runs << 40) | wedges: runs <= nb < 2^24 (host check)
            // run ends from the per-slot next-window table (k_run_table): one
            // load instead of a gallop, when this window is on the global grid
            // (not re-cut, top below the span clamp)
            bool grid_ends = KIND == 0 && nxt_rev != nullptr && (u64)nb * ((u64)kWalkWords << 4) < (1ull << 40);
            for (;;) {
                // run ends of the b's with a c in [lo, hi); runs are ordered
                // thread-major (thread t owns b = t + i*THREADS), so one block scan
                // of per-thread (runs, wedges) places them
                my_runs = 0, my_wedges = 0;
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
                        u32 h = re, cn = kEmpty;
                        bool have_cn = false;
                        // the row's last window needs no search: its run ends at re
                        if (WIN && S.lastc[j] >= hi) {
                            if (grid_ends) {
                                // first slot after rb + c0 on a later window (or row start)
                                // and the c there, in one load
                                const u64 p1 = rb + c0 + 1;
                                const u64 v = p1 < 2 * g.m ? ld_u64_stream(nxt_rev + (2 * g.m - 1 - p1)) : ~0ull;
                                const u64 qe = (v >> 32) - rb;
                                if (qe < (u64)re) {
                                    h = (u32)qe;
                                    cn = (u32)v;
                                    have_cn = true;
                                }
                            } else {
                                const u32 pl = S.plen[j];
                                h = (u32)(gallop_from(g.adj, rb + c0, rb + re, rb + c0 + (pl ? pl - 1 : 0), hi) - rb);
                                S.plen[j] = h - c0;
                            }
                        }
                        S.hpos[j] = c0; // run start
                        S.rwin[j] = win;
                        S.cur[j] = h;
                        S.nextc[j] = h < re ? (have_cn ? cn : g.adj[rb + h]) : kEmpty;
                        ++my_runs;
                        my_wedges += h - c0;
                    }
                }
                GL_PROF_SYNC_MARK(6);
                u64 tot;
                mine = ((u64)my_runs << kRunShift) | my_wedges;
                {
                    using BlockScan = cub::BlockScan<u64, THREADS>;
                    __shared__ typename BlockScan::TempStorage tmp;
                    BlockScan(tmp).ExclusiveSum(mine, mine, tot);
                }
                nnz = (u32)(tot >> kRunShift);
                const u64 T64 = tot & ((1ull << kRunShift) - 1);
                T = (u32)T64;
                // a dense window above 2^31 wedges (u32 walk indices; only a
                // top with a huge lower neighbourhood): restore its b's cursors
                // and halve it (the run ends are then off the window grid: the
                // gallop finds them)
                if constexpr (KIND == 0) {
                    if (T64 < (1ull << 31)) break;
                    for (u32 j = threadIdx.x; j < nb; j += THREADS) {
                        if (S.rwin[j] != win) continue;
                        const u32 c0 = S.hpos[j];
                        S.cur[j] = c0;
                        S.nextc[j] = g.adj[S.rb[j] + c0];
                        S.rwin[j] = kEmpty;
                    }
                    __syncthreads(); // BlockScan storage reuse
                    hi = lo + std::max<u32>((hi - lo) / 2, 32u);
                    grid_ends = false;
                    continue;
                }
                // a KIND 3 window over its wedge cap: restore its b's cursors
                // and re-cut it narrower (a window of <= kHashWinMax ids is
                // always accepted: its distinct c ids fit the slots anyway)
                if constexpr (KIND == 3) {
                    if (T <= kHashWinMax || hi - lo <= kHashWinMax) break;
#ifdef GL_CYCLE_PROF
                    if (threadIdx.x == 0) atomicAdd(&g_cycle_prof[29], 1ull); // KIND 3 re-cuts
#endif
                    for (u32 j = threadIdx.x; j < nb; j += THREADS) {
                        if (S.rwin[j] != win) continue;
                        const u32 c0 = S.hpos[j];
                        S.cur[j] = c0;
                        S.nextc[j] = g.adj[S.rb[j] + c0];
                        S.rwin[j] = kEmpty;
                    }
                    __syncthreads(); // BlockScan storage reuse
                    const u64 nspan = (u64)(hi - lo) * kHashWinTarget / T;
                    hi = lo + (u32)(nspan ? nspan : 1);
                } else {
                    break;
                }
            }
            rem = rem > T ? rem - T : 0;
#ifdef GL_CYCLE_PROF
            if (KIND == 3 && threadIdx.x == 0) {
                atomicAdd(&g_cycle_prof[30], 1ull);
                atomicAdd(&g_cycle_prof[31], (unsigned long long)T);
            }
#endif
            GL_PROF_MARK(1);
            GL_PROF_ADD(8, 1);
            GL_PROF_ADD(9, T);
#ifdef GL_CYCLE_PROF
            if (KIND == 0 && threadIdx.x == 0) {
                // per counter tier cl (4 = 2-bit ... 0 = 32-bit): windows, runs, wedges
                atomicAdd(&g_cycle_prof[32 + 4 * cl], 1ull);
                atomicAdd(&g_cycle_prof[33 + 4 * cl], (unsigned long long)nnz);
                atomicAdd(&g_cycle_prof[34 + 4 * cl], (unsigned long long)T);
                atomicAdd(&g_cycle_prof[11], (unsigned long long)nnz);
                if (nnz > kMeta) {
                    atomicAdd(&g_cycle_prof[14], 1ull);
                    atomicAdd(&g_cycle_prof[15], (unsigned long long)T);
                }
            }
#endif
            const RunMeta M = nnz <= kMeta ? Msm : Mgl;
            if (!HASH) meta_dirty = true;
            if (my_runs) {
                u32 q = (u32)(mine >> kRunShift), w = (u32)(mine & ((1ull << kRunShift) - 1));
                for (u32 j0 = threadIdx.x; j0 < nb && q < (u32)(mine >> kRunShift) + my_runs; j0 += kNcBatch * THREADS) {
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
                    meta_pass<KIND, 0>(g, Msm, Mgl, nnz, T, &s_work[0], W, lo, cl, abase, cr);
                }
                __syncthreads();
                GL_PROF_MARK(3);
                {
                    meta_pass<KIND, 1>(g, Msm, Mgl, nnz, T, &s_work[1], W, lo, cl, abase, cr);
                }
                __syncthreads();
                GL_PROF_MARK(4);
                if (bulk_clear) {
                    const u32 words = HASH ? kWords : (hi - lo + (1u << cl) - 1u) >> cl;
                    table_clear(W, (words + 3u) & ~3u, HASH ? kSlots : 0u, THREADS);
                } else if (!HASH) {
                    meta_pass<KIND, 2>(g, Msm, Mgl, nnz, T, &s_work[2], W, lo, cl, abase, cr);
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
__global__ void k_fold_slots(DevGraph g, Credits cr, i64* __restrict__ part) {
    for (u64 e = blockIdx.x * (u64)blockDim.x + threadIdx.x; e < g.m; e += (u64)gridDim.x * blockDim.x) {
        const u32 v = g.ev[e], u = g.eu[e];
        const u64 p1 = g.off[v] + (e - g.loff[v]), p2 = g.off[u] + g.epos[e];
        const i64 s = cr.s64[p1] + cr.s64[p2] + (i64)cr.s32[p1] + (i64)cr.s32[p2];
        if (s) part[2 * e + 1] += s;
    }
}

