// graph.cuh -- device-resident preprocessed graph (the B200 counterpart of
// graphlet::Graph, /root/reference/proj/include/graphlet/graph.hpp:41-93).
//
// HBM layout (one replica per GPU):
//   off   u64[n+1]  row offsets of the symmetric CSR
//   adj   u32[2m]   neighbours, ascending internal id per row (P1-relabelled)
//   eid   u32[2m]   oriented edge id of every adjacency slot
//   lcnt  u32[n]    |L(v)| = # neighbours with smaller id; L(v) is the row
//                   prefix, U(v) the suffix (degree-ordered DAG)
//   loff  u64[n+1]  exclusive prefix of lcnt = first edge id with v as the
//                   high endpoint (orient_edges order, graph.cpp:180-193)
//   ev/eu u32[m]    endpoints of edge id e (v high, u low)
//   epos  u32[m]    position of v inside u's row (so U(u) after v starts at
//                   off[u] + epos + 1, and |{c in N(u) : c < v}| = epos)
//   deg   u32[n], label u64[n]
#pragma once

#include <atomic>

#include "common.cuh"

namespace gl {

struct DevGraph {
    u64 n = 0, m = 0;
    u32 dmax = 0;
    u64* off = nullptr;
    u32* adj = nullptr;
    u32* eid = nullptr;
    u32* lcnt = nullptr;
    u64* loff = nullptr;
    u32* ev = nullptr;
    u32* eu = nullptr;
    u32* epos = nullptr;
    u32* deg = nullptr;
    u64* label = nullptr;
};

// Process-wide caching allocator (host.cpp): freed blocks are kept per device
// and handed out again for requests of at most their size and at least half
// of it, so building and counting a new graph every step does not pay
// cudaMalloc / cudaFree of the multi-GB working set each time.
void* pool_alloc(size_t bytes, int device, size_t* got);
void pool_free(void* p, size_t bytes, int device);
void pool_trim();

// RAII device buffer (pool-backed)
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    int dev = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { reset(); }
    void reset() {
        if (p) pool_free(p, bytes, dev);
        p = nullptr;
        bytes = 0;
    }
    void alloc(size_t b) {
        if (b <= bytes && p) return;
        reset();
        if (b == 0) b = 16;
        GL_CUDA(cudaGetDevice(&dev));
        p = pool_alloc(b, dev, &bytes);
    }
    template <typename T> T* as() const { return static_cast<T*>(p); }
};

// Per-graph counting state (device arrays reused across calls).
struct CountState {
    DevBuf t;        // u32[m]   triangles per edge
    DevBuf x7, x10;  // u64[m]   micro outputs of the last shard
    DevBuf part;     // i64[2m]  partials for the single-process path
    DevBuf slots;    // i64[2m]  C4 credits per adjacency slot (folded into y): hub c and the (a,b) run sums
    DevBuf slots32;  // u32[2m]  the same for c of degree < 65536 (cycles.cuh Credits)
    DevBuf hlist;    // per-block H-edge lists of the clique pass
    DevBuf tlist, tl_base, tl_n; // persistent H-edge records for the triangle-sum pass
    u64 tl_cap = 0;
    bool tl_sized = false;
    u32 tl_exact = 0;   // exact record reservations (hpass.cuh TriList::exact)
    DevBuf wpre;     // u64[m+1] wedge prefix per edge for the cycle kernels
    DevBuf items2, items3s, items3m, items3b, items3x; // work lists
    DevBuf keys, tmp, scratch, cursor, cursor2, acc; // sort keys, cub temp, kernel scratch
    DevBuf keys_c, items_c, tmp_c; // the cycle pass's own (it runs concurrently on s2)
    DevBuf pieces;                 // uint4 (a, clo, chi, wedge estimate): windowed-top pieces, then the rank's share
    u64 cycle_pieces = 0;
    DevBuf runtab;                 // u64[2m] run-end table of the dense cycle windows: (end slot, c there) (count.cu k_run_flags)
    // early copy-out (gl_count_edges): t and x7 are final after the H-pass, so
    // they go to these host buffers on s3 while the cycle pass runs
    std::uint32_t* out_t = nullptr;
    std::uint64_t* out_x7 = nullptr;
    cudaStream_t s3 = nullptr;
    cudaEvent_t ev_out = nullptr;
    u32 runtab_key = 0;            // walk_cl + 1 it was built for (0: none)
    DevBuf tierbuf;                // u32[4] degree tiers of the window counters (count.cu k_tiers)
    uint4 tiers = {0, 0, 0, 0};
    bool tiers_valid = false;
    cudaStream_t s2 = nullptr;     // cycle-pass stream (owned)
    cudaEvent_t ev[8] = {};        // phase events: 0/1 H-pass, 2/3 cycles, 4/5 sums, 6 fork, 7 end of count_mid
    u64 n_items2 = 0, n_items3s = 0, n_items3m = 0, n_items3b = 0, n_items3x = 0;
    u64 shard_begin = 0, shard_end = 0;
    bool have_micro = false;
    bool began = false;
    bool mid_done = false;
    int rank = 0, world = 1;
    u64 s1 = 0, h_gstride = 0; // H-pass streamed entries, global workspace stride
    u32 h_kmax = 0;            // largest |U(a)| of the last count
    float ms[5] = {0, 0, 0, 0, 0};
    u32 launches = 0;
    u64 work[4] = {0, 0, 0, 0};
};

struct Graph {
    int device = 0;
    cudaStream_t stream = nullptr;
    DevGraph d;
    DevBuf b_off, b_adj, b_eid, b_lcnt, b_loff, b_ev, b_eu, b_epos, b_deg, b_label;
    CountState cs;
    ~Graph() {
        // kernels of an unfinished count may still write the buffers that go
        // back to the (stream-unaware) pool below, on the graph's streams or a
        // caller's: drain the device before releasing them
        cudaSetDevice(device);
        cudaDeviceSynchronize();
        if (cs.s3) {
            cudaStreamSynchronize(cs.s3);
            cudaStreamDestroy(cs.s3);
            if (cs.ev_out) cudaEventDestroy(cs.ev_out);
        }
        if (cs.s2) {
            cudaStreamSynchronize(cs.s2);
            for (auto e : cs.ev)
                if (e) cudaEventDestroy(e);
            cudaStreamDestroy(cs.s2);
        }
        if (stream) cudaStreamDestroy(stream);
    }
};

// build.cu
Graph* build_graph_device(const u64* d_pairs, u64 count, int device);
void generate_rmat_device(const RmatParams& p, u64 count, u64* d_pairs, cudaStream_t s);

// parse.cu
u64 parse_edge_list_device(const char* host_text, u64 len, int device, DevBuf& d_pairs, cudaStream_t s);

// count.cu
extern std::atomic<int> g_overlap;
void count_begin(Graph& g, int rank, int world, i64* d_partials, cudaStream_t s);
void count_mid(Graph& g, i64* d_partials, cudaStream_t s);
void count_finish(Graph& g, const i64* d_partials, u64 begin, u64 end, u128 C[17],
                  cudaStream_t s);
void micro_records(const Graph& g, u64 first, u64 count, u64* host_out /* count*10 */);
void edge_motif_records(const Graph& g, u64 first, u64 count, u64* host_out /* count*5 */);

// algebra.cpp
void global_from_unrestricted(const u128 C[17], u64 n, u64 m, u128 X[18]);

} // namespace gl
