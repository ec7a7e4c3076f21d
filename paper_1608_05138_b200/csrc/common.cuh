// common.cuh -- shared types, error plumbing and device helpers.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace gl {

using u32 = std::uint32_t;
using u64 = std::uint64_t;
using i64 = std::int64_t;
using u128 = unsigned __int128;

// Exceptions mirror the reference's classes; the C-ABI maps them to codes.
struct invalid_argument : std::runtime_error { using std::runtime_error::runtime_error; };
struct parse_error : std::runtime_error {
    parse_error(u64 line, const std::string& w)
        : std::runtime_error("line " + std::to_string(line) + ": " + w), line(line) {}
    u64 line;
};
struct io_error : std::runtime_error { using std::runtime_error::runtime_error; };
struct cuda_error : std::runtime_error { using std::runtime_error::runtime_error; };
struct oom_error : std::runtime_error { using std::runtime_error::runtime_error; };
struct consistency_error : std::runtime_error { using std::runtime_error::runtime_error; };
struct overflow_error : std::runtime_error { using std::runtime_error::runtime_error; };
struct state_error : std::runtime_error { using std::runtime_error::runtime_error; };

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e == cudaSuccess) return;
    std::string msg = std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                      std::to_string(line) + ")";
    if (e == cudaErrorMemoryAllocation) throw oom_error(msg);
    throw cuda_error(msg);
}
#define GL_CUDA(x) ::gl::cuda_check((x), #x, __FILE__, __LINE__)
#define GL_LAUNCH_CHECK() ::gl::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

// ---------------------------------------------------------------------------
// Counter-based hashing for the synthetic generators: identical on host and
// device so a graph generated in HBM equals the one generated on the host.
__host__ __device__ inline u64 mix64(u64 z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__host__ __device__ inline u64 hash2(u64 seed, u64 ctr) { return mix64(seed ^ mix64(ctr)); }

struct RmatParams {
    u32 scale;
    u32 ta, tb, tc; // cumulative 32-bit thresholds for quadrants a, a+b, a+b+c
    u64 seed;
};

// Edge i of an RMAT graph: one 32-bit draw per level, quadrant by threshold.
__host__ __device__ inline void rmat_edge(const RmatParams& p, u64 i, u64& src, u64& dst) {
    u64 r = 0, c = 0;
    for (u32 l = 0; l < p.scale; ++l) {
        u32 x = (u32)(hash2(p.seed, i * 64 + l) >> 32);
        r <<= 1;
        c <<= 1;
        if (x < p.ta) {
        } else if (x < p.tb) {
            c |= 1;
        } else if (x < p.tc) {
            r |= 1;
        } else {
            r |= 1;
            c |= 1;
        }
    }
    src = r;
    dst = c;
}

RmatParams make_rmat_params(u32 scale, double a, double b, double c, u64 seed);

// ---------------------------------------------------------------------------
// Device helpers
#ifdef __CUDACC__

// first index in [lo, hi) with a[idx] >= x
template <typename T, typename I>
__device__ __forceinline__ I lower_bound_dev(const T* __restrict__ a, I lo, I hi, T x) {
    while (lo < hi) {
        I mid = lo + ((hi - lo) >> 1);
        if (a[mid] < x)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}
// last index in [lo, hi) with a[idx] <= x, for monotone prefix arrays
template <typename T, typename I>
__device__ __forceinline__ I upper_bound_dev(const T* __restrict__ a, I lo, I hi, T x) {
    while (lo < hi) {
        I mid = lo + ((hi - lo) >> 1);
        if (a[mid] <= x)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

__device__ __forceinline__ u32 lane_id() { return threadIdx.x & 31u; }

// Segmented inclusive sum over consecutive lanes sharing `key` (keys of a
// warp's items are non-decreasing).  Returns true on the segment's last lane
// (the "tail"), with *sum = the segment total.  All 32 lanes must call.
__device__ __forceinline__ bool seg_tail_sum(u64 key, u64 val, u64* sum) {
    const u32 lane = lane_id();
    u64 s = val;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        u64 ov = __shfl_up_sync(0xffffffffu, s, d);
        u64 ok = __shfl_up_sync(0xffffffffu, key, d);
        if (lane >= (u32)d && ok == key) s += ov;
    }
    u64 nk = __shfl_down_sync(0xffffffffu, key, 1);
    *sum = s;
    return lane == 31 || nk != key;
}
#endif // __CUDACC__

} // namespace gl
