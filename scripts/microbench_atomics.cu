// Throughput probes for the cycle pass's per-wedge operations on one B200
// (not product code): shared-memory RED on spread / clustered addresses,
// global RED.64 on spread addresses, coalesced 32- vs 128-bit adjacency loads.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/mb scripts/microbench_atomics.cu && /tmp/mb
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// MODE 0: red.shared spread (random word in 32K words)
// MODE 1: red.shared clustered: lane -> word (base + lane/16) (16 lanes per word, packed 2-bit tier)
// MODE 2: red.shared clustered: lane -> word (base + lane/2)
// MODE 3: ld.shared spread + add (no atomic) as an LDS floor
template <int MODE>
__global__ void __launch_bounds__(1024, 1) k_smem(int iters, uint32_t* out) {
    extern __shared__ uint32_t W[];
    for (int i = threadIdx.x; i < 32768; i += blockDim.x) W[i] = 0;
    __syncthreads();
    uint32_t s = hsh(threadIdx.x * 7919u + blockIdx.x), acc = 0;
    const uint32_t lane = threadIdx.x & 31;
    for (int it = 0; it < iters; ++it) {
        s = s * 1664525u + 1013904223u;
        uint32_t w;
        if (MODE == 0 || MODE == 3) w = (s >> 8) & 32767u;
        else if (MODE == 1) w = ((__shfl_sync(0xffffffffu, s, 0) >> 8) & 32767u & ~1u) + lane / 16;
        else w = ((__shfl_sync(0xffffffffu, s, 0) >> 8) & 32767u & ~15u) + lane / 2;
        if (MODE == 3) acc += W[w];
        else {
            uint32_t addr = (uint32_t)__cvta_generic_to_shared(W + w);
            asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(1u << (lane & 15) * 2) : "memory");
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = W[5] + acc;
}

// global RED.64 spread over n8 u64 slots (predicated like the kernel)
__global__ void __launch_bounds__(1024, 1) k_redg(int iters, unsigned long long* slots, uint64_t n8) {
    uint32_t s = hsh(threadIdx.x * 7919u + blockIdx.x);
    for (int it = 0; it < iters; ++it) {
        s = s * 1664525u + 1013904223u;
        uint64_t i = ((uint64_t)hsh(s) * n8) >> 32;
        asm volatile("red.global.add.u64 [%0], %1;" ::"l"(slots + i), "l"(1ull) : "memory");
    }
}

// coalesced streaming of a u32 array: VEC=1 (LDG.32) or 4 (LDG.128), UNR loads in flight
template <int VEC, int UNR>
__global__ void __launch_bounds__(1024, 1) k_stream(const uint32_t* __restrict__ a, uint64_t n, uint32_t* out) {
    uint32_t acc = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * VEC * UNR;
    for (uint64_t base = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * VEC; base < n; base += stride) {
        if (VEC == 4) {
            uint4 v[UNR];
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                uint64_t p = base + (uint64_t)u * gridDim.x * blockDim.x * 4;
                v[u] = p + 3 < n ? __ldg(reinterpret_cast<const uint4*>(a + p)) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < UNR; ++u) acc += v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
        } else {
            uint32_t v[UNR];
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                uint64_t p = base + (uint64_t)u * gridDim.x * blockDim.x;
                v[u] = p < n ? __ldg(a + p) : 0;
            }
#pragma unroll
            for (int u = 0; u < UNR; ++u) acc += v[u];
        }
    }
    if (acc == 0x12345678u) out[0] = acc;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    uint32_t* out;
    cudaMalloc(&out, 4096 * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    const int iters = 4096;
    auto smem_run = [&](auto kern, const char* name) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
        kern<<<sms, 1024, 131072>>>(iters, out);
        cudaEventRecord(e0);
        kern<<<sms, 1024, 131072>>>(iters, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double lanes = (double)sms * 1024 * iters;
        double cyc = ms * 1e-3 * clk * 1e3;
        printf("%-40s %8.3f ms  %6.2f lanes/clk/SM\n", name, ms, lanes / sms / cyc);
    };
    smem_run(k_smem<0>, "red.shared spread");
    smem_run(k_smem<1>, "red.shared 16 lanes/word");
    smem_run(k_smem<2>, "red.shared 2 lanes/word");
    smem_run(k_smem<3>, "ld.shared spread");
    const uint64_t n8 = 1ull << 25; // 256 MB of u64 slots
    unsigned long long* slots;
    cudaMalloc(&slots, n8 * 8);
    cudaMemset(slots, 0, n8 * 8);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        k_redg<<<sms, 1024>>>(1024, slots, n8);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
    }
    {
        double lanes = (double)sms * 1024 * 1024, cyc = ms * 1e-3 * clk * 1e3;
        printf("%-40s %8.3f ms  %6.2f lanes/clk/SM  %.1f G/s\n", "red.global.add.u64 spread 256MB", ms,
               lanes / sms / cyc, lanes / ms / 1e6);
    }
    const uint64_t n = 126ull << 20 >> 2; // 126 MB of u32 (RMAT-20 adjacency)
    uint32_t* a;
    cudaMalloc(&a, n * 4 + 64);
    cudaMemset(a, 1, n * 4);
    auto st = [&](auto kern, const char* name) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            kern<<<sms, 1024>>>(a, n, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
        }
        printf("%-40s %8.3f ms  %7.1f GB/s\n", name, ms, n * 4 / ms / 1e6);
    };
    st(k_stream<1, 4>, "stream LDG.32 x4 (126 MB, L2-warm)");
    st(k_stream<1, 8>, "stream LDG.32 x8");
    st(k_stream<4, 1>, "stream LDG.128 x1");
    st(k_stream<4, 2>, "stream LDG.128 x2");
    st(k_stream<4, 4>, "stream LDG.128 x4");
    printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
