// DSMEM throughput probes for cluster-wide cycle windows (not product code):
// red.shared::cluster.add.u32 to a peer CTA's shared memory (spread addresses)
// vs the local red.shared.add, and ld.shared::cluster (remote load) throughput.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/_mbd scripts/microbench_dsmem.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// MODE 0: local red.shared; 1: remote red to rank (r+1)%CL; 2: spread over all ranks (1/CL local);
// 3: remote ld.shared::cluster (sum) from rank (r+1)%CL; 4: local ld.shared
template <int MODE, int CL>
__global__ void __launch_bounds__(1024, 1) k_ds(int iters, uint32_t* out) {
    extern __shared__ uint32_t W[];
    cg::cluster_group cl = cg::this_cluster();
    for (int i = threadIdx.x; i < 32768; i += blockDim.x) W[i] = 0;
    cl.sync();
    const uint32_t me = cl.block_rank();
    uint32_t s = hsh(threadIdx.x * 7919u + blockIdx.x), acc = 0;
    uint32_t base_local = (uint32_t)__cvta_generic_to_shared(W);
    for (int it = 0; it < iters; ++it) {
        s = s * 1664525u + 1013904223u;
        const uint32_t w = (s >> 8) & 32767u;
        uint32_t tgt = MODE == 1 || MODE == 3 ? (me + 1) % CL : MODE == 2 ? (s >> 28) % CL : me;
        uint32_t addr = base_local + 4 * w, raddr;
        if (MODE == 0) {
            asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(addr) : "memory");
        } else if (MODE == 4) {
            uint32_t v;
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
            acc += v;
        } else {
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(addr), "r"(tgt));
            if (MODE == 3) {
                uint32_t v;
                asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(raddr));
                acc += v;
            } else {
                asm volatile("red.shared::cluster.add.u32 [%0], 1;" ::"r"(raddr) : "memory");
            }
        }
    }
    cl.sync();
    if (threadIdx.x == 0) out[blockIdx.x] = W[5] + acc;
}

template <int MODE, int CL>
void run(const char* name, int sms, int clk, uint32_t* out) {
    auto kern = k_ds<MODE, CL>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
    cudaLaunchConfig_t cfg = {};
    int grid = (sms / CL) * CL;
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(1024);
    cfg.dynamicSmemBytes = 131072;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const int iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms = 0;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        cudaError_t err = cudaLaunchKernelEx(&cfg, kern, iters, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        if (err != cudaSuccess) { printf("%s: launch %s\n", name, cudaGetErrorString(err)); return; }
        cudaEventElapsedTime(&ms, e0, e1);
    }
    double lanes = (double)grid * 1024 * iters;
    double cyc = ms * 1e-3 * clk * 1e3;
    printf("%-44s cl=%d %8.3f ms  %6.2f lanes/clk/SM\n", name, CL, ms, lanes / grid / cyc);
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    uint32_t* out;
    cudaMalloc(&out, 4096 * 4);
    run<0, 2>("local red.shared", sms, clk, out);
    run<1, 2>("remote red.shared::cluster (peer)", sms, clk, out);
    run<2, 2>("red.shared::cluster spread over cluster", sms, clk, out);
    run<2, 4>("red.shared::cluster spread over cluster", sms, clk, out);
    run<2, 8>("red.shared::cluster spread over cluster", sms, clk, out);
    run<4, 2>("local ld.shared", sms, clk, out);
    run<3, 2>("remote ld.shared::cluster (peer)", sms, clk, out);
    run<3, 4>("remote ld.shared::cluster (peer)", sms, clk, out);
    printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
