// Microbenchmark: random 32-bit atomicOr throughput on a bitmap held in shared
// memory, local (one CTA) or distributed over a thread-block cluster (DSMEM),
// to size a per-seed visited bitmap kept on chip instead of in L2.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a scripts/ubench_smem.cu -o scripts/ubench_smem
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16;
    return x;
}

// MODE 0: atomicOr, result unused; 1: atomicOr with result consumed;
// 2: plain load (bank-conflict floor)
template <int ILP, int MODE>
__global__ void kern(uint32_t words_per_cta, uint32_t iters, uint32_t* sink) {
    extern __shared__ uint32_t bm[];
    cg::cluster_group cl = cg::this_cluster();
    const uint32_t csize = cl.num_blocks();
    for (uint32_t i = threadIdx.x; i < words_per_cta; i += blockDim.x) bm[i] = 0;
    cl.sync();
    const uint32_t total = words_per_cta * csize;
    uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t smem_base = (uint32_t)__cvta_generic_to_shared(bm);
    uint32_t acc = 0;
    for (uint32_t it = 0; it < iters; ++it) {
        uint32_t v[ILP];
#pragma unroll
        for (int r = 0; r < ILP; ++r) {
            const uint32_t h = hash32(tid * 7919u + it * 104729u + r * 31u);
            const uint32_t w = h % total;
            const uint32_t owner = w / words_per_cta, off = w - owner * words_per_cta;
            uint32_t a = smem_base + off * 4;
            const uint32_t bit = 1u << (h >> 27);
            if (csize == 1) {
                if (MODE == 0) { asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"(bit) : "memory"); v[r] = 0; }
                else if (MODE == 1) asm volatile("atom.shared.or.b32 %0, [%1], %2;" : "=r"(v[r]) : "r"(a), "r"(bit) : "memory");
                else asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v[r]) : "r"(a) : "memory");
            } else {
                uint32_t ra;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(owner));
                if (MODE == 0) { asm volatile("red.shared::cluster.or.b32 [%0], %1;" ::"r"(ra), "r"(bit) : "memory"); v[r] = 0; }
                else if (MODE == 1) asm volatile("atom.shared::cluster.or.b32 %0, [%1], %2;" : "=r"(v[r]) : "r"(ra), "r"(bit) : "memory");
                else asm volatile("ld.volatile.shared::cluster.u32 %0, [%1];" : "=r"(v[r]) : "r"(ra) : "memory");
            }
        }
#pragma unroll
        for (int r = 0; r < ILP; ++r) acc += v[r];
    }
    cl.sync();
    if (acc == 0x12345678) sink[0] = acc;
}

template <int ILP, int MODE>
void run(const char* name, int csize, uint32_t bytes_per_cta, int threads, uint32_t* sink) {
    auto k = kern<ILP, MODE>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes_per_cta);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = bytes_per_cta;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = csize; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int nclusters = 0;
    cfg.gridDim = dim3(csize * 256);
    cudaOccupancyMaxActiveClusters(&nclusters, k, &cfg);
    if (nclusters <= 0) { printf("%s: no cluster fits (%s)\n", name, cudaGetErrorString(cudaGetLastError())); return; }
    cfg.gridDim = dim3(nclusters * csize);
    const uint32_t words = bytes_per_cta / 4, iters = 256;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaLaunchKernelEx(&cfg, k, words, 8u, sink);
    cudaEventRecord(a);
    cudaLaunchKernelEx(&cfg, k, words, iters, sink);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
    float ms = 0; cudaEventElapsedTime(&ms, a, b);
    double ops = (double)cfg.gridDim.x * threads * iters * ILP;
    printf("%-16s C=%2d clusters=%3d smem=%6u threads=%4d ILP=%d  %8.3f ms  %7.1f Gop/s  (%.2f op/clk/SM @1.965GHz)\n",
           name, csize, nclusters, bytes_per_cta, threads, ILP, ms, ops / ms / 1e6,
           ops / ms / 1e6 / sms / 1.965);
}

int main() {
    uint32_t* sink; cudaMalloc(&sink, 4);
    const uint32_t B = 150 * 1024;
    for (int t : {512, 1024}) {
        run<8, 0>("smem_or", 1, B, t, sink);
        run<8, 1>("smem_or_ret", 1, B, t, sink);
        run<8, 2>("smem_ld", 1, B, t, sink);
    }
    for (int c : {2, 4, 8}) {
        for (int t : {512, 1024}) {
            run<8, 0>("dsmem_or", c, B, t, sink);
            run<8, 1>("dsmem_or_ret", c, B, t, sink);
        }
    }
    run<16, 0>("dsmem_or", 2, B, 1024, sink);
    return 0;
}
