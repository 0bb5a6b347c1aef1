// Microbenchmark: stream a 32-bit id array from global memory (coalesced, like
// a CSR col_idx) and set the ids' bits in a shared-memory bitmap (ATOMS.OR),
// one CTA of 1024 threads per SM. Separates the load stream, the smem atomics
// and their combination, with random ids and with sorted runs (CSR rows).
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a scripts/ubench_stream_smem.cu -o scripts/ubench_stream_smem
#include <cstdint>
#include <cstdio>
#include <vector>
#include <algorithm>
#include <random>
#include <cstdlib>
#include <cuda_runtime.h>

template <int ILP, int MODE>  // MODE 0 loads only, 1 loads + atomics, 2 atomics only (ids from hash)
__global__ void __launch_bounds__(1024, 1) kern(const uint32_t* __restrict__ ids, uint64_t n_per_cta, uint32_t nbits,
                                                uint32_t keep_lo, uint32_t keep_n, uint32_t* sink) {
    extern __shared__ uint32_t bm[];
    const uint32_t nw = nbits / 32;
    for (uint32_t i = threadIdx.x; i < nw; i += blockDim.x) bm[i] = 0;
    __syncthreads();
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(bm);
    const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint64_t beg = (uint64_t)blockIdx.x * n_per_cta, per_warp = n_per_cta / 32;
    const uint64_t ws = beg + wib * per_warp, we = ws + per_warp;
    uint32_t acc = 0;
    for (uint64_t x = ws + lane; x < we; x += 32 * ILP) {
        uint32_t u[ILP];
#pragma unroll
        for (int q = 0; q < ILP; ++q) {
            const uint64_t p = x + 32 * q;
            if (MODE == 2) {
                uint32_t h = (uint32_t)p * 0x9E3779B1u;
                h ^= h >> 15;
                u[q] = (h % keep_n);
            } else {
                u[q] = p < we ? __ldg(ids + p) - keep_lo : 0xFFFFFFFFu;
            }
        }
#pragma unroll
        for (int q = 0; q < ILP; ++q) {
            if (MODE == 0) acc += u[q];
            else if (u[q] < keep_n)
                asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(base + (u[q] >> 5) * 4), "r"(1u << (u[q] & 31)));
        }
    }
    __syncthreads();
    if (acc == 0x1234567 || bm[threadIdx.x] == 0x1234567) sink[0] = acc;
}

template <int ILP, int MODE>
void run(const char* name, const uint32_t* ids, uint64_t n, uint32_t nbits, uint32_t keep_lo, uint32_t keep_n,
         uint32_t* sink) {
    auto k = kern<ILP, MODE>;
    const size_t smem = nbits / 8;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = 148;
    const uint64_t per = n / grid / 32 * 32;
    printf("%s: launching\n", name);
    fflush(stdout);
    k<<<grid, 1024, smem>>>(ids, per, nbits, keep_lo, keep_n, sink);
    cudaError_t e0 = cudaDeviceSynchronize();
    if (e0 != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e0)); fflush(stdout); return; }
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) k<<<grid, 1024, smem>>>(ids, per, nbits, keep_lo, keep_n, sink);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    ms /= 5;
    const double tot = (double)per * grid;
    printf("%-28s ILP=%2d  %8.3f ms  %7.1f G ids/s  (%.2f ids/clk/SM)\n", name, ILP, ms, tot / ms / 1e6,
           tot / ms / 1e6 / 148 / 1.965);
}

int main(int argc, char** argv) {
    const uint64_t n = (argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 32ull) << 20;  // default 32M ids = 128 MB
    const uint32_t N = 2412345, half = 1206272;
    std::vector<uint32_t> h(n);
    std::mt19937_64 rng(1);
    for (auto& x : h) x = (uint32_t)(rng() % N);
    uint32_t *d_rand, *d_sorted, *sink;
    if (cudaMalloc(&d_rand, n * 4) || cudaMalloc(&d_sorted, n * 4) || cudaMalloc(&sink, 4)) {
        printf("cudaMalloc failed\n");
        return 1;
    }
    printf("allocated\n");
    fflush(stdout);
    cudaMemcpy(d_rand, h.data(), n * 4, cudaMemcpyHostToDevice);
    // "CSR rows": runs of 2048 sorted ids (a row of degree 2048 over N ids)
    for (uint64_t i = 0; i < n; i += 2048) std::sort(h.begin() + i, h.begin() + std::min(n, i + 2048));
    cudaMemcpy(d_sorted, h.data(), n * 4, cudaMemcpyHostToDevice);
    // every id in the CTA's slice (each read ends in an atomic): ids mod half, sorted runs
    uint32_t* d_inrange;
    if (cudaMalloc(&d_inrange, n * 4)) return 1;
    for (auto& x : h) x %= half;
    for (uint64_t i = 0; i < n; i += 2048) std::sort(h.begin() + i, h.begin() + std::min(n, i + 2048));
    cudaMemcpy(d_inrange, h.data(), n * 4, cudaMemcpyHostToDevice);
    const uint32_t nbits = half;
    run<8, 0>("loads only (random)", d_rand, n, nbits, 0, half, sink);
    run<8, 1>("loads+atoms random R=2", d_rand, n, nbits, 0, half, sink);
    run<8, 1>("loads+atoms rows R=2", d_sorted, n, nbits, 0, half, sink);
    run<8, 2>("atoms only (hash)", d_rand, n, nbits, 0, half, sink);
    run<16, 0>("loads only (random)", d_rand, n, nbits, 0, half, sink);
    run<16, 1>("loads+atoms random R=2", d_rand, n, nbits, 0, half, sink);
    run<16, 1>("loads+atoms rows R=2", d_sorted, n, nbits, 0, half, sink);
    run<4, 1>("loads+atoms random R=2", d_rand, n, nbits, 0, half, sink);
    run<16, 1>("loads+atoms rows all-kept", d_inrange, n, nbits, 0, half, sink);
    run<8, 1>("loads+atoms rows all-kept", d_inrange, n, nbits, 0, half, sink);
    return 0;
}
