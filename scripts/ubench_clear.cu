// Microbenchmark: popcount + zero of S bitmap rows (the SINGLE engine's dense clearing pass).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <bool CS, int U>
__global__ void pass(uint32_t* V, uint32_t rs, uint32_t S, unsigned long long* pop) {
    constexpr uint32_t CH = U * 4 * 512;
    const uint32_t chunks = (rs + CH - 1) / CH;
    for (uint32_t t = blockIdx.x; t < S * chunks; t += gridDim.x) {
        const uint32_t slot = t / chunks;
        const uint32_t base = (t % chunks) * CH + threadIdx.x * 4;
        uint4* row = reinterpret_cast<uint4*>(V + (size_t)slot * rs);
        uint4 v[U];
#pragma unroll
        for (int i = 0; i < U; ++i) {
            const uint32_t w = base + i * 4 * 512;
            v[i] = w < rs ? (CS ? __ldcs(row + w / 4) : row[w / 4]) : make_uint4(0, 0, 0, 0);
        }
        uint32_t pc = 0;
#pragma unroll
        for (int i = 0; i < U; ++i) {
            const uint32_t w = base + i * 4 * 512;
            pc += __popc(v[i].x) + __popc(v[i].y) + __popc(v[i].z) + __popc(v[i].w);
            if (w < rs) { if (CS) __stcs(row + w / 4, make_uint4(0, 0, 0, 0)); else row[w / 4] = make_uint4(0, 0, 0, 0); }
        }
        for (int d = 16; d > 0; d >>= 1) pc += __shfl_xor_sync(0xffffffff, pc, d);
        if ((threadIdx.x & 31) == 0 && pc) atomicAdd(&pop[slot], (unsigned long long)pc);
    }
}
__global__ void fill(uint32_t* V, size_t n) { for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) atomicOr(V + i, 0x10101u); }
template <bool CS, int U> void run(const char* nm, uint32_t* V, uint32_t rs, uint32_t S, unsigned long long* pop, int grid) {
    fill<<<1184, 512>>>(V, (size_t)rs * S); cudaDeviceSynchronize();
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); pass<CS, U><<<grid, 512>>>(V, rs, S, pop); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%-10s U=%d grid=%d: %.1f us  %.0f GB/s (r+w)\n", nm, U, grid, ms * 1e3, 2.0 * rs * S * 4 / ms / 1e6);
}
int main() {
    const uint32_t rs = 75392, S = 300;
    uint32_t* V; unsigned long long* pop;
    cudaMalloc(&V, (size_t)rs * S * 4); cudaMalloc(&pop, S * 8);
    run<true, 4>("cs", V, rs, S, pop, 296);
    run<false, 4>("plain", V, rs, S, pop, 296);
    run<false, 8>("plain", V, rs, S, pop, 296);
    run<false, 2>("plain", V, rs, S, pop, 592);
    run<true, 4>("cs", V, rs, S, pop, 296);
    run<false, 4>("plain", V, rs, S, pop, 1184);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
