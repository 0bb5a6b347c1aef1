// Microbenchmark: random 32-bit atomicOr / load throughput on B200 over a
// bitmap the size of the SINGLE engine's working set (the ceiling for the
// per-edge visited test). nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <string>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16;
    return x;
}

template <int ILP, int MODE>  // MODE 0 atomicOr w/ return, 1 red (no return), 2 load, 3 load+cond atomic, 4 st.b32, 5 st 32 B
__global__ void kern(uint32_t* bits, uint32_t nwords, uint32_t iters, uint32_t* sink) {
    uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    for (uint32_t it = 0; it < iters; ++it) {
        uint32_t idx[ILP];
#pragma unroll
        for (int r = 0; r < ILP; ++r) idx[r] = hash32(tid * 7919u + it * 104729u + r * 31u) % nwords;
        uint32_t v[ILP];
#pragma unroll
        for (int r = 0; r < ILP; ++r) {
            const uint32_t bit = 1u << (idx[r] & 31);
            if (MODE == 0) v[r] = atomicOr(bits + idx[r], bit);
            else if (MODE == 1) { atomicOr(bits + idx[r], bit); v[r] = 0; }
            else if (MODE == 4) { bits[idx[r]] = 0; v[r] = 0; }
            else if (MODE == 5) {
                asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(bits + (idx[r] & ~7u)),
                             "r"(0u) : "memory");
                v[r] = 0;
            }
            else v[r] = __ldcg(bits + idx[r]);
        }
        if (MODE == 3) {
#pragma unroll
            for (int r = 0; r < ILP; ++r)
                if (!(v[r] & 1u)) v[r] = atomicOr(bits + idx[r], 1u);
        }
#pragma unroll
        for (int r = 0; r < ILP; ++r) acc += v[r];
    }
    if (acc == 0x12345678) sink[0] = acc;
}

template <int ILP, int MODE>
void run(const char* name, uint32_t* bits, uint32_t nwords, int blocks, int threads, uint32_t* sink) {
    const uint32_t iters = 64;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    kern<ILP, MODE><<<blocks, threads>>>(bits, nwords, 4, sink);
    cudaEventRecord(a);
    kern<ILP, MODE><<<blocks, threads>>>(bits, nwords, iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0; cudaEventElapsedTime(&ms, a, b);
    double ops = (double)blocks * threads * iters * ILP;
    printf("%-22s ILP=%d blocks=%5d threads=%4d  %7.3f ms  %7.1f Gop/s\n", name, ILP, blocks, threads, ms,
           ops / ms / 1e6);
}

int main(int argc, char** argv) {
    if (argc > 1 && std::string(argv[1]) == "--red-sweep") {  // the red.or ceiling over configurations
        for (size_t mb : {8ul, 16ul, 32ul, 64ul, 90ul}) {
            const uint32_t nwords = (uint32_t)(mb * 1024 * 1024 / 4);
            uint32_t *bits, *sink;
            cudaMalloc(&bits, (size_t)nwords * 4);
            cudaMalloc(&sink, 4);
            cudaMemset(bits, 0, (size_t)nwords * 4);
            printf("== %zu MB array\n", mb);
            for (int blocks : {296, 592, 1184})
                for (int threads : {256, 512, 1024}) {
                    run<4, 1>("red.or", bits, nwords, blocks, threads, sink);
                    run<8, 1>("red.or", bits, nwords, blocks, threads, sink);
                    run<16, 1>("red.or", bits, nwords, blocks, threads, sink);
                }
            cudaFree(bits);
            cudaFree(sink);
        }
        return 0;
    }
    for (size_t mb : {1ul, 16ul, 90ul, 512ul}) {
        const uint32_t nwords = (uint32_t)(mb * 1024 * 1024 / 4);
        uint32_t *bits, *sink;
        cudaMalloc(&bits, (size_t)nwords * 4);
        cudaMalloc(&sink, 4);
        cudaMemset(bits, 0, (size_t)nwords * 4);
        printf("== %zu MB array\n", mb);
        run<4, 0>("atomicOr+ret", bits, nwords, 296, 512, sink);
        run<8, 0>("atomicOr+ret", bits, nwords, 296, 512, sink);
        run<4, 0>("atomicOr+ret", bits, nwords, 148 * 4, 512, sink);
        run<4, 1>("red.or", bits, nwords, 296, 512, sink);
        run<8, 1>("red.or", bits, nwords, 296, 512, sink);
        run<4, 2>("ld.cg", bits, nwords, 296, 512, sink);
        run<8, 2>("ld.cg", bits, nwords, 296, 512, sink);
        run<4, 2>("ld.cg", bits, nwords, 148 * 4, 512, sink);
        run<4, 4>("st.b32 zero", bits, nwords, 296, 512, sink);
        run<4, 4>("st.b32 zero", bits, nwords, 148 * 4, 512, sink);
        run<4, 5>("st.v8 sector zero", bits, nwords, 296, 512, sink);
        run<4, 5>("st.v8 sector zero", bits, nwords, 148 * 4, 512, sink);
        cudaMemset(bits, 0, (size_t)nwords * 4);
        run<4, 3>("ld+cond atomic", bits, nwords, 296, 512, sink);
        cudaFree(bits);
        cudaFree(sink);
    }
    return 0;
}
