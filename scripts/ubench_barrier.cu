// Microbenchmark: cost of the engines' software grid barrier at different grid shapes.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void grid_barrier(unsigned int* bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int gen = *reinterpret_cast<volatile unsigned int*>(bar + 1);
        __threadfence();
        if (atomicAdd(bar, 1u) == gridDim.x - 1) {
            *reinterpret_cast<volatile unsigned int*>(bar) = 0;
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*reinterpret_cast<volatile unsigned int*>(bar + 1) == gen) __nanosleep(20);
        }
        __threadfence();
    }
    __syncthreads();
}
__global__ void kern(unsigned int* bar, int n) { for (int i = 0; i < n; ++i) grid_barrier(bar); }
int main() {
    unsigned int* bar; cudaMalloc(&bar, 8); cudaMemset(bar, 0, 8);
    int shapes[][2] = {{148, 1024}, {296, 512}, {592, 256}, {148, 512}};
    for (auto& s : shapes) {
        kern<<<s[0], s[1]>>>(bar, 10); cudaDeviceSynchronize();
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a); kern<<<s[0], s[1]>>>(bar, 1000); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("grid %d x %d: %.2f us per barrier (%s)\n", s[0], s[1], ms, cudaGetErrorString(cudaGetLastError()));
    }
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); for (int i = 0; i < 100; ++i) kern<<<296, 512>>>(bar, 0); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); printf("empty launch: %.2f us\n", ms * 10);
}
