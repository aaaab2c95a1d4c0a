// Development probe: dependent random-load latency vs working-set size (TLB reach).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void chase(const unsigned long long* __restrict__ a, unsigned long long n, int steps, unsigned long long* out,
                      long long* cyc) {
    unsigned long long i = (blockIdx.x * 7919ull + threadIdx.x * 104729ull) % n;
    long long t0 = clock64();
    for (int s = 0; s < steps; ++s) i = a[i];
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = i;
    if (threadIdx.x == 0) atomicAdd((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}
__global__ void fill(unsigned long long* a, unsigned long long n) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n; i += gridDim.x * (unsigned long long)blockDim.x) {
        unsigned long long x = i * 0x9E3779B97F4A7C15ull;
        x ^= x >> 29; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 32;
        a[i] = x % n;
    }
}
int main() {
    unsigned long long maxb = 16ull << 30;
    unsigned long long* a; cudaMalloc(&a, maxb);
    unsigned long long* out; cudaMalloc(&out, 1 << 24);
    long long* cyc; cudaMalloc(&cyc, 8);
    for (unsigned long long bytes : {64ull << 20, 256ull << 20, 1ull << 30, 4ull << 30, 8ull << 30, 16ull << 30}) {
        unsigned long long n = bytes / 8;
        fill<<<1184, 256>>>(a, n);
        for (int blocks : {1, 148, 148 * 8}) {
            cudaMemset(cyc, 0, 8);
            chase<<<blocks, 32>>>(a, n, 200, out, cyc);
            long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
            printf("ws %6llu MB  warps %5d  cycles/load %.0f\n", bytes >> 20, blocks, (double)h / blocks / 200);
        }
    }
    return 0;
}
