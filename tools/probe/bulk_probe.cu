// Development probe: 1-D bulk async copy global -> shared with an mbarrier.
#include <cstdio>
__global__ void k(const float* src, float* out, int fence) {
    __shared__ alignas(128) float buf[256];
    __shared__ alignas(8) unsigned long long bar;
    const unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
        if (fence) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(1024) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                         "r"((unsigned)__cvta_generic_to_shared(buf)), "l"(src), "r"(1024), "r"(b) : "memory");
    }
    __syncthreads();
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}" ::"r"(b) : "memory");
    out[threadIdx.x] = buf[threadIdx.x];
}
int main(int argc, char** argv) {
    float *s, *o;
    cudaMalloc(&s, 1024); cudaMalloc(&o, 1024);
    float h[256];
    for (int i = 0; i < 256; ++i) h[i] = i;
    cudaMemcpy(s, h, 1024, cudaMemcpyHostToDevice);
    k<<<1, 256>>>(s, o, argc > 1);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, o, 1024, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < 256; ++i) bad += h[i] != i;
    printf("bulk copy: %s, mismatches %d\n", cudaGetErrorString(e), bad);
}
