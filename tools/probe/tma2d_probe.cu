// Development probe: 2-D TMA box load (32 x 8 f32).
#include <cuda.h>
#include <cstdio>
#include <vector>
__global__ void k(const __grid_constant__ CUtensorMap tm, float* out, int mode) {
    __shared__ alignas(1024) float buf[8][32];
    __shared__ alignas(8) unsigned long long bar;
    const unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(1024) : "memory");
        if (mode == 0)
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
                             "r"((unsigned)__cvta_generic_to_shared(&buf[0][0])), "l"(&tm), "r"(0), "r"(0), "r"(b) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
                             "r"((unsigned)__cvta_generic_to_shared(&buf[0][0])), "l"(&tm), "r"(0), "r"(0), "r"(b) : "memory");
    }
    __syncthreads();
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}" ::"r"(b) : "memory");
    out[threadIdx.x] = (&buf[0][0])[threadIdx.x];
}
int main(int argc, char** argv) {
    const int n = 64;
    std::vector<float> h(n * n);
    for (int i = 0; i < n * n; ++i) h[i] = i;
    float *d, *o;
    cudaMalloc(&d, h.size() * 4); cudaMalloc(&o, 1024);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    CUtensorMap tm;
    cuuint64_t dims[2] = {n, n}, str[1] = {n * 4ull};
    cuuint32_t box[2] = {32, 8}, es[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    k<<<1, 256>>>(tm, o, argc > 1);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> ho(256);
    cudaMemcpy(ho.data(), o, 1024, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int y = 0; y < 8; ++y) for (int x = 0; x < 32; ++x) bad += ho[x + 32 * y] != h[x + n * y];
    printf("2d tma (encode %d, mode %d): %s, mismatches %d\n", (int)r, argc > 1, cudaGetErrorString(e), bad);
}
