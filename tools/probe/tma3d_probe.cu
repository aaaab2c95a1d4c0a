// Development probe: 2-D TMA box load (32 x 8 f32).
#include <cuda.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
__global__ void k(const __grid_constant__ CUtensorMap tm, float* out, int mode, int cx) {
    __shared__ alignas(1024) float buf[4][6][36];
    __shared__ alignas(8) unsigned long long bar;
    const unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(3456) : "memory");
        if (mode == 0)
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %5}], [%4];" ::
                             "r"((unsigned)__cvta_generic_to_shared(&buf[0][0][0])), "l"(&tm), "r"(cx), "r"(0), "r"(b), "r"(0) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.3d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %5}], [%4];" ::
                             "r"((unsigned)__cvta_generic_to_shared(&buf[0][0][0])), "l"(&tm), "r"(cx), "r"(0), "r"(b), "r"(0) : "memory");
    }
    __syncthreads();
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}" ::"r"(b) : "memory");
    for (int i = threadIdx.x; i < 864; i += blockDim.x) out[i] = (&buf[0][0][0])[i];
}
int main(int argc, char** argv) {
    const int n = 64;
    std::vector<float> h(n * n * n);
    for (int i = 0; i < n * n * n; ++i) h[i] = i;
    float *d, *o;
    cudaMalloc(&d, h.size() * 4); cudaMalloc(&o, 4096);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    CUtensorMap tm;
    cuuint64_t dims[3] = {n, n, n}, str[2] = {n * 4ull, n * n * 4ull};
    cuuint32_t box[3] = {36, 6, 4}, es[3] = {1, 1, 1};
    CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int cx = argc > 2 ? atoi(argv[2]) : 0;
    k<<<1, 256>>>(tm, o, argc > 1 && argv[1][0] == 'x', cx);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> ho(864);
    cudaMemcpy(ho.data(), o, 864 * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int z = 0; z < 4; ++z) for (int y = 0; y < 6; ++y) for (int x = 0; x < 36; ++x) { const int gx = x + cx; const float w = (gx < 0 || gx >= n) ? 0.f : h[gx + n * (y + n * z)]; bad += ho[x + 36 * (y + 6 * z)] != w; }
    printf("3d tma (encode %d, mode %d): %s, mismatches %d\n", (int)r, argc > 1, cudaGetErrorString(e), bad);
}
