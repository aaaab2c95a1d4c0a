// Development probe: one 3-D TMA box load (36 x 6 x 4 f32) into shared memory, with the
// tensor map as a __grid_constant__ parameter or in global memory.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ void bar_init(unsigned long long* b) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(b)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
template <int kMode>
__global__ void k(const __grid_constant__ CUtensorMap tm, const CUtensorMap* gtm, float* out, int x, int y, int z, unsigned txb) {
    __shared__ alignas(128) float buf[4][6][36];
    __shared__ alignas(8) unsigned long long bar;
    if (threadIdx.x == 0) {
        bar_init(&bar);
        const CUtensorMap* m = kMode == 1 ? gtm : &tm;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar)), "r"(txb) : "memory");
        if (kMode == 2)
            asm volatile("cp.async.bulk.tensor.3d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
                             "r"((unsigned)__cvta_generic_to_shared(&buf[0][0][0])), "l"((unsigned long long)m), "r"(x), "r"(y), "r"(z),
                             "r"((unsigned)__cvta_generic_to_shared(&bar)) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
                             "r"((unsigned)__cvta_generic_to_shared(&buf[0][0][0])), "l"((unsigned long long)m), "r"(x), "r"(y), "r"(z),
                             "r"((unsigned)__cvta_generic_to_shared(&bar)) : "memory");
    }
    __syncthreads();
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}" ::"r"((unsigned)__cvta_generic_to_shared(&bar)) : "memory");
    for (int i = threadIdx.x; i < 864; i += blockDim.x) out[i] = (&buf[0][0][0])[i];
}
int main(int argc, char** argv) {
    const int want_mode = argc > 1 ? atoi(argv[1]) : 0;
    const int promo = argc > 2 ? atoi(argv[2]) : 1;
    const unsigned bw = argc > 3 ? atoi(argv[3]) : 36;
    const int n = 64;
    std::vector<float> h(n * n * n);
    for (int i = 0; i < n * n * n; ++i) h[i] = i;
    float *d, *o; CUtensorMap* g;
    cudaMalloc(&d, h.size() * 4); cudaMalloc(&o, 864 * 4); cudaMalloc(&g, sizeof(CUtensorMap));
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    void* fn = nullptr; cudaDriverEntryPointQueryResult q;
    if (argc > 4) cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q);
    else cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    CUtensorMap tm;
    cuuint64_t dims[3] = {n, n, n}, str[2] = {n * 4ull, n * n * 4ull};
    cuuint32_t box[3] = {bw, 6, 4}, es[3] = {1, 1, 1};
    CUresult r = (argc > 5) ? cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, (promo ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_NONE), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)
        : enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, (promo ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_NONE), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("map:");
    for (int i = 0; i < 16; ++i) printf(" %016llx", (unsigned long long)tm.opaque[i]);
    printf("\n");
    printf("encode %d q %d box %u sizeof %zu align %zu\n", (int)r, (int)q, bw, sizeof(CUtensorMap), alignof(CUtensorMap));
    cudaMemcpy(g, &tm, sizeof tm, cudaMemcpyHostToDevice);
    for (int mode = want_mode; mode <= want_mode; ++mode)
        for (int c = 0; c < 2; ++c) {
            int x = c ? -1 : 3, y = c ? -1 : 5, z = c ? -1 : 7;
            if (mode == 0) k<0><<<1, 128>>>(tm, g, o, x, y, z, bw * 24 * 4);
            else if (mode == 1) k<1><<<1, 128>>>(tm, g, o, x, y, z, bw * 24 * 4);
            else k<2><<<1, 128>>>(tm, g, o, x, y, z, bw * 24 * 4);
            cudaError_t e = cudaDeviceSynchronize();
            std::vector<float> ho(864);
            cudaMemcpy(ho.data(), o, 864 * 4, cudaMemcpyDeviceToHost);
            int bad = 0;
            for (int zz = 0; zz < 4; ++zz) for (int yy = 0; yy < 6; ++yy) for (int xx = 0; xx < 36; ++xx) {
                int gx = x + xx, gy = y + yy, gz = z + zz;
                float want = (gx < 0 || gy < 0 || gz < 0 || gx >= n || gy >= n || gz >= n) ? 0.f : h[gx + n * (gy + n * gz)];
                bad += ho[xx + 36 * (yy + 6 * zz)] != want;
            }
            printf("mode %d corner %d: %s, mismatches %d\n", mode, c, cudaGetErrorString(e), bad);
            if (e != cudaSuccess) return 1;
        }
    return 0;
}
