// Standalone check of the 3-D TMA tile load used by brick_kernel_tma.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ CUtensorMap g_map;
__global__ void k(const __grid_constant__ CUtensorMap tmap_param, float* out, int bx, int by, int bz, int c0, int c1, int c2, int variant) {
    const CUtensorMap& tmap = (variant & 2) ? g_map : tmap_param;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) unsigned long long bar;
    unsigned char* smem = (unsigned char*)(((unsigned long long)smem_raw + 127) & ~127ull);
    const int boxv = bx * by * bz;
    if (threadIdx.x == 0) {
        unsigned a = (unsigned)__cvta_generic_to_shared(&bar);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a));
        if ((variant & 1) == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        else asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned a = (unsigned)__cvta_generic_to_shared(&bar);
        unsigned d = (unsigned)__cvta_generic_to_shared(smem);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"((variant & 8) ? 0 : boxv * 4) : "memory");
        if (variant & 8) {
            // mbarrier only (no copy): arrive with zero tx
        } else if (variant & 16) {
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(d), "l"(&tmap), "r"(c2), "r"(c1), "r"(c0), "r"(a) : "memory");
        } else {
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(d), "l"(&tmap), "r"(c2), "r"(c1), "r"(c0), "r"(a) : "memory");
        }
    }
    {
        unsigned a = (unsigned)__cvta_generic_to_shared(&bar);
        asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(a) : "memory");
    }
    const float* t = (const float*)smem;
    for (int e = threadIdx.x; e < boxv; e += blockDim.x) out[e] = t[e];
}

#include <cstdlib>
int main(int argc, char** argv) {
    const int only = argc > 1 ? atoi(argv[1]) : -1;
    const int E0 = 16, E1 = 16, E2 = 16;
    std::vector<float> h(E0 * E1 * E2);
    for (int i = 0; i < (int)h.size(); ++i) h[i] = (float)i;
    float *d, *o;
    cudaMalloc(&d, h.size() * 4);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    const int big = argc > 2 ? atoi(argv[2]) : 0;   // box shape: 1 = 16^3, else 12x11x11
    const int neg = argc > 3 ? atoi(argv[3]) : 1;   // coords: 1 = (-2,3,6), 0 = (0,0,0), 2 = (2,3,6)
    const int bx = big ? 16 : 12, by = big ? 16 : 11, bz = big ? 16 : 11;
    const int C0 = neg == 1 ? -2 : (neg == 2 ? 2 : 0), C1 = neg ? 3 : 0, C2 = neg == 3 ? -4 : (neg == 4 ? 5 : (neg == 5 ? -3 : (neg ? 8 : 0)));
    cudaMalloc(&o, bx * by * bz * 4);
    EncodeTiledFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    for (int l2 = 0; l2 < 2; ++l2) {
        for (int variant = 0; variant < 32; ++variant) {
            if (only >= 0 && variant != only) continue;
            CUtensorMap map;
            cuuint64_t dims[3] = {E2, E1, E0}, str[2] = {E2 * 4, E2 * E1 * 4};
            cuuint32_t box[3] = {bx, by, bz}, es[3] = {1, 1, 1};
            CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_NONE, l2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (variant & 2) cudaMemcpyToSymbol(g_map, &map, sizeof map);
            if (variant & 4) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(1); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = bx * by * bz * 4 + 128;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
                cfg.attrs = at; cfg.numAttrs = 1;
                cudaLaunchKernelEx(&cfg, k, map, o, bx, by, bz, C0, C1, C2, variant);
            } else {
                k<<<1, 128, bx * by * bz * 4 + 128>>>(map, o, bx, by, bz, C0, C1, C2, variant);
            }
            cudaError_t e = cudaDeviceSynchronize();
            std::vector<float> ho(bx * by * bz);
            cudaMemcpy(ho.data(), o, ho.size() * 4, cudaMemcpyDeviceToHost);
            int bad = 0;
            for (int z = 0; z < bz; ++z)
                for (int y = 0; y < by; ++y)
                    for (int x = 0; x < bx; ++x) {
                        int gz = z + C0, gy = y + C1, gx = x + C2;
                        float want = (gz >= 0 && gz < E0 && gy < E1 && gx < E2) ? h[(gz * E1 + gy) * E2 + gx] : 0.f;
                        if (ho[(z * by + y) * bx + x] != want) ++bad;
                    }
            printf("encode=%d l2=%d variant=%d err=%s bad=%d\n", (int)r, l2, variant, cudaGetErrorString(e), bad);
            if (e != cudaSuccess) return 1;
        }
    }
    return 0;
}
