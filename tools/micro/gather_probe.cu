// Probe: random 12-byte point gathers (protocol B reads the caller's points through the sort
// permutation) with different load flavours — time and, under ncu, DRAM bytes per point.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/gather_probe tools/micro/gather_probe.cu
//   /tmp/gather_probe [n]
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

__global__ void init_kernel(float* p, int* perm, long long n, unsigned long long a) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        p[3 * i] = (float)(i % 251);
        p[3 * i + 1] = (float)(i % 241);
        p[3 * i + 2] = (float)(i % 239);
        perm[i] = (int)((i * a + 12345) % n);  // a coprime to n: a permutation
    }
}

template <int MODE>
__device__ __forceinline__ float ld(const float* p) {
    float v;
    if (MODE == 0) v = __ldg(p);
    else if (MODE == 1) asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    else if (MODE == 2) asm volatile("ld.global.cs.f32 %0, [%1];" : "=f"(v) : "l"(p));
    else if (MODE == 3) asm volatile("ld.global.nc.L1::no_allocate.L2::64B.f32 %0, [%1];" : "=f"(v) : "l"(p));
    else v = *(volatile const float*)p;
    return v;
}

template <int MODE>
__global__ void gather_kernel(const float* __restrict__ p, const int* __restrict__ perm, long long n, float* __restrict__ out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long j = perm[i];
        const float* q = p + 3 * j;
        out[i] = ld<MODE>(q) + ld<MODE>(q + 1) + ld<MODE>(q + 2);
    }
}

// 4 independent gathers per thread in flight
template <int MODE>
__global__ void gather4_kernel(const float* __restrict__ p, const int* __restrict__ perm, long long n, float* __restrict__ out) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += 4 * stride) {
        float r[4];
        long long j[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) j[u] = i + u * stride < n ? perm[i + u * stride] : 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const float* q = p + 3 * j[u];
            r[u] = ld<MODE>(q) + ld<MODE>(q + 1) + ld<MODE>(q + 2);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (i + u * stride < n) out[i + u * stride] = r[u];
    }
}

int main(int argc, char** argv) {
    const long long n = argc > 1 ? atoll(argv[1]) : 100000000;
    float *p, *out;
    int* perm;
    CK(cudaMalloc(&p, 12 * n));
    CK(cudaMalloc(&perm, 4 * n));
    CK(cudaMalloc(&out, 4 * n));
    init_kernel<<<148 * 16, 256>>>(p, perm, n, 2654435761ull);
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char* name, void (*k)(const float*, const int*, long long, float*), int blocks) {
        k<<<blocks, 256>>>(p, perm, n, out);
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) k<<<blocks, 256>>>(p, perm, n, out);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-28s %.3f ms  %.2f Gpts/s\n", name, ms / 5, n / (ms / 5) / 1e6);
    };
    run("ldg", gather_kernel<0>, 148 * 16);
    run("nc.L1::no_allocate", gather_kernel<1>, 148 * 16);
    run("cs", gather_kernel<2>, 148 * 16);
    run("nc.no_alloc.L2::64B", gather_kernel<3>, 148 * 16);
    run("ldg x4 in flight", gather4_kernel<0>, 148 * 16);
    run("no_alloc x4 in flight", gather4_kernel<1>, 148 * 16);
    return 0;
}
