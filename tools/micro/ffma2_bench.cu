// Microbenchmark: FP32 FFMA vs packed FFMA2 (fma.rn.f32x2, sm_100a) issue throughput.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long f2(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long r;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

__global__ void k_ffma(float* out, int iters, float s) {
    float a[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j] = threadIdx.x * 0.001f + j;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 16; ++j) a[j] = fmaf(a[j], s, 0.5f * j);
    }
    float t = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) t += a[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

__global__ void k_ffma_reg(float* out, int iters, float s, float c) {
    float a[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j] = threadIdx.x * 0.001f + j;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 16; ++j) a[j] = fmaf(a[j], s, c);
    }
    float t = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) t += a[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

__global__ void k_ffma2(float* out, int iters, float s, float c) {
    unsigned long long a[8];
    float2 sv = make_float2(s, s), cv = make_float2(c, c);
    unsigned long long S = *reinterpret_cast<unsigned long long*>(&sv), C = *reinterpret_cast<unsigned long long*>(&cv);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        float2 v = make_float2(threadIdx.x * 0.001f + 2 * j, threadIdx.x * 0.001f + 2 * j + 1);
        a[j] = *reinterpret_cast<unsigned long long*>(&v);
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = f2(a[j], S, C);
    }
    float t = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        float2 v = *reinterpret_cast<float2*>(&a[j]);
        t += v.x + v.y;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

int main() {
    int blocks = 148 * 8, threads = 256, iters = 4096;
    float* out;
    cudaMalloc(&out, blocks * threads * sizeof(float));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int v = 0; v < 3; ++v) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (v == 0) k_ffma<<<blocks, threads>>>(out, iters, 0.999f);
            else if (v == 1) k_ffma_reg<<<blocks, threads>>>(out, iters, 0.999f, 0.25f);
            else k_ffma2<<<blocks, threads>>>(out, iters, 0.999f, 0.25f);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double fmas = (double)blocks * threads * iters * 16;
        printf("%s: %.3f ms  %.1f TFMA/s  (%.1f TFLOP/s)\n", v == 0 ? "FFMA imm" : (v == 1 ? "FFMA reg" : "FFMA2   "), ms,
               fmas / ms / 1e9, 2 * fmas / ms / 1e9);
    }
    return 0;
}
