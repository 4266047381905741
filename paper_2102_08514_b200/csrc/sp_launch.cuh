// sp_launch.cuh — kernel launch helpers and the generated-kernel registry entry type.
#pragma once

#include "sp_common.cuh"
#include "sp_evaluators.cuh"

namespace sp {

template <typename T>
using LaunchFn = cudaError_t (*)(const EvalArgs<T>&, int, size_t, cudaStream_t);

template <typename T, class Ev>
static cudaError_t launch_eval(const EvalArgs<T>& a, int blocks, size_t smem, cudaStream_t st) {
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(eval_kernel<T, Ev>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    eval_kernel<T, Ev><<<blocks, kThreads, smem, st>>>(a);
    return cudaGetLastError();
}

template <typename T>
using BrickLaunchFn = cudaError_t (*)(const EvalArgs<T>&, const long long*, int, int, int, size_t, cudaStream_t);

template <typename T, class Ev>
static cudaError_t launch_bricks(const EvalArgs<T>& a, const long long* bstart, int nbricks, int log2b, int blocks,
                                 size_t smem, cudaStream_t st) {
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(brick_kernel<T, Ev>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    brick_kernel<T, Ev><<<blocks, kThreads, smem, st>>>(a, bstart, nbricks, log2b);
    return cudaGetLastError();
}

template <typename T, class Ev>
static int occupancy_bricks(size_t smem) {
    int per_sm = 0;
    cudaFuncSetAttribute(brick_kernel<T, Ev>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, brick_kernel<T, Ev>, kThreads, smem) != cudaSuccess)
        per_sm = 1;
    return per_sm < 1 ? 1 : per_sm;
}

template <typename T, class Ev>
static int occupancy_blocks(size_t smem) {
    int per_sm = 0;
    cudaFuncSetAttribute(eval_kernel<T, Ev>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, eval_kernel<T, Ev>, kThreads, smem) != cudaSuccess)
        per_sm = 1;
    return per_sm < 1 ? 1 : per_sm;
}

struct GenEntry {
    const char* name;
    const uint64_t* blob;
    int blob_len;
    LaunchFn<float> launch_f32;
    LaunchFn<double> launch_f64;
    int (*occ_f32)(size_t);
    int (*occ_f64)(size_t);
    BrickLaunchFn<float> brick_f32;
    BrickLaunchFn<double> brick_f64;
    int (*bocc_f32)(size_t);
    int (*bocc_f64)(size_t);
};

}  // namespace sp
