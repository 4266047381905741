// sp_launch.cuh — kernel launch helpers and the generated-kernel registry entry type.
#pragma once

#include <map>
#include <mutex>
#include <utility>

#include "sp_common.cuh"
#include "sp_evaluators.cuh"

namespace sp {

// Blocks per SM of `kern` at `smem` bytes, memoised per (kernel, smem): the occupancy query
// costs tens of microseconds of host time, which short launches cannot hide.
template <typename K>
static int cached_occupancy(K kern, size_t smem) {
    // keyed by the kernel too: every kernel of one signature shares this instantiation
    static std::mutex mu;
    static std::map<std::pair<const void*, size_t>, int> memo;
    std::lock_guard<std::mutex> lock(mu);
    const auto key = std::make_pair(reinterpret_cast<const void*>(kern), smem);
    auto it = memo.find(key);
    if (it != memo.end()) return it->second;
    int per_sm = 0;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    memo[key] = per_sm;
    return per_sm;
}

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
    return cached_occupancy(brick_kernel<T, Ev>, smem);
}

template <typename T, class Ev>
static int occupancy_blocks(size_t smem) {
    return cached_occupancy(eval_kernel<T, Ev>, smem);
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
    int trec_bytes;  // per-tile address records (+ tables) in smem
};

}  // namespace sp
