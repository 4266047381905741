// sp_launch.cuh — kernel launch helpers and the generated-kernel registry entry type.
#pragma once

#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>
#include <utility>

#include "sp_common.cuh"
#include "sp_evaluators.cuh"

namespace sp {

// cudaFuncSetAttribute acts on the current device: done once per (kernel, device).  Keyed by
// the kernel address (kernels of one signature share any per-instantiation static).
template <typename K>
static cudaError_t ensure_smem_limit(K kern, int dev) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, cudaError_t> done;
    std::lock_guard<std::mutex> lock(mu);
    const auto key = std::make_pair(reinterpret_cast<const void*>(kern), dev);
    auto it = done.find(key);
    if (it != done.end()) return it->second;
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    if (e == cudaSuccess) done[key] = e;
    return e;
}

template <typename K>
static cudaError_t ensure_smem_limit(K kern) {
    int dev = 0;
    cudaGetDevice(&dev);
    return ensure_smem_limit(kern, dev);
}

// Blocks per SM of `kern` at `smem` bytes, memoised per (kernel, smem, device): the occupancy
// query costs tens of microseconds of host time, which short launches cannot hide.  Also
// raises the kernel's dynamic shared-memory limit on this device.
template <typename K>
static int cached_occupancy(K kern, size_t smem) {
    int dev = 0;
    cudaGetDevice(&dev);
    static std::mutex mu;
    static std::map<std::tuple<const void*, size_t, int>, int> memo;
    {
        std::lock_guard<std::mutex> lock(mu);
        auto it = memo.find(std::make_tuple(reinterpret_cast<const void*>(kern), smem, dev));
        if (it != memo.end()) return it->second;
    }
    int per_sm = 0;
    ensure_smem_limit(kern, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    std::lock_guard<std::mutex> lock(mu);
    memo[std::make_tuple(reinterpret_cast<const void*>(kern), smem, dev)] = per_sm;
    return per_sm;
}

template <typename T>
using LaunchFn = cudaError_t (*)(const EvalArgs<T>&, int, size_t, cudaStream_t);

template <typename T, class Ev>
static cudaError_t launch_eval(const EvalArgs<T>& a, int blocks, size_t smem, cudaStream_t st) {
    const cudaError_t e = ensure_smem_limit(eval_kernel<T, Ev>);
    if (e != cudaSuccess) return e;
    eval_kernel<T, Ev><<<blocks, kThreads, smem, st>>>(a);
    return cudaGetLastError();
}

template <typename T>
using BrickLaunchFn = cudaError_t (*)(const EvalArgs<T>&, const long long*, int, int, int, size_t, cudaStream_t);

template <typename T, class Ev>
static cudaError_t launch_bricks(const EvalArgs<T>& a, const long long* bstart, int nbricks, int log2b, int blocks,
                                 size_t smem, cudaStream_t st) {
    const cudaError_t e = ensure_smem_limit(brick_kernel<T, Ev>);
    if (e != cudaSuccess) return e;
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

// Texture-filtered variant of a generated plan (TexFetch, sp_eval_texture): thread per point,
// plan tables in shared memory, every fetch from the cosets' texture objects.
template <class Ev>
__global__ void __launch_bounds__(kThreads) tex_eval_kernel(const EvalArgs<float> a, const TexArgs targs) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ TileGeom geom;  // not read by the texture fetcher
    const int tb = (a.table_bytes + 15) & ~15;
    if (a.table_bytes > 0) {
        const int4* src = reinterpret_cast<const int4*>(a.tables);
        int4* dst = reinterpret_cast<int4*>(smem);
        for (int i = threadIdx.x; i < tb / 16; i += kThreads) dst[i] = src[i];
    }
    __syncthreads();
    EvalCtx<float, Ev> ctx;
    ctx.a = &a;
    ctx.tables = smem;
    ctx.geom = &geom;
    ctx.trec = nullptr;
    ctx.err = 0;
    for (long long i = blockIdx.x * (long long)kThreads + threadIdx.x; i < a.n; i += (long long)gridDim.x * kThreads) {
        const float x[3] = {a.pts[3 * i], a.pts[3 * i + 1], a.pts[3 * i + 2]};
        float v = NAN;
        if (isfinite(x[0]) && isfinite(x[1]) && isfinite(x[2])) {
            ctx.index = i;
            ctx.X[0] = clamp_cell(x[0]);
            ctx.X[1] = clamp_cell(x[1]);
            ctx.X[2] = clamp_cell(x[2]);
            TexFetch f;
            f.targs = &targs;
            v = Ev::template eval<TexFetch>(x, f, ctx);
        }
        a.out[i] = v;
    }
    if (ctx.err && a.err) atomicOr(a.err, 1);
}

using TexLaunchFn = cudaError_t (*)(const EvalArgs<float>&, const TexArgs&, cudaStream_t);

template <class Ev>
static cudaError_t launch_tex(const EvalArgs<float>& a, const TexArgs& t, cudaStream_t st) {
    const long long blocks = std::min<long long>((a.n + kThreads - 1) / kThreads, 148ll * 16);
    tex_eval_kernel<Ev><<<(int)std::max<long long>(1, blocks), kThreads, (a.table_bytes + 15) & ~15, st>>>(a, t);
    return cudaGetLastError();
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
    TexLaunchFn tex_f32;  // hardware-texture variant (float32)
    const uint32_t* cube_tab;  // unit-cube class-word table (codegen.cube_table), or null
    int cube_len;
    int smem_table_bytes;      // leading bytes of the plan tables staged into shared memory
    int tile_kb;               // shared-memory tile budget of the brick kernels (codegen.tile_budget_kb)
};

}  // namespace sp
