// sp_tma.cuh — brick kernel with TMA (cp.async.bulk.tensor) double-buffered staging.
//
// For single-coset tensor-product plans with the 'zero' boundary policy the staged brick box
// has the same shape for every brick, so one tensor map (box = brick + site reach, padded to
// 16 bytes) covers all of them: one elected thread issues the 3-D bulk tensor copy of the
// NEXT brick into the other shared-memory buffer (mbarrier complete_tx) while the CTA
// evaluates the current one; out-of-range texels are zero-filled by the TMA unit, which is
// exactly the 'zero' policy (runtime.py:155-161).  No per-element staging instructions.
#pragma once

#include <cuda.h>

#include "sp_common.cuh"
#include "sp_evaluators.cuh"

namespace sp {

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, unsigned long long* bar, int c0, int c1,
                                            int c2) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
            "r"(d),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(b)
        : "memory");
}

// Row-vector copy of a staged box: vtile[(z*vy + y)*vx + x] = tile[(z*by + y)*bx + x .. +kVec)
// (the (vx, vy) pitches may be padded for conflict-free row loads).
template <typename T, int kVec>
__device__ __forceinline__ void build_vtile(const T* tile, typename VecT<T, kVec>::type* vtile, int boxv, bool padded,
                                            int bx, int by, int vx, int vy, unsigned mx, unsigned sx, unsigned my,
                                            unsigned sy, int tid) {
    using V = typename VecT<T, kVec>::type;
    for (int e = tid; e < boxv; e += kThreads) {
        V v;
        T* pv = reinterpret_cast<T*>(&v);
#pragma unroll
        for (int q = 0; q < kVec; ++q) pv[q] = e + q < boxv ? tile[e + q] : T(0);
        int d = e;
        if (padded) {
            const int r = (int)fastdiv((unsigned)e, mx, sx);  // z*by + y
            const int z = (int)fastdiv((unsigned)r, my, sy);
            d = (r + z * (vy - by)) * vx + (e - r * bx);
        }
        vtile[d] = v;
    }
}

// G = geometry known at compile time (0: runtime arguments): {log2b, bx, by, bz, vx, vy}.
template <int L2B = 0, int BX = 0, int BY = 0, int BZ = 0, int VX = 0, int VY = 0>
struct TmaGeom {};

template <class G, int I>
struct GeomVal;
template <int L2B, int BX, int BY, int BZ, int VX, int VY, int I>
struct GeomVal<TmaGeom<L2B, BX, BY, BZ, VX, VY>, I> {
    static constexpr int v[6] = {L2B, BX, BY, BZ, VX, VY};
    static constexpr int value = v[I];
};
// compile-time value when the geometry fixes it, else the runtime argument
template <class G, int I>
__device__ __forceinline__ int geom_or(int runtime) {
    constexpr int c = GeomVal<G, I>::value;
    return c > 0 ? c : runtime;
}

// Single-coset (M = 1) brick kernel, T = float, evaluators with a row-vector tile.
// box = (bz, by, bx) coset cells; bx is a multiple of 4 (16-byte TMA rows) and 3 wider than
// needed, because the box's innermost start coordinate must be 16-byte aligned; the host may
// widen bx / by further so that the row loads are bank-conflict free (choose_box_pitch).
template <typename T, class Ev, class G = TmaGeom<>>
__global__ void __launch_bounds__(kThreads, Ev::kMinBlocks)
    brick_kernel_tma(const EvalArgs<T> a, const __grid_constant__ CUtensorMap tmap,
                     const long long* __restrict__ brick_start, int nbricks, int log2b_, int bx_, int by_, int bz_,
                     int vx_, int vy_) {
    const int log2b = geom_or<G, 0>(log2b_), bx = geom_or<G, 1>(bx_), by = geom_or<G, 2>(by_);
    const int bz = geom_or<G, 3>(bz_), vx = geom_or<G, 4>(vx_), vy = geom_or<G, 5>(vy_);
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ TileGeom geom;
    __shared__ __align__(8) unsigned long long mbar[2];
    __shared__ int corner[2][3];
    constexpr int kVec = Ev::template vec_width<T>();
    using V = typename VecT<T, kVec>::type;
    static_assert(kVec > 0, "TMA brick path is for row-vector evaluators");

    const int tid = threadIdx.x;
    const int boxv = bx * by * bz;
    const int buf_bytes = (boxv * (int)sizeof(T) + 127) & ~127;
    auto buf = [&](int slot) { return reinterpret_cast<T*>(smem + slot * buf_bytes); };
    V* vtile = reinterpret_cast<V*>(smem + 2 * buf_bytes);
    const int B = 1 << log2b;
    const bool padded = vx != bx || vy != by;
    unsigned mx, sx, my, sy;
    fastdiv_magic((unsigned)bx, mx, sx);
    fastdiv_magic((unsigned)by, my, sy);

    if (tid == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    // thread 0: brick corner from its first point, then the bulk tensor copy of its box
    auto issue = [&](int b, int slot) {
        const T* x = point_ptr(a, brick_start[b]);
        int c[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            c[i] = (clamp_cell(x[i]) >> log2b) << log2b;
            corner[slot][i] = c[i];
        }
        // array index of the box origin (may be negative: TMA zero-fills out of range); the
        // innermost coordinate must be 16-byte aligned, so it is rounded down to 4 floats
        // (the host widens the box by 3 to cover it)
        const int z0 = c[0] + a.fr.reach_lo[0] - a.grid.org[0][0];
        const int z1 = c[1] + a.fr.reach_lo[1] - a.grid.org[0][1];
        const int z2 = (c[2] + a.fr.reach_lo[2] - a.grid.org[0][2]) & ~3;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&mbar[slot], (unsigned)(boxv * sizeof(T)));
        tma_load_3d(buf(slot), &tmap, &mbar[slot], z2, z1, z0);
        // and the brick's points into L2 (bulk prefetch, 16-byte granules inside the array): the
        // per-point loads of the brick then hit L2 instead of waiting on HBM
        if (a.prefetch_pts && !a.in_index32) prefetch_points_l2(a, brick_start[b], brick_start[b + 1]);
    };

    if (a.nbricks_dev) nbricks = min(nbricks, *a.nbricks_dev);
    const bool plain = !a.in_index32 && !a.out_index && !a.out_index32 && !a.dbg && a.plain_pts;
    if (tid == 0 && (int)blockIdx.x < nbricks) issue(blockIdx.x, 0);
    unsigned phase = 0u;  // bit s = mbarrier parity of buffer s
    int it = 0;
    for (int b = blockIdx.x; b < nbricks; b += gridDim.x, ++it) {
        const int cur = it & 1;
        const int nb = b + gridDim.x;
        if (tid == 0 && nb < nbricks) issue(nb, cur ^ 1);  // overlaps this brick's evaluation
        mbar_wait(&mbar[cur], (phase >> cur) & 1u);
        phase ^= 1u << cur;
        const T* tile = buf(cur);
        const int c0 = corner[cur][0], c1 = corner[cur][1], c2 = corner[cur][2];
        const int lo0 = c0 + a.fr.reach_lo[0], lo1 = c1 + a.fr.reach_lo[1];
        const int lo2 = ((c2 + a.fr.reach_lo[2] - a.grid.org[0][2]) & ~3) + a.grid.org[0][2];
        build_vtile<T, kVec>(tile, vtile, boxv, padded, bx, by, vx, vy, mx, sx, my, sy, tid);
        if (tid == 0) {
            geom.staged = 1;
            geom.total = boxv;
            geom.off[0] = 0;
            geom.lo[0][0] = lo0;
            geom.lo[0][1] = lo1;
            geom.lo[0][2] = lo2;
            geom.ex[0][0] = bz;
            geom.ex[0][1] = by;
            geom.ex[0][2] = bx;
            geom.vx = vx;
            geom.vy = vy;
            geom.vtotal = vx * vy * bz;
            geom.vbase = -lo0 * vy * vx - lo1 * vx - lo2;
            geom.st0[0] = by * bx;  // scalar (TMA) tile pitches
            geom.st1[0] = bx;
            geom.cbase[0] = -lo0 * by * bx - lo1 * bx - lo2;
        }
        __syncthreads();

        EvalCtx<T, Ev> ctx;
        ctx.a = &a;
        ctx.tables = smem;
        ctx.geom = &geom;
        ctx.trec = nullptr;
        ctx.err = 0;
        ctx.load_geom(geom, 1);
        const long long p0 = brick_start[b], p1 = brick_start[b + 1];
        if (plain) {
            // plain brick-order points (no permutations, no debug output): direct point loads and
            // stores, and "inside the staged brick" from the saturating floor conversions (far
            // points fail it) plus one NaN test (x0 + x1 + x2 != itself); the others take
            // eval_one's paths
            // bricks at the clamp limit (corner + B > 2^30) keep the clamped path for every point
            const bool bexact = c0 + B <= kCellClamp && c1 + B <= kCellClamp && c2 + B <= kCellClamp;
            const T* px = a.pts + 3 * (p0 + tid);
            T y0 = T(0), y1 = T(0), y2 = T(0);
            if (p0 + tid < p1) {
                y0 = __ldg(px);
                y1 = __ldg(px + 1);
                y2 = __ldg(px + 2);
            }
#pragma unroll 1
            for (long long j = p0 + tid; j < p1; j += kThreads) {
                const T x[3] = {y0, y1, y2};
                px += 3 * kThreads;
                if (j + kThreads < p1) {
                    y0 = __ldg(px);
                    y1 = __ldg(px + 1);
                    y2 = __ldg(px + 2);
                }
                T v;
                const int X0 = floor_int(x[0]), X1 = floor_int(x[1]), X2 = floor_int(x[2]);
                const T sum = x[0] + x[1] + x[2];
                if (bexact & ((unsigned)(X0 - c0) < (unsigned)B) & ((unsigned)(X1 - c1) < (unsigned)B) &
                    ((unsigned)(X2 - c2) < (unsigned)B) & (sum == sum)) {
                    ctx.X[0] = X0;  // = clamp_cell(x): |X| < 2^30 inside an exact brick
                    ctx.X[1] = X1;
                    ctx.X[2] = X2;
                    TileFetch<T, V> f;
                    f.tile = tile;
                    f.vtile = vtile;
                    SP_TILE_LIMIT(f, ctx.geom->total);
                    v = Ev::template eval<TileFetch<T, V>>(x, f, ctx);
                } else {
                    ctx.index = j;
                    ctx.X[0] = clamp_cell(x[0]);
                    ctx.X[1] = clamp_cell(x[1]);
                    ctx.X[2] = clamp_cell(x[2]);
                    v = eval_one<T, Ev, V>(x, true, c0, c1, c2, B, tile, vtile, ctx);
                }
                SP_CHECK(j >= 0 && j < a.n);
                a.out[j] = v;
            }
            if (ctx.err && a.err) atomicOr(a.err, 1);
            __syncthreads();  // vtile / geom / this buffer are rewritten next iteration
            continue;
        }
        T xn0 = T(0), xn1 = T(0), xn2 = T(0);
        if (p0 + tid < p1) {
            const T* px = point_ptr(a, p0 + tid);
            xn0 = __ldg(px);
            xn1 = __ldg(px + 1);
            xn2 = __ldg(px + 2);
        }
#pragma unroll 1
        for (long long j = p0 + tid; j < p1; j += kThreads) {
            ctx.index = j;
            const T x[3] = {xn0, xn1, xn2};
            if (j + kThreads < p1) {
                const T* px = point_ptr(a, j + kThreads);
                xn0 = __ldg(px);
                xn1 = __ldg(px + 1);
                xn2 = __ldg(px + 2);
            }
            ctx.X[0] = clamp_cell(x[0]);
            ctx.X[1] = clamp_cell(x[1]);
            ctx.X[2] = clamp_cell(x[2]);
            store_out(a, j, eval_one<T, Ev, V>(x, true, c0, c1, c2, B, tile, vtile, ctx));
        }
        if (ctx.err && a.err) atomicOr(a.err, 1);
        __syncthreads();  // vtile / geom / this buffer are rewritten next iteration
    }
}

}  // namespace sp
