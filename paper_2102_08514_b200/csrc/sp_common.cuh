// sp_common.cuh — shared device machinery of the reconstruction kernels (sm_100a).
//
// The reference evaluates Algorithm 1 as numpy passes over the whole
// batch (runtime.py:363-408) with fancy-index gathers into per-coset float64 arrays
// (runtime.py:151-188).  Here one CTA owns a chunk of kThreads*ppt consecutive query points:
//
//   1. it loads the chunk, reduces the bounding box of the points' unit cells,
//   2. if the box (+ the plan's site reach, per coset) fits the shared-memory budget it
//      stages those coefficients ONCE into shared memory, applying the grid's boundary
//      policy while staging (zero / clamp / mirror, runtime.py:109-123, :151-168, :191-204),
//      so the per-point gathers are unchecked shared-memory reads,
//   3. otherwise (incoherent point order) every read goes to global memory (L2) through
//      the same policy function.
//
// Points presented in Morton order (sp_morton_keys) make step 2 the common case; any order
// is correct.  The per-point evaluators (TP B-spline, generated plan kernels, generic plan
// interpreter) only see the Fetch interface below.
#pragma once

#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/splinerecon.h"

namespace sp {

constexpr int kThreads = 256;
constexpr int kMaxPPT = 8;                    // points per thread per chunk (runtime <= this)
constexpr int kCellClamp = 1 << 30;           // |cell| clamp (mirror exact below this)

template <typename T>
struct GridArgs {
    const T* data[SP_MAX_COSETS];
    int ext[SP_MAX_COSETS][3];
    int org[SP_MAX_COSETS][3];
    int M;
    int boundary;
};

struct FrameArgs {
    int M;
    int diag[3];
    int shift[SP_MAX_COSETS][3];
    int reach_lo[3];  // site reach in coset cells, relative to floor((x - l_k)/d)
    int reach_hi[3];
    int dlog2[3];     // log2(d_i) when d_i is a power of two, else -1
};

template <typename T>
struct EvalArgs {
    GridArgs<T> grid;
    FrameArgs fr;
    const T* pts;
    T* out;
    long long n;
    int* dbg;           // nullable [n*M*4]
    int* err;           // nullable
    const void* tables; // evaluator tables (device), copied to smem when table_bytes > 0
    int table_bytes;
    int tile_cap;       // staged-tile capacity in elements
    int ppt;            // points per thread per chunk (chunk = kThreads * ppt)
    int margin;         // extra halo cells (1 for float64 points on shifted cosets, else 0)
    unsigned long long* stats;  // nullable: [0] staged chunks, [1] unstaged chunks, [2] staged elements
    const long long* out_index; // nullable: value of point i goes to out[out_index[i]]
    const int* out_index32;     // nullable: same with int32 indices (sp_sort_points' permutation)
    const int* in_index32;      // nullable: brick-order point j is pts[in_index32[j]] (unsorted input, no gather)
    int trec_bytes;             // per-(coset, class) tile records (generated kernels), in smem
    int vec_cap;                // row-vector tile capacity in elements (0: no row-vector tile)
    const int* nbricks_dev;     // nullable: brick count in device memory (sync-free brick runs)
    int prefetch_pts;           // TMA brick kernel: bulk-prefetch each next brick's points into L2
    int plain_pts;              // brick kernels: plain-point loop (SP_PLAIN_PTS, default on)
    int box_pad[3];             // single-coset plans: extra staged cells at the high end per axis
                                // (bank-conflict-free tile pitches for scalar float64 rows)
};

// Checked build (build.py --checked -> libsplinerecon_checked.so, loaded with SP_CHECKED=1):
// shared-tile, point and output indices are bounds-checked and a violation traps with a
// message (compute-sanitizer is not available on the GPU pool).  Compiled out otherwise.
#ifdef SP_BOUNDS_CHECK
#define SP_CHECK(cond)                                                                              \
    do {                                                                                            \
        if (!(cond)) {                                                                              \
            printf("splinerecon bounds check failed: %s (%s:%d) block %d thread %d\n", #cond,      \
                   __FILE__, __LINE__, (int)blockIdx.x, (int)threadIdx.x);                          \
            __trap();                                                                               \
        }                                                                                           \
    } while (0)
#define SP_TILE_LIMIT(f, n) ((f).lim = (n))
#else
#define SP_CHECK(cond) \
    do {               \
    } while (0)
#define SP_TILE_LIMIT(f, n) ((void)0)
#endif

struct TileGeom {
    int staged;
    int total;
    int off[SP_MAX_COSETS];
    int lo[SP_MAX_COSETS][3];  // box origin in coset-cell coordinates
    int ex[SP_MAX_COSETS][3];  // box extents
    unsigned fdm[SP_MAX_COSETS][3];  // fast-division magic / shift for ex[k][1], ex[k][2]
    unsigned fds[SP_MAX_COSETS][3];
    // tile address of coset cell (c0,c1,c2) = cbase[k] + c0*st0[k] + c1*st1[k] + c2
    int cbase[SP_MAX_COSETS];
    int st0[SP_MAX_COSETS];
    int st1[SP_MAX_COSETS];
    // row-vector tile (coset 0): padded pitches vx, vy (vx = 6 mod 8, vy = 2 mod 4 makes the
    // 16-byte rows of any 2x2x2 cell block fall in distinct bank groups), address base
    int vx, vy, vtotal, vbase;
    unsigned vfm_x, vfs_x, vfm_y, vfs_y;
};

__device__ __forceinline__ int floordiv_i(int a, int d) {
    int q = a / d;
    return (a % d != 0 && ((a < 0) != (d < 0))) ? q - 1 : q;
}

// floor(v) as int, clamped to +-kCellClamp.  cvt.rmi saturates out-of-range values and maps
// NaN to 0, so this is branch-free (non-finite points are masked out by the callers).
__device__ __forceinline__ int clamp_cell(float v) { return min(max(__float2int_rd(v), -kCellClamp), kCellClamp); }
__device__ __forceinline__ int clamp_cell(double v) { return min(max(__double2int_rd(v), -kCellClamp), kCellClamp); }
// floor(v) as int, saturating (cvt.rmi), NaN -> 0: equals clamp_cell(v) for |v| < 2^30
__device__ __forceinline__ int floor_int(float v) { return __float2int_rd(v); }
__device__ __forceinline__ int floor_int(double v) { return __double2int_rd(v); }

__device__ __forceinline__ int mirror_index(int v, int n) {
    // runtime.py:191-196 (period 2n-2)
    if (n == 1) return 0;
    int p = 2 * n - 2;
    v = abs(v) % p;
    return v >= n ? p - v : v;
}

// Policy read of array index (z0,z1,z2) of coset k (index = cell - origin).
template <typename T>
__device__ __forceinline__ T policy_read(const GridArgs<T>& g, int k, int z0, int z1, int z2) {
    const int e0 = g.ext[k][0], e1 = g.ext[k][1], e2 = g.ext[k][2];
    const bool in = (unsigned)z0 < (unsigned)e0 && (unsigned)z1 < (unsigned)e1 && (unsigned)z2 < (unsigned)e2;
    if (!in) {
        if (g.boundary == SP_ZERO) return T(0);
        if (g.boundary == SP_CLAMP) {
            z0 = min(max(z0, 0), e0 - 1);
            z1 = min(max(z1, 0), e1 - 1);
            z2 = min(max(z2, 0), e2 - 1);
        } else {
            z0 = mirror_index(z0, e0);
            z1 = mirror_index(z1, e1);
            z2 = mirror_index(z2, e2);
        }
    }
    return __ldg(g.data[k] + ((long long)z0 * e1 + z1) * (long long)e2 + z2);
}

// Out-of-line variant for the (rare) unstaged path: keeps the kernels' code small.  Scalar
// arguments only (a pointer to the kernel-parameter struct would force a local copy of it).
template <typename T>
__device__ __noinline__ T policy_read_slow(const T* data, int e0, int e1, int e2, int boundary, int z0, int z1,
                                           int z2) {
    const bool in = (unsigned)z0 < (unsigned)e0 && (unsigned)z1 < (unsigned)e1 && (unsigned)z2 < (unsigned)e2;
    if (!in) {
        if (boundary == SP_ZERO) return T(0);
        if (boundary == SP_CLAMP) {
            z0 = min(max(z0, 0), e0 - 1);
            z1 = min(max(z1, 0), e1 - 1);
            z2 = min(max(z2, 0), e2 - 1);
        } else {
            z0 = mirror_index(z0, e0);
            z1 = mirror_index(z1, e1);
            z2 = mirror_index(z2, e2);
        }
    }
    return __ldg(data + ((long long)z0 * e1 + z1) * (long long)e2 + z2);
}

// ---------------------------------------------------------------------------------------
// Fetchers.  A "frame" fixes the coset, the base cell and the class's site renaming
// (piA = signed permutation rho/tau, probe12 of SURVEY.md §9): the site with zero-coset
// offsets (s0,s1,s2)/d reads coset cell  base_i + tau_i * s[rho_i].  Generated kernels call
// get() with compile-time offsets, so the address arithmetic folds to IMADs.

template <typename T, typename V = T>
struct TileFetch {
    static constexpr bool kIsTile = true;
    const T* tile;
    const V* vtile;  // row-vector copy of the tile (evaluators with vec_width > 0)
    int a0;
    int c0, c1, c2;
#ifdef SP_BOUNDS_CHECK
    int lim;  // staged scalar tile elements
#endif

    __device__ __forceinline__ void frame(const TileGeom& tg, int k, const int base[3], const int rho[3],
                                          const int tau[3]) {
        const int ex1 = tg.ex[k][1], ex2 = tg.ex[k][2];
        const int st[3] = {ex1 * ex2, ex2, 1};
        a0 = tg.off[k] + (base[0] - tg.lo[k][0]) * st[0] + (base[1] - tg.lo[k][1]) * st[1] + (base[2] - tg.lo[k][2]);
        int c[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) c[i] = 0;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const int v = tau[i] * st[i];
            c[0] = rho[i] == 0 ? v : c[0];
            c[1] = rho[i] == 1 ? v : c[1];
            c[2] = rho[i] == 2 ? v : c[2];
        }
        c0 = c[0];
        c1 = c[1];
        c2 = c[2];
    }
    __device__ __forceinline__ void frame_identity(const TileGeom& tg, int k, const int base[3]) {
        const int ex1 = tg.ex[k][1], ex2 = tg.ex[k][2];
        c0 = ex1 * ex2;
        c1 = ex2;
        c2 = 1;
        a0 = tg.off[k] + (base[0] - tg.lo[k][0]) * c0 + (base[1] - tg.lo[k][1]) * c1 + (base[2] - tg.lo[k][2]);
    }
    __device__ __forceinline__ T get(int s0, int s1, int s2) const {
        SP_CHECK((unsigned)(a0 + s0 * c0 + s1 * c1 + s2 * c2) < (unsigned)lim);
        return tile[a0 + s0 * c0 + s1 * c1 + s2 * c2];
    }
    // a 2-site fetch group (the paper's linear-fetch merge, §4.4) done exactly in software:
    // acc + g*c0 + t_num*(c1 - c0)  (plancompile.py:669-697 up to the local-lerp rounding)
    __device__ __forceinline__ T lerp2(T acc, T g, T tn, int a0_, int a1_, int a2_, int b0_, int b1_, int b2_) const {
        const T c0 = get(a0_, a1_, a2_);
        const T c1 = get(b0_, b1_, b2_);
        acc = fma(g, c0, acc);
        return fma(tn, c1 - c0, acc);
    }
};

template <typename T>
struct GlobalFetch {
    static constexpr bool kIsTile = false;
    const T* data;
    int e0, e1, e2, boundary;
    int b0, b1, b2;       // base array index (cell - origin)
    int p[3][3];          // p[j][i] = tau_i if rho_i == j

    __device__ __forceinline__ void frame(const GridArgs<T>& grid, int kk, const int base[3], const int rho[3],
                                          const int tau[3]) {
        data = grid.data[kk];
        e0 = grid.ext[kk][0];
        e1 = grid.ext[kk][1];
        e2 = grid.ext[kk][2];
        boundary = grid.boundary;
        b0 = base[0] - grid.org[kk][0];
        b1 = base[1] - grid.org[kk][1];
        b2 = base[2] - grid.org[kk][2];
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int i = 0; i < 3; ++i) p[j][i] = rho[i] == j ? tau[i] : 0;
    }
    __device__ __forceinline__ void frame_identity(const GridArgs<T>& grid, int kk, const int base[3]) {
        const int rho[3] = {0, 1, 2}, tau[3] = {1, 1, 1};
        frame(grid, kk, base, rho, tau);
    }
    __device__ __forceinline__ T get(int s0, int s1, int s2) const {
        const int z0 = b0 + s0 * p[0][0] + s1 * p[1][0] + s2 * p[2][0];
        const int z1 = b1 + s0 * p[0][1] + s1 * p[1][1] + s2 * p[2][1];
        const int z2 = b2 + s0 * p[0][2] + s1 * p[1][2] + s2 * p[2][2];
        return policy_read_slow(data, e0, e1, e2, boundary, z0, z1, z2);
    }
    // a 2-site fetch group (the paper's linear-fetch merge, §4.4) done exactly in software:
    // acc + g*c0 + t_num*(c1 - c0)  (plancompile.py:669-697 up to the local-lerp rounding)
    __device__ __forceinline__ T lerp2(T acc, T g, T tn, int a0_, int a1_, int a2_, int b0_, int b1_, int b2_) const {
        const T c0 = get(a0_, a1_, a2_);
        const T c1 = get(b0_, b1_, b2_);
        acc = fma(g, c0, acc);
        return fma(tn, c1 - c0, acc);
    }
};

// Hardware-texture fetcher (the paper's GPU path, PAPER.md:334 / §4.4): one texture object
// per coset (cudaFilterModeLinear, unnormalised coordinates, texel i = array index i, centre
// at i + 0.5; border = 'zero', clamp = 'clamp').  get() samples a texel centre (exact); a
// 2-site group is ONE filtered fetch at c0's centre + (t_num/g) toward c1 — the filtering
// weight is 9-bit fixed point, so this variant is NOT exact (reported separately).
struct TexArgs {
    cudaTextureObject_t tex[SP_MAX_COSETS];
};
struct TexFetch {
    static constexpr bool kIsTile = false;
    const TexArgs* targs;
    cudaTextureObject_t t;
    int b0, b1, b2;
    int p[3][3];
    __device__ __forceinline__ void frame(const GridArgs<float>& grid, int kk, const int base[3], const int rho[3],
                                          const int tau[3]) {
        t = targs->tex[kk];
        b0 = base[0] - grid.org[kk][0];
        b1 = base[1] - grid.org[kk][1];
        b2 = base[2] - grid.org[kk][2];
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int i = 0; i < 3; ++i) p[j][i] = rho[i] == j ? tau[i] : 0;
    }
    __device__ __forceinline__ void index(int s0, int s1, int s2, int z[3]) const {
        z[0] = b0 + s0 * p[0][0] + s1 * p[1][0] + s2 * p[2][0];
        z[1] = b1 + s0 * p[0][1] + s1 * p[1][1] + s2 * p[2][1];
        z[2] = b2 + s0 * p[0][2] + s1 * p[1][2] + s2 * p[2][2];
    }
    __device__ __forceinline__ float get(int s0, int s1, int s2) const {
        int z[3];
        index(s0, s1, s2, z);
        return tex3D<float>(t, (float)z[2] + 0.5f, (float)z[1] + 0.5f, (float)z[0] + 0.5f);
    }
    __device__ __forceinline__ float lerp2(float acc, float g, float tn, int a0_, int a1_, int a2_, int b0_, int b1_,
                                           int b2_) const {
        int za[3], zb[3];
        index(a0_, a1_, a2_, za);
        index(b0_, b1_, b2_, zb);
        const float tt = g == 0.0f ? 0.5f : tn / g;
        const float v = tex3D<float>(t, (float)za[2] + 0.5f + tt * (float)(zb[2] - za[2]),
                                     (float)za[1] + 0.5f + tt * (float)(zb[1] - za[1]),
                                     (float)za[0] + 0.5f + tt * (float)(zb[0] - za[0]));
        return fma(g, v, acc);
    }
};

// ---------------------------------------------------------------------------------------
// The chunk driver.  Ev provides:
//   static constexpr bool kNeedsTables;
//   template <class F, class Ctx> static T eval(const T x[3], F& fetch, const Ctx& ctx)
// where Ctx gives the evaluator access to its smem tables, the tile geometry and args.

template <typename T, class Ev>
struct EvalCtx {
    const EvalArgs<T>* a;
    const unsigned char* tables;  // smem copy (or global when not staged)
    const TileGeom* geom;
    const int4* trec;             // per-(coset, class) tile address records (generated kernels)
    long long index;              // point index (for debug output)
    int X[3];                     // floor(x) of the current point (clamped), computed once
    mutable int err;              // sigma-sentinel hits, flushed with one atomic per thread
    int cbase[SP_MAX_COSETS];     // register copies of the tile geometry (staged path)
    int st0[SP_MAX_COSETS];
    int st1[SP_MAX_COSETS];
    int vbase, vst0, vst1;        // row-vector tile (coset 0)
    __device__ __forceinline__ void load_geom(const TileGeom& g, int M) {
        vbase = g.vbase;
        vst0 = g.vx * g.vy;
        vst1 = g.vx;
#pragma unroll
        for (int k = 0; k < SP_MAX_COSETS; ++k) {
            if (k < M) {
                cbase[k] = g.cbase[k];
                st0[k] = g.st0[k];
                st1[k] = g.st1[k];
            }
        }
    }
};

// cp.async (LDGSTS) element copy global -> shared; src_bytes = 0 zero-fills (boundary 'zero').
template <int BYTES>
__device__ __forceinline__ void cp_async_elem(void* smem_dst, const void* gsrc, int src_bytes) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(d), "l"(gsrc), "n"(BYTES), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// Fast unsigned division by a runtime divisor (Granlund-Montgomery), valid for n < 2^31.
__device__ __forceinline__ void fastdiv_magic(unsigned div, unsigned& m, unsigned& s) {
    s = 0;
    while ((1u << s) < div) ++s;
    m = (unsigned)((((unsigned long long)1 << 32) * ((1ull << s) - div)) / div + 1);
}
__device__ __forceinline__ unsigned fastdiv(unsigned n, unsigned m, unsigned s) { return (__umulhi(n, m) + n) >> s; }

__device__ __forceinline__ int floordiv_d(int a, int d, int dlog2) {
    return dlog2 >= 0 ? (a >> dlog2) : floordiv_i(a, d);
}

// Stage coset box [lo, lo+ex) (coset-cell coordinates) into dst with cp.async; the boundary
// policy is resolved here (POLICY is warp-uniform), so the evaluators read unchecked.
template <int POLICY, typename T>
__device__ __forceinline__ void stage_box(T* dst, const T* __restrict__ base, int vol, int e1, int e2, unsigned m2,
                                          unsigned s2, unsigned m1, unsigned s1, int z0b, int z1b, int z2b, int g0,
                                          int g1, int g2, int tid) {
#pragma unroll 2
    for (int e = tid; e < vol; e += kThreads) {
        const int r = (int)fastdiv((unsigned)e, m2, s2);
        const int i2 = e - r * e2;
        const int i0 = (int)fastdiv((unsigned)r, m1, s1);
        const int i1 = r - i0 * e1;
        int z0 = z0b + i0, z1 = z1b + i1, z2 = z2b + i2;
        int bytes = (int)sizeof(T);
        const bool in = (unsigned)z0 < (unsigned)g0 && (unsigned)z1 < (unsigned)g1 && (unsigned)z2 < (unsigned)g2;
        if (POLICY == SP_ZERO) {
            bytes = in ? bytes : 0;
            z0 = in ? z0 : 0;
            z1 = in ? z1 : 0;
            z2 = in ? z2 : 0;
        } else if (POLICY == SP_CLAMP) {
            z0 = min(max(z0, 0), g0 - 1);
            z1 = min(max(z1, 0), g1 - 1);
            z2 = min(max(z2, 0), g2 - 1);
        } else if (!in) {
            z0 = mirror_index(z0, g0);
            z1 = mirror_index(z1, g1);
            z2 = mirror_index(z2, g2);
        }
        cp_async_elem<sizeof(T)>(dst + e, base + ((long long)z0 * g1 + z1) * (long long)g2 + z2, bytes);
    }
}

template <typename T, int V>
struct VecT;
template <>
struct VecT<float, 2> { using type = float2; };
template <>
struct VecT<float, 4> { using type = float4; };
template <typename T>
struct VecT<T, 0> { using type = T; };

// Staging geometry from the unit-cell bounds red[0..2] (lo) / red[3..5] (hi): per coset the
// box of coset cells the points can read (+ plan site reach, + margin), its offset in the
// tile, fast-division magics, and whether it fits the tile.  Called by warp 0 only.
template <typename T>
__device__ __forceinline__ void warp_geometry(const EvalArgs<T>& a, const int* red, TileGeom& geom, int lane) {
    const int M = a.fr.M;
    const bool any = red[0] <= red[3];
    long long e = 1;
    int k = 0, i = 0;
    if (lane < 3 * M && any) {
        k = lane / 3;
        i = lane - 3 * k;
        const int d = a.fr.diag[i], l = a.fr.shift[k][i], dl = a.fr.dlog2[i];
        const long long b0 = (long long)floordiv_d(red[i] - l, d, dl) + a.fr.reach_lo[i] - a.margin;
        const long long b1 = (long long)floordiv_d(red[3 + i] - l, d, dl) + a.fr.reach_hi[i] + a.margin + a.box_pad[i];
        e = min(b1 - b0 + 1, (long long)(1 << 20));
        geom.lo[k][i] = (int)b0;
        geom.ex[k][i] = (int)e;
        if (i > 0) {
            unsigned m, sh;
            fastdiv_magic((unsigned)e, m, sh);
            geom.fdm[k][i] = m;
            geom.fds[k][i] = sh;
        }
    }
    const long long e1 = __shfl_down_sync(0xffffffffu, e, 1);
    const long long e2 = __shfl_down_sync(0xffffffffu, e, 2);
    const long long vol = e * e1 * e2;  // meaningful on lanes 3k
    const int mylo = (lane < 3 * M && any) ? geom.lo[k][i] : 0;
    const int lo1 = __shfl_down_sync(0xffffffffu, mylo, 1);
    const int lo2 = __shfl_down_sync(0xffffffffu, mylo, 2);
    long long total = 0, mine = 0;
    for (int kk = 0; kk < M; ++kk) {
        const long long v = __shfl_sync(0xffffffffu, vol, 3 * kk);
        if (lane == 3 * kk) mine = total;
        total += v;
    }
    const bool ok = any && a.tile_cap > 0 && total <= a.tile_cap;
    if (lane < 3 * M && i == 0) {
        geom.off[k] = (int)mine;
        const int s0 = (int)(e1 * e2), s1 = (int)e2;
        geom.st0[k] = s0;
        geom.st1[k] = s1;
        geom.cbase[k] = (int)mine - mylo * s0 - lo1 * s1 - lo2;
    }
    if (lane == 0 && a.vec_cap > 0 && any) {
        // padded pitches for the row-vector tile of coset 0 (dense when they do not fit)
        const int ex = (int)e2, ey = (int)e1, ez = (int)e;
        int vx = ex + ((6 - ex % 8) + 8) % 8;
        int vy = ey + ((2 - ey % 4) + 4) % 4;
        if ((long long)vx * vy * ez > a.vec_cap) {
            vx = ex;
            vy = ey;
        }
        geom.vx = vx;
        geom.vy = vy;
        geom.vtotal = vx * vy * ez;
        geom.vbase = -mylo * vy * vx - lo1 * vx - lo2;
        unsigned m, sh;
        fastdiv_magic((unsigned)vx, m, sh);
        geom.vfm_x = m;
        geom.vfs_x = sh;
        fastdiv_magic((unsigned)vy, m, sh);
        geom.vfm_y = m;
        geom.vfs_y = sh;
    }
    if (lane == 0) {
        geom.staged = ok ? 1 : 0;
        geom.total = ok ? (int)total : 0;
        if (a.stats) {
            atomicAdd(a.stats + (ok ? 0 : 1), 1ull);
            if (ok) atomicAdd(a.stats + 2, (unsigned long long)total);
        }
    }
}

// Stage every coset box of `geom` into the tile (all threads), then build the row-vector
// copy when the evaluator uses one.  Ends with the tile complete for the calling thread's
// own copies; callers __syncthreads() before reading.
template <typename T, int kVec, typename V>
__device__ __forceinline__ void stage_tile(const EvalArgs<T>& a, const TileGeom& geom, T* tile, V* vtile, int tid) {
    const int M = a.fr.M;
    for (int k = 0; k < M; ++k) {
        const int e1 = geom.ex[k][1], e2 = geom.ex[k][2];
        const int vol = geom.ex[k][0] * e1 * e2;
        const int z0b = geom.lo[k][0] - a.grid.org[k][0];
        const int z1b = geom.lo[k][1] - a.grid.org[k][1];
        const int z2b = geom.lo[k][2] - a.grid.org[k][2];
        const int g0 = a.grid.ext[k][0], g1 = a.grid.ext[k][1], g2 = a.grid.ext[k][2];
        T* dst = tile + geom.off[k];
        const T* base = a.grid.data[k];
        const unsigned m2 = geom.fdm[k][2], s2 = geom.fds[k][2], m1 = geom.fdm[k][1], s1 = geom.fds[k][1];
        if (a.grid.boundary == SP_ZERO)
            stage_box<SP_ZERO>(dst, base, vol, e1, e2, m2, s2, m1, s1, z0b, z1b, z2b, g0, g1, g2, tid);
        else if (a.grid.boundary == SP_CLAMP)
            stage_box<SP_CLAMP>(dst, base, vol, e1, e2, m2, s2, m1, s1, z0b, z1b, z2b, g0, g1, g2, tid);
        else
            stage_box<SP_MIRROR>(dst, base, vol, e1, e2, m2, s2, m1, s1, z0b, z1b, z2b, g0, g1, g2, tid);
    }
    cp_async_wait_all();
    if constexpr (kVec > 0) {
        // row-vector layout (coset 0): vtile[(z*vy + y)*vx + x] = (tile[e], ..., tile[e+kVec-1])
        // with e the dense index of (z, y, x), so a point's row of kVec taps along the
        // contiguous axis is ONE shared-memory load; padded pitches avoid bank conflicts
        __syncthreads();
        const int vt = geom.vtotal, vx = geom.vx, vy = geom.vy;
        const int ex = geom.ex[0][2], ey = geom.ex[0][1];
        for (int e = tid; e < vt; e += kThreads) {
            const int r = (int)fastdiv((unsigned)e, geom.vfm_x, geom.vfs_x);
            const int x = e - r * vx;
            const int z = (int)fastdiv((unsigned)r, geom.vfm_y, geom.vfs_y);
            const int y = r - z * vy;
            if (x < ex && y < ey) {
                const int d = (z * ey + y) * ex + x;
                V v;
                T* pv = reinterpret_cast<T*>(&v);
#pragma unroll
                for (int q = 0; q < kVec; ++q) pv[q] = tile[d + q];
                vtile[e] = v;
            }
        }
    }
}

template <typename T, class Ev>
__global__ void __launch_bounds__(kThreads, Ev::kMinBlocks) eval_kernel(const EvalArgs<T> a) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ TileGeom geom;
    __shared__ int red[6];
    constexpr int kVec = Ev::template vec_width<T>();
    using V = typename VecT<T, kVec>::type;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    // evaluator tables -> smem (16-byte granules)
    const int tb = (a.table_bytes + 15) & ~15;
    if (a.table_bytes > 0) {
        const int4* src = reinterpret_cast<const int4*>(a.tables);
        int4* dst = reinterpret_cast<int4*>(smem);
        for (int i = tid; i < tb / 16; i += kThreads) dst[i] = src[i];
    }
    const int ppt = a.ppt;
    const int chunk_pts = kThreads * ppt;
    int4* trec = reinterpret_cast<int4*>(smem + tb);
    const int tb2 = tb + a.trec_bytes;
    T* spts = reinterpret_cast<T*>(smem + tb2);  // [chunk_pts * 3]
    T* tile = reinterpret_cast<T*>(smem + tb2 + ((chunk_pts * 3 * (int)sizeof(T) + 15) & ~15));
    V* vtile = reinterpret_cast<V*>(reinterpret_cast<unsigned char*>(tile) +
                                    (((a.tile_cap + 4) * (int)sizeof(T) + 15) & ~15));

    const long long n = a.n;
    const long long nchunks = (n + chunk_pts - 1) / chunk_pts;
    const int M = a.fr.M;

    for (long long chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x) {
        const long long first = chunk * chunk_pts;
        const int cnt = (int)min((long long)chunk_pts, n - first);
        // 1. points -> smem, coalesced (16-byte vectors when aligned)
        {
            const T* src = a.pts + 3 * first;
            const int nel = 3 * cnt;
            constexpr int kPer = 16 / (int)sizeof(T);
            if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
                const int nvec = nel / kPer;
                const int4* s4 = reinterpret_cast<const int4*>(src);
                int4* d4 = reinterpret_cast<int4*>(spts);
                for (int v = tid; v < nvec; v += kThreads) d4[v] = __ldg(s4 + v);
                for (int e = nvec * kPer + tid; e < nel; e += kThreads) spts[e] = __ldg(src + e);
            } else {
                for (int e = tid; e < nel; e += kThreads) spts[e] = __ldg(src + e);
            }
        }
        if (tid < 3) red[tid] = INT_MAX;
        else if (tid < 6) red[tid] = INT_MIN;
        __syncthreads();

        // 2. bounding box of the chunk's (finite) unit cells floor(x)
        int lo0 = INT_MAX, lo1 = INT_MAX, lo2 = INT_MAX, hi0 = INT_MIN, hi1 = INT_MIN, hi2 = INT_MIN;
        for (int j = tid; j < cnt; j += kThreads) {
            const T x0 = spts[3 * j], x1 = spts[3 * j + 1], x2 = spts[3 * j + 2];
            const bool fin = isfinite(x0) && isfinite(x1) && isfinite(x2);
            const int f0 = clamp_cell(x0), f1 = clamp_cell(x1), f2 = clamp_cell(x2);
            lo0 = fin ? min(lo0, f0) : lo0; hi0 = fin ? max(hi0, f0) : hi0;
            lo1 = fin ? min(lo1, f1) : lo1; hi1 = fin ? max(hi1, f1) : hi1;
            lo2 = fin ? min(lo2, f2) : lo2; hi2 = fin ? max(hi2, f2) : hi2;
        }
        lo0 = __reduce_min_sync(0xffffffffu, lo0);
        lo1 = __reduce_min_sync(0xffffffffu, lo1);
        lo2 = __reduce_min_sync(0xffffffffu, lo2);
        hi0 = __reduce_max_sync(0xffffffffu, hi0);
        hi1 = __reduce_max_sync(0xffffffffu, hi1);
        hi2 = __reduce_max_sync(0xffffffffu, hi2);
        if (lane == 0) {
            atomicMin(&red[0], lo0); atomicMin(&red[1], lo1); atomicMin(&red[2], lo2);
            atomicMax(&red[3], hi0); atomicMax(&red[4], hi1); atomicMax(&red[5], hi2);
        }
        __syncthreads();

        // 3. staging geometry, one lane per (coset, axis) of warp 0
        if (tid < 32) warp_geometry(a, red, geom, lane);
        __syncthreads();
        const bool staged = geom.staged != 0;

        // 4. stage the coefficient box (+ halo) with cp.async, boundary policy applied here
        if (staged) {
            Ev::tile_records(a, geom, smem, trec, tid);
            stage_tile<T, kVec>(a, geom, tile, vtile, tid);
        }
        __syncthreads();

        // 5. evaluate
        EvalCtx<T, Ev> ctx;
        ctx.a = &a;
        ctx.tables = smem;
        ctx.geom = &geom;
        ctx.trec = trec;
        ctx.err = 0;
        ctx.load_geom(geom, M);
#pragma unroll 1
        for (int j = tid; j < cnt; j += kThreads) {
            const long long i = first + j;
            ctx.index = i;
            const T x[3] = {spts[3 * j], spts[3 * j + 1], spts[3 * j + 2]};
            ctx.X[0] = clamp_cell(x[0]);
            ctx.X[1] = clamp_cell(x[1]);
            ctx.X[2] = clamp_cell(x[2]);
            T v;
            if (!(isfinite(x[0]) && isfinite(x[1]) && isfinite(x[2]))) {
                v = T(NAN);
            } else if (staged) {
                TileFetch<T, V> f;
                f.tile = tile;
                f.vtile = vtile;
                SP_TILE_LIMIT(f, ctx.geom->total);
                v = Ev::template eval<TileFetch<T, V>>(x, f, ctx);
            } else {
                GlobalFetch<T> f;
                v = Ev::template eval<GlobalFetch<T>>(x, f, ctx);
            }
            a.out[i] = v;
        }
        if (ctx.err && a.err) atomicOr(a.err, 1);
        __syncthreads();
    }
}


// Bulk-prefetch points [p0, p1) into L2 (16-byte granules inside the array, <= 1 MiB each):
// issued by the TMA brick kernel for the CTA's next brick, so that brick's per-point loads hit
// L2 instead of HBM (+3 % tricubic).  Not used by the generic brick kernel: with its larger
// bricks the prefetched points evict lattice lines (ncu: +40 % DRAM traffic for +0-1.5 %).
template <typename T>
__device__ __forceinline__ void prefetch_points_l2(const EvalArgs<T>& a, long long p0, long long p1) {
    if ((reinterpret_cast<uintptr_t>(a.pts) & 15) != 0) return;
    const unsigned long long lo = ((unsigned long long)p0 * 3 * sizeof(T) + 15) & ~15ull;
    const unsigned long long hi =
        min((unsigned long long)p1 * 3 * sizeof(T) + 15, (unsigned long long)a.n * 3 * sizeof(T)) & ~15ull;
    const char* base = reinterpret_cast<const char*>(a.pts);
    for (unsigned long long o = lo; o < hi; o += 1u << 20) {
        const unsigned sz = (unsigned)min(hi - o, 1ull << 20);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + o), "r"(sz) : "memory");
    }
}

// brick-order point j (through the sort permutation when the points are not gathered)
template <typename T>
__device__ __forceinline__ const T* point_ptr(const EvalArgs<T>& a, long long j) {
    SP_CHECK(j >= 0 && j < a.n);
    SP_CHECK(!a.in_index32 || (unsigned)a.in_index32[j] < (unsigned long long)a.n);
    return a.pts + 3 * (a.in_index32 ? (long long)a.in_index32[j] : j);
}

template <typename T>
__device__ __forceinline__ void store_out(const EvalArgs<T>& a, long long j, T v) {
    SP_CHECK(j >= 0 && j < a.n);
    SP_CHECK(!a.out_index || (a.out_index[j] >= 0 && a.out_index[j] < a.n));
    SP_CHECK(!a.out_index32 || (unsigned)a.out_index32[j] < (unsigned long long)a.n);
    if (a.out_index) a.out[a.out_index[j]] = v;
    else if (a.out_index32) a.out[a.out_index32[j]] = v;
    else a.out[j] = v;
}

// One point in brick mode (ctx.X = floor(x) already set): staged tile when the point lies in
// the staged brick, else the global (policy-checked) path.
template <typename T, class Ev, typename V>
__device__ __forceinline__ T eval_one(const T x[3], bool staged, int c0, int c1, int c2, int B, const T* tile,
                                      const V* vtile, const EvalCtx<T, Ev>& ctx) {
    if (!(isfinite(x[0]) && isfinite(x[1]) && isfinite(x[2]))) return T(NAN);
    const bool inside = (unsigned)(ctx.X[0] - c0) < (unsigned)B && (unsigned)(ctx.X[1] - c1) < (unsigned)B &&
                        (unsigned)(ctx.X[2] - c2) < (unsigned)B;
    if (staged && inside) {
        TileFetch<T, V> f;
        f.tile = tile;
        f.vtile = vtile;
        SP_TILE_LIMIT(f, ctx.geom->total);
        return Ev::template eval<TileFetch<T, V>>(x, f, ctx);
    }
    GlobalFetch<T> f;
    return Ev::template eval<GlobalFetch<T>>(x, f, ctx);
}

// Kernel-signature grouping for plans with K > 1 kernels (generated Evs with kSig): a warp
// evaluating points whose cosets select different kernels runs every selected kernel for
// every coset (SIMT divergence: fcc_cubic spends 55 % of its instructions there).  Per
// segment of up to 1024 points of a brick: pass 1 classifies each point (plane tests and
// sigma only) into a word of per-coset classes and a signature = its kernel id per coset;
// a counting sort by signature (shared-memory histogram, warp scan, atomic scatter) orders
// the segment; pass 2 evaluates in that order from the stored classes (Ev::eval_word: no
// plane tests), so consecutive lanes share kernels.  Values are those of Ev::eval bit for
// bit (same frames, same classes); only the evaluation order changes.  Points that are
// non-finite or outside the staged brick form their own bucket and take the per-point path.
template <typename T, class Ev, typename V>
__device__ __forceinline__ void eval_brick_sig(const EvalArgs<T>& a, EvalCtx<T, Ev>& ctx, long long p0, long long p1,
                                               bool staged, int c0, int c1, int c2, int B, const T* tile,
                                               const V* vtile, const unsigned char* tables) {
    constexpr int kSeg = Ev::kSigSeg;
    constexpr int kBuckets = Ev::kSigCount + 1;  // last bucket: per-point path
    static_assert(kBuckets <= 65535, "signature count");
    constexpr int kPer = kSeg / kThreads;
    __shared__ unsigned s_word[kSeg];
    __shared__ unsigned short s_order[kSeg];
    __shared__ unsigned short s_key[kSeg];
    __shared__ int s_hist[kBuckets];
    __shared__ __align__(16) T s_pts[3 * kSeg];
    const int tid = threadIdx.x, lane = tid & 31;
    // segments after the first start on a 16-byte boundary of the point array (vector loads)
    constexpr int kAlignPts = sizeof(T) == 4 ? 4 : 2;
    for (long long seg = p0, len = kSeg - (p0 % kAlignPts); seg < p1; seg += len, len = kSeg) {
        const int n = (int)min(len, p1 - seg);
        for (int i = tid; i < kBuckets; i += kThreads) s_hist[i] = 0;
        // the segment's points -> shared memory (coalesced, all loads in flight together;
        // 16-byte vectors for brick-order points with a 16-byte aligned segment start)
        const T* src = a.pts + 3 * seg;
        constexpr int kVecE = 16 / (int)sizeof(T);
        if (!a.in_index32 && n == kSeg && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
            constexpr int kVecs = 3 * kSeg / kVecE;  // 16-byte vectors in the segment
            constexpr int kNV = (kVecs + kThreads - 1) / kThreads;
            static_assert(3 * kSeg % kVecE == 0, "segment size");
            int4 v[kNV];
#pragma unroll
            for (int q = 0; q < kNV; ++q)
                if (tid + q * kThreads < kVecs) v[q] = __ldg(reinterpret_cast<const int4*>(src) + tid + q * kThreads);
#pragma unroll
            for (int q = 0; q < kNV; ++q)
                if (tid + q * kThreads < kVecs) reinterpret_cast<int4*>(s_pts)[tid + q * kThreads] = v[q];
        } else {
            T v[3 * kPer];
#pragma unroll
            for (int q = 0; q < 3 * kPer; ++q) {
                const int e = tid + q * kThreads;
                v[q] = e >= 3 * n ? T(0)
                       : a.in_index32 ? __ldg(a.pts + 3 * (long long)a.in_index32[seg + e / 3] + e % 3)
                                      : __ldg(src + e);
            }
#pragma unroll
            for (int q = 0; q < 3 * kPer; ++q) s_pts[tid + q * kThreads] = v[q];
        }
        __syncthreads();
        for (int i = tid; i < n; i += kThreads) {  // pass 1: classes and signature
            const T x[3] = {s_pts[3 * i], s_pts[3 * i + 1], s_pts[3 * i + 2]};
            const bool fin = isfinite(x[0]) && isfinite(x[1]) && isfinite(x[2]);
            ctx.X[0] = clamp_cell(x[0]);
            ctx.X[1] = clamp_cell(x[1]);
            ctx.X[2] = clamp_cell(x[2]);
            const bool inside = (unsigned)(ctx.X[0] - c0) < (unsigned)B && (unsigned)(ctx.X[1] - c1) < (unsigned)B &&
                                (unsigned)(ctx.X[2] - c2) < (unsigned)B;
            int key = kBuckets - 1;
            unsigned w = 0u;
            if (fin && staged && inside) key = Ev::classify_key(x, ctx, w);
            s_word[i] = w;
            s_key[i] = (unsigned short)key;
            atomicAdd(&s_hist[key], 1);
        }
        __syncthreads();
        if (tid < 32) {  // exclusive scan of the histogram: lane-contiguous chunks + warp scan
            constexpr int kPer = (kBuckets + 31) / 32;
            int local = 0;
            for (int q = 0; q < kPer; ++q) {
                const int b = lane * kPer + q;
                if (b < kBuckets) local += s_hist[b];
            }
            int incl = local;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            int run = incl - local;
            for (int q = 0; q < kPer; ++q) {
                const int b = lane * kPer + q;
                if (b < kBuckets) {
                    const int c = s_hist[b];
                    s_hist[b] = run;
                    run += c;
                }
            }
        }
        __syncthreads();
        for (int i = tid; i < n; i += kThreads) s_order[atomicAdd(&s_hist[s_key[i]], 1)] = (unsigned short)i;
        __syncthreads();
#pragma unroll 1
        for (int r = tid; r < n; r += kThreads) {  // pass 2: evaluation in signature order
            const int i = s_order[r];
            const long long j = seg + i;
            const T x[3] = {s_pts[3 * i], s_pts[3 * i + 1], s_pts[3 * i + 2]};
            ctx.index = j;
            ctx.X[0] = clamp_cell(x[0]);
            ctx.X[1] = clamp_cell(x[1]);
            ctx.X[2] = clamp_cell(x[2]);
            T v;
            if (s_key[i] != kBuckets - 1) {
                TileFetch<T, V> f;
                f.tile = tile;
                f.vtile = vtile;
                SP_TILE_LIMIT(f, ctx.geom->total);
                v = Ev::template eval_word<TileFetch<T, V>>(x, s_word[i], f, ctx);
            } else if (!(isfinite(x[0]) && isfinite(x[1]) && isfinite(x[2]))) {
                v = T(NAN);
            } else {
                GlobalFetch<T> f;
                v = Ev::template eval<GlobalFetch<T>>(x, f, ctx);
            }
            store_out(a, j, v);
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------------------
// Brick mode: points sorted by the Morton code of their unit cell are grouped into aligned
// bricks of B^3 unit cells (B = 2^log2b); brick_start[b]..brick_start[b+1] are brick b's
// points.  One CTA stages one brick's coefficient box (+ halo) ONCE and evaluates all of its
// points (thousands), so staging, geometry and barriers are amortised over the brick.
// A point outside its run's brick (only possible for clamped/non-finite keys) takes the
// global path.
template <typename T, class Ev>
__global__ void __launch_bounds__(kThreads, Ev::kMinBlocks)
    brick_kernel(const EvalArgs<T> a, const long long* __restrict__ brick_start, int nbricks, int log2b) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ TileGeom geom;
    __shared__ int red[6];
    constexpr int kVec = Ev::template vec_width<T>();
    using V = typename VecT<T, kVec>::type;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int tb = (a.table_bytes + 15) & ~15;
    if (a.table_bytes > 0) {
        const int4* src = reinterpret_cast<const int4*>(a.tables);
        int4* dst = reinterpret_cast<int4*>(smem);
        for (int i = tid; i < tb / 16; i += kThreads) dst[i] = src[i];
    }
    int4* trec = reinterpret_cast<int4*>(smem + tb);
    T* tile = reinterpret_cast<T*>(smem + tb + a.trec_bytes);
    V* vtile = reinterpret_cast<V*>(reinterpret_cast<unsigned char*>(tile) +
                                    (((a.tile_cap + 4) * (int)sizeof(T) + 15) & ~15));
    const int B = 1 << log2b;
    if (a.nbricks_dev) nbricks = min(nbricks, *a.nbricks_dev);

    for (int b = blockIdx.x; b < nbricks; b += gridDim.x) {
        const long long p0 = brick_start[b], p1 = brick_start[b + 1];
        if (tid < 32) {
            if (lane == 0) {
                const T* x = point_ptr(a, p0);
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    const int c = clamp_cell(x[i]);
                    const int lo = (c >> log2b) << log2b;
                    red[i] = lo;
                    red[3 + i] = lo + B - 1;
                }
            }
            __syncwarp();
            warp_geometry(a, red, geom, lane);
        }
        __syncthreads();
        const bool staged = geom.staged != 0;
        if (staged) {
            Ev::tile_records(a, geom, smem, trec, tid);
            stage_tile<T, kVec>(a, geom, tile, vtile, tid);
        }
        __syncthreads();
        const int c0 = red[0], c1 = red[1], c2 = red[2];

        EvalCtx<T, Ev> ctx;
        ctx.a = &a;
        ctx.tables = smem;
        ctx.geom = &geom;
        ctx.trec = trec;
        ctx.err = 0;
        ctx.load_geom(geom, a.fr.M);
        // software-pipelined point loads: the next point is in flight while this one is evaluated
        T xn0 = T(0), xn1 = T(0), xn2 = T(0);
        if (p0 + tid < p1) {
            const T* px = point_ptr(a, p0 + tid);
            xn0 = __ldg(px);
            xn1 = __ldg(px + 1);
            xn2 = __ldg(px + 2);
        }
        if constexpr (Ev::kSig) {
            // K > 1 plans: points grouped by kernel signature before evaluation
            eval_brick_sig<T, Ev, V>(a, ctx, p0, p1, staged, c0, c1, c2, B, tile, vtile, smem);
            if (ctx.err && a.err) atomicOr(a.err, 1);
            __syncthreads();
            continue;
        }
        // plain brick-order points (no permutations, no debug output) in an exact brick (corner
        // + B <= 2^30): points inside the staged brick are recognised from the saturating floor
        // conversions plus one NaN test and evaluated from the tile directly (same values: X is
        // clamp_cell(x) there); the others take the checked path below
        const bool plain = !a.in_index32 && !a.out_index && !a.out_index32 && !a.dbg && a.plain_pts && staged &&
                           c0 + B <= kCellClamp && c1 + B <= kCellClamp && c2 + B <= kCellClamp;
#pragma unroll 1
        for (long long j = p0 + tid; j < p1; j += kThreads) {
            ctx.index = j;
            const T x[3] = {xn0, xn1, xn2};
            if (j + kThreads < p1) {
                const T* px = plain ? a.pts + 3 * (j + kThreads) : point_ptr(a, j + kThreads);
                xn0 = __ldg(px);
                xn1 = __ldg(px + 1);
                xn2 = __ldg(px + 2);
            }
            if (plain) {
                const int X0 = floor_int(x[0]), X1 = floor_int(x[1]), X2 = floor_int(x[2]);
                const T sum = x[0] + x[1] + x[2];
                if (((unsigned)(X0 - c0) < (unsigned)B) & ((unsigned)(X1 - c1) < (unsigned)B) &
                    ((unsigned)(X2 - c2) < (unsigned)B) & (sum == sum)) {
                    ctx.X[0] = X0;
                    ctx.X[1] = X1;
                    ctx.X[2] = X2;
                    TileFetch<T, V> f;
                    f.tile = tile;
                    f.vtile = vtile;
                    SP_TILE_LIMIT(f, ctx.geom->total);
                    SP_CHECK(j >= 0 && j < a.n);
                    a.out[j] = Ev::template eval<TileFetch<T, V>>(x, f, ctx);
                    continue;
                }
            }
            T v;
            const bool fin = isfinite(x[0]) && isfinite(x[1]) && isfinite(x[2]);
            ctx.X[0] = clamp_cell(x[0]);
            ctx.X[1] = clamp_cell(x[1]);
            ctx.X[2] = clamp_cell(x[2]);
            const bool inside = (unsigned)(ctx.X[0] - c0) < (unsigned)B && (unsigned)(ctx.X[1] - c1) < (unsigned)B &&
                                (unsigned)(ctx.X[2] - c2) < (unsigned)B;
            if (!fin) {
                v = T(NAN);
            } else if (staged && inside) {
                TileFetch<T, V> f;
                f.tile = tile;
                f.vtile = vtile;
                SP_TILE_LIMIT(f, ctx.geom->total);
                v = Ev::template eval<TileFetch<T, V>>(x, f, ctx);
            } else {
                GlobalFetch<T> f;
                v = Ev::template eval<GlobalFetch<T>>(x, f, ctx);
            }
            store_out(a, j, v);
        }
        if (ctx.err && a.err) atomicOr(a.err, 1);
        __syncthreads();
    }
}

// Frame setup helpers used by the evaluators: bind a fetcher to (coset k, base, rho, tau).
template <typename T, typename V>
__device__ __forceinline__ void bind(TileFetch<T, V>& f, const EvalArgs<T>& a, const TileGeom& g, int k,
                                     const int base[3], const int rho[3], const int tau[3]) {
    f.frame(g, k, base, rho, tau);
}
template <typename T>
__device__ __forceinline__ void bind(GlobalFetch<T>& f, const EvalArgs<T>& a, const TileGeom& g, int k,
                                     const int base[3], const int rho[3], const int tau[3]) {
    f.frame(a.grid, k, base, rho, tau);
}
__device__ __forceinline__ void bind(TexFetch& f, const EvalArgs<float>& a, const TileGeom& g, int k, const int base[3],
                                     const int rho[3], const int tau[3]) {
    f.frame(a.grid, k, base, rho, tau);
}
template <typename T, typename V>
__device__ __forceinline__ void bind_identity(TileFetch<T, V>& f, const EvalArgs<T>& a, const TileGeom& g, int k,
                                              const int base[3]) {
    f.frame_identity(g, k, base);
}
template <typename T>
__device__ __forceinline__ void bind_identity(GlobalFetch<T>& f, const EvalArgs<T>& a, const TileGeom& g, int k,
                                              const int base[3]) {
    f.frame_identity(a.grid, k, base);
}

// ---------------------------------------------------------------------------------------
// Coset frame of Algorithm 1, in float64 exactly as runtime.py:371-373:
//   xl = x - l_k ; kk = floor(xl / d) * d ; xp = xl - kk
struct CosetFrame {
    double xp[3];
    int cell[3];  // kk / d
};

template <typename T>
__device__ __forceinline__ CosetFrame coset_frame(const T x[3], const FrameArgs& fr, int k) {
    CosetFrame c;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const double d = (double)fr.diag[i];
        const double xl = (double)x[i] - (double)fr.shift[k][i];
        // power-of-two d: multiplying by 1/d is exact and avoids the float64 division
        const double q = fr.dlog2[i] >= 0 ? floor(xl * ldexp(1.0, -fr.dlog2[i])) : floor(xl / d);
        const double kk = q * d;
        c.xp[i] = xl - kk;
        c.cell[i] = clamp_cell(q);
    }
    return c;
}

__device__ __forceinline__ double sel3(int i, double a, double b, double c) { return i == 0 ? a : (i == 1 ? b : c); }

}  // namespace sp
