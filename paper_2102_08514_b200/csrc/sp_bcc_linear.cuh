// sp_bcc_linear.cuh — closed-form brick kernel for the BCC linear box spline (bcc_linear_rd).
//
// The reference evaluates bcc_linear_rd (4 body diagonals on BCC, scale |det L| = 4) as
// Algorithm 1 (runtime.py:363-408): per coset the coset frame, six plane
// tests, sigma, a class transform (signed permutation) and two affine weight polynomials
// of one 2-site fetch group.  The spline is the linear rhombic-dodecahedron box spline
// (Table 1, 4 lookups), i.e. barycentric interpolation on the BCC Delaunay
// tetrahedra, and the whole per-class machinery folds into a few warp-uniform min/max
// operations (the paper's symmetry folding, done arithmetically):
//
//   y = x - (1,1,1)                  (non-centred support sum [0, xi])
//   E = 2 rint(y/2)                  nearest even site (coset 0), d = y - E in [-1,1]^3
//   s = sign(d), w = |d|; a = argmax w, b = argmin w, m = the middle axis
//   f = (1 - (w_a+w_m)/2) c[E] + (w_a-w_m)/2 c[E + 2 s_a e_a]
//     + (w_m+w_b)/2 c[E + s] + (w_m-w_b)/2 c[E + s - 2 s_b e_b]          (odd sites: coset 1)
//
// Every reflection / permutation is a select on lane-local data, so all lanes run the same
// instruction stream (no sigma table, no class records, no kernel switch).  The formula is the
// plan's function exactly (tests/test_codegen_affine.py checks it against the reference
// outputs in float64 to ~1e-16); ties between tetrahedra pick a neighbour with the same
// (continuous) value.  Points are read four per thread (3 x 16-byte loads) and the results
// written with one 16-byte store.  Non-finite points give NaN (as every evaluator); points
// outside the fast domain (|x| >= kFast) or outside their run's brick take the same formula in
// float64 with policy-checked global reads.
#pragma once

#include "sp_common.cuh"

namespace sp {

template <typename T>
struct BccTetTraits;
template <>
struct BccTetTraits<float> {
    static constexpr float kFast = 4194304.0f;  // 2^22: x - 1 and the cell indices are exact
};
template <>
struct BccTetTraits<double> {
    static constexpr double kFast = 1073741824.0;  // 2^30: cell indices fit int
};

// Tetrahedron selection, shared by every path (same operations -> same bits everywhere).
template <typename R>
struct TetSel {
    int e0, e1, e2;     // coset-0 cell of the nearest even site E = 2 e
    bool n0, n1, n2;    // d_i < 0 (s_i = -1)
    bool c01, c02, c12; // |d_0| >= |d_1| etc.
    R wa, wb, wm;       // largest, smallest, middle |d_i|
};

template <typename R>
__device__ __forceinline__ TetSel<R> tet_select(R y0, R y1, R y2) {
    TetSel<R> t;
    const R f0 = rint(y0 * R(0.5)), f1 = rint(y1 * R(0.5)), f2 = rint(y2 * R(0.5));
    const R d0 = fma(f0, R(-2), y0), d1 = fma(f1, R(-2), y1), d2 = fma(f2, R(-2), y2);
    t.e0 = (int)f0;
    t.e1 = (int)f1;
    t.e2 = (int)f2;
    t.n0 = d0 < R(0);
    t.n1 = d1 < R(0);
    t.n2 = d2 < R(0);
    const R w0 = fabs(d0), w1 = fabs(d1), w2 = fabs(d2);
    t.c01 = w0 >= w1;
    t.c02 = w0 >= w2;
    t.c12 = w1 >= w2;
    const R mx01 = fmax(w0, w1), mn01 = fmin(w0, w1);
    t.wa = fmax(mx01, w2);
    t.wb = fmin(mn01, w2);
    t.wm = fmax(mn01, fmin(mx01, w2));
    return t;
}

// axis (0/1/2) of the largest / smallest |d| (distinct, also at ties)
template <typename R>
__device__ __forceinline__ int tet_axis_a(const TetSel<R>& t) { return t.c01 ? (t.c02 ? 0 : 2) : (t.c12 ? 1 : 2); }
template <typename R>
__device__ __forceinline__ int tet_axis_b(const TetSel<R>& t) { return t.c01 ? (t.c12 ? 2 : 1) : (t.c02 ? 2 : 0); }

// sites E, E + 2 s_a e_a (coset 0) and E + s, E + s - 2 s_b e_b (coset 1)
template <typename R>
__device__ __forceinline__ R tet_combine(const TetSel<R>& t, R cE, R cA, R cO, R cB) {
    R acc = (R(2) - t.wa - t.wm) * cE;
    acc = fma(t.wa - t.wm, cA, acc);
    acc = fma(t.wm + t.wb, cO, acc);
    acc = fma(t.wm - t.wb, cB, acc);
    return acc * R(0.5);
}

// One point from the staged brick tile (selection already made): both coset boxes have
// strides (E*E, E, 1), coset 1 at offset E^3; `base` = tile index of coset-0 cell (0,0,0).
template <int E, typename T>
__device__ __forceinline__ T bcc_tet_tile(const TetSel<T>& t, const T* __restrict__ tile, int base) {
    constexpr int S0 = E * E, S1 = E, ODD = E * E * E;
    const int ss0 = t.n0 ? -S0 : S0, ss1 = t.n1 ? -S1 : S1, ss2 = t.n2 ? -1 : 1;
    const int sa = t.c01 ? (t.c02 ? ss0 : ss2) : (t.c12 ? ss1 : ss2);
    const int sb = t.c01 ? (t.c12 ? ss2 : ss1) : (t.c02 ? ss2 : ss0);
    const int iE = base + t.e0 * S0 + t.e1 * S1 + t.e2;
    const int iO = iE + ODD - ((t.n0 ? S0 : 0) + (t.n1 ? S1 : 0) + (t.n2 ? 1 : 0));
    // E + s - 2 s_b e_b leaves the spline's support only when its weight w_m - w_b is 0
    // (all |d_i| = 1): read E + s instead (tet_guard_b), so the box is exactly the support
    const int iB = t.wm > t.wb ? iO - sb : iO;
    SP_CHECK(iE >= 0 && iE + sa >= 0 && iE + sa < ODD && iO < 2 * ODD && iB >= ODD && iB < 2 * ODD);
    return tet_combine<T>(t, tile[iE], tile[iE + sa], tile[iO], tile[iB]);
}

// Stage an E^3 box of one coset (coset-cell origin z0b.. as array indices) with the policy
// resolved per element; E is a compile-time constant (divisions fold to multiply-shifts).
template <int POLICY, int E, typename T>
__device__ __forceinline__ void stage_cube(T* dst, const T* __restrict__ base, int z0b, int z1b, int z2b, int g0,
                                           int g1, int g2, int tid) {
    constexpr int VOL = E * E * E;
#pragma unroll 2
    for (int e = tid; e < VOL; e += kThreads) {
        const int i0 = e / (E * E);
        const int r = e - i0 * (E * E);
        const int i1 = r / E;
        const int i2 = r - i1 * E;
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

// Any point through two coset fetchers (TileFetch / GlobalFetch, bound per coset by `bindk`).
template <typename R, typename T, class F, class Bind>
__device__ __forceinline__ R bcc_tet_fetch(R y0, R y1, R y2, F& f, Bind bindk) {
    const TetSel<R> t = tet_select<R>(y0, y1, y2);
    const int ia = tet_axis_a(t), ib = tet_axis_b(t);
    const int s0 = t.n0 ? -1 : 1, s1 = t.n1 ? -1 : 1, s2 = t.n2 ? -1 : 1;
    const int e[3] = {t.e0, t.e1, t.e2};
    bindk(f, 0, e);
    const R cE = (R)f.get(0, 0, 0);
    const R cA = (R)f.get(ia == 0 ? s0 : 0, ia == 1 ? s1 : 0, ia == 2 ? s2 : 0);
    const int o[3] = {t.e0 - (int)t.n0, t.e1 - (int)t.n1, t.e2 - (int)t.n2};
    bindk(f, 1, o);
    const R cO = (R)f.get(0, 0, 0);
    const bool gb = t.wm > t.wb;  // same guard as bcc_tet_tile
    const R cB = (R)f.get(gb && ib == 0 ? -s0 : 0, gb && ib == 1 ? -s1 : 0, gb && ib == 2 ? -s2 : 0);
    return tet_combine<R>(t, cE, cA, cO, cB);
}

// Slow path of the brick kernel: policy-checked global reads; R = T inside the fast domain
// (the same arithmetic as the tile path and BccTetEval), float64 beyond it.
template <typename R, typename T>
__device__ __forceinline__ T bcc_tet_global(const EvalArgs<T>& a, R y0, R y1, R y2) {
    GlobalFetch<T> f;
    return (T)bcc_tet_fetch<R, T>(y0, y1, y2, f, [&](GlobalFetch<T>& ff, int k, const int* base) {
        ff.frame_identity(a.grid, k, base);
    });
}

// The same function as an evaluator for the generic drivers (chunk kernel, indirect brick
// kernel): identical values, bit for bit, to bcc_tet_brick_kernel.  Reads coset cells up to
// 2 around floor((x - l)/2) (sp_plan_create widens the plan's reach for it).
template <typename T>
struct BccTetEval {
    static constexpr int kMinBlocks = 4;
    static constexpr bool kSig = false;
    static constexpr int kSigCount = 1;
    template <typename U>
    static constexpr int vec_width() {
        return 0;
    }
    __device__ static void tile_records(const EvalArgs<T>&, const TileGeom&, const unsigned char*, int4*, int) {}
    template <class Ctx>
    __device__ __forceinline__ static unsigned classify_word(const T*, const Ctx&) { return 0u; }
    __device__ __forceinline__ static int signature(unsigned, const unsigned char*) { return 0; }
    template <class F, class Ctx>
    __device__ __forceinline__ static T eval_word(const T x[3], unsigned, F& f, const Ctx& ctx) {
        return eval<F, Ctx>(x, f, ctx);
    }
    template <class F, class Ctx>
    __device__ __forceinline__ static T eval(const T x[3], F& f, const Ctx& ctx) {
        constexpr T kF = BccTetTraits<T>::kFast;
        auto bindk = [&](F& ff, int k, const int* base) { bind_identity(ff, *ctx.a, *ctx.geom, k, base); };
        if (fabs(x[0]) < kF && fabs(x[1]) < kF && fabs(x[2]) < kF)
            return bcc_tet_fetch<T, T>(x[0] - T(1), x[1] - T(1), x[2] - T(1), f, bindk);
        return (T)bcc_tet_fetch<double, T>((double)x[0] - 1.0, (double)x[1] - 1.0, (double)x[2] - 1.0, f, bindk);
    }
};

// Persistent CTAs over bricks (grid-strided).  Box per coset: coset cells [c/2 - 1, c/2 + B/2]
// per axis (E = B/2 + 2) — exactly the spline's support for unit cells [c, c+B) (with the
// zero-weight guard of bcc_tet_tile) — same shape for both cosets, staged with the grid's
// boundary policy; optionally double-buffered (the next brick's boxes in flight while the
// current one is evaluated).  Points: quads of 4 consecutive brick-order points per thread
// (3 x 16-byte loads; PF: the next quad's loads issued before the current one is evaluated).
// A point takes the tile path iff c <= x < c + B on every axis (false for NaN) and the brick
// lies inside the fast domain (|x| < kFast); others take the global path.
template <typename T, int L2B, bool PF = true, int MINB = (sizeof(T) == 4 ? 3 : 2), bool DB = false>
__global__ void __launch_bounds__(kThreads, MINB)
    bcc_tet_brick_kernel(const EvalArgs<T> a, const long long* __restrict__ brick_start, int nbricks) {
    constexpr int B = 1 << L2B;
    constexpr int E = B / 2 + 2;
    constexpr int VOL = E * E * E;
    constexpr T kF = BccTetTraits<T>::kFast;
    extern __shared__ __align__(16) unsigned char smem[];
    T* const tiles = reinterpret_cast<T*>(smem);  // [1 or 2][2 * VOL]
    const int tid = threadIdx.x;
    if (a.nbricks_dev) nbricks = min(nbricks, *a.nbricks_dev);

    auto corner_of = [&](int b, int c[3]) {  // uniform loads (broadcast)
        const T* x = a.pts + 3 * brick_start[b];
#pragma unroll
        for (int i = 0; i < 3; ++i) c[i] = (clamp_cell(x[i]) >> L2B) << L2B;
    };
    auto stage = [&](int b, T* tile) {
        int c[3];
        corner_of(b, c);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int z0b = (c[0] >> 1) - 1 - a.grid.org[k][0];
            const int z1b = (c[1] >> 1) - 1 - a.grid.org[k][1];
            const int z2b = (c[2] >> 1) - 1 - a.grid.org[k][2];
            const int g0 = a.grid.ext[k][0], g1 = a.grid.ext[k][1], g2 = a.grid.ext[k][2];
            if (a.grid.boundary == SP_ZERO)
                stage_cube<SP_ZERO, E>(tile + k * VOL, a.grid.data[k], z0b, z1b, z2b, g0, g1, g2, tid);
            else if (a.grid.boundary == SP_CLAMP)
                stage_cube<SP_CLAMP, E>(tile + k * VOL, a.grid.data[k], z0b, z1b, z2b, g0, g1, g2, tid);
            else
                stage_cube<SP_MIRROR, E>(tile + k * VOL, a.grid.data[k], z0b, z1b, z2b, g0, g1, g2, tid);
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    auto load_quad = [&](long long j0, T xs[12]) {
        if (j0 + 4 <= a.n) {
            if constexpr (sizeof(T) == 4) {
                const float4* src = reinterpret_cast<const float4*>(a.pts + 3 * j0);
#pragma unroll
                for (int v = 0; v < 3; ++v) {
                    const float4 t = __ldg(src + v);
                    xs[4 * v] = t.x;
                    xs[4 * v + 1] = t.y;
                    xs[4 * v + 2] = t.z;
                    xs[4 * v + 3] = t.w;
                }
            } else {
                const double2* src = reinterpret_cast<const double2*>(a.pts + 3 * j0);
#pragma unroll
                for (int v = 0; v < 6; ++v) {
                    const double2 t = __ldg(src + v);
                    xs[2 * v] = t.x;
                    xs[2 * v + 1] = t.y;
                }
            }
        } else {
#pragma unroll
            for (int e = 0; e < 12; ++e) xs[e] = j0 + e / 3 < a.n ? __ldg(a.pts + 3 * j0 + e) : T(0);
        }
    };

    if (DB && (int)blockIdx.x < nbricks) stage(blockIdx.x, tiles);
    int it = 0;
    for (int b = blockIdx.x; b < nbricks; b += gridDim.x, ++it) {
        T* tile = tiles + (DB ? (it & 1) * 2 * VOL : 0);
        const int nb = b + gridDim.x;
        if (!DB) {
            stage(b, tile);
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        } else if (nb < nbricks) {
            stage(nb, tiles + ((it + 1) & 1) * 2 * VOL);  // overlaps this brick's evaluation
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncthreads();
        int c[3];
        corner_of(b, c);
        const long long p0 = brick_start[b], p1 = brick_start[b + 1];
        // tile index of coset-0 cell (0,0,0)
        const int lo0 = (c[0] >> 1) - 1, lo1 = (c[1] >> 1) - 1, lo2 = (c[2] >> 1) - 1;
        const int base = -(lo0 * E * E + lo1 * E + lo2);
        // tile path: c <= x < c + B per axis, brick inside the fast domain
        const bool dom = (T)c[0] > -kF && (T)c[1] > -kF && (T)c[2] > -kF && (T)(c[0] + B) < kF &&
                         (T)(c[1] + B) < kF && (T)(c[2] + B) < kF;
        const T blo0 = dom ? (T)c[0] : kF, blo1 = (T)c[1], blo2 = (T)c[2];  // dom false: no point passes
        const T bhi0 = (T)(c[0] + B), bhi1 = (T)(c[1] + B), bhi2 = (T)(c[2] + B);
        const long long q0 = p0 >> 2, q1 = (p1 + 3) >> 2;
        T xn[12];
        if (PF && q0 + tid < q1) load_quad((q0 + tid) << 2, xn);
#pragma unroll 1
        for (long long q = q0 + tid; q < q1; q += kThreads) {
            const long long j0 = q << 2;
            T xs[12];
            if constexpr (PF) {
#pragma unroll
                for (int e = 0; e < 12; ++e) xs[e] = xn[e];
                if (q + kThreads < q1) load_quad((q + kThreads) << 2, xn);
            } else {
                load_quad(j0, xs);
            }
            T r[4];
            unsigned slow = 0u;  // points for the global path (outside the brick, far or non-finite)
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const T x0 = xs[3 * u], x1 = xs[3 * u + 1], x2 = xs[3 * u + 2];
                const bool fast = x0 >= blo0 && x0 < bhi0 && x1 >= blo1 && x1 < bhi1 && x2 >= blo2 && x2 < bhi2;
                T v = T(0);
                if (fast) v = bcc_tet_tile<E, T>(tet_select<T>(x0 - T(1), x1 - T(1), x2 - T(1)), tile, base);
                r[u] = v;
                slow |= fast ? 0u : (1u << u);
            }
#pragma unroll 1
            while (slow) {  // rare: one call site, registers selected (no local-memory arrays)
                const int u = __ffs(slow) - 1;
                slow &= slow - 1;
                auto pick = [&](int o) { return u == 0 ? xs[o] : u == 1 ? xs[3 + o] : u == 2 ? xs[6 + o] : xs[9 + o]; };
                const T x0 = pick(0), x1 = pick(1), x2 = pick(2);
                T v = T(NAN);
                if (fabs(x0) < kF && fabs(x1) < kF && fabs(x2) < kF)
                    v = bcc_tet_global<T, T>(a, x0 - T(1), x1 - T(1), x2 - T(1));
                else if (isfinite(x0) && isfinite(x1) && isfinite(x2))
                    v = bcc_tet_global<double, T>(a, (double)x0 - 1.0, (double)x1 - 1.0, (double)x2 - 1.0);
                r[0] = u == 0 ? v : r[0];
                r[1] = u == 1 ? v : r[1];
                r[2] = u == 2 ? v : r[2];
                r[3] = u == 3 ? v : r[3];
            }
            if (j0 >= p0 && j0 + 4 <= p1) {
                if constexpr (sizeof(T) == 4) {
                    *reinterpret_cast<float4*>(a.out + j0) = make_float4(r[0], r[1], r[2], r[3]);
                } else {
                    reinterpret_cast<double2*>(a.out + j0)[0] = make_double2(r[0], r[1]);
                    reinterpret_cast<double2*>(a.out + j0)[1] = make_double2(r[2], r[3]);
                }
            } else {
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (j0 + u >= p0 && j0 + u < p1) a.out[j0 + u] = r[u];
            }
        }
        __syncthreads();  // the tile is restaged for the next brick
    }
}


// ---------------------------------------------------------------------------------------------
// Leaner tile path (bcc_tet_brick_kernel_v2).  Same values, bit for bit, as bcc_tet_tile:
//  * rint(y/2) by the magic-number add: t = fma(y, 1/2, 1.5*2^p) rounds y/2 (exact) to the
//    nearest integer, ties to even (the magic is even), so f = t - magic is rint(y/2) and the
//    low mantissa bits of t hold that integer: no FRND / F2I on the conversion pipe;
//  * tile reads through one 32-bit shared-window address (no generic->shared conversion per
//    point), byte offsets folded into the strides;
//  * the brick test is made once per quad of points: four straight-line evaluations when all
//    four lie in the brick (always, for brick runs of finite in-range points);
//  * points in groups of three 16-byte vectors (4 float32 / 2 float64 points), two groups in
//    flight per thread in two register sets used alternately (no copies).
template <typename T>
struct TetMagic;
template <>
struct TetMagic<float> {
    static constexpr float kM = 12582912.0f;                // 1.5 * 2^23
    static constexpr unsigned kBits = 0x4B400000u;          // its bit pattern: k = bits(t) - kBits
    __device__ static __forceinline__ unsigned bits(float t) { return __float_as_uint(t); }
};
template <>
struct TetMagic<double> {
    static constexpr double kM = 6755399441055744.0;        // 1.5 * 2^52: low word of bits(t) is k
    static constexpr unsigned kBits = 0u;
    __device__ static __forceinline__ unsigned bits(double t) { return (unsigned)__double2loint(t); }
};

template <typename T>
__device__ __forceinline__ T lds_at(unsigned addr);
template <>
__device__ __forceinline__ float lds_at<float>(unsigned addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}
template <>
__device__ __forceinline__ double lds_at<double>(unsigned addr) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
    return v;
}

// One in-brick point from the staged tile; `sbias` = shared address of the tile element of
// coset-0 cell (0,0,0) minus kBits * (S0 + S1 + S2) bytes (so the raw magic bits index it).
template <int E, typename T>
__device__ __forceinline__ T bcc_tet_tile_v2(T x0, T x1, T x2, unsigned sbias, unsigned sbase) {
    constexpr T kM = TetMagic<T>::kM;
    constexpr int SZ = (int)sizeof(T);
    constexpr int S0 = E * E * SZ, S1 = E * SZ, S2 = SZ, ODD = E * E * E * SZ;
    const T y0 = x0 - T(1), y1 = x1 - T(1), y2 = x2 - T(1);
    const T t0 = fma(y0, T(0.5), kM), t1 = fma(y1, T(0.5), kM), t2 = fma(y2, T(0.5), kM);
    const T d0 = fma(t0 - kM, T(-2), y0), d1 = fma(t1 - kM, T(-2), y1), d2 = fma(t2 - kM, T(-2), y2);
    TetSel<T> t;
    t.n0 = d0 < T(0);
    t.n1 = d1 < T(0);
    t.n2 = d2 < T(0);
    const T w0 = fabs(d0), w1 = fabs(d1), w2 = fabs(d2);
    t.c01 = w0 >= w1;
    t.c02 = w0 >= w2;
    t.c12 = w1 >= w2;
    const T mx01 = fmax(w0, w1), mn01 = fmin(w0, w1);
    t.wa = fmax(mx01, w2);
    t.wb = fmin(mn01, w2);
    t.wm = fmax(mn01, fmin(mx01, w2));
    const int ss0 = t.n0 ? -S0 : S0, ss1 = t.n1 ? -S1 : S1, ss2 = t.n2 ? -S2 : S2;
    const int sa = t.c01 ? (t.c02 ? ss0 : ss2) : (t.c12 ? ss1 : ss2);
    const int sb = t.c01 ? (t.c12 ? ss2 : ss1) : (t.c02 ? ss2 : ss0);
    const unsigned aE = sbias + TetMagic<T>::bits(t0) * (unsigned)S0 + TetMagic<T>::bits(t1) * (unsigned)S1 +
                        TetMagic<T>::bits(t2) * (unsigned)S2;
    const unsigned aO = aE + (unsigned)ODD - (unsigned)((t.n0 ? S0 : 0) + (t.n1 ? S1 : 0) + (t.n2 ? S2 : 0));
    const unsigned aB = t.wm > t.wb ? aO - (unsigned)sb : aO;  // tet_guard_b (see bcc_tet_tile)
    SP_CHECK(aE - sbase < (unsigned)ODD && aE + sa - sbase < (unsigned)ODD && aO - sbase - ODD < (unsigned)ODD &&
             aB - sbase - ODD < (unsigned)ODD);
    (void)sbase;
    return tet_combine<T>(t, lds_at<T>(aE), lds_at<T>(aE + (unsigned)sa), lds_at<T>(aO), lds_at<T>(aB));
}

template <typename T, int L2B, int MINB = (sizeof(T) == 4 ? 3 : 2)>
__global__ void __launch_bounds__(kThreads, MINB)
    bcc_tet_brick_kernel_v2(const EvalArgs<T> a, const long long* __restrict__ brick_start, int nbricks) {
    constexpr int B = 1 << L2B;
    constexpr int E = B / 2 + 2;
    constexpr int VOL = E * E * E;
    constexpr int SZ = (int)sizeof(T);
    constexpr T kF = BccTetTraits<T>::kFast;
    extern __shared__ __align__(16) unsigned char smem[];
    T* const tile = reinterpret_cast<T*>(smem);  // [2 * VOL]: coset 0 | coset 1
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(tile);
    const int tid = threadIdx.x;
    if (a.nbricks_dev) nbricks = min(nbricks, *a.nbricks_dev);

    // a group = the G points of three 16-byte vectors (4 float32 / 2 float64 points)
    constexpr int G = 16 / SZ, LG = SZ == 4 ? 2 : 1;
    auto load_group = [&](long long j0, T xs[3 * G]) {
        if (j0 + G <= a.n) {
            if constexpr (sizeof(T) == 4) {
                const float4* src = reinterpret_cast<const float4*>(a.pts + 3 * j0);
#pragma unroll
                for (int v = 0; v < 3; ++v) {
                    const float4 t = __ldg(src + v);
                    xs[4 * v] = t.x;
                    xs[4 * v + 1] = t.y;
                    xs[4 * v + 2] = t.z;
                    xs[4 * v + 3] = t.w;
                }
            } else {
                const double2* src = reinterpret_cast<const double2*>(a.pts + 3 * j0);
#pragma unroll
                for (int v = 0; v < 3; ++v) {
                    const double2 t = __ldg(src + v);
                    xs[2 * v] = t.x;
                    xs[2 * v + 1] = t.y;
                }
            }
        } else {
#pragma unroll
            for (int e = 0; e < 3 * G; ++e) xs[e] = j0 + e / 3 < a.n ? __ldg(a.pts + 3 * j0 + e) : T(0);
        }
    };

    for (int b = blockIdx.x; b < nbricks; b += gridDim.x) {
        int c[3];
        {
            const T* x = a.pts + 3 * brick_start[b];  // uniform loads (broadcast)
#pragma unroll
            for (int i = 0; i < 3; ++i) c[i] = (clamp_cell(x[i]) >> L2B) << L2B;
        }
        const long long p0 = brick_start[b], p1 = brick_start[b + 1];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int z0b = (c[0] >> 1) - 1 - a.grid.org[k][0];
            const int z1b = (c[1] >> 1) - 1 - a.grid.org[k][1];
            const int z2b = (c[2] >> 1) - 1 - a.grid.org[k][2];
            const int g0 = a.grid.ext[k][0], g1 = a.grid.ext[k][1], g2 = a.grid.ext[k][2];
            if (a.grid.boundary == SP_ZERO)
                stage_cube<SP_ZERO, E>(tile + k * VOL, a.grid.data[k], z0b, z1b, z2b, g0, g1, g2, tid);
            else if (a.grid.boundary == SP_CLAMP)
                stage_cube<SP_CLAMP, E>(tile + k * VOL, a.grid.data[k], z0b, z1b, z2b, g0, g1, g2, tid);
            else
                stage_cube<SP_MIRROR, E>(tile + k * VOL, a.grid.data[k], z0b, z1b, z2b, g0, g1, g2, tid);
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
        const long long q0 = p0 >> LG, q1 = (p1 + G - 1) >> LG;
        // two groups in flight per thread, ping-ponged between two register sets (no copies);
        // the first one is loaded while the tile lands
        T xa[3 * G], xb[3 * G];
        long long q = q0 + tid;
        if (q < q1) load_group(q << LG, xa);
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        __syncthreads();
        const int lo0 = (c[0] >> 1) - 1, lo1 = (c[1] >> 1) - 1, lo2 = (c[2] >> 1) - 1;
        const int base = -(lo0 * E * E + lo1 * E + lo2);  // tile index of coset-0 cell (0,0,0)
        const unsigned sbias = sbase + (unsigned)(base * SZ) -
                               TetMagic<T>::kBits * (unsigned)(E * E * SZ + E * SZ + SZ);
        const bool dom = (T)c[0] > -kF && (T)c[1] > -kF && (T)c[2] > -kF && (T)(c[0] + B) < kF &&
                         (T)(c[1] + B) < kF && (T)(c[2] + B) < kF;
        const T blo0 = dom ? (T)c[0] : kF, blo1 = (T)c[1], blo2 = (T)c[2];  // dom false: no point passes
        const T bhi0 = (T)(c[0] + B), bhi1 = (T)(c[1] + B), bhi2 = (T)(c[2] + B);

        auto process = [&](long long q, const T xs[3 * G]) {
            const long long j0 = q << LG;
            T r[G];
            auto in_brick = [&](int u) {  // non-short-circuit: one predicate chain
                return (xs[3 * u] >= blo0) & (xs[3 * u] < bhi0) & (xs[3 * u + 1] >= blo1) & (xs[3 * u + 1] < bhi1) &
                       (xs[3 * u + 2] >= blo2) & (xs[3 * u + 2] < bhi2);
            };
            bool all = true;
#pragma unroll
            for (int u = 0; u < G; ++u) all &= in_brick(u);
            if (all) {
#pragma unroll
                for (int u = 0; u < G; ++u) r[u] = bcc_tet_tile_v2<E, T>(xs[3 * u], xs[3 * u + 1], xs[3 * u + 2], sbias, sbase);
            } else {
#pragma unroll 1
                for (int u = 0; u < G; ++u) {  // rare: one call site each, registers selected
                    auto pick = [&](int o) {
                        T v = xs[o];
#pragma unroll
                        for (int w = 1; w < G; ++w) v = u == w ? xs[3 * w + o] : v;
                        return v;
                    };
                    const T x0 = pick(0), x1 = pick(1), x2 = pick(2);
                    T v;
                    if ((x0 >= blo0) & (x0 < bhi0) & (x1 >= blo1) & (x1 < bhi1) & (x2 >= blo2) & (x2 < bhi2))
                        v = bcc_tet_tile_v2<E, T>(x0, x1, x2, sbias, sbase);
                    else if (fabs(x0) < kF && fabs(x1) < kF && fabs(x2) < kF)
                        v = bcc_tet_global<T, T>(a, x0 - T(1), x1 - T(1), x2 - T(1));
                    else if (isfinite(x0) && isfinite(x1) && isfinite(x2))
                        v = bcc_tet_global<double, T>(a, (double)x0 - 1.0, (double)x1 - 1.0, (double)x2 - 1.0);
                    else
                        v = T(NAN);
#pragma unroll
                    for (int w = 0; w < G; ++w) r[w] = u == w ? v : r[w];
                }
            }
            if (j0 >= p0 && j0 + G <= p1) {
                if constexpr (sizeof(T) == 4) {
                    *reinterpret_cast<float4*>(a.out + j0) = make_float4(r[0], r[1], r[2], r[3]);
                } else {
                    *reinterpret_cast<double2*>(a.out + j0) = make_double2(r[0], r[1]);
                }
            } else {
#pragma unroll
                for (int u = 0; u < G; ++u)
                    if (j0 + u >= p0 && j0 + u < p1) a.out[j0 + u] = r[u];
            }
        };

#pragma unroll 1
        for (; q < q1; q += 2 * kThreads) {
            const bool has_b = q + kThreads < q1;
            if (has_b) load_group((q + kThreads) << LG, xb);
            process(q, xa);
            if (!has_b) break;
            if (q + 2 * kThreads < q1) load_group((q + 2 * kThreads) << LG, xa);
            process(q + kThreads, xb);
        }
        __syncthreads();  // the tile is restaged for the next brick
    }
}

}  // namespace sp
