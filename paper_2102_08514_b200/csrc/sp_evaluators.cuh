// sp_evaluators.cuh — per-point evaluators: tensor-product B-spline and generic plan.
//
// Both implement the sum of Algorithm 1 for one point:
//   f(x) = sum_k sum_{groups} g(y) * fetch(...)     (runtime.py:370-407)
// with the sub-region classification done in float64 exactly as runtime.py:371-379.
#pragma once

#include "sp_common.cuh"

namespace sp {

__device__ __forceinline__ void write_dbg(int* dbg, long long i, int M, int k, int cls, const int cell[3]) {
    if (dbg) {
        int* p = dbg + ((long long)i * M + k) * 4;
        p[0] = cls;
        p[1] = cell[0];
        p[2] = cell[1];
        p[3] = cell[2];
    }
}

// ---------------------------------------------------------------------------------------
// Tensor-product B-spline of degree DEG on the Cartesian lattice (non-centred: support
// [0, DEG+1]^3).  Site floor(x) + o (o in [-DEG, 0]^3) has weight
// prod_i w[o_i + DEG](t_i), t = x - floor(x).  The host proves the plan equals this form
// exactly (plan.py: EvaluationPlan.tensor_bspline_degree) before selecting it; for the
// reference's cc_tricubic plan this replaces 8 grouped fetches with degree-9 weight
// programs (1,360 Horner mults) by 3x4 weights + a 64-tap separable sum.

template <int DEG>
struct BWeights;

template <>
struct BWeights<1> {
    template <typename T>
    __device__ __forceinline__ static void w(T t, T* w) {
        w[0] = T(1) - t;
        w[1] = t;
    }
};

template <>
struct BWeights<2> {
    template <typename T>
    __device__ __forceinline__ static void w(T t, T* w) {
        const T s = T(1) - t;
        w[0] = T(0.5) * s * s;
        w[2] = T(0.5) * t * t;
        w[1] = fma(t, s, T(0.5));  // (-2t^2 + 2t + 1)/2
    }
};

template <>
struct BWeights<3> {
    template <typename T>
    __device__ __forceinline__ static void w(T t, T* w) {
        const T s = T(1) - t;
        const T t2 = t * t;
        const T s2 = s * s;
        const T sixth = T(1) / T(6);
        w[0] = sixth * s2 * s;                                // (1-t)^3/6
        w[3] = sixth * t2 * t;                                // t^3/6
        w[1] = fma(t2, fma(T(0.5), t, T(-1)), T(2) / T(3));   // (3t^3 - 6t^2 + 4)/6
        w[2] = fma(s2, fma(T(0.5), s, T(-1)), T(2) / T(3));   // same polynomial in 1-t
    }
};

// S0, S1 > 0: the row-vector tile's pitches as compile-time constants (the headline TMA
// configuration), so the (DEG+1)^2 row loads use immediate offsets.
template <typename T, int DEG, int S0 = 0, int S1 = 0>
struct TensorBSplineEval {
    static constexpr int kMinBlocks = sizeof(T) == 4 ? 4 : 3;  // <= 64 / 80 registers
    static constexpr bool kSig = false;
    __device__ static void tile_records(const EvalArgs<T>&, const TileGeom&, const unsigned char*, int4*, int) {}
    // fp32: rows of DEG+1 taps are one LDS.64 / LDS.128 from the row-vector tile
    template <typename U>
    static constexpr int vec_width() {
        return sizeof(U) == 4 ? (DEG == 1 ? 2 : 4) : 0;
    }
    template <class F, class Ctx>
    __device__ __forceinline__ static T eval(const T x[3], F& f, const Ctx& ctx) {
        int cell[3];
        T w[3][DEG + 1];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const T fl = floor(x[i]);
            BWeights<DEG>::w(x[i] - fl, w[i]);
            cell[i] = ctx.X[i];
        }
        bind_identity(f, *ctx.a, *ctx.geom, 0, cell);
        write_dbg(ctx.a->dbg, ctx.index, 1, 0, 0, cell);
        T acc = T(0);
        if constexpr (F::kIsTile && vec_width<T>() > 0) {
            // staged row-vector tile: one vector load per (a0, a1) row
            const int s0 = S0 > 0 ? S0 : ctx.vst0, s1 = S1 > 0 ? S1 : ctx.vst1;
            const auto* p = f.vtile + (ctx.vbase + cell[0] * s0 + cell[1] * s1 + cell[2] - DEG * (s0 + s1 + 1));
            SP_CHECK(ctx.vbase + cell[0] * s0 + cell[1] * s1 + cell[2] - DEG * (s0 + s1 + 1) >= 0 &&
                     ctx.vbase + cell[0] * s0 + cell[1] * s1 + cell[2] < ctx.geom->vtotal);
#pragma unroll
            for (int a0 = 0; a0 <= DEG; ++a0) {
                T acc1 = T(0);
#pragma unroll
                for (int a1 = 0; a1 <= DEG; ++a1) {
                    const auto q = p[a0 * s0 + a1 * s1];
                    const T* qv = reinterpret_cast<const T*>(&q);
                    T acc2 = T(0);
#pragma unroll
                    for (int a2 = 0; a2 <= DEG; ++a2) acc2 = fma(w[2][a2], qv[a2], acc2);
                    acc1 = fma(w[1][a1], acc2, acc1);
                }
                acc = fma(w[0][a0], acc1, acc);
            }
        } else if constexpr (F::kIsTile) {
            // staged tile, identity frame: rows along the contiguous axis, immediate offsets
            const T* p = f.tile + (f.a0 - DEG * (f.c0 + f.c1 + 1));
#pragma unroll
            for (int a0 = 0; a0 <= DEG; ++a0) {
                T acc1 = T(0);
#pragma unroll
                for (int a1 = 0; a1 <= DEG; ++a1) {
                    const T* row = p + a0 * f.c0 + a1 * f.c1;
                    T acc2 = T(0);
#pragma unroll
                    for (int a2 = 0; a2 <= DEG; ++a2) acc2 = fma(w[2][a2], row[a2], acc2);
                    acc1 = fma(w[1][a1], acc2, acc1);
                }
                acc = fma(w[0][a0], acc1, acc);
            }
        } else {
#pragma unroll
            for (int a0 = 0; a0 <= DEG; ++a0) {
                T acc1 = T(0);
#pragma unroll
                for (int a1 = 0; a1 <= DEG; ++a1) {
                    T acc2 = T(0);
#pragma unroll
                    for (int a2 = 0; a2 <= DEG; ++a2) acc2 = fma(w[2][a2], f.get(a0 - DEG, a1 - DEG, a2 - DEG), acc2);
                    acc1 = fma(w[1][a1], acc2, acc1);
                }
                acc = fma(w[0][a0], acc1, acc);
            }
        }
        return acc;
    }
};

// ---------------------------------------------------------------------------------------
// Generic plan evaluator: any s=3 plan, full T / piA matrices, tables in global memory.
// Used for plans without a compiled-in specialisation; same semantics, slower.

struct GenericTables {
    int Q, r, N, K, n_sites;
    const int* normals;           // [Q*3]
    const double* offsets;        // [Q]
    const int* sigma;             // [r]
    const int* cls_kernel;        // [N]
    const double* cls_T;          // [N*9]
    const double* cls_t;          // [N*3]
    const int* kernel_group_start;// [K+1]
    const int* group_nspan;       // [G]
    const int* group_site_start;  // [G+1]
    const int* group_poly_start;  // [G+1]
    const int* site_off;          // [N*n_sites*3]  (piA site + pib)/d
    const int* poly_term_start;   // [P+1]
    const int* term_exps;         // [T*3]
    const double* term_coeffs;    // [T]
};

template <typename T>
__device__ __forceinline__ T generic_poly(const GenericTables& gt, int p, const T y[3]) {
    T acc = T(0);
    const int e = __ldg(gt.poly_term_start + p + 1);
    for (int t = __ldg(gt.poly_term_start + p); t < e; ++t) {
        T m = (T)__ldg(gt.term_coeffs + t);
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const int ex = __ldg(gt.term_exps + 3 * t + i);
            for (int q = 0; q < ex; ++q) m *= y[i];
        }
        acc += m;
    }
    return acc;
}

template <typename T>
struct GenericEval {
    static constexpr int kMinBlocks = 1;
    static constexpr bool kSig = false;

    __device__ static void tile_records(const EvalArgs<T>&, const TileGeom&, const unsigned char*, int4*, int) {}
    template <typename U>
    static constexpr int vec_width() {
        return 0;
    }
    template <class F, class Ctx>
    __device__ static T eval(const T x[3], F& f, const Ctx& ctx) {
        const EvalArgs<T>& a = *ctx.a;
        const GenericTables& gt = *reinterpret_cast<const GenericTables*>(a.tables);
        T total = T(0);
        for (int k = 0; k < a.fr.M; ++k) {
            const CosetFrame cf = coset_frame(x, a.fr, k);
            long long q = 0;
            for (int j = 0; j < gt.Q; ++j) {
                double dot = 0.0;
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    const int nv = __ldg(gt.normals + 3 * j + i);
                    if (nv) dot += (double)nv * cf.xp[i];
                }
                if (dot >= __ldg(gt.offsets + j)) q |= 1LL << j;
            }
            int cls = __ldg(gt.sigma + (int)(q % gt.r));
            write_dbg(a.dbg, ctx.index, a.fr.M, k, cls, cf.cell);  // raw class: -1 for the sentinel
            if (cls < 0) {
                ctx.err = 1;
                cls = 0;
            }
            T y[3];
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                double v = 0.0;
#pragma unroll
                for (int j = 0; j < 3; ++j) v += __ldg(gt.cls_T + 9 * cls + 3 * i + j) * cf.xp[j];
                y[i] = (T)(v - __ldg(gt.cls_t + 3 * cls + i));
            }
            bind_identity(f, a, *ctx.geom, k, cf.cell);
            const int kern = __ldg(gt.cls_kernel + cls);
            T acc = T(0);
            const int g1 = __ldg(gt.kernel_group_start + kern + 1);
            for (int g = __ldg(gt.kernel_group_start + kern); g < g1; ++g) {
                const int p0 = __ldg(gt.group_poly_start + g);
                const int ns = __ldg(gt.group_nspan + g);
                const int s0 = __ldg(gt.group_site_start + g);
                const T gv = generic_poly(gt, p0, y);
                const int* so = gt.site_off + ((long long)cls * gt.n_sites + s0) * 3;
                if (ns == 0) {
                    acc = fma(gv, f.get(__ldg(so), __ldg(so + 1), __ldg(so + 2)), acc);
                    continue;
                }
                T t[3];
                for (int j = 0; j < ns; ++j) {
                    const T tn = generic_poly(gt, p0 + 1 + j, y);
                    t[j] = gv == T(0) ? T(0.5) : tn / gv;  // plancompile.py:684-688
                }
                T v[8];
                const int size = 1 << ns;
                for (int c = 0; c < size; ++c) v[c] = f.get(__ldg(so + 3 * c), __ldg(so + 3 * c + 1), __ldg(so + 3 * c + 2));
                // local multilinear lerp over the group's corners (bit j <-> span axis j)
                for (int j = 0; j < ns; ++j) {
                    const int step = 1 << j;
                    for (int c = 0; c < size; c += 2 * step) v[c] = fma(t[j], v[c + step] - v[c], v[c]);
                }
                acc = fma(gv, v[0], acc);
            }
            total += acc;
        }
        return total;
    }
};

}  // namespace sp
