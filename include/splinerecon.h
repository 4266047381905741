/*
 * splinerecon.h — C ABI of the B200 reconstruction hot path (libsplinerecon.so).
 *
 * Drop-in boundary for the reference's batch evaluator
 *     PlanInterpreter(plan).eval_batch(grid, pts)        runtime.py:219-248
 * i.e. Algorithm 1 of arXiv 2102.08514 over a compiled
 * EvaluationPlan (plancompile.py:94-143) and a coset-decomposed CoefficientGrid
 * (runtime.py:38-105).  The reference is pure Python with no FFI; the binding a
 * maintainer adds on the reference side is a ctypes stub.
 *
 * Conventions: plain pointers and sizes only, no torch types.  All device pointers
 * are CUDA device memory; calls are stream-ordered and asynchronous unless noted.
 * Functions return SP_OK (0) or a negative sp_status; sp_last_error() gives a
 * thread-local message.  No exception crosses the ABI.  Concurrent sp_eval calls on
 * different streams with the same plan are safe (a plan is immutable after create).
 */
#ifndef SPLINERECON_H
#define SPLINERECON_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SP_MAX_DIM 3
#define SP_MAX_COSETS 8

typedef enum sp_status {
    SP_OK = 0,
    SP_ERR_INVALID = -1,     /* malformed descriptor / argument            (PlanError)     */
    SP_ERR_UNSUPPORTED = -2, /* valid but not implemented (e.g. s != 3)    (NotImplemented) */
    SP_ERR_CUDA = -3,        /* CUDA runtime failure                                         */
    SP_ERR_SENTINEL = -4,    /* sigma sentinel hit      runtime.py:380-381 (RuntimeError_)   */
    SP_ERR_MISMATCH = -5     /* grid decomposition != plan header, runtime.py:250-254         */
} sp_status;

typedef enum sp_dtype { SP_F32 = 0, SP_F64 = 1 } sp_dtype;

/* CoefficientGrid boundary policies, runtime.py:35 and :109-123 / :151-168 / :191-204 */
typedef enum sp_boundary { SP_ZERO = 0, SP_CLAMP = 1, SP_MIRROR = 2 } sp_boundary;

/* Which kernel family a created plan dispatches to (sp_plan_kernel_kind). */
typedef enum sp_kernel_kind {
    SP_KIND_TENSOR_BSPLINE = 0, /* separable closed form, proven equal to the plan      */
    SP_KIND_GENERATED = 1,      /* plan-specialised kernel compiled into this library   */
    SP_KIND_GENERIC = 2         /* table-driven kernel for any other plan (still GPU)   */
} sp_kernel_kind;

/*
 * Flattened EvaluationPlan (plancompile.py:94-143; ClassTransform analysis.py:89-100;
 * FetchGroup plancompile.py:55-77).  Replaces the Python object the reference passes to
 * PlanInterpreter(plan) (runtime.py:219).  All arrays are host memory, row-major, and
 * are copied by sp_plan_create.
 */
typedef struct sp_plan_desc {
    int32_t s;                              /* dimension; kernels implement s == 3          */
    int32_t M;                              /* cosets                                         */
    int32_t diag[SP_MAX_DIM];               /* D = diag(d_i)              lattice.py:104-133 */
    int32_t shifts[SP_MAX_COSETS][SP_MAX_DIM]; /* l_k                                          */
    int32_t Q;                              /* plane count                                     */
    const int32_t* normals;                 /* [Q*s] integer normals                           */
    const double* offsets;                  /* [Q]  float(offset), as runtime.py:263           */
    int32_t r;                              /* sigma modulus                                   */
    const int32_t* sigma;                   /* [r]  class id or -1 sentinel                    */
    int32_t N;                              /* classes                                         */
    const int32_t* cls_kernel;              /* [N]                                             */
    const double* cls_T;                    /* [N*s*s] float(T)                                */
    const double* cls_t;                    /* [N*s]   float(t)                                */
    const int32_t* cls_piA;                 /* [N*s*s]                                         */
    const int32_t* cls_pib;                 /* [N*s]                                           */
    int32_t K;                              /* kernels                                         */
    const int32_t* kernel_group_start;      /* [K+1] into groups                               */
    int32_t n_groups;
    const int32_t* group_span;              /* [n_groups*SP_MAX_DIM] span axes, -1 padded     */
    const int32_t* group_nspan;             /* [n_groups] len(span_axes); size = 1 << nspan   */
    const int32_t* group_site_start;        /* [n_groups+1] into sites                         */
    const int32_t* sites;                   /* [n_sites*s] zero-coset lattice vectors          */
    const int32_t* group_poly_start;        /* [n_groups+1] into polys: g, then t_nums[j]      */
    int32_t n_polys;
    const int32_t* poly_term_start;         /* [n_polys+1] into terms                          */
    const int32_t* term_exps;               /* [n_terms*s]                                     */
    const double* term_coeffs;              /* [n_terms]  float(coefficient)                   */
    int32_t texel_offset_half;              /* PlanOptions.texel_offset_half                   */
    int32_t tp_degree;                      /* >= 0: caller asserts a tensor-product B-spline  */
                                            /* plan of this degree; verified in create.        */
                                            /* -1: automatic; -2: force the generic kernel.     */
} sp_plan_desc;

/* One coset-decomposed grid: per-coset contiguous C-order device arrays (axis s-1
 * fastest), site D z + l_k at arrays[k][z - origin[k]] (runtime.py:38-43). */
typedef struct sp_grid_desc {
    int32_t s;
    int32_t M;
    int32_t dtype;                              /* sp_dtype of the arrays                   */
    int32_t boundary;                           /* sp_boundary                               */
    int32_t diag[SP_MAX_DIM];
    int32_t shifts[SP_MAX_COSETS][SP_MAX_DIM];
    const void* data[SP_MAX_COSETS];            /* device pointers                           */
    int64_t extent[SP_MAX_COSETS][SP_MAX_DIM];
    int64_t origin[SP_MAX_COSETS][SP_MAX_DIM];
} sp_grid_desc;

typedef struct sp_plan sp_plan; /* opaque; owns device copies of the packed tables */

/* Validate + specialise a plan.  Replaces PlanInterpreter.__init__ / _batch_tables
 * (runtime.py:219-230, :256-272).  Requires a CUDA device. */
int sp_plan_create(const sp_plan_desc* desc, sp_plan** out);
void sp_plan_destroy(sp_plan* plan);
int sp_plan_kernel_kind(const sp_plan* plan); /* sp_kernel_kind */
/* Name of the specialised kernel (e.g. "tensor_bspline_3", "gen:bcc_linear_rd", "generic"). */
const char* sp_plan_kernel_name(const sp_plan* plan);

/*
 * Batch reconstruction: out[i] = sum_k sum_{m in C_k(x_i)} c_m phi(x_i - m)   (Eq. 7).
 * Replaces PlanInterpreter.eval_batch (runtime.py:244-248) -> _eval_batch (:363-408).
 *   pts  device [n*s] of `dtype`; out device [n] of `dtype`; grid arrays must be `dtype`.
 *   dbg  nullable device int32 [n*M*4]: per point and coset (class id, cell_0..2), the
 *        classification of runtime.py:371-379 (cell = kk/d).
 *   err_flag nullable device int32, OR-ed with 1 when a sigma sentinel is hit.
 *   stream  cudaStream_t (0 = legacy default stream).
 * Asynchronous; returns before the kernel finishes.  n == 0 is a no-op.
 */
int sp_eval(const sp_plan* plan, const sp_grid_desc* grid, const void* pts, int64_t n, int32_t dtype,
            void* out, int32_t* dbg, int32_t* err_flag, void* stream);

/*
 * Brick mode (the fast path for coherent point sets).  Points sorted by sp_morton_keys are
 * grouped into aligned bricks of (2^log2_brick)^3 unit cells; brick_start (device int64,
 * n_bricks+1 entries) delimits each brick's run of points.  One CTA stages a brick's
 * coefficient box (+ halo) once and evaluates all its points.  Results go to
 * out[out_index[i]] when out_index (device int64 [n]) is given, else out[i].  Same
 * arithmetic as sp_eval, bit-identical results.  Any brick partition is correct (points
 * outside their run's brick are evaluated without staging).
 */
int sp_eval_bricks(const sp_plan* plan, const sp_grid_desc* grid, const void* pts, int64_t n, int32_t dtype,
                   const int64_t* brick_start, int32_t n_bricks, int32_t log2_brick, const int64_t* out_index,
                   void* out, int32_t* err_flag, void* stream);

/* Recommended log2 brick edge for a plan and dtype (largest brick whose box fits the tile),
 * or a negative value when brick mode is not applicable. */
int sp_brick_log2(const sp_plan* plan, int32_t dtype);

/* Sync-free brick mode.  sp_brick_runs finds the brick runs of Morton-ordered points from
 * their sp_morton_keys (brick id = key >> 3*log2_brick): brick_start (device, capacity
 * n + 1) and the brick count (device int32), without a host round trip.
 * sp_eval_bricks_dev is sp_eval_bricks with the brick count read from device memory
 * (n_bricks_cap bounds it and sizes the launch), so a host pipeline can queue chunk after
 * chunk without synchronising (runtime.py:244-248 over pinned host batches). */
int sp_brick_runs(const uint64_t* keys, int64_t n, int32_t log2_brick, int64_t* brick_start, int32_t* n_bricks,
                  void* temp, int64_t temp_bytes, void* stream);
/* device scratch bytes sp_brick_runs needs for n points (pass it as temp/temp_bytes to avoid
 * a stream-ordered allocation per call; temp may be NULL). */
int64_t sp_brick_runs_temp_bytes(int64_t n);
/* sp_brick_runs_points: the same brick runs computed straight from Morton-ordered points
 * (dtype SP_F32 / SP_F64): a point's brick is the Morton code of its clamped unit cell shifted
 * by 3*log2_brick — identical runs to sp_morton_keys + sp_brick_runs, without the key array.
 * temp: sp_brick_runs_points_temp_bytes(n) bytes (NULL: stream-ordered allocation). */
int64_t sp_brick_runs_points_temp_bytes(int64_t n);
int sp_brick_runs_points(const void* pts, int64_t n, int32_t dtype, int32_t log2_brick, int64_t* brick_start,
                         int32_t* n_bricks, void* temp, int64_t temp_bytes, void* stream);
int sp_eval_bricks_dev(const sp_plan* plan, const sp_grid_desc* grid, const void* pts, int64_t n, int32_t dtype,
                       const int64_t* brick_start, const int32_t* n_bricks_dev, int32_t n_bricks_cap,
                       int32_t log2_brick, const int64_t* out_index, void* out, int32_t* err_flag, void* stream);

/* Input-order protocol B (arbitrary point order) without a host round trip.
 * sp_sort_points: 30-bit Morton keys of the points' unit cells relative to (lo0, lo1, lo2)
 * with `bits` (<= 10) per axis — cells outside [lo, lo + 2^bits) are clamped, which only
 * affects the order (any brick partition is evaluated correctly) — a radix sort of (key,
 * index) pairs over whole 8-bit digits (the lowest 3*bits % 8 key bits, inside a brick, are
 * left unsorted), the points gathered into key order (sorted_pts, same dtype/shape as pts),
 * (skipped when sorted_pts is NULL), the int32 permutation (perm[i] = caller index of sorted
 * point i) and the brick runs
 * (brick_start [n+1], brick count in device memory), all stream-ordered; n < 2^31.
 * temp: device scratch of sp_sort_points_temp_bytes(n) bytes (NULL: stream-ordered alloc).
 * sp_eval_bricks_perm32: sp_eval_bricks_dev writing point i's value to out[perm[i]] — the
 * results come back in the caller's order. */
int64_t sp_sort_points_temp_bytes(int64_t n);
int sp_sort_points(const void* pts, int64_t n, int32_t dtype, int32_t lo0, int32_t lo1, int32_t lo2, int32_t bits,
                   int32_t log2_brick, void* sorted_pts, int32_t* perm, int64_t* brick_start, int32_t* n_bricks,
                   void* temp, int64_t temp_bytes, void* stream);
/* sp_sort_points_payload: protocol B with the points as the sort payload — brick-id keys
 * (Morton order of the bricks of 2^log2_brick cells in the frame lo + [0, 2^bits)^3, cells
 * clamped into the frame), a radix sort of (key, {point, index}) over the brick-id bits only,
 * the sorted points written to sorted_pts ((n,3), required) and their caller indices to perm,
 * and the brick runs; the points are read once, coalesced, instead of through the permutation
 * by the brick kernel.  Pair with sp_eval_bricks_perm32 (results in the caller's order) or
 * sp_eval_bricks_dev (brick order).  temp: sp_sort_points_payload_temp_bytes(n, dtype) bytes. */
int64_t sp_sort_points_payload_temp_bytes(int64_t n, int32_t dtype);
int sp_sort_points_payload(const void* pts, int64_t n, int32_t dtype, int32_t lo0, int32_t lo1, int32_t lo2,
                           int32_t bits, int32_t log2_brick, void* sorted_pts, int32_t* perm, int64_t* brick_start,
                           int32_t* n_bricks, void* temp, int64_t temp_bytes, void* stream);
int sp_eval_bricks_perm32(const sp_plan* plan, const sp_grid_desc* grid, const void* pts, int64_t n, int32_t dtype,
                          const int64_t* brick_start, const int32_t* n_bricks_dev, int32_t n_bricks_cap,
                          int32_t log2_brick, const int32_t* perm, void* out, int32_t* err_flag, void* stream);
/* sp_eval_bricks_indirect: the same without the gathered copy — `pts` are the caller's
 * (unsorted) points, brick-order point i is pts[perm[i]] and its value goes to out[perm[i]]
 * (sp_sort_points may then be called with sorted_pts = NULL, skipping its gather). */
int sp_eval_bricks_indirect(const sp_plan* plan, const sp_grid_desc* grid, const void* pts, int64_t n, int32_t dtype,
                            const int64_t* brick_start, const int32_t* n_bricks_dev, int32_t n_bricks_cap,
                            int32_t log2_brick, const int32_t* perm, void* out, int32_t* err_flag, void* stream);

/* sp_eval_bricks_unordered: as sp_eval_bricks_indirect, but the value of brick-order point i
 * (= pts[perm[i]]) is written to out[i] — results stay in brick order, pairing with perm,
 * for callers that reduce over the batch (error norms, sums) and need no caller order: the
 * random result writes (a read-modify-write of a whole DRAM burst per 4-byte value) vanish. */
int sp_eval_bricks_unordered(const sp_plan* plan, const sp_grid_desc* grid, const void* pts, int64_t n, int32_t dtype,
                             const int64_t* brick_start, const int32_t* n_bricks_dev, int32_t n_bricks_cap,
                             int32_t log2_brick, const int32_t* perm, void* out, int32_t* err_flag, void* stream);

/* Synchronous convenience: sp_eval + stream sync + sentinel check (SP_ERR_SENTINEL). */
int sp_eval_sync(const sp_plan* plan, const sp_grid_desc* grid, const void* pts, int64_t n, int32_t dtype,
                 void* out, void* stream);

/* Number of kernel launches sp_eval issues for n points (for launch accounting). */
int sp_eval_launch_count(const sp_plan* plan, int64_t n);

/* Morton (Z-order) keys of the points' unit cells floor(x): used to present query points
 * in the coherent order the staged kernels exploit (input-order protocol).
 * keys device uint64 [n]. */
int sp_morton_keys(const void* pts, int64_t n, int32_t dtype, uint64_t* keys, void* stream);

/* 30-bit Morton keys of (floor(x) - lo), each axis clamped to [0, 2^bits), bits <= 10:
 * the same order as sp_morton_keys inside the box, half the sort width. keys device int32 [n]. */
int sp_morton_keys32(const void* pts, int64_t n, int32_t dtype, int32_t lo0, int32_t lo1, int32_t lo2, int32_t bits,
                     int32_t* keys, void* stream);

/* out[perm[i]] = src[i]  (float or double, by dtype) — unpermute results of a sorted batch. */
int sp_scatter(const void* src, const int64_t* perm, int64_t n, int32_t dtype, void* out, void* stream);
/* L2-blocked variant with an int32 permutation: one pass over (perm, src) per destination window
 * of `window` elements (<= 0: one pass), each writing only the values landing in its window, so
 * every output sector is written whole while L2-resident (a random 4-byte scatter costs a DRAM
 * read-modify-write per value).  Same result as out[perm[i]] = src[i]. */
int sp_scatter32_blocked(const void* src, const int32_t* perm, int64_t n, int32_t dtype, int64_t window, void* out,
                         void* stream);
/* out[perm[i]] = src[i] for a PERMUTATION perm of [0, n): the (perm, src) pairs are radix-sorted
 * by the destination's bits >= 11 (two 8-bit passes at 1e8), then one CTA per 2048-element
 * destination window writes it with full coalesced stores (no partial-sector writes).  temp:
 * >= sp_scatter32_perm_temp_bytes(n, dtype) bytes of device memory (NULL: allocated on the
 * stream). */
int64_t sp_scatter32_perm_temp_bytes(int64_t n, int32_t dtype);
int sp_scatter32_perm(const void* src, const int32_t* perm, int64_t n, int32_t dtype, void* out, void* temp,
                      int64_t temp_bytes, void* stream);
/* dst[i] = pts[perm[i]] (s=3 points) — gather points into sorted order. */
int sp_gather_points(const void* pts, const int64_t* perm, int64_t n, int32_t dtype, void* dst, void* stream);

/*
 * Hardware-texture-filtered variant (the paper's GPU fetch path),
 * reported separately from the exact kernels because texture filtering weights are 9-bit
 * fixed point: 3-D CUDA array copy of a single-coset float32 grid with linear filtering
 * (boundary zero -> border, clamp -> clamp; mirror is not expressible: the hardware mirror
 * period is 2n, runtime.py:191-196 uses 2n-2).  Tensor-product plans of degree 1 (one
 * filtered fetch per point) and 3 (eight fetches per point).
 */
typedef struct sp_texture sp_texture;
int sp_texture_create(const sp_grid_desc* grid, sp_texture** out);
void sp_texture_destroy(sp_texture* tex);
int sp_eval_texture(const sp_plan* plan, const sp_texture* tex, const void* pts, int64_t n, void* out, void* stream);

/*
 * Quasi-interpolation prefilter on coset grids (taps from
 * corpus.prefilter_taps, corpus.py:71-111): the lattice correlation
 *     out[site] = sum_t w_t * in[site + o_t]
 * resolved per output coset k into taps (source coset, coset-cell offset dz, weight):
 * out_k[z] = sum_{t in [tap_start[k], tap_start[k+1])} weight[t] * in_{src[t]}[z + dz[t]],
 * taps summed in the given order with separate multiply and add (no FMA contraction), the
 * input read through the grid's boundary policy (runtime.py:109-123, as site_value does).
 * `out[k]` are device arrays of the same dtype and extents as in->data[k] (must not alias).
 * At most SP_MAX_STENCIL taps per output coset.  Stream-ordered.
 */
#define SP_MAX_STENCIL 64
typedef struct sp_stencil_desc {
    int32_t M;                                 /* output cosets (= grid M)                    */
    int32_t tap_start[SP_MAX_COSETS + 1];      /* CSR over taps per output coset              */
    const int32_t* src_coset;                  /* [T] host array                              */
    const int32_t* dz;                         /* [T][3] host array                           */
    const double* weight;                      /* [T] host array                              */
} sp_stencil_desc;
int sp_prefilter(const sp_grid_desc* in, const sp_stencil_desc* stencil, void* const* out, void* stream);

/*
 * Ray-marcher around the reconstruction (SPEC.md render_volume, which
 * the reference describes but does not ship).  A frame = per slab of steps:
 *   sp_ray_points -> sp_eval (the slab's points) -> sp_composite.
 * sp_ray_points writes the lattice coordinates of steps [k0, k1) of every pixel's ray,
 * pixel-major (row-major pixels, steps of one ray contiguous), float32 [(w*h*(k1-k0))][3]:
 * orthographic rays from position + v*span_y*up + u*fov*right along forward, sample t =
 * (k + 0.5)*step, lattice = world*lattice_scale + lattice_offset, computed in float64.
 * sp_composite folds one slab of values [npix][nsteps] (float32 or float64 device array) into
 * the per-pixel state [npix][4] = (r, g, b, transmittance) in float64 (initialise to
 * (0, 0, 0, 1)): front to back, colour += T * alpha * rgb, T *= 1 - alpha, with (rgb, alpha)
 * piecewise linear in the value over the transfer function's control points (clamped).
 */
#define SP_MAX_TRANSFER 16
typedef struct sp_camera {
    double position[3], right[3], up[3], forward[3];
    double fov, step, lattice_scale, lattice_offset[3];
} sp_camera;
typedef struct sp_transfer {
    int32_t n;                              /* control points, 2..SP_MAX_TRANSFER, increasing value */
    double points[5 * SP_MAX_TRANSFER];     /* (value, r, g, b, alpha) per control point           */
} sp_transfer;
int sp_ray_points(const sp_camera* cam, int32_t width, int32_t height, int32_t k0, int32_t k1, float* out,
                  void* stream);
int sp_composite(const void* values, int32_t dtype, int64_t npix, int32_t nsteps, const sp_transfer* tf, double* state,
                 void* stream);

/* Staging statistics for tuning (not thread-safe): copies the counters accumulated since the
 * last call into out[4] = {staged chunks, unstaged chunks, staged tile elements, 0} (when
 * out != NULL), then enables (1, counters reset) or disables (0) collection. */
int sp_debug_stats(int enable, uint64_t* out);

const char* sp_last_error(void);
const char* sp_version(void);

#ifdef __cplusplus
}
#endif

#endif /* SPLINERECON_H */
