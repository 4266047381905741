// sp_prefilter.cu — quasi-interpolation prefilter on coset grids.
//
// The step before reconstruction in the paper's convergence study (§5.2):
// the samples are replaced by their lattice correlation with the spline's quasi-
// interpolation taps (corpus.py:71-111).  On the coset layout one output coset k reads a
// fixed list of (source coset, cell offset, weight) taps; the kernel is a streaming stencil
// over shared-memory tiles, so the HBM traffic is one read of every input coset plus one
// write of every output coset.
// Separate multiply / add roundings in the given tap order, boundary policy on every read
// (runtime.py:109-123), so float64 results equal the reference's per-site loop bit for bit.
#include <cuda.h>
#include <cuda_runtime.h>

#include <string>

#include "../../include/splinerecon.h"
#include "sp_common.cuh"

namespace sp {
void set_error(const std::string& msg);  // splinerecon.cu (feeds sp_last_error)
}

namespace {

__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

// Tiled kernel.  One block = an output tile of kTX (z2) x kTY (z1) samples of one plane z0
// of one output coset k; blockIdx.z interleaves (z0, k) so the tiles of all output cosets
// over one input region run close together (each input coset is read from HBM once per
// step).  The block first stages, per source coset its taps read, the box of input samples
// the tile needs (tile + the taps' cell-offset range) into shared memory — warp per row,
// lanes along the contiguous axis, boundary policy resolved here — then every output is
// sum_t w_t * box[t][...] with the tap's box offset precomputed on the host: one LDS, one
// multiply, one add per tap, separate roundings, taps in the given order.
constexpr int kTX = 128, kTY = 16, kThreadsPF = 256, kZChunk = 32;
constexpr int kAhead = 1;  // prefetch depth: planes staged ahead of the step being computed (2 measured no faster)

template <typename T>
struct TileTaps {             // one output coset
    int n;                    // taps
    int nbox;                 // source boxes
    int box_src[SP_MAX_COSETS];
    int box_lo[SP_MAX_COSETS][3];   // min tap offset per axis (box origin relative to the tile)
    int box_ex[SP_MAX_COSETS][3];   // box extents
    int box_off[SP_MAX_COSETS];     // smem element offset of the box's plane ring
    int ring[SP_MAX_COSETS];        // planes in the ring: power of two >= box_ex[0] + 1 (one prefetched ahead)
    int slot_elems[SP_MAX_COSETS];  // ring slot stride (elements; 128-byte multiple)
    int pitch[SP_MAX_COSETS];       // staged row pitch (elements)
    int tap_box[SP_MAX_STENCIL];
    int tap_dz0[SP_MAX_STENCIL];    // plane offset of the tap
    int tap_off[SP_MAX_STENCIL];    // in-plane offset of (dz1 - lo1, dz2 - lo2)
    T w[SP_MAX_STENCIL];
};

template <typename T>
struct TileParams {
    TileTaps<T> c[SP_MAX_COSETS];
    T* out[SP_MAX_COSETS];
};

constexpr int kChunks = (kTX + 31) / 32 + 1;  // box rows up to kTX + 32 wide (tap offsets span <= 32)

// Linear index of array index (a0, a1, a2) of coset s after the boundary policy
// (runtime.py:109-123); ok is cleared when the 'zero' policy reads outside (value 0).
template <typename T>
__device__ __forceinline__ long long policy_index(const sp::GridArgs<T>& g, int s, int a0, int a1, int a2, bool& ok) {
    const int e0 = g.ext[s][0], e1 = g.ext[s][1], e2 = g.ext[s][2];
    const bool in = (unsigned)a0 < (unsigned)e0 && (unsigned)a1 < (unsigned)e1 && (unsigned)a2 < (unsigned)e2;
    if (!in) {
        if (g.boundary == SP_ZERO) {
            ok = false;
            a0 = a1 = a2 = 0;
        } else if (g.boundary == SP_CLAMP) {
            a0 = min(max(a0, 0), e0 - 1);
            a1 = min(max(a1, 0), e1 - 1);
            a2 = min(max(a2, 0), e2 - 1);
        } else {
            a0 = sp::mirror_index(a0, e0);
            a1 = sp::mirror_index(a1, e1);
            a2 = sp::mirror_index(a2, e2);
        }
    }
    return ((long long)a0 * e1 + a1) * e2 + a2;
}

// Staging modes of the z-marching kernel.
//   kCpAsync: every thread copies its share of a plane element by element (cp.async, boundary
//             policy folded into the source index) — any grid, any policy.
//   kTmaPlane: one thread copies whole box planes with a 3-D tensor map (TMA zero-fills out
//             of range = the 'zero' policy) — coset rows that are 16-byte multiples.
enum PfMode { kCpAsync = 0, kTmaPlane = 1 };

// Copy plane `p` (coset-cell index along axis 0) of box b's rows [y0 + lo1, ...) x
// [x0 + lo2, ...) into ring slot `slot` with cp.async (4 / 8-byte elements, zero-filled for the
// 'zero' policy outside the array, clamp / mirror indices otherwise): warp per row.
template <typename T>
__device__ __forceinline__ void stage_plane(const sp::GridArgs<T>& g, const TileTaps<T>& tp, int b, int p, int slot,
                                            int y0, int x0, int hv, int wv, T* sm, int lane, int warp) {
    const int s = tp.box_src[b];
    const int ex1 = tp.box_ex[b][1], ex2 = tp.box_ex[b][2];
    const int ex1c = ex1 - (kTY - hv), ex2c = ex2 - (kTX - wv);  // rows / columns the valid outputs read
    const int s1 = y0 + tp.box_lo[b][1], s2 = x0 + tp.box_lo[b][2];
    const T* src = g.data[s];
    T* dst = sm + tp.box_off[b] + slot * tp.slot_elems[b];
    const int e0 = g.ext[s][0], e1 = g.ext[s][1], e2 = g.ext[s][2];
    const bool inside = p >= 0 && p < e0 && s1 >= 0 && s2 >= 0 && s1 + ex1c <= e1 && s2 + ex2c <= e2;
    for (int i1 = warp; i1 < ex1c; i1 += kThreadsPF / 32) {
        T* drow = dst + i1 * tp.pitch[b];
        if (inside) {
            const T* rp = src + ((long long)p * e1 + (s1 + i1)) * e2 + s2;
            for (int c = lane; c < ex2c; c += 32) sp::cp_async_elem<sizeof(T)>(drow + c, rp + c, (int)sizeof(T));
        } else {
            for (int c = lane; c < ex2c; c += 32) {
                bool ok = true;
                const long long idx = policy_index(g, s, p, s1 + i1, s2 + c, ok);
                sp::cp_async_elem<sizeof(T)>(drow + c, src + (ok ? idx : 0), ok ? (int)sizeof(T) : 0);
            }
        }
    }
}

// Tensor maps of the TMA variant: one per (output coset, source box), box = one plane of the
// source box (rows x 16-byte aligned columns); out-of-range texels are zero-filled by the TMA
// unit, which is the 'zero' policy.
constexpr int kMaxMaps = 16;
struct PfMaps {
    CUtensorMap m[kMaxMaps];
    int nbox_max;
    unsigned set_bytes[SP_MAX_COSETS];  // bytes of one plane of every box, per output coset
};

__device__ __forceinline__ void pf_mbar_init(unsigned long long* bar) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a) : "memory");
}
__device__ __forceinline__ void pf_mbar_expect(unsigned long long* bar, unsigned bytes) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void pf_mbar_wait(unsigned long long* bar, unsigned parity) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void pf_tma_plane(void* dst, const CUtensorMap* map, unsigned long long* bar, int c0, int c1,
                                             int c2) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
            "r"(d), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(b)
        : "memory");
}

// z-marching kernel.  One block = an output tile of kTX (z2) x kTY (z1) samples of output
// coset k, marching over kZChunk planes z0: each source box keeps a ring of box_ex[0] + 1 (or
// more: a power of two) staged planes, so every input plane is copied into shared memory
// once per tile column, one plane ahead of the computation, instead of once per output
// plane.  Each output is sum_t w_t * box[t][...] — one LDS, one multiply, one add per tap,
// separate roundings, taps in the given order (bit-identical to a per-site loop over
// site_value).
template <typename T, int NT, int kMode>
__global__ void __launch_bounds__(kThreadsPF) prefilter_zmarch(const sp::GridArgs<T> g, const TileParams<T> P,
                                                               const __grid_constant__ PfMaps maps) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* sm = reinterpret_cast<T*>(smem_raw);
    __shared__ __align__(8) unsigned long long mbar[2];
    constexpr bool kAsyncBar = kMode == kTmaPlane;  // mbarrier-tracked copies
    const int k = blockIdx.z % g.M;
    const int zc = blockIdx.z / g.M;
    const TileTaps<T>& tp = P.c[k];
    const int e0 = g.ext[k][0], e1 = g.ext[k][1], e2 = g.ext[k][2];
    const int x0 = blockIdx.x * kTX, y0 = blockIdx.y * kTY;
    const int za = zc * kZChunk, zb = min(za + kZChunk, e0);
    if (za >= e0 || y0 >= e1 || x0 >= e2) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wv = min(kTX, e2 - x0), hv = min(kTY, e1 - y0);
    auto slot_of = [&](int b, int p) { return p & (tp.ring[b] - 1); };  // ring sizes are powers of two
    if constexpr (kAsyncBar) {
        if (tid == 0) {
            pf_mbar_init(&mbar[0]);
            pf_mbar_init(&mbar[1]);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
    }
    // stage one set of planes: plane p(b) of every box b, tracked by `bar`
    auto stage_set = [&](auto plane_of, int nplanes, unsigned long long* bar) {
        if constexpr (kMode == kCpAsync) {
            for (int b = 0; b < tp.nbox; ++b)
                for (int i = 0; i < nplanes; ++i) {
                    const int p = plane_of(b, i);
                    if (p != INT_MIN) stage_plane<T>(g, tp, b, p, slot_of(b, p), y0, x0, hv, wv, sm, lane, warp);
                }
            asm volatile("cp.async.commit_group;\n" ::: "memory");
        } else if constexpr (kMode == kTmaPlane) {
            if (tid == 0) {
                unsigned bytes = 0;
                for (int b = 0; b < tp.nbox; ++b)
                    for (int i = 0; i < nplanes; ++i)
                        if (plane_of(b, i) != INT_MIN) bytes += (unsigned)(tp.box_ex[b][1] * tp.box_ex[b][2] * (int)sizeof(T));
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                pf_mbar_expect(bar, bytes);
                for (int b = 0; b < tp.nbox; ++b)
                    for (int i = 0; i < nplanes; ++i) {
                        const int p = plane_of(b, i);
                        if (p != INT_MIN)
                            pf_tma_plane(sm + tp.box_off[b] + slot_of(b, p) * tp.slot_elems[b],
                                         &maps.m[k * maps.nbox_max + b], bar, x0 + tp.box_lo[b][2], y0 + tp.box_lo[b][1], p);
                    }
            }
        }
    };
    // prologue: set 0 = planes za + lo0 .. za + hi0 of every box (mbar[0]); set a < kAhead = the
    // plane step za + a adds; set i + kAhead is issued during step i (mbar[(i + kAhead) & 1])
    int maxex0 = 0;
    for (int b = 0; b < tp.nbox; ++b) maxex0 = max(maxex0, tp.box_ex[b][0]);
    stage_set([&](int b, int i) { return i < tp.box_ex[b][0] ? za + tp.box_lo[b][0] + i : INT_MIN; }, maxex0, &mbar[0]);
    for (int a = 1; a < kAhead; ++a) {
        if (za + a < zb) stage_set([&](int b, int) { return za + a + tp.box_lo[b][0] + tp.box_ex[b][0] - 1; }, 1, &mbar[a & 1]);
        else if constexpr (kMode != kTmaPlane) asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    const int tx = tid % kTX, ty = tid / kTX;
    constexpr int kRowsPerThread = kTY / (kThreadsPF / kTX);
    const bool col_ok = x0 + tx < e2;
    for (int z0 = za; z0 < zb; ++z0) {
        const int it = z0 - za;
        if constexpr (kMode != kTmaPlane) asm volatile("cp.async.wait_group %0;\n" ::"n"(kAhead - 1) : "memory");
        if constexpr (kAsyncBar) pf_mbar_wait(&mbar[it & 1], (unsigned)(it >> 1) & 1u);
        __syncthreads();  // set it landed for every thread; every thread is past step it - 1
        // prefetch set it + kAhead (the plane per box that step adds) into the slot step it - 1 read
        if (z0 + kAhead < zb)
            stage_set([&](int b, int) { return z0 + kAhead + tp.box_lo[b][0] + tp.box_ex[b][0] - 1; }, 1,
                      &mbar[(it + kAhead) & 1]);
        else if constexpr (kMode != kTmaPlane)
            asm volatile("cp.async.commit_group;\n" ::: "memory");
        if (col_ok) {
            T* out = P.out[k] + ((long long)z0 * e1 + y0) * e2 + x0 + tx;
            if constexpr (NT > 0) {
                int base[NT], pitch[NT];
                T w[NT];
#pragma unroll
                for (int t = 0; t < NT; ++t) {
                    const int b = tp.tap_box[t];
                    pitch[t] = tp.pitch[b];
                    base[t] = tp.box_off[b] + slot_of(b, z0 + tp.tap_dz0[t]) * tp.slot_elems[b] + tp.tap_off[t] +
                              ty * pitch[t] + tx;
                    w[t] = tp.w[t];
                }
#pragma unroll
                for (int j = 0; j < kRowsPerThread; ++j) {
                    const int r = ty + j * (kThreadsPF / kTX);
                    if (y0 + r >= e1) break;
                    T acc = T(0);
#pragma unroll
                    for (int t = 0; t < NT; ++t)
                        acc = add_rn(acc, mul_rn(w[t], sm[base[t] + j * (kThreadsPF / kTX) * pitch[t]]));
                    out[(long long)r * e2] = acc;
                }
            } else {
                for (int j = 0; j < kRowsPerThread; ++j) {
                    const int r = ty + j * (kThreadsPF / kTX);
                    if (y0 + r >= e1) break;
                    T acc = T(0);
                    for (int t = 0; t < tp.n; ++t) {
                        const int b = tp.tap_box[t];
                        const int pl = tp.box_off[b] + slot_of(b, z0 + tp.tap_dz0[t]) * tp.slot_elems[b];
                        acc = add_rn(acc, mul_rn(tp.w[t], sm[pl + tp.tap_off[t] + r * tp.pitch[b] + tx]));
                    }
                    out[(long long)r * e2] = acc;
                }
            }
        }
    }
    if constexpr (kMode != kTmaPlane) asm volatile("cp.async.wait_all;\n" ::: "memory");
}

int pfail(int code, const std::string& msg) {
    sp::set_error(msg);
    return code;
}

typedef CUresult (*PfEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PfEncodeFn pf_encoder() {
    // initialised once, thread-safely (function-local static)
    static const PfEncodeFn fn = [] {
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<PfEncodeFn>(f);
        return (PfEncodeFn) nullptr;
    }();
    return fn;
}

template <typename T>
int run(const sp_grid_desc* in, const sp_stencil_desc* st, void* const* out, cudaStream_t stream) {
    sp::GridArgs<T> g{};
    g.M = in->M;
    g.boundary = in->boundary;
    long long max_e[3] = {0, 0, 0};
    for (int k = 0; k < in->M; ++k) {
        if (!in->data[k] || !out[k]) return pfail(SP_ERR_INVALID, "null coset array");
        g.data[k] = reinterpret_cast<const T*>(in->data[k]);
        for (int i = 0; i < 3; ++i) {
            if (in->extent[k][i] < 1 || in->extent[k][i] > (1ll << 30))
                return pfail(SP_ERR_INVALID, "coset extent out of range");
            g.ext[k][i] = (int)in->extent[k][i];
            g.org[k][i] = (int)in->origin[k][i];
            max_e[i] = std::max(max_e[i], (long long)in->extent[k][i]);
        }
    }
    if ((max_e[1] + kTY - 1) / kTY > 65535 || (max_e[0] + kZChunk - 1) / kZChunk * in->M > 65535)
        return pfail(SP_ERR_UNSUPPORTED, "prefilter: coset extents too large for the launch grid");
    // 1. per output coset: one source box per source coset = tile + the taps' offset range
    TileParams<T> P{};
    int lo[SP_MAX_COSETS][SP_MAX_COSETS][3], box_of[SP_MAX_COSETS][SP_MAX_COSETS];
    int nbox_max = 0;
    for (int k = 0; k < in->M; ++k) {
        TileTaps<T>& tp = P.c[k];
        const int t0 = st->tap_start[k], t1 = st->tap_start[k + 1];
        tp.n = t1 - t0;
        if (tp.n < 0 || tp.n > SP_MAX_STENCIL) return pfail(SP_ERR_INVALID, "tap count out of range");
        int hi[SP_MAX_COSETS][3];
        for (int s2 = 0; s2 < SP_MAX_COSETS; ++s2) box_of[k][s2] = -1;
        for (int t = 0; t < tp.n; ++t) {
            const int s2 = st->src_coset[t0 + t];
            if (s2 < 0 || s2 >= in->M) return pfail(SP_ERR_INVALID, "tap source coset out of range");
            const int* dz = st->dz + 3 * (t0 + t);
            for (int i = 0; i < 3; ++i)
                if (dz[i] < -(1 << 20) || dz[i] > (1 << 20)) return pfail(SP_ERR_INVALID, "tap offset out of range");
            if (box_of[k][s2] < 0) {
                box_of[k][s2] = tp.nbox++;
                for (int i = 0; i < 3; ++i) lo[k][s2][i] = hi[s2][i] = dz[i];
            }
            for (int i = 0; i < 3; ++i) {
                lo[k][s2][i] = std::min(lo[k][s2][i], dz[i]);
                hi[s2][i] = std::max(hi[s2][i], dz[i]);
            }
        }
        for (int s2 = 0; s2 < in->M; ++s2) {
            const int b = box_of[k][s2];
            if (b < 0) continue;
            tp.box_src[b] = s2;
            const int tile[3] = {1, kTY, kTX};
            for (int i = 0; i < 3; ++i) {
                tp.box_lo[b][i] = lo[k][s2][i];
                tp.box_ex[b][i] = tile[i] + hi[s2][i] - lo[k][s2][i];
            }
            if (tp.box_ex[b][2] > kTX + 32) return pfail(SP_ERR_UNSUPPORTED, "prefilter: tap offsets span more than 32 cells along axis 2");
        }
        nbox_max = std::max(nbox_max, tp.nbox);
        P.out[k] = reinterpret_cast<T*>(out[k]);
    }
    if (nbox_max == 0) {  // no taps anywhere: zero output
        for (int k = 0; k < in->M; ++k)
            cudaMemsetAsync(out[k], 0, (size_t)(in->extent[k][0] * in->extent[k][1] * in->extent[k][2]) * sizeof(T),
                            stream);
        return SP_OK;
    }
    // 2. staging mode: TMA planes when the policy is 'zero' (the TMA unit zero-fills out of
    //    range) and every coset row is a multiple of 16 bytes (tensor-map strides), else
    //    element-wise cp.async; the TMA layout (aligned, wider boxes) must fit shared memory.
    //    (1-D bulk row copies and 16-byte cp.async of the aligned row spans were measured slower
    //    than element-wise cp.async on 1,624-byte rows and are not kept.)
    constexpr int kVecE = 16 / (int)sizeof(T);
    PfEncodeFn enc = pf_encoder();
    bool aligned16 = true;
    for (int k = 0; k < in->M; ++k) {
        aligned16 &= (in->extent[k][2] * (long long)sizeof(T)) % 16 == 0;
        if ((reinterpret_cast<uintptr_t>(in->data[k]) & 15) != 0) aligned16 = false;
    }
    const TileParams<T> P0 = P;
    // lay out mode `m` into P; returns the shared-memory bytes, or -1 if the mode does not apply
    auto layout = [&](int m) -> long long {
        P = P0;
        long long need = 0;
        for (int k = 0; k < in->M; ++k) {
            TileTaps<T>& tp = P.c[k];
            long long off = 0;
            for (int b = 0; b < tp.nbox; ++b) {
                if (m == kTmaPlane) {  // 16-byte aligned box columns
                    const int l2 = tp.box_lo[b][2];
                    const int al = l2 >= 0 ? l2 / kVecE * kVecE : -((-l2 + kVecE - 1) / kVecE) * kVecE;
                    tp.box_ex[b][2] = (tp.box_ex[b][2] + (l2 - al) + kVecE - 1) / kVecE * kVecE;
                    tp.box_lo[b][2] = al;
                    if (tp.box_ex[b][2] > 256 || tp.box_ex[b][1] > 256) return -1;
                }
                tp.pitch[b] = tp.box_ex[b][2];
                tp.ring[b] = 1;
                while (tp.ring[b] < tp.box_ex[b][0] + kAhead) tp.ring[b] *= 2;  // kAhead planes ahead; slot = plane & (ring-1)
                const int plane = tp.box_ex[b][1] * tp.pitch[b];
                tp.slot_elems[b] = (plane * (int)sizeof(T) + 127) / 128 * 128 / (int)sizeof(T);
                tp.box_off[b] = (int)off;
                off += (long long)tp.ring[b] * tp.slot_elems[b];
            }
            need = std::max(need, off * (long long)sizeof(T));
            const int t0 = st->tap_start[k];
            for (int t = 0; t < tp.n; ++t) {
                const int s2 = st->src_coset[t0 + t];
                const int bx = box_of[k][s2];
                const int* dz = st->dz + 3 * (t0 + t);
                tp.tap_box[t] = bx;
                tp.tap_dz0[t] = dz[0];
                tp.tap_off[t] = (dz[1] - tp.box_lo[bx][1]) * tp.pitch[bx] + (dz[2] - tp.box_lo[bx][2]);
                tp.w[t] = (T)st->weight[t0 + t];
            }
        }
        return need <= 160 * 1024 ? need : -1;
    };
    int mode = -1;
    long long smem_need = -1;
    if (in->boundary == SP_ZERO && enc != nullptr && in->M * nbox_max <= kMaxMaps && aligned16 &&
        (smem_need = layout(kTmaPlane)) >= 0)
        mode = kTmaPlane;
    if (mode < 0 && (smem_need = layout(kCpAsync)) >= 0) mode = kCpAsync;
    if (mode < 0) return pfail(SP_ERR_UNSUPPORTED, "prefilter: tap offsets span too large a box");
    bool use_tma = mode == kTmaPlane;
    PfMaps maps{};
    maps.nbox_max = nbox_max;
    if (use_tma) {
        for (int k = 0; k < in->M && use_tma; ++k) {
            const TileTaps<T>& tp = P.c[k];
            unsigned bytes = 0;
            for (int b = 0; b < tp.nbox; ++b) {
                const int src = tp.box_src[b];
                const cuuint64_t dims[3] = {(cuuint64_t)in->extent[src][2], (cuuint64_t)in->extent[src][1],
                                            (cuuint64_t)in->extent[src][0]};
                const cuuint64_t strides[2] = {(cuuint64_t)(in->extent[src][2] * sizeof(T)),
                                               (cuuint64_t)(in->extent[src][2] * in->extent[src][1] * sizeof(T))};
                const cuuint32_t box[3] = {(cuuint32_t)tp.box_ex[b][2], (cuuint32_t)tp.box_ex[b][1], 1u};
                const cuuint32_t estr[3] = {1, 1, 1};
                if (enc(&maps.m[k * nbox_max + b], sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                        3, const_cast<void*>(in->data[src]), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
                    use_tma = false;
                bytes += (unsigned)(tp.box_ex[b][1] * tp.box_ex[b][2] * (int)sizeof(T));
            }
            maps.set_bytes[k] = bytes;
        }
    }
    if (mode == kTmaPlane && !use_tma) {  // tensor-map encoding refused: next mode
        mode = -1;
        if ((smem_need = layout(kCpAsync)) >= 0) mode = kCpAsync;
        if (mode < 0) return pfail(SP_ERR_UNSUPPORTED, "prefilter: tap offsets span too large a box");
    }
    const int smem_bytes = (int)smem_need;
    int nt = P.c[0].n;
    for (int k = 1; k < in->M; ++k)
        if (P.c[k].n != nt) nt = 0;
    const dim3 grid((unsigned)((max_e[2] + kTX - 1) / kTX), (unsigned)((max_e[1] + kTY - 1) / kTY),
                    (unsigned)((max_e[0] + kZChunk - 1) / kZChunk * in->M));
    cudaError_t e = cudaSuccess;
    auto launch = [&](auto kern) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
        if (e == cudaSuccess) kern<<<grid, kThreadsPF, smem_bytes, stream>>>(g, P, maps);
    };
    switch (nt) {
#define SP_PF_CASE(N)                                                                  \
    case N:                                                                            \
        if (mode == kTmaPlane) launch(prefilter_zmarch<T, N, kTmaPlane>);              \
        else launch(prefilter_zmarch<T, N, kCpAsync>);                                 \
        break;
        SP_PF_CASE(1) SP_PF_CASE(2) SP_PF_CASE(3) SP_PF_CASE(4) SP_PF_CASE(5) SP_PF_CASE(7) SP_PF_CASE(9)
        SP_PF_CASE(27)
        default:
            if (mode == kTmaPlane) launch(prefilter_zmarch<T, 0, kTmaPlane>);
            else launch(prefilter_zmarch<T, 0, kCpAsync>);
            break;
#undef SP_PF_CASE
    }
    if (e != cudaSuccess) return pfail(SP_ERR_CUDA, std::string("prefilter: ") + cudaGetErrorString(e));
    e = cudaGetLastError();
    if (e != cudaSuccess) return pfail(SP_ERR_CUDA, std::string("prefilter launch: ") + cudaGetErrorString(e));
    return SP_OK;
}

}  // namespace

extern "C" int sp_prefilter(const sp_grid_desc* in, const sp_stencil_desc* stencil, void* const* out, void* stream) {
    if (!in || !stencil || !out) return pfail(SP_ERR_INVALID, "null argument");
    if (in->s != 3) return pfail(SP_ERR_UNSUPPORTED, "prefilter: 3-D grids only");
    if (stencil->M != in->M || in->M < 1 || in->M > SP_MAX_COSETS)
        return pfail(SP_ERR_MISMATCH, "stencil coset count does not match the grid");
    if (in->boundary < SP_ZERO || in->boundary > SP_MIRROR) return pfail(SP_ERR_INVALID, "unknown boundary policy");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (in->dtype == SP_F32) return run<float>(in, stencil, out, st);
    if (in->dtype == SP_F64) return run<double>(in, stencil, out, st);
    return pfail(SP_ERR_INVALID, "unknown dtype");
}
