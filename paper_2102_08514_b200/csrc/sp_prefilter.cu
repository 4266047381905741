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
constexpr int kTX = 128, kTY = 32, kThreadsPF = 256;

template <typename T>
struct TileTaps {             // one output coset
    int n;                    // taps
    int nbox;                 // source boxes
    int box_src[SP_MAX_COSETS];
    int box_lo[SP_MAX_COSETS][3];   // min tap offset per axis (box origin relative to the tile)
    int box_ex[SP_MAX_COSETS][3];   // box extents
    int box_off[SP_MAX_COSETS];     // smem element offset of the box
    int tap_box[SP_MAX_STENCIL];
    int tap_off[SP_MAX_STENCIL];    // box_off + linear offset of (dz - lo) in the box
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

template <typename T, int NT>
__global__ void __launch_bounds__(kThreadsPF) prefilter_tiled(const sp::GridArgs<T> g, const TileParams<T> P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* sm = reinterpret_cast<T*>(smem_raw);
    const int k = blockIdx.z % g.M;
    const int z0 = blockIdx.z / g.M;
    const TileTaps<T>& tp = P.c[k];
    const int e1 = g.ext[k][1], e2 = g.ext[k][2];
    const int x0 = blockIdx.x * kTX, y0 = blockIdx.y * kTY;
    if (z0 >= g.ext[k][0] || y0 >= e1 || x0 >= e2) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // stage the source boxes: warp per box row, each lane issues all of its row's loads
    // before storing any (up to kChunks in flight), boundary policy folded into the index.
    // Only the part of each box the tile's VALID outputs read is staged (edge tiles are
    // clipped to the array), so interior-vs-policy is decided on what is actually read.
    const int wv = min(kTX, e2 - x0), hv = min(kTY, e1 - y0);
    for (int b = 0; b < tp.nbox; ++b) {
        const int s = tp.box_src[b];
        const int ex1 = tp.box_ex[b][1], ex2 = tp.box_ex[b][2];
        const int ex1c = ex1 - (kTY - hv), ex2c = ex2 - (kTX - wv);  // clipped extents
        const int ex0 = tp.box_ex[b][0];
        const int s0 = z0 + tp.box_lo[b][0], s1 = y0 + tp.box_lo[b][1], s2 = x0 + tp.box_lo[b][2];
        const T* src = g.data[s];
        T* dst = sm + tp.box_off[b];
        const bool inside = s0 >= 0 && s1 >= 0 && s2 >= 0 && s0 + ex0 <= g.ext[s][0] && s1 + ex1c <= g.ext[s][1] &&
                            s2 + ex2c <= g.ext[s][2];
        for (int i0 = 0; i0 < ex0; ++i0) {
            for (int i1 = warp; i1 < ex1c; i1 += kThreadsPF / 32) {
                T* drow = dst + (i0 * ex1 + i1) * ex2;
                T v[kChunks];
                if (inside) {
                    const T* rp = src + ((long long)(s0 + i0) * g.ext[s][1] + (s1 + i1)) * g.ext[s][2] + s2;
#pragma unroll
                    for (int c = 0; c < kChunks; ++c) v[c] = lane + 32 * c < ex2c ? __ldg(rp + lane + 32 * c) : T(0);
                } else {
#pragma unroll
                    for (int c = 0; c < kChunks; ++c) {
                        bool ok = lane + 32 * c < ex2c;
                        const long long idx = policy_index(g, s, s0 + i0, s1 + i1, s2 + lane + 32 * c, ok);
                        v[c] = ok ? __ldg(src + idx) : T(0);
                    }
                }
#pragma unroll
                for (int c = 0; c < kChunks; ++c)
                    if (lane + 32 * c < ex2c) drow[lane + 32 * c] = v[c];
            }
        }
    }
    __syncthreads();
    const int tx = tid % kTX;
    const int z2 = x0 + tx;
    if (z2 >= e2) return;
    const int ty = tid / kTX;
    constexpr int kRowsPerThread = kTY / (kThreadsPF / kTX);
    T* out = P.out[k] + ((long long)z0 * e1 + y0) * e2 + z2;
    if constexpr (NT > 0) {
        int base[NT], pitch[NT];
        T w[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            pitch[t] = tp.box_ex[tp.tap_box[t]][2];
            base[t] = tp.tap_off[t] + ty * pitch[t] + tx;
            w[t] = tp.w[t];
        }
#pragma unroll
        for (int j = 0; j < kRowsPerThread; ++j) {
            const int r = ty + j * (kThreadsPF / kTX);
            if (y0 + r >= e1) break;
            T acc = T(0);
#pragma unroll
            for (int t = 0; t < NT; ++t) acc = add_rn(acc, mul_rn(w[t], sm[base[t] + j * (kThreadsPF / kTX) * pitch[t]]));
            out[(long long)r * e2] = acc;
        }
    } else {
        for (int j = 0; j < kRowsPerThread; ++j) {
            const int r = ty + j * (kThreadsPF / kTX);
            if (y0 + r >= e1) break;
            T acc = T(0);
            for (int t = 0; t < tp.n; ++t) {
                const int b = tp.tap_box[t];
                acc = add_rn(acc, mul_rn(tp.w[t], sm[tp.tap_off[t] + r * tp.box_ex[b][2] + tx]));
            }
            out[(long long)r * e2] = acc;
        }
    }
}

int pfail(int code, const std::string& msg) {
    sp::set_error(msg);
    return code;
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
    if ((max_e[1] + kTY - 1) / kTY > 65535 || max_e[0] * in->M > 65535)
        return pfail(SP_ERR_UNSUPPORTED, "prefilter: coset extents too large for the launch grid");
    TileParams<T> P{};
    int smem_max = 0;
    for (int k = 0; k < in->M; ++k) {
        TileTaps<T>& tp = P.c[k];
        const int t0 = st->tap_start[k], t1 = st->tap_start[k + 1];
        tp.n = t1 - t0;
        if (tp.n < 0 || tp.n > SP_MAX_STENCIL) return pfail(SP_ERR_INVALID, "tap count out of range");
        int lo[SP_MAX_COSETS][3], hi[SP_MAX_COSETS][3], box_of[SP_MAX_COSETS];
        for (int s = 0; s < SP_MAX_COSETS; ++s) box_of[s] = -1;
        for (int t = 0; t < tp.n; ++t) {
            const int s = st->src_coset[t0 + t];
            if (s < 0 || s >= in->M) return pfail(SP_ERR_INVALID, "tap source coset out of range");
            const int* dz = st->dz + 3 * (t0 + t);
            for (int i = 0; i < 3; ++i)
                if (dz[i] < -(1 << 20) || dz[i] > (1 << 20)) return pfail(SP_ERR_INVALID, "tap offset out of range");
            if (box_of[s] < 0) {
                box_of[s] = tp.nbox++;
                for (int i = 0; i < 3; ++i) lo[s][i] = hi[s][i] = dz[i];
            }
            for (int i = 0; i < 3; ++i) {
                lo[s][i] = std::min(lo[s][i], dz[i]);
                hi[s][i] = std::max(hi[s][i], dz[i]);
            }
        }
        long long off = 0;
        for (int s = 0; s < in->M; ++s) {
            const int b = box_of[s];
            if (b < 0) continue;
            tp.box_src[b] = s;
            const int tile[3] = {1, kTY, kTX};
            for (int i = 0; i < 3; ++i) {
                tp.box_lo[b][i] = lo[s][i];
                tp.box_ex[b][i] = tile[i] + hi[s][i] - lo[s][i];
            }
            if (tp.box_ex[b][2] > 32 * kChunks)
                return pfail(SP_ERR_UNSUPPORTED, "prefilter: tap offsets span more than 32 cells along axis 2");
            tp.box_off[b] = (int)off;
            off += (long long)tp.box_ex[b][0] * tp.box_ex[b][1] * tp.box_ex[b][2];
            off = (off + 3) & ~3ll;
            if (off * (long long)sizeof(T) > 160 * 1024)
                return pfail(SP_ERR_UNSUPPORTED, "prefilter: tap offsets span too large a box");
        }
        smem_max = std::max(smem_max, (int)(off * sizeof(T)));
        for (int t = 0; t < tp.n; ++t) {
            const int s = st->src_coset[t0 + t];
            const int b = box_of[s];
            const int* dz = st->dz + 3 * (t0 + t);
            tp.tap_box[t] = b;
            tp.tap_off[t] = tp.box_off[b] + ((dz[0] - lo[s][0]) * tp.box_ex[b][1] + (dz[1] - lo[s][1])) * tp.box_ex[b][2] +
                            (dz[2] - lo[s][2]);
            tp.w[t] = (T)st->weight[t0 + t];
        }
        P.out[k] = reinterpret_cast<T*>(out[k]);
    }
    if (smem_max == 0) {  // no taps anywhere: zero output
        for (int k = 0; k < in->M; ++k)
            cudaMemsetAsync(out[k], 0, (size_t)(in->extent[k][0] * in->extent[k][1] * in->extent[k][2]) * sizeof(T),
                            stream);
        return SP_OK;
    }
    int nt = P.c[0].n;
    for (int k = 1; k < in->M; ++k)
        if (P.c[k].n != nt) nt = 0;
    const dim3 grid((unsigned)((max_e[2] + kTX - 1) / kTX), (unsigned)((max_e[1] + kTY - 1) / kTY),
                    (unsigned)(max_e[0] * in->M));
    cudaError_t e = cudaSuccess;
    switch (nt) {
#define SP_PF_CASE(N)                                                                                      \
    case N:                                                                                                \
        e = cudaFuncSetAttribute(prefilter_tiled<T, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024); \
        if (e == cudaSuccess) prefilter_tiled<T, N><<<grid, kThreadsPF, smem_max, stream>>>(g, P);        \
        break;
        SP_PF_CASE(1) SP_PF_CASE(2) SP_PF_CASE(3) SP_PF_CASE(4) SP_PF_CASE(5) SP_PF_CASE(7) SP_PF_CASE(9)
        SP_PF_CASE(27)
        default:
            e = cudaFuncSetAttribute(prefilter_tiled<T, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
            if (e == cudaSuccess) prefilter_tiled<T, 0><<<grid, kThreadsPF, smem_max, stream>>>(g, P);
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
