// sp_texture.cu — hardware-texture-filtered variant of the tensor-product reconstruction.
//
// The paper's GPU path (§4.4) merges adjacent coefficient reads into
// hardware (tri)linear texture fetches: TEX3D(tex_coset, a' + t(x)(b' - a')).  The exact
// kernels of this library do that merge in software (local lerp on exact integer cells,
// SURVEY.md fact 4) because texture filtering weights are 9-bit fixed point (8 fractional
// bits).  This file provides the hardware variant for comparison, reported separately with
// its measured error (bench.py "texture_variant"):
//   * trilinear: one filtered fetch per point,
//   * tricubic: 8 filtered fetches per point (per axis the 4 B-spline weights fold into two
//     lerps, g0 = w0 + w1 at a0 + w1/g0 and g1 = w2 + w3 at a2 + w3/g1).
// Non-centred convention: site floor(x) - DEG + a carries weight w_a.
// Texel i of axis k holds array index i, i.e. lattice site i + origin_k; texel centres are at
// i + 0.5 in unnormalised coordinates.
#include <cuda_runtime.h>

#include <cstdio>
#include <string>

#include "../../include/splinerecon.h"
#include "sp_evaluators.cuh"
#include "sp_launch.cuh"

struct sp_texture {
    int M = 0;
    cudaArray_t array[SP_MAX_COSETS] = {};
    cudaTextureObject_t texs[SP_MAX_COSETS] = {};
    cudaTextureObject_t tex = 0;  // coset 0 (tensor-product kernels)
    int origin[3] = {0, 0, 0};    // coset 0
    sp_grid_desc desc{};          // extents / origins / policy of every coset (data pointers unused)
};

namespace sp {
void set_error(const std::string& msg);  // splinerecon.cu (feeds sp_last_error)
int eval_texture_generated(const sp_plan* p, const sp_grid_desc* g, const TexArgs& targs, const void* pts, int64_t n,
                           void* out, int32_t* err, cudaStream_t st);  // splinerecon.cu
}

namespace {

int tfail(int code, const char* msg, cudaError_t e = cudaSuccess) {
    std::string m = msg;
    if (e != cudaSuccess) {
        m += ": ";
        m += cudaGetErrorString(e);
    }
    sp::set_error(m);
    return code;
}

__device__ __forceinline__ float tap(cudaTextureObject_t t, float u0, float u1, float u2) {
    return tex3D<float>(t, u2, u1, u0);  // x = contiguous axis 2
}

__global__ void __launch_bounds__(256) tex_trilinear(cudaTextureObject_t t, const float* __restrict__ pts, long long n,
                                                     float* __restrict__ out, int o0, int o1, int o2) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const float x0 = pts[3 * i], x1 = pts[3 * i + 1], x2 = pts[3 * i + 2];
        // sites floor(x)-1 (weight 1-t) and floor(x) (weight t): texel coordinate x - 1 - o + 0.5
        out[i] = tap(t, x0 - (float)o0 - 0.5f, x1 - (float)o1 - 0.5f, x2 - (float)o2 - 0.5f);
    }
}

__global__ void __launch_bounds__(256) tex_tricubic(cudaTextureObject_t t, const float* __restrict__ pts, long long n,
                                                    float* __restrict__ out, int o0, int o1, int o2) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const float x[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
        const int o[3] = {o0, o1, o2};
        float g[3][2], h[3][2];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float fl = floorf(x[k]);
            float w[4];
            sp::BWeights<3>::w(x[k] - fl, w);
            const float base = fl - (float)o[k];  // array index of site floor(x)
            g[k][0] = w[0] + w[1];
            g[k][1] = w[2] + w[3];
            h[k][0] = base - 3.0f + w[1] / g[k][0] + 0.5f;
            h[k][1] = base - 1.0f + w[3] / g[k][1] + 0.5f;
        }
        float acc = 0.0f;
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int b = 0; b < 2; ++b)
#pragma unroll
                for (int c = 0; c < 2; ++c)
                    acc = fmaf(g[0][a] * g[1][b] * g[2][c], tap(t, h[0][a], h[1][b], h[2][c]), acc);
        out[i] = acc;
    }
}

}  // namespace

extern "C" void sp_texture_destroy(sp_texture* t) {
    if (!t) return;
    for (int k = 0; k < t->M; ++k) {
        if (t->texs[k]) cudaDestroyTextureObject(t->texs[k]);
        if (t->array[k]) cudaFreeArray(t->array[k]);
    }
    delete t;
}

extern "C" int sp_texture_create(const sp_grid_desc* grid, sp_texture** out) {
    if (!grid || !out) return tfail(SP_ERR_INVALID, "null argument");
    *out = nullptr;
    if (grid->s != 3 || grid->M < 1 || grid->M > SP_MAX_COSETS) return tfail(SP_ERR_UNSUPPORTED, "texture variant: 3-D grids only");
    if (grid->dtype != SP_F32) return tfail(SP_ERR_UNSUPPORTED, "texture variant: float32 grids only");
    if (grid->boundary == SP_MIRROR)
        return tfail(SP_ERR_UNSUPPORTED, "texture variant: hardware mirror (period 2n) differs from runtime.py:191-196");
    sp_texture* t = new sp_texture();
    t->M = grid->M;
    t->desc = *grid;
    for (int i = 0; i < 3; ++i) t->origin[i] = (int)grid->origin[0][i];
    for (int k = 0; k < grid->M; ++k) {  // one 3-D array + linear-filtered texture object per coset
        const cudaExtent ext = make_cudaExtent(grid->extent[k][2], grid->extent[k][1], grid->extent[k][0]);
        cudaChannelFormatDesc ch = cudaCreateChannelDesc<float>();
        cudaError_t e = cudaMalloc3DArray(&t->array[k], &ch, ext);
        if (e != cudaSuccess) { sp_texture_destroy(t); return tfail(SP_ERR_CUDA, "cudaMalloc3DArray", e); }
        cudaMemcpy3DParms cp = {};
        cp.srcPtr = make_cudaPitchedPtr(const_cast<void*>(grid->data[k]), grid->extent[k][2] * sizeof(float),
                                        grid->extent[k][2], grid->extent[k][1]);
        cp.dstArray = t->array[k];
        cp.extent = ext;
        cp.kind = cudaMemcpyDeviceToDevice;
        e = cudaMemcpy3D(&cp);
        if (e != cudaSuccess) { sp_texture_destroy(t); return tfail(SP_ERR_CUDA, "cudaMemcpy3D", e); }
        cudaResourceDesc rd = {};
        rd.resType = cudaResourceTypeArray;
        rd.res.array.array = t->array[k];
        cudaTextureDesc td = {};
        const cudaTextureAddressMode am = grid->boundary == SP_ZERO ? cudaAddressModeBorder : cudaAddressModeClamp;
        td.addressMode[0] = td.addressMode[1] = td.addressMode[2] = am;
        td.filterMode = cudaFilterModeLinear;
        td.readMode = cudaReadModeElementType;
        td.normalizedCoords = 0;
        e = cudaCreateTextureObject(&t->texs[k], &rd, &td, nullptr);
        if (e != cudaSuccess) { sp_texture_destroy(t); return tfail(SP_ERR_CUDA, "cudaCreateTextureObject", e); }
    }
    t->tex = t->texs[0];
    *out = t;
    return SP_OK;
}

extern "C" int sp_eval_texture(const sp_plan* plan, const sp_texture* t, const void* pts, int64_t n, void* out,
                               void* stream) {
    if (!plan || !t) return tfail(SP_ERR_INVALID, "null plan or texture");
    if (n <= 0) return SP_OK;
    cudaStream_t st0 = reinterpret_cast<cudaStream_t>(stream);
    if (sp_plan_kernel_kind(plan) == SP_KIND_GENERATED) {  // box splines: per-coset textures, TexFetch
        sp::TexArgs targs{};
        for (int k = 0; k < t->M; ++k) targs.tex[k] = t->texs[k];
        sp_grid_desc g = t->desc;
        return sp::eval_texture_generated(plan, &g, targs, pts, n, out, nullptr, st0);
    }
    if (sp_plan_kernel_kind(plan) != SP_KIND_TENSOR_BSPLINE || t->M != 1)
        return tfail(SP_ERR_UNSUPPORTED, "texture variant: tensor-product or compiled box-spline plans only");
    const std::string name = sp_plan_kernel_name(plan);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const long long blocks = std::min<long long>((n + 255) / 256, 148ll * 32);
    if (name == "tensor_bspline_1")
        tex_trilinear<<<(int)blocks, 256, 0, st>>>(t->tex, (const float*)pts, n, (float*)out, t->origin[0], t->origin[1],
                                                  t->origin[2]);
    else if (name == "tensor_bspline_3")
        tex_tricubic<<<(int)blocks, 256, 0, st>>>(t->tex, (const float*)pts, n, (float*)out, t->origin[0], t->origin[1],
                                                 t->origin[2]);
    else
        return tfail(SP_ERR_UNSUPPORTED, "texture variant: degrees 1 and 3");
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return tfail(SP_ERR_CUDA, "texture kernel launch", e);
    return SP_OK;
}
