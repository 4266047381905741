// sp_render.cu — ray-marcher kernels around the reconstruction (SURVEY.md §8f rank 3,
// SPEC.md render_volume): the sample points of a slab of ray steps, and front-to-back
// compositing of the reconstructed values through a piecewise-linear transfer function.
//
// A frame is: for each slab of steps, sp_ray_points -> sp_eval (chunk kernel; the points of
// one ray are contiguous, so each CTA stages a compact box) -> sp_composite.  Both kernels
// here are streaming (12 B written per point, 4 B read per value, 32 B of state per pixel
// per slab) and negligible next to the reconstruction.
//
// sp_ray_points reproduces render.ray_points' float64 arithmetic operation for operation
// (no FMA contraction: __dmul_rn / __dadd_rn), so the float32 points are identical to the
// host's; sp_composite is the textbook sequential front-to-back loop in float64.
#include <cuda_runtime.h>

#include <string>

#include "../../include/splinerecon.h"

namespace sp {
void set_error(const std::string& msg);  // splinerecon.cu (feeds sp_last_error)
}

namespace {

constexpr int kMaxTf = SP_MAX_TRANSFER;

__global__ void ray_points_kernel(const sp_camera cam, int width, int height, int k0, int k1, float* __restrict__ out) {
    const int ns = k1 - k0;
    const long long total = (long long)width * height * ns;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long pix = i / ns;
        const int s = (int)(i - pix * ns);
        const int py = (int)(pix / width), px = (int)(pix - (long long)py * width);
        // render.ray_points: u = (px + 0.5) / w - 0.5, v = 0.5 - (py + 0.5) / h
        const double u = __dadd_rn(__ddiv_rn(__dadd_rn((double)px, 0.5), (double)width), -0.5);
        const double v = __dadd_rn(0.5, -__ddiv_rn(__dadd_rn((double)py, 0.5), (double)height));
        const double span_y = __ddiv_rn(__dmul_rn(cam.fov, (double)height), (double)width);
        const double t = __dmul_rn(__dadd_rn((double)(k0 + s), 0.5), cam.step);
        const double vs = __dmul_rn(v, span_y), uf = __dmul_rn(u, cam.fov);
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            // org = (position + (v*span_y)*up) + (u*fov)*right ; p = org + t*fwd ; lattice = p*scale + off
            const double org = __dadd_rn(__dadd_rn(cam.position[a], __dmul_rn(vs, cam.up[a])), __dmul_rn(uf, cam.right[a]));
            const double p = __dadd_rn(org, __dmul_rn(t, cam.forward[a]));
            out[3 * i + a] = (float)__dadd_rn(__dmul_rn(p, cam.lattice_scale), cam.lattice_offset[a]);
        }
    }
}

__device__ __forceinline__ void transfer(const double* tf, int ntf, double v, double c[4]) {
    // piecewise-linear (value, r, g, b, a) control points, clamped outside (render.TransferFunction)
    v = fmin(fmax(v, tf[0]), tf[5 * (ntf - 1)]);
    int i = 1;
    while (i < ntf - 1 && tf[5 * i] <= v) ++i;
    const double x0 = tf[5 * (i - 1)], x1 = tf[5 * i];
    const double w = (v - x0) / (x1 - x0);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const double a = tf[5 * (i - 1) + 1 + q], b = tf[5 * i + 1 + q];
        c[q] = a + w * (b - a);
    }
}

template <typename T>
__global__ void composite_kernel(const T* __restrict__ values, long long npix, int nsteps, const sp_transfer tfd,
                                 double* __restrict__ state) {
    __shared__ double tf[5 * kMaxTf];
    for (int i = threadIdx.x; i < 5 * tfd.n; i += blockDim.x) tf[i] = tfd.points[i];  // by-value kernel parameter
    __syncthreads();
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < npix; p += (long long)gridDim.x * blockDim.x) {
        double* st = state + 4 * p;  // r, g, b, transmittance
        double r = st[0], g = st[1], b = st[2], tr = st[3];
        const T* vp = values + p * nsteps;
        for (int s = 0; s < nsteps; ++s) {
            double c[4];
            transfer(tf, tfd.n, (double)vp[s], c);
            const double w = tr * c[3];
            r += w * c[0];
            g += w * c[1];
            b += w * c[2];
            tr *= 1.0 - c[3];
        }
        st[0] = r;
        st[1] = g;
        st[2] = b;
        st[3] = tr;
    }
}

int grid_for(long long work, int threads) {
    long long b = (work + threads - 1) / threads;
    return (int)(b < 1 ? 1 : (b > 148 * 64 ? 148 * 64 : b));
}

}  // namespace

extern "C" int sp_ray_points(const sp_camera* cam, int32_t width, int32_t height, int32_t k0, int32_t k1, float* out,
                             void* stream) {
    if (!cam || !out || width <= 0 || height <= 0 || k1 <= k0 || k0 < 0) {
        sp::set_error("sp_ray_points: invalid arguments");
        return SP_ERR_INVALID;
    }
    const long long total = (long long)width * height * (k1 - k0);
    ray_points_kernel<<<grid_for(total, 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(*cam, width, height, k0,
                                                                                                 k1, out);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        sp::set_error(std::string("sp_ray_points: ") + cudaGetErrorString(e));
        return SP_ERR_CUDA;
    }
    return SP_OK;
}

extern "C" int sp_composite(const void* values, int32_t dtype, int64_t npix, int32_t nsteps, const sp_transfer* tf,
                            double* state, void* stream) {
    if (!values || !tf || !state || npix < 0 || nsteps < 0 || tf->n < 2 || tf->n > SP_MAX_TRANSFER) {
        sp::set_error("sp_composite: invalid arguments");
        return SP_ERR_INVALID;
    }
    if (npix == 0 || nsteps == 0) return SP_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (dtype == SP_F32)
        composite_kernel<float><<<grid_for(npix, 128), 128, 0, st>>>(static_cast<const float*>(values), npix, nsteps, *tf, state);
    else if (dtype == SP_F64)
        composite_kernel<double><<<grid_for(npix, 128), 128, 0, st>>>(static_cast<const double*>(values), npix, nsteps, *tf, state);
    else {
        sp::set_error("sp_composite: unknown dtype");
        return SP_ERR_INVALID;
    }
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        sp::set_error(std::string("sp_composite: ") + cudaGetErrorString(e));
        return SP_ERR_CUDA;
    }
    return SP_OK;
}
