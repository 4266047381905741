// Probe: MSD multisplit of {x, y, z, index} records by Morton-key digits with CTA-staged,
// coalesced run writes (protocol B without a radix sort of the points).
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/msd_probe tools/micro/msd_probe.cu
//   /tmp/msd_probe [n]
//
// Level 0: histogram of the brick key (top KB bits of the 24-bit Morton key of a point in
// [0,256)^3) + exclusive scan -> brick starts.  Pass 1: split by the top K1 bits into
// bucket order.  Pass 2: split each pass-1 bucket by the remaining brick bits.  Pass 3: sort
// each brick by the in-brick Morton bits in shared memory.
#include <cuda_runtime.h>
#include <cub/cub.cuh>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

constexpr int KEYB = 24;  // 8 bits per axis
constexpr int KB = 15;    // brick key bits (8^3-cell bricks)
constexpr int K1 = 10;    // pass-1 digit
constexpr int K2 = KB - K1;

__device__ __forceinline__ unsigned spread3(unsigned v) {
    v &= 0x3ff;
    v = (v | (v << 16)) & 0x030000FF;
    v = (v | (v << 8)) & 0x0300F00F;
    v = (v | (v << 4)) & 0x030C30C3;
    v = (v | (v << 2)) & 0x09249249;
    return v;
}
__device__ __forceinline__ unsigned morton(float x, float y, float z) {
    const unsigned a = min(max((int)x, 0), 255), b = min(max((int)y, 0), 255), c = min(max((int)z, 0), 255);
    return (spread3(a) << 2) | (spread3(b) << 1) | spread3(c);
}

__global__ void gen_kernel(float* p, long long n, unsigned seed) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < 3 * n; i += (long long)gridDim.x * blockDim.x) {
        unsigned h = (unsigned)i * 2654435761u ^ seed;
        h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
        p[i] = (h >> 8) * (256.0f / 16777216.0f);
    }
}

__global__ void hist_kernel(const float* __restrict__ p, int n, int* __restrict__ ghist) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const unsigned k = morton(p[3 * i], p[3 * i + 1], p[3 * i + 2]) >> (KEYB - KB);
        atomicAdd(&ghist[k], 1);
    }
}

__global__ void hist_smem_kernel(const float* __restrict__ p, int n, int* __restrict__ ghist) {
    extern __shared__ int sh[];
    constexpr int NB = 1 << KB;
    for (int i = threadIdx.x; i < NB; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const unsigned k = morton(p[3 * i], p[3 * i + 1], p[3 * i + 2]) >> (KEYB - KB);
        atomicAdd(&sh[k], 1);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < NB; i += blockDim.x)
        if (sh[i]) atomicAdd(&ghist[i], sh[i]);
}

// Pass 1 / pass 2: split tiles of T records by a digit; cursors are per digit value (global).
template <int NT, int T, int DB, bool FIRST>
__global__ void __launch_bounds__(NT) split_kernel(const float* __restrict__ pts, const float4* __restrict__ in, int n,
                                                   const int* __restrict__ tile_begin, int ntiles,
                                                   const int* __restrict__ tile_end, int* __restrict__ cursor,
                                                   float4* __restrict__ out) {
    constexpr int NB = 1 << DB;
    constexpr int PPT = T / NT;
    extern __shared__ float4 stage[];
    __shared__ int h[NB], gb[NB];
    typedef cub::BlockScan<int, NT> Scan;
    __shared__ typename Scan::TempStorage scan_tmp;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int b0 = FIRST ? t * T : tile_begin[t];
        const int b1 = FIRST ? min(n, b0 + T) : tile_end[t];
        for (int i = threadIdx.x; i < NB; i += NT) h[i] = 0;
        __syncthreads();
        float4 rec[PPT];
        int dig[PPT], rk[PPT];
        unsigned hi_pref = 0;
#pragma unroll
        for (int j = 0; j < PPT; ++j) {
            const int i = b0 + j * NT + threadIdx.x;
            dig[j] = -1;
            if (i < b1) {
                if (FIRST) rec[j] = make_float4(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], __int_as_float(i));
                else rec[j] = in[i];
                const unsigned k = morton(rec[j].x, rec[j].y, rec[j].z) >> (KEYB - KB);
                dig[j] = FIRST ? (int)(k >> (KB - DB)) : (int)(k & (NB - 1));
                if (!FIRST) hi_pref = k >> DB;
                rk[j] = atomicAdd(&h[dig[j]], 1);
            }
        }
        __syncthreads();
        // exclusive scan of the digit histogram
        constexpr int IPT = (NB + NT - 1) / NT;
        int v[IPT];
#pragma unroll
        for (int q = 0; q < IPT; ++q) { const int d = threadIdx.x * IPT + q; v[q] = d < NB ? h[d] : 0; }
        int cnt[IPT];
#pragma unroll
        for (int q = 0; q < IPT; ++q) cnt[q] = v[q];
        Scan(scan_tmp).ExclusiveSum(v, v);
        __syncthreads();
        // reserve global runs; keep the local offsets in h, the global bases in gb
        unsigned pref = 0;
        if (!FIRST) {
            // all records of a pass-2 tile share the pass-1 digit
            __shared__ unsigned s_pref;
            if (threadIdx.x == 0) s_pref = 0;
            __syncthreads();
            if (dig[0] >= 0) s_pref = hi_pref;
            __syncthreads();
            pref = s_pref;
        }
#pragma unroll
        for (int q = 0; q < IPT; ++q) {
            const int d = threadIdx.x * IPT + q;
            if (d < NB) {
                gb[d] = cnt[q] ? atomicAdd(&cursor[FIRST ? d : (int)(pref << DB) + d], cnt[q]) : 0;
                h[d] = v[q];
            }
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < PPT; ++j)
            if (dig[j] >= 0) stage[h[dig[j]] + rk[j]] = rec[j];
        __syncthreads();
        const int m = b1 - b0;
        for (int s = threadIdx.x; s < m; s += NT) {
            const float4 r = stage[s];
            const unsigned k = morton(r.x, r.y, r.z) >> (KEYB - KB);
            const int d = FIRST ? (int)(k >> (KB - DB)) : (int)(k & (NB - 1));
            out[gb[d] + s - h[d]] = r;
        }
        __syncthreads();
    }
}

// Pass 3: one CTA per brick (grid-stride), counting sort by the 9 in-brick Morton bits.
template <int NT, int CAP>
__global__ void __launch_bounds__(NT) brick_sort_kernel(float4* __restrict__ rec, const int* __restrict__ start, int nbricks) {
    extern __shared__ float4 stage[];
    __shared__ int h[512];
    typedef cub::BlockScan<int, NT> Scan;
    __shared__ typename Scan::TempStorage scan_tmp;
    for (int b = blockIdx.x; b < nbricks; b += gridDim.x) {
        const int p0 = start[b], p1 = start[b + 1], m = p1 - p0;
        if (m > CAP) continue;  // left unsorted (correct, just slower to evaluate)
        for (int i = threadIdx.x; i < 512; i += NT) h[i] = 0;
        __syncthreads();
        for (int s = threadIdx.x; s < m; s += NT) {
            const float4 r = rec[p0 + s];
            stage[s] = r;
            atomicAdd(&h[morton(r.x, r.y, r.z) & 511], 1);
        }
        __syncthreads();
        constexpr int IPT = 512 / NT;
        int v[IPT];
#pragma unroll
        for (int q = 0; q < IPT; ++q) v[q] = h[threadIdx.x * IPT + q];
        Scan(scan_tmp).ExclusiveSum(v, v);
        __syncthreads();
#pragma unroll
        for (int q = 0; q < IPT; ++q) h[threadIdx.x * IPT + q] = v[q];
        __syncthreads();
        for (int s = threadIdx.x; s < m; s += NT) {
            const float4 r = stage[s];
            rec[p0 + atomicAdd(&h[morton(r.x, r.y, r.z) & 511], 1)] = r;
        }
        __syncthreads();
    }
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 100000000;
    constexpr int NBR = 1 << KB;
    float* pts;
    float4 *r1, *r2;
    int *hist, *start, *cur1, *cur2, *tb, *te;
    CK(cudaMalloc(&pts, 12ll * n));
    CK(cudaMalloc(&r1, 16ll * n));
    CK(cudaMalloc(&r2, 16ll * n));
    CK(cudaMalloc(&hist, 4 * (NBR + 1)));
    CK(cudaMalloc(&start, 4 * (NBR + 1)));
    CK(cudaMalloc(&cur1, 4 * (1 << K1)));
    CK(cudaMalloc(&cur2, 4 * NBR));
    const int maxt2 = n / 2048 + (1 << K1) + 8;
    CK(cudaMalloc(&tb, 4 * maxt2));
    CK(cudaMalloc(&te, 4 * maxt2));
    gen_kernel<<<1184, 256>>>(pts, n, 12345u);
    void* tmp = nullptr;
    size_t tmpb = 0;
    cub::DeviceScan::ExclusiveSum(tmp, tmpb, hist, start, NBR + 1);
    CK(cudaMalloc(&tmp, tmpb));
#ifndef PNT
#define PNT 512
#define PT 8192
#endif
    constexpr int NT = PNT, T = PT;
    CK(cudaFuncSetAttribute(hist_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 << KB));
    int occ1 = 0;
    auto k1 = split_kernel<NT, T, K1, true>;
    auto k2 = split_kernel<NT, T, K2, false>;
    auto k3 = brick_sort_kernel<256, 12288>;
    CK(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, T * 16));
    CK(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, T * 16));
    CK(cudaFuncSetAttribute(k3, cudaFuncAttributeMaxDynamicSharedMemorySize, 12288 * 16));
    cudaEvent_t e[6];
    for (auto& x : e) cudaEventCreate(&x);
    std::vector<int> hs(NBR + 1);
    for (int it = 0; it < 6; ++it) {
        cudaEventRecord(e[0]);
        CK(cudaMemsetAsync(hist, 0, 4 * (NBR + 1)));
        if (getenv("HIST_GLOBAL")) hist_kernel<<<148 * 8, 256>>>(pts, n, hist);
        else hist_smem_kernel<<<148, 1024, 4 << KB>>>(pts, n, hist);
        cub::DeviceScan::ExclusiveSum(tmp, tmpb, hist, start, NBR + 1);
        cudaEventRecord(e[1]);
        // cursors: pass 1 at bucket starts, pass 2 at brick starts (device copies)
        CK(cudaMemcpyAsync(cur2, start, 4 * NBR, cudaMemcpyDeviceToDevice));
        CK(cudaMemcpy(hs.data(), start, 4 * (NBR + 1), cudaMemcpyDeviceToHost));  // probe only: tile lists on the host
        std::vector<int> c1(1 << K1), vb, ve;
        for (int d = 0; d < (1 << K1); ++d) {
            c1[d] = hs[d << K2];
            const int a = hs[d << K2], z = hs[(d + 1) << K2];
            for (int q = a; q < z; q += T) { vb.push_back(q); ve.push_back(std::min(z, q + T)); }
        }
        CK(cudaMemcpy(cur1, c1.data(), 4 * c1.size(), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(tb, vb.data(), 4 * vb.size(), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(te, ve.data(), 4 * ve.size(), cudaMemcpyHostToDevice));
        cudaEventRecord(e[2]);
        const int nt1 = (n + T - 1) / T;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ1, k1, NT, T * 16);
        k1<<<148 * occ1, NT, T * 16>>>(pts, nullptr, n, nullptr, nt1, nullptr, cur1, r1);
        cudaEventRecord(e[3]);
        k2<<<148 * occ1, NT, T * 16>>>(nullptr, r1, n, tb, (int)vb.size(), te, cur2, r2);
        cudaEventRecord(e[4]);
        k3<<<148 * 2, 256, 12288 * 16>>>(r2, start, NBR);
        cudaEventRecord(e[5]);
        CK(cudaEventSynchronize(e[5]));
        float t[5];
        for (int q = 0; q < 5; ++q) cudaEventElapsedTime(&t[q], e[q], e[q + 1]);
        printf("occ %d  hist+scan %.3f  (host tiles %.3f)  pass1 %.3f  pass2 %.3f  pass3 %.3f ms\n", occ1, t[0], t[1], t[2], t[3], t[4]);
    }
    CK(cudaGetLastError());
    // verify: r2 grouped by brick, every index once, sorted within bricks
    std::vector<float4> h2(n);
    CK(cudaMemcpy(h2.data(), r2, 16ll * n, cudaMemcpyDeviceToHost));
    std::vector<char> seen(n, 0);
    auto mort = [](float x, float y, float z) {
        auto sp = [](unsigned v) { unsigned r = 0; for (int b = 0; b < 8; ++b) r |= ((v >> b) & 1u) << (3 * b); return r; };
        unsigned a = std::min(std::max((int)x, 0), 255), b = std::min(std::max((int)y, 0), 255), c = std::min(std::max((int)z, 0), 255);
        return (sp(a) << 2) | (sp(b) << 1) | sp(c);
    };
    long long bad = 0, unsorted = 0;
    for (int br = 0; br < NBR; ++br)
        for (int i = hs[br]; i < hs[br + 1]; ++i) {
            const float4 r = h2[i];
            int idx; memcpy(&idx, &r.w, 4);
            if (idx < 0 || idx >= n || seen[idx]) { ++bad; continue; }
            seen[idx] = 1;
            const unsigned k = mort(r.x, r.y, r.z);
            if ((int)(k >> (KEYB - KB)) != br) ++bad;
            if (i > hs[br] && k < mort(h2[i - 1].x, h2[i - 1].y, h2[i - 1].z)) ++unsorted;
        }
    printf("verify: bad %lld unsorted-pairs %lld\n", bad, unsorted);
    return bad != 0;
}
