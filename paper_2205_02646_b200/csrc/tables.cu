// tables.cu -- K1 "phase_tables": per-offset-class RL-JSDE tables, built on the
// device once per class and kept resident (replaces build_transform + fill_planes,
// /root/reference/proj/src/rljsde.cpp:22-102, and precompute_kernels 186-201).
//
//   k_transform : T_mk = sum_{3 px} (1/3) conj(unit[(eta*sigma + gamma*rho) mod W]),
//                 B_mk = w_m T_mk (rljsde.cpp:22-48, 60-68), fp64, k-major [k*L+m]
//   k_gram      : C[s,u] = sum_m B_{m,s} conj(T_{m,u}) for s >= u, fp64 accumulate in
//                 m order, upper half written as the exact conjugate (rljsde.cpp:77-99)
//   k_pack32    : D = Re diag C (rljsde.cpp:100); the fp32 product tables in rank
//                 order: s_r = sqrt(q/D), C'[s,u] = s_s C[s,u] (rounded once from fp64),
//                 fac_u = gamma/(s_u D_u)
//
// All classes that a frame needs are built in one batched launch per stage
// (grid.z = class), so the one-off precompute fills the GPU even at P = 8. The fp64
// planes are the cache (the reference's KernelSet); the fp32 product tables depend on
// per-call options (q through the frequency exponent, gamma) and are derived from the
// planes lazily per option set (launch_tables_derive).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "tqsb_internal.hpp"

namespace tqsb {
namespace {



__global__ void k_transform(const ClassBuild* __restrict__ cls, int W,
                            const double* __restrict__ unit64) {
    const ClassBuild c = cls[blockIdx.z];
    const int K = W * W, L = c.local;
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    const int k = blockIdx.y;
    if (m >= L || k >= K) return;
    const int sigma = k / W, rho = k % W;
    const double third = 1.0 / 3.0;
    double re = 0.0, im = 0.0;
#pragma unroll
    for (int t = 0; t < 3; ++t) {
        const int eta = c.px[m * 6 + 2 * t], gam = c.px[m * 6 + 2 * t + 1];
        const int idx = (eta * sigma + gam * rho) % W;
        re += third * unit64[2 * idx];
        im -= third * unit64[2 * idx + 1];  // conjugate basis
    }
    const size_t o = (size_t(k) * L + m) * 2;
    c.t64[o] = re;
    c.t64[o + 1] = im;
    const double w = c.w[m];
    c.b64[o] = w * re;
    c.b64[o + 1] = w * im;
}

// Lower-triangular complex GEMM, 64x64 output tiles, 16x16 threads x (4x4) outputs.
constexpr int GT = 64, GM = 16;

__global__ void __launch_bounds__(256) k_gram(const ClassBuild* __restrict__ cls, int W,
                                              int n_tiles) {
    const ClassBuild c = cls[blockIdx.z];
    const int K = W * W, L = c.local;
    // map the linear tile index to (si >= ui)
    int t = blockIdx.x, si = 0;
    while (t > si) { t -= si + 1; ++si; }
    const int ui = t;
    if (si >= n_tiles) return;
    const int s0 = si * GT, u0 = ui * GT;

    __shared__ double bre[GM][GT + 1], bim[GM][GT + 1], tre[GM][GT + 1], tim[GM][GT + 1];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    double ar[4][4], ai[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) ar[i][j] = ai[i][j] = 0.0;

    for (int m0 = 0; m0 < L; m0 += GM) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int idx = threadIdx.x + 256 * r;
            const int mm = idx % GM, kk = idx / GM;
            const int m = m0 + mm;
            const int s = s0 + kk, u = u0 + kk;
            double br = 0, bi = 0, tr = 0, ti = 0;
            if (m < L && s < K) {
                const size_t o = (size_t(s) * L + m) * 2;
                br = c.b64[o];
                bi = c.b64[o + 1];
            }
            if (m < L && u < K) {
                const size_t o = (size_t(u) * L + m) * 2;
                tr = c.t64[o];
                ti = c.t64[o + 1];
            }
            bre[mm][kk] = br;
            bim[mm][kk] = bi;
            tre[mm][kk] = tr;
            tim[mm][kk] = ti;
        }
        __syncthreads();
        const int mlim = min(GM, L - m0);
        for (int mm = 0; mm < mlim; ++mm) {
            double sr[4], sim[4], ur[4], uim[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                sr[i] = bre[mm][ty + 16 * i];
                sim[i] = bim[mm][ty + 16 * i];
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                ur[j] = tre[mm][tx + 16 * j];
                uim[j] = tim[mm][tx + 16 * j];
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    // accRe += sRe*uRe + sIm*uIm; accIm += sIm*uRe - sRe*uIm (rljsde.cpp:86-89),
                    // rounded like the reference build: acc + fma(a, b, c*d) per m
                    ar[i][j] = __dadd_rn(ar[i][j], __fma_rn(sr[i], ur[j], __dmul_rn(sim[i], uim[j])));
                    ai[i][j] = __dadd_rn(ai[i][j], __fma_rn(sim[i], ur[j], -__dmul_rn(sr[i], uim[j])));
                }
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int s = s0 + ty + 16 * i, u = u0 + tx + 16 * j;
            if (s >= K || u >= K || s < u) continue;
            const size_t lo = (size_t(u) * K + s) * 2;
            c.c64[lo] = ar[i][j];
            c.c64[lo + 1] = ai[i][j];
            if (s != u) {
                const size_t hi = (size_t(s) * K + u) * 2;
                c.c64[hi] = ar[i][j];
                c.c64[hi + 1] = -ai[i][j];
            }
        }
}

__global__ void k_diag(const ClassBuild* __restrict__ cls, int W) {
    const ClassBuild c = cls[blockIdx.z];
    const int K = W * W;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < K) c.d64[k] = c.c64[(size_t(k) * K + k) * 2];
}

// scale / fac in rank order
__global__ void k_scale(const ClassBuild* __restrict__ cls, int W, int k_pad,
                        const int* __restrict__ perm, const double* __restrict__ q64,
                        double step) {
    const ClassBuild c = cls[blockIdx.z];
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= k_pad || c.scale == nullptr) return;
    const int k = perm[r];
    float sc = __int_as_float(0x7fc00000), fa = 0.f;  // NaN marks inadmissible (D <= 0)
    if (k >= 0) {
        const double d = c.d64[k];
        if (d > 0.0) {
            const double s = sqrt(q64[k] / d);
            sc = float(s);
            fa = float(step / (s * d));
        }
    }
    c.scale[r] = sc;
    c.fac[r] = fa;
}

// C'[s,u] = s_s * C[s,u], column u_rank, float4 (re_a, re_b, im_a, im_b) per rank pair
__global__ void k_pack32(const ClassBuild* __restrict__ cls, int W, int k_pad,
                         const int* __restrict__ perm, const double* __restrict__ q64) {
    const ClassBuild c = cls[blockIdx.z];
    if (c.cpack == nullptr) return;
    const int K = W * W;
    const int ur = blockIdx.y;                                 // column rank
    const int pair = blockIdx.x * blockDim.x + threadIdx.x;    // rank pair index
    if (pair >= k_pad / 2) return;
    const int u = perm[ur];
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    const bool ucol = u >= 0 && c.d64[u] > 0.0;
    float o[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int b = 0; b < 2; ++b) {
        const int sr = 2 * pair + b;
        const int s = perm[sr];
        if (!ucol || s < 0) continue;
        const double d = c.d64[s];
        if (d > 0.0) {
            const double sc = sqrt(q64[s] / d);
            const size_t idx = (size_t(u) * K + s) * 2;
            o[b] = float(sc * c.c64[idx]);
            o[2 + b] = float(sc * c.c64[idx + 1]);
        } else {
            o[b] = __int_as_float(0x7fc00000);
            o[2 + b] = __int_as_float(0x7fc00000);
        }
    }
    v = make_float4(o[0], o[1], o[2], o[3]);
    // slot i = pair / 32, lane j = pair % 32  ->  float4 index i*32 + j == pair
    reinterpret_cast<float4*>(c.cpack)[size_t(ur) * (k_pad / 2) + pair] = v;
}

// bt[m*K + k] = b[k*L + m] (complex), into the T scratch once the Gram kernel is done
// with it: 32x32 tiles through shared memory, coalesced both ways
__global__ void k_transpose_b(const ClassBuild* __restrict__ cls, int W) {
    const ClassBuild c = cls[blockIdx.z];
    const int K = W * W, L = c.local;
    __shared__ double2 tile[32][33];
    const int k0 = blockIdx.y * 32, m0 = blockIdx.x * 32;
    const double2* b = reinterpret_cast<const double2*>(c.b64);
    double2* bt = reinterpret_cast<double2*>(c.t64);
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int k = k0 + i, m = m0 + threadIdx.x;
        if (k < K && m < L) tile[i][threadIdx.x] = b[size_t(k) * L + m];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int m = m0 + i, k = k0 + threadIdx.x;
        if (k < K && m < L) bt[size_t(m) * K + k] = tile[threadIdx.x][i];
    }
}

// The reference's Precision::Single planes (fill_planes<float>, rljsde.cpp:70-100): B, C
// and D stored as float from the double accumulations, widened to double in the loop
// (KernelPlanes::dAt and the update's casts) -- here rounded in place in the fp64 planes.
__global__ void k_round_single(const ClassBuild* __restrict__ cls, int W) {
    const ClassBuild c = cls[blockIdx.z];
    const size_t K = size_t(W) * W;
    const size_t nb = K * c.local * 2, nc = K * K * 2;
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nc; i += stride) {
        c.c64[i] = double(float(c.c64[i]));
        if (i < nb) c.b64[i] = double(float(c.b64[i]));
        if (i < K) c.d64[i] = double(float(c.d64[i]));
    }
}

} // namespace

// Batched fp64 plane build over n classes (k_transform, k_gram, k_diag, and the
// Precision::Single rounding); `descs` is a host array copied to the device here.
int launch_tables_build(const void* host_descs, int n, int window, const double* unit64,
                        int max_local, void* stream_, int* launches, int round_single) {
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    const ClassBuild* hd = static_cast<const ClassBuild*>(host_descs);
    ClassBuild* dd = nullptr;
    cudaError_t e = cudaMallocAsync(&dd, sizeof(ClassBuild) * n, stream);
    if (e != cudaSuccess) return e;
    e = cudaMemcpyAsync(dd, hd, sizeof(ClassBuild) * n, cudaMemcpyHostToDevice, stream);
    if (e != cudaSuccess) return e;
    const int K = window * window;
    for (int z0 = 0; z0 < n; z0 += 65535) {
        const int nz = n - z0 < 65535 ? n - z0 : 65535;
        const ClassBuild* d = dd + z0;
        {
            dim3 g((max_local + 127) / 128, K, nz);
            k_transform<<<g, 128, 0, stream>>>(d, window, unit64);
        }
        {
            const int nt = (K + GT - 1) / GT;
            dim3 g(nt * (nt + 1) / 2, 1, nz);
            k_gram<<<g, 256, 0, stream>>>(d, window, nt);
        }
        {
            dim3 g((K + 255) / 256, 1, nz);
            k_diag<<<g, 256, 0, stream>>>(d, window);
        }
        if (launches) *launches += 3;
        if (round_single) {
            dim3 g(4 * 148, 1, nz);
            k_round_single<<<g, 256, 0, stream>>>(d, window);
            if (launches) *launches += 1;
        }
        {
            dim3 g((max_local + 31) / 32, (K + 31) / 32, nz);
            k_transpose_b<<<g, dim3(32, 8), 0, stream>>>(d, window);
            if (launches) *launches += 1;
        }
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return cudaFreeAsync(dd, stream);
}

int launch_tables_transpose(const void* host_descs, int n, int window, int max_local, void* stream_,
                            int* launches) {
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    ClassBuild* dd = nullptr;
    cudaError_t e = cudaMallocAsync(&dd, sizeof(ClassBuild) * n, stream);
    if (e != cudaSuccess) return e;
    e = cudaMemcpyAsync(dd, host_descs, sizeof(ClassBuild) * n, cudaMemcpyHostToDevice, stream);
    if (e != cudaSuccess) return e;
    const int K = window * window;
    for (int z0 = 0; z0 < n; z0 += 65535) {
        const int nz = n - z0 < 65535 ? n - z0 : 65535;
        dim3 g((max_local + 31) / 32, (K + 31) / 32, nz);
        k_transpose_b<<<g, dim3(32, 8), 0, stream>>>(dd + z0, window);
        if (launches) *launches += 1;
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return cudaFreeAsync(dd, stream);
}

// The fp32 product tables of n classes for one (frequency exponent, step width):
// scale / fac (k_scale) and C' (k_pack32), derived from the resident fp64 planes.
int launch_tables_derive(const void* host_descs, int n, int window, int k_pad, double step,
                         const double* q64, const int* perm, void* stream_, int* launches) {
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    const ClassBuild* hd = static_cast<const ClassBuild*>(host_descs);
    ClassBuild* dd = nullptr;
    cudaError_t e = cudaMallocAsync(&dd, sizeof(ClassBuild) * n, stream);
    if (e != cudaSuccess) return e;
    e = cudaMemcpyAsync(dd, hd, sizeof(ClassBuild) * n, cudaMemcpyHostToDevice, stream);
    if (e != cudaSuccess) return e;
    (void)window;
    for (int z0 = 0; z0 < n; z0 += 65535) {
        const int nz = n - z0 < 65535 ? n - z0 : 65535;
        const ClassBuild* d = dd + z0;
        {
            dim3 g((k_pad + 255) / 256, 1, nz);
            k_scale<<<g, 256, 0, stream>>>(d, window, k_pad, perm, q64, step);
        }
        {
            dim3 g((k_pad / 2 + 127) / 128, k_pad, nz);
            k_pack32<<<g, 128, 0, stream>>>(d, window, k_pad, perm, q64);
        }
        if (launches) *launches += 2;
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return cudaFreeAsync(dd, stream);
}

} // namespace tqsb
