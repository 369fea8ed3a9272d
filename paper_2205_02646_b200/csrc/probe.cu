// probe.cu -- roofline denominators that MEASURED_PEAKS.json does not carry:
// the FP32 pipe peak (FFMA2, the instruction the solve kernel's update runs on)
// and the shared-memory load bandwidth (LDS.128, the path its C' columns take).
// Timed with CUDA events on the device; used by bench.py for roofline.peak.
#include <cuda_runtime.h>

#include "tqsb_internal.hpp"

namespace tqsb {
namespace {

__global__ void __launch_bounds__(256) k_ffma2(float* out, int iters, float a0) {
    float2 acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = make_float2(a0 + j, a0 - j + threadIdx.x * 1e-7f);
    const float2 m = make_float2(0.9999f, 1.0001f), c = make_float2(1e-7f, -1e-7f);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = __ffma2_rn(acc[j], m, c);
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += acc[j].x + acc[j].y;
    if (s == 12345.678f) out[threadIdx.x] = s;  // keep the chain alive
}

__global__ void __launch_bounds__(512) k_lds(float* out, int iters) {
    extern __shared__ float4 sh[];
    const int n = 8192;  // 128 KB
    for (int i = threadIdx.x; i < n; i += blockDim.x) sh[i] = make_float4(i, i, i, i);
    __syncthreads();
    float4 acc = make_float4(0, 0, 0, 0);
    int idx = threadIdx.x;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const float4 v = sh[(idx + j * 512) & (n - 1)];
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
        idx += 37;
    }
    if (acc.x + acc.y + acc.z + acc.w == 1.2345f) out[threadIdx.x] = acc.x;
}

} // namespace

int probe_peaks(int device, double* fp32_tflops, double* smem_tbps) {
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return e;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    float* out = nullptr;
    if ((e = cudaMalloc(&out, 4096))) return e;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms = 0.f;
    // FP32: 8 CTAs x 256 threads per SM, 8 independent FFMA2 chains per thread. The
    // clocks ramp from idle first (~0.3 s of the same load), then the median of five
    // ~40 ms launches is taken -- a single short launch reads low (clock ramp).
    const int iters = 4096 * 72, grid = sms * 8;
    k_ffma2<<<grid, 256>>>(out, 64, 1.f);
    for (int w = 0; w < 8; ++w) k_ffma2<<<grid, 256>>>(out, iters, 1.f);
    float runs[5];
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a);
        k_ffma2<<<grid, 256>>>(out, iters, 1.f);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&runs[r], a, b);
    }
    for (int i = 0; i < 5; ++i)  // median of five
        for (int j = i + 1; j < 5; ++j)
            if (runs[j] < runs[i]) { const float t = runs[i]; runs[i] = runs[j]; runs[j] = t; }
    ms = runs[2];
    const double flops = double(grid) * 256 * iters * 8 * 4;  // FFMA2 = 2 FMA = 4 flop
    if (fp32_tflops) *fp32_tflops = flops / (ms * 1e-3) / 1e12;
    // shared memory: 1 CTA of 512 threads per SM, LDS.128 stream
    cudaFuncSetAttribute(k_lds, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
    const int liters = 2048;
    k_lds<<<sms, 512, 131072>>>(out, 16);
    cudaEventRecord(a);
    k_lds<<<sms, 512, 131072>>>(out, liters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = double(sms) * 512 * liters * 8 * 16;
    if (smem_tbps) *smem_tbps = bytes / (ms * 1e-3) / 1e12;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(out);
    return cudaGetLastError();
}

} // namespace tqsb
