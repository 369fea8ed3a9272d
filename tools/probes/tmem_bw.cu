// TMEM read-bandwidth probe (tcgen05.ld.32x32b.x64) vs shared-memory LDS.128,
// 12 warps per CTA, 1 CTA per SM -- decides whether hot C' columns belong in TMEM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void __launch_bounds__(384, 1) k_tmem(float* out, int iters) {
    __shared__ uint32_t taddr_s;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&taddr_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = taddr_s + ((uint32_t)(32 * (warp & 3)) << 16);
    // fill: each warp of quadrant q (warps 0..3) writes its lane rows, 8 x 64 columns
    if (warp < 4) {
        for (int j = 0; j < 8; ++j) {
            uint32_t v[64];
#pragma unroll
            for (int i = 0; i < 64; ++i) v[i] = __float_as_uint(1.0f + 1e-3f * (i + lane + j));
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x64.b32 [%0], {"
                "%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,"
                "%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,"
                "%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63,%64};"
                ::"r"(base + 64 * j),
                "r"(v[0]),"r"(v[1]),"r"(v[2]),"r"(v[3]),"r"(v[4]),"r"(v[5]),"r"(v[6]),"r"(v[7]),
                "r"(v[8]),"r"(v[9]),"r"(v[10]),"r"(v[11]),"r"(v[12]),"r"(v[13]),"r"(v[14]),"r"(v[15]),
                "r"(v[16]),"r"(v[17]),"r"(v[18]),"r"(v[19]),"r"(v[20]),"r"(v[21]),"r"(v[22]),"r"(v[23]),
                "r"(v[24]),"r"(v[25]),"r"(v[26]),"r"(v[27]),"r"(v[28]),"r"(v[29]),"r"(v[30]),"r"(v[31]),
                "r"(v[32]),"r"(v[33]),"r"(v[34]),"r"(v[35]),"r"(v[36]),"r"(v[37]),"r"(v[38]),"r"(v[39]),
                "r"(v[40]),"r"(v[41]),"r"(v[42]),"r"(v[43]),"r"(v[44]),"r"(v[45]),"r"(v[46]),"r"(v[47]),
                "r"(v[48]),"r"(v[49]),"r"(v[50]),"r"(v[51]),"r"(v[52]),"r"(v[53]),"r"(v[54]),"r"(v[55]),
                "r"(v[56]),"r"(v[57]),"r"(v[58]),"r"(v[59]),"r"(v[60]),"r"(v[61]),"r"(v[62]),"r"(v[63]));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
        uint32_t r[64];
        const uint32_t a = base + 64 * ((it + warp) & 7);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x64.b32 {"
            "%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"
            "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,"
            "%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
            : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),
              "=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]),
              "=r"(r[16]),"=r"(r[17]),"=r"(r[18]),"=r"(r[19]),"=r"(r[20]),"=r"(r[21]),"=r"(r[22]),"=r"(r[23]),
              "=r"(r[24]),"=r"(r[25]),"=r"(r[26]),"=r"(r[27]),"=r"(r[28]),"=r"(r[29]),"=r"(r[30]),"=r"(r[31]),
              "=r"(r[32]),"=r"(r[33]),"=r"(r[34]),"=r"(r[35]),"=r"(r[36]),"=r"(r[37]),"=r"(r[38]),"=r"(r[39]),
              "=r"(r[40]),"=r"(r[41]),"=r"(r[42]),"=r"(r[43]),"=r"(r[44]),"=r"(r[45]),"=r"(r[46]),"=r"(r[47]),
              "=r"(r[48]),"=r"(r[49]),"=r"(r[50]),"=r"(r[51]),"=r"(r[52]),"=r"(r[53]),"=r"(r[54]),"=r"(r[55]),
              "=r"(r[56]),"=r"(r[57]),"=r"(r[58]),"=r"(r[59]),"=r"(r[60]),"=r"(r[61]),"=r"(r[62]),"=r"(r[63])
            : "r"(a));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        uint32_t x = 0;
#pragma unroll
        for (int i = 0; i < 64; ++i) x ^= r[i];
        acc += __uint_as_float(x);
    }
    if (acc == 12345.f) out[threadIdx.x] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr_s));
}

__global__ void __launch_bounds__(384, 1) k_lds(float* out, int iters) {
    extern __shared__ float4 sh[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 8 * 512; i += blockDim.x) sh[i] = make_float4(i, 1, 2, 3);
    __syncthreads();
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
        const float4* col = sh + 512 * ((it + warp) & 7);
        float4 r[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const unsigned ad = (unsigned)__cvta_generic_to_shared(col + i * 32 + lane);
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r[i].x), "=f"(r[i].y), "=f"(r[i].z), "=f"(r[i].w) : "r"(ad));
        }
        uint32_t x = 0;
#pragma unroll
        for (int i = 0; i < 16; ++i)
            x ^= __float_as_uint(r[i].x) ^ __float_as_uint(r[i].y) ^ __float_as_uint(r[i].z) ^ __float_as_uint(r[i].w);
        acc += __uint_as_float(x);
    }
    if (acc == 12345.f) out[threadIdx.x] = acc;
}


__global__ void __launch_bounds__(512, 1) k_tmem_rw(float* out, int iters) {
    __shared__ uint32_t taddr_s;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&taddr_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    // 16 warps: warp w owns columns 64*(w/4) .. +63 of quadrant w%4 (an R' mirror)
    const uint32_t base = taddr_s + ((uint32_t)(32 * (warp & 3)) << 16) + 64 * (warp >> 2);
    uint32_t x = lane;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t r[16];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),
                  "=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15])
                : "r"(base + 16 * q));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
            for (int i = 0; i < 16; ++i) r[i] ^= x + i;
            asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                :: "r"(base + 16 * q), "r"(r[0]),"r"(r[1]),"r"(r[2]),"r"(r[3]),"r"(r[4]),"r"(r[5]),"r"(r[6]),"r"(r[7]),
                  "r"(r[8]),"r"(r[9]),"r"(r[10]),"r"(r[11]),"r"(r[12]),"r"(r[13]),"r"(r[14]),"r"(r[15]));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;");
        x += 7;
    }
    if (x == 12345u) out[threadIdx.x] = x;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr_s));
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    CK(cudaMalloc(&out, 4096));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 20000;
    float ms;
    k_tmem<<<sms, 384>>>(out, 100);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    k_tmem<<<sms, 384>>>(out, iters);
    CK(cudaGetLastError());
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    double bytes = double(sms) * 12 * iters * 8192;
    printf("tmem  ld.32x32b.x64: %.3f ms  %.1f TB/s  %.1f B/clk/SM\n", ms, bytes / ms / 1e9,
           bytes / sms / (ms * 1e-3 * 1.965e9));
    CK(cudaFuncSetAttribute(k_lds, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    k_lds<<<sms, 384, 65536>>>(out, 100);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    k_lds<<<sms, 384, 65536>>>(out, iters);
    CK(cudaGetLastError());
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    printf("smem  LDS.128     : %.3f ms  %.1f TB/s  %.1f B/clk/SM\n", ms, bytes / ms / 1e9,
           bytes / sms / (ms * 1e-3 * 1.965e9));
    k_tmem_rw<<<sms, 512>>>(out, 100);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    k_tmem_rw<<<sms, 512>>>(out, iters);
    CK(cudaGetLastError());
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    bytes = double(sms) * 16 * iters * 8192;  // read + write each
    printf("tmem  R-mirror rw (4x ld.x16 + wait + st.x16, 16 warps): %.3f ms  %.1f B/clk/SM each way, %.0f cyc/warp-iter\n",
           ms, bytes / sms / (ms * 1e-3 * 1.965e9), ms * 1e-3 * 1.965e9 / iters);
    return 0;
}
