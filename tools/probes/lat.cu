// lat.cu -- dependent-chain latencies of the instructions on the solve kernel's
// selection chain (one warp, clock64 around N chained ops):
//   CREDUX (redux.sync.max.f32), REDUX (redux.sync.max.u32), SHFL, VOTE+FLO,
//   LDS, LDTM (tcgen05.ld.32x32b.x4 + wait::ld), a 5-deep uniform branch tree.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lat lat.cu && ./lat
#include <cstdio>
#include <cstdint>

__device__ unsigned long long g_out[16];

__global__ void k_lat(int n, float seed, int sel) {
    const int lane = threadIdx.x & 31;
    __shared__ float sh[1024];
    __shared__ uint32_t s_tmem;
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sh[i] = float(i & 7);
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
        static_cast<unsigned>(__cvta_generic_to_shared(&s_tmem))));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = s_tmem;
    {
        const uint32_t v = 0;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %1, %1, %1};" ::"r"(tm), "r"(v) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    float x = seed + lane;
    unsigned u = __float_as_uint(x);
    unsigned long long t0 = 0, t1 = 0;
    // 0: CREDUX f32
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
        float m;
        asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(m) : "f"(x));
        x = m * 0.5f + lane;
    }
    t1 = clock64();
    if (lane == 0) g_out[0] = (t1 - t0);
    // 1: REDUX u32
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
        unsigned m;
        asm volatile("redux.sync.max.u32 %0, %1, 0xffffffff;" : "=r"(m) : "r"(u));
        u = (m >> 1) + lane;
    }
    t1 = clock64();
    if (lane == 0) g_out[1] = (t1 - t0);
    // 2: SHFL
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31) + 1.f;
    t1 = clock64();
    if (lane == 0) g_out[2] = (t1 - t0);
    // 3: VOTE + FLO
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
        const unsigned b = __ballot_sync(0xffffffffu, (u & 31) == unsigned(lane));
        u += __ffs(b);
    }
    t1 = clock64();
    if (lane == 0) g_out[3] = (t1 - t0);
    // 4: LDS chain
    int idx = lane;
    t0 = clock64();
    for (int i = 0; i < n; ++i) idx = int(sh[idx & 1023]) + lane;
    t1 = clock64();
    if (lane == 0) g_out[4] = (t1 - t0);
    // 5: LDTM x4 + wait::ld chain (address depends on the previous value)
    unsigned a = 0;
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
        unsigned r0, r1, r2, r3;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(tm + (a & 3)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        a = r0 + r1 + r2 + r3 + (a & 1);
    }
    t1 = clock64();
    if (lane == 0) g_out[5] = (t1 - t0);
    // 6: FFMA dependent chain (reference latency)
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = fmaf(x, 0.999f, 0.5f);
    t1 = clock64();
    if (lane == 0) g_out[6] = (t1 - t0);
    // 7: uniform switch on a runtime value (32 cases) -> pick from a register array
    float R[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) R[j] = float(j + lane);
    int t = sel;
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
        float v = 0.f;
        switch (t & 31) {
#define C(k) case k: v = R[k]; break;
            C(0) C(1) C(2) C(3) C(4) C(5) C(6) C(7) C(8) C(9) C(10) C(11) C(12) C(13) C(14) C(15)
            C(16) C(17) C(18) C(19) C(20) C(21) C(22) C(23) C(24) C(25) C(26) C(27) C(28) C(29) C(30) C(31)
#undef C
        }
        t = int(v) + 7 - lane;
        t = __shfl_sync(0xffffffffu, t, 0);
    }
    t1 = clock64();
    if (lane == 0) g_out[7] = (t1 - t0);
    if (lane == 0) g_out[8] = __float_as_uint(x) + u + idx + a + t;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tm));
}

int main() {
    const int n = 4096;
    k_lat<<<1, 32>>>(64, 1.f, 5);
    k_lat<<<1, 32>>>(n, 1.f, 5);
    cudaDeviceSynchronize();
    unsigned long long h[16];
    cudaMemcpyFromSymbol(h, g_out, sizeof h);
    const char* names[] = {"CREDUX.f32 (+FFMA)", "REDUX.u32 (+SHF+IADD)", "SHFL (+FADD)", "VOTE+FLO (+IADD)",
                           "LDS (+F2I+IADD)", "LDTM.x4+wait (+3 IADD)", "FFMA", "switch32+SHFL"};
    for (int k = 0; k < 8; ++k) printf("%-26s %7.1f cycles/iter\n", names[k], double(h[k]) / n);
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
