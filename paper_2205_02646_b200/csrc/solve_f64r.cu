// solve_f64r.cu -- the fp64 parity / exact-reproduction solve with the residual in
// registers (W <= 32). Same arithmetic as solve_f64.cu (the reference build's rounding,
// expression for expression: bitwise equal to tqs::reconstruct), laid out for the B200:
//
//   * one warp per block; lane j holds R_k for k = j + 32 i, i < NE, in registers
//     (64 doubles per lane at W = 32), so the per-iteration selection scan and the column
//     cascade are unrolled register code with independent loads in flight instead of
//     shared-memory read-modify-write loops;
//   * selection: per lane the strict '>' first maximum over its k ascending, then a warp
//     reduction with ties to the smaller k (= the reference's scan from k = 0,
//     rljsde.cpp:144-158);
//   * the picked R_u from its owner lane (uniform register switch + SHFL);
//   * coefficients (ModelCoefficients: += per pick, first-touch active list, basis.hpp:40-58)
//     in a per-warp shared-memory list; synthesis over the kept B x B pixels at the end
//     (basis.cpp:52-73 restricted, pipeline.cpp:157-166);
//   * the init R = B y runs as its own kernel (k_init_f64r: the 8 blocks of a class group
//     share one pass over B, R to an HBM slab in register order, 32 K tasks per pass);
//     the solve CTA takes 8 consecutive (class-sorted) tasks behind a group barrier, loads
//     R from the slab and issues a pick's whole column (NE LDG.128) before the cascade.
//     12.94 -> 13.20 MP/s at 2160^2 P=8 over the fused-init kernel, bitwise
//     (profiles/r01_variants_fp64_init.jsonl).
// Tracing and windows above 32 use solve_f64.cu.
#include <cuda_runtime.h>

#include <cstdint>

#include "tqsb_internal.hpp"

namespace tqsb {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kWarpsF64R = 8;     // warps per CTA, both kernels
constexpr int kTileM = 4;         // m columns per cp.async stage of a warp's B rows
constexpr int kChunkTasks = 32768;  // tasks per init/solve pass (R slab: 512 MB at W = 32)

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool ok) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(ok ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// R = B y (rljsde.cpp:127-138) in the reference build's rounding: the init sum runs m
// ascending per k, unfused (mul, add) over the vectorised m < n_unfused and fused in the
// scalar epilogue (see solve_f64.cu)
__device__ __forceinline__ void init_term(double& re, double& im, double2 b, double ym, int m, int n_unfused) {
    if (m < n_unfused) {
        re = __dadd_rn(re, __dmul_rn(b.x, ym));
        im = __dadd_rn(im, __dmul_rn(b.y, ym));
    } else {
        re = __fma_rn(b.x, ym, re);
        im = __fma_rn(b.y, ym, im);
    }
}

// ---- K2a: the init as its own kernel. A CTA takes 8 consecutive (class-sorted) tasks;
// when they share a class, warp w sums rows k of B for register slots i = w, w + 8, ...
// for all 8 blocks at once (8 independent sums per lane; B read from L2 once per group
// through a cp.async double-buffered tile, the blocks' y_m as four broadcast LDS.128 from
// yT[m][block]); otherwise each warp sums its own block. R goes to an HBM slab in the
// solve kernel's register order: rs[task][i][lane] (double2), one coalesced 512 B row per
// slot. Keeping the init out of the solve kernel leaves that kernel's register budget to
// the greedy loop (tools/experiments/solve_f64r_exchange_init.cu: fused, the loop lost
// its batched column loads).
__global__ void __launch_bounds__(kWarpsF64R * 32) k_init_f64r(const SolveArgs a, int ne, double2* __restrict__ rs) {
    extern __shared__ __align__(16) unsigned char smi[];
    const int W = a.window, K = W * W;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int LM = K / 4 + 1;
    double* yT = reinterpret_cast<double*>(smi);  // [LM][8]
    double2* wt = reinterpret_cast<double2*>(smi + size_t(LM) * kWarpsF64R * 8) + warp * 2 * 32 * (kTileM + 1);
    __shared__ int s_same, s_cls0;
    const int t0 = blockIdx.x * kWarpsF64R;
    const int ti = t0 + warp;
    const bool active = ti < a.n_tasks;
    const int my_cls = active ? __ldg(a.task_cls + ti) : -1;
    if (threadIdx.x == 0) {
        s_cls0 = my_cls;
        s_same = 1;
    }
    __syncthreads();
    if (lane == 0 && active && my_cls != s_cls0) s_same = 0;
    const int cls = active ? my_cls : s_cls0;
    const ClassTab ct = a.tabs[cls];
    const int L = ct.local;
    const int n_unfused = 8 * (L / 8) + (L % 8 >= 4 ? 4 : 0);
    const Task tk = active ? a.tasks[ti] : a.tasks[t0];
    {  // gather_local_values (grid.cpp:104-114); pad_frame by clamping (pipeline.cpp:44-52)
        const int r0 = (tk.origin_row + 1) / 2;
        const int c0 = (tk.origin_col + 1) / 2, c1 = (tk.origin_col + W - 2) / 2;
        const int ncol = c1 - c0 + 1;
        for (int m = lane; m < L; m += 32) {
            int fr = r0 + m / ncol, fc = c0 + m % ncol;
            fr = fr < a.frame_rows - 1 ? fr : a.frame_rows - 1;
            fc = fc < a.frame_cols - 1 ? fc : a.frame_cols - 1;
            yT[m * kWarpsF64R + warp] = a.frame[size_t(fr - a.frame_row0) * a.frame_pitch + fc];
        }
    }
    __syncthreads();
    const double2* bk = reinterpret_cast<const double2*>(ct.b64);
    if (s_same) {
        const int nmt = (L + kTileM - 1) / kTileM;
        for (int i = warp; i < ne; i += kWarpsF64R) {
            auto issue = [&](int mt) {
                double2* buf = wt + (mt & 1) * 32 * (kTileM + 1);
                const int m0 = mt * kTileM;
#pragma unroll
                for (int e = lane; e < 32 * kTileM; e += 32) {
                    const int rr = e / kTileM, mm = e % kTileM;
                    const int k = 32 * i + rr, m = m0 + mm;
                    const bool ok = k < K && m < L;
                    cp_async16(buf + rr * (kTileM + 1) + mm, ok ? bk + size_t(k) * L + m : bk, ok);
                }
                cp_async_commit();
            };
            double re[kWarpsF64R], im[kWarpsF64R];
#pragma unroll
            for (int q = 0; q < kWarpsF64R; ++q) re[q] = im[q] = 0.0;
            issue(0);
            for (int mt = 0; mt < nmt; ++mt) {
                if (mt + 1 < nmt) {
                    issue(mt + 1);
                    cp_async_wait<1>();
                } else {
                    cp_async_wait<0>();
                }
                __syncwarp();
                const double2* row = wt + (mt & 1) * 32 * (kTileM + 1) + lane * (kTileM + 1);
                const int m0 = mt * kTileM;
#pragma unroll
                for (int mm = 0; mm < kTileM; ++mm) {
                    const int m = m0 + mm;
                    if (m < L) {
                        const double2 bv = row[mm];
                        const double2* yr = reinterpret_cast<const double2*>(yT + m * kWarpsF64R);
#pragma unroll
                        for (int q2 = 0; q2 < kWarpsF64R / 2; ++q2) {
                            const double2 ym = yr[q2];
                            init_term(re[2 * q2], im[2 * q2], bv, ym.x, m, n_unfused);
                            init_term(re[2 * q2 + 1], im[2 * q2 + 1], bv, ym.y, m, n_unfused);
                        }
                    }
                }
                __syncwarp();  // this buffer is refilled by the next iteration's issue
            }
#pragma unroll
            for (int q = 0; q < kWarpsF64R; ++q)
                if (t0 + q < a.n_tasks)
                    rs[(size_t(t0 + q) * ne + i) * 32 + lane] = make_double2(re[q], im[q]);
        }
    } else if (active) {
        for (int i = 0; i < ne; ++i) {
            const int k = lane + 32 * i;
            double re = 0.0, im = 0.0;
            if (k < K) {
                const double2* col = bk + size_t(k) * L;
                for (int m = 0; m < L; ++m) init_term(re, im, __ldg(col + m), yT[m * kWarpsF64R + warp], m, n_unfused);
            }
            rs[(size_t(ti) * ne + i) * 32 + lane] = make_double2(re, im);
        }
    }
}

struct F64RLayout {  // per-warp shared memory, in bytes
    int K, nact_max;
    __host__ __device__ size_t re_off() const { return 0; }
    __host__ __device__ size_t im_off() const { return re_off() + align(size_t(nact_max) * 8); }
    __host__ __device__ size_t f_off() const { return im_off() + align(size_t(nact_max) * 8); }
    __host__ __device__ size_t idx_off() const { return f_off() + align(size_t(nact_max) * 4); }
    __host__ __device__ size_t d_off() const { return idx_off() + align(size_t(K) * 2); }
    __host__ __device__ size_t bytes() const { return d_off() + align(size_t(K) * 8); }
    __host__ __device__ static size_t align(size_t b) { return (b + 15) & ~size_t(15); }
};

// R[i] of this lane for a warp-uniform i: a binary branch tree over the register array
// (log2 NE uniform branches, no local memory)
template <int LO, int HI, int NE>
__device__ __forceinline__ double pick_bs(const double (&R)[NE], int i) {
    if constexpr (HI - LO == 1) {
        return R[LO];
    } else {
        constexpr int MID = (LO + HI) / 2;
        return i < MID ? pick_bs<LO, MID, NE>(R, i) : pick_bs<MID, HI, NE>(R, i);
    }
}
template <int NE>
__device__ __forceinline__ double pick(const double (&R)[NE], int i) {
    return pick_bs<0, NE, NE>(R, i);
}

// ---- K2b: the greedy loop. A CTA takes 8 consecutive tasks (a class group) per barrier,
// each warp loads its R from the slab into registers and run select / update / synthesis.
template <int NE>
__global__ void __launch_bounds__(kWarpsF64R * 32, 1)
    k_solve_f64r(const SolveArgs a, F64RLayout lay, const double2* __restrict__ rs) {
    extern __shared__ __align__(16) unsigned char smr[];
    const int W = a.window, K = W * W, B = a.block;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned char* base = smr + size_t(warp) * lay.bytes();
    double* act_re = reinterpret_cast<double*>(base + lay.re_off());
    double* act_im = reinterpret_cast<double*>(base + lay.im_off());
    int* act_f = reinterpret_cast<int*>(base + lay.f_off());
    short* idx_of = reinterpret_cast<short*>(base + lay.idx_off());
    double* dsm = reinterpret_cast<double*>(base + lay.d_off());  // the block's class D
    double* qsm = reinterpret_cast<double*>(smr + size_t(kWarpsF64R) * lay.bytes());  // q
    const double* __restrict__ unit = a.wc.unit64;
    for (int k = threadIdx.x; k < K; k += blockDim.x) qsm[k] = a.wc.q64[k];
    __syncthreads();
    __shared__ int grp_s;
    for (;;) {
        __syncthreads();  // every warp has read the previous group's index
        if (threadIdx.x == 0) grp_s = atomicAdd(a.counter, kWarpsF64R);
        __syncthreads();  // the CTA's 8 warps start their (same-class) loops together
        const int ti = grp_s + warp;
        if (grp_s >= a.n_tasks) break;
        if (ti >= a.n_tasks) continue;
        const ClassTab ct = a.tabs[__ldg(a.task_cls + ti)];
        const Task tk = a.tasks[ti];
        double Rr[NE], Ri[NE];
        const double2* rt = rs + size_t(ti) * NE * 32 + lane;
#pragma unroll
        for (int i = 0; i < NE; ++i) {
            const double2 v = __ldcs(rt + 32 * i);  // read once: stream past L1/L2
            Rr[i] = v.x;
            Ri[i] = v.y;
        }
        for (int k = lane; k < K; k += 32) {
            idx_of[k] = -1;
            dsm[k] = __ldg(ct.d64 + k);
        }
        __syncwarp();

        int nact = 0;
        for (int it = 0; it < a.iterations; ++it) {
            // ---- selection: q |R|^2 / D, strict first maximum ----
            int best = -1;
            double bs = 0.0;
#pragma unroll
            for (int i = 0; i < NE; ++i) {
                const int k = lane + 32 * i;
                if (k < K) {
                    const double dk = dsm[k];
                    if (dk > 0.0) {
                        const double s = __ddiv_rn(
                            __dmul_rn(qsm[k], __fma_rn(Rr[i], Rr[i], __dmul_rn(Ri[i], Ri[i]))), dk);
                        if (best < 0 || s > bs) {
                            best = k;
                            bs = s;
                        }
                    }
                }
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const double os = __shfl_xor_sync(FULL, bs, off);
                const int ok = __shfl_xor_sync(FULL, best, off);
                if (ok >= 0 && (best < 0 || os > bs || (os == bs && ok < best))) {
                    bs = os;
                    best = ok;
                }
            }
            if (best < 0) break;  // no admissible frequency (rljsde.cpp:159)
            const int u = best;
            const double ur = __shfl_sync(FULL, pick<NE>(Rr, u >> 5), u & 31);
            const double ui = __shfl_sync(FULL, pick<NE>(Ri, u >> 5), u & 31);
            const double du = dsm[u];
            const double gr = a.step * (ur / du), gi = a.step * (ui / du);
            // ---- coefficients (ModelCoefficients::add, first-touch active list) ----
            const int idx = idx_of[u];
            __syncwarp();
            if (lane == 0) {
                if (idx < 0) {
                    idx_of[u] = short(nact);
                    act_f[nact] = u;
                    act_re[nact] = gr;
                    act_im[nact] = gi;
                } else {
                    act_re[idx] += gr;
                    act_im[idx] += gi;
                }
            }
            if (idx < 0) ++nact;
            __syncwarp();  // lane 0's list writes are visible to the next iteration's reads
            // ---- column cascade: R_s -= g C[s,u] (rljsde.cpp:160-172) ----
            const double2* col = reinterpret_cast<const double2*>(ct.c64) + size_t(u) * K + lane;
            constexpr int CH = NE < 32 ? NE : 32;
#pragma unroll
            for (int i0 = 0; i0 < NE; i0 += CH) {
                double2 c[CH];
#pragma unroll
                for (int j = 0; j < CH; ++j)
                    c[j] = (lane + 32 * (i0 + j) < K) ? __ldg(col + 32 * (i0 + j)) : make_double2(0.0, 0.0);
#pragma unroll
                for (int j = 0; j < CH; ++j) {
                    const int i = i0 + j;
                    Rr[i] = __dsub_rn(Rr[i], __fma_rn(gr, c[j].x, -__dmul_rn(gi, c[j].y)));
                    Ri[i] = __dsub_rn(Ri[i], __fma_rn(gr, c[j].y, __dmul_rn(gi, c[j].x)));
                }
            }
        }
        __syncwarp();
        // ---- synthesize_real over the kept pixels (basis.cpp:52-73), place ----
        const int rw = tk.block_row - tk.origin_row, cw = tk.block_col - tk.origin_col;
        for (int p = lane; p < B * B; p += 32) {
            const int eta = rw + p / B, gam = cw + p % B;
            double v = 0.0;
            for (int t = 0; t < nact; ++t) {
                const int f = act_f[t];
                const int ix = (eta * (f / W) + gam * (f % W)) % W;
                v = __dadd_rn(v, __fma_rn(act_re[t], unit[2 * ix], -__dmul_rn(act_im[t], unit[2 * ix + 1])));
            }
            const int orow = tk.block_row + p / B, ocol = tk.block_col + p % B;
            if (orow < a.out_rows && ocol < a.out_cols) {
                if (a.clip) v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
                a.out[size_t(orow - a.out_row0) * a.out_cols + ocol] = v;
            }
        }
        __syncwarp();  // the next task reuses this warp's shared region
    }
}

template <int NE>
int launch_ne(const SolveArgs& a, cudaStream_t st, int num_sms) {
    const int K = a.window * a.window;
    F64RLayout lay{K, a.iterations < K ? (a.iterations > 0 ? a.iterations : 1) : K};
    const size_t smem = lay.bytes() * kWarpsF64R + size_t(K) * sizeof(double);
    const size_t smem_init = size_t(K / 4 + 1) * kWarpsF64R * 8 + size_t(kWarpsF64R) * 2 * 32 * (kTileM + 1) * 16;
    // the per-warp coefficient lists grow with nu (W = 32, nu >= ~890 exceeds 227 KB):
    // hand such launches to the generic kernel, which keeps its state in global memory
    int dev = 0, smem_max = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess)
        e = cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (e != cudaSuccess) return e;
    if (smem > size_t(smem_max) || smem_init > size_t(smem_max)) return cudaErrorNotSupported;
    e = cudaFuncSetAttribute(k_solve_f64r<NE>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_init_f64r, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_init));
    if (e != cudaSuccess) return e;
    const int chunk = a.n_tasks < kChunkTasks ? a.n_tasks : kChunkTasks;
    if (chunk <= 0) return cudaSuccess;
    double2* rs = nullptr;
    e = cudaMallocAsync(reinterpret_cast<void**>(&rs), size_t(chunk) * NE * 32 * sizeof(double2), st);
    if (e != cudaSuccess) return e;
    for (int t0 = 0; t0 < a.n_tasks && e == cudaSuccess; t0 += chunk) {
        SolveArgs c = a;
        c.tasks = a.tasks + t0;
        c.task_cls = a.task_cls + t0;
        c.n_tasks = a.n_tasks - t0 < chunk ? a.n_tasks - t0 : chunk;
        if (t0 > 0) e = cudaMemsetAsync(a.counter, 0, sizeof(int), st);
        if (e != cudaSuccess) break;
        k_init_f64r<<<(c.n_tasks + kWarpsF64R - 1) / kWarpsF64R, kWarpsF64R * 32, smem_init, st>>>(c, NE, rs);
        k_solve_f64r<NE><<<num_sms, kWarpsF64R * 32, smem, st>>>(c, lay, rs);
        e = cudaGetLastError();
    }
    const cudaError_t f = cudaFreeAsync(rs, st);
    return e != cudaSuccess ? e : f;
}

} // namespace

// fp64 mode for W <= 32 without tracing; returns cudaErrorNotSupported otherwise
int launch_solve_f64r(const SolveArgs& a, void* stream, int num_sms) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int K = a.window * a.window;
    if (a.window > 32 || a.trace_picks || !a.counter || !a.task_cls || force_global_state())
        return cudaErrorNotSupported;
    const int ne = (K + 31) / 32;
    if (ne <= 1) return launch_ne<1>(a, st, num_sms);
    if (ne <= 2) return launch_ne<2>(a, st, num_sms);
    if (ne <= 4) return launch_ne<4>(a, st, num_sms);
    if (ne <= 8) return launch_ne<8>(a, st, num_sms);
    if (ne <= 16) return launch_ne<16>(a, st, num_sms);
    return launch_ne<32>(a, st, num_sms);
}

} // namespace tqsb
