// solve_ljsde.cu -- the L-JSDE baseline on the device.
//
// The reference's baseline block solver (ljsde.cpp:131-185): every iteration the
// selection numerator N_k = sum_m (w T)_mk r_m is re-evaluated by direct summation
// over the local measurement system for all K frequencies (O(K L) per iteration,
// no Gram table), the best q |N|^2 / den is chosen with the strict '>' first-max
// rule, and the complex measurement residual is updated in place,
// r_m -= gamma delta conj(T_mu) with T recovered as (w T) / w (ljsde.cpp:163-170).
// The optional energy stop (ljsde.cpp:178-183) ends a block once
// sum_m |r_m|^2 w_m < earlyStopScale * L.
//
// Double precision throughout, in the reference's summation order (m ascending per
// k), on the class's resident B = w T (k-major) and den = D (tables.cu), so its
// output matches the reference's L-JSDE to ~1e-15 and the RL-JSDE fp64 mode to the
// reference's own L <-> RL equivalence bar (bench, pipeline.cpp:258-329).
//
// One CTA of kThreadsL threads per block: thread j owns frequencies j, j + kThreadsL,
// ... (each summed over m in order, so the arithmetic per k is the reference's), the
// first-max selection is a CTA reduction with ties to the smaller k, and the residual
// (L <= K/4 complex) lives in shared memory. Synthesis and placement as in solve_f64.cu.
#include <cuda_runtime.h>

#include <cstdint>

#include "tqsb_internal.hpp"

namespace tqsb {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kThreadsL = 256;
constexpr int kWarpsL = kThreadsL / 32;

struct Best {
    double s;
    int k;
};

// strict first-max: a candidate wins on a larger score, or an equal score at a smaller k
__device__ __forceinline__ Best better(Best a, Best b) {
    if (b.k < 0) return a;
    if (a.k < 0) return b;
    return (b.s > a.s || (b.s == a.s && b.k < a.k)) ? b : a;
}

// per-CTA state in doubles (see the layout below)
__host__ __device__ inline size_t ljsde_state_doubles(int K) {
    return size_t(4) * K + 2 * (K / 4 + 1) + K / 2 + K / 8 + 8;
}

// state in shared memory, or in a global slab (gscratch) when it exceeds shared memory
__global__ void __launch_bounds__(kThreadsL) k_solve_ljsde(const SolveArgs a, double* gscratch) {
    extern __shared__ __align__(16) double smL_dyn[];
    const int W = a.window, K = W * W, B = a.block;
    double* smL = gscratch ? gscratch + size_t(blockIdx.x) * ljsde_state_doubles(K) : smL_dyn;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // N (2K), coef (2K), r (2 * (K/4 + 1)), order (K ints), touched (K bytes)
    double* Nr = smL;
    double* Ni = Nr + K;
    double* cr = Ni + K;
    double* ci = cr + K;
    double* rr = ci + K;
    double* ri = rr + K / 4 + 1;
    int* order = reinterpret_cast<int*>(ri + K / 4 + 1);
    unsigned char* touched = reinterpret_cast<unsigned char*>(order + K);
    __shared__ Best s_best[kWarpsL];
    __shared__ int s_stop;

    // every CTA strides over the whole class-sorted task list (a work item holds only a
    // few dozen tasks, far fewer than the grid's CTAs)
    {
        for (int ti = blockIdx.x; ti < a.n_tasks; ti += gridDim.x) {
            const ClassTab& ct = a.tabs[a.task_cls ? a.task_cls[ti] : a.items[0].cls];
            const int L = ct.local;
            const Task tk = a.tasks[ti];
            // r = y^local (extract_local_system / gather_local_values, grid.cpp:104-114)
            const int r0 = (tk.origin_row + 1) / 2;
            const int c0 = (tk.origin_col + 1) / 2, c1 = (tk.origin_col + W - 2) / 2;
            const int ncol = c1 - c0 + 1;
            for (int m = tid; m < L; m += kThreadsL) {
                int fr = r0 + m / ncol, fc = c0 + m % ncol;
                fr = fr < a.frame_rows - 1 ? fr : a.frame_rows - 1;
                fc = fc < a.frame_cols - 1 ? fc : a.frame_cols - 1;
                rr[m] = a.frame[size_t(fr - a.frame_row0) * a.frame_pitch + fc];
                ri[m] = 0.0;
            }
            for (int k = tid; k < K; k += kThreadsL) {
                cr[k] = 0.0;
                ci[k] = 0.0;
                touched[k] = 0;
            }
            __syncthreads();
            const double floor = a.early_stop ? a.early_stop_scale * L : -1.0;
            const bool tracing = a.trace_picks != nullptr && ti == 0;
            int nactive = 0, it = 0;
            for (; it < a.iterations; ++it) {
                // numerators for every frequency + first-max selection (score_all)
                Best best{0.0, -1};
                for (int k = tid; k < K; k += kThreadsL) {
                    const double* col = ct.b64 + size_t(k) * L * 2;
                    double nr = 0.0, ni = 0.0;
                    for (int m = 0; m < L; ++m) {
                        const double br = col[2 * m], bi = col[2 * m + 1];
                        nr += br * rr[m] - bi * ri[m];
                        ni += br * ri[m] + bi * rr[m];
                    }
                    Nr[k] = nr;
                    Ni[k] = ni;
                    const double den = ct.d64[k];
                    if (den <= 0.0) continue;
                    const double s = a.wc.q64[k] * (nr * nr + ni * ni) / den;
                    if (best.k < 0 || s > best.s) best = Best{s, k};  // k ascending per thread
                }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                    Best o;
                    o.s = __shfl_xor_sync(FULL, best.s, off);
                    o.k = __shfl_xor_sync(FULL, best.k, off);
                    best = better(best, o);
                }
                if (lane == 0) s_best[warp] = best;
                __syncthreads();
                best = s_best[0];
#pragma unroll
                for (int w = 1; w < kWarpsL; ++w) best = better(best, s_best[w]);
                if (best.k < 0) break;  // no admissible frequency (uniform across the CTA)
                const int u = best.k;
                const double den = ct.d64[u];
                const double gr = a.step * (Nr[u] / den), gi = a.step * (Ni[u] / den);
                const bool fresh = touched[u] == 0;
                __syncthreads();  // all reads of s_best / touched precede the writes below
                if (tid == 0) {
                    cr[u] += gr;
                    ci[u] += gi;
                    if (fresh) {
                        touched[u] = 1;
                        order[nactive] = u;
                    }
                    if (tracing) {
                        a.trace_picks[it] = u;
                        a.trace_gd[2 * it] = gr;
                        a.trace_gd[2 * it + 1] = gi;
                    }
                }
                if (fresh) ++nactive;
                // r_m -= g conj(T_mu), T from the stored w T (ljsde.cpp:163-170)
                const double* col = ct.b64 + size_t(u) * L * 2;
                for (int m = tid; m < L; m += kThreadsL) {
                    const double wm = ct.w64[m];
                    const double tr = col[2 * m] / wm, tim = -col[2 * m + 1] / wm;
                    rr[m] -= gr * tr - gi * tim;
                    ri[m] -= gr * tim + gi * tr;
                }
                __syncthreads();
                if (a.early_stop) {  // energy stop, summed in m order like the reference
                    if (tid == 0) {
                        double es = 0.0;
                        for (int m = 0; m < L; ++m) es += (rr[m] * rr[m] + ri[m] * ri[m]) * ct.w64[m];
                        s_stop = es < floor;
                    }
                    __syncthreads();
                    if (s_stop) {
                        ++it;  // this iteration completed (the hook ran) before the stop
                        break;
                    }
                }
            }
            if (tracing && tid == 0) *a.trace_n = it;
            __syncthreads();
            // synthesize_real (basis.cpp:52-73) over the kept pixels, then place
            const int rw = tk.block_row - tk.origin_row, cw = tk.block_col - tk.origin_col;
            for (int p = tid; p < B * B; p += kThreadsL) {
                const int eta = rw + p / B, gam = cw + p % B;
                double v = 0.0;
                for (int t = 0; t < nactive; ++t) {
                    const int f = order[t];
                    const int idx = (eta * (f / W) + gam * (f % W)) % W;
                    v += cr[f] * a.wc.unit64[2 * idx] - ci[f] * a.wc.unit64[2 * idx + 1];
                }
                const int orow = tk.block_row + p / B, ocol = tk.block_col + p % B;
                if (orow < a.out_rows && ocol < a.out_cols) {
                    if (a.clip) v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
                    a.out[size_t(orow - a.out_row0) * a.out_cols + ocol] = v;
                }
            }
            if (tracing && a.trace_window) {
                for (int p = tid; p < K; p += kThreadsL) {
                    const int eta = p / W, gam = p % W;
                    double v = 0.0;
                    for (int t = 0; t < nactive; ++t) {
                        const int f = order[t];
                        const int idx = (eta * (f / W) + gam * (f % W)) % W;
                        v += cr[f] * a.wc.unit64[2 * idx] - ci[f] * a.wc.unit64[2 * idx + 1];
                    }
                    a.trace_window[p] = v;
                }
            }
            __syncthreads();
        }
    }
}

}  // namespace

int launch_solve_ljsde(const SolveArgs& a, void* stream, int num_sms) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int K = a.window * a.window;
    const size_t smem = ljsde_state_doubles(K) * sizeof(double);
    if (smem > 227 * 1024 || force_global_state()) {  // W >= 74: state in global memory, one CTA per SM
        double* scratch = nullptr;
        cudaError_t e = cudaMallocAsync(&scratch, smem * size_t(num_sms), st);
        if (e != cudaSuccess) return e;
        k_solve_ljsde<<<num_sms, kThreadsL, 0, st>>>(a, scratch);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        return cudaFreeAsync(scratch, st);
    }
    cudaError_t e = cudaFuncSetAttribute(k_solve_ljsde, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(smem));
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_solve_ljsde, kThreadsL, smem);
    if (e != cudaSuccess) return e;
    const int grid = num_sms * (per_sm > 0 ? per_sm : 1);
    k_solve_ljsde<<<grid, kThreadsL, smem, st>>>(a, nullptr);
    return cudaGetLastError();
}

}  // namespace tqsb
