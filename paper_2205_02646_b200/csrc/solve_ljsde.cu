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
// One warp per block; synthesis and placement as in solve_f64.cu.
#include <cuda_runtime.h>

#include <cstdint>

#include "tqsb_internal.hpp"

namespace tqsb {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kWarpsL = 4;

__global__ void __launch_bounds__(kWarpsL * 32) k_solve_ljsde(const SolveArgs a) {
    extern __shared__ __align__(16) double smL[];
    const int W = a.window, K = W * W, B = a.block;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // per warp: N (2K), coef (2K), r (2 * K/4), order (K ints), touched (K bytes)
    const size_t per = size_t(4) * K + K / 2 + K / 2 + K / 8 + 8;
    double* base = smL + warp * per;
    double* Nr = base;
    double* Ni = Nr + K;
    double* cr = Ni + K;
    double* ci = cr + K;
    double* rr = ci + K;
    double* ri = rr + K / 4 + 1;
    int* order = reinterpret_cast<int*>(ri + K / 4 + 1);
    unsigned char* touched = reinterpret_cast<unsigned char*>(order + K);

    const int gw = blockIdx.x * kWarpsL + warp, nw = gridDim.x * kWarpsL;
    for (int it_item = 0; it_item < a.n_items; ++it_item) {
        const WorkItem item = a.items[it_item];
        const ClassTab& ct = a.tabs[item.cls];
        const int L = ct.local;
        for (int ti = item.start + gw; ti < item.start + item.count; ti += nw) {
            const Task tk = a.tasks[ti];
            // r = y^local (extract_local_system / gather_local_values, grid.cpp:104-114)
            const int r0 = (tk.origin_row + 1) / 2;
            const int c0 = (tk.origin_col + 1) / 2, c1 = (tk.origin_col + W - 2) / 2;
            const int ncol = c1 - c0 + 1;
            for (int m = lane; m < L; m += 32) {
                int fr = r0 + m / ncol, fc = c0 + m % ncol;
                fr = fr < a.frame_rows - 1 ? fr : a.frame_rows - 1;
                fc = fc < a.frame_cols - 1 ? fc : a.frame_cols - 1;
                rr[m] = a.frame[size_t(fr - a.frame_row0) * a.frame_pitch + fc];
                ri[m] = 0.0;
            }
            for (int k = lane; k < K; k += 32) {
                cr[k] = 0.0;
                ci[k] = 0.0;
                touched[k] = 0;
            }
            __syncwarp();
            const double floor = a.early_stop ? a.early_stop_scale * L : -1.0;
            const bool tracing = a.trace_picks != nullptr && ti == 0;
            int nactive = 0, it = 0;
            for (; it < a.iterations; ++it) {
                // numerators for every frequency + first-max selection (score_all)
                int best = -1;
                double bs = 0.0;
                for (int k = lane; k < K; k += 32) {
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
                    if (best < 0 || s > bs) {
                        best = k;
                        bs = s;
                    }
                }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                    const double os = __shfl_xor_sync(FULL, bs, off);
                    const int ok = __shfl_xor_sync(FULL, best, off);
                    const bool take = ok >= 0 && (best < 0 || os > bs || (os == bs && ok < best));
                    if (take) {
                        bs = os;
                        best = ok;
                    }
                }
                if (best < 0) break;  // no admissible frequency
                __syncwarp();
                const int u = best;
                const double den = ct.d64[u];
                const double gr = a.step * (Nr[u] / den), gi = a.step * (Ni[u] / den);
                const bool fresh = touched[u] == 0;
                __syncwarp();
                if (lane == 0) {
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
                for (int m = lane; m < L; m += 32) {
                    const double wm = ct.w64[m];
                    const double tr = col[2 * m] / wm, tim = -col[2 * m + 1] / wm;
                    rr[m] -= gr * tr - gi * tim;
                    ri[m] -= gr * tim + gi * tr;
                }
                __syncwarp();
                if (a.early_stop) {  // energy stop, summed in m order like the reference
                    double es = 0.0;
                    if (lane == 0)
                        for (int m = 0; m < L; ++m) es += (rr[m] * rr[m] + ri[m] * ri[m]) * ct.w64[m];
                    es = __shfl_sync(FULL, es, 0);
                    if (es < floor) {
                        ++it;  // this iteration completed (the hook ran) before the stop
                        break;
                    }
                }
            }
            if (tracing && lane == 0) *a.trace_n = it;
            __syncwarp();
            // synthesize_real (basis.cpp:52-73) over the kept pixels, then place
            const int rw = tk.block_row - tk.origin_row, cw = tk.block_col - tk.origin_col;
            for (int p = lane; p < B * B; p += 32) {
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
                for (int p = lane; p < K; p += 32) {
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
            __syncwarp();
        }
    }
}

}  // namespace

int launch_solve_ljsde(const SolveArgs& a, void* stream, int num_sms) {
    const int K = a.window * a.window;
    const size_t per = size_t(4) * K + K / 2 + K / 2 + K / 8 + 8;
    const size_t smem = per * sizeof(double) * kWarpsL;
    cudaError_t e = cudaFuncSetAttribute(k_solve_ljsde, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(smem));
    if (e != cudaSuccess) return e;
    k_solve_ljsde<<<num_sms * 2, kWarpsL * 32, smem, static_cast<cudaStream_t>(stream)>>>(a);
    return cudaGetLastError();
}

}  // namespace tqsb
