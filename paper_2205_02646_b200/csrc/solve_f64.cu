// solve_f64.cu -- the fp64 PARITY mode of the block solve (TQSB_COMPUTE_FP64).
//
// The reference's block_impl (rljsde.cpp:122-182) restated per warp on device
// in double precision on the reference-ordered tables (B k-major, C column-major,
// D; tables.cu): init R = B y in m order (127-138), selection q|R|^2/D with the
// strict '>' first-max rule (144-158, basis.hpp:90-92), the coefficient step and
// column cascade (160-172), then synthesize_real (basis.cpp:52-73) restricted to
// the kept B x B pixels over the active list in first-touch order, placement
// with optional clip (pipeline.cpp:157-166). Every floating-point expression is spelled
// with explicit-rounding intrinsics in the reference build's own contraction pattern (g++
// -O3 with FMA: init R += rnd(B y) unfused; score = q * fma(Re, Re, Im*Im) / d; R -= fma(g_re, c_re, -(g_im*c_im))
// and fma(g_re, c_im, g_im*c_re); synthesis += fma(c_re, cos, -(c_im*sin))), so the
// greedy paths match the reference's even at near-ties. Its purpose is to prove that the
// device pipeline (enumeration, classes, tables, gather, placement) reproduces
// the reference's greedy paths; the fp32 kernel (solve_f32.cu) is the product.
#include <cuda_runtime.h>

#include <cstdint>

#include <cstdlib>

#include "tqsb_internal.hpp"

namespace tqsb {
namespace {

constexpr unsigned FULL = 0xffffffffu;

// per-warp state in doubles: R (2K), coef (2K), y (K), order (K ints), touched (K bytes)
__host__ __device__ inline size_t f64_state_doubles(int K) { return size_t(5) * K + K / 2 + K / 8 + 8; }

// State in shared memory (warps per CTA chosen by the launcher to fit), or, for windows
// whose state exceeds shared memory (W >= 68), in a global scratch slab (gscratch).
__global__ void __launch_bounds__(kWarpsF64 * 32) k_solve_f64(const SolveArgs a, double* gscratch) {
    extern __shared__ __align__(16) double sm64[];
    const int W = a.window, K = W * W, B = a.block;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wpc = blockDim.x >> 5;  // warps per CTA
    const size_t per = f64_state_doubles(K);
    double* base = gscratch ? gscratch + (size_t(blockIdx.x) * wpc + warp) * per : sm64 + warp * per;
    double* Rr = base;
    double* Ri = Rr + K;
    double* cr = Ri + K;
    double* ci = cr + K;
    double* y = ci + K;
    int* order = reinterpret_cast<int*>(y + K);
    unsigned char* touched = reinterpret_cast<unsigned char*>(order + K);

    const int gw = blockIdx.x * wpc + warp, nw = gridDim.x * wpc;
    // every warp strides over the whole class-sorted task list
    {
        for (int ti = gw; ti < a.n_tasks; ti += nw) {
            const ClassTab& ct = a.tabs[a.task_cls ? a.task_cls[ti] : a.items[0].cls];
            const int L = ct.local;
            const int n_unfused = 8 * (L / 8) + (L % 8 >= 4 ? 4 : 0);
            const Task tk = a.tasks[ti];
            // gather_local_values (grid.cpp:104-114); pad_frame by clamping (pipeline.cpp:44-52)
            const int r0 = (tk.origin_row + 1) / 2, r1 = (tk.origin_row + W - 2) / 2;
            const int c0 = (tk.origin_col + 1) / 2, c1 = (tk.origin_col + W - 2) / 2;
            const int ncol = c1 - c0 + 1;
            for (int m = lane; m < L; m += 32) {
                int fr = r0 + m / ncol, fc = c0 + m % ncol;
                fr = fr < a.frame_rows - 1 ? fr : a.frame_rows - 1;
                fc = fc < a.frame_cols - 1 ? fc : a.frame_cols - 1;
                y[m] = a.frame[size_t(fr - a.frame_row0) * a.frame_pitch + fc];
                (void)r1;
            }
            for (int k = lane; k < K; k += 32) {
                cr[k] = 0.0;
                ci[k] = 0.0;
                touched[k] = 0;
            }
            __syncwarp();
            for (int k = lane; k < K; k += 32) {  // R = B y  (rljsde.cpp:127-138)
                const double* col = ct.b64 + size_t(k) * L * 2;
                double re = 0.0, im = 0.0;
                for (int m = 0; m < L; ++m) {
                    // the reference build (g++ -O3, x86-64-v4) vectorises this in-order
                    // reduction: products of m < n_unfused come from 8- and 4-wide vector
                    // multiplies added one by one (acc + rnd(b y)); the last L mod 4 terms
                    // run in the scalar epilogue as FMAs (acc = fma(b, y, acc))
                    if (m < n_unfused) {
                        re = __dadd_rn(re, __dmul_rn(col[2 * m], y[m]));
                        im = __dadd_rn(im, __dmul_rn(col[2 * m + 1], y[m]));
                    } else {
                        re = __fma_rn(col[2 * m], y[m], re);
                        im = __fma_rn(col[2 * m + 1], y[m], im);
                    }
                }
                Rr[k] = re;
                Ri[k] = im;
            }
            __syncwarp();
            const bool tracing = a.trace_picks != nullptr && ti == 0;
            int nactive = 0, it = 0;
            for (; it < a.iterations; ++it) {
                int best = -1;
                double bs = 0.0;
                for (int k = lane; k < K; k += 32) {
                    const double dk = ct.d64[k];
                    if (dk <= 0.0) continue;
                    const double s = __ddiv_rn(
                        __dmul_rn(a.wc.q64[k], __fma_rn(Rr[k], Rr[k], __dmul_rn(Ri[k], Ri[k]))), dk);
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
                if (best < 0) break;
                const int u = best;
                const double du = ct.d64[u];
                const double gr = a.step * (Rr[u] / du), gi = a.step * (Ri[u] / du);
                __syncwarp();
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
                const double* col = ct.c64 + size_t(u) * K * 2;
                for (int s = lane; s < K; s += 32) {
                    const double c_r = col[2 * s], c_i = col[2 * s + 1];
                    Rr[s] = __dsub_rn(Rr[s], __fma_rn(gr, c_r, -__dmul_rn(gi, c_i)));
                    Ri[s] = __dsub_rn(Ri[s], __fma_rn(gr, c_i, __dmul_rn(gi, c_r)));
                }
                __syncwarp();
            }
            __syncwarp();
            // synthesize_real over the kept pixels (basis.cpp:52-73), then place
            const int rw = tk.block_row - tk.origin_row, cw = tk.block_col - tk.origin_col;
            for (int p = lane; p < B * B; p += 32) {
                const int eta = rw + p / B, gam = cw + p % B;
                double v = 0.0;
                for (int t = 0; t < nactive; ++t) {
                    const int f = order[t];
                    const int idx = (eta * (f / W) + gam * (f % W)) % W;
                    v = __dadd_rn(v, __fma_rn(cr[f], a.wc.unit64[2 * idx],
                                              -__dmul_rn(ci[f], a.wc.unit64[2 * idx + 1])));
                }
                const int orow = tk.block_row + p / B, ocol = tk.block_col + p % B;
                if (orow < a.out_rows && ocol < a.out_cols) {
                    if (a.clip) v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
                    a.out[size_t(orow - a.out_row0) * a.out_cols + ocol] = v;
                }
            }
            if (tracing) {
                if (lane == 0) *a.trace_n = it;
                if (a.trace_window) {
                    for (int p = lane; p < K; p += 32) {
                        const int eta = p / W, gam = p % W;
                        double v = 0.0;
                        for (int t = 0; t < nactive; ++t) {
                            const int f = order[t];
                            const int idx = (eta * (f / W) + gam * (f % W)) % W;
                            v = __dadd_rn(v, __fma_rn(cr[f], a.wc.unit64[2 * idx],
                                                      -__dmul_rn(ci[f], a.wc.unit64[2 * idx + 1])));
                        }
                        a.trace_window[p] = v;
                    }
                }
            }
            __syncwarp();
        }
    }
}

} // namespace

int launch_solve_f64(const SolveArgs& a, void* stream, int num_sms) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int K = a.window * a.window;
    const size_t per_bytes = f64_state_doubles(K) * sizeof(double);
    constexpr size_t kSmemMax = 227 * 1024;
    // as many warps per CTA (<= kWarpsF64) as shared memory holds; none -> global state
    int wpc = int(kSmemMax / per_bytes);
    wpc = wpc > kWarpsF64 ? kWarpsF64 : wpc;
    if (force_global_state()) wpc = 0;  // test hook: exercise the large-window path
    const int grid = num_sms * 2;
    if (wpc >= 1) {
        const size_t smem = per_bytes * wpc;
        cudaError_t e = cudaFuncSetAttribute(k_solve_f64, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(smem));
        if (e != cudaSuccess) return e;
        k_solve_f64<<<grid, wpc * 32, smem, st>>>(a, nullptr);
        return cudaGetLastError();
    }
    wpc = kWarpsF64;
    double* scratch = nullptr;
    cudaError_t e = cudaMallocAsync(&scratch, per_bytes * size_t(grid) * wpc, st);
    if (e != cudaSuccess) return e;
    k_solve_f64<<<grid, wpc * 32, 0, st>>>(a, scratch);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return cudaFreeAsync(scratch, st);
}

} // namespace tqsb
