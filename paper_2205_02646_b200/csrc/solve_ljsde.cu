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
// For W <= 32 the batched variant below (NB blocks of a class per CTA) is launched; this
// per-block kernel serves larger windows and single-block tracing.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

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

// ---------------------------------------------------------------------------
// Batched L-JSDE (W <= 32): NB blocks of one class per CTA, in lock step. Every
// iteration each thread takes its frequencies k (tid, tid + 256, ...) and sums the
// numerators of all NB blocks in one pass over m, reading the class's B in its
// transposed, m-major copy (ClassTab::bt64: one coalesced 16 B load per thread per m,
// shared by the NB blocks, instead of one strided B row per block). Per block and k
// the sum still runs over m in ascending order with the same expression, and the
// selection, step, residual update, energy stop, coefficient accumulation and
// synthesis are the per-block kernel's, so the output is identical to it (and to the
// reference's greedy paths). The residuals of the NB blocks live in shared memory; the
// dense coefficients and first-touch order in a per-CTA global scratch.
// ---------------------------------------------------------------------------
struct BestN {
    double s, nr, ni;
    int k;
};

__device__ __forceinline__ BestN betterN(BestN a, BestN b) {
    if (b.k < 0) return a;
    if (a.k < 0) return b;
    return (b.s > a.s || (b.s == a.s && b.k < a.k)) ? b : a;
}

template <int NB, int KT>
__global__ void __launch_bounds__(kThreadsL, 2)
    k_solve_ljsde_b(const SolveArgs a, int groups_per_item, double* coef_g, int* order_g,
                    unsigned char* touched_g) {
    extern __shared__ __align__(16) double2 smr[];  // [NB][L] residuals
    __shared__ BestN s_best[kWarpsL][NB];
    __shared__ int s_u[NB], s_done[NB], s_nact[NB], s_alive;
    __shared__ double s_gr[NB], s_gi[NB];
    const int W = a.window, K = W * W, B = a.block;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double2* coef = reinterpret_cast<double2*>(coef_g) + size_t(blockIdx.x) * NB * K;
    int* order = order_g + size_t(blockIdx.x) * NB * K;
    unsigned char* touched = touched_g + size_t(blockIdx.x) * NB * K;
    const int n_groups = a.n_items * groups_per_item;
    for (int gi = blockIdx.x; gi < n_groups; gi += gridDim.x) {
        const WorkItem item = a.items[gi / groups_per_item];
        const int t0 = item.start + (gi % groups_per_item) * NB;
        const int cnt = min(NB, item.start + item.count - t0);
        if (cnt <= 0) continue;  // CTA-uniform
        const ClassTab& ct = a.tabs[item.cls];
        const int L = ct.local;
        const double2* bt = reinterpret_cast<const double2*>(ct.bt64);
        // r = y^local per block (gather_local_values, grid.cpp:104-114)
        for (int idx = tid; idx < NB * L; idx += kThreadsL) {
            const int b = idx / L, m = idx % L;
            double v = 0.0;
            if (b < cnt) {
                const Task tk = a.tasks[t0 + b];
                const int r0 = (tk.origin_row + 1) / 2;
                const int c0 = (tk.origin_col + 1) / 2, c1 = (tk.origin_col + W - 2) / 2;
                const int ncol = c1 - c0 + 1;
                int fr = r0 + m / ncol, fc = c0 + m % ncol;
                fr = fr < a.frame_rows - 1 ? fr : a.frame_rows - 1;
                fc = fc < a.frame_cols - 1 ? fc : a.frame_cols - 1;
                v = a.frame[size_t(fr - a.frame_row0) * a.frame_pitch + fc];
            }
            smr[idx] = make_double2(v, 0.0);
        }
        for (int idx = tid; idx < NB * K; idx += kThreadsL) {
            coef[idx] = make_double2(0.0, 0.0);
            touched[idx] = 0;
        }
        if (tid < NB) {
            s_done[tid] = tid >= cnt;
            s_nact[tid] = 0;
        }
        __syncthreads();
        const double floor = a.early_stop ? a.early_stop_scale * L : -1.0;
        for (int it = 0; it < a.iterations; ++it) {
            unsigned live = 0;
#pragma unroll
            for (int b = 0; b < NB; ++b) live |= s_done[b] ? 0u : 1u << b;
            if (!live) break;  // CTA-uniform
            BestN best[NB];
#pragma unroll
            for (int b = 0; b < NB; ++b) best[b] = BestN{0.0, 0.0, 0.0, -1};
            // KT frequencies per thread at once (k0 + 256 t), so each residual value read
            // from shared memory feeds KT x 4 multiply-adds; k ascending per thread
            for (int k0 = tid; k0 < K; k0 += kThreadsL * KT) {
                double nr[KT][NB], ni[KT][NB];
#pragma unroll
                for (int t = 0; t < KT; ++t)
#pragma unroll
                    for (int b = 0; b < NB; ++b) nr[t][b] = ni[t][b] = 0.0;
                const double2* col[KT];
#pragma unroll
                for (int t = 0; t < KT; ++t) {
                    const int k = k0 + kThreadsL * t;
                    col[t] = bt + (k < K ? k : 0);
                }
                // PF rows of B in flight (L2 hits of ~250+ cycles), sums in m order
                constexpr int PF = 2;
                int m = 0;
                for (; m + PF <= L; m += PF) {
                    double2 bb[PF][KT];
#pragma unroll
                    for (int j = 0; j < PF; ++j)
#pragma unroll
                        for (int t = 0; t < KT; ++t) bb[j][t] = __ldg(col[t] + size_t(m + j) * K);
#pragma unroll
                    for (int j = 0; j < PF; ++j) {
#pragma unroll
                        for (int b = 0; b < NB; ++b) {
                            const double2 r = smr[b * L + m + j];
#pragma unroll
                            for (int t = 0; t < KT; ++t) {
                                const double br = bb[j][t].x, bi = bb[j][t].y;
                                nr[t][b] += br * r.x - bi * r.y;
                                ni[t][b] += br * r.y + bi * r.x;
                            }
                        }
                    }
                }
                for (; m < L; ++m) {
#pragma unroll
                    for (int b = 0; b < NB; ++b) {
                        const double2 r = smr[b * L + m];
#pragma unroll
                        for (int t = 0; t < KT; ++t) {
                            const double2 bb = __ldg(col[t] + size_t(m) * K);
                            nr[t][b] += bb.x * r.x - bb.y * r.y;
                            ni[t][b] += bb.x * r.y + bb.y * r.x;
                        }
                    }
                }
#pragma unroll
                for (int t = 0; t < KT; ++t) {
                    const int k = k0 + kThreadsL * t;
                    if (k >= K) break;
                    const double den = ct.d64[k];
                    if (den <= 0.0) continue;
                    const double q = a.wc.q64[k];
#pragma unroll
                    for (int b = 0; b < NB; ++b) {
                        if (!(live >> b & 1u)) continue;
                        const double s = q * (nr[t][b] * nr[t][b] + ni[t][b] * ni[t][b]) / den;
                        if (best[b].k < 0 || s > best[b].s) best[b] = BestN{s, nr[t][b], ni[t][b], k};
                    }
                }
            }
#pragma unroll
            for (int b = 0; b < NB; ++b) {
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                    BestN o;
                    o.s = __shfl_xor_sync(FULL, best[b].s, off);
                    o.nr = __shfl_xor_sync(FULL, best[b].nr, off);
                    o.ni = __shfl_xor_sync(FULL, best[b].ni, off);
                    o.k = __shfl_xor_sync(FULL, best[b].k, off);
                    best[b] = betterN(best[b], o);
                }
                if (lane == 0) s_best[warp][b] = best[b];
            }
            __syncthreads();
            if (tid < NB && (live >> tid & 1u)) {
                const int b = tid;
                BestN bb = s_best[0][b];
                for (int w = 1; w < kWarpsL; ++w) bb = betterN(bb, s_best[w][b]);
                if (bb.k < 0) {  // no admissible frequency: this block stops (ljsde.cpp:150)
                    s_done[b] = 1;
                    s_u[b] = -1;
                } else {
                    const int u = bb.k;
                    const double den = ct.d64[u];
                    const double gr = a.step * (bb.nr / den), gi = a.step * (bb.ni / den);
                    double2& c = coef[size_t(b) * K + u];
                    c.x += gr;
                    c.y += gi;
                    if (!touched[size_t(b) * K + u]) {
                        touched[size_t(b) * K + u] = 1;
                        order[size_t(b) * K + s_nact[b]++] = u;
                    }
                    s_u[b] = u;
                    s_gr[b] = gr;
                    s_gi[b] = gi;
                }
            } else if (tid < NB) {
                s_u[tid] = -1;
            }
            __syncthreads();
            // r_m -= g conj(T_mu), T from the stored w T (ljsde.cpp:163-170)
            for (int idx = tid; idx < cnt * L; idx += kThreadsL) {
                const int b = idx / L, m = idx % L;
                const int u = s_u[b];
                if (u < 0) continue;
                const double* col = ct.b64 + size_t(u) * L * 2;
                const double gr = s_gr[b], gi = s_gi[b];
                const double wm = ct.w64[m];
                const double tr = col[2 * m] / wm, tim = -col[2 * m + 1] / wm;
                double2 r = smr[idx];
                r.x -= gr * tr - gi * tim;
                r.y -= gr * tim + gi * tr;
                smr[idx] = r;
            }
            __syncthreads();
            if (a.early_stop) {  // energy stop, summed in m order like the reference
                if (tid < cnt && s_u[tid] >= 0) {
                    double es = 0.0;
                    for (int m = 0; m < L; ++m) {
                        const double2 r = smr[tid * L + m];
                        es += (r.x * r.x + r.y * r.y) * ct.w64[m];
                    }
                    if (es < floor) s_done[tid] = 1;
                }
                __syncthreads();
            }
        }
        __syncthreads();
        // synthesize_real (basis.cpp:52-73) over the kept pixels, then place
        for (int p = tid; p < cnt * B * B; p += kThreadsL) {
            const int b = p / (B * B), q = p % (B * B);
            const Task tk = a.tasks[t0 + b];
            const int rw = tk.block_row - tk.origin_row, cw = tk.block_col - tk.origin_col;
            const int eta = rw + q / B, gam = cw + q % B;
            double v = 0.0;
            const int na = s_nact[b];
            for (int t = 0; t < na; ++t) {
                const int f = order[size_t(b) * K + t];
                const int idx = (eta * (f / W) + gam * (f % W)) % W;
                const double2 c = coef[size_t(b) * K + f];
                v += c.x * a.wc.unit64[2 * idx] - c.y * a.wc.unit64[2 * idx + 1];
            }
            const int orow = tk.block_row + q / B, ocol = tk.block_col + q % B;
            if (orow < a.out_rows && ocol < a.out_cols) {
                if (a.clip) v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
                a.out[size_t(orow - a.out_row0) * a.out_cols + ocol] = v;
            }
        }
        __syncthreads();  // the next group reuses the shared residuals and the scratch
    }
}

template <int NB, int KT>
int launch_batched(const SolveArgs& a, cudaStream_t st, int num_sms, int max_item) {
    const int K = a.window * a.window;
    const size_t smem = size_t(NB) * (K / 4 + 1) * sizeof(double2);
    cudaError_t e = cudaFuncSetAttribute(k_solve_ljsde_b<NB, KT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(smem));
    if (e != cudaSuccess) return e;
    const int gpi = (max_item + NB - 1) / NB;
    const int groups = a.n_items * gpi;
    int grid = 2 * num_sms;
    grid = groups < grid ? groups : grid;
    if (grid < 1) grid = 1;
    const size_t per = size_t(NB) * K;
    char* scratch = nullptr;
    e = cudaMallocAsync(reinterpret_cast<void**>(&scratch), size_t(grid) * per * (16 + 4 + 1), st);
    if (e != cudaSuccess) return e;
    double* coef = reinterpret_cast<double*>(scratch);
    int* order = reinterpret_cast<int*>(scratch + size_t(grid) * per * 16);
    unsigned char* touched = reinterpret_cast<unsigned char*>(scratch + size_t(grid) * per * 20);
    k_solve_ljsde_b<NB, KT><<<grid, kThreadsL, smem, st>>>(a, gpi, coef, order, touched);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return cudaFreeAsync(scratch, st);
}

}  // namespace

int launch_solve_ljsde(const SolveArgs& a, void* stream, int num_sms) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int K = a.window * a.window;
    // the batched kernel for W <= 32 (L <= K / 4 residuals per block in shared memory,
    // the m-major B copy present); tracing and the forced global-state test path keep
    // the per-block kernel
    if (a.window <= 32 && !a.trace_picks && !force_global_state() && a.items && a.n_items > 0) {
        // tasks per work item (plan.cpp prepare_band: 4 x the warps of the kernel family);
        // the largest family bounds it, so no task of an item is left out
        const int max_item = 4 * (kWarpsF32 > kWarpsF64 ? kWarpsF32 : kWarpsF64);
        // enough groups to fill two CTAs per SM: 8 blocks per CTA when the frame allows
        const int n_tasks = a.n_tasks;
        const char* nbv = std::getenv("TQSB_LJSDE_NB");  // experiment override
        // measured at 512^2 / P = 32 (tools/ljsde_bench.py): 2 blocks x 4 frequencies per
        // thread 0.57 s, 4 x 2 0.94 s, 1 x 4 0.75 s -- two blocks once the frame fills the
        // GPU with two CTAs per SM, else one
        const int nb = nbv ? std::atoi(nbv) : n_tasks >= 2 * 2 * num_sms ? 2 : 1;
        // frequencies per thread: K / 256 rounded up (no lanes on k >= K)
        const int kt = K > 512 ? 4 : K > 256 ? 2 : 1;
        if (nb == 4) return launch_batched<4, 2>(a, st, num_sms, max_item);
        if (nb == 2) {
            if (kt == 4) return launch_batched<2, 4>(a, st, num_sms, max_item);
            if (kt == 2) return launch_batched<2, 2>(a, st, num_sms, max_item);
            return launch_batched<2, 1>(a, st, num_sms, max_item);
        }
        if (kt == 4) return launch_batched<1, 4>(a, st, num_sms, max_item);
        if (kt == 2) return launch_batched<1, 2>(a, st, num_sms, max_item);
        return launch_batched<1, 1>(a, st, num_sms, max_item);
    }
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
