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
//   * warps take blocks from a global counter (the class-sorted task list).
// Tracing and windows above 32 use solve_f64.cu.
#include <cuda_runtime.h>

#include <cstdint>

#include "tqsb_internal.hpp"

namespace tqsb {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kWarpsF64R = 8;
constexpr int kTileM = 32;  // m columns of the shared B tile

struct F64RLayout {  // per-warp shared memory, in bytes
    int K, nact_max, L_max;
    __host__ __device__ size_t y_off() const { return 0; }
    __host__ __device__ size_t re_off() const { return align(size_t(L_max) * 8); }
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

template <int NE>
__global__ void __launch_bounds__(kWarpsF64R * 32, 1) k_solve_f64r(const SolveArgs a, F64RLayout lay) {
    extern __shared__ __align__(16) unsigned char smr[];
    const int W = a.window, K = W * W, B = a.block;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned char* base = smr + size_t(warp) * lay.bytes();
    double* y = reinterpret_cast<double*>(base + lay.y_off());
    double* act_re = reinterpret_cast<double*>(base + lay.re_off());
    double* act_im = reinterpret_cast<double*>(base + lay.im_off());
    int* act_f = reinterpret_cast<int*>(base + lay.f_off());
    short* idx_of = reinterpret_cast<short*>(base + lay.idx_off());
    double* dsm = reinterpret_cast<double*>(base + lay.d_off());  // the block's class D
    const double* __restrict__ q64 = a.wc.q64;
    const double* __restrict__ unit = a.wc.unit64;

    // the CTA takes kWarpsF64R consecutive tasks at a time (one per warp); when they share a
    // class, the init R = B y streams the class's B through shared memory once for all of
    // them (B: K x L complex = 4 MB at W = 32, otherwise re-read from L2 by every block)
    double2* tile = reinterpret_cast<double2*>(smr + size_t(kWarpsF64R) * lay.bytes());
    double* qsm = reinterpret_cast<double*>(tile + 32 * (kTileM + 1));  // q (class independent)
    for (int k = threadIdx.x; k < K; k += blockDim.x) qsm[k] = q64[k];
    __shared__ int s_t0, s_cls0, s_same;
    for (;;) {
        if (threadIdx.x == 0) s_t0 = atomicAdd(a.counter, kWarpsF64R);
        __syncthreads();
        const int t0 = s_t0;
        if (t0 >= a.n_tasks) break;
        const int ti = t0 + warp;
        const bool active = ti < a.n_tasks;
        const int my_cls = active ? __ldg(a.task_cls + ti) : -1;
        if (threadIdx.x == 0) {
            s_cls0 = my_cls;
            s_same = 1;
        }
        __syncthreads();
        if (lane == 0 && active && my_cls != s_cls0) s_same = 0;
        __syncthreads();
        const bool shared_init = s_same != 0;
        const int cls = active ? my_cls : s_cls0;
        const ClassTab ct = a.tabs[cls];
        const int L = ct.local;
        const int n_unfused = 8 * (L / 8) + (L % 8 >= 4 ? 4 : 0);  // see solve_f64.cu
        const Task tk = active ? a.tasks[ti] : a.tasks[t0];
        // gather_local_values (grid.cpp:104-114); pad_frame by clamping (pipeline.cpp:44-52)
        {
            const int r0 = (tk.origin_row + 1) / 2;
            const int c0 = (tk.origin_col + 1) / 2, c1 = (tk.origin_col + W - 2) / 2;
            const int ncol = c1 - c0 + 1;
            for (int m = lane; m < L; m += 32) {
                int fr = r0 + m / ncol, fc = c0 + m % ncol;
                fr = fr < a.frame_rows - 1 ? fr : a.frame_rows - 1;
                fc = fc < a.frame_cols - 1 ? fc : a.frame_cols - 1;
                y[m] = a.frame[size_t(fr - a.frame_row0) * a.frame_pitch + fc];
            }
            for (int k = lane; k < K; k += 32) {
                idx_of[k] = -1;
                dsm[k] = __ldg(ct.d64 + k);
            }
        }
        __syncwarp();
        // R = B y (rljsde.cpp:127-138) in the reference build's rounding, m ascending per k
        double Rr[NE], Ri[NE];
        auto term = [&](double& re, double& im, double2 b, int m) {
            if (m < n_unfused) {
                re = __dadd_rn(re, __dmul_rn(b.x, y[m]));
                im = __dadd_rn(im, __dmul_rn(b.y, y[m]));
            } else {
                re = __fma_rn(b.x, y[m], re);
                im = __fma_rn(b.y, y[m], im);
            }
        };
        if (shared_init) {
            const double2* bk = reinterpret_cast<const double2*>(ct.b64);
#pragma unroll
            for (int i = 0; i < NE; ++i) {
                double re = 0.0, im = 0.0;
                for (int m0 = 0; m0 < L; m0 += kTileM) {
                    const int mc = L - m0 < kTileM ? L - m0 : kTileM;
                    // rows k = 32 i .. 32 i + 31, columns m0 .. m0 + mc: one 512 B row piece
                    // per warp load, padded row stride (kTileM + 1) double2: conflict-free reads
                    for (int e = threadIdx.x; e < 32 * kTileM; e += kWarpsF64R * 32) {
                        const int r = e / kTileM, mm = e % kTileM;
                        const int k = 32 * i + r;
                        tile[r * (kTileM + 1) + mm] =
                            (k < K && mm < mc) ? __ldg(bk + size_t(k) * L + m0 + mm) : make_double2(0.0, 0.0);
                    }
                    __syncthreads();
                    if (active && lane + 32 * i < K) {
                        const double2* row = tile + lane * (kTileM + 1);
                        for (int mm = 0; mm < mc; ++mm) term(re, im, row[mm], m0 + mm);
                    }
                    __syncthreads();
                }
                Rr[i] = re;
                Ri[i] = im;
            }
        } else {
#pragma unroll
            for (int i = 0; i < NE; ++i) {
                const int k = lane + 32 * i;
                double re = 0.0, im = 0.0;
                if (k < K && active) {
                    const double2* col = reinterpret_cast<const double2*>(ct.b64) + size_t(k) * L;
                    for (int m = 0; m < L; ++m) term(re, im, __ldg(col + m), m);
                }
                Rr[i] = re;
                Ri[i] = im;
            }
        }
        if (!active) {  // a short last group: idle warps only joined the shared init
            __syncthreads();
            continue;
        }

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
            constexpr int CH = NE < 8 ? NE : 8;
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
        __syncthreads();  // the group ends together (s_t0 and the tile are reused)
    }
}

template <int NE>
int launch_ne(const SolveArgs& a, cudaStream_t st, int num_sms) {
    const int K = a.window * a.window;
    F64RLayout lay{K, a.iterations < K ? (a.iterations > 0 ? a.iterations : 1) : K, K / 4 + 1};
    const size_t smem = lay.bytes() * kWarpsF64R + size_t(32) * (kTileM + 1) * sizeof(double2) +
                        size_t(K) * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(k_solve_f64r<NE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(smem));
    if (e != cudaSuccess) return e;
    k_solve_f64r<NE><<<num_sms, kWarpsF64R * 32, smem, st>>>(a, lay);
    return cudaGetLastError();
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
