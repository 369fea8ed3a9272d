// solve_f32.cu -- K2+K3+K4: the fused per-block RL-JSDE solve, fp32 product path.
//
// One warp owns one B x B target block end to end (the reference's per-block
// work item, pipeline.cpp:141-166 -> rljsde_block, rljsde.cpp:258-271):
//
//  init (K2)   R_k = sum_m B_mk y_m (rljsde.cpp:127-138) evaluated as the separable
//              2-D DFT of the window image a(eta,gamma) = (w_m/3) y_m at the three
//              transparent pixels of every included cell -- the same sum, factorised
//              (B_mk = w_m (1/3) sum_px conj(unit[(eta sigma + gamma rho) mod W])).
//              Only sigma <= W/2 is computed; the other half is written as the
//              exact conjugate, so conjugate pairs tie bitwise like the reference's.
//  loop (K3)   nu x { argmax_k q_k |R_k|^2 / D_k over D_k > 0, smallest k on ties
//              (rljsde.cpp:144-158, basis.hpp:90-92); R -= gamma (R_u/D_u) C[:,u]
//              (160-172) } on the SCALED residual R'_k = sqrt(q_k/D_k) R_k, so the
//              score is |R'_k|^2 and the update streams C'[s,u] = s_s C[s,u] --
//              2 FFMA2 per complex element, 2 more for the score, FMNMX3 for the max.
//  synth (K4)  only the B x B target pixels of sum Re(g unit[(eta sigma + gamma rho)])
//              (basis.cpp:52-73 restricted to the kept block, pipeline.cpp:157-166),
//              accumulated per pick, clipped and stored straight into the output.
//
// Register layout: lane j, slot i holds ranks r = 64 i + 2 j + {0,1} as one float4
// (re_a, re_b, im_a, im_b); ranks order frequencies by centred radius (hot first).
// The C' column of rank u is the same float4 array, so a column read is 32 lanes x
// 16 B = one fully coalesced 512 B line per slot. The first `hot` columns of the
// CTA's class are cached in shared memory; the rest stream from L2.
#include <cuda_runtime.h>

#include <cstdint>

#include "tqsb_internal.hpp"

namespace tqsb {
namespace {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ float qnan() { return __int_as_float(0x7fc00000); }

__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

template <int NS>
__device__ __forceinline__ float4 pick_slot(const float4 (&R)[NS], int i) {
    float4 v = R[0];
    switch (i) {
#define TQSB_CASE(n) \
    case n:          \
        if (n < NS) v = R[n < NS ? n : 0]; \
        break;
        TQSB_CASE(0) TQSB_CASE(1) TQSB_CASE(2) TQSB_CASE(3) TQSB_CASE(4) TQSB_CASE(5)
        TQSB_CASE(6) TQSB_CASE(7) TQSB_CASE(8) TQSB_CASE(9) TQSB_CASE(10) TQSB_CASE(11)
        TQSB_CASE(12) TQSB_CASE(13) TQSB_CASE(14) TQSB_CASE(15)
#undef TQSB_CASE
        default: break;
    }
    return v;
}

// Scores |R'|^2 of every slot: slot maxima to sbuf (STS.128 per 4 slots), lane max returned.
template <int NS>
__device__ __forceinline__ float score_pass(const float4 (&R)[NS], int lane, float* sbuf) {
    float lmax = qnan();
#pragma unroll
    for (int i0 = 0; i0 < NS; i0 += 4) {
        float m[4] = {qnan(), qnan(), qnan(), qnan()};
#pragma unroll
        for (int j = 0; j < 4 && i0 + j < NS; ++j) {
            const float2 re = make_float2(R[i0 + j].x, R[i0 + j].y);
            const float2 im = make_float2(R[i0 + j].z, R[i0 + j].w);
            float2 s = __fmul2_rn(re, re);
            s = __ffma2_rn(im, im, s);
            m[j] = fmaxf(s.x, s.y);
        }
        if constexpr (NS >= 4) {
            *reinterpret_cast<float4*>(sbuf + lane * kSbufStride + i0) =
                make_float4(m[0], m[1], m[2], m[3]);
        } else {
#pragma unroll
            for (int j = 0; j < NS; ++j) sbuf[lane * kSbufStride + j] = m[j];
        }
        lmax = fmax3(lmax, fmax3(m[0], m[1], m[2]), m[3]);
    }
    return lmax;
}

// R' -= g C'[:,u] for every slot (2 FFMA2 per complex element), fused with the scores.
template <int NS>
__device__ __forceinline__ float update_pass(float4 (&R)[NS], const float4* __restrict__ col,
                                             int lane, float gre, float gim, float* sbuf) {
    const float2 ngre = make_float2(-gre, -gre);
    const float2 pgim = make_float2(gim, gim);
    const float2 ngim = make_float2(-gim, -gim);
    float lmax = qnan();
#pragma unroll
    for (int i0 = 0; i0 < NS; i0 += 4) {
        float m[4] = {qnan(), qnan(), qnan(), qnan()};
#pragma unroll
        for (int j = 0; j < 4 && i0 + j < NS; ++j) {
            const int i = i0 + j;
            const float4 c = col[i * 32 + lane];
            const float2 cre = make_float2(c.x, c.y), cim = make_float2(c.z, c.w);
            float2 re = make_float2(R[i].x, R[i].y), im = make_float2(R[i].z, R[i].w);
            re = __ffma2_rn(ngre, cre, re);
            re = __ffma2_rn(pgim, cim, re);
            im = __ffma2_rn(ngre, cim, im);
            im = __ffma2_rn(ngim, cre, im);
            R[i] = make_float4(re.x, re.y, im.x, im.y);
            float2 s = __fmul2_rn(re, re);
            s = __ffma2_rn(im, im, s);
            m[j] = fmaxf(s.x, s.y);
        }
        if constexpr (NS >= 4) {
            *reinterpret_cast<float4*>(sbuf + lane * kSbufStride + i0) =
                make_float4(m[0], m[1], m[2], m[3]);
        } else {
#pragma unroll
            for (int j = 0; j < NS; ++j) sbuf[lane * kSbufStride + j] = m[j];
        }
        lmax = fmax3(lmax, fmax3(m[0], m[1], m[2]), m[3]);
    }
    return lmax;
}

// per-warp scratch floats: init half-spectrum buffer (W/2+1 rows x 32 complex,
// row stride 18 complex for the transpose) vs the slot-max buffer (32 x 20)
template <int W>
struct Scratch {
    static constexpr int kHalf = W / 2 + 1;
    static constexpr int kZ = 32 * 18 * 2;           // zbuf[gamma][sigma] (float2), stride 18
    static constexpr int kR = kHalf * 32 * 2;        // r0buf[sigma][rho] (float2)
    static constexpr int kS = 32 * kSbufStride;      // sbuf[lane][slot]
    static constexpr int kFloats = (kZ > kR ? (kZ > kS ? kZ : kS) : (kR > kS ? kR : kS));
};

template <int NS, int W, int PPL>
__global__ void __launch_bounds__(kWarpsF32 * 32, 1) k_solve_f32(const SolveArgs a) {
    extern __shared__ __align__(16) float smem[];
    constexpr int COLF4 = NS * 32;  // float4 per column
    constexpr int SCR = Scratch<W>::kFloats;
    float4* hot = reinterpret_cast<float4*>(smem);
    float2* unit = reinterpret_cast<float2*>(smem + size_t(a.hot) * COLF4 * 4);
    float* scr_all = smem + size_t(a.hot) * COLF4 * 4 + 2 * 32;
    __shared__ int s_cls;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float* scr = scr_all + warp * SCR;
    float2* zbuf = reinterpret_cast<float2*>(scr);
    float* sbuf = scr;

    if (threadIdx.x < W) unit[threadIdx.x] = make_float2(a.wc.unit32[2 * threadIdx.x],
                                                         a.wc.unit32[2 * threadIdx.x + 1]);
    if (threadIdx.x == 0) s_cls = -1;
    __syncthreads();

    const int B = a.block;
    const int nb2 = B * B;

    for (int it_item = blockIdx.x; it_item < a.n_items; it_item += gridDim.x) {
        const WorkItem item = a.items[it_item];
        if (item.cls != s_cls) {  // CTA-uniform: refill the hot-column cache
            __syncthreads();
            const float4* src = reinterpret_cast<const float4*>(a.tabs[item.cls].cpack);
            const int n = a.hot * COLF4;
            for (int i = threadIdx.x; i < n; i += blockDim.x) hot[i] = __ldg(src + i);
            __syncthreads();
            if (threadIdx.x == 0) s_cls = item.cls;
            __syncthreads();
        }
        const ClassTab& ct = a.tabs[item.cls];
        const float4* gcols = reinterpret_cast<const float4*>(ct.cpack);
        const float2* scale2 = reinterpret_cast<const float2*>(ct.scale);

        for (int ti = item.start + warp; ti < item.start + item.count; ti += kWarpsF32) {
            const Task tk = a.tasks[ti];
            // ---------------- init: window image column per lane ----------------
            float colv[W];
            {
                const int gc = tk.origin_col + lane;
                int fc = gc >> 1;
                fc = fc < a.frame_cols - 1 ? fc : a.frame_cols - 1;
#pragma unroll
                for (int eta = 0; eta < W; ++eta) {
                    float v = 0.f;
                    if (lane < W) {
                        const float mk = __ldg(ct.mask32 + eta * W + lane);
                        int fr = (tk.origin_row + eta) >> 1;
                        fr = fr < a.frame_rows - 1 ? fr : a.frame_rows - 1;
                        const double y =
                            __ldg(a.frame + size_t(fr - a.frame_row0) * a.frame_pitch + fc);
                        v = mk * float(y);
                    }
                    colv[eta] = v;
                }
            }
            // step 1 (lane = gamma): Z(sigma, gamma) = sum_eta a(eta,gamma) conj(U(eta sigma))
            constexpr int H = W / 2 + 1;
#pragma unroll
            for (int sg = 0; sg < H; ++sg) {
                float zr = 0.f, zi = 0.f;
#pragma unroll
                for (int eta = 0; eta < W; ++eta) {
                    const float2 u = unit[(eta * sg) % W];
                    zr = fmaf(colv[eta], u.x, zr);
                    zi = fmaf(-colv[eta], u.y, zi);
                }
                zbuf[lane * 18 + sg] = make_float2(zr, zi);
            }
            __syncwarp();
            // step 2 (lane = rho): R0(sigma, rho) = sum_gamma Z(sigma,gamma) conj(U(gamma rho))
            float2 r0[H];
#pragma unroll
            for (int sg = 0; sg < H; ++sg) r0[sg] = make_float2(0.f, 0.f);
#pragma unroll 4
            for (int g = 0; g < W; ++g) {
                const float2 u = unit[(g * lane) % W];  // conj: (u.x, -u.y)
#pragma unroll
                for (int sg = 0; sg < H; ++sg) {
                    const float2 z = zbuf[g * 18 + sg];
                    // (z.x + i z.y)(u.x - i u.y)
                    r0[sg].x = fmaf(z.x, u.x, fmaf(z.y, u.y, r0[sg].x));
                    r0[sg].y = fmaf(z.y, u.x, fmaf(-z.x, u.y, r0[sg].y));
                }
            }
            __syncwarp();
            float2* r0buf = zbuf;
            if (lane < W) {
#pragma unroll
                for (int sg = 0; sg < H; ++sg) r0buf[sg * W + lane] = r0[sg];
            }
            __syncwarp();
            // gather into rank order, scale, first scores
            float4 R[NS];
#pragma unroll
            for (int i = 0; i < NS; ++i) {
                const int r = 64 * i + 2 * lane;
                const int s0 = __ldg(a.wc.src + r), s1 = __ldg(a.wc.src + r + 1);
                const float2 sc = __ldg(scale2 + 32 * i + lane);
                float2 v0 = r0buf[s0 & 0xffff], v1 = r0buf[s1 & 0xffff];
                if (s0 & (1 << 30)) v0.y = -v0.y;
                if (s1 & (1 << 30)) v1.y = -v1.y;
                float2 re = make_float2(v0.x, v1.x), im = make_float2(v0.y, v1.y);
                re = __fmul2_rn(sc, re);
                im = __fmul2_rn(sc, im);
                R[i] = make_float4(re.x, re.y, im.x, im.y);
            }
            __syncwarp();
            float lmax = score_pass<NS>(R, lane, sbuf);

            // synthesis accumulators: pixel p = lane + 32 j of the B x B block
            float acc[PPL];
#pragma unroll
            for (int j = 0; j < PPL; ++j) acc[j] = 0.f;
            const int rw = tk.block_row - tk.origin_row, cw = tk.block_col - tk.origin_col;
            const bool tracing = a.trace_picks != nullptr && ti == 0;

            int it = 0;
            for (; it < a.iterations; ++it) {
                __syncwarp();
                // ---- argmax over the warp (NaN = inadmissible, ignored by max) ----
                float gmax = lmax;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1)
                    gmax = fmaxf(gmax, __shfl_xor_sync(FULL, gmax, off));
                if (gmax != gmax) break;  // no admissible frequency (rljsde.cpp:159)
                const unsigned cand = __ballot_sync(FULL, lmax == gmax);
                const int L0 = __ffs(cand) - 1;
                const float sv = lane < NS ? sbuf[L0 * kSbufStride + lane] : qnan();
                const unsigned sm = __ballot_sync(FULL, sv == gmax);
                int u, Lw, slot, b;
                float4 v;
                if (__popc(cand) == 1 && __popc(sm) == 1) {
                    Lw = L0;
                    slot = __ffs(sm) - 1;
                    v = pick_slot<NS>(R, slot);
                    const float e0 = fmaf(v.z, v.z, v.x * v.x);
                    const float e1 = fmaf(v.w, v.w, v.y * v.y);
                    const int b0 = e0 == gmax, b1 = e1 == gmax;
                    int bb = b0 ? 0 : 1;
                    if (b0 && b1) {
                        const int r0i = 64 * slot + 2 * lane;
                        bb = __ldg(a.wc.perm + r0i) < __ldg(a.wc.perm + r0i + 1) ? 0 : 1;
                    }
                    b = __shfl_sync(FULL, bb, Lw);
                    u = 64 * slot + 2 * Lw + b;
                } else {
                    // general tie path: smallest flat index among all maxima
                    unsigned key = 0xffffffffu;
#pragma unroll
                    for (int i = 0; i < NS; ++i) {
                        const float e0 = fmaf(R[i].z, R[i].z, R[i].x * R[i].x);
                        const float e1 = fmaf(R[i].w, R[i].w, R[i].y * R[i].y);
                        const int r = 64 * i + 2 * lane;
                        if (e0 == gmax) key = min(key, (unsigned(__ldg(a.wc.perm + r)) << 12) | r);
                        if (e1 == gmax)
                            key = min(key, (unsigned(__ldg(a.wc.perm + r + 1)) << 12) | (r + 1));
                    }
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1)
                        key = min(key, __shfl_xor_sync(FULL, key, off));
                    u = key & 0xfff;
                    slot = u >> 6;
                    Lw = (u >> 1) & 31;
                    b = u & 1;
                    v = pick_slot<NS>(R, slot);
                }
                const float ure = __shfl_sync(FULL, b ? v.y : v.x, Lw);
                const float uim = __shfl_sync(FULL, b ? v.w : v.z, Lw);
                const float f = __ldg(ct.fac + u);
                const float gre = f * ure, gim = f * uim;
                const int kflat = __ldg(a.wc.perm + u);
                const int sigma = kflat / W, rho = kflat % W;
                // ---- synthesis of the kept block pixels ----
#pragma unroll
                for (int j = 0; j < PPL; ++j) {
                    const int p = lane + 32 * j;
                    if (p < nb2) {
                        const int eta = rw + p / B, gam = cw + p % B;
                        const float2 ph = unit[(eta * sigma + gam * rho) % W];
                        acc[j] = fmaf(gre, ph.x, fmaf(-gim, ph.y, acc[j]));
                    }
                }
                if (tracing && lane == 0) {
                    a.trace_picks[it] = kflat;
                    a.trace_gd[2 * it] = gre;
                    a.trace_gd[2 * it + 1] = gim;
                }
                // ---- rank-1 update streamed from C'[:,u], fused with the next scores ----
                __syncwarp();  // locate reads of sbuf complete before it is rewritten
                const float4* col = (u < a.hot ? hot : gcols) + size_t(u) * COLF4;
                lmax = update_pass<NS>(R, col, lane, gre, gim, sbuf);
            }
            // ---- placement: clip + crop straight into the output ----
#pragma unroll
            for (int j = 0; j < PPL; ++j) {
                const int p = lane + 32 * j;
                if (p < nb2) {
                    const int orow = tk.block_row + p / B, ocol = tk.block_col + p % B;
                    if (orow < a.out_rows && ocol < a.out_cols) {
                        float val = acc[j];
                        if (a.clip) val = fminf(fmaxf(val, 0.f), 1.f);
                        a.out[size_t(orow - a.out_row0) * a.out_cols + ocol] = double(val);
                    }
                }
            }
            if (tracing) {
                if (lane == 0) *a.trace_n = it;
                if (a.trace_window) {
                    __syncwarp();
                    for (int p = lane; p < W * W; p += 32) {
                        const int eta = p / W, gam = p % W;
                        float s = 0.f;
                        for (int t = 0; t < it; ++t) {
                            const int k = a.trace_picks[t];
                            const float2 ph = unit[(eta * (k / W) + gam * (k % W)) % W];
                            s = fmaf(float(a.trace_gd[2 * t]), ph.x,
                                     fmaf(-float(a.trace_gd[2 * t + 1]), ph.y, s));
                        }
                        a.trace_window[p] = s;
                    }
                }
            }
        }
    }
}

template <int NS, int W, int PPL>
int launch_one(const SolveArgs& a, cudaStream_t stream, int num_sms) {
    const size_t smem = solve_f32_smem_bytes(NS, a.hot) ;
    auto kern = k_solve_f32<NS, W, PPL>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(smem));
    if (e != cudaSuccess) return e;
    int grid = a.n_items < num_sms ? a.n_items : num_sms;
    if (grid < 1) grid = 1;
    kern<<<grid, kWarpsF32 * 32, smem, stream>>>(a);
    return cudaGetLastError();
}

template <int W>
int launch_w(const SolveArgs& a, int n_slots, cudaStream_t s, int num_sms) {
    const int nb2 = a.block * a.block;
    constexpr int NSW = (W * W + 63) / 64 <= 1   ? 1
                        : (W * W + 63) / 64 <= 2 ? 2
                        : (W * W + 63) / 64 <= 4 ? 4
                        : (W * W + 63) / 64 <= 8 ? 8
                                                 : 16;
    if (n_slots != NSW) return cudaErrorInvalidValue;
    if (nb2 <= 32) return launch_one<NSW, W, 1>(a, s, num_sms);
    if (nb2 <= 64) return launch_one<NSW, W, 2>(a, s, num_sms);
    if (nb2 <= 128) return launch_one<NSW, W, 4>(a, s, num_sms);
    if (nb2 <= 256) return launch_one<NSW, W, 8>(a, s, num_sms);
    return cudaErrorInvalidValue;
}

} // namespace

size_t solve_f32_smem_bytes(int n_slots, int hot) {
    // hot columns + unit table + per-warp scratch (sized for W = 32, the largest)
    return size_t(hot) * n_slots * 32 * 16 + 2 * 32 * 4 +
           size_t(kWarpsF32) * Scratch<32>::kFloats * 4;
}

int solve_f32_max_hot(int n_slots, int device) {
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    const long base = long(solve_f32_smem_bytes(n_slots, 0)) + 64;  // static smem margin
    const long col = long(n_slots) * 32 * 16;
    const long h = (long(optin) - base) / col;
    return h < 0 ? 0 : int(h);
}

int launch_solve_f32(const SolveArgs& a, int n_slots, void* stream, int num_sms) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    switch (a.window) {
        case 2: return launch_w<2>(a, n_slots, s, num_sms);
        case 4: return launch_w<4>(a, n_slots, s, num_sms);
        case 6: return launch_w<6>(a, n_slots, s, num_sms);
        case 8: return launch_w<8>(a, n_slots, s, num_sms);
        case 10: return launch_w<10>(a, n_slots, s, num_sms);
        case 12: return launch_w<12>(a, n_slots, s, num_sms);
        case 14: return launch_w<14>(a, n_slots, s, num_sms);
        case 16: return launch_w<16>(a, n_slots, s, num_sms);
        case 18: return launch_w<18>(a, n_slots, s, num_sms);
        case 20: return launch_w<20>(a, n_slots, s, num_sms);
        case 22: return launch_w<22>(a, n_slots, s, num_sms);
        case 24: return launch_w<24>(a, n_slots, s, num_sms);
        case 26: return launch_w<26>(a, n_slots, s, num_sms);
        case 28: return launch_w<28>(a, n_slots, s, num_sms);
        case 30: return launch_w<30>(a, n_slots, s, num_sms);
        case 32: return launch_w<32>(a, n_slots, s, num_sms);
        default: return cudaErrorInvalidValue;
    }
}

} // namespace tqsb
