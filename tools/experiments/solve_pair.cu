// EXPERIMENT (not built; measured slower than the product kernel):
// TMEM-resident residuals with two target blocks per warp. Build it by copying into
// paper_2205_02646_b200/csrc/, adding it to build.py's CU list and routing
// launch_solve_f32 to launch_solve_pair for NS == 16 (and declaring launch_solve_pair /
// solve_pair_smem_bytes in tqsb_internal.hpp). Results are bitwise identical to k_solve_f32.
//
// solve_pair.cu -- the fp32 product solve with TMEM-resident residuals, two target
// blocks per warp (K2+K3+K4, same algorithm and arithmetic as solve_f32.cu).
//
// Why: the per-iteration chain of one block (argmax -> owner lane and position ->
// R'_u -> step g -> column) is serial, and with one block per warp (64 registers of
// residual per lane) only 3 warps per SM sub-partition fit, so ~45 % of issue slots
// stayed empty waiting on that chain. Here each lane keeps its
// residual slots in tensor memory (TMEM, 512 columns x 128 lanes per SM) instead of
// registers, and each warp owns two blocks A and B and alternates between them:
//
//     half(A, B): update A (stream R'_A chunks TMEM -> registers -> TMEM, fused with
//                 the next keys) while B's chain resolves (CREDUX, ballot, the TMEM
//                 read of B's picked slot, the step, B's first column chunks)
//     half(B, A): the same with the roles swapped
//
// so one block's chain latency hides behind the other block's update in the same
// instruction stream. The register pick (a 5-deep branch tree over 32 elements) is
// replaced by one tcgen05.ld of the picked slot. Per block and iteration the
// arithmetic is exactly the one of solve_f32.cu (same FFMA2 sequences, same packed
// selection keys, same per-pick synthesis order), so results are bitwise identical.
//
// TMEM layout: warp w uses lane quadrant w % 4; its blocks A/B own the 64 columns at
// 128 * (w / 4) + {0, 64}; column 4 i + j of a block holds component j of slot i
// (re_a, re_b, im_a, im_b), i.e. the register float4 R[i] of solve_f32.cu.
#include <cuda_runtime.h>

#include <cstdint>

#include "tqsb_internal.hpp"
#include "solve_common.cuh"

#ifndef TQSB_WARPS_PAIR
#define TQSB_WARPS_PAIR 12
#endif

namespace tqsb {
namespace dev {
// ---------------------------------------------------------------------------
// K2 init of one block (rljsde.cpp:127-138) as the separable 2-D DFT of the window
// image a(eta,gamma) = (w_m/3) y_m (see solve_f32.cu's header), gathered into rank
// order and scaled: R[i] = (re_a, re_b, im_a, im_b) of ranks 64 i + 2 lane + {0,1}.
// scr: per-warp scratch of InitScratch<W>::kFloats floats.
// ---------------------------------------------------------------------------
template <int W>
struct InitScratch {
    static constexpr int kZ = 32 * 18 * 2;
    static constexpr int kR = (W / 2 + 1) * 32 * 2;
    static constexpr int kFloats = kZ > kR ? kZ : kR;
};

template <int NS, int W>
__device__ __forceinline__ void init_residual(const SolveArgs& a, const Task& tk, const ClassTab& ct,
                                              int lane, const float2* unit, float* scr,
                                              float4 (&R)[NS]) {
    const float2* __restrict__ scale2 = reinterpret_cast<const float2*>(ct.scale);
    float2* zbuf = reinterpret_cast<float2*>(scr);
    float colv[W];
    {
        int fc = (tk.origin_col + lane) >> 1;
        fc = fc < a.frame_cols - 1 ? fc : a.frame_cols - 1;
#pragma unroll
        for (int eta = 0; eta < W; ++eta) {
            float v = 0.f;
            if (lane < W) {
                const float mk = __ldg(ct.mask32 + eta * W + lane);
                int fr = (tk.origin_row + eta) >> 1;
                fr = fr < a.frame_rows - 1 ? fr : a.frame_rows - 1;
                const double y = __ldg(a.frame + size_t(fr - a.frame_row0) * a.frame_pitch + fc);
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
        const float2 u = unit[(g * lane) % W];
#pragma unroll
        for (int sg = 0; sg < H; ++sg) {
            const float2 z = zbuf[g * 18 + sg];
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
    // gather into rank order and scale: R'_r = s_r R0[perm r]
#pragma unroll
    for (int i = 0; i < NS; ++i) {
        const int r = 64 * i + 2 * lane;
        const int s0 = __ldg(a.wc.src + r), s1 = __ldg(a.wc.src + r + 1);
        const float2 sc = __ldg(scale2 + 32 * i + lane);
        float2 v0 = r0buf[s0 & 0xffff], v1 = r0buf[s1 & 0xffff];
        if (s0 & (1 << 30)) v0.y = -v0.y;
        if (s1 & (1 << 30)) v1.y = -v1.y;
        const float2 re = __fmul2_rn(sc, make_float2(v0.x, v1.x));
        const float2 im = __fmul2_rn(sc, make_float2(v0.y, v1.y));
        R[i] = make_float4(re.x, re.y, im.x, im.y);
    }
    __syncwarp();
}

}  // namespace dev
}  // namespace tqsb

namespace tqsb {
size_t solve_pair_smem_bytes();
int launch_solve_pair(const SolveArgs& a, void* stream, int num_sms);
namespace {

using namespace dev;

#ifndef TQSB_PAIR_DEP
#define TQSB_PAIR_DEP 1
#endif
#ifndef TQSB_PAIR_PF
#define TQSB_PAIR_PF 2  // column prefetch into L1: 1 prefetch.global.L1, 2 dummy loads
#endif
constexpr int kWarpsPair = TQSB_WARPS_PAIR;
static_assert(kWarpsPair % 4 == 0 && kWarpsPair / 4 * 128 <= 512, "TMEM: 128 columns per warp");

// ---- TMEM helpers (16 / 4 consecutive 32-bit columns per lane) ----
__device__ __forceinline__ void tm_ld16(uint32_t ta, float4 (&r)[4]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=f"(r[0].x), "=f"(r[0].y), "=f"(r[0].z), "=f"(r[0].w), "=f"(r[1].x), "=f"(r[1].y),
          "=f"(r[1].z), "=f"(r[1].w), "=f"(r[2].x), "=f"(r[2].y), "=f"(r[2].z), "=f"(r[2].w),
          "=f"(r[3].x), "=f"(r[3].y), "=f"(r[3].z), "=f"(r[3].w)
        : "r"(ta));
}
__device__ __forceinline__ void tm_st16(uint32_t ta, const float4 (&r)[4]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
        ::"r"(ta), "f"(r[0].x), "f"(r[0].y), "f"(r[0].z), "f"(r[0].w), "f"(r[1].x), "f"(r[1].y),
          "f"(r[1].z), "f"(r[1].w), "f"(r[2].x), "f"(r[2].y), "f"(r[2].z), "f"(r[2].w),
          "f"(r[3].x), "f"(r[3].y), "f"(r[3].z), "f"(r[3].w));
}
__device__ __forceinline__ void tm_ld4(uint32_t ta, float4& v) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(ta));
}
// wait::ld completes every outstanding tcgen05.ld of the thread; the registers they
// write are threaded through as in/out operands so no use is scheduled above it
__device__ __forceinline__ void tm_wait_ld_rr(float4 (&r)[4], float4 (&s)[4]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+f"(r[0].x), "+f"(r[0].y), "+f"(r[0].z), "+f"(r[0].w), "+f"(r[1].x), "+f"(r[1].y),
                   "+f"(r[1].z), "+f"(r[1].w), "+f"(r[2].x), "+f"(r[2].y), "+f"(r[2].z), "+f"(r[2].w),
                   "+f"(r[3].x), "+f"(r[3].y), "+f"(r[3].z), "+f"(r[3].w), "+f"(s[0].x), "+f"(s[0].y),
                   "+f"(s[0].z), "+f"(s[0].w), "+f"(s[1].x), "+f"(s[1].y), "+f"(s[1].z), "+f"(s[1].w),
                   "+f"(s[2].x), "+f"(s[2].y), "+f"(s[2].z), "+f"(s[2].w), "+f"(s[3].x), "+f"(s[3].y),
                   "+f"(s[3].z), "+f"(s[3].w)::"memory");
}
__device__ __forceinline__ void tm_wait_ld2(float4 (&r)[4], float4 (&s)[4], float4& v) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+f"(r[0].x), "+f"(r[0].y), "+f"(r[0].z), "+f"(r[0].w), "+f"(r[1].x), "+f"(r[1].y),
                   "+f"(r[1].z), "+f"(r[1].w), "+f"(r[2].x), "+f"(r[2].y), "+f"(r[2].z), "+f"(r[2].w),
                   "+f"(r[3].x), "+f"(r[3].y), "+f"(r[3].z), "+f"(r[3].w), "+f"(s[0].x), "+f"(s[0].y),
                   "+f"(s[0].z), "+f"(s[0].w), "+f"(s[1].x), "+f"(s[1].y), "+f"(s[1].z), "+f"(s[1].w),
                   "+f"(s[2].x), "+f"(s[2].y), "+f"(s[2].z), "+f"(s[2].w), "+f"(s[3].x), "+f"(s[3].y),
                   "+f"(s[3].z), "+f"(s[3].w), "+f"(v.x), "+f"(v.y), "+f"(v.z), "+f"(v.w)::"memory");
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// One block's state between half-steps (all warp-uniform except the per-lane parts).
template <int PPL>
struct Blk {
    const float4* cols;  // C' of the block's class (+ lane)
    const float* fac;    // gamma / (s_u D_u) per rank
    uint32_t tm;         // TMEM address of the block's 64 residual columns
    float lmax;          // lane key max after the last update
    float gre, gim;      // step of the pending pick
    int kflat;           // flat k of the pending pick (synthesis)
    bool live;           // false once no admissible frequency remains (rljsde.cpp:159)
    const float4* col;   // column of the pending pick (+ lane)
    float acc[PPL];
    unsigned pe[PPL], pg[PPL];
};

template <int W, int PPL>
__global__ void __launch_bounds__(kWarpsPair * 32, 1) k_solve_pair(const SolveArgs a) {
    constexpr int NS = 16;
    constexpr int COLF4 = NS * 32;
    constexpr int SCR = InitScratch<W>::kFloats;
    extern __shared__ __align__(16) float smem[];
    float2* unit = reinterpret_cast<float2*>(smem);  // W (cos, sin)
    float* scr_all = reinterpret_cast<float*>(unit + 32);
    __shared__ uint32_t s_tmem;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float* scr = scr_all + warp * SCR;
    if (threadIdx.x < W)
        unit[threadIdx.x] = make_float2(a.wc.unit32[2 * threadIdx.x], a.wc.unit32[2 * threadIdx.x + 1]);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            static_cast<unsigned>(__cvta_generic_to_shared(&s_tmem))));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tmem_sync_all();
    const uint32_t tw = s_tmem + (uint32_t(32 * (warp & 3)) << 16) + uint32_t(128 * (warp >> 2));

    const int B = a.block, nb2 = B * B;
    int p_r[PPL], p_c[PPL];
#pragma unroll
    for (int j = 0; j < PPL; ++j) {
        const int p = lane + 32 * j;
        p_r[j] = p < nb2 ? p / B : -1;
        p_c[j] = p < nb2 ? p % B : 0;
    }
    const int* __restrict__ perm = a.wc.perm;

    // init of one block (solve_f32.cu's K2, shared helper) -> TMEM, lane key max
    auto start = [&](Blk<PPL>& X, int ti, uint32_t tm) {
        const ClassTab& ct = a.tabs[__ldg(a.task_cls + ti)];
        const Task tk = a.tasks[ti];
        float4 R[NS];
        init_residual<NS, W>(a, tk, ct, lane, unit, scr, R);
        X.lmax = score_pass_keys<NS>(R);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            float4 t4[4] = {R[4 * k], R[4 * k + 1], R[4 * k + 2], R[4 * k + 3]};
            tm_st16(tm + uint32_t(16 * k), t4);
        }
        X.cols = reinterpret_cast<const float4*>(ct.cpack) + lane;
        X.fac = ct.fac;
        X.tm = tm;
        X.live = true;
        const int rw = tk.block_row - tk.origin_row, cw = tk.block_col - tk.origin_col;
#pragma unroll
        for (int j = 0; j < PPL; ++j) {
            X.acc[j] = 0.f;
            X.pe[j] = unsigned(rw + (p_r[j] < 0 ? 0 : p_r[j]));
            X.pg[j] = unsigned(cw + p_c[j]);
        }
    };

    // chain of Y: argmax -> (lane, position) -> u; first column chunks, factor, flat k;
    // the picked slot from TMEM. Returns the slot's (re, im) candidates in v (still
    // in flight: completed by the next tcgen05.wait::ld) and the owner lane.
    auto chain = [&](Blk<PPL>& Y, float4& v, int& Lw, int& half, float& fac) {
        const float gmax = warp_max_f32(Y.lmax);
        if (gmax != gmax) {  // no admissible frequency
            Y.live = false;
            return;
        }
        int t;
        asm volatile("mov.b32 %0, %1;" : "=r"(t) : "r"(31 - int(__float_as_uint(gmax) & 31u)));
        Lw = __ffs(__ballot_sync(FULL, Y.lmax == gmax)) - 1;
        const int slot = t >> 1;
        half = t & 1;
        const int u = 64 * slot + 2 * Lw + half;
        Y.col = Y.cols + size_t(u) * COLF4;
        // the column's 64 lines of 128 B into L1 (no registers held across the
        // half-step; the update streams it from L1)
        {
            const char* cl = reinterpret_cast<const char*>(Y.col - lane) + 128 * lane;
#if TQSB_PAIR_PF == 1
            asm volatile("prefetch.global.L1 [%0];" ::"l"(cl));
            asm volatile("prefetch.global.L1 [%0];" ::"l"(cl + 4096));
#else
            // two 4-byte loads per lane into registers that are never read: the lines
            // land in L1 like any ld.global.nc, the registers free once they arrive
            unsigned d0, d1;
            asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(d0) : "l"(cl));
            asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(d1) : "l"(cl + 4096));
#endif
        }
        fac = __ldg(Y.fac + u);
        Y.kflat = __ldg(perm + u);
        tm_wait_st();  // Y's residual stores (its last update) are complete
        tm_ld4(Y.tm + uint32_t(4 * slot), v);
    };
    auto finish_chain = [&](Blk<PPL>& Y, const float4& v, int Lw, int half, float fac) {
        const float pre = half ? v.y : v.x, pim = half ? v.w : v.z;
        const float ure = __shfl_sync(FULL, pre, Lw), uim = __shfl_sync(FULL, pim, Lw);
        Y.gre = fac * ure;
        Y.gim = fac * uim;
    };
    auto synth = [&](Blk<PPL>& Y) {
        const unsigned sigma = unsigned(Y.kflat) / W, rho = unsigned(Y.kflat) % W;
#pragma unroll
        for (int j = 0; j < PPL; ++j) {
            const float2 ph = unit[(Y.pe[j] * sigma + Y.pg[j] * rho) % unsigned(W)];
            Y.acc[j] = fmaf(Y.gre, ph.x, fmaf(-Y.gim, ph.y, Y.acc[j]));
        }
    };

    // update X with its pending pick (R'_X -= g C'[:,u], fused keys), TMEM round trip;
    // Y's chain is interleaved (do_chain: Y is live and needs a pick this half-step)
    auto half_step = [&](Blk<PPL>& X, Blk<PPL>& Y, bool do_chain) {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        int Lw = 0, hf = 0;
        float fac = 0.f;
        if (do_chain) chain(Y, v, Lw, hf, fac);
        const bool yc = do_chain && Y.live;
        if (X.live) {
            float4 r0[4], r1[4], ca[4], cb[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) ca[q] = __ldg(X.col + 32 * q);
#pragma unroll
            for (int q = 0; q < 4; ++q) cb[q] = __ldg(X.col + 32 * (4 + q));
            tm_wait_st();
            tm_ld16(X.tm, r0);
            tm_ld16(X.tm + 16u, r1);
            tm_wait_ld2(r0, r1, v);
            if (yc) finish_chain(Y, v, Lw, hf, fac);
            const float2 ngre = make_float2(-X.gre, -X.gre), pgim = make_float2(X.gim, X.gim),
                         ngim = make_float2(-X.gim, -X.gim);
            float m4[4] = {qnan(), qnan(), qnan(), qnan()};
            const unsigned kmask = keymask();
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                float4(&r)[4] = (k & 1) ? r1 : r0;
                float4(&cc)[4] = (k & 1) ? cb : ca;
                if (k == 2) tm_wait_ld_rr(r0, r1);  // residual chunks 2 and 3
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int i = 4 * k + q;
                    const float2 cre = make_float2(cc[q].x, cc[q].y), cim = make_float2(cc[q].z, cc[q].w);
                    float2 re = make_float2(r[q].x, r[q].y), im = make_float2(r[q].z, r[q].w);
                    re = __ffma2_rn(ngre, cre, re);
                    re = __ffma2_rn(pgim, cim, re);
                    im = __ffma2_rn(ngre, cim, im);
                    im = __ffma2_rn(ngim, cre, im);
                    r[q] = make_float4(re.x, re.y, im.x, im.y);
                    const float2 sc = __ffma2_rn(im, im, __fmul2_rn(re, re));
                    m4[i & 3] = fmax3(m4[i & 3], score_key(sc.x, 2 * i, kmask), score_key(sc.y, 2 * i + 1, kmask));
                }
                tm_st16(X.tm + uint32_t(16 * k), r);
                if (k < 2) {  // chunk k + 2 of the residual (TMEM) and of the column (L1)
                    tm_ld16(X.tm + uint32_t(16 * (k + 2)), r);
                    // (zero) dependency on this chunk's keys: ptxas may not hoist the load
                    // above the chunk, so the column never holds more than 32 registers
                    const int dep = TQSB_PAIR_DEP ? int(__float_as_uint(m4[3]) >> 31) : 0;
#pragma unroll
                    for (int q = 0; q < 4; ++q) cc[q] = __ldg(X.col + dep + 32 * (4 * (k + 2) + q));
                }
            }
            X.lmax = fmax3(fmax3(m4[0], m4[1], m4[2]), m4[3], qnan());
            synth(X);
        } else if (yc) {
            asm volatile("tcgen05.wait::ld.sync.aligned;" : "+f"(v.x), "+f"(v.y), "+f"(v.z), "+f"(v.w)::"memory");
            finish_chain(Y, v, Lw, hf, fac);
        }
    };

    auto place = [&](const Blk<PPL>& X, int ti) {
        const Task tk = a.tasks[ti];
#pragma unroll
        for (int j = 0; j < PPL; ++j) {
            const int pr = p_r[j], pcc = p_c[j];
            if (pr >= 0) {
                const int orow = tk.block_row + pr, ocol = tk.block_col + pcc;
                if (orow < a.out_rows && ocol < a.out_cols) {
                    float val = X.acc[j];
                    if (a.clip) val = fminf(fmaxf(val, 0.f), 1.f);
                    a.out[size_t(orow - a.out_row0) * a.out_cols + ocol] = double(val);
                }
            }
        }
    };

    Blk<PPL> A, Bk;
    for (;;) {
        int ti = 0;
        if (lane == 0) ti = atomicAdd(a.counter, 2);
        ti = __shfl_sync(FULL, ti, 0);
        if (ti >= a.n_tasks) break;
        const bool hasB = ti + 1 < a.n_tasks;
        start(A, ti, tw);
        if (hasB) {
            start(Bk, ti + 1, tw + 64u);
        } else {
            Bk.live = false;
            Bk.lmax = qnan();
#pragma unroll
            for (int j = 0; j < PPL; ++j) Bk.acc[j] = 0.f, Bk.pe[j] = 0u, Bk.pg[j] = 0u;
        }
        const int iters = a.iterations;
        if (iters > 0) {
            // A's first pick, unoverlapped
            {
                float4 v;
                int Lw = 0, hf = 0;
                float fac = 0.f;
                tm_wait_st();
                chain(A, v, Lw, hf, fac);
                if (A.live) {
                    asm volatile("tcgen05.wait::ld.sync.aligned;" : "+f"(v.x), "+f"(v.y), "+f"(v.z), "+f"(v.w)::"memory");
                    finish_chain(A, v, Lw, hf, fac);
                }
            }
            for (int it = 0; it < iters; ++it) {
                half_step(A, Bk, Bk.live);                  // update A (pick it), chain B (pick it)
                half_step(Bk, A, A.live && it + 1 < iters);  // update B (pick it), chain A (pick it+1)
                if (!A.live && !Bk.live) break;
            }
        }
        place(A, ti);
        if (hasB) place(Bk, ti + 1);
        tm_wait_st();
        __syncwarp();
    }
    tmem_sync_all();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s_tmem));
}

template <int W>
int launch_pair_w(const SolveArgs& a, cudaStream_t stream, int num_sms) {
    const int nb2 = a.block * a.block;
    const size_t smem = solve_pair_smem_bytes();
    auto pick = [&](auto kern) -> int {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return e;
        kern<<<num_sms, kWarpsPair * 32, smem, stream>>>(a);
        return cudaGetLastError();
    };
    if (nb2 <= 32) return pick(k_solve_pair<W, 1>);
    if (nb2 <= 64) return pick(k_solve_pair<W, 2>);
    if (nb2 <= 128) return pick(k_solve_pair<W, 4>);
    if (nb2 <= 256) return pick(k_solve_pair<W, 8>);
    return cudaErrorInvalidValue;
}

} // namespace

size_t solve_pair_smem_bytes() {
    return 32 * 8 + size_t(kWarpsPair) * InitScratch<32>::kFloats * 4;
}

// NS == 16 windows (W = 24..32) only; smaller windows use solve_f32.cu
int launch_solve_pair(const SolveArgs& a, void* stream, int num_sms) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    switch (a.window) {
        case 32: return launch_pair_w<32>(a, s, num_sms);
#ifndef TQSB_ONLY_W32
        case 30: return launch_pair_w<30>(a, s, num_sms);
        case 28: return launch_pair_w<28>(a, s, num_sms);
        case 26: return launch_pair_w<26>(a, s, num_sms);
        case 24: return launch_pair_w<24>(a, s, num_sms);
#endif
        default: return cudaErrorInvalidValue;
    }
}

} // namespace tqsb
