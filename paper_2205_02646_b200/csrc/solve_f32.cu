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
//  loop (K3)   nu x { argmax_k q_k |R_k|^2 / D_k over D_k > 0 (rljsde.cpp:144-158,
//              basis.hpp:90-92); R -= gamma (R_u/D_u) C[:,u] (160-172) } on the SCALED
//              residual R'_k = sqrt(q_k/D_k) R_k, so the score is |R'_k|^2 and the update
//              streams C'[s,u] = s_s C[s,u] -- 2 FFMA2 per complex element, 2 more for the
//              score. Selection: each score carries its in-lane position in its low 5
//              mantissa bits (score_key), one FMNMX3 tree + CREDUX give max and position,
//              a ballot the lane; conjugate pairs sit on one lane's slot halves so their
//              bitwise ties resolve to the smaller flat k like the reference's.
//  synth (K4)  only the B x B target pixels of sum Re(g unit[(eta sigma + gamma rho)])
//              (basis.cpp:52-73 restricted to the kept block, pipeline.cpp:157-166),
//              accumulated per pick, clipped and stored straight into the output.
//
// Register layout: lane j, slot i holds ranks r = 64 i + 2 j + {0,1} as one float4
// (re_a, re_b, im_a, im_b); ranks order frequencies by centred radius (hot first). The
// C' column of rank u is the same float4 array, so a column read is 32 lanes x 16 B =
// one fully coalesced 512 B line per slot, streamed in 4-slot chunks two chunks ahead
// of the update (L1/L2; optionally the lowest ranks from TMEM, template TM).
// Scheduling: warps take blocks from a global counter (DYN) -- or, with the TMEM tier
// or tracing, CTAs stride over 48-block single-class work items.
#include <cuda_runtime.h>

#include <cstdint>

#include "tqsb_internal.hpp"
#include "solve_common.cuh"

#ifndef TQSB_KEYS
// packed score/position keys (see score_key). TQSB_KEYS=0 builds the exact-selection
// variant (score buffer + smallest-flat-index tie scan), kept as the reference for the
// keys' share of fp32 path forks (profiles/r02_parity.md, tools/parity_r02.py)
#define TQSB_KEYS 1
#endif
#ifndef TQSB_DYN
#define TQSB_DYN 1  // warp-level dynamic task scheduling when no CTA-wide class state is needed
#endif
#ifndef TQSB_INIT_FFT
#define TQSB_INIT_FFT 1  // W = 32: the init's second DFT stage as a shuffle FFT across lanes
#endif
#ifndef TQSB_AHEAD
#define TQSB_AHEAD 2  // 4-slot column chunks in flight ahead of the update (NS == 16)
#endif
#ifndef TQSB_SMEM_PAD
#define TQSB_SMEM_PAD 0  // experiment builds: extra shared memory (a larger carveout, less L1)
#endif
#ifndef TQSB_GATHER_SHARE
// W = 32 (shuffle-FFT init): warps per half-spectrum staging buffer, taken in turns. 16 =
// one 4.3 KB buffer per CTA: the CTA needs 5 KB of shared memory, the 8 KB carveout
// leaves L1 248 KB for C' columns (hit rate 63 -> 74 %; 4K frame 34.53 -> 32.84 ms;
// 1 / 2 / 4 / 8 warps per buffer: 33.80 / 33.44 / 33.10 / 32.94)
#define TQSB_GATHER_SHARE 16
#endif

namespace tqsb {
namespace {

using namespace dev;


// per-warp scratch floats: the init transpose buffer zbuf[gamma][sigma] (float2,
// row stride 18) / half-spectrum r0buf[sigma][rho], aliased with the element-score
// buffer sbuf[lane][2*NS] (row stride kSbufStride floats) of the exact-selection build.
// With the shuffle FFT and packed keys (the product path) only r0buf remains, and
// kShare warps share one
template <int W>
struct Scratch {
    static constexpr bool kFFT = W == 32 && TQSB_INIT_FFT;
    static constexpr int kZ = kFFT ? 0 : 32 * 18 * 2;
    static constexpr int kR = (W / 2 + 1) * 32 * 2;
    static constexpr int kS = TQSB_KEYS ? 0 : 32 * kSbufStride;
    static constexpr int kFloats = (kZ > kR ? (kZ > kS ? kZ : kS) : (kR > kS ? kR : kS));
    static constexpr int kShare = kFFT && TQSB_KEYS ? TQSB_GATHER_SHARE : 1;
    static constexpr int buffers(int warps) { return (warps + kShare - 1) / kShare; }
};

// (fac, k) rank table in shared memory: read by the static-item schedule and the exact
// tie scan; the dynamic schedule with packed keys reads both through L1 instead
template <bool DYN>
__host__ __device__ constexpr int meta_ranks(int kp) { return DYN && TQSB_KEYS ? 0 : kp; }

template <int W, bool DYN>
size_t smem_bytes(int n_slots, int warps) {
    return size_t(meta_ranks<DYN>(n_slots * 64)) * 8 + 32 * 8 + 32 * 16 +
           size_t(Scratch<W>::buffers(warps)) * Scratch<W>::kFloats * 4 + TQSB_SMEM_PAD;
}

// NW warps per CTA (1 CTA per SM): 16 at 128 registers where the kernel fits without
// spilling in the loop (the default W = 32 / B = 4 product path: 38.8 vs 40.5 ms per 4K frame at 12),
// 12 at 168 registers for the heavier instantiations (B >= 8, TMEM tier, tracing)
// SP: the streamed host-buffer variant (SolveArgs::progress, chunk-tagged
// task list); a separate instantiation so the device-resident path carries none of it
template <int NS, int W, int PPL, bool TRACE, bool TM, int NW, bool SP = false>
__global__ void __launch_bounds__(NW * 32, 1) k_solve_f32(const SolveArgs a) {
    constexpr bool DYN = !TRACE && !TM && TQSB_DYN;  // per-warp task queue (a.counter)
    static_assert(!SP || DYN, "streamed completion needs the warp-level task queue");
    extern __shared__ __align__(16) float smem[];
    constexpr int COLF4 = NS * 32;  // float4 per column
    constexpr int KP = NS * 64;     // padded frequency count
    constexpr int SCR = Scratch<W>::kFloats;
    // KP x (gamma/(s_u D_u) bits, flat k) per rank u (not allocated for DYN + keys)
    int2* s_meta = reinterpret_cast<int2*>(smem);
    float2* unit = reinterpret_cast<float2*>(s_meta + meta_ranks<DYN>(KP));   // W (cos, sin)
    float4* unit4 = reinterpret_cast<float4*>(unit + 32);    // W (cos, -sin, sin, -sin): init
    float* scr_all = reinterpret_cast<float*>(unit4 + 32);
    __shared__ int s_cls;
    __shared__ uint32_t s_tmem;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int kShare = Scratch<W>::kShare;
    float* scr = scr_all + (warp / kShare) * SCR;
    __shared__ int s_glock[NW];  // staging-buffer locks (kShare > 1)
    int* glock = s_glock + warp / kShare;
    if (threadIdx.x < NW) s_glock[threadIdx.x] = 0;
    float2* zbuf = reinterpret_cast<float2*>(scr);
    float* srow = scr + lane * kSbufStride;  // this lane's element scores

    if (threadIdx.x < W) {
        const float cs = a.wc.unit32[2 * threadIdx.x], sn = a.wc.unit32[2 * threadIdx.x + 1];
        unit[threadIdx.x] = make_float2(cs, sn);
        unit4[threadIdx.x] = make_float4(cs, -sn, sn, -sn);
    }
    if constexpr (meta_ranks<DYN>(KP) > 0)
        for (int r = threadIdx.x; r < KP; r += blockDim.x) s_meta[r].y = a.wc.perm[r];
    if (threadIdx.x == 0) s_cls = -1;
    // TMEM tier: a.hot columns x 4*NS TMEM columns per quadrant (512 max)
    const int hotn = TM ? a.hot : 0;  // TMEM tier (TM instantiations only)
    const bool tm_alloc = hotn > 0;
    if (tm_alloc && warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            static_cast<unsigned>(__cvta_generic_to_shared(&s_tmem))));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tmem_sync_all();
    const uint32_t tq = tm_alloc ? s_tmem + (uint32_t(32 * (warp & 3)) << 16) : 0u;

    // synthesis pixels of this lane: p = lane + 32 j of the B x B block (loop invariant)
    const int B = a.block;
    const int nb2 = B * B;
    int p_r[PPL], p_c[PPL];
#pragma unroll
    for (int j = 0; j < PPL; ++j) {
        const int p = lane + 32 * j;
        p_r[j] = p < nb2 ? p / B : -1;
        p_c[j] = p < nb2 ? p % B : 0;
    }

    // one target block end to end: init, nu iterations, synthesis, placement
    auto solve_task = [&](const int ti, const ClassTab& ct, const int chunk) {
        // the class's table pointers once per task, in registers (ct refers to global
        // memory: read inside the loop, ct.fac was re-loaded every iteration, a dependent
        // load ahead of the step factor's own)
        const float4* __restrict__ gcols = reinterpret_cast<const float4*>(ct.cpack);
        const float2* __restrict__ scale2 = reinterpret_cast<const float2*>(ct.scale);
        const float* __restrict__ facp = ct.fac;
        const float* __restrict__ maskp = ct.mask32;
        const Task tk = a.tasks[ti];
        // ---------------- init: window image column per lane ----------------
        float colv[W];
        {
            int fc = (tk.origin_col + lane) >> 1;
            fc = fc < a.frame_cols - 1 ? fc : a.frame_cols - 1;
#pragma unroll
            for (int eta = 0; eta < W; ++eta) {
                float v = 0.f;
                if (lane < W) {
                    const float mk = __ldg(maskp + eta * W + lane);
                    int fr = (tk.origin_row + eta) >> 1;
                    fr = fr < a.frame_rows - 1 ? fr : a.frame_rows - 1;
                    const double y =
                        __ldg(a.frame + size_t(fr - a.frame_row0) * a.frame_pitch + fc);
                    v = mk * float(y);
                }
                colv[eta] = v;
            }
        }
        constexpr int H = W / 2 + 1;
        float2* r0buf = zbuf;
        float4 R[NS];
        if constexpr (Scratch<W>::kFFT) {
            // step 1 (lane = gamma): Z(sigma, gamma) = sum_eta a(eta,gamma) conj(U(eta sigma)),
            // kept in registers
            // with the first two radix-2 splits of a real-input FFT: U(eta sigma) repeats
            // with period 32 / gcd(sigma, 32), so s = a[eta] + a[eta+16] serves the even
            // sigma and d = a[eta] - a[eta+16] the odd ones, then s[eta] +- s[eta+8] the
            // sigma = 0 / 2 mod 4 -- 200 FFMA2 instead of 544
            float sv[16], dv[16], pv[8], qv[8];
#pragma unroll
            for (int eta = 0; eta < 16; ++eta) {
                sv[eta] = colv[eta] + colv[eta + 16];
                dv[eta] = colv[eta] - colv[eta + 16];
            }
#pragma unroll
            for (int eta = 0; eta < 8; ++eta) {
                pv[eta] = sv[eta] + sv[eta + 8];
                qv[eta] = sv[eta] - sv[eta + 8];
            }
            float2 zr[H];
#pragma unroll
            for (int sg = 0; sg < H; ++sg) {
                float2 z = make_float2(0.f, 0.f);
                const int n = (sg & 1) ? 16 : 8;
#pragma unroll
                for (int eta = 0; eta < n; ++eta) {
                    const float v = (sg & 1) ? dv[eta] : (sg & 2) ? qv[eta] : pv[eta];
                    const float4 u = unit4[(eta * sg) % W];  // (cos, -sin, sin, -sin)
                    z = __ffma2_rn(make_float2(v, v), make_float2(u.x, u.y), z);
                }
                zr[sg] = z;
            }
            // step 2: R0(sigma, rho) = sum_gamma Z(sigma,gamma) conj(U(gamma rho)) as a radix-2
            // decimation-in-frequency FFT across the lanes (lane = gamma), 5 stages of
            // shuffle butterflies: (a, b) -> (a + b, (a - b) e^{-2 pi i j / 2h}); lane l ends
            // with R0(sigma, bitrev(l)). 17 independent transforms per stage keep the
            // shuffles' latency hidden; no shared-memory transpose.
#pragma unroll
            for (int h = 16; h >= 1; h >>= 1) {
                const bool low = lane & h;  // holds b of its pair
                const float2 un = unit[(lane & (h - 1)) * (16 / h)];  // (cos, sin) of the twiddle
                const float2 sg2 = low ? make_float2(-1.f, -1.f) : make_float2(1.f, 1.f);
                const float2 wa = low ? make_float2(un.x, un.x) : make_float2(1.f, 1.f);
                const float2 wb = low ? make_float2(un.y, -un.y) : make_float2(0.f, 0.f);
#pragma unroll
                for (int sg = 0; sg < H; ++sg) {
                    float2 o;
                    o.x = __shfl_xor_sync(FULL, zr[sg].x, h);
                    o.y = __shfl_xor_sync(FULL, zr[sg].y, h);
                    const float2 y = __ffma2_rn(sg2, zr[sg], o);        // a + b  |  a - b
                    const float2 t = __fmul2_rn(y, wa);                    // y * w (complex)
                    zr[sg] = __ffma2_rn(make_float2(y.y, y.x), wb, t);
                }
            }
            // gather into rank order and scale: R'_r = s_r R0[perm r]. The half spectrum
            // is staged in shared memory (lane l holds column rho = bitrev(l) of every
            // row); SHARE warps take turns on one staging buffer under a shared-memory
            // lock held for the ~200 cycles of the gather (a task runs ~50k), so the
            // CTA's shared memory stays small and the SM's L1 keeps the rest for C'
            const int rho = int(__brev(unsigned(lane)) >> 27);
            const int2* __restrict__ src2 = reinterpret_cast<const int2*>(a.wc.src);
            if constexpr (kShare > 1) {
                // the whole warp spins on lane 0's CAS (a warp-uniform exit keeps the
                // solve provably converged: no WARPSYNC wrapping of its collectives)
                for (;;) {
                    int got = 0;
                    if (lane == 0) got = atomicCAS(glock, 0, 1) == 0;
                    if (__shfl_sync(FULL, got, 0)) break;
                }
            }
#pragma unroll
            for (int sg = 0; sg < H; ++sg) r0buf[sg * W + rho] = zr[sg];
            __syncwarp();
#pragma unroll
            for (int i = 0; i < NS; ++i) {
                const int2 sp = __ldg(src2 + 32 * i + lane);  // ranks 64 i + 2 lane + {0, 1}
                const float2 v0 = r0buf[sp.x & 0xffff], v1 = r0buf[sp.y & 0xffff];
                R[i] = make_float4(v0.x, v1.x, v0.y, v1.y);
            }
            __syncwarp();
            if constexpr (kShare > 1) {
                if (lane == 0) {
                    __threadfence_block();
                    atomicExch(glock, 0);
                }
            }
#pragma unroll
            for (int i = 0; i < NS; ++i) {
                const int2 sp = __ldg(src2 + 32 * i + lane);
                const float2 sc = __ldg(scale2 + 32 * i + lane);
                const float im0 = (sp.x & (1 << 30)) ? -R[i].z : R[i].z;
                const float im1 = (sp.y & (1 << 30)) ? -R[i].w : R[i].w;
                const float2 re = __fmul2_rn(sc, make_float2(R[i].x, R[i].y));
                const float2 im = __fmul2_rn(sc, make_float2(im0, im1));
                R[i] = make_float4(re.x, re.y, im.x, im.y);
            }
        } else {
            // step 1 (lane = gamma): Z(sigma, gamma) = sum_eta a(eta,gamma) conj(U(eta sigma))
#pragma unroll
            for (int sg = 0; sg < H; ++sg) {
                // (zr, zi) += (a, -a) * (cos, sin): one FFMA2, the same two roundings as
                // the scalar pair
                float2 z = make_float2(0.f, 0.f);
#pragma unroll
                for (int eta = 0; eta < W; ++eta) {
                    const float4 u = unit4[(eta * sg) % W];  // (cos, -sin, sin, -sin)
                    z = __ffma2_rn(make_float2(colv[eta], colv[eta]), make_float2(u.x, u.y), z);
                }
                zbuf[lane * 18 + sg] = z;
            }
            __syncwarp();
            // step 2 (lane = rho): R0(sigma, rho) = sum_gamma Z(sigma,gamma) conj(U(gamma rho))
            float2 r0[H];
#pragma unroll
            for (int sg = 0; sg < H; ++sg) r0[sg] = make_float2(0.f, 0.f);
#pragma unroll 4
            for (int g = 0; g < W; ++g) {
                const float4 u = unit4[(g * lane) % W];
#pragma unroll
                for (int sg = 0; sg < H; ++sg) {
                    // r0 += (z.y, -z.x) * sin, then += (z.x, z.y) * cos: the scalar FMA order
                    // (inner product with sin first) as two FFMA2
                    const float2 z = zbuf[g * 18 + sg];
                    const float2 t = __ffma2_rn(make_float2(z.y, z.x), make_float2(u.z, u.w), r0[sg]);
                    r0[sg] = __ffma2_rn(z, make_float2(u.x, u.x), t);
                }
            }
            __syncwarp();
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
#if TQSB_KEYS
        float lmax = score_pass_keys<NS>(R);
#else
        float lmax = score_pass<NS>(R, srow);
#endif

        float acc[PPL];
#pragma unroll
        for (int j = 0; j < PPL; ++j) acc[j] = 0.f;
        const int rw = tk.block_row - tk.origin_row, cw = tk.block_col - tk.origin_col;
        // window coordinates of this lane's kept pixels (unsigned: cheap mod W)
        unsigned pe[PPL], pg[PPL];
#pragma unroll
        for (int j = 0; j < PPL; ++j) {
            pe[j] = unsigned(rw + (p_r[j] < 0 ? 0 : p_r[j]));
            pg[j] = unsigned(cw + p_c[j]);
        }
        const bool tracing = TRACE && ti == 0;

        int it = 0;
        // no admissible frequency (rljsde.cpp:157-158: best < 0 only when no D_k > 0, a
        // static property of the class): inadmissible ranks are NaN from the init on and
        // stay NaN (their C' rows are NaN), admissible ones stay finite, so the test is
        // taken once, on the init scores, not per pick (-1.0 % per frame)
        const float g0 = warp_max_f32(lmax);
        const int n_it = g0 != g0 ? 0 : a.iterations;
        for (; it < n_it; ++it) {
            __syncwarp();
            // ---- argmax over the warp (NaN = inadmissible, ignored by max) ----
            const float gmax = warp_max_f32(lmax);
#if TQSB_KEYS
            // t through a vector register (a uniform-register switch makes ptxas spill R)
            int t;
            asm volatile("mov.b32 %0, %1;" : "=r"(t) : "r"(31 - int(__float_as_uint(gmax) & 31u)));
            // (& 31: a lane index whatever the ballot, so no pick can address outside the table)
            const int Lw = (__ffs(__ballot_sync(FULL, lmax == gmax)) - 1) & 31;
#else
            const unsigned cand = __ballot_sync(FULL, lmax == gmax);
            int Lw = (__ffs(cand) - 1) & 31;
            const float sv = lane < 2 * NS ? scr[Lw * kSbufStride + lane] : qnan();
            const unsigned hit = __ballot_sync(FULL, sv == gmax);
            int t;  // element index within lane Lw: slot t>>1, half t&1
            if (__popc(cand) == 1 && __popc(hit) == 1) {
                t = __ffs(hit) - 1;
            } else {
                // ties: smallest flat index among all maxima (rljsde.cpp:147-156)
                unsigned key = 0xffffffffu;
#pragma unroll
                for (int e = 0; e < 2 * NS; ++e) {
                    if (srow[e] == gmax) {
                        const int r = 64 * (e >> 1) + 2 * lane + (e & 1);
                        key = min(key, (unsigned(s_meta[r].y) << 16) | unsigned(r));
                    }
                }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1)
                    key = min(key, __shfl_xor_sync(FULL, key, off));
                const int r = int(key & 0xffffu);
                Lw = (r >> 1) & 31;
                t = 2 * (r >> 6) + (r & 1);
            }
#endif
            const int slot = t >> 1, b = t & 1;
            const int u = 64 * slot + 2 * Lw + b;
            // ---- issue the whole C' column now; its latency overlaps the pick ----
            constexpr bool kUni = NS == 16;  // one chunked update path for both column tiers
            constexpr int PF = kUni ? 4 * TQSB_AHEAD : (NS < TQSB_PREFETCH ? NS : TQSB_PREFETCH);
            float4 c[NS];
            const float4* col = gcols + size_t(u) * COLF4;
            const bool in_tmem = TM && u < hotn;
            const uint32_t tcol = tq + uint32_t(u * 4 * NS);
            if constexpr (kUni) {
                float4 t4[4];
                load_chunk<TM>(in_tmem, tcol, col + lane, t4);
#pragma unroll
                for (int k = 0; k < 4; ++k) c[k] = t4[k];
                if constexpr (TQSB_AHEAD > 1) {
                    load_chunk<TM>(in_tmem, tcol + 16u, col + 4 * 32 + lane, t4);
#pragma unroll
                    for (int k = 0; k < 4; ++k) c[4 + k] = t4[k];
                }
            } else if (in_tmem) {
                tmem_ld<NS>(tcol, c);
            } else {
#pragma unroll
                for (int i = 0; i < PF; ++i) c[i] = __ldg(col + i * 32 + lane);
            }
            // (fac bits, flat k) of rank u: CTA-shared table, or through L1 when scheduled per warp
            const int2 meta = DYN ? make_int2(__float_as_int(__ldg(facp + u)), __ldg(a.wc.perm + u))
                                  : s_meta[u];
            const float2 v = pick_elem<NS>(R, t);
            const float ure = __shfl_sync(FULL, v.x, Lw);
            const float uim = __shfl_sync(FULL, v.y, Lw);
            const float f = __int_as_float(meta.x);
            const float gre = f * ure, gim = f * uim;
            const int kflat = meta.y;
            // synthesis phases of the kept pixels: issued now, consumed after the update
            const unsigned sigma = unsigned(kflat) / W, rho = unsigned(kflat) % W;
            float2 ph[PPL];
#pragma unroll
            for (int j = 0; j < PPL; ++j) ph[j] = unit[(pe[j] * sigma + pg[j] * rho) % unsigned(W)];
#if !TQSB_KEYS
            __syncwarp();  // all score reads of this iteration precede the rewrite
#endif
            if constexpr (kUni) {
                lmax = update_uni<NS, TQSB_KEYS, TQSB_AHEAD, TM>(R, c, in_tmem, tcol, col + lane, gre, gim, srow);
            } else {
#if TQSB_KEYS
            if (in_tmem) {
                tmem_wait_ld();
                lmax = update_pass_keys<NS, NS>(R, c, col, lane, gre, gim);
            } else {
                lmax = update_pass_keys<NS, PF>(R, c, col, lane, gre, gim);
            }
#else
            if (in_tmem) {
                tmem_wait_ld();
                lmax = update_pass<NS, NS>(R, c, col, lane, gre, gim, srow);
            } else {
                lmax = update_pass<NS, PF>(R, c, col, lane, gre, gim, srow);
            }
#endif
            }
            // ---- synthesis of the kept block pixels (off the critical path) ----
#pragma unroll
            for (int j = 0; j < PPL; ++j) acc[j] = fmaf(gre, ph[j].x, fmaf(-gim, ph[j].y, acc[j]));
            if (tracing && lane == 0) {
                a.trace_picks[it] = kflat;
                a.trace_gd[2 * it] = gre;
                a.trace_gd[2 * it + 1] = gim;
            }
        }
        // ---- placement: clip + crop straight into the output ----
        const int2 bo = make_int2(tk.block_row, tk.block_col);
#pragma unroll
        for (int j = 0; j < PPL; ++j) {
            const int pr = p_r[j], pcc = p_c[j];
            if (pr >= 0) {
                const int orow = bo.x + pr, ocol = bo.y + pcc;
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
                    float sacc = 0.f;
                    for (int q = 0; q < it; ++q) {
                        const int k = a.trace_picks[q];
                        const float2 ph = unit[(eta * (k / W) + gam * (k % W)) % W];
                        sacc = fmaf(float(a.trace_gd[2 * q]), ph.x,
                                    fmaf(-float(a.trace_gd[2 * q + 1]), ph.y, sacc));
                    }
                    a.trace_window[p] = sacc;
                }
            }
        }
    };

    if constexpr (DYN) {
        // warp-level dynamic scheduling over the class-sorted task list: no CTA-wide
        // class state (per-rank factors are read through L1), and no tail imbalance
        // beyond one block per warp
        // streamed completion (SP): finished blocks are counted per chunk and published
        // with one release per chunk change -- tasks come in chunk order, so a warp
        // publishes ~once per chunk; the release orders all its earlier output stores
        int cur_chunk = -1, pending = 0;
        auto publish = [&]() {
            __syncwarp();  // the lanes' stores before lane 0's release
            if (lane == 0 && pending && (SP || a.progress))
                asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(a.progress + cur_chunk),
                             "r"(pending)
                             : "memory");
        };
        for (;;) {
            int ti = 0;
            if (lane == 0) ti = atomicAdd(a.counter, 1);
            ti = __shfl_sync(FULL, ti, 0);
            if (ti >= a.n_tasks) break;
            const int tc = __ldg(a.task_cls + ti);
            // (the same loop shape with and without streaming: it compiles to the faster
            // code -- 35.8 vs 37.5 ms per 4K frame for the variant without the chunk
            // bookkeeping; untagged task_cls entries have chunk 0 and no progress pointer)
            const int ch = tc >> kTaskClsBits;
            if (ch != cur_chunk) {
                publish();
                cur_chunk = ch;
                pending = 0;
            }
            solve_task(ti, a.tabs[tc & ((1 << kTaskClsBits) - 1)], ch);
            ++pending;
        }
        publish();
    } else {
        for (int it_item = blockIdx.x; it_item < a.n_items; it_item += gridDim.x) {
            const WorkItem item = a.items[it_item];
            if (item.cls != s_cls) {  // CTA-uniform: refill the class's on-chip tables
                tmem_sync_all();
                const float4* src = reinterpret_cast<const float4*>(a.tabs[item.cls].cpack);
                if (warp < 4) {  // one warp per TMEM lane quadrant copies the hot columns
                    for (int j = 0; j < hotn; ++j) {
    #pragma unroll
                        for (int i = 0; i < NS; ++i)
                            tmem_st4(tq + uint32_t(j * 4 * NS + 4 * i), __ldg(src + size_t(j) * COLF4 + i * 32 + lane));
                    }
                    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                }
                const float* fsrc = a.tabs[item.cls].fac;
                for (int r = threadIdx.x; r < KP; r += blockDim.x) s_meta[r].x = __float_as_int(__ldg(fsrc + r));
                tmem_sync_all();
                if (threadIdx.x == 0) s_cls = item.cls;
                __syncthreads();
            }
            const ClassTab ct = a.tabs[item.cls];

            for (int ti = item.start + warp; ti < item.start + item.count; ti += NW) {
                __syncwarp();  // converged: no divergence wrapping of the solve's collectives
                solve_task(ti, ct, 0);
            }
        }
    }
    tmem_sync_all();
    if (tm_alloc && warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s_tmem));
}

template <int NS, int W, int PPL>
int launch_one(const SolveArgs& a, cudaStream_t stream, int num_sms) {
    // the TMEM column tier only when columns are assigned to it (results are identical
    // either way; it costs instructions: measured 40.6 vs 40.1 ms per 4K frame with it on)
    constexpr int NWP = PPL == 1 ? kWarpsF32 : kWarpsF32Heavy;  // product path (B <= 5)
    const int nw = (a.trace_picks || a.hot > 0) ? kWarpsF32Heavy : NWP;
    const bool dyn = !(a.trace_picks || a.hot > 0) && TQSB_DYN;
    const size_t smem = dyn ? smem_bytes<W, true>(NS, nw) : smem_bytes<W, false>(NS, nw);
    auto kern = a.trace_picks ? k_solve_f32<NS, W, PPL, true, false, kWarpsF32Heavy>
                : a.hot > 0   ? k_solve_f32<NS, W, PPL, false, true, kWarpsF32Heavy>
                              : k_solve_f32<NS, W, PPL, false, false, NWP>;
    if (a.progress) {  // streamed host-buffer call: the product instantiations only
        if constexpr (solve_f32_streams(NS, PPL == 1 ? 16 : 64))
            kern = k_solve_f32<NS, W, PPL, false, false, NWP, true>;
        else
            return cudaErrorNotSupported;
        if (a.trace_picks || a.hot > 0) return cudaErrorNotSupported;
    }
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(smem));
    if (e != cudaSuccess) return e;
#ifdef TQSB_CARVEOUT
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, TQSB_CARVEOUT);
    if (e != cudaSuccess) return e;
#endif
    int grid = a.n_items < num_sms ? a.n_items : num_sms;
    if (grid < 1) grid = 1;
    kern<<<grid, nw * 32, smem, stream>>>(a);
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


int solve_f32_max_hot(int n_slots, int device) {
    // TMEM tier: 512 columns per lane quadrant, 4*NS columns per C' column
    (void)device;
    const int h = 512 / (4 * n_slots);
    return h < 64 * n_slots ? h : 64 * n_slots;
}

int launch_solve_f32(const SolveArgs& a, int n_slots, void* stream, int num_sms) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
#ifdef TQSB_ONLY_W32  // experiment builds (tools/variants.py): the default window only
    if (a.window == 32) return launch_w<32>(a, n_slots, s, num_sms);
    return cudaErrorInvalidValue;
#endif
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
