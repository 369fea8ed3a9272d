// solve_common.cuh -- device helpers shared by the fp32 solve kernels
// (solve_f32.cu): selection keys, the register pick, score and update passes,
// chunked column loads (global or TMEM) and the TMEM helpers.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "tqsb_internal.hpp"

namespace tqsb {
namespace dev {

constexpr unsigned FULL = 0xffffffffu;

#ifndef TQSB_PREFETCH
#define TQSB_PREFETCH 16  // C' slots in flight ahead of the update (register budget)
#endif

__device__ __forceinline__ float qnan() { return __int_as_float(0x7fc00000); }

// STS.64 straight from an FFMA2 register pair (inline PTX keeps ptxas from fusing
// neighbouring stores into an STS.128 that needs register copies to pack)
__device__ __forceinline__ void st_shared_f2(float* p, float2 v) {
    asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(
                     static_cast<unsigned>(__cvta_generic_to_shared(p))),
                 "f"(v.x), "f"(v.y)
                 : "memory");
}

// warp-wide max in one CREDUX (redux.sync .f32, sm_100a); NaN inputs are ignored,
// so the result is NaN only when every lane holds NaN (no admissible frequency)
__device__ __forceinline__ float warp_max_f32(float x) {
    float m;
    asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(m) : "f"(x));
    return m;
}

__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

// (re, im) of element t (slot t>>1, half t&1) of this lane's residual; t is
// warp-uniform, so the switch is a uniform branch, not a local-memory array.
template <int NS>
__device__ __forceinline__ float2 pick_elem(const float4 (&R)[NS], int t) {
    float re = 0.f, im = 0.f;
    switch (t) {
#define TQSB_CASE(n)                                                            \
    case n:                                                                     \
        if ((n >> 1) < NS) {                                                    \
            re = (n & 1) ? R[(n >> 1) < NS ? (n >> 1) : 0].y : R[(n >> 1) < NS ? (n >> 1) : 0].x; \
            im = (n & 1) ? R[(n >> 1) < NS ? (n >> 1) : 0].w : R[(n >> 1) < NS ? (n >> 1) : 0].z; \
        }                                                                       \
        break;
        TQSB_CASE(0) TQSB_CASE(1) TQSB_CASE(2) TQSB_CASE(3) TQSB_CASE(4) TQSB_CASE(5)
        TQSB_CASE(6) TQSB_CASE(7) TQSB_CASE(8) TQSB_CASE(9) TQSB_CASE(10) TQSB_CASE(11)
        TQSB_CASE(12) TQSB_CASE(13) TQSB_CASE(14) TQSB_CASE(15) TQSB_CASE(16) TQSB_CASE(17)
        TQSB_CASE(18) TQSB_CASE(19) TQSB_CASE(20) TQSB_CASE(21) TQSB_CASE(22) TQSB_CASE(23)
        TQSB_CASE(24) TQSB_CASE(25) TQSB_CASE(26) TQSB_CASE(27) TQSB_CASE(28) TQSB_CASE(29)
        TQSB_CASE(30) TQSB_CASE(31)
#undef TQSB_CASE
        default: break;
    }
    return make_float2(re, im);
}

// Scores |R'|^2 of every element go to this lane's row of the score buffer (one
// STS.64 per slot, straight from the FFMA2 register pair) and into the lane maximum (FMNMX3;
// NaN marks an inadmissible frequency and is ignored by max).
template <int NS>
__device__ __forceinline__ float score_pass(const float4 (&R)[NS], float* srow) {
    float m4[4] = {qnan(), qnan(), qnan(), qnan()};  // 4 short FMNMX3 chains
#pragma unroll
    for (int i = 0; i < NS; ++i) {
        const float2 re = make_float2(R[i].x, R[i].y), im = make_float2(R[i].z, R[i].w);
        const float2 sc = __ffma2_rn(im, im, __fmul2_rn(re, re));
        m4[i & 3] = fmax3(m4[i & 3], sc.x, sc.y);
        st_shared_f2(srow + 2 * i, sc);
    }
    return fmax3(fmax3(m4[0], m4[1], m4[2]), m4[3], qnan());
}

// Packed selection key (TQSB_KEYS): the score's top 27 bits with the element's
// position t = 2*slot + half stored as 31 - t in the low 5 mantissa bits, so one
// FMNMX3/CREDUX max yields both the maximum and (with a lane ballot) its position.
// Scores that differ by less than 2^-18 relative compare by position instead.
// one LOP3 per element: (bits & mask) | (31 - t) with the mask held in a register
// (keymask(), opaque to constant folding) and 31 - t as the instruction immediate
__device__ __forceinline__ unsigned keymask() {
    unsigned m;
    asm volatile("mov.b32 %0, 0xffffffe0;" : "=r"(m));
    return m;
}
__device__ __forceinline__ float score_key(float s, int t, unsigned mask) {
    unsigned d;
    asm("lop3.b32 %0, %1, %2, %3, 0xEC;" : "=r"(d) : "r"(__float_as_uint(s)), "r"(unsigned(31 - t)), "r"(mask));
    return __uint_as_float(d);
}

template <int NS>
__device__ __forceinline__ float score_pass_keys(const float4 (&R)[NS]) {
    float m4[4] = {qnan(), qnan(), qnan(), qnan()};
    const unsigned kmask = keymask();
#pragma unroll
    for (int i = 0; i < NS; ++i) {
        const float2 re = make_float2(R[i].x, R[i].y), im = make_float2(R[i].z, R[i].w);
        const float2 sc = __ffma2_rn(im, im, __fmul2_rn(re, re));
        m4[i & 3] = fmax3(m4[i & 3], score_key(sc.x, 2 * i, kmask), score_key(sc.y, 2 * i + 1, kmask));
    }
    return fmax3(fmax3(m4[0], m4[1], m4[2]), m4[3], qnan());
}

template <int NS, int PF>
__device__ __forceinline__ float update_pass_keys(float4 (&R)[NS], float4 (&c)[NS],
                                                  const float4* __restrict__ col, int lane,
                                                  float gre, float gim) {
    const float2 ngre = make_float2(-gre, -gre);
    const float2 pgim = make_float2(gim, gim);
    const float2 ngim = make_float2(-gim, -gim);
    float m4[4] = {qnan(), qnan(), qnan(), qnan()};
    const unsigned kmask = keymask();
#pragma unroll
    for (int i = 0; i < NS; ++i) {
        if (i + PF < NS) c[i + PF] = col[(i + PF) * 32 + lane];
        const float2 cre = make_float2(c[i].x, c[i].y), cim = make_float2(c[i].z, c[i].w);
        float2 re = make_float2(R[i].x, R[i].y), im = make_float2(R[i].z, R[i].w);
        re = __ffma2_rn(ngre, cre, re);
        re = __ffma2_rn(pgim, cim, re);
        im = __ffma2_rn(ngre, cim, im);
        im = __ffma2_rn(ngim, cre, im);
        R[i] = make_float4(re.x, re.y, im.x, im.y);
        const float2 sc = __ffma2_rn(im, im, __fmul2_rn(re, re));
        m4[i & 3] = fmax3(m4[i & 3], score_key(sc.x, 2 * i, kmask), score_key(sc.y, 2 * i + 1, kmask));
    }
    return fmax3(fmax3(m4[0], m4[1], m4[2]), m4[3], qnan());
}

// R' -= g C'[:,u] for every slot (4 FFMA2 per rank pair) from the prefetched
// column c[], fused with the next scores.
// PF slots of the column were issued before the pick (c[0..PF-1]); the rest stream
// in a sliding window PF slots ahead of the update.
template <int NS, int PF>
__device__ __forceinline__ float update_pass(float4 (&R)[NS], float4 (&c)[NS],
                                             const float4* __restrict__ col, int lane, float gre,
                                             float gim, float* srow) {
    const float2 ngre = make_float2(-gre, -gre);
    const float2 pgim = make_float2(gim, gim);
    const float2 ngim = make_float2(-gim, -gim);
    float m4[4] = {qnan(), qnan(), qnan(), qnan()};  // 4 short FMNMX3 chains
#pragma unroll
    for (int i = 0; i < NS; ++i) {
        if (i + PF < NS) c[i + PF] = col[(i + PF) * 32 + lane];
        const float2 cre = make_float2(c[i].x, c[i].y), cim = make_float2(c[i].z, c[i].w);
        float2 re = make_float2(R[i].x, R[i].y), im = make_float2(R[i].z, R[i].w);
        re = __ffma2_rn(ngre, cre, re);
        re = __ffma2_rn(pgim, cim, re);
        im = __ffma2_rn(ngre, cim, im);
        im = __ffma2_rn(ngim, cre, im);
        R[i] = make_float4(re.x, re.y, im.x, im.y);
        const float2 sc = __ffma2_rn(im, im, __fmul2_rn(re, re));
        m4[i & 3] = fmax3(m4[i & 3], sc.x, sc.y);
        st_shared_f2(srow + 2 * i, sc);
    }
    return fmax3(fmax3(m4[0], m4[1], m4[2]), m4[3], qnan());
}

// ---------------------------------------------------------------------------
// Tensor memory as the hot-column tier. TMEM is 512 columns x 128 lanes x 32 bit
// per SM and a warp reaches only its lane quadrant (lanes 32*(warp%4)..+31), so
// each quadrant holds its own copy of the class's lowest-rank C' columns: lane j
// of a quadrant keeps the 4*NS floats that lane j of a warp would load for that
// column (the same float4 layout as global memory). Reads are tcgen05.ld
// (LDTM), which bypasses the L1/shared-memory data path that the rest of the
// loop saturates (measured on B200: ~450 B/clk/SM vs 128 for LDS.128).
// ---------------------------------------------------------------------------
template <int NS> struct TmemShape;  // 32x32b.x(4*NS): 4*NS consecutive columns per lane
#define TQSB_TM_REGS16(P) P(0) P(1) P(2) P(3)
template <int NS>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, float4 (&c)[NS]) {
    uint32_t r[4 * NS];
    if constexpr (NS == 16) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x64.b32 {"
            "%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"
            "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,"
            "%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
              "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
              "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
              "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
              "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
              "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]),
              "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]),
              "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]),
              "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]),
              "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]),
              "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
            : "r"(taddr));
    } else if constexpr (NS == 8) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {"
            "%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
              "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
              "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
              "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
              "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
              "=r"(r[31])
            : "r"(taddr));
    } else if constexpr (NS == 4) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {"
            "%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
              "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
              "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr));
    } else if constexpr (NS == 2) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                       "=r"(r[6]), "=r"(r[7])
                     : "r"(taddr));
    } else {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                     : "r"(taddr));
    }
#pragma unroll
    for (int i = 0; i < NS; ++i)
        c[i] = make_float4(__uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1]),
                           __uint_as_float(r[4 * i + 2]), __uint_as_float(r[4 * i + 3]));
}

// Four column slots (16 floats per lane) into d[] from TMEM (tm) or global memory
// (g = column + slot0 * 32 + lane): one code path for both tiers, so the residual
// registers keep a single allocation. The tcgen05.ld is predicated on a warp-uniform
// flag; a following tcgen05.wait::ld (unconditional) completes it.
template <bool TM>
__device__ __forceinline__ void load_chunk(bool tm, uint32_t taddr, const float4* g, float4 (&d)[4]) {
    if constexpr (!TM) {  // no TMEM tier: four coalesced 512 B global reads
        (void)tm;
        (void)taddr;
#pragma unroll
        for (int k = 0; k < 4; ++k) d[k] = __ldg(g + 32 * k);
        return;
    }
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %18, 0;\n\t"
        "@p tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n\t"
        "@!p ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%17];\n\t"
        "@!p ld.global.nc.v4.f32 {%4,%5,%6,%7}, [%17+512];\n\t"
        "@!p ld.global.nc.v4.f32 {%8,%9,%10,%11}, [%17+1024];\n\t"
        "@!p ld.global.nc.v4.f32 {%12,%13,%14,%15}, [%17+1536];\n\t}"
        : "=f"(d[0].x), "=f"(d[0].y), "=f"(d[0].z), "=f"(d[0].w), "=f"(d[1].x), "=f"(d[1].y),
          "=f"(d[1].z), "=f"(d[1].w), "=f"(d[2].x), "=f"(d[2].y), "=f"(d[2].z), "=f"(d[2].w),
          "=f"(d[3].x), "=f"(d[3].y), "=f"(d[3].z), "=f"(d[3].w)
        : "r"(taddr), "l"(g), "r"(int(tm))
        : "memory");
}

// One update path for both tiers (NS == 16): chunks 0 and 1 (slots 0-7) were issued
// before the pick; chunk k+2 is issued at the start of chunk k, after the wait::ld
// that completes chunk k+1.
template <int NS, bool KEYS, int AHEAD, bool TM>
__device__ __forceinline__ float update_uni(float4 (&R)[NS], float4 (&c)[NS], bool tm,
                                            uint32_t taddr, const float4* __restrict__ gl,
                                            float gre, float gim, float* srow) {
    static_assert(NS == 16, "update_uni streams four 4-slot chunks");
    const float2 ngre = make_float2(-gre, -gre);
    const float2 pgim = make_float2(gim, gim);
    const float2 ngim = make_float2(-gim, -gim);
    float m4[4] = {qnan(), qnan(), qnan(), qnan()};
    [[maybe_unused]] const unsigned kmask = keymask();
#pragma unroll
    for (int i = 0; i < NS; ++i) {
        if (i % 4 == 0) {
            if constexpr (TM) asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            constexpr int A = 4 * AHEAD;  // slots issued ahead of the update
            if (i + A < NS) {
                float4 t4[4];
                load_chunk<TM>(tm, taddr + uint32_t(4 * (i + A)), gl + (i + A) * 32, t4);
#pragma unroll
                for (int k = 0; k < 4; ++k) c[i + A + k] = t4[k];
            }
        }
        const float2 cre = make_float2(c[i].x, c[i].y), cim = make_float2(c[i].z, c[i].w);
        float2 re = make_float2(R[i].x, R[i].y), im = make_float2(R[i].z, R[i].w);
        re = __ffma2_rn(ngre, cre, re);
        re = __ffma2_rn(pgim, cim, re);
        im = __ffma2_rn(ngre, cim, im);
        im = __ffma2_rn(ngim, cre, im);
        R[i] = make_float4(re.x, re.y, im.x, im.y);
        const float2 sc = __ffma2_rn(im, im, __fmul2_rn(re, re));
        if constexpr (KEYS) {
            if (i == NS - 1)  // the last slot's keys enter at the final level: one FMNMX3
                              // less between the last update and the warp max (the max of
                              // the same set, NaN-ignoring: bitwise the same key)
                return fmax3(fmax3(fmax3(m4[0], m4[1], m4[2]), m4[3], qnan()),
                             score_key(sc.x, 2 * i, kmask), score_key(sc.y, 2 * i + 1, kmask));
            m4[i & 3] = fmax3(m4[i & 3], score_key(sc.x, 2 * i, kmask), score_key(sc.y, 2 * i + 1, kmask));
        } else {
            m4[i & 3] = fmax3(m4[i & 3], sc.x, sc.y);
            st_shared_f2(srow + 2 * i, sc);
        }
    }
    return fmax3(fmax3(m4[0], m4[1], m4[2]), m4[3], qnan());
}

// the whole residual (16 float4 per lane) into 64 consecutive TMEM columns of this
// warp's lane quadrant: 32x32b.x64, asynchronous (tcgen05.wait::st before reading back)
__device__ __forceinline__ void tmem_st64(uint32_t taddr, const float4 (&R)[16]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x64.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63,%64};"
                 :: "r"(taddr), "r"(__float_as_uint(R[0].x)), "r"(__float_as_uint(R[0].y)), "r"(__float_as_uint(R[0].z)), "r"(__float_as_uint(R[0].w)), "r"(__float_as_uint(R[1].x)), "r"(__float_as_uint(R[1].y)), "r"(__float_as_uint(R[1].z)), "r"(__float_as_uint(R[1].w)), "r"(__float_as_uint(R[2].x)), "r"(__float_as_uint(R[2].y)), "r"(__float_as_uint(R[2].z)), "r"(__float_as_uint(R[2].w)), "r"(__float_as_uint(R[3].x)), "r"(__float_as_uint(R[3].y)), "r"(__float_as_uint(R[3].z)), "r"(__float_as_uint(R[3].w)), "r"(__float_as_uint(R[4].x)), "r"(__float_as_uint(R[4].y)), "r"(__float_as_uint(R[4].z)), "r"(__float_as_uint(R[4].w)), "r"(__float_as_uint(R[5].x)), "r"(__float_as_uint(R[5].y)), "r"(__float_as_uint(R[5].z)), "r"(__float_as_uint(R[5].w)), "r"(__float_as_uint(R[6].x)), "r"(__float_as_uint(R[6].y)), "r"(__float_as_uint(R[6].z)), "r"(__float_as_uint(R[6].w)), "r"(__float_as_uint(R[7].x)), "r"(__float_as_uint(R[7].y)), "r"(__float_as_uint(R[7].z)), "r"(__float_as_uint(R[7].w)), "r"(__float_as_uint(R[8].x)), "r"(__float_as_uint(R[8].y)), "r"(__float_as_uint(R[8].z)), "r"(__float_as_uint(R[8].w)), "r"(__float_as_uint(R[9].x)), "r"(__float_as_uint(R[9].y)), "r"(__float_as_uint(R[9].z)), "r"(__float_as_uint(R[9].w)), "r"(__float_as_uint(R[10].x)), "r"(__float_as_uint(R[10].y)), "r"(__float_as_uint(R[10].z)), "r"(__float_as_uint(R[10].w)), "r"(__float_as_uint(R[11].x)), "r"(__float_as_uint(R[11].y)), "r"(__float_as_uint(R[11].z)), "r"(__float_as_uint(R[11].w)), "r"(__float_as_uint(R[12].x)), "r"(__float_as_uint(R[12].y)), "r"(__float_as_uint(R[12].z)), "r"(__float_as_uint(R[12].w)), "r"(__float_as_uint(R[13].x)), "r"(__float_as_uint(R[13].y)), "r"(__float_as_uint(R[13].z)), "r"(__float_as_uint(R[13].w)), "r"(__float_as_uint(R[14].x)), "r"(__float_as_uint(R[14].y)), "r"(__float_as_uint(R[14].z)), "r"(__float_as_uint(R[14].w)), "r"(__float_as_uint(R[15].x)), "r"(__float_as_uint(R[15].y)), "r"(__float_as_uint(R[15].z)), "r"(__float_as_uint(R[15].w))
                 : "memory");
}

// one slot (4 floats: re_a, re_b, im_a, im_b) of the residual shadow back
__device__ __forceinline__ float4 tmem_ld_slot(uint32_t taddr) {
    uint32_t r0, r1, r2, r3;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(taddr));
    return make_float4(__uint_as_float(r0), __uint_as_float(r1), __uint_as_float(r2), __uint_as_float(r3));
}

__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// store 4 columns (one float4) per call: 32x32b.x4
__device__ __forceinline__ void tmem_st4(uint32_t taddr, float4 v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr),
                 "r"(__float_as_uint(v.x)), "r"(__float_as_uint(v.y)), "r"(__float_as_uint(v.z)),
                 "r"(__float_as_uint(v.w))
                 : "memory");
}

__device__ __forceinline__ void tmem_sync_all() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}


}  // namespace dev
}  // namespace tqsb
