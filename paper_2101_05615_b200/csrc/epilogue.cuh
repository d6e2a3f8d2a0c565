// epilogue.cuh — the fused back-end on the TMEM -> register -> global drain,
// shared by the large-M GEMM kernels (gemm_tc.cu 1-CTA, gemm_tc2w.cu CTA
// pair): 16 accumulator columns of one output row per call.
//
// MODE 0: raw int32 (+ BiasAdd; WriteRawI32, pipeline.hpp:191-198)
// MODE 1: requantize F32_RNE; MODE 2: REF (quant.hpp:127-133)
// ReluQuantized folded into the clamp (pipeline.hpp:51-53, 176-190).
#pragma once
#include <stdint.h>

#include "q8g_internal.cuh"
#include "requant.cuh"

namespace q8g {

struct EpiArgs {
    const EpiRecord* rec;     // requant records (null for raw)
    int32_t zp_c;
    int relu;
    int fast;                 // q8g_epilogue::fast_f32
    const int32_t* bias_add;  // raw writer only
    void* c;
    int ldc;
    int n;                    // logical N
};

// d = {c[15:0], sat_u8(a), sat_u8(b)} (one I2IP)
__device__ __forceinline__ uint32_t pack_sat_u8(int32_t a, int32_t b, uint32_t c) {
    uint32_t d;
    asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// F32_RNE when fast: adj (wrapping int32), x = RN(float(adj) * m), floor at 0
// (ReLU) or -2^23, magic add y = x + 1.5*2^23 and the saturating pack of
// bits(y) - (0x4B400000 - zp_c) = clamp(rint(x) + zp_c, relu ? zp_c : 0, 255)
// exactly (bits(y) - 0x4B400000 = rint(x) for |x| <= 2^22 and monotone beyond;
// requires 0 <= zp_c <= 255 and finite multipliers: fast_f32)
__device__ __forceinline__ uint32_t requant4_f32_fast(const uint32_t* v, const int4* r4, uint32_t nrowsum,
                                                      int32_t zoff, float floor_x) {
    int32_t rr[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const int32_t adj = (int32_t)(v[b] + ((uint32_t)r4[b].x + (uint32_t)r4[b].y * nrowsum));
        float x = __fmul_rn(__int2float_rn(adj), __int_as_float(r4[b].z));
        x = fmaxf(x, floor_x);
        rr[b] = __float_as_int(__fadd_rn(x, 12582912.0f)) - zoff;
    }
    return pack_sat_u8(rr[1], rr[0], pack_sat_u8(rr[3], rr[2], 0u));
}

template <int MODE>
__device__ __forceinline__ void store_chunk16(const EpiArgs& p, int row, int col0, const uint32_t (&v)[16],
                                              int32_t rowsum) {
    if (MODE == 0) {
        int32_t* dst = reinterpret_cast<int32_t*>(p.c) + (size_t)row * p.ldc + col0;
        int32_t out[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            int32_t x = (int32_t)v[j];
            if (p.bias_add && col0 + j < p.n) x = (int32_t)((uint32_t)x + (uint32_t)__ldg(p.bias_add + col0 + j));
            out[j] = x;
        }
        const bool vec = (col0 + 16 <= p.n) && ((p.ldc & 3) == 0) && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0);
        if (vec) {
#pragma unroll
            for (int j = 0; j < 16; j += 4)
                *reinterpret_cast<int4*>(dst + j) = make_int4(out[j], out[j + 1], out[j + 2], out[j + 3]);
        } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (col0 + j < p.n) dst[j] = out[j];
        }
        return;
    }
    uint32_t packed[4];
    const int4* recs = reinterpret_cast<const int4*>(p.rec + col0);
    if (MODE == 1 && p.fast) {
        const int32_t zoff = 0x4B400000 - p.zp_c;
        const float floor_x = p.relu ? 0.0f : -8388608.0f;
        const uint32_t nrowsum = 0u - (uint32_t)rowsum;  // adj = v + c + zp_b * (-rowsum)
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            int4 r4[4];
#pragma unroll
            for (int b = 0; b < 4; ++b) r4[b] = __ldg(recs + w * 4 + b);
            packed[w] = requant4_f32_fast(v + w * 4, r4, nrowsum, zoff, floor_x);
        }
    } else {
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            uint32_t word = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int j = w * 4 + b;
                const int4 r4 = __ldg(recs + j);
                EpiRecord rc;
                rc.c = r4.x;
                rc.zpb = r4.y;
                const int32_t adj = adjust((int32_t)v[j], rowsum, rc);
                const uint32_t q = MODE == 1 ? requant_f32(adj, __int_as_float(r4.z), p.zp_c, p.relu)
                                             : requant_ref(adj, __hiloint2double(r4.w, r4.z), p.zp_c, p.relu);
                word |= q << (8 * b);
            }
            packed[w] = word;
        }
    }
    uint8_t* dst = reinterpret_cast<uint8_t*>(p.c) + (size_t)row * p.ldc + col0;
    const bool vec = (col0 + 16 <= p.n) && ((p.ldc & 15) == 0) && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0);
    if (vec) {
        *reinterpret_cast<uint4*>(dst) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
    } else {
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if (col0 + j < p.n) dst[j] = (uint8_t)(packed[j / 4] >> (8 * (j % 4)));
    }
}

}  // namespace q8g
