// requant.cuh — the fused back-end, device side.
//
// Restates quant.hpp:115-133 (requantize_adjust / requantize_scalar) and
// pipeline.hpp:51-53,176-190 (ReluQuantized folded into Requantize) with the
// per-column constants folded at epilogue-create time:
//   adj = acc - zp_b[j]*rowsum[i] + c[j]
//       c[j] = bias[j] - zp_a*colsum[j] + K*zp_a*zp_b[j]
// All int32 arithmetic wraps mod 2^32.  The reference computes `adj` in
// int64; whenever the true |adj| < 2^31 the wrapped int32 value equals it,
// and q8g_epilogue_create rejects parameters for which some column's bound
// K*max|A - zp_a|*(max|B| + |zp_b|) + |(k_total - K) zp_a zp_b| + |bias|
// reaches 2^31 (abi.cu).
#pragma once

#include <stdint.h>

#include "q8g_internal.cuh"

namespace q8g {

__device__ __forceinline__ int32_t adjust(int32_t acc, int32_t rowsum, const EpiRecord& r) {
    // unsigned arithmetic: defined wrap-around
    return (int32_t)((uint32_t)acc - (uint32_t)r.zpb * (uint32_t)rowsum + (uint32_t)r.c);
}

__device__ __forceinline__ int32_t sat_add(int32_t a, int32_t b) {
    int32_t d;
    asm("add.sat.s32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}

// ReluQuantized after the [0,255] clamp: q < zp_c ? (uint8)zp_c : q
__device__ __forceinline__ uint32_t finish_u8(int32_t q, int32_t zp_c, bool relu) {
    q = q < 0 ? 0 : (q > 255 ? 255 : q);
    if (relu && q < zp_c) q = zp_c & 255;
    return (uint32_t)q;
}

// F32_RNE: one RN int->fp32 conversion, one RN fp32
// multiply (no FMA contraction possible: __fmul_rn), cvt.rni (ties to even,
// saturating), saturating + zp_c, clamp.
__device__ __forceinline__ uint32_t requant_f32(int32_t adj, float mult, int32_t zp_c, bool relu) {
    const float x = __fmul_rn(__int2float_rn(adj), mult);
    const int32_t r = __float2int_rn(x);
    return finish_u8(sat_add(r, zp_c), zp_c, relu);
}

// REF (quant.hpp:127-133): double(adj) exact, one RN fp64 multiply,
// llround (round half away from zero, quant.hpp:45-47), + zp_c, clamp.
__device__ __forceinline__ uint32_t requant_ref(int32_t adj, double mult, int32_t zp_c, bool relu) {
    const double x = __dmul_rn(mult, (double)adj);
    const double t = trunc(x);
    const double frac = x - t;  // exact: |x - trunc(x)| < 1 and same binade
    double r = t;
    if (fabs(frac) >= 0.5) r += (x < 0.0 ? -1.0 : 1.0);
    // saturate to int32; with |zp_c| <= 2^30 (host-validated) the saturating
    // add below then clamps exactly like the reference's long long sum
    r = fmin(fmax(r, -2147483648.0), 2147483647.0);
    return finish_u8(sat_add((int32_t)r, zp_c), zp_c, relu);
}

}  // namespace q8g
