// common.cuh — device helpers shared by the pmap kernels (sm_100a).
// Product code: no dependency on oracle/ (the oracle is a separate C library
// written from the same paper; the two share no code).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/pmap.h"

#define PM_DEVINL __device__ __forceinline__

namespace pm {

constexpr int kWarp = 32;

// Depth validity (Q4 / S:69): > 0 and finite.  Positive finite floats are the
// bit patterns [0x00000001, 0x7F7FFFFF]; one unsigned compare covers 0, -0,
// negatives, inf and NaN.
PM_DEVINL bool valid_depth(float z) { return (__float_as_uint(z) - 1u) < 0x7F7FFFFFu; }

// exp2 on the MUFU unit (flush-to-zero; c_p underflows harmlessly to 0).
PM_DEVINL float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Philox4x32-10 (Salmon et al., SC'11), written for the device.  Counter
// {h, region, frame, 0}, key {lo32(seed), hi32(seed)} (north_star; Q17).
struct U4 { uint32_t x, y, z, w; };
PM_DEVINL U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int i = 0; i < 10; ++i) {
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

// Packed compacted point: (u | v << 16, z bits).
struct __align__(8) PackedPoint { uint32_t uv; float z; };

// Deprojection in the exact f32 order of DESIGN.md §3 (Alg. 2 ℓ3):
// X = (((float)u - cx) * ifx) * z.  Explicit _rn intrinsics: never contracted.
PM_DEVINL float3 deproject(PackedPoint p, float cx, float cy, float ifx, float ify) {
    const float u = (float)(p.uv & 0xFFFFu), v = (float)(p.uv >> 16);
    float3 P;
    P.x = __fmul_rn(__fmul_rn(__fsub_rn(u, cx), ifx), p.z);
    P.y = __fmul_rn(__fmul_rn(__fsub_rn(v, cy), ify), p.z);
    P.z = p.z;
    return P;
}

// Point-plane distance |n.p + d| as the explicit fused chain (Eq. 3 rho).
PM_DEVINL float plane_dist(float4 pl, float3 P) {
    return fabsf(__fmaf_rn(pl.z, P.z, __fmaf_rn(pl.y, P.y, __fmaf_rn(pl.x, P.x, pl.w))));
}

}  // namespace pm
