// common.cuh — device helpers shared by the pmap kernels (sm_100a).
// Product code: no dependency on oracle/ (the oracle is a separate C library
// written from the same paper; the two share no code).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/pmap.h"

#define PM_DEVINL __device__ __forceinline__

// Checked build (compute-sanitizer substitute, tools/checked_run.sh): device
// bounds checks on the shared- and global-memory indices of the hot kernels;
// a failed check traps (the launch then fails with an illegal-instruction
// error).  Empty in the product build.
#ifdef PM_CHECKED
#define PM_CHECK(cond)               \
    do {                             \
        if (!(cond)) __trap();       \
    } while (0)
#else
#define PM_CHECK(cond) \
    do {               \
    } while (0)
#endif

namespace pm {

constexpr int kWarp = 32;

// Depth validity (Q4 / S:69): > 0 and finite.  Positive finite floats are the
// bit patterns [0x00000001, 0x7F7FFFFF]; one unsigned compare covers 0, -0,
// negatives, inf and NaN.
// ---- packed fp32 pairs (sm_100a FADD2 / FMUL2 / FFMA2: two fp32 lanes per
// instruction, the FP32-pipe work of two scalar ops in one issue slot).
// Packed fp32 ops as inline PTX (the __fmul2_rn/__fadd2_rn intrinsics get
// contracted into FFMA2 even under --fmad=false: measured, the divergence
// scheme lost bitwise equality with the scalar path).
PM_DEVINL uint64_t f2pk(float2 a) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
    return r;
}
PM_DEVINL float2 f2up(uint64_t r) {
    float2 a;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
    return a;
}
PM_DEVINL float2 f2add(float2 a, float2 b) {
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2pk(a)), "l"(f2pk(b)));
    return f2up(r);
}
PM_DEVINL float2 f2sub(float2 a, float2 b) {
    uint64_t r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2pk(a)), "l"(f2pk(b)));
    return f2up(r);
}
PM_DEVINL float2 f2mul(float2 a, float2 b) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2pk(a)), "l"(f2pk(b)));
    return f2up(r);
}
PM_DEVINL float2 f2fma(float2 a, float2 b, float2 c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2pk(a)), "l"(f2pk(b)), "l"(f2pk(c)));
    return f2up(r);
}
PM_DEVINL float2 f2s(float a) { return make_float2(a, a); }

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
// Exact u16 -> f32 without the XU pipe: 2^23 + k has k in its low mantissa bits.
PM_DEVINL float u16_to_f32(uint32_t k) { return __fsub_rn(__uint_as_float(0x4B000000u | k), 8388608.0f); }

PM_DEVINL float3 deproject(PackedPoint p, float cx, float cy, float ifx, float ify) {
    const float u = u16_to_f32(p.uv & 0xFFFFu), v = u16_to_f32(p.uv >> 16);
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

// ---------------------------------------------------------------------------
// TMA (cp.async.bulk.tensor) + mbarrier helpers, sm_90+/sm_100a.
#include <cuda.h>

namespace pm {

PM_DEVINL uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

PM_DEVINL void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// Order this CTA's earlier generic-proxy shared-memory accesses (made visible
// to the issuing thread by a barrier) before a following async-proxy (TMA) write.
PM_DEVINL void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

PM_DEVINL void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

PM_DEVINL void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// Bulk copy shared -> global (cp.async.bulk, bulk-group completion): 16-B
// aligned addresses, size a multiple of 16.  Pair with bulk_commit() and
// bulk_wait_read() (the source may be overwritten / the CTA exit after it).
PM_DEVINL void bulk_store_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"((uint64_t)dst),
                 "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
}
PM_DEVINL void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
PM_DEVINL void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }

// 3-D tile load global -> shared, completion signalled on `bar` (tx bytes).
PM_DEVINL void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"((uint64_t)map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

// Host: encode a 3-D fp32 tensor map over [B][H][W] with a boxW x boxH x 1
// box (zero fill out of bounds).  Returns false when TMA cannot describe the
// buffer (row stride not a multiple of 16 B, misaligned base, entry point
// unavailable) -- callers then use the LDG path.
bool make_tmap_f32_3d(CUtensorMap* map, const void* base, int W, int H, int B, int boxW, int boxH);

}  // namespace pm
