// adf_cell.cuh — the per-cell arithmetic of Alg. 1 shared by
// the two ADF engines (adf.cu: shared-memory tiles; adf_reg.cu: register
// tiles), so that both evaluate the identical _rn expression on identical
// operands (bitwise invariance).
#pragma once
#include <float.h>
#include <stdint.h>

#include <type_traits>

#include "common.cuh"

namespace pm {
namespace adfk {

struct AdfParams {
    float kc;         // -log2(e) / (4 kappa^2)
    float l2lam;      // log2(lambda): lambda * c = 2^(kc * g2 + log2(lambda))
    float kd;         // -log2(e) / kappa^2 (divergence scheme: c(d) = 2^(kd d^2))
    float lam;
    float negz;       // -0.0f (run-time operand, see f2mul_nf)
    float fx, fy, cx, cy;
    float ifx, ify;   // 1/fx, 1/fy (Eq. 2 as printed)
    int scheme;       // PM_ADF_ALG1 | PM_ADF_DIVERGENCE
    int nmode;        // PM_NORMALS_GEOMETRIC | PM_NORMALS_AS_PRINTED
    int keep_valid;   // lambda > kNoCheckMaxLambda: floor valid updates at the
                      // smallest positive float (see keep_valid() below)
    unsigned* hole_note;   // mapped host word: the first pass stores call_id on a tile with
    unsigned call_id;      // an invalid pixel (AUTO engine choice, adf.cu), or null
};

// Q4 fixes validity from the INPUT of the filter.  For lambda <= 0.249 no
// valid pixel can filter to a value <= 0 (adf.cu fast_depth); above, a pixel
// next to much smaller neighbours can round to 0 (or, through the ex2
// approximation, slightly below) and would read as invalid in the next
// pass.  The hole-aware paths therefore floor a valid pixel's update at
// 2^-149 when keep_valid is set, so validity is carried across passes.
constexpr float kTinyPos = 1.40129846e-45f;   // 2^-149, bits 0x00000001
PM_DEVINL float keep_valid(float o, int on) { return on ? fmaxf(o, kTinyPos) : o; }

// Alg. 1 ℓ4-6 at a valid centre C with neighbour values N, S, W, E (already
// replaced by C where the zero-flux rule applies):
//   2gx = E - W;  2gy = S - N;  lap = ((N + S) + (W + E)) - 4 C
//   lambda * c = 2^(kc (2gx^2 + 2gy^2) + log2 lambda),  c = exp(-|grad|^2 / k^2)
//   I' = C + (lambda c) * lap
// (pairwise sums keep a constant image an exact fixed point; the f32
// rounding of the sums costs < 1e-6 m over 100 sweeps)
PM_DEVINL float adf_cell(float C, float N, float S, float W, float E, float kc, float l2lam) {
    const float gx2 = __fsub_rn(E, W);
    const float gy2 = __fsub_rn(S, N);
    const float g2 = __fmaf_rn(gx2, gx2, __fmul_rn(gy2, gy2));
    const float lc = ex2_approx(__fmaf_rn(g2, kc, l2lam));
    const float lap = __fmaf_rn(-4.0f, C, __fadd_rn(__fadd_rn(N, S), __fadd_rn(W, E)));
    return __fmaf_rn(lc, lap, C);
}

// Eq. 1 as the 4-flux Perona-Malik scheme (NEXT-1, reading Q1):
//   I' = C + lambda * ((c(dN) dN + c(dS) dS) + (c(dW) dW + c(dE) dE)),
//   dX = X - C, c(d) = exp(-(d / k)^2) = 2^(kd d^2)
PM_DEVINL float adf_cell_div(float C, float N, float S, float W, float E, float kd, float lam) {
    const float dn = __fsub_rn(N, C), ds = __fsub_rn(S, C);
    const float dw = __fsub_rn(W, C), de = __fsub_rn(E, C);
    const float fn = __fmul_rn(ex2_approx(__fmul_rn(__fmul_rn(dn, dn), kd)), dn);
    const float fs = __fmul_rn(ex2_approx(__fmul_rn(__fmul_rn(ds, ds), kd)), ds);
    const float fw = __fmul_rn(ex2_approx(__fmul_rn(__fmul_rn(dw, dw), kd)), dw);
    const float fe = __fmul_rn(ex2_approx(__fmul_rn(__fmul_rn(de, de), kd)), de);
    return __fmaf_rn(lam, __fadd_rn(__fadd_rn(fn, fs), __fadd_rn(fw, fe)), C);
}

template <bool CHECK, bool DIV>
PM_DEVINL float cell(float C, float N, float S, float W, float E, const AdfParams& p) {
    if (CHECK) {
        if (!valid_depth(C)) return C;                 // invalid pixels never change
        N = valid_depth(N) ? N : C;
        S = valid_depth(S) ? S : C;
        W = valid_depth(W) ? W : C;
        E = valid_depth(E) ? E : C;
        return keep_valid(DIV ? adf_cell_div(C, N, S, W, E, p.kd, p.lam) : adf_cell(C, N, S, W, E, p.kc, p.l2lam),
                          p.keep_valid);
    }
    return DIV ? adf_cell_div(C, N, S, W, E, p.kd, p.lam) : adf_cell(C, N, S, W, E, p.kc, p.l2lam);
}

// ---------------------------------------------------------------------------
// Packed fp32 (sm_100a FADD2 / FMUL2 / FFMA2): one instruction updates both
// cells of a thread's pair (x, x+1) -- the same FP32-pipe work as two scalar
// ops in half the issue slots.  With P = (W, E) (the pair's outer neighbours,
// two scalar loads into one register pair) and Cs = (C.y, C.x) (the pair
// swapped: a free operand swizzle, .F32x2.LO_HI), the low cell's west / east
// neighbours are (W, C.y) and the high cell's are (C.x, E), so
//   Cs - P = (E - W | lo, -(E - W) | hi)   and   P + Cs = (W + E | lo, E + W | hi).
// The cell formula uses W and E only through (E - W)^2 and W + E, so both
// cells get exactly the rounding sequence of adf_cell() / adf_cell_div()
// (bitwise invariance).
// A product that feeds an add: ptxas fuses mul.rn.f32x2 + add.rn.f32x2 into
// FFMA2 even under --fmad=false (measured), and folds fma(a, b, -0) back into
// a mul.  fma(a, b, z) with z = -0 passed in at run time is the same rounded
// product for every input (a -0 addend keeps the sign of a zero product) and
// cannot be fused with the add.
PM_DEVINL float2 f2mul_nf(float2 a, float2 b, float z) { return f2fma(a, b, f2s(z)); }

PM_DEVINL float2 adf_cell2(float2 C, float2 N, float2 S, float2 Wv, float2 Ev, float kc, float l2lam) {
    const float2 gx2 = f2sub(Ev, Wv);
    const float2 gy2 = f2sub(S, N);
    const float2 g2 = f2fma(gx2, gx2, f2mul(gy2, gy2));
    const float2 e = f2fma(g2, f2s(kc), f2s(l2lam));
    const float2 lc = make_float2(ex2_approx(e.x), ex2_approx(e.y));
    const float2 lap = f2fma(f2s(-4.0f), C, f2add(f2add(N, S), f2add(Wv, Ev)));
    return f2fma(lc, lap, C);
}

PM_DEVINL float2 flux2(float2 d, float kd, float z) {
    const float2 a = f2mul(f2mul(d, d), f2s(kd));
    return f2mul_nf(make_float2(ex2_approx(a.x), ex2_approx(a.y)), d, z);
}

PM_DEVINL float2 adf_cell2_div(float2 C, float2 N, float2 S, float2 Wv, float2 Ev, float kd, float lam, float z) {
    const float2 fn = flux2(f2sub(N, C), kd, z), fs = flux2(f2sub(S, C), kd, z);
    const float2 fw = flux2(f2sub(Wv, C), kd, z), fe = flux2(f2sub(Ev, C), kd, z);
    return f2fma(f2s(lam), f2add(f2add(fn, fs), f2add(fw, fe)), C);
}

template <bool DIV>
PM_DEVINL float2 cell2(float2 C, float2 N, float2 S, float2 Wv, float2 Ev, const AdfParams& p) {
    return DIV ? adf_cell2_div(C, N, S, Wv, Ev, p.kd, p.lam, p.negz) : adf_cell2(C, N, S, Wv, Ev, p.kc, p.l2lam);
}


// Hole-aware pair cell with arbitrary neighbour pairs (register engine): the
// substitution of cell<true> per element, so each cell gets the scalar
// rounding sequence.
template <bool DIV>
PM_DEVINL float2 cell2_chk(float2 C, float2 N, float2 S, float2 Wv, float2 Ev, const AdfParams& p) {
    const bool vx = valid_depth(C.x), vy = valid_depth(C.y);
    N = make_float2(valid_depth(N.x) ? N.x : C.x, valid_depth(N.y) ? N.y : C.y);
    S = make_float2(valid_depth(S.x) ? S.x : C.x, valid_depth(S.y) ? S.y : C.y);
    Wv = make_float2(valid_depth(Wv.x) ? Wv.x : C.x, valid_depth(Wv.y) ? Wv.y : C.y);
    Ev = make_float2(valid_depth(Ev.x) ? Ev.x : C.x, valid_depth(Ev.y) ? Ev.y : C.y);
    float2 o = cell2<DIV>(C, N, S, Wv, Ev, p);
    o.x = vx ? keep_valid(o.x, p.keep_valid) : C.x;
    o.y = vy ? keep_valid(o.y, p.keep_valid) : C.y;
    return o;
}

// Sobel (1/8-normalised, clamp-to-edge) + geometric normal (Eq. 2 read as
// Q7): m = (fx Gx, fy Gy, -(Z + (u-cx) Gx + (v-cy) Gy)), n = m/|m|; (0,0,0)
// if any window pixel is invalid (Q9).  z[a][b] = window row a, column b.
// CHECK = false: the caller knows every window pixel is valid (hole-free tile).
// NM: the normals mode (PM_NORMALS_*), -1 = read p.nmode.
template <bool CHECK = true, int NM = -1>
PM_DEVINL float3 sobel_normal(const float z[3][3], float u, float v, const AdfParams& p) {
    if (CHECK) {
        bool ok = true;
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) ok = ok && valid_depth(z[a][b]);
        if (!ok) return make_float3(0.f, 0.f, 0.f);
    }
    const int nmode = NM >= 0 ? NM : p.nmode;
    const float gx = __fmul_rn(__fadd_rn(__fadd_rn(__fsub_rn(z[0][2], z[0][0]),
                                                   __fmul_rn(2.0f, __fsub_rn(z[1][2], z[1][0]))),
                                         __fsub_rn(z[2][2], z[2][0])), 0.125f);
    const float gy = __fmul_rn(__fadd_rn(__fadd_rn(__fsub_rn(z[2][0], z[0][0]),
                                                   __fmul_rn(2.0f, __fsub_rn(z[2][1], z[0][1]))),
                                         __fsub_rn(z[2][2], z[0][2])), 0.125f);
    float mx, my, mz;
    if (nmode == PM_NORMALS_AS_PRINTED) {        // Eq. 2 literally: -K^-1 [Gx, Gy, 1]^T (NEXT-1)
        mx = -__fmul_rn(__fsub_rn(gx, p.cx), p.ifx);
        my = -__fmul_rn(__fsub_rn(gy, p.cy), p.ify);
        mz = -1.0f;
    } else {
        mx = __fmul_rn(p.fx, gx);
        my = __fmul_rn(p.fy, gy);
        mz = -__fmaf_rn(__fsub_rn(v, p.cy), gy, __fmaf_rn(__fsub_rn(u, p.cx), gx, z[1][1]));
    }
    const float ss = __fmaf_rn(mx, mx, __fmaf_rn(my, my, __fmul_rn(mz, mz)));
    if (!(ss > 0.0f) || !(ss <= FLT_MAX)) return make_float3(0.f, 0.f, 0.f);
    float inv;                                   // MUFU.RSQ (ss < 2^-126 would flush: |m| >= ~|Z| here)
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(ss));
    return make_float3(__fmul_rn(mx, inv), __fmul_rn(my, inv), __fmul_rn(mz, inv));
}

// Fast-path ("hole-free") depth: valid and in [2^-100, 2^100).  For such
// tiles and lambda <= kNoCheckMaxLambda (internal.h) an update
// C + (lambda c) lap >= (1 - 4 lambda c) C >= 0.0036 C stays a positive normal
// float (lap >= -4C holds after rounding: the neighbour sum is >= 0, finite,
// and rounding is monotone), so no filtered pixel turns invalid: the normals
// epilogue may skip its window checks, and pm_process_frames' compaction
// count its depth reads.  Other tiles take the checked path.
PM_DEVINL bool fast_depth(float z) { return (__float_as_uint(z) - 0x0D800000u) < (0x71800000u - 0x0D800000u); }

}  // namespace adfk

// ---- adf_reg.cu (register-tile engine), host side
constexpr int kMaxItersRegPass = 16;
cudaError_t adf_reg_setup_attributes();
// Launches one pass on the register engine when applicable (*launched = true);
// otherwise returns cudaSuccess with *launched = false and launches nothing.
cudaError_t adf_reg_pass(const float* src, float* dst, float* normals, int W, int H, int B, int sweeps,
                         const adfk::AdfParams& p, cudaStream_t stream, int* frame_flags, int flag_mode,
                         bool* launched);

}  // namespace pm
