// adf_reg.cu — Algorithm 1 of arXiv 2411.01919 with the tile
// held in REGISTERS: the T Jacobi sweeps of a pass (ℓ2-8) and, in the last
// pass, the Sobel + normal stage (ℓ9-13), one HBM read and one write per
// pass.
//
// Why registers: the shared-memory column walk of adf.cu
// moves 12-16 B of shared memory per cell-sweep (south pair, west / east
// neighbours, the store) and ran at ~75 % of the SM's 128 B/clk shared-memory
// bandwidth, below both its FP32 and HBM rooflines.  Here every cell lives in
// a register; a thread only exchanges its block's perimeter through shared
// memory, ~8 B per cell-sweep at 128-bit width, so the pass is bound by the
// FP32 pipe (the method's 10 lane-ops per cell-sweep) instead.
//
// Layout.  A CTA owns a tile of kCH = 128 rows x cw = 4 ncg columns of one
// frame (ncg = 34..36 column groups for 640-wide frames), run by ncg x 16
// threads: thread (g, s) holds columns 4g .. 4g+3 of rows s*4 .. s*4+3 of
// the tile's TOP half and the same rows of its BOTTOM half.  The pair
// (top-half cell, bottom-half cell) of a column is one float2, so every cell
// update is packed FP32 (FADD2/FMUL2/FFMA2: two cells per instruction) and
// the north / south / west / east neighbours of a pair are themselves pairs:
// in-thread neighbours are registers, the rest come from the neighbouring
// threads' perimeter in shared memory.  The seam between the halves is
// exact: the bottom half's row -1 is the top half's last row.
//
// Tiles never extend beyond the frame: the last tile column / row is
// clamped to end at the image border.  A tile edge on the image border is
// the zero-flux boundary of Q4 (neighbour outside = centre, i.e. replicate),
// and any other tile edge is replicated too -- there the values are wrong
// but stay inside the halo (hr = T (+1 with normals) rows, hc = hr rounded
// up to 4 columns) that the tile does not output.
//
// Passes are persistent: one CTA per SM walks the tiles of the launch; the
// TMA load of its next tile lands in the shared tile buffer while the
// current tile's sweeps run in registers.  Results go to HBM straight from
// registers (128-bit stores).
//
// Every cell evaluates the identical _rn expression of adf_cell.cuh on
// identical operands, so the result is bitwise equal to the shared-memory
// engine (and independent of T, tiling and batching).
#include <cuda_runtime.h>
#include <float.h>
#include <stdint.h>

#include <mutex>

#include "adf_cell.cuh"
#include "common.cuh"
#include "internal.h"

namespace pm {

namespace {
using namespace adfk;

#ifndef PM_REG_NRS
#define PM_REG_NRS 16
#endif
#ifndef PM_REG_STS64
#define PM_REG_STS64 1
#endif
constexpr int kRS = 4;                  // rows per thread in each half
constexpr int kNRS = PM_REG_NRS;        // row strips per CTA
constexpr int kCtasPerSm = kNRS == 16 ? 1 : 2;
constexpr int kCH = 2 * kNRS * kRS;     // computed rows per tile
constexpr int kMaxNCG = 32;             // <= 128 computed columns: <= 16 warps (128 registers)
constexpr int kMinNCG = 8;

// shared memory: tile [kCH][cw] floats + exchange [2 parity][4 kind][kNRS][2 half][ncg] float4
__host__ __device__ constexpr size_t reg_smem_bytes(int ncg) {
    return sizeof(float) * (size_t)kCH * 4 * ncg + sizeof(float4) * (size_t)2 * 4 * kNRS * 2 * ncg;
}
// exchange kinds: left column, right column, top row, bottom row of a block
enum { XL = 0, XR = 1, XT = 2, XB = 3 };

struct RegGeom {
    int W, H;
    int ncg, cw;     // column groups per CTA, computed columns
    int ntx, nty;    // tiles per frame
    int hc, hr;      // halos
    int ntiles;      // B * ntx * nty
};

PM_DEVINL int tile_x(const RegGeom& G, int tx) { return tx >= G.ntx - 1 ? G.W - G.cw : tx * (G.cw - 2 * G.hc); }
PM_DEVINL int tile_y(const RegGeom& G, int ty) { return ty >= G.nty - 1 ? G.H - kCH : ty * (kCH - 2 * G.hr); }

// ---- packed pairs as 64-bit registers: every pair lives in an aligned
// register pair for its whole life, so the packed FP32 instructions take it
// without moves (a float2 would be split and re-paired by the allocator).
typedef uint64_t P2;
PM_DEVINL P2 pk(float a, float b) {
    P2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
PM_DEVINL float plo(P2 r) { return __uint_as_float((uint32_t)r); }
PM_DEVINL float phi(P2 r) { return __uint_as_float((uint32_t)(r >> 32)); }
PM_DEVINL P2 padd(P2 a, P2 b) { P2 r; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
PM_DEVINL P2 psub(P2 a, P2 b) { P2 r; asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
PM_DEVINL P2 pmul(P2 a, P2 b) { P2 r; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
PM_DEVINL P2 pfma(P2 a, P2 b, P2 c) {
    P2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
PM_DEVINL P2 pex2(P2 a) { return pk(ex2_approx(plo(a)), ex2_approx(phi(a))); }

// Broadcast constants of the cell formula.
struct PConst {
    P2 kc, l2lam, m4, kd, lam, negz;
};

// adf_cell2() / adf_cell2_div() of adf_cell.cuh on packed registers: the
// same operations in the same order (bitwise equal, tested).
template <bool DIV>
PM_DEVINL P2 pcell(P2 C, P2 N, P2 S, P2 W, P2 E, const PConst& k) {
    if (!DIV) {
        const P2 gx2 = psub(E, W);
        const P2 gy2 = psub(S, N);
        const P2 g2 = pfma(gx2, gx2, pmul(gy2, gy2));
        const P2 lc = pex2(pfma(g2, k.kc, k.l2lam));
        const P2 lap = pfma(k.m4, C, padd(padd(N, S), padd(W, E)));
        return pfma(lc, lap, C);
    } else {
        auto flux = [&](P2 d) { return pfma(pex2(pmul(pmul(d, d), k.kd)), d, k.negz); };
        const P2 fn = flux(psub(N, C)), fs = flux(psub(S, C));
        const P2 fw = flux(psub(W, C)), fe = flux(psub(E, C));
        return pfma(k.lam, padd(padd(fn, fs), padd(fw, fe)), C);
    }
}

// Hole-aware: cell2_chk() of adf_cell.cuh on packed registers.
PM_DEVINL float subst(float x, float c) { return valid_depth(x) ? x : c; }
template <bool DIV>
PM_DEVINL P2 pcell_chk(P2 C, P2 N, P2 S, P2 W, P2 E, const PConst& k, int keep) {
    const float cx = plo(C), cy = phi(C);
    N = pk(subst(plo(N), cx), subst(phi(N), cy));
    S = pk(subst(plo(S), cx), subst(phi(S), cy));
    W = pk(subst(plo(W), cx), subst(phi(W), cy));
    E = pk(subst(plo(E), cx), subst(phi(E), cy));
    const P2 o = pcell<DIV>(C, N, S, W, E, k);
    return pk(valid_depth(cx) ? keep_valid(plo(o), keep) : cx, valid_depth(cy) ? keep_valid(phi(o), keep) : cy);
}

// Shared-memory exchange of block perimeters, 2 parities x 4 kinds x kNRS x
// 2 halves x ncg entries of two pairs (16 B).  Per thread the word offsets of
// its own entries and of the entries it reads are fixed for the tile walk:
// a block edge on the tile border reads the thread's own entry instead
// (replicate = zero flux, Q4).
struct Xchg {
    P2* base;          // pairs
    int par_stride;    // pairs per parity
    int h_stride;      // pairs per half (2 ncg)
    int own[4];        // XL, XR, XT, XB entries of this thread (pair index of half 0)
    int rd_w, rd_e, rd_n, rd_s;
};

PM_DEVINL int xidx(int kind, int s, int h, int g, int ncg) { return (((kind * kNRS + s) * 2 + h) * ncg + g) * 2; }

PM_DEVINL void ld2(const P2* a, P2& x, P2& y) {
    asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "r"(smem_u32(a)));
}
PM_DEVINL void st2(P2* a, P2 x, P2 y) {
    asm volatile("st.shared.v2.b64 [%0], {%1, %2};" ::"r"(smem_u32(a)), "l"(x), "l"(y) : "memory");
}

struct Halo {
    P2 Wv[kRS], Ev[kRS], Nv[4], Sv[4];
};

// Neighbour pairs of the block in iterate `par`.  Seam: for s = 0 the north
// row of the top half replicates row 0 and that of the bottom half is the top
// half's last row (strip kNRS - 1); symmetric for the south row of s = kNRS - 1.
PM_DEVINL void load_halo(const P2 (&X)[4][kRS], const Xchg& x, int par, int s, Halo& h) {
    const P2* b = x.base + par * x.par_stride;
    ld2(b + x.rd_w, h.Wv[0], h.Wv[1]);
    ld2(b + x.rd_w + x.h_stride, h.Wv[2], h.Wv[3]);
    ld2(b + x.rd_e, h.Ev[0], h.Ev[1]);
    ld2(b + x.rd_e + x.h_stride, h.Ev[2], h.Ev[3]);
    ld2(b + x.rd_n, h.Nv[0], h.Nv[1]);
    ld2(b + x.rd_n + x.h_stride, h.Nv[2], h.Nv[3]);
    ld2(b + x.rd_s, h.Sv[0], h.Sv[1]);
    ld2(b + x.rd_s + x.h_stride, h.Sv[2], h.Sv[3]);
    if (s == 0) {
#pragma unroll
        for (int c = 0; c < 4; ++c) h.Nv[c] = pk(plo(X[c][0]), plo(h.Nv[c]));
    }
    if (s == kNRS - 1) {
#pragma unroll
        for (int c = 0; c < 4; ++c) h.Sv[c] = pk(phi(h.Sv[c]), phi(X[c][kRS - 1]));
    }
}

PM_DEVINL void st1(P2* a, P2 v) { asm volatile("st.shared.b64 [%0], %1;" ::"r"(smem_u32(a)), "l"(v) : "memory"); }

PM_DEVINL void store_edges(const P2 (&Y)[4][kRS], const Xchg& x, int par) {
    P2* b = x.base + par * x.par_stride;
    if (PM_REG_STS64) {   // one 8-byte store per pair: no moves to build 16-byte quads
        const int hs = x.h_stride;
        st1(b + x.own[XL], Y[0][0]); st1(b + x.own[XL] + 1, Y[0][1]);
        st1(b + x.own[XL] + hs, Y[0][2]); st1(b + x.own[XL] + hs + 1, Y[0][3]);
        st1(b + x.own[XR], Y[3][0]); st1(b + x.own[XR] + 1, Y[3][1]);
        st1(b + x.own[XR] + hs, Y[3][2]); st1(b + x.own[XR] + hs + 1, Y[3][3]);
        st1(b + x.own[XT], Y[0][0]); st1(b + x.own[XT] + 1, Y[1][0]);
        st1(b + x.own[XT] + hs, Y[2][0]); st1(b + x.own[XT] + hs + 1, Y[3][0]);
        st1(b + x.own[XB], Y[0][kRS - 1]); st1(b + x.own[XB] + 1, Y[1][kRS - 1]);
        st1(b + x.own[XB] + hs, Y[2][kRS - 1]); st1(b + x.own[XB] + hs + 1, Y[3][kRS - 1]);
        return;
    }
    st2(b + x.own[XL], Y[0][0], Y[0][1]);
    st2(b + x.own[XL] + x.h_stride, Y[0][2], Y[0][3]);
    st2(b + x.own[XR], Y[3][0], Y[3][1]);
    st2(b + x.own[XR] + x.h_stride, Y[3][2], Y[3][3]);
    st2(b + x.own[XT], Y[0][0], Y[1][0]);
    st2(b + x.own[XT] + x.h_stride, Y[2][0], Y[3][0]);
    st2(b + x.own[XB], Y[0][kRS - 1], Y[1][kRS - 1]);
    st2(b + x.own[XB] + x.h_stride, Y[2][kRS - 1], Y[3][kRS - 1]);
}

#ifndef PM_REG_SPLIT
#define PM_REG_SPLIT 1
#endif

// Exchange synchronisation.  PM_REG_SPLIT: two mbarriers (one per exchange
// parity, all threads arrive) split the barrier into arrive (after a
// thread's edges are stored) and wait (before it reads its neighbours'),
// so two interior pairs of the block -- which read no neighbour -- are
// computed while the slower threads catch up.  Otherwise one __syncthreads.
struct Sync {
    uint64_t* bar;     // [2] (PM_REG_SPLIT)
    uint32_t ph[2];    // phase bit per parity
    PM_DEVINL void arrive(int par) {
        if (PM_REG_SPLIT)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar + par)) : "memory");
        else
            __syncthreads();
    }
    PM_DEVINL void wait(int par) {
        if (PM_REG_SPLIT) {
            mbar_wait(bar + par, ph[par]);
            ph[par] ^= 1;
        }
    }
    // a phase that completed without this thread waiting on it
    PM_DEVINL void skip(int par) {
        if (PM_REG_SPLIT) ph[par] ^= 1;
    }
};

// One Jacobi sweep X (iterate k, edges in exchange parity par = k & 1) -> Y
// (edges to parity par ^ 1).  Order: the interior pairs (1..2, 1..2) read no
// neighbour, so two of them cover the latency of the halo loads, the edge
// pairs follow, their values are published, and the last two interior pairs
// run after the arrive.
template <bool CHECK, bool DIV>
PM_DEVINL void reg_sweep(const P2 (&X)[4][kRS], P2 (&Y)[4][kRS], const Xchg& x, Sync& sy, int par, int s,
                         const PConst& k, int keep) {
    sy.wait(par);
    Halo h;
#ifdef PM_REG_EXP_NOXCHG   // timing experiment only (wrong results): no halo exchange
    for (int i = 0; i < kRS; ++i) { h.Wv[i] = X[0][i]; h.Ev[i] = X[3][i]; h.Nv[i] = X[i][0]; h.Sv[i] = X[i][kRS - 1]; }
#else
    load_halo(X, x, par, s, h);
#endif
    auto upd = [&](int c, int i) {
        const P2 C = X[c][i];
        const P2 N = i > 0 ? X[c][i - 1] : h.Nv[c];
        const P2 S = i < kRS - 1 ? X[c][i + 1] : h.Sv[c];
        const P2 Wp = c > 0 ? X[c - 1][i] : h.Wv[i];
        const P2 Ep = c < 3 ? X[c + 1][i] : h.Ev[i];
        Y[c][i] = CHECK ? pcell_chk<DIV>(C, N, S, Wp, Ep, k, keep) : pcell<DIV>(C, N, S, Wp, Ep, k);
    };
    upd(1, 1);
    upd(2, 1);
#pragma unroll
    for (int i = 0; i < kRS; ++i)
#pragma unroll
        for (int c = 0; c < 4; ++c)
            if (c == 0 || c == 3 || i == 0 || i == kRS - 1) upd(c, i);
#ifndef PM_REG_EXP_NOXCHG
    store_edges(Y, x, par ^ 1);
#endif
#ifndef PM_REG_EXP_NOSYNC
    sy.arrive(par ^ 1);
#endif
    upd(1, 2);
    upd(2, 2);
}

template <bool CHECK, bool DIV>
PM_DEVINL void reg_sweeps(P2 (&A)[4][kRS], P2 (&B)[4][kRS], const Xchg& x, Sync& sy, int s, int T,
                          const PConst& k, int keep) {
    int t = 0;
    for (; t + 2 <= T; t += 2) {
        reg_sweep<CHECK, DIV>(A, B, x, sy, 0, s, k, keep);
        reg_sweep<CHECK, DIV>(B, A, x, sy, 1, s, k, keep);
    }
    if (t < T) {
        reg_sweep<CHECK, DIV>(A, B, x, sy, 0, s, k, keep);
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int i = 0; i < kRS; ++i) A[c][i] = B[c][i];
    }
}

// Sobel + normal of a pixel pair from its 3x3 window of pairs z[row][col]:
// the expression of sobel_normal() (adf_cell.cuh) per element, packed.
// CHECK: a window holding an invalid depth was made NaN by the caller, which
// makes ss NaN -> (0, 0, 0) (Q9).
template <bool CHECK, int NM>
PM_DEVINL void normal2(const P2 (&z)[3][3], P2 u, P2 v, const AdfParams& p, const PConst& k, P2& nx, P2& ny,
                       P2& nz) {
    const P2 two = pk(2.0f, 2.0f), eighth = pk(0.125f, 0.125f);
    const P2 gx = pmul(padd(padd(psub(z[0][2], z[0][0]), pmul(two, psub(z[1][2], z[1][0]))),
                            psub(z[2][2], z[2][0])), eighth);
    const P2 gy = pmul(padd(padd(psub(z[2][0], z[0][0]), pmul(two, psub(z[2][1], z[0][1]))),
                            psub(z[2][2], z[0][2])), eighth);
    P2 mx, my, mz;
    if (NM == PM_NORMALS_AS_PRINTED) {
        mx = pmul(psub(gx, pk(p.cx, p.cx)), pk(-p.ifx, -p.ifx));
        my = pmul(psub(gy, pk(p.cy, p.cy)), pk(-p.ify, -p.ify));
        mz = pk(-1.0f, -1.0f);
    } else {
        mx = pmul(pk(p.fx, p.fx), gx);
        my = pmul(pk(p.fy, p.fy), gy);
        const P2 t = pfma(psub(v, pk(p.cy, p.cy)), gy, pfma(psub(u, pk(p.cx, p.cx)), gx, z[1][1]));
        mz = pk(-plo(t), -phi(t));
    }
    const P2 ss = pfma(mx, mx, pfma(my, my, pfma(mz, mz, k.negz)));
    float ix, iy;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(ix) : "f"(plo(ss)));
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(iy) : "f"(phi(ss)));
    const P2 inv = pk(ix, iy);
    nx = pmul(mx, inv);
    ny = pmul(my, inv);
    nz = pmul(mz, inv);
    // (ss > 0 && ss <= FLT_MAX): positive finite, one unsigned compare
    bool okx = valid_depth(plo(ss)), oky = valid_depth(phi(ss));
    if (CHECK && NM == PM_NORMALS_AS_PRINTED) {   // Eq. 2 as printed does not read the centre: test it here
        okx = okx && plo(z[1][1]) == plo(z[1][1]);
        oky = oky && phi(z[1][1]) == phi(z[1][1]);
    }
    if (!okx || !oky) {
        nx = pk(okx ? plo(nx) : 0.f, oky ? phi(nx) : 0.f);
        ny = pk(okx ? plo(ny) : 0.f, oky ? phi(ny) : 0.f);
        nz = pk(okx ? plo(nz) : 0.f, oky ? phi(nz) : 0.f);
    }
}

PM_DEVINL P2 nan_if_invalid(P2 a) {
    const float q = __int_as_float(0x7fffffff);
    return pk(valid_depth(plo(a)) ? plo(a) : q, valid_depth(phi(a)) ? phi(a) : q);
}

struct TileIO {
    float* out;        // frame depth out (nullable)
    float* nrm;        // frame normals (nullable)
    size_t HW;
    int W;
    int x0, y0;        // tile origin (image coords)
    int bx0, bx1, by0, by1;   // output band
};

PM_DEVINL void stg4(float* a, float x, float y, float z, float w) {
    *reinterpret_cast<float4*>(a) = make_float4(x, y, z, w);
}

// Stores of the thread's depth block (rows in the band, column group in the band).
PM_DEVINL void store_depth(const P2 (&A)[4][kRS], const TileIO& io, int g, int s) {
    const int cx = io.x0 + 4 * g;
    if (cx < io.bx0 || cx >= io.bx1) return;
#pragma unroll
    for (int i = 0; i < kRS; ++i) {
        const int yt = io.y0 + s * kRS + i, yb = yt + kNRS * kRS;
        if (yt >= io.by0 && yt < io.by1)
            stg4(io.out + (size_t)yt * io.W + cx, plo(A[0][i]), plo(A[1][i]), plo(A[2][i]), plo(A[3][i]));
        if (yb >= io.by0 && yb < io.by1)
            stg4(io.out + (size_t)yb * io.W + cx, phi(A[0][i]), phi(A[1][i]), phi(A[2][i]), phi(A[3][i]));
    }
}

// Sobel + normals of the thread's block from the final iterate A (edges in
// exchange parity par).  Diagonal neighbours come from the edge columns of
// the diagonal threads; tile borders replicate (clamp-to-edge, Q8).
template <bool CHECK, int NM>
PM_DEVINL void normals_block(const P2 (&A)[4][kRS], const Xchg& x, int par, int g, int s, int ncg,
                             const TileIO& io, const AdfParams& p, const PConst& k) {
    Halo h;
    load_halo(A, x, par, s, h);
    const P2* b = x.base + par * x.par_stride;
    // corners (pairs): NW, NE, SW, SE from the diagonal threads' edge columns
    P2 NW, NE, SW, SE, t0, t1;
    auto colpair = [&](int kind, int ss, int hh, int gg, P2& a0, P2& a1) {
        ld2(b + xidx(kind, ss, hh, gg, ncg), a0, a1);
    };
    if (g > 0) {
        if (s > 0) { colpair(XR, s - 1, 1, g - 1, t0, NW); }
        else { colpair(XR, kNRS - 1, 1, g - 1, t0, t1); NW = pk(plo(h.Wv[0]), plo(t1)); }
        if (s < kNRS - 1) { colpair(XR, s + 1, 0, g - 1, SW, t0); }
        else { colpair(XR, 0, 0, g - 1, t0, t1); SW = pk(phi(t0), phi(h.Wv[kRS - 1])); }
    } else {
        NW = h.Nv[0];
        SW = h.Sv[0];
    }
    if (g < ncg - 1) {
        if (s > 0) { colpair(XL, s - 1, 1, g + 1, t0, NE); }
        else { colpair(XL, kNRS - 1, 1, g + 1, t0, t1); NE = pk(plo(h.Ev[0]), plo(t1)); }
        if (s < kNRS - 1) { colpair(XL, s + 1, 0, g + 1, SE, t0); }
        else { colpair(XL, 0, 0, g + 1, t0, t1); SE = pk(phi(t0), phi(h.Ev[kRS - 1])); }
    } else {
        NE = h.Nv[3];
        SE = h.Sv[3];
    }
    // extended block E[col + 1][row + 1], col -1..4, row -1..kRS
    P2 E[6][kRS + 2];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
#pragma unroll
        for (int i = 0; i < kRS; ++i) E[c + 1][i + 1] = A[c][i];
        E[c + 1][0] = h.Nv[c];
        E[c + 1][kRS + 1] = h.Sv[c];
    }
#pragma unroll
    for (int i = 0; i < kRS; ++i) {
        E[0][i + 1] = h.Wv[i];
        E[5][i + 1] = h.Ev[i];
    }
    E[0][0] = NW; E[5][0] = NE; E[0][kRS + 1] = SW; E[5][kRS + 1] = SE;
    if (CHECK) {
#pragma unroll
        for (int c = 0; c < 6; ++c)
#pragma unroll
            for (int i = 0; i < kRS + 2; ++i) E[c][i] = nan_if_invalid(E[c][i]);
    }
    const int cx = io.x0 + 4 * g;
    if (cx < io.bx0 || cx >= io.bx1) return;
    const int yt = io.y0 + s * kRS, yb = yt + kNRS * kRS;
#pragma unroll
    for (int i = 0; i < kRS; ++i) {
        const P2 v = pk((float)(yt + i), (float)(yb + i));
        P2 nx[4], ny[4], nz[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const float uf = (float)(cx + c);
            P2 z[3][3];
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int bb = 0; bb < 3; ++bb) z[a][bb] = E[c + bb][i + a];
            normal2<CHECK, NM>(z, pk(uf, uf), v, p, k, nx[c], ny[c], nz[c]);
        }
        if (yt + i >= io.by0 && yt + i < io.by1) {
            const size_t o = (size_t)(yt + i) * io.W + cx;
            stg4(io.nrm + o, plo(nx[0]), plo(nx[1]), plo(nx[2]), plo(nx[3]));
            stg4(io.nrm + io.HW + o, plo(ny[0]), plo(ny[1]), plo(ny[2]), plo(ny[3]));
            stg4(io.nrm + 2 * io.HW + o, plo(nz[0]), plo(nz[1]), plo(nz[2]), plo(nz[3]));
        }
        if (yb + i >= io.by0 && yb + i < io.by1) {
            const size_t o = (size_t)(yb + i) * io.W + cx;
            stg4(io.nrm + o, phi(nx[0]), phi(nx[1]), phi(nx[2]), phi(nx[3]));
            stg4(io.nrm + io.HW + o, phi(ny[0]), phi(ny[1]), phi(ny[2]), phi(ny[3]));
            stg4(io.nrm + 2 * io.HW + o, phi(nz[0]), phi(nz[1]), phi(nz[2]), phi(nz[3]));
        }
    }
}

#ifdef PM_REG_TIMING
// Per-phase SM-cycle counters (variant builds only; tools/): wait, load,
// edges, sweeps, depth stores, normals.
__device__ unsigned long long g_reg_prof[8];
#define PM_TSTAMP(v) const long long v = clock64()
#define PM_TACC(k, a, b) if (threadIdx.x == 0) atomicAdd(&g_reg_prof[k], (unsigned long long)((b) - (a)))
#else
#define PM_TSTAMP(v)
#define PM_TACC(k, a, b)
#endif

// One pass: T sweeps (+ normals when NRM) over every tile of the launch.
//   src [B][H][W] -> dst [B][H][W] (nullable when NRM) and normals [B][3][H][W].
// grid = min(tiles, SMs), block = ncg * kNRS threads, one CTA per SM.
template <bool DIV, bool NRM, int NM>
__global__ void __launch_bounds__(kMaxNCG * kNRS, kCtasPerSm)
adf_reg_kernel(float* __restrict__ dst, float* __restrict__ normals, RegGeom G, int T, AdfParams p,
               const __grid_constant__ CUtensorMap tmap, int* __restrict__ frame_flags, int flag_mode) {
    extern __shared__ __align__(128) float smem[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ __align__(8) uint64_t xbar[2];
    const int ncg = G.ncg;
    const int tid = threadIdx.x;
    const int g = tid % ncg, s = tid / ncg;
    float* tile = smem;
    Xchg x;
    x.base = reinterpret_cast<P2*>(smem + (size_t)kCH * G.cw);
    x.par_stride = 4 * kNRS * 2 * ncg * 2;
    x.h_stride = 2 * ncg;
#pragma unroll
    for (int kd = 0; kd < 4; ++kd) x.own[kd] = xidx(kd, s, 0, g, ncg);
    x.rd_w = g > 0 ? xidx(XR, s, 0, g - 1, ncg) : x.own[XL];
    x.rd_e = g < ncg - 1 ? xidx(XL, s, 0, g + 1, ncg) : x.own[XR];
    x.rd_n = xidx(XB, s > 0 ? s - 1 : kNRS - 1, 0, g, ncg);
    x.rd_s = xidx(XT, s < kNRS - 1 ? s + 1 : 0, 0, g, ncg);
    PConst k;
    k.kc = pk(p.kc, p.kc);
    k.l2lam = pk(p.l2lam, p.l2lam);
    k.m4 = pk(-4.0f, -4.0f);
    k.kd = pk(p.kd, p.kd);
    k.lam = pk(p.lam, p.lam);
    k.negz = pk(p.negz, p.negz);
    const int per_frame = G.ntx * G.nty;
    const size_t HW = (size_t)G.W * G.H;

    auto coords = [&](int t, int& f, int& tx, int& ty) {
        f = t / per_frame;
        const int r = t - f * per_frame;
        ty = r / G.ntx;
        tx = r - ty * G.ntx;
    };
    auto issue = [&](int t) {
        int f, tx, ty;
        coords(t, f, tx, ty);
        mbar_arrive_expect_tx(&bar, (uint32_t)(sizeof(float) * kCH * G.cw));
        tma_load_3d(tile, &tmap, tile_x(G, tx), tile_y(G, ty), f, &bar);
    };
    if (tid == 0) {
        mbar_init(&bar, 1);
        mbar_init(&xbar[0], blockDim.x);
        mbar_init(&xbar[1], blockDim.x);
    }
    __syncthreads();
    Sync sy;
    sy.bar = xbar;
    sy.ph[0] = sy.ph[1] = 0;
    if (tid == 0 && (int)blockIdx.x < G.ntiles) issue(blockIdx.x);
    uint32_t phase = 0;
    for (int t = blockIdx.x; t < G.ntiles; t += gridDim.x) {
        int f, tx, ty;
        coords(t, f, tx, ty);
        TileIO io;
        io.HW = HW;
        io.W = G.W;
        io.out = dst ? dst + (size_t)f * HW : nullptr;
        io.nrm = NRM ? normals + (size_t)f * 3 * HW : nullptr;
        io.x0 = tile_x(G, tx);
        io.y0 = tile_y(G, ty);
        io.bx0 = tx == 0 ? 0 : io.x0 + G.hc;
        io.bx1 = tx == G.ntx - 1 ? G.W : tile_x(G, tx + 1) + G.hc;
        io.by0 = ty == 0 ? 0 : io.y0 + G.hr;
        io.by1 = ty == G.nty - 1 ? G.H : tile_y(G, ty + 1) + G.hr;

        PM_TSTAMP(t0);
        mbar_wait(&bar, phase);
        phase ^= 1;
        PM_TSTAMP(t1);
        P2 A[4][kRS], B[4][kRS];
        // validity scan, skipped when the first pass found the frame hole-free
        // (validity is fixed by the input, Q4)
        const bool scan = flag_mode != 2 || frame_flags[f] != 0;
        bool fast = true;
#pragma unroll
        for (int i = 0; i < kRS; ++i) {
            const float4 a = *reinterpret_cast<const float4*>(tile + (size_t)(s * kRS + i) * G.cw + 4 * g);
            const float4 b = *reinterpret_cast<const float4*>(tile + (size_t)(kNRS * kRS + s * kRS + i) * G.cw + 4 * g);
            A[0][i] = pk(a.x, b.x); A[1][i] = pk(a.y, b.y);
            A[2][i] = pk(a.z, b.z); A[3][i] = pk(a.w, b.w);
            if (scan)
                fast &= fast_depth(a.x) && fast_depth(a.y) && fast_depth(a.z) && fast_depth(a.w) &&
                        fast_depth(b.x) && fast_depth(b.y) && fast_depth(b.z) && fast_depth(b.w);
        }
        fast = __syncthreads_and(fast);   // also: every thread is done with the tile buffer
        if (tid == 0) {
            if (flag_mode == 1 && !fast) atomicOr(frame_flags + f, 1);
            if (t + (int)gridDim.x < G.ntiles) {
                fence_proxy_async_smem();
                issue(t + gridDim.x);
            }
        }
        PM_TSTAMP(t2);
        store_edges(A, x, 0);
        sy.arrive(0);
        PM_TSTAMP(t3);
        // the unchecked sweeps only where no update can turn a pixel invalid
        const bool sweep_fast = fast && !p.keep_valid;
        if (sweep_fast) reg_sweeps<false, DIV>(A, B, x, sy, s, T, k, 0);
        else reg_sweeps<true, DIV>(A, B, x, sy, s, T, k, p.keep_valid);
        PM_TSTAMP(t4);
        if (io.out) store_depth(A, io, g, s);
        PM_TSTAMP(t5);
        PM_TACC(0, t0, t1); PM_TACC(1, t1, t2); PM_TACC(2, t2, t3); PM_TACC(3, t3, t4); PM_TACC(4, t4, t5);
        if (NRM) sy.wait(T & 1);    // the final iterate's edges
        else sy.skip(T & 1);
        if (NRM) {
            // hole-free tile: every window is valid for lambda <= kNoCheckMaxLambda (adf.cu fast_depth)
            const bool nocheck = fast && (T == 0 || p.lam <= kNoCheckMaxLambda);
            if (nocheck) normals_block<false, NM>(A, x, T & 1, g, s, ncg, io, p, k);
            else normals_block<true, NM>(A, x, T & 1, g, s, ncg, io, p, k);
            PM_TSTAMP(t6);
            PM_TACC(5, t5, t6);
        }
    }
}

using RegFn = void (*)(float*, float*, RegGeom, int, AdfParams, const CUtensorMap, int*, int);

RegFn reg_fn(bool div, bool nrm, int nmode) {
    if (!nrm) return div ? adf_reg_kernel<true, false, 0> : adf_reg_kernel<false, false, 0>;
    if (nmode == PM_NORMALS_AS_PRINTED)
        return div ? adf_reg_kernel<true, true, PM_NORMALS_AS_PRINTED> : adf_reg_kernel<false, true, PM_NORMALS_AS_PRINTED>;
    return div ? adf_reg_kernel<true, true, PM_NORMALS_GEOMETRIC> : adf_reg_kernel<false, true, PM_NORMALS_GEOMETRIC>;
}

// Tiling of one axis: n tiles of `cw` computed cells with halo h, the first
// and last clamped to the border.  Valid when every output band is
// non-empty and inside its tile's valid region.
bool axis_ok(int W, int cw, int h, int n) {
    if (cw > W || n < 1) return false;
    if (n == 1) return cw == W;
    if (cw - 2 * h <= 0) return false;
    auto xs = [&](int j) { return j >= n - 1 ? W - cw : j * (cw - 2 * h); };
    int b0 = 0;
    for (int j = 0; j < n; ++j) {
        const int b1 = j == n - 1 ? W : xs(j + 1) + h;
        const int lo = xs(j) + (j > 0 ? h : 0), hi = xs(j) + cw - (j < n - 1 ? h : 0);
        if (xs(j) < 0 || b1 <= b0 || b0 < lo || b1 > hi) return false;
        b0 = b1;
    }
    return true;
}

bool make_geom(int W, int H, int B, int sweeps, bool nrm, RegGeom& G) {
    if ((W & 3) != 0 || H < kCH) return false;
    const int hr = sweeps + (nrm ? 1 : 0);
    const int hc = (hr + 3) & ~3;
    G.W = W; G.H = H; G.hr = hr; G.hc = hc;
    G.ncg = 0;
    for (int n = 1; n <= W / (4 * kMinNCG) + 1 && G.ncg == 0; ++n) {
        const int need = (W + 2 * hc * (n - 1) + n - 1) / n;
        const int cw = (need + 3) & ~3;
        if (cw > 4 * kMaxNCG) continue;
        if (cw < 4 * kMinNCG || !axis_ok(W, cw, hc, n)) continue;
        G.ncg = cw / 4; G.cw = cw; G.ntx = n;
    }
    if (G.ncg == 0) return false;
    G.nty = 0;
    for (int n = 1; n <= H / 8 + 1 && G.nty == 0; ++n)
        if ((long)n * kCH - 2L * hr * (n - 1) >= H && axis_ok(H, kCH, hr, n)) G.nty = n;
    if (G.nty == 0) return false;
    const long tiles = (long)B * G.ntx * G.nty;
    if (tiles > (1L << 30)) return false;
    G.ntiles = (int)tiles;
    return true;
}

constexpr int kMaxDev = 64;
std::once_flag g_sm_once[kMaxDev];
int g_sms[kMaxDev];

}  // namespace

cudaError_t adf_reg_setup_attributes() {
    const size_t smem = reg_smem_bytes(kMaxNCG);
    for (int d = 0; d < 2; ++d)
        for (int n = 0; n < 2; ++n)
            for (int m = 0; m < 2; ++m) {
                cudaError_t e = cudaFuncSetAttribute(reg_fn(d, n, m), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     (int)smem);
                if (e != cudaSuccess) return e;
            }
    return cudaSuccess;
}

cudaError_t adf_reg_pass(const float* src, float* dst, float* normals, int W, int H, int B, int sweeps,
                         const AdfParams& p, cudaStream_t stream, int* frame_flags, int flag_mode, bool* launched) {
    *launched = false;
    RegGeom G;
    if (((uintptr_t)src & 15u) != 0 || sweeps > kMaxItersRegPass) return cudaSuccess;
    if (!make_geom(W, H, B, sweeps, normals != nullptr, G)) return cudaSuccess;
    CUtensorMap tmap;
    if (!make_tmap_f32_3d(&tmap, src, W, H, B, G.cw, kCH)) return cudaSuccess;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= kMaxDev) return cudaErrorInvalidDevice;
    std::call_once(g_sm_once[dev], [dev] {
        if (cudaDeviceGetAttribute(&g_sms[dev], cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) g_sms[dev] = 148;
    });
    const int grid = G.ntiles < kCtasPerSm * g_sms[dev] ? G.ntiles : kCtasPerSm * g_sms[dev];
    const RegFn fn = reg_fn(p.scheme == PM_ADF_DIVERGENCE, normals != nullptr, p.nmode);
    int T = sweeps;
    AdfParams pv = p;
    void* args[] = {(void*)&dst, (void*)&normals, (void*)&G, (void*)&T, (void*)&pv, (void*)&tmap,
                    (void*)&frame_flags, (void*)&flag_mode};
    e = cudaLaunchKernel((const void*)fn, dim3(grid), dim3(G.ncg * kNRS), args, reg_smem_bytes(G.ncg), stream);
    if (e == cudaSuccess) *launched = true;
    return e;
}

#ifdef PM_REG_TIMING
extern "C" __attribute__((visibility("default"))) int pm_debug_reg_prof(unsigned long long* out, int reset) {
    if (cudaMemcpyFromSymbol(out, pm::g_reg_prof, sizeof(unsigned long long) * 8) != cudaSuccess) return 1;
    if (reset) {
        unsigned long long z[8] = {};
        cudaMemcpyToSymbol(pm::g_reg_prof, z, sizeof(z));
    }
    return 0;
}
#endif
}  // namespace pm
