// adf_stream.cu — Algorithm 1 as a streaming wavefront: one CTA
// owns a vertical strip of 2 x blockDim.x columns of one frame and walks it
// top to bottom once, carrying all T sweeps ("levels") at the same time.
//
//   * level 0 is the input row; level t computes row r = s - 2t at step s
//     from level t-1's rows r-1, r, r+1 (the lag of 2 rows per level lets
//     every level of a step read only values produced in earlier steps, so a
//     step needs one CTA barrier for all T levels);
//   * each thread owns two adjacent columns; its own north/centre/south
//     values of every level live in registers (a 3-row ring per level whose
//     slots are compile-time constants: the step loop is unrolled by 3), the
//     west / east neighbours come from a 3-row shared-memory ring per level
//     (one 8-byte store and two 4-byte loads per pair and level);
//   * no halo in y at all and one HBM pass for all T sweeps: the only
//     redundant work is the T-column halo on each side of the strip;
//   * the last level is also staged in a 4-row ring from which the Sobel /
//     normal of row r - 2 is computed at step s (Alg. 1 ℓ9-13);
//   * the zero-flux image border (Q4) costs nothing per cell in the steady
//     state: the pair on the first / last image column points its W / E
//     address at itself, and rows 0 / H-1 are handled by the boundary steps;
//   * frames with holes are detected on the fly (the per-step barrier is a
//     __syncthreads_or over "an invalid input was loaded") and switch to the
//     hole-aware step for the rest of the walk.
// Every cell evaluates the same _rn expression as adf.cu on the same
// operands, so the output is bitwise identical to the tiled kernel.
#include <cuda_runtime.h>
#include <float.h>
#include <stdint.h>

#include "common.cuh"
#include "internal.h"

namespace pm {

namespace {

constexpr int kMaxStreamLevels = 20;

PM_DEVINL float s_cell_alg1(float C, float N, float S, float W, float E, float kc, float l2lam) {
    const float gx2 = __fsub_rn(E, W);
    const float gy2 = __fsub_rn(S, N);
    const float g2 = __fmaf_rn(gx2, gx2, __fmul_rn(gy2, gy2));
    const float lc = ex2_approx(__fmaf_rn(g2, kc, l2lam));
    const float lap = __fmaf_rn(-4.0f, C, __fadd_rn(__fadd_rn(N, S), __fadd_rn(W, E)));
    return __fmaf_rn(lc, lap, C);
}

PM_DEVINL float s_cell_div(float C, float N, float S, float W, float E, float kd, float lam) {
    const float dn = __fsub_rn(N, C), ds = __fsub_rn(S, C);
    const float dw = __fsub_rn(W, C), de = __fsub_rn(E, C);
    const float fn = __fmul_rn(ex2_approx(__fmul_rn(__fmul_rn(dn, dn), kd)), dn);
    const float fs = __fmul_rn(ex2_approx(__fmul_rn(__fmul_rn(ds, ds), kd)), ds);
    const float fw = __fmul_rn(ex2_approx(__fmul_rn(__fmul_rn(dw, dw), kd)), dw);
    const float fe = __fmul_rn(ex2_approx(__fmul_rn(__fmul_rn(de, de), kd)), de);
    return __fmaf_rn(lam, __fadd_rn(__fadd_rn(fn, fs), __fadd_rn(fw, fe)), C);
}

template <bool CHECK, bool DIV>
PM_DEVINL float s_cell(float C, float N, float S, float W, float E, const AdfStreamParams& p) {
    if (CHECK) {
        if (!valid_depth(C)) return C;
        N = valid_depth(N) ? N : C;
        S = valid_depth(S) ? S : C;
        W = valid_depth(W) ? W : C;
        E = valid_depth(E) ? E : C;
    }
    return DIV ? s_cell_div(C, N, S, W, E, p.kd, p.lam) : s_cell_alg1(C, N, S, W, E, p.kc, p.l2lam);
}

PM_DEVINL float3 s_sobel_normal(const float z[3][3], float u, float v, const AdfStreamParams& p) {
    bool ok = true;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) ok = ok && valid_depth(z[a][b]);
    if (!ok) return make_float3(0.f, 0.f, 0.f);
    const float gx = __fmul_rn(__fadd_rn(__fadd_rn(__fsub_rn(z[0][2], z[0][0]),
                                                   __fmul_rn(2.0f, __fsub_rn(z[1][2], z[1][0]))),
                                         __fsub_rn(z[2][2], z[2][0])), 0.125f);
    const float gy = __fmul_rn(__fadd_rn(__fadd_rn(__fsub_rn(z[2][0], z[0][0]),
                                                   __fmul_rn(2.0f, __fsub_rn(z[2][1], z[0][1]))),
                                         __fsub_rn(z[2][2], z[0][2])), 0.125f);
    float mx, my, mz;
    if (p.nmode == PM_NORMALS_AS_PRINTED) {
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
    const float inv = rsqrtf(ss);
    return make_float3(__fmul_rn(mx, inv), __fmul_rn(my, inv), __fmul_rn(mz, inv));
}

struct StreamCtx {
    const float* in;      // frame input
    float* out;           // frame output (depth)
    float* nrm;           // frame normals or nullptr
    size_t HW;
    int W, H;
    int c;                // strip column of this thread's pair (even)
    int gx;               // image column of the pair
    int offW, offE;       // shared-ring offsets of the west / east neighbour
    bool in_img;          // pair inside the image
    bool out_col;         // pair inside the strip's output range and the image
    int SW;               // strip width (floats)
    float* pub;           // [T][3][SW] level rings (levels 0 .. T-1)
    float* ring_out;      // [4][SW] last level
};

// One step of the wavefront, phase PH = s % 3 (compile time), all levels.
// GENERAL: rows outside [0, H) are skipped, rows 0 / H-1 use the zero-flux
// rule, the hole-aware cell is used; otherwise (steady state) every level is
// interior and the fast cell is used.
template <int T, int PH, bool GENERAL, bool DIV>
PM_DEVINL void stream_step(const int s, float2 (&Rg)[T + 1][3], float2 (&IN)[3], bool& bad,
                           const StreamCtx& x, const AdfStreamParams& p) {
    // ---- levels T .. 1 (descending: level t reads level t-1's ring before
    // level t-1 overwrites its oldest slot in this step)
#pragma unroll
    for (int t = T; t >= 1; --t) {
        const int r = s - 2 * t;
        if (GENERAL && (r < 0 || r >= x.H)) continue;
        const int kC = ((PH - 2 * t) % 3 + 3) % 3;       // slot of level t-1's row r
        const int kS = (kC + 1) % 3;                     // row r + 1
        const int kN = (kC + 2) % 3;                     // row r - 1
        const float2 C = Rg[t - 1][kC];
        float2 N = Rg[t - 1][kN], S = Rg[t - 1][kS];
        if (GENERAL) {
            if (r == 0) N = C;
            if (r == x.H - 1) S = C;
        }
        const float* rowp = x.pub + (size_t)(t - 1) * 3 * x.SW + kC * x.SW;
        const float Wv = rowp[x.c + x.offW];
        const float Ev = rowp[x.c + x.offE];
        float2 o;
        o.x = s_cell<GENERAL, DIV>(C.x, N.x, S.x, Wv, C.y, p);
        o.y = s_cell<GENERAL, DIV>(C.y, N.y, S.y, C.x, Ev, p);
        Rg[t][kC] = o;
        if (t < T) {
            *reinterpret_cast<float2*>(x.pub + (size_t)t * 3 * x.SW + kC * x.SW + x.c) = o;
        } else {
            *reinterpret_cast<float2*>(x.ring_out + (r & 3) * x.SW + x.c) = o;
            if (x.out_col) *reinterpret_cast<float2*>(x.out + (size_t)r * x.W + x.gx) = o;
        }
    }
    // ---- level 0 last (level 1 above read its oldest slot first): input
    // row s (loaded 3 steps ago), prefetch row s + 3
    if (!GENERAL || s < x.H) {
        const float2 v = IN[PH];
        Rg[0][PH] = v;
        bad |= x.in_img && !(valid_depth(v.x) && valid_depth(v.y));
        *reinterpret_cast<float2*>(x.pub + PH * x.SW + x.c) = v;
    }
    if (!GENERAL || s + 3 < x.H) {
        if (x.in_img) IN[PH] = __ldg(reinterpret_cast<const float2*>(x.in + (size_t)(s + 3) * x.W + x.gx));
    }
    // ---- normals of row rn = s - 2T - 2 from the last level's 4-row ring
    if (x.nrm) {
        const int rn = s - 2 * T - 2;
        if (!GENERAL || (rn >= 0 && rn < x.H)) {
            if (x.out_col) {
                const int rows[3] = {max(rn - 1, 0), rn, min(rn + 1, x.H - 1)};
                float z[3][4];
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    const float* rp = x.ring_out + (rows[a] & 3) * x.SW + x.c;
                    const float2 m = *reinterpret_cast<const float2*>(rp);
                    z[a][1] = m.x;
                    z[a][2] = m.y;
                    z[a][0] = x.offW == 0 ? m.x : rp[-1];
                    z[a][3] = x.offE == 1 ? m.y : rp[2];
                }
                const float w0[3][3] = {{z[0][0], z[0][1], z[0][2]}, {z[1][0], z[1][1], z[1][2]},
                                        {z[2][0], z[2][1], z[2][2]}};
                const float w1[3][3] = {{z[0][1], z[0][2], z[0][3]}, {z[1][1], z[1][2], z[1][3]},
                                        {z[2][1], z[2][2], z[2][3]}};
                const float3 n0 = s_sobel_normal(w0, (float)x.gx, (float)rn, p);
                const float3 n1 = s_sobel_normal(w1, (float)(x.gx + 1), (float)rn, p);
                const size_t o = (size_t)rn * x.W + x.gx;
                *reinterpret_cast<float2*>(x.nrm + o) = make_float2(n0.x, n1.x);
                *reinterpret_cast<float2*>(x.nrm + x.HW + o) = make_float2(n0.y, n1.y);
                *reinterpret_cast<float2*>(x.nrm + 2 * x.HW + o) = make_float2(n0.z, n1.z);
            }
        }
    }
}

// grid = (n_strips, B); block = SW / 2 threads; dynamic smem (T + 4/3) * 3 * SW floats.
template <int T, bool DIV>
__global__ void __launch_bounds__(256, 1)
adf_stream_kernel(const float* __restrict__ src, float* __restrict__ dst, float* __restrict__ normals, int W,
                  int H, int halo, AdfStreamParams p) {
    extern __shared__ __align__(16) float smem[];
    StreamCtx x;
    x.SW = 2 * blockDim.x;
    x.pub = smem;
    x.ring_out = smem + (size_t)T * 3 * x.SW;
    x.W = W;
    x.H = H;
    x.HW = (size_t)W * H;
    const size_t f = blockIdx.y;
    x.in = src + f * x.HW;
    x.out = dst + f * x.HW;
    x.nrm = normals ? normals + f * 3 * x.HW : nullptr;
    const int TWs = x.SW - 2 * halo;
    const int x0 = blockIdx.x * TWs - halo;
    x.c = 2 * threadIdx.x;
    x.gx = x0 + x.c;
    x.in_img = x.gx >= 0 && x.gx < W;               // W even: a pair is fully in or out
    x.out_col = x.in_img && x.c >= halo && x.c < halo + TWs;
    x.offW = (x.gx == 0 || x.c == 0) ? 0 : -1;      // zero flux at the image border (Q4)
    x.offE = (x.gx + 2 == W || x.c + 2 == x.SW) ? 1 : 2;
    float2 Rg[T + 1][3];
    float2 IN[3];
#pragma unroll
    for (int t = 0; t <= T; ++t)
#pragma unroll
        for (int k = 0; k < 3; ++k) Rg[t][k] = make_float2(0.f, 0.f);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        IN[k] = make_float2(0.f, 0.f);
        if (x.in_img && k < H) IN[k] = __ldg(reinterpret_cast<const float2*>(x.in + (size_t)k * W + x.gx));
    }
    // out-of-image pairs publish zeros (never read by in-image cells)
    bool bad = false;
    bool holes = false;
    const int n_steps = H + 2 * T + 2;               // s = 0 .. H + 2T + 1
    // steady state: every level interior (1 <= s - 2t <= H - 2), an input row
    // to read (s < H) and one to prefetch (s + 3 < H), normals row >= 0
    const int fast_lo = 2 * T + 2, fast_hi = H - 4;
    auto general = [&](int st) {
        const int ph = st % 3;
        if (ph == 0) stream_step<T, 0, true, DIV>(st, Rg, IN, bad, x, p);
        else if (ph == 1) stream_step<T, 1, true, DIV>(st, Rg, IN, bad, x, p);
        else stream_step<T, 2, true, DIV>(st, Rg, IN, bad, x, p);
    };
    int s = 0;
    while (s < n_steps && (s < fast_lo || s % 3 != 0)) {
        general(s);
        holes = __syncthreads_or(bad);
        ++s;
    }
    while (!holes && s + 2 <= fast_hi) {             // s % 3 == 0 here
        stream_step<T, 0, false, DIV>(s, Rg, IN, bad, x, p);
        holes = __syncthreads_or(bad);
        ++s;
        if (holes) break;
        stream_step<T, 1, false, DIV>(s, Rg, IN, bad, x, p);
        holes = __syncthreads_or(bad);
        ++s;
        if (holes) break;
        stream_step<T, 2, false, DIV>(s, Rg, IN, bad, x, p);
        holes = __syncthreads_or(bad);
        ++s;
    }
    while (s < n_steps) {
        general(s);
        __syncthreads();
        ++s;
    }
}

}  // namespace

// ---------------------------------------------------------------------------
// host side
using StreamFn = void (*)(const float*, float*, float*, int, int, int, AdfStreamParams);

template <int T>
struct StreamTable {
    static void fill(StreamFn (*fns)[2]) {
        fns[T][0] = adf_stream_kernel<T, false>;
        fns[T][1] = adf_stream_kernel<T, true>;
        StreamTable<T - 1>::fill(fns);
    }
};
template <>
struct StreamTable<0> {
    static void fill(StreamFn (*)[2]) {}
};

static const StreamFn (&stream_fns())[kMaxStreamLevels + 1][2] {
    static StreamFn fns[kMaxStreamLevels + 1][2] = {};
    static bool init = false;
    if (!init) { StreamTable<kMaxStreamLevels>::fill(fns); init = true; }
    return fns;
}

int adf_stream_max_levels() { return kMaxStreamLevels; }

static size_t stream_smem(int T, int SW) { return sizeof(float) * ((size_t)T * 3 * SW + 4 * (size_t)SW); }

cudaError_t adf_stream_setup_attributes() {
    const auto& F = stream_fns();
    for (int T = 1; T <= kMaxStreamLevels; ++T)
        for (int d = 0; d < 2; ++d) {
            cudaError_t e = cudaFuncSetAttribute(F[T][d], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)stream_smem(T, 512));
            if (e != cudaSuccess) return e;
        }
    return cudaSuccess;
}

// Strip width for this frame width: multiple of 64 columns in [256, 512],
// minimising computed columns (strips x width), ties to the narrower strip.
static int pick_strip(int W, int halo) {
    int best = 256;
    long best_cost = -1;
    for (int sw = 256; sw <= 512; sw += 64) {
        const int tw = sw - 2 * halo;
        if (tw <= 0) continue;
        const long cost = (long)((W + tw - 1) / tw) * sw;
        if (best_cost < 0 || cost < best_cost) { best_cost = cost; best = sw; }
    }
    return best;
}

bool adf_stream_applicable(int W, int H, int levels) {
    return (W % 2) == 0 && levels >= 1 && levels <= kMaxStreamLevels && H >= 3;
}

cudaError_t adf_stream_pass(const float* src, float* dst, float* normals, int W, int H, int B, int levels,
                            const AdfStreamParams& p, cudaStream_t stream) {
    const int halo = ((levels + (normals ? 1 : 0)) + 1) & ~1;   // even, so pairs align with the image
    const int SW = pick_strip(W, halo);
    const int TWs = SW - 2 * halo;
    dim3 grid((W + TWs - 1) / TWs, B);
    const int Wv = W, Hv = H, hv = halo;
    const AdfStreamParams pv = p;
    void* args[] = {(void*)&src, (void*)&dst, (void*)&normals, (void*)&Wv, (void*)&Hv, (void*)&hv, (void*)&pv};
    const StreamFn fn = stream_fns()[levels][p.scheme == PM_ADF_DIVERGENCE ? 1 : 0];
    return cudaLaunchKernel((const void*)fn, grid, dim3(SW / 2), args, stream_smem(levels, SW), stream);
}

}  // namespace pm
