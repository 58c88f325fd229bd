// adf.cu — Algorithm 1 of arXiv 2411.01919 on sm_100a:
// temporally blocked Perona–Malik diffusion (ℓ1-8) with the Sobel/normal
// stage (ℓ9-13) fused into the last pass.
//
// One CTA owns an output tile of TW x TH pixels of one frame.  It loads the
// tile plus an R-pixel halo (R = iterations of this pass, +1 when the normal
// stage is fused) into shared memory once, runs the pass's T Jacobi sweeps in
// shared memory on a region that shrinks by one pixel per sweep (ping-pong
// buffers), and writes the tile back: one HBM read and one write per pass
// instead of one per sweep.  Every cell update uses the same explicit _rn
// arithmetic, so the result is bitwise independent of T, tile shape and
// batch.
#include <cuda_runtime.h>
#include <float.h>
#include <stdint.h>

#include "common.cuh"
#include "internal.h"

namespace pm {

namespace {

constexpr int kThreads = 256;      // 32 x 8
constexpr int kSmemW = 128;        // smem row pitch (floats); TW = kSmemW - 2R
constexpr int kTileH = 32;         // output rows per CTA

struct AdfParams {
    float lam;        // gamma of Alg. 1
    float kc;         // -log2(e) / (4 kappa^2): c = 2^(kc * (2gx)^2 + (2gy)^2))
    float fx, fy, cx, cy;
};

// One Jacobi update of Alg. 1 ℓ4-6 at a valid centre value I with the four
// neighbour values (zero-flux rule Q4: invalid or out-of-image neighbours
// were stored as non-positive values and are replaced by the centre).
// dN = N - I etc.; gx2 = 2 gx = dE - dW, gy2 = 2 gy = dS - dN;
// c = exp(-(gx^2 + gy^2)/k^2) = 2^(kc (gx2^2 + gy2^2)); lap = (dN+dS)+(dE+dW).
PM_DEVINL float adf_update(float I, float n, float s, float w, float e, float lam, float kc) {
    const float dn = valid_depth(n) ? __fsub_rn(n, I) : 0.0f;
    const float ds = valid_depth(s) ? __fsub_rn(s, I) : 0.0f;
    const float dw = valid_depth(w) ? __fsub_rn(w, I) : 0.0f;
    const float de = valid_depth(e) ? __fsub_rn(e, I) : 0.0f;
    const float gx2 = __fsub_rn(de, dw);
    const float gy2 = __fsub_rn(ds, dn);
    const float g2 = __fmaf_rn(gx2, gx2, __fmul_rn(gy2, gy2));
    const float c = ex2_approx(__fmul_rn(g2, kc));
    const float lap = __fadd_rn(__fadd_rn(dn, ds), __fadd_rn(de, dw));
    return __fmaf_rn(__fmul_rn(lam, c), lap, I);
}

// Sobel (1/8-normalised, clamp-to-edge) + geometric normal (Eq. 2 read as
// Q7): m = (fx Gx, fy Gy, -(Z + (u-cx) Gx + (v-cy) Gy)), n = m/|m|; (0,0,0)
// if any window pixel is invalid (Q9).  z[a][b] = window row a, column b.
PM_DEVINL float3 sobel_normal(const float z[3][3], float u, float v, const AdfParams& p) {
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
    const float mx = __fmul_rn(p.fx, gx);
    const float my = __fmul_rn(p.fy, gy);
    const float mz = -__fmaf_rn(__fsub_rn(v, p.cy), gy, __fmaf_rn(__fsub_rn(u, p.cx), gx, z[1][1]));
    const float ss = __fmaf_rn(mx, mx, __fmaf_rn(my, my, __fmul_rn(mz, mz)));
    if (!(ss > 0.0f) || !(ss <= FLT_MAX)) return make_float3(0.f, 0.f, 0.f);
    const float inv = rsqrtf(ss);
    return make_float3(mx * inv, my * inv, mz * inv);
}

// One pass: `iters` sweeps on a tile; halo R = iters + (fuse ? 1 : 0).
//   src [B][H][W] -> dst [B][H][W] (if write_depth) and normals [B][3][H][W].
__global__ void __launch_bounds__(kThreads)
adf_pass_kernel(const float* __restrict__ src, float* __restrict__ dst,
                float* __restrict__ normals, int W, int H, int iters, int R,
                int write_depth, AdfParams p) {
    extern __shared__ float smem[];
    const int TW = kSmemW - 2 * R;
    const int SH = kTileH + 2 * R;
    float* buf0 = smem;
    float* buf1 = smem + kSmemW * SH;
    const size_t frame = blockIdx.z;
    const size_t HW = (size_t)H * W;
    const float* in = src + frame * HW;
    const int x0 = blockIdx.x * TW - R;     // image coords of smem (0, 0)
    const int y0 = blockIdx.y * kTileH - R;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;

    // load tile + halo; out-of-image cells get 0 (invalid => zero flux)
    for (int y = ty; y < SH; y += kThreads / 32) {
        const int gy = y0 + y;
        const bool rowok = gy >= 0 && gy < H;
        for (int x = tx; x < kSmemW; x += 32) {
            const int gx = x0 + x;
            float v = 0.0f;
            if (rowok && gx >= 0 && gx < W) v = __ldg(in + (size_t)gy * W + gx);
            buf0[y * kSmemW + x] = v;
        }
    }
    __syncthreads();

    float* cur = buf0;
    float* nxt = buf1;
    for (int t = 1; t <= iters; ++t) {
        for (int y = t + ty; y < SH - t; y += kThreads / 32) {
            const float* row = cur + y * kSmemW;
            float* orow = nxt + y * kSmemW;
            for (int x = t + tx; x < kSmemW - t; x += 32) {
                const float I = row[x];
                float o = I;
                if (valid_depth(I))
                    o = adf_update(I, row[x - kSmemW], row[x + kSmemW], row[x - 1], row[x + 1], p.lam, p.kc);
                orow[x] = o;
            }
        }
        __syncthreads();
        float* tmp = cur; cur = nxt; nxt = tmp;
    }

    // write the tile (and its normals)
    const int ox = blockIdx.x * TW, oy = blockIdx.y * kTileH;
    float* out = dst + frame * HW;
    float* nrm = normals ? normals + frame * 3 * HW : nullptr;
    for (int y = ty; y < kTileH; y += kThreads / 32) {
        const int gy = oy + y;
        if (gy >= H) break;
        for (int x = tx; x < TW; x += 32) {
            const int gx = ox + x;
            if (gx >= W) break;
            const int sx = x + R, sy = y + R;
            if (write_depth) out[(size_t)gy * W + gx] = cur[sy * kSmemW + sx];
            if (nrm) {
                // clamp-to-edge window in image coords, mapped to smem coords
                const int xm = max(gx - 1, 0) - x0, xp = min(gx + 1, W - 1) - x0;
                const int ym = max(gy - 1, 0) - y0, yp = min(gy + 1, H - 1) - y0;
                const int xs[3] = {xm, sx, xp}, ys[3] = {ym, sy, yp};
                float z[3][3];
#pragma unroll
                for (int a = 0; a < 3; ++a)
#pragma unroll
                    for (int b = 0; b < 3; ++b) z[a][b] = cur[ys[a] * kSmemW + xs[b]];
                const float3 n = sobel_normal(z, (float)gx, (float)gy, p);
                const size_t o = (size_t)gy * W + gx;
                nrm[o] = n.x;
                nrm[HW + o] = n.y;
                nrm[2 * HW + o] = n.z;
            }
        }
    }
}

size_t pass_smem_bytes(int R) { return sizeof(float) * 2 * kSmemW * (kTileH + 2 * R); }

}  // namespace

constexpr int kMaxItersPerPass = 16;

cudaError_t adf_setup_attributes() {
    return cudaFuncSetAttribute(adf_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)pass_smem_bytes(kMaxItersPerPass + 1));
}

static cudaError_t launch_pass(const float* src, float* dst, float* normals, int W, int H, int B,
                               int iters, bool fuse, bool write_depth, const AdfParams& p,
                               cudaStream_t stream) {
    const int R = iters + (fuse ? 1 : 0);
    const int TW = kSmemW - 2 * R;
    dim3 grid((W + TW - 1) / TW, (H + kTileH - 1) / kTileH, B);
    adf_pass_kernel<<<grid, kThreads, pass_smem_bytes(R), stream>>>(src, dst, normals, W, H, iters, R,
                                                                     write_depth ? 1 : 0, p);
    return cudaGetLastError();
}

int adf_default_iters_per_pass() { return 4; }

cudaError_t adf_run(const float* in, float* out, float* normals, float* ws, int W, int H, int B,
                    const pm_intrinsics* K, float lam, float kappa, int iters, int iters_per_pass,
                    cudaStream_t stream) {
    AdfParams p;
    p.lam = lam;
    p.kc = (float)(-1.4426950408889634 / (4.0 * (double)kappa * (double)kappa));
    p.fx = K ? K->fx : 1.f;
    p.fy = K ? K->fy : 1.f;
    p.cx = K ? K->cx : 0.f;
    p.cy = K ? K->cy : 0.f;
    int T = iters_per_pass > 0 ? iters_per_pass : adf_default_iters_per_pass();
    if (T > kMaxItersPerPass) T = kMaxItersPerPass;
    if (iters == 0) {
        // N = 0: I_smooth = I; normals of the input
        return launch_pass(in, out, normals, W, H, B, 0, normals != nullptr, true, p, stream);
    }
    const int passes = (iters + T - 1) / T;
    const float* src = in;
    int done = 0;
    for (int k = 0; k < passes; ++k) {
        const int it = (iters - done) / (passes - k);   // near-equal split, sums to iters
        // ping-pong so that the last pass lands in `out`
        float* dst = (((passes - 1 - k) & 1) == 0) ? out : ws;
        const bool last = k == passes - 1;
        cudaError_t e = launch_pass(src, dst, last ? normals : nullptr, W, H, B, it,
                                    last && normals != nullptr, true, p, stream);
        if (e != cudaSuccess) return e;
        src = dst;
        done += it;
    }
    return cudaSuccess;
}

cudaError_t normals_run(const float* depth, float* normals, int W, int H, int B,
                        const pm_intrinsics* K, cudaStream_t stream) {
    AdfParams p{};
    p.fx = K->fx; p.fy = K->fy; p.cx = K->cx; p.cy = K->cy;
    return launch_pass(depth, nullptr, normals, W, H, B, 0, true, false, p, stream);
}

}  // namespace pm
