/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded CPU implementation of the hot path of
 * arXiv 2411.01919 ("real-time planar semantic mapping"): Algorithm 1
 * (anisotropic diffusion + normals) and Algorithm 2 (RANSAC plane fitting).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path
 * (paper_2411_01919_b200/) never links, imports or calls it, and this file
 * shares no code, header or constant table with the CUDA path.
 *
 * Citations: "P:n" = PAPER.md line n, "S:n" = SPEC.md line n (the
 * reference text), "Qk" = reading k of DESIGN.md §3 / SURVEY §8(c).
 *
 * Precision: ADF and normals in fp64 (rounded to f32 once at the end).
 * RANSAC decisions (distances, inlier counts) are taken in f32 with the
 * operation sequence DESIGN.md §3 prescribes, because the kernel takes them in
 * f32 and an integer decided by floating point must be decided in the same
 * precision on both sides; the least-squares refit is fp64.
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math (no FMA contraction; the
 * only fused multiply-adds are the explicit fmaf() calls below).
 *
 * Parity pins: see tests/test_oracle_*.py.  Every exported function has at
 * least one pin except where a comment says "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_API __attribute__((visibility("default")))

/* ------------------------------------------------------------------------ */
/* Depth validity.  The paper is silent (Q4); sensor convention S:69 "0 =
 * invalid", plus non-finite values.                                          */
static int orc_valid_f(float z) { return z > 0.0f && isfinite(z); }
static int orc_valid_d(double z) { return z > 0.0 && isfinite(z); }

enum { ORC_ADF_ALG1 = 0, ORC_ADF_DIVERGENCE = 1 };
enum { ORC_NORMALS_GEOMETRIC = 0, ORC_NORMALS_AS_PRINTED = 1 };

/* ------------------------------------------------------------------------ */
/* Algorithm 1, lines 1-8: anisotropic diffusion.
 *   ℓ1  I_smooth <- I
 *   ℓ2  for i = 1..N
 *   ℓ3    for each pixel p (parallel  -> Jacobi, Q2)
 *   ℓ4      compute grad I at p      (central differences, Q3)
 *   ℓ5      c_p = exp(-(|grad I_p| / k)^2)
 *   ℓ6      I_p <- I_p + gamma * c_p * lap(I_p)   (5-point Laplacian)
 * Boundary / invalid depth (Q4): an out-of-image or invalid neighbour takes
 * the centre pixel's value (zero flux); invalid pixels never change.
 * in/out: f32 [H][W] metres.  Computes in double, rounds once at the end.
 * scheme ORC_ADF_DIVERGENCE: Eq. 1 as the 4-flux Perona-Malik scheme instead
 * (NEXT-1; same zero-flux rule).
 * Returns 0, or -1 on bad arguments / allocation failure.                   */
ORC_API int orc_adf_ex(const float* in, float* out, int W, int H,
                       double lambda, double kappa, int iters, int scheme)
{
    if (!in || !out || W < 1 || H < 1 || iters < 0 || !(kappa > 0)) return -1;
    size_t n = (size_t)W * H;
    double* I = (double*)malloc(n * sizeof(double));
    double* J = (double*)malloc(n * sizeof(double));
    unsigned char* valid = (unsigned char*)malloc(n);
    if (!I || !J || !valid) { free(I); free(J); free(valid); return -1; }
    for (size_t p = 0; p < n; ++p) {
        valid[p] = (unsigned char)orc_valid_f(in[p]);   /* fixed from the input */
        I[p] = valid[p] ? (double)in[p] : 0.0;
    }
    const double k2 = kappa * kappa;
    for (int it = 0; it < iters; ++it) {                     /* ℓ2 */
        for (int v = 0; v < H; ++v) {
            for (int u = 0; u < W; ++u) {                    /* ℓ3 */
                size_t p = (size_t)v * W + u;
                if (!valid[p]) { J[p] = I[p]; continue; }
                double c0 = I[p];
                double vn = (v > 0     && valid[p - W]) ? I[p - W] : c0;
                double vs = (v < H - 1 && valid[p + W]) ? I[p + W] : c0;
                double vw = (u > 0     && valid[p - 1]) ? I[p - 1] : c0;
                double ve = (u < W - 1 && valid[p + 1]) ? I[p + 1] : c0;
                if (scheme == ORC_ADF_DIVERGENCE) {
                    /* Eq. 1 discretised as the classic 4-flux
                     * Perona-Malik scheme: I += lambda sum_d c(|grad_d I|) grad_d I,
                     * grad_d I = I_d - I_p, c(x) = exp(-(x/k)^2) (Q1) */
                    double dn = vn - c0, ds = vs - c0, dw = vw - c0, de = ve - c0;
                    J[p] = c0 + lambda * (exp(-dn * dn / k2) * dn + exp(-ds * ds / k2) * ds +
                                          exp(-dw * dw / k2) * dw + exp(-de * de / k2) * de);
                } else {
                    double gx = 0.5 * (ve - vw);             /* ℓ4 */
                    double gy = 0.5 * (vs - vn);
                    double c = exp(-(gx * gx + gy * gy) / k2);   /* ℓ5 */
                    double lap = (vn + vs + ve + vw) - 4.0 * c0;
                    J[p] = c0 + lambda * c * lap;            /* ℓ6 */
                }
            }
        }
        double* t = I; I = J; J = t;                         /* Jacobi swap */
    }
    for (size_t p = 0; p < n; ++p)
        out[p] = valid[p] ? (float)I[p] : in[p];             /* invalid: bitwise copy */
    free(I); free(J); free(valid);
    return 0;
}

ORC_API int orc_adf(const float* in, float* out, int W, int H,
                    double lambda, double kappa, int iters)
{
    return orc_adf_ex(in, out, W, H, lambda, kappa, iters, ORC_ADF_ALG1);
}

/* ------------------------------------------------------------------------ */
/* Algorithm 1, lines 9-13 and Eq. 2: per-pixel
 * normal from Sobel gradients and the intrinsics K, read geometrically (Q7):
 *   Gx, Gy = 3x3 Sobel of the depth Z, normalised by 1/8 (Q8), clamp-to-edge;
 *   m = dP/du x dP/dv for P(u,v) = Z(u,v) K^-1 [u v 1]^T, scaled by fx fy / Z:
 *   m = ( fx Gx, fy Gy, -(Z + (u-cx) Gx + (v-cy) Gy) ),  n = m / |m|  (ℓ12).
 * Invalid marker (Q9): n = (0,0,0) if any pixel of the clamped 3x3 window is
 * invalid.  mode ORC_NORMALS_AS_PRINTED: Eq. 2 literally, n = -K^-1[Gx,Gy,1]^T
 * normalised (NEXT-1; not a geometric normal, Q7).
 * depth: [H][W] double; out: [3][H][W] double (SoA).                        */
ORC_API int orc_normals_f64_ex(const double* D, int W, int H,
                               double fx, double fy, double cx, double cy, int mode,
                               double* out)
{
    if (!D || !out || W < 1 || H < 1) return -1;
    size_t n = (size_t)W * H;
    for (int v = 0; v < H; ++v) {
        for (int u = 0; u < W; ++u) {
            int um = u > 0 ? u - 1 : 0, up = u < W - 1 ? u + 1 : W - 1;
            int vm = v > 0 ? v - 1 : 0, vp = v < H - 1 ? v + 1 : H - 1;
#define Z(vv, uu) D[(size_t)(vv) * W + (uu)]
            int ok = 1;
            int rows[3] = {vm, v, vp}, cols[3] = {um, u, up};
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b)
                    if (!orc_valid_d(Z(rows[a], cols[b]))) ok = 0;
            size_t p = (size_t)v * W + u;
            if (!ok) { out[p] = 0.0; out[n + p] = 0.0; out[2 * n + p] = 0.0; continue; }
            double gx = ((Z(vm, up) - Z(vm, um)) + 2.0 * (Z(v, up) - Z(v, um))
                         + (Z(vp, up) - Z(vp, um))) / 8.0;
            double gy = ((Z(vp, um) - Z(vm, um)) + 2.0 * (Z(vp, u) - Z(vm, u))
                         + (Z(vp, up) - Z(vm, up))) / 8.0;
            double z = Z(v, u);
#undef Z
            double mx, my, mz;
            if (mode == ORC_NORMALS_AS_PRINTED) {
                /* Eq. 2 / Alg. 1 ℓ11 taken literally: n = -K^-1 [Gx, Gy, 1]^T */
                mx = -(gx - cx) / fx; my = -(gy - cy) / fy; mz = -1.0;
            } else {
                mx = fx * gx; my = fy * gy;
                mz = -(z + ((double)u - cx) * gx + ((double)v - cy) * gy);
            }
            double len = sqrt(mx * mx + my * my + mz * mz);
            if (!(len > 0.0) || !isfinite(len)) { out[p] = 0.0; out[n + p] = 0.0; out[2 * n + p] = 0.0; continue; }
            out[p] = mx / len; out[n + p] = my / len; out[2 * n + p] = mz / len;
        }
    }
    return 0;
}

ORC_API int orc_normals_f64(const double* D, int W, int H,
                            double fx, double fy, double cx, double cy, double* out)
{
    return orc_normals_f64_ex(D, W, H, fx, fy, cx, cy, ORC_NORMALS_GEOMETRIC, out);
}

/* f32-depth entry (the ABI's input type): promotes to double, then as above. */
ORC_API int orc_normals_ex(const float* depth, int W, int H,
                           double fx, double fy, double cx, double cy, int mode, double* out)
{
    if (!depth) return -1;
    size_t n = (size_t)W * H;
    double* D = (double*)malloc(n * sizeof(double));
    if (!D) return -1;
    for (size_t p = 0; p < n; ++p) D[p] = (double)depth[p];
    int rc = orc_normals_f64_ex(D, W, H, fx, fy, cx, cy, mode, out);
    free(D);
    return rc;
}

ORC_API int orc_normals(const float* depth, int W, int H,
                        double fx, double fy, double cx, double cy, double* out)
{
    return orc_normals_ex(depth, W, H, fx, fy, cx, cy, ORC_NORMALS_GEOMETRIC, out);
}

/* Sobel gradients alone (the Gx, Gy of Alg. 1 ℓ10), same convention as above;
 * no validity masking.  out: [2][H][W].                                     */
ORC_API int orc_sobel_f64(const double* D, int W, int H, double* out)
{
    if (!D || !out || W < 1 || H < 1) return -1;
    size_t n = (size_t)W * H;
    for (int v = 0; v < H; ++v)
        for (int u = 0; u < W; ++u) {
            int um = u > 0 ? u - 1 : 0, up = u < W - 1 ? u + 1 : W - 1;
            int vm = v > 0 ? v - 1 : 0, vp = v < H - 1 ? v + 1 : H - 1;
#define Z(vv, uu) D[(size_t)(vv) * W + (uu)]
            out[(size_t)v * W + u] = ((Z(vm, up) - Z(vm, um)) + 2.0 * (Z(v, up) - Z(v, um))
                                      + (Z(vp, up) - Z(vp, um))) / 8.0;
            out[n + (size_t)v * W + u] = ((Z(vp, um) - Z(vm, um)) + 2.0 * (Z(vp, u) - Z(vm, u))
                                          + (Z(vp, up) - Z(vm, up))) / 8.0;
#undef Z
        }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon et al., SC'11 "Parallel random numbers: as easy as
 * 1, 2, 3"): the counter-based RNG keyed by (seed, region, hypothesis,
 * frame) that north_star names for RANSAC sampling (Q17).  Pinned by the
 * Random123 known-answer vectors (tests/golden/philox4x32_10_kat.txt).      */
static void orc_mulhilo32(uint32_t a, uint32_t b, uint32_t* hi, uint32_t* lo)
{
    uint64_t p = (uint64_t)a * (uint64_t)b;
    *hi = (uint32_t)(p >> 32);
    *lo = (uint32_t)p;
}

ORC_API void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint32_t hi0, lo0, hi1, lo1;
        orc_mulhilo32(0xD2511F53u, c0, &hi0, &lo0);
        orc_mulhilo32(0xCD9E8D57u, c2, &hi1, &lo1);
        uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Alg. 2 ℓ6 "Select random subset of 3 points", uniform without
 * replacement (Q17): three distinct indices in [0, n) from three u32 draws by
 * multiply-high scaling and skip-insertion.  Requires n >= 3.               */
ORC_API void orc_sample_triple(uint32_t r0, uint32_t r1, uint32_t r2, uint32_t n, uint32_t idx[3])
{
    uint32_t i0 = (uint32_t)(((uint64_t)r0 * n) >> 32);
    uint32_t i1 = (uint32_t)(((uint64_t)r1 * (n - 1)) >> 32);
    if (i1 >= i0) i1++;
    uint32_t a = i0 < i1 ? i0 : i1, b = i0 < i1 ? i1 : i0;
    uint32_t i2 = (uint32_t)(((uint64_t)r2 * (n - 2)) >> 32);
    if (i2 >= a) i2++;
    if (i2 >= b) i2++;
    idx[0] = i0; idx[1] = i1; idx[2] = i2;
}

/* Test-mode sampler ENUMERATE: hypothesis h is the h-th 3-combination
 * {c0 < c1 < c2} of [0, n) in colexicographic order (pin P11: exhaustive
 * search).  Returns 0 when h >= C(n,3).                                     */
static uint64_t orc_binom(uint64_t n, uint64_t k)
{
    if (k > n) return 0;
    uint64_t r = 1;
    for (uint64_t i = 1; i <= k; ++i) r = r * (n - k + i) / i;
    return r;
}

ORC_API int orc_colex_unrank3(uint64_t h, uint32_t n, uint32_t idx[3])
{
    if (h >= orc_binom(n, 3)) return 0;
    uint32_t c2 = 2;
    while (orc_binom(c2 + 1, 3) <= h) c2++;
    h -= orc_binom(c2, 3);
    uint32_t c1 = 1;
    while (orc_binom(c1 + 1, 2) <= h) c1++;
    h -= orc_binom(c1, 2);
    idx[0] = (uint32_t)h; idx[1] = c1; idx[2] = c2;
    return 1;
}

/* ------------------------------------------------------------------------ */
/* Alg. 2 ℓ3 "Convert depth values to 3D points P using K", pinhole
 * model (Q24).  f32, in this exact order:
 *   X = (((float)u - cx) * (1/fx)) * z,  Y = (((float)v - cy) * (1/fy)) * z,  Z = z */
ORC_API void orc_deproject(int u, int v, float z, float fx, float fy, float cx, float cy, float P[3])
{
    float ifx = 1.0f / fx, ify = 1.0f / fy;
    P[0] = (((float)u - cx) * ifx) * z;
    P[1] = (((float)v - cy) * ify) * z;
    P[2] = z;
}

/* Alg. 2 ℓ7 "Fit plane model to these points".  f32 in
 * this exact order (no contraction).  Plane n.X + d = 0, |n| = 1, d >= 0
 * (camera on the front side).  Returns 0 for a collinear sample (Q18):
 * !(|e1 x e2|^2 > 1e-12 |e1|^2 |e2|^2).                                     */
ORC_API int orc_plane_from_3pts(const float p0[3], const float p1[3], const float p2[3], float plane[4])
{
    float e1x = p1[0] - p0[0], e1y = p1[1] - p0[1], e1z = p1[2] - p0[2];
    float e2x = p2[0] - p0[0], e2y = p2[1] - p0[1], e2z = p2[2] - p0[2];
    float cxv = e1y * e2z - e1z * e2y;
    float cyv = e1z * e2x - e1x * e2z;
    float czv = e1x * e2y - e1y * e2x;
    float s2 = (cxv * cxv + cyv * cyv) + czv * czv;
    float l1 = (e1x * e1x + e1y * e1y) + e1z * e1z;
    float l2 = (e2x * e2x + e2y * e2y) + e2z * e2z;
    if (!(s2 > 1e-12f * (l1 * l2))) return 0;
    float len = sqrtf(s2);
    float nx = cxv / len, ny = cyv / len, nz = czv / len;
    float d = -((nx * p0[0] + ny * p0[1]) + nz * p0[2]);
    if (d < 0.0f) { nx = -nx; ny = -ny; nz = -nz; d = -d; }
    plane[0] = nx; plane[1] = ny; plane[2] = nz; plane[3] = d;
    return 1;
}

/* Eq. 3 rho and Alg. 2 ℓ10: point-plane distance |n.p + d|,
 * f32, explicit fused chain fmaf(nz, Z, fmaf(ny, Y, fmaf(nx, X, d))).        */
ORC_API float orc_point_plane_dist(const float plane[4], const float P[3])
{
    return fabsf(fmaf(plane[2], P[2], fmaf(plane[1], P[1], fmaf(plane[0], P[0], plane[3]))));
}

/* ------------------------------------------------------------------------ */
/* Symmetric 3x3 eigen-decomposition by cyclic Jacobi rotations (textbook,
 * e.g. Golub & Van Loan §8.5), until the off-diagonal norm is below
 * 1e-15 * trace.  Returns the unit eigenvector of the smallest eigenvalue.   */
static void orc_jacobi3_smallest(const double M[3][3], double vec[3])
{
    double a[3][3], V[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
    memcpy(a, M, sizeof(a));
    double tr = fabs(a[0][0]) + fabs(a[1][1]) + fabs(a[2][2]);
    for (int sweep = 0; sweep < 64; ++sweep) {
        double off = sqrt(a[0][1] * a[0][1] + a[0][2] * a[0][2] + a[1][2] * a[1][2]);
        if (off <= 1e-15 * tr || off == 0.0) break;
        static const int PQ[3][2] = {{0, 1}, {0, 2}, {1, 2}};
        for (int k = 0; k < 3; ++k) {
            int p = PQ[k][0], q = PQ[k][1];
            if (a[p][q] == 0.0) continue;
            double theta = (a[q][q] - a[p][p]) / (2.0 * a[p][q]);
            double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
            double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
            /* A <- J^T A J with J the (p,q) rotation */
            for (int i = 0; i < 3; ++i) {
                double aip = a[i][p], aiq = a[i][q];
                a[i][p] = c * aip - s * aiq;
                a[i][q] = s * aip + c * aiq;
            }
            for (int i = 0; i < 3; ++i) {
                double api = a[p][i], aqi = a[q][i];
                a[p][i] = c * api - s * aqi;
                a[q][i] = s * api + c * aqi;
            }
            for (int i = 0; i < 3; ++i) {
                double vip = V[i][p], viq = V[i][q];
                V[i][p] = c * vip - s * viq;
                V[i][q] = s * vip + c * viq;
            }
        }
    }
    int m = 0;
    if (a[1][1] < a[m][m]) m = 1;
    if (a[2][2] < a[m][m]) m = 2;
    double nrm = sqrt(V[0][m] * V[0][m] + V[1][m] * V[1][m] + V[2][m] * V[2][m]);
    vec[0] = V[0][m] / nrm; vec[1] = V[1][m] / nrm; vec[2] = V[2][m] / nrm;
}

/* Least-squares (total least squares) refit over an inlier set (north_star
 * "least-squares refit"; S:318 / S:342; reading Q19): o = first point,
 * centroid = o + mean(p - o); M = sum (p - c)(p - c)^T (second pass);
 * normal = smallest eigenvector of M; d = -n.c, oriented so d >= 0.
 * pts: [n][3] double.  out: n[3], d, centroid[3].  Returns 0 if n < 1.      */
ORC_API int orc_refit_plane(const double* pts, int n, double out[7])
{
    if (n < 1) return 0;
    double o[3] = {pts[0], pts[1], pts[2]}, s[3] = {0, 0, 0};
    for (int i = 0; i < n; ++i)
        for (int k = 0; k < 3; ++k) s[k] += pts[3 * i + k] - o[k];
    double c[3];
    for (int k = 0; k < 3; ++k) c[k] = o[k] + s[k] / n;
    double M[3][3] = {{0}};
    for (int i = 0; i < n; ++i) {
        double q[3] = {pts[3 * i] - c[0], pts[3 * i + 1] - c[1], pts[3 * i + 2] - c[2]};
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) M[a][b] += q[a] * q[b];
    }
    double nv[3];
    orc_jacobi3_smallest(M, nv);
    double d = -(nv[0] * c[0] + nv[1] * c[1] + nv[2] * c[2]);
    if (d < 0) { nv[0] = -nv[0]; nv[1] = -nv[1]; nv[2] = -nv[2]; d = -d; }
    out[0] = nv[0]; out[1] = nv[1]; out[2] = nv[2]; out[3] = d;
    out[4] = c[0]; out[5] = c[1]; out[6] = c[2];
    return 1;
}

/* ------------------------------------------------------------------------ */
/* Algorithm 2, batched over every labelled region of one frame.
 *   ℓ1   for each region r (a label image replaces the polygon contours C)
 *   ℓ2-3 P <- valid labelled pixels of r in RASTER order, deprojected (f32)
 *   ℓ5   for h = 0..n_hyp-1
 *   ℓ6-7   3 distinct points (Philox keyed {h, r, frame, 0} / {seed lo, hi},
 *          or ENUMERATE) -> f32 plane; collinear -> hypothesis invalid (-1)
 *   ℓ9-13  for every point: d = |n.p + d|; inliers += (d < tau) (strict, Q14);
 *          error += d  (fixed point: rint(min(d, 64) * 2^24), exact, Q12)
 *   ℓ14-17 best = argmax inliers, ties -> lowest h (SELECT_COUNT, Q11), or
 *          argmin error, ties -> lowest h (SELECT_ERROR, the paper as printed)
 *   refit  fp64 least squares over S = {i : d_best(i) < tau} (Q19)
 *   ℓ19  status = OK iff 10 * inliers > 9 * n (Q15), else REJECTED;
 *        TOO_FEW if n < 3; DEGENERATE if no hypothesis is valid.
 * Outputs per region r:
 *   out_f64[r*7 ..]  n[3], d, centroid[3]           (double)
 *   out_i32[r*4 ..]  inliers, n_points, best_hyp, status
 *   out_errq[r]      fixed-point error of the winner (units 2^-24 m)
 *   counts  [r*n_hyp + h] (nullable) inlier count per hypothesis (-1 invalid)
 *   errq_all[r*n_hyp + h] (nullable) fixed-point error per hypothesis        */
enum { ORC_OK = 0, ORC_REJECTED = 1, ORC_TOO_FEW = 2, ORC_DEGENERATE = 3 };
enum { ORC_SAMPLER_PHILOX = 0, ORC_SAMPLER_ENUMERATE = 1 };
/* *_EARLY: "This process iterates until the maximum iterations are reached or
 * a satisfactory model is found", reading "satisfactory" as the
 * acceptance gate of ℓ19 (inliers / points > 0.9): the hypothesis loop stops
 * after the first h at which the best model so far passes it (Q20). */
enum { ORC_SELECT_COUNT = 0, ORC_SELECT_ERROR = 1, ORC_SELECT_COUNT_EARLY = 2, ORC_SELECT_ERROR_EARLY = 3 };

ORC_API int orc_ransac(const float* depth, const int32_t* labels, int W, int H,
                       float fx, float fy, float cx, float cy,
                       int n_regions, int n_hyp, float tau, uint64_t seed, uint32_t frame_id,
                       int sampler, int select_mode,
                       double* out_f64, int32_t* out_i32, uint64_t* out_errq,
                       int32_t* counts, uint64_t* errq_all)
{
    if (!depth || !labels || W < 1 || H < 1 || n_regions < 0 || n_hyp < 1) return -1;
    size_t npx = (size_t)W * H;
    float ifx = 1.0f / fx, ify = 1.0f / fy;
    float* P = (float*)malloc(npx * 3 * sizeof(float));
    int32_t* cnt = (int32_t*)malloc((size_t)n_hyp * sizeof(int32_t));
    uint64_t* err = (uint64_t*)malloc((size_t)n_hyp * sizeof(uint64_t));
    double* S = (double*)malloc(npx * 3 * sizeof(double));
    if (!P || !cnt || !err || !S) { free(P); free(cnt); free(err); free(S); return -1; }
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};

    for (int r = 0; r < n_regions; ++r) {
        /* ℓ2-3: raster-order gather + deprojection */
        uint32_t n = 0;
        for (int v = 0; v < H; ++v)
            for (int u = 0; u < W; ++u) {
                size_t p = (size_t)v * W + u;
                float z = depth[p];
                if (labels[p] != r || !orc_valid_f(z)) continue;
                P[3 * n + 0] = (((float)u - cx) * ifx) * z;
                P[3 * n + 1] = (((float)v - cy) * ify) * z;
                P[3 * n + 2] = z;
                n++;
            }
        double* of = out_f64 + (size_t)r * 7;
        int32_t* oi = out_i32 + (size_t)r * 4;
        for (int k = 0; k < 7; ++k) of[k] = 0.0;
        oi[0] = 0; oi[1] = (int32_t)n; oi[2] = -1; oi[3] = ORC_TOO_FEW;
        out_errq[r] = 0;
        if (counts) for (int h = 0; h < n_hyp; ++h) counts[(size_t)r * n_hyp + h] = -1;
        if (errq_all) for (int h = 0; h < n_hyp; ++h) errq_all[(size_t)r * n_hyp + h] = 0;
        if (n < 3) continue;

        for (int h = 0; h < n_hyp; ++h) {                      /* ℓ5 */
            uint32_t idx[3];
            cnt[h] = -1; err[h] = 0;
            if (sampler == ORC_SAMPLER_ENUMERATE) {
                if (!orc_colex_unrank3((uint64_t)h, n, idx)) continue;
            } else {
                uint32_t ctr[4] = {(uint32_t)h, (uint32_t)r, frame_id, 0u}, rnd[4];
                orc_philox4x32_10(ctr, key, rnd);
                orc_sample_triple(rnd[0], rnd[1], rnd[2], n, idx);
            }
            float pl[4];
            if (!orc_plane_from_3pts(&P[3 * idx[0]], &P[3 * idx[1]], &P[3 * idx[2]], pl)) continue;
            int32_t c = 0;
            uint64_t e = 0;
            for (uint32_t i = 0; i < n; ++i) {                 /* ℓ9-13 */
                float dist = orc_point_plane_dist(pl, &P[3 * i]);
                c += (dist < tau);
                e += (uint64_t)rintf(fminf(dist, 64.0f) * 16777216.0f);
            }
            cnt[h] = c; err[h] = e;
        }
        if (counts) memcpy(counts + (size_t)r * n_hyp, cnt, (size_t)n_hyp * sizeof(int32_t));
        if (errq_all) memcpy(errq_all + (size_t)r * n_hyp, err, (size_t)n_hyp * sizeof(uint64_t));

        int best = -1;                                         /* ℓ14-17 */
        const int by_error = select_mode == ORC_SELECT_ERROR || select_mode == ORC_SELECT_ERROR_EARLY;
        const int early = select_mode == ORC_SELECT_COUNT_EARLY || select_mode == ORC_SELECT_ERROR_EARLY;
        for (int h = 0; h < n_hyp; ++h) {
            if (cnt[h] < 0) continue;
            if (best < 0) best = h;
            else if (by_error ? (err[h] < err[best]) : (cnt[h] > cnt[best])) best = h;
            if (early && (int64_t)10 * cnt[best] > (int64_t)9 * n) break;   /* satisfactory */
        }
        if (best < 0) { oi[3] = ORC_DEGENERATE; continue; }

        /* re-derive the winner's plane, collect its inliers S */
        uint32_t idx[3];
        if (sampler == ORC_SAMPLER_ENUMERATE) {
            orc_colex_unrank3((uint64_t)best, n, idx);
        } else {
            uint32_t ctr[4] = {(uint32_t)best, (uint32_t)r, frame_id, 0u}, rnd[4];
            orc_philox4x32_10(ctr, key, rnd);
            orc_sample_triple(rnd[0], rnd[1], rnd[2], n, idx);
        }
        float pl[4];
        orc_plane_from_3pts(&P[3 * idx[0]], &P[3 * idx[1]], &P[3 * idx[2]], pl);
        int ns = 0;
        for (uint32_t i = 0; i < n; ++i) {
            if (orc_point_plane_dist(pl, &P[3 * i]) < tau) {
                S[3 * ns + 0] = P[3 * i + 0]; S[3 * ns + 1] = P[3 * i + 1]; S[3 * ns + 2] = P[3 * i + 2];
                ns++;
            }
        }
        if (ns >= 3) {
            orc_refit_plane(S, ns, of);
        } else {
            /* refit impossible (tau below rounding): keep the 3-point model,
             * centroid = mean of the three sample points (Q19). */
            of[0] = pl[0]; of[1] = pl[1]; of[2] = pl[2]; of[3] = pl[3];
            for (int k = 0; k < 3; ++k)
                of[4 + k] = ((double)P[3 * idx[0] + k] + (double)P[3 * idx[1] + k] + (double)P[3 * idx[2] + k]) / 3.0;
        }
        oi[0] = cnt[best];
        oi[2] = best;
        oi[3] = ((int64_t)10 * cnt[best] > (int64_t)9 * n) ? ORC_OK : ORC_REJECTED;   /* ℓ19 */
        out_errq[r] = err[best];
    }
    free(P); free(cnt); free(err); free(S);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* NEXT-2: region labels from the normal image, the step the
 * paper places between Alg. 1 and Alg. 2: "edges are detected from the normal
 * vector image using the Canny edge detection algorithm. Subsequently,
 * contours are extracted from these edges".  Readings
 * (Q26-Q29): Canny runs on the 8-bit RGB normal image
 * c = rint((n + 1) * 127.5) (the visualisation of fig:ADF_ex), with
 * 3x3 Sobel, replicated borders, L2 magnitude, the channel of largest
 * magnitude per pixel, non-maximum suppression and 8-connected
 * hysteresis; pixels with an invalid normal are edges; the edge mask is
 * dilated by one pixel (3x3); regions = 4-connected components of non-edge
 * pixels with >= min_area pixels, numbered by descending size, ties
 * by smallest raster index, at most max_regions; others -1.       */

/* f32 normals [3][H][W] -> interleaved u8 [H][W][3]. */
ORC_API void orc_normals_to_u8(const float* nrm, int W, int H, uint8_t* img)
{
    size_t n = (size_t)W * H;
    for (size_t p = 0; p < n; ++p)
        for (int c = 0; c < 3; ++c) {
            float v = rintf((nrm[c * n + p] + 1.0f) * 127.5f);
            int q = (int)v;
            img[3 * p + c] = (uint8_t)(q < 0 ? 0 : (q > 255 ? 255 : q));
        }
}

/* Canny on an interleaved u8 image with C channels; edges [H][W] 0/255. */
ORC_API int orc_canny_u8(const uint8_t* img, int W, int H, int C, double low_thresh, double high_thresh,
                         uint8_t* edges)
{
    if (!img || !edges || W < 1 || H < 1 || C < 1) return -1;
    if (low_thresh > high_thresh) { double t = low_thresh; low_thresh = high_thresh; high_thresh = t; }
    /* L2 magnitude compared with squared thresholds, as integers */
    long long low = (long long)floor(low_thresh > 0 ? low_thresh * low_thresh : low_thresh);
    long long high = (long long)floor(high_thresh > 0 ? high_thresh * high_thresh : high_thresh);
    size_t n = (size_t)W * H;
    int* dx = (int*)malloc(n * sizeof(int));
    int* dy = (int*)malloc(n * sizeof(int));
    long long* mag = (long long*)malloc(n * sizeof(long long));
    unsigned char* cand = (unsigned char*)calloc(n, 1);   /* 1 = NMS survivor above low */
    int* stack = (int*)malloc(n * sizeof(int));
    if (!dx || !dy || !mag || !cand || !stack) { free(dx); free(dy); free(mag); free(cand); free(stack); return -1; }
#define PX(vv, uu, cc) ((int)img[(((size_t)(vv) * W) + (uu)) * C + (cc)])
    for (int v = 0; v < H; ++v)
        for (int u = 0; u < W; ++u) {
            int um = u > 0 ? u - 1 : 0, up = u < W - 1 ? u + 1 : W - 1;
            int vm = v > 0 ? v - 1 : 0, vp = v < H - 1 ? v + 1 : H - 1;
            long long best = -1;
            int bx = 0, by = 0;
            for (int c = 0; c < C; ++c) {
                int gx = (PX(vm, up, c) - PX(vm, um, c)) + 2 * (PX(v, up, c) - PX(v, um, c)) + (PX(vp, up, c) - PX(vp, um, c));
                int gy = (PX(vp, um, c) - PX(vm, um, c)) + 2 * (PX(vp, u, c) - PX(vm, u, c)) + (PX(vp, up, c) - PX(vm, up, c));
                long long m = (long long)gx * gx + (long long)gy * gy;
                if (m > best) { best = m; bx = gx; by = gy; }      /* first channel wins ties */
            }
            size_t p = (size_t)v * W + u;
            dx[p] = bx; dy[p] = by; mag[p] = best;
        }
#undef PX
    /* non-maximum suppression along the quantised gradient direction
     * (tan 22.5 deg in 15-bit fixed point); neighbours outside the image
     * count as 0 */
    const long long TG22 = (long long)(0.4142135623730950488016887242097 * (1 << 15) + 0.5);
#define MAG(vv, uu) (((vv) < 0 || (vv) >= H || (uu) < 0 || (uu) >= W) ? 0LL : mag[(size_t)(vv) * W + (uu)])
    for (int v = 0; v < H; ++v)
        for (int u = 0; u < W; ++u) {
            size_t p = (size_t)v * W + u;
            long long m = mag[p];
            if (!(m > low)) continue;
            long long xs = dx[p], ys = dy[p];
            long long x = xs < 0 ? -xs : xs, y = (ys < 0 ? -ys : ys) << 15;
            long long tg22x = x * TG22;
            int keep;
            if (y < tg22x) {
                keep = m > MAG(v, u - 1) && m >= MAG(v, u + 1);
            } else {
                long long tg67x = tg22x + (x << 16);
                if (y > tg67x) {
                    keep = m > MAG(v - 1, u) && m >= MAG(v + 1, u);
                } else {
                    int s = ((xs ^ ys) < 0) ? -1 : 1;
                    keep = m > MAG(v - 1, u - s) && m > MAG(v + 1, u + s);
                }
            }
            if (keep) cand[p] = 1;
        }
#undef MAG
    /* hysteresis: candidates 8-connected (through candidates) to a strong one */
    memset(edges, 0, n);
    int top = 0;
    for (size_t p = 0; p < n; ++p)
        if (cand[p] && mag[p] > high) { edges[p] = 255; stack[top++] = (int)p; }
    while (top > 0) {
        int p = stack[--top];
        int v = p / W, u = p % W;
        for (int dv = -1; dv <= 1; ++dv)
            for (int du = -1; du <= 1; ++du) {
                int vv = v + dv, uu = u + du;
                if ((dv == 0 && du == 0) || vv < 0 || vv >= H || uu < 0 || uu >= W) continue;
                size_t q = (size_t)vv * W + uu;
                if (cand[q] && !edges[q]) { edges[q] = 255; stack[top++] = (int)q; }
            }
    }
    free(dx); free(dy); free(mag); free(cand); free(stack);
    return 0;
}

/* Region labels from f32 normals [3][H][W] (see the block comment above).
 * labels [H][W] int32 (-1 = none), *n_regions = number of regions kept,
 * edges_out [H][W] (nullable): the final (dilated) edge mask 0/1.        */
ORC_API int orc_segment_regions(const float* nrm, int W, int H, double low, double high, int min_area,
                                int max_regions, int32_t* labels, int32_t* n_regions, uint8_t* edges_out)
{
    if (!nrm || !labels || !n_regions || W < 1 || H < 1) return -1;
    size_t n = (size_t)W * H;
    uint8_t* img = (uint8_t*)malloc(3 * n);
    uint8_t* e0 = (uint8_t*)malloc(n);
    uint8_t* e1 = (uint8_t*)malloc(n);
    int32_t* comp = (int32_t*)malloc(n * sizeof(int32_t));
    int* queue = (int*)malloc(n * sizeof(int));
    if (!img || !e0 || !e1 || !comp || !queue) { free(img); free(e0); free(e1); free(comp); free(queue); return -1; }
    orc_normals_to_u8(nrm, W, H, img);
    orc_canny_u8(img, W, H, 3, low, high, e0);
    for (size_t p = 0; p < n; ++p)                         /* invalid normal -> edge */
        if (nrm[p] == 0.0f && nrm[n + p] == 0.0f && nrm[2 * n + p] == 0.0f) e0[p] = 255;
    for (int v = 0; v < H; ++v)                            /* 3x3 dilation */
        for (int u = 0; u < W; ++u) {
            int any = 0;
            for (int dv = -1; dv <= 1 && !any; ++dv)
                for (int du = -1; du <= 1; ++du) {
                    int vv = v + dv, uu = u + du;
                    if (vv < 0 || vv >= H || uu < 0 || uu >= W) continue;
                    if (e0[(size_t)vv * W + uu]) { any = 1; break; }
                }
            e1[(size_t)v * W + u] = (uint8_t)any;
        }
    /* 4-connected components of non-edge pixels by BFS in raster order: the
     * component's seed is its smallest raster index */
    for (size_t p = 0; p < n; ++p) comp[p] = -1;
    int n_comp = 0;
    int cap = 1024;
    int* seed = (int*)malloc(cap * sizeof(int));
    int* size = (int*)malloc(cap * sizeof(int));
    for (size_t p0 = 0; p0 < n; ++p0) {
        if (e1[p0] || comp[p0] >= 0) continue;
        if (n_comp == cap) { cap *= 2; seed = (int*)realloc(seed, cap * sizeof(int)); size = (int*)realloc(size, cap * sizeof(int)); }
        int head = 0, tail = 0;
        queue[tail++] = (int)p0;
        comp[p0] = n_comp;
        while (head < tail) {
            int p = queue[head++];
            int v = p / W, u = p % W;
            const int nb[4][2] = {{-1, 0}, {1, 0}, {0, -1}, {0, 1}};
            for (int k = 0; k < 4; ++k) {
                int vv = v + nb[k][0], uu = u + nb[k][1];
                if (vv < 0 || vv >= H || uu < 0 || uu >= W) continue;
                size_t q = (size_t)vv * W + uu;
                if (!e1[q] && comp[q] < 0) { comp[q] = n_comp; queue[tail++] = (int)q; }
            }
        }
        seed[n_comp] = (int)p0;
        size[n_comp] = tail;
        n_comp++;
    }
    /* keep components >= min_area, order by (size desc, seed asc) */
    int* order = (int*)malloc((n_comp > 0 ? n_comp : 1) * sizeof(int));
    int* rank = (int*)malloc((n_comp > 0 ? n_comp : 1) * sizeof(int));
    int kept = 0;
    for (int c = 0; c < n_comp; ++c) if (size[c] >= min_area) order[kept++] = c;
    for (int i = 1; i < kept; ++i) {                       /* insertion sort (stable, small) */
        int c = order[i], j = i - 1;
        while (j >= 0 && (size[order[j]] < size[c] || (size[order[j]] == size[c] && seed[order[j]] > seed[c]))) {
            order[j + 1] = order[j];
            j--;
        }
        order[j + 1] = c;
    }
    for (int c = 0; c < n_comp; ++c) rank[c] = -1;
    if (kept > max_regions) kept = max_regions;
    for (int i = 0; i < kept; ++i) rank[order[i]] = i;
    for (size_t p = 0; p < n; ++p) labels[p] = comp[p] >= 0 ? rank[comp[p]] : -1;
    *n_regions = kept;
    if (edges_out) for (size_t p = 0; p < n; ++p) edges_out[p] = e1[p];
    free(img); free(e0); free(e1); free(comp); free(queue); free(seed); free(size); free(order); free(rank);
    return 0;
}

/* ======================================================================
 * NEXT-3: polygon glue between region labels and planes
 * ("contours are extracted from these edges and simplified into
 * polygons", Alg. 2 "for each detected contour c").
 * Readings Q35-Q39 in DESIGN.md.
 * ====================================================================== */

/* Q35: outer boundary of region `region` of a label image by Moore-neighbour
 * tracing.  Start: the region's first pixel in raster order, backtrack = its
 * west neighbour.  Neighbours are visited clockwise on screen (x right, y
 * down) starting just after the backtrack direction: E, SE, S, SW, W, NW, N,
 * NE.  Pixels outside the image or of another label are background.  Stops
 * when the walk is back at the start pixel about to repeat its first move
 * (Jacob's criterion).  Writes up to max_pts (x, y) pairs to pts, returns the
 * contour length (which may exceed max_pts: the output is then truncated), 0
 * when the region is empty.                                                  */
static const int ORC_MOORE[8][2] = {{1, 0}, {1, 1}, {0, 1}, {-1, 1}, {-1, 0}, {-1, -1}, {0, -1}, {1, -1}};

static int orc_in_region(const int32_t* labels, int W, int H, int x, int y, int region)
{
    return x >= 0 && y >= 0 && x < W && y < H && labels[(size_t)y * W + x] == region;
}

ORC_API int orc_trace_contour(const int32_t* labels, int W, int H, int region, int32_t* pts, int max_pts)
{
    size_t n = (size_t)W * H, s = n;
    for (size_t p = 0; p < n; ++p) if (labels[p] == region) { s = p; break; }
    if (s == n) return 0;
    int sx = (int)(s % W), sy = (int)(s / W);
    int len = 0;
    int px = sx, py = sy, bdir = 4;                  /* backtrack: west */
    int first_dir = -1;
    for (;;) {
        int found = -1;
        for (int k = 1; k <= 8; ++k) {
            int d = (bdir + k) & 7;
            if (orc_in_region(labels, W, H, px + ORC_MOORE[d][0], py + ORC_MOORE[d][1], region)) { found = d; break; }
        }
        if (found < 0) {                             /* isolated pixel */
            if (max_pts > 0) { pts[0] = px; pts[1] = py; }
            return 1;
        }
        if (px == sx && py == sy) {
            if (first_dir < 0) first_dir = found;
            else if (found == first_dir) break;      /* Jacob's stopping criterion */
        }
        if (len < max_pts) { pts[2 * len] = px; pts[2 * len + 1] = py; }
        len++;
        /* move; the new backtrack is the background neighbour examined just
         * before `found`, seen from the new pixel */
        int bd = (found + 7) & 7;                    /* previous direction examined (background) */
        int bx = px + ORC_MOORE[bd][0], by = py + ORC_MOORE[bd][1];
        px += ORC_MOORE[found][0];
        py += ORC_MOORE[found][1];
        int dxb = bx - px, dyb = by - py;
        for (int d = 0; d < 8; ++d) if (ORC_MOORE[d][0] == dxb && ORC_MOORE[d][1] == dyb) { bdir = d; break; }
    }
    return len;
}

/* Q36: Douglas-Peucker simplification of a closed contour of n integer
 * points.  Anchors: point 0 and the point farthest from it
 * (largest squared distance, ties -> lowest index); each open chain i..j is
 * split at the point k of largest distance to the LINE through p_i, p_j
 * (to p_i itself when p_i == p_j), ties -> lowest k, if that distance > eps.
 * Exact: |cross| compared among k, then cross^2 > eps^2 |p_j - p_i|^2 in
 * 128-bit integers with eps given in 1/16 px (eps16).  keep[n] (0/1) marks
 * the retained vertices; returns their number.                             */
static void orc_dp_rec(const int32_t* pts, int n, int i, int j, int64_t eps16, uint8_t* keep)
{
    /* chain i, i+1, ..., j (indices mod n) */
    int cnt = (j - i + n) % n;
    if (cnt < 2) return;
    int64_t ax = pts[2 * i], ay = pts[2 * i + 1], bx = pts[2 * (j % n)], by = pts[2 * (j % n) + 1];
    int64_t dx = bx - ax, dy = by - ay;
    int best = -1;
    unsigned __int128 bestv = 0;
    for (int s = 1; s < cnt; ++s) {
        int k = (i + s) % n;
        int64_t px = pts[2 * k] - ax, py = pts[2 * k + 1] - ay;
        unsigned __int128 v;
        if (dx == 0 && dy == 0) v = (unsigned __int128)(px * px + py * py);
        else {
            int64_t c = dx * py - dy * px;
            if (c < 0) c = -c;
            v = (unsigned __int128)c;
        }
        if (best < 0 || v > bestv) { best = k; bestv = v; }
    }
    /* distance > eps:  point case: d2 > eps^2 ; line case: cross^2 > eps^2 len^2 */
    unsigned __int128 lhs, rhs;
    if (dx == 0 && dy == 0) { lhs = bestv * 256u; rhs = (unsigned __int128)(eps16 * eps16); }
    else {
        lhs = bestv * bestv * 256u;
        rhs = (unsigned __int128)(eps16 * eps16) * (unsigned __int128)(dx * dx + dy * dy);
    }
    if (lhs > rhs) {
        keep[best] = 1;
        orc_dp_rec(pts, n, i, best, eps16, keep);
        orc_dp_rec(pts, n, best, j, eps16, keep);
    }
}

ORC_API int orc_simplify_dp(const int32_t* pts, int n, int eps16, uint8_t* keep)
{
    if (n <= 0) return 0;
    for (int k = 0; k < n; ++k) keep[k] = 0;
    keep[0] = 1;
    if (n == 1) return 1;
    int far = 0;
    int64_t fd = -1;
    for (int k = 1; k < n; ++k) {
        int64_t dx = pts[2 * k] - pts[0], dy = pts[2 * k + 1] - pts[1];
        int64_t d2 = dx * dx + dy * dy;
        if (d2 > fd) { fd = d2; far = k; }
    }
    keep[far] = 1;
    orc_dp_rec(pts, n, 0, far, eps16, keep);
    orc_dp_rec(pts, n, far, n, eps16, keep);   /* far .. n-1, 0 (index n == 0 mod n) */
    int m = 0;
    for (int k = 0; k < n; ++k) m += keep[k];
    return m;
}

/* Q37/Q38: rasterise polygons (integer vertices = pixel centres) to a label
 * image: pixel (x, y) is inside polygon q by the even-odd rule on its centre
 * with half-open crossings -- edge a->b counts iff (a.y > y) != (b.y > y) and
 * x < a.x + (y - a.y)(b.x - a.x)/(b.y - a.y), evaluated exactly in integers;
 * a pixel inside several polygons takes the lowest polygon index, -1 when in
 * none.  Polygon q has n_v[q] vertices at verts + 2*off[q].                 */
ORC_API int orc_rasterize_polygons(const int32_t* verts, const int32_t* off, const int32_t* n_v, int n_poly,
                                   int W, int H, int32_t* labels)
{
    for (size_t p = 0; p < (size_t)W * H; ++p) labels[p] = -1;
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x)
            for (int q = 0; q < n_poly; ++q) {
                const int32_t* v = verts + 2 * (size_t)off[q];
                int m = n_v[q], inside = 0;
                for (int e = 0; e < m; ++e) {
                    int64_t ax = v[2 * e], ay = v[2 * e + 1];
                    int64_t bx = v[2 * ((e + 1) % m)], by = v[2 * ((e + 1) % m) + 1];
                    if ((ay > y) == (by > y)) continue;
                    /* x < ax + (y - ay)(bx - ax)/(by - ay)  <=>  (x - ax)(by - ay) < (y - ay)(bx - ax) * sign */
                    int64_t lhs = (x - ax) * (by - ay), rhs = (y - ay) * (bx - ax);
                    int cross = (by > ay) ? (lhs < rhs) : (lhs > rhs);
                    if (cross) inside ^= 1;
                }
                if (inside) { labels[(size_t)y * W + x] = q; break; }
            }
    return 0;
}

/* Q39: lift pixel vertices onto a plane n.X + d = 0 along their camera rays
 * (S:327): r = ((u - cx)/fx, (v - cy)/fy, 1), X = -d/(n.r) r in fp64; NaN
 * when n.r == 0 or the intersection is behind the camera.                   */
ORC_API void orc_lift_vertices(const int32_t* uv, int n, const double plane[4], double fx, double fy, double cx,
                               double cy, double* X)
{
    for (int k = 0; k < n; ++k) {
        double r0 = ((double)uv[2 * k] - cx) / fx, r1 = ((double)uv[2 * k + 1] - cy) / fy, r2 = 1.0;
        double den = plane[0] * r0 + plane[1] * r1 + plane[2] * r2;
        double t = den != 0.0 ? -plane[3] / den : NAN;
        if (!(t > 0.0)) { X[3 * k] = X[3 * k + 1] = X[3 * k + 2] = NAN; continue; }
        X[3 * k] = t * r0; X[3 * k + 1] = t * r1; X[3 * k + 2] = t * r2;
    }
}
