// ransac.cu — Algorithm 2 of arXiv 2411.01919, batched over every
// region of every frame in five launches:
//   hyp      : one thread per (frame, region, hypothesis): Philox sample ->
//              3 points -> f32 plane (Alg. 2 ℓ6-7); also the plane pairs
//              (h, h + L) the packed scoring loop reads
//   score    : the hot loop (ℓ9-13).  The compacted points of a frame are cut
//              into fixed 4096-point chunks, one CTA per chunk regardless of
//              region sizes (load balance); a chunk's points are deprojected
//              once into shared memory and scored against every hypothesis
//              of the region(s) it overlaps: K hypotheses per lane in
//              registers, two per packed FFMA2 chain; counts reduced by
//              shuffles + shared memory and added to global integer counters
//              with one atomic per hypothesis (exact, order-free)
//   select   : one warp per (frame, region): argmax count (or argmin error),
//              ties -> lowest h (ℓ14-17)
//   refit    : 8192-point chunks, 1024 contiguous points per warp: the
//              winner's inliers recounted with the same f32 arithmetic, fp64
//              shifted moments, one slot per (chunk + region, warp) -- no
//              float atomics
//   finalize : one thread per (frame, region): slots summed in a fixed order,
//              3x3 eigen-solve, gate (ℓ19), pm_plane output.
// All plane and distance arithmetic uses explicit _rn intrinsics in the f32
// order DESIGN.md §3 fixes, so counts are bit-identical to the oracle's.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "common.cuh"
#include "internal.h"

namespace pm {

// fp64 refit moments of one (region, chunk) slot (declared in internal.h)
struct __align__(16) Sums {
    double s[3];     // sum of q = p - o over inliers (o = the region's first point)
    double m[6];     // sum of q q^T (xx, xy, xz, yy, yz, zz)
    unsigned long long err;   // sum over ALL points of rint(min(d, 64) * 2^24)
    int n;           // inliers
    int pad;
};

namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kScoreThreads = 256;
constexpr int kScoreChunk = 4096;     // points per scoring CTA (dynamic shared memory)
constexpr int kHB = 8;                // hypothesis array padding
constexpr int kRefitChunk = 8192;     // points per refit CTA
constexpr int kRefitWarps = kScoreThreads / 32;   // refit moment slots per (chunk + region)

struct SampleIdx { uint32_t i0, i1, i2; bool ok; };

// Alg. 2 ℓ6 (Q17): three distinct uniform indices in [0, n) from Philox draws.
PM_DEVINL SampleIdx sample_philox(uint32_t h, uint32_t r, uint32_t f, uint64_t seed, uint32_t n) {
    const U4 x = philox4x32_10(U4{h, r, f, 0u}, (uint32_t)seed, (uint32_t)(seed >> 32));
    uint32_t i0 = __umulhi(x.x, n);
    uint32_t i1 = __umulhi(x.y, n - 1);
    if (i1 >= i0) i1++;
    const uint32_t a = min(i0, i1), b = max(i0, i1);
    uint32_t i2 = __umulhi(x.z, n - 2);
    if (i2 >= a) i2++;
    if (i2 >= b) i2++;
    return SampleIdx{i0, i1, i2, true};
}

// Test sampler ENUMERATE: h -> h-th 3-combination of [0, n) in colex order.
PM_DEVINL uint64_t binom3(uint64_t m) { return m < 3 ? 0 : m * (m - 1) * (m - 2) / 6; }
PM_DEVINL uint64_t binom2(uint64_t m) { return m < 2 ? 0 : m * (m - 1) / 2; }
PM_DEVINL SampleIdx sample_colex(uint32_t h, uint32_t n) {
    uint64_t hh = h;
    uint32_t c2 = 2;
    while (binom3(c2 + 1) <= hh) c2++;
    hh -= binom3(c2);
    uint32_t c1 = 1;
    while (binom2(c1 + 1) <= hh) c1++;
    hh -= binom2(c1);
    return SampleIdx{(uint32_t)hh, c1, c2, c2 < n};
}

PM_DEVINL SampleIdx sample(int sampler, uint32_t h, uint32_t r, uint32_t f, uint64_t seed, uint32_t n) {
    return sampler == PM_SAMPLER_ENUMERATE ? sample_colex(h, n) : sample_philox(h, r, f, seed, n);
}

// Alg. 2 ℓ7: plane through three points, f32 in the fixed order; d >= 0.
// Returns false for a collinear sample: !(|e1 x e2|^2 > 1e-12 |e1|^2 |e2|^2).
PM_DEVINL bool plane_from_3pts(float3 p0, float3 p1, float3 p2, float4& pl) {
    const float e1x = __fsub_rn(p1.x, p0.x), e1y = __fsub_rn(p1.y, p0.y), e1z = __fsub_rn(p1.z, p0.z);
    const float e2x = __fsub_rn(p2.x, p0.x), e2y = __fsub_rn(p2.y, p0.y), e2z = __fsub_rn(p2.z, p0.z);
    const float cx = __fsub_rn(__fmul_rn(e1y, e2z), __fmul_rn(e1z, e2y));
    const float cy = __fsub_rn(__fmul_rn(e1z, e2x), __fmul_rn(e1x, e2z));
    const float cz = __fsub_rn(__fmul_rn(e1x, e2y), __fmul_rn(e1y, e2x));
    const float s2 = __fadd_rn(__fadd_rn(__fmul_rn(cx, cx), __fmul_rn(cy, cy)), __fmul_rn(cz, cz));
    const float l1 = __fadd_rn(__fadd_rn(__fmul_rn(e1x, e1x), __fmul_rn(e1y, e1y)), __fmul_rn(e1z, e1z));
    const float l2 = __fadd_rn(__fadd_rn(__fmul_rn(e2x, e2x), __fmul_rn(e2y, e2y)), __fmul_rn(e2z, e2z));
    if (!(s2 > __fmul_rn(1e-12f, __fmul_rn(l1, l2)))) return false;
    const float len = __fsqrt_rn(s2);
    float nx = __fdiv_rn(cx, len), ny = __fdiv_rn(cy, len), nz = __fdiv_rn(cz, len);
    float d = -__fadd_rn(__fadd_rn(__fmul_rn(nx, p0.x), __fmul_rn(ny, p0.y)), __fmul_rn(nz, p0.z));
    if (d < 0.0f) { nx = -nx; ny = -ny; nz = -nz; d = -d; }
    pl = make_float4(nx, ny, nz, d);
    return true;
}

__global__ void __launch_bounds__(256)
ransac_hyp_kernel(RansacWorkspace ws, RansacArgs a, int need_err) {
    const int idx = blockIdx.x * 256 + threadIdx.x;
    const int R = ws.R, HP = ws.n_hyp_pad, KL = ws.score_K * ws.score_L;
    const int HS = max(HP, KL);
    if (idx >= R * HS) return;
    const int r = idx / HS, h = idx % HS;
    const size_t f = blockIdx.y;
    const size_t slot = (f * R + r) * HP + h;
    const int32_t* off = ws.region_off + f * (size_t)(R + 1);
    const uint32_t n = (uint32_t)(off[r + 1] - off[r]);
    float4 pl = make_float4(__int_as_float(0x7FC00000), 0.f, 0.f, 0.f);   // NaN = invalid
    int c0 = -1;
    if (h < ws.n_hyp && n >= 3) {
        const SampleIdx s = sample(a.sampler, (uint32_t)h, (uint32_t)r, a.first_frame + (uint32_t)f, a.seed, n);
        if (s.ok) {
            const uint2* pts = ws.points + f * (size_t)ws.W * ws.H + off[r];
            const float ifx = 1.0f / a.K.fx, ify = 1.0f / a.K.fy;   // host-identical IEEE division
            PM_CHECK(s.i0 < n && s.i1 < n && s.i2 < n && off[r] + n <= ws.W * ws.H);
            const uint2 q0 = pts[s.i0], q1 = pts[s.i1], q2 = pts[s.i2];
            const float3 p0 = deproject(PackedPoint{q0.x, __uint_as_float(q0.y)}, a.K.cx, a.K.cy, ifx, ify);
            const float3 p1 = deproject(PackedPoint{q1.x, __uint_as_float(q1.y)}, a.K.cx, a.K.cy, ifx, ify);
            const float3 p2 = deproject(PackedPoint{q2.x, __uint_as_float(q2.y)}, a.K.cx, a.K.cy, ifx, ify);
            float4 t;
            if (plane_from_3pts(p0, p1, p2, t)) { pl = t; c0 = 0; }
        }
    }
    if (h < HP) {
        ws.planes[slot] = pl;
        ws.counts[slot] = c0;
        if (need_err) ws.errq[slot] = 0ull;
    }
    if ((ws.score_K & 1) == 0 && h < KL) {      // packed-scoring copy: pair (h, h + L) per component
        const int L = ws.score_L, k = h / L, l = h % L, j = k >> 1, half = k & 1;
        float* q = reinterpret_cast<float*>(ws.pairs) + ((f * R + r) * (size_t)(2 * KL) + (j * L + l) * 4) * 2 + half;
        q[0] = pl.x;
        q[2] = pl.y;
        q[4] = pl.z;
        q[6] = pl.w;
    }
}

// ---- chunk staging shared by the score and refit kernels: the compacted
// points [s, e) of frame f, deprojected once into shared memory, and the
// first region overlapping the chunk.
struct Chunk {
    int s, e, r0;
};

// max{r < R : off[r] <= s} for nondecreasing off[] with off[0] = 0 <= s, by
// one full warp: a 32-ary search (every lane probes one offset per level; the
// ballot is a prefix), log32(R) dependent loads instead of log2(R).
PM_DEVINL int first_region(const int32_t* off, int R, int s, int lane) {
    int r0 = 0;
    for (int hi = R; hi - r0 > 1;) {
        const int step = (hi - r0 + 31) >> 5;
        const int p = r0 + lane * step;
        const unsigned le = __ballot_sync(kFull, lane == 0 || (p < hi && off[p] <= s));
        r0 += (31 - __clz(le)) * step;
        hi = min(hi, r0 + step);
    }
    return r0;
}

PM_DEVINL bool stage_chunk(const RansacWorkspace& ws, const RansacArgs& a, size_t f, float4* sp, int* s_r0,
                           Chunk& ck) {
    // points per CTA: kScoreChunk
    const int R = ws.R;
    const int32_t* off = ws.region_off + f * (size_t)(R + 1);
    const int total = off[R];
    ck.s = blockIdx.x * kScoreChunk;
    if (ck.s >= total) return false;
    ck.e = min(ck.s + kScoreChunk, total);
    const uint2* pts = ws.points + f * (size_t)ws.W * ws.H;
    const float ifx = 1.0f / a.K.fx, ify = 1.0f / a.K.fy;   // IEEE division, as on the host
    for (int i = threadIdx.x; i < ck.e - ck.s; i += kScoreThreads) {
        PM_CHECK(i < kScoreChunk && ck.s + i < ws.W * ws.H);
        const uint2 q = pts[ck.s + i];
        const float3 P = deproject(PackedPoint{q.x, __uint_as_float(q.y)}, a.K.cx, a.K.cy, ifx, ify);
        sp[i] = make_float4(P.x, P.y, P.z, 0.f);
    }
    if (threadIdx.x < 32) {                 // region with off[r] <= s < off[r+1]
        const int r0 = first_region(off, R, ck.s, threadIdx.x);
        if (threadIdx.x == 0) *s_r0 = r0;
    }
    __syncthreads();
    ck.r0 = *s_r0;
    return true;
}

// c += (a < b): one FSETP and one predicated IADD (NaN never counts)
PM_DEVINL void count_lt(int& c, float a, float b) {
    asm("{\n.reg .pred p;\nsetp.lt.f32 p, %1, %2;\n@p add.s32 %0, %0, 1;\n}" : "+r"(c) : "f"(a), "f"(b));
}

// pairs j with bit (j mod 4) set count on the FMA pipe (FSET + FADD2), the
// others on the ALU pipe (FSETP + predicated IADD).  Measured on the bench
// step (tools/ab_fadd_mask.sh): mask 0 (all on the ALU pipe) 3.031 ms,
// 5 (even pairs) 3.048, 1: 3.076, 7: 3.112, 15: 3.134 ms RANSAC stage.
#ifndef PM_SCORE_FADD_MASK
#define PM_SCORE_FADD_MASK 0
#endif
// pairs j with bit (j mod 4) set count by the sign of fl(|d| - tau) (FADD on
// the FMA pipe with the |.| operand modifier, then LEA.HI / shift-add of the
// sign bit on the ALU pipe): fl(|d| - tau) < 0 exactly when |d| < tau (the
// rounded difference keeps its sign and is +0 only at |d| == tau; |NaN| - tau
// is a positive NaN), so the counts stay bit-exact.
#ifndef PM_SCORE_SIGN_MASK
#define PM_SCORE_SIGN_MASK 0
#endif

// Packed-pair scoring (two hypotheses per FFMA2 chain) for even K without the
// error sum, reading the plane pairs the hyp kernel lays out (ws.pairs).
template <int K, int L, bool WITH_ERR>
__host__ __device__ constexpr bool score_packed() { return !WITH_ERR && (K % 2) == 0; }
template <int K, int L, bool WITH_ERR>
constexpr size_t score_smem_bytes() {
    return sizeof(float4) * kScoreChunk + sizeof(int) * kScoreThreads * K;
}

// The hot loop (Alg. 2 ℓ9-13).  grid = (ceil(W*H / kScoreChunk), B).  The CTA's
// threads form G = 256 / L groups of L lanes; lane l of every group holds
// hypotheses l, l + L, ..., l + (K-1) L of the current region in registers;
// group g walks points g, g + G, ... of the segment, each point a broadcast
// shared load.  An evaluation costs 3 FFMA + FSETP + a predicated IADD; the
// only reduction is one shared-memory sum over the G groups per segment and
// one integer atomic per hypothesis (exact and order-free).
template <int K, int L, bool WITH_ERR>
__global__ void __launch_bounds__(kScoreThreads)
ransac_score_kernel(RansacWorkspace ws, RansacArgs a) {
    extern __shared__ __align__(16) float4 sp[];                 // kScoreChunk points
    __shared__ int s_r0;
    constexpr int G = kScoreThreads / L;
    constexpr bool kSmemReduce = G > 1;
    int* s_cnt = reinterpret_cast<int*>(sp + kScoreChunk);      // [G][L * K]
    const size_t f = blockIdx.y;
    Chunk ck;
    if (!stage_chunk(ws, a, f, sp, &s_r0, ck)) return;
    const int R = ws.R, HP = ws.n_hyp_pad, NH = ws.n_hyp;
    const int g = threadIdx.x / L, l = threadIdx.x % L;
    const int32_t* off = ws.region_off + f * (size_t)(R + 1);
    const float tau = a.tau;
    const float4 nan4 = make_float4(__int_as_float(0x7FC00000), 0.f, 0.f, 0.f);
    for (int r = ck.r0; r < R && off[r] < ck.e; ++r) {
        const int lo = max(ck.s, off[r]) - ck.s, hi = min(ck.e, off[r + 1]) - ck.s;
        if (hi <= lo || off[r + 1] - off[r] < 3) continue;
        const float4* planes = ws.planes + (f * R + r) * HP;
        int32_t* counts = ws.counts + (f * R + r) * HP;
        uint64_t* errq = ws.errq + (f * R + r) * HP;
        float4 pl[K];
        int c[K];
        uint64_t eq[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int h = l + k * L;
            pl[k] = (!score_packed<K, L, WITH_ERR>() && h < NH) ? __ldg(planes + h) : nan4;
            c[k] = 0;
            eq[k] = 0;
        }
        if (!score_packed<K, L, WITH_ERR>()) {
#pragma unroll 4
            for (int i = lo + g; i < hi; i += G) {
                const float4 p4 = sp[i];
                const float3 P = make_float3(p4.x, p4.y, p4.z);
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const float dist = plane_dist(pl[k], P);
                    count_lt(c[k], dist, tau);
                    if (WITH_ERR) eq[k] += __float2ull_rn(__fmul_rn(fminf(dist, 64.0f), 16777216.0f));
                }
            }
        } else {
            // two hypotheses per packed FFMA2 chain: the same per-lane fma
            // sequence as plane_dist(), so the counts stay bit-exact
            // plane pairs as written by the hyp kernel ([K/2][L] x (x, y, z, w)
            // pairs): they reach the registers as 64-bit pairs (pairs built from
            // scalars get re-paired with moves on every use)
            constexpr int K2 = K / 2 > 0 ? K / 2 : 1;
            const ulonglong2* pp = reinterpret_cast<const ulonglong2*>(ws.pairs) + (f * R + r) * (size_t)(K * L);
            uint64_t X[K2], Y[K2], Z[K2], D[K2];
#pragma unroll
            for (int j = 0; j < K2; ++j) {
                const ulonglong2 u = __ldg(pp + (j * L + l) * 2);
                const ulonglong2 v = __ldg(pp + (j * L + l) * 2 + 1);
                X[j] = u.x; Y[j] = u.y; Z[j] = v.x; D[j] = v.y;
            }
            // inlier indicators as 1.0f / 0.0f (FSET, NaN -> 0) summed two at a
            // time (FADD2); exact: a thread adds at most kScoreChunk ones
            uint64_t acc[K2];
#pragma unroll
            for (int j = 0; j < K2; ++j) acc[j] = 0ull;
#pragma unroll 8
            for (int i = lo + g; i < hi; i += G) {
                const float4 p4 = sp[i];
                const uint64_t px = f2pk(f2s(p4.x)), py = f2pk(f2s(p4.y)), pz = f2pk(f2s(p4.z));
#pragma unroll
                for (int j = 0; j < K2; ++j) {
                    uint64_t d;
                    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(X[j]), "l"(px), "l"(D[j]));
                    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(Y[j]), "l"(py));
                    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(Z[j]), "l"(pz));
                    const float2 df = f2up(d);
                    if ((PM_SCORE_SIGN_MASK >> (j & 3)) & 1) {
                        c[2 * j] += (int)(__float_as_uint(__fsub_rn(fabsf(df.x), tau)) >> 31);
                        c[2 * j + 1] += (int)(__float_as_uint(__fsub_rn(fabsf(df.y), tau)) >> 31);
                    } else if (!((PM_SCORE_FADD_MASK >> (j & 3)) & 1)) {
                        // ALU-pipe count (FSETP + predicated IADD): the FMA pipe
                        // keeps the three FFMA2 of the distance
                        count_lt(c[2 * j], fabsf(df.x), tau);
                        count_lt(c[2 * j + 1], fabsf(df.y), tau);
                    } else {
                        float i0, i1;
                        asm("set.lt.f32.f32 %0, %1, %2;" : "=f"(i0) : "f"(fabsf(df.x)), "f"(tau));
                        asm("set.lt.f32.f32 %0, %1, %2;" : "=f"(i1) : "f"(fabsf(df.y)), "f"(tau));
                        asm("add.rn.f32x2 %0, %0, %1;" : "+l"(acc[j]) : "l"(f2pk(make_float2(i0, i1))));
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < K2; ++j) {
                if (!((PM_SCORE_FADD_MASK >> (j & 3)) & 1)) continue;
                const float2 a2 = f2up(acc[j]);
                c[2 * j] = (int)a2.x;
                c[2 * j + 1] = (int)a2.y;
            }
        }
        if (WITH_ERR) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int h = l + k * L;
                if (h < NH && eq[k] > 0 && !isnan(pl[k].x))
                    atomicAdd((unsigned long long*)(errq + h), (unsigned long long)eq[k]);
            }
        }
        if (!kSmemReduce) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int h = l + k * L;
                if (h < NH && c[k] > 0) atomicAdd(counts + h, c[k]);
            }
        } else {
            // groups of one warp first meet by shuffles (L < 32), then one
            // partial per warp (or per group) in shared memory
            constexpr int NP = L < 32 ? kScoreThreads / 32 : G;   // partials per hypothesis
            const int lane = threadIdx.x & 31;
            if (L < 32) {
#pragma unroll
                for (int k = 0; k < K; ++k)
#pragma unroll
                    for (int o = L; o < 32; o <<= 1) c[k] += __shfl_xor_sync(kFull, c[k], o);
            }
            if (L >= 32 || lane < L) {
                const int q = L < 32 ? (int)(threadIdx.x >> 5) : g;
#pragma unroll
                for (int k = 0; k < K; ++k) s_cnt[q * (L * K) + k * L + l] = c[k];
            }
            __syncthreads();
            for (int h = threadIdx.x; h < L * K; h += kScoreThreads) {
                int sum = 0;
#pragma unroll 8
                for (int q = 0; q < NP; ++q) sum += s_cnt[q * (L * K) + h];
                if (h < NH && sum > 0) atomicAdd(counts + h, sum);
            }
            __syncthreads();
        }
    }
}

// Many small regions (a chunk holding ~10+ region segments): the kernel above
// spreads every segment over all 256 threads and pays a block reduction with
// two barriers per segment.  Here each warp takes whole segments (regions
// r0 + w, r0 + w + 8, ...) with its 32 / L groups of L lanes, reduces them by
// shuffles and adds one atomic per hypothesis -- no barrier after staging.
// The same packed evaluation and ALU-pipe count as above (bit-exact counts).
// Used for the count-only packed layouts when the frame's average region is
// smaller than kSmallRegionPx points (host dispatch; measured: 640x480 frames
// with R = 1024, 300-point regions: scoring 0.43 -> 0.71 of its issue bound,
// with R = 256, 1200-point regions, the CTA-wide kernel stays ahead).
constexpr int kSmallRegionPx = kScoreChunk / 8;   // ~8+ segments per chunk: every warp has one
template <int K, int L>
__global__ void __launch_bounds__(kScoreThreads)
ransac_score_small_kernel(RansacWorkspace ws, RansacArgs a) {
    static_assert(K % 2 == 0 && L <= 32 && 32 % L == 0, "packed count layouts with L <= 32");
    extern __shared__ __align__(16) float4 sp[];                 // kScoreChunk points
    __shared__ int s_r0;
    constexpr int GW = 32 / L;                                   // groups per warp
    constexpr int K2 = K / 2;
    const size_t f = blockIdx.y;
    Chunk ck;
    if (!stage_chunk(ws, a, f, sp, &s_r0, ck)) return;
    const int R = ws.R, NH = ws.n_hyp;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int g = lane / L, l = lane % L;
    const int32_t* off = ws.region_off + f * (size_t)(R + 1);
    const float tau = a.tau;
    for (int r = ck.r0 + w; r < R && off[r] < ck.e; r += kScoreThreads / 32) {   // warp-uniform
        const int lo = max(ck.s, off[r]) - ck.s, hi = min(ck.e, off[r + 1]) - ck.s;
        if (hi <= lo || off[r + 1] - off[r] < 3) continue;
        const ulonglong2* pp = reinterpret_cast<const ulonglong2*>(ws.pairs) + (f * R + r) * (size_t)(K * L);
        uint64_t X[K2], Y[K2], Z[K2], D[K2];
#pragma unroll
        for (int j = 0; j < K2; ++j) {
            const ulonglong2 u = __ldg(pp + (j * L + l) * 2);
            const ulonglong2 v = __ldg(pp + (j * L + l) * 2 + 1);
            X[j] = u.x; Y[j] = u.y; Z[j] = v.x; D[j] = v.y;
        }
        int c[K];
#pragma unroll
        for (int k = 0; k < K; ++k) c[k] = 0;
#pragma unroll 4
        for (int i = lo + g; i < hi; i += GW) {
            PM_CHECK(i >= 0 && i < kScoreChunk);
            const float4 p4 = sp[i];
            const uint64_t px = f2pk(f2s(p4.x)), py = f2pk(f2s(p4.y)), pz = f2pk(f2s(p4.z));
#pragma unroll
            for (int j = 0; j < K2; ++j) {
                uint64_t d;
                asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(X[j]), "l"(px), "l"(D[j]));
                asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(Y[j]), "l"(py));
                asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(Z[j]), "l"(pz));
                const float2 df = f2up(d);
                count_lt(c[2 * j], fabsf(df.x), tau);
                count_lt(c[2 * j + 1], fabsf(df.y), tau);
            }
        }
        int32_t* counts = ws.counts + (f * R + r) * ws.n_hyp_pad;
#pragma unroll
        for (int k = 0; k < K; ++k) {
#pragma unroll
            for (int o = L; o < 32; o <<= 1) c[k] += __shfl_xor_sync(kFull, c[k], o);
            const int h = l + k * L;                 // pair j holds k = 2j, 2j + 1 (the hyp kernel's layout)
            if (g == 0 && h < NH && c[k] > 0) atomicAdd(counts + h, c[k]);
        }
    }
}

// ---- ℓ14-17 selection: argmax count (or argmin error), ties -> lowest h.
// Every caller evaluates the same order-free rule, so results agree.
struct Best {
    unsigned long long score;   // 0 = no valid hypothesis
    int h;
};
PM_DEVINL void best_merge(Best& b, unsigned long long sc, int h) {
    if (sc > b.score || (sc == b.score && h < b.h)) { b.score = sc; b.h = h; }
}
PM_DEVINL bool select_by_error(int select) { return select == PM_SELECT_ERROR || select == PM_SELECT_ERROR_EARLY; }
PM_DEVINL unsigned long long hyp_score(int select, int32_t c, uint64_t e) {
    if (c < 0) return 0ull;
    return select_by_error(select) ? ~(unsigned long long)e : (unsigned long long)(c + 1);
}
// warp-cooperative: all lanes return the result
PM_DEVINL Best warp_select(const int32_t* counts, const uint64_t* errq, int NH, int select) {
    Best b{0ull, 0x7FFFFFFF};
    for (int h = (int)(threadIdx.x & 31); h < NH; h += 32) best_merge(b, hyp_score(select, counts[h], errq[h]), h);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long sc = __shfl_xor_sync(kFull, b.score, o);
        const int h = __shfl_xor_sync(kFull, b.h, o);
        best_merge(b, sc, h);
    }
    return b;
}

// ---- fp64 refit: shifted moments of the winner's inliers, per (region,
// chunk) slot, reduced in a fixed order (deterministic).
PM_DEVINL void sums_add(Sums& a, const Sums& b) {
#pragma unroll
    for (int k = 0; k < 3; ++k) a.s[k] += b.s[k];
#pragma unroll
    for (int k = 0; k < 6; ++k) a.m[k] += b.m[k];
    a.n += b.n;
    a.err += b.err;
}

PM_DEVINL Sums sums_shfl_xor(const Sums& a, int o) {
    Sums b;
#pragma unroll
    for (int k = 0; k < 3; ++k) b.s[k] = __shfl_xor_sync(kFull, a.s[k], o);
#pragma unroll
    for (int k = 0; k < 6; ++k) b.m[k] = __shfl_xor_sync(kFull, a.m[k], o);
    b.n = __shfl_xor_sync(kFull, a.n, o);
    b.err = __shfl_xor_sync(kFull, a.err, o);
    b.pad = 0;
    return b;
}

// P:292 "iterates until ... a satisfactory model is found" (the *_EARLY
// select modes, Q20): the sequential loop of ℓ5-18 stops after the
// first h at which the best model so far passes the acceptance gate of ℓ19.
// Every hypothesis is scored anyway (no work to save in a batched launch);
// the warp replays the loop's selection in chunks of 32: an inclusive
// prefix-best scan per chunk, then the first lane whose prefix best is
// satisfactory.  Warp-cooperative: all lanes return the result.
PM_DEVINL int early_select(const int32_t* counts, const uint64_t* errq, int NH, int select, int n) {
    const int lane = (int)(threadIdx.x & 31);
    Best run{0ull, 0x7FFFFFFF};                 // best of the chunks before
    int run_cnt = -1;
    for (int h0 = 0; h0 < NH; h0 += 32) {
        const int h = h0 + lane;
        const int32_t c = h < NH ? counts[h] : -1;
        Best b{h < NH ? hyp_score(select, c, errq[h]) : 0ull, h};
        int bc = c;                             // count of the prefix best
        // inclusive prefix scan of best_merge (lowest index wins ties: the
        // sequential loop keeps the earlier model unless strictly better)
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long sc = __shfl_up_sync(kFull, b.score, o);
            const int hh = __shfl_up_sync(kFull, b.h, o);
            const int cc = __shfl_up_sync(kFull, bc, o);
            if (lane >= o && (sc > b.score || (sc == b.score && hh < b.h))) { b.score = sc; b.h = hh; bc = cc; }
        }
        if (run.score > b.score || (run.score == b.score && run.h < b.h)) { b = run; bc = run_cnt; }
        const bool ok = b.score != 0ull && (long long)10 * bc > (long long)9 * n;
        const unsigned m = __ballot_sync(kFull, ok && h < NH);
        if (m) {
            const int l = __ffs(m) - 1;
            return __shfl_sync(kFull, b.h, l);
        }
        run.score = __shfl_sync(kFull, b.score, 31);
        run.h = __shfl_sync(kFull, b.h, 31);
        run_cnt = __shfl_sync(kFull, bc, 31);
    }
    return run.score == 0ull ? -1 : run.h;
}

// ℓ14-17 once per region: one warp per (frame, region) -> best[f][r] (-1:
// none / too few points).  grid = (ceil(R / 8), B).
__global__ void __launch_bounds__(256)
ransac_select_kernel(RansacWorkspace ws, RansacArgs a) {
    const int r = blockIdx.x * 8 + (threadIdx.x >> 5);
    const size_t f = blockIdx.y;
    if (r >= ws.R) return;
    const int R = ws.R, HP = ws.n_hyp_pad;
    const int32_t* off = ws.region_off + f * (size_t)(R + 1);
    int best = -1;
    const int n = off[r + 1] - off[r];
    if (n >= 3) {
        const int32_t* cnt = ws.counts + (f * R + r) * HP;
        const uint64_t* eq = ws.errq + (f * R + r) * HP;
        if (a.select == PM_SELECT_COUNT_EARLY || a.select == PM_SELECT_ERROR_EARLY) {
            best = early_select(cnt, eq, ws.n_hyp, a.select, n);
        } else {
            const Best b = warp_select(cnt, eq, ws.n_hyp, a.select);
            best = b.score == 0ull ? -1 : b.h;
        }
    }
    if ((threadIdx.x & 31) == 0) ws.best[f * R + r] = best;
}

// grid = (ceil(W*H / kRefitChunk), B).  For every region segment of the
// chunk: take the winner (ransac_select_kernel), recount its inliers with the same f32
// arithmetic, accumulate fp64 moments, write slot (chunk + region).
// Warp w owns the contiguous sub-chunk [wlo, whi) of kWarpSpan points; it meets
// one or two regions, so a warp runs ~1.2 moment reductions per chunk.  Its
// points arrive in shared memory by two bulk copies (cp.async.bulk, one per
// half span, each on its own mbarrier) issued before any arithmetic, so the
// second half streams in while the first is processed and the whole chunk is
// in flight at once (64 KB per CTA) instead of 8 loads per thread.
constexpr int kWarpSpan = kRefitChunk / kRefitWarps;       // 1024 points
constexpr int kHalfSpan = kWarpSpan / 2;
constexpr int kHalfSlot = kHalfSpan + 2;                    // + 16 B alignment slack
constexpr size_t kRefitSmem = sizeof(uint2) * kRefitWarps * 2 * kHalfSlot;

PM_DEVINL void bulk_load_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"((uint64_t)src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__global__ void __launch_bounds__(kScoreThreads)
ransac_refit_kernel(RansacWorkspace ws, RansacArgs a) {
    extern __shared__ __align__(16) uint2 s_pts[];            // [warp][half][kHalfSlot]
    __shared__ __align__(8) uint64_t s_bar[kRefitWarps][2];
    const size_t f = blockIdx.y;
    const int R = ws.R, HP = ws.n_hyp_pad;
    const int32_t* off = ws.region_off + f * (size_t)(R + 1);
    const int total = off[R];
    const int cs = blockIdx.x * kRefitChunk;
    if (cs >= total) return;
    const int ce = min(cs + kRefitChunk, total);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint2* pts = ws.points + f * (size_t)ws.W * ws.H;
    const int wlo = cs + w * kWarpSpan, whi = min(wlo + kWarpSpan, ce), wmid = min(wlo + kHalfSpan, whi);
    // half h covers [hs[h], he[h]); its first point sits at s_pts index sb[h] + sh[h]
    const int hs0 = wlo, he0 = wmid, hs1 = wmid, he1 = whi;
    uint2* sb0 = s_pts + (w * 2 + 0) * kHalfSlot;
    uint2* sb1 = s_pts + (w * 2 + 1) * kHalfSlot;
    // the workspace is 256-B aligned, so a point's byte address is 8-B aligned:
    // copy from the 16-B boundary at or below it (the extra point is unused;
    // the rounded-up end stays inside the points buffer's 256-B padding)
    const int sh0 = (int)(((uintptr_t)(pts + hs0) >> 3) & 1), sh1 = (int)(((uintptr_t)(pts + hs1) >> 3) & 1);
    if (lane == 0) {
        mbar_init(&s_bar[w][0], 1);
        mbar_init(&s_bar[w][1], 1);
        if (he0 > hs0) {
            const uint32_t bytes = (uint32_t)(((he0 - hs0 + sh0) * 8 + 15) & ~15);
            mbar_arrive_expect_tx(&s_bar[w][0], bytes);
            bulk_load_g2s(sb0, pts + hs0 - sh0, bytes, &s_bar[w][0]);
        }
        if (he1 > hs1) {
            const uint32_t bytes = (uint32_t)(((he1 - hs1 + sh1) * 8 + 15) & ~15);
            mbar_arrive_expect_tx(&s_bar[w][1], bytes);
            bulk_load_g2s(sb1, pts + hs1 - sh1, bytes, &s_bar[w][1]);
        }
    }
    const int r0 = first_region(off, R, cs, lane);          // first region of the chunk
    // lane j prefetches region r0 + j (offsets, winner, winner's plane, first
    // point) in two rounds of independent loads; the region loop below takes
    // them by shuffle instead of four dependent loads per region
    const int rl = r0 + lane;
    const int offL = rl <= R ? off[rl] : 0;
    const int bestL = rl < R ? ws.best[f * R + rl] : -1;
    float4 plL = make_float4(0.f, 0.f, 0.f, 0.f);
    uint2 q0L = make_uint2(0u, 0u);
    if (bestL >= 0 && offL < ce) {                           // best >= 0: >= 3 points
        plL = ws.planes[(f * R + rl) * HP + bestL];
        q0L = pts[offL];
    }
    __syncthreads();          // the mbarrier inits visible before any wait
    const float ifx = 1.0f / a.K.fx, ify = 1.0f / a.K.fy;
    int ready = 0;                                           // bit h: half h waited on
    for (int r = r0; r < R; ++r) {
        const int j = r - r0;                                // warp-uniform
        const bool pre = j < 31;
        const int o0 = pre ? __shfl_sync(kFull, offL, j) : off[r];
        if (o0 >= ce) break;
        const int o1 = pre ? __shfl_sync(kFull, offL, j + 1) : off[r + 1];
        const int lo = max(cs, o0), hi = min(ce, o1);
        if (hi <= lo) continue;
        const int best = pre ? __shfl_sync(kFull, bestL, j) : ws.best[f * R + r];
        if (best >= 0) {
            const int a0 = max(lo, wlo), a1 = min(hi, whi);
            Sums acc = {};
            if (a0 < a1) {                                    // warp-uniform
                float4 pl;
                uint2 q0;
                if (pre) {
                    pl = make_float4(__shfl_sync(kFull, plL.x, j), __shfl_sync(kFull, plL.y, j),
                                     __shfl_sync(kFull, plL.z, j), __shfl_sync(kFull, plL.w, j));
                    q0 = make_uint2(__shfl_sync(kFull, q0L.x, j), __shfl_sync(kFull, q0L.y, j));
                } else {
                    pl = ws.planes[(f * R + r) * HP + best];
                    q0 = pts[o0];
                }
                const float3 o3 = deproject(PackedPoint{q0.x, __uint_as_float(q0.y)}, a.K.cx, a.K.cy, ifx, ify);
                const double ox = o3.x, oy = o3.y, oz = o3.z;
#pragma unroll 1
                for (int half = 0; half < 2; ++half) {
                    const int b0 = max(a0, half ? hs1 : hs0), b1 = min(a1, half ? he1 : he0);
                    if (b0 >= b1) continue;
                    if (!(ready >> half & 1)) { mbar_wait(&s_bar[w][half], 0); ready |= 1 << half; }
                    const uint2* sp = (half ? sb1 + sh1 - hs1 : sb0 + sh0 - hs0);
#pragma unroll 4
                    for (int i = b0 + lane; i < b1; i += 32) {
                        PM_CHECK(&sp[i] >= s_pts && &sp[i] < s_pts + kRefitWarps * 2 * kHalfSlot);
                        const uint2 q = sp[i];
                        const float3 P = deproject(PackedPoint{q.x, __uint_as_float(q.y)}, a.K.cx, a.K.cy, ifx, ify);
                        const float dist = plane_dist(pl, P);
                        // <= 2^30: a 32-bit conversion (F2I.U32), widened for the sum
                        acc.err += (unsigned long long)__float2uint_rn(__fmul_rn(fminf(dist, 64.0f), 16777216.0f));
                        if (dist < a.tau) {
                            const double x = (double)P.x - ox, y = (double)P.y - oy, z = (double)P.z - oz;
                            acc.s[0] += x; acc.s[1] += y; acc.s[2] += z;
                            acc.m[0] = fma(x, x, acc.m[0]); acc.m[1] = fma(x, y, acc.m[1]); acc.m[2] = fma(x, z, acc.m[2]);
                            acc.m[3] = fma(y, y, acc.m[3]); acc.m[4] = fma(y, z, acc.m[4]); acc.m[5] = fma(z, z, acc.m[5]);
                            acc.n += 1;
                        }
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) sums_add(acc, sums_shfl_xor(acc, o));
            }
            // one slot per (chunk + region, warp), zero when the warp's span
            // misses the region: no block barrier; the finalize kernel sums
            // them in (chunk, warp) order (deterministic)
            PM_CHECK(blockIdx.x + r < ws.n_slots);
            if (lane == 0) ws.slots[(f * (size_t)ws.n_slots + blockIdx.x + r) * kRefitWarps + w] = acc;
        }
    }
    // a warp whose copies were never waited on must not exit with them in flight
    if (!(ready & 1) && he0 > hs0) mbar_wait(&s_bar[w][0], 0);
    if (!(ready & 2) && he1 > hs1) mbar_wait(&s_bar[w][1], 0);
}

// Smallest-eigenvalue eigenvector of a symmetric 3x3 (double) by cyclic
// Jacobi rotations (Golub & Van Loan, symmetric Schur decomposition).
PM_DEVINL void smallest_eigvec(double A[3][3], double out[3]) {
    double V[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
    const double scale = fabs(A[0][0]) + fabs(A[1][1]) + fabs(A[2][2]);
    for (int sweep = 0; sweep < 64; ++sweep) {
        const double off = sqrt(A[0][1] * A[0][1] + A[0][2] * A[0][2] + A[1][2] * A[1][2]);
        if (off == 0.0 || off <= 1e-15 * scale) break;
        for (int k = 0; k < 3; ++k) {
            const int p = k == 2 ? 1 : 0, q = k == 0 ? 1 : 2;
            const double apq = A[p][q];
            if (apq == 0.0) continue;
            const double tau = (A[q][q] - A[p][p]) / (2.0 * apq);
            const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            const double c = rsqrt(1.0 + t * t), sn = t * c;
            for (int i = 0; i < 3; ++i) {            // A <- A J
                const double aip = A[i][p], aiq = A[i][q];
                A[i][p] = c * aip - sn * aiq;
                A[i][q] = sn * aip + c * aiq;
            }
            for (int i = 0; i < 3; ++i) {            // A <- J^T A
                const double api = A[p][i], aqi = A[q][i];
                A[p][i] = c * api - sn * aqi;
                A[q][i] = sn * api + c * aqi;
            }
            for (int i = 0; i < 3; ++i) {            // V <- V J
                const double vip = V[i][p], viq = V[i][q];
                V[i][p] = c * vip - sn * viq;
                V[i][q] = sn * vip + c * viq;
            }
        }
    }
    int m = 0;
    if (A[1][1] < A[m][m]) m = 1;
    if (A[2][2] < A[m][m]) m = 2;
    const double nn = sqrt(V[0][m] * V[0][m] + V[1][m] * V[1][m] + V[2][m] * V[2][m]);
    out[0] = V[0][m] / nn;
    out[1] = V[1][m] / nn;
    out[2] = V[2][m] / nn;
}

// One thread per (frame, region): selection, slot reduction in chunk order,
// eigen-solve, gate (ℓ19), pm_plane output.
constexpr int kFinalThreads = 128;
__global__ void __launch_bounds__(kFinalThreads)
ransac_finalize_kernel(RansacWorkspace ws, RansacArgs a, pm_plane* __restrict__ planes_out) {
    const int r = blockIdx.x * kFinalThreads + threadIdx.x;
    const size_t f = blockIdx.y;
    const int R = ws.R, HP = ws.n_hyp_pad, NH = ws.n_hyp;
    if (r >= R) return;
    const int32_t* off = ws.region_off + f * (size_t)(R + 1);
    const int base = off[r];
    const int n = off[r + 1] - base;
    const int32_t* counts = ws.counts + (f * R + r) * HP;
    const uint64_t* errq = ws.errq + (f * R + r) * HP;
    if (a.counts_out)
        for (int h = 0; h < NH; ++h) a.counts_out[(f * R + r) * NH + h] = counts[h];
    if (a.errq_out)
        for (int h = 0; h < NH; ++h) a.errq_out[(f * R + r) * NH + h] = errq[h];
    pm_plane res;
    for (int k = 0; k < 3; ++k) { res.n[k] = 0.f; res.centroid[k] = 0.f; }
    res.d = 0.f; res.inliers = 0; res.n_points = n; res.best_hyp = -1; res.sum_dist = 0.f;
    pm_plane* out = planes_out + f * R + r;
    if (n < 3) { res.status = PM_PLANE_TOO_FEW; *out = res; return; }
    const int best = ws.best[f * R + r];
    if (best < 0) { res.status = PM_PLANE_DEGENERATE; *out = res; return; }
    const float4 pl = ws.planes[(f * R + r) * HP + best];
    // slots of this region: chunks c0..c1 -> slot c + r (ascending order)
    const int c0 = base / kRefitChunk, c1 = (base + n - 1) / kRefitChunk;
    const Sums* sl = ws.slots + f * (size_t)ws.n_slots * kRefitWarps;
    Sums t = sl[(c0 + r) * kRefitWarps];
    for (int k = 1; k < kRefitWarps; ++k) sums_add(t, sl[(c0 + r) * kRefitWarps + k]);
    for (int c = c0 + 1; c <= c1; ++c)
        for (int k = 0; k < kRefitWarps; ++k) sums_add(t, sl[(c + r) * kRefitWarps + k]);
    const uint2* pts = ws.points + f * (size_t)ws.W * ws.H + base;
    const float ifx = 1.0f / a.K.fx, ify = 1.0f / a.K.fy;
    const uint2 q0 = pts[0];
    const float3 o3 = deproject(PackedPoint{q0.x, __uint_as_float(q0.y)}, a.K.cx, a.K.cy, ifx, ify);
    double nv[3], cen[3], dd;
    if (t.n >= 3) {
        const double inv = 1.0 / t.n;
        const double mx = t.s[0] * inv, my = t.s[1] * inv, mz = t.s[2] * inv;
        double A[3][3];
        A[0][0] = t.m[0] - t.n * mx * mx; A[0][1] = t.m[1] - t.n * mx * my; A[0][2] = t.m[2] - t.n * mx * mz;
        A[1][1] = t.m[3] - t.n * my * my; A[1][2] = t.m[4] - t.n * my * mz; A[2][2] = t.m[5] - t.n * mz * mz;
        A[1][0] = A[0][1]; A[2][0] = A[0][2]; A[2][1] = A[1][2];
        smallest_eigvec(A, nv);
        cen[0] = (double)o3.x + mx; cen[1] = (double)o3.y + my; cen[2] = (double)o3.z + mz;
        dd = -(nv[0] * cen[0] + nv[1] * cen[1] + nv[2] * cen[2]);
    } else {
        // refit impossible (tau below rounding): keep the 3-point model,
        // centroid = mean of its three sample points (Q19)
        const SampleIdx s = sample(a.sampler, (uint32_t)best, (uint32_t)r, a.first_frame + (uint32_t)f, a.seed,
                                   (uint32_t)n);
        const uint32_t id[3] = {s.i0, s.i1, s.i2};
        cen[0] = cen[1] = cen[2] = 0.0;
        for (int k = 0; k < 3; ++k) {
            const uint2 q = pts[id[k]];
            const float3 P = deproject(PackedPoint{q.x, __uint_as_float(q.y)}, a.K.cx, a.K.cy, ifx, ify);
            cen[0] += P.x; cen[1] += P.y; cen[2] += P.z;
        }
        for (int k = 0; k < 3; ++k) cen[k] /= 3.0;
        nv[0] = pl.x; nv[1] = pl.y; nv[2] = pl.z;
        dd = pl.w;
    }
    if (dd < 0.0) { nv[0] = -nv[0]; nv[1] = -nv[1]; nv[2] = -nv[2]; dd = -dd; }
    for (int k = 0; k < 3; ++k) { res.n[k] = (float)nv[k]; res.centroid[k] = (float)cen[k]; }
    res.d = (float)dd;
    res.inliers = counts[best];
    res.best_hyp = best;
    res.status = (10ll * counts[best] > 9ll * n) ? PM_PLANE_OK : PM_PLANE_REJECTED;   // ℓ19
    res.sum_dist = (float)((double)t.err * (1.0 / 16777216.0));
    *out = res;
}

}  // namespace

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

cudaError_t ransac_setup_attributes() {
    cudaError_t e = cudaSuccess;
#define PM_ATTR(KK, LL)                                                                                    \
    for (int wr = 0; wr < 2 && e == cudaSuccess; ++wr)                                                     \
        e = cudaFuncSetAttribute(wr ? (const void*)ransac_score_kernel<KK, LL, true>                        \
                                    : (const void*)ransac_score_kernel<KK, LL, false>,                      \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,                              \
                                 (int)(wr ? score_smem_bytes<KK, LL, true>() : score_smem_bytes<KK, LL, false>()));
    PM_ATTR(1, 8) PM_ATTR(2, 8) PM_ATTR(4, 8) PM_ATTR(8, 8) PM_ATTR(8, 16) PM_ATTR(8, 32)
    PM_ATTR(8, 64) PM_ATTR(8, 128) PM_ATTR(8, 256) PM_ATTR(16, 256)
#undef PM_ATTR
#define PM_ATTR_SMALL(KK, LL)                                                                              \
    if (e == cudaSuccess)                                                                                  \
        e = cudaFuncSetAttribute((const void*)ransac_score_small_kernel<KK, LL>,                           \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(sizeof(float4) * kScoreChunk));
    PM_ATTR_SMALL(2, 8) PM_ATTR_SMALL(4, 8) PM_ATTR_SMALL(8, 8) PM_ATTR_SMALL(8, 16) PM_ATTR_SMALL(8, 32)
#undef PM_ATTR_SMALL
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute((const void*)ransac_refit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kRefitSmem);
    return e;
}

RansacWorkspace ransac_workspace_layout(void* base, int W, int H, int R, int n_hyp, int B) {
    RansacWorkspace ws{};
    ws.W = W; ws.H = H; ws.B = B; ws.R = R; ws.n_hyp = n_hyp;
    ws.n_hyp_pad = ((n_hyp + kHB - 1) / kHB) * kHB;
    // scoring layout: K hypotheses per lane, L lanes per group (L * K >= n_hyp);
    // small L means more points in flight per warp, cheaper per-point overhead
    auto pow2ceil = [](int x) { int p = 1; while (p < x) p <<= 1; return p; };
    int L = pow2ceil((n_hyp + 7) / 8);
    L = L < 8 ? 8 : (L > 256 ? 256 : L);
    ws.score_L = L;
    ws.score_K = pow2ceil((n_hyp + L - 1) / L);     // <= 8 except n_hyp > 2048 -> 16
    const size_t WH = (size_t)W * H;
    int st = 1024;
    while (st < 4 * R && st < (1 << 24)) st <<= 1;      // hist entries <= ~W*H/4 per frame
    ws.sub_tile = st;
    ws.n_sub = (int)((WH + st - 1) / st);
    ws.n_slots = (int)((WH + kRefitChunk - 1) / kRefitChunk) + R;
    const size_t Rm = R > 0 ? R : 1;
    size_t o = 0;
    char* p = (char*)base;
    auto take = [&](size_t bytes) { char* q = p ? p + o : nullptr; o += align256(bytes); return (void*)q; };
    ws.points = (uint2*)take(sizeof(uint2) * B * WH);
    ws.hist = (int32_t*)take(sizeof(int32_t) * B * Rm * ws.n_sub);
    ws.region_cnt = (int32_t*)take(sizeof(int32_t) * B * Rm);
    ws.region_off = (int32_t*)take(sizeof(int32_t) * B * (Rm + 1));
    ws.planes = (float4*)take(sizeof(float4) * B * Rm * ws.n_hyp_pad);
    ws.pairs = (float2*)take(sizeof(float4) * B * Rm * (size_t)ws.score_K * ws.score_L);
    ws.counts = (int32_t*)take(sizeof(int32_t) * B * Rm * ws.n_hyp_pad);
    ws.errq = (uint64_t*)take(sizeof(uint64_t) * B * Rm * ws.n_hyp_pad);
    ws.slots = (Sums*)take(sizeof(Sums) * B * (size_t)ws.n_slots * kRefitWarps);
    ws.best = (int32_t*)take(sizeof(int32_t) * B * Rm);
    ws.total_bytes = o;
    return ws;
}

cudaError_t ransac_run(const RansacWorkspace& ws, const RansacArgs& a, pm_plane* planes,
                       cudaStream_t stream) {
    const bool need_err = a.select == PM_SELECT_ERROR || a.select == PM_SELECT_ERROR_EARLY || a.errq_out != nullptr;
    const int K = ws.score_K, L = ws.score_L;
    const int n_hyp_slots = ws.R * (ws.n_hyp_pad > K * L ? ws.n_hyp_pad : K * L);
    auto mark = [&](int k) {
        if (a.stage_events) cudaEventRecord((cudaEvent_t)a.stage_events[k], stream);
    };
    ransac_hyp_kernel<<<dim3((n_hyp_slots + 255) / 256, ws.B), 256, 0, stream>>>(ws, a, need_err ? 1 : 0);
    mark(0);
    const dim3 g_score((unsigned)(((size_t)ws.W * ws.H + kScoreChunk - 1) / kScoreChunk), ws.B);
    bool launched = false;
    // many small regions: the warp-per-segment kernel (count-only packed layouts)
    const bool small = !need_err && (size_t)ws.W * ws.H < (size_t)kSmallRegionPx * (size_t)ws.R;
#define PM_SCORE_SMALL(KK, LL)                                                                             \
    if (!launched && small && K == KK && L == LL) {                                                        \
        ransac_score_small_kernel<KK, LL><<<g_score, kScoreThreads, sizeof(float4) * kScoreChunk, stream>>>(ws, a); \
        launched = true;                                                                                   \
    }
    PM_SCORE_SMALL(2, 8) PM_SCORE_SMALL(4, 8) PM_SCORE_SMALL(8, 8) PM_SCORE_SMALL(8, 16) PM_SCORE_SMALL(8, 32)
#undef PM_SCORE_SMALL
#define PM_SCORE(KK, LL)                                                                                   \
    if (!launched && K == KK && L == LL) {                                                                 \
        if (need_err)                                                                                      \
            ransac_score_kernel<KK, LL, true>                                                              \
                <<<g_score, kScoreThreads, score_smem_bytes<KK, LL, true>(), stream>>>(ws, a);             \
        else                                                                                               \
            ransac_score_kernel<KK, LL, false>                                                             \
                <<<g_score, kScoreThreads, score_smem_bytes<KK, LL, false>(), stream>>>(ws, a);            \
        launched = true;                                                                                   \
    }
    PM_SCORE(1, 8) PM_SCORE(2, 8) PM_SCORE(4, 8) PM_SCORE(8, 8) PM_SCORE(8, 16) PM_SCORE(8, 32)
    PM_SCORE(8, 64) PM_SCORE(8, 128) PM_SCORE(8, 256) PM_SCORE(16, 256)
#undef PM_SCORE
    if (!launched) return cudaErrorInvalidConfiguration;
    mark(1);
    const dim3 g_refit((unsigned)(((size_t)ws.W * ws.H + kRefitChunk - 1) / kRefitChunk), ws.B);
    ransac_select_kernel<<<dim3((ws.R + 7) / 8, ws.B), 256, 0, stream>>>(ws, a);
    ransac_refit_kernel<<<g_refit, kScoreThreads, kRefitSmem, stream>>>(ws, a);
    mark(2);
    ransac_finalize_kernel<<<dim3((ws.R + kFinalThreads - 1) / kFinalThreads, ws.B), kFinalThreads, 0, stream>>>(
        ws, a, planes);
    mark(3);
    return cudaGetLastError();
}

}  // namespace pm
