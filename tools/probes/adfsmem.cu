// Microbenchmark (round 2): the tiled engine's shared-memory pair walk in
// isolation -- 8 warps per CTA, 4 CTAs per SM, a 52 x 128 double-buffered
// f32 tile, 4 row parts x 2 column groups, one barrier per sweep, no global
// memory -- with variants of the neighbour loads and of the cell, to see
// which limiter binds the sweep rate (cycles per 64 cell-updates per SMSP).
//   MODE 0: as adf.cu: LDS.64 south pair, scalar W (x-1) and E (x+2) loads
//           (2-way bank conflicts), STS.64
//   MODE 1: W / E from conflict-free addresses (wrong values; timing only)
//   MODE 2: no W / E loads (the pair's own cells stand in)
//   MODE 3: MODE 0 without the per-sweep barrier (wrong; timing only)
//   MODE 6: W / E by SHFL of the neighbour lanes' centre pair (+ one edge LDS)
//   MODE 9: W / E by one aligned LDS.64 (wrong cells; timing only)
//   MODE 10 (kernel kq): the quad walk, 4 columns per thread
//   MODE 11: odd rows take 2^x from a polynomial on the FMA pipe (fewer MUFU)
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/probes/adfsmem tools/probes/adfsmem.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

typedef uint64_t P2;
__device__ __forceinline__ P2 pk(float a, float b) { P2 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float plo(P2 r) { float a, b; asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); return a; }
__device__ __forceinline__ float phi(P2 r) { float a, b; asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); return b; }
__device__ __forceinline__ P2 padd(P2 a, P2 b) { P2 r; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ P2 psub(P2 a, P2 b) { P2 r; asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ P2 pmul(P2 a, P2 b) { P2 r; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ P2 pfma(P2 a, P2 b, P2 c) { P2 r; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__device__ __forceinline__ float ex2(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ P2 swp(P2 a) { return pk(phi(a), plo(a)); }

constexpr int kSW = 128, T = 4;

// 2^x for x <= 0 on the FMA pipe (+ integer exponent add): round-to-nearest
// range reduction by the 1.5 * 2^23 magic, degree-5 polynomial on [-0.5, 0.5]
__device__ __forceinline__ P2 pex2_poly(P2 x) {
    const P2 MAG = pk(12582912.0f, 12582912.0f);
    x = pk(fmaxf(plo(x), -126.f), fmaxf(phi(x), -126.f));
    const P2 t = padd(x, MAG);
    const P2 f = psub(x, psub(t, MAG));
    P2 q = pfma(f, pk(1.3333558e-3f, 1.3333558e-3f), pk(9.6181291e-3f, 9.6181291e-3f));
    q = pfma(q, f, pk(5.5504109e-2f, 5.5504109e-2f));
    q = pfma(q, f, pk(2.4022651e-1f, 2.4022651e-1f));
    q = pfma(q, f, pk(6.9314718e-1f, 6.9314718e-1f));
    q = pfma(q, f, pk(1.0f, 1.0f));
    const int n0 = __float_as_int(plo(t)) - 0x4B400000, n1 = __float_as_int(phi(t)) - 0x4B400000;
    return pk(__int_as_float(__float_as_int(plo(q)) + (n0 << 23)), __int_as_float(__float_as_int(phi(q)) + (n1 << 23)));
}

template <int MODE>
__device__ __forceinline__ P2 cell(P2 C, P2 N, P2 S, P2 P, P2 KC, P2 L2, P2 M4, bool poly = false) {
    const P2 Cs = swp(C);
    const P2 gx = psub(Cs, P), gy = psub(S, N);
    const P2 e = pfma(pfma(gx, gx, pmul(gy, gy)), KC, L2);
    const P2 lc = poly ? pex2_poly(e) : pk(ex2(plo(e)), ex2(phi(e)));
    const P2 lap = pfma(M4, C, padd(padd(N, S), padd(P, Cs)));
    return pfma(lc, lap, C);
}

template <int MODE, int SH, int PD>
__global__ void __launch_bounds__(256, 4) k(float* out, int reps, float kc, float l2lam) {
    extern __shared__ __align__(16) float sm[];
    float* b0 = sm;
    float* b1 = sm + kSW * (SH + 2);
    for (int i = threadIdx.x; i < kSW * (SH + 2); i += 256) {
        b0[i] = 1.0f + 1e-4f * (i & 63);
        b1[i] = b0[i];
    }
    __syncthreads();
    const P2 KC = pk(kc, kc), L2 = pk(l2lam, l2lam), M4 = pk(-4.f, -4.f);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int x = ((warp & 1) * 32 + lane) * 2;
    for (int rep = 0; rep < reps; ++rep) {
#pragma unroll 1
        for (int t = 1; t <= T; ++t) {
            const float* cur = (t & 1) ? b0 : b1;
            float* nxt = (t & 1) ? b1 : b0;
            const int ylo = t, yhi = SH - t;
            const int q = (yhi - ylo + 3) / 4;
            const int ys = ylo + (warp >> 1) * q, ye = min(ys + q, yhi);
            if (ys < ye) {                                  // warp-uniform (SHFL in MODE 6)
                const float* col = cur + x + ys * kSW;
                const float* colW = MODE == 1 ? cur + ys * kSW + (warp & 1) * 64 + lane : col - 1;
                const float* colE = MODE == 1 ? colW + 32 : col + 2;
                float* ocol = nxt + x + ys * kSW;
                auto ld2 = [](const float* a) { return *reinterpret_cast<const P2*>(a); };
                P2 C = ld2(col), N = ld2(col - kSW);
                P2 S = ld2(col + kSW);
                P2 S2 = PD == 2 ? ld2(col + 2 * kSW) : S;
                P2 Pn = (MODE == 2 || MODE == 6 || MODE == 9) ? C : pk(colW[0], colE[0]);
                const int n = ye - ys;
                auto step = [&]() {
                    const P2 S1 = PD == 2 ? S2 : ld2(col + 2 * kSW);
                    if (PD == 2) S2 = ld2(col + 3 * kSW);
                    P2 P1;
                    if (MODE == 2) {
                        P1 = S;
                    } else if (MODE == 6) {
                        float w = __shfl_up_sync(0xffffffffu, phi(S), 1);
                        float e = __shfl_down_sync(0xffffffffu, plo(S), 1);
                        const float edge = col[kSW + (lane == 0 ? -1 : 2)];   // the other column group's cell
                        if (lane == 0) w = edge;
                        if (lane == 31) e = edge;
                        P1 = pk(w, e);
                    } else if (MODE == 9) {
                        P1 = ld2(col + kSW + 2);          // one aligned 64-bit load (wrong cells; timing only)
                    } else {
                        P1 = pk(colW[kSW], colE[kSW]);
                    }
                    *reinterpret_cast<P2*>(ocol) = cell<MODE>(C, N, S, Pn, KC, L2, M4, MODE == 11 && (((ocol - nxt) >> 7) & 1));
                    N = C;
                    C = S;
                    S = S1;
                    Pn = P1;
                    col += kSW;
                    colW += kSW;
                    colE += kSW;
                    ocol += kSW;
                };
                int i = 0;
                for (; i + 4 <= n; i += 4) {
                    step(); step(); step(); step();
                }
                for (; i < n; ++i) step();
            }
            if (MODE != 3) __syncthreads();
        }
    }
    __syncthreads();
    out[blockIdx.x * 256 + threadIdx.x] = b0[threadIdx.x * 7 % (kSW * SH)];
}

// MODE 10: quad walk -- 4 columns per thread as two packed pairs, one warp
// per 128-column row strip, 8 row parts: per row one LDS.128 (south quad),
// scalar W (x-1) and E (x+4), one STS.128; the pairs' outer neighbours
// (W, c2) and (c1, E) built by register moves
template <int SH>
__global__ void __launch_bounds__(256, 4) kq(float* out, int reps, float kc, float l2lam) {
    extern __shared__ __align__(16) float sm[];
    float* b0 = sm;
    float* b1 = sm + kSW * (SH + 2);
    for (int i = threadIdx.x; i < kSW * (SH + 2); i += 256) {
        b0[i] = 1.0f + 1e-4f * (i & 63);
        b1[i] = b0[i];
    }
    __syncthreads();
    const P2 KC = pk(kc, kc), L2 = pk(l2lam, l2lam), M4 = pk(-4.f, -4.f);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int x = lane * 4;
    for (int rep = 0; rep < reps; ++rep) {
#pragma unroll 1
        for (int t = 1; t <= T; ++t) {
            const float* cur = (t & 1) ? b0 : b1;
            float* nxt = (t & 1) ? b1 : b0;
            const int ylo = t, yhi = SH - t;
            const int q = (yhi - ylo + 7) / 8;
            const int ys = ylo + warp * q, ye = min(ys + q, yhi);
            if (ys < ye) {
                const float* col = cur + x + ys * kSW;
                float* ocol = nxt + x + ys * kSW;
                const int offW = x == 0 ? 0 : -1, offE = x == kSW - 4 ? 3 : 4;
                auto ld4 = [](const float* a) { return *reinterpret_cast<const float4*>(a); };
                float4 C = ld4(col), N = ld4(col - kSW), S = ld4(col + kSW);
                float w = col[offW], e = col[offE];
                for (int y = ys; y < ye; ++y) {
                    const float4 S1 = ld4(col + 2 * kSW);
                    const float w1 = col[kSW + offW], e1 = col[kSW + offE];
                    const P2 c01 = pk(C.x, C.y), c23 = pk(C.z, C.w);
                    const P2 o0 = cell<0>(c01, pk(N.x, N.y), pk(S.x, S.y), pk(w, C.z), KC, L2, M4);
                    const P2 o1 = cell<0>(c23, pk(N.z, N.w), pk(S.z, S.w), pk(C.y, e), KC, L2, M4);
                    *reinterpret_cast<float4*>(ocol) = make_float4(plo(o0), phi(o0), plo(o1), phi(o1));
                    N = C; C = S; S = S1; w = w1; e = e1;
                    col += kSW; ocol += kSW;
                }
            }
            __syncthreads();
        }
    }
    out[blockIdx.x * 256 + threadIdx.x] = b0[threadIdx.x * 7 % (kSW * SH)];
}

template <int SH, int CPS>
void runq(const char* name) {
    int sms, clk;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const size_t smem = sizeof(float) * 2 * kSW * (SH + 2);
    cudaFuncSetAttribute(kq<SH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    float* o;
    const int blocks = sms * CPS * 8;
    cudaMalloc(&o, (size_t)blocks * 256 * 4);
    const int reps = 50;
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        kq<SH><<<blocks, 256, smem>>>(o, reps, -400.f, -2.7f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    double per_tile = 0;
    for (int t = 1; t <= T; ++t) per_tile += (double)(SH - 2 * t) * kSW;
    const double cells = per_tile * reps * blocks;
    const double cyc = best * 1e-3 * clk * 1e3;
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, kq<SH>);
    const double rate = cells / cyc / sms;
    printf("%-58s regs %3d  %.3f ms  %.2f cells/clk/SM  %.1f cyc per 64 cells per SMSP\n", name, fa.numRegs, best,
           rate, 4.0 * 64 / rate);
    cudaFree(o);
}

template <int MODE, int SH = 52, int CPS = 4, int PD = 1>
void run(const char* name) {
    int sms, clk;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const size_t smem = sizeof(float) * 2 * kSW * (SH + 2);
    cudaFuncSetAttribute(k<MODE, SH, PD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    float* o;
    const int blocks = sms * CPS * 8;
    cudaMalloc(&o, (size_t)blocks * 256 * 4);
    const int reps = 50;
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k<MODE, SH, PD><<<blocks, 256, smem>>>(o, reps, -400.f, -2.7f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    // cell-updates: per sweep t the region is (SH - 2t) rows x kSW columns
    double per_tile = 0;
    for (int t = 1; t <= T; ++t) per_tile += (double)(SH - 2 * t) * kSW;
    const double cells = per_tile * reps * blocks;
    const double cyc = best * 1e-3 * clk * 1e3;
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k<MODE, SH, PD>);
    const double rate = cells / cyc / sms;
    printf("%-58s regs %3d  %.3f ms  %.2f cells/clk/SM  %.1f cyc per 64 cells per SMSP\n", name, fa.numRegs, best,
           rate, 4.0 * 64 / rate);
    cudaFree(o);
}

int main() {
    run<0>("0 as adf.cu (LDS.64 S, conflicted W/E, STS.64, barrier)");
    run<1>("1 W/E conflict-free addresses");
    run<2>("2 no W/E loads");
    run<3>("3 no barrier");
    run<6>("6 W/E by SHFL + one edge LDS");
    run<9>("9 W/E as one aligned LDS.64 (1 instr, 2 wavefronts)");
    run<0, 52, 4, 2>("0, S loaded two rows ahead");
    run<0, 40, 5>("0, 40-row tile, 5 CTAs/SM (10 warps/SMSP)");
    run<0, 32, 6>("0, 32-row tile, 6 CTAs/SM (12 warps/SMSP)");
    run<2, 40, 5>("2, 40-row tile, 5 CTAs/SM");
    runq<52, 4>("10 quad walk (LDS.128, 2 pairs per thread)");
    run<11>("11 odd rows: exp2 by polynomial on the FMA pipe");
    run<0>("0 again");
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
