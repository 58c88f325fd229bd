// Microbenchmark (round 2): the Alg. 1 cell update (10 packed FP32 ops + 2
// MUFU.EX2 per pair of cells) on NP independent register pairs per thread,
// no shared memory and no barriers -- the attainable sweep rate of a
// register-resident ADF at a given occupancy.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/probes/adfmix tools/probes/adfmix.cu
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

template <int NC, int NR, int MODE>
__global__ void k(float* out, int iters, float kc, float l2lam) {
    P2 A[NC][NR], B[NC][NR];
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int i = 0; i < NR; ++i) A[c][i] = pk(1.0f + 1e-3f * (threadIdx.x + c + i), 1.5f + 1e-3f * (c * i));
    const P2 KC = pk(kc, kc), L2 = pk(l2lam, l2lam), M4 = pk(-4.f, -4.f);
    auto sweep = [&](P2 (&X)[NC][NR], P2 (&Y)[NC][NR]) {
#pragma unroll
        for (int i = 0; i < NR; ++i)
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const P2 C = X[c][i];
                const P2 N = X[c][(i + NR - 1) % NR], S = X[c][(i + 1) % NR];
                const P2 W = X[(c + NC - 1) % NC][i], E = X[(c + 1) % NC][i];
                const P2 gx2 = psub(E, W), gy2 = psub(S, N);
                const P2 g2 = pfma(gx2, gx2, pmul(gy2, gy2));
                const P2 e = pfma(g2, KC, L2);
                const P2 lc = MODE == 0 ? pk(ex2(plo(e)), ex2(phi(e))) : e;
                const P2 lap = pfma(M4, C, padd(padd(N, S), padd(W, E)));
                Y[c][i] = pfma(lc, lap, C);
            }
    };
    for (int it = 0; it < iters; ++it) {
        sweep(A, B);
        sweep(B, A);
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int i = 0; i < NR; ++i) s += plo(A[c][i]) + phi(A[c][i]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NC, int NR, int MODE>
void run(const char* name, int threads, int blocks_per_sm) {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float* o;
    cudaMalloc(&o, (size_t)sms * blocks_per_sm * threads * 4);
    const int iters = 200;
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k<NC, NR, MODE><<<sms * blocks_per_sm, threads>>>(o, iters, -400.f, -2.7f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double cells = (double)sms * blocks_per_sm * threads * iters * 2 * NC * NR * 2;
    const double cyc = best * 1e-3 * clk * 1e3;
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k<NC, NR, MODE>);
    printf("%-34s regs %3d  %.3f ms  %.2f cells/clk/SM  (%.1f cyc per pair-group per SMSP)\n", name, fa.numRegs, best,
           cells / cyc / sms, 4.0 * 64 / (cells / cyc / sms));
    cudaFree(o);
}

int main() {
    run<4, 4, 0>("4x4 pairs, 512 thr x1 (4 w/SMSP)", 512, 1);
    run<4, 4, 0>("4x4 pairs, 256 thr x2 (4 w/SMSP)", 256, 2);
    run<4, 2, 0>("4x2 pairs, 256 thr x4 (8 w/SMSP)", 256, 4);
    run<2, 2, 0>("2x2 pairs, 256 thr x8 (16 w/SMSP)", 256, 8);
    run<4, 4, 1>("4x4 no MUFU, 512x1", 512, 1);
    run<4, 2, 1>("4x2 no MUFU, 256x4", 256, 4);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
