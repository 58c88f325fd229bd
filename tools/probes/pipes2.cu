// Microbenchmark: FFMA vs packed FFMA2/FADD2 (sm_100a f32x2) throughput per SM,
// and an ADF-like mix (5 FFMA2 : 1 MUFU.EX2 : 2 LDS.64).
#include <cstdio>
#include <cuda_runtime.h>

typedef unsigned long long u64;

template <int OP>
__global__ void k(float* out, int iters, float a, float b) {
    __shared__ float2 sm[1024];
    sm[threadIdx.x] = make_float2(threadIdx.x, 1.f);
    __syncthreads();
    float x[8];
    u64 y[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) { x[j] = threadIdx.x * 1e-3f + j; float2 t = make_float2(x[j], x[j] + 0.5f); y[j] = *reinterpret_cast<u64*>(&t); }
    float2 ab = make_float2(a, a), bb = make_float2(b, b);
    u64 A = *reinterpret_cast<u64*>(&ab), B = *reinterpret_cast<u64*>(&bb);
    const float2* p = sm + (threadIdx.x & 511);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (OP == 0) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[j]) : "f"(a), "f"(b));
            if (OP == 1) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(y[j]) : "l"(A), "l"(B));
            if (OP == 2) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(y[j]) : "l"(A));
            if (OP == 3) {
                asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(y[j]) : "l"(A), "l"(B));
                asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(y[j]) : "l"(A), "l"(B));
                asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(y[j]) : "l"(A), "l"(B));
                asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(y[j]) : "l"(A), "l"(B));
                asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(y[j]) : "l"(A), "l"(B));
                if (j & 1) {
                    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[j]));
                    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[j - 1]));
                    float2 q = p[(i * 8 + j) & 511 ? 32 : 0];
                    x[j] += q.x;
                }
            }
        }
    }
    float s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) { float2 t = *reinterpret_cast<float2*>(&y[j]); s += x[j] + t.x + t.y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float* o; cudaMalloc(&o, sms * 8 * 1024 * 4);
    const char* names[] = {"ffma", "ffma2", "fadd2", "mix 5ffma2:1ex2"};
    const double per[] = {8, 16, 16, 80};  // fp32 lane-ops per thread per iteration
    for (int op = 0; op < 4; ++op) {
        int iters = 4096;
        auto fn = op == 0 ? k<0> : op == 1 ? k<1> : op == 2 ? k<2> : k<3>;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            fn<<<sms * 4, 512>>>(o, iters, 0.999f, 1e-3f);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            double ops = (double)sms * 4 * 512 * iters * per[op];
            printf("%-16s %.3f ms  %.1f fp32 lane-ops/clk/SM at %d MHz max\n", names[op], ms,
                   ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
        }
    }
    return 0;
}
