// Microbenchmark: per-SM throughput of MUFU.EX2, FFMA (3 reg), FADD on this GPU.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(float* out, int iters, float a, float b) {
    float x0 = threadIdx.x * 1e-3f, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#define OP1(x)                                                                     \
    if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x));             \
    if (OP == 1) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x) : "f"(a), "f"(b)); \
    if (OP == 2) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(x) : "f"(a));
        OP1(x0) OP1(x1) OP1(x2) OP1(x3) OP1(x4) OP1(x5) OP1(x6) OP1(x7)
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float* o; cudaMalloc(&o, sms * 8 * 1024 * 4);
    const char* names[] = {"ex2.approx", "ffma", "fadd"};
    for (int op = 0; op < 3; ++op) {
        int iters = 4096;
        auto fn = op == 0 ? k<0> : op == 1 ? k<1> : k<2>;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            fn<<<sms * 4, 512>>>(o, iters, 0.999f, 1e-3f);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            double ops = (double)sms * 4 * 512 * iters * 8;
            printf("%-10s %.3f ms  %.3e ops/s  = %.1f ops/clk/SM at %d MHz max\n", names[op], ms, ops / (ms * 1e-3),
                   ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
        }
    }
    return 0;
}
