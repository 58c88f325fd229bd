// Dependent-chain latency (cycles) of FFMA, FFMA2, FADD2, MUFU.EX2, LDS.64 on one warp.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
template <int OP>
__global__ void k(float* out, long long* cyc, float a, float b) {
    __shared__ float2 sm[64];
    sm[threadIdx.x] = make_float2(0.f, 0.f);
    __syncthreads();
    float x = threadIdx.x * 1e-3f;
    float2 t = make_float2(x, x);
    u64 y = *reinterpret_cast<u64*>(&t);
    float2 ab = make_float2(a, a), bb = make_float2(b, b);
    u64 A = *reinterpret_cast<u64*>(&ab), B = *reinterpret_cast<u64*>(&bb);
    int idx = threadIdx.x;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 256; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            if (OP == 0) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x) : "f"(a), "f"(b));
            if (OP == 1) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(y) : "l"(A), "l"(B));
            if (OP == 2) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(y) : "l"(A));
            if (OP == 3) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x));
            if (OP == 4) { float2 v = sm[idx & 63]; idx = __float_as_int(v.x) + threadIdx.x; }
        }
    }
    long long t1 = clock64();
    float2 r = *reinterpret_cast<float2*>(&y);
    out[threadIdx.x] = x + r.x + idx;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    float* o; long long* c; cudaMalloc(&o, 4096); cudaMalloc(&c, 8);
    const char* names[] = {"ffma", "ffma2", "fadd2", "ex2", "lds.64"};
    for (int op = 0; op < 5; ++op) {
        auto fn = op == 0 ? k<0> : op == 1 ? k<1> : op == 2 ? k<2> : op == 3 ? k<3> : k<4>;
        for (int rep = 0; rep < 2; ++rep) {
            fn<<<1, 32>>>(o, c, 0.999f, 1e-3f);
            long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
            if (rep) printf("%-8s %.2f cycles/op\n", names[op], h / 4096.0);
        }
    }
    return 0;
}
