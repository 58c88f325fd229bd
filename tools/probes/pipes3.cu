// Microbenchmark (round 2): per-SM issue / pipe throughput of the
// instruction mixes the ADF and RANSAC inner loops are built from, on this
// B200.  Each kernel runs 8 independent chains per thread, 64 warps per SM.
// Output: warp-instructions per clock per SM and lane-ops per clock per SM.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/pipes3 tools/probes/pipes3.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define PK(a, b) asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b))

template <int OP>
__global__ void __launch_bounds__(512) k(float* out, int iters, float a, float b, float c) {
    __shared__ float4 sm[512 + 64];
    float x[8];
    uint64_t p[8];
    uint32_t cnt[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        x[j] = threadIdx.x * 1e-3f + j;
        asm("mov.b64 %0, {%1, %2};" : "=l"(p[j]) : "f"(x[j]), "f"(x[j] + 0.5f));
        cnt[j] = j;
    }
    sm[threadIdx.x] = make_float4(x[0], x[1], x[2], x[3]);
    __syncthreads();
    uint64_t pa, pb;
    asm("mov.b64 %0, {%1, %2};" : "=l"(pa) : "f"(a), "f"(b));
    asm("mov.b64 %0, {%1, %2};" : "=l"(pb) : "f"(c), "f"(a));
    float4 acc = make_float4(0, 0, 0, 0);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (OP == 0) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[j]) : "f"(a), "f"(b));
            if (OP == 1) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[j]) : "l"(pa), "l"(pb));
            if (OP == 2) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[j]) : "l"(pa));
            if (OP == 3) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[j]));
            if (OP == 4) {   // FSETP |x| < c + predicated IADD
                asm volatile("{.reg .pred q; setp.lt.f32 q, %1, %2; @q add.u32 %0, %0, 1;}"
                             : "+r"(cnt[j]) : "f"(fabsf(x[j])), "f"(c));
                asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(x[j]) : "f"(a));
            }
            if (OP == 5) asm volatile("add.u32 %0, %0, %1;" : "+r"(cnt[j]) : "r"(cnt[(j + 1) & 7]));
            if (OP == 6) asm volatile("shfl.sync.idx.b32 %0, %0, %1, 31, -1;" : "+f"(x[j]) : "r"((int)(threadIdx.x + 1) & 31));
            if (OP == 7) {
                float4 v = sm[(threadIdx.x + j * 7 + i) & 511];
                acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
            }
            if (OP == 8) asm volatile("fma.rn.f32 %0, %0, 0f3F800347, 0f3A83126F;" : "+f"(x[j]));
            if (OP == 9) {   // ADF-like mix: 5 FFMA2 : 1 MUFU
                asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[j]) : "l"(pa), "l"(pb));
                if ((j % 5) == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[j]));
            }
            if (OP == 10) {   // LEA.HI sign-bit accumulate: cnt += x >> 31 (unsigned)
                asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(x[j]) : "f"(a));
                asm volatile("{.reg .u32 t; shr.u32 t, %1, 31; add.u32 %0, %0, t;}" : "+r"(cnt[j]) : "r"(__float_as_uint(x[j])));
            }
            if (OP == 11) asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(p[j]) : "l"(pa));
            if (OP == 12) {   // FFMA2 with one scalar-broadcast operand (pa) and a register pair
                asm volatile("fma.rn.f32x2 %0, %1, %0, %2;" : "+l"(p[j]) : "l"(pa), "l"(p[(j + 1) & 7]));
            }
            if (OP == 13) asm volatile("fma.rn.f32 %0, %0, %1, %0;" : "+f"(x[j]) : "f"(a));
        }
    }
    float s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        float lo, hi;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(p[j]));
        s += x[j] + lo + hi + (float)cnt[j];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc.x + acc.y + acc.z + acc.w;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* o;
    cudaMalloc(&o, sms * 4 * 512 * 4);
    const char* names[] = {"FFMA 3reg", "FFMA2", "FADD2", "MUFU.EX2", "FSETP+IADD(+FADD)", "IADD",
                           "SHFL", "LDS.128(+4FADD)", "FFMA imm", "5FFMA2:1EX2 (per FFMA2)",
                           "FADD+SHR+IADD", "FMUL2", "FFMA2 chain-pairs", "FFMA 2reg"};
    // warp-instructions issued per j-iteration (for the per-instr rate)
    const double wi[] = {1, 1, 1, 1, 3, 1, 1, 5, 1, 1.2, 3, 1, 1, 1};
    const double lanes[] = {1, 2, 2, 1, 1, 1, 1, 1, 1, 2, 1, 2, 2, 1};
    for (int op = 0; op < 14; ++op) {
        void (*fn)(float*, int, float, float, float) = nullptr;
        switch (op) {
            case 0: fn = k<0>; break; case 1: fn = k<1>; break; case 2: fn = k<2>; break;
            case 3: fn = k<3>; break; case 4: fn = k<4>; break; case 5: fn = k<5>; break;
            case 6: fn = k<6>; break; case 7: fn = k<7>; break; case 8: fn = k<8>; break;
            case 9: fn = k<9>; break; case 10: fn = k<10>; break; case 11: fn = k<11>; break;
            case 12: fn = k<12>; break; case 13: fn = k<13>; break;
        }
        const int iters = 2048;
        float best = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            fn<<<sms * 4, 512>>>(o, iters, 0.9999f, 1e-4f, 0.5f);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        int clk_khz;
        cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
        const double warps = (double)sms * 4 * 512 / 32;
        const double winstr = warps * iters * 8 * wi[op];
        const double cyc = best * 1e-3 * clk_khz * 1e3;   // at max clock (approximation)
        printf("%-28s %.3f ms  warp-instr/clk/SM %.2f  main-op lanes/clk/SM %.1f\n", names[op], best,
               winstr / cyc / sms, warps * iters * 8 * 32 * lanes[op] / cyc / sms);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
