// Standalone probe of the TMA path used by adf.cu (debug tool).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../../paper_2411_01919_b200/csrc/common.cuh"

template <int MODE>
__global__ void k(const __grid_constant__ CUtensorMap tmap, float* out, int x0, int y0, int boxW, int boxH) {
    extern __shared__ __align__(128) float sm[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) pm::mbar_init(&bar, 1);
    __syncthreads();
    if (threadIdx.x == 0) {
        pm::mbar_arrive_expect_tx(&bar, boxW * boxH * 4);
        if (MODE == 0) {
            pm::tma_load_3d(sm, &tmap, x0, y0, 0, &bar);
        } else {
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(pm::smem_u32(sm)), "l"((uint64_t)&tmap), "r"(x0), "r"(y0), "r"(0), "r"(pm::smem_u32(&bar)) : "memory");
        }
    }
    pm::mbar_wait(&bar, 0);
    for (int i = threadIdx.x; i < boxW * boxH; i += blockDim.x) out[i] = sm[i];
}

int main(int argc, char** argv) {
    int only = argc > 1 ? atoi(argv[1]) : -1;
    int W = 64, H = 48;
    float* d; cudaMalloc(&d, W * H * 4);
    float h[64 * 48]; for (int i = 0; i < W * H; ++i) h[i] = 1 + i;
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    float* o; cudaMalloc(&o, 128 * 128 * 4);
    struct { int boxW, boxH, x0, y0; } cases[] = {{64, 48, -3, 0}, {64, 48, -5, 0}, {64, 32, -4, -3}, {32, 16, 3, 0}, {32, 16, 1, 1}, {32, 16, 2, 5}, {64, 32, -8, -3}, {32, 16, 6, 1}};
    int ci = -1;
    for (int mode = 0; mode < 1; ++mode)
    for (auto c : cases) {
        ++ci; if (only >= 0 && ci != only) continue;
        CUtensorMap m;
        bool ok = pm::make_tmap_f32_3d(&m, d, W, H, 1, c.boxW, c.boxH);
        cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 128 * 4);
        cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 128 * 4);
        if (!ok) { printf("box %dx%d rejected by encode\n", c.boxW, c.boxH); continue; }
        if (mode == 0) k<0><<<1, 128, c.boxW * c.boxH * 4>>>(m, o, c.x0, c.y0, c.boxW, c.boxH);
        else k<1><<<1, 128, c.boxW * c.boxH * 4>>>(m, o, c.x0, c.y0, c.boxW, c.boxH);
        cudaError_t e = cudaDeviceSynchronize();
        float r[4] = {0};
        if (e == cudaSuccess) cudaMemcpy(r, o, 16, cudaMemcpyDeviceToHost);
        printf("mode %d box %dx%d at (%d,%d): encode=%d err=%s first=%g %g %g\n", mode, c.boxW, c.boxH, c.x0, c.y0, ok,
               cudaGetErrorString(e), r[0], r[1], r[2]);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
