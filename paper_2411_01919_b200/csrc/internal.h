// internal.h — launch functions behind the C ABI (not exported).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/pmap.h"

#include <nvtx3/nvToolsExt.h>

namespace pm {

// NVTX range around a C-ABI call (header-only NVTX v3: a no-op unless a tool
// such as nsys / ncu injects itself), so host timelines show the pmap calls.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// ---- adf.cu
cudaError_t adf_setup_attributes();
int adf_default_iters_per_pass();
// byte offset of the per-frame validity flags inside the adf workspace
size_t adf_flags_offset(int W, int H, int B);
size_t adf_flags_region_bytes(int W, int H, int B);   // frame flags + per-tile hole lists
// lambda bound under which a frame whose ADF flag is 0 (every input depth
// valid and in [2^-100, 2^100), adf.cu fast_depth) filters to valid depths only
constexpr float kNoCheckMaxLambda = 0.249f;
// in -> out (B frames); ws: B*H*W floats (used when >= 2 passes); normals nullable.
cudaError_t adf_run(const float* in, float* out, float* normals, float* ws, int W, int H, int B,
                    const pm_intrinsics* K, float lam, float kappa, int iters, int iters_per_pass,
                    int scheme, int nmode, int engine, cudaStream_t stream);
// ---- adf_reg.cu (register-tile engine; the pass launcher is declared in adf_cell.cuh)
cudaError_t adf_reg_setup_attributes();
cudaError_t normals_run(const float* depth, float* normals, int W, int H, int B,
                        const pm_intrinsics* K, int nmode, cudaStream_t stream);

// ---- api.cu: the argument checks of pm_process_frames, without launching
pm_status pipeline_validate(int32_t W, int32_t H, int32_t B, const pm_intrinsics* K, float lam, float kappa,
                            int32_t iters, int32_t R, int32_t n_hyp, float tau);

// ---- compact.cu / ransac.cu
struct Sums;
struct RansacWorkspace {
    // sizes
    int W, H, B, R, n_hyp, n_hyp_pad, sub_tile, n_sub, n_slots;
    int score_K, score_L;  // scoring layout: K hypotheses per lane, L lanes per group (K * L >= n_hyp)
    // buffers (device)
    uint2* points;        // [B][W*H] packed (u | v<<16, z bits), region-major, raster order
    int32_t* hist;        // [B][R][n_sub] count -> exclusive prefix per region
    int32_t* region_cnt;  // [B][R]
    int32_t* region_off;  // [B][R+1]
    float4* planes;       // [B][R][n_hyp_pad] hypothesis planes (NaN = invalid)
    float2* pairs;        // [B][R][K/2][L][4] plane pairs (h, h + L) per component, for packed scoring
    int32_t* counts;      // [B][R][n_hyp_pad] inlier counts (-1 = invalid)
    uint64_t* errq;       // [B][R][n_hyp_pad] fixed-point error sums (select=ERROR / debug)
    Sums* slots;          // [B][n_slots] refit moments per (region, chunk): slot chunk + region
    int32_t* best;        // [B][R] selected hypothesis (-1: none)
    size_t total_bytes;
};
// Carve `base` (nullable: sizing only) into the ransac workspace.
RansacWorkspace ransac_workspace_layout(void* base, int W, int H, int R, int n_hyp, int B);

// depth_all_valid (nullable): per-frame flags, 0 = every depth of the frame is
// known valid (pm_process_frames passes the ADF's fast-depth flags), so the
// count reads labels only
cudaError_t compact_run(const float* depth, const int32_t* labels, const RansacWorkspace& ws,
                        cudaStream_t stream, const int* depth_all_valid = nullptr);

struct RansacArgs {
    pm_intrinsics K;
    float tau;
    uint64_t seed;
    uint32_t first_frame;
    int sampler;
    int select;
    int32_t* counts_out;   // nullable debug
    uint64_t* errq_out;    // nullable debug
    void* const* stage_events;   // nullable: 4 cudaEvent_t recorded after hyp, score, refit, finalize
};
cudaError_t ransac_setup_attributes();
cudaError_t ransac_run(const RansacWorkspace& ws, const RansacArgs& a, pm_plane* planes,
                       cudaStream_t stream);

}  // namespace pm
