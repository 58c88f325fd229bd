// api.cu — the C ABI of include/pmap.h: argument validation, workspace
// carving and launch sequencing on the caller's stream.  No allocation on the
// hot path; the only global state is the one-time (per device) kernel attribute setup.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <mutex>

#include "../../include/pmap.h"
#include "internal.h"

namespace {

constexpr int32_t kVersion = 200;   // 0.2.0: pm_ransac_options.stage_events, PM_LABELS_RUNS, pm_process_frames_host_async, PM_ADF_ENGINE_REG / _HOLES

// Kernel attributes (> 48 KB dynamic shared memory) are per device context:
// set once per device, on first use from any thread.
constexpr int kMaxDevices = 64;
std::once_flag g_once[kMaxDevices];
cudaError_t g_setup_err[kMaxDevices];

cudaError_t setup() {
    int dev = 0;
    if (cudaError_t e = cudaGetDevice(&dev); e != cudaSuccess) return e;
    if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
    std::call_once(g_once[dev], [dev] {
        cudaError_t e = pm::adf_setup_attributes();
        if (e == cudaSuccess) e = pm::adf_reg_setup_attributes();
        if (e == cudaSuccess) e = pm::ransac_setup_attributes();
        g_setup_err[dev] = e;
    });
    return g_setup_err[dev];
}

bool finite_pos(float x) { return x > 0.0f && isfinite(x); }

bool dims_ok(int32_t W, int32_t H, int32_t B) {
    return W >= 3 && H >= 3 && W <= 65535 && H <= 65535 && B >= 1 && B <= 65535;
}

bool intrinsics_ok(const pm_intrinsics* K) {
    return K && finite_pos(K->fx) && finite_pos(K->fy) && isfinite(K->cx) && isfinite(K->cy);
}

bool overlap(const void* a, size_t na, const void* b, size_t nb) {
    const char* pa = (const char*)a;
    const char* pb = (const char*)b;
    return pa < pb + nb && pb < pa + na;
}

bool aligned256(const void* p) { return ((uintptr_t)p & 255u) == 0; }

pm_status cuda_status(cudaError_t e) { return e == cudaSuccess ? PM_OK : PM_ERR_CUDA; }

pm_status adf_impl(const float* in, float* out, int32_t W, int32_t H, int32_t B, const pm_intrinsics* K,
                   float lam, float kappa, int32_t iters, float* normals, void* ws, size_t ws_bytes,
                   int32_t iters_per_pass, int32_t scheme, int32_t nmode, int32_t engine, cudaStream_t stream) {
    const pm::NvtxRange nvtx_("pmap:adf_filter");
    if (engine != PM_ADF_ENGINE_AUTO && engine != PM_ADF_ENGINE_TILED && engine != PM_ADF_ENGINE_REG &&
        engine != PM_ADF_ENGINE_HOLES)
        return PM_ERR_INVALID_ARGUMENT;
    if (scheme != PM_ADF_ALG1 && scheme != PM_ADF_DIVERGENCE) return PM_ERR_INVALID_ARGUMENT;
    if (nmode != PM_NORMALS_GEOMETRIC && nmode != PM_NORMALS_AS_PRINTED) return PM_ERR_INVALID_ARGUMENT;
    if (!in || !out || !dims_ok(W, H, B) || iters < 0) return PM_ERR_INVALID_ARGUMENT;
    // the kernels write rows as float4 / bulk copies: 16-byte aligned outputs
    if (((reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(normals)) & 15) != 0)
        return PM_ERR_INVALID_ARGUMENT;
    if (!(lam > 0.0f && lam <= 0.25f) || !finite_pos(kappa)) return PM_ERR_INVALID_ARGUMENT;
    if (normals && !intrinsics_ok(K)) return PM_ERR_INVALID_ARGUMENT;
    const size_t bytes = sizeof(float) * (size_t)B * W * H;
    if (overlap(in, bytes, out, bytes)) return PM_ERR_INVALID_ARGUMENT;
    if (normals && (overlap(normals, 3 * bytes, in, bytes) || overlap(normals, 3 * bytes, out, bytes)))
        return PM_ERR_INVALID_ARGUMENT;
    if (iters_per_pass < 0 || iters_per_pass > 16) return PM_ERR_INVALID_ARGUMENT;   // 16 = adf.cu kMaxItersPerPass
    // the ping-pong workspace is required whenever one pass does not hold all the sweeps
    const int T = iters_per_pass > 0 ? iters_per_pass : pm::adf_default_iters_per_pass();
    const bool needs_ws = iters > T;
    if (needs_ws && (!ws || ws_bytes < pm_adf_workspace_bytes(W, H, B) || !aligned256(ws))) return PM_ERR_WORKSPACE;
    if (needs_ws && (overlap(ws, bytes, in, bytes) || overlap(ws, bytes, out, bytes))) return PM_ERR_INVALID_ARGUMENT;
    if (cudaError_t e = setup(); e != cudaSuccess) return PM_ERR_CUDA;
    return cuda_status(pm::adf_run(in, out, normals, (float*)ws, W, H, B, K, lam, kappa, iters,
                                   iters_per_pass, scheme, nmode, engine, stream));
}

pm_status ransac_impl(const float* depth, int32_t W, int32_t H, int32_t B, uint32_t first_frame,
                      const pm_intrinsics* K, const int32_t* labels, int32_t R, int32_t n_hyp,
                      float tau, uint64_t seed, pm_plane* planes, void* ws, size_t ws_bytes,
                      const pm_ransac_options* opt, cudaStream_t stream, const int* depth_all_valid = nullptr) {
    const pm::NvtxRange nvtx_("pmap:ransac_planes");
    if (!depth || !labels || !dims_ok(W, H, B) || !intrinsics_ok(K)) return PM_ERR_INVALID_ARGUMENT;
    if (R < 0 || R > 65536 || n_hyp < 1 || n_hyp > 4096 || !finite_pos(tau)) return PM_ERR_INVALID_ARGUMENT;
    if (R > 0 && !planes) return PM_ERR_INVALID_ARGUMENT;
    int sampler = PM_SAMPLER_PHILOX, select = PM_SELECT_COUNT;
    int32_t* counts_out = nullptr;
    uint64_t* errq_out = nullptr;
    void* const* ev = nullptr;
    if (opt) {
        sampler = opt->sampler;
        select = opt->select;
        counts_out = opt->counts_out;
        errq_out = opt->errq_out;
        ev = opt->stage_events;
        if (sampler != PM_SAMPLER_PHILOX && sampler != PM_SAMPLER_ENUMERATE) return PM_ERR_INVALID_ARGUMENT;
        if (select < PM_SELECT_COUNT || select > PM_SELECT_ERROR_EARLY) return PM_ERR_INVALID_ARGUMENT;
    }
    if (R == 0) return PM_OK;
    const size_t need = pm_ransac_workspace_bytes(W, H, R, n_hyp, B);
    if (!ws || ws_bytes < need || !aligned256(ws)) return PM_ERR_WORKSPACE;
    if (cudaError_t e = setup(); e != cudaSuccess) return PM_ERR_CUDA;
    const pm::RansacWorkspace L = pm::ransac_workspace_layout(ws, W, H, R, n_hyp, B);
    if (ev && cudaEventRecord((cudaEvent_t)ev[0], stream) != cudaSuccess) return PM_ERR_CUDA;
    cudaError_t e = pm::compact_run(depth, labels, L, stream, depth_all_valid);
    if (e != cudaSuccess) return PM_ERR_CUDA;
    if (ev && cudaEventRecord((cudaEvent_t)ev[1], stream) != cudaSuccess) return PM_ERR_CUDA;
    pm::RansacArgs a;
    a.K = *K;
    a.tau = tau;
    a.seed = seed;
    a.first_frame = first_frame;
    a.sampler = sampler;
    a.select = select;
    a.counts_out = counts_out;
    a.errq_out = errq_out;
    a.stage_events = ev ? ev + 2 : nullptr;
    return cuda_status(pm::ransac_run(L, a, planes, stream));
}

}  // namespace

namespace pm {
pm_status pipeline_validate(int32_t W, int32_t H, int32_t B, const pm_intrinsics* K, float lam, float kappa,
                            int32_t iters, int32_t R, int32_t n_hyp, float tau) {
    if (!dims_ok(W, H, B) || !intrinsics_ok(K) || iters < 0) return PM_ERR_INVALID_ARGUMENT;
    if (!(lam > 0.0f && lam <= 0.25f) || !finite_pos(kappa)) return PM_ERR_INVALID_ARGUMENT;
    if (R < 0 || R > 65536 || n_hyp < 1 || n_hyp > 4096 || !finite_pos(tau)) return PM_ERR_INVALID_ARGUMENT;
    return PM_OK;
}
}  // namespace pm

extern "C" {

PM_API size_t pm_adf_workspace_bytes(int32_t W, int32_t H, int32_t n_frames) {
    if (W < 1 || H < 1 || n_frames < 1) return 0;
    return pm::adf_flags_offset(W, H, n_frames) + pm::adf_flags_region_bytes(W, H, n_frames);
}

PM_API pm_status pm_adf_filter(const float* depth_in, float* depth_out, int32_t W, int32_t H,
                               const pm_intrinsics* K, float lambda, float kappa, int32_t iters,
                               float* normals_out, void* workspace, size_t ws_bytes, pm_stream_t stream) {
    return adf_impl(depth_in, depth_out, W, H, 1, K, lambda, kappa, iters, normals_out, workspace,
                    ws_bytes, 0, PM_ADF_ALG1, PM_NORMALS_GEOMETRIC, PM_ADF_ENGINE_AUTO, (cudaStream_t)stream);
}

PM_API pm_status pm_adf_filter_batched(const float* depth_in, float* depth_out, int32_t W, int32_t H,
                                       int32_t n_frames, const pm_intrinsics* K, float lambda,
                                       float kappa, int32_t iters, float* normals_out, void* workspace,
                                       size_t ws_bytes, pm_stream_t stream) {
    return adf_impl(depth_in, depth_out, W, H, n_frames, K, lambda, kappa, iters, normals_out, workspace,
                    ws_bytes, 0, PM_ADF_ALG1, PM_NORMALS_GEOMETRIC, PM_ADF_ENGINE_AUTO, (cudaStream_t)stream);
}

PM_API pm_status pm_adf_filter_ex(const float* depth_in, float* depth_out, int32_t W, int32_t H,
                                  int32_t n_frames, const pm_intrinsics* K, float lambda, float kappa,
                                  int32_t iters, float* normals_out, void* workspace, size_t ws_bytes,
                                  const pm_adf_options* opt, pm_stream_t stream) {
    return adf_impl(depth_in, depth_out, W, H, n_frames, K, lambda, kappa, iters, normals_out, workspace,
                    ws_bytes, opt ? opt->iters_per_pass : 0, opt ? opt->scheme : PM_ADF_ALG1,
                    opt ? opt->normals_mode : PM_NORMALS_GEOMETRIC, opt ? opt->engine : PM_ADF_ENGINE_AUTO,
                    (cudaStream_t)stream);
}

PM_API pm_status pm_normals_from_depth(const float* depth, int32_t W, int32_t H, const pm_intrinsics* K,
                                       float* normals_out, pm_stream_t stream) {
    return pm_normals_from_depth_batched(depth, W, H, 1, K, normals_out, stream);
}

PM_API pm_status pm_normals_from_depth_batched(const float* depth, int32_t W, int32_t H, int32_t n_frames,
                                               const pm_intrinsics* K, float* normals_out,
                                               pm_stream_t stream) {
    return pm_normals_from_depth_ex(depth, W, H, n_frames, K, PM_NORMALS_GEOMETRIC, normals_out, stream);
}

PM_API pm_status pm_normals_from_depth_ex(const float* depth, int32_t W, int32_t H, int32_t n_frames,
                                          const pm_intrinsics* K, int32_t mode, float* normals_out,
                                          pm_stream_t stream) {
    const pm::NvtxRange nvtx_("pmap:normals_from_depth");
    if (!depth || !normals_out || !dims_ok(W, H, n_frames) || !intrinsics_ok(K)) return PM_ERR_INVALID_ARGUMENT;
    if ((reinterpret_cast<uintptr_t>(normals_out) & 15) != 0) return PM_ERR_INVALID_ARGUMENT;   // float4 rows
    if (mode != PM_NORMALS_GEOMETRIC && mode != PM_NORMALS_AS_PRINTED) return PM_ERR_INVALID_ARGUMENT;
    const size_t bytes = sizeof(float) * (size_t)n_frames * W * H;
    if (overlap(depth, bytes, normals_out, 3 * bytes)) return PM_ERR_INVALID_ARGUMENT;
    if (cudaError_t e = setup(); e != cudaSuccess) return PM_ERR_CUDA;
    return cuda_status(pm::normals_run(depth, normals_out, W, H, n_frames, K, mode, (cudaStream_t)stream));
}

PM_API size_t pm_ransac_workspace_bytes(int32_t W, int32_t H, int32_t n_regions, int32_t n_hyp,
                                        int32_t n_frames) {
    if (W < 1 || H < 1 || n_regions < 0 || n_hyp < 1 || n_frames < 1) return 0;
    return pm::ransac_workspace_layout(nullptr, W, H, n_regions, n_hyp, n_frames).total_bytes;
}

PM_API pm_status pm_ransac_planes(const float* depth, int32_t W, int32_t H, const pm_intrinsics* K,
                                  const int32_t* region_labels, int32_t n_regions, int32_t n_hyp,
                                  float inlier_thresh, uint64_t seed, pm_plane* planes_out, void* workspace,
                                  size_t ws_bytes, pm_stream_t stream) {
    return ransac_impl(depth, W, H, 1, 0u, K, region_labels, n_regions, n_hyp, inlier_thresh, seed, planes_out,
                       workspace, ws_bytes, nullptr, (cudaStream_t)stream);
}

PM_API pm_status pm_ransac_planes_batched(const float* depth, int32_t W, int32_t H, int32_t n_frames,
                                          uint32_t first_frame_id, const pm_intrinsics* K,
                                          const int32_t* region_labels, int32_t n_regions, int32_t n_hyp,
                                          float inlier_thresh, uint64_t seed, pm_plane* planes_out,
                                          void* workspace, size_t ws_bytes, pm_stream_t stream) {
    return ransac_impl(depth, W, H, n_frames, first_frame_id, K, region_labels, n_regions, n_hyp, inlier_thresh,
                       seed, planes_out, workspace, ws_bytes, nullptr, (cudaStream_t)stream);
}

PM_API pm_status pm_ransac_planes_ex(const float* depth, int32_t W, int32_t H, int32_t n_frames,
                                     uint32_t first_frame_id, const pm_intrinsics* K,
                                     const int32_t* region_labels, int32_t n_regions, int32_t n_hyp,
                                     float inlier_thresh, uint64_t seed, pm_plane* planes_out, void* workspace,
                                     size_t ws_bytes, const pm_ransac_options* opt, pm_stream_t stream) {
    return ransac_impl(depth, W, H, n_frames, first_frame_id, K, region_labels, n_regions, n_hyp, inlier_thresh,
                       seed, planes_out, workspace, ws_bytes, opt, (cudaStream_t)stream);
}

PM_API size_t pm_pipeline_workspace_bytes(int32_t W, int32_t H, int32_t n_regions, int32_t n_hyp,
                                          int32_t n_frames) {
    const size_t a = pm_adf_workspace_bytes(W, H, n_frames);
    const size_t r = pm_ransac_workspace_bytes(W, H, n_regions, n_hyp, n_frames);
    return a > r ? a : r;   // adf's ping-pong buffer is dead before ransac starts
}

PM_API pm_status pm_process_frames(const float* depth_in, const int32_t* region_labels, int32_t W, int32_t H,
                                   int32_t n_frames, uint32_t first_frame_id, const pm_intrinsics* K,
                                   float lambda, float kappa, int32_t iters, int32_t n_regions, int32_t n_hyp,
                                   float inlier_thresh, uint64_t seed, float* depth_out, float* normals_out,
                                   pm_plane* planes_out, void* workspace, size_t ws_bytes, pm_stream_t stream) {
    const pm::NvtxRange nvtx_("pmap:process_frames");
    if (!depth_out || !normals_out) return PM_ERR_INVALID_ARGUMENT;
    if (ws_bytes < pm_pipeline_workspace_bytes(W, H, n_regions, n_hyp, n_frames)) return PM_ERR_WORKSPACE;
    pm_status s = adf_impl(depth_in, depth_out, W, H, n_frames, K, lambda, kappa, iters, normals_out, workspace,
                           ws_bytes, 0, PM_ADF_ALG1, PM_NORMALS_GEOMETRIC, PM_ADF_ENGINE_AUTO, (cudaStream_t)stream);
    if (s != PM_OK) return s;
    // The ADF's per-frame flags (written by its first pass when it runs more
    // than one; 0 = every input depth valid and in [2^-100, 2^100)) say which
    // filtered frames hold valid depths only (lambda <= kNoCheckMaxLambda,
    // adf.cu fast_depth): their compaction count skips the depth reads.  The
    // flags sit in the ping-pong region, inside the compaction's point buffer
    // (checked: not in the histogram it clears first), which is written only
    // after the count.
    const int T = pm::adf_default_iters_per_pass();
    const size_t flags_off = pm::adf_flags_offset(W, H, n_frames);
    const bool flags_live = iters > T && lambda <= pm::kNoCheckMaxLambda &&
                            flags_off + sizeof(int) * (size_t)n_frames <= sizeof(uint64_t) * (size_t)n_frames * W * H;
    const int* fast =
        flags_live ? reinterpret_cast<const int*>(static_cast<const char*>(workspace) + flags_off) : nullptr;
    return ransac_impl(depth_out, W, H, n_frames, first_frame_id, K, region_labels, n_regions, n_hyp,
                       inlier_thresh, seed, planes_out, workspace, ws_bytes, nullptr, (cudaStream_t)stream, fast);
}

PM_API int32_t pm_pipeline_kernel_launches(int32_t iters, int32_t n_regions) {
    const int T = pm::adf_default_iters_per_pass();
    const int adf = iters <= 0 ? 1 : (iters + T - 1) / T;
    return adf + (n_regions > 0 ? 4 /* compaction */ + 5 /* hyp, score, select, refit, finalize */ : 0);
}

PM_API const char* pm_status_string(pm_status s) {
    switch (s) {
        case PM_OK: return "ok";
        case PM_ERR_INVALID_ARGUMENT: return "invalid argument";
        case PM_ERR_WORKSPACE: return "workspace missing, misaligned or too small";
        case PM_ERR_UNSUPPORTED: return "unsupported";
        case PM_ERR_CUDA: return "CUDA launch failed";
    }
    return "unknown status";
}

PM_API int32_t pm_version(void) { return kVersion; }

}  // extern "C"
