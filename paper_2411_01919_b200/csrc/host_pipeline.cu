// host_pipeline.cu — the whole path for frames in HOST memory
// (pm_process_frames_host): chunked, double-buffered H2D / compute / D2H on
// the caller's stream plus two internal copy streams per device (one per
// direction: a D2H waiting for chunk k's kernels must not hold back the H2D
// of chunk k+1), so the upload of chunk k+1 overlaps the kernels of chunk k
// and the link stays busy.  Sensor-native inputs (uint16 millimetres,
// S:26-28; uint16 / uint8 labels) cut the PCIe bytes.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <mutex>

#include "../../include/pmap.h"
#include "common.cuh"
#include "internal.h"

namespace pm {

namespace {

constexpr int kConvThreads = 256;

// Alg. 1 input convention: uint16 millimetres -> f32 metres, 0 stays 0 (invalid)
__global__ void __launch_bounds__(kConvThreads)
u16_to_metres_kernel(const uint16_t* __restrict__ mm, float* __restrict__ out, size_t n, float scale) {
    const size_t i0 = ((size_t)blockIdx.x * kConvThreads + threadIdx.x) * 4;
    if (i0 + 3 < n && ((reinterpret_cast<uintptr_t>(mm + i0) & 7) == 0) &&
        ((reinterpret_cast<uintptr_t>(out + i0) & 15) == 0)) {
        const ushort4 v = *reinterpret_cast<const ushort4*>(mm + i0);
        *reinterpret_cast<float4*>(out + i0) =
            make_float4(__fmul_rn((float)v.x, scale), __fmul_rn((float)v.y, scale), __fmul_rn((float)v.z, scale),
                        __fmul_rn((float)v.w, scale));
        return;
    }
    for (size_t i = i0; i < n && i < i0 + 4; ++i) out[i] = __fmul_rn((float)mm[i], scale);
}

// uint16 labels -> int32, 0xFFFF -> -1 (unlabelled)
__global__ void __launch_bounds__(kConvThreads)
u16_labels_kernel(const uint16_t* __restrict__ in, int32_t* __restrict__ out, size_t n) {
    const size_t i = (size_t)blockIdx.x * kConvThreads + threadIdx.x;
    if (i < n) out[i] = in[i] == 0xFFFFu ? -1 : (int32_t)in[i];
}

// uint8 labels -> int32, 0xFF -> -1 (unlabelled)
__global__ void __launch_bounds__(kConvThreads)
u8_labels_kernel(const uint8_t* __restrict__ in, int32_t* __restrict__ out, size_t n) {
    const size_t i = (size_t)blockIdx.x * kConvThreads + threadIdx.x;
    if (i < n) out[i] = in[i] == 0xFFu ? -1 : (int32_t)in[i];
}

// row runs -> int32 labels: one warp per image row, the row's runs written in
// turn by the whole warp (coalesced); 0xFFFF -> -1; pixels past the last run
// -> -1, runs past W cut.  row_start is relative to the chunk's first run.
__global__ void __launch_bounds__(kConvThreads)
runs_labels_kernel(const uint32_t* __restrict__ row_start, uint32_t base, const uint32_t* __restrict__ runs,
                   uint32_t nruns, int32_t* __restrict__ out, int W, int rows) {
    const int row = blockIdx.x * (kConvThreads / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    // a malformed (non-monotonic) row_start never reads past the chunk's runs
    const uint32_t r0 = min(row_start[row] - base, nruns), r1 = min(row_start[row + 1] - base, nruns);
    int32_t* o = out + (size_t)row * W;
    int x = 0;
    for (uint32_t r = r0; r < r1 && x < W; ++r) {
        const uint32_t run = runs[r];
        const int len = min((int)(run >> 16), W - x);
        const int32_t lab = (run & 0xFFFFu) == 0xFFFFu ? -1 : (int32_t)(run & 0xFFFFu);
        for (int i = lane; i < len; i += 32) o[x + i] = lab;
        x += len;
    }
    for (int i = x + lane; i < W; i += 32) o[i] = -1;
}

struct DeviceStreams {
    cudaStream_t copy = nullptr;      // H2D
    cudaStream_t down = nullptr;      // D2H
    cudaStream_t comp[2] = {};        // kernels of slot 0 / 1 (chunks k and k+1 may overlap: wave tails)
    cudaEvent_t h2d[2] = {}, done[2] = {}, freed[2] = {};
    cudaEvent_t start = nullptr;      // the caller's stream at entry
    std::mutex mu;            // one host pipeline at a time per device
    cudaError_t err = cudaSuccess;
};

DeviceStreams* streams_for_current_device() {
    static std::mutex g;
    static DeviceStreams* per_dev[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    std::lock_guard<std::mutex> lk(g);
    if (!per_dev[dev]) {
        DeviceStreams* d = new DeviceStreams();
        d->err = cudaStreamCreateWithFlags(&d->copy, cudaStreamNonBlocking);
        if (d->err == cudaSuccess) d->err = cudaStreamCreateWithFlags(&d->down, cudaStreamNonBlocking);
        for (int s = 0; s < 2 && d->err == cudaSuccess; ++s)
            d->err = cudaStreamCreateWithFlags(&d->comp[s], cudaStreamNonBlocking);
        if (d->err == cudaSuccess) d->err = cudaEventCreateWithFlags(&d->start, cudaEventDisableTiming);
        // (the freed events are recorded below, once every event exists: both slots start free)
        for (int s = 0; s < 2 && d->err == cudaSuccess; ++s) {
            d->err = cudaEventCreateWithFlags(&d->h2d[s], cudaEventDisableTiming);
            if (d->err == cudaSuccess) d->err = cudaEventCreateWithFlags(&d->done[s], cudaEventDisableTiming);
            if (d->err == cudaSuccess) d->err = cudaEventCreateWithFlags(&d->freed[s], cudaEventDisableTiming);
        }
        for (int s = 0; s < 2 && d->err == cudaSuccess; ++s) d->err = cudaEventRecord(d->freed[s], d->copy);
        per_dev[dev] = d;
    }
    return per_dev[dev];
}

size_t a256(size_t x) { return (x + 255) & ~(size_t)255; }

struct Slot {
    void* raw_depth;      // host-format depth staging (u16) or f32 depth directly
    void* raw_labels;     // host-format labels (u16 / u8 / run row starts) or int32 directly
    uint32_t* raw_runs;   // PM_LABELS_RUNS: the chunk's runs (<= one per pixel)
    float* depth;         // f32 metres (== raw_depth for f32 input)
    int32_t* labels;      // int32 (== raw_labels for int32 input)
    float* depth_out;
    float* normals;
    pm_plane* planes;
    void* ws;
    size_t ws_bytes;
};

struct Arena {
    size_t slot_bytes;
    Slot slot[2];
};

Arena arena_layout(void* base, int W, int H, int R, int n_hyp, int C, int depth_fmt, int label_fmt) {
    Arena a{};
    const size_t px = (size_t)C * W * H;
    const size_t ws = pm_pipeline_workspace_bytes(W, H, R, n_hyp, C);
    size_t o = 0;
    char* p = (char*)base;
    for (int s = 0; s < 2; ++s) {
        auto take = [&](size_t b) { void* q = p ? p + o : nullptr; o += a256(b); return q; };
        Slot& sl = a.slot[s];
        sl.depth = (float*)take(sizeof(float) * px);
        sl.raw_depth = depth_fmt == PM_DEPTH_U16_MM ? take(sizeof(uint16_t) * px) : (void*)sl.depth;
        sl.labels = (int32_t*)take(sizeof(int32_t) * px);
        sl.raw_labels = label_fmt == PM_LABELS_U16    ? take(sizeof(uint16_t) * px)
                        : label_fmt == PM_LABELS_U8   ? take(sizeof(uint8_t) * px)
                        : label_fmt == PM_LABELS_RUNS ? take(sizeof(uint32_t) * ((size_t)C * H + 1))
                                                      : (void*)sl.labels;
        sl.raw_runs = label_fmt == PM_LABELS_RUNS ? (uint32_t*)take(sizeof(uint32_t) * px) : nullptr;
        sl.depth_out = (float*)take(sizeof(float) * px);
        sl.normals = (float*)take(sizeof(float) * 3 * px);
        sl.planes = (pm_plane*)take(sizeof(pm_plane) * (size_t)C * (R > 0 ? R : 1));
        sl.ws = take(ws);
        sl.ws_bytes = ws;
    }
    a.slot_bytes = o / 2;
    return a;
}

}  // namespace

}  // namespace pm

extern "C" {

PM_API size_t pm_host_pipeline_arena_bytes(int32_t W, int32_t H, int32_t n_regions, int32_t n_hyp,
                                           int32_t chunk_frames, int32_t depth_format, int32_t label_format) {
    if (W < 1 || H < 1 || n_regions < 0 || n_hyp < 1 || chunk_frames < 1) return 0;
    pm::Arena a = pm::arena_layout(nullptr, W, H, n_regions, n_hyp, chunk_frames, depth_format, label_format);
    return 2 * a.slot_bytes;
}

PM_API pm_status pm_depth_u16_to_metres(const uint16_t* depth_mm, float* depth_m, size_t n, float scale,
                                        pm_stream_t stream) {
    if (!depth_mm || !depth_m || !(scale > 0.0f)) return PM_ERR_INVALID_ARGUMENT;
    if (n == 0) return PM_OK;
    const size_t quads = (n + 3) / 4;
    pm::u16_to_metres_kernel<<<(unsigned)((quads + pm::kConvThreads - 1) / pm::kConvThreads), pm::kConvThreads, 0,
                               (cudaStream_t)stream>>>(depth_mm, depth_m, n, scale);
    return cudaGetLastError() == cudaSuccess ? PM_OK : PM_ERR_CUDA;
}

}  // extern "C"

namespace pm {
namespace {
pm_status host_pipeline(const void* depth_host, int32_t depth_format, const void* labels_host, int32_t label_format,
                        int32_t W, int32_t H, int32_t n_frames, uint32_t first_frame_id, const pm_intrinsics* K,
                        float lambda, float kappa, int32_t iters, int32_t n_regions, int32_t n_hyp,
                        float inlier_thresh, uint64_t seed, pm_plane* planes_host, float* depth_out_host,
                        float* normals_host, int32_t chunk_frames, void* arena, size_t arena_bytes,
                        pm_stream_t stream, bool async) {
    const pm::NvtxRange nvtx_("pmap:process_frames_host");
    if (!depth_host || !labels_host || !planes_host || chunk_frames < 1 || n_frames < 1)
        return PM_ERR_INVALID_ARGUMENT;
    if (depth_format != PM_DEPTH_F32_M && depth_format != PM_DEPTH_U16_MM) return PM_ERR_INVALID_ARGUMENT;
    if (label_format != PM_LABELS_I32 && label_format != PM_LABELS_U16 && label_format != PM_LABELS_U8 &&
        label_format != PM_LABELS_RUNS)
        return PM_ERR_INVALID_ARGUMENT;
    const pm_label_runs* lr = label_format == PM_LABELS_RUNS ? (const pm_label_runs*)labels_host : nullptr;
    if (lr && (!lr->row_start || !lr->runs)) return PM_ERR_INVALID_ARGUMENT;
    if (lr && W > 65535) return PM_ERR_INVALID_ARGUMENT;
    if (label_format == PM_LABELS_U16 && n_regions > 65535) return PM_ERR_INVALID_ARGUMENT;
    if (label_format == PM_LABELS_U8 && n_regions > 255) return PM_ERR_INVALID_ARGUMENT;
    const int C = chunk_frames < n_frames ? chunk_frames : n_frames;
    if (!arena || arena_bytes < pm_host_pipeline_arena_bytes(W, H, n_regions, n_hyp, C, depth_format, label_format) ||
        ((uintptr_t)arena & 255u))
        return PM_ERR_WORKSPACE;
    // every argument check before the first copy is queued
    if (pm_status v = pipeline_validate(W, H, n_frames, K, lambda, kappa, iters, n_regions, n_hyp, inlier_thresh);
        v != PM_OK)
        return v;
    DeviceStreams* ds = streams_for_current_device();
    if (!ds || ds->err != cudaSuccess) return PM_ERR_CUDA;
    std::lock_guard<std::mutex> lk(ds->mu);
    const Arena A = arena_layout(arena, W, H, n_regions, n_hyp, C, depth_format, label_format);
    cudaStream_t cs = (cudaStream_t)stream;
    const size_t frame_px = (size_t)W * H;
    const size_t dsz = depth_format == PM_DEPTH_U16_MM ? 2 : 4;
    const size_t lsz = label_format == PM_LABELS_U16 ? 2 : label_format == PM_LABELS_U8 ? 1 : 4;   // not RUNS
    const int n_chunks = (n_frames + C - 1) / C;
    // every exit waits for the copies already queued on the internal streams
    // (and the kernels feeding them): the caller may free or reuse its host
    // buffers and the arena as soon as this returns, also on error
    auto finish = [&](pm_status st) {
        const cudaError_t e1 = cudaStreamSynchronize(ds->copy);
        const cudaError_t e2 = cudaStreamSynchronize(ds->comp[0]);
        const cudaError_t e4 = cudaStreamSynchronize(ds->comp[1]);
        const cudaError_t e3 = cudaStreamSynchronize(ds->down);
        const cudaError_t e5 = cudaStreamSynchronize(cs);
        if (st == PM_OK && (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess || e4 != cudaSuccess ||
                            e5 != cudaSuccess))
            st = PM_ERR_CUDA;
        return st;
    };
    cudaError_t e = cudaSuccess;
    if (!async) {
        // everything after the caller's earlier work on `stream`
        e = cudaEventRecord(ds->start, cs);
        for (int s = 0; s < 2 && e == cudaSuccess; ++s) e = cudaStreamWaitEvent(ds->comp[s], ds->start, 0);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(ds->copy, ds->start, 0);
    }
    // (async: the inputs are host memory the caller has ready; each slot is
    // reused after its previous download -- possibly a previous call's --
    // through the freed events, so consecutive calls overlap: the next call's
    // first upload runs under this call's last kernels)
    for (int k = 0; k < n_chunks && e == cudaSuccess; ++k) {
        const int s = k & 1;
        const Slot& sl = A.slot[s];
        const int f0 = k * C;
        const int nf = (n_frames - f0) < C ? (n_frames - f0) : C;
        const size_t px = (size_t)nf * frame_px;
        // H2D on the copy stream once the slot's previous results are out
        e = cudaStreamWaitEvent(ds->copy, ds->freed[s], 0);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(sl.raw_depth, (const char*)depth_host + (size_t)f0 * frame_px * dsz, px * dsz,
                                cudaMemcpyHostToDevice, ds->copy);
        uint32_t run_base = 0, run_count = 0;
        if (lr) {   // the chunk's row starts and runs (a contiguous slice of each)
            const size_t g0 = (size_t)f0 * H, g1 = (size_t)(f0 + nf) * H;
            run_base = lr->row_start[g0];
            const size_t nruns = lr->row_start[g1] - run_base;
            if (nruns > px) return finish(PM_ERR_INVALID_ARGUMENT);      // > one run per pixel
            run_count = (uint32_t)nruns;
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(sl.raw_labels, lr->row_start + g0, sizeof(uint32_t) * (g1 - g0 + 1),
                                    cudaMemcpyHostToDevice, ds->copy);
            if (e == cudaSuccess && nruns)
                e = cudaMemcpyAsync(sl.raw_runs, lr->runs + run_base, sizeof(uint32_t) * nruns,
                                    cudaMemcpyHostToDevice, ds->copy);
        } else if (e == cudaSuccess) {
            e = cudaMemcpyAsync(sl.raw_labels, (const char*)labels_host + (size_t)f0 * frame_px * lsz, px * lsz,
                                cudaMemcpyHostToDevice, ds->copy);
        }
        if (e == cudaSuccess) e = cudaEventRecord(ds->h2d[s], ds->copy);
        // the chunk's kernels on the slot's compute stream (the other slot's
        // chunk may still be running: its last wave overlaps this one's first)
        cudaStream_t ks = ds->comp[s];
        if (e == cudaSuccess) e = cudaStreamWaitEvent(ks, ds->h2d[s], 0);
        if (e != cudaSuccess) break;
        if (depth_format == PM_DEPTH_U16_MM) {
            pm_status st = pm_depth_u16_to_metres((const uint16_t*)sl.raw_depth, sl.depth, px, 1e-3f, ks);
            if (st != PM_OK) return finish(st);
        }
        if (label_format == PM_LABELS_U16) {
            u16_labels_kernel<<<(unsigned)((px + kConvThreads - 1) / kConvThreads), kConvThreads, 0, ks>>>(
                (const uint16_t*)sl.raw_labels, sl.labels, px);
            if ((e = cudaGetLastError()) != cudaSuccess) break;
        } else if (label_format == PM_LABELS_U8) {
            u8_labels_kernel<<<(unsigned)((px + kConvThreads - 1) / kConvThreads), kConvThreads, 0, ks>>>(
                (const uint8_t*)sl.raw_labels, sl.labels, px);
            if ((e = cudaGetLastError()) != cudaSuccess) break;
        } else if (lr) {
            const int rows = nf * H;
            runs_labels_kernel<<<(unsigned)((rows + kConvThreads / 32 - 1) / (kConvThreads / 32)), kConvThreads, 0,
                                 ks>>>((const uint32_t*)sl.raw_labels, run_base, sl.raw_runs, run_count, sl.labels, W,
                                       rows);
            if ((e = cudaGetLastError()) != cudaSuccess) break;
        }
        pm_status st = pm_process_frames(sl.depth, sl.labels, W, H, nf, first_frame_id + (uint32_t)f0, K, lambda,
                                         kappa, iters, n_regions, n_hyp, inlier_thresh, seed, sl.depth_out,
                                         sl.normals, sl.planes, sl.ws, sl.ws_bytes, ks);
        if (st != PM_OK) return finish(st);
        e = cudaEventRecord(ds->done[s], ks);
        // D2H of the results on the download stream; the slot is free afterwards
        if (e == cudaSuccess) e = cudaStreamWaitEvent(ds->down, ds->done[s], 0);
        if (e == cudaSuccess && n_regions > 0)
            e = cudaMemcpyAsync(planes_host + (size_t)f0 * n_regions, sl.planes, sizeof(pm_plane) * nf * n_regions,
                                cudaMemcpyDeviceToHost, ds->down);
        if (e == cudaSuccess && depth_out_host)
            e = cudaMemcpyAsync(depth_out_host + (size_t)f0 * frame_px, sl.depth_out, sizeof(float) * px,
                                cudaMemcpyDeviceToHost, ds->down);
        if (e == cudaSuccess && normals_host)
            e = cudaMemcpyAsync(normals_host + (size_t)f0 * 3 * frame_px, sl.normals, sizeof(float) * 3 * px,
                                cudaMemcpyDeviceToHost, ds->down);
        if (e == cudaSuccess) e = cudaEventRecord(ds->freed[s], ds->down);
    }
    // the caller's stream completes after the last download of both slots
    for (int s = 0; s < 2 && e == cudaSuccess; ++s) e = cudaStreamWaitEvent(cs, ds->freed[s], 0);
    if (async && e == cudaSuccess) return PM_OK;
    return finish(e == cudaSuccess ? PM_OK : PM_ERR_CUDA);
}
}  // namespace
}  // namespace pm

extern "C" {

PM_API pm_status pm_process_frames_host(const void* depth_host, int32_t depth_format, const void* labels_host,
                                        int32_t label_format, int32_t W, int32_t H, int32_t n_frames,
                                        uint32_t first_frame_id, const pm_intrinsics* K, float lambda, float kappa,
                                        int32_t iters, int32_t n_regions, int32_t n_hyp, float inlier_thresh,
                                        uint64_t seed, pm_plane* planes_host, float* depth_out_host,
                                        float* normals_host, int32_t chunk_frames, void* arena, size_t arena_bytes,
                                        pm_stream_t stream) {
    return pm::host_pipeline(depth_host, depth_format, labels_host, label_format, W, H, n_frames, first_frame_id, K,
                             lambda, kappa, iters, n_regions, n_hyp, inlier_thresh, seed, planes_host,
                             depth_out_host, normals_host, chunk_frames, arena, arena_bytes, stream, false);
}

PM_API pm_status pm_process_frames_host_async(const void* depth_host, int32_t depth_format, const void* labels_host,
                                              int32_t label_format, int32_t W, int32_t H, int32_t n_frames,
                                              uint32_t first_frame_id, const pm_intrinsics* K, float lambda,
                                              float kappa, int32_t iters, int32_t n_regions, int32_t n_hyp,
                                              float inlier_thresh, uint64_t seed, pm_plane* planes_host,
                                              float* depth_out_host, float* normals_host, int32_t chunk_frames,
                                              void* arena, size_t arena_bytes, pm_stream_t stream) {
    return pm::host_pipeline(depth_host, depth_format, labels_host, label_format, W, H, n_frames, first_frame_id, K,
                             lambda, kappa, iters, n_regions, n_hyp, inlier_thresh, seed, planes_host,
                             depth_out_host, normals_host, chunk_frames, arena, arena_bytes, stream, true);
}

}  // extern "C"
