/*
 * pmap.h — C ABI of the B200-native hot path of arXiv 2411.01919
 * ("real-time planar semantic mapping"): iterated Perona–Malik anisotropic
 * diffusion of a depth frame, the per-pixel normal image fused into the last
 * diffusion pass, and batched RANSAC plane fitting over every labelled region.
 *
 * Citations: "P:n" = line n of the paper text, "S:n" = line n of
 * SPEC.md, "Qk" = reading k in DESIGN.md §3 (where the paper is silent or
 * ambiguous).
 *
 * Conventions (all calls)
 *  - Every pointer is a DEVICE pointer unless marked "host".  The caller owns
 *    every buffer, including the workspace; the library allocates nothing.
 *  - Work is enqueued asynchronously on `stream` (a cudaStream_t; NULL = the
 *    legacy default stream).  No call synchronises the host except the
 *    *_host pipeline entry, which synchronises its own stream before return.
 *  - Frames are row-major f32 [H][W] in metres; u = column, v = row (Q25).
 *    A depth value is VALID iff it is > 0 and finite (Q4).  Batched
 *    calls take n_frames contiguous frames [B][H][W].
 *  - Argument errors are detected before any launch and return
 *    PM_ERR_INVALID_ARGUMENT; too-small workspaces return PM_ERR_WORKSPACE;
 *    a failed launch returns PM_ERR_CUDA (asynchronous faults surface at the
 *    caller's next synchronisation).  Per-region RANSAC failures are
 *    statuses in pm_plane, not errors.
 *  - Limits: 3 <= W, H <= 65535; 0 <= n_regions <= 65536; 1 <= n_hyp <= 4096;
 *    1 <= n_frames <= 65535.
 *  - Calls are re-entrant and thread-safe (the only global state is a
 *    one-time kernel-attribute setup guarded by std::call_once).
 */
#ifndef PMAP_H_
#define PMAP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define PM_API __attribute__((visibility("default")))
#else
#define PM_API
#endif

typedef struct CUstream_st* pm_stream_t;   /* == cudaStream_t */

typedef enum {
    PM_OK = 0,
    PM_ERR_INVALID_ARGUMENT = 1,
    PM_ERR_WORKSPACE = 2,
    PM_ERR_UNSUPPORTED = 3,
    PM_ERR_CUDA = 4
} pm_status;

/* Pinhole intrinsics K ("camera intrinsic matrix"; Q24): fx, fy > 0
 * and finite; cx, cy in pixels.  Always passed by HOST pointer. */
typedef struct { float fx, fy, cx, cy; } pm_intrinsics;

/* One fitted plane per (frame, region): n.X + d = 0 in the camera frame,
 * |n| = 1, d >= 0 (metres); centroid = mean of the refit inliers (Q22).
 * inliers = best hypothesis' inlier count (Alg. 2 ℓ16), n_points = valid
 * labelled pixels of the region, best_hyp = winning hypothesis index or -1,
 * status = PM_PLANE_*; sum_dist = the winner's total distance Σ min(d,64)
 * (Alg. 2 ℓ11, error), from the exact fixed-point sum, informative. 48 bytes. */
typedef struct {
    float n[3];
    float d;
    float centroid[3];
    int32_t inliers;
    int32_t n_points;
    int32_t best_hyp;
    int32_t status;
    float sum_dist;
} pm_plane;

enum {
    PM_PLANE_OK = 0,          /* 10 * inliers > 9 * n_points (Alg. 2 ℓ19) */
    PM_PLANE_REJECTED = 1,    /* gate failed: outliers >= 10 %            */
    PM_PLANE_TOO_FEW = 2,     /* n_points < 3                              */
    PM_PLANE_DEGENERATE = 3   /* every hypothesis collinear (Q18)                  */
};

/* ---------------------------------------------------------------------- */
/* adf_filter — Algorithm 1: N Jacobi sweeps of
 *   I_p <- I_p + lambda * c_p * lap(I_p),  c_p = exp(-|grad I_p|^2 / kappa^2)
 * (ℓ2-8; Eq. 1; central-difference gradient Q3; 5-point Laplacian;
 * zero-flux rule Q4: an out-of-image or invalid neighbour takes the centre
 * value; invalid pixels are copied bit for bit), then, if normals_out is not
 * NULL, the normal image of the result (ℓ9-13, see normals_from_depth) fused
 * into the last diffusion pass.
 *   depth_in   [B][H][W] f32, read only; must not overlap depth_out.
 *   depth_out  [B][H][W] f32, written (I_smooth); 16-byte aligned (float4 /
 *              bulk-copy rows; a tensor view at an element offset may not be:
 *              PM_ERR_INVALID_ARGUMENT).
 *   K          host pointer; required iff normals_out != NULL.
 *   lambda     gamma of Alg. 1, 0 < lambda <= 0.25 (stability).
 *   kappa      k of Alg. 1 in metres, > 0.
 *   iters      N >= 0 (N = 0 copies depth_in).
 *   normals_out [B][3][H][W] f32 (SoA: nx plane, ny plane, nz plane) or NULL;
 *              16-byte aligned like depth_out.
 *   workspace  >= pm_adf_workspace_bytes(W, H, n_frames) bytes, 256-B aligned.
 * The result is bitwise independent of n_frames and of the blocking depth. */
PM_API pm_status pm_adf_filter(const float* depth_in, float* depth_out, int32_t W, int32_t H,
                               const pm_intrinsics* K, float lambda, float kappa, int32_t iters,
                               float* normals_out, void* workspace, size_t ws_bytes,
                               pm_stream_t stream);
PM_API pm_status pm_adf_filter_batched(const float* depth_in, float* depth_out, int32_t W, int32_t H,
                                       int32_t n_frames, const pm_intrinsics* K, float lambda,
                                       float kappa, int32_t iters, float* normals_out,
                                       void* workspace, size_t ws_bytes, pm_stream_t stream);
PM_API size_t pm_adf_workspace_bytes(int32_t W, int32_t H, int32_t n_frames);

/* Options for adf.  iters_per_pass is a tuning knob (results do not depend
 * on it); scheme / normals_mode select the paper-literal variants (NEXT-1):
 *   PM_ADF_ALG1        Alg. 1 as printed, c_p * lap(I) (default, Q1)
 *   PM_ADF_DIVERGENCE  Eq. 1 as the 4-flux Perona-Malik scheme
 *                      I += lambda * sum_d exp(-((I_d - I)/k)^2) (I_d - I)
 *   PM_NORMALS_GEOMETRIC   the tangent-cross-product normal (default, Q7)
 *   PM_NORMALS_AS_PRINTED  Eq. 2 literally: n = -K^-1 [Gx, Gy, 1]^T, normalised */
enum { PM_ADF_ALG1 = 0, PM_ADF_DIVERGENCE = 1 };
enum { PM_NORMALS_GEOMETRIC = 0, PM_NORMALS_AS_PRINTED = 1 };
/* engine: AUTO = TILED (the faster engine on B200), switching
 * to HOLES while a call on the device within the last 16 multi-pass calls met
 * an invalid pixel (the first pass notes it in a mapped host word; results
 * are the same either way);
 * REG = register-resident tiles (csrc/adf_reg.cu; W % 4 == 0, H >= 128,
 * 16-B aligned depth), falls back to TILED where it does not apply;
 * TILED = shared-memory tiles, iters_per_pass sweeps (default 4) per HBM pass;
 * HOLES = TILED whose tiles with a few invalid pixels (<= ~1.5 %: sensor
 * dropout) run the unchecked walk and then recompute the cells next to a hole
 * with the checked cell, instead of checking every cell (1 % dropout: ~1.3x
 * faster ADF; hole-free frames ~1-4 % slower, hence not the default).
 * All engines give bitwise identical results.  (Value 2, a wavefront engine
 * of round 1, was removed: 2.6x slower than TILED.) */
enum { PM_ADF_ENGINE_AUTO = 0, PM_ADF_ENGINE_TILED = 1, PM_ADF_ENGINE_REG = 3, PM_ADF_ENGINE_HOLES = 4 };
typedef struct {
    int32_t iters_per_pass;   /* sweeps per HBM pass (1..16); 0 = engine default */
    int32_t scheme;           /* PM_ADF_*        */
    int32_t normals_mode;     /* PM_NORMALS_*    */
    int32_t engine;           /* PM_ADF_ENGINE_* */
} pm_adf_options;
PM_API pm_status pm_adf_filter_ex(const float* depth_in, float* depth_out, int32_t W, int32_t H,
                                  int32_t n_frames, const pm_intrinsics* K, float lambda,
                                  float kappa, int32_t iters, float* normals_out,
                                  void* workspace, size_t ws_bytes, const pm_adf_options* opt,
                                  pm_stream_t stream);

/* ---------------------------------------------------------------------- */
/* normals_from_depth — Alg. 1 ℓ9-13, Eq. 2 read
 * geometrically (Q7): with 3x3 Sobel gradients of Z normalised by 1/8 and
 * clamp-to-edge indexing (Q8),
 *   m = ( fx Gx, fy Gy, -(Z + (u - cx) Gx + (v - cy) Gy) ),  n = m / |m|
 * (the tangent cross product dP/du x dP/dv of P = Z K^-1 [u v 1]^T; it faces
 * the camera).  n = (0,0,0) if any pixel of the clamped 3x3 window is
 * invalid (Q9).  depth [B][H][W] f32; normals_out [B][3][H][W] f32. */
PM_API pm_status pm_normals_from_depth(const float* depth, int32_t W, int32_t H,
                                       const pm_intrinsics* K, float* normals_out,
                                       pm_stream_t stream);
PM_API pm_status pm_normals_from_depth_batched(const float* depth, int32_t W, int32_t H,
                                               int32_t n_frames, const pm_intrinsics* K,
                                               float* normals_out, pm_stream_t stream);
/* mode: PM_NORMALS_GEOMETRIC (default) or PM_NORMALS_AS_PRINTED (see pm_adf_options). */
PM_API pm_status pm_normals_from_depth_ex(const float* depth, int32_t W, int32_t H, int32_t n_frames,
                                          const pm_intrinsics* K, int32_t mode, float* normals_out,
                                          pm_stream_t stream);

/* ---------------------------------------------------------------------- */
/* ransac_planes — Algorithm 2, batched over every region of every
 * frame.  For region r of frame f (f = first_frame_id + batch index):
 *   P  = its valid labelled pixels in raster order, deprojected in f32 as
 *        X = (((float)u - cx) * (1/fx)) * z, Y likewise, Z = z  (ℓ2-3)
 *   hypothesis h (0 <= h < n_hyp): Philox4x32-10 of counter {h, r, f, 0},
 *        key {lo32(seed), hi32(seed)} -> 3 distinct indices (Q17) -> f32 plane
 *        (ℓ6-7); collinear samples are invalid (Q18)
 *   score: inliers_h = #{ |n.p + d| < inlier_thresh } (ℓ9-13, strict, Q14)
 *   select: argmax inliers, ties to the lowest h (Q11)
 *   refit: fp64 total least squares over the winner's inliers (Q19)
 *   gate: PM_PLANE_OK iff 10 * inliers > 9 * n_points (ℓ19, Q15).
 * The exact float32 operation sequence is DESIGN.md §3 (shared with the
 * oracle by specification, not by code).
 *   depth          [B][H][W] f32 (raw or filtered, Q10).
 *   region_labels  [B][H][W] int32; labels outside [0, n_regions) are ignored.
 *   planes_out     [B][n_regions] pm_plane.
 *   inlier_thresh  tau in metres, > 0 and finite.
 *   workspace      >= pm_ransac_workspace_bytes(W, H, n_regions, n_hyp, n_frames).
 * Results are bitwise independent of batching and launch geometry. */
PM_API pm_status pm_ransac_planes(const float* depth, int32_t W, int32_t H, const pm_intrinsics* K,
                                  const int32_t* region_labels, int32_t n_regions, int32_t n_hyp,
                                  float inlier_thresh, uint64_t seed, pm_plane* planes_out,
                                  void* workspace, size_t ws_bytes, pm_stream_t stream);
PM_API pm_status pm_ransac_planes_batched(const float* depth, int32_t W, int32_t H, int32_t n_frames,
                                          uint32_t first_frame_id, const pm_intrinsics* K,
                                          const int32_t* region_labels, int32_t n_regions,
                                          int32_t n_hyp, float inlier_thresh, uint64_t seed,
                                          pm_plane* planes_out, void* workspace, size_t ws_bytes,
                                          pm_stream_t stream);
PM_API size_t pm_ransac_workspace_bytes(int32_t W, int32_t H, int32_t n_regions, int32_t n_hyp,
                                        int32_t n_frames);

/* Test / paper-literal options for ransac (NEXT-1 rows of SURVEY §8(f)). */
enum { PM_SAMPLER_PHILOX = 0, PM_SAMPLER_ENUMERATE = 1 };   /* ENUMERATE: h -> h-th 3-combination, colex */
enum { PM_SELECT_COUNT = 0, PM_SELECT_ERROR = 1,            /* ERROR: argmin Σd as printed       */
       PM_SELECT_COUNT_EARLY = 2, PM_SELECT_ERROR_EARLY = 3 }; /* *_EARLY: the hypothesis loop stops once the
                                                                  best model so far passes the 0.9 gate
                                                                  ("until ... a satisfactory model is found",
                                                                  P:292; Q20)                     */
typedef struct {
    int32_t sampler;          /* PM_SAMPLER_*                                          */
    int32_t select;           /* PM_SELECT_*                                           */
    int32_t* counts_out;      /* nullable device [B][n_regions][n_hyp]: inliers per h,
                                 -1 = invalid hypothesis                                */
    uint64_t* errq_out;       /* nullable device [B][n_regions][n_hyp]: Σ rint(min(d,64)
                                 * 2^24) per h (required work for PM_SELECT_ERROR)     */
    void* const* stage_events;/* nullable host array of PM_RANSAC_STAGE_EVENTS
                                 cudaEvent_t (created by the caller): recorded on the
                                 stream before compaction and after compaction,
                                 hypotheses, scoring, selection + refit and the plane
                                 table -- per-kernel timing with CUDA events (bench) */
} pm_ransac_options;
enum { PM_RANSAC_STAGE_EVENTS = 6 };
PM_API pm_status pm_ransac_planes_ex(const float* depth, int32_t W, int32_t H, int32_t n_frames,
                                     uint32_t first_frame_id, const pm_intrinsics* K,
                                     const int32_t* region_labels, int32_t n_regions,
                                     int32_t n_hyp, float inlier_thresh, uint64_t seed,
                                     pm_plane* planes_out, void* workspace, size_t ws_bytes,
                                     const pm_ransac_options* opt, pm_stream_t stream);

/* ---------------------------------------------------------------------- */
/* Whole per-frame path (adf_filter with fused normals, then ransac_planes on
 * the FILTERED depth, Q10) for n_frames device-resident frames.
 * depth_out, normals_out, planes_out as above; workspace >=
 * pm_pipeline_workspace_bytes(...). */
PM_API pm_status pm_process_frames(const float* depth_in, const int32_t* region_labels,
                                   int32_t W, int32_t H, int32_t n_frames, uint32_t first_frame_id,
                                   const pm_intrinsics* K, float lambda, float kappa, int32_t iters,
                                   int32_t n_regions, int32_t n_hyp, float inlier_thresh,
                                   uint64_t seed, float* depth_out, float* normals_out,
                                   pm_plane* planes_out, void* workspace, size_t ws_bytes,
                                   pm_stream_t stream);
PM_API size_t pm_pipeline_workspace_bytes(int32_t W, int32_t H, int32_t n_regions, int32_t n_hyp,
                                          int32_t n_frames);

/* ---------------------------------------------------------------------- */
/* segment_regions — NEXT-2 of SURVEY §8(f): region labels from the normal
 * image, the paper's step between Alg. 1 and Alg. 2 ("edges are detected from
 * the normal vector image using the Canny edge detection algorithm.
 * Subsequently, contours are extracted from these edges").
 * Readings (Q26-Q29): Canny on the 8-bit RGB normal image
 * c = rint((n + 1) * 127.5) with 3x3 Sobel, replicated borders, the
 * L2 magnitude of the strongest channel, non-maximum suppression and
 * 8-connected hysteresis (canny_low / canny_high on that magnitude, as
 * OpenCV's Canny with L2gradient); pixels with an invalid normal are edges;
 * the edge mask is dilated by one pixel (3x3); regions are the 4-connected
 * components of non-edge pixels with >= min_area pixels, numbered
 * 0.. by descending size, ties by smallest raster index, at most
 * max_regions; all other pixels -1.  Integer decisions only: bit-exact.
 *   normals      [B][3][H][W] f32 (from adf_filter / normals_from_depth)
 *   labels_out   [B][H][W] int32
 *   n_regions_out [B] int32 (device, nullable): regions kept per frame
 *   edges_out    [B][H][W] uint8 0/1 (device, nullable): the dilated edge mask
 *   workspace    >= pm_segment_workspace_bytes(W, H, n_frames, min_area). */
typedef struct {
    float canny_low;          /* default 30 */
    float canny_high;         /* default 90         */
    int32_t min_area;         /* default 300 px     */
    int32_t max_regions;      /* <= 65536           */
} pm_segment_params;
PM_API pm_status pm_segment_regions(const float* normals, int32_t W, int32_t H, int32_t n_frames,
                                    const pm_segment_params* params, int32_t* labels_out,
                                    int32_t* n_regions_out, uint8_t* edges_out, void* workspace,
                                    size_t ws_bytes, pm_stream_t stream);
PM_API size_t pm_segment_workspace_bytes(int32_t W, int32_t H, int32_t n_frames, int32_t min_area);

/* ---------------------------------------------------------------------- */
/* The whole path for frames in HOST memory: chunks of chunk_frames frames
 * are copied to the device, processed by pm_process_frames and the plane
 * tables (and, if the pointers are not NULL, the filtered depth [B][H][W] and
 * normals [B][3][H][W]) copied back, double-buffered so that the copies of
 * one chunk overlap the kernels of the previous one (the caller's stream plus
 * two internal copy streams per device -- upload, download -- created on first use).  Host buffers
 * should be pinned (cudaHostAlloc / cudaHostRegister) for the copies to be
 * asynchronous.  Synchronises before returning.
 *   depth_host   [B][H][W] in depth_format: PM_DEPTH_F32_M (f32 metres) or
 *                PM_DEPTH_U16_MM (uint16 millimetres, the sensor's native
 *                format; 0 = invalid; converted as (float)mm * 1e-3f)
 *   labels_host  [B][H][W] in label_format: PM_LABELS_I32 (int32, -1 = none),
 *                PM_LABELS_U16 (uint16, 0xFFFF = none; n_regions <= 65535) or
 *                PM_LABELS_U8 (uint8, 0xFF = none; n_regions <= 255); or, for
 *                PM_LABELS_RUNS, a pointer to a pm_label_runs: the same label
 *                image as row runs (region labels are piecewise constant --
 *                the paper's regions are polygons, P:287 -- so a frame's
 *                labels take a few KB instead of W*H bytes on the link)
 *   planes_host  [B][n_regions] pm_plane (host)
 *   arena        device memory >= pm_host_pipeline_arena_bytes(...), 256-B aligned.
 * Other arguments as pm_process_frames. */
enum { PM_DEPTH_F32_M = 0, PM_DEPTH_U16_MM = 1 };
enum { PM_LABELS_I32 = 0, PM_LABELS_U16 = 1, PM_LABELS_U8 = 2, PM_LABELS_RUNS = 3 };
/* Run-length labels of B frames (host memory, pinned for asynchronous copies).
 * Row y of frame f (global row index g = f * H + y) is the runs
 * runs[row_start[g] .. row_start[g + 1]), left to right; a run is
 * (label | length << 16): label in the low 16 bits (0xFFFF = none; labels
 * >= n_regions are ignored like any out-of-range label), length >= 1 pixels.
 * A row's lengths should sum to W: pixels past the last run are unlabelled,
 * runs past W are cut.  row_start has B * H + 1 entries, row_start[0] = 0. */
typedef struct {
    const uint32_t* row_start;
    const uint32_t* runs;
} pm_label_runs;
PM_API pm_status pm_process_frames_host(const void* depth_host, int32_t depth_format, const void* labels_host,
                                        int32_t label_format, int32_t W, int32_t H, int32_t n_frames,
                                        uint32_t first_frame_id, const pm_intrinsics* K, float lambda,
                                        float kappa, int32_t iters, int32_t n_regions, int32_t n_hyp,
                                        float inlier_thresh, uint64_t seed, pm_plane* planes_host,
                                        float* depth_out_host, float* normals_host, int32_t chunk_frames,
                                        void* arena, size_t arena_bytes, pm_stream_t stream);
/* The same, asynchronous: returns once every copy and kernel is queued.  The
 * host buffers (inputs and outputs) and the arena must stay untouched until
 * `stream` has completed (cudaStreamSynchronize(stream), or an event recorded
 * on it after the call); the inputs must be ready when the call is made.
 * Consecutive calls on the same device overlap: the next call's first upload
 * runs under this call's last kernels (the arena's two slots are reused only
 * after their previous downloads).  Errors found before anything is queued
 * return as for the synchronous call; a failure after that drains the
 * internal streams before returning. */
PM_API pm_status pm_process_frames_host_async(const void* depth_host, int32_t depth_format,
                                              const void* labels_host, int32_t label_format, int32_t W,
                                              int32_t H, int32_t n_frames, uint32_t first_frame_id,
                                              const pm_intrinsics* K, float lambda, float kappa, int32_t iters,
                                              int32_t n_regions, int32_t n_hyp, float inlier_thresh,
                                              uint64_t seed, pm_plane* planes_host, float* depth_out_host,
                                              float* normals_host, int32_t chunk_frames, void* arena,
                                              size_t arena_bytes, pm_stream_t stream);
PM_API size_t pm_host_pipeline_arena_bytes(int32_t W, int32_t H, int32_t n_regions, int32_t n_hyp,
                                           int32_t chunk_frames, int32_t depth_format, int32_t label_format);
/* uint16 millimetres -> f32 metres (device buffers, n values): m = (float)mm * scale. */
PM_API pm_status pm_depth_u16_to_metres(const uint16_t* depth_mm, float* depth_m, size_t n, float scale,
                                        pm_stream_t stream);

/* ---------------------------------------------------------------------- */
/* NEXT-3 of SURVEY §8(f): polygon glue between region labels and planes
 * ("contours are extracted from these edges and simplified into
 * polygons"; readings Q35-Q39 in DESIGN.md).
 * All buffers device memory, batched over n_frames x n_regions slots. */
typedef struct {
    int32_t eps16;         /* Douglas-Peucker tolerance in 1/16 px (S:262 default 3 px = 48) */
    int32_t max_contour;   /* capacity of a traced contour (points) */
    int32_t max_vertices;  /* capacity of a simplified polygon (vertices, >= 3) */
} pm_polygon_params;

/* Per region r of each frame's label image [B][H][W] (int32, r in
 * [0, n_regions), others ignored): the outer boundary by Moore-neighbour
 * tracing from the region's first pixel in raster order (clockwise on
 * screen; Q35), then closed Douglas-Peucker with exact integer distance tests
 * (anchors: the start and the farthest point; Q36).
 *   contour_len  [B][R]   traced length (> max_contour: truncated), 0 = empty
 *   vertices     [B][R][max_vertices][2] int32 (x, y) in contour order
 *   n_vertices   [B][R]   kept vertices (> max_vertices: truncated)
 *   workspace    >= pm_region_polygons_workspace_bytes(B, R, max_contour), 256-B aligned */
PM_API pm_status pm_region_polygons(const int32_t* labels, int32_t W, int32_t H, int32_t n_frames,
                                    int32_t n_regions, const pm_polygon_params* prm, int32_t* contour_len,
                                    int32_t* vertices, int32_t* n_vertices, void* workspace, size_t ws_bytes,
                                    pm_stream_t stream);
PM_API size_t pm_region_polygons_workspace_bytes(int32_t n_frames, int32_t n_regions, int32_t max_contour);

/* Rasterise the polygons back to labels ("rasterize its interior"):
 * pixel (x, y) gets the lowest region index whose polygon contains the pixel
 * centre by the even-odd rule with half-open crossings (Q37, Q38), -1 if
 * none; polygons with < 3 vertices cover nothing.
 *   labels_out [B][H][W] int32; workspace >= 16 * B * max(R, 1) bytes, 256-B aligned. */
PM_API pm_status pm_rasterize_polygons(const int32_t* vertices, const int32_t* n_vertices, int32_t max_vertices,
                                       int32_t W, int32_t H, int32_t n_frames, int32_t n_regions,
                                       int32_t* labels_out, void* workspace, size_t ws_bytes, pm_stream_t stream);

/* Lift every polygon vertex onto its region's fitted plane along the camera
 * ray: X = -d / (n.r) r, r = ((u-cx)/fx, (v-cy)/fy, 1), fp64 (Q39).
 *   planes [B][R] (from pm_ransac_planes); X_out [B][R][max_vertices][3]
 *   double, NaN for missing vertices, planes not PM_PLANE_OK, rays parallel
 *   to the plane or hitting it behind the camera. */
PM_API pm_status pm_lift_polygon_vertices(const int32_t* vertices, const int32_t* n_vertices,
                                          int32_t max_vertices, const pm_plane* planes, int32_t n_frames,
                                          int32_t n_regions, const pm_intrinsics* K, double* X_out,
                                          pm_stream_t stream);

/* ---------------------------------------------------------------------- */
/* NEXT-4 of SURVEY §8(f), HOST code (no device work): the paper's map merge
 * gate and vertical-drift Kalman filter (§III-E) applied to the
 * plane table (one plane per region in place of the paper's polygon;
 * DESIGN.md readings Q30-Q34).  All in fp64. */
typedef struct {
    double x;      /* drift estimate x_k|k (metres, world z) */
    double P;      /* its covariance P_k|k */
} pm_drift_filter;

/* Eqs. 6-10 in order: x_pred = x (6); P_pred = P + sigma_p (7);
 * K = P_pred / (P_pred + sigma_m) (8); x = x_pred + K (z - x_pred) (9);
 * P = (1 - K) P_pred (10).  Updates *f, returns K (NaN if f is NULL). */
PM_API double pm_drift_kalman_step(pm_drift_filter* f, double z, double sigma_p, double sigma_m);

/* Eqs. 4-5: dz = |z_new - z_map| (written to *dz_out if not
 * NULL); returns 1 iff dz <= drift_tol ("merge"), else 0. */
PM_API int32_t pm_merge_gate(double z_new, double z_map, double drift_tol, double* dz_out);

typedef struct {
    double n[3];   /* unit normal, world frame */
    double c[3];   /* centroid, world frame (drift-compensated z) */
    double w;      /* merge weight: accumulated inlier count */
    int32_t n_obs; /* observations merged into this plane */
    int32_t pad;
} pm_map_plane;

typedef struct {
    double drift_tol;   /* Eq. 5 tolerance (paper: 0.05 m) */
    double normal_tol;  /* max angle between normals to match (rad) */
    double xy_radius;   /* max horizontal centroid distance to match (m) */
    double sigma_p;     /* Eq. 7 process noise */
    double sigma_m;     /* Eq. 8 measurement noise */
} pm_map_params;

/* One frame's plane table into the map (Q31-Q34): PM_PLANE_OK
 * planes to the world frame with `pose` (row-major 4x4 camera-to-world),
 * z minus the drift estimate; each is matched to the map plane (as it was
 * before this frame) that passes the gate -- normals within normal_tol,
 * horizontal centroid distance <= xy_radius, Eq. 5 on the centroid heights --
 * with the smallest horizontal distance (ties: lowest index); if any matched,
 * z_k = mean signed (z_new - z_map) + x and one Kalman step (Eqs. 6-10), the
 * incoming heights re-adjusted by the change of x; matched planes are merged
 * (inlier-weighted normal and centroid), the others appended in frame order.
 *   map          [map_capacity] pm_map_plane, *map_count in use (in/out)
 *   match_out    [n_planes] matched map index or -1 (inserted / not OK), nullable
 *   z_k_out      the drift measurement, NaN when nothing matched, nullable
 * Returns PM_ERR_WORKSPACE (map untouched) if the inserts exceed capacity. */
PM_API pm_status pm_plane_map_merge_frame(pm_map_plane* map, int32_t* map_count, int32_t map_capacity,
                                          const pm_plane* frame, int32_t n_planes, const double pose[16],
                                          pm_drift_filter* filter, const pm_map_params* prm,
                                          int32_t* match_out, double* z_k_out);

/* Number of kernel launches one pm_process_frames call enqueues (for the
 * bench's launch accounting; memsets excluded). */
PM_API int32_t pm_pipeline_kernel_launches(int32_t iters, int32_t n_regions);

/* Human-readable status. */
PM_API const char* pm_status_string(pm_status s);
/* ABI version (major * 10000 + minor * 100 + patch).  0.2.0 (200):
 * pm_ransac_options gained stage_events
 * (a caller built against 0.1 passes a shorter struct -- rebuild), PM_LABELS_RUNS,
 * pm_process_frames_host_async, PM_ADF_ENGINE_REG; engine value 2 removed. */
PM_API int32_t pm_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PMAP_H_ */
