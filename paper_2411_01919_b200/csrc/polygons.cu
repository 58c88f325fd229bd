// polygons.cu — NEXT-3 of SURVEY §8(f): the polygon glue between region
// labels and planes ("contours are extracted from these edges and
// simplified into polygons", Alg. 2 "for each detected contour c";
// S:236-251), batched over frames and regions:
//   start    : first pixel of every region in raster order (atomicMin)
//   trace    : one thread per (frame, region): Moore-neighbour walk of the
//              outer boundary (Q35) -- a sequential chain per region, the
//              parallelism is across regions and frames
//   simplify : one thread per contour: closed Douglas-Peucker (Q36) with an
//              explicit stack, exact 128-bit integer distance tests
//   raster   : one thread per pixel: lowest-index polygon containing the
//              pixel centre, half-open even-odd rule in exact integers (Q37/38)
//   lift     : one thread per vertex: ray / plane intersection in fp64 (Q39)
// Integer outputs are bit-identical to the oracle; lifted vertices follow
// the oracle's fp64 expression order.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "../../include/pmap.h"
#include "internal.h"

namespace pm {

namespace {

constexpr int kThreads = 256;
constexpr int32_t kNoStart = 0x7F7F7F7F;   // the byte-wise memset fill of `start` (no pixel)

__device__ __constant__ int kMoore[8][2] = {{1, 0}, {1, 1}, {0, 1}, {-1, 1}, {-1, 0}, {-1, -1}, {0, -1}, {1, -1}};

__global__ void __launch_bounds__(kThreads)
region_start_kernel(const int32_t* __restrict__ labels, int WH, int R, int32_t* __restrict__ start) {
    const size_t f = blockIdx.y;
    const int p = blockIdx.x * kThreads + threadIdx.x;
    const int l = p < WH ? labels[f * WH + p] : -1;
    // warp-aggregated: the lowest lane of each label group holds the group's
    // smallest raster index (p grows with the lane); one atomic per group
    const unsigned m = __match_any_sync(0xFFFFFFFFu, l);
    if (l >= 0 && l < R && (int)(threadIdx.x & 31) == __ffs(m) - 1) atomicMin(start + f * R + l, p);
}

__device__ __forceinline__ bool in_region(const int32_t* lab, int W, int H, int x, int y, int r) {
    return x >= 0 && y >= 0 && x < W && y < H && __ldg(lab + (size_t)y * W + x) == r;
}

// Q35 (oracle orc_trace_contour): clockwise Moore walk from the region's first
// raster pixel, backtrack west, Jacob's stopping criterion.  Points packed as
// x | y << 16; the full length is returned even beyond `cap`.
__global__ void __launch_bounds__(kThreads)
trace_kernel(const int32_t* __restrict__ labels, int W, int H, int R, const int32_t* __restrict__ start, int cap,
             uint32_t* __restrict__ pts, int32_t* __restrict__ len_out) {
    const int r = blockIdx.x * kThreads + threadIdx.x;
    const size_t f = blockIdx.y;
    if (r >= R) return;
    const int32_t s = start[f * R + r];
    int32_t* lo = len_out + f * R + r;
    if (s == kNoStart) { *lo = 0; return; }
    const int32_t* lab = labels + f * (size_t)W * H;
    uint32_t* out = pts + (f * R + r) * (size_t)cap;
    const int sx = s % W, sy = s / W;
    int px = sx, py = sy, bdir = 4, first_dir = -1, len = 0;
    for (;;) {
        // all 8 neighbour loads issued together (the step's latency is one
        // load, not up to eight), then the first region pixel clockwise after
        // the backtrack direction
        uint32_t mask = 0;
#pragma unroll
        for (int d = 0; d < 8; ++d)
            mask |= in_region(lab, W, H, px + kMoore[d][0], py + kMoore[d][1], r) ? (1u << d) : 0u;
        const int s0 = (bdir + 1) & 7;
        const uint32_t rot = ((mask >> s0) | (mask << (8 - s0))) & 0xFFu;
        const int found = rot ? (s0 + __ffs(rot) - 1) & 7 : -1;
        if (found < 0) {
            if (cap > 0) out[0] = (uint32_t)px | ((uint32_t)py << 16);
            len = 1;
            break;
        }
        if (px == sx && py == sy) {
            if (first_dir < 0) first_dir = found;
            else if (found == first_dir) break;
        }
        if (len < cap) out[len] = (uint32_t)px | ((uint32_t)py << 16);
        len++;
        const int bd = (found + 7) & 7;
        const int bx = px + kMoore[bd][0], by = py + kMoore[bd][1];
        px += kMoore[found][0];
        py += kMoore[found][1];
        const int dxb = bx - px, dyb = by - py;
#pragma unroll
        for (int d = 0; d < 8; ++d)
            if (kMoore[d][0] == dxb && kMoore[d][1] == dyb) bdir = d;
    }
    *lo = len;
}

__device__ __forceinline__ int px_x(uint32_t p) { return (int)(p & 0xFFFFu); }
__device__ __forceinline__ int px_y(uint32_t p) { return (int)(p >> 16); }

// Q36 (oracle orc_simplify_dp): anchors 0 and the farthest point; chain i..j
// (mod n) split at the point of largest |cross| (ties -> lowest index) if
// cross^2 * 256 > eps16^2 * len^2 (point distance when p_i == p_j).  keep[n]
// flags, then the kept points written in contour order.
__global__ void __launch_bounds__(128)
simplify_kernel(const uint32_t* __restrict__ pts, const int32_t* __restrict__ len_in, int R, int cap, int eps16,
                uint8_t* __restrict__ keep_ws, int2* __restrict__ stack_ws, int max_vertices,
                int32_t* __restrict__ verts, int32_t* __restrict__ n_verts) {
    const int r = blockIdx.x * 128 + threadIdx.x;
    const size_t f = blockIdx.y;
    if (r >= R) return;
    const size_t slot = f * R + r;
    const int n = min(len_in[slot], cap);
    const uint32_t* c = pts + slot * (size_t)cap;
    uint8_t* keep = keep_ws + slot * (size_t)cap;
    int2* stack = stack_ws + slot * (size_t)(cap + 4);
    int32_t* vout = verts + slot * (size_t)max_vertices * 2;
    if (n <= 0) { n_verts[slot] = 0; return; }
    for (int k = 0; k < n; ++k) keep[k] = 0;
    keep[0] = 1;
    if (n > 1) {
        int far = 0;
        long long fd = -1;
        const int x0 = px_x(c[0]), y0 = px_y(c[0]);
        for (int k = 1; k < n; ++k) {
            const long long dx = px_x(c[k]) - x0, dy = px_y(c[k]) - y0;
            const long long d2 = dx * dx + dy * dy;
            if (d2 > fd) { fd = d2; far = k; }
        }
        keep[far] = 1;
        // explicit stack; the oracle recurses on (i, best) before (best, j),
        // the order does not change the kept set
        int sp = 0;
        stack[sp++] = make_int2(far, n);
        stack[sp++] = make_int2(0, far);
        while (sp > 0) {
            const int2 seg = stack[--sp];
            const int i = seg.x, j = seg.y;
            const int cnt = (j - i + n) % n;
            if (cnt < 2) continue;
            const long long ax = px_x(c[i]), ay = px_y(c[i]);
            const long long bx = px_x(c[j % n]), by = px_y(c[j % n]);
            const long long dx = bx - ax, dy = by - ay;
            int best = -1;
            unsigned long long bestv = 0;
            for (int s = 1; s < cnt; ++s) {
                const int k = (i + s) % n;
                const long long qx = px_x(c[k]) - ax, qy = px_y(c[k]) - ay;
                unsigned long long v;
                if (dx == 0 && dy == 0) v = (unsigned long long)(qx * qx + qy * qy);
                else {
                    long long cr = dx * qy - dy * qx;
                    v = (unsigned long long)(cr < 0 ? -cr : cr);
                }
                if (best < 0 || v > bestv) { best = k; bestv = v; }
            }
            unsigned __int128 lhs, rhs;
            if (dx == 0 && dy == 0) {
                lhs = (unsigned __int128)bestv * 256u;
                rhs = (unsigned __int128)((long long)eps16 * eps16);
            } else {
                lhs = (unsigned __int128)bestv * bestv * 256u;
                rhs = (unsigned __int128)((long long)eps16 * eps16) * (unsigned __int128)(dx * dx + dy * dy);
            }
            if (lhs > rhs) {                     // depth <= kept points + 2 <= cap + 2
                keep[best] = 1;
                stack[sp++] = make_int2(best, j);
                stack[sp++] = make_int2(i, best);
            }
        }
    }
    int m = 0;
    for (int k = 0; k < n; ++k)
        if (keep[k]) {
            if (m < max_vertices) { vout[2 * m] = px_x(c[k]); vout[2 * m + 1] = px_y(c[k]); }
            ++m;
        }
    n_verts[slot] = m;
}

// bounding boxes of the polygons (x0, y0, x1, y1), empty -> x0 > x1
__global__ void __launch_bounds__(kThreads)
poly_bbox_kernel(const int32_t* __restrict__ verts, const int32_t* __restrict__ n_verts, int R, int max_vertices,
                 int4* __restrict__ bbox) {
    const int r = blockIdx.x * kThreads + threadIdx.x;
    const size_t f = blockIdx.y;
    if (r >= R) return;
    const size_t slot = f * R + r;
    const int m = min(n_verts[slot], max_vertices);
    const int32_t* v = verts + slot * (size_t)max_vertices * 2;
    int4 b = make_int4(1 << 30, 1 << 30, -(1 << 30), -(1 << 30));
    for (int k = 0; k < m; ++k) {
        b.x = min(b.x, v[2 * k]); b.y = min(b.y, v[2 * k + 1]);
        b.z = max(b.z, v[2 * k]); b.w = max(b.w, v[2 * k + 1]);
    }
    if (m < 3) b = make_int4(1, 1, 0, 0);       // fewer than 3 vertices: covers no pixel
    bbox[slot] = b;
}

// Q37/Q38 (oracle orc_rasterize_polygons): lowest polygon index whose
// half-open even-odd test holds at the pixel centre, else -1.
__global__ void __launch_bounds__(kThreads)
raster_kernel(const int32_t* __restrict__ verts, const int32_t* __restrict__ n_verts, const int4* __restrict__ bbox,
              int R, int max_vertices, int W, int H, int32_t* __restrict__ labels) {
    const size_t f = blockIdx.y;
    const int p = blockIdx.x * kThreads + threadIdx.x;
    if (p >= W * H) return;
    const int x = p % W, y = p / W;
    int lab = -1;
    for (int q = 0; q < R && lab < 0; ++q) {
        const size_t slot = f * R + q;
        const int4 b = __ldg(bbox + slot);
        if (x < b.x || x > b.z || y < b.y || y > b.w) continue;
        const int m = min(__ldg(n_verts + slot), max_vertices);
        const int32_t* v = verts + slot * (size_t)max_vertices * 2;
        int inside = 0;
        long long ax = __ldg(v + 2 * (m - 1)), ay = __ldg(v + 2 * (m - 1) + 1);
        for (int e = 0; e < m; ++e) {
            // edge a = v[e-1] -> b = v[e] (the oracle's edge set, visited from
            // the closing edge; parity is order-free), the oracle's exact test
            const long long bx = __ldg(v + 2 * e), by = __ldg(v + 2 * e + 1);
            if ((ay > y) != (by > y)) {
                const long long lhs = (x - ax) * (by - ay), rhs = (y - ay) * (bx - ax);
                if ((by > ay) ? (lhs < rhs) : (lhs > rhs)) inside ^= 1;
            }
            ax = bx; ay = by;
        }
        if (inside) lab = q;
    }
    labels[f * (size_t)W * H + p] = lab;
}

// Q39 (oracle orc_lift_vertices): X = -d/(n.r) r, r = ((u-cx)/fx, (v-cy)/fy, 1), fp64
__global__ void __launch_bounds__(kThreads)
lift_kernel(const int32_t* __restrict__ verts, const int32_t* __restrict__ n_verts, int R, int max_vertices,
            const pm_plane* __restrict__ planes, double fx, double fy, double cx, double cy, double* __restrict__ X) {
    const int t = blockIdx.x * kThreads + threadIdx.x;
    const size_t f = blockIdx.y;
    if (t >= R * max_vertices) return;
    const int r = t / max_vertices, k = t % max_vertices;
    const size_t slot = f * R + r;
    double* o = X + (slot * (size_t)max_vertices + k) * 3;
    const int m = min(n_verts[slot], max_vertices);
    const pm_plane pl = planes[slot];
    if (k >= m || pl.status != PM_PLANE_OK) { o[0] = o[1] = o[2] = NAN; return; }
    const int32_t* v = verts + slot * (size_t)max_vertices * 2;
    const double r0 = ((double)v[2 * k] - cx) / fx, r1 = ((double)v[2 * k + 1] - cy) / fy, r2 = 1.0;
    const double den = (double)pl.n[0] * r0 + (double)pl.n[1] * r1 + (double)pl.n[2] * r2;
    const double tt = den != 0.0 ? -(double)pl.d / den : NAN;
    if (!(tt > 0.0)) { o[0] = o[1] = o[2] = NAN; return; }
    o[0] = tt * r0; o[1] = tt * r1; o[2] = tt * r2;
}

size_t a256(size_t x) { return (x + 255) & ~(size_t)255; }

struct PolyWs {
    int32_t* start;
    uint32_t* pts;
    uint8_t* keep;
    int2* stack;
    int4* bbox;
    size_t bytes;
};

PolyWs poly_ws(void* base, int B, int R, int cap) {
    PolyWs w{};
    size_t o = 0;
    char* p = (char*)base;
    auto take = [&](size_t b) { void* q = p ? p + o : nullptr; o += a256(b); return q; };
    const size_t slots = (size_t)B * (R > 0 ? R : 1);
    w.start = (int32_t*)take(sizeof(int32_t) * slots);
    w.pts = (uint32_t*)take(sizeof(uint32_t) * slots * cap);
    w.keep = (uint8_t*)take(slots * cap);
    w.stack = (int2*)take(sizeof(int2) * slots * (cap + 4));
    w.bbox = (int4*)take(sizeof(int4) * slots);
    w.bytes = o;
    return w;
}

bool params_ok(const pm_polygon_params* p) {
    return p && p->eps16 >= 0 && p->max_contour >= 1 && p->max_vertices >= 3 && p->max_contour <= (1 << 24);
}

}  // namespace

}  // namespace pm

extern "C" {

PM_API size_t pm_region_polygons_workspace_bytes(int32_t n_frames, int32_t n_regions, int32_t max_contour) {
    if (n_frames < 1 || n_regions < 0 || max_contour < 1) return 0;
    return pm::poly_ws(nullptr, n_frames, n_regions, max_contour).bytes;
}

PM_API pm_status pm_region_polygons(const int32_t* labels, int32_t W, int32_t H, int32_t n_frames, int32_t n_regions,
                                    const pm_polygon_params* prm, int32_t* contour_len, int32_t* vertices,
                                    int32_t* n_vertices, void* workspace, size_t ws_bytes, pm_stream_t stream) {
    const pm::NvtxRange nvtx_("pmap:region_polygons");
    using namespace pm;
    if (!labels || !contour_len || !vertices || !n_vertices || W < 1 || H < 1 || W > 65535 || H > 65535 ||
        n_frames < 1 || n_regions < 0 || !params_ok(prm))
        return PM_ERR_INVALID_ARGUMENT;
    if (n_regions == 0) return PM_OK;
    if (!workspace || ((uintptr_t)workspace & 255u) ||
        ws_bytes < pm_region_polygons_workspace_bytes(n_frames, n_regions, prm->max_contour))
        return PM_ERR_WORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    const PolyWs w = poly_ws(workspace, n_frames, n_regions, prm->max_contour);
    const int WH = W * H;
    cudaError_t e = cudaMemsetAsync(w.start, 0x7F, sizeof(int32_t) * (size_t)n_frames * n_regions, st);
    if (e != cudaSuccess) return PM_ERR_CUDA;
    region_start_kernel<<<dim3((WH + kThreads - 1) / kThreads, n_frames), kThreads, 0, st>>>(labels, WH, n_regions,
                                                                                             w.start);
    trace_kernel<<<dim3((n_regions + kThreads - 1) / kThreads, n_frames), kThreads, 0, st>>>(
        labels, W, H, n_regions, w.start, prm->max_contour, w.pts, contour_len);
    simplify_kernel<<<dim3((n_regions + 127) / 128, n_frames), 128, 0, st>>>(
        w.pts, contour_len, n_regions, prm->max_contour, prm->eps16, w.keep, w.stack, prm->max_vertices, vertices,
        n_vertices);
    return cudaGetLastError() == cudaSuccess ? PM_OK : PM_ERR_CUDA;
}

PM_API pm_status pm_rasterize_polygons(const int32_t* vertices, const int32_t* n_vertices, int32_t max_vertices,
                                       int32_t W, int32_t H, int32_t n_frames, int32_t n_regions, int32_t* labels_out,
                                       void* workspace, size_t ws_bytes, pm_stream_t stream) {
    const pm::NvtxRange nvtx_("pmap:rasterize_polygons");
    using namespace pm;
    if (!vertices || !n_vertices || !labels_out || W < 1 || H < 1 || W > 65535 || H > 65535 || n_frames < 1 ||
        n_regions < 0 || max_vertices < 3)
        return PM_ERR_INVALID_ARGUMENT;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t need = sizeof(int4) * (size_t)n_frames * (n_regions > 0 ? n_regions : 1);
    if (!workspace || ((uintptr_t)workspace & 255u) || ws_bytes < need) return PM_ERR_WORKSPACE;
    int4* bbox = (int4*)workspace;
    if (n_regions > 0)
        poly_bbox_kernel<<<dim3((n_regions + kThreads - 1) / kThreads, n_frames), kThreads, 0, st>>>(
            vertices, n_vertices, n_regions, max_vertices, bbox);
    raster_kernel<<<dim3((W * H + kThreads - 1) / kThreads, n_frames), kThreads, 0, st>>>(
        vertices, n_vertices, bbox, n_regions, max_vertices, W, H, labels_out);
    return cudaGetLastError() == cudaSuccess ? PM_OK : PM_ERR_CUDA;
}

PM_API pm_status pm_lift_polygon_vertices(const int32_t* vertices, const int32_t* n_vertices, int32_t max_vertices,
                                          const pm_plane* planes, int32_t n_frames, int32_t n_regions,
                                          const pm_intrinsics* K, double* X_out, pm_stream_t stream) {
    const pm::NvtxRange nvtx_("pmap:lift_polygon_vertices");
    using namespace pm;
    if (!vertices || !n_vertices || !planes || !X_out || !K || n_frames < 1 || n_regions < 0 || max_vertices < 3 ||
        !(K->fx > 0.0f) || !(K->fy > 0.0f))
        return PM_ERR_INVALID_ARGUMENT;
    if (n_regions == 0) return PM_OK;
    const int tot = n_regions * max_vertices;
    lift_kernel<<<dim3((tot + kThreads - 1) / kThreads, n_frames), kThreads, 0, (cudaStream_t)stream>>>(
        vertices, n_vertices, n_regions, max_vertices, planes, (double)K->fx, (double)K->fy, (double)K->cx,
        (double)K->cy, X_out);
    return cudaGetLastError() == cudaSuccess ? PM_OK : PM_ERR_CUDA;
}

}  // extern "C"
