// segment.cu — NEXT-2: region labels from the normal image on the device,
// the step the paper puts between Alg. 1 and Alg. 2 ("edges are detected from
// the normal vector image using the Canny edge detection algorithm.
// Subsequently, contours are extracted from these edges").
// Readings (Q26-Q29): Canny on the 8-bit RGB normal image
// c = rint((n + 1) * 127.5), 3x3 Sobel with replicated borders, L2 magnitude
// of the strongest channel (integers: exact), OpenCV's non-maximum
// suppression, 8-connected hysteresis; invalid normals are edges; a 3x3
// dilation; regions = 4-connected components of non-edge pixels with
// >= min_area pixels, numbered by (size desc, smallest raster index).
//
// Kernels: candidates (tile + 2-pixel halo in shared memory: u8 conversion,
// Sobel, NMS) -> union-find over candidates (8-conn, lock-free atomicMin
// linking, roots = smallest index) -> strong flags -> edges -> dilation ->
// union-find over non-edge pixels (4-conn) -> sizes -> kept roots -> ranks
// (each kept root counts the keys ahead of it: deterministic) -> labels.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/pmap.h"
#include "common.cuh"
#include "internal.h"

namespace pm {

namespace {

constexpr int kTX = 32, kTY = 8;          // candidate kernel block
constexpr int kTW = 32, kTH = 16;         // candidate tile
constexpr int kEW = kTW + 4, kEH = kTH + 4;   // + 2-pixel halo

PM_DEVINL int to_u8(float n) {
    const int q = __float2int_rn(__fmul_rn(__fadd_rn(n, 1.0f), 127.5f));
    return q < 0 ? 0 : (q > 255 ? 255 : q);
}

// cls bits: 0-1 Canny class (0 none, 1 weak candidate, 2 strong), bit 2 invalid normal
__global__ void __launch_bounds__(kTX * kTY)
seg_candidates_kernel(const float* __restrict__ normals, int W, int H, long long low2, long long high2,
                      uint8_t* __restrict__ cls) {
    __shared__ uint8_t img[3][kEH][kEW];
    __shared__ int mag[kTH + 2][kTW + 2];
    const size_t f = blockIdx.z;
    const size_t HW = (size_t)W * H;
    const float* nrm = normals + f * 3 * HW;
    const int x0 = blockIdx.x * kTW, y0 = blockIdx.y * kTH;
    const int tid = threadIdx.y * kTX + threadIdx.x;
    for (int i = tid; i < kEW * kEH; i += kTX * kTY) {
        const int sy = i / kEW, sx = i % kEW;
        const int gy = min(max(y0 + sy - 2, 0), H - 1), gx = min(max(x0 + sx - 2, 0), W - 1);
        const size_t o = (size_t)gy * W + gx;
#pragma unroll
        for (int c = 0; c < 3; ++c) img[c][sy][sx] = (uint8_t)to_u8(__ldg(nrm + c * HW + o));
    }
    __syncthreads();
    // L2 magnitude of the strongest channel on tile + 1 (0 outside the image)
    auto sobel = [&](int sy, int sx, int c, int& gx, int& gy) {
        gx = ((int)img[c][sy - 1][sx + 1] - img[c][sy - 1][sx - 1]) + 2 * ((int)img[c][sy][sx + 1] - img[c][sy][sx - 1]) +
             ((int)img[c][sy + 1][sx + 1] - img[c][sy + 1][sx - 1]);
        gy = ((int)img[c][sy + 1][sx - 1] - img[c][sy - 1][sx - 1]) + 2 * ((int)img[c][sy + 1][sx] - img[c][sy - 1][sx]) +
             ((int)img[c][sy + 1][sx + 1] - img[c][sy - 1][sx + 1]);
    };
    for (int i = tid; i < (kTW + 2) * (kTH + 2); i += kTX * kTY) {
        const int my = i / (kTW + 2), mx = i % (kTW + 2);
        const int gy = y0 + my - 1, gx = x0 + mx - 1;
        int best = 0;
        if (gy >= 0 && gy < H && gx >= 0 && gx < W) {
            best = -1;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                int sx_, sy_;
                sobel(my + 1, mx + 1, c, sx_, sy_);
                const int m = sx_ * sx_ + sy_ * sy_;
                if (m > best) best = m;
            }
        }
        mag[my][mx] = best;
    }
    __syncthreads();
    const int TG22 = (int)(0.4142135623730950488016887242097 * (1 << 15) + 0.5);
    for (int i = tid; i < kTW * kTH; i += kTX * kTY) {
        const int ty = i / kTW, tx = i % kTW;
        const int gy = y0 + ty, gx = x0 + tx;
        if (gy >= H || gx >= W) continue;
        const int sy = ty + 2, sx = tx + 2, my = ty + 1, mx = tx + 1;
        int best = -1, bx = 0, by = 0;
#pragma unroll
        for (int c = 0; c < 3; ++c) {                       // first channel wins ties
            int gxc, gyc;
            sobel(sy, sx, c, gxc, gyc);
            const int m = gxc * gxc + gyc * gyc;
            if (m > best) { best = m; bx = gxc; by = gyc; }
        }
        const long long m = best;
        uint8_t c_out = 0;
        if (m > low2) {
            const long long x = bx < 0 ? -bx : bx, y = (long long)(by < 0 ? -by : by) << 15;
            const long long tg22x = x * TG22;
            bool keep;
            if (y < tg22x) {
                keep = m > mag[my][mx - 1] && m >= mag[my][mx + 1];
            } else {
                const long long tg67x = tg22x + (x << 16);
                if (y > tg67x) {
                    keep = m > mag[my - 1][mx] && m >= mag[my + 1][mx];
                } else {
                    const int s = ((bx ^ by) < 0) ? -1 : 1;
                    keep = m > mag[my - 1][mx - s] && m > mag[my + 1][mx + s];
                }
            }
            if (keep) c_out = m > high2 ? 2 : 1;
        }
        const size_t o = (size_t)gy * W + gx;
        if (nrm[o] == 0.0f && nrm[HW + o] == 0.0f && nrm[2 * HW + o] == 0.0f) c_out |= 4;
        cls[f * HW + o] = c_out;
    }
}

// ---- lock-free union-find (roots are the smallest index of their component)
PM_DEVINL int uf_find(const int* parent, int p) {
    int q = __ldcg(parent + p);
    while (q != p) {
        p = q;
        q = __ldcg(parent + p);
    }
    return p;
}

PM_DEVINL void uf_unite(int* parent, int a, int b) {
    while (true) {
        a = uf_find(parent, a);
        b = uf_find(parent, b);
        if (a == b) return;
        if (a > b) { const int t = a; a = b; b = t; }
        const int old = atomicMin(parent + b, a);
        if (old == b) return;
        b = old;
    }
}

constexpr int kT = 256;


__global__ void __launch_bounds__(kT) seg_uf_flatten(int HW, int* __restrict__ parent) {
    const size_t i = (size_t)blockIdx.x * kT + threadIdx.x;
    const size_t f = blockIdx.y;
    if (i >= (size_t)HW) return;
    int* par = parent + f * HW;
    if (par[i] >= 0) par[i] = uf_find(par, (int)i);
}

// strong candidates flag their root
__global__ void __launch_bounds__(kT)
seg_strong(const uint8_t* __restrict__ cls, int HW, const int* __restrict__ parent, int* __restrict__ flag) {
    const size_t i = (size_t)blockIdx.x * kT + threadIdx.x;
    const size_t f = blockIdx.y;
    if (i >= (size_t)HW) return;
    if ((cls[f * HW + i] & 3) == 2) atomicOr(flag + f * HW + parent[f * HW + i], 1);
}

// edge0 = (candidate of a component with a strong pixel) | invalid normal; then 3x3 dilation
__global__ void __launch_bounds__(kT)
seg_edges(const uint8_t* __restrict__ cls, int HW, const int* __restrict__ parent, const int* __restrict__ flag,
          uint8_t* __restrict__ e0) {
    const size_t i = (size_t)blockIdx.x * kT + threadIdx.x;
    const size_t f = blockIdx.y;
    if (i >= (size_t)HW) return;
    const uint8_t c = cls[f * HW + i];
    bool e = (c & 4) != 0;
    if ((c & 3) != 0) e = e || flag[f * HW + parent[f * HW + i]] != 0;
    e0[f * HW + i] = e ? 1 : 0;
}

__global__ void __launch_bounds__(kT)
seg_dilate(const uint8_t* __restrict__ e0, int W, int H, uint8_t* __restrict__ e1) {
    const size_t i = (size_t)blockIdx.x * kT + threadIdx.x;
    const size_t f = blockIdx.y;
    const size_t HW = (size_t)W * H;
    if (i >= HW) return;
    const int v = (int)(i / W), u = (int)(i % W);
    const uint8_t* e = e0 + f * HW;
    uint8_t any = 0;
    for (int dv = -1; dv <= 1; ++dv) {
        const int vv = v + dv;
        if (vv < 0 || vv >= H) continue;
        for (int du = -1; du <= 1; ++du) {
            const int uu = u + du;
            if (uu < 0 || uu >= W) continue;
            any |= e[(size_t)vv * W + uu];
        }
    }
    e1[f * HW + i] = any;
}

// component sizes; neighbouring pixels share roots, so lanes with the same
// root combine their increments first (one atomic per root per warp)
__global__ void __launch_bounds__(kT)
seg_sizes(int HW, const int* __restrict__ parent, int* __restrict__ size) {
    const size_t i = (size_t)blockIdx.x * kT + threadIdx.x;
    const size_t f = blockIdx.y;
    const int r = i < (size_t)HW ? parent[f * HW + i] : -1;
    const unsigned m = __match_any_sync(0xFFFFFFFFu, r);
    if (r >= 0 && (int)(threadIdx.x & 31) == __ffs(m) - 1) atomicAdd(size + f * HW + r, __popc(m));
}

// Block-local labelling of the non-edge pixels (4-connectivity) of a
// 32 x 32 tile in shared memory, then the global parent of every pixel is the
// global index of its tile-local root (the tile's smallest raster index of
// that piece: tile-local order is monotone in global raster order).  Only
// pixels on the tile's west / north border are merged globally afterwards.
constexpr int kCT = 32;
PM_DEVINL int l_find(const int* lp, int p) {
    int q = lp[p];
    while (q != p) { p = q; q = lp[p]; }
    return p;
}
PM_DEVINL void l_unite(int* lp, int a, int b) {
    while (true) {
        a = l_find(lp, a);
        b = l_find(lp, b);
        if (a == b) return;
        if (a > b) { const int t = a; a = b; b = t; }
        const int old = atomicMin(lp + b, a);
        if (old == b) return;
        b = old;
    }
}

__global__ void __launch_bounds__(256)
seg_local_ccl4(const uint8_t* __restrict__ edge, int W, int H, int* __restrict__ parent) {
    __shared__ int lp[kCT * kCT];
    __shared__ unsigned rowmask[kCT];
    const size_t f = blockIdx.z;
    const size_t HW = (size_t)W * H;
    const int x0 = blockIdx.x * kCT, y0 = blockIdx.y * kCT;
    const uint8_t* e = edge + f * HW;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // run start of lane's column in a row mask (first pixel after the last
    // edge pixel to its left)
    auto run_start = [&](unsigned m) {
        const unsigned bg = ~m & ((1u << lane) - 1u);
        return bg ? 32 - __clz(bg) : 0;
    };
    // (1) horizontal runs: one warp per row (kCT = 32 columns), every pixel
    // points at its run's first pixel, which is the run's root
    for (int ly = warp; ly < kCT; ly += 8) {
        const int gy = y0 + ly, gx = x0 + lane;
        const bool fg = gy < H && gx < W && e[(size_t)gy * W + gx] == 0;
        const unsigned m = __ballot_sync(0xFFFFFFFFu, fg);
        if (lane == 0) rowmask[ly] = m;
        lp[ly * kCT + lane] = fg ? ly * kCT + run_start(m) : -1;
    }
    __syncthreads();
    // (2) one union per pair of vertically overlapping runs, at the first
    // column of their overlap (union by minimum index: canonical roots)
    for (int ly = 1 + warp; ly < kCT; ly += 8) {
        const unsigned m = rowmask[ly], mn = rowmask[ly - 1];
        if (((m & mn) >> lane) & 1u) {
            const int s = run_start(m), sn = run_start(mn);
            if (lane == max(s, sn)) l_unite(lp, ly * kCT + s, (ly - 1) * kCT + sn);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kCT * kCT; i += 256) {
        const int ly = i / kCT, lx = i % kCT;
        const int gy = y0 + ly, gx = x0 + lx;
        if (gy >= H || gx >= W) continue;
        int g = -1;
        if (lp[i] >= 0) {
            const int r = l_find(lp, i);
            g = (y0 + r / kCT) * W + (x0 + r % kCT);
        }
        parent[f * HW + (size_t)gy * W + gx] = g;
    }
}

// Hysteresis components (8-connectivity over Canny candidates, cls & 3 != 0),
// tile-local first: horizontal runs per row (one warp per row), then one union
// per pair of 8-adjacent runs in consecutive rows at the first column where
// they touch (run A in row y touches run B in row y-1 at column x iff B holds
// one of x-1, x, x+1; the first such x in A is max(sA, sB - 1)).  Roots are
// the minimum local index (canonical), written as global indices.
__global__ void __launch_bounds__(256)
seg_local_ccl8(const uint8_t* __restrict__ cls, int W, int H, int* __restrict__ parent) {
    __shared__ int lp[kCT * kCT];
    __shared__ unsigned rowmask[kCT];
    const size_t f = blockIdx.z;
    const size_t HW = (size_t)W * H;
    const int x0 = blockIdx.x * kCT, y0 = blockIdx.y * kCT;
    const uint8_t* c = cls + f * HW;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    auto start_at = [](unsigned m, int x) {          // run start of column x (x in the run)
        const unsigned bg = ~m & ((1u << x) - 1u);
        return bg ? 32 - __clz(bg) : 0;
    };
    for (int ly = warp; ly < kCT; ly += 8) {
        const int gy = y0 + ly, gx = x0 + lane;
        const bool fg = gy < H && gx < W && (c[(size_t)gy * W + gx] & 3) != 0;
        const unsigned m = __ballot_sync(0xFFFFFFFFu, fg);
        if (lane == 0) rowmask[ly] = m;
        lp[ly * kCT + lane] = fg ? ly * kCT + start_at(m, lane) : -1;
    }
    __syncthreads();
    for (int ly = 1 + warp; ly < kCT; ly += 8) {
        const unsigned m = rowmask[ly], mn = rowmask[ly - 1];
        if (!((m >> lane) & 1u)) continue;
        const int sA = start_at(m, lane);
#pragma unroll
        for (int dx = -1; dx <= 1; ++dx) {
            const int p = lane + dx;
            if (p < 0 || p >= 32 || !((mn >> p) & 1u)) continue;
            const int sB = start_at(mn, p);
            if (lane == max(sA, sB - 1)) l_unite(lp, ly * kCT + sA, (ly - 1) * kCT + sB);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kCT * kCT; i += 256) {
        const int ly = i / kCT, lx = i % kCT;
        const int gy = y0 + ly, gx = x0 + lx;
        if (gy >= H || gx >= W) continue;
        int g = -1;
        if (lp[i] >= 0) {
            const int r = l_find(lp, i);
            g = (y0 + r / kCT) * W + (x0 + r % kCT);
        }
        parent[f * HW + (size_t)gy * W + gx] = g;
    }
}

// 8-connected merge across tile borders: pixels of a tile's west column and
// north row unite with their W, NW, N, NE neighbours in other tiles
__global__ void __launch_bounds__(kT)
seg_border_merge8(int W, int H, int* __restrict__ parent) {
    const size_t i = (size_t)blockIdx.x * kT + threadIdx.x;
    const size_t f = blockIdx.y;
    const size_t HW = (size_t)W * H;
    if (i >= HW) return;
    const int v = (int)(i / W), u = (int)(i % W);
    const bool west = u > 0 && (u % kCT) == 0, north = v > 0 && (v % kCT) == 0;
    const bool east_edge = u < W - 1 && ((u + 1) % kCT) == 0;   // NE neighbour in the next tile column
    if (!west && !north && !(east_edge && v > 0)) return;
    int* par = parent + f * HW;
    if (__ldcg(par + i) < 0) return;
    if (west && __ldcg(par + i - 1) >= 0) uf_unite(par, (int)i, (int)i - 1);
    if (v > 0) {
        // NW crosses a border if west or north; N if north; NE if north or east_edge
        if (u > 0 && (west || north) && __ldcg(par + i - W - 1) >= 0) uf_unite(par, (int)i, (int)(i - W - 1));
        if (north && __ldcg(par + i - W) >= 0) uf_unite(par, (int)i, (int)(i - W));
        if (u < W - 1 && (north || east_edge) && __ldcg(par + i - W + 1) >= 0)
            uf_unite(par, (int)i, (int)(i - W + 1));
    }
}

// global merge across tile borders (west column and north row of each tile)
__global__ void __launch_bounds__(kT)
seg_border_merge4(int W, int H, int* __restrict__ parent) {
    const size_t i = (size_t)blockIdx.x * kT + threadIdx.x;
    const size_t f = blockIdx.y;
    const size_t HW = (size_t)W * H;
    if (i >= HW) return;
    const int v = (int)(i / W), u = (int)(i % W);
    const bool west = u > 0 && (u % kCT) == 0, north = v > 0 && (v % kCT) == 0;
    if (!west && !north) return;
    int* par = parent + f * HW;
    if (__ldcg(par + i) < 0) return;
    if (west && __ldcg(par + i - 1) >= 0) uf_unite(par, (int)i, (int)i - 1);
    if (north && __ldcg(par + i - W) >= 0) uf_unite(par, (int)i, (int)(i - W));
}

// roots of components with >= min_area pixels -> key list; every root's rank = -1
__global__ void __launch_bounds__(kT)
seg_collect(int HW, int min_area, const int* __restrict__ parent, const int* __restrict__ size,
            int* __restrict__ rank, unsigned long long* __restrict__ keys, int cap, int* __restrict__ count) {
    const size_t i = (size_t)blockIdx.x * kT + threadIdx.x;
    const size_t f = blockIdx.y;
    if (i >= (size_t)HW) return;
    if (parent[f * HW + i] != (int)i) return;
    rank[f * HW + i] = -1;
    const int s = size[f * HW + i];
    if (s < min_area) return;
    const int slot = atomicAdd(count + f, 1);
    if (slot < cap)
        keys[f * (size_t)cap + slot] = ((unsigned long long)(0xFFFFFFFFu - (unsigned)s) << 32) | (unsigned)i;
}

// rank of each kept root = number of keys before it (size desc, index asc)
__global__ void __launch_bounds__(kT)
seg_rank(const unsigned long long* __restrict__ keys, int cap, const int* __restrict__ count, int HW, int max_regions,
         int* __restrict__ rank, int32_t* __restrict__ n_regions) {
    const size_t f = blockIdx.y;
    const int n = min(count[f], cap);
    const int j = blockIdx.x * kT + threadIdx.x;
    if (j == 0 && n_regions) n_regions[f] = min(n, max_regions);
    if (j >= n) return;
    const unsigned long long* k = keys + f * (size_t)cap;
    const unsigned long long mine = k[j];
    int r = 0;
    for (int q = 0; q < n; ++q) r += k[q] < mine;
    if (r < max_regions) rank[f * HW + (int)(mine & 0xFFFFFFFFu)] = r;
}

__global__ void __launch_bounds__(kT)
seg_labels(int HW, const int* __restrict__ parent, const int* __restrict__ rank, int32_t* __restrict__ labels) {
    const size_t i = (size_t)blockIdx.x * kT + threadIdx.x;
    const size_t f = blockIdx.y;
    if (i >= (size_t)HW) return;
    const int r = parent[f * HW + i];
    labels[f * HW + i] = r >= 0 ? rank[f * HW + r] : -1;
}

size_t a256(size_t x) { return (x + 255) & ~(size_t)255; }

}  // namespace

struct SegLayout {
    uint8_t* cls;
    uint8_t* e0;
    uint8_t* e1;
    int* parent;
    int* aux;            // flags, then sizes
    int* rank;
    unsigned long long* keys;
    int* count;
    int cap;
    size_t total;
};

static SegLayout seg_layout(void* base, int W, int H, int B, int min_area) {
    SegLayout L{};
    const size_t HW = (size_t)W * H;
    L.cap = (int)(HW / (size_t)(min_area > 0 ? min_area : 1)) + 1;
    size_t o = 0;
    char* p = (char*)base;
    auto take = [&](size_t b) { void* q = p ? p + o : nullptr; o += a256(b); return q; };
    L.cls = (uint8_t*)take(B * HW);
    L.e0 = (uint8_t*)take(B * HW);
    L.e1 = (uint8_t*)take(B * HW);
    L.parent = (int*)take(sizeof(int) * B * HW);
    L.aux = (int*)take(sizeof(int) * B * HW);
    L.rank = (int*)take(sizeof(int) * B * HW);
    L.keys = (unsigned long long*)take(sizeof(unsigned long long) * B * (size_t)L.cap);
    L.count = (int*)take(sizeof(int) * B);
    L.total = o;
    return L;
}

}  // namespace pm

extern "C" {

PM_API size_t pm_segment_workspace_bytes(int32_t W, int32_t H, int32_t n_frames, int32_t min_area) {
    if (W < 1 || H < 1 || n_frames < 1 || min_area < 1) return 0;
    return pm::seg_layout(nullptr, W, H, n_frames, min_area).total;
}

PM_API pm_status pm_segment_regions(const float* normals, int32_t W, int32_t H, int32_t n_frames,
                                    const pm_segment_params* prm, int32_t* labels_out, int32_t* n_regions_out,
                                    uint8_t* edges_out, void* workspace, size_t ws_bytes, pm_stream_t stream) {
    const pm::NvtxRange nvtx_("pmap:segment_regions");
    using namespace pm;
    if (!normals || !labels_out || !prm || W < 3 || H < 3 || W > 65535 || H > 65535 || n_frames < 1 ||
        n_frames > 65535)
        return PM_ERR_INVALID_ARGUMENT;
    if (!(prm->canny_low >= 0.0f) || !(prm->canny_high >= 0.0f) || prm->min_area < 1 || prm->max_regions < 0 ||
        prm->max_regions > 65536)
        return PM_ERR_INVALID_ARGUMENT;
    if ((size_t)W * H > (size_t)0x7FFFFFFF) return PM_ERR_UNSUPPORTED;
    const size_t need = pm_segment_workspace_bytes(W, H, n_frames, prm->min_area);
    if (!workspace || ws_bytes < need || ((uintptr_t)workspace & 255u)) return PM_ERR_WORKSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    const SegLayout L = seg_layout(workspace, W, H, n_frames, prm->min_area);
    double lo = prm->canny_low, hi = prm->canny_high;
    if (lo > hi) { const double t = lo; lo = hi; hi = t; }
    const long long low2 = (long long)floor(lo > 0 ? lo * lo : lo);
    const long long high2 = (long long)floor(hi > 0 ? hi * hi : hi);
    const int HW = W * H;
    const dim3 gp((HW + kT - 1) / kT, n_frames);
    const size_t bytes = (size_t)n_frames * HW;
    seg_candidates_kernel<<<dim3((W + kTW - 1) / kTW, (H + kTH - 1) / kTH, n_frames), dim3(kTX, kTY), 0, s>>>(
        normals, W, H, low2, high2, L.cls);
    // hysteresis: components of candidates (8-conn) containing a strong pixel
    seg_local_ccl8<<<dim3((W + kCT - 1) / kCT, (H + kCT - 1) / kCT, n_frames), 256, 0, s>>>(L.cls, W, H, L.parent);
    seg_border_merge8<<<gp, kT, 0, s>>>(W, H, L.parent);
    seg_uf_flatten<<<gp, kT, 0, s>>>(HW, L.parent);
    if (cudaMemsetAsync(L.aux, 0, sizeof(int) * bytes, s) != cudaSuccess) return PM_ERR_CUDA;
    seg_strong<<<gp, kT, 0, s>>>(L.cls, HW, L.parent, L.aux);
    seg_edges<<<gp, kT, 0, s>>>(L.cls, HW, L.parent, L.aux, L.e0);
    seg_dilate<<<gp, kT, 0, s>>>(L.e0, W, H, L.e1);
    // regions: 4-connected components of non-edge pixels (tile-local first)
    seg_local_ccl4<<<dim3((W + kCT - 1) / kCT, (H + kCT - 1) / kCT, n_frames), 256, 0, s>>>(L.e1, W, H, L.parent);
    seg_border_merge4<<<gp, kT, 0, s>>>(W, H, L.parent);
    seg_uf_flatten<<<gp, kT, 0, s>>>(HW, L.parent);
    if (cudaMemsetAsync(L.aux, 0, sizeof(int) * bytes, s) != cudaSuccess) return PM_ERR_CUDA;
    if (cudaMemsetAsync(L.count, 0, sizeof(int) * n_frames, s) != cudaSuccess) return PM_ERR_CUDA;
    seg_sizes<<<gp, kT, 0, s>>>(HW, L.parent, L.aux);
    seg_collect<<<gp, kT, 0, s>>>(HW, prm->min_area, L.parent, L.aux, L.rank, L.keys, L.cap, L.count);
    seg_rank<<<dim3((L.cap + kT - 1) / kT, n_frames), kT, 0, s>>>(L.keys, L.cap, L.count, HW, prm->max_regions,
                                                                 L.rank, n_regions_out);
    seg_labels<<<gp, kT, 0, s>>>(HW, L.parent, L.rank, labels_out);
    if (edges_out && cudaMemcpyAsync(edges_out, L.e1, bytes, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
        return PM_ERR_CUDA;
    return cudaGetLastError() == cudaSuccess ? PM_OK : PM_ERR_CUDA;
}

}  // extern "C"
