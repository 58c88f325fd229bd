// compact.cu — Alg. 2 ℓ2 "Extract depth values within c from I" for
// every region of every frame at once: a stable, deterministic compaction of
// the valid labelled pixels into per-region lists in raster order (the order
// hypothesis indices refer to).
//
//   count   : each warp owns a sub-tile of `sub_tile` consecutive pixels and
//             counts (region, sub-tile) occurrences.  Labels are spatially
//             coherent, so the warp keeps a run-length cache (current label,
//             running count) in registers and touches memory only when the
//             label changes; a step with several labels falls back to
//             __match_any_sync groups.  hist entries are owned by one warp:
//             no atomics, no ordering dependence.  For R <= 256 the
//             count_lane variant keeps the run cache per lane instead (shared
//             histogram row per warp), and skips the depth reads for frames
//             known to hold valid depths only (pm_process_frames).
//   scan    : per (frame, region) exclusive prefix over sub-tiles -> counts;
//             per frame exclusive prefix over regions -> region offsets.
//   scatter : the same warp walk, writing packed (u, v, z) points to
//             region_off + prefix + rank-in-step.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "internal.h"

namespace pm {

namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kWarpsPerBlock = 8;
constexpr int kPrefetch = 8;          // 32-pixel steps whose loads are issued together

PM_DEVINL unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__global__ void __launch_bounds__(kWarpsPerBlock * 32)
compact_count_kernel(const float* __restrict__ depth, const int32_t* __restrict__ labels,
                     int WH, int R, int sub_tile, int n_sub, int32_t* __restrict__ hist) {
    const int lane = threadIdx.x & 31;
    const int st = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    if (st >= n_sub) return;
    const size_t f = blockIdx.y;
    const float* d = depth + f * WH;
    const int32_t* l = labels + f * WH;
    int32_t* h = hist + f * (size_t)R * n_sub;
    const size_t beg = (size_t)st * sub_tile;
    const size_t end = min(beg + (size_t)sub_tile, (size_t)WH);
    int cur = -1, cnt = 0;
    for (size_t i00 = beg; i00 < end; i00 += 32 * kPrefetch) {
        int lraw[kPrefetch];
        float zraw[kPrefetch];
#pragma unroll
        for (int u = 0; u < kPrefetch; ++u) {        // all loads of kPrefetch steps in flight
            const size_t i = i00 + u * 32 + lane;
            lraw[u] = i < end ? __ldg(l + i) : -1;
            zraw[u] = i < end ? __ldg(d + i) : 0.0f;
        }
#pragma unroll
        for (int u = 0; u < kPrefetch; ++u) {
            if (i00 + u * 32 >= end) break;
            const int lab = (valid_depth(zraw[u]) && (unsigned)lraw[u] < (unsigned)R) ? lraw[u] : -1;
            if (__all_sync(kFull, lab == cur || lab < 0)) {
                cnt += __popc(__ballot_sync(kFull, lab >= 0));
                continue;
            }
            const int L = __reduce_max_sync(kFull, lab);
            if (cur >= 0 && lane == 0) h[(size_t)cur * n_sub + st] += cnt;
            __syncwarp();
            if (__all_sync(kFull, lab == L || lab < 0)) {          // one new label
                cur = L;
                cnt = __popc(__ballot_sync(kFull, lab >= 0));
                continue;
            }
            cur = -1;                                              // mixed step
            cnt = 0;
            const unsigned m = __match_any_sync(kFull, lab);
            if (lab >= 0 && lane == __ffs(m) - 1) h[(size_t)lab * n_sub + st] += __popc(m);
            __syncwarp();
        }
    }
    if (cur >= 0 && lane == 0) h[(size_t)cur * n_sub + st] += cnt;
}

// Count with a run cache per LANE (R <= kLaneCountMaxR): lane l walks pixels
// l, l+32, ... of the warp's sub-tile and flushes its (label, run length) into
// the warp's shared-memory histogram row only when its label changes, so a
// 32-pixel step costs ~8-12 instructions (the warp-vote walk above: ~37).
// The warp then writes its nonzero (region, sub-tile) entries -- the same
// owner-exclusive hist the scatter reads.  NEED_Z = false: the frame is known
// to hold valid depths only (depth_all_valid[f] == 0) and only labels are read.
constexpr int kLaneCountMaxR = 256;
template <bool NEED_Z>
PM_DEVINL void count_lane_walk(const float* __restrict__ d, const int32_t* __restrict__ l, unsigned beg, unsigned end,
                               int R, int lane, int* __restrict__ row) {
    int cur = -1, cnt = 0;
    for (unsigned i00 = beg; i00 < end; i00 += 32 * kPrefetch) {
        int lraw[kPrefetch];
        float zraw[kPrefetch];
#pragma unroll
        for (int u = 0; u < kPrefetch; ++u) {        // all loads of kPrefetch steps in flight
            const unsigned i = i00 + u * 32 + lane;
            lraw[u] = i < end ? __ldg(l + i) : -1;
            if (NEED_Z) zraw[u] = i < end ? __ldg(d + i) : 0.0f;
        }
#pragma unroll
        for (int u = 0; u < kPrefetch; ++u) {
            const int lab = ((!NEED_Z || valid_depth(zraw[u])) && (unsigned)lraw[u] < (unsigned)R) ? lraw[u] : -1;
            if (lab >= 0) {
                if (lab != cur) {                      // rare: a region boundary in this lane's column
                    if (cur >= 0) atomicAdd(row + cur, cnt);
                    cur = lab;
                    cnt = 0;
                }
                ++cnt;
            }
        }
    }
    if (cur >= 0) atomicAdd(row + cur, cnt);
}

// The same walk with 16-byte loads: lane l takes pixels 4l..4l+3 of every
// 128-pixel step (the histogram does not depend on the order a lane sees
// its pixels); a quarter of the load instructions.  Needs W*H % 4 == 0 and
// 16-byte aligned frame bases.
constexpr int kPrefetch4 = 4;
template <bool NEED_Z>
PM_DEVINL void count_lane_walk4(const float* __restrict__ d, const int32_t* __restrict__ l, unsigned beg,
                                unsigned end, int R, int lane, int* __restrict__ row) {
    int cur = -1, cnt = 0;
    auto take = [&](int lab, float z) {
        const int lb = ((!NEED_Z || valid_depth(z)) && (unsigned)lab < (unsigned)R) ? lab : -1;
        if (lb >= 0) {
            if (lb != cur) {                           // rare: a region boundary in this lane's pixels
                if (cur >= 0) atomicAdd(row + cur, cnt);
                cur = lb;
                cnt = 0;
            }
            ++cnt;
        }
    };
    for (unsigned i00 = beg; i00 < end; i00 += 128 * kPrefetch4) {
        int4 lr[kPrefetch4];
        float4 zr[kPrefetch4];
#pragma unroll
        for (int u = 0; u < kPrefetch4; ++u) {         // all loads of kPrefetch4 steps in flight
            const unsigned i = i00 + u * 128 + lane * 4;
            lr[u] = i < end ? __ldg(reinterpret_cast<const int4*>(l + i)) : make_int4(-1, -1, -1, -1);
            if (NEED_Z) zr[u] = i < end ? __ldg(reinterpret_cast<const float4*>(d + i)) : make_float4(0.f, 0.f, 0.f, 0.f);
            else zr[u] = make_float4(1.f, 1.f, 1.f, 1.f);
        }
#pragma unroll
        for (int u = 0; u < kPrefetch4; ++u) {
            take(lr[u].x, zr[u].x);
            take(lr[u].y, zr[u].y);
            take(lr[u].z, zr[u].z);
            take(lr[u].w, zr[u].w);
        }
    }
    if (cur >= 0) atomicAdd(row + cur, cnt);
}

__global__ void __launch_bounds__(kWarpsPerBlock * 32)
compact_count_lane_kernel(const float* __restrict__ depth, const int32_t* __restrict__ labels,
                          int WH, int R, int sub_tile, int n_sub, int32_t* __restrict__ hist,
                          const int* __restrict__ depth_all_valid) {
    __shared__ int s_h[kWarpsPerBlock][kLaneCountMaxR];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int st = blockIdx.x * kWarpsPerBlock + w;
    if (st >= n_sub) return;                     // warp-level only: no block barrier below
    const size_t f = blockIdx.y;
    int* row = s_h[w];
    for (int r = lane; r < R; r += 32) row[r] = 0;
    __syncwarp();
    const unsigned beg = (unsigned)st * (unsigned)sub_tile;
    const unsigned end = min(beg + (unsigned)sub_tile, (unsigned)WH);
    const float* d = depth + f * WH;
    const int32_t* l = labels + f * WH;
    const bool need_z = depth_all_valid == nullptr || depth_all_valid[f] != 0;
    const bool vec = (WH & 3) == 0 && ((reinterpret_cast<uintptr_t>(depth) | reinterpret_cast<uintptr_t>(labels)) & 15) == 0;
    if (vec) {
        if (need_z) count_lane_walk4<true>(d, l, beg, end, R, lane, row);
        else count_lane_walk4<false>(d, l, beg, end, R, lane, row);
    } else if (need_z) {
        count_lane_walk<true>(d, l, beg, end, R, lane, row);
    } else {
        count_lane_walk<false>(d, l, beg, end, R, lane, row);
    }
    __syncwarp();
    int32_t* h = hist + f * (size_t)R * n_sub;
    for (int r = lane; r < R; r += 32) {
        const int v = row[r];
        if (v) h[(size_t)r * n_sub + st] = v;
    }
}

// one warp per (frame, region): exclusive prefix over sub-tiles, total count
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
compact_scan_kernel(int R, int n_sub, int32_t* __restrict__ hist, int32_t* __restrict__ region_cnt) {
    const int lane = threadIdx.x & 31;
    const int r = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    if (r >= R) return;
    const size_t f = blockIdx.y;
    int32_t* row = hist + (f * R + r) * (size_t)n_sub;
    int carry = 0;
    for (int s0 = 0; s0 < n_sub; s0 += 32) {
        const int s = s0 + lane;
        const int v = s < n_sub ? row[s] : 0;
        int incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += t;
        }
        if (s < n_sub) row[s] = carry + incl - v;
        carry += __shfl_sync(kFull, incl, 31);
    }
    if (lane == 0) region_cnt[f * R + r] = carry;
}

// one block per frame: region_off[f][0..R] = exclusive prefix of region_cnt
__global__ void __launch_bounds__(1024)
compact_offsets_kernel(int R, const int32_t* __restrict__ region_cnt, int32_t* __restrict__ region_off) {
    __shared__ int warp_tot[32];
    __shared__ int carry_s;
    const size_t f = blockIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int32_t* cnt = region_cnt + f * R;
    int32_t* off = region_off + f * (size_t)(R + 1);
    if (threadIdx.x == 0) carry_s = 0;
    __syncthreads();
    for (int base = 0; base < R; base += 1024) {
        const int r = base + threadIdx.x;
        const int v = r < R ? cnt[r] : 0;
        int incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) warp_tot[w] = incl;
        __syncthreads();
        if (w == 0) {
            int x = warp_tot[lane];
            int xi = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(kFull, xi, o);
                if (lane >= o) xi += t;
            }
            warp_tot[lane] = xi - x;                         // exclusive warp prefix
        }
        __syncthreads();
        const int carry = carry_s;
        if (r < R) off[r] = carry + warp_tot[w] + incl - v;
        __syncthreads();
        if (threadIdx.x == 1023) carry_s = carry + warp_tot[w] + incl;
        __syncthreads();
    }
    if (threadIdx.x == 0) off[R] = carry_s;
}

__global__ void __launch_bounds__(kWarpsPerBlock * 32)
compact_scatter_kernel(const float* __restrict__ depth, const int32_t* __restrict__ labels,
                       int W, int WH, int R, int sub_tile, int n_sub, int32_t* __restrict__ hist,
                       const int32_t* __restrict__ region_off, uint2* __restrict__ points) {
    const int lane = threadIdx.x & 31;
    const int st = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    if (st >= n_sub) return;
    const size_t f = blockIdx.y;
    const float* d = depth + f * WH;
    const int32_t* l = labels + f * WH;
    int32_t* h = hist + f * (size_t)R * n_sub;
    const int32_t* off = region_off + f * (size_t)(R + 1);
    uint2* pts = points + f * WH;
    const size_t beg = (size_t)st * sub_tile;
    const size_t end = min(beg + (size_t)sub_tile, (size_t)WH);
    const unsigned lt = lanemask_lt();
    int cur = -1, rel = 0, roff = 0;       // cached label, next rank within region, region offset
    // image coordinates (pu, pv) of this lane's pixel, advanced by 32 pixels
    // per step (one division per sub-tile instead of a div/mod per step)
    unsigned pu = (unsigned)((beg + lane) % (unsigned)W), pv = (unsigned)((beg + lane) / (unsigned)W);
    for (size_t i00 = beg; i00 < end; i00 += 32 * kPrefetch) {
        int lraw[kPrefetch];
        float zraw[kPrefetch];
#pragma unroll
        for (int u = 0; u < kPrefetch; ++u) {        // all loads of kPrefetch steps in flight
            const size_t i = i00 + u * 32 + lane;
            lraw[u] = i < end ? __ldg(l + i) : -1;
            zraw[u] = i < end ? __ldg(d + i) : 0.0f;
        }
#pragma unroll
        for (int u = 0; u < kPrefetch; ++u) {
            const size_t i0 = i00 + u * 32;
            if (i0 >= end) break;
            const int lab = (valid_depth(zraw[u]) && (unsigned)lraw[u] < (unsigned)R) ? lraw[u] : -1;
            const uint2 pk = make_uint2(pu | (pv << 16), __float_as_uint(zraw[u]));   // used iff lab >= 0
            pu += 32;
            while (pu >= (unsigned)W) { pu -= (unsigned)W; ++pv; }
            bool fast = __all_sync(kFull, lab == cur || lab < 0);
            if (!fast) {
                const int L = __reduce_max_sync(kFull, lab);
                if (cur >= 0 && lane == 0) h[(size_t)cur * n_sub + st] = rel;     // flush
                __syncwarp();
                if (__all_sync(kFull, lab == L || lab < 0)) {
                    cur = L;
                    rel = h[(size_t)L * n_sub + st];
                    roff = off[L];
                    fast = true;
                } else {
                    cur = -1;
                    const unsigned m = __match_any_sync(kFull, lab);
                    const int leader = __ffs(m) - 1;
                    int b = 0;
                    if (lab >= 0 && lane == leader) {
                        const int r0 = h[(size_t)lab * n_sub + st];
                        h[(size_t)lab * n_sub + st] = r0 + __popc(m);
                        b = off[lab] + r0;
                    }
                    b = __shfl_sync(kFull, b, leader);
                    PM_CHECK(lab < 0 || (b + __popc(m & lt) >= 0 && b + __popc(m & lt) < WH));
                    if (lab >= 0) pts[b + __popc(m & lt)] = pk;
                    __syncwarp();
                }
            }
            if (fast) {
                const unsigned bal = __ballot_sync(kFull, lab >= 0);
                PM_CHECK(lab < 0 || (roff + rel + __popc(bal & lt) >= 0 && roff + rel + __popc(bal & lt) < WH));
                if (lab >= 0) pts[roff + rel + __popc(bal & lt)] = pk;
                rel += __popc(bal);
            }
        }
    }
    if (cur >= 0 && lane == 0) h[(size_t)cur * n_sub + st] = rel;
}

}  // namespace

cudaError_t compact_run(const float* depth, const int32_t* labels, const RansacWorkspace& ws,
                        cudaStream_t stream, const int* depth_all_valid) {
    const int WH = ws.W * ws.H;
    cudaError_t e = cudaMemsetAsync(ws.hist, 0, sizeof(int32_t) * (size_t)ws.B * ws.R * ws.n_sub, stream);
    if (e != cudaSuccess) return e;
    const dim3 blk(kWarpsPerBlock * 32);
    const dim3 g_tiles((ws.n_sub + kWarpsPerBlock - 1) / kWarpsPerBlock, ws.B);
    if (ws.R <= kLaneCountMaxR && (long long)ws.W * ws.H < (1ll << 31))
        compact_count_lane_kernel<<<g_tiles, blk, 0, stream>>>(depth, labels, WH, ws.R, ws.sub_tile, ws.n_sub,
                                                               ws.hist, depth_all_valid);
    else
        compact_count_kernel<<<g_tiles, blk, 0, stream>>>(depth, labels, WH, ws.R, ws.sub_tile, ws.n_sub, ws.hist);
    const dim3 g_regions((ws.R + kWarpsPerBlock - 1) / kWarpsPerBlock, ws.B);
    compact_scan_kernel<<<g_regions, blk, 0, stream>>>(ws.R, ws.n_sub, ws.hist, ws.region_cnt);
    compact_offsets_kernel<<<ws.B, 1024, 0, stream>>>(ws.R, ws.region_cnt, ws.region_off);
    compact_scatter_kernel<<<g_tiles, blk, 0, stream>>>(depth, labels, ws.W, WH, ws.R, ws.sub_tile,
                                                        ws.n_sub, ws.hist, ws.region_off, ws.points);
    return cudaGetLastError();
}

}  // namespace pm
