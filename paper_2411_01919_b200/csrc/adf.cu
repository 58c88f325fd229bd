// adf.cu — Algorithm 1 of arXiv 2411.01919 on sm_100a:
// temporally blocked Perona–Malik diffusion (ℓ1-8) with the Sobel/normal
// stage (ℓ9-13) fused into the last pass.
//
// One CTA owns an output tile of (128 - 2RA) x 44 pixels of one frame.  It
// loads the tile plus an R-pixel halo (R = sweeps of this pass, +1 when the
// normal stage is fused; RA = R rounded up to 4 columns) into shared memory
// once with one TMA box, runs the pass's T Jacobi sweeps in shared memory on
// a region that shrinks by one pixel per sweep (ping-pong buffers), and
// writes the tile back: one HBM read and one write per T sweeps.
//
// Sweep inner loop ("column walk"): each thread owns a pair of adjacent
// columns of a row strip and walks down it keeping the north and centre pairs
// in registers; per row and pair: 3 shared loads (S pair, W, E), 1 store, 10
// packed FP32 instructions (FADD2/FMUL2/FFMA2, see below) and two MUFU.EX2,
// the next row's loads issued before this row's store.  The zero-flux image border (Q4) costs nothing per cell: a
// thread whose column is the first / last image column points its W / E
// address at the centre cell, the strip that starts on the first image row
// seeds N with the centre, and the last image row is peeled with S = centre.
// Tiles whose loaded region contains an invalid depth (holes) run the same
// walk with per-neighbour validity substitution (zero flux at holes, Q4), or
// -- the FIX kernels (PM_ADF_ENGINE_HOLES, or AUTO after dropout was seen) --
// the unchecked walk plus a recomputation of the cells next to a hole.
// Plain passes write their rows back by cp.async.bulk copies.
// Every path evaluates the identical _rn expression on identical operands,
// so the result is bitwise independent of tile shape, sweeps per pass,
// batching and engine.
#include <cuda_runtime.h>
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <atomic>
#include <mutex>
#include <type_traits>

#include "adf_cell.cuh"
#include "common.cuh"
#include "internal.h"

namespace pm {

namespace {
using namespace adfk;

constexpr int kThreads = 256;      // 8 warps (4 CTAs / SM for halo R <= 5)
constexpr int kWarps = kThreads / 32;
constexpr int kMaxItersPerPass = 16;

// Shared tile: kSW = 128 columns (four 32-lane column groups) x SH rows; the
// output tile is (kSW - 2R) x TH; smem cell (sx, sy) is image pixel
// (x0 + sx, y0 + sy); the image covers smem columns [ix0, ix1), rows [iy0, iy1).
constexpr int kSW = 128;
// Output rows per CTA.  44: a (44 + 2R)-row tile pair fits 4 CTAs per SM in
// shared memory for R <= 5 (the default passes), and 480-row frames split
// into 11 tiles wasting 4 rows (64-row tiles: 8 tiles, 32 wasted rows).
constexpr int kTH = 44;
// Hole lists: one per warp of the validity scan, kWarpHoles uint16 entries
// each, in the 512-B spare row.  A tile takes the fix-up path when every warp's
// list fits and the 5 stencil cells of all its holes fit 2 per thread
// (<= 102 invalid cells, ~1.5 % of a 52-row tile); otherwise the checked walk.
constexpr int kWarpHoles = kSW * 2 / kWarps;
constexpr int kFixItems = 2;
constexpr int kHoleCap = kFixItems * kThreads / 5;
// Per-tile record of the first pass's hole lists (list_mode 1 writes, 2
// reads): 8 uint16 counts, then the 512-B lists -- kListVecs + 1 uint4.
constexpr int kListVecs = kSW * 2 * 2 / 16;
static_assert(kWarps == 8, "the hole-list record header holds 8 uint16 per-warp counts (one uint4)");
PM_DEVINL size_t tile_index() { return ((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x; }

struct Box { int ix0, ix1, iy0, iy1; };

// One Jacobi sweep over smem rows [t, SH - t) x columns [PAD + t, kSW - PAD - t)
// (PAD = unused alignment columns), clipped to the image.  Warp w walks
// column group (w & 3), row half (w >> 2).
template <int SH, int PAD, bool CHECK, bool DIV>
PM_DEVINL void sweep(const float* __restrict__ cur, float* __restrict__ nxt, int t, const Box& b,
                     const AdfParams& p) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int kParts = kWarps / 4;
    const int x = (warp & 3) * 32 + lane;
    const int ylo = max(t, b.iy0), yhi = min(SH - t, b.iy1);
    const int half = (yhi - ylo + kParts - 1) / kParts;
    const int ys = ylo + (warp >> 2) * half;
    const int ye = min(ys + half, yhi);
    if (x < max(PAD + t, b.ix0) || x >= min(kSW - PAD - t, b.ix1) || ys >= ye) return;
    const int ylast = b.iy1 - 1;
    const int ymid = min(ye, ylast);            // rows [ys, ymid) have a real south neighbour
    const int offW = x == b.ix0 ? 0 : -1;       // zero flux at the image border (Q4)
    const int offE = x == b.ix1 - 1 ? 0 : 1;
    const float* col = cur + x;
    const float* colW = col + offW;
    const float* colE = col + offE;
    float* ocol = nxt + x;
    float C = col[ys * kSW];
    float N = ys == b.iy0 ? C : col[(ys - 1) * kSW];
    int y = ys;
#pragma unroll 4
    for (; y < ymid; ++y) {
        const float S = col[(y + 1) * kSW];
        const float W = colW[y * kSW];
        const float E = colE[y * kSW];
        PM_CHECK(ocol + y * kSW - nxt >= 0 && ocol + y * kSW - nxt < kSW * SH);
        PM_CHECK(col + (y + 1) * kSW - cur < kSW * (SH + 1) && colW + y * kSW - cur >= 0);
        ocol[y * kSW] = cell<CHECK, DIV>(C, N, S, W, E, p);
        N = C;
        C = S;
    }
    if (ye > ylast)                             // last image row: S = C
        ocol[y * kSW] = cell<CHECK, DIV>(C, N, C, colW[y * kSW], colE[y * kSW], p);
}

// Same sweep with two horizontally adjacent cells per thread (columns x, x+1,
// x even): per row one 8-byte load of the south pair, one load each for the
// outer west / east neighbours (the inner ones are the pair itself), one
// 8-byte store -- 2 shared accesses per cell instead of 4.  Requires the image
// columns [ix0, ix1) to start and end on even smem columns, so that a pair is
// entirely inside or outside the image.  A pair straddling the sweep region's
// edge also updates its outer cell; that cell lies outside every later
// region and is never read again.
template <int SH, int PAD, bool CHECK, bool DIV>
PM_DEVINL void sweep_pairs(const float* __restrict__ cur, float* __restrict__ nxt, int t, const Box& b,
                           const AdfParams& p) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int kParts = kWarps / 2;
    const int x = ((warp & 1) * 32 + lane) * 2;
    const int ylo = max(t, b.iy0), yhi = min(SH - t, b.iy1);
    const int q = (yhi - ylo + kParts - 1) / kParts;
    const int ys = ylo + (warp >> 1) * q;
    const int ye = min(ys + q, yhi);
    const int xa = max(PAD + t, b.ix0), xb = min(kSW - PAD - t, b.ix1);
    if (x + 2 <= xa || x >= xb || ys >= ye) return;
    const int ylast = b.iy1 - 1;
    const int ymid = min(ye, ylast);
    const int offW = x == b.ix0 ? 0 : -1;           // zero flux at the image border (Q4)
    const int offE = x + 2 == b.ix1 ? 1 : 2;
    const float* __restrict__ col = cur + x + ys * kSW;
    const float* __restrict__ colW = col + offW;
    const float* __restrict__ colE = col + offE;
    float* __restrict__ ocol = nxt + x + ys * kSW;
    auto ld2 = [](const float* a) { return *reinterpret_cast<const float2*>(a); };
    float2 C = ld2(col);
    float2 N = ys == b.iy0 ? C : ld2(col - kSW);
    // The cell pair in packed FP32.  CHECK (tiles with invalid depth, Q4):
    // every invalid neighbour -- outer (P) or inner (the other cell of the
    // pair, in Cs) -- is replaced by the centre (zero flux) and invalid
    // centres keep their value: the substitution of cell<true>, so both
    // cells still get the scalar rounding sequence.
    auto cellp = [&](float2 C, float2 N, float2 S, float2 P) -> float2 {
        if (!CHECK) return cell2<DIV>(C, N, S, P, make_float2(C.y, C.x), p);
        const bool vx = valid_depth(C.x), vy = valid_depth(C.y);
        const float2 Nv = make_float2(valid_depth(N.x) ? N.x : C.x, valid_depth(N.y) ? N.y : C.y);
        const float2 Sv = make_float2(valid_depth(S.x) ? S.x : C.x, valid_depth(S.y) ? S.y : C.y);
        const float2 Pv = make_float2(valid_depth(P.x) ? P.x : C.x, valid_depth(P.y) ? P.y : C.y);
        const float2 Cs = make_float2(vy ? C.y : C.x, vx ? C.x : C.y);
        float2 o = cell2<DIV>(C, Nv, Sv, Pv, Cs, p);
        o.x = vx ? keep_valid(o.x, p.keep_valid) : C.x;
        o.y = vy ? keep_valid(o.y, p.keep_valid) : C.y;
        return o;
    };
    // software-pipelined: the next row's S, W, E are loaded before this row's
    // store (loads are not hoisted above a possibly aliasing store).  The last
    // step prefetches one row past the region (at most row SH: the buffers
    // carry one spare row), never used.
    const int n = ymid - ys;
    float2 S = ld2(col + kSW);
    float2 P = make_float2(colW[0], colE[0]);
    auto step = [&]() {
        PM_CHECK(col + 2 * kSW - cur + 2 <= kSW * (SH + 1) && colW + kSW - cur >= 0 && colE + kSW - cur < kSW * (SH + 1));
        PM_CHECK(ocol - nxt >= 0 && ocol - nxt + 2 <= kSW * SH);
        const float2 S1 = ld2(col + 2 * kSW);
        const float2 P1 = make_float2(colW[kSW], colE[kSW]);
        *reinterpret_cast<float2*>(ocol) = cellp(C, N, S, P);
        N = C;
        C = S;
        S = S1;
        P = P1;
        col += kSW;
        colW += kSW;
        colE += kSW;
        ocol += kSW;
    };
    int i = 0;
#ifndef PM_ADF_WALK_UNROLL
    for (; i + 4 <= n; i += 4) {
        step(); step(); step(); step();
    }
    if (i < n) {                                    // 0-3 last rows, straight-line
        step();
        if (i + 1 < n) {
            step();
            if (i + 2 < n) step();
        }
    }
#else   // A/B knob (tools/build_variant.sh): rows per unrolled step
    constexpr int kWalkUnroll = PM_ADF_WALK_UNROLL;
#pragma unroll(kWalkUnroll)
    for (; i < n; ++i) step();
#endif
    if (ye > ylast)                                 // last image row: S = C
        *reinterpret_cast<float2*>(ocol) = cellp(C, N, C, P);
}

#ifdef PM_ADF_TIMING
// Per-phase SM-cycle counters of adf_pass_kernel (variant builds, tools/):
// load+scan, sweeps, epilogue (stores / normals); [3] = plain, [4..6] fused.
__device__ unsigned long long g_adf_prof[8];
#define PM_ATS(v) const long long v = clock64()
#define PM_AACC(k, a, b) if (threadIdx.x == 0) atomicAdd(&g_adf_prof[k], (unsigned long long)((b) - (a)))
#else
#define PM_ATS(v)
#define PM_AACC(k, a, b)
#endif

template <int R>
constexpr size_t pass_smem_bytes() { return sizeof(float) * ((size_t)2 * kSW * (kTH + 2 * R) + kSW); }

// Left halo rounded up to 4 columns: the TMA box must start on a 16-byte
// column boundary (measured on B200: other starts raise an illegal-instruction
// fault), so smem column 0 is image column bx * TW - RA.
template <int R>
__host__ __device__ constexpr int halo_x() { return (R + 3) & ~3; }
template <int R>
__host__ __device__ constexpr int tile_w() { return kSW - 2 * halo_x<R>(); }

// One pass of `iters` sweeps; halo R = iters (+1 when the normals are fused).
//   src [B][H][W] -> dst [B][H][W] (if dst) and normals [B][3][H][W] (if normals).
// FIX (PM_ADF_ENGINE_HOLES): tiles with a few holes run the unchecked walk
// plus the fix-up of the cells next to a hole (below) instead of the checked
// walk.  Its bookkeeping stays out of the FIX = false kernels, which are the
// default: it costs the hole-free tiles 1-4 %.
template <int R, bool DIV, bool FIX>
__global__ void __launch_bounds__(kThreads, 4)   // <= 64 registers: 4 CTAs / SM
adf_pass_kernel(const float* __restrict__ src, float* __restrict__ dst, float* __restrict__ normals,
                int W, int H, int iters, AdfParams p, const __grid_constant__ CUtensorMap tmap, int use_tma,
                int* __restrict__ frame_flags, int flag_mode, uint4* __restrict__ tile_lists, int list_mode) {
    constexpr int SH = kTH + 2 * R;
    constexpr int RA = halo_x<R>();
    constexpr int TW = tile_w<R>();
    constexpr int PAD = RA - R;
    extern __shared__ __align__(128) float smem[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ int s_wn[kWarps];               // invalid cells found by each warp's scan
    float* buf0 = smem;
    float* buf1 = smem + kSW * SH;
    // hole lists (smem (sy << 7) | sx of the invalid in-image cells, warp w's
    // at [w * kWarpHoles, ...)) in the spare row after buf1: the walks'
    // one-row-ahead prefetch reads that row but never uses it, nothing writes it
    uint16_t* hl = reinterpret_cast<uint16_t*>(smem + 2 * kSW * SH);
    const size_t frame = blockIdx.z;
    const size_t HW = (size_t)H * W;
    const float* in = src + frame * HW;
    const int x0 = blockIdx.x * TW - RA;       // image coords of smem (0, 0)
    const int y0 = blockIdx.y * kTH - R;
    Box b;
    b.ix0 = max(0, -x0); b.ix1 = min(kSW, W - x0);
    b.iy0 = max(0, -y0); b.iy1 = min(SH, H - y0);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    PM_ATS(t0);

    // load tile + halo: one TMA box (out-of-image cells zero-filled, never
    // read) or coalesced LDG rows; note whether every in-image pixel is valid
    // (fast path) or not (hole-aware path)
    bool all_valid = true;
    int wn = 0;                                // this warp's invalid cells (warp-uniform)
    if (use_tma) {
#ifndef PM_ADF_EXP_NOLOAD   // timing experiment only (wrong results): no tile load
        if (threadIdx.x == 0) mbar_init(&bar, 1);
        __syncthreads();
        if (threadIdx.x == 0) {
            mbar_arrive_expect_tx(&bar, (uint32_t)(sizeof(float) * kSW * SH));
            tma_load_3d(buf0, &tmap, x0, y0, (int)frame, &bar);
        }
        // fetched while the tile streams in: the frame flag (flag_mode 2) and,
        // FIX with list_mode 2, this tile's hole-list record (speculatively)
        int lflag = 1;
        uint4 lrec = make_uint4(0u, 0u, 0u, 0u);
        if (flag_mode == 2) lflag = frame_flags[frame];
        if (FIX && flag_mode == 2 && list_mode == 2 && threadIdx.x <= kListVecs)
            lrec = tile_lists[tile_index() * (kListVecs + 1) + threadIdx.x];   // (speculative)
        mbar_wait(&bar, 0);
#else
        const int lflag = flag_mode == 2 ? frame_flags[frame] : 1;
        uint4 lrec = make_uint4(0u, 0u, 0u, 0u);
        for (int i = threadIdx.x; i < kSW * SH; i += kThreads) buf0[i] = 1.0f + 1e-3f * (i & 7);
        __syncthreads();
#endif
        // validity scan (skipped when an earlier pass found the frame hole-free:
        // validity never changes, Q4): each lane checks 4 consecutive columns.
        // Passes with the first pass's tile geometry read that pass's hole
        // lists instead (list_mode 2; loads overlap the tile load).
        if (FIX && flag_mode == 2 && list_mode == 2) {
            if (lflag != 0 && threadIdx.x <= kListVecs) {
                const uint4 v = lrec;
                if (threadIdx.x == 0) {
                    const uint32_t c[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int w = 0; w < kWarps; ++w) s_wn[w] = (int)((c[w >> 1] >> (16 * (w & 1))) & 0xFFFFu);
                } else {
                    reinterpret_cast<uint4*>(hl)[threadIdx.x - 1] = v;
                }
            } else if (threadIdx.x < kWarps) {
                s_wn[threadIdx.x] = 0;
            }
        } else if (lflag != 0) {
            const int c0 = 4 * lane;  // (4 columns per lane: 32 lanes cover the 128-column tile)
            bool in[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) in[j] = c0 + j >= b.ix0 && c0 + j < b.ix1;
#pragma unroll(FIX ? 1 : (SH + kWarps - 1) / kWarps)
            for (int sy = b.iy0 + warp; sy < b.iy1; sy += kWarps) {
                const float4 v = *reinterpret_cast<const float4*>(buf0 + sy * kSW + c0);
                if constexpr (!FIX) {
                    all_valid &= (fast_depth(v.x) || !in[0]) && (fast_depth(v.y) || !in[1]) &&
                                 (fast_depth(v.z) || !in[2]) && (fast_depth(v.w) || !in[3]);
                    continue;
                }
                const unsigned bad = (fast_depth(v.x) || !in[0] ? 0u : 1u) | (fast_depth(v.y) || !in[1] ? 0u : 2u) |
                                     (fast_depth(v.z) || !in[2] ? 0u : 4u) | (fast_depth(v.w) || !in[3] ? 0u : 8u);
                all_valid &= bad == 0;
                // rare (warp-uniform branch): append the row's invalid cells to
                // the warp's list, lanes ranked by ballot, one cell per lane per round
                if (__any_sync(0xffffffffu, bad != 0)) {
                    unsigned m = bad;
                    for (unsigned any = __ballot_sync(0xffffffffu, m != 0); any;
                         any = __ballot_sync(0xffffffffu, m != 0)) {
                        const int k = wn + __popc(any & ((1u << lane) - 1u));
                        if (m && k < kWarpHoles) hl[warp * kWarpHoles + k] = (uint16_t)((sy << 7) | (c0 + __ffs(m) - 1));
                        m &= m - 1;
                        wn += __popc(any);
                    }
                }
            }
        }
    } else {
        for (int sy = b.iy0 + warp; sy < b.iy1; sy += kWarps) {
            const float* row = in + (size_t)(y0 + sy) * W + x0;
#pragma unroll
            for (int k = 0; k < kSW / 32; ++k) {
                const int sx = k * 32 + lane;
                if (sx >= b.ix0 && sx < b.ix1) {
                    const float v = __ldg(row + sx);
                    all_valid &= fast_depth(v);
                    buf0[sy * kSW + sx] = v;
                }
            }
        }
    }
    if constexpr (FIX) {
        // (the row-load path keeps no lists: its hole tiles take the checked walk)
        if (!use_tma) wn = __any_sync(0xffffffffu, !all_valid) ? kWarpHoles + 1 : 0;
        if (lane == 0 && !(flag_mode == 2 && list_mode == 2)) s_wn[warp] = wn;
    }
    all_valid = __syncthreads_and(all_valid);
    if (flag_mode == 1 && !all_valid && threadIdx.x == 0) {
        atomicOr(frame_flags + frame, 1);
        if (p.hole_note) *(volatile unsigned*)p.hole_note = p.call_id;
    }
    // tiles with a few holes: the unchecked walk everywhere, then the cells
    // whose stencil touches a listed cell (the cell itself and its 4
    // neighbours) recomputed with the checked cell -- every other cell's
    // unchecked result is the checked one (all five operands fast_depth)
    int pre[kWarps + 1] = {};                  // prefix of the per-warp counts
    int wmax = 0;
    if (FIX && (!all_valid || (flag_mode == 2 && list_mode == 2))) {
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const int c = s_wn[w];
            pre[w + 1] = pre[w] + c;
            wmax = max(wmax, c);
        }
    }
    const int nh = pre[kWarps];
    if (FIX && flag_mode == 2 && list_mode == 2) all_valid = nh == 0;
    else if (FIX && list_mode == 1 && threadIdx.x <= (all_valid ? 0 : kListVecs)) {   // keep them for the later passes
        uint4 v;
        if (threadIdx.x == 0) {
            uint32_t c[4];
#pragma unroll
            for (int j = 0; j < 4; ++j)
                c[j] = (uint32_t)min(s_wn[2 * j], 0xFFFF) | ((uint32_t)min(s_wn[2 * j + 1], 0xFFFF) << 16);
            v = make_uint4(c[0], c[1], c[2], c[3]);
        } else {
            v = reinterpret_cast<const uint4*>(hl)[threadIdx.x - 1];
        }
        tile_lists[tile_index() * (kListVecs + 1) + threadIdx.x] = v;
    }
    // the unchecked sweeps only where no update can turn a pixel invalid
    const bool fast = all_valid && !p.keep_valid;
    const bool fixup = FIX && !all_valid && !p.keep_valid && nh <= kHoleCap && wmax <= kWarpHoles;
    // this thread's stencil cells (items k = tid + 256 r of the 5 * nh: a
    // listed cell and its 4 neighbours) as smem indices (sy << 7 | sx), -1 =
    // none; fixed for the pass (holes never move)
    int item[kFixItems];
#pragma unroll
    for (int r = 0; r < kFixItems; ++r) {
        item[r] = -1;
        const int k = threadIdx.x + r * kThreads;
        if (fixup && k < 5 * nh) {
            const int h = k / 5;
            const int d = k - 5 * h;
            int slot = h;                              // the h-th hole of the flattened lists
#pragma unroll
            for (int w = 1; w < kWarps; ++w)
                if (h >= pre[w]) slot = h - pre[w] + w * kWarpHoles;
            PM_CHECK(slot >= 0 && slot < kWarps * kWarpHoles);
            const int e = hl[slot];
            item[r] = e + (d == 1 ? -kSW : d == 2 ? kSW : d == 3 ? -1 : d == 4 ? 1 : 0);
            if ((d == 3 && (e & 127) == 0) || (d == 4 && (e & 127) == kSW - 1)) item[r] = -1;
        }
    }

    const bool pairs = ((b.ix0 | b.ix1) & 1) == 0;

    PM_ATS(t1);
    float* cur = buf0;
    float* nxt = buf1;
    // Interior, hole-free tiles (the loaded region lies inside the image: ~55 %
    // of a 640x480 frame's tiles): the sweep geometry is a compile-time
    // constant -- sweeps unrolled, Box literal -- so the per-warp-sweep setup
    // (row split, clipping, border offsets) folds to a few instructions.  Same
    // cells, same operands, same order: bitwise the generic loop's result.
    // after sweep t's walk: the checked cell (border rule of the walks: an
    // out-of-image neighbour is the centre) at this thread's stencil cells in
    // the sweep region
    auto fix = [&](int t) {
        __syncthreads();                              // the walk's stores first
        const int ylo = max(t, b.iy0), yhi = min(SH - t, b.iy1);
        const int xlo = max(PAD + t, b.ix0), xhi = min(kSW - PAD - t, b.ix1);
#pragma unroll
        for (int r = 0; r < kFixItems; ++r) {
            const int e = item[r];
            const int sy = e >> 7, sx = e & 127;
            if (e < 0 || sy < ylo || sy >= yhi || sx < xlo || sx >= xhi) continue;
            PM_CHECK(e - kSW >= 0 && e + kSW < kSW * SH && sx >= 1 && sx + 1 < kSW);
            const float* c = cur + e;
            const float C = c[0];
            const float N = sy == b.iy0 ? C : c[-kSW];
            const float S = sy == b.iy1 - 1 ? C : c[kSW];
            const float Wv = sx == b.ix0 ? C : c[-1];
            const float E = sx == b.ix1 - 1 ? C : c[1];
            nxt[e] = cell<true, DIV>(C, N, S, Wv, E, p);
        }
    };
    bool done = false;
    if constexpr (R <= 6) {
        if ((fast || fixup) && b.ix0 == 0 && b.ix1 == kSW && b.iy0 == 0 && b.iy1 == SH) {
            constexpr Box kIn{0, kSW, 0, SH};
#pragma unroll
            for (int t = 1; t <= R; ++t) {
                if (t > iters) break;
                sweep_pairs<SH, PAD, false, DIV>(cur, nxt, t, kIn, p);
                if (FIX && fixup) fix(t);
                __syncthreads();
                float* tmp = cur; cur = nxt; nxt = tmp;
            }
            done = true;
        }
    }
    // generic tiles: one sweep loop per variant (the variant test outside the
    // loop lets the sweep-invariant column setup be hoisted out of it)
    auto sweeps = [&](auto FN) {
        for (int t = 1; t <= iters; ++t) {
            FN(t);
            __syncthreads();
            float* tmp = cur; cur = nxt; nxt = tmp;
        }
    };
    if (!done) {
        // (the fix-up tiles share the unchecked walk's code: one copy of each walk)
#define PM_SWEEPS(FN, CK) sweeps([&](int t) { FN<SH, PAD, CK, DIV>(cur, nxt, t, b, p); if (FIX && !CK && fixup) fix(t); })
        if constexpr (FIX) {
            if (pairs) { if (fast || fixup) PM_SWEEPS(sweep_pairs, false); else PM_SWEEPS(sweep_pairs, true); }
            else { if (fast || fixup) PM_SWEEPS(sweep, false); else PM_SWEEPS(sweep, true); }
        } else {
            if (pairs) { if (fast) PM_SWEEPS(sweep_pairs, false); else PM_SWEEPS(sweep_pairs, true); }
            else { if (fast) PM_SWEEPS(sweep, false); else PM_SWEEPS(sweep, true); }
        }
#undef PM_SWEEPS
    }

    PM_ATS(t2);
    [[maybe_unused]] const int pk_ = normals ? 4 : 0;
    PM_AACC(pk_ + 0, t0, t1);
    PM_AACC(pk_ + 1, t1, t2);
    // write the tile (and its normals).  Rows of float4 quads when W % 4 == 0
    // (the tile origin is then 16-byte aligned in global and shared memory).
    const int ox = blockIdx.x * TW, oy = blockIdx.y * kTH;
    float* out = dst ? dst + frame * HW : nullptr;
    float* nrm = normals ? normals + frame * 3 * HW : nullptr;
#ifndef PM_ADF_QUAD_STORES
    // plain passes: each output row leaves shared memory as one bulk copy
    // (cp.async.bulk), issued by one thread per row -- the tile's stores
    // cost 44 instructions instead of a load / store pair per float4
    if (!nrm && out && (W & 3) == 0 && ((uintptr_t)out & 15) == 0) {
        const int y = threadIdx.x, gy = oy + y;
        if (y < kTH && gy < H) {
            const int w = min(TW, W - ox);
            PM_CHECK(w > 0 && ox + w <= W && y + R < SH && RA + w <= kSW && ((w * 4) & 15) == 0);
            fence_proxy_async_smem();             // the last sweep's stores, before the async proxy reads
            bulk_store_s2g(out + (size_t)gy * W + ox, cur + (y + R) * kSW + RA, (uint32_t)(sizeof(float) * w));
            bulk_commit();
            bulk_wait_read();
        }
        PM_ATS(t3);
        PM_AACC(pk_ + 2, t2, t3);
        return;
    }
#endif
    if ((W & 3) == 0) {
        constexpr int QW = TW / 4;
        // CK: window validity checks (tiles with holes); NMC: normals mode
        auto quads = [&](auto CK, auto NMC) {
        for (int y = warp; y < kTH; y += kWarps) {
            const int gy = oy + y;
            if (gy >= H) break;
            const int q = lane;
            const int gx = ox + 4 * q;
            if (q >= QW || gx >= W) continue;
            const int sx = RA + 4 * q, sy = y + R;
            const size_t o = (size_t)gy * W + gx;
            const float4 c = *reinterpret_cast<const float4*>(cur + sy * kSW + sx);
            if (out) *reinterpret_cast<float4*>(out + o) = c;
            if (nrm) {
                // clamp-to-edge 3x6 window: rows ym, sy, yp; columns gx-1 .. gx+4
                const int rows[3] = {max(gy - 1, 0) - y0, sy, min(gy + 1, H - 1) - y0};
                float z[3][6];
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    const float* rp = cur + rows[a] * kSW + sx;
                    const float4 m = *reinterpret_cast<const float4*>(rp);
                    z[a][1] = m.x; z[a][2] = m.y; z[a][3] = m.z; z[a][4] = m.w;
                    z[a][0] = gx == 0 ? m.x : rp[-1];
                    z[a][5] = gx + 4 >= W ? m.w : rp[4];
                }
                float4 nx, ny, nz;
                float* px = &nx.x; float* py = &ny.x; float* pz = &nz.x;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float w3[3][3] = {{z[0][j], z[0][j + 1], z[0][j + 2]},
                                            {z[1][j], z[1][j + 1], z[1][j + 2]},
                                            {z[2][j], z[2][j + 1], z[2][j + 2]}};
                    const float3 n = sobel_normal<decltype(CK)::value, decltype(NMC)::value>(
                        w3, (float)(gx + j), (float)gy, p);
                    px[j] = n.x; py[j] = n.y; pz[j] = n.z;
                }
                *reinterpret_cast<float4*>(nrm + o) = nx;
                *reinterpret_cast<float4*>(nrm + HW + o) = ny;
                *reinterpret_cast<float4*>(nrm + 2 * HW + o) = nz;
            }
        }
        };
        using T_ = std::true_type;
        using F_ = std::false_type;
        using GEO = std::integral_constant<int, PM_NORMALS_GEOMETRIC>;
        using PRN = std::integral_constant<int, PM_NORMALS_AS_PRINTED>;
        // hole-free tile: every window is valid -- no filtered pixel turns
        // invalid for lambda <= kNoCheckMaxLambda (fast_depth); at lambda ~ 1/4
        // a pixel can round to 0 (c = 1 next to much smaller neighbours), so
        // the windows are checked
        const bool nocheck = all_valid && (iters == 0 || p.lam <= kNoCheckMaxLambda);
        if (!nrm) quads(F_{}, GEO{});
        else if (p.nmode == PM_NORMALS_AS_PRINTED) { if (nocheck) quads(F_{}, PRN{}); else quads(T_{}, PRN{}); }
        else { if (nocheck) quads(F_{}, GEO{}); else quads(T_{}, GEO{}); }
        PM_ATS(t3);
        PM_AACC(pk_ + 2, t2, t3);
        return;
    }
    for (int y = warp; y < kTH; y += kWarps) {
        const int gy = oy + y;
        if (gy >= H) break;
        for (int x = lane; x < TW; x += 32) {
            const int gx = ox + x;
            if (gx >= W) break;
            const int sx = x + RA, sy = y + R;
            if (out) out[(size_t)gy * W + gx] = cur[sy * kSW + sx];
            if (nrm) {
                // clamp-to-edge window in image coords, mapped to smem coords
                const int xm = max(gx - 1, 0) - x0, xp = min(gx + 1, W - 1) - x0;
                const int ym = max(gy - 1, 0) - y0, yp = min(gy + 1, H - 1) - y0;
                const int xs[3] = {xm, sx, xp}, ys[3] = {ym, sy, yp};
                float z[3][3];
#pragma unroll
                for (int a = 0; a < 3; ++a)
#pragma unroll
                    for (int c = 0; c < 3; ++c) z[a][c] = cur[ys[a] * kSW + xs[c]];
                const float3 n = sobel_normal(z, (float)gx, (float)gy, p);
                const size_t o = (size_t)gy * W + gx;
                nrm[o] = n.x;
                nrm[HW + o] = n.y;
                nrm[2 * HW + o] = n.z;
            }
        }
    }
}

using PassFn = void (*)(const float*, float*, float*, int, int, int, AdfParams, const CUtensorMap, int, int*, int,
                        uint4*, int);

template <int R>
struct PassTable {
    static void fill(PassFn (*fns)[2][2], size_t* smem, int* tw) {
        fns[R][0][0] = adf_pass_kernel<R, false, false>;
        fns[R][1][0] = adf_pass_kernel<R, true, false>;
        fns[R][0][1] = adf_pass_kernel<R, false, true>;
        fns[R][1][1] = adf_pass_kernel<R, true, true>;
        smem[R] = pass_smem_bytes<R>();
        tw[R] = tile_w<R>();
        PassTable<R - 1>::fill(fns, smem, tw);
    }
};
template <>
struct PassTable<0> {
    static void fill(PassFn (*)[2][2], size_t*, int*) {}
};

struct Passes {
    PassFn fn[kMaxItersPerPass + 2][2][2] = {};   // [R][scheme == PM_ADF_DIVERGENCE][FIX]
    size_t smem[kMaxItersPerPass + 2] = {};
    int tw[kMaxItersPerPass + 2] = {};
    Passes() { PassTable<kMaxItersPerPass + 1>::fill(fn, smem, tw); }
};
const Passes& passes() {
    static const Passes p;
    return p;
}

}  // namespace

cudaError_t adf_setup_attributes() {
    const Passes& P = passes();
    for (int R = 1; R <= kMaxItersPerPass + 1; ++R)
        for (int d = 0; d < 2; ++d)
            for (int f = 0; f < 2; ++f) {
                cudaError_t e = cudaFuncSetAttribute(P.fn[R][d][f], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     (int)P.smem[R]);
                if (e != cudaSuccess) return e;
            }
    return cudaSuccess;
}

static cudaError_t launch_pass(const float* src, float* dst, float* normals, int W, int H, int B,
                               int iters, bool fuse, const AdfParams& p, cudaStream_t stream,
                               int* frame_flags = nullptr, int flag_mode = 0, uint4* tile_lists = nullptr,
                               int list_mode = 0, bool fix = false) {
    const int R = iters + (fuse ? 1 : 0);
    const Passes& P = passes();
    const int TW = P.tw[R];
    dim3 grid((W + TW - 1) / TW, (H + kTH - 1) / kTH, B);
    CUtensorMap tmap;
    int use_tma = make_tmap_f32_3d(&tmap, src, W, H, B, kSW, kTH + 2 * R) ? 1 : 0;
    if (!use_tma) memset(&tmap, 0, sizeof(tmap));
    void* args[] = {(void*)&src,  (void*)&dst,  (void*)&normals, (void*)&W,           (void*)&H,
                    (void*)&iters, (void*)&p,   (void*)&tmap,    (void*)&use_tma,     (void*)&frame_flags,
                    (void*)&flag_mode, (void*)&tile_lists, (void*)&list_mode};
    return cudaLaunchKernel((const void*)P.fn[R][p.scheme == PM_ADF_DIVERGENCE ? 1 : 0][fix ? 1 : 0], grid,
                            dim3(kThreads), args, P.smem[R], stream);
}

int adf_default_iters_per_pass() { return 4; }

size_t adf_flags_offset(int W, int H, int B) { return (sizeof(float) * (size_t)B * W * H + 255) & ~(size_t)255; }

// the hole-list records after the flags: one per tile of the narrowest
// plain-pass tiling (tile_w<kMaxItersPerPass>() = 96 columns)
static size_t adf_lists_offset(int B) { return ((sizeof(int) * (size_t)B + 255) & ~(size_t)255); }
size_t adf_flags_region_bytes(int W, int H, int B) {
    const size_t tiles = (size_t)((W + tile_w<kMaxItersPerPass>() - 1) / tile_w<kMaxItersPerPass>()) *
                         ((H + kTH - 1) / kTH) * B;
    return (adf_lists_offset(B) + tiles * (kListVecs + 1) * sizeof(uint4) + 255) & ~(size_t)255;
}

static AdfParams make_params(const pm_intrinsics* K, float lam, float kappa, int scheme, int nmode) {
    AdfParams p;
    p.kc = (float)(-1.4426950408889634 / (4.0 * (double)kappa * (double)kappa));
    p.l2lam = (float)log2((double)lam);
    p.kd = (float)(-1.4426950408889634 / ((double)kappa * (double)kappa));
    p.lam = lam;
    p.negz = -0.0f;
    p.fx = K ? K->fx : 1.f;
    p.fy = K ? K->fy : 1.f;
    p.cx = K ? K->cx : 0.f;
    p.cy = K ? K->cy : 0.f;
    p.ifx = 1.0f / p.fx;
    p.ify = 1.0f / p.fy;
    p.scheme = scheme;
    p.nmode = nmode;
    p.keep_valid = lam > kNoCheckMaxLambda ? 1 : 0;
    p.hole_note = nullptr;
    p.call_id = 0;
    return p;
}

// AUTO engine choice: the hole engine (FIX kernels) while a recent call on
// this device saw an invalid pixel, the lean tiled kernels otherwise.  The
// first pass of a multi-pass call stores the call's id into a mapped host
// word when one of its tiles holds an invalid pixel (the frame-flag branch);
// the host reads it when the next call is made -- no copy, no stream
// operation.  Results do not depend on the choice (the engines are bitwise
// equal); only the speed on frames with dropout does.
namespace {
constexpr unsigned kHoleMemory = 16;   // calls a hole observation keeps AUTO on the hole engine
struct HoleNote {
    std::once_flag once;
    unsigned* host = nullptr;          // mapped pinned word (host view)
    unsigned* dev = nullptr;           // its device view
    std::atomic<unsigned> calls{0};
};
HoleNote g_hole_note[64];
HoleNote* hole_note(cudaStream_t stream) {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= 64) return nullptr;
    HoleNote& n = g_hole_note[d];
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
        (void)cudaGetLastError();
        return n.host ? &n : nullptr;  // (no allocation inside a graph capture)
    }
    std::call_once(n.once, [&] {
        unsigned* h = nullptr;
        unsigned* dp = nullptr;
        if (cudaHostAlloc(&h, sizeof(unsigned), cudaHostAllocMapped) != cudaSuccess) {
            (void)cudaGetLastError();
            return;
        }
        *h = 0;
        if (cudaHostGetDevicePointer(&dp, h, 0) != cudaSuccess) {
            (void)cudaGetLastError();
            cudaFreeHost(h);
            return;
        }
        n.dev = dp;
        n.host = h;
    });
    return n.host ? &n : nullptr;
}
}  // namespace

cudaError_t adf_run(const float* in, float* out, float* normals, float* ws, int W, int H, int B,
                    const pm_intrinsics* K, float lam, float kappa, int iters, int iters_per_pass,
                    int scheme, int nmode, int engine, cudaStream_t stream) {
    AdfParams p = make_params(K, lam, kappa, scheme, nmode);
    int T = iters_per_pass > 0 ? iters_per_pass : adf_default_iters_per_pass();
    if (T > kMaxItersPerPass) T = kMaxItersPerPass;
    if (iters == 0) {   // N = 0: I_smooth = I (Alg. 1 ℓ1); normals of the input
        if (!normals)
            return cudaMemcpyAsync(out, in, sizeof(float) * (size_t)B * W * H, cudaMemcpyDeviceToDevice, stream);
        if (engine == PM_ADF_ENGINE_REG) {
            bool launched = false;
            cudaError_t e = adf_reg_pass(in, out, normals, W, H, B, 0, p, stream, nullptr, 0, &launched);
            if (e != cudaSuccess || launched) return e;
        }
        return launch_pass(in, out, normals, W, H, B, 0, true, p, stream);
    }
    const int passes = (iters + T - 1) / T;
    // per-frame "has an invalid pixel" flags after the ping-pong buffer
    int* flags = passes > 1 ? reinterpret_cast<int*>(reinterpret_cast<char*>(ws) + adf_flags_offset(W, H, B))
                            : nullptr;
    if (flags) {
        cudaError_t e = cudaMemsetAsync(flags, 0, sizeof(int) * (size_t)B, stream);
        if (e != cudaSuccess) return e;
    }
    const float* src = in;
    int done = 0;
    // the register engine is opt-in: measured slower than the tiled engine on B200
    const bool try_reg = engine == PM_ADF_ENGINE_REG;
    bool fix = engine == PM_ADF_ENGINE_HOLES;         // the tiled engine with the fix-up walk
    if (flags && (engine == PM_ADF_ENGINE_AUTO || engine == PM_ADF_ENGINE_HOLES)) {
        if (HoleNote* n = hole_note(stream)) {
            const unsigned id = n->calls.fetch_add(1) + 1u;
            const unsigned seen = *(volatile unsigned*)n->host;
            if (engine == PM_ADF_ENGINE_AUTO && seen != 0 && id - seen <= kHoleMemory) fix = true;
            p.hole_note = n->dev;
            p.call_id = id;
        }
    }
    bool lists_written = false;   // by a tiled first pass
    for (int k = 0; k < passes; ++k) {
        const int it = (iters - done) / (passes - k);   // near-equal split, sums to iters
        float* dst = (((passes - 1 - k) & 1) == 0) ? out : ws;   // the last pass lands in `out`
        const bool last = k == passes - 1;
        const int mode = flags ? (k == 0 ? 1 : 2) : 0;
        // hole lists: written by the first pass, read by the later plain
        // passes that use its tile geometry (same sweep count, not fused)
        const int it0 = iters / passes;
        const bool fused = last && normals != nullptr;
        int lmode = !flags || !fix ? 0 : k == 0 ? (fused ? 0 : 1) : (!fused && it == it0 && lists_written ? 2 : 0);
#ifdef PM_ADF_EXP_NOLISTS
        lmode = 0;
#endif
        uint4* lists = flags ? reinterpret_cast<uint4*>(reinterpret_cast<char*>(flags) + adf_lists_offset(B)) : nullptr;
        bool launched = false;
        if (try_reg) {
            cudaError_t e = adf_reg_pass(src, dst, last ? normals : nullptr, W, H, B, it, p, stream, flags, mode,
                                         &launched);
            if (e != cudaSuccess) return e;
        }
        if (!launched) {
            cudaError_t e = launch_pass(src, dst, last ? normals : nullptr, W, H, B, it, fused, p, stream, flags,
                                        mode, lists, lmode, fix);
            if (e != cudaSuccess) return e;
            if (lmode == 1) lists_written = true;
        }
        src = dst;
        done += it;
    }
    return cudaSuccess;
}

cudaError_t normals_run(const float* depth, float* normals, int W, int H, int B,
                        const pm_intrinsics* K, int nmode, cudaStream_t stream) {
    const AdfParams p = make_params(K, 0.25f, 1.0f, PM_ADF_ALG1, nmode);
    return launch_pass(depth, nullptr, normals, W, H, B, 0, true, p, stream);
}

#ifdef PM_ADF_TIMING
extern "C" __attribute__((visibility("default"))) int pm_debug_adf_prof(unsigned long long* out, int reset) {
    if (cudaMemcpyFromSymbol(out, pm::g_adf_prof, sizeof(unsigned long long) * 8) != cudaSuccess) return 1;
    if (reset) {
        unsigned long long z[8] = {};
        cudaMemcpyToSymbol(pm::g_adf_prof, z, sizeof(z));
    }
    return 0;
}
#endif
}  // namespace pm
