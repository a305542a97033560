// hs_tiles.cu -- tile-major binning on sm_100a (the training path's binner).
//
// The per-(frame, tile) lists the reference order implies (S/render.py:221-223:
// a stable depth argsort per frame, then the splats covering each tile in that
// order) are built tile-first instead of by a global key sort:
//
//   counts         every (frame, splat) adds one to each tile of its pixel bbox -- in
//                  the projection kernel (hs_project_avatar_fwd's tile_counts, which
//                  also packs each item's tile rectangle) or hs_tile_count
//   hs_tile_scan   exclusive scan of the counts -> ranges + scatter cursors (1,024 lists
//                  per CTA, decoupled look-back), the lists longer than kWarpShort, and
//                  the step's single device->host summary (key total, error word, depth
//                  range, longest list)
//   hs_tile_fill   scatter (per-CTA slot blocks, arrival order inside a list), then each
//                  list sorted on chip by (depth bits, Gaussian index): warps sort lists
//                  up to kWarpShort entries in registers (32-bit keys: depth offset |
//                  slot, ties settled on the full keys), CTAs sort lists up to kWarpCap
//                  (register runs merged by rank) -- concurrently on two streams -- and
//                  up to kCtaCap (shared-memory bitonic); lists the 32-bit path cannot
//                  settle are sorted on their full 64-bit keys in shared memory
//
// Sorting each list by (depth bits, index) is exactly the reference's order: positive
// float depths compare like their bit patterns and the stable argsort breaks ties by
// the lower index (oracle/binning.py).  Lists longer than kCtaCap are left to the
// caller, which sees the longest length in the summary and falls back to the global
// two-level sort (hs_depth_order + hs_bin_emit_sorted + hs_sort_pairs32) for that step.
#include <algorithm>

#include "hs_common.cuh"

namespace hs {

#ifndef HS_WARP_SHORT
#define HS_WARP_SHORT 256
#endif
constexpr int kWarpShort = HS_WARP_SHORT;   // longest list one warp sorts (in registers)
constexpr int kWarpCap = 1024;        // longest list one CTA sorts as merged register runs
constexpr int kCtaCap = 8192;         // longest list one CTA sorts in shared memory
constexpr int kCtaSortThreads = 512;
constexpr int kWarpSortWarps = 4;     // warps per CTA of the warp-level sort

// list_counts = [the half the next scan uses | half 0 | half 1], halves of `half` words:
// [1] / [2] the CTA-sorted list counts, [5] scan ticket, [6] scan done, [7] longest,
// [8 + t] scan CTA t's flagged total.  A scan works in its half and zeroes the other one
// (the previous step's, whose fill has finished) for the next, so no memset is needed.
__device__ __forceinline__ uint32_t *counts_half(uint32_t *list_counts, int half, uint32_t p) {
    return list_counts + 1 + (size_t)p * half;
}
__device__ __forceinline__ const uint32_t *filled_half(const uint32_t *list_counts, int half) {
    return list_counts + 1 + (size_t)(1u - list_counts[0]) * half;   // the scan flipped [0]
}

// ------------------------------------------------------------------- count

// A CTA covers kTileItems consecutive (frame, Gaussian) items -- neighbours on the
// UV grid, so they hit few, shared tiles.  Items of the CTA's first frame count
// into a shared-memory histogram over that frame's tiles (flushed with one global
// atomic per touched tile); items past a frame boundary, or every item when the
// frame has too many tiles for shared memory, add to the global counters directly.
#ifndef HS_TILE_ITEMS
#define HS_TILE_ITEMS 512
#endif
constexpr int kTileItems = HS_TILE_ITEMS;
constexpr int kTileThreads = 256;
constexpr int kTileSmemBins = 12288;   // tiles per frame the shared histogram holds (48 KB)

struct TileBox {
    int ty0, ty1, tx0, tx1;
};


// The CTA's items, kPer per thread (item k = threadIdx.x + j * kTileThreads), loaded
// up front so the loads overlap: count, pixel bbox, frame.
constexpr int kPer = kTileItems / kTileThreads;

struct CtaItems {
    uint32_t rows[kPer], cols[kPer], n[kPer], b[kPer], mask[kPer];
    bool live[kPer];
};

// rects (optional, hs_project_avatar_fwd's tile_rects): per item the tile rectangle packed
// ty0 | ty1 << 8 | tx0 << 16 | tx1 << 24 (dead items: ty0 > ty1) and its kept-tile mask
// (hs_common.cuh:mask_keeps) -- 8 coalesced bytes instead of the count and two words of
// the 48-byte record
__device__ __forceinline__ void load_items(CtaItems &it, int64_t items, int64_t N, const float *__restrict__ records,
                                           const uint32_t *__restrict__ counts, const uint32_t *__restrict__ rects) {
    const int64_t i0 = blockIdx.x * (int64_t)kTileItems;
    const int64_t b0 = i0 / N;
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        const int64_t i = i0 + threadIdx.x + j * kTileThreads;
        const bool in = i < items;
        it.mask[j] = 0xFFFFFFFFu;
        if (rects) {
            const uint2 rm = in ? reinterpret_cast<const uint2 *>(rects)[i] : make_uint2(0x00010001u, 0u);
            it.rows[j] = rm.x;
            it.mask[j] = rm.y;
            it.live[j] = (rm.x & 0xFFu) <= ((rm.x >> 8) & 0xFFu);
        } else {
            it.live[j] = in && counts[i] != 0u;
            it.rows[j] = in ? __float_as_uint(records[i * kRec + 7]) : 0u;
            it.cols[j] = in ? __float_as_uint(records[i * kRec + 8]) : 0u;
        }
        int64_t b = b0, n = i - b0 * N;
        if (n >= N) {                            // past the CTA's first frame (rare)
            b = item_frame(i, N);
            n = i - b * N;
        }
        it.b[j] = (uint32_t)b;
        it.n[j] = (uint32_t)n;
    }
}

__device__ __forceinline__ TileBox item_box(const CtaItems &it, int j, bool packed) {
    if (packed) {
        const uint32_t r = it.rows[j];
        return {(int)(r & 0xFFu), (int)((r >> 8) & 0xFFu), (int)((r >> 16) & 0xFFu), (int)(r >> 24)};
    }
    return {unpack_lo(it.rows[j]) / kTile, unpack_hi(it.rows[j]) / kTile, unpack_lo(it.cols[j]) / kTile,
            unpack_hi(it.cols[j]) / kTile};
}

__global__ void __launch_bounds__(kTileThreads) tile_count_kernel(int64_t items, int64_t N, int tiles_x, int tiles,
                                                                  int tile_bits, const float *__restrict__ records,
                                                                  const uint32_t *__restrict__ counts,
                                                                  uint32_t *__restrict__ tile_counts) {
    pdl_prologue();
    extern __shared__ uint32_t hist[];
    const uint32_t b0 = (uint32_t)(blockIdx.x * (int64_t)kTileItems / N);
    const bool shared = tiles <= kTileSmemBins;
    CtaItems it;
    load_items(it, items, N, records, counts, nullptr);
    if (shared)
        for (int t = threadIdx.x; t < tiles; t += kTileThreads) hist[t] = 0u;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        if (!it.live[j]) continue;
        const TileBox bx = item_box(it, j, false);
        uint32_t *dst = (shared && it.b[j] == b0) ? hist : tile_counts + ((size_t)it.b[j] << tile_bits);
        for (int ty = bx.ty0; ty <= bx.ty1; ++ty)
            for (int tx = bx.tx0; tx <= bx.tx1; ++tx) atomicAdd(dst + ty * tiles_x + tx, 1u);
    }
    if (!shared) return;
    __syncthreads();
    uint32_t *row = tile_counts + ((size_t)b0 << tile_bits);
    for (int t = threadIdx.x; t < tiles; t += kTileThreads) {
        const uint32_t c = hist[t];
        if (c) atomicAdd(row + t, c);
    }
}

// -------------------------------------------------------------------- scan

// One CTA: the exclusive scan of the per-(frame, tile) counts -> ranges, scatter
// cursors, the key total and the longest list; resets the fill's counters.  (The list
// sorts stride over all segments and pick their length class themselves.)
constexpr int kScanThreads = 1024;
constexpr int kScanPer = 16;          // segments per thread and round: tid + k * kScanThreads

__global__ void __launch_bounds__(kScanThreads) tile_scan_kernel(int nseg, uint32_t *__restrict__ tile_counts,
                                                                 uint32_t *__restrict__ ranges,
                                                                 uint32_t *__restrict__ cursor,
                                                                 uint32_t *__restrict__ lists,
                                                                 uint32_t *__restrict__ list_counts, int half,
                                                                 unsigned long long *__restrict__ err,
                                                                 uint32_t *__restrict__ depth_range,
                                                                 unsigned long long *__restrict__ summary) {
    pdl_prologue();
    __shared__ uint32_t wt[kScanPer][kScanThreads / 32];   // per k: inclusive scan over warps
    __shared__ uint32_t s_max, s_big[2];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (tid == 0) s_max = s_big[0] = s_big[1] = 0u;
    __syncthreads();
    uint32_t carry = 0, mx = 0;
    for (int base = 0; base < nseg; base += kScanThreads * kScanPer) {
        uint32_t c[kScanPer], incl[kScanPer];
#pragma unroll
        for (int k = 0; k < kScanPer; ++k) {
            const int i = base + k * kScanThreads + tid;
            c[k] = i < nseg ? tile_counts[i] : 0u;
        }
#pragma unroll
        for (int k = 0; k < kScanPer; ++k) {
            mx = max(mx, c[k]);
            uint32_t v = c[k];
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += t;
            }
            incl[k] = v;
            if (lane == 31) wt[k][w] = v;
        }
        __syncthreads();
        if (w < kScanPer) {
            uint32_t v = wt[w][lane];
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += t;
            }
            wt[w][lane] = v;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kScanPer; ++k) {
            const int i = base + k * kScanThreads + tid;
            const uint32_t run = carry + (w > 0 ? wt[k][w - 1] : 0u) + incl[k] - c[k];
            carry += wt[k][kScanThreads / 32 - 1];
            if (i < nseg) {
                // empty lists: (0, 0), as the sorts leave them
                reinterpret_cast<uint2 *>(ranges)[i] = c[k] ? make_uint2(run, run + c[k]) : make_uint2(0u, 0u);
                cursor[i] = run;
                if (c[k]) tile_counts[i] = 0u;       // ready for the next step's count
            }
            // the CTA-sorted lists, one shared atomic per warp: kWarpShort+1..kWarpCap
            // entries from the front of lists, kWarpCap+1..kCtaCap from the back
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const bool big = q == 0 ? c[k] > (uint32_t)kWarpShort && c[k] <= (uint32_t)kWarpCap
                                        : c[k] > (uint32_t)kWarpCap && c[k] <= (uint32_t)kCtaCap;
                const uint32_t m = __ballot_sync(0xffffffffu, big);
                if (m) {
                    const int leader = __ffs(m) - 1;
                    uint32_t first = 0;
                    if (lane == leader) first = atomicAdd(&s_big[q], (uint32_t)__popc(m));
                    first = __shfl_sync(0xffffffffu, first, leader);
                    const uint32_t r = first + __popc(m & ((1u << lane) - 1u));
                    if (big) lists[q == 0 ? r : nseg - 1 - r] = (uint32_t)i;
                }
            }
        }
        __syncthreads();   // wt is rewritten by the next round
    }
    for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) atomicMax(&s_max, mx);
    __syncthreads();
    // [1] / [2]: the long / longer lists, in this step's half; the other half zeroed
    const uint32_t p = list_counts[0];
    __syncthreads();
    uint32_t *lc = counts_half(list_counts, half, p), *other = counts_half(list_counts, half, 1u - p);
    if (tid == 1) lc[1] = s_big[0];
    if (tid == 2) lc[2] = s_big[1];
    for (int k = tid; k < half; k += blockDim.x) other[k] = 0u;
    __syncthreads();
    if (tid == 0) {
        list_counts[0] = 1u - p;
        summary[0] = carry;
        summary[1] = err ? *err : HS_NO_ERROR;
        if (err) *err = HS_NO_ERROR;                 // read once per step: reset for the next
        summary[2] = depth_range ? ((unsigned long long)depth_range[1] << 32) | depth_range[0] : 0xFFFFFFFFull;
        summary[3] = s_max;
        if (depth_range && s_max <= (uint32_t)kCtaCap) {   // (a fallback step still needs it)
            depth_range[0] = 0xFFFFFFFFu;
            depth_range[1] = 0u;
        }
    }
}

// Many-CTA variant (the training path's): CTA t (a ticket, so predecessors are
// resident first) scans kScanSpan consecutive segments, publishes its total, adds the
// totals of all CTAs before it (decoupled look-back on aggregates only) and writes its
// ranges; list appends and the longest list go through global atomics, and the last
// CTA to finish writes the summary.  list_counts alternates between two halves of
// `half` words (word 0 selects the half being filled; counts_half): in the half of
// this step [1] / [2] count the long / longer lists, [5] is the CTA ticket, [6] the
// done count, [7] the longest list and [8 + t] CTA t's flagged total; the last CTA
// zeroes the other half for the next step, so no host-side reset is needed.
constexpr int kScanSpan = 1024;
constexpr uint32_t kAggFlag = 1u << 31;

__global__ void __launch_bounds__(kScanSpan) tile_scan_multi_kernel(int nseg, uint32_t *__restrict__ tile_counts,
                                                                    uint32_t *__restrict__ ranges,
                                                                    uint32_t *__restrict__ cursor,
                                                                    uint32_t *__restrict__ lists,
                                                                    uint32_t *__restrict__ all_counts, int half,
                                                                    unsigned long long *__restrict__ err,
                                                                    uint32_t *__restrict__ depth_range,
                                                                    unsigned long long *__restrict__ summary) {
    pdl_prologue();
    __shared__ uint32_t wsum[kScanSpan / 32];
    __shared__ uint32_t s_tile, s_prefix;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const uint32_t p = all_counts[0];            // flipped only by the last CTA, after all read it
    uint32_t *list_counts = counts_half(all_counts, half, p);
    if (tid == 0) s_tile = atomicAdd(list_counts + 5, 1u);
    __syncthreads();
    const uint32_t t = s_tile;
    const int i = (int)t * kScanSpan + tid;
    const uint32_t c = i < nseg ? tile_counts[i] : 0u;
    uint32_t incl = c;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) wsum[w] = incl;
    const uint32_t mx = __reduce_max_sync(0xffffffffu, c);
    if (lane == 0 && mx) atomicMax(list_counts + 7, mx);
    __syncthreads();
    if (w == 0) {
        uint32_t v = wsum[lane];
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t x = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += x;
        }
        wsum[lane] = v;                              // inclusive over warps
        if (lane == 31) {
            __threadfence();
            atomicExch(list_counts + 8 + t, kAggFlag | v);
        }
        // the totals of all CTAs before this one, 32 at a time
        uint32_t pre = 0;
        for (int j0 = 0; j0 < (int)t; j0 += 32) {
            const int j = j0 + lane;
            uint32_t st = 0u;
            if (j < (int)t)
                do {
                    st = atomicAdd(list_counts + 8 + j, 0u);
                } while (!(st & kAggFlag));
            pre += st & ~kAggFlag;
        }
        pre = __reduce_add_sync(0xffffffffu, pre);
        if (lane == 0) s_prefix = pre;
    }
    __syncthreads();
    const uint32_t run = s_prefix + (w > 0 ? wsum[w - 1] : 0u) + incl - c;
    if (i < nseg) {
        reinterpret_cast<uint2 *>(ranges)[i] = c ? make_uint2(run, run + c) : make_uint2(0u, 0u);
        cursor[i] = run;
        if (c) tile_counts[i] = 0u;                  // ready for the next step's count
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const bool big = q == 0 ? c > (uint32_t)kWarpShort && c <= (uint32_t)kWarpCap
                                : c > (uint32_t)kWarpCap && c <= (uint32_t)kCtaCap;
        const uint32_t m = __ballot_sync(0xffffffffu, big);
        if (m) {
            const int leader = __ffs(m) - 1;
            uint32_t first = 0;
            if (lane == leader) first = atomicAdd(list_counts + 1 + q, (uint32_t)__popc(m));
            first = __shfl_sync(0xffffffffu, first, leader);
            const uint32_t r = first + __popc(m & ((1u << lane) - 1u));
            if (big) lists[q == 0 ? r : nseg - 1 - r] = (uint32_t)i;
        }
    }
    // the last CTA to finish: the summary (total = the last segment's end)
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        if (atomicAdd(list_counts + 6, 1u) == gridDim.x - 1) {
            __threadfence();
            uint32_t total = 0;
            for (int j = 0; j < (int)gridDim.x; ++j) total += atomicAdd(list_counts + 8 + j, 0u) & ~kAggFlag;
            summary[0] = total;
            summary[1] = err ? *err : HS_NO_ERROR;
            if (err) *err = HS_NO_ERROR;             // read once per step: reset for the next
            summary[2] = depth_range ? ((unsigned long long)depth_range[1] << 32) | depth_range[0] : 0xFFFFFFFFull;
            const uint32_t longest = atomicAdd(list_counts + 7, 0u);
            summary[3] = longest;
            if (depth_range && longest <= (uint32_t)kCtaCap) {   // (a fallback step still needs it)
                depth_range[0] = 0xFFFFFFFFu;
                depth_range[1] = 0u;
            }
            uint32_t *other = counts_half(all_counts, half, 1u - p);
            for (int k = 0; k < half; ++k) other[k] = 0u;
            all_counts[0] = 1u - p;
        }
    }
}

// ----------------------------------------------------------------- scatter

// Same CTA partition as the count: the shared histogram of the CTA's first frame
// reserves one block of slots per touched tile (one global atomic each), then the
// items take slots inside their block with shared atomics.  Slot order inside a list
// is arbitrary; the list sort below fixes it.
__global__ void __launch_bounds__(kTileThreads) tile_scatter_kernel(int64_t items, int64_t N, int tiles_x, int tiles,
                                                                    int tile_bits, const float *__restrict__ records,
                                                                    const uint32_t *__restrict__ counts,
                                                                    const uint32_t *__restrict__ rects,
                                                                    uint32_t *__restrict__ cursor, uint64_t capacity,
                                                                    const unsigned long long *__restrict__ summary,
                                                                    uint32_t *__restrict__ keys,
                                                                    uint32_t *__restrict__ vals) {
    pdl_prologue();
    extern __shared__ uint32_t hist[];
    if (summary[0] > capacity) return;               // the caller grows the buffers and re-runs
    const uint32_t b0 = (uint32_t)(blockIdx.x * (int64_t)kTileItems / N);
    const bool shared = tiles <= kTileSmemBins;
    CtaItems it;
    load_items(it, items, N, records, counts, rects);
    const bool packed = rects != nullptr;
    if (shared) {
        for (int t = threadIdx.x; t < tiles; t += kTileThreads) hist[t] = 0u;
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            if (!it.live[j] || it.b[j] != b0) continue;
            const TileBox bx = item_box(it, j, packed);
            const int area = (bx.ty1 - bx.ty0 + 1) * (bx.tx1 - bx.tx0 + 1);
            int idx = 0;
            for (int ty = bx.ty0; ty <= bx.ty1; ++ty)
                for (int tx = bx.tx0; tx <= bx.tx1; ++tx, ++idx)
                    if (mask_keeps(it.mask[j], area, idx)) atomicAdd(hist + ty * tiles_x + tx, 1u);
        }
        __syncthreads();
        uint32_t *row = cursor + ((size_t)b0 << tile_bits);
        for (int t = threadIdx.x; t < tiles; t += kTileThreads) {
            const uint32_t c = hist[t];
            if (c) hist[t] = atomicAdd(row + t, c);  // the block's first slot
        }
        __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        if (!it.live[j]) continue;
        const TileBox bx = item_box(it, j, packed);
        const bool local = shared && it.b[j] == b0;
        const uint32_t hi = it.b[j] << tile_bits;
        const int area = (bx.ty1 - bx.ty0 + 1) * (bx.tx1 - bx.tx0 + 1);
        int idx = 0;
        for (int ty = bx.ty0; ty <= bx.ty1; ++ty)
            for (int tx = bx.tx0; tx <= bx.tx1; ++tx, ++idx) {
                if (!mask_keeps(it.mask[j], area, idx)) continue;
                const uint32_t t = (uint32_t)(ty * tiles_x + tx);
                const uint32_t pos = local ? atomicAdd(hist + t, 1u) : atomicAdd(cursor + (hi | t), 1u);
                HS_CHECK(pos < capacity, "tile scatter slot", pos);
                if (keys) keys[pos] = hi | t;
                vals[pos] = it.n[j];
            }
    }
}

// Warp-flattened scatter (the training path, packed tile rectangles): a warp takes 32
// consecutive (frame, Gaussian) items, scans their rectangle areas, and then walks the
// resulting (item, tile) keys 32 at a time -- every lane one key, whatever the rectangle
// sizes (the per-item tile loops of tile_scatter_kernel left ~12 of 32 lanes active).
// A key finds its item by a binary search over the scan (shuffles), and lanes holding
// the same (frame, tile) key take consecutive slots behind one global atomic per group
// (__match_any_sync).  Slot order inside a list is arbitrary; the list sorts fix it.
#ifndef HS_SCATTER_MATCH
#define HS_SCATTER_MATCH 1           // lanes with equal (frame, tile) keys share one atomic
#endif
#ifndef HS_SCATTER_WARP_ROUNDS
#define HS_SCATTER_WARP_ROUNDS 1
#endif
constexpr int kSwRounds = HS_SCATTER_WARP_ROUNDS;   // 32-item rounds per warp
__global__ void __launch_bounds__(256) tile_scatter_warp_kernel(int64_t items, int64_t N, int tiles_x, int tile_bits,
                                                                const uint32_t *__restrict__ rects,
                                                                uint32_t *__restrict__ cursor, uint64_t capacity,
                                                                const unsigned long long *__restrict__ summary,
                                                                uint32_t *__restrict__ keys,
                                                                uint32_t *__restrict__ vals) {
    pdl_prologue();
    if (summary[0] > capacity) return;               // the caller grows the buffers and re-runs
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const uint32_t lt_mask = (1u << lane) - 1u;
#pragma unroll 1
    for (int rd = 0; rd < kSwRounds; ++rd) {
        const int64_t i = (warp * kSwRounds + rd) * 32 + lane;
        if ((warp * kSwRounds + rd) * 32 >= items) break;                 // warp-uniform
        const uint2 rm = i < items ? reinterpret_cast<const uint2 *>(rects)[i] : make_uint2(0x00010001u, 0u);
        const uint32_t r = rm.x, msk = rm.y;                              // dead: ty0 > ty1
        const int ty0 = r & 0xFF, ty1 = (r >> 8) & 0xFF, tx0 = (r >> 16) & 0xFF, tx1 = r >> 24;
        const int w = tx1 - tx0 + 1;
        const uint32_t area = ty0 <= ty1 ? (uint32_t)((ty1 - ty0 + 1) * w) : 0u;
        const uint32_t c = area > (uint32_t)kMaskTiles ? area : (uint32_t)__popc(msk);   // kept tiles
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        const uint32_t excl = incl - c, total = __shfl_sync(0xffffffffu, incl, 31);
        const int64_t b = item_frame(i, N);
        const uint32_t n = (uint32_t)(i - b * N), hi = (uint32_t)b << tile_bits;
        for (uint32_t k0 = 0; k0 < total; k0 += 32) {
            const uint32_t k = k0 + lane;
            const bool act = k < total;
            // the item of key k: the largest lane whose exclusive offset is <= k (lanes with
            // no keys share their offset with the next lane, so the search lands past them)
            int o = 0;
#pragma unroll
            for (int st = 16; st; st >>= 1) {
                const uint32_t e = __shfl_sync(0xffffffffu, excl, o + st);
                if (e <= k) o += st;
            }
            uint32_t lo = k - __shfl_sync(0xffffffffu, excl, o);
            const uint32_t ro = __shfl_sync(0xffffffffu, r, o), mo = __shfl_sync(0xffffffffu, msk, o);
            const uint32_t no = __shfl_sync(0xffffffffu, n, o), ho = __shfl_sync(0xffffffffu, hi, o);
            const uint32_t wo = (ro >> 24) - ((ro >> 16) & 0xFFu) + 1u;
            const uint32_t ao = (((ro >> 8) & 0xFFu) - (ro & 0xFFu) + 1u) * wo;
            if (act && ao <= (uint32_t)kMaskTiles) lo = nth_set_bit(mo, lo);        // the lo-th kept tile
            HS_CHECK(!act || lo < ao, "tile scatter rectangle index", lo);
            // lo / wo without an integer division (hs_project.cu: the tile pass)
            const uint32_t dy = (uint32_t)__fdividef((float)lo + 0.5f, (float)wo), dx = lo - dy * wo;
            const uint32_t key = ho | ((( ro & 0xFFu) + dy) * (uint32_t)tiles_x + ((ro >> 16) & 0xFFu) + dx);
#if HS_SCATTER_MATCH
            const uint32_t grp = __match_any_sync(0xffffffffu, act ? key : 0xFFFFFFFFu);
            const int leader = __ffs(grp) - 1;
            uint32_t base = 0;
            if (act && lane == leader) base = atomicAdd(cursor + key, (uint32_t)__popc(grp));
            base = __shfl_sync(0xffffffffu, base, leader);
            if (act) {
                const uint32_t pos = base + (uint32_t)__popc(grp & lt_mask);
#else
            if (act) {
                const uint32_t pos = atomicAdd(cursor + key, 1u);
#endif
                HS_CHECK(pos < capacity, "tile scatter slot", pos);
                vals[pos] = no;
                if (keys) keys[pos] = key;
            }
        }
    }
}

// -------------------------------------------------------------------- sort

__device__ __forceinline__ unsigned long long sort_key(const float *__restrict__ depth, int64_t frame_base,
                                                       uint32_t n) {
    return ((unsigned long long)__float_as_uint(depth[frame_base + n]) << 32) | n;
}

// bitonic compare-exchange network over P (a power of two) keys in shared memory,
// `threads` cooperating threads with index t (one warp, or the whole CTA)
template <bool kCta>
__device__ __forceinline__ void bitonic_smem(unsigned long long *s, int P, int t, int threads) {
    for (int k = 2; k <= P; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int q = t; q < (P >> 1); q += threads) {
                const int i = ((q & ~(j - 1)) << 1) | (q & (j - 1));
                const int l = i + j;
                const unsigned long long a = s[i], c = s[l];
                if ((a > c) == ((i & k) == 0)) {
                    s[i] = c;
                    s[l] = a;
                }
            }
            if (kCta) __syncthreads();
            else __syncwarp();
        }
}

// Register bitonic sort of one list by one warp: E keys per lane, key q = e * 32 +
// lane (padding ~0 sorts last).  Strides below 32 exchange across lanes with
// shuffles; strides of 32 and up swap registers of the same lane.  The stage loops
// stay rolled (small code: the kernels run out of the instruction cache otherwise).
template <int E, int JE, typename K>
__device__ __forceinline__ void swap_regs(K (&key)[E], int k) {
    const int kd = k >> 5;                       // k >= 64 here: lane bits do not matter
#pragma unroll
    for (int e = 0; e < E; ++e) {
        if (e & JE) continue;
        const bool up = (e & kd) == 0;
        const K a = key[e], b = key[e | JE];
        key[e] = up ? min(a, b) : max(a, b);
        key[e | JE] = up ? max(a, b) : min(a, b);
    }
}


// The common case in 32-bit keys: ((depth bits - the list's smallest) >> sh) << IB |
// slot, slot = the entry's position in the unsorted list, whose full 64-bit key
// (depth bits << 32 | index) waits in shared memory; sh drops just enough low depth
// bits to fit.  Entries left next to each other with equal 32-bit depth fields (exact
// depth ties, or depths that differ only in the dropped bits) are then put in full-key
// order by odd-even transposition over the sorted slots.  Returns false -- `vals`
// untouched -- when that does not settle within kFixRounds rounds (long runs of equal
// depths); the caller then sorts the full 64-bit keys in shared memory.
constexpr int kFixRounds = 32;
#ifndef HS_SORT_LANE_MAJOR
#define HS_SORT_LANE_MAJOR 1         // short lists: lane-major register layout (fewer shuffle stages)
#endif

// ascending bitonic network over the 32 * E 32-bit keys of a warp (key q = e * 32 + lane)
template <int E>
__device__ __forceinline__ void bitonic_u32(uint32_t (&key)[E], int lane) {
    constexpr int P = 32 * E;
#pragma unroll 1
    for (int k = 2; k <= P; k <<= 1) {
#pragma unroll 1
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= 32) {
                const int je = j >> 5;
                if (E >= 32 && je == 16) swap_regs<E, (E >= 32 ? 16 : 0)>(key, k);
                else if (E >= 16 && je == 8) swap_regs<E, (E >= 16 ? 8 : 0)>(key, k);
                else if (E >= 8 && je == 4) swap_regs<E, (E >= 8 ? 4 : 0)>(key, k);
                else if (E >= 4 && je == 2) swap_regs<E, (E >= 4 ? 2 : 0)>(key, k);
                else if (E >= 2 && je == 1) swap_regs<E, (E >= 2 ? 1 : 0)>(key, k);
            } else {
                const bool lower = (lane & j) == 0;
                // this slot keeps the smaller key when its half runs ascending: the
                // direction bit is the lane's (k < 32) or the register's (k >= 32)
                const int kd = k >> 5;
                const bool lane_up = (lane & k) == 0;
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const bool up = kd ? (e & kd) == 0 : lane_up;
                    const uint32_t o = __shfl_xor_sync(0xffffffffu, key[e], j);
                    key[e] = (lower == up) ? min(key[e], o) : max(key[e], o);
                }
            }
        }
    }
}

// Lane-major variant (HS_SORT_LANE_MAJOR): key q = lane * E + e, so strides below E swap
// registers of the same lane and only strides of E and up exchange across lanes -- for
// E = 4 / 8, 15 shuffle stages instead of 25 / 30.
template <int E, int J>
__device__ __forceinline__ void swap_in_lane(uint32_t (&key)[E], int lane, int k) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
        if (e & J) continue;
        const bool up = (((lane * E) + e) & k) == 0;
        const uint32_t a = key[e], b = key[e | J];
        key[e] = up ? min(a, b) : max(a, b);
        key[e | J] = up ? max(a, b) : min(a, b);
    }
}
template <int E>
__device__ __forceinline__ void bitonic_u32_lm(uint32_t (&key)[E], int lane) {
    constexpr int P = 32 * E;
#pragma unroll 1
    for (int k = 2; k <= P; k <<= 1) {
#pragma unroll 1
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j < E) {
                if (E >= 16 && j == 8) swap_in_lane<E, (E >= 16 ? 8 : 0)>(key, lane, k);
                else if (E >= 8 && j == 4) swap_in_lane<E, (E >= 8 ? 4 : 0)>(key, lane, k);
                else if (E >= 4 && j == 2) swap_in_lane<E, (E >= 4 ? 2 : 0)>(key, lane, k);
                else if (E >= 2 && j == 1) swap_in_lane<E, (E >= 2 ? 1 : 0)>(key, lane, k);
            } else {
                const int jl = j / E;                 // lane stride
                const bool lower = (lane & jl) == 0;
                const bool up = (lane & (k / E)) == 0;  // k >= 2j >= 2E: direction by lane
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const uint32_t o = __shfl_xor_sync(0xffffffffu, key[e], jl);
                    key[e] = (lower == up) ? min(key[e], o) : max(key[e], o);
                }
            }
        }
    }
}

template <int E>
__device__ __forceinline__ bool sort_list_warp32(const float *__restrict__ depth, int64_t fb, uint32_t start,
                                                 uint32_t len, uint32_t *__restrict__ vals, int lane,
                                                 unsigned long long *__restrict__ s_k64,
                                                 uint32_t *__restrict__ s_q) {
    constexpr int IB = E == 1 ? 5 : E == 2 ? 6 : E == 4 ? 7 : E == 8 ? 8 : E == 16 ? 9 : 10;
    constexpr uint32_t kSlot = (1u << IB) - 1u;
    // the list position of register e of this lane
    auto kQ = [&](int e) -> uint32_t { return HS_SORT_LANE_MAJOR ? (uint32_t)(lane * E + e) : (uint32_t)(e * 32 + lane); };
    // the entries are read into the registers e-major (slot e * 32 + lane: coalesced loads,
    // conflict-free 8-byte stores); the network sorts any placement, and the slot only
    // names the entry's full key in s_k64
#ifndef HS_SORT_LOAD_EMAJOR
#define HS_SORT_LOAD_EMAJOR 1
#endif
    auto kL = [&](int e) -> uint32_t { return HS_SORT_LOAD_EMAJOR ? (uint32_t)(e * 32 + lane) : kQ(e); };
    uint32_t key[E];
    uint32_t dmin = 0xFFFFFFFFu, dmax = 0u;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const uint32_t q = kL(e);
        key[e] = 0xFFFFFFFFu;
        if (q < len) {
            const uint32_t n = vals[start + q];
            key[e] = __float_as_uint(depth[fb + n]);
            s_k64[q] = ((unsigned long long)key[e] << 32) | n;
            dmin = min(dmin, key[e]);
            dmax = max(dmax, key[e]);
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        dmin = min(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
        dmax = max(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    }
    const int span = 32 - __clz(dmax - dmin);
    const int sh = max(0, span - (31 - IB));           // real keys stay below 2^31
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const uint32_t q = kL(e);
        if (q < len) key[e] = (((key[e] - dmin) >> sh) << IB) | q;
    }
    if (HS_SORT_LANE_MAJOR) bitonic_u32_lm<E>(key, lane);
    else bitonic_u32<E>(key, lane);
    // neighbours with equal depth fields?
    bool tie = false;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        uint32_t prev;
        if (HS_SORT_LANE_MAJOR) {          // q - 1: the previous register, or lane - 1's last
            const uint32_t up_last = __shfl_up_sync(0xffffffffu, key[E - 1], 1);
            prev = e > 0 ? key[e > 0 ? e - 1 : 0] : up_last;
        } else {
            prev = __shfl_up_sync(0xffffffffu, key[e], 1);
            if (e > 0) {
                const uint32_t wrap = __shfl_sync(0xffffffffu, key[e > 0 ? e - 1 : 0], 31);
                if (lane == 0) prev = wrap;
            }
        }
        const uint32_t q = kQ(e);
        if (q > 0 && q < len && (prev >> IB) == (key[e] >> IB)) tie = true;
    }
    __syncwarp();
    if (!__any_sync(0xffffffffu, tie)) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const uint32_t q = kQ(e);
            if (q < len) vals[start + q] = (uint32_t)s_k64[key[e] & kSlot];
        }
        return true;
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const uint32_t q = kQ(e);
        if (q < len) s_q[q] = key[e];
    }
    __syncwarp();
    int quiet = 0;
    for (int round = 0; round < kFixRounds && quiet < 2; ++round) {
        bool swapped = false;
        for (uint32_t i = 2 * (uint32_t)lane + (round & 1); i + 1 < len; i += 64) {
            const uint32_t a = s_q[i], b = s_q[i + 1];
            if ((a >> IB) == (b >> IB) && s_k64[a & kSlot] > s_k64[b & kSlot]) {
                s_q[i] = b;
                s_q[i + 1] = a;
                swapped = true;
            }
        }
        __syncwarp();
        quiet = __any_sync(0xffffffffu, swapped) ? 0 : quiet + 1;
    }
    if (quiet < 2) return false;
    for (uint32_t q = lane; q < len; q += 32) vals[start + q] = (uint32_t)s_k64[s_q[q] & kSlot];
    return true;
}

// a list the 32-bit sort declines is sorted on its 64-bit keys in the warp's shared memory
template <int E>
__device__ __forceinline__ void sort_list(const float *__restrict__ depth, int64_t fb, uint32_t start,
                                          uint32_t len, uint32_t *__restrict__ vals, int lane,
                                          unsigned long long *__restrict__ s_k64, uint32_t *__restrict__ s_q) {
    if (!sort_list_warp32<E>(depth, fb, start, len, vals, lane, s_k64, s_q)) {
        // the full 64-bit keys are still in shared memory: sort them there (rare)
        int P = 32;
        while (P < (int)len) P <<= 1;
        for (int q = (int)len + lane; q < P; q += 32) s_k64[q] = ~0ull;
        __syncwarp();
        bitonic_smem<false>(s_k64, P, lane, 32);
        for (uint32_t q = lane; q < len; q += 32) vals[start + q] = (uint32_t)s_k64[q];
    }
    __syncwarp();
}

// One warp per list of 2..kWarpShort entries, the warps striding over all segments.
#ifndef HS_SHORT_SORT_MINB
#define HS_SHORT_SORT_MINB 8
#endif
__global__ void __launch_bounds__(32 * kWarpSortWarps, HS_SHORT_SORT_MINB) tile_sort_warp_kernel(
    int64_t N, int tile_bits, int nseg, const float *__restrict__ depth, const uint32_t *__restrict__ ranges,
    uint32_t *__restrict__ lists, uint32_t *__restrict__ list_counts, uint64_t capacity,
    const unsigned long long *__restrict__ summary, uint32_t *__restrict__ vals) {
    pdl_prologue();
    __shared__ unsigned long long s_k64_all[kWarpSortWarps][kWarpShort];
    __shared__ uint32_t s_q_all[kWarpSortWarps][kWarpShort];
    if (summary[0] > capacity) return;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned long long *s_k64 = s_k64_all[w];
    uint32_t *s_q = s_q_all[w];
    // warp g takes segments g + j * stride; 32 candidates are read at once (one per lane)
    const uint32_t stride = gridDim.x * kWarpSortWarps;
    for (uint32_t base = blockIdx.x * kWarpSortWarps + w; base < (uint32_t)nseg; base += 32 * stride) {
        const uint32_t seg_l = base + lane * stride;
        const uint2 rg_l = seg_l < (uint32_t)nseg ? reinterpret_cast<const uint2 *>(ranges)[seg_l] : make_uint2(0u, 0u);
        const uint32_t len_l = rg_l.y - rg_l.x;
        uint32_t pick = __ballot_sync(0xffffffffu, len_l >= 2u && len_l <= (uint32_t)kWarpShort);
        while (pick) {
            const int b = __ffs(pick) - 1;
            pick &= pick - 1u;
            const uint32_t seg = base + b * stride;
            const uint32_t start = __shfl_sync(0xffffffffu, rg_l.x, b), len = __shfl_sync(0xffffffffu, len_l, b);
            const int64_t fb = (int64_t)(seg >> tile_bits) * N;
            if (len <= 32u) sort_list<1>(depth, fb, start, len, vals, lane, s_k64, s_q);
            else if (len <= 64u) sort_list<2>(depth, fb, start, len, vals, lane, s_k64, s_q);
            else if (len <= 128u) sort_list<4>(depth, fb, start, len, vals, lane, s_k64, s_q);
            else if (kWarpShort <= 256 || len <= 256u) sort_list<8>(depth, fb, start, len, vals, lane, s_k64, s_q);
            else sort_list<(kWarpShort > 256 ? 16 : 8)>(depth, fb, start, len, vals, lane, s_k64, s_q);
        }
    }
}

// Lists of kWarpShort+1..kWarpCap entries: one CTA of kLongWarps warps per list.
// Each warp sorts a run of kWarpShort entries in registers (the 32-bit keys of
// sort_list_warp32, on the list-wide depth offset and shift, 10 slot bits); every key
// then finds its merged position by binary search in the other runs (keys are unique),
// and the equal-depth-field fix-up runs over the merged list.  A list the fix-up does
// not settle is sorted on its full 64-bit keys in place, in the same shared memory.
#ifndef HS_LONG_RUN
#define HS_LONG_RUN 256
#endif
constexpr int kRun = HS_LONG_RUN;               // entries per warp-sorted run
constexpr int kLongWarps = kWarpCap / kRun;
static_assert(kRun >= 32 && kRun <= kWarpCap / 2 && kWarpCap % kRun == 0,
              "a long list is merged from >= 2 warp runs that fill s_k64[kWarpCap]");

__global__ void __launch_bounds__(32 * kLongWarps) tile_sort_long_kernel(
    int64_t N, int tile_bits, int nseg, const float *__restrict__ depth, const uint32_t *__restrict__ ranges,
    uint32_t *__restrict__ lists, uint32_t *__restrict__ list_counts, int half, uint64_t capacity,
    const unsigned long long *__restrict__ summary, uint32_t *__restrict__ vals) {
    pdl_prologue();
    constexpr int E = kRun / 32, IB = 10;
    constexpr uint32_t kSlot = (1u << IB) - 1u;
    __shared__ unsigned long long s_k64[kWarpCap];
    __shared__ uint32_t s_run[kWarpCap], s_out[kWarpCap];
    __shared__ uint32_t s_min[kLongWarps], s_max[kLongWarps];
    __shared__ int s_flag;
    if (summary[0] > capacity) return;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    // the lists longer than kWarpShort, collected by the scan: CTA c takes c + j * gridDim.x
    const uint32_t nbig = filled_half(list_counts, half)[1];
    for (uint32_t li = blockIdx.x; li < nbig; li += gridDim.x) {
      {
        const uint32_t seg = lists[li];
        const uint2 rg = reinterpret_cast<const uint2 *>(ranges)[seg];
        const uint32_t start = rg.x, len = rg.y - rg.x;
        const int64_t fb = (int64_t)(seg >> tile_bits) * N;
        uint32_t key[E];
        uint32_t dmin = 0xFFFFFFFFu, dmax = 0u;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const uint32_t q = (uint32_t)(w * kRun + e * 32 + lane);
            key[e] = 0xFFFFFFFFu;
            if (q < len) {
                const uint32_t n = vals[start + q];
                key[e] = __float_as_uint(depth[fb + n]);
                s_k64[q] = ((unsigned long long)key[e] << 32) | n;
                dmin = min(dmin, key[e]);
                dmax = max(dmax, key[e]);
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            dmin = min(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
            dmax = max(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
        }
        if (lane == 0) {
            s_min[w] = dmin;
            s_max[w] = dmax;
        }
        __syncthreads();
#pragma unroll
        for (int v = 0; v < kLongWarps; ++v) {
            dmin = min(dmin, s_min[v]);
            dmax = max(dmax, s_max[v]);
        }
        const int sh = max(0, (32 - __clz(dmax - dmin)) - (31 - IB));
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const uint32_t q = (uint32_t)(w * kRun + e * 32 + lane);
            if (q < len) key[e] = (((key[e] - dmin) >> sh) << IB) | q;
        }
        if (w * kRun < (int)len) {                            // (runs past the end: padding)
            if (HS_SORT_LANE_MAJOR) bitonic_u32_lm<E>(key, lane);
            else bitonic_u32<E>(key, lane);
        }
#pragma unroll
        for (int e = 0; e < E; ++e) s_run[w * kRun + (HS_SORT_LANE_MAJOR ? lane * E + e : e * 32 + lane)] = key[e];
        __syncthreads();
        // merged position: own rank + the keys below it in every other run (runs past
        // the list's end hold padding only and count nothing)
        const int runs = (int)((len + kRun - 1) / kRun);
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const uint32_t x = key[e];
            if (x == 0xFFFFFFFFu) continue;          // padding (real keys stay below 2^31)
            uint32_t pos = (uint32_t)(HS_SORT_LANE_MAJOR ? lane * E + e : e * 32 + lane);
            for (int v = 0; v < runs; ++v) {
                if (v == w) continue;
                // count of run v's keys below x: a branch-free search over its kRun keys
                int lo = v * kRun;
#pragma unroll
                for (int step = kRun / 2; step > 0; step >>= 1)
                    if (s_run[lo + step - 1] < x) lo += step;
                if (s_run[lo] < x) ++lo;
                pos += (uint32_t)(lo - v * kRun);
            }
            if (pos < len) s_out[pos] = x;
        }
        __syncthreads();
        // equal depth fields next to each other: odd-even transposition on full keys
        if (threadIdx.x == 0) s_flag = 0;
        __syncthreads();
        for (uint32_t i = threadIdx.x + 1; i < len; i += blockDim.x)
            if ((s_out[i - 1] >> IB) == (s_out[i] >> IB)) s_flag = 1;
        __syncthreads();
        bool ok = true;
        if (s_flag) {
            int quiet = 0;
            for (int round = 0; round < kFixRounds && quiet < 2; ++round) {
                __syncthreads();
                if (threadIdx.x == 0) s_flag = 0;
                __syncthreads();
                for (uint32_t i = 2 * threadIdx.x + (round & 1); i + 1 < len; i += 2 * blockDim.x) {
                    const uint32_t a = s_out[i], b = s_out[i + 1];
                    if ((a >> IB) == (b >> IB) && s_k64[a & kSlot] > s_k64[b & kSlot]) {
                        s_out[i] = b;
                        s_out[i + 1] = a;
                        s_flag = 1;
                    }
                }
                __syncthreads();
                quiet = s_flag ? 0 : quiet + 1;
            }
            ok = quiet >= 2;
        }
        if (ok) {
            for (uint32_t q = threadIdx.x; q < len; q += blockDim.x) vals[start + q] = (uint32_t)s_k64[s_out[q] & kSlot];
        } else {
            // the full 64-bit keys are still in shared memory: sort them there (rare); P is
            // the next power of two >= len (<= kWarpCap: these lists hold at most kWarpCap)
            int P = 32;
            while (P < (int)len) P <<= 1;
            for (int q = (int)len + threadIdx.x; q < P; q += blockDim.x) s_k64[q] = ~0ull;
            __syncthreads();
            bitonic_smem<true>(s_k64, P, threadIdx.x, blockDim.x);
            for (uint32_t q = threadIdx.x; q < len; q += blockDim.x) vals[start + q] = (uint32_t)s_k64[q];
        }
        __syncthreads();
      }
    }
}

// one CTA per list of kWarpCap+1..kCtaCap entries
__global__ void __launch_bounds__(kCtaSortThreads) tile_sort_cta_kernel(
    int64_t N, int tile_bits, int nseg, const float *__restrict__ depth, const uint32_t *__restrict__ ranges,
    const uint32_t *__restrict__ lists, const uint32_t *__restrict__ list_counts, int half, uint64_t capacity,
    const unsigned long long *__restrict__ summary, uint32_t *__restrict__ vals) {
    pdl_prologue();
    extern __shared__ unsigned long long s_keys[];
    if (summary[0] > capacity) return;
    const uint32_t nbig = filled_half(list_counts, half)[2];
    for (uint32_t li = blockIdx.x; li < nbig; li += gridDim.x) {
      {
        const uint32_t seg = lists[nseg - 1 - li];
        const uint2 rg = reinterpret_cast<const uint2 *>(ranges)[seg];
        const uint32_t start = rg.x, len = rg.y - rg.x;
        const int64_t fb = (int64_t)(seg >> tile_bits) * N;
        int P = 2 * kWarpCap;
        while (P < (int)len) P <<= 1;
        for (int q = threadIdx.x; q < P; q += kCtaSortThreads)
            s_keys[q] = q < (int)len ? sort_key(depth, fb, vals[start + q]) : ~0ull;
        __syncthreads();
        bitonic_smem<true>(s_keys, P, threadIdx.x, kCtaSortThreads);
        for (int q = threadIdx.x; q < (int)len; q += kCtaSortThreads) vals[start + q] = (uint32_t)s_keys[q];
        __syncthreads();
      }
    }
}

}  // namespace hs

using namespace hs;

namespace hs {
// caller-owned fork context of hs_tile_fill (see hs_api.h)
struct HsFork {
    int device = 0;
    cudaStream_t side = nullptr;
    cudaEvent_t forked = nullptr, joined = nullptr;
};
}  // namespace hs

extern "C" {

int hs_tile_sort_cap(void) { return kCtaCap; }
int hs_tile_cta_sort_min(void) { return kWarpCap + 1; }

int hs_tile_count(int B, int64_t N, int width, int height, const float *records, const uint32_t *counts,
                  uint32_t *tile_counts, void *stream) {
    const int64_t items = (int64_t)B * N;
    if (items <= 0) return HS_OK;
    const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
    const int tile_bits = bit_length_u32((uint32_t)(tiles_x * tiles_y - 1));
    if (tile_bits + bit_length_u32((uint32_t)(B - 1)) > 31) {
        set_error("hs_tile_count: frame/tile bits exceed 31");
        return HS_ERR_SHAPE;
    }
    const int tiles = tiles_x * tiles_y;
    const size_t smem = tiles <= kTileSmemBins ? sizeof(uint32_t) * tiles : 0;
    launch_k(tile_count_kernel, grid_for(items, kTileItems), kTileThreads, smem, HS_CHECK_STREAM(stream), 
        items, N, tiles_x, tiles, tile_bits, records, counts, tile_counts);
    return check_launch("hs_tile_count");
}

int hs_tile_scan(int B, int width, int height, uint32_t *tile_counts, uint32_t *ranges, uint32_t *cursor,
                 uint32_t *lists, uint32_t *list_counts, int list_half, unsigned long long *err,
                 uint32_t *depth_range, unsigned long long *summary, void *stream) {
    const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
    const int tile_bits = bit_length_u32((uint32_t)(tiles_x * tiles_y - 1));
    const int64_t nseg = (int64_t)B << tile_bits;
    if (B <= 0 || nseg > (1ll << 30)) {
        set_error("hs_tile_scan: bad segment count");
        return HS_ERR_SHAPE;
    }
    cudaStream_t s = HS_CHECK_STREAM(stream);
#ifndef HS_SCAN_MULTI
#define HS_SCAN_MULTI 1
#endif
    if (HS_SCAN_MULTI && nseg > kScanSpan) {
        const int ctas = (int)((nseg + kScanSpan - 1) / kScanSpan);
        if (list_half < 8 + ctas) {
            set_error("hs_tile_scan: list_counts halves of %d words, need %d", list_half, 8 + ctas);
            return HS_ERR_SHAPE;
        }
        launch_k(tile_scan_multi_kernel, ctas, kScanSpan, 0, s, (int)nseg, tile_counts, ranges, cursor, lists, list_counts,
                                                          list_half, err, depth_range, summary);
    } else {
        if (list_half < 8) {
            set_error("hs_tile_scan: list_counts halves of %d words, need >= 8", list_half);
            return HS_ERR_SHAPE;
        }
        launch_k(tile_scan_kernel, 1, 1024, 0, s, (int)nseg, tile_counts, ranges, cursor, lists, list_counts, list_half,
                                            err, depth_range, summary);
    }
    return check_launch("hs_tile_scan");
}

void *hs_fork_create(void) {
    HsFork *f = new HsFork();
    cudaGetDevice(&f->device);
    if (cudaStreamCreateWithFlags(&f->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&f->forked, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&f->joined, cudaEventDisableTiming) != cudaSuccess) {
        set_error("hs_fork_create: %s", cudaGetErrorString(cudaGetLastError()));
        delete f;
        return nullptr;
    }
    return f;
}

void hs_fork_destroy(void *fork) {
    HsFork *f = reinterpret_cast<HsFork *>(fork);
    if (!f) return;
    cudaStreamSynchronize(f->side);
    cudaEventDestroy(f->forked);
    cudaEventDestroy(f->joined);
    cudaStreamDestroy(f->side);
    delete f;
}

int hs_tile_fill(int B, int64_t N, int width, int height, const float *records, const uint32_t *counts,
                 const uint32_t *tile_rects, const float *depth, const uint32_t *ranges, uint32_t *cursor, uint32_t *lists,
                 uint32_t *list_counts, int list_half, const unsigned long long *summary, uint64_t capacity,
                 uint32_t *keys, uint32_t *values, int flags, void *fork, void *stream) {
    const int64_t items = (int64_t)B * N;
    if (items <= 0) return HS_OK;
    cudaStream_t s = HS_CHECK_STREAM(stream);
    const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
    const int tile_bits = bit_length_u32((uint32_t)(tiles_x * tiles_y - 1));
    const int nseg = B << tile_bits;
    const int tiles = tiles_x * tiles_y;
    const size_t tsmem = tiles <= kTileSmemBins ? sizeof(uint32_t) * tiles : 0;
#ifndef HS_SCATTER_WARP
#define HS_SCATTER_WARP 1
#endif
    if (HS_SCATTER_WARP && tile_rects && tiles_x <= 256) {
        const int64_t warps = (items + 32 * kSwRounds - 1) / (32 * kSwRounds);
        launch_k(tile_scatter_warp_kernel, (unsigned)((warps + 7) / 8), 256, 0, s, items, N, tiles_x, tile_bits, tile_rects,
                                                                            cursor, capacity, summary, keys, values);
    } else {
        launch_k(tile_scatter_kernel, grid_for(items, kTileItems), kTileThreads, tsmem, s, 
            items, N, tiles_x, tiles, tile_bits, records, counts, tile_rects, cursor, capacity, summary, keys, values);
    }
    const int sms = current_sm_count();
    // the long lists first (fewer, longer: their tail overlaps nothing otherwise); the
    // short lists sort on the fork context's side stream alongside them (each kernel
    // leaves SMs idle in its tail), and the caller's stream waits for both
    HsFork *f = reinterpret_cast<HsFork *>(fork);
    cudaStream_t side = s;
    if (f) {
        cudaEventRecord(f->forked, s);
        cudaStreamWaitEvent(f->side, f->forked, 0);
        side = f->side;
    }
    if (flags & HS_FILL_CTA_SORT) {
        // lists of kWarpCap+1..kCtaCap entries expected: their CTA sorts go first on the
        // side stream, so they start beside the long-list sort instead of after it
        const int csmem = kCtaCap * (int)sizeof(unsigned long long);
        cudaFuncSetAttribute(tile_sort_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, csmem);
        launch_k(tile_sort_cta_kernel, (unsigned)sms * 2, kCtaSortThreads, csmem, side, N, tile_bits, nseg, depth,
                 ranges, lists, list_counts, list_half, capacity, summary, values);
    }
#ifndef HS_SHORT_SORT_CTAS_PER_SM
#define HS_SHORT_SORT_CTAS_PER_SM 16
#endif
    launch_k(tile_sort_warp_kernel, (unsigned)sms * HS_SHORT_SORT_CTAS_PER_SM, 32 * kWarpSortWarps, 0, side, 
        N, tile_bits, nseg, depth, ranges, lists, list_counts, capacity, summary, values);
    if (f) cudaEventRecord(f->joined, f->side);
#ifndef HS_LONG_SORT_CTAS_PER_SM
#define HS_LONG_SORT_CTAS_PER_SM 16
#endif
    launch_k(tile_sort_long_kernel, (unsigned)sms * HS_LONG_SORT_CTAS_PER_SM, 32 * kLongWarps, 0, s, 
        N, tile_bits, nseg, depth, ranges, lists, list_counts, list_half, capacity, summary, values);
    if (f) cudaStreamWaitEvent(s, f->joined, 0);
    return check_launch("hs_tile_fill");
}

int hs_tile_fill_longest(int B, int64_t N, int width, int height, const float *depth, const uint32_t *ranges,
                         uint32_t *lists, uint32_t *list_counts, int list_half,
                         const unsigned long long *summary, uint64_t capacity, uint32_t *values, void *stream) {
    if ((int64_t)B * N <= 0) return HS_OK;
    cudaStream_t s = HS_CHECK_STREAM(stream);
    const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
    const int tile_bits = bit_length_u32((uint32_t)(tiles_x * tiles_y - 1));
    const int nseg = B << tile_bits;
    const int sms = current_sm_count();
    const int csmem = kCtaCap * (int)sizeof(unsigned long long);
    // (a per-device function attribute: set on every call, so any device a caller drives
    // has it -- a cheap host call)
    cudaFuncSetAttribute(tile_sort_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, csmem);
    launch_k(tile_sort_cta_kernel, (unsigned)sms * 2, kCtaSortThreads, csmem, s, N, tile_bits, nseg, depth, ranges, lists,
                                                                          list_counts, list_half, capacity, summary,
                                                                          values);
    return check_launch("hs_tile_fill_longest");
}

}  // extern "C"
