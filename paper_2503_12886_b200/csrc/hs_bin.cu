// hs_bin.cu -- batched tile binning on sm_100a: key-offset scan, key emission,
// a stable LSD radix sort of (frame, tile, depth) keys and per-tile ranges.
//
// The reference has no tiles: one global stable depth argsort per frame
// (S/render.py:221-223) and a per-splat pixel-bbox scatter (:248-251).  The
// device path keys every (frame, splat, tile) overlap and sorts all frames of a
// step in one pass; oracle/binning.py is the bit-exact CPU restatement
// (SURVEY Appendix B).  Stable sorting of keys emitted in Gaussian order makes
// equal depth bits resolve to the lower index, the reference's tie-break.
#include <algorithm>

#include "hs_common.cuh"

namespace hs {

// ------------------------------------------------------------- offsets scan

// One CTA: exclusive scan of the per-256-item tile-count sums.  Writes the key
// total and the error word to `summary` (the step's single device->host read).
__global__ void __launch_bounds__(1024) scan_kernel(int nb, const uint32_t *__restrict__ sums,
                                                    uint32_t *__restrict__ offs,
                                                    const unsigned long long *__restrict__ err,
                                                    const uint32_t *__restrict__ depth_range,
                                                    unsigned long long *__restrict__ summary) {
    pdl_prologue();
    __shared__ unsigned long long warp_tot[32];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int per = (nb + blockDim.x - 1) / blockDim.x;
    const int lo = min(nb, tid * per), hi = min(nb, lo + per);
    unsigned long long local = 0;
    for (int i = lo; i < hi; ++i) local += sums[i];
    unsigned long long incl = local;
    for (int o = 1; o < 32; o <<= 1) {
        unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) warp_tot[w] = incl;
    __syncthreads();
    if (w == 0) {
        unsigned long long v = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0ull;
        for (int o = 1; o < 32; o <<= 1) {
            unsigned long long t = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += t;
        }
        warp_tot[lane] = v;  // inclusive over warps
    }
    __syncthreads();
    unsigned long long run = (w > 0 ? warp_tot[w - 1] : 0ull) + incl - local;
    for (int i = lo; i < hi; ++i) {
        offs[i] = (uint32_t)run;
        run += sums[i];
    }
    if (tid == 0 && summary) {
        summary[0] = warp_tot[(blockDim.x >> 5) - 1];
        summary[1] = err ? *err : HS_NO_ERROR;
        summary[2] = depth_range ? ((unsigned long long)depth_range[1] << 32) | depth_range[0] : 0xFFFFFFFFull;
    }
}

// ------------------------------------------------------------------ emission

#ifdef HS_BIN_STATS
__device__ unsigned long long g_bin_stats[2];
#endif

// Same 256-item partition as the projection kernel: block-local exclusive scan of
// the tile counts plus the block offset gives each (frame, Gaussian) its slot.
__global__ void __launch_bounds__(kScanBlock) emit_kernel(int B, int64_t N, int tiles_x, int tile_bits,
                                                          const float *__restrict__ records,
                                                          const float *__restrict__ depth,
                                                          const uint32_t *__restrict__ counts,
                                                          const uint32_t *__restrict__ offs,
                                                          const uint32_t *__restrict__ rects,
                                                          uint64_t *__restrict__ keys,
                                                          uint32_t *__restrict__ vals) {
    pdl_prologue();
    __shared__ uint32_t warp_tot[kScanBlock / 32];
    const int64_t i = blockIdx.x * (int64_t)kScanBlock + threadIdx.x;
    const bool in = i < (int64_t)B * N;
    const uint32_t cnt = in ? counts[i] : 0u;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t incl = cnt;
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) warp_tot[w] = incl;
    __syncthreads();
    uint32_t wpre = 0;
    for (int k = 0; k < w; ++k) wpre += warp_tot[k];
    if (!in || cnt == 0) return;
    uint32_t pos = offs[blockIdx.x] + wpre + incl - cnt;
    const int b = (int)item_frame(i, N);
    const uint32_t n = (uint32_t)(i - (int64_t)b * N);
    const float *rec = records + i * kRec;
    const uint32_t rows = __float_as_uint(rec[7]), cols = __float_as_uint(rec[8]);
    const int ty0 = unpack_lo(rows) / kTile, ty1 = unpack_hi(rows) / kTile;
    const int tx0 = unpack_lo(cols) / kTile, tx1 = unpack_hi(cols) / kTile;
    const uint64_t hi = ((uint64_t)b << (tile_bits + 32)) | (uint64_t)__float_as_uint(depth[i]);
    // with the projection's tile_rects: only its kept tiles (counts[i] of them)
    const uint32_t mask = rects ? rects[2 * i + 1] : 0xFFFFFFFFu;
    const int area = (ty1 - ty0 + 1) * (tx1 - tx0 + 1);
    int idx = 0;
    for (int ty = ty0; ty <= ty1; ++ty)
        for (int tx = tx0; tx <= tx1; ++tx, ++idx) {
            if (!mask_keeps(mask, area, idx)) continue;
            keys[pos] = hi | ((uint64_t)(ty * tiles_x + tx) << 32);
            vals[pos] = n;
            ++pos;
#ifdef HS_BIN_STATS
            {   // would the exact ellipse-rectangle test cull this (splat, tile) key?
                const float mx = rec[0], my = rec[1], a = rec[2], bb = rec[3], c = rec[4], qmax = rec[6];
                const int rl = unpack_lo(rows), rh = unpack_hi(rows), cl = unpack_lo(cols), ch = unpack_hi(cols);
                const int xs = max(tx * kTile, cl), xe = min(tx * kTile + kTile - 1, ch);
                const int ys = max(ty * kTile, rl), ye = min(ty * kTile + kTile - 1, rh);
                bool cull = xs > xe || ys > ye || !(qmax >= 0.f);
                const float det = a * c - bb * bb;
                if (!cull && det > 0.f && a > 0.f && c > 0.f) {
                    const float dxlo = (float)xs + 0.5f - mx, dxhi = (float)xe + 0.5f - mx;
                    const float dylo = (float)ys + 0.5f - my, dyhi = (float)ye + 0.5f - my;
                    const float dxv = fminf(fmaxf(0.f, dxlo), dxhi);
                    const float dyv = fminf(fmaxf(-bb * dxv / c, dylo), dyhi);
                    const float dyh = fminf(fmaxf(0.f, dylo), dyhi);
                    const float dxh = fminf(fmaxf(-bb * dyh / a, dxlo), dxhi);
                    const float qv = a * dxv * dxv + 2.f * bb * dxv * dyv + c * dyv * dyv;
                    const float qh = a * dxh * dxh + 2.f * bb * dxh * dyh + c * dyh * dyh;
                    cull = fminf(qv, qh) * 0.999f - 1e-3f > qmax;
                }
                atomicAdd(&g_bin_stats[0], 1ull);
                if (cull) atomicAdd(&g_bin_stats[1], 1ull);
            }
#endif
        }
}

// ---------------------------------------------------- two-level binning
//
// Same lists, fewer key bits per sort pass: the (frame, Gaussian) items are first
// sorted by depth alone (32-bit keys over B*N items -- the float depth bits, stable,
// ties to the lower frame-major index), then each item emits its tiles in that
// order with 32-bit (frame, tile) keys, and a stable 2-pass sort by (frame, tile)
// leaves every tile's list in depth order with ties to the lower Gaussian index --
// the lists the one-level (frame, tile, depth) sort produces.

// per 256 sorted items: sum of their tile counts (the emission-offset scan input)
__global__ void __launch_bounds__(kScanBlock) sorted_block_sums_kernel(int64_t items, const uint32_t *__restrict__ order,
                                                                       const uint32_t *__restrict__ counts,
                                                                       uint32_t *__restrict__ block_sums) {
    pdl_prologue();
    const int64_t j = blockIdx.x * (int64_t)kScanBlock + threadIdx.x;
    uint32_t v = j < items ? counts[order[j]] : 0u;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __shared__ uint32_t ws[kScanBlock / 32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int k = 0; k < kScanBlock / 32; ++k) t += ws[k];
        block_sums[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(kScanBlock) emit_sorted_kernel(int64_t items, int64_t N, int tiles_x, int tile_bits,
                                                                 const float *__restrict__ records,
                                                                 const uint32_t *__restrict__ order,
                                                                 const uint32_t *__restrict__ counts,
                                                                 const uint32_t *__restrict__ offs,
                                                                 const uint32_t *__restrict__ rects,
                                                                 uint32_t *__restrict__ keys,
                                                                 uint32_t *__restrict__ vals) {
    pdl_prologue();
    __shared__ uint32_t warp_tot[kScanBlock / 32];
    const int64_t j = blockIdx.x * (int64_t)kScanBlock + threadIdx.x;
    const bool in = j < items;
    const uint32_t i = in ? order[j] : 0u;
    const uint32_t cnt = in ? counts[i] : 0u;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t incl = cnt;
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) warp_tot[w] = incl;
    __syncthreads();
    uint32_t wpre = 0;
    for (int k = 0; k < w; ++k) wpre += warp_tot[k];
    if (in && cnt) {
        uint32_t pos = offs[blockIdx.x] + wpre + incl - cnt;
        const uint32_t b = (uint32_t)item_frame(i, N);
        const uint32_t n = (uint32_t)(i - (int64_t)b * N);
        const float *rec = records + (int64_t)i * kRec;
        const uint32_t rows = __float_as_uint(rec[7]), cols = __float_as_uint(rec[8]);
        const int ty0 = unpack_lo(rows) / kTile, ty1 = unpack_hi(rows) / kTile;
        const int tx0 = unpack_lo(cols) / kTile, tx1 = unpack_hi(cols) / kTile;
        const uint32_t hi = b << tile_bits;
        const uint32_t mask = rects ? rects[2 * (int64_t)i + 1] : 0xFFFFFFFFu;
        const int area = (ty1 - ty0 + 1) * (tx1 - tx0 + 1);
        int idx = 0;
        for (int ty = ty0; ty <= ty1; ++ty)
            for (int tx = tx0; tx <= tx1; ++tx, ++idx) {
                if (!mask_keeps(mask, area, idx)) continue;
                const uint32_t key = hi | (uint32_t)(ty * tiles_x + tx);
                keys[pos] = key;
                vals[pos] = n;
                ++pos;
            }
    }
}

__global__ void tile_ranges32_kernel(int64_t n, const uint32_t *__restrict__ keys, uint32_t *__restrict__ ranges) {
    pdl_prologue();
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t t = keys[i];
    if (i == 0 || keys[i - 1] != t) ranges[2 * (uint64_t)t] = (uint32_t)i;
    if (i == n - 1 || keys[i + 1] != t) ranges[2 * (uint64_t)t + 1] = (uint32_t)(i + 1);
}

// --------------------------------------------------------------- radix sort
//
// Stable LSD radix sort, onesweep style: one kernel computes the digit histograms
// of every pass in a single read of the keys; each pass is then ONE kernel whose
// CTAs take tile ids in launch order, rank their 2048 keys per digit (warp
// match.any), publish per-digit counts and resolve their global digit offsets by
// decoupled look-back over the predecessor tiles, and scatter through shared
// memory so every digit run is written contiguously.  Only the 8-bit digit
// windows that intersect `bit_mask` are sorted (digits that are constant across all
// keys cannot change the order).

#ifndef HS_SORT_MINB
#define HS_SORT_MINB 4
#endif
constexpr int kSortThreads = 256;
#ifndef HS_SORT_ITEMS
#define HS_SORT_ITEMS 8
#endif
constexpr int kSortItems = HS_SORT_ITEMS;
constexpr int kSortTile = kSortThreads * kSortItems;   // 2048 keys per CTA
constexpr int kRadix = 256;
#ifndef HS_LOOKBACK
#define HS_LOOKBACK 8
#endif
constexpr int kLookback = HS_LOOKBACK;
constexpr int kMaxPasses = 8;
constexpr uint32_t kFlagAgg = 1u << 30, kFlagInc = 2u << 30, kCountMask = (1u << 30) - 1u;

struct PassShifts {
    int shift[kMaxPasses];
    int n;
    int plain_below;   // windows below this shift count with plain shared atomics
};

#ifndef HS_HIST32_PLAIN_BELOW
#define HS_HIST32_PLAIN_BELOW 16   // depth-order histogram: plain atomics for the two low windows
#endif
#ifndef HS_TILE_PLAIN_BELOW
#define HS_TILE_PLAIN_BELOW 16     // tile sort: plain atomics for both windows (measured best)
#endif
template <typename KT>
__global__ void __launch_bounds__(256) radix_hist_all_kernel(int64_t n, const KT *__restrict__ keys,
                                                             PassShifts ps, uint32_t *__restrict__ hist) {
    pdl_prologue();
    __shared__ uint32_t h[kMaxPasses][kRadix];
    for (int i = threadIdx.x; i < kMaxPasses * kRadix; i += blockDim.x) (&h[0][0])[i] = 0;
    __syncthreads();
    // warp-uniform trip count so the digit counts can be aggregated per warp with
    // match.any (the frame/tile digits are nearly constant within a warp)
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); i0 < n; i0 += stride) {
        const int64_t i = i0 + lane;
        const bool valid = i < n;
        const uint64_t k = valid ? (uint64_t)keys[i] : 0ull;
        const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
        for (int p = 0; p < ps.n; ++p) {
            const uint32_t d = (uint32_t)(k >> ps.shift[p]) & (kRadix - 1);
            if (!valid) continue;
            if (ps.shift[p] < ps.plain_below) {
                // digits close to random across neighbouring keys (the low depth-mantissa
                // bytes, the tile's low byte): plain shared atomics beat the match
                atomicAdd(&h[p][d], 1u);
            } else {
                const uint32_t peers = __match_any_sync(vmask, d);
                if ((peers & ((1u << lane) - 1u)) == 0u) atomicAdd(&h[p][d], (uint32_t)__popc(peers));
            }
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < ps.n * kRadix; i += blockDim.x) {
        const uint32_t v = (&h[0][0])[i];
        if (v) atomicAdd(hist + i, v);
    }
}

// exclusive scan of each pass's 256 digit counts (one CTA, one thread per digit)
__global__ void __launch_bounds__(kRadix) radix_digit_scan_kernel(int npass, uint32_t *__restrict__ hist) {
    pdl_prologue();
    __shared__ uint32_t warp_tot[kRadix / 32];
    const int d = threadIdx.x, lane = d & 31, w = d >> 5;
    for (int p = 0; p < npass; ++p) {
        const uint32_t v = hist[p * kRadix + d];
        uint32_t incl = v;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) warp_tot[w] = incl;
        __syncthreads();
        uint32_t pre = 0;
        for (int k = 0; k < w; ++k) pre += warp_tot[k];
        hist[p * kRadix + d] = pre + incl - v;
        __syncthreads();
    }
}

// Bits of the float depth keys that can differ among key-emitting splats: every bit at
// or below the highest bit in which the smallest and largest emitted depth differ
// (depth_range = {min, max} float bits; none emitted -> min > max -> 0).
__device__ __forceinline__ uint32_t depth_live_bits(const uint32_t *depth_range) {
    const uint32_t lo = depth_range[0], hi = depth_range[1];
    if (lo > hi) return 0u;
    const uint32_t diff = lo ^ hi;
    return diff ? (0xFFFFFFFFu >> __clz(diff)) : 0u;
}

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t *p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// vals_in == nullptr: the values are the input positions (an implicit iota).
// live_bits != nullptr: a device word of the key bits that may vary (the depth sort
// decides this on the device, before the step's host read): a pass whose 8-bit window
// holds none of them copies its input unchanged (same order, parity kept).
template <typename KT>
__global__ void __launch_bounds__(kSortThreads, HS_SORT_MINB) radix_onesweep_kernel(int64_t n, int shift,
                                                                      const KT *__restrict__ keys_in,
                                                                      const uint32_t *__restrict__ vals_in,
                                                                      KT *__restrict__ keys_out,
                                                                      uint32_t *__restrict__ vals_out,
                                                                      const uint32_t *__restrict__ digit_base,
                                                                      uint32_t *__restrict__ status,
                                                                      uint32_t *__restrict__ counter,
                                                                      const uint32_t *__restrict__ live_bits) {
    pdl_prologue();
    if (live_bits && ((depth_live_bits(live_bits) >> shift) & (kRadix - 1)) == 0u) {
        for (int64_t i = blockIdx.x * (int64_t)kSortTile + threadIdx.x; i < n && i < (blockIdx.x + 1) * (int64_t)kSortTile;
             i += kSortThreads) {
            keys_out[i] = keys_in[i];
            vals_out[i] = vals_in ? vals_in[i] : (uint32_t)i;
        }
        return;
    }
    __shared__ KT s_keys[kSortTile];
    __shared__ uint32_t s_vals[kSortTile];
    __shared__ uint32_t warp_hist[kSortThreads / 32][kRadix];
    __shared__ uint32_t digit_off[kRadix];
    __shared__ uint32_t glob[kRadix];
    __shared__ uint32_t warp_tot[8];
    __shared__ uint32_t s_tile;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(counter, 1u);          // tile ids in launch order
    for (int k = 0; k < kSortThreads / 32; ++k) warp_hist[k][tid] = 0;
    __syncthreads();
    const uint32_t tile = s_tile;
    const int64_t base = (int64_t)tile * kSortTile;

    KT k_reg[kSortItems];
    uint32_t v_reg[kSortItems];
    uint32_t local[kSortItems];
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
        const int64_t idx = base + w * (32 * kSortItems) + i * 32 + lane;
        const bool valid = idx < n;
        k_reg[i] = valid ? keys_in[idx] : (KT)0;
        v_reg[i] = valid ? (vals_in ? vals_in[idx] : (uint32_t)idx) : 0u;
    }
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
        const int64_t idx = base + w * (32 * kSortItems) + i * 32 + lane;
        const bool valid = idx < n;
        const uint32_t d = (uint32_t)(k_reg[i] >> shift) & (kRadix - 1);
        const uint32_t mask = __ballot_sync(0xffffffffu, valid);
        local[i] = 0;
        if (valid) {
            const uint32_t peers = __match_any_sync(mask, d);
            const uint32_t rank = __popc(peers & lt);
            const uint32_t cur = warp_hist[w][d];
            __syncwarp(mask);
            if (rank == 0) warp_hist[w][d] = cur + __popc(peers);
            __syncwarp(mask);
            local[i] = cur + rank;
        }
    }
    __syncthreads();
    // per digit (thread tid = digit): prefix over warps, CTA count, block-exclusive scan
    uint32_t cnt;
    {
        uint32_t run = 0;
#pragma unroll
        for (int k = 0; k < kSortThreads / 32; ++k) {
            const uint32_t t = warp_hist[k][tid];
            warp_hist[k][tid] = run;
            run += t;
        }
        cnt = run;
        uint32_t incl = run;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) warp_tot[w] = incl;
        __syncthreads();
        uint32_t wpre = 0;
        for (int k = 0; k < w; ++k) wpre += warp_tot[k];
        digit_off[tid] = wpre + incl - run;
    }
    // decoupled look-back for digit `tid`
    {
        uint32_t *st = status + (size_t)tile * kRadix + tid;
        uint32_t excl = 0;
        if (tile == 0) {
            st_relaxed(st, kFlagInc | cnt);
        } else {
            st_relaxed(st, kFlagAgg | cnt);
            // windowed look-back: kLookback predecessor words per round (independent
            // loads), consumed in order until an inclusive prefix is found
            int64_t j = (int64_t)tile - 1;
            bool found = false;
            while (!found) {
                uint32_t v[kLookback];
#pragma unroll
                for (int k = 0; k < kLookback; ++k)
                    v[k] = (j - k >= 0) ? ld_relaxed(status + (size_t)(j - k) * kRadix + tid) : kFlagInc;
#pragma unroll
                for (int k = 0; k < kLookback; ++k) {
                    if (found) break;
                    if (v[k] == 0u) break;          // not published yet: retry from this tile
                    excl += v[k] & kCountMask;
                    if (v[k] & kFlagInc) found = true;
                    --j;
                }
            }
            st_relaxed(st, kFlagInc | (excl + cnt));
        }
        glob[tid] = digit_base[tid] + excl;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
        const int64_t idx = base + w * (32 * kSortItems) + i * 32 + lane;
        if (idx < n) {
            const uint32_t d = (uint32_t)(k_reg[i] >> shift) & (kRadix - 1);
            const uint32_t p = digit_off[d] + warp_hist[w][d] + local[i];
            s_keys[p] = k_reg[i];
            s_vals[p] = v_reg[i];
        }
    }
    __syncthreads();
    const int cnt_tile = (int)min((int64_t)kSortTile, n - base);
    for (int j = tid; j < cnt_tile; j += kSortThreads) {
        const KT key = s_keys[j];
        const uint32_t d = (uint32_t)(key >> shift) & (kRadix - 1);
        const uint32_t p = glob[d] + (uint32_t)j - digit_off[d];
        keys_out[p] = key;
        vals_out[p] = s_vals[j];
    }
}

// ----------------------------------------------------------------- ranges

__global__ void tile_ranges_kernel(int64_t n, const uint64_t *__restrict__ keys, uint32_t *__restrict__ ranges) {
    pdl_prologue();
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t t = keys[i] >> 32;
    if (i == 0 || (keys[i - 1] >> 32) != t) ranges[2 * t] = (uint32_t)i;
    if (i == n - 1 || (keys[i + 1] >> 32) != t) ranges[2 * t + 1] = (uint32_t)(i + 1);
}

}  // namespace hs

using namespace hs;

extern "C" {

int hs_bin_scan(int num_blocks, const uint32_t *block_sums, uint32_t *block_offsets, const unsigned long long *err,
                const uint32_t *depth_range, unsigned long long *summary, void *stream) {
    launch_k(scan_kernel, 1, 1024, 0, HS_CHECK_STREAM(stream), num_blocks, block_sums, block_offsets, err, depth_range,
                                                         summary);
    return check_launch("hs_bin_scan");
}

int hs_bin_emit(int B, int64_t N, int width, int height, const float *records, const float *depth,
                const uint32_t *counts, const uint32_t *block_offsets, const uint32_t *tile_rects, uint64_t *keys,
                uint32_t *values, void *stream) {
    const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
    const int tile_bits = bit_length_u32((uint32_t)(tiles_x * tiles_y - 1));
    const int frame_bits = bit_length_u32((uint32_t)(B - 1));
    if (tile_bits + frame_bits > 32) {
        set_error("hs_bin_emit: frame/tile key bits %d + %d exceed 32", frame_bits, tile_bits);
        return HS_ERR_SHAPE;
    }
    const int64_t items = (int64_t)B * N;
    launch_k(emit_kernel, hs_scan_blocks(items), kScanBlock, 0, HS_CHECK_STREAM(stream), 
        B, N, tiles_x, tile_bits, records, depth, counts, block_offsets, tile_rects, keys, values);
    return check_launch("hs_bin_emit");
}

size_t hs_sort_workspace_size(int64_t num_keys) {
    const int64_t tiles = (num_keys + kSortTile - 1) / kSortTile;
    // digit bases [8][256] + status [8][tiles][256] + tile counters [8]
    return sizeof(uint32_t) * ((size_t)kMaxPasses * kRadix + (size_t)kMaxPasses * (size_t)(tiles > 0 ? tiles : 1) *
                               kRadix + kMaxPasses);
}

}  // extern "C"

template <typename KT>
static int sort_pairs_impl(const char *what, int64_t num_keys, uint64_t bit_mask, const KT *keys_in,
                           const uint32_t *values_in, KT *keys, uint32_t *values, KT *keys_alt,
                           uint32_t *values_alt, void *workspace,
                           size_t workspace_bytes, int *result_in_alt, const uint32_t *depth_range,
                           cudaStream_t s, int plain_below = 0) {
    if (result_in_alt) *result_in_alt = 0;
    if (num_keys <= 0) return HS_OK;
    if (workspace_bytes < hs_sort_workspace_size(num_keys)) {
        set_error("%s: workspace too small (%zu < %zu)", what, workspace_bytes, hs_sort_workspace_size(num_keys));
        return HS_ERR_SHAPE;
    }
    if (num_keys > (int64_t)kCountMask) {
        set_error("%s: too many keys", what);
        return HS_ERR_SHAPE;
    }
    PassShifts ps{};
    ps.plain_below = plain_below;
    for (int sh = 0; sh < (int)(8 * sizeof(KT)); sh += 8)
        if ((bit_mask >> sh) & 0xFFull) ps.shift[ps.n++] = sh;
    if (ps.n == 0) return HS_OK;
    const int tiles = (int)((num_keys + kSortTile - 1) / kSortTile);
    uint32_t *hist = reinterpret_cast<uint32_t *>(workspace);
    uint32_t *status = hist + (size_t)kMaxPasses * kRadix;
    uint32_t *counters = status + (size_t)kMaxPasses * tiles * kRadix;
    cudaMemsetAsync(workspace, 0,
                    sizeof(uint32_t) * ((size_t)kMaxPasses * kRadix + (size_t)ps.n * tiles * kRadix), s);
    cudaMemsetAsync(counters, 0, sizeof(uint32_t) * kMaxPasses, s);
    const int sms = current_sm_count();
#ifndef HS_HIST_CTAS_PER_SM
#define HS_HIST_CTAS_PER_SM 4
#endif
    const unsigned hgrid = (unsigned)std::min<int64_t>(grid_for(num_keys, 256 * 8), (int64_t)sms * HS_HIST_CTAS_PER_SM);
    launch_k(radix_hist_all_kernel<KT>, hgrid, 256, 0, s, num_keys, keys_in, ps, hist);
    launch_k(radix_digit_scan_kernel, 1, kRadix, 0, s, ps.n, hist);
    // pass 0 reads keys_in (values implicit when values_in is null), then ping-pong;
    // the caller passes (keys, values) as pass 0's source when they are the input
    const KT *ki = keys_in;
    const uint32_t *vi = values_in;
    KT *ko = keys_alt;
    uint32_t *vo = values_alt;
    int alt = 1;
    for (int p = 0; p < ps.n; ++p) {
        launch_k(radix_onesweep_kernel<KT>, tiles, kSortThreads, 0, s, num_keys, ps.shift[p], ki, vi, ko, vo,
                                                                 hist + (size_t)p * kRadix,
                                                                 status + (size_t)p * tiles * kRadix, counters + p,
                                                                 depth_range);
        ki = ko;
        vi = vo;
        ko = alt ? keys : keys_alt;
        vo = alt ? values : values_alt;
        alt ^= 1;
    }
    if (result_in_alt) *result_in_alt = alt ^ 1;
    return check_launch(what);
}

extern "C" {

int hs_sort_pairs(int64_t num_keys, uint64_t bit_mask, uint64_t *keys, uint32_t *values, uint64_t *keys_alt,
                  uint32_t *values_alt, void *workspace, size_t workspace_bytes, int *result_in_alt,
                  void *stream) {
    return sort_pairs_impl<uint64_t>("hs_sort_pairs", num_keys, bit_mask, keys, values, keys, values, keys_alt,
                                     values_alt, workspace, workspace_bytes, result_in_alt, nullptr,
                                     HS_CHECK_STREAM(stream));
}

int hs_sort_pairs32(int64_t num_keys, uint32_t bit_mask, uint32_t *keys, uint32_t *values, uint32_t *keys_alt,
                    uint32_t *values_alt, void *workspace, size_t workspace_bytes, int *result_in_alt,
                    void *stream) {
    return sort_pairs_impl<uint32_t>("hs_sort_pairs32", num_keys, bit_mask, keys, values, keys, values, keys_alt,
                                     values_alt, workspace, workspace_bytes, result_in_alt, nullptr,
                                     HS_CHECK_STREAM(stream), HS_TILE_PLAIN_BELOW);
}

int hs_depth_order(int64_t num_items, const float *depth, const uint32_t *depth_range, uint32_t *order,
                   uint32_t *order_alt, uint32_t *keys_a, uint32_t *keys_b, void *workspace, size_t workspace_bytes,
                   void *stream) {
    if (num_items <= 0) return HS_OK;
    // 4 passes over the depth bits; windows that the device-side depth range shows to be
    // constant copy through, so the result lands in `order` without a host read
    int alt = 0;
    const int rc = sort_pairs_impl<uint32_t>("hs_depth_order", num_items, 0xFFFFFFFFull,
                                             reinterpret_cast<const uint32_t *>(depth), nullptr, keys_b, order,
                                             keys_a, order_alt, workspace, workspace_bytes, &alt, depth_range,
                                             HS_CHECK_STREAM(stream), HS_HIST32_PLAIN_BELOW);
    if (rc == HS_OK && alt) {
        set_error("hs_depth_order: internal parity error");
        return HS_ERR_CUDA;
    }
    return rc;
}

int hs_bin_emit_sorted(int B, int64_t N, int width, int height, const float *records, const uint32_t *counts,
                       const uint32_t *tile_rects, const uint32_t *order, uint32_t *block_sums,
                       uint32_t *block_offsets, uint32_t *keys, uint32_t *values, void *stream) {
    const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
    const int tile_bits = bit_length_u32((uint32_t)(tiles_x * tiles_y - 1));
    const int frame_bits = bit_length_u32((uint32_t)(B - 1));
    if (tile_bits + frame_bits > 32) {
        set_error("hs_bin_emit_sorted: frame/tile key bits %d + %d exceed 32", frame_bits, tile_bits);
        return HS_ERR_SHAPE;
    }
    const int64_t items = (int64_t)B * N;
    const int nb = hs_scan_blocks(items);
    cudaStream_t s = HS_CHECK_STREAM(stream);
    launch_k(sorted_block_sums_kernel, nb, kScanBlock, 0, s, items, order, counts, block_sums);
    launch_k(scan_kernel, 1, 1024, 0, s, nb, block_sums, block_offsets, nullptr, nullptr, nullptr);
    launch_k(emit_sorted_kernel, nb, kScanBlock, 0, s, items, N, tiles_x, tile_bits, records, order, counts, block_offsets,
                                                 tile_rects, keys, values);
    return check_launch("hs_bin_emit_sorted");
}

int hs_tile_ranges32(int64_t num_keys, const uint32_t *keys, uint32_t *ranges, void *stream) {
    if (num_keys <= 0) return HS_OK;
    launch_k(tile_ranges32_kernel, grid_for(num_keys, 256), 256, 0, HS_CHECK_STREAM(stream), num_keys, keys, ranges);
    return check_launch("hs_tile_ranges32");
}

int hs_bin_stats(unsigned long long *host_out, int reset) {
#ifdef HS_BIN_STATS
    cudaMemcpyFromSymbol(host_out, g_bin_stats, sizeof(unsigned long long) * 2);
    if (reset) {
        const unsigned long long z[2] = {0, 0};
        cudaMemcpyToSymbol(g_bin_stats, z, sizeof(z));
    }
#else
    host_out[0] = host_out[1] = 0;
    (void)reset;
#endif
    return check_launch("hs_bin_stats");
}

int hs_tile_ranges(int64_t num_keys, const uint64_t *keys, uint32_t *ranges, void *stream) {
    if (num_keys <= 0) return HS_OK;
    launch_k(tile_ranges_kernel, grid_for(num_keys, 256), 256, 0, HS_CHECK_STREAM(stream), num_keys, keys, ranges);
    return check_launch("hs_tile_ranges");
}

}  // extern "C"
