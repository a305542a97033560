// hs_raster.cu -- tile rasterizer (forward + adjoint) on sm_100a.
//
// One warp (a one-warp CTA) per (frame, 16x16 tile, 8x8 pixel block): each lane
// holds two pixels of the block (rows r and r+4 of one column), so the per-splat
// overhead (list walk, shared loads, the warp reduction of the adjoint) is paid
// once per 64 pixels.  The four warps of a tile walk its depth-ordered key range
// independently, 32 splats per batch: each lane gathers one 48-byte record, pre-transforms it
// into a 64-byte staged form in the warp's private shared slot and votes whether
// the warp's 8x8 block can be touched at all: the splat's integer pixel bbox must
// admit a pixel of the block and its alpha >= 1/255 ellipse (q <= qmax) must reach
// the rectangle of those pixel centres (exact minimum of q over the rectangle,
// padded for rounding).  Skipping a block is exact: every pixel in it fails the
// reference's bbox or q test anyway.  Each CTA is a single warp, so there is no
// CTA barrier and blocks retire independently.
//
// Per pixel the math is the reference's front-to-back compositing
// (S/render.py:233-273): same bbox test, q / qmax and alpha >= 1/255 cutoffs, no
// alpha clamp, termination at T < 1e-14 with the stop index recorded for the
// adjoint.  Fused epilogue: background (:402), the L1 loss and its sign
// (S/metrics.py:10-22, :80-85, S/train.py:238-247), the black-background L1, and
// for colour init the per-(frame, Gaussian) max blend weight and Eq. 3 weight
// sums (S/render.py:339-377) reduced across the warp before one atomic per value.
//
// The adjoint (S/render.py:276-336) walks the same lists back to front per pixel
// with the suffix recurrence; each lane first adds its two pixels' contributions,
// then the 9 per-splat gradients are reduce-scattered across the warp (12 shuffles)
// before one RED per value.
#include <algorithm>

#include "hs_common.cuh"

namespace hs {

#ifndef HS_RASTER_PX
#define HS_RASTER_PX 2               // pixels per lane (a warp owns an 8 x 4*PX block)
#endif
#ifndef HS_RASTER_CTA_WARPS
#define HS_RASTER_CTA_WARPS 1        // warps per CTA (each warp owns one 8 x 4*PX block)
#endif
#ifndef HS_RASTER_MINB
#define HS_RASTER_MINB (56 / HS_RASTER_PX / HS_RASTER_CTA_WARPS)   // resident CTAs per SM (28 one-warp CTAs: 72 registers)
#endif

#ifndef HS_RASTER_EXACT_CULL
#define HS_RASTER_EXACT_CULL 1       // cull blocks with the exact ellipse-rectangle distance
#endif
#ifndef HS_RASTER_DIRECT
#define HS_RASTER_DIRECT 5           // adjoint: up to this many contributing lanes add directly
#endif

constexpr int kPX = HS_RASTER_PX;
constexpr int kCW = HS_RASTER_CTA_WARPS;

// Optional instrumentation (-DHS_RASTER_STATS): forward-pass counts of warp
// iterations and pixel tests, read with hs_raster_stats().
__device__ unsigned long long g_raster_stats[16];
constexpr int kBlocks = kTile * kTile / (32 * kPX);   // 8 x 4*PX pixel blocks per tile
constexpr int kRT = 32 * kCW;                          // threads per CTA
static_assert(kBlocks % kCW == 0, "CTA warps must divide the blocks of a tile");
constexpr unsigned kFull = 0xffffffffu;

struct RasterArgs {
    int B;
    int64_t N;
    int W, H, tiles_x, tile_bits;
    const float *records;
    const uint32_t *vals;
    const uint32_t *ranges;
    const float *bgs;
    const uint8_t *targets;
    const float *wsum_image;
    const uint8_t *visited;
    float *pix_T;
    uint32_t *pix_state;
    float *image;
    float *maxw;
    float *wsums;
    float *loss_partials;
    // backward
    const float *grad_image;
    float grad_scale;
    float *g_splat;
};

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(kFull, v, o));
    return v;
}

// ---- staged splat layout (shared memory, 64 B per splat) -------------------
//   p0: mx - 0.5, my - 0.5, k*a, 2k*b     with k = -0.5 log2(e), so that
//       e2 = k*q = dx (k a dx + 2k b dy) + k c dy^2 and alpha = op * 2^e2;
//       q <= qmax  <=>  e2 >= k*qmax  (k < 0)
//   p1: k*c, k*qmax, opacity, gidx | visited << 31   (gidx = frame * N + n)
//   p2: c_lo, c_hi, r_lo, r_hi  (the reference's pixel bbox, S/render.py:248-251)
//   p3: colour r, g, b, 0
// Forward and adjoint evaluate e2 / alpha with the same explicit-rounding
// expression, so both make identical pair decisions.
constexpr float kK = -0.72134752044448170f;      // -0.5 * log2(e)
constexpr float kMeanScale = -2.0f / kK;         // d q / d(k q) folded into g_mean
constexpr int kStageBytes = 64;

__device__ __forceinline__ float4 lds4(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}
__device__ __forceinline__ int4 lds4i(uint32_t addr) {
    int4 v;
    asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}
// 1/x for x in (0, 1] (x = 1 - alpha, alpha < 1): the MUFU reciprocal without the
// denormal-range fix-up __fdividef adds (same result for normal x)
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// 1 - alpha for the transmittance update, floored at 2^-24 (the spacing of fp32 below 1).
// The floor only changes alpha == 1.0f exactly: fp32 rounds sigmoid(logit) to 1 above
// logit ~16.6 and the Gaussian to 1 at a pixel within ~1e-3 px of the mean, where the
// reference's float64 alpha is still < 1 (its opacity saturates only near logit 36.7).
// Unfloored, T would become exactly 0 and the adjoint's t_rev / (1 - alpha) would be
// 0 * inf = NaN (S/render.py:318-319).  Forward and adjoint use the same floor, so
// t_rev * rcp(one_minus_alpha) still recovers the transmittance before the splat.
#ifndef HS_ONE_MINUS_FLOOR
#define HS_ONE_MINUS_FLOOR 5.9604644775390625e-8f               // 2^-24 (0: the unguarded A/B build)
#endif
constexpr float kOneMinusFloor = HS_ONE_MINUS_FLOOR;
__device__ __forceinline__ float one_minus_alpha(float alpha) { return fmaxf(1.0f - alpha, kOneMinusFloor); }

// e2 = k q(dx, dy) given kadx = k a dx; one rounding per operation
__device__ __forceinline__ float splat_e2(float dx, float dy, float kadx, float kb2, float kc) {
    return __fmaf_rn(__fmul_rn(kc, dy), dy, __fmul_rn(dx, __fmaf_rn(kb2, dy, kadx)));
}

// Pixels of lane l in block w of a tile: block w covers cols (w & 1) * 8 .. +7 and
// rows (w >> 1) * 4 kPX .. +4 kPX - 1; lane l holds column l & 7 and rows
// (l >> 3) + 4 p for p < kPX.
__device__ __forceinline__ void pixels_of(int w, int l, int tx, int ty, int &px, int &py0) {
    px = tx * kTile + (w & 1) * 8 + (l & 7);
    py0 = ty * kTile + (w >> 1) * 4 * kPX + (l >> 3);
}

// Stage one splat record into the lane's slot.  Returns bit 0: the warp's block
// [x0, x0+7] x [y0, y0+4 kPX-1] can hold a contributing pixel; bit 1: the splat's
// integer bbox covers the whole block (the per-pixel bbox test can be skipped);
// bit 2+p: row group p (every lane's p-th pixel) can hold one -- a group the splat
// cannot reach is skipped by the whole warp.
template <bool kCull = true>
__device__ __forceinline__ uint32_t stage_splat(const float *__restrict__ rec, uint32_t gflag, int x0, int y0,
                                            uint32_t saddr) {
    const float4 *r = reinterpret_cast<const float4 *>(rec);
    const float4 A = __ldg(r), Bv = __ldg(r + 1), Cv = __ldg(r + 2);
    const uint32_t rows = __float_as_uint(Bv.w), cols = __float_as_uint(Cv.x);
    const int rl = unpack_lo(rows), rh = unpack_hi(rows), cl = unpack_lo(cols), ch = unpack_hi(cols);
    const float a = A.z, b = A.w, c = Bv.x, qmax = Bv.z;
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(saddr), "f"(A.x - 0.5f), "f"(A.y - 0.5f),
                 "f"(kK * a), "f"(2.0f * kK * b));
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(saddr + 16), "f"(kK * c), "f"(kK * qmax),
                 "f"(Bv.y), "f"(__uint_as_float(gflag)));
    asm volatile("st.shared.v4.s32 [%0], {%1, %2, %3, %4};" ::"r"(saddr + 32), "r"(cl), "r"(ch), "r"(rl), "r"(rh));
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(saddr + 48), "f"(Cv.y), "f"(Cv.z), "f"(Cv.w),
                 "f"(0.f));
    if (!kCull) return 0u;
    if (!(qmax >= 0.f)) return 0u;
    // columns of the block the reference's bbox admits
    const int xs = max(x0, cl), xe = min(x0 + 7, ch);
    if (xs > xe) return 0u;
    const bool full = cl <= x0 && ch >= x0 + 7 && rl <= y0 && rh >= y0 + 4 * kPX - 1;
    const float det = a * c - b * b;
    const bool exact = HS_RASTER_EXACT_CULL && det > 0.f && a > 0.f && c > 0.f;
    const float dxlo = (float)xs + 0.5f - A.x, dxhi = (float)xe + 0.5f - A.x;
    const float dxv = fminf(fmaxf(0.f, dxlo), dxhi);
    const float dyv0 = __fdividef(-b * dxv, c);                 // (margin covers the approx.)
    uint32_t groups = 0u;
#pragma unroll
    for (int p = 0; p < kPX; ++p) {
        // row group p (the lanes' p-th pixels: rows y0 + 4p .. y0 + 4p + 3)
        const int ys = max(y0 + 4 * p, rl), ye = min(y0 + 4 * p + 3, rh);
        if (ys > ye) continue;
        bool hit = true;
        if (exact) {
            // minimum of q(d) = a dx^2 + 2b dx dy + c dy^2 over the rectangle spanned
            // by those pixel centres (d = centre - mean).  For a positive-definite q the
            // minimiser is the mean if it lies inside, else on a rectangle edge facing
            // it; the two candidate segments (x nearest the mean with the best y, and
            // vice versa) are both inside the rectangle, so their minimum is exact.
            const float dylo = (float)ys + 0.5f - A.y, dyhi = (float)ye + 0.5f - A.y;
            const float dyv = fminf(fmaxf(dyv0, dylo), dyhi);
            const float dyh = fminf(fmaxf(0.f, dylo), dyhi);
            const float dxh = fminf(fmaxf(__fdividef(-b * dyh, a), dxlo), dxhi);
            const float qv = a * dxv * dxv + 2.f * b * dxv * dyv + c * dyv * dyv;
            const float qh = a * dxh * dxh + 2.f * b * dxh * dyh + c * dyh * dyh;
            // margin for the fp32 rounding of this bound and of the per-pixel q
            hit = !(fminf(qv, qh) * 0.999f - 1e-3f > qmax);
        }
        if (hit) groups |= 4u << p;
    }
    if (!groups) return 0u;
    return 1u | ((uint32_t)full << 1) | groups;
}

// CI: 0 none, 1 max weight (all splats), 2 max weight + weight sums (all splats),
//     3 max weight + weight sums for splats whose Gaussian is not yet visited.
constexpr int kMaskBatches = 64;     // per-warp hit masks kept from the forward for the fused adjoint
constexpr int kMaskWords = 2 + kPX;  // per batch: hit, full-cover, one per row group

template <bool kExplicitGrad>
__device__ __forceinline__ void raster_bwd_loop(const RasterArgs &a, int b, int px, int py0, int x0, int y0,
                                                uint32_t start, uint32_t last, const float (&g)[kPX][3],
                                                float (&t_rev)[kPX], float (&suffix)[kPX], const uint32_t (&stop)[kPX],
                                                int lane, uint32_t wbase, const uint32_t *masks);

template <bool kLoss, bool kImage, int CI, bool kTrain = false>
__device__ __forceinline__ void raster_fwd_block(const RasterArgs &a, int b, int gw, int nblk, int lane,
                                                 uint32_t wbase, uint32_t *masks = nullptr) {
    // gw = tile * kBlocks + blk: the pixel block of frame b this warp composites
    const int tile = gw / kBlocks, blk = gw % kBlocks;
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    int px, py0;
    pixels_of(blk, lane, tx, ty, px, py0);
    const int x0 = tx * kTile + (blk & 1) * 8, y0 = ty * kTile + (blk >> 1) * 4 * kPX;
    const uint2 rg = reinterpret_cast<const uint2 *>(a.ranges)[((int64_t)b << a.tile_bits) + tile];
    const uint32_t start = rg.x, end = rg.y;
    const float bg[3] = {a.bgs[3 * b], a.bgs[3 * b + 1], a.bgs[3 * b + 2]};
    const float fpx = (float)px;

    // live state across the splat loop is kept small (T, C, stop, and the colour-init
    // source only when needed); the target is re-read in the epilogue
    float fpy[kPX], T[kPX], C[kPX][3], src[CI >= 2 ? kPX : 1][3];
    uint32_t stop[kPX];
    bool live[kPX];
#pragma unroll
    for (int p = 0; p < kPX; ++p) {
        const int py = py0 + 4 * p;
        const bool inside = px < a.W && py < a.H;
        fpy[p] = (float)py;
        T[p] = 1.0f;
        live[p] = inside;
        stop[p] = end - start;
#pragma unroll
        for (int c = 0; c < 3; ++c) C[p][c] = 0.f;
        if constexpr (CI >= 2) {
            const int64_t pix = ((int64_t)b * a.H + (inside ? py : 0)) * a.W + (inside ? px : 0);
#pragma unroll
            for (int c = 0; c < 3; ++c) src[p][c] = 0.f;
            if (inside && a.wsum_image) {
#pragma unroll
                for (int c = 0; c < 3; ++c) src[p][c] = a.wsum_image[pix * 3 + c];
            } else if (inside && a.targets) {
                const uchar4 t = reinterpret_cast<const uchar4 *>(a.targets)[pix];
                const float al = (float)t.w / 255.0f;
                const float rgb[3] = {(float)t.x / 255.0f, (float)t.y / 255.0f, (float)t.z / 255.0f};
#pragma unroll
                for (int c = 0; c < 3; ++c) src[p][c] = rgb[c] * al + (1.0f - al) * bg[c];
            }
        }
    }

#ifdef HS_RASTER_STATS
    unsigned long long st_iter = 0, st_test = 0, st_q = 0, st_c = 0, st_empty = 0, st_full = 0, st_batches = 0;
#endif
    for (uint32_t c0 = start; c0 < end; c0 += 32) {
        bool any_live = false;
#pragma unroll
        for (int p = 0; p < kPX; ++p) any_live = any_live || live[p];
        if (!__any_sync(kFull, any_live)) break;
        const uint32_t idx = c0 + lane;
        uint32_t code = 0u;
        bool want = false;
        if (idx < end) {
            const uint32_t n = a.vals[idx];
            const uint32_t gflag = (uint32_t)((int64_t)b * a.N + n);
            code = stage_splat(a.records + ((int64_t)b * a.N + n) * kRec, gflag, x0, y0, wbase + lane * kStageBytes);
            want = CI > 0 && (code & 1u) && (CI != 3 || !a.visited[n]);   // visited: no colour-init work
        }
        uint32_t bits = __ballot_sync(kFull, code & 1u);
        const uint32_t fullb = __ballot_sync(kFull, code & 2u);
        const uint32_t wantb = __ballot_sync(kFull, want);
        uint32_t grpb[kPX];
#pragma unroll
        for (int p = 0; p < kPX; ++p) grpb[p] = __ballot_sync(kFull, code & (4u << p));
        if (kTrain && lane == 0) {
            const uint32_t k = (c0 - start) >> 5;
            if (k < (uint32_t)kMaskBatches)
            {
                uint32_t *m = masks + k * kMaskWords;
                m[0] = bits;
                m[1] = fullb;
#pragma unroll
                for (int p = 0; p < kPX; ++p) m[2 + p] = grpb[p];
            }
        }
#ifdef HS_RASTER_STATS
        st_batches += lane == 0;
#endif
        __syncwarp();
        while (bits) {
            const int j = __ffs(bits) - 1;
            bits &= bits - 1u;
            const uint32_t ad = wbase + j * kStageBytes;
            const float4 p0 = lds4(ad), p1 = lds4(ad + 16), col = lds4(ad + 48);
            bool inb[kPX];
            if ((fullb >> j) & 1u) {                 // warp-uniform: bbox covers the block
#pragma unroll
                for (int p = 0; p < kPX; ++p) inb[p] = true;
            } else {
                const int4 bb = lds4i(ad + 32);
                const bool inx = px >= bb.x && px <= bb.y;
#pragma unroll
                for (int p = 0; p < kPX; ++p) inb[p] = inx && py0 + 4 * p >= bb.z && py0 + 4 * p <= bb.w;
            }
            const float dx = fpx - p0.x;
            const float kadx = __fmul_rn(p0.z, dx);
            float w[kPX];
#pragma unroll
            for (int p = 0; p < kPX; ++p) w[p] = 0.f;
#ifdef HS_RASTER_STATS
            st_iter += (lane == 0);
            st_full += (lane == 0) && ((fullb >> j) & 1u);
            bool anyq = false;
#endif
            // branch-free per pixel: alpha is evaluated for every slot and the
            // update predicated on the reference's tests (bbox, q <= qmax, cutoff)
#pragma unroll
            for (int p = 0; p < kPX; ++p) {
                if (!((grpb[p] >> j) & 1u)) continue;          // warp-uniform: group out of reach
                const float e2 = splat_e2(dx, fpy[p] - p0.y, kadx, p0.w, p1.x);
                const float alpha = __fmul_rn(p1.z, ex2_approx(e2));
                const bool ok = live[p] && inb[p] && e2 >= p1.y && alpha >= kAlphaCutoff;
#ifdef HS_RASTER_STATS
                st_test += live[p] && inb[p];
                st_q += live[p] && inb[p] && e2 >= p1.y;
                anyq = anyq || (live[p] && inb[p] && e2 >= p1.y);
                st_c += ok;
#endif
                if (ok) {
                    w[p] = alpha * T[p];
                    C[p][0] += w[p] * col.x;
                    C[p][1] += w[p] * col.y;
                    C[p][2] += w[p] * col.z;
                    T[p] = T[p] * one_minus_alpha(alpha);
                    if (T[p] < kTermEps) {
                        live[p] = false;
                        stop[p] = c0 - start + (uint32_t)j + 1u;
                    }
                }
            }
#ifdef HS_RASTER_STATS
            st_empty += !__any_sync(kFull, anyq) && lane == 0;
#endif
            if (CI > 0 && ((wantb >> j) & 1u)) {
                float wmax = 0.f;
#pragma unroll
                for (int p = 0; p < kPX; ++p) wmax = fmaxf(wmax, w[p]);
                if (__any_sync(kFull, wmax > 0.f)) {
                    const int64_t g = __float_as_uint(p1.w);
                    const float wm = warp_max(wmax);
                    if (CI >= 2) {
                        float v[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                        for (int p = 0; p < kPX; ++p) {
                            v[0] += w[p] * src[p][0];
                            v[1] += w[p] * src[p][1];
                            v[2] += w[p] * src[p][2];
                            v[3] += w[p];
                        }
                        int vi;
                        bool issue;
                        const float s = reduce_scatter(v, lane, vi, issue);
                        if (issue) atomicAdd(a.wsums + g * 4 + vi, s);
                    }
                    if (lane == 0) atomicMax(reinterpret_cast<int *>(a.maxw) + g, __float_as_int(wm));
                }
            }
        }
        __syncwarp();
    }

#ifdef HS_RASTER_STATS
    atomicAdd(&g_raster_stats[0], st_iter);
    atomicAdd(&g_raster_stats[1], st_test);
    atomicAdd(&g_raster_stats[2], st_q);
    atomicAdd(&g_raster_stats[3], st_c);
    atomicAdd(&g_raster_stats[4], st_empty);
    atomicAdd(&g_raster_stats[5], st_full);
    atomicAdd(&g_raster_stats[6], st_batches);
#endif
    float l1 = 0.f, black = 0.f;
    float g[kTrain ? kPX : 1][3];            // fused adjoint: the L1 gradient of each pixel
#pragma unroll
    for (int p = 0; p < kPX; ++p) {
        const int py = py0 + 4 * p;
        if (kTrain) {
#pragma unroll
            for (int c = 0; c < 3; ++c) g[p][c] = 0.f;
        }
        if (px >= a.W || py >= a.H) continue;
        const int64_t pix = ((int64_t)b * a.H + py) * a.W + px;
        float pred[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) pred[c] = C[p][c] + T[p] * bg[c];
        uint32_t signs = 0;
        if (kLoss) {
            const uchar4 t = reinterpret_cast<const uchar4 *>(a.targets)[pix];
            const float al = (float)t.w / 255.0f;
            const float rgb[3] = {(float)t.x / 255.0f, (float)t.y / 255.0f, (float)t.z / 255.0f};
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const float tgt = rgb[c] * al + (1.0f - al) * bg[c];
                const float d = pred[c] - tgt;
                l1 += fabsf(d);
                black += fabsf(C[p][c] - rgb[c] * al);
                signs |= (d > 0.f ? 1u : d < 0.f ? 2u : 0u) << (2 * c);
                if (kTrain) g[p][c] = d > 0.f ? a.grad_scale : d < 0.f ? -a.grad_scale : 0.f;
            }
        }
        if (!kTrain || a.pix_T) {
            a.pix_T[pix] = T[p];
            a.pix_state[pix] = stop[p] | (signs << 26);
        }
        if (kImage) {
#pragma unroll
            for (int c = 0; c < 3; ++c) a.image[pix * 3 + c] = pred[c];
        }
    }
    if (kLoss) {            // per-block partials: no CTA barrier, warps retire independently
        l1 = warp_sum(l1);
        black = warp_sum(black);
        if (lane == 0) {
            const int64_t o = ((int64_t)b * nblk + gw) * 2;
            a.loss_partials[o] = l1;
            a.loss_partials[o + 1] = black;
        }
    }
    if constexpr (kTrain) {
        // the adjoint of this block right away: T, stop and the loss gradient are in
        // registers and the forward's hit masks are in shared memory
        if (start >= end) return;
        float t_rev[kPX], suffix[kPX];
        uint32_t smax = 0;
#pragma unroll
        for (int p = 0; p < kPX; ++p) {
            const bool inside = px < a.W && py0 + 4 * p < a.H;
            if (!inside) stop[p] = 0;
            t_rev[p] = inside ? T[p] : 0.f;
            suffix[p] = inside ? T[p] * (g[p][0] * bg[0] + g[p][1] * bg[1] + g[p][2] * bg[2]) : 0.f;
            smax = max(smax, stop[p]);
        }
        const uint32_t last = start + __reduce_max_sync(kFull, smax);
        __syncwarp();
        raster_bwd_loop<false>(a, b, px, py0, x0, y0, start, last, g, t_rev, suffix, stop, lane, wbase, masks);
    }
}

// Work distribution (HS_RASTER_PERSIST, default): a persistent grid of resident
// one-warp CTAs where every warp pulls (frame, block) items from a global counter
// (frame-major, tile order), so short and long blocks mix freely and no CTA launch
// happens per block (-8 % raster time vs one CTA per block).  The last warp to
// finish resets the counters for the next launch, so raster launches of one process
// must not run concurrently on different streams (hs_api.h).  HS_RASTER_PERSIST=0:
// one CTA per block.
#ifndef HS_RASTER_PERSIST
#define HS_RASTER_PERSIST 1
#endif
__device__ unsigned int g_raster_work[6];   // [fwd next, done, bwd next, done, train next, done]

// Longest-first item order (HS_RASTER_LPT): tiles bucketed by the bit length of their
// key count, heaviest bucket first, so the long tiles start early and the persistent
// grid's tail is made of short items.  One small CTA per launch builds it.
#ifndef HS_RASTER_LPT
#define HS_RASTER_LPT 1
#endif
#ifndef HS_RASTER_LPT_SUB
#define HS_RASTER_LPT_SUB 2
#endif
constexpr int kMaxOrder = 1 << 20;
__device__ uint32_t g_tile_order[kMaxOrder];

__global__ void __launch_bounds__(1024) tile_order_kernel(int total_tiles, int tile_bits, int tiles,
                                                          const uint32_t *__restrict__ ranges) {
    constexpr int kSub = HS_RASTER_LPT_SUB;         // sub-buckets per octave
    constexpr int kNB = 33 << kSub;
    __shared__ uint32_t hist[kNB], cursor[kNB];
    for (int i = threadIdx.x; i < kNB; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    auto bucket = [&](int t) {
        const int b = t / tiles, tile = t % tiles;
        const uint2 rg = reinterpret_cast<const uint2 *>(ranges)[((int64_t)b << tile_bits) + tile];
        const uint32_t len = rg.y - rg.x;
        const int bl = 32 - __clz(len);            // 0 (empty) .. 32
        const uint32_t sub = bl > kSub ? (len >> (bl - 1 - kSub)) & ((1u << kSub) - 1u) : 0u;
        return (bl << kSub) | (int)sub;            // log-linear: heavier = larger
    };
    for (int t = threadIdx.x; t < total_tiles; t += blockDim.x) atomicAdd(&hist[bucket(t)], 1u);
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t run = 0;
        for (int k = kNB - 1; k >= 0; --k) {
            cursor[k] = run;
            run += hist[k];
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < total_tiles; t += blockDim.x) g_tile_order[atomicAdd(&cursor[bucket(t)], 1u)] = t;
}

template <typename F>
__device__ __forceinline__ void for_each_block(int B, int nblk, int lane, int warp, unsigned int *work, F &&fn) {
    if (!HS_RASTER_PERSIST) {
        fn((int)blockIdx.y, (int)blockIdx.x * kCW + warp);
        return;
    }
    const int total = B * nblk;
    const bool lpt = HS_RASTER_LPT && total / kBlocks <= kMaxOrder;
    const int tiles = nblk / kBlocks;
    for (;;) {
        int item = 0;
        if (lane == 0) item = (int)atomicAdd(work, 1u);
        item = __shfl_sync(kFull, item, 0);
        if (item >= total) break;
        if (lpt) {
            const uint32_t bt = g_tile_order[item / kBlocks];
            fn((int)(bt / tiles), (int)(bt % tiles) * kBlocks + item % kBlocks);
        } else {
            fn(item / nblk, item % nblk);
        }
        __syncwarp();
    }
    if (lane == 0) {
        const unsigned int warps = gridDim.x * gridDim.y * kCW;
        if (atomicAdd(work + 1, 1u) == warps - 1) {
            work[0] = 0u;
            work[1] = 0u;
        }
    }
}

template <bool kLoss, bool kImage, int CI>
__global__ void __launch_bounds__(kRT, HS_RASTER_MINB) raster_fwd_kernel(RasterArgs a, int nblk) {
    __shared__ __align__(16) unsigned char s_stage[kRT * kStageBytes];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t wbase = (uint32_t)__cvta_generic_to_shared(s_stage) + warp * 32 * kStageBytes;
    for_each_block(a.B, nblk, lane, warp, g_raster_work,
                   [&](int b, int gw) { raster_fwd_block<kLoss, kImage, CI>(a, b, gw, nblk, lane, wbase); });
}

template <bool kExplicitGrad>
__device__ __forceinline__ void raster_bwd_block(const RasterArgs &a, int b, int gw, int lane, uint32_t wbase) {
    const int tile = gw / kBlocks, blk = gw % kBlocks;
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    int px, py0;
    pixels_of(blk, lane, tx, ty, px, py0);
    const int x0 = tx * kTile + (blk & 1) * 8, y0 = ty * kTile + (blk >> 1) * 4 * kPX;
    const uint2 rg = reinterpret_cast<const uint2 *>(a.ranges)[((int64_t)b << a.tile_bits) + tile];
    const uint32_t start = rg.x, end = rg.y;
    if (start >= end) return;
    const float bg[3] = {a.bgs[3 * b], a.bgs[3 * b + 1], a.bgs[3 * b + 2]};

    float g[kPX][3], t_rev[kPX], suffix[kPX];
    uint32_t stop[kPX];
#pragma unroll
    for (int p = 0; p < kPX; ++p) {
        const int py = py0 + 4 * p;
        const bool inside = px < a.W && py < a.H;
        const int64_t pix = ((int64_t)b * a.H + (inside ? py : 0)) * a.W + (inside ? px : 0);
        g[p][0] = g[p][1] = g[p][2] = 0.f;
        stop[p] = 0;
        t_rev[p] = 0.f;
        suffix[p] = 0.f;
        if (inside) {
            const uint32_t st = a.pix_state[pix];
            stop[p] = st & kStopMask;
            const float Tf = a.pix_T[pix];
            if (kExplicitGrad) {
#pragma unroll
                for (int c = 0; c < 3; ++c) g[p][c] = a.grad_image[pix * 3 + c];
            } else {
                const uint32_t sg = st >> 26;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const uint32_t s2 = (sg >> (2 * c)) & 3u;
                    g[p][c] = s2 == 1u ? a.grad_scale : s2 == 2u ? -a.grad_scale : 0.f;
                }
            }
            t_rev[p] = Tf;
            suffix[p] = Tf * (g[p][0] * bg[0] + g[p][1] * bg[1] + g[p][2] * bg[2]);
        }
    }
    // this warp only needs the list up to its pixels' largest stop index
    uint32_t smax = 0;
#pragma unroll
    for (int p = 0; p < kPX; ++p) smax = max(smax, stop[p]);
    const uint32_t last = start + __reduce_max_sync(kFull, smax);
    raster_bwd_loop<kExplicitGrad>(a, b, px, py0, x0, y0, start, last, g, t_rev, suffix, stop, lane, wbase, nullptr);
}

// Back-to-front walk of [start, last) in the forward's 32-key batches.  With the
// forward's hit masks (fused kernel) a batch is staged only by its hit lanes and
// skipped when empty; otherwise each batch is staged and culled again.
template <bool kExplicitGrad>
__device__ __forceinline__ void raster_bwd_loop(const RasterArgs &a, int b, int px, int py0, int x0, int y0,
                                                uint32_t start, uint32_t last, const float (&g)[kPX][3],
                                                float (&t_rev)[kPX], float (&suffix)[kPX], const uint32_t (&stop)[kPX],
                                                int lane, uint32_t wbase, const uint32_t *masks) {
    const float fpx = (float)px;
    int py[kPX];
    float fpy[kPX];
#pragma unroll
    for (int p = 0; p < kPX; ++p) {
        py[p] = py0 + 4 * p;
        fpy[p] = (float)py[p];
    }
    if (last <= start) return;
    for (int k = (int)((last - 1 - start) >> 5); k >= 0; --k) {
        const uint32_t c0 = start + 32u * (uint32_t)k;
        const uint32_t c_end = min(c0 + 32u, last);
        const uint32_t live_lanes = c_end - c0 >= 32u ? kFull : (1u << (c_end - c0)) - 1u;
        uint32_t bits, fullb, grpb[kPX];
        const uint32_t idx = c0 + lane;
        if (masks != nullptr && k < kMaskBatches) {
            const uint32_t *m = masks + k * kMaskWords;
            bits = m[0] & live_lanes;
            fullb = m[1];
#pragma unroll
            for (int p = 0; p < kPX; ++p) grpb[p] = m[2 + p];
            if (bits == 0u) continue;                      // warp-uniform
            if ((bits >> lane) & 1u) {
                const uint32_t n = a.vals[idx];
                stage_splat<false>(a.records + ((int64_t)b * a.N + n) * kRec, (uint32_t)((int64_t)b * a.N + n), x0,
                                   y0, wbase + lane * kStageBytes);
            }
        } else {
            uint32_t code = 0u;
            if (idx < c_end) {
                const uint32_t n = a.vals[idx];
                code = stage_splat(a.records + ((int64_t)b * a.N + n) * kRec, (uint32_t)((int64_t)b * a.N + n), x0,
                                   y0, wbase + lane * kStageBytes);
            }
            bits = __ballot_sync(kFull, code & 1u);
            fullb = __ballot_sync(kFull, code & 2u);
#pragma unroll
            for (int p = 0; p < kPX; ++p) grpb[p] = __ballot_sync(kFull, code & (4u << p));
        }
        __syncwarp();
        while (bits) {
            const int j = 31 - __clz(bits);
            bits &= ~(1u << j);
            const uint32_t jl = c0 - start + (uint32_t)j;
            const uint32_t ad = wbase + j * kStageBytes;
            const float4 p0 = lds4(ad), p1 = lds4(ad + 16), col = lds4(ad + 48);
            bool inb[kPX];
            if ((fullb >> j) & 1u) {                 // warp-uniform: bbox covers the block
#pragma unroll
                for (int p = 0; p < kPX; ++p) inb[p] = true;
            } else {
                const int4 bb = lds4i(ad + 32);
                const bool inx = px >= bb.x && px <= bb.y;
#pragma unroll
                for (int p = 0; p < kPX; ++p) inb[p] = inx && py[p] >= bb.z && py[p] <= bb.w;
            }
            const float dx = fpx - p0.x;
            const float kadx = __fmul_rn(p0.z, dx);
            const float hb2 = 0.5f * p0.w;
            float gv[9];
#pragma unroll
            for (int k = 0; k < 9; ++k) gv[k] = 0.f;
            bool contrib = false;
            // branch-free per pixel: a slot failing the reference's tests runs the same
            // instructions with alpha = G = 0, which leaves t_rev and suffix unchanged
            // (1 / (1 - 0) == 1 exactly) and adds zeros to the gradients
#pragma unroll
            for (int p = 0; p < kPX; ++p) {
                if (!((grpb[p] >> j) & 1u)) continue;          // warp-uniform: group out of reach
                const float dy = fpy[p] - p0.y;
                const float e2 = splat_e2(dx, dy, kadx, p0.w, p1.x);
                const float G0 = ex2_approx(e2);
                const float alpha0 = __fmul_rn(p1.z, G0);
                const bool ok = jl < stop[p] && inb[p] && e2 >= p1.y && alpha0 >= kAlphaCutoff;
                contrib = contrib || ok;
                const float G = ok ? G0 : 0.f, alpha = ok ? alpha0 : 0.f;
                const float inv = rcp_approx(one_minus_alpha(alpha));
                const float t_prior = t_rev[p] * inv;
                const float gw = g[p][0] * col.x + g[p][1] * col.y + g[p][2] * col.z;
                const float wgt = alpha * t_prior;
                gv[6] += wgt * g[p][0];
                gv[7] += wgt * g[p][1];
                gv[8] += wgt * g[p][2];
                const float d_alpha = t_prior * gw - suffix[p] * inv;
                gv[5] += G * d_alpha;
                // dq = -0.5 alpha d_alpha; the constant factors are applied once per
                // reduced value (kGradScale) instead of per pixel
                const float dq = alpha * d_alpha;
                const float dqx = dq * dx, dqy = dq * dy;
                gv[2] += dqx * dx;
                gv[3] += dqx * dy;
                gv[4] += dqy * dy;
                // -2 dq (a dx + b dy) with the k-scaled conic: (-2/k) dq (ka dx + kb dy)
                gv[0] += p0.z * dqx + hb2 * dqy;
                gv[1] += hb2 * dqx + p1.x * dqy;
                suffix[p] += wgt * gw;
                t_rev[p] = t_prior;
            }
#ifdef HS_RASTER_STATS
            {
                const int nc = __popc(__ballot_sync(kFull, contrib));
                if (lane == 0) {
                    const int bin = nc == 0 ? 0 : nc == 1 ? 1 : nc == 2 ? 2 : nc <= 4 ? 3 : nc <= 8 ? 4 : nc <= 16 ? 5 : 6;
                    atomicAdd(&g_raster_stats[8 + bin], 1ull);
                }
            }
#endif
            const uint32_t cmask = __ballot_sync(kFull, contrib);
            if (HS_RASTER_DIRECT && cmask && __popc(cmask) <= HS_RASTER_DIRECT) {
                // few contributing pixels: their lanes add directly (9 atomics each) instead
                // of the 9-value warp reduce-scatter
                if (contrib) {
                    float *gp = a.g_splat + (uint64_t)(__float_as_uint(p1.w)) * kGS;
#pragma unroll
                    for (int k = 0; k < 9; ++k) {
                        const float sc = k < 2 ? -0.5f * kMeanScale : k == 3 ? -1.0f : k < 5 ? -0.5f : 1.0f;
                        atomicAdd(gp + k, gv[k] * sc);
                    }
                }
            } else if (cmask) {
                int vi;
                bool issue;
                const float s = reduce_scatter(gv, lane, vi, issue);
                const float sc = vi < 2 ? -0.5f * kMeanScale : vi == 3 ? -1.0f : vi < 5 ? -0.5f : 1.0f;
                if (issue) atomicAdd(a.g_splat + (uint64_t)(__float_as_uint(p1.w)) * kGS + vi, s * sc);
            }
        }
        __syncwarp();
    }
}


// Training step: forward (L1 loss, colour-init sums) and adjoint of each pixel block in
// one pass -- no per-pixel state round trip through HBM, and the adjoint reuses the
// forward's per-batch hit masks.
template <int CI>
__global__ void __launch_bounds__(kRT, HS_RASTER_MINB) raster_train_kernel(RasterArgs a, int nblk) {
    __shared__ __align__(16) unsigned char s_stage[kRT * kStageBytes];
    __shared__ uint32_t s_masks[kCW][kMaskBatches * kMaskWords];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t wbase = (uint32_t)__cvta_generic_to_shared(s_stage) + warp * 32 * kStageBytes;
    for_each_block(a.B, nblk, lane, warp, g_raster_work + 4, [&](int b, int gw) {
        raster_fwd_block<true, false, CI, true>(a, b, gw, nblk, lane, wbase, s_masks[warp]);
    });
}

template <bool kExplicitGrad>
__global__ void __launch_bounds__(kRT, HS_RASTER_MINB) raster_bwd_kernel(RasterArgs a, int nblk) {
    __shared__ __align__(16) unsigned char s_stage[kRT * kStageBytes];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t wbase = (uint32_t)__cvta_generic_to_shared(s_stage) + warp * 32 * kStageBytes;
    for_each_block(a.B, nblk, lane, warp, g_raster_work + 2,
                   [&](int b, int gw) { raster_bwd_block<kExplicitGrad>(a, b, gw, lane, wbase); });
}

// partials[b][tiles * kBlocks][2] (one pair per pixel block)
__global__ void loss_reduce_kernel(int B, int tiles, float inv_count, const float *__restrict__ partials,
                                   float *__restrict__ out) {
    __shared__ float red[2][32];
    const int b = blockIdx.x, tid = threadIdx.x;
    float s0 = 0.f, s1 = 0.f;
    for (int t = tid; t < tiles; t += blockDim.x) {
        s0 += partials[((int64_t)b * tiles + t) * 2];
        s1 += partials[((int64_t)b * tiles + t) * 2 + 1];
    }
    s0 = warp_sum(s0);
    s1 = warp_sum(s1);
    if ((tid & 31) == 0) { red[0][tid >> 5] = s0; red[1][tid >> 5] = s1; }
    __syncthreads();
    if (tid == 0) {
        float a0 = 0.f, a1 = 0.f;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) { a0 += red[0][i]; a1 += red[1][i]; }
        out[b] = a0 * inv_count;
        out[B + b] = a1 * inv_count;
    }
}

__global__ void loss_mean_kernel(int B, float *__restrict__ out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        float s = 0.f;
        for (int b = 0; b < B; ++b) s += out[b];
        out[2 * B] = s / (float)B;
    }
}

static RasterArgs make_args(int B, int64_t N, int W, int H, const float *records, const uint32_t *values,
                            const uint32_t *ranges, int tile_bits, const float *bgs) {
    RasterArgs a{};
    a.B = B;
    a.N = N;
    a.W = W;
    a.H = H;
    a.tiles_x = (W + kTile - 1) / kTile;
    a.tile_bits = tile_bits;
    a.records = records;
    a.vals = values;
    a.ranges = ranges;
    a.bgs = bgs;
    return a;
}

template <bool L, bool I>
static void launch_fwd_ci(int ci, dim3 grid, int nblk, cudaStream_t s, const RasterArgs &a) {
    switch (ci) {
        case 0: raster_fwd_kernel<L, I, 0><<<grid, kRT, 0, s>>>(a, nblk); break;
        case 1: raster_fwd_kernel<L, I, 1><<<grid, kRT, 0, s>>>(a, nblk); break;
        case 2: raster_fwd_kernel<L, I, 2><<<grid, kRT, 0, s>>>(a, nblk); break;
        default: raster_fwd_kernel<L, I, 3><<<grid, kRT, 0, s>>>(a, nblk); break;
    }
}

// grid of the raster kernels: one CTA per kCW blocks, or a persistent grid of
// resident CTAs (HS_RASTER_PERSIST)
static void launch_tile_order(int B, int nblk, int tile_bits, const uint32_t *ranges, cudaStream_t s) {
    const int tiles = nblk / kBlocks;
    if (HS_RASTER_PERSIST && HS_RASTER_LPT && B * tiles <= kMaxOrder)
        tile_order_kernel<<<1, 1024, 0, s>>>(B * tiles, tile_bits, tiles, ranges);
}

static dim3 raster_grid(int nblk, int B) {
    if (!HS_RASTER_PERSIST) return dim3(nblk / kCW, B);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int64_t want = (int64_t)sms * HS_RASTER_MINB, items = (int64_t)nblk * B / kCW;
    return dim3((unsigned)std::max<int64_t>(1, std::min(want, items)), 1);
}

}  // namespace hs

using namespace hs;

extern "C" {

int hs_raster_tile_order(int B, int width, int height, const uint32_t *ranges, int tile_bits, void *stream) {
    const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
    launch_tile_order(B, tiles_x * tiles_y * kBlocks, tile_bits, ranges, HS_CHECK_STREAM(stream));
    return check_launch("hs_raster_tile_order");
}

int hs_raster_fwd(int B, int64_t N, int width, int height, int flags, const float *records, const uint32_t *values,
                  const uint32_t *ranges, int tile_bits, const float *backgrounds, const uint8_t *targets,
                  const float *wsum_image, const uint8_t *visited, float *pix_T, uint32_t *pix_state, float *image,
                  float *maxw, float *wsums, float *loss_partials, void *stream) {
    const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
    const bool loss = flags & HS_RASTER_LOSS, img = flags & HS_RASTER_IMAGE;
    int ci = 0;
    if (flags & HS_RASTER_MAXW_UNVISITED) ci = 3;
    else if ((flags & HS_RASTER_MAXW_ALL) && (flags & HS_RASTER_WSUMS)) ci = 2;
    else if (flags & HS_RASTER_MAXW_ALL) ci = 1;
    if ((loss && !targets) || (img && !image) || (ci && !maxw) || (ci >= 2 && !wsums) || (ci == 3 && !visited) ||
        (ci >= 2 && !targets && !wsum_image) || (loss && !loss_partials)) {
        set_error("hs_raster_fwd: flags 0x%x need a buffer that is NULL", flags);
        return HS_ERR_SHAPE;
    }
    RasterArgs a = make_args(B, N, width, height, records, values, ranges, tile_bits, backgrounds);
    a.targets = targets;
    a.wsum_image = (flags & HS_RASTER_WSUMS_IMAGE) ? wsum_image : nullptr;
    a.visited = visited;
    a.pix_T = pix_T;
    a.pix_state = pix_state;
    a.image = image;
    a.maxw = maxw;
    a.wsums = wsums;
    a.loss_partials = loss_partials;
    const int nblk = tiles_x * tiles_y * kBlocks;
    const dim3 grid = raster_grid(nblk, B);
    cudaStream_t s = HS_CHECK_STREAM(stream);
    if (!(flags & HS_RASTER_ORDER_READY)) launch_tile_order(B, nblk, tile_bits, ranges, s);
    if (loss && img) launch_fwd_ci<true, true>(ci, grid, nblk, s, a);
    else if (loss) launch_fwd_ci<true, false>(ci, grid, nblk, s, a);
    else if (img) launch_fwd_ci<false, true>(ci, grid, nblk, s, a);
    else launch_fwd_ci<false, false>(ci, grid, nblk, s, a);
    return check_launch("hs_raster_fwd");
}

int hs_raster_bwd(int B, int64_t N, int width, int height, const float *records, const uint32_t *values,
                  const uint32_t *ranges, int tile_bits, const float *backgrounds, const float *pix_T,
                  const uint32_t *pix_state, const float *grad_image, float grad_scale, float *g_splat,
                  void *stream) {
    const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
    RasterArgs a = make_args(B, N, width, height, records, values, ranges, tile_bits, backgrounds);
    a.pix_T = const_cast<float *>(pix_T);
    a.pix_state = const_cast<uint32_t *>(pix_state);
    a.grad_image = grad_image;
    a.grad_scale = grad_scale;
    a.g_splat = g_splat;
    const int nblk = tiles_x * tiles_y * kBlocks;
    const dim3 grid = raster_grid(nblk, B);
    cudaStream_t s = HS_CHECK_STREAM(stream);
    launch_tile_order(B, nblk, tile_bits, ranges, s);
    if (grad_image) raster_bwd_kernel<true><<<grid, kRT, 0, s>>>(a, nblk);
    else raster_bwd_kernel<false><<<grid, kRT, 0, s>>>(a, nblk);
    return check_launch("hs_raster_bwd");
}

int hs_raster_train(int B, int64_t N, int width, int height, int flags, const float *records, const uint32_t *values,
                    const uint32_t *ranges, int tile_bits, const float *backgrounds, const uint8_t *targets,
                    const uint8_t *visited, float *maxw, float *wsums, float *loss_partials, float grad_scale,
                    float *g_splat, float *pix_T, uint32_t *pix_state, void *stream) {
    const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
    int ci = 0;
    if (flags & HS_RASTER_MAXW_UNVISITED) ci = 3;
    else if ((flags & HS_RASTER_MAXW_ALL) && (flags & HS_RASTER_WSUMS)) ci = 2;
    else if (flags & HS_RASTER_MAXW_ALL) ci = 1;
    if (!targets || !loss_partials || !g_splat || (ci && !maxw) || (ci >= 2 && !wsums) || (ci == 3 && !visited) ||
        (flags & (HS_RASTER_IMAGE | HS_RASTER_WSUMS_IMAGE)) || (!pix_T != !pix_state)) {
        set_error("hs_raster_train: flags 0x%x / buffers not supported (needs targets, loss_partials, g_splat)", flags);
        return HS_ERR_SHAPE;
    }
    RasterArgs a = make_args(B, N, width, height, records, values, ranges, tile_bits, backgrounds);
    a.targets = targets;
    a.visited = visited;
    a.maxw = maxw;
    a.wsums = wsums;
    a.loss_partials = loss_partials;
    a.grad_scale = grad_scale;
    a.g_splat = g_splat;
    a.pix_T = pix_T;
    a.pix_state = pix_state;
    const int nblk = tiles_x * tiles_y * kBlocks;
    const dim3 grid = raster_grid(nblk, B);
    cudaStream_t s = HS_CHECK_STREAM(stream);
    if (!(flags & HS_RASTER_ORDER_READY)) launch_tile_order(B, nblk, tile_bits, ranges, s);
    switch (ci) {
        case 0: raster_train_kernel<0><<<grid, kRT, 0, s>>>(a, nblk); break;
        case 1: raster_train_kernel<1><<<grid, kRT, 0, s>>>(a, nblk); break;
        case 2: raster_train_kernel<2><<<grid, kRT, 0, s>>>(a, nblk); break;
        default: raster_train_kernel<3><<<grid, kRT, 0, s>>>(a, nblk); break;
    }
    return check_launch("hs_raster_train");
}

int hs_raster_stats(unsigned long long *host_out, int reset) {
    cudaMemcpyFromSymbol(host_out, g_raster_stats, sizeof(unsigned long long) * 16);
    if (reset) {
        const unsigned long long z[16] = {};
        cudaMemcpyToSymbol(g_raster_stats, z, sizeof(z));
    }
    return check_launch("hs_raster_stats");
}

int hs_loss_reduce(int B, int num_tiles, int width, int height, const float *loss_partials, float *loss_out,
                   void *stream) {
    cudaStream_t s = HS_CHECK_STREAM(stream);
    const float inv = (float)(1.0 / ((double)width * height * 3.0));
    static_assert(HS_LOSS_PARTIALS_PER_TILE >= 2 * kBlocks, "hs_api.h partial count");
    loss_reduce_kernel<<<B, 256, 0, s>>>(B, num_tiles * kBlocks, inv, loss_partials, loss_out);
    loss_mean_kernel<<<1, 32, 0, s>>>(B, loss_out);
    return check_launch("hs_loss_reduce");
}

}  // extern "C"
