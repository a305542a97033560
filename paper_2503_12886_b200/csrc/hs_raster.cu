// hs_raster.cu -- tile rasterizer (forward + adjoint) on sm_100a.
//
// One 256-thread CTA per (frame, 16x16 tile); one pixel per thread; each warp
// owns an 8x4 pixel block of the tile.  The frame's depth-sorted key range for
// the tile is walked in chunks of 256 splat records staged in shared memory (one
// coalesced gather per chunk).  While staging, the loading thread also computes
// which of the 8 warp blocks the splat can touch at all -- the intersection of
// its integer pixel bbox with the exact extent of its alpha >= 1/255 ellipse
// (q <= qmax), padded for rounding -- and each warp then iterates only over its
// own splats (ballot-compacted bit lists).  Skipping a warp is exact: every pixel
// of a skipped block fails the reference's bbox or q test anyway.
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
// with the suffix recurrence and reduces the 9 per-splat gradients across the
// warp with a reduce-scatter (12 shuffles instead of 45) before the atomics.
#include "hs_common.cuh"

namespace hs {

#ifndef HS_RASTER_MINB
#define HS_RASTER_MINB 4             // resident CTAs per SM the register budget must allow
#endif

constexpr int kRT = kTile * kTile;   // 256 pixels / threads per CTA
constexpr int kWarps = kRT / 32;     // 8 warps, each an 8x4 pixel block
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

// Pixel of thread `tid` in the tile: warp w covers cols (w & 1) * 8 .. +7 and
// rows (w >> 1) * 4 .. +3; lane l is (col l & 7, row l >> 3) of that block.
__device__ __forceinline__ void pixel_of(int tid, int tx, int ty, int &px, int &py) {
    const int w = tid >> 5, l = tid & 31;
    px = tx * kTile + (w & 1) * 8 + (l & 7);
    py = ty * kTile + (w >> 1) * 4 + (l >> 3);
}

// ---- staged splat layout (shared memory, 64 B per splat) -------------------
//   p0: mx - 0.5, my - 0.5, k*a, 2k*b     with k = -0.5 log2(e), so that
//       e2 = k*q = dx (k a dx + 2k b dy) + k c dy^2 and alpha = op * 2^e2;
//       q <= qmax  <=>  e2 >= k*qmax  (k < 0)
//   p1: k*c, k*qmax, opacity, gidx | visited << 31   (gidx = frame * N + n)
//   p2: c_lo, c_hi, r_lo, r_hi  (the reference's pixel bbox, S/render.py:248-251)
//   p3: colour r, g, b, 0
// Forward and adjoint evaluate e2 / alpha through the same explicit-rounding
// helpers, so both make identical pair decisions.
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
__device__ __forceinline__ uint32_t lds1(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// e2 = k q(dx, dy), one rounding per operation (no contraction differences between kernels)
__device__ __forceinline__ float splat_e2(float dx, float dy, float ka, float kb2, float kc) {
    const float t = __fmaf_rn(kb2, dy, __fmul_rn(ka, dx));
    return __fmaf_rn(__fmul_rn(kc, dy), dy, __fmul_rn(dx, t));
}

// Stage one splat record into shared memory and return its 8-bit warp-block mask:
// warp w's 8x4 block can hold a contributing pixel only if it intersects the
// integer bbox AND the extent of the q <= qmax ellipse (padded for rounding).
__device__ __forceinline__ uint32_t stage_splat(const float *__restrict__ rec, uint32_t gflag, int tx, int ty,
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
    if (qmax < 0.f) return 0u;
    int r0 = rl, r1 = rh, c0 = cl, c1 = ch;
    const float det = a * c - b * b;
    const float ex = sqrtf(qmax * c / det), ey = sqrtf(qmax * a / det);
    if (det > 0.f && ex < 1e6f && ey < 1e6f) {
        const float hx = ex * 1.001f + 1e-3f, hy = ey * 1.001f + 1e-3f;   // rounding margin
        // pixel p passes |p + 0.5 - m| <= e  <=>  p in [m - e - 0.5, m + e - 0.5]
        r0 = max(r0, (int)floorf(A.y - hy - 0.5f));
        r1 = min(r1, (int)ceilf(A.y + hy - 0.5f));
        c0 = max(c0, (int)floorf(A.x - hx - 0.5f));
        c1 = min(c1, (int)ceilf(A.x + hx - 0.5f));
    }
    uint32_t mask = 0u;
    const int bx = tx * kTile, by = ty * kTile;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        const int x0 = bx + (w & 1) * 8, y0 = by + (w >> 1) * 4;
        if (c0 <= x0 + 7 && c1 >= x0 && r0 <= y0 + 3 && r1 >= y0) mask |= 1u << w;
    }
    return mask;
}

// CI: 0 none, 1 max weight (all splats), 2 max weight + weight sums (all splats),
//     3 max weight + weight sums for splats whose Gaussian is not yet visited.
template <bool kLoss, bool kImage, int CI>
__global__ void __launch_bounds__(kRT, HS_RASTER_MINB) raster_fwd_kernel(RasterArgs a) {
    __shared__ __align__(16) unsigned char s_stage[kRT * kStageBytes];
    __shared__ uint32_t s_mask[kRT];
    __shared__ float red[2][kWarps];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tile = blockIdx.x, b = blockIdx.y;
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    int px, py;
    pixel_of(tid, tx, ty, px, py);
    const bool inside = px < a.W && py < a.H;
    const uint2 rg = reinterpret_cast<const uint2 *>(a.ranges)[((int64_t)b << a.tile_bits) + tile];
    const uint32_t start = rg.x, end = rg.y;
    const float fpx = (float)px, fpy = (float)py;
    const int64_t pix = ((int64_t)b * a.H + (inside ? py : 0)) * a.W + (inside ? px : 0);
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(s_stage);

    float tgt[3] = {0.f, 0.f, 0.f}, rgba_a = 0.f, rgb[3] = {0.f, 0.f, 0.f};
    const float bg[3] = {a.bgs[3 * b], a.bgs[3 * b + 1], a.bgs[3 * b + 2]};
    if ((kLoss || CI >= 2) && inside && a.targets) {
        const uchar4 t = reinterpret_cast<const uchar4 *>(a.targets)[pix];
        rgba_a = (float)t.w / 255.0f;
        rgb[0] = (float)t.x / 255.0f;
        rgb[1] = (float)t.y / 255.0f;
        rgb[2] = (float)t.z / 255.0f;
#pragma unroll
        for (int c = 0; c < 3; ++c) tgt[c] = rgb[c] * rgba_a + (1.0f - rgba_a) * bg[c];
    }
    float ws_src[3] = {tgt[0], tgt[1], tgt[2]};
    if (CI >= 2 && a.wsum_image && inside) {
#pragma unroll
        for (int c = 0; c < 3; ++c) ws_src[c] = a.wsum_image[pix * 3 + c];
    }

    float T = 1.0f, C[3] = {0.f, 0.f, 0.f};
    uint32_t stop = end - start;
    bool done = !inside;
    for (uint32_t c0 = start; c0 < end; c0 += kRT) {
        if (__syncthreads_count(!done) == 0) break;
        const uint32_t idx = c0 + tid;
        uint32_t m = 0u;
        if (idx < end) {
            const uint32_t n = a.vals[idx];
            uint32_t gflag = (uint32_t)((int64_t)b * a.N + n);
            if (CI == 3 && a.visited[n]) gflag |= 0x80000000u;   // visited: skip colour-init work
            m = stage_splat(a.records + ((int64_t)b * a.N + n) * kRec, gflag, tx, ty, sbase + tid * kStageBytes);
        }
        s_mask[tid] = m;
        __syncthreads();
        const int cnt = (int)min((uint32_t)kRT, end - c0);
        if (!__all_sync(kFull, done)) {
            for (int i = 0; i < (cnt + 31) / 32; ++i) {
                uint32_t bits = __ballot_sync(kFull, (s_mask[i * 32 + lane] >> warp) & 1u);
                while (bits) {
                    const int j = i * 32 + __ffs(bits) - 1;
                    bits &= bits - 1u;
                    const uint32_t ad = sbase + j * kStageBytes;
                    float w = 0.f;
                    if (!done) {
                        const int4 bb = lds4i(ad + 32);
                        if (px >= bb.x && px <= bb.y && py >= bb.z && py <= bb.w) {
                            const float4 p0 = lds4(ad), p1 = lds4(ad + 16);
                            const float dx = fpx - p0.x, dy = fpy - p0.y;
                            const float e2 = splat_e2(dx, dy, p0.z, p0.w, p1.x);
                            if (e2 >= p1.y) {
                                const float alpha = __fmul_rn(p1.z, ex2_approx(e2));
                                if (alpha >= kAlphaCutoff) {
                                    const float4 col = lds4(ad + 48);
                                    w = alpha * T;
                                    C[0] += w * col.x;
                                    C[1] += w * col.y;
                                    C[2] += w * col.z;
                                    T = T * (1.0f - alpha);
                                    if (T < kTermEps) {
                                        done = true;
                                        stop = c0 - start + (uint32_t)j + 1u;
                                    }
                                }
                            }
                        }
                    }
                    if (CI > 0) {
                        const uint32_t gf = lds1(ad + 28);
                        const bool want = CI != 3 || !(gf & 0x80000000u);
                        if (want && __any_sync(kFull, w > 0.f)) {
                            const int64_t g = gf & 0x7FFFFFFFu;
                            const float wm = warp_max(w);
                            if (CI >= 2) {
                                const float v[4] = {w * ws_src[0], w * ws_src[1], w * ws_src[2], w};
                                int vi;
                                bool issue;
                                const float s = reduce_scatter(v, lane, vi, issue);
                                if (issue) atomicAdd(a.wsums + g * 4 + vi, s);
                            }
                            if (lane == 0) atomicMax(reinterpret_cast<int *>(a.maxw) + g, __float_as_int(wm));
                        }
                    }
                }
            }
        }
        __syncthreads();
    }

    float l1 = 0.f, black = 0.f;
    if (inside) {
        float pred[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) pred[c] = C[c] + T * bg[c];
        uint32_t signs = 0;
        if (kLoss) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const float d = pred[c] - tgt[c];
                l1 += fabsf(d);
                black += fabsf(C[c] - rgb[c] * rgba_a);
                signs |= (d > 0.f ? 1u : d < 0.f ? 2u : 0u) << (2 * c);
            }
        }
        a.pix_T[pix] = T;
        a.pix_state[pix] = stop | (signs << 26);
        if (kImage) {
#pragma unroll
            for (int c = 0; c < 3; ++c) a.image[pix * 3 + c] = pred[c];
        }
    }
    if (kLoss) {
        l1 = warp_sum(l1);
        black = warp_sum(black);
        if (lane == 0) {
            red[0][warp] = l1;
            red[1][warp] = black;
        }
        __syncthreads();
        if (tid == 0) {
            float s0 = 0.f, s1 = 0.f;
            for (int i = 0; i < kWarps; ++i) { s0 += red[0][i]; s1 += red[1][i]; }
            const int tiles = gridDim.x;
            a.loss_partials[((int64_t)b * tiles + tile) * 2] = s0;
            a.loss_partials[((int64_t)b * tiles + tile) * 2 + 1] = s1;
        }
    }
}

template <bool kExplicitGrad>
__global__ void __launch_bounds__(kRT, HS_RASTER_MINB) raster_bwd_kernel(RasterArgs a) {
    __shared__ __align__(16) unsigned char s_stage[kRT * kStageBytes];
    __shared__ uint32_t s_mask[kRT];
    __shared__ uint32_t s_max[kWarps];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tile = blockIdx.x, b = blockIdx.y;
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    int px, py;
    pixel_of(tid, tx, ty, px, py);
    const bool inside = px < a.W && py < a.H;
    const uint2 rg = reinterpret_cast<const uint2 *>(a.ranges)[((int64_t)b << a.tile_bits) + tile];
    const uint32_t start = rg.x, end = rg.y;
    if (start >= end) return;
    const float fpx = (float)px, fpy = (float)py;
    const int64_t pix = ((int64_t)b * a.H + (inside ? py : 0)) * a.W + (inside ? px : 0);
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(s_stage);

    float g[3] = {0.f, 0.f, 0.f};
    uint32_t stop = 0;
    float t_rev = 0.f, suffix = 0.f;
    if (inside) {
        const uint32_t st = a.pix_state[pix];
        stop = st & kStopMask;
        const float Tf = a.pix_T[pix];
        if (kExplicitGrad) {
#pragma unroll
            for (int c = 0; c < 3; ++c) g[c] = a.grad_image[pix * 3 + c];
        } else {
            const uint32_t sg = st >> 26;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const uint32_t s2 = (sg >> (2 * c)) & 3u;
                g[c] = s2 == 1u ? a.grad_scale : s2 == 2u ? -a.grad_scale : 0.f;
            }
        }
        t_rev = Tf;
        suffix = Tf * (g[0] * a.bgs[3 * b] + g[1] * a.bgs[3 * b + 1] + g[2] * a.bgs[3 * b + 2]);
    }
    // last local index any pixel of the tile needs
    const uint32_t wmax = __reduce_max_sync(kFull, stop);
    if (lane == 0) s_max[warp] = wmax;
    __syncthreads();
    uint32_t maxstop = 0;
#pragma unroll
    for (int i = 0; i < kWarps; ++i) maxstop = max(maxstop, s_max[i]);
    const uint32_t last = start + maxstop;

    for (uint32_t c_end = last; c_end > start;) {
        const uint32_t c0 = c_end - start > (uint32_t)kRT ? c_end - kRT : start;
        const uint32_t idx = c0 + tid;
        __syncthreads();
        uint32_t m = 0u;
        if (idx < c_end) {
            const uint32_t n = a.vals[idx];
            m = stage_splat(a.records + ((int64_t)b * a.N + n) * kRec, (uint32_t)((int64_t)b * a.N + n), tx, ty,
                            sbase + tid * kStageBytes);
        }
        s_mask[tid] = m;
        __syncthreads();
        const int cnt = (int)(c_end - c0);
        for (int i = (cnt - 1) / 32; i >= 0; --i) {
            uint32_t bits = __ballot_sync(kFull, (s_mask[i * 32 + lane] >> warp) & 1u);
            while (bits) {
                const int hb = 31 - __clz(bits);
                bits &= ~(1u << hb);
                const int j = i * 32 + hb;
                const uint32_t jl = c0 - start + (uint32_t)j;
                const uint32_t ad = sbase + j * kStageBytes;
                float gv[9];
                bool contrib = false;
                if (jl < stop) {
                    const int4 bb = lds4i(ad + 32);
                    if (px >= bb.x && px <= bb.y && py >= bb.z && py <= bb.w) {
                        const float4 p0 = lds4(ad), p1 = lds4(ad + 16);
                        const float dx = fpx - p0.x, dy = fpy - p0.y;
                        const float e2 = splat_e2(dx, dy, p0.z, p0.w, p1.x);
                        if (e2 >= p1.y) {
                            const float G = ex2_approx(e2);
                            const float alpha = __fmul_rn(p1.z, G);
                            if (alpha >= kAlphaCutoff) {
                                contrib = true;
                                const float4 col = lds4(ad + 48);
                                const float inv = __fdividef(1.0f, 1.0f - alpha);
                                const float t_prior = t_rev * inv;
                                const float gw = g[0] * col.x + g[1] * col.y + g[2] * col.z;
                                const float wgt = alpha * t_prior;
                                gv[6] = wgt * g[0];
                                gv[7] = wgt * g[1];
                                gv[8] = wgt * g[2];
                                const float d_alpha = t_prior * gw - suffix * inv;
                                gv[5] = G * d_alpha;
                                const float dq = -0.5f * alpha * d_alpha;
                                const float dqx = dq * dx, dqy = dq * dy;
                                gv[2] = dqx * dx;
                                gv[3] = 2.0f * dqx * dy;
                                gv[4] = dqy * dy;
                                // -2 dq (a dx + b dy) with the k-scaled conic: (-2/k) dq (ka dx + kb dy)
                                const float hb2 = 0.5f * p0.w;
                                gv[0] = kMeanScale * (p0.z * dqx + hb2 * dqy);
                                gv[1] = kMeanScale * (hb2 * dqx + p1.x * dqy);
                                suffix += wgt * gw;
                                t_rev = t_prior;
                            }
                        }
                    }
                }
                if (__any_sync(kFull, contrib)) {
                    if (!contrib) {
#pragma unroll
                        for (int k = 0; k < 9; ++k) gv[k] = 0.f;
                    }
                    int vi;
                    bool issue;
                    const float s = reduce_scatter(gv, lane, vi, issue);
                    if (issue) atomicAdd(a.g_splat + (uint64_t)lds1(ad + 28) * kGS + vi, s);
                }
            }
        }
        c_end = c0;
    }
}

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
static void launch_fwd_ci(int ci, dim3 grid, cudaStream_t s, const RasterArgs &a) {
    switch (ci) {
        case 0: raster_fwd_kernel<L, I, 0><<<grid, kRT, 0, s>>>(a); break;
        case 1: raster_fwd_kernel<L, I, 1><<<grid, kRT, 0, s>>>(a); break;
        case 2: raster_fwd_kernel<L, I, 2><<<grid, kRT, 0, s>>>(a); break;
        default: raster_fwd_kernel<L, I, 3><<<grid, kRT, 0, s>>>(a); break;
    }
}

}  // namespace hs

using namespace hs;

extern "C" {

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
    dim3 grid(tiles_x * tiles_y, B);
    cudaStream_t s = HS_CHECK_STREAM(stream);
    if (loss && img) launch_fwd_ci<true, true>(ci, grid, s, a);
    else if (loss) launch_fwd_ci<true, false>(ci, grid, s, a);
    else if (img) launch_fwd_ci<false, true>(ci, grid, s, a);
    else launch_fwd_ci<false, false>(ci, grid, s, a);
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
    dim3 grid(tiles_x * tiles_y, B);
    cudaStream_t s = HS_CHECK_STREAM(stream);
    if (grad_image) raster_bwd_kernel<true><<<grid, kRT, 0, s>>>(a);
    else raster_bwd_kernel<false><<<grid, kRT, 0, s>>>(a);
    return check_launch("hs_raster_bwd");
}

int hs_loss_reduce(int B, int num_tiles, int width, int height, const float *loss_partials, float *loss_out,
                   void *stream) {
    cudaStream_t s = HS_CHECK_STREAM(stream);
    const float inv = (float)(1.0 / ((double)width * height * 3.0));
    loss_reduce_kernel<<<B, 256, 0, s>>>(B, num_tiles, inv, loss_partials, loss_out);
    loss_mean_kernel<<<1, 32, 0, s>>>(B, loss_out);
    return check_launch("hs_loss_reduce");
}

}  // extern "C"
