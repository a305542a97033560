// hs_raster.cu -- tile rasterizer (forward + adjoint) on sm_100a.
//
// One warp (a one-warp CTA) per (frame, 16x16 tile, 8x8 pixel block): each lane
// holds two pixels of the block (rows r and r+4 of one column), so the per-splat
// overhead (list walk, shared loads, the warp reduction of the adjoint) is paid
// once per 64 pixels.  The four warps of a tile walk its depth-ordered key range
// independently, 32 splats per batch: each lane gathers one 48-byte record, pre-transforms it
// into a 64-byte staged form in the warp's private shared slots (four 512-byte quarter
// blocks: conflict-free 16-byte stores) and votes whether
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
// then the 9 per-splat gradients go out as vector REDs from each contributing lane (at
// most HS_RASTER_DIRECT of them) or are reduce-scattered across the warp (12 shuffles)
// before one RED per value.
#include <algorithm>
#include <type_traits>

#include "hs_common.cuh"

namespace hs {

#ifndef HS_RASTER_CTA_WARPS
#define HS_RASTER_CTA_WARPS 1        // warps per CTA (each warp owns one 8 x 8 block)
#endif
#ifndef HS_RASTER_MINB
#define HS_RASTER_MINB (28 / HS_RASTER_CTA_WARPS)   // resident CTAs per SM (28 one-warp CTAs: <= 72 registers)
#endif

// The training raster with the colour-init sums (CI >= 2) fits 64 registers without spills:
// 32 resident one-warp CTAs per SM (-2 % against 28 at 72 registers); the CI 0 / 1 variants
// would spill there and keep HS_RASTER_MINB.
#ifndef HS_RASTER_MINB_CI
#define HS_RASTER_MINB_CI 32
#endif
constexpr int train_minb(int ci) { return ci >= 2 ? HS_RASTER_MINB_CI : HS_RASTER_MINB; }
#ifndef HS_RASTER_MINB_FWD
#define HS_RASTER_MINB_FWD 32        // the forward-only (render / compat) raster: 64 registers (render +0.7 %)
#endif

#ifndef HS_RASTER_EXACT_CULL
#define HS_RASTER_EXACT_CULL 1       // cull row groups with the exact ellipse-rectangle distance
#endif
#ifndef HS_QTEST
#define HS_QTEST 1                   // the reference's q <= qmax test next to alpha >= 1/255 (0: A/B only)
#endif
#ifndef HS_RASTER_FWD_ASM
#define HS_RASTER_FWD_ASM 1          // forward: per-pixel decision as one predicate chain
#endif
#ifndef HS_RASTER_DIRECT
#define HS_RASTER_DIRECT 12          // adjoint: up to this many contributing lanes add directly
#endif

// Two pixels per lane (rows r and r + 4 of one column of the warp's 8 x 8 block): the
// pair is evaluated with sm_100a's packed FP32 (fma/mul/add.rn.f32x2 -> FFMA2 / FMUL2 /
// FADD2), one instruction for both pixels.
constexpr int kPX = 2;
constexpr int kCW = HS_RASTER_CTA_WARPS;

// Optional instrumentation (-DHS_RASTER_STATS): forward-pass counts of warp
// iterations and pixel tests, read with hs_raster_stats().
__device__ unsigned long long g_raster_stats[16];
#ifdef HS_RASTER_TIMING
__device__ unsigned long long g_raster_times[3 * 8192];   // per warp: start, end (globaltimer ns), items
#endif
constexpr int kBlocks = kTile * kTile / (32 * kPX);   // 8 x 8 pixel blocks per tile
constexpr int kRT = 32 * kCW;                          // threads per CTA
static_assert(kBlocks % kCW == 0, "CTA warps must divide the blocks of a tile");
constexpr unsigned kFull = 0xffffffffu;

struct RasterArgs {
    int B;
    int64_t N;
    int W, H, tiles_x, tile_bits;
    float inv_tiles_x;
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
    // persistent scheduling (caller workspace, see hs_raster_workspace_size)
    unsigned int *work;
    const uint32_t *tile_order;
    // HS_RASTER_DETERMINISTIC: g_splat / wsums are int64 fixed-point accumulators
    int det;
    // float mode with a 16-byte aligned g_splat: the adjoint may use vector REDs
    int vec;
    // speculative launch guard (hs_raster_guard_t): the binning summary and the limits
    // under which its lists are complete; NULL: no guard
    const unsigned long long *guard;
    unsigned long long guard_capacity;
    unsigned int guard_longest;
};

// A raster enqueued before the host has read the step's binning summary (the one host
// sync) exits at once unless the lists are complete: the fill ran (key total within the
// buffers), no list needs the CTA / two-level sorts, and no error was flagged.  The host
// re-launches it after fixing up the rare case.
__device__ __forceinline__ bool guard_blocks(const RasterArgs &a) {
    if (a.guard == nullptr) return false;
    return a.guard[0] > a.guard_capacity || a.guard[3] > a.guard_longest || a.guard[1] != HS_NO_ERROR;
}

// Deterministic accumulation (HS_RASTER_DETERMINISTIC): every contribution rounded once to
// a fixed-point int64 (2^-48 resolution for the splat gradients, 2^-40 for the colour-init
// sums) and added with integer atomics, which are associative -- the totals no longer
// depend on the order in which warps finish (float atomics do, by an ulp or so).
constexpr float kFxGrad = 281474976710656.0f;     // 2^48
constexpr float kFxSums = 1099511627776.0f;       // 2^40
__device__ __forceinline__ void acc_add(const RasterArgs &a, float *fp, int64_t i, float v, float fx) {
    HS_CHECK(i >= 0 && i < (int64_t)a.B * a.N * (fp == a.wsums ? 4 : kGS), "raster accumulator index", i);
    if (a.det)
        atomicAdd(reinterpret_cast<unsigned long long *>(fp) + i, (unsigned long long)__float2ll_rn(v * fx));
    else
        atomicAdd(fp + i, v);
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(kFull, v, o));
    return v;
}

// ---- staged splat layout (shared memory, 64 B per splat) -------------------------------
//   q0: nmx nmy ka  kb2        nm = 0.5 - mean: dx = px + nmx = px + 0.5 - mx;
//                              k = -0.5 log2(e): e2 = k q = dx (ka dx + kb2 dy) + kc dy^2
//   q1: kc  nop ncr ncg        alpha = op 2^e2; nop = -op (clamped, kOpacityMax); nc = -colour
//   q2: ncb kqmax gidx kb      q <= qmax <=> e2 >= k qmax; gidx = frame * N + n;
//                              kb = kb2 / 2 (the non-raw adjoint's conic term)
//   q3: mlo mhi                64-bit pixel mask of the warp's 8 x 8 block (bit 32 p + lane:
//                              pixel p of the lane) = the reference's integer bbox
//                              (S/render.py:248-251) minus row groups the alpha >= 1/255
//                              ellipse cannot reach
// The packed instructions take each per-splat scalar as a broadcast operand (the .F32
// form of FFMA2 / FMUL2 / FADD2), so one value serves both pixels of a lane.  Negated
// opacity / colour make 1 - alpha an FADD2 and the weighted colour an FFMA2 with no extra
// negation.  Forward and adjoint evaluate e2 / alpha with the same explicitly rounded
// operations (per element identical to __fmaf_rn / __fmul_rn), so both make identical
// decisions.
constexpr float kK = -0.72134752044448170f;      // -0.5 * log2(e)
constexpr float kMeanScale = -2.0f / kK;         // d q / d(k q) folded into g_mean
// the adjoint's constant factor of gradient value v (g_mean 2, g_conic 3, g_opacity,
// g_colour 3): the mean and conic partial sums carry -dq = -alpha d_alpha (S/render.py:323-330)
//   kRaw (the training path, HS_RASTER_RAW_MEAN): g_mean's two sums are the raw -sum dq dx,
//   -sum dq dy; hs_project_avatar_bwd applies the conic, g_mean = [[a b] [b c]] (..)
template <bool kRaw = false>
__device__ __forceinline__ float grad_factor(int v) {
    return v < 2 ? (kRaw ? -1.0f : 0.5f * kMeanScale) : v == 3 ? 1.0f : v < 5 ? 0.5f : 1.0f;
}
// Each value stored once (64 B per splat); the packed instructions take the scalar as a
// broadcast operand (the .F32 form of FFMA2 / FMUL2 / FADD2).
// HS_STAGE_SOA: the warp's 32 slots as four 512-byte blocks (q0 of every slot, then q1, q2,
// q3 at a 16-byte stride), so a lane's 16-byte stores of its own slot hit consecutive
// addresses across the warp (conflict-free) instead of a 64-byte stride (4-way bank
// conflicts on every staging store); the broadcast loads of one slot are one wavefront
// either way.  The record prefetch slots likewise (three 512-byte blocks).
#ifndef HS_STAGE_SOA
#define HS_STAGE_SOA 1
#endif
constexpr int kStageBytes = 64;
constexpr int kQStride = HS_STAGE_SOA ? 512 : 16;      // byte offset between a slot's q0, q1, q2, q3
constexpr int kSlotStride = HS_STAGE_SOA ? 16 : kStageBytes;
constexpr int kWarpSmem = 32 * (kStageBytes + 48);    // staged splats + the record prefetch slots

__device__ __forceinline__ float4 lds4(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}
__device__ __forceinline__ void sts4(uint32_t addr, float a, float b, float c, float d) {
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

// 1/x for x in [2^-24, 1] (x = 1 - alpha, >= 2^-24 by the opacity clamp): the MUFU reciprocal without the
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
// Saturation guard: 1 - alpha must stay >= 2^-24 (the spacing of fp32 below 1).  fp32
// rounds sigmoid(logit) to 1.0f above logit ~16.6 and the Gaussian to 1 at a pixel within
// ~1e-3 px of the mean, where the reference's float64 alpha is still < 1 (its opacity
// saturates only near logit 36.7); alpha == 1.0f would make T exactly 0 and the adjoint's
// t_rev / (1 - alpha) 0 * inf = NaN (S/render.py:318-319).  The staging clamps the opacity
// at 1 - 2^-24 (the largest float below 1, nearer the reference's value than 1.0f), so
// alpha = op G <= 1 - 2^-24 and 1 - alpha >= 2^-24 exactly (Sterbenz) at every pixel: no
// per-pixel floor in either pass.  HS_ONE_MINUS_FLOOR=0: the unguarded A/B build.
#ifndef HS_ONE_MINUS_FLOOR
#define HS_ONE_MINUS_FLOOR 5.9604644775390625e-8f               // 2^-24 (0: the unguarded A/B build)
#endif
constexpr float kOneMinusFloor = HS_ONE_MINUS_FLOOR;
constexpr float kOpacityMax = 1.0f - kOneMinusFloor;

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }

// The staged splat of slot `ad`, unpacked into register pairs.
struct Staged {
    float2 nmx, nmy, ka, kb2, kc, nop, ncr, ncg, ncb, kb;
    float kq;
    uint32_t gidx, mlo, mhi;
};
__device__ __forceinline__ Staged load_staged(uint32_t ad) {
    Staged t;
    const float4 q0 = lds4(ad), q1 = lds4(ad + kQStride), q2 = lds4(ad + 2 * kQStride);
    uint32_t mlo, mhi;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(mlo), "=r"(mhi) : "r"(ad + 3 * kQStride));
    t.nmx = f2(q0.x, q0.x);
    t.nmy = f2(q0.y, q0.y);
    t.ka = f2(q0.z, q0.z);
    t.kb2 = f2(q0.w, q0.w);
    t.kc = f2(q1.x, q1.x);
    t.nop = f2(q1.y, q1.y);
    t.ncr = f2(q1.z, q1.z);
    t.ncg = f2(q1.w, q1.w);
    t.ncb = f2(q2.x, q2.x);
    t.kq = q2.y;
    t.gidx = __float_as_uint(q2.z);
    t.kb = f2(q2.w, q2.w);
    t.mlo = mlo;
    t.mhi = mhi;
    return t;
}

// e2 = k q at both pixels of the lane: per element
// __fmaf_rn(__fmul_rn(kc, dy), dy, __fmul_rn(dx, __fmaf_rn(kb2, dy, __fmul_rn(ka, dx))))
__device__ __forceinline__ float2 splat_e2(const Staged &t, float2 fpx2, float2 fpy2, float2 &dx2, float2 &dy2) {
    dx2 = add2(fpx2, t.nmx);
    dy2 = add2(fpy2, t.nmy);
    const float2 kadx = mul2(t.ka, dx2);
    return fma2(mul2(t.kc, dy2), dy2, mul2(dx2, fma2(t.kb2, dy2, kadx)));
}

// Forward per-pixel decision, one predicate chain (LOP3 + 3 FSETP.AND + FSEL):
//   live = pixel in the splat's mask && T >= 1e-14   (stop = live ? jl1 : stop)
//   returns live && e2 >= k qmax && -alpha <= -1/255 ? -alpha : 0
__device__ __forceinline__ float fwd_gate(uint32_t mask, uint32_t lanebit, float T, float e2, float kq, float nal,
                                          uint32_t jl1, uint32_t &stop) {
    float out;
    asm("{\n\t.reg .pred p, q;\n\t.reg .b32 m;\n\t"
        "and.b32 m, %2, %3;\n\t"
        "setp.ne.u32 p, m, 0;\n\t"
        "setp.ge.and.f32 p, %4, %5, p;\n\t"
        "selp.u32 %1, %9, %1, p;\n\t"
#if HS_QTEST
        "setp.ge.and.f32 q, %6, %7, p;\n\t"
#else
        "mov.pred q, p;\n\t"
#endif
        "setp.le.and.f32 q, %8, %10, q;\n\t"
        "selp.f32 %0, %8, 0f00000000, q;\n\t}"
        : "=f"(out), "+r"(stop)
        : "r"(mask), "r"(lanebit), "f"(T), "f"(kTermEps), "f"(e2), "f"(kq), "f"(nal), "r"(jl1), "f"(-kAlphaCutoff));
    return out;
}

// the same without the stop index (a forward that no adjoint follows: render)
__device__ __forceinline__ float fwd_gate_ns(uint32_t mask, uint32_t lanebit, float T, float e2, float kq, float nal) {
    float out;
    asm("{\n\t.reg .pred p, q;\n\t.reg .b32 m;\n\t"
        "and.b32 m, %1, %2;\n\t"
        "setp.ne.u32 p, m, 0;\n\t"
        "setp.ge.and.f32 p, %3, %4, p;\n\t"
#if HS_QTEST
        "setp.ge.and.f32 q, %5, %6, p;\n\t"
#else
        "mov.pred q, p;\n\t"
#endif
        "setp.le.and.f32 q, %7, %8, q;\n\t"
        "selp.f32 %0, %7, 0f00000000, q;\n\t}"
        : "=f"(out)
        : "r"(mask), "r"(lanebit), "f"(T), "f"(kTermEps), "f"(e2), "f"(kq), "f"(nal), "f"(-kAlphaCutoff));
    return out;
}

// Stage one splat record into the lane's slot for the warp's 8 x 8 block with origin
// (x0, y0).  Returns true when a pixel of the block can be touched (its mask is nonzero).
// The record prefetch (HS_RASTER_PREFETCH): while a warp works through one 32-key batch,
// each lane's 48-byte record of the NEXT batch streams into a per-lane shared slot with
// cp.async (the list value for it was loaded a batch earlier), so staging a batch reads
// shared memory instead of waiting on two dependent global loads (list value, then record).
#ifndef HS_RASTER_PREFETCH
#define HS_RASTER_PREFETCH 1
#endif
constexpr int kRecBytes = 48;
constexpr int kRecQStride = HS_STAGE_SOA ? 512 : 16;
constexpr int kRecSlotStride = HS_STAGE_SOA ? 16 : kRecBytes;
__device__ __forceinline__ void cp_async_record(uint32_t dst, const float *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(dst + kRecQStride), "l"(src + 4) : "memory");
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(dst + 2 * kRecQStride), "l"(src + 8) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

struct RawRec {
    float4 A, B, C;
};
__device__ __forceinline__ RawRec load_rec_global(const float *rec) {
    const float4 *r = reinterpret_cast<const float4 *>(rec);
    return {__ldg(r), __ldg(r + 1), __ldg(r + 2)};
}
__device__ __forceinline__ RawRec load_rec_shared(uint32_t addr) {
    return {lds4(addr), lds4(addr + kRecQStride), lds4(addr + 2 * kRecQStride)};
}

// The pixel mask of the 8 x 8 block at (x0, y0) for a splat record: the block's pixels inside
// the reference's integer bbox minus the row groups (4 rows) its alpha >= 1/255 ellipse cannot reach.
template <bool kCull = true>
__device__ __forceinline__ uint64_t block_mask(const RawRec &rr, int x0, int y0) {
    const float4 A = rr.A, Bv = rr.B, Cv = rr.C;
    const uint32_t rows = __float_as_uint(Bv.w), cols = __float_as_uint(Cv.x);
    const int rl = unpack_lo(rows), rh = unpack_hi(rows), cl = unpack_lo(cols), ch = unpack_hi(cols);
    const float a = A.z, b = A.w, c = Bv.x, qmax = Bv.z;
    // the block's pixels inside the reference's bbox
    const int cs = max(cl - x0, 0), ce = min(ch - x0, 7), rs = max(rl - y0, 0), re = min(rh - y0, 7);
    uint64_t mask = 0;
    if (qmax >= 0.f && cs <= ce && rs <= re) {
        const uint32_t colbits = (0xFFu >> (7 - (ce - cs))) << cs;
        const uint64_t rowsp = (0x0101010101010101ull >> (8 * (7 - (re - rs)))) << (8 * rs);
        mask = rowsp * colbits;
        if (kCull && HS_RASTER_EXACT_CULL) {
            const float det = a * c - b * b;
            if (det > 0.f && a > 0.f && c > 0.f) {
                const float dxlo = (float)(x0 + cs) + 0.5f - A.x, dxhi = (float)(x0 + ce) + 0.5f - A.x;
                const float dxv = fminf(fmaxf(0.f, dxlo), dxhi);
                const float dyv0 = __fdividef(-b * dxv, c);                 // (margin covers the approx.)
#pragma unroll
                for (int p = 0; p < kPX; ++p) {
                    // row group p (rows y0 + 4p .. y0 + 4p + 3) within the bbox rows: the minimum
                    // of q(d) = a dx^2 + 2b dx dy + c dy^2 over the rectangle of those pixel
                    // centres (d = centre - mean).  For a positive-definite q the minimiser is
                    // the mean if it lies inside, else on an edge facing it; the two candidate
                    // segments (x nearest the mean with the best y, and vice versa) are inside
                    // the rectangle, so their minimum is exact.
                    const int ys = max(4 * p, rs), ye = min(4 * p + 3, re);
                    if (ys > ye) continue;
                    const float dylo = (float)(y0 + ys) + 0.5f - A.y, dyhi = (float)(y0 + ye) + 0.5f - A.y;
                    const float dyv = fminf(fmaxf(dyv0, dylo), dyhi);
                    const float dyh = fminf(fmaxf(0.f, dylo), dyhi);
                    const float dxh = fminf(fmaxf(__fdividef(-b * dyh, a), dxlo), dxhi);
                    const float qv = a * dxv * dxv + 2.f * b * dxv * dyv + c * dyv * dyv;
                    const float qh = a * dxh * dxh + 2.f * b * dxh * dyh + c * dyh * dyh;
                    // margin for the fp32 rounding of this bound and of the per-pixel q
                    if (fminf(qv, qh) * 0.999f - 1e-3f > qmax) mask &= ~(0xFFFFFFFFull << (32 * p));
                }
            }
        }
    }
    return mask;
}

template <bool kCull = true>
__device__ __forceinline__ bool stage_splat(const RawRec &rr, uint32_t gflag, int x0, int y0, uint32_t saddr) {
    const float4 A = rr.A, Bv = rr.B, Cv = rr.C;
    const float a = A.z, b = A.w, c = Bv.x, qmax = Bv.z;
    const float opv = kOneMinusFloor > 0.f ? fminf(Bv.y, kOpacityMax) : Bv.y;   // (the saturation guard)
    const float nmx = 0.5f - A.x, nmy = 0.5f - A.y, ka = kK * a, kb2 = 2.0f * kK * b, kb = kK * b, kc = kK * c;
    const uint64_t mask = block_mask<kCull>(rr, x0, y0);
    sts4(saddr, nmx, nmy, ka, kb2);
    sts4(saddr + kQStride, kc, -opv, -Cv.y, -Cv.z);
    sts4(saddr + 2 * kQStride, -Cv.w, kK * qmax, __uint_as_float(gflag), kb);
    asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(saddr + 3 * kQStride), "r"((uint32_t)mask), "r"((uint32_t)(mask >> 32))
                 : "memory");
    return mask != 0;
}

// CI: 0 none, 1 max weight (all splats), 2 max weight + weight sums (all splats),
//     3 max weight + weight sums for splats whose Gaussian is not yet visited.
constexpr int kMaskBatches = 64;

// HS_FLUSH_VEC: the adjoint's direct adds as vector REDs.  Splat gidx's 9 sums start at
// float 9 gidx, whose offset mod 4 is gidx mod 4; each alignment class splits the 9 values
// into 16 / 8 / 4-byte aligned pieces (3 or 4 REDs instead of 9).  Needs a 16-byte
// aligned g_splat (checked by the launcher) and the float mode.
#ifndef HS_FLUSH_VEC
#define HS_FLUSH_VEC 1
#endif
#ifndef HS_RASTER_SPLIT_SLOW
#define HS_RASTER_SPLIT_SLOW 1       // adjoint: separate loop bodies with / without the stop test
#endif
__device__ __forceinline__ void red4(float *p, float x, float y, float z, float w) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(x), "f"(y), "f"(z), "f"(w) : "memory");
}
__device__ __forceinline__ void red2(float *p, float x, float y) {
    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(x), "f"(y) : "memory");
}
__device__ __forceinline__ void red_splat9(float *gp, uint32_t gidx, const float (&f)[9]) {
    switch (gidx & 3u) {
        case 0:
            red4(gp, f[0], f[1], f[2], f[3]);
            red4(gp + 4, f[4], f[5], f[6], f[7]);
            atomicAdd(gp + 8, f[8]);
            break;
        case 1:
            atomicAdd(gp, f[0]);
            red2(gp + 1, f[1], f[2]);
            red4(gp + 3, f[3], f[4], f[5], f[6]);
            red2(gp + 7, f[7], f[8]);
            break;
        case 2:
            red2(gp, f[0], f[1]);
            red4(gp + 2, f[2], f[3], f[4], f[5]);
            red2(gp + 6, f[6], f[7]);
            atomicAdd(gp + 8, f[8]);
            break;
        default:
            atomicAdd(gp, f[0]);
            red4(gp + 1, f[1], f[2], f[3], f[4]);
            red4(gp + 5, f[5], f[6], f[7], f[8]);
            break;
    }
}     // per-warp hit masks kept from the forward for the fused adjoint

template <bool kExplicitGrad, bool kRaw>
__device__ __forceinline__ void raster_bwd_loop(const RasterArgs &a, int b, float2 fpx2, float2 fpy2, int x0, int y0,
                                                uint32_t start, uint32_t last, const float2 (&ng)[3], float2 t_rev,
                                                float2 nsuf, uint2 stop, int lane, uint32_t wbase,
                                                const uint32_t *masks);

// kState: track each pixel's stop index and write pix_T / pix_state (for an adjoint); false
// for a forward nothing follows (render)
template <bool kLoss, bool kImage, int CI, bool kTrain = false, bool kState = true>
__device__ __forceinline__ void raster_fwd_block(const RasterArgs &a, int b, int gw, int nblk, int lane,
                                                 uint32_t wbase, uint32_t *masks = nullptr) {
    // gw = tile * kBlocks + blk: the pixel block of frame b this warp composites
    const int tile = gw / kBlocks, blk = gw % kBlocks;
    // tile / tiles_x without an integer division: (tile + 1/2) / tiles_x is >= 1 / (2 tiles_x)
    // from an integer, far above the product's rounding (tile < 2^16)
    const int ty = (int)(((float)tile + 0.5f) * a.inv_tiles_x), tx = tile - ty * a.tiles_x;
    const int x0 = tx * kTile + (blk & 1) * 8, y0 = ty * kTile + (blk >> 1) * 8;
    const int px = x0 + (lane & 7), py0 = y0 + (lane >> 3);      // pixel p: (px, py0 + 4 p)
    const uint2 rg = reinterpret_cast<const uint2 *>(a.ranges)[((int64_t)b << a.tile_bits) + tile];
    const uint32_t start = rg.x, end = rg.y;
    HS_CHECK(start <= end && b < a.B, "raster range", (int64_t)end - start);
    const float bg[3] = {a.bgs[3 * b], a.bgs[3 * b + 1], a.bgs[3 * b + 2]};
    const float2 fpx2 = f2((float)px, (float)px), fpy2 = f2((float)py0, (float)(py0 + 4));
    const uint32_t lanebit = 1u << lane;
    const bool in0 = px < a.W && py0 < a.H, in1 = px < a.W && py0 + 4 < a.H;

    // per pixel pair: transmittance, colour (C[c] = channel c of both pixels), stop index
    float2 T = f2(1.f, 1.f), C[3] = {f2(0.f, 0.f), f2(0.f, 0.f), f2(0.f, 0.f)};
    uint2 stop = make_uint2(0u, 0u);
    // the colour-init source colours of the two pixels (target over bg, or wsum_image): loaded
    // on the first batch that has colour-init work -- most blocks have none once the
    // Gaussians in view are visited
    float src[CI >= 2 ? kPX : 1][3];
    bool src_ready = false;
    auto load_src = [&]() {
        if constexpr (CI >= 2) {
#pragma unroll
            for (int p = 0; p < kPX; ++p) {
                const bool inside = p ? in1 : in0;
                const int64_t pix = ((int64_t)b * a.H + (inside ? py0 + 4 * p : 0)) * a.W + (inside ? px : 0);
#pragma unroll
                for (int c = 0; c < 3; ++c) src[p][c] = 0.f;
                if (inside && a.wsum_image) {
#pragma unroll
                    for (int c = 0; c < 3; ++c) src[p][c] = a.wsum_image[pix * 3 + c];
                } else if (inside && a.targets) {
                    const uchar4 t = reinterpret_cast<const uchar4 *>(a.targets)[pix];
                    const float al = u8_unit(t.w);
                    const float rgb[3] = {u8_unit(t.x), u8_unit(t.y), u8_unit(t.z)};
#pragma unroll
                    for (int c = 0; c < 3; ++c) src[p][c] = rgb[c] * al + (1.0f - al) * bg[c];
                }
            }
        }
    };
    const float2 one2 = f2(1.f, 1.f);

#ifdef HS_RASTER_STATS
    unsigned long long st_iter = 0, st_c = 0, st_batches = 0, st_empty = 0, st_live = 0;
#endif
    // record prefetch: slot of this lane, and the list value of the next batch
    const uint32_t rslot = wbase + 32 * kStageBytes + lane * kRecSlotStride;
    const float *frec = a.records + (int64_t)b * a.N * kRec;
    uint32_t n_cur = start + lane < end ? a.vals[start + lane] : 0u;
    uint32_t n_next = 0u;
    if (HS_RASTER_PREFETCH) {
        if (start + lane < end) cp_async_record(rslot, frec + (int64_t)n_cur * kRec);
        cp_async_commit();
        n_next = start + 32 + lane < end ? a.vals[start + 32 + lane] : 0u;
    }
    for (uint32_t c0 = start; c0 < end; c0 += 32) {
        // pixels outside the image have no mask bits; the loop ends when every pixel of
        // the block has terminated
        if (!__any_sync(kFull, (in0 && T.x >= kTermEps) || (in1 && T.y >= kTermEps))) break;
        const uint32_t idx = c0 + lane;
        bool hit = false, want = false;
        if (idx < end) {
            const uint32_t n = n_cur;
            HS_CHECK(n < a.N, "raster list value", n);
            const uint32_t gflag = (uint32_t)((int64_t)b * a.N + n);
            RawRec rr;
            if (HS_RASTER_PREFETCH) {
                cp_async_wait_all();
                rr = load_rec_shared(rslot);
            } else {
                rr = load_rec_global(frec + (int64_t)n * kRec);
            }
            hit = stage_splat(rr, gflag, x0, y0, wbase + lane * kSlotStride);
            want = CI > 0 && hit && (CI != 3 || !a.visited[n]);   // visited: no colour-init work
        }
        // the next batch: its records start streaming into the slots (this lane's slot was
        // just read), and its successor's list values are loaded
        if (HS_RASTER_PREFETCH) {
            if (idx + 32 < end) cp_async_record(rslot, frec + (int64_t)n_next * kRec);
            cp_async_commit();
            n_cur = n_next;
            n_next = idx + 64 < end ? a.vals[idx + 64] : 0u;
        } else {
            n_cur = idx + 32 < end ? a.vals[idx + 32] : 0u;
        }
        uint32_t bits = __ballot_sync(kFull, hit);
        const uint32_t wantb = __ballot_sync(kFull, want);
        if (kTrain && lane == 0) {
            const uint32_t k = (c0 - start) >> 5;
            if (k < (uint32_t)kMaskBatches) masks[k] = bits;
        }
#ifdef HS_RASTER_STATS
        st_batches += lane == 0;
#endif
        __syncwarp();
        // one splat of the batch (kCI: with the colour-init sums); the batch runs the loop
        // without the colour-init test when no staged splat wants it
        auto splat = [&](int j, auto ci_tag) {
            constexpr bool kCI = decltype(ci_tag)::value;
            const Staged t = load_staged(wbase + j * kSlotStride);
            float2 dx2, dy2;
            const float2 e2 = splat_e2(t, fpx2, fpy2, dx2, dy2);
            float2 nal = mul2(t.nop, f2(ex2_approx(e2.x), ex2_approx(e2.y)));     // -alpha
            // the reference's tests (S/render.py:248-266): bbox, not terminated, q <= qmax,
            // alpha >= 1/255; a failing pixel gets alpha = 0 (no change to C or T); stop
            // records the list position after the last splat tested while live
            const uint32_t jl1 = c0 - start + (uint32_t)j + 1u;
            if (HS_RASTER_FWD_ASM && !kState && !kTrain) {
                nal.x = fwd_gate_ns(t.mlo, lanebit, T.x, e2.x, t.kq, nal.x);
                nal.y = fwd_gate_ns(t.mhi, lanebit, T.y, e2.y, t.kq, nal.y);
            } else if (HS_RASTER_FWD_ASM) {
                nal.x = fwd_gate(t.mlo, lanebit, T.x, e2.x, t.kq, nal.x, jl1, stop.x);
                nal.y = fwd_gate(t.mhi, lanebit, T.y, e2.y, t.kq, nal.y, jl1, stop.y);
            } else {
                const bool live0 = (t.mlo & lanebit) && T.x >= kTermEps, live1 = (t.mhi & lanebit) && T.y >= kTermEps;
                if (live0) stop.x = jl1;
                if (live1) stop.y = jl1;
                const bool ok0 = live0 && e2.x >= t.kq && nal.x <= -kAlphaCutoff;
                const bool ok1 = live1 && e2.y >= t.kq && nal.y <= -kAlphaCutoff;
                nal.x = ok0 ? nal.x : 0.f;
                nal.y = ok1 ? nal.y : 0.f;
            }
#ifdef HS_RASTER_STATS
            st_iter += (lane == 0);
            st_c += (nal.x != 0.f) + (nal.y != 0.f);
            {
                const bool any_c = __any_sync(kFull, nal.x != 0.f || nal.y != 0.f);
                const int nlive = __popc(__ballot_sync(kFull, (t.mlo & lanebit) && T.x >= kTermEps)) +
                                  __popc(__ballot_sync(kFull, (t.mhi & lanebit) && T.y >= kTermEps));
                st_empty += (lane == 0) && !any_c;
                st_live += (lane == 0) ? nlive : 0;
            }
#endif
            const float2 nw = mul2(nal, T);                    // -alpha T
            C[0] = fma2(nw, t.ncr, C[0]);
            C[1] = fma2(nw, t.ncg, C[1]);
            C[2] = fma2(nw, t.ncb, C[2]);
            float2 om = add2(one2, nal);                       // 1 - alpha
            T = mul2(T, om);
            if (kCI && ((wantb >> j) & 1u)) {
                const float wmax = -fminf(nw.x, nw.y);
                if (__any_sync(kFull, wmax > 0.f)) {
                    const int64_t g = t.gidx;
                    const float wm = warp_max(wmax);
                    if (CI >= 2) {
                        const float v[4] = {-(nw.x * src[0][0] + nw.y * src[1][0]),
                                            -(nw.x * src[0][1] + nw.y * src[1][1]),
                                            -(nw.x * src[0][2] + nw.y * src[1][2]), -(nw.x + nw.y)};
                        int vi;
                        bool issue;
                        const float s = reduce_scatter(v, lane, vi, issue);
                        if (issue) acc_add(a, a.wsums, g * 4 + vi, s, kFxSums);
                    }
                    if (lane == 0) atomicMax(reinterpret_cast<int *>(a.maxw) + g, __float_as_int(wm));
                }
            }
        };
        if (CI >= 2 && wantb && !src_ready) {      // (warp-uniform)
            load_src();
            src_ready = true;
        }
        if (CI > 0 && wantb) {
            while (bits) {
                const int j = __ffs(bits) - 1;
                bits &= bits - 1u;
                splat(j, std::true_type{});
            }
        } else {
            while (bits) {
                const int j = __ffs(bits) - 1;
                bits &= bits - 1u;
                splat(j, std::false_type{});
            }
        }
        __syncwarp();
    }

    if (HS_RASTER_PREFETCH) cp_async_wait_all();            // (the loop may break early)
#ifdef HS_RASTER_STATS
    atomicAdd(&g_raster_stats[0], st_iter);
    atomicAdd(&g_raster_stats[3], st_c);
    atomicAdd(&g_raster_stats[6], st_batches);
    atomicAdd(&g_raster_stats[4], st_empty);
    atomicAdd(&g_raster_stats[1], st_live);
#endif
    // pixel p: a terminated pixel keeps the stop index found above (its terminating
    // splat + 1); a live one gets the list length (S/render.py:254-259: no stop)
    const uint32_t len = end - start;
    if (T.x >= kTermEps) stop.x = len;
    if (T.y >= kTermEps) stop.y = len;
    float l1 = 0.f, black = 0.f;
    float2 ng[3];                            // fused adjoint: minus the L1 gradient of each pixel
#pragma unroll
    for (int p = 0; p < kPX; ++p) {
        const int py = py0 + 4 * p;
        const float Tp = p ? T.y : T.x;
        float g3[3] = {0.f, 0.f, 0.f};
        if (px < a.W && py < a.H) {
            const int64_t pix = ((int64_t)b * a.H + py) * a.W + px;
            float pred[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) pred[c] = (p ? C[c].y : C[c].x) + Tp * bg[c];
            uint32_t signs = 0;
            if (kLoss) {
                const uchar4 t = reinterpret_cast<const uchar4 *>(a.targets)[pix];
                const float al = u8_unit(t.w);
                const float rgb[3] = {u8_unit(t.x), u8_unit(t.y), u8_unit(t.z)};
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const float tgt = rgb[c] * al + (1.0f - al) * bg[c];
                    const float d = pred[c] - tgt;
                    l1 += fabsf(d);
                    black += fabsf((p ? C[c].y : C[c].x) - rgb[c] * al);
                    signs |= (d > 0.f ? 1u : d < 0.f ? 2u : 0u) << (2 * c);
                    if (kTrain) g3[c] = d > 0.f ? -a.grad_scale : d < 0.f ? a.grad_scale : 0.f;
                }
            }
            if (kTrain ? a.pix_T != nullptr : kState) {
                a.pix_T[pix] = Tp;
                a.pix_state[pix] = (p ? stop.y : stop.x) | (signs << 26);
            }
            if (kImage) {
#pragma unroll
                for (int c = 0; c < 3; ++c) a.image[pix * 3 + c] = pred[c];
            }
        }
        if (kTrain) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                if (p) ng[c].y = g3[c];
                else ng[c].x = g3[c];
            }
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
        if (!in0) stop.x = 0;
        if (!in1) stop.y = 0;
        const float2 t_rev = f2(in0 ? T.x : 0.f, in1 ? T.y : 0.f);
        // -suffix = -T <g, bg> = T <ng, bg>
        const float2 nsuf = mul2(t_rev, fma2(ng[2], f2(bg[2], bg[2]), fma2(ng[1], f2(bg[1], bg[1]),
                                                                          mul2(ng[0], f2(bg[0], bg[0])))));
        const uint32_t last = start + __reduce_max_sync(kFull, max(stop.x, stop.y));
        __syncwarp();
        raster_bwd_loop<false, true>(a, b, fpx2, fpy2, x0, y0, start, last, ng, t_rev, nsuf, stop, lane, wbase, masks);
    }
}

// Work distribution (HS_RASTER_PERSIST, default): a persistent grid of resident
// one-warp CTAs where every warp pulls (frame, block) items from a counter, so short and
// long blocks mix freely and no CTA launch happens per block (-8 % raster time vs one CTA
// per block).  The counters and the item order live in a caller-provided workspace
// (hs_raster_workspace_size; zeroed once at allocation): the last warp to finish resets
// the counters, so launches on different workspaces are independent and one workspace
// serves its stream's launches back to back.  HS_RASTER_PERSIST=0: one CTA per block.
#ifndef HS_RASTER_PERSIST
#define HS_RASTER_PERSIST 1
#endif

// Longest-first item order (HS_RASTER_LPT): tiles bucketed by the bit length of their
// key count, heaviest bucket first, so the long tiles start early and the persistent
// grid's tail is made of short items.  One small CTA per launch builds it.
#ifndef HS_RASTER_LPT
#define HS_RASTER_LPT 1
#endif
#ifndef HS_RASTER_LPT_SUB
#define HS_RASTER_LPT_SUB 2
#endif
constexpr int kWsCounters = 16;      // workspace head: [next, done] (+ padding), then the order

__global__ void __launch_bounds__(1024) tile_order_kernel(int total_tiles, int tile_bits, int tiles,
                                                          const uint32_t *__restrict__ ranges,
                                                          uint32_t *__restrict__ order) {
    pdl_prologue();
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
    // (the entries are b << tile_bits | tile: the raster splits them with a shift)
    for (int t = threadIdx.x; t < total_tiles; t += blockDim.x)
        order[atomicAdd(&cursor[bucket(t)], 1u)] = ((uint32_t)(t / tiles) << tile_bits) | (uint32_t)(t % tiles);
}

template <typename F>
__device__ __forceinline__ void for_each_block(const RasterArgs &a, int nblk, int lane, int warp, F &&fn) {
    if (!HS_RASTER_PERSIST) {
        fn((int)blockIdx.y, (int)blockIdx.x * kCW + warp);
        return;
    }
    const int total = a.B * nblk;
    const int tiles = nblk / kBlocks;
    unsigned int *work = a.work;
#ifdef HS_RASTER_TIMING
    unsigned long long t_start;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    unsigned int n_items = 0;
#endif
    for (;;) {
        int item = 0;
        if (lane == 0) item = (int)atomicAdd(work, 1u);
        item = __shfl_sync(kFull, item, 0);
        if (item >= total) break;
        if (HS_RASTER_LPT) {
            const uint32_t bt = a.tile_order[item / kBlocks];
            fn((int)(bt >> a.tile_bits), (int)(bt & ((1u << a.tile_bits) - 1u)) * kBlocks + item % kBlocks);
        } else {
            fn(item / nblk, item % nblk);
        }
        __syncwarp();
#ifdef HS_RASTER_TIMING
        ++n_items;
#endif
    }
#ifdef HS_RASTER_TIMING
    if (lane == 0) {
        unsigned long long t_end;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        const unsigned int wid = blockIdx.x * kCW + warp;
        if (wid < 8192) {
            g_raster_times[3 * wid] = t_start;
            g_raster_times[3 * wid + 1] = t_end;
            g_raster_times[3 * wid + 2] = n_items;
        }
    }
#endif
    if (lane == 0) {
        const unsigned int warps = gridDim.x * gridDim.y * kCW;
        if (atomicAdd(work + 1, 1u) == warps - 1) {
            work[0] = 0u;
            work[1] = 0u;
        }
    }
}

template <bool kLoss, bool kImage, int CI, bool kState = true>
__global__ void __launch_bounds__(kRT, HS_RASTER_MINB_FWD) raster_fwd_kernel(RasterArgs a, int nblk) {
    pdl_prologue();
    if (guard_blocks(a)) return;
    __shared__ __align__(16) unsigned char s_stage[kCW * kWarpSmem];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t wbase = (uint32_t)__cvta_generic_to_shared(s_stage) + warp * kWarpSmem;
    for_each_block(a, nblk, lane, warp, [&](int b, int gw) {
        raster_fwd_block<kLoss, kImage, CI, false, kState>(a, b, gw, nblk, lane, wbase);
    });
}

template <bool kExplicitGrad, bool kRaw>
__device__ __forceinline__ void raster_bwd_block(const RasterArgs &a, int b, int gw, int lane, uint32_t wbase) {
    const int tile = gw / kBlocks, blk = gw % kBlocks;
    // tile / tiles_x without an integer division: (tile + 1/2) / tiles_x is >= 1 / (2 tiles_x)
    // from an integer, far above the product's rounding (tile < 2^16)
    const int ty = (int)(((float)tile + 0.5f) * a.inv_tiles_x), tx = tile - ty * a.tiles_x;
    const int x0 = tx * kTile + (blk & 1) * 8, y0 = ty * kTile + (blk >> 1) * 8;
    const int px = x0 + (lane & 7), py0 = y0 + (lane >> 3);
    const uint2 rg = reinterpret_cast<const uint2 *>(a.ranges)[((int64_t)b << a.tile_bits) + tile];
    const uint32_t start = rg.x, end = rg.y;
    if (start >= end) return;
    const float bg[3] = {a.bgs[3 * b], a.bgs[3 * b + 1], a.bgs[3 * b + 2]};
    float2 ng[3], t_rev, nsuf;
    uint2 stop;
#pragma unroll
    for (int p = 0; p < kPX; ++p) {
        const int py = py0 + 4 * p;
        const bool inside = px < a.W && py < a.H;
        const int64_t pix = ((int64_t)b * a.H + (inside ? py : 0)) * a.W + (inside ? px : 0);
        float g[3] = {0.f, 0.f, 0.f}, Tf = 0.f;
        uint32_t st = 0;
        if (inside) {
            const uint32_t w = a.pix_state[pix];
            st = w & kStopMask;
            Tf = a.pix_T[pix];
            if (kExplicitGrad) {
#pragma unroll
                for (int c = 0; c < 3; ++c) g[c] = -a.grad_image[pix * 3 + c];
            } else {
                const uint32_t sg = w >> 26;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const uint32_t s2 = (sg >> (2 * c)) & 3u;
                    g[c] = s2 == 1u ? -a.grad_scale : s2 == 2u ? a.grad_scale : 0.f;
                }
            }
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            if (p) ng[c].y = g[c];
            else ng[c].x = g[c];
        }
        if (p) { stop.y = st; t_rev.y = Tf; }
        else { stop.x = st; t_rev.x = Tf; }
    }
    nsuf = mul2(t_rev, fma2(ng[2], f2(bg[2], bg[2]), fma2(ng[1], f2(bg[1], bg[1]), mul2(ng[0], f2(bg[0], bg[0])))));
    // this warp only needs the list up to its pixels' largest stop index
    const uint32_t last = start + __reduce_max_sync(kFull, max(stop.x, stop.y));
    raster_bwd_loop<kExplicitGrad, kRaw>(a, b, f2((float)px, (float)px), f2((float)py0, (float)(py0 + 4)), x0, y0, start,
                                   last, ng, t_rev, nsuf, stop, lane, wbase, nullptr);
}

// Back-to-front walk of [start, last) in the forward's 32-key batches (S/render.py:
// 276-336, the suffix recurrence per pixel).  With the forward's hit masks (fused kernel)
// a batch is staged only by its hit lanes and skipped when empty; otherwise each batch is
// staged and culled again.  A batch holding no pixel's stop index takes the fast path
// (no per-splat stop test).
template <bool kExplicitGrad, bool kRaw>
__device__ __forceinline__ void raster_bwd_loop(const RasterArgs &a, int b, float2 fpx2, float2 fpy2, int x0, int y0,
                                                uint32_t start, uint32_t last, const float2 (&ng)[3], float2 t_rev,
                                                float2 nsuf, uint2 stop, int lane, uint32_t wbase,
                                                const uint32_t *masks) {
    if (last <= start) return;
    const uint32_t lanebit = 1u << lane;
    const float2 one2 = f2(1.f, 1.f);
    const uint32_t rslot = wbase + 32 * kStageBytes + lane * kRecSlotStride;
    const float *frec = a.records + (int64_t)b * a.N * kRec;
    // batch k's staging set: the forward's hit mask (fused kernel), or every list entry
    auto need = [&](int k) -> uint32_t {
        const uint32_t c0 = start + 32u * (uint32_t)k, c_end = min(c0 + 32u, last);
        const uint32_t live_lanes = c_end - c0 >= 32u ? kFull : (1u << (c_end - c0)) - 1u;
        return (masks != nullptr && k < kMaskBatches) ? masks[k] & live_lanes : live_lanes;
    };
#if HS_FLUSH_VEC
    // the reduce-scatter's result slot of this lane (a function of the lane only)
    int rs_vi;
    bool rs_issue;
    {
        const float z[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        (void)reduce_scatter(z, lane, rs_vi, rs_issue);
    }
    const float rs_factor = grad_factor<kRaw>(rs_vi);
#endif
    // back to front: the records of the next batch to walk (k - 1) prefetch while this one runs
    int k = (int)((last - 1 - start) >> 5);
    uint32_t nb_cur = need(k);
    if (HS_RASTER_PREFETCH) {
        if ((nb_cur >> lane) & 1u) cp_async_record(rslot, frec + (int64_t)a.vals[start + 32u * k + lane] * kRec);
        cp_async_commit();
    }
    for (; k >= 0; --k) {
        const uint32_t c0 = start + 32u * (uint32_t)k;
        const uint32_t c_end = min(c0 + 32u, last);
        const uint32_t idx = c0 + lane;
        const bool fused = masks != nullptr && k < kMaskBatches;
        const uint32_t stage_set = nb_cur;
        const uint32_t nb_next = k > 0 ? need(k - 1) : 0u;
        uint32_t bits;
        bool hit = false;
        if ((stage_set >> lane) & 1u) {
            const uint32_t n = a.vals[idx];
            HS_CHECK(n < a.N, "raster list value", n);
            RawRec rr;
            if (HS_RASTER_PREFETCH) {
                cp_async_wait_all();
                rr = load_rec_shared(rslot);
            } else {
                rr = load_rec_global(frec + (int64_t)n * kRec);
            }
            const uint32_t gflag = (uint32_t)((int64_t)b * a.N + n);
            if (fused) hit = stage_splat<false>(rr, gflag, x0, y0, wbase + lane * kSlotStride);
            else hit = stage_splat(rr, gflag, x0, y0, wbase + lane * kSlotStride);
        }
        if (HS_RASTER_PREFETCH) {
            if ((nb_next >> lane) & 1u) cp_async_record(rslot, frec + (int64_t)a.vals[idx - 32] * kRec);
            cp_async_commit();
        }
        nb_cur = nb_next;
        if (fused) {
            bits = stage_set;
            if (bits == 0u) continue;                      // warp-uniform
        } else {
            bits = __ballot_sync(kFull, hit);
        }
        // pixels whose stop index lies inside this batch need the per-splat test
        // jl < stop; a pixel with stop <= c0 takes no part in this batch at all
        const uint32_t b0 = stop.x > c0 - start ? lanebit : 0u, b1 = stop.y > c0 - start ? lanebit : 0u;
        const bool partial = (stop.x > c0 - start && stop.x < c_end - start) ||
                             (stop.y > c0 - start && stop.y < c_end - start);
        const bool slow = __any_sync(kFull, partial);
        __syncwarp();
        // the adjoint of splat j at this lane's two pixels: its 9 gradient partial sums
        // (returns whether a pixel of this lane contributed); advances t_rev / suffix
        auto splat = [&](int j, float (&gv)[9], uint32_t &gidx, auto slow_tag) -> bool {
            constexpr bool kSlow = decltype(slow_tag)::value;
            const uint32_t jl = c0 - start + (uint32_t)j;
            const Staged t = load_staged(wbase + j * kSlotStride);
            gidx = t.gidx;
            float2 dx2, dy2;
            const float2 e2 = splat_e2(t, fpx2, fpy2, dx2, dy2);
            float2 G = f2(ex2_approx(e2.x), ex2_approx(e2.y));
            float2 nal = mul2(t.nop, G);
            bool in0 = (t.mlo & b0) != 0u, in1 = (t.mhi & b1) != 0u;
            if (kSlow) {
                in0 = in0 && jl < stop.x;
                in1 = in1 && jl < stop.y;
            }
            const bool ok0 = in0 && (!HS_QTEST || e2.x >= t.kq) && nal.x <= -kAlphaCutoff;
            const bool ok1 = in1 && (!HS_QTEST || e2.y >= t.kq) && nal.y <= -kAlphaCutoff;
            // a failing pixel runs the same instructions with alpha = G = 0, which leaves
            // t_rev and the suffix unchanged (1 / (1 - 0) == 1 exactly) and adds zeros
            G.x = ok0 ? G.x : 0.f;
            G.y = ok1 ? G.y : 0.f;
            nal = mul2(t.nop, G);                                  // -alpha
            float2 om = add2(one2, nal);
            const float2 inv = f2(rcp_approx(om.x), rcp_approx(om.y));
            const float2 tp = mul2(t_rev, inv);                    // T before the splat
            const float2 gw = fma2(ng[2], t.ncb, fma2(ng[1], t.ncg, mul2(ng[0], t.ncr)));   // <g, colour>
            const float2 nwg = mul2(nal, tp);                      // -alpha T
            // colour: alpha T g = (-alpha T)(-g)
            gv[6] = nwg.x * ng[0].x + nwg.y * ng[0].y;
            gv[7] = nwg.x * ng[1].x + nwg.y * ng[1].y;
            gv[8] = nwg.x * ng[2].x + nwg.y * ng[2].y;
            // d alpha = T gw - suffix / (1 - alpha)
            const float2 da = fma2(nsuf, inv, mul2(tp, gw));
            gv[5] = G.x * da.x + G.y * da.y;
            const float2 ndq = mul2(nal, da);                      // -alpha d_alpha
            const float2 dqx = mul2(ndq, dx2), dqy = mul2(ndq, dy2);
            const float2 d2 = mul2(dqx, dx2), d3 = mul2(dqx, dy2), d4 = mul2(dqy, dy2);
            gv[2] = d2.x + d2.y;
            gv[3] = d3.x + d3.y;
            gv[4] = d4.x + d4.y;
            if constexpr (kRaw) {
                // the raw sums; the conic is applied once per splat by hs_project_avatar_bwd
                gv[0] = dqx.x + dqx.y;
                gv[1] = dqy.x + dqy.y;
            } else {
                // -2 dq (a dx + b dy) with the k-scaled conic: (-2/k) dq (ka dx + kb dy)
                const float2 m0 = fma2(t.kb, dqy, mul2(t.ka, dqx)), m1 = fma2(t.kc, dqy, mul2(t.kb, dqx));
                gv[0] = m0.x + m0.y;
                gv[1] = m1.x + m1.y;
            }
            nsuf = fma2(nwg, gw, nsuf);                            // suffix += alpha T gw
            t_rev = tp;
            return ok0 || ok1;
        };
        // one splat's 9 sums into g_splat: few contributing pixels (<= HS_RASTER_DIRECT
        // lanes) add directly (9 atomics each), otherwise the 9-value warp reduce-scatter
        // and one atomic per value.  Constant factors are applied once per reduced value
        // (the mean and conic sums carry -dq, sign folded here).
        auto flush1 = [&](const float (&gv)[9], uint32_t gidx, bool contrib, uint32_t cmask) {
#if HS_FLUSH_VEC
            float *gp = a.g_splat + (size_t)gidx * kGS;
            if (HS_RASTER_DIRECT && __popc(cmask) <= HS_RASTER_DIRECT) {
                if (contrib) {
                    if (a.vec) {
                        float f[9];
#pragma unroll
                        for (int v = 0; v < 9; ++v) f[v] = gv[v] * grad_factor<kRaw>(v);
                        red_splat9(gp, gidx, f);
                    } else {
#pragma unroll
                        for (int v = 0; v < 9; ++v) acc_add(a, a.g_splat, (int64_t)gidx * kGS + v, gv[v] * grad_factor<kRaw>(v), kFxGrad);
                    }
                }
            } else {
                const float s = reduce_scatter_value(gv, lane);
                if (rs_issue) {
                    if (a.det) acc_add(a, a.g_splat, (int64_t)gidx * kGS + rs_vi, s * rs_factor, kFxGrad);
                    else atomicAdd(gp + rs_vi, s * rs_factor);
                }
            }
#else
            if (HS_RASTER_DIRECT && __popc(cmask) <= HS_RASTER_DIRECT) {
                if (contrib) {
#pragma unroll
                    for (int v = 0; v < 9; ++v) acc_add(a, a.g_splat, (int64_t)gidx * kGS + v, gv[v] * grad_factor<kRaw>(v), kFxGrad);
                }
            } else {
                int vi;
                bool issue;
                const float s = reduce_scatter(gv, lane, vi, issue);
                if (issue) acc_add(a, a.g_splat, (int64_t)gidx * kGS + vi, s * grad_factor<kRaw>(vi), kFxGrad);
            }
#endif
        };
        // (a batch holding no pixel's stop index runs the loop without the per-splat stop test)
        auto walk = [&](auto slow_tag) {
            while (bits) {
                const int j = 31 - __clz(bits);
                bits &= ~(1u << j);
                float gv[9];
                uint32_t gidx;
                const bool contrib = splat(j, gv, gidx, slow_tag);
                const uint32_t cmask = __ballot_sync(kFull, contrib);
#ifdef HS_RASTER_STATS
                if (lane == 0) {
                    const int nc = __popc(cmask);
                    const int bin = nc == 0 ? 0 : nc == 1 ? 1 : nc == 2 ? 2 : nc <= 4 ? 3 : nc <= 8 ? 4 : nc <= 16 ? 5 : 6;
                    atomicAdd(&g_raster_stats[8 + bin], 1ull);
                }
#endif
                if (cmask) flush1(gv, gidx, contrib, cmask);
            }
        };
        if (HS_RASTER_SPLIT_SLOW && !slow) walk(std::false_type{});
        else walk(std::true_type{});
        __syncwarp();
    }
    if (HS_RASTER_PREFETCH) cp_async_wait_all();
}


// Training step: forward (L1 loss, colour-init sums) and adjoint of each pixel block in
// one pass -- no per-pixel state round trip through HBM, and the adjoint reuses the
// forward's per-batch hit masks.
template <int CI>
__global__ void __launch_bounds__(kRT, train_minb(CI)) raster_train_kernel(RasterArgs a, int nblk) {
    pdl_prologue();
    if (guard_blocks(a)) return;
    __shared__ __align__(16) unsigned char s_stage[kCW * kWarpSmem];
    __shared__ uint32_t s_masks[kCW][kMaskBatches];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t wbase = (uint32_t)__cvta_generic_to_shared(s_stage) + warp * kWarpSmem;
    for_each_block(a, nblk, lane, warp, [&](int b, int gw) {
        raster_fwd_block<true, false, CI, true>(a, b, gw, nblk, lane, wbase, s_masks[warp]);
    });
}

template <bool kExplicitGrad, bool kRaw>
__global__ void __launch_bounds__(kRT, HS_RASTER_MINB) raster_bwd_kernel(RasterArgs a, int nblk) {
    pdl_prologue();
    __shared__ __align__(16) unsigned char s_stage[kCW * kWarpSmem];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t wbase = (uint32_t)__cvta_generic_to_shared(s_stage) + warp * kWarpSmem;
    for_each_block(a, nblk, lane, warp,
                   [&](int b, int gw) { raster_bwd_block<kExplicitGrad, kRaw>(a, b, gw, lane, wbase); });
}

// partials[b][tiles * kBlocks][2] (one pair per pixel block)
__global__ void loss_reduce_kernel(int B, int tiles, float inv_count, const float *__restrict__ partials,
                                   float *__restrict__ out) {
    pdl_prologue();
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
    pdl_prologue();
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        float s = 0.f;
        for (int b = 0; b < B; ++b) s += out[b];
        out[2 * B] = s / (float)B;
    }
}

__global__ void fixed_to_float_kernel(int64_t n, const long long *__restrict__ fixed, float *__restrict__ out,
                                      float inv) {
    pdl_prologue();
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = (float)((double)fixed[i] * (double)inv);
}

static RasterArgs make_args(int B, int64_t N, int W, int H, const float *records, const uint32_t *values,
                            const uint32_t *ranges, int tile_bits, const float *bgs, void *workspace) {
    RasterArgs a{};
    a.B = B;
    a.N = N;
    a.W = W;
    a.H = H;
    a.tiles_x = (W + kTile - 1) / kTile;
    a.inv_tiles_x = 1.0f / (float)a.tiles_x;
    a.tile_bits = tile_bits;
    a.records = records;
    a.vals = values;
    a.ranges = ranges;
    a.bgs = bgs;
    a.work = reinterpret_cast<unsigned int *>(workspace);
    a.tile_order = reinterpret_cast<const uint32_t *>(workspace) + kWsCounters;
    return a;
}

template <bool L, bool I>
static void launch_fwd_ci(int ci, dim3 grid, int nblk, cudaStream_t s, const RasterArgs &a) {
    if (!a.pix_T && ci == 0) {            // no per-pixel state: no adjoint follows (render)
        launch_k(raster_fwd_kernel<L, I, 0, false>, grid, kRT, 0, s, a, nblk);
        return;
    }
    switch (ci) {
        case 0: launch_k(raster_fwd_kernel<L, I, 0>, grid, kRT, 0, s, a, nblk); break;
        case 1: launch_k(raster_fwd_kernel<L, I, 1>, grid, kRT, 0, s, a, nblk); break;
        case 2: launch_k(raster_fwd_kernel<L, I, 2>, grid, kRT, 0, s, a, nblk); break;
        default: launch_k(raster_fwd_kernel<L, I, 3>, grid, kRT, 0, s, a, nblk); break;
    }
}

static size_t workspace_bytes(int B, int W, int H) {
    const int64_t tiles = (int64_t)((W + kTile - 1) / kTile) * ((H + kTile - 1) / kTile);
    return sizeof(uint32_t) * (size_t)(kWsCounters + B * tiles);
}

// the persistent raster's longest-first item order, into the workspace
static void launch_tile_order(int B, int nblk, int tile_bits, const uint32_t *ranges, void *ws, cudaStream_t s) {
    const int tiles = nblk / kBlocks;
    if (HS_RASTER_PERSIST && HS_RASTER_LPT)
        launch_k(tile_order_kernel, 1, 1024, 0, s, B * tiles, tile_bits, tiles, ranges,
                                             reinterpret_cast<uint32_t *>(ws) + kWsCounters);
}

// grid of the raster kernels: one CTA per kCW blocks, or a persistent grid of
// resident CTAs (HS_RASTER_PERSIST) sized by the current device's SM count
static dim3 raster_grid(int nblk, int B, int minb = HS_RASTER_MINB) {
    if (!HS_RASTER_PERSIST) return dim3(nblk / kCW, B);
    const int64_t want = (int64_t)current_sm_count() * minb, items = (int64_t)nblk * B / kCW;
    return dim3((unsigned)std::max<int64_t>(1, std::min(want, items)), 1);
}

static void take_guard(RasterArgs &a, const hs_raster_guard_t *g) {
    if (g != nullptr && g->summary != nullptr) {
        a.guard = g->summary;
        a.guard_capacity = g->capacity;
        a.guard_longest = g->longest_max;
    }
}

static int check_ws(const char *fn, void *ws) {
    if (ws == nullptr || (reinterpret_cast<uintptr_t>(ws) & 15u)) {
        set_error("%s: workspace must be a 16-byte aligned device buffer of hs_raster_workspace_size() bytes", fn);
        return HS_ERR_SHAPE;
    }
    return HS_OK;
}

}  // namespace hs

using namespace hs;

extern "C" {

size_t hs_raster_workspace_size(int B, int width, int height) { return workspace_bytes(B, width, height); }



int hs_raster_tile_order(int B, int width, int height, const uint32_t *ranges, int tile_bits, void *workspace,
                         void *stream) {
    if (int e = check_ws("hs_raster_tile_order", workspace)) return e;
    const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
    launch_tile_order(B, tiles_x * tiles_y * kBlocks, tile_bits, ranges, workspace, HS_CHECK_STREAM(stream));
    return check_launch("hs_raster_tile_order");
}

int hs_raster_fwd(int B, int64_t N, int width, int height, int flags, const float *records, const uint32_t *values,
                  const uint32_t *ranges, int tile_bits, const float *backgrounds, const uint8_t *targets,
                  const float *wsum_image, const uint8_t *visited, float *pix_T, uint32_t *pix_state, float *image,
                  float *maxw, float *wsums, float *loss_partials, const hs_raster_guard_t *guard, void *workspace,
                  void *stream) {
    const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
    const bool loss = flags & HS_RASTER_LOSS, img = flags & HS_RASTER_IMAGE;
    int ci = 0;
    if (flags & HS_RASTER_MAXW_UNVISITED) ci = 3;
    else if ((flags & HS_RASTER_MAXW_ALL) && (flags & HS_RASTER_WSUMS)) ci = 2;
    else if (flags & HS_RASTER_MAXW_ALL) ci = 1;
    if ((loss && !targets) || (img && !image) || (ci && !maxw) || (ci >= 2 && !wsums) || (ci == 3 && !visited) ||
        (ci >= 2 && !targets && !wsum_image) || (loss && !loss_partials) || (!pix_T != !pix_state) ||
        (ci && !pix_T)) {
        set_error("hs_raster_fwd: flags 0x%x need a buffer that is NULL (pix_T and pix_state: both or neither, "
                  "both with the colour-init flags)", flags);
        return HS_ERR_SHAPE;
    }
    if (int e = check_ws("hs_raster_fwd", workspace)) return e;
    RasterArgs a = make_args(B, N, width, height, records, values, ranges, tile_bits, backgrounds, workspace);
    a.det = (flags & HS_RASTER_DETERMINISTIC) != 0;
    take_guard(a, guard);
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
    const dim3 grid = raster_grid(nblk, B, HS_RASTER_MINB_FWD);
    cudaStream_t s = HS_CHECK_STREAM(stream);
    if (!(flags & HS_RASTER_ORDER_READY)) launch_tile_order(B, nblk, tile_bits, ranges, workspace, s);
    if (loss && img) launch_fwd_ci<true, true>(ci, grid, nblk, s, a);
    else if (loss) launch_fwd_ci<true, false>(ci, grid, nblk, s, a);
    else if (img) launch_fwd_ci<false, true>(ci, grid, nblk, s, a);
    else launch_fwd_ci<false, false>(ci, grid, nblk, s, a);
    return check_launch("hs_raster_fwd");
}

int hs_raster_bwd(int B, int64_t N, int width, int height, const float *records, const uint32_t *values,
                  const uint32_t *ranges, int tile_bits, const float *backgrounds, const float *pix_T,
                  const uint32_t *pix_state, const float *grad_image, float grad_scale, float *g_splat,
                  int flags, void *workspace, void *stream) {
    if (int e = check_ws("hs_raster_bwd", workspace)) return e;
    const int tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
    RasterArgs a = make_args(B, N, width, height, records, values, ranges, tile_bits, backgrounds, workspace);
    a.pix_T = const_cast<float *>(pix_T);
    a.pix_state = const_cast<uint32_t *>(pix_state);
    a.grad_image = grad_image;
    a.grad_scale = grad_scale;
    a.g_splat = g_splat;
    a.vec = !a.det && (reinterpret_cast<uintptr_t>(g_splat) & 15u) == 0;
    const int nblk = tiles_x * tiles_y * kBlocks;
    const dim3 grid = raster_grid(nblk, B);
    cudaStream_t s = HS_CHECK_STREAM(stream);
    launch_tile_order(B, nblk, tile_bits, ranges, workspace, s);
    const bool raw = (flags & HS_RASTER_RAW_MEAN) != 0;
    if (grad_image) {
        if (raw) launch_k(raster_bwd_kernel<true, true>, grid, kRT, 0, s, a, nblk);
        else launch_k(raster_bwd_kernel<true, false>, grid, kRT, 0, s, a, nblk);
    } else {
        if (raw) launch_k(raster_bwd_kernel<false, true>, grid, kRT, 0, s, a, nblk);
        else launch_k(raster_bwd_kernel<false, false>, grid, kRT, 0, s, a, nblk);
    }
    return check_launch("hs_raster_bwd");
}

int hs_raster_train(int B, int64_t N, int width, int height, int flags, const float *records, const uint32_t *values,
                    const uint32_t *ranges, int tile_bits, const float *backgrounds, const uint8_t *targets,
                    const uint8_t *visited, float *maxw, float *wsums, float *loss_partials, float grad_scale,
                    float *g_splat, float *pix_T, uint32_t *pix_state, const hs_raster_guard_t *guard,
                    void *workspace, void *stream) {
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
    if (int e = check_ws("hs_raster_train", workspace)) return e;
    RasterArgs a = make_args(B, N, width, height, records, values, ranges, tile_bits, backgrounds, workspace);
    a.det = (flags & HS_RASTER_DETERMINISTIC) != 0;
    take_guard(a, guard);
    a.targets = targets;
    a.visited = visited;
    a.maxw = maxw;
    a.wsums = wsums;
    a.loss_partials = loss_partials;
    a.grad_scale = grad_scale;
    a.g_splat = g_splat;
    a.vec = !a.det && (reinterpret_cast<uintptr_t>(g_splat) & 15u) == 0;
    a.pix_T = pix_T;
    a.pix_state = pix_state;
    const int nblk = tiles_x * tiles_y * kBlocks;
    const dim3 grid = raster_grid(nblk, B, train_minb(ci));
    cudaStream_t s = HS_CHECK_STREAM(stream);
    if (!(flags & HS_RASTER_ORDER_READY)) launch_tile_order(B, nblk, tile_bits, ranges, workspace, s);
    switch (ci) {
        case 0: launch_k(raster_train_kernel<0>, grid, kRT, 0, s, a, nblk); break;
        case 1: launch_k(raster_train_kernel<1>, grid, kRT, 0, s, a, nblk); break;
        case 2: launch_k(raster_train_kernel<2>, grid, kRT, 0, s, a, nblk); break;
        default: launch_k(raster_train_kernel<3>, grid, kRT, 0, s, a, nblk); break;
    }
    return check_launch("hs_raster_train");
}

int hs_raster_warp_times(unsigned long long *host_out, int n) {
#ifdef HS_RASTER_TIMING
    cudaMemcpyFromSymbol(host_out, g_raster_times, sizeof(unsigned long long) * 3 * std::min(n, 8192));
    return check_launch("hs_raster_warp_times");
#else
    (void)host_out;
    (void)n;
    set_error("hs_raster_warp_times: build with -DHS_RASTER_TIMING");
    return HS_ERR_SHAPE;
#endif
}

int hs_raster_stats(unsigned long long *host_out, int reset) {
    cudaMemcpyFromSymbol(host_out, g_raster_stats, sizeof(unsigned long long) * 16);
    if (reset) {
        const unsigned long long z[16] = {};
        cudaMemcpyToSymbol(g_raster_stats, z, sizeof(z));
    }
    return check_launch("hs_raster_stats");
}

int hs_fixed_to_float(int64_t n, const long long *fixed, float *out, int sums, void *stream) {
    if (n <= 0) return HS_OK;
    launch_k(fixed_to_float_kernel, grid_for(n, 256), 256, 0, HS_CHECK_STREAM(stream), n, fixed, out,
                                                                                1.0f / (sums ? kFxSums : kFxGrad));
    return check_launch("hs_fixed_to_float");
}

int hs_loss_reduce(int B, int num_tiles, int width, int height, const float *loss_partials, float *loss_out,
                   void *stream) {
    cudaStream_t s = HS_CHECK_STREAM(stream);
    const float inv = (float)(1.0 / ((double)width * height * 3.0));
    static_assert(HS_LOSS_PARTIALS_PER_TILE >= 2 * kBlocks, "hs_api.h partial count");
    launch_k(loss_reduce_kernel, B, 256, 0, s, B, num_tiles * kBlocks, inv, loss_partials, loss_out);
    launch_k(loss_mean_kernel, 1, 32, 0, s, B, loss_out);
    return check_launch("hs_loss_reduce");
}

}  // extern "C"
