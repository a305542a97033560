// hs_project.cu -- batched projection (forward + adjoint) on sm_100a.
//
// One thread per (frame, Gaussian) over the whole B x N batch in ONE launch
// (the frame dimension is a grid dimension, replacing the reference's per-item
// thread-pool tasks, S/scheduler.py:57-72).  The avatar variant fuses
//   activate (S/model.py:219-234) -> transform_to_deformed (S/binding.py:174-188)
//   -> _project_kernel (S/render.py:132-198)
// and writes the 48-byte splat record, the camera depth and the number of 16x16
// tiles its pixel bbox touches, plus one partial sum of tile
// counts per 256 items for the key-offset scan.  The adjoint recomputes the same
// chain and applies _preprocess_backward (S/render.py:432-497), transform_backward
// (S/binding.py:191-204) and activate_backward (S/model.py:237-248).
#include "hs_common.cuh"

namespace hs {

struct Proj {
    float xc, yc, zc;             // camera-space position
    float m[9];                   // M = Rc R(q)
    float cov[6];                 // camera covariance c00 c01 c02 c11 c12 c22
    float j00, j02, j11, j12;     // EWA Jacobian
    float s00, s01, s11;          // 2D covariance
    float det, rad;
    float ca, cb, cc;             // conic
    float mx, my;
    bool valid;
};

// S/render.py:136-197, same operation order (fp32).
__device__ __forceinline__ void project_one(const float pw[3], const float q[4], const float s[3],
                                            const float *__restrict__ cam, Proj &p) {
    const float *rc = cam, *tc = cam + 9;
    const float fx = cam[12], fy = cam[13], cx = cam[14], cy = cam[15];
    p.xc = rc[0] * pw[0] + rc[1] * pw[1] + rc[2] * pw[2] + tc[0];
    p.yc = rc[3] * pw[0] + rc[4] * pw[1] + rc[5] * pw[2] + tc[1];
    p.zc = rc[6] * pw[0] + rc[7] * pw[1] + rc[8] * pw[2] + tc[2];
    p.valid = false;
    if (!(p.zc > kNearPlane)) return;
    float r[9];
    quat_to_mat(q, r);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            p.m[i * 3 + j] = rc[i * 3] * r[j] + rc[i * 3 + 1] * r[3 + j] + rc[i * 3 + 2] * r[6 + j];
    const float s0 = s[0] * s[0], s1 = s[1] * s[1], s2 = s[2] * s[2];
    const float *m = p.m;
    const float c00 = s0 * m[0] * m[0] + s1 * m[1] * m[1] + s2 * m[2] * m[2];
    const float c01 = s0 * m[0] * m[3] + s1 * m[1] * m[4] + s2 * m[2] * m[5];
    const float c02 = s0 * m[0] * m[6] + s1 * m[1] * m[7] + s2 * m[2] * m[8];
    const float c11 = s0 * m[3] * m[3] + s1 * m[4] * m[4] + s2 * m[5] * m[5];
    const float c12 = s0 * m[3] * m[6] + s1 * m[4] * m[7] + s2 * m[5] * m[8];
    const float c22 = s0 * m[6] * m[6] + s1 * m[7] * m[7] + s2 * m[8] * m[8];
    p.cov[0] = c00; p.cov[1] = c01; p.cov[2] = c02; p.cov[3] = c11; p.cov[4] = c12; p.cov[5] = c22;
    const float inv_z = __fdividef(1.0f, p.zc);
    p.j00 = fx * inv_z;
    p.j02 = -fx * p.xc * inv_z * inv_z;
    p.j11 = fy * inv_z;
    p.j12 = -fy * p.yc * inv_z * inv_z;
    p.s00 = p.j00 * (p.j00 * c00 + p.j02 * c02) + p.j02 * (p.j00 * c02 + p.j02 * c22);
    p.s01 = p.j11 * (p.j00 * c01 + p.j02 * c12) + p.j12 * (p.j00 * c02 + p.j02 * c22);
    p.s11 = p.j11 * (p.j11 * c11 + p.j12 * c12) + p.j12 * (p.j11 * c12 + p.j12 * c22);
    p.det = p.s00 * p.s11 - p.s01 * p.s01;
    const float mid = 0.5f * (p.s00 + p.s11);
    float disc = mid * mid - p.det;
    if (disc < 0.0f) disc = 0.0f;
    const float lam = mid + sqrtf(disc);
    p.rad = lam > 0.0f ? 3.0f * sqrtf(lam) : 0.0f;
    if (!(p.det > 0.0f) || !(p.rad >= kMinRadius)) return;
    const float inv_det = __fdividef(1.0f, p.det);
    p.ca = p.s11 * inv_det;
    p.cb = -p.s01 * inv_det;
    p.cc = p.s00 * inv_det;
    p.mx = fx * p.xc * inv_z + cx;
    p.my = fy * p.yc * inv_z + cy;
    p.valid = true;
}

// Record + tile count.  Pixel bbox per SURVEY Appendix B step 2: IEEE fp32, one
// rounding per op (the __f*_rn intrinsics forbid FMA contraction) so the key
// list is bit-exact against oracle/binning.py.
struct TileRect {
    int ty0, ty1, tx0, tx1;
    int rl, rh, cl, ch;            // the pixel bbox
    float qmax;
};

__device__ __forceinline__ uint32_t write_record(const Proj &p, float op, const float col[3], int W, int H,
                                                 float *__restrict__ rec, TileRect *rect = nullptr) {
    int r_lo = 1, r_hi = 0, c_lo = 1, c_hi = 0;
    if (p.valid) {
        const float rl = ceilf(__fsub_rn(__fsub_rn(p.my, p.rad), 0.5f));
        const float rh = floorf(__fsub_rn(__fadd_rn(p.my, p.rad), 0.5f));
        const float cl = ceilf(__fsub_rn(__fsub_rn(p.mx, p.rad), 0.5f));
        const float ch = floorf(__fsub_rn(__fadd_rn(p.mx, p.rad), 0.5f));
        // clamp in float first so the int conversion is exact and in range
        r_lo = (int)fmaxf(rl, 0.0f);
        r_hi = (int)fminf(rh, (float)(H - 1));
        c_lo = (int)fmaxf(cl, 0.0f);
        c_hi = (int)fminf(ch, (float)(W - 1));
        if (rh < 0.0f) r_hi = -1;
        if (ch < 0.0f) c_hi = -1;
        if (rl > (float)(H - 1)) r_lo = H;
        if (cl > (float)(W - 1)) c_lo = W;
    }
    const bool live = p.valid && op >= kAlphaCutoff && r_lo <= r_hi && c_lo <= c_hi;
    if (!live) { r_lo = 1; r_hi = 0; c_lo = 1; c_hi = 0; }
    float4 *r4 = reinterpret_cast<float4 *>(rec);
    const float qmax = op > 0.f ? 2.0f * logf(op * 255.0f) + 1e-9f : -1.0f;
    r4[0] = make_float4(p.mx, p.my, p.ca, p.cb);
    r4[1] = make_float4(p.cc, op, qmax, __uint_as_float(pack_lohi(r_lo, r_hi)));
    r4[2] = make_float4(__uint_as_float(pack_lohi(c_lo, c_hi)), col[0], col[1], col[2]);
    if (!live) return 0u;
    if (rect) *rect = {r_lo / kTile, r_hi / kTile, c_lo / kTile, c_hi / kTile, r_lo, r_hi, c_lo, c_hi, qmax};
    return (uint32_t)((r_hi / kTile - r_lo / kTile + 1) * (c_hi / kTile - c_lo / kTile + 1));
}

// Tile-major binning's count (hs_tile_count), fused: each (frame, splat) adds one per
// tile of its bbox -- into a shared histogram over the CTA's first frame's tiles,
// flushed with one global atomic per touched tile, or straight to the global counters.
constexpr int kProjHistBins = 4096;

// Per-256-item sum of tile counts (the key-offset scan input) and the range of the
// float bits of the depths that emit keys: the radix sort skips digit windows that
// are constant over [min, max] (positive floats order like their bit patterns).
__device__ __forceinline__ void block_sum_store(uint32_t v, float depth, uint32_t *block_sums,
                                                uint32_t *depth_range) {
    __shared__ uint32_t warp_sums[32], warp_min[32], warp_max[32];
    const uint32_t db = __float_as_uint(depth);
    const uint32_t dmin = __reduce_min_sync(0xffffffffu, v ? db : 0xFFFFFFFFu);
    const uint32_t dmax = __reduce_max_sync(0xffffffffu, v ? db : 0u);
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) {
        warp_sums[w] = v;
        warp_min[w] = dmin;
        warp_max[w] = dmax;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t s = 0, mn = 0xFFFFFFFFu, mx = 0u;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
            s += warp_sums[i];
            mn = min(mn, warp_min[i]);
            mx = max(mx, warp_max[i]);
        }
        block_sums[blockIdx.x] = s;
        if (depth_range && s) {
            atomicMin(depth_range, mn);
            atomicMax(depth_range + 1, mx);
        }
    }
}

__device__ __forceinline__ bool all_finite(const float *v, int n) {
    bool ok = true;
    for (int i = 0; i < n; ++i) ok &= isfinite(v[i]);
    return ok;
}

// world attributes of (b, n) in the avatar mode; returns false on a zero quaternion
struct AvatarWorld {
    float xt[3], qraw[4], qn[4], qf[4], qr[4], qw[4], s[3], op, col[3], pw[3];
    const float *R;
};

__device__ __forceinline__ bool avatar_world(int64_t N, int b, int64_t n, int F,
                                             const float *__restrict__ raw10,
                                             const float *__restrict__ base14,
                                             const int32_t *__restrict__ tri,
                                             const float *__restrict__ bary,
                                             const float *__restrict__ frames, AvatarWorld &a) {
    const float *raw = raw10 + (int64_t)b * 10 * N;
#pragma unroll
    for (int c = 0; c < 3; ++c) a.xt[c] = raw[3 * n + c];
#pragma unroll
    for (int c = 0; c < 4; ++c) a.qraw[c] = raw[3 * N + 4 * n + c];
    float colr[3], sr[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) colr[c] = raw[7 * N + 3 * n + c];
#pragma unroll
    for (int c = 0; c < 3; ++c) sr[c] = __ldg(base14 + 10 * N + 3 * n + c);
    const float opr = __ldg(base14 + 13 * N + n);
    // activate (S/model.py:219-234)
    const float nrm = sqrtf(a.qraw[0] * a.qraw[0] + a.qraw[1] * a.qraw[1] + a.qraw[2] * a.qraw[2] +
                            a.qraw[3] * a.qraw[3]);
    const bool ok = nrm >= 1e-30f;
    const float rn = __fdividef(1.0f, nrm);
#pragma unroll
    for (int c = 0; c < 4; ++c) a.qn[c] = a.qraw[c] * rn;
#pragma unroll
    for (int c = 0; c < 3; ++c) a.s[c] = __expf(sr[c]);
    a.op = sigmoid_fast(opr);
#pragma unroll
    for (int c = 0; c < 3; ++c) a.col[c] = sigmoid_fast(colr[c]);
    // transform (S/binding.py:174-188)
    const float *fr = frames + ((int64_t)b * F + __ldg(tri + n)) * kFrame;
    a.R = fr;
    const float bb[3] = {__ldg(bary + 3 * n), __ldg(bary + 3 * n + 1), __ldg(bary + 3 * n + 2)};
#pragma unroll
    for (int j = 0; j < 3; ++j)
        a.pw[j] = (fr[j * 3] * a.xt[0] + fr[j * 3 + 1] * a.xt[1] + fr[j * 3 + 2] * a.xt[2]) +
                  (bb[0] * fr[13 + j] + bb[1] * fr[16 + j] + bb[2] * fr[19 + j]);
#pragma unroll
    for (int c = 0; c < 4; ++c) a.qf[c] = fr[9 + c];
    quat_mul(a.qf, a.qn, a.qr);
    const float n2 = sqrtf(a.qr[0] * a.qr[0] + a.qr[1] * a.qr[1] + a.qr[2] * a.qr[2] + a.qr[3] * a.qr[3]);
    const float rn2 = __fdividef(1.0f, n2);
#pragma unroll
    for (int c = 0; c < 4; ++c) a.qw[c] = a.qr[c] * rn2;
    return ok;
}

__device__ __forceinline__ void check_world(const float pw[3], const float q[4], const float s[3], float op,
                                            const float col[3], int b, int64_t n,
                                            unsigned long long *err) {
    int attr = -1;
    if (!all_finite(pw, 3)) attr = 0;
    else if (!all_finite(q, 4)) attr = 1;
    else if (!all_finite(s, 3)) attr = 2;
    else if (!isfinite(op)) attr = 3;
    else if (!all_finite(col, 3)) attr = 4;
    if (attr >= 0) atomicMin(err, err_code(1, b, attr, n));
}

#ifndef HS_PFWD_MINB
#define HS_PFWD_MINB 6                 // 40 registers: 6 CTAs (48 warps) per SM (61.5 -> 57.3 us against 48 registers)
#endif
__global__ void __launch_bounds__(256, HS_PFWD_MINB) project_avatar_fwd_kernel(
    int B, int64_t N, int F, int W, int H, const float *__restrict__ raw10, const float *__restrict__ base14,
    const int32_t *__restrict__ tri, const float *__restrict__ bary, const float *__restrict__ frames,
    const float *__restrict__ cams, float *__restrict__ records, float *__restrict__ depth,
    uint32_t *__restrict__ counts, uint32_t *__restrict__ block_sums, uint32_t *__restrict__ depth_range,
    float *__restrict__ radius, float *__restrict__ zero_gsplat, float *__restrict__ zero_maxw,
    float *__restrict__ zero_wsums, uint32_t *__restrict__ tile_counts, uint32_t *__restrict__ tile_rects,
    unsigned long long *err) {
    pdl_prologue();
    extern __shared__ uint32_t hist[];
    // (launched with kScanBlock threads and B * N < 2^31, so the index math is 32-bit and the
    // loop trip counts are compile-time shifts)
    const int64_t i = blockIdx.x * (int64_t)kScanBlock + threadIdx.x;
    uint32_t cnt = 0;
    float dz = 0.f;
    const int tiles_x = (W + kTile - 1) / kTile, tiles = tiles_x * ((H + kTile - 1) / kTile);
    const int tile_bits = bit_length_u32((uint32_t)(tiles - 1));
    const int b0 = (int)((blockIdx.x * (uint32_t)kScanBlock) / (uint32_t)N);
    const bool shared = tile_counts && tiles <= kProjHistBins;
    // (the histogram is padded to a multiple of 4 bins: 16-byte clears and reads)
    const int tiles4 = (tiles + 3) >> 2;
    if (shared) {
        for (int t = threadIdx.x; t < tiles4; t += kScanBlock) reinterpret_cast<uint4 *>(hist)[t] = make_uint4(0u, 0u, 0u, 0u);
        __syncthreads();
    }
    // the step's per-(frame, splat) accumulators, zeroed here instead of by separate
    // fills (the raster adds into them with atomics); g_splat: the CTA's contiguous
    // 256 x kGS floats with coalesced 16-byte stores (a full CTA's span is 9216 bytes)
    if (zero_gsplat) {
        float *z = zero_gsplat + blockIdx.x * (int64_t)kScanBlock * kGS;
        const int items = (int)min((int64_t)kScanBlock, (int64_t)B * N - blockIdx.x * (int64_t)kScanBlock);
        if (items == kScanBlock && (reinterpret_cast<uintptr_t>(z) & 15u) == 0) {
#pragma unroll
            for (int k = 0; k < kScanBlock * kGS / 4; k += kScanBlock)
                if (k + (int)threadIdx.x < kScanBlock * kGS / 4)
                    reinterpret_cast<float4 *>(z)[k + threadIdx.x] = make_float4(0.f, 0.f, 0.f, 0.f);
        } else {
            for (int k = threadIdx.x; k < items * kGS; k += kScanBlock) z[k] = 0.f;
        }
    }
    const int lane = threadIdx.x & 31;
    TileRect rect{1, 0, 1, 0, 1, 0, 1, 0, -1.f};
    TileCull tc{};
    int b = 0;
    if (i < (int64_t)B * N) {
        if (zero_maxw) zero_maxw[i] = 0.f;
        if (zero_wsums) reinterpret_cast<float4 *>(zero_wsums)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        b = (int)((uint32_t)i / (uint32_t)N);
        const int64_t n = i - (int64_t)b * N;
        AvatarWorld a;
        const bool ok = avatar_world(N, b, n, F, raw10, base14, tri, bary, frames, a);
        if (!ok) atomicMin(err, err_code(0, b, 1, n));
        check_world(a.pw, a.qw, a.s, a.op, a.col, b, n, err);
        Proj p;
        project_one(a.pw, a.qw, a.s, cams + b * kCam, p);
        if (!ok) p.valid = false;
        cnt = write_record(p, a.op, a.col, W, H, records + i * kRec, &rect);
        if (tile_rects && cnt) tc = tile_cull(p.mx, p.my, p.ca, p.cb, p.cc, rect.qmax, rect.rl, rect.rh, rect.cl, rect.ch);
        depth[i] = p.zc;
        dz = p.zc;
        if (radius) radius[i] = p.valid ? p.rad : 0.f;
    }
    // The tiles: every lane takes one (item, tile) candidate of the warp's 32 items at a
    // time (no per-item loops of different lengths), tests it against the item's tile cull
    // when the item's rectangle carries a mask (tile_rects given, <= kMaskTiles tiles), and
    // counts a kept tile into the per-(frame, tile) counters; the ballot of kept candidates
    // gives each item its mask.  The item data the candidate lanes read is staged in shared
    // memory, one 48-byte slot per lane.
    uint32_t tmask = 0xFFFFFFFFu;
    if (tile_counts || tile_rects) {
        const uint32_t area = cnt;
        const bool cullable = tile_rects != nullptr && area != 0u && (int)area <= kMaskTiles;
        float4 *slots = reinterpret_cast<float4 *>(hist + (shared ? tiles4 * 4 : 0)) + (threadIdx.x & ~31) * 3;
        const uint32_t rp = (uint32_t)rect.ty0 | (uint32_t)rect.ty1 << 8 | (uint32_t)rect.tx0 << 16 | (uint32_t)rect.tx1 << 24;
        slots[3 * lane] = make_float4(tc.mx, tc.my, tc.a, tc.b);
        slots[3 * lane + 1] = make_float4(tc.c, tc.qmax, tc.inv_a, tc.inv_c);
        slots[3 * lane + 2] = make_float4(__uint_as_float(pack_lohi(tc.rl, tc.rh)), __uint_as_float(pack_lohi(tc.cl, tc.ch)),
                                          __uint_as_float(rp),
                                          __uint_as_float((uint32_t)b << 2 | (tc.pd ? 2u : 0u) | (cullable ? 1u : 0u)));
        __syncwarp();
        uint32_t incl = area;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        const uint32_t excl = incl - area, total = __shfl_sync(0xffffffffu, incl, 31);
        uint32_t bits = 0u;
        for (uint32_t k0 = 0; k0 < total; k0 += 32) {
            const uint32_t k = k0 + lane;
            const bool act = k < total;
            int o = 0;                     // the candidate's item: the last lane with excl <= k
#pragma unroll
            for (int st = 16; st; st >>= 1) {
                const uint32_t e = __shfl_sync(0xffffffffu, excl, o + st);
                if (e <= k) o += st;
            }
            const uint32_t lo = k - __shfl_sync(0xffffffffu, excl, o);
            bool keep = false;
            if (act) {
                const float4 s2 = slots[3 * o + 2];
                const uint32_t ro = __float_as_uint(s2.z), fo = __float_as_uint(s2.w);
                const int wo = (int)(ro >> 24) - (int)((ro >> 16) & 0xFFu) + 1;
                // lo / wo without an integer division: (lo + 1/2) / wo is at least 1 / (2 wo)
                // >= 2^-9 from an integer, far beyond the approximate quotient's error
                const int qy = (int)__fdividef((float)lo + 0.5f, (float)wo);
                const int ty = (int)(ro & 0xFFu) + qy, tx = (int)((ro >> 16) & 0xFFu) + (int)lo - qy * wo;
                keep = true;
                if (fo & 1u) {
                    const float4 s0 = slots[3 * o], s1 = slots[3 * o + 1];
                    TileCull t;
                    t.mx = s0.x; t.my = s0.y; t.a = s0.z; t.b = s0.w;
                    t.c = s1.x; t.qmax = s1.y; t.inv_a = s1.z; t.inv_c = s1.w;
                    t.rl = unpack_lo(__float_as_uint(s2.x)); t.rh = unpack_hi(__float_as_uint(s2.x));
                    t.cl = unpack_lo(__float_as_uint(s2.y)); t.ch = unpack_hi(__float_as_uint(s2.y));
                    t.pd = (fo & 2u) != 0u;
                    keep = tile_reaches(t, tx, ty);
                }
                if (keep && tile_counts) {
                    const int bo = (int)(fo >> 2);
                    const int t = ty * tiles_x + tx;
                    HS_CHECK(t >= 0 && t < tiles && bo < B, "projection tile count index", t);
                    if (shared && bo == b0) atomicAdd(hist + t, 1u);
                    else atomicAdd(tile_counts + ((size_t)bo << tile_bits) + t, 1u);
                }
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, keep);
            if (cullable) {        // this item's candidates of the round: [s, e)
                const uint32_t s = max(excl, k0), e = min(excl + area, k0 + 32u);
                if (s < e) bits |= ((bal >> (s - k0)) & (0xFFFFFFFFu >> (32u - (e - s)))) << (s - excl);
            }
        }
        if (cullable) {
            tmask = bits;
            cnt = (uint32_t)__popc(bits);
        }
    }
    if (i < (int64_t)B * N) {
        counts[i] = cnt;
        if (tile_rects)
            reinterpret_cast<uint2 *>(tile_rects)[i] =
                make_uint2(cnt ? (uint32_t)rect.ty0 | (uint32_t)rect.ty1 << 8 | (uint32_t)rect.tx0 << 16 |
                                     (uint32_t)rect.tx1 << 24
                               : 0x00010001u,
                           cnt ? tmask : 0u);
    }
    block_sum_store(cnt, dz, block_sums, depth_range);   // (a CTA barrier: the histogram is complete)
    if (shared) {
        uint32_t *row = tile_counts + ((size_t)b0 << tile_bits);
        for (int t = threadIdx.x; t < tiles4; t += kScanBlock) {
            const uint4 c = reinterpret_cast<const uint4 *>(hist)[t];
            if (c.x) atomicAdd(row + 4 * t, c.x);
            if (c.y) atomicAdd(row + 4 * t + 1, c.y);
            if (c.z) atomicAdd(row + 4 * t + 2, c.z);
            if (c.w) atomicAdd(row + 4 * t + 3, c.w);
        }
    }
}

__global__ void __launch_bounds__(256) project_world_fwd_kernel(
    int B, int64_t N, int W, int H, const float *__restrict__ world14, const float *__restrict__ cams,
    float *__restrict__ records, float *__restrict__ depth, uint32_t *__restrict__ counts,
    uint32_t *__restrict__ block_sums, uint32_t *__restrict__ depth_range, float *__restrict__ radius,
    float *__restrict__ x_cam, float *__restrict__ cov_cam, unsigned long long *err) {
    pdl_prologue();
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    uint32_t cnt = 0;
    float dz = 0.f;
    if (i < (int64_t)B * N) {
        const int b = (int)item_frame(i, N);
        const int64_t n = i - (int64_t)b * N;
        const float *w = world14 + (int64_t)b * 14 * N;
        float pw[3], q[4], s[3], col[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) { pw[c] = w[3 * n + c]; col[c] = w[7 * N + 3 * n + c]; s[c] = w[10 * N + 3 * n + c]; }
#pragma unroll
        for (int c = 0; c < 4; ++c) q[c] = w[3 * N + 4 * n + c];
        const float op = w[13 * N + n];
        check_world(pw, q, s, op, col, b, n, err);
        Proj p;
        project_one(pw, q, s, cams + b * kCam, p);
        cnt = write_record(p, op, col, W, H, records + i * kRec);
        depth[i] = p.zc;
        dz = p.zc;
        counts[i] = cnt;
        if (radius) radius[i] = p.valid ? p.rad : 0.f;
        if (x_cam) { x_cam[3 * i] = p.xc; x_cam[3 * i + 1] = p.yc; x_cam[3 * i + 2] = p.zc; }
        if (cov_cam) {
            const float *c = p.cov;
            const float full[9] = {c[0], c[1], c[2], c[1], c[3], c[4], c[2], c[4], c[5]};
#pragma unroll
            for (int k = 0; k < 9; ++k) cov_cam[9 * i + k] = p.valid ? full[k] : 0.f;
        }
    }
    block_sum_store(cnt, dz, block_sums, depth_range);
}

// _preprocess_backward for one splat (S/render.py:444-490).  gs = g_splat (9 floats).
// Outputs the world-space gradients of position, normalized quaternion and scale.
__device__ __forceinline__ void preprocess_bwd_one(const Proj &p, const float q[4], const float s[3],
                                                   const float *__restrict__ cam, const float gs[9],
                                                   float g_pos[3], float g_q[4], float g_s[3]) {
    const float *rc = cam;
    const float fx = cam[12], fy = cam[13];
    const float inv_z = __fdividef(1.0f, p.zc);
    const float ca = p.ca, cb = p.cb, cc = p.cc;
    const float ga = gs[2], gb = 0.5f * gs[3], gc = gs[4];
    const float g00 = -(ca * (ca * ga + cb * gb) + cb * (ca * gb + cb * gc));
    const float g01 = -(ca * (cb * ga + cc * gb) + cb * (cb * gb + cc * gc));
    const float g11 = -(cb * (cb * ga + cc * gb) + cc * (cb * gb + cc * gc));
    // J = [[j00, 0, j02], [0, j11, j12]]
    const float J[6] = {p.j00, 0.f, p.j02, 0.f, p.j11, p.j12};
    const float G[4] = {g00, g01, g01, g11};
    // g_cov_cam = J^T G J
    float gcc[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int l = 0; l < 3; ++l) {
            float acc = 0.f;
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int k = 0; k < 2; ++k) acc += J[j * 3 + i] * G[j * 2 + k] * J[k * 3 + l];
            gcc[i * 3 + l] = acc;
        }
    // g_J = (G + G^T) J cov_cam  (only the 4 non-structural-zero entries are used)
    const float C[9] = {p.cov[0], p.cov[1], p.cov[2], p.cov[1], p.cov[3], p.cov[4], p.cov[2], p.cov[4], p.cov[5]};
    float JC[6];
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int l = 0; l < 3; ++l) JC[j * 3 + l] = J[j * 3] * C[l] + J[j * 3 + 1] * C[3 + l] + J[j * 3 + 2] * C[6 + l];
    float gj[6];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int l = 0; l < 3; ++l) gj[i * 3 + l] = 2.f * (G[i * 2] * JC[l] + G[i * 2 + 1] * JC[3 + l]);
    // g_cov_world = Rc^T gcc Rc
    float t[9], gw[9];
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int l = 0; l < 3; ++l) t[j * 3 + l] = gcc[j * 3] * rc[l] + gcc[j * 3 + 1] * rc[3 + l] + gcc[j * 3 + 2] * rc[6 + l];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int l = 0; l < 3; ++l) gw[i * 3 + l] = rc[i] * t[l] + rc[3 + i] * t[3 + l] + rc[6 + i] * t[6 + l];
    float R[9];
    quat_to_mat(q, R);
    const float ss[3] = {s[0] * s[0], s[1] * s[1], s[2] * s[2]};
    float grot[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            float acc = 0.f;
#pragma unroll
            for (int j = 0; j < 3; ++j) acc += (gw[i * 3 + j] + gw[j * 3 + i]) * (R[j * 3 + k] * ss[k]);
            grot[i * 3 + k] = acc;
        }
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int k = 0; k < 3; ++k) acc += R[j * 3 + i] * gw[j * 3 + k] * R[k * 3 + i];
        g_s[i] = 2.0f * s[i] * acc;
    }
    quat_to_mat_bwd(q, grot, g_q);
    const float iz2 = inv_z * inv_z, iz3 = iz2 * inv_z;
    const float gmx = gs[0], gmy = gs[1];
    const float gx = gmx * fx * inv_z + gj[2] * (-fx * iz2);
    const float gy = gmy * fy * inv_z + gj[5] * (-fy * iz2);
    const float gz = -gmx * fx * p.xc * iz2 - gmy * fy * p.yc * iz2 + gj[0] * (-fx * iz2) +
                     gj[2] * (2.0f * fx * p.xc * iz3) + gj[4] * (-fy * iz2) + gj[5] * (2.0f * fy * p.yc * iz3);
#pragma unroll
    for (int j = 0; j < 3; ++j) g_pos[j] = gx * rc[j] + gy * rc[3 + j] + gz * rc[6 + j];
}

#ifndef HS_PBWD_MINB
#define HS_PBWD_MINB 3
#endif
__global__ void __launch_bounds__(256, HS_PBWD_MINB) project_avatar_bwd_kernel(
    int B, int64_t N, int F, const float *__restrict__ raw10, const float *__restrict__ base14,
    const int32_t *__restrict__ tri, const float *__restrict__ bary, const float *__restrict__ frames,
    const float *__restrict__ cams, const float *__restrict__ g_splat, int raw_mean, float *__restrict__ g_raw14) {
    pdl_prologue();
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= (int64_t)B * N) return;
    const int b = (int)item_frame(i, N);
    const int64_t n = i - (int64_t)b * N;
    float *o = g_raw14 + (int64_t)b * 14 * N;
    // the splat gradients first: their loads overlap the forward recomputation
    float gs[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) gs[k] = __ldcs(g_splat + i * kGS + k);
    AvatarWorld a;
    avatar_world(N, b, n, F, raw10, base14, tri, bary, frames, a);
    Proj p;
    project_one(a.pw, a.qw, a.s, cams + b * kCam, p);
    float g_xt[3] = {0.f, 0.f, 0.f}, g_qraw[4] = {0.f, 0.f, 0.f, 0.f}, g_sr[3] = {0.f, 0.f, 0.f};
    float g_colr[3] = {0.f, 0.f, 0.f}, g_opr = 0.f;
    if (p.valid) {
        if (raw_mean) {            // HS_RASTER_RAW_MEAN: g_mean = [[a b][b c]] (raw sums)
            const float sx = gs[0], sy = gs[1];
            gs[0] = p.ca * sx + p.cb * sy;
            gs[1] = p.cb * sx + p.cc * sy;
        }
        float g_pw[3], g_qw[4], g_s[3];
        preprocess_bwd_one(p, a.qw, a.s, cams + b * kCam, gs, g_pw, g_qw, g_s);
        // transform_backward (S/binding.py:191-204)
        const float *R = a.R;
#pragma unroll
        for (int k = 0; k < 3; ++k) g_xt[k] = R[k] * g_pw[0] + R[3 + k] * g_pw[1] + R[6 + k] * g_pw[2];
        float g_qr[4], g_qn[4];
        quat_normalize_bwd(a.qr, g_qw, g_qr);
        quat_mul_bwd_right(a.qf, g_qr, g_qn);
        // activate_backward (S/model.py:237-248)
        quat_normalize_bwd(a.qraw, g_qn, g_qraw);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            g_sr[k] = g_s[k] * a.s[k];
            g_colr[k] = gs[6 + k] * a.col[k] * (1.f - a.col[k]);
        }
        g_opr = gs[5] * a.op * (1.f - a.op);
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        o[3 * n + k] = g_xt[k];
        o[7 * N + 3 * n + k] = g_colr[k];
        o[10 * N + 3 * n + k] = g_sr[k];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) o[3 * N + 4 * n + k] = g_qraw[k];
    o[13 * N + n] = g_opr;
}

__global__ void __launch_bounds__(256) project_world_bwd_kernel(int B, int64_t N, const float *__restrict__ world14,
                                                                const float *__restrict__ cams,
                                                                const float *__restrict__ g_splat,
                                                                float *__restrict__ g_world14) {
    pdl_prologue();
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= (int64_t)B * N) return;
    const int b = (int)item_frame(i, N);
    const int64_t n = i - (int64_t)b * N;
    const float *w = world14 + (int64_t)b * 14 * N;
    float *o = g_world14 + (int64_t)b * 14 * N;
    float pw[3], q[4], s[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) { pw[c] = w[3 * n + c]; s[c] = w[10 * N + 3 * n + c]; }
#pragma unroll
    for (int c = 0; c < 4; ++c) q[c] = w[3 * N + 4 * n + c];
    Proj p;
    project_one(pw, q, s, cams + b * kCam, p);
    float g_pw[3] = {0.f, 0.f, 0.f}, g_q[4] = {0.f, 0.f, 0.f, 0.f}, g_s[3] = {0.f, 0.f, 0.f};
    float gs[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (p.valid) {
#pragma unroll
        for (int k = 0; k < 9; ++k) gs[k] = g_splat[i * kGS + k];
        preprocess_bwd_one(p, q, s, cams + b * kCam, gs, g_pw, g_q, g_s);
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        o[3 * n + k] = g_pw[k];
        o[7 * N + 3 * n + k] = gs[6 + k];
        o[10 * N + 3 * n + k] = g_s[k];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) o[3 * N + 4 * n + k] = g_q[k];
    o[13 * N + n] = gs[5];
}

}  // namespace hs

using namespace hs;

extern "C" {

int hs_scan_blocks(int64_t num_items) { return (int)((num_items + kScanBlock - 1) / kScanBlock); }

int hs_project_avatar_fwd(int B, int64_t N, int F, int width, int height, const float *raw10,
                          const float *base14, const int32_t *tri_index, const float *bary, const float *frames,
                          const float *cameras, float *records, float *depth, uint32_t *counts,
                          uint32_t *block_sums, uint32_t *depth_range, float *radius, float *zero_gsplat,
                          float *zero_maxw, float *zero_wsums, uint32_t *tile_counts, uint32_t *tile_rects,
                          unsigned long long *err, void *stream) {
    if (B < 1 || N < 1 || width < 1 || height < 1 || width > 32767 || height > 32767 ||
        (int64_t)B * N >= (int64_t(1) << 31)) {
        set_error("hs_project_avatar_fwd: bad sizes B=%d N=%lld %dx%d (B*N < 2^31)", B, (long long)N, width, height);
        return HS_ERR_SHAPE;
    }
    const int64_t items = (int64_t)B * N;
    const int tiles = ((width + kTile - 1) / kTile) * ((height + kTile - 1) / kTile);
    if (tile_counts && bit_length_u32((uint32_t)(tiles - 1)) + bit_length_u32((uint32_t)(B - 1)) > 31) {
        set_error("hs_project_avatar_fwd: frame/tile bits exceed 31");
        return HS_ERR_SHAPE;
    }
    if (tile_rects && (((width + kTile - 1) / kTile) > 256 || ((height + kTile - 1) / kTile) > 256)) {
        set_error("hs_project_avatar_fwd: tile_rects needs at most 256 tiles per image axis");
        return HS_ERR_SHAPE;
    }
    // the shared tile histogram (tiles padded to 4) + the tile pass's item slots (48 B per thread)
    const size_t smem = (tile_counts && tiles <= kProjHistBins ? sizeof(uint32_t) * ((tiles + 3) & ~3) : 0) +
                        ((tile_counts || tile_rects) ? 48 * (size_t)kScanBlock : 0);
    launch_k(project_avatar_fwd_kernel, hs_scan_blocks(items), kScanBlock, smem, HS_CHECK_STREAM(stream), 
        B, N, F, width, height, raw10, base14, tri_index, bary, frames, cameras, records, depth, counts,
        block_sums, depth_range, radius, zero_gsplat, zero_maxw, zero_wsums, tile_counts, tile_rects, err);
    return check_launch("hs_project_avatar_fwd");
}

int hs_project_world_fwd(int B, int64_t N, int width, int height, const float *world14, const float *cameras,
                         float *records, float *depth, uint32_t *counts, uint32_t *block_sums,
                         uint32_t *depth_range, float *radius, float *x_cam, float *cov_cam,
                         unsigned long long *err, void *stream) {
    if (B < 1 || N < 1 || width < 1 || height < 1 || width > 32767 || height > 32767) {
        set_error("hs_project_world_fwd: bad sizes B=%d N=%lld %dx%d", B, (long long)N, width, height);
        return HS_ERR_SHAPE;
    }
    const int64_t items = (int64_t)B * N;
    launch_k(project_world_fwd_kernel, hs_scan_blocks(items), kScanBlock, 0, HS_CHECK_STREAM(stream), 
        B, N, width, height, world14, cameras, records, depth, counts, block_sums, depth_range, radius, x_cam, cov_cam,
        err);
    return check_launch("hs_project_world_fwd");
}

int hs_project_avatar_bwd(int B, int64_t N, int F, const float *raw10, const float *base14,
                          const int32_t *tri_index, const float *bary, const float *frames, const float *cameras,
                          const float *g_splat, int raw_mean, float *g_raw14, void *stream) {
    const int64_t items = (int64_t)B * N;
    launch_k(project_avatar_bwd_kernel, grid_for(items, 256), 256, 0, HS_CHECK_STREAM(stream), 
        B, N, F, raw10, base14, tri_index, bary, frames, cameras, g_splat, raw_mean, g_raw14);
    return check_launch("hs_project_avatar_bwd");
}

int hs_project_world_bwd(int B, int64_t N, const float *world14, const float *cameras, const float *g_splat,
                         float *g_world14, void *stream) {
    const int64_t items = (int64_t)B * N;
    launch_k(project_world_bwd_kernel, grid_for(items, 256), 256, 0, HS_CHECK_STREAM(stream), B, N, world14, cameras,
                                                                                         g_splat, g_world14);
    return check_launch("hs_project_world_bwd");
}

}  // extern "C"
