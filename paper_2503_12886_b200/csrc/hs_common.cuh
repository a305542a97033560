// hs_common.cuh -- shared device helpers for the sm_100a RGBAvatar hot path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

#include "../../include/hs_api.h"

namespace hs {

// Device-side bounds checks of the debug build (-DHS_DEBUG_BOUNDS; compute-sanitizer is not
// available on the GPU pool): a violated index bound prints its site and traps, which
// fails the launch loudly.  Compiled out otherwise.
#ifdef HS_DEBUG_BOUNDS
#define HS_CHECK(cond, what, v)                                                                        \
    do {                                                                                               \
        if (!(cond)) {                                                                                 \
            printf("HS_CHECK failed: %s (%lld) at %s:%d block %d thread %d\n", what, (long long)(v),   \
                   __FILE__, __LINE__, (int)blockIdx.x, (int)threadIdx.x);                             \
            __trap();                                                                                  \
        }                                                                                              \
    } while (0)
#else
#define HS_CHECK(cond, what, v) \
    do {                        \
    } while (0)
#endif

// S/render.py:34-37
constexpr float kNearPlane = 0.01f;
constexpr float kMinRadius = 0.3f;
constexpr float kAlphaCutoff = 1.0f / 255.0f;
// x / 255 correctly rounded for a byte value x (0..255), without the IEEE division's
// instruction sequence: the product with the rounded reciprocal, then one FMA residual
// correction -- identical to (float)x / 255.0f for all 256 inputs (checked exhaustively
// against exact rationals, tests/test_abi.py::test_u8_unit_is_exact).
__device__ __forceinline__ float u8_unit(uint32_t x) {
    const float xf = (float)x, r = 1.0f / 255.0f;
    const float q = xf * r;
    return __fmaf_rn(__fmaf_rn(-q, 255.0f, xf), r, q);
}
constexpr float kTermEps = 1e-14f;
constexpr int kTile = 16;
constexpr int kRec = 12;            // floats per splat record
constexpr int kGS = 9;              // floats per splat gradient
constexpr int kFrame = 22;          // floats per mesh frame
constexpr int kCam = 16;            // floats per camera
constexpr int kScanBlock = 256;     // items per project/emit scan block
constexpr uint32_t kStopMask = (1u << 26) - 1u;

// error codes (see hs_api.h)
__host__ __device__ inline unsigned long long err_code(int stage, int frame, int attr, int64_t n) {
    return ((unsigned long long)stage << 62) | ((unsigned long long)frame << 40) |
           ((unsigned long long)attr << 32) | (unsigned long long)(uint32_t)n;
}

void set_error(const char *fmt, ...);
int check_launch(const char *what);
// SM count of the calling thread's current device (cached per device)
int current_sm_count();

inline unsigned grid_for(int64_t n, int threads) { return (unsigned)((n + threads - 1) / threads); }

// ---- programmatic dependent launch (PDL) -------------------------------------------
// Every kernel of the library is launched with programmatic stream serialization, and
// every kernel starts with pdl_prologue(): it lets its dependents launch right away
// (griddepcontrol.launch_dependents: the next kernel in the stream may be scheduled once
// all of this grid's CTAs are resident) and then waits until the grids it depends on have
// completed and their memory is visible (griddepcontrol.wait) -- so the next kernel's launch
// latency hides behind the tail of the previous one instead of idling the GPU between
// them.  Without a programmatic dependency both instructions are no-ops.  HS_PDL=0 in the
// environment launches normally.
__device__ __forceinline__ void pdl_prologue() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                            Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

__device__ __forceinline__ float sigmoidf_ref(float x) {
    // S/model.py:251-257 two-branch stable sigmoid
    if (x >= 0.0f) return 1.0f / (1.0f + expf(-x));
    float ex = expf(x);
    return ex / (1.0f + ex);
}

// The same two-branch sigmoid with the MUFU exp / reciprocal (a few ulp): the
// projection's activations feed only tolerance-checked values (the key list is built
// from the device's own fp32 projection, so binning stays bit-exact against it).
__device__ __forceinline__ float sigmoid_fast(float x) {
    if (x >= 0.0f) return __fdividef(1.0f, 1.0f + __expf(-x));
    const float ex = __expf(x);
    return __fdividef(ex, 1.0f + ex);
}

// S/quatmath.py:28-40 Hamilton product a (x) b
__device__ __forceinline__ void quat_mul(const float a[4], const float b[4], float o[4]) {
    o[0] = a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3];
    o[1] = a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2];
    o[2] = a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1];
    o[3] = a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0];
}

// S/quatmath.py:43-55 adjoint of b -> a (x) b
__device__ __forceinline__ void quat_mul_bwd_right(const float a[4], const float g[4], float o[4]) {
    o[0] = a[0] * g[0] + a[1] * g[1] + a[2] * g[2] + a[3] * g[3];
    o[1] = -a[1] * g[0] + a[0] * g[1] + a[3] * g[2] - a[2] * g[3];
    o[2] = -a[2] * g[0] - a[3] * g[1] + a[0] * g[2] + a[1] * g[3];
    o[3] = -a[3] * g[0] + a[2] * g[1] - a[1] * g[2] + a[0] * g[3];
}

// S/quatmath.py:58-76 (unit formula, no renormalization), row-major 3x3
__device__ __forceinline__ void quat_to_mat(const float q[4], float m[9]) {
    float w = q[0], x = q[1], y = q[2], z = q[3];
    m[0] = 1.f - 2.f * (y * y + z * z);
    m[1] = 2.f * (x * y - w * z);
    m[2] = 2.f * (x * z + w * y);
    m[3] = 2.f * (x * y + w * z);
    m[4] = 1.f - 2.f * (x * x + z * z);
    m[5] = 2.f * (y * z - w * x);
    m[6] = 2.f * (x * z - w * y);
    m[7] = 2.f * (y * z + w * x);
    m[8] = 1.f - 2.f * (x * x + y * y);
}

// S/quatmath.py:79-102
__device__ __forceinline__ void quat_to_mat_bwd(const float q[4], const float g[9], float o[4]) {
    float w = q[0], x = q[1], y = q[2], z = q[3];
    o[0] = 2.f * (x * (g[7] - g[5]) + y * (g[2] - g[6]) + z * (g[3] - g[1]));
    o[1] = 2.f * (w * (g[7] - g[5]) + y * (g[3] + g[1]) + z * (g[6] + g[2]) - 2.f * x * (g[4] + g[8]));
    o[2] = 2.f * (w * (g[2] - g[6]) + x * (g[3] + g[1]) + z * (g[7] + g[5]) - 2.f * y * (g[0] + g[8]));
    o[3] = 2.f * (w * (g[3] - g[1]) + x * (g[6] + g[2]) + y * (g[7] + g[5]) - 2.f * z * (g[0] + g[4]));
}

// S/quatmath.py:21-25 adjoint of q -> q/|q|
__device__ __forceinline__ void quat_normalize_bwd(const float q[4], const float g[4], float o[4]) {
    float nrm = sqrtf(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    float inv = 1.0f / nrm;
    float y0 = q[0] * inv, y1 = q[1] * inv, y2 = q[2] * inv, y3 = q[3] * inv;
    float dot = y0 * g[0] + y1 * g[1] + y2 * g[2] + y3 * g[3];
    o[0] = (g[0] - y0 * dot) * inv;
    o[1] = (g[1] - y1 * dot) * inv;
    o[2] = (g[2] - y2 * dot) * inv;
    o[3] = (g[3] - y3 * dot) * inv;
}

__device__ __forceinline__ uint32_t pack_lohi(int lo, int hi) {
    return (uint32_t)(lo & 0xFFFF) | ((uint32_t)(hi & 0xFFFF) << 16);
}
__device__ __forceinline__ int unpack_lo(uint32_t v) { return (int)(int16_t)(v & 0xFFFF); }
__device__ __forceinline__ int unpack_hi(uint32_t v) { return (int)(int16_t)(v >> 16); }

// The binning's tile cull (tile-major path, oracle/binning.py:tile_reaches): can splat (mean,
// conic a b c, qmax, integer pixel bbox [rl, rh] x [cl, ch]) reach a pixel of tile (tx, ty)?
// The minimum of q(d) = a dx^2 + 2 b dx dy + c dy^2 over the rectangle of the tile's pixel
// centres inside the bbox (d = centre - mean): for a positive-definite q the minimiser lies
// on one of the two segments through the point nearest the mean (x clamped with the best y
// for it, and y clamped with the best x), both inside the rectangle; q there is the minimum
// up to second-order rounding.  No pixel can pass the reference's q <= qmax test
// (S/render.py:260-262) when it exceeds qmax by the margin (0.1 % + 1e-3, far above the fp32
// rounding of q at a pixel).  IEEE fp32, one rounding per operation, inv_a / inv_c the
// correctly rounded reciprocals (TileCull), so every emitter and the oracle decide alike;
// non-positive-definite or non-finite input keeps the tile.
struct TileCull {
    float mx, my, a, b, c, qmax, inv_a, inv_c;
    int rl, rh, cl, ch;
    bool pd;
};
__device__ __forceinline__ TileCull tile_cull(float mx, float my, float a, float b, float c, float qmax, int rl, int rh,
                                              int cl, int ch) {
    TileCull t;
    t.mx = mx; t.my = my; t.a = a; t.b = b; t.c = c; t.qmax = qmax;
    t.rl = rl; t.rh = rh; t.cl = cl; t.ch = ch;
    const float det = __fsub_rn(__fmul_rn(a, c), __fmul_rn(b, b));
    t.pd = det > 0.f && a > 0.f && c > 0.f;
    t.inv_a = t.pd ? __frcp_rn(a) : 0.f;
    t.inv_c = t.pd ? __frcp_rn(c) : 0.f;
    return t;
}
__device__ __forceinline__ bool tile_reaches(const TileCull &t, int tx, int ty) {
    const int xs = max(tx * kTile, t.cl), xe = min(tx * kTile + kTile - 1, t.ch);
    const int ys = max(ty * kTile, t.rl), ye = min(ty * kTile + kTile - 1, t.rh);
    if (xs > xe || ys > ye) return false;
    if (!t.pd) return true;
    const float dxlo = __fsub_rn(__fadd_rn((float)xs, 0.5f), t.mx), dxhi = __fsub_rn(__fadd_rn((float)xe, 0.5f), t.mx);
    const float dylo = __fsub_rn(__fadd_rn((float)ys, 0.5f), t.my), dyhi = __fsub_rn(__fadd_rn((float)ye, 0.5f), t.my);
    const float dxv = fminf(fmaxf(0.f, dxlo), dxhi);
    const float dyv = fminf(fmaxf(__fmul_rn(__fmul_rn(-t.b, dxv), t.inv_c), dylo), dyhi);
    const float dyh = fminf(fmaxf(0.f, dylo), dyhi);
    const float dxh = fminf(fmaxf(__fmul_rn(__fmul_rn(-t.b, dyh), t.inv_a), dxlo), dxhi);
    const float b2 = __fmul_rn(2.f, t.b);
    const float qv = __fadd_rn(__fadd_rn(__fmul_rn(__fmul_rn(t.a, dxv), dxv), __fmul_rn(__fmul_rn(b2, dxv), dyv)),
                               __fmul_rn(__fmul_rn(t.c, dyv), dyv));
    const float qh = __fadd_rn(__fadd_rn(__fmul_rn(__fmul_rn(t.a, dxh), dxh), __fmul_rn(__fmul_rn(b2, dxh), dyh)),
                               __fmul_rn(__fmul_rn(t.c, dyh), dyh));
    return !(__fsub_rn(__fmul_rn(fminf(qv, qh), 0.999f), 1e-3f) > t.qmax);
}
// Position of the n-th (0-based) set bit of m (n < popc(m)): a branch-free popc search
// (__fns compiles to a loop)
__device__ __forceinline__ uint32_t nth_set_bit(uint32_t m, uint32_t n) {
    uint32_t pos = 0;
#pragma unroll
    for (int w = 16; w; w >>= 1) {
        const uint32_t c = __popc(m & ((1u << w) - 1u));
        const bool hi = n >= c;
        n = hi ? n - c : n;
        m = hi ? m >> w : m;
        pos = hi ? pos + w : pos;
    }
    return pos;
}
// Tile rectangles of at most kMaskTiles tiles carry a kept-tile mask (bit dy * w + dx);
// larger ones keep every tile (mask all ones).
constexpr int kMaskTiles = 32;
__device__ __forceinline__ bool mask_keeps(uint32_t mask, int area, int idx) {
    return area > kMaskTiles || ((mask >> idx) & 1u);
}

// i / N for a (frame, Gaussian) item index: 32-bit when both fit (always, in practice; a
// 64-bit division is ~70 instructions)
__device__ __forceinline__ int64_t item_frame(int64_t i, int64_t N) {
    if (((uint64_t)i | (uint64_t)N) < (1ull << 32)) return (int64_t)((uint32_t)i / (uint32_t)N);
    return i / N;
}

__host__ __device__ inline int bit_length_u32(uint32_t x) {
    int n = 0;
    while (x) { ++n; x >>= 1; }
    return n;
}

// Warp reduce-scatter of S values: each round halves the slot count, exchanging
// only the half the partner keeps (S=9: 12 shuffles instead of 45).  On return the
// lane holds the warp total of value `idx`; exactly one lane per value has `issue`.
template <int S, int R>
struct ReduceScatter {
    static __device__ __forceinline__ float run(const float *w, int lane, int &idx, int &cnt, int &dup) {
        constexpr int O = 16 >> R;
        if constexpr (R == 5) {
            return w[0];
        } else if constexpr (S == 1) {
            const float t[1] = {w[0] + __shfl_xor_sync(0xffffffffu, w[0], O)};
            dup |= O;
            return ReduceScatter<1, R + 1>::run(t, lane, idx, cnt, dup);
        } else {
            constexpr int L = (S + 1) / 2;
            const bool up = lane & O;
            float nw[L];
#pragma unroll
            for (int s = 0; s < L; ++s) {
                const float hi = (L + s < S) ? w[L + s] : 0.f;
                const float lo = w[s];
                nw[s] = (up ? hi : lo) + __shfl_xor_sync(0xffffffffu, up ? lo : hi, O);
            }
            if (up) {
                idx += L;
                cnt -= L;
            } else {
                cnt = min(cnt, L);
            }
            return ReduceScatter<L, R + 1>::run(nw, lane, idx, cnt, dup);
        }
    }
};

template <int S>
__device__ __forceinline__ float reduce_scatter(const float (&v)[S], int lane, int &idx, bool &issue) {
    int cnt = S, dup = 0;
    idx = 0;
    const float r = ReduceScatter<S, 0>::run(v, lane, idx, cnt, dup);
    issue = cnt >= 1 && (lane & dup) == 0;
    return r;
}

// the value only (the slot index is a function of the lane: compute it once)
template <int S>
__device__ __forceinline__ float reduce_scatter_value(const float (&v)[S], int lane) {
    int cnt = S, dup = 0, idx = 0;
    return ReduceScatter<S, 0>::run(v, lane, idx, cnt, dup);
}

// ---- 1D bulk async copies (the TMA engine without a tensor map) + mbarriers ----------
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// global -> shared, `bytes` a multiple of 16 with both addresses 16-byte aligned; completes
// `bytes` transactions on `bar`
__device__ __forceinline__ void bulk_g2s(void *dst_smem, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst_smem)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace hs

#define HS_CHECK_STREAM(s) (reinterpret_cast<cudaStream_t>(s))
