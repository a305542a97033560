// hs_model.cu -- reduced-blendshape model ops on sm_100a: MLP, blend (+adjoint),
// multi-group Adam, colour-init apply, and the elementwise compat ops.
//
// Reference: S/model.py (map_params :130, mlp_backward :145, blend :165,
// blend_backward :188, activate :219, activate_backward :237), S/optim.py:28-40,
// S/train.py:164-199 (Adam groups), :253-255 (item-order reduce), :263-278 and
// S/color_init.py:45-80 (colour init), S/binding.py:174-204 (transform).
#include <cstdarg>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <cmath>

#include "hs_common.cuh"

namespace hs {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

bool pdl_enabled() {
    static const bool on = [] {
        const char *e = getenv("HS_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

int current_sm_count() {
    static int cache[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    if (dev < 0 || dev >= 64) dev = 0;
    int v = __atomic_load_n(&cache[dev], __ATOMIC_RELAXED);
    if (v == 0) {
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
        __atomic_store_n(&cache[dev], v, __ATOMIC_RELAXED);
    }
    return v;
}

int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: %s", what, cudaGetErrorString(e));
        return HS_ERR_CUDA;
    }
    return HS_OK;
}

// ------------------------------------------------------------------- MLP

// One CTA per frame.  S/model.py:130-142.  Each GEMV row is one warp-cooperative
// dot product (lanes split the row: coalesced loads, many in flight).
__device__ __forceinline__ float row_dot(const float *__restrict__ row, const float *__restrict__ x, int n, int lane) {
    float acc = 0.f;
#pragma unroll 4
    for (int j = lane; j < n; j += 32) acc = fmaf(row[j], x[j], acc);
    return warp_sum(acc);
}

__global__ void mlp_fwd_kernel(int H, int D, int K, const float *__restrict__ mlp,
                               const float *__restrict__ theta, float *__restrict__ cache,
                               float *__restrict__ psi, unsigned long long *err) {
    pdl_prologue();
    extern __shared__ float sm[];
    float *th = sm, *h1 = th + H, *h2 = h1 + D;
    const int b = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const float *w1 = mlp, *b1 = w1 + D * H, *w2 = b1 + D, *b2 = w2 + D * D, *w3 = b2 + D, *b3 = w3 + K * D;
    for (int i = threadIdx.x; i < H; i += blockDim.x) {
        float t = theta[b * H + i];
        th[i] = t;
        if (!isfinite(t)) atomicMin(err, err_code(0, b, 0, 0));
    }
    __syncthreads();
    float *c = cache + (int64_t)b * 4 * D;
    // layer 1 is narrow (H = 13): one thread per output row, loads issued back to back
    for (int i = threadIdx.x; i < D; i += blockDim.x) {
        const float *row = w1 + (int64_t)i * H;
        float acc = 0.f;
#pragma unroll 8
        for (int j = 0; j < H; ++j) acc = fmaf(row[j], th[j], acc);
        const float z = acc + b1[i];
        const float h = z > 0.f ? z : 0.f;
        c[i] = z;
        c[D + i] = h;
        h1[i] = h;
    }
    __syncthreads();
    for (int i = warp; i < D; i += nw) {
        const float z = row_dot(w2 + (int64_t)i * D, h1, D, lane) + b2[i];
        if (lane == 0) {
            const float h = z > 0.f ? z : 0.f;
            c[2 * D + i] = z;
            c[3 * D + i] = h;
            h2[i] = h;
        }
    }
    __syncthreads();
    for (int k = warp; k < K; k += nw) {
        const float p = row_dot(w3 + (int64_t)k * D, h2, D, lane) + b3[k];
        if (lane == 0) psi[b * K + k] = p;
    }
}

// Per frame: reduce the blend_bwd partials into g_psi (fixed order), then the
// hidden-layer adjoints gz2 = relu'(z2) W3^T g_psi and gz1 = relu'(z1) W2^T gz2
// (S/model.py:151-160).  The transposed GEMVs walk W rows (coalesced) with each
// warp owning a slice of rows; warp partials are summed through shared memory.
__global__ void mlp_bwd_frame_kernel(int H, int D, int K, const float *__restrict__ mlp,
                                     const float *__restrict__ cache,
                                     const float *__restrict__ partials, int P,
                                     float *__restrict__ gpsi, float *__restrict__ scratch) {
    pdl_prologue();
    extern __shared__ float sm[];
    const int nw = blockDim.x >> 5;
    float *gp = sm, *gz2 = gp + K, *part = gz2 + D;     // part: [nw][D]
    const int b = blockIdx.x;
    const int B = gridDim.x;
    const float *w2 = mlp + D * H + D, *w3 = w2 + D * D + D;
    const float *c = cache + (int64_t)b * 4 * D;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int k = warp; k < K; k += nw) {
        const float *row = partials + ((int64_t)b * K + k) * P;
        float s = 0.f;
        for (int p = lane; p < P; p += 32) s += row[p];
        s = warp_sum(s);
        if (lane == 0) {
            gp[k] = s;
            gpsi[b * K + k] = s;
        }
    }
    __syncthreads();
    float *s_gz2 = scratch + (int64_t)b * D;             // [B][D]
    float *s_gz1 = scratch + (int64_t)B * D + (int64_t)b * D;
    // gz2[j] = sum_k w3[k][j] gp[k]   (K rows of length D)
    for (int j = threadIdx.x; j < D; j += blockDim.x) {
        float acc = 0.f;
#pragma unroll 4
        for (int k = 0; k < K; ++k) acc = fmaf(w3[(int64_t)k * D + j], gp[k], acc);
        const float g = c[2 * D + j] > 0.f ? acc : 0.f;
        gz2[j] = g;
        s_gz2[j] = g;
    }
    __syncthreads();
    // gz1[j] = sum_i w2[i][j] gz2[i]: warp w sums rows i = w, w + nw, ...
    for (int j = lane; j < D; j += 32) {
        float acc = 0.f;
#pragma unroll 4
        for (int i = warp; i < D; i += nw) acc = fmaf(w2[(int64_t)i * D + j], gz2[i], acc);
        part[warp * D + j] = acc;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < D; j += blockDim.x) {
        float acc = 0.f;
        for (int w = 0; w < nw; ++w) acc += part[w * D + j];
        s_gz1[j] = c[j] > 0.f ? acc : 0.f;
    }
}

// One thread per MLP parameter, frames summed in order b = 0..B-1.
__global__ void mlp_bwd_weights_kernel(int B, int H, int D, int K, const float *__restrict__ theta,
                                       const float *__restrict__ cache,
                                       const float *__restrict__ gpsi,
                                       const float *__restrict__ scratch, float *__restrict__ g) {
    pdl_prologue();
    const int64_t total = (int64_t)D * H + D + (int64_t)D * D + D + (int64_t)K * D + K;
    const float *gz2 = scratch, *gz1 = scratch + (int64_t)B * D;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = i;
        float acc = 0.f;
        if (r < (int64_t)D * H) {                   // w1[i][j] += gz1[i] theta[j]
            int ii = r / H, j = r % H;
            for (int b = 0; b < B; ++b) acc += gz1[b * D + ii] * theta[b * H + j];
        } else if ((r -= (int64_t)D * H) < D) {     // b1
            for (int b = 0; b < B; ++b) acc += gz1[b * D + r];
        } else if ((r -= D) < (int64_t)D * D) {     // w2[i][j] += gz2[i] h1[j]
            int ii = r / D, j = r % D;
            for (int b = 0; b < B; ++b) acc += gz2[b * D + ii] * cache[(int64_t)b * 4 * D + D + j];
        } else if ((r -= (int64_t)D * D) < D) {     // b2
            for (int b = 0; b < B; ++b) acc += gz2[b * D + r];
        } else if ((r -= D) < (int64_t)K * D) {     // w3[k][j] += gpsi[k] h2[j]
            int k = r / D, j = r % D;
            for (int b = 0; b < B; ++b) acc += gpsi[b * K + k] * cache[(int64_t)b * 4 * D + 3 * D + j];
        } else {                                    // b3
            r -= (int64_t)K * D;
            for (int b = 0; b < B; ++b) acc += gpsi[b * K + r];
        }
        g[i] = acc;
    }
}

// ----------------------------------------------------------------- blend

// raw[b] = base + sum_k psi[b,k] delta_k (S/model.py:165-185: k ascending, fmaf, psi == 0
// skipped), TMA-staged: a persistent CTA streams 512-channel tiles of the K delta rows and
// the base row into shared memory with 1D bulk async copies (one elected thread, an mbarrier
// per stage, two stages), so ~42 KB per CTA are in flight with no register staging; its 256
// threads then own 2 channels x all frames each, reading the deltas from shared memory
// (psi, transposed, broadcast from shared memory four frames per load) and storing each
// frame's 2 KB row of raw coalesced.  Every delta byte is read from HBM once per step.
#ifndef HS_BLEND_TE
#define HS_BLEND_TE 256
#endif
#ifndef HS_BLEND_STAGES
#define HS_BLEND_STAGES 2
#endif
constexpr int kBfTE = HS_BLEND_TE;        // channels per tile
constexpr int kBfT = kBfTE / 2;           // threads per CTA (2 channels each)
constexpr int kBfS = HS_BLEND_STAGES;     // pipeline stages

__host__ __device__ inline int blend_fwd_bc(int B) { return B <= 4 ? 4 : B <= 8 ? 8 : 16; }
__host__ __device__ inline int blend_fwd_bpad(int B) {
    const int bc = blend_fwd_bc(B);
    return (B + bc - 1) / bc * bc;
}
__host__ inline size_t blend_fwd_smem(int K, int B) {
    return 64 + sizeof(float) * (2 * (size_t)K * blend_fwd_bpad(B) + kBfS * (size_t)(K + 1) * kBfTE);
}

// One tile: thread owns channels (c, c+1); frames in chunks of BC accumulators (pairs of
// channels, updated with FFMA2 -- per element exactly fmaf(psi, delta, acc)).  s_psi2 holds
// psi[b][k] twice per frame ([k][Bp][2]) so one LDS.128 yields two frames' (w, w) pairs.
template <int BC, bool kAllNonzero>
__device__ __forceinline__ void blend_fwd_tile(int64_t E, int K, int B, int Bp, const float *s_psi2,
                                               const float *stage, int64_t e0, float *__restrict__ raw) {
    const int c = 2 * threadIdx.x;
    const int64_t e = e0 + c;
    if (e >= E) return;
    const float2 bv = *reinterpret_cast<const float2 *>(stage + (size_t)K * kBfTE + c);
    for (int b0 = 0; b0 < B; b0 += BC) {
        float2 acc[BC];
#pragma unroll
        for (int j = 0; j < BC; ++j) acc[j] = bv;
        #pragma unroll 4
        for (int k = 0; k < K; ++k) {
            const float2 d = *reinterpret_cast<const float2 *>(stage + (size_t)k * kBfTE + c);
            const float4 *w = reinterpret_cast<const float4 *>(s_psi2 + ((size_t)k * Bp + b0) * 2);
#pragma unroll
            for (int j2 = 0; j2 < BC / 2; ++j2) {
                const float4 w4 = w[j2];                       // (w_j, w_j, w_j+1, w_j+1)
                if (kAllNonzero) {
                    acc[2 * j2] = __ffma2_rn(make_float2(w4.x, w4.y), d, acc[2 * j2]);
                    acc[2 * j2 + 1] = __ffma2_rn(make_float2(w4.z, w4.w), d, acc[2 * j2 + 1]);
                } else {
                    if (w4.x != 0.0f) acc[2 * j2] = __ffma2_rn(make_float2(w4.x, w4.y), d, acc[2 * j2]);
                    if (w4.z != 0.0f) acc[2 * j2 + 1] = __ffma2_rn(make_float2(w4.z, w4.w), d, acc[2 * j2 + 1]);
                }
            }
        }
#pragma unroll
        for (int j = 0; j < BC; ++j)
            if (b0 + j < B) __stcs(reinterpret_cast<float2 *>(raw + (int64_t)(b0 + j) * E + e), acc[j]);
    }
}

// HS_BLEND_V2: thread owns channels 4 cg .. 4 cg + 3 of the tile and one half of the
// frames (FB = Bp / 2 of them): per basis one LDS.128 of deltas and FB / 4 LDS.128 of
// weights feed 2 FB FFMA2 (the weight is the packed instruction's broadcast operand, so
// psi is stored once per frame); per element still exactly fmaf(psi, delta, acc).
#ifndef HS_BLEND_V2
#define HS_BLEND_V2 1
#endif
#ifndef HS_BF_DIAG
#define HS_BF_DIAG 0                 // diagnostics: 1 loads only, 2 no stores
#endif
template <int FB, bool kAllNonzero>
__device__ __forceinline__ void blend_fwd_tile4(int64_t E, int K, int B, int Bp, const float *s_psi,
                                                const float *stage, int64_t e0, float *__restrict__ raw) {
    constexpr int kGroups = kBfTE / 4;                 // channel groups per tile
    const int cg = threadIdx.x % kGroups, fg = threadIdx.x / kGroups;
    const int c = 4 * cg;
    const int64_t e = e0 + c;
    if (e >= E) return;
    const float4 bv = *reinterpret_cast<const float4 *>(stage + (size_t)K * kBfTE + c);
    for (int f0 = fg * FB; f0 < B; f0 += 2 * FB) {          // (Bp > 2 FB: frame blocks in turn)
        float2 acc[FB][2];
#pragma unroll
        for (int j = 0; j < FB; ++j) {
            acc[j][0] = make_float2(bv.x, bv.y);
            acc[j][1] = make_float2(bv.z, bv.w);
        }
#pragma unroll 2
        for (int k = 0; k < K; ++k) {
            const float4 d = *reinterpret_cast<const float4 *>(stage + (size_t)k * kBfTE + c);
            const float2 d01 = make_float2(d.x, d.y), d23 = make_float2(d.z, d.w);
            float w[FB];
            if constexpr (FB >= 4) {
#pragma unroll
                for (int q = 0; q < FB / 4; ++q) {
                    const float4 w4 = *reinterpret_cast<const float4 *>(s_psi + (size_t)k * Bp + f0 + 4 * q);
                    w[4 * q] = w4.x;
                    w[4 * q + 1] = w4.y;
                    w[4 * q + 2] = w4.z;
                    w[4 * q + 3] = w4.w;
                }
            } else {
#pragma unroll
                for (int q = 0; q < FB; ++q) w[q] = s_psi[(size_t)k * Bp + f0 + q];
            }
#pragma unroll
            for (int j = 0; j < FB; ++j) {
                if (kAllNonzero || w[j] != 0.0f) {
                    acc[j][0] = __ffma2_rn(make_float2(w[j], w[j]), d01, acc[j][0]);
                    acc[j][1] = __ffma2_rn(make_float2(w[j], w[j]), d23, acc[j][1]);
                }
            }
        }
#pragma unroll
        for (int j = 0; j < FB; ++j)
            if (f0 + j < B && (HS_BF_DIAG != 2 || acc[j][0].x == 1234.5f))
                __stcs(reinterpret_cast<float4 *>(raw + (int64_t)(f0 + j) * E + e),
                       make_float4(acc[j][0].x, acc[j][0].y, acc[j][1].x, acc[j][1].y));
    }
}

__global__ void __launch_bounds__(kBfT) blend_fwd_tma_kernel(int64_t E, int K, int B, const float *__restrict__ base,
                                                             const float *__restrict__ deltas,
                                                             const float *__restrict__ psi, float *__restrict__ raw) {
    pdl_prologue();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw);
    const int Bp = blend_fwd_bpad(B);
    float *s_psi2 = reinterpret_cast<float *>(smem_raw + 64);          // [K][Bp][2]
    float *stages = s_psi2 + 2 * K * Bp;                                 // kBfS x [(K + 1)][kBfTE]
    const int64_t ntiles = (E + kBfTE - 1) / kBfTE;
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int st = 0; st < kBfS; ++st) mbar_init(&bars[st], 1);
        mbar_fence_init();
    }
    int nz = 1;
    for (int i = tid; i < K * Bp; i += kBfT) {
        const int k = i / Bp, b = i % Bp;
        const float w = b < B ? psi[b * K + k] : 0.f;
        if (HS_BLEND_V2) {
            s_psi2[i] = w;                                   // [K][Bp]
        } else {
            s_psi2[2 * i] = w;
            s_psi2[2 * i + 1] = w;
        }
        nz &= (b >= B) || (w != 0.0f);
    }
    const bool all_nonzero = __syncthreads_and(nz);
    auto issue = [&](int64_t t, int st) {
        const int64_t e0 = t * kBfTE;
        const uint32_t bytes = (uint32_t)((E - e0 < kBfTE ? E - e0 : (int64_t)kBfTE) * 4);
        float *dst = stages + (size_t)st * (K + 1) * kBfTE;
        mbar_expect_tx(&bars[st], bytes * (K + 1));
        for (int k = 0; k < K; ++k) bulk_g2s(dst + (size_t)k * kBfTE, deltas + (int64_t)k * E + e0, bytes, &bars[st]);
        bulk_g2s(dst + (size_t)K * kBfTE, base + e0, bytes, &bars[st]);
    };
    if (tid == 0) {
        for (int st = 0; st < kBfS; ++st)
            if (blockIdx.x + (int64_t)st * gridDim.x < ntiles) issue(blockIdx.x + (int64_t)st * gridDim.x, st);
    }
    uint32_t phase = 0;         // bit st: parity of stage st's next completion
    int it = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int st = it % kBfS;
        mbar_wait(&bars[st], (phase >> st) & 1u);
        phase ^= 1u << st;
        const float *stage = stages + (size_t)st * (K + 1) * kBfTE;
        const int64_t e0 = t * kBfTE;
        if (HS_BF_DIAG == 1) {
            if (stage[threadIdx.x] == 1234.5f) raw[threadIdx.x] = 0.f;     // loads only
        } else if (HS_BLEND_V2) {
            if (Bp <= 4) {
                if (all_nonzero) blend_fwd_tile4<2, true>(E, K, B, Bp, s_psi2, stage, e0, raw);
                else blend_fwd_tile4<2, false>(E, K, B, Bp, s_psi2, stage, e0, raw);
            } else if (Bp <= 8) {
                if (all_nonzero) blend_fwd_tile4<4, true>(E, K, B, Bp, s_psi2, stage, e0, raw);
                else blend_fwd_tile4<4, false>(E, K, B, Bp, s_psi2, stage, e0, raw);
            } else {
                if (all_nonzero) blend_fwd_tile4<8, true>(E, K, B, Bp, s_psi2, stage, e0, raw);
                else blend_fwd_tile4<8, false>(E, K, B, Bp, s_psi2, stage, e0, raw);
            }
        } else if (Bp <= 4) {
            if (all_nonzero) blend_fwd_tile<4, true>(E, K, B, Bp, s_psi2, stage, e0, raw);
            else blend_fwd_tile<4, false>(E, K, B, Bp, s_psi2, stage, e0, raw);
        } else if (Bp <= 8) {
            if (all_nonzero) blend_fwd_tile<8, true>(E, K, B, Bp, s_psi2, stage, e0, raw);
            else blend_fwd_tile<8, false>(E, K, B, Bp, s_psi2, stage, e0, raw);
        } else {
            if (all_nonzero) blend_fwd_tile<16, true>(E, K, B, Bp, s_psi2, stage, e0, raw);
            else blend_fwd_tile<16, false>(E, K, B, Bp, s_psi2, stage, e0, raw);
        }
        __syncthreads();                      // every thread is done with this stage
        if (tid == 0 && t + kBfS * (int64_t)gridDim.x < ntiles) issue(t + kBfS * (int64_t)gridDim.x, st);
    }
}

// Rows only 8-byte aligned (odd N: E = 10 N = 2 mod 4, and the deltas start at float 14 N of
// the parameters): the same TMA pipeline, shared row stride TE + 4.  A row whose address is
// 8 mod 16 is copied from 2 floats before the tile (its compute offset 2); the first tile
// copies from 2 floats after the row start instead (nothing before a row is read), and the
// aligned rows' 2-float tails on the last tile (a bulk copy moves multiples of 16 bytes) are
// read by threads.  Compute as blend_fwd_tile4, with 8-byte shared loads on the offset rows
// and 8-byte stores into the frames whose output row is offset.
constexpr int kBmRS = kBfTE + 4;
#ifndef HS_BLEND_MIS_WIDE_B
#define HS_BLEND_MIS_WIDE_B 16
#endif
__host__ inline size_t blend_fwd_mis_smem(int K, int B) {
    return 64 + sizeof(float) * ((size_t)K * blend_fwd_bpad(B) + kBfS * (size_t)(K + 1) * kBmRS);
}
__device__ __forceinline__ int row_off(const float *rowp) { return ((uintptr_t)rowp & 15u) ? 2 : 0; }
template <int FB, bool kAllNonzero>
__device__ __forceinline__ void blend_fwd_tile4_mis(int64_t E, int K, int B, int Bp, const float *s_psi,
                                                    const float *stage, int64_t e0, const float *__restrict__ deltas,
                                                    const float *__restrict__ base, float *__restrict__ raw) {
    constexpr int kGroups = kBfTE / 4;
    const int cg = threadIdx.x % kGroups, fg = threadIdx.x / kGroups, ng = blockDim.x / kGroups;
    const int c = 4 * cg;
    const int64_t e = e0 + c;
    if (e >= E) return;
    const bool full = e + 4 <= E;                      // (else 2 channels: E = 2 mod 4)
    const float *brow = stage + (size_t)K * kBmRS + row_off(base) + c;
    const float2 b01 = *reinterpret_cast<const float2 *>(brow), b23 = *reinterpret_cast<const float2 *>(brow + 2);
    for (int f0 = fg * FB; f0 < B; f0 += ng * FB) {
        float2 acc[FB][2];
#pragma unroll
        for (int j = 0; j < FB; ++j) {
            acc[j][0] = b01;
            acc[j][1] = b23;
        }
#pragma unroll 2
        for (int k = 0; k < K; ++k) {
            const float *row = stage + (size_t)k * kBmRS + row_off(deltas + (int64_t)k * E) + c;
            const float2 d01 = *reinterpret_cast<const float2 *>(row), d23 = *reinterpret_cast<const float2 *>(row + 2);
            float w[FB];
            if constexpr (FB >= 4) {
#pragma unroll
                for (int q = 0; q < FB / 4; ++q) {
                    const float4 w4 = *reinterpret_cast<const float4 *>(s_psi + (size_t)k * Bp + f0 + 4 * q);
                    w[4 * q] = w4.x;
                    w[4 * q + 1] = w4.y;
                    w[4 * q + 2] = w4.z;
                    w[4 * q + 3] = w4.w;
                }
            } else {
#pragma unroll
                for (int q = 0; q < FB; ++q) w[q] = s_psi[(size_t)k * Bp + f0 + q];
            }
#pragma unroll
            for (int j = 0; j < FB; ++j) {
                if (kAllNonzero || w[j] != 0.0f) {
                    acc[j][0] = __ffma2_rn(make_float2(w[j], w[j]), d01, acc[j][0]);
                    acc[j][1] = __ffma2_rn(make_float2(w[j], w[j]), d23, acc[j][1]);
                }
            }
        }
#pragma unroll
        for (int j = 0; j < FB; ++j) {
            const int f = f0 + j;
            if (f >= B) continue;
            float *o = raw + (int64_t)f * E + e;
            if (full && ((uintptr_t)o & 15u) == 0) {
                __stcs(reinterpret_cast<float4 *>(o), make_float4(acc[j][0].x, acc[j][0].y, acc[j][1].x, acc[j][1].y));
            } else {
                __stcs(reinterpret_cast<float2 *>(o), acc[j][0]);
                if (full) __stcs(reinterpret_cast<float2 *>(o + 2), acc[j][1]);
            }
        }
    }
}

// row r (< K: delta row r, K: base) for the tile at e0: the bulk copy global [src, src + len)
// -> shared index dst, and up to 2 floats (global g, shared index g - e0 + off) for threads
struct RowPlan {
    const float *rowp;
    int64_t src, len;
    int dst, off, nfill;
    int64_t fill[8];
};
__device__ __forceinline__ RowPlan row_plan(int r, int64_t e0, int64_t E, int K, const float *deltas,
                                            const float *base) {
    RowPlan p;
    p.rowp = r < K ? deltas + (int64_t)r * E : base;
    p.off = row_off(p.rowp);
    if (p.off && e0 > 0) {                    // from 2 floats before the tile
        p.src = e0 - 2;
        p.dst = 0;
    } else if (p.off) {                       // the first tile: from float 2 (nothing before the row)
        p.src = 2;
        p.dst = 4;
    } else {
        p.src = e0;
        p.dst = 0;
    }
    p.len = max((int64_t)0, min((int64_t)(kBmRS - p.dst), E - p.src)) & ~(int64_t)3;
    // the floats the tile's compute reads that the copy does not cover (first / last tile)
    const int64_t hi = min(e0 + (int64_t)kBfTE, E);
    p.nfill = 0;
    for (int64_t g = e0; g < min(p.src, hi); ++g) p.fill[p.nfill++] = g;
    for (int64_t g = max(p.src + p.len, e0); g < hi && p.nfill < 8; ++g) p.fill[p.nfill++] = g;
    return p;
}

__global__ void __launch_bounds__(2 * kBfT) blend_fwd_tma_mis_kernel(int64_t E, int K, int B,
                                                                 const float *__restrict__ base,
                                                                 const float *__restrict__ deltas,
                                                                 const float *__restrict__ psi,
                                                                 float *__restrict__ raw) {
    pdl_prologue();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw);
    const int Bp = blend_fwd_bpad(B);
    float *s_psi = reinterpret_cast<float *>(smem_raw + 64);           // [K][Bp]
    float *stages = s_psi + K * Bp;                                      // kBfS x [(K + 1)][kBmRS]
    const int64_t ntiles = (E + kBfTE - 1) / kBfTE;
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int st = 0; st < kBfS; ++st) mbar_init(&bars[st], 1);
        mbar_fence_init();
    }
    int nz = 1;
    for (int i = tid; i < K * Bp; i += blockDim.x) {
        const int k = i / Bp, b = i % Bp;
        const float w = b < B ? psi[b * K + k] : 0.f;
        s_psi[i] = w;
        nz &= (b >= B) || (w != 0.0f);
    }
    const bool all_nonzero = __syncthreads_and(nz);
    auto issue = [&](int64_t t, int st) {
        const int64_t e0 = t * kBfTE;
        float *dst = stages + (size_t)st * (K + 1) * kBmRS;
        uint32_t bytes = 0;
        for (int r = 0; r <= K; ++r) bytes += (uint32_t)(row_plan(r, e0, E, K, deltas, base).len * 4);
        mbar_expect_tx(&bars[st], bytes);
        for (int r = 0; r <= K; ++r) {
            const RowPlan p = row_plan(r, e0, E, K, deltas, base);
            if (p.len > 0) bulk_g2s(dst + (size_t)r * kBmRS + p.dst, p.rowp + p.src, (uint32_t)(p.len * 4), &bars[st]);
        }
    };
    if (tid == 0) {
        for (int st = 0; st < kBfS; ++st)
            if (blockIdx.x + (int64_t)st * gridDim.x < ntiles) issue(blockIdx.x + (int64_t)st * gridDim.x, st);
    }
    uint32_t phase = 0;
    int it = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int st = it % kBfS;
        mbar_wait(&bars[st], (phase >> st) & 1u);
        phase ^= 1u << st;
        float *stage = stages + (size_t)st * (K + 1) * kBmRS;
        const int64_t e0 = t * kBfTE;
        if (e0 == 0 || e0 + kBfTE > E) {        // the first / last tile: the floats no copy moved
            for (int r = tid; r <= K; r += blockDim.x) {
                const RowPlan p = row_plan(r, e0, E, K, deltas, base);
                for (int q = 0; q < p.nfill; ++q)
                    stage[(size_t)r * kBmRS + (p.fill[q] - e0 + p.off)] = p.rowp[p.fill[q]];
            }
            __syncthreads();
        }
        if (Bp <= 4) {
            if (all_nonzero) blend_fwd_tile4_mis<2, true>(E, K, B, Bp, s_psi, stage, e0, deltas, base, raw);
            else blend_fwd_tile4_mis<2, false>(E, K, B, Bp, s_psi, stage, e0, deltas, base, raw);
        } else if (Bp <= 8) {
            if (all_nonzero) blend_fwd_tile4_mis<4, true>(E, K, B, Bp, s_psi, stage, e0, deltas, base, raw);
            else blend_fwd_tile4_mis<4, false>(E, K, B, Bp, s_psi, stage, e0, deltas, base, raw);
        } else {
            if (all_nonzero) blend_fwd_tile4_mis<8, true>(E, K, B, Bp, s_psi, stage, e0, deltas, base, raw);
            else blend_fwd_tile4_mis<8, false>(E, K, B, Bp, s_psi, stage, e0, deltas, base, raw);
        }
        __syncthreads();                      // every thread is done with this stage
        if (tid == 0 && t + kBfS * (int64_t)gridDim.x < ntiles) issue(t + kBfS * (int64_t)gridDim.x, st);
    }
}

// raw[b] = base + sum_k psi[b,k] delta_k over the 10N blended channels.  Each
// thread owns VEC consecutive channels and keeps BC frames of accumulators, so
// every delta element is read from HBM once per BC frames (once per step for
// B <= BC).  S/model.py:165-185 (k ascending, psi == 0 skipped).
#ifndef HS_BLEND_KB
#define HS_BLEND_KB 4
#endif
constexpr int kKB = HS_BLEND_KB;
#ifndef HS_BLEND_FWD_PF
#define HS_BLEND_FWD_PF 0   // 1: next round prefetched (111 registers; measured 33 -> 39 us, slower)
#endif
template <int VEC, int BC>
__global__ void __launch_bounds__(256) blend_fwd_kernel(int64_t E, int K, int B,
                                                        const float *__restrict__ base,
                                                        const float *__restrict__ deltas,
                                                        const float *__restrict__ psi,
                                                        float *__restrict__ raw) {
    pdl_prologue();
    extern __shared__ float s_psi[];
    for (int i = threadIdx.x; i < B * K; i += blockDim.x) s_psi[i] = psi[i];
    __syncthreads();
    const int64_t nvec = E / VEC;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvec;
         v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = v * VEC;
        float bv[VEC];
        if constexpr (VEC == 4) {
            float4 t = __ldg(reinterpret_cast<const float4 *>(base + e));
            bv[0] = t.x; bv[1] = t.y; bv[2] = t.z; bv[3] = t.w;
        } else if constexpr (VEC == 2) {
            float2 t = __ldg(reinterpret_cast<const float2 *>(base + e));
            bv[0] = t.x; bv[1] = t.y;
        } else {
            bv[0] = base[e];
        }
        for (int b0 = blockIdx.y * BC; b0 < B; b0 += BC * gridDim.y) {
            const int nb = min(BC, B - b0);
            float acc[BC][VEC];
#pragma unroll
            for (int j = 0; j < BC; ++j)
#pragma unroll
                for (int c = 0; c < VEC; ++c) acc[j][c] = bv[c];
            // kKB bases per round: all their loads are issued before any use, so a
            // thread keeps kKB * 16 B in flight instead of one dependent load per basis
            // software pipeline (HS_BLEND_FWD_PF): the next round's loads are issued
            // before this round's FMAs
            float dn[kKB][VEC];
            auto load_round = [&](int k0) {
#pragma unroll
                for (int q = 0; q < kKB; ++q) {
                    const int k = min(k0 + q, K - 1);
                    if constexpr (VEC == 4) {
                        float4 t = __ldg(reinterpret_cast<const float4 *>(deltas + (int64_t)k * E + e));
                        dn[q][0] = t.x; dn[q][1] = t.y; dn[q][2] = t.z; dn[q][3] = t.w;
                    } else if constexpr (VEC == 2) {
                        float2 t = __ldg(reinterpret_cast<const float2 *>(deltas + (int64_t)k * E + e));
                        dn[q][0] = t.x; dn[q][1] = t.y;
                    } else {
                        dn[q][0] = __ldcs(deltas + (int64_t)k * E + e);
                    }
                }
            };
            if (HS_BLEND_FWD_PF) load_round(0);
            for (int k0 = 0; k0 < K; k0 += kKB) {
                float dv[kKB][VEC];
                if (!HS_BLEND_FWD_PF) load_round(k0);
#pragma unroll
                for (int q = 0; q < kKB; ++q)
#pragma unroll
                    for (int c = 0; c < VEC; ++c) dv[q][c] = dn[q][c];
                if (HS_BLEND_FWD_PF && k0 + kKB < K) load_round(k0 + kKB);
#pragma unroll
                for (int q = 0; q < kKB; ++q) {
                    if (k0 + q < K) {
#pragma unroll
                        for (int j = 0; j < BC; ++j) {
                            if (j < nb) {
                                const float w = s_psi[(b0 + j) * K + k0 + q];
#pragma unroll
                                for (int c = 0; c < VEC; ++c)
                                    acc[j][c] = w != 0.0f ? fmaf(w, dv[q][c], acc[j][c]) : acc[j][c];
                            }
                        }
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < BC; ++j) {
                if (j < nb) {
                    float *o = raw + (int64_t)(b0 + j) * E + e;
                    if constexpr (VEC == 4) {
                        *reinterpret_cast<float4 *>(o) = make_float4(acc[j][0], acc[j][1], acc[j][2], acc[j][3]);
                    } else if constexpr (VEC == 2) {
                        __stcs(reinterpret_cast<float2 *>(o), make_float2(acc[j][0], acc[j][1]));
                    } else {
                        o[0] = acc[j][0];
                    }
                }
            }
        }
    }
}

// Adjoint of blend, reduced over the frame batch in-kernel (S/model.py:188-216 +
// the item-order sum of S/train.py:253-255):
//   g_base[e]     = sum_b g[b][e]                              (all 14N channels)
//   g_delta[k][e] = sum_b psi[b][k] g[b][e]                    (10N blended channels)
//   g_psi[b][k]   = sum_e delta[k][e] g[b][e]   -> one partial per CTA (deterministic)
// Each warp streams 32 consecutive channels at a time with the BP frame values in
// registers (coalesced loads, no shared-memory staging); the g_psi products of a
// basis k are reduce-scattered across the warp (16 values in 16 shuffles) and
// accumulated per warp in shared memory, then summed over the CTA's warps.
#ifndef HS_BLEND_MINB
#define HS_BLEND_MINB 2
#endif
constexpr int kBT = 256;
constexpr int kBMaxB = 16;
constexpr int kBMaxK = 32;
#ifndef HS_BLEND_BLOCKS
#define HS_BLEND_BLOCKS 296          // one wave at 2 CTAs per SM (148 x 2)
#endif
constexpr int kBBlocks = HS_BLEND_BLOCKS;   // persistent grid
#ifndef HS_BLEND_CPI
#define HS_BLEND_CPI 4
#endif
constexpr int kCPI = HS_BLEND_CPI;  // chunks per warp iteration

template <int BP>
__global__ void __launch_bounds__(kBT, HS_BLEND_MINB) blend_bwd_kernel(int64_t N, int K, int Bc, int b0,
                                                       const float *__restrict__ deltas,
                                                       const float *__restrict__ psi,
                                                       const float *__restrict__ g_raw,
                                                       float *__restrict__ g_base,
                                                       float *__restrict__ g_deltas,
                                                       float *__restrict__ partials, int P,
                                                       int accumulate) {
    pdl_prologue();
    static_assert(BP % 4 == 0, "frames per pass: a multiple of 4");
    // psi transposed to [k][b]: a basis' BP weights are BP / 4 16-byte loads
    __shared__ __align__(16) float p_t[kBMaxK * kBMaxB];
    __shared__ float accw[kBT / 32][BP * kBMaxK];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < BP * K; i += kBT) {
        const int k = i / BP, b = i % BP;
        p_t[i] = b < Bc ? psi[(b0 + b) * K + k] : 0.f;
    }
    for (int i = lane; i < BP * K; i += 32) accw[warp][i] = 0.f;
    __syncthreads();
    const int64_t E10 = 10 * N, E14 = 14 * N;
    const int64_t chunks = (E14 + 31) / 32;
    // kCPI consecutive 32-channel chunks per warp iteration: the g_psi products of the
    // chunks are summed in registers before the one reduce-scatter per basis.  The frame
    // values are register pairs (frames b, b + 1): the FMAs are packed FFMA2.
    for (int64_t c0 = ((int64_t)blockIdx.x * (kBT / 32) + warp) * kCPI; c0 < chunks;
         c0 += (int64_t)gridDim.x * (kBT / 32) * kCPI) {
        float2 g[kCPI][BP / 2];
        bool in10[kCPI];
#pragma unroll
        for (int j = 0; j < kCPI; ++j) {
            const int64_t e = (c0 + j) * 32 + lane;
            const bool in = e < E14;
            in10[j] = e < E10;
            float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
            for (int h = 0; h < BP / 2; ++h) {
                const int b = 2 * h;
                g[j][h].x = (in && b < Bc) ? __ldcs(g_raw + (int64_t)(b0 + b) * E14 + e) : 0.f;
                g[j][h].y = (in && b + 1 < Bc) ? __ldcs(g_raw + (int64_t)(b0 + b + 1) * E14 + e) : 0.f;
                s2 = __fadd2_rn(s2, g[j][h]);
            }
            const float s = s2.x + s2.y;
            if (in) g_base[e] = accumulate ? g_base[e] + s : s;
        }
        if (c0 * 32 >= E10) continue;                      // warp-uniform
        const int64_t e0 = c0 * 32 + lane;
        // software pipeline over the bases: basis k+1's delta loads are issued before
        // basis k's FMAs and reduce-scatter, so a load's latency hides behind a whole
        // basis of work instead of stalling the warp once per basis
        float dn[kCPI];
#pragma unroll
        for (int j = 0; j < kCPI; ++j) dn[j] = in10[j] ? __ldcs(deltas + e0 + 32 * j) : 0.f;
        for (int k = 0; k < K; ++k) {
            float dk[kCPI];
#pragma unroll
            for (int j = 0; j < kCPI; ++j) dk[j] = dn[j];
            if (k + 1 < K) {
#pragma unroll
                for (int j = 0; j < kCPI; ++j)
                    dn[j] = in10[j] ? __ldcs(deltas + (int64_t)(k + 1) * E10 + e0 + 32 * j) : 0.f;
            }
            float2 pk[BP / 2];
#pragma unroll
            for (int q = 0; q < BP / 4; ++q) {
                const float4 w = *reinterpret_cast<const float4 *>(p_t + k * BP + 4 * q);
                pk[2 * q] = make_float2(w.x, w.y);
                pk[2 * q + 1] = make_float2(w.z, w.w);
            }
            float2 gd[kCPI], v[BP / 2];
#pragma unroll
            for (int j = 0; j < kCPI; ++j) gd[j] = make_float2(0.f, 0.f);
#pragma unroll
            for (int h = 0; h < BP / 2; ++h) v[h] = make_float2(0.f, 0.f);
#pragma unroll
            for (int h = 0; h < BP / 2; ++h)
#pragma unroll
                for (int j = 0; j < kCPI; ++j) {
                    gd[j] = __ffma2_rn(pk[h], g[j][h], gd[j]);
                    v[h] = __ffma2_rn(make_float2(dk[j], dk[j]), g[j][h], v[h]);
                }
#pragma unroll
            for (int j = 0; j < kCPI; ++j)
                if (in10[j]) {
                    float *o = g_deltas + (int64_t)k * E10 + e0 + 32 * j;
                    const float r = gd[j].x + gd[j].y;
                    *o = accumulate ? *o + r : r;
                }
            float vf[BP];
#pragma unroll
            for (int h = 0; h < BP / 2; ++h) {
                vf[2 * h] = v[h].x;
                vf[2 * h + 1] = v[h].y;
            }
            int vi;
            bool issue;
            const float r = reduce_scatter(vf, lane, vi, issue);
            if (issue) accw[warp][k * BP + vi] += r;
        }
    }
    __syncthreads();
    for (int i = tid; i < Bc * K; i += kBT) {
        const int b = i / K, k = i % K;
        float s = 0.f;
#pragma unroll
        for (int w = 0; w < kBT / 32; ++w) s += accw[w][k * BP + b];
        partials[((int64_t)(b0 + b) * K + k) * P + blockIdx.x] = s;
    }
}

// HS_BLEND_BWD_TMA: the same adjoint over kBbTE-channel tiles staged in shared memory by
// 1D bulk copies (the frames' g rows and the bases' delta rows, kBbS stages in flight)
// for 9..16-frame passes with K <= 20 and N % (kBbTE / 2) == 0 (every tile full, every
// row 16-byte aligned).  Per tile, with 256 threads:
//   g_base / g_delta: thread (cg = t % (TE / 4), kg = t / (TE / 4)) owns channels 4 cg ..
//     4 cg + 3 and bases kg, kg + kBbKG, ...: its frames' g (LDS.128 each) times psi (the
//     packed FFMA2's broadcast operand), one 16-byte store per basis;
//   g_psi: thread (c = t % 16, blk = t / 16) accumulates frames 4 (blk % 4) .. + 3 x bases
//     5 (blk / 4) .. + 4 over channels 64 h + 4 c .. + 3 (packed pairs of channels, 40
//     FFMA2 per 64 channels), kept in registers across the CTA's tiles and reduced over
//     the 16 channel groups once at the end (one partial per CTA).
// Per tile the FFMA2 count is the floor of both products (2 x 16 x 20 x TE / 2 / 256 per
// thread); the loads are 36 rows of 4 TE bytes.
#ifndef HS_BLEND_BWD_TMA
#define HS_BLEND_BWD_TMA 1
#endif
#ifndef HS_BLEND_BWD_STAGES
#define HS_BLEND_BWD_STAGES 2
#endif
#ifndef HS_BB_DIAG
#define HS_BB_DIAG 0                 // diagnostics: 1 skips g_psi, 2 skips the g_delta stores
#endif
#ifndef HS_BB_TE
#define HS_BB_TE 256                 // (1 KB rows: 128-channel tiles' 512-byte copies load at ~2/3 the rate)
#endif
constexpr int kBbTE = HS_BB_TE;                    // channels per tile
constexpr int kBbKG = 1024 / kBbTE;                // g_delta: basis groups (threads per channel quad: 256 / (TE / 4))
constexpr int kBbKPT = (20 + kBbKG - 1) / kBbKG;   // bases per thread
constexpr int kBbS = HS_BLEND_BWD_STAGES;
constexpr int kBbK = 20;                           // max bases of this path (4 blocks of 5)
constexpr int kBbStage = (16 + kBbK) * kBbTE;      // floats per stage: 16 g rows + 20 delta rows
__host__ inline size_t blend_bwd_tma_smem() {
    return 64 + sizeof(float) * ((size_t)kBbS * kBbStage + kBbK * 16 + 16 * 16 * 20);
}

#ifndef HS_BB_MINB
#define HS_BB_MINB 2
#endif
__global__ void __launch_bounds__(256, HS_BB_MINB) blend_bwd_tma_kernel(int64_t N, int K, int Bc, int b0,
                                                               const float *__restrict__ deltas,
                                                               const float *__restrict__ psi,
                                                               const float *__restrict__ g_raw,
                                                               float *__restrict__ g_base,
                                                               float *__restrict__ g_deltas,
                                                               float *__restrict__ partials, int P, int accumulate) {
    pdl_prologue();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw);
    float *stages = reinterpret_cast<float *>(smem_raw + 64);          // kBbS x [16 g | K d] x kBbTE
    float *p_t = stages + (size_t)kBbS * kBbStage;                     // psi [k][16]
    float *red = p_t + kBbK * 16;                                      // [16 blk][16 c][20] g_psi reduce
    const int tid = threadIdx.x;
    const int64_t E10 = 10 * N, E14 = 14 * N;
    const int64_t ntiles = E14 / kBbTE, ntiles10 = E10 / kBbTE;
    if (tid == 0) {
        for (int st = 0; st < kBbS; ++st) mbar_init(&bars[st], 1);
        mbar_fence_init();
    }
    for (int i = tid; i < kBbK * 16; i += 256) {
        const int k = i / 16, b = i % 16;
        p_t[i] = (k < K && b < Bc) ? psi[(b0 + b) * K + k] : 0.f;
    }
    __syncthreads();
    // warp 0 issues a stage: lane 0 registers the bytes, lanes issue one row each
    auto issue = [&](int64_t t, int st) {
        const int lane = tid & 31;
        const int64_t e0 = t * kBbTE;
        const int rows = Bc + (t < ntiles10 ? K : 0);
        float *dst = stages + (size_t)st * kBbStage;
        if (lane == 0) mbar_expect_tx(&bars[st], (uint32_t)(rows * kBbTE * 4));
        __syncwarp();
        for (int r = lane; r < rows; r += 32) {
            if (r < Bc) bulk_g2s(dst + (size_t)r * kBbTE, g_raw + (int64_t)(b0 + r) * E14 + e0, kBbTE * 4, &bars[st]);
            else bulk_g2s(dst + (size_t)(16 + r - Bc) * kBbTE, deltas + (int64_t)(r - Bc) * E10 + e0, kBbTE * 4, &bars[st]);
        }
    };
    if (tid < 32) {
        for (int st = 0; st < kBbS; ++st)
            if (blockIdx.x + (int64_t)st * gridDim.x < ntiles) issue(blockIdx.x + (int64_t)st * gridDim.x, st);
    }
    // g_psi accumulators: frames 4 bb .. 4 bb + 3, bases 5 kb .. 5 kb + 4, channel pairs
    const int rc = tid & 15, blk = tid >> 4, bb = blk & 3, kb = blk >> 2;
    float2 acc[4][5];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < 5; ++q) acc[i][q] = make_float2(0.f, 0.f);
    const int cg = tid % (kBbTE / 4), kg = tid / (kBbTE / 4);
    uint32_t phase = 0;
    int it = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int st = it % kBbS;
        mbar_wait(&bars[st], (phase >> st) & 1u);
        phase ^= 1u << st;
        const float *sg = stages + (size_t)st * kBbStage, *sd = sg + 16 * kBbTE;
        const int64_t e0 = t * kBbTE;
        const bool blended = t < ntiles10;
        // g_base and g_delta
        if (blended || kg == 0) {
            // frames in two halves of 8 (registers); each thread's <= 3 bases accumulate
            float2 a[kBbKPT][2], s01 = make_float2(0.f, 0.f), s23 = make_float2(0.f, 0.f);
#pragma unroll
            for (int j = 0; j < kBbKPT; ++j) a[j][0] = a[j][1] = make_float2(0.f, 0.f);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                float4 g[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int b = 8 * h + i;
                    g[i] = b < Bc ? *reinterpret_cast<const float4 *>(sg + b * kBbTE + 4 * cg)
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
                }
                if (kg == 0) {
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        s01 = __fadd2_rn(s01, make_float2(g[i].x, g[i].y));
                        s23 = __fadd2_rn(s23, make_float2(g[i].z, g[i].w));
                    }
                }
                if (blended) {
#pragma unroll
                    for (int j = 0; j < kBbKPT; ++j) {
                        const int k = kg + kBbKG * j;
                        if (k < K) {
#pragma unroll
                            for (int q = 0; q < 2; ++q) {
                                const float4 w = *reinterpret_cast<const float4 *>(p_t + k * 16 + 8 * h + 4 * q);
                                const float wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                                for (int i = 0; i < 4; ++i) {
                                    const float4 gb = g[4 * q + i];
                                    a[j][0] = __ffma2_rn(make_float2(wv[i], wv[i]), make_float2(gb.x, gb.y), a[j][0]);
                                    a[j][1] = __ffma2_rn(make_float2(wv[i], wv[i]), make_float2(gb.z, gb.w), a[j][1]);
                                }
                            }
                        }
                    }
                }
            }
            if (kg == 0) {
                float4 *o = reinterpret_cast<float4 *>(g_base + e0 + 4 * cg);
                float4 r = make_float4(s01.x, s01.y, s23.x, s23.y);
                if (accumulate) {
                    const float4 q = *o;
                    r = make_float4(q.x + r.x, q.y + r.y, q.z + r.z, q.w + r.w);
                }
                *o = r;
            }
            if (blended && !(HS_BB_DIAG & 2)) {
#pragma unroll
                for (int j = 0; j < kBbKPT; ++j) {
                    const int k = kg + kBbKG * j;
                    if (k < K) {
                        float4 *o = reinterpret_cast<float4 *>(g_deltas + (int64_t)k * E10 + e0 + 4 * cg);
                        float4 r = make_float4(a[j][0].x, a[j][0].y, a[j][1].x, a[j][1].y);
                        if (accumulate) {
                            const float4 q = *o;
                            r = make_float4(q.x + r.x, q.y + r.y, q.z + r.z, q.w + r.w);
                        }
                        __stcs(o, r);
                    }
                }
            }
        }
        // g_psi partial sums
        if (blended && !(HS_BB_DIAG & 1)) {
#pragma unroll
            for (int h = 0; h < kBbTE / 64; ++h) {
                const int c = 64 * h + 4 * rc;
                float4 gv[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) gv[i] = *reinterpret_cast<const float4 *>(sg + (4 * bb + i) * kBbTE + c);
#pragma unroll
                for (int q = 0; q < 5; ++q) {
                    const int k = 5 * kb + q;
                    if (k < K) {
                        const float4 dv = *reinterpret_cast<const float4 *>(sd + k * kBbTE + c);
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            acc[i][q] = __ffma2_rn(make_float2(gv[i].x, gv[i].y), make_float2(dv.x, dv.y), acc[i][q]);
                            acc[i][q] = __ffma2_rn(make_float2(gv[i].z, gv[i].w), make_float2(dv.z, dv.w), acc[i][q]);
                        }
                    }
                }
            }
        }
        __syncthreads();                     // every thread is done with this stage
        if (tid < 32 && t + kBbS * (int64_t)gridDim.x < ntiles) issue(t + kBbS * (int64_t)gridDim.x, st);
    }
    // g_psi: sum the 16 channel groups of each (frame, basis) block in a fixed order
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < 5; ++q) red[(blk * 16 + rc) * 20 + i * 5 + q] = acc[i][q].x + acc[i][q].y;
    __syncthreads();
    for (int o = tid; o < Bc * K; o += 256) {
        const int b = o / K, k = o % K;
        const int ob = (b >> 2) | ((k / 5) << 2), oi = (b & 3) * 5 + k % 5;
        float s = 0.f;
        for (int c = 0; c < 16; ++c) s += red[(ob * 16 + c) * 20 + oi];
        partials[((int64_t)(b0 + b) * K + k) * P + blockIdx.x] = s;
    }
}

// HS_BLEND_BWD_SPLIT: the adjoint as two streaming kernels, for any N alignment and any
// frame count in one pass over g (the fused kernels above take <= 16 frames per launch,
// so more frames mean read-modify-write passes over g_delta, and the TMA tiles need
// N % 128 == 0):
// (a) blend_bwd_gd_kernel -- g_base and g_delta.  One thread per channel pair (e, e + 1):
//     the B frames' g[b][e..e+1] (8-byte loads, coalesced, 4 in flight) in ascending frame
//     order into the running sum and, for e < 10N, into K packed accumulators with
//     psi[b][k] as the FFMA2's broadcast operand (psi staged 128 frames at a time).  One
//     store per output.
// (b) blend_bwd_psi_kernel -- g_psi, one partial per CTA (fixed order).  The CTA's range
//     of 64-channel tiles, double-buffered with cp.async (8-byte g pairs, zero-filled past
//     10N; the delta rows transposed to [channel][basis] so basis pairs are adjacent).
//     Thread item = 4 frames x 10 bases, G = 256 / items threads per item over the
//     tile's channel pairs: 40 FFMA2 per 14 shared loads; the G channel groups are summed
//     in a fixed order at the end.
#ifndef HS_BLEND_BWD_SPLIT
#define HS_BLEND_BWD_SPLIT 1          // 0: never, 1: for more than 16 frames, 2: always
#endif
constexpr int kGdT = 256;
constexpr int kGdFrames = 128;        // psi frames staged per shared-memory round
constexpr int kPsT = 256, kPsTE = 64;
constexpr int kPsMaxB = 128;          // frames per psi launch

#ifndef HS_GD_UNROLL
#define HS_GD_UNROLL 16               // frames whose loads are in flight together
#endif
#ifndef HS_GD_MINB
#define HS_GD_MINB 2
#endif
template <int KM>
__global__ void __launch_bounds__(kGdT, HS_GD_MINB) blend_bwd_gd_kernel(int64_t N, int K, int B,
                                                                        const float *__restrict__ psi,
                                                                        const float *__restrict__ g_raw,
                                                                        float *__restrict__ g_base,
                                                                        float *__restrict__ g_deltas) {
    constexpr int U = KM > 20 ? 8 : HS_GD_UNROLL;     // (32 bases: registers)
    pdl_prologue();
    __shared__ __align__(16) float s_psi[kGdFrames * KM];
    const int64_t E10 = 10 * N, E14 = 14 * N;
    const int64_t e = 2 * ((int64_t)blockIdx.x * kGdT + threadIdx.x);
    const bool in = e < E14, blended = e < E10;      // (10N even: a pair is wholly in or out)
    float2 acc[KM], sum = make_float2(0.f, 0.f);
#pragma unroll
    for (int k = 0; k < KM; ++k) acc[k] = make_float2(0.f, 0.f);
    for (int b0 = 0; b0 < B; b0 += kGdFrames) {
        const int Bc = min(kGdFrames, B - b0);
        __syncthreads();
        for (int i = threadIdx.x; i < Bc * KM; i += kGdT) {
            const int b = i / KM, k = i % KM;
            s_psi[i] = k < K ? psi[(int64_t)(b0 + b) * K + k] : 0.f;
        }
        __syncthreads();
        if (!in) continue;
        const float *gp = g_raw + (int64_t)b0 * E14 + e;
        auto frame = [&](float2 g, int b) {
            sum = __fadd2_rn(sum, g);
            if (blended) {
#pragma unroll
                for (int k = 0; k < KM; ++k) {
                    const float w = s_psi[b * KM + k];
                    acc[k] = __ffma2_rn(make_float2(w, w), g, acc[k]);
                }
            }
        };
        int b = 0;
        for (; b + U <= Bc; b += U) {
            float2 g[U];
#pragma unroll
            for (int j = 0; j < U; ++j) g[j] = __ldcs(reinterpret_cast<const float2 *>(gp + (int64_t)(b + j) * E14));
#pragma unroll
            for (int j = 0; j < U; ++j) frame(g[j], b + j);
        }
        for (; b < Bc; ++b) frame(__ldcs(reinterpret_cast<const float2 *>(gp + (int64_t)b * E14)), b);
    }
    if (!in) return;
    *reinterpret_cast<float2 *>(g_base + e) = sum;
    if (blended) {
#pragma unroll
        for (int k = 0; k < KM; ++k)
            if (k < K) __stcs(reinterpret_cast<float2 *>(g_deltas + (int64_t)k * E10 + e), acc[k]);
    }
}

__device__ __forceinline__ void cp_async_zfill(void *dst, const void *src, int bytes, bool ok) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
    if (bytes == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(ok ? 8 : 0) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(src), "r"(ok ? 4 : 0) : "memory");
}

__host__ __device__ inline int psi_kpad(int K) { return (K + 9) / 10 * 10; }
constexpr int kPsRow = kPsTE + 2;     // g row stride (pad: the frame blocks of a warp on distinct banks)
__host__ __device__ inline int psi_stage(int Bc, int K) { return ((Bc + 3) & ~3) * kPsRow + kPsTE * psi_kpad(K); }
__host__ inline size_t blend_bwd_psi_smem(int Bc, int K) {
    return sizeof(float) * (size_t)std::max(2 * psi_stage(Bc, K), kPsT * 40);
}

__global__ void __launch_bounds__(kPsT) blend_bwd_psi_kernel(int64_t N, int K, int Bc, int b0,
                                                             const float *__restrict__ deltas,
                                                             const float *__restrict__ g_raw,
                                                             float *__restrict__ partials, int P) {
    pdl_prologue();
    extern __shared__ __align__(16) float sm[];
    const int Bp = (Bc + 3) & ~3, Kp = psi_kpad(K);
    const int nfb = Bp / 4, items = nfb * (Kp / 10);
    const int G = kPsT / items;                      // (host: items <= 128)
    const int tid = threadIdx.x, item = tid / G, cg = tid % G;
    const bool active = item < items;
    const int fb = item % nfb, kb = item / nfb;
    const int stage = psi_stage(Bc, K);
    const int64_t E10 = 10 * N, E14 = 14 * N;
    const int64_t ntiles = (E10 + kPsTE - 1) / kPsTE;
    const int64_t per = (ntiles + gridDim.x - 1) / gridDim.x;
    const int64_t t_lo = (int64_t)blockIdx.x * per, t_hi = min(ntiles, t_lo + per);
    for (int i = tid; i < 2 * stage; i += kPsT) sm[i] = 0.f;    // (padding rows / bases stay zero)
    __syncthreads();
    auto issue = [&](int64_t t, int buf) {
        float *sg = sm + buf * stage, *sd = sg + Bp * kPsRow;
        const int64_t e0 = t * kPsTE;
        for (int i = tid; i < Bc * (kPsTE / 2); i += kPsT) {
            const int b = i / (kPsTE / 2), c = 2 * (i % (kPsTE / 2));
            const bool ok = e0 + c < E10;
            cp_async_zfill(sg + b * kPsRow + c, g_raw + (int64_t)(b0 + b) * E14 + (ok ? e0 + c : 0), 8, ok);
        }
        for (int i = tid; i < K * kPsTE; i += kPsT) {
            const int k = i / kPsTE, c = i % kPsTE;
            const bool ok = e0 + c < E10;
            cp_async_zfill(sd + c * Kp + k, deltas + (int64_t)k * E10 + (ok ? e0 + c : 0), 4, ok);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    float2 acc[4][5];
#pragma unroll
    for (int f = 0; f < 4; ++f)
#pragma unroll
        for (int q = 0; q < 5; ++q) acc[f][q] = make_float2(0.f, 0.f);
    if (t_lo < t_hi) issue(t_lo, 0);
    int it = 0;
    for (int64_t t = t_lo; t < t_hi; ++t, ++it) {
        const int buf = it & 1;
        if (t + 1 < t_hi) {
            issue(t + 1, buf ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        if (active) {
            const float *sg = sm + buf * stage, *sd = sg + Bp * kPsRow;
            for (int c = 2 * cg; c < kPsTE; c += 2 * G) {
                float2 gv[4];
#pragma unroll
                for (int f = 0; f < 4; ++f) gv[f] = *reinterpret_cast<const float2 *>(sg + (4 * fb + f) * kPsRow + c);
                const float *d0 = sd + c * Kp + 10 * kb, *d1 = d0 + Kp;
#pragma unroll
                for (int q = 0; q < 5; ++q) {
                    const float2 da = *reinterpret_cast<const float2 *>(d0 + 2 * q);
                    const float2 db = *reinterpret_cast<const float2 *>(d1 + 2 * q);
#pragma unroll
                    for (int f = 0; f < 4; ++f) {
                        acc[f][q] = __ffma2_rn(make_float2(gv[f].x, gv[f].x), da, acc[f][q]);
                        acc[f][q] = __ffma2_rn(make_float2(gv[f].y, gv[f].y), db, acc[f][q]);
                    }
                }
            }
        }
        __syncthreads();                             // before this buffer is refilled
    }
    // the G channel groups of each item, summed in a fixed order
    float *red = sm;                                 // [items][G][40]
    if (active) {
#pragma unroll
        for (int f = 0; f < 4; ++f)
#pragma unroll
            for (int q = 0; q < 5; ++q) {
                red[(item * G + cg) * 40 + f * 10 + 2 * q] = acc[f][q].x;
                red[(item * G + cg) * 40 + f * 10 + 2 * q + 1] = acc[f][q].y;
            }
    }
    __syncthreads();
    for (int o = tid; o < Bc * K; o += kPsT) {
        const int b = o / K, k = o % K;
        const int itm = b / 4 + (k / 10) * nfb, slot = (b % 4) * 10 + k % 10;
        float s = 0.f;
        for (int c = 0; c < G; ++c) s += red[(itm * G + c) * 40 + slot];
        partials[((int64_t)(b0 + b) * K + k) * P + blockIdx.x] = s;
    }
}

// ------------------------------------------------------------------ Adam

// S/optim.py:28-40, one update of the flat parameter buffer [base | deltas | mlp]:
// a multi-tensor Adam whose learning rate comes from the element's group
// (S/train.py:184-199: 5 base groups, 3 delta groups repeated per basis, the MLP).
// Optionally restricted to [begin, end) so that it can run per allreduce bucket
// as the buckets arrive, and optionally fused with the colour-init apply
// (S/train.py:263-278, S/color_init.py:45-80, S/model.py:260-263): colour init
// runs after Adam in the reference and leaves the moments alone, so the colour
// segment's threads do the Adam update and then overwrite the parameter.
struct AdamArgs {
    int64_t N, begin, end;
    int K;
    float *p;
    const float *g;
    float *m, *v;
    float lr[9];
    float b1, b2, inv_bc1, inv_bc2, eps;
    // colour init: mode 1 = local frames (maxw/wsums), 2 = reduced across ranks (packed/est4)
    int B;
    const float *maxw, *wsums;
    const int64_t *packed;
    const float *est4;
    float thr;
    uint8_t *visited;
    int *n_init;
    unsigned long long *err;
};

__device__ __forceinline__ float adam_lr(const AdamArgs &a, int64_t i) {
    const int64_t N = a.N, base = 14 * N, dend = base + (int64_t)a.K * 10 * N;
    if (i < base) return i < 3 * N ? a.lr[0] : i < 7 * N ? a.lr[1] : i < 10 * N ? a.lr[2] : i < 13 * N ? a.lr[3] : a.lr[4];
    if (i < dend) {
        const int64_t j = (i - base) % (10 * N);
        return j < 3 * N ? a.lr[5] : j < 7 * N ? a.lr[6] : a.lr[7];
    }
    return a.lr[8];
}

__device__ __forceinline__ float adam_one(const AdamArgs &a, float lr, float p, float gi, float &mi, float &vi) {
    mi = mi * a.b1;
    mi = mi + (1.0f - a.b1) * gi;
    vi = vi * a.b2;
    vi = vi + (1.0f - a.b2) * (gi * gi);
    const float mh = mi * a.inv_bc1, vh = vi * a.inv_bc2;
    return p - lr * mh / (sqrtf(vh) + a.eps);
}

__device__ __forceinline__ float logit_clip(float e) {
    const float q = fminf(fmaxf(e, 1e-4f), 1.0f - 1e-4f);
    return logf(q) - log1pf(-q);
}

template <int CI, bool kVec>
__global__ void __launch_bounds__(256) adam_kernel(AdamArgs a) {
    pdl_prologue();
    const int64_t N = a.N, c0 = 7 * N, c1 = 10 * N;      // base colour segment
    // element ranges of the generic update: [begin, end) minus the colour segment when fused
    int64_t lo0 = a.begin, hi0 = a.end, lo1 = 0, hi1 = 0;
    if (CI && a.begin <= c0 && a.end >= c1) {
        hi0 = c0;
        lo1 = c1;
        hi1 = a.end;
    }
    constexpr int W = kVec ? 4 : 1;
    const int64_t n0 = (hi0 - lo0) / W, n1 = (hi1 - lo1) / W;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n0 + n1; t += stride) {
        const int64_t i = t < n0 ? lo0 + t * W : lo1 + (t - n0) * W;
        const float lr = adam_lr(a, i);      // group boundaries are multiples of N (N % 4 == 0 when kVec)
        if constexpr (kVec) {
            const float4 gv = __ldcs(reinterpret_cast<const float4 *>(a.g + i));
            float4 mv = __ldcs(reinterpret_cast<const float4 *>(a.m + i));
            float4 vv = __ldcs(reinterpret_cast<const float4 *>(a.v + i));
            float4 pv = *reinterpret_cast<const float4 *>(a.p + i);
            pv.x = adam_one(a, lr, pv.x, gv.x, mv.x, vv.x);
            pv.y = adam_one(a, lr, pv.y, gv.y, mv.y, vv.y);
            pv.z = adam_one(a, lr, pv.z, gv.z, mv.z, vv.z);
            pv.w = adam_one(a, lr, pv.w, gv.w, mv.w, vv.w);
            __stcs(reinterpret_cast<float4 *>(a.m + i), mv);
            __stcs(reinterpret_cast<float4 *>(a.v + i), vv);
            *reinterpret_cast<float4 *>(a.p + i) = pv;
        } else {
            float mi = a.m[i], vi = a.v[i];
            a.p[i] = adam_one(a, lr, a.p[i], a.g[i], mi, vi);
            a.m[i] = mi;
            a.v[i] = vi;
        }
    }
    if (!CI || hi1 == 0) return;
    // colour segment: one thread per Gaussian (its 3 channels), Adam then colour init
    for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < N; n += stride) {
        float col[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const int64_t i = c0 + 3 * n + c;
            float mi = a.m[i], vi = a.v[i];
            col[c] = adam_one(a, a.lr[2], a.p[i], a.g[i], mi, vi);
            a.m[i] = mi;
            a.v[i] = vi;
        }
        bool init = false;
        float est[3];
        if (!a.visited[n]) {
            if (CI == 1) {
                int best = 0;
                float bw = a.maxw[n];
                for (int b = 1; b < a.B; ++b) {
                    const float w = a.maxw[(int64_t)b * N + n];
                    if (w > bw) { bw = w; best = b; }   // first max wins (np.argmax)
                }
                if (bw > a.thr) {
                    const float4 sm = reinterpret_cast<const float4 *>(a.wsums)[(int64_t)best * N + n];
                    if (sm.w <= 0.f) {
                        atomicMin(a.err, err_code(2, best, 0, n));
                    } else {
                        init = true;
                        est[0] = sm.x / sm.w;
                        est[1] = sm.y / sm.w;
                        est[2] = sm.z / sm.w;
                    }
                }
            } else {
                const float w = __uint_as_float((uint32_t)((unsigned long long)a.packed[n] >> 32));
                const float4 e = reinterpret_cast<const float4 *>(a.est4)[n];
                if (w > a.thr && e.w > 0.f) {
                    init = true;
                    est[0] = e.x;
                    est[1] = e.y;
                    est[2] = e.z;
                }
            }
        }
        if (init) {
#pragma unroll
            for (int c = 0; c < 3; ++c) col[c] = logit_clip(est[c]);
            a.visited[n] = 1;
            if (a.n_init) atomicAdd(a.n_init, 1);
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) a.p[c0 + 3 * n + c] = col[c];
    }
}

// ------------------------------------------------------------ colour init

// S/train.py:263-278 + S/color_init.py:45-80 + S/model.py:260-263 (logit with clamp).
__global__ void color_init_kernel(int B, int64_t N, const float *__restrict__ maxw,
                                  const float *__restrict__ wsums, float thr,
                                  uint8_t *__restrict__ visited, float *__restrict__ color,
                                  int *n_init, unsigned long long *err) {
    pdl_prologue();
    const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (n >= N) return;
    if (visited[n]) return;
    int best = 0;
    float bw = maxw[n];
    for (int b = 1; b < B; ++b) {
        float w = maxw[(int64_t)b * N + n];
        if (w > bw) { bw = w; best = b; }   // first max wins (np.argmax)
    }
    if (!(bw > thr)) return;
    const float4 s = reinterpret_cast<const float4 *>(wsums)[(int64_t)best * N + n];
    if (s.w <= 0.f) {
        atomicMin(err, err_code(2, best, 0, n));
        return;
    }
    const float den = s.w;
    const float est[3] = {s.x / den, s.y / den, s.z / den};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        float p = fminf(fmaxf(est[c], 1e-4f), 1.0f - 1e-4f);
        color[3 * n + c] = logf(p) - log1pf(-p);
    }
    visited[n] = 1;
    if (n_init) atomicAdd(n_init, 1);
}

// Multi-GPU colour init: order-preserving pack of (weight, -frame) into a signed
// int64 (non-negative weights keep the top bit clear).
__global__ void color_pack_kernel(int B, int64_t N, int frame_offset, const float *__restrict__ maxw,
                                  const uint8_t *__restrict__ visited, int64_t *__restrict__ packed) {
    pdl_prologue();
    const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (n >= N) return;
    unsigned long long best = 0;
    if (!visited[n]) {
        for (int b = 0; b < B; ++b) {
            const float w = maxw[(int64_t)b * N + n];
            const unsigned long long v = ((unsigned long long)__float_as_uint(fmaxf(w, 0.f)) << 32) |
                                         (unsigned long long)(0xFFFFFFFFu - (uint32_t)(frame_offset + b));
            best = v > best ? v : best;
        }
    }
    packed[n] = (int64_t)best;
}

__global__ void color_select_kernel(int B, int64_t N, int frame_offset, const int64_t *__restrict__ packed,
                                    const float *__restrict__ wsums, float *__restrict__ est4,
                                    unsigned long long *err) {
    pdl_prologue();
    const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (n >= N) return;
    const unsigned long long v = (unsigned long long)packed[n];
    const int f = (int)(0xFFFFFFFFu - (uint32_t)(v & 0xFFFFFFFFull));
    const int b = f - frame_offset;
    float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
    if (v != 0ull && b >= 0 && b < B) {
        const float4 s = reinterpret_cast<const float4 *>(wsums)[(int64_t)b * N + n];
        if (s.w > 0.f) o = make_float4(s.x / s.w, s.y / s.w, s.z / s.w, 1.f);
        else if (__uint_as_float((uint32_t)(v >> 32)) > 0.f) atomicMin(err, err_code(2, f, 0, n));
    }
    reinterpret_cast<float4 *>(est4)[n] = o;
}

__global__ void color_apply_kernel(int64_t N, const int64_t *__restrict__ packed, const float *__restrict__ est4,
                                   float thr, uint8_t *__restrict__ visited, float *__restrict__ color,
                                   int *n_init) {
    pdl_prologue();
    const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (n >= N || visited[n]) return;
    const float w = __uint_as_float((uint32_t)((unsigned long long)packed[n] >> 32));
    const float4 e = reinterpret_cast<const float4 *>(est4)[n];
    if (!(w > thr) || !(e.w > 0.f)) return;
    const float est[3] = {e.x, e.y, e.z};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        float p = fminf(fmaxf(est[c], 1e-4f), 1.0f - 1e-4f);
        color[3 * n + c] = logf(p) - log1pf(-p);
    }
    visited[n] = 1;
    if (n_init) atomicAdd(n_init, 1);
}

// ---------------------------------------------------------- compat ops

// S/model.py:219-234 (layout [pos 3N | rot 4N | color 3N | scale 3N | opacity N])
__global__ void activate_fwd_kernel(int64_t N, const float *__restrict__ raw, float *__restrict__ act,
                                    unsigned long long *err) {
    pdl_prologue();
    const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (n >= N) return;
    const float *q = raw + 3 * N + 4 * n;
    float nrm = sqrtf(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    if (!(nrm >= 1e-30f)) atomicMin(err, err_code(0, 0, 1, n));
    for (int c = 0; c < 3; ++c) act[3 * n + c] = raw[3 * n + c];
    for (int c = 0; c < 4; ++c) act[3 * N + 4 * n + c] = q[c] / nrm;
    for (int c = 0; c < 3; ++c) act[7 * N + 3 * n + c] = sigmoidf_ref(raw[7 * N + 3 * n + c]);
    for (int c = 0; c < 3; ++c) act[10 * N + 3 * n + c] = expf(raw[10 * N + 3 * n + c]);
    act[13 * N + n] = sigmoidf_ref(raw[13 * N + n]);
}

// S/model.py:237-248
__global__ void activate_bwd_kernel(int64_t N, const float *__restrict__ raw,
                                    const float *__restrict__ act, const float *__restrict__ g,
                                    float *__restrict__ o) {
    pdl_prologue();
    const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (n >= N) return;
    for (int c = 0; c < 3; ++c) o[3 * n + c] = g[3 * n + c];
    float q[4], gq[4], oq[4];
    for (int c = 0; c < 4; ++c) { q[c] = raw[3 * N + 4 * n + c]; gq[c] = g[3 * N + 4 * n + c]; }
    quat_normalize_bwd(q, gq, oq);
    for (int c = 0; c < 4; ++c) o[3 * N + 4 * n + c] = oq[c];
    for (int c = 0; c < 3; ++c) {
        float a = act[7 * N + 3 * n + c];
        o[7 * N + 3 * n + c] = g[7 * N + 3 * n + c] * a * (1.f - a);
        o[10 * N + 3 * n + c] = g[10 * N + 3 * n + c] * act[10 * N + 3 * n + c];
    }
    float a = act[13 * N + n];
    o[13 * N + n] = g[13 * N + n] * a * (1.f - a);
}

// S/binding.py:174-188
__global__ void transform_fwd_kernel(int64_t N, const float *__restrict__ t, const float *__restrict__ frames,
                                     const int32_t *__restrict__ tri, const float *__restrict__ bary,
                                     float *__restrict__ w) {
    pdl_prologue();
    const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (n >= N) return;
    const float *fr = frames + (int64_t)tri[n] * kFrame;
    const float *R = fr, *fq = fr + 9, *V = fr + 13;
    const float x[3] = {t[3 * n], t[3 * n + 1], t[3 * n + 2]};
    const float bb[3] = {bary[3 * n], bary[3 * n + 1], bary[3 * n + 2]};
    for (int j = 0; j < 3; ++j)
        w[3 * n + j] = (R[j * 3] * x[0] + R[j * 3 + 1] * x[1] + R[j * 3 + 2] * x[2]) +
                       (bb[0] * V[j] + bb[1] * V[3 + j] + bb[2] * V[6 + j]);
    float q[4], qf[4], qr[4];
    for (int c = 0; c < 4; ++c) { q[c] = t[3 * N + 4 * n + c]; qf[c] = fq[c]; }
    quat_mul(qf, q, qr);
    float nrm = sqrtf(qr[0] * qr[0] + qr[1] * qr[1] + qr[2] * qr[2] + qr[3] * qr[3]);
    for (int c = 0; c < 4; ++c) w[3 * N + 4 * n + c] = qr[c] / nrm;
    for (int c = 0; c < 3; ++c) w[7 * N + 3 * n + c] = t[7 * N + 3 * n + c];
    for (int c = 0; c < 3; ++c) w[10 * N + 3 * n + c] = t[10 * N + 3 * n + c];
    w[13 * N + n] = t[13 * N + n];
}

// S/binding.py:191-204
__global__ void transform_bwd_kernel(int64_t N, const float *__restrict__ t, const float *__restrict__ frames,
                                     const int32_t *__restrict__ tri, const float *__restrict__ g,
                                     float *__restrict__ o) {
    pdl_prologue();
    const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (n >= N) return;
    const float *fr = frames + (int64_t)tri[n] * kFrame;
    const float *R = fr, *fq = fr + 9;
    for (int i = 0; i < 3; ++i)
        o[3 * n + i] = R[i] * g[3 * n] + R[3 + i] * g[3 * n + 1] + R[6 + i] * g[3 * n + 2];
    float q[4], qf[4], qr[4], gq[4], gn[4], go[4];
    for (int c = 0; c < 4; ++c) { q[c] = t[3 * N + 4 * n + c]; qf[c] = fq[c]; gq[c] = g[3 * N + 4 * n + c]; }
    quat_mul(qf, q, qr);
    quat_normalize_bwd(qr, gq, gn);
    quat_mul_bwd_right(qf, gn, go);
    for (int c = 0; c < 4; ++c) o[3 * N + 4 * n + c] = go[c];
    for (int c = 0; c < 3; ++c) o[7 * N + 3 * n + c] = g[7 * N + 3 * n + c];
    for (int c = 0; c < 3; ++c) o[10 * N + 3 * n + c] = g[10 * N + 3 * n + c];
    o[13 * N + n] = g[13 * N + n];
}

}  // namespace hs

using namespace hs;

extern "C" {

const char *hs_last_error(void) { return g_err; }
int hs_version(void) { return 1; }

int hs_device_sm_count(int device) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
    return v;
}

int64_t hs_mlp_size(int H, int D, int K) {
    return (int64_t)D * H + D + (int64_t)D * D + D + (int64_t)K * D + K;
}

int hs_mlp_fwd(int B, int H, int D, int K, const float *mlp, const float *theta, float *cache,
               float *psi, unsigned long long *err, void *stream) {
    if (B < 1 || H < 1 || D < 1 || K < 1) {
        set_error("hs_mlp_fwd: bad sizes B=%d H=%d D=%d K=%d", B, H, D, K);
        return HS_ERR_SHAPE;
    }
    size_t smem = sizeof(float) * (H + 2 * D);
    launch_k(mlp_fwd_kernel, B, 1024, smem, HS_CHECK_STREAM(stream), H, D, K, mlp, theta, cache, psi, err);
    return check_launch("hs_mlp_fwd");
}

int hs_mlp_bwd(int B, int H, int D, int K, const float *mlp, const float *theta, const float *cache,
               const float *gpsi_partials, int num_partials, float *gpsi, float *scratch, float *g_mlp,
               void *stream) {
    cudaStream_t s = HS_CHECK_STREAM(stream);
    size_t smem = sizeof(float) * (K + D + 32 * D);
    launch_k(mlp_bwd_frame_kernel, B, 1024, smem, s, H, D, K, mlp, cache, gpsi_partials, num_partials, gpsi, scratch);
    int64_t total = hs_mlp_size(H, D, K);
    launch_k(mlp_bwd_weights_kernel, grid_for(total, 256), 256, 0, s, B, H, D, K, theta, cache, gpsi, scratch, g_mlp);
    return check_launch("hs_mlp_bwd");
}

int hs_blend_fwd(int64_t N, int K, int B, const float *base14, const float *deltas, const float *psi,
                 float *raw10, void *stream) {
    if (N < 1 || K < 1 || B < 1) {
        set_error("hs_blend_fwd: bad sizes N=%lld K=%d B=%d", (long long)N, K, B);
        return HS_ERR_SHAPE;
    }
    cudaStream_t s = HS_CHECK_STREAM(stream);
    const int64_t E = 10 * N;
    size_t smem = sizeof(float) * B * K;
#ifndef HS_BLEND_VEC4
#define HS_BLEND_VEC4 1
#endif
    const bool vec = HS_BLEND_VEC4 && (E % 4 == 0) && ((uintptr_t)base14 % 16 == 0) &&
                     ((uintptr_t)deltas % 16 == 0) && ((uintptr_t)raw10 % 16 == 0);
    const int sms = current_sm_count();
#ifndef HS_BLEND_BC
#define HS_BLEND_BC 8
#endif
#ifndef HS_BLEND_TMA
#define HS_BLEND_TMA 1
#endif
    const size_t tsm = blend_fwd_smem(K, B);
    if (HS_BLEND_TMA && vec && tsm <= 200 * 1024) {
        static_assert(kBfTE == 2 * kBfT, "two channels per thread");
        cudaFuncSetAttribute(blend_fwd_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm);
        const int per_sm = std::max(1, (int)((220 * 1024) / tsm));
        const int64_t ntiles = (E + kBfTE - 1) / kBfTE;
#ifndef HS_BLEND_CTAS_PER_SM
#define HS_BLEND_CTAS_PER_SM 8
#endif
        const unsigned grid = (unsigned)std::min<int64_t>(ntiles, (int64_t)sms * std::min(per_sm, HS_BLEND_CTAS_PER_SM));
        launch_k(blend_fwd_tma_kernel, grid, kBfT, tsm, s, E, K, B, base14, deltas, psi, raw10);
    } else if (vec) {
        // grid.y splits the frames into chunks of HS_BLEND_BC: few accumulators per
        // thread (occupancy) while the 40 MB of deltas stay L2-resident across chunks
        int64_t nv = E / 4;
        const unsigned gy = (unsigned)((B + HS_BLEND_BC - 1) / HS_BLEND_BC);
        const dim3 grid((unsigned)grid_for(nv, 256), gy);
        launch_k(blend_fwd_kernel<4, HS_BLEND_BC>, grid, 256, smem, s, E, K, B, base14, deltas, psi, raw10);
    } else if (HS_BLEND_TMA && E % 2 == 0 && (uintptr_t)base14 % 8 == 0 && (uintptr_t)deltas % 8 == 0 &&
               (uintptr_t)raw10 % 8 == 0 && E > 2 && blend_fwd_mis_smem(K, B) <= 200 * 1024) {
        const size_t msm = blend_fwd_mis_smem(K, B);
        cudaFuncSetAttribute(blend_fwd_tma_mis_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)msm);
        const int per_sm = std::max(1, (int)((220 * 1024) / msm));
        const int64_t ntiles = (E + kBfTE - 1) / kBfTE;
        const unsigned grid = (unsigned)std::min<int64_t>(ntiles, (int64_t)sms * std::min(per_sm, HS_BLEND_CTAS_PER_SM));
        // more than 16 frames: 4 frame groups per tile (256 threads) instead of 2, twice the
        // warps in flight at the same shared memory per CTA
        launch_k(blend_fwd_tma_mis_kernel, grid, B > HS_BLEND_MIS_WIDE_B ? 2 * kBfT : kBfT, msm, s, E, K, B, base14,
                 deltas, psi, raw10);
    } else if (E % 2 == 0 && (uintptr_t)base14 % 8 == 0 && (uintptr_t)deltas % 8 == 0 && (uintptr_t)raw10 % 8 == 0) {
        // odd N (every other delta / frame row only 8-byte aligned): float2 channel pairs,
        // frames in chunks over grid.y (render at 100,489 Gaussians: 367 us -> see DESIGN)
#ifndef HS_BLEND_BC2
#define HS_BLEND_BC2 8
#endif
        int64_t nv = E / 2;
        const unsigned gy = (unsigned)((B + HS_BLEND_BC2 - 1) / HS_BLEND_BC2);
        const dim3 grid((unsigned)grid_for(nv, 256), gy);
        launch_k(blend_fwd_kernel<2, HS_BLEND_BC2>, grid, 256, smem, s, E, K, B, base14, deltas, psi, raw10);
    } else {
        unsigned grid = (unsigned)std::min<int64_t>(grid_for(E, 256), (int64_t)sms * 16);
        launch_k(blend_fwd_kernel<1, 16>, grid, 256, smem, s, E, K, B, base14, deltas, psi, raw10);
    }
    return check_launch("hs_blend_fwd");
}

int hs_blend_bwd_partials(int64_t N) {
    const int64_t warps = ((14 * N + 31) / 32 + (kBT / 32) - 1) / (kBT / 32);
    return (int)std::min<int64_t>(kBBlocks, std::max<int64_t>(1, warps));
}

int hs_blend_bwd_kernels(int64_t N, int K, int B) {
    if (N >= 17 && (HS_BLEND_BWD_SPLIT == 2 || (HS_BLEND_BWD_SPLIT == 1 && B > kBMaxB)))
        return 1 + (B + kPsMaxB - 1) / kPsMaxB;
    return (B + kBMaxB - 1) / kBMaxB;
}

int hs_blend_bwd(int64_t N, int K, int B, const float *deltas, const float *psi, const float *g_raw14,
                 float *g_base14, float *g_deltas, float *gpsi_partials, int *num_partials, void *stream) {
    if (K > kBMaxK || K < 1 || B < 1 || N < 1) {
        set_error("hs_blend_bwd: unsupported sizes N=%lld K=%d (max %d) B=%d", (long long)N, K, kBMaxK, B);
        return HS_ERR_SHAPE;
    }
    cudaStream_t s = HS_CHECK_STREAM(stream);
    const int P = hs_blend_bwd_partials(N);
    const bool tma = HS_BLEND_BWD_TMA && N % (kBbTE / 2) == 0 && K <= kBbK &&
                     (uintptr_t)deltas % 16 == 0 && (uintptr_t)g_raw14 % 16 == 0 && (uintptr_t)g_base14 % 16 == 0 &&
                     (uintptr_t)g_deltas % 16 == 0;
    const bool split_ok = N >= 17 && (uintptr_t)deltas % 8 == 0 && (uintptr_t)g_raw14 % 8 == 0 &&
                          (uintptr_t)g_base14 % 8 == 0 && (uintptr_t)g_deltas % 8 == 0;
    const bool split = split_ok && (HS_BLEND_BWD_SPLIT == 2 || (HS_BLEND_BWD_SPLIT == 1 && B > kBMaxB));
    if (split) {
        // g_base / g_delta over all frames in one launch, then g_psi per <= 128 frames
        const int64_t pairs = 7 * N;
        if (K <= 20)
            launch_k(blend_bwd_gd_kernel<20>, (unsigned)((pairs + kGdT - 1) / kGdT), kGdT, 0, s, N, K, B, psi, g_raw14,
                     g_base14, g_deltas);
        else
            launch_k(blend_bwd_gd_kernel<32>, (unsigned)((pairs + kGdT - 1) / kGdT), kGdT, 0, s, N, K, B, psi, g_raw14,
                     g_base14, g_deltas);
        for (int b0 = 0; b0 < B; b0 += kPsMaxB) {
            const int Bc = std::min(kPsMaxB, B - b0);
            const size_t smem = blend_bwd_psi_smem(Bc, K);
            cudaFuncSetAttribute(blend_bwd_psi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            launch_k(blend_bwd_psi_kernel, P, kPsT, smem, s, N, K, Bc, b0, deltas, g_raw14, gpsi_partials, P);
        }
        if (num_partials) *num_partials = P;
        return check_launch("hs_blend_bwd");
    }
    if (tma) cudaFuncSetAttribute(blend_bwd_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)blend_bwd_tma_smem());
    for (int b0 = 0; b0 < B; b0 += kBMaxB) {
        const int Bc = std::min(kBMaxB, B - b0);
        const int acc = b0 > 0;
        if (tma && Bc > 8)
            launch_k(blend_bwd_tma_kernel, P, 256, blend_bwd_tma_smem(), s, N, K, Bc, b0, deltas, psi, g_raw14,
                     g_base14, g_deltas, gpsi_partials, P, acc);
        else if (Bc <= 4)
            launch_k(blend_bwd_kernel<4>, P, kBT, 0, s, N, K, Bc, b0, deltas, psi, g_raw14, g_base14, g_deltas,
                                                  gpsi_partials, P, acc);
        else if (Bc <= 8)
            launch_k(blend_bwd_kernel<8>, P, kBT, 0, s, N, K, Bc, b0, deltas, psi, g_raw14, g_base14, g_deltas,
                                                  gpsi_partials, P, acc);
        else
            launch_k(blend_bwd_kernel<16>, P, kBT, 0, s, N, K, Bc, b0, deltas, psi, g_raw14, g_base14, g_deltas,
                                                   gpsi_partials, P, acc);
    }
    if (num_partials) *num_partials = P;
    return check_launch("hs_blend_bwd");
}

int hs_adam_fused(int64_t N, int K, int64_t mlp_size, float *params, const float *grads, float *m, float *v,
                  const float *lrs, int step, float beta1, float beta2, float eps, int64_t begin, int64_t end,
                  int ci_mode, int B, const float *maxw, const float *wsums, const int64_t *packed,
                  const float *est4, float threshold, uint8_t *visited, int *n_init, unsigned long long *err,
                  void *stream) {
    const int64_t total = 14 * N + (int64_t)K * 10 * N + mlp_size;
    if (step < 1) {
        set_error("hs_adam: step must be >= 1");
        return HS_ERR_SHAPE;
    }
    if (begin < 0 || end > total || begin > end) {
        set_error("hs_adam: range [%lld, %lld) outside [0, %lld)", (long long)begin, (long long)end,
                  (long long)total);
        return HS_ERR_SHAPE;
    }
    const int64_t c0 = 7 * N, c1 = 10 * N;
    const bool has_colour = begin <= c0 && end >= c1;
    if (ci_mode != 0 && !has_colour && begin < c1 && end > c0) {
        set_error("hs_adam: a colour-init bucket must hold the whole colour segment [%lld, %lld)", (long long)c0,
                  (long long)c1);
        return HS_ERR_SHAPE;
    }
    if (ci_mode < 0 || ci_mode > 2 || (ci_mode && has_colour && (!visited || (ci_mode == 1 && (!maxw || !wsums || !err || B < 1)) ||
                                                                 (ci_mode == 2 && (!packed || !est4))))) {
        set_error("hs_adam: colour-init mode %d needs a buffer that is NULL", ci_mode);
        return HS_ERR_SHAPE;
    }
    if (end == begin) return HS_OK;
    AdamArgs a{};
    a.N = N;
    a.K = K;
    a.begin = begin;
    a.end = end;
    a.p = params;
    a.g = grads;
    a.m = m;
    a.v = v;
    for (int i = 0; i < 9; ++i) a.lr[i] = lrs[i];
    a.b1 = beta1;
    a.b2 = beta2;
    a.inv_bc1 = (float)(1.0 / (1.0 - std::pow((double)beta1, step)));
    a.inv_bc2 = (float)(1.0 / (1.0 - std::pow((double)beta2, step)));
    a.eps = eps;
    a.B = B;
    a.maxw = maxw;
    a.wsums = wsums;
    a.packed = packed;
    a.est4 = est4;
    a.thr = threshold;
    a.visited = visited;
    a.n_init = n_init;
    a.err = err;
    const int ci = has_colour ? ci_mode : 0;
    const bool vec = N % 4 == 0 && begin % 4 == 0 && end % 4 == 0 && (uintptr_t)params % 16 == 0 &&
                     (uintptr_t)grads % 16 == 0 && (uintptr_t)m % 16 == 0 && (uintptr_t)v % 16 == 0;
    const int sms = current_sm_count();
#ifndef HS_ADAM_CTAS_PER_SM
#define HS_ADAM_CTAS_PER_SM 8
#endif
    const unsigned grid = (unsigned)std::min<int64_t>(grid_for((end - begin) / (vec ? 4 : 1), 256),
                                                      (int64_t)sms * HS_ADAM_CTAS_PER_SM);
    cudaStream_t s = HS_CHECK_STREAM(stream);
    if (vec) {
        if (ci == 0) launch_k(adam_kernel<0, true>, grid, 256, 0, s, a);
        else if (ci == 1) launch_k(adam_kernel<1, true>, grid, 256, 0, s, a);
        else launch_k(adam_kernel<2, true>, grid, 256, 0, s, a);
    } else {
        if (ci == 0) launch_k(adam_kernel<0, false>, grid, 256, 0, s, a);
        else if (ci == 1) launch_k(adam_kernel<1, false>, grid, 256, 0, s, a);
        else launch_k(adam_kernel<2, false>, grid, 256, 0, s, a);
    }
    return check_launch("hs_adam");
}

int hs_adam(int64_t N, int K, int64_t mlp_size, float *params, const float *grads, float *m, float *v,
            const float *lrs, int step, float beta1, float beta2, float eps, void *stream) {
    const int64_t total = 14 * N + (int64_t)K * 10 * N + mlp_size;
    return hs_adam_fused(N, K, mlp_size, params, grads, m, v, lrs, step, beta1, beta2, eps, 0, total, 0, 0, nullptr,
                         nullptr, nullptr, nullptr, 0.f, nullptr, nullptr, nullptr, stream);
}

int hs_color_init(int B, int64_t N, const float *maxw, const float *wsums, float threshold,
                  uint8_t *visited, float *params, int *n_init, unsigned long long *err, void *stream) {
    launch_k(color_init_kernel, grid_for(N, 256), 256, 0, HS_CHECK_STREAM(stream), 
        B, N, maxw, wsums, threshold, visited, params + 7 * N, n_init, err);
    return check_launch("hs_color_init");
}

int hs_color_pack(int B, int64_t N, int frame_offset, const float *maxw, const uint8_t *visited, int64_t *packed,
                  void *stream) {
    launch_k(color_pack_kernel, grid_for(N, 256), 256, 0, HS_CHECK_STREAM(stream), B, N, frame_offset, maxw, visited,
                                                                              packed);
    return check_launch("hs_color_pack");
}

int hs_color_select(int B, int64_t N, int frame_offset, const int64_t *packed, const float *wsums, float *est4,
                    unsigned long long *err, void *stream) {
    launch_k(color_select_kernel, grid_for(N, 256), 256, 0, HS_CHECK_STREAM(stream), B, N, frame_offset, packed, wsums,
                                                                                est4, err);
    return check_launch("hs_color_select");
}

int hs_color_apply(int64_t N, const int64_t *packed, const float *est4, float threshold, uint8_t *visited,
                   float *params, int *n_init, void *stream) {
    launch_k(color_apply_kernel, grid_for(N, 256), 256, 0, HS_CHECK_STREAM(stream), N, packed, est4, threshold, visited,
                                                                               params + 7 * N, n_init);
    return check_launch("hs_color_apply");
}

int hs_activate_fwd(int64_t N, const float *raw14, float *act14, unsigned long long *err, void *stream) {
    launch_k(activate_fwd_kernel, grid_for(N, 256), 256, 0, HS_CHECK_STREAM(stream), N, raw14, act14, err);
    return check_launch("hs_activate_fwd");
}

int hs_activate_bwd(int64_t N, const float *raw14, const float *act14, const float *g_act14, float *g_raw14,
                    void *stream) {
    launch_k(activate_bwd_kernel, grid_for(N, 256), 256, 0, HS_CHECK_STREAM(stream), N, raw14, act14, g_act14, g_raw14);
    return check_launch("hs_activate_bwd");
}

int hs_transform_fwd(int64_t N, const float *tangent14, const float *frames, const int32_t *tri_index,
                     const float *bary, float *world14, void *stream) {
    launch_k(transform_fwd_kernel, grid_for(N, 256), 256, 0, HS_CHECK_STREAM(stream), N, tangent14, frames, tri_index,
                                                                                  bary, world14);
    return check_launch("hs_transform_fwd");
}

int hs_transform_bwd(int64_t N, const float *tangent14, const float *frames, const int32_t *tri_index,
                     const float *g_world14, float *g_tangent14, void *stream) {
    launch_k(transform_bwd_kernel, grid_for(N, 256), 256, 0, HS_CHECK_STREAM(stream), N, tangent14, frames, tri_index,
                                                                                  g_world14, g_tangent14);
    return check_launch("hs_transform_bwd");
}

}  // extern "C"
