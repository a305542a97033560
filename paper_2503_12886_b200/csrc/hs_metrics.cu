// hs_metrics.cu -- evaluation metrics on device: PSNR / SSIM / L1 of
// a rendered batch against its targets composited over black, as S/train.py:342-360
// `evaluate` computes per frame (S/metrics.py:25-77 psnr, ssim, composite_over).
//
// Everything in fp64 like the reference (values in [0, 1]; the SSIM variance terms
// E[x^2] - mu^2 cancel badly in fp32).  One launch accumulates, per frame, the sum of
// squared and absolute errors and, per channel, the sum of the SSIM map over the
// valid-mode window positions; the host divides.  SSIM: Gaussian window (size 11,
// sigma 1.5, normalised), separable valid filtering -- each CTA owns a 16 x 32 tile
// of window positions of one (frame, channel), filters the 5 moment images
// horizontally into shared memory, then vertically, then evaluates the SSIM map.
#include <algorithm>
#include <cmath>

#include "hs_common.cuh"

namespace hs {

constexpr int kWin = 11;
constexpr int kTH = 16, kTW = 32;           // window positions per CTA
constexpr int kRows = kTH + kWin - 1;

struct Window {
    double w[kWin];
};

__device__ __forceinline__ void load_px(const float *__restrict__ pred, const uint8_t *__restrict__ target,
                                        int64_t pix, int c, double &x, double &y) {
    x = (double)pred[pix * 3 + c];
    const uchar4 t = reinterpret_cast<const uchar4 *>(target)[pix];
    const double a = (double)t.w / 255.0;
    const double v = (double)(c == 0 ? t.x : c == 1 ? t.y : t.z) / 255.0;
    y = v * a;                                   // composite_over(rgba, black)
}

__global__ void __launch_bounds__(256) ssim_kernel(int H, int W, const float *__restrict__ pred,
                                                   const uint8_t *__restrict__ target, Window win, double c1,
                                                   double c2, double *__restrict__ out) {
    pdl_prologue();
    __shared__ double hrow[5][kRows][kTW];
    __shared__ double red[8];
    const int Hv = H - kWin + 1, Wv = W - kWin + 1;
    const int b = blockIdx.z / 3, c = blockIdx.z % 3;
    const int r0 = blockIdx.y * kTH, c0 = blockIdx.x * kTW;
    const int64_t fbase = (int64_t)b * H * W;
    for (int e = threadIdx.x; e < kRows * kTW; e += blockDim.x) {
        const int r = e / kTW, cc = e % kTW;
        const int gy = r0 + r, gx = c0 + cc;
        double s[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        if (gy < H && gx < Wv) {
            for (int k = 0; k < kWin; ++k) {
                double x, y;
                load_px(pred, target, fbase + (int64_t)gy * W + gx + k, c, x, y);
                const double w = win.w[k];
                s[0] += w * x;
                s[1] += w * y;
                s[2] += w * (x * x);
                s[3] += w * (y * y);
                s[4] += w * (x * y);
            }
        }
        for (int q = 0; q < 5; ++q) hrow[q][r][cc] = s[q];
    }
    __syncthreads();
    double acc = 0.0;
    for (int e = threadIdx.x; e < kTH * kTW; e += blockDim.x) {
        const int r = e / kTW, cc = e % kTW;
        if (r0 + r >= Hv || c0 + cc >= Wv) continue;
        double m[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        for (int k = 0; k < kWin; ++k) {
            const double w = win.w[k];
            for (int q = 0; q < 5; ++q) m[q] += w * hrow[q][r + k][cc];
        }
        const double mx = m[0], my = m[1];
        const double xx = m[2] - mx * mx, yy = m[3] - my * my, xy = m[4] - mx * my;
        acc += ((2.0 * mx * my + c1) * (2.0 * xy + c2)) / ((mx * mx + my * my + c1) * (xx + yy + c2));
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
        atomicAdd(out + (int64_t)b * 5 + 2 + c, s);
    }
}

// per frame: sum (pred - target)^2 and sum |pred - target| over H x W x 3
__global__ void __launch_bounds__(256) err_sums_kernel(int64_t HW, const float *__restrict__ pred,
                                                       const uint8_t *__restrict__ target,
                                                       double *__restrict__ out) {
    pdl_prologue();
    __shared__ double red[2][8];
    const int b = blockIdx.y;
    double sq = 0.0, ab = 0.0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < HW; p += (int64_t)gridDim.x * blockDim.x) {
        for (int c = 0; c < 3; ++c) {
            double x, y;
            load_px(pred, target, (int64_t)b * HW + p, c, x, y);
            const double d = x - y;
            sq += d * d;
            ab += fabs(d);
        }
    }
    for (int o = 16; o; o >>= 1) {
        sq += __shfl_xor_sync(0xffffffffu, sq, o);
        ab += __shfl_xor_sync(0xffffffffu, ab, o);
    }
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = sq;
        red[1][threadIdx.x >> 5] = ab;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s0 = 0.0, s1 = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
            s0 += red[0][i];
            s1 += red[1][i];
        }
        atomicAdd(out + (int64_t)b * 5, s0);
        atomicAdd(out + (int64_t)b * 5 + 1, s1);
    }
}

}  // namespace hs

using namespace hs;

extern "C" {

int hs_image_metrics(int B, int H, int W, const float *pred, const uint8_t *target_rgba, double *sums, void *stream) {
    if (B < 1 || H < kWin || W < kWin) {
        set_error("hs_image_metrics: images must be at least %dx%d (got B=%d %dx%d)", kWin, kWin, B, H, W);
        return HS_ERR_SHAPE;
    }
    cudaStream_t s = HS_CHECK_STREAM(stream);
    cudaMemsetAsync(sums, 0, sizeof(double) * 5 * (size_t)B, s);
    Window win;
    double tot = 0.0;
    for (int k = 0; k < kWin; ++k) {                 // S/metrics.py:33-37
        const double x = k - (kWin - 1) / 2.0;
        win.w[k] = std::exp(-(x * x) / (2.0 * 1.5 * 1.5));
        tot += win.w[k];
    }
    for (int k = 0; k < kWin; ++k) win.w[k] /= tot;
    const int Hv = H - kWin + 1, Wv = W - kWin + 1;
    const dim3 sgrid((Wv + kTW - 1) / kTW, (Hv + kTH - 1) / kTH, 3 * B);
    launch_k(ssim_kernel, sgrid, 256, 0, s, H, W, pred, target_rgba, win, 0.01 * 0.01, 0.03 * 0.03, sums);
    const dim3 egrid((unsigned)std::min<int64_t>(grid_for((int64_t)H * W, 256), 148), B);
    launch_k(err_sums_kernel, egrid, 256, 0, s, (int64_t)H * W, pred, target_rgba, sums);
    return check_launch("hs_image_metrics");
}

}  // extern "C"
