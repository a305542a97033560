/*
 * hs_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * A float64 CPU restatement of the RGBAvatar reference hot path
 * (/root/reference/pkg/src/headsplat, abbreviated S/ below).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library.  The product path (paper_2503_12886_b200) never links
 * or calls it.
 *
 * Parity is PINNED: tests/test_oracle_golden.py checks every function here
 * against golden vectors produced by running the reference package itself
 * (tests/golden/make_golden.py, committed with its outputs).
 *
 * Arithmetic follows the reference operation by operation in IEEE double
 * (compiled with -ffp-contract=off, no -ffast-math) so results agree with the
 * reference to a few ulp; numpy reductions (BLAS dots, einsum) may order sums
 * differently, which is why golden comparisons use 1e-12-level tolerances.
 *
 * Every frame-level function is a pure function of its inputs and touches no
 * global state, so a caller may run frames on concurrent threads (ctypes drops
 * the GIL for the duration of each call), mirroring the reference's
 * ThreadPoolExecutor scheduler (S/scheduler.py:26-82).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* S/render.py:34-37 */
#define NEAR_PLANE 0.01
#define MIN_RADIUS 0.3
#define ALPHA_CUTOFF (1.0 / 255.0)
#define TERMINATION_EPS 1e-14

/* ------------------------------------------------------------------ MLP */

/* S/model.py:130-142  map_params: psi = W3 relu(W2 relu(W1 theta + b1) + b2) + b3 */
void or_mlp_fwd(int H, int D, int K,
                const double *w1, const double *b1, const double *w2, const double *b2,
                const double *w3, const double *b3, const double *theta,
                double *z1, double *h1, double *z2, double *h2, double *psi) {
    for (int i = 0; i < D; ++i) {
        double acc = 0.0;
        for (int j = 0; j < H; ++j) acc += w1[i * H + j] * theta[j];
        z1[i] = acc + b1[i];
        h1[i] = z1[i] > 0.0 ? z1[i] : 0.0;
    }
    for (int i = 0; i < D; ++i) {
        double acc = 0.0;
        for (int j = 0; j < D; ++j) acc += w2[i * D + j] * h1[j];
        z2[i] = acc + b2[i];
        h2[i] = z2[i] > 0.0 ? z2[i] : 0.0;
    }
    for (int k = 0; k < K; ++k) {
        double acc = 0.0;
        for (int j = 0; j < D; ++j) acc += w3[k * D + j] * h2[j];
        psi[k] = acc + b3[k];
    }
}

/* S/model.py:145-162  mlp_backward; weight grads are ACCUMULATED (+=) so a
 * caller can sum frames in item order like ParamGradients.add_ (S/train.py:86-93). */
void or_mlp_bwd(int H, int D, int K, const double *w2, const double *w3,
                const double *theta, const double *z1, const double *h1,
                const double *z2, const double *h2, const double *gpsi,
                double *gw1, double *gb1, double *gw2, double *gb2,
                double *gw3, double *gb3) {
    double *gz2 = (double *)malloc(sizeof(double) * D);
    double *gz1 = (double *)malloc(sizeof(double) * D);
    for (int k = 0; k < K; ++k) {
        for (int j = 0; j < D; ++j) gw3[k * D + j] += gpsi[k] * h2[j];
        gb3[k] += gpsi[k];
    }
    for (int j = 0; j < D; ++j) {
        double acc = 0.0;
        for (int k = 0; k < K; ++k) acc += w3[k * D + j] * gpsi[k];
        gz2[j] = z2[j] > 0.0 ? acc : 0.0;
    }
    for (int i = 0; i < D; ++i) {
        for (int j = 0; j < D; ++j) gw2[i * D + j] += gz2[i] * h1[j];
        gb2[i] += gz2[i];
    }
    for (int j = 0; j < D; ++j) {
        double acc = 0.0;
        for (int i = 0; i < D; ++i) acc += w2[i * D + j] * gz2[i];
        gz1[j] = z1[j] > 0.0 ? acc : 0.0;
    }
    for (int i = 0; i < D; ++i) {
        for (int j = 0; j < H; ++j) gw1[i * H + j] += gz1[i] * theta[j];
        gb1[i] += gz1[i];
    }
    free(gz2);
    free(gz1);
}

/* --------------------------------------------------------------- blend */

/* S/model.py:165-185  blend.  base10/out10 = [pos 3N | rot 4N | color 3N];
 * deltas = K consecutive blocks of the same 10N layout.  k ascending, psi_k == 0
 * skipped, `out += w * d` with one rounding for the product and one for the sum. */
void or_blend(int64_t N, int K, const double *base10, const double *deltas,
              const double *psi, double *out10) {
    const int64_t E = 10 * N;
    memcpy(out10, base10, sizeof(double) * E);
    for (int k = 0; k < K; ++k) {
        const double w = psi[k];
        if (w == 0.0) continue;
        const double *d = deltas + (int64_t)k * E;
        for (int64_t e = 0; e < E; ++e) {
            double t = w * d[e];
            out10[e] = out10[e] + t;
        }
    }
}

/* S/model.py:188-216  blend_backward for one frame.  g_raw14 = [pos 3N | rot 4N |
 * color 3N | scale 3N | opacity N].  grad_base = copy of g_raw (ACCUMULATED into
 * g_base14), grad_delta_k = psi_k * g (ACCUMULATED into g_deltas), grad_psi_k =
 * <d_k, g> over the blended channels (written). */
void or_blend_backward(int64_t N, int K, const double *deltas, const double *psi,
                       const double *g_raw14, double *g_base14, double *g_deltas,
                       double *g_psi) {
    const int64_t E = 10 * N;
    for (int64_t e = 0; e < 14 * N; ++e) g_base14[e] += g_raw14[e];
    for (int k = 0; k < K; ++k) {
        const double *d = deltas + (int64_t)k * E;
        double *gd = g_deltas + (int64_t)k * E;
        double acc = 0.0;
        for (int64_t e = 0; e < E; ++e) {
            gd[e] += psi[k] * g_raw14[e];
            acc += d[e] * g_raw14[e];
        }
        g_psi[k] = acc;
    }
}

/* ------------------------------------------------------------ activate */

static double sigmoid_ref(double x) {
    /* S/model.py:251-257 two-branch stable sigmoid */
    if (x >= 0.0) return 1.0 / (1.0 + exp(-x));
    double ex = exp(x);
    return ex / (1.0 + ex);
}

/* S/model.py:219-234  activate.  Returns -1, or the first index whose quaternion
 * norm is below 1e-30 (FloatingPointError in the reference, :224-227). */
int64_t or_activate(int64_t N, const double *rot_raw, const double *scale_raw,
                    const double *opac_raw, const double *col_raw, double *rot,
                    double *scale, double *opac, double *col) {
    for (int64_t n = 0; n < N; ++n) {
        const double *q = rot_raw + 4 * n;
        double s = q[0] * q[0];
        s = s + q[1] * q[1];
        s = s + q[2] * q[2];
        s = s + q[3] * q[3];
        double nrm = sqrt(s);
        if (nrm < 1e-30) return n;
        for (int c = 0; c < 4; ++c) rot[4 * n + c] = q[c] / nrm;
        for (int c = 0; c < 3; ++c) scale[3 * n + c] = exp(scale_raw[3 * n + c]);
        opac[n] = sigmoid_ref(opac_raw[n]);
        for (int c = 0; c < 3; ++c) col[3 * n + c] = sigmoid_ref(col_raw[3 * n + c]);
    }
    return -1;
}

/* S/model.py:237-248  activate_backward.  Writes g_raw (pos, rot, scale, opac, col). */
void or_activate_backward(int64_t N, const double *rot_raw, const double *rot_act,
                          const double *scale_act, const double *opac_act,
                          const double *col_act, const double *g_pos, const double *g_rot,
                          const double *g_scale, const double *g_opac, const double *g_col,
                          double *o_pos, double *o_rot, double *o_scale, double *o_opac,
                          double *o_col) {
    for (int64_t n = 0; n < N; ++n) {
        const double *q = rot_raw + 4 * n;
        double s = q[0] * q[0];
        s = s + q[1] * q[1];
        s = s + q[2] * q[2];
        s = s + q[3] * q[3];
        double nrm = sqrt(s);
        const double *y = rot_act + 4 * n;
        const double *g = g_rot + 4 * n;
        double dot = y[0] * g[0];
        dot = dot + y[1] * g[1];
        dot = dot + y[2] * g[2];
        dot = dot + y[3] * g[3];
        for (int c = 0; c < 4; ++c) o_rot[4 * n + c] = (g[c] - y[c] * dot) / nrm;
        for (int c = 0; c < 3; ++c) {
            o_pos[3 * n + c] = g_pos[3 * n + c];
            o_scale[3 * n + c] = g_scale[3 * n + c] * scale_act[3 * n + c];
            double cc = col_act[3 * n + c];
            o_col[3 * n + c] = g_col[3 * n + c] * cc * (1.0 - cc);
        }
        double o = opac_act[n];
        o_opac[n] = g_opac[n] * o * (1.0 - o);
    }
}

/* ---------------------------------------------------------- quaternions */

/* S/quatmath.py:28-40  Hamilton product a (x) b */
static void quat_mul(const double *a, const double *b, double *o) {
    double aw = a[0], ax = a[1], ay = a[2], az = a[3];
    double bw = b[0], bx = b[1], by = b[2], bz = b[3];
    o[0] = aw * bw - ax * bx - ay * by - az * bz;
    o[1] = aw * bx + ax * bw + ay * bz - az * by;
    o[2] = aw * by - ax * bz + ay * bw + az * bx;
    o[3] = aw * bz + ax * by - ay * bx + az * bw;
}

/* S/quatmath.py:58-76  unit-quaternion rotation matrix (no renormalization) */
static void quat_to_mat(const double *q, double *m) {
    double w = q[0], x = q[1], y = q[2], z = q[3];
    m[0] = 1 - 2 * (y * y + z * z);
    m[1] = 2 * (x * y - w * z);
    m[2] = 2 * (x * z + w * y);
    m[3] = 2 * (x * y + w * z);
    m[4] = 1 - 2 * (x * x + z * z);
    m[5] = 2 * (y * z - w * x);
    m[6] = 2 * (x * z - w * y);
    m[7] = 2 * (y * z + w * x);
    m[8] = 1 - 2 * (x * x + y * y);
}

/* S/quatmath.py:79-102  adjoint of quat_to_matrix; g is 3x3 row-major */
static void quat_to_mat_bwd(const double *q, const double *g, double *o) {
    double w = q[0], x = q[1], y = q[2], z = q[3];
    o[0] = 2 * (x * (g[7] - g[5]) + y * (g[2] - g[6]) + z * (g[3] - g[1]));
    o[1] = 2 * (w * (g[7] - g[5]) + y * (g[3] + g[1]) + z * (g[6] + g[2]) - 2 * x * (g[4] + g[8]));
    o[2] = 2 * (w * (g[2] - g[6]) + x * (g[3] + g[1]) + z * (g[7] + g[5]) - 2 * y * (g[0] + g[8]));
    o[3] = 2 * (w * (g[3] - g[1]) + x * (g[6] + g[2]) + y * (g[7] + g[5]) - 2 * z * (g[0] + g[4]));
}

/* ------------------------------------------------------------ transform */

/* S/binding.py:174-188  transform_to_deformed.  frames: frot F*9 (row-major, columns
 * T,B,N), fquat F*4, ftri F*9 (vertex-major: ftri[f*9 + k*3 + j] = vertex k coord j). */
void or_transform(int64_t N, const double *pos_t, const double *rot_t,
                  const double *frot, const double *fquat, const double *ftri,
                  const int64_t *tri_idx, const double *bary,
                  double *pos_w, double *rot_w) {
    for (int64_t n = 0; n < N; ++n) {
        int64_t f = tri_idx[n];
        const double *R = frot + 9 * f;
        const double *V = ftri + 9 * f;
        const double *b = bary + 3 * n;
        const double *x = pos_t + 3 * n;
        for (int j = 0; j < 3; ++j) {
            double t = b[0] * V[0 * 3 + j];
            t = t + b[1] * V[1 * 3 + j];
            t = t + b[2] * V[2 * 3 + j];
            double r = R[j * 3 + 0] * x[0];
            r = r + R[j * 3 + 1] * x[1];
            r = r + R[j * 3 + 2] * x[2];
            pos_w[3 * n + j] = r + t;
        }
        double qr[4];
        quat_mul(fquat + 4 * f, rot_t + 4 * n, qr);
        double s = qr[0] * qr[0];
        s = s + qr[1] * qr[1];
        s = s + qr[2] * qr[2];
        s = s + qr[3] * qr[3];
        double nrm = sqrt(s);
        for (int c = 0; c < 4; ++c) rot_w[4 * n + c] = qr[c] / nrm;
    }
}

/* S/binding.py:191-204 (+ S/quatmath.py:21-25, :43-55)  transform_backward:
 * g_x = R^T g_xw; quaternion: normalize adjoint then left-multiply adjoint. */
void or_transform_backward(int64_t N, const double *rot_t, const double *frot,
                           const double *fquat, const int64_t *tri_idx,
                           const double *g_pos_w, const double *g_rot_w,
                           double *g_pos_t, double *g_rot_t) {
    for (int64_t n = 0; n < N; ++n) {
        int64_t f = tri_idx[n];
        const double *R = frot + 9 * f;
        const double *g = g_pos_w + 3 * n;
        for (int i = 0; i < 3; ++i) {
            double acc = R[0 * 3 + i] * g[0];
            acc = acc + R[1 * 3 + i] * g[1];
            acc = acc + R[2 * 3 + i] * g[2];
            g_pos_t[3 * n + i] = acc;
        }
        const double *a = fquat + 4 * f;
        double qr[4];
        quat_mul(a, rot_t + 4 * n, qr);
        double s = qr[0] * qr[0];
        s = s + qr[1] * qr[1];
        s = s + qr[2] * qr[2];
        s = s + qr[3] * qr[3];
        double nrm = sqrt(s);
        double y[4];
        for (int c = 0; c < 4; ++c) y[c] = qr[c] / nrm;
        const double *go = g_rot_w + 4 * n;
        double dot = y[0] * go[0];
        dot = dot + y[1] * go[1];
        dot = dot + y[2] * go[2];
        dot = dot + y[3] * go[3];
        double gq[4];
        for (int c = 0; c < 4; ++c) gq[c] = (go[c] - y[c] * dot) / nrm;
        double aw = a[0], ax = a[1], ay = a[2], az = a[3];
        double *o = g_rot_t + 4 * n;
        o[0] = aw * gq[0] + ax * gq[1] + ay * gq[2] + az * gq[3];
        o[1] = -ax * gq[0] + aw * gq[1] + az * gq[2] - ay * gq[3];
        o[2] = -ay * gq[0] - az * gq[1] + aw * gq[2] + ax * gq[3];
        o[3] = -az * gq[0] + ay * gq[1] - ax * gq[2] + aw * gq[3];
    }
}

/* ------------------------------------------------------------- project */

/* S/render.py:132-198  _project_kernel, verbatim arithmetic order.
 * cam = [R(9) row-major, t(3), fx, fy, cx, cy]. */
void or_project(int64_t N, const double *position, const double *rotation,
                const double *scale, const double *cam, double *x_cam, double *cov_cam,
                double *mean2d, double *conic, double *radius, uint8_t *valid) {
    const double *rc = cam;
    const double *tc = cam + 9;
    const double fx = cam[12], fy = cam[13], cx = cam[14], cy = cam[15];
    for (int64_t i = 0; i < N; ++i) {
        double px = position[3 * i], py = position[3 * i + 1], pz = position[3 * i + 2];
        double xc = rc[0] * px + rc[1] * py + rc[2] * pz + tc[0];
        double yc = rc[3] * px + rc[4] * py + rc[5] * pz + tc[1];
        double zc = rc[6] * px + rc[7] * py + rc[8] * pz + tc[2];
        x_cam[3 * i] = xc; x_cam[3 * i + 1] = yc; x_cam[3 * i + 2] = zc;
        if (zc <= NEAR_PLANE) { valid[i] = 0; continue; }
        double w = rotation[4 * i], x = rotation[4 * i + 1], y = rotation[4 * i + 2], z = rotation[4 * i + 3];
        double r00 = 1.0 - 2.0 * (y * y + z * z), r01 = 2.0 * (x * y - w * z), r02 = 2.0 * (x * z + w * y);
        double r10 = 2.0 * (x * y + w * z), r11 = 1.0 - 2.0 * (x * x + z * z), r12 = 2.0 * (y * z - w * x);
        double r20 = 2.0 * (x * z - w * y), r21 = 2.0 * (y * z + w * x), r22 = 1.0 - 2.0 * (x * x + y * y);
        double m00 = rc[0] * r00 + rc[1] * r10 + rc[2] * r20;
        double m01 = rc[0] * r01 + rc[1] * r11 + rc[2] * r21;
        double m02 = rc[0] * r02 + rc[1] * r12 + rc[2] * r22;
        double m10 = rc[3] * r00 + rc[4] * r10 + rc[5] * r20;
        double m11 = rc[3] * r01 + rc[4] * r11 + rc[5] * r21;
        double m12 = rc[3] * r02 + rc[4] * r12 + rc[5] * r22;
        double m20 = rc[6] * r00 + rc[7] * r10 + rc[8] * r20;
        double m21 = rc[6] * r01 + rc[7] * r11 + rc[8] * r21;
        double m22 = rc[6] * r02 + rc[7] * r12 + rc[8] * r22;
        double s0 = scale[3 * i] * scale[3 * i];
        double s1 = scale[3 * i + 1] * scale[3 * i + 1];
        double s2 = scale[3 * i + 2] * scale[3 * i + 2];
        double c00 = s0 * m00 * m00 + s1 * m01 * m01 + s2 * m02 * m02;
        double c01 = s0 * m00 * m10 + s1 * m01 * m11 + s2 * m02 * m12;
        double c02 = s0 * m00 * m20 + s1 * m01 * m21 + s2 * m02 * m22;
        double c11 = s0 * m10 * m10 + s1 * m11 * m11 + s2 * m12 * m12;
        double c12 = s0 * m10 * m20 + s1 * m11 * m21 + s2 * m12 * m22;
        double c22 = s0 * m20 * m20 + s1 * m21 * m21 + s2 * m22 * m22;
        double *cv = cov_cam + 9 * i;
        cv[0] = c00; cv[1] = c01; cv[2] = c02;
        cv[3] = c01; cv[4] = c11; cv[5] = c12;
        cv[6] = c02; cv[7] = c12; cv[8] = c22;
        double inv_z = 1.0 / zc;
        double j00 = fx * inv_z;
        double j02 = -fx * xc * inv_z * inv_z;
        double j11 = fy * inv_z;
        double j12 = -fy * yc * inv_z * inv_z;
        double s00 = j00 * (j00 * c00 + j02 * c02) + j02 * (j00 * c02 + j02 * c22);
        double s01 = j11 * (j00 * c01 + j02 * c12) + j12 * (j00 * c02 + j02 * c22);
        double s11 = j11 * (j11 * c11 + j12 * c12) + j12 * (j11 * c12 + j12 * c22);
        double det = s00 * s11 - s01 * s01;
        double mid = 0.5 * (s00 + s11);
        double disc = mid * mid - det;
        if (disc < 0.0) disc = 0.0;
        double lam_max = mid + sqrt(disc);
        double rad = lam_max > 0.0 ? 3.0 * sqrt(lam_max) : 0.0;
        if (det <= 0.0 || rad < MIN_RADIUS) { valid[i] = 0; continue; }
        double inv_det = 1.0 / det;
        conic[3 * i] = s11 * inv_det;
        conic[3 * i + 1] = -s01 * inv_det;
        conic[3 * i + 2] = s00 * inv_det;
        radius[i] = rad;
        mean2d[2 * i] = fx * xc / zc + cx;
        mean2d[2 * i + 1] = fy * yc / zc + cy;
        valid[i] = 1;
    }
}

/* S/render.py:221-223  np.argsort(z, kind="stable"): ascending depth, ties by index.
 * Implemented as a stable merge sort (thread-safe). */
/* merge sort (thread-safe, stable) */
static void msort(int64_t *a, int64_t *tmp, int64_t n, const double *key) {
    if (n < 2) return;
    int64_t h = n / 2;
    msort(a, tmp, h, key);
    msort(a + h, tmp, n - h, key);
    int64_t i = 0, j = h, k = 0;
    while (i < h && j < n) {
        if (key[a[j]] < key[a[i]]) tmp[k++] = a[j++];
        else tmp[k++] = a[i++];
    }
    while (i < h) tmp[k++] = a[i++];
    while (j < n) tmp[k++] = a[j++];
    memcpy(a, tmp, sizeof(int64_t) * n);
}
void or_stable_argsort(int64_t M, const double *depth, int64_t *order) {
    int64_t *tmp = (int64_t *)malloc(sizeof(int64_t) * (M > 0 ? M : 1));
    for (int64_t i = 0; i < M; ++i) order[i] = i;
    msort(order, tmp, M, depth);
    free(tmp);
}

/* ---------------------------------------------------------- rasterize */

/* Pixel bbox of S/render.py:248-251.  When `bbox` is non-NULL the caller supplies
 * it (r_lo, r_hi, c_lo, c_hi per splat) so a checker can replay exactly the pair
 * set another implementation used; otherwise it is derived as in the reference. */
static void splat_bbox(const int32_t *bbox, int64_t s, double mx, double my, double rad,
                       int h, int w, int *r_lo, int *r_hi, int *c_lo, int *c_hi) {
    if (bbox) {
        *r_lo = bbox[4 * s]; *r_hi = bbox[4 * s + 1];
        *c_lo = bbox[4 * s + 2]; *c_hi = bbox[4 * s + 3];
        return;
    }
    int a = (int)ceil(my - rad - 0.5); *r_lo = a > 0 ? a : 0;
    int b = (int)floor(my + rad - 0.5); *r_hi = b < h - 1 ? b : h - 1;
    int c = (int)ceil(mx - rad - 0.5); *c_lo = c > 0 ? c : 0;
    int d = (int)floor(mx + rad - 0.5); *c_hi = d < w - 1 ? d : w - 1;
}

/* S/render.py:233-273  _composite_kernel (arrays already in depth order).
 * image (h*w*3), trans (h*w, init 1), stop (h*w, init M), maxw (M, init 0) are
 * in/out exactly as in the reference; the caller initializes them. */
void or_composite(int64_t M, const double *mean2d, const double *conic,
                  const double *opacity, const double *color, const double *radius,
                  const int32_t *bbox, int h, int w, double *image, double *trans,
                  int64_t *stop, double *maxw) {
    for (int64_t s = 0; s < M; ++s) {
        double op = opacity[s];
        if (op < ALPHA_CUTOFF) continue;
        double qmax = 2.0 * log(op * 255.0) + 1e-9;
        double mx = mean2d[2 * s], my = mean2d[2 * s + 1], rad = radius[s];
        double a = conic[3 * s], b = conic[3 * s + 1], c = conic[3 * s + 2];
        int r_lo, r_hi, c_lo, c_hi;
        splat_bbox(bbox, s, mx, my, rad, h, w, &r_lo, &r_hi, &c_lo, &c_hi);
        for (int r = r_lo; r <= r_hi; ++r) {
            double dy = r + 0.5 - my;
            for (int cc = c_lo; cc <= c_hi; ++cc) {
                int64_t p = (int64_t)r * w + cc;
                double t = trans[p];
                if (t < TERMINATION_EPS) {
                    if (stop[p] > s) stop[p] = s;
                    continue;
                }
                double dx = cc + 0.5 - mx;
                double q = a * dx * dx + 2.0 * b * dx * dy + c * dy * dy;
                if (q > qmax) continue;
                double alpha = op * exp(-0.5 * q);
                if (alpha < ALPHA_CUTOFF) continue;
                double wgt = alpha * t;
                image[3 * p] += wgt * color[3 * s];
                image[3 * p + 1] += wgt * color[3 * s + 1];
                image[3 * p + 2] += wgt * color[3 * s + 2];
                if (wgt > maxw[s]) maxw[s] = wgt;
                trans[p] = t * (1.0 - alpha);
            }
        }
    }
}

/* S/render.py:276-336  _backward_kernel (arrays in depth order).  Outputs are
 * accumulated (+=) into zero-initialized caller buffers. */
void or_composite_backward(int64_t M, const double *mean2d, const double *conic,
                           const double *opacity, const double *color, const double *radius,
                           const int32_t *bbox, int h, int w, const double *trans_final,
                           const int64_t *stop, const double *grad_image,
                           const double *background, double *g_mean, double *g_conic,
                           double *g_opacity, double *g_color) {
    int64_t P = (int64_t)h * w;
    double *t_rev = (double *)malloc(sizeof(double) * P);
    double *suffix = (double *)malloc(sizeof(double) * P);
    for (int64_t p = 0; p < P; ++p) {
        t_rev[p] = trans_final[p];
        suffix[p] = trans_final[p] * (grad_image[3 * p] * background[0]
                                      + grad_image[3 * p + 1] * background[1]
                                      + grad_image[3 * p + 2] * background[2]);
    }
    for (int64_t s = M - 1; s >= 0; --s) {
        double op = opacity[s];
        if (op < ALPHA_CUTOFF) continue;
        double qmax = 2.0 * log(op * 255.0) + 1e-9;
        double mx = mean2d[2 * s], my = mean2d[2 * s + 1], rad = radius[s];
        double a = conic[3 * s], b = conic[3 * s + 1], c = conic[3 * s + 2];
        int r_lo, r_hi, c_lo, c_hi;
        splat_bbox(bbox, s, mx, my, rad, h, w, &r_lo, &r_hi, &c_lo, &c_hi);
        for (int r = r_lo; r <= r_hi; ++r) {
            double dy = r + 0.5 - my;
            for (int cc = c_lo; cc <= c_hi; ++cc) {
                int64_t p = (int64_t)r * w + cc;
                if (s >= stop[p]) continue;
                double dx = cc + 0.5 - mx;
                double q = a * dx * dx + 2.0 * b * dx * dy + c * dy * dy;
                if (q > qmax) continue;
                double g = exp(-0.5 * q);
                double alpha = op * g;
                if (alpha < ALPHA_CUTOFF) continue;
                double one_m = 1.0 - alpha;
                double t_prior = t_rev[p] / one_m;
                const double *gi = grad_image + 3 * p;
                double gw = gi[0] * color[3 * s] + gi[1] * color[3 * s + 1] + gi[2] * color[3 * s + 2];
                double wgt = alpha * t_prior;
                g_color[3 * s] += wgt * gi[0];
                g_color[3 * s + 1] += wgt * gi[1];
                g_color[3 * s + 2] += wgt * gi[2];
                double d_alpha = t_prior * gw - suffix[p] / one_m;
                g_opacity[s] += g * d_alpha;
                double dq = -0.5 * alpha * d_alpha;
                g_conic[3 * s] += dq * dx * dx;
                g_conic[3 * s + 1] += 2.0 * dq * dx * dy;
                g_conic[3 * s + 2] += dq * dy * dy;
                g_mean[2 * s] += -2.0 * dq * (a * dx + b * dy);
                g_mean[2 * s + 1] += -2.0 * dq * (b * dx + c * dy);
                suffix[p] += wgt * gw;
                t_rev[p] = t_prior;
            }
        }
    }
    free(t_rev);
    free(suffix);
}

/* Checker extension (not in the reference): the pixels where one of the
 * compositing decisions of S/render.py:233-273 sits within fp32 noise of its
 * threshold, so an fp32 implementation and this float64 restatement may decide
 * it differently.  The loop is or_composite's; a pixel is flagged when, for some
 * splat it tests,
 *   |alpha - 1/255| < 2e-6         (alpha cutoff, :266)
 *   |q - qmax| < 1e-4 (1 + qmax)   (ellipse cutoff, :262)
 *   alpha > 1 - 1e-6               (fp32 rounds alpha to 1, T to ~0)
 *   T (1 - alpha) within 1e-3 relative of 1e-14 (termination, :254)
 * mask (h*w bytes) is OR-ed, so a caller can accumulate over frames. */
void or_flip_mask(int64_t M, const double *mean2d, const double *conic,
                  const double *opacity, const double *radius, const int32_t *bbox,
                  int h, int w, uint8_t *mask) {
    int64_t P = (int64_t)h * w;
    double *trans = (double *)malloc(sizeof(double) * P);
    for (int64_t p = 0; p < P; ++p) trans[p] = 1.0;
    for (int64_t s = 0; s < M; ++s) {
        double op = opacity[s];
        if (op < ALPHA_CUTOFF) continue;
        double qmax = 2.0 * log(op * 255.0) + 1e-9;
        double mx = mean2d[2 * s], my = mean2d[2 * s + 1], rad = radius[s];
        double a = conic[3 * s], b = conic[3 * s + 1], c = conic[3 * s + 2];
        int r_lo, r_hi, c_lo, c_hi;
        splat_bbox(bbox, s, mx, my, rad, h, w, &r_lo, &r_hi, &c_lo, &c_hi);
        for (int r = r_lo; r <= r_hi; ++r) {
            double dy = r + 0.5 - my;
            for (int cc = c_lo; cc <= c_hi; ++cc) {
                int64_t p = (int64_t)r * w + cc;
                double t = trans[p];
                if (t < TERMINATION_EPS) continue;
                double dx = cc + 0.5 - mx;
                double q = a * dx * dx + 2.0 * b * dx * dy + c * dy * dy;
                if (fabs(q - qmax) < 1e-4 * (1.0 + fabs(qmax))) mask[p] = 1;
                if (q > qmax) continue;
                double alpha = op * exp(-0.5 * q);
                if (fabs(alpha - ALPHA_CUTOFF) < 2e-6) mask[p] = 1;
                if (alpha < ALPHA_CUTOFF) continue;
                if (alpha > 1.0 - 1e-6) mask[p] = 1;
                double tn = t * (1.0 - alpha);
                if (fabs(tn - TERMINATION_EPS) < 1e-3 * TERMINATION_EPS) mask[p] = 1;
                trans[p] = tn;
            }
        }
    }
    free(trans);
}

/* S/render.py:339-377  _weight_sums_kernel (arrays in depth order); num (M*3) and
 * den (M) accumulate into zero-initialized caller buffers. */
void or_weight_sums(int64_t M, const double *mean2d, const double *conic,
                    const double *opacity, const double *radius, const int32_t *bbox,
                    int h, int w, const double *image, double *num, double *den) {
    int64_t P = (int64_t)h * w;
    double *trans = (double *)malloc(sizeof(double) * P);
    for (int64_t p = 0; p < P; ++p) trans[p] = 1.0;
    for (int64_t s = 0; s < M; ++s) {
        double op = opacity[s];
        if (op < ALPHA_CUTOFF) continue;
        double qmax = 2.0 * log(op * 255.0) + 1e-9;
        double mx = mean2d[2 * s], my = mean2d[2 * s + 1], rad = radius[s];
        double a = conic[3 * s], b = conic[3 * s + 1], c = conic[3 * s + 2];
        int r_lo, r_hi, c_lo, c_hi;
        splat_bbox(bbox, s, mx, my, rad, h, w, &r_lo, &r_hi, &c_lo, &c_hi);
        for (int r = r_lo; r <= r_hi; ++r) {
            double dy = r + 0.5 - my;
            for (int cc = c_lo; cc <= c_hi; ++cc) {
                int64_t p = (int64_t)r * w + cc;
                double t = trans[p];
                if (t < TERMINATION_EPS) continue;
                double dx = cc + 0.5 - mx;
                double q = a * dx * dx + 2.0 * b * dx * dy + c * dy * dy;
                if (q > qmax) continue;
                double alpha = op * exp(-0.5 * q);
                if (alpha < ALPHA_CUTOFF) continue;
                double wgt = alpha * t;
                num[3 * s] += wgt * image[3 * p];
                num[3 * s + 1] += wgt * image[3 * p + 1];
                num[3 * s + 2] += wgt * image[3 * p + 2];
                den[s] += wgt;
                trans[p] = t * (1.0 - alpha);
            }
        }
    }
    free(trans);
}

/* S/render.py:432-497  _preprocess_backward for the kept subset (M splats in
 * source-index order, idx maps to the world set).  Writes the world grads of the
 * kept Gaussians; the caller zero-fills culled ones. */
void or_preprocess_backward(int64_t M, const int64_t *idx, const double *x_cam,
                            const double *cov_cam, const double *conic,
                            const double *world_rot, const double *world_scale,
                            const double *cam, const double *g_mean, const double *g_conic,
                            const double *g_opacity, const double *g_color,
                            double *o_pos, double *o_rot, double *o_scale, double *o_opac,
                            double *o_col) {
    const double *rc = cam;
    const double fx = cam[12], fy = cam[13];
    for (int64_t s = 0; s < M; ++s) {
        int64_t n = idx[s];
        const double *xc = x_cam + 3 * s;
        double z = xc[2];
        double inv_z = 1.0 / z;
        double ca = conic[3 * s], cb = conic[3 * s + 1], cc = conic[3 * s + 2];
        double ga = g_conic[3 * s], gb = 0.5 * g_conic[3 * s + 1], gc = g_conic[3 * s + 2];
        double gs00 = -(ca * (ca * ga + cb * gb) + cb * (ca * gb + cb * gc));
        double gs01 = -(ca * (cb * ga + cc * gb) + cb * (cb * gb + cc * gc));
        double gs11 = -(cb * (cb * ga + cc * gb) + cc * (cb * gb + cc * gc));
        double G[4] = {gs00, gs01, gs01, gs11};
        double J[6] = {fx * inv_z, 0.0, -fx * xc[0] * inv_z * inv_z,
                       0.0, fy * inv_z, -fy * xc[1] * inv_z * inv_z};
        /* g_cov_cam = J^T G J  (einsum "nji,njk,nkl->nil") */
        double gcc[9];
        for (int i = 0; i < 3; ++i)
            for (int l = 0; l < 3; ++l) {
                double acc = 0.0;
                for (int j = 0; j < 2; ++j)
                    for (int k = 0; k < 2; ++k) acc += J[j * 3 + i] * G[j * 2 + k] * J[k * 3 + l];
                gcc[i * 3 + l] = acc;
            }
        /* g_j = (G + G^T) J cov_cam  (einsum "nij,njk,nkl->nil") */
        const double *C = cov_cam + 9 * s;
        double GG[4] = {G[0] + G[0], G[1] + G[2], G[2] + G[1], G[3] + G[3]};
        double gj[6];
        for (int i = 0; i < 2; ++i)
            for (int l = 0; l < 3; ++l) {
                double acc = 0.0;
                for (int j = 0; j < 2; ++j)
                    for (int k = 0; k < 3; ++k) acc += GG[i * 2 + j] * J[j * 3 + k] * C[k * 3 + l];
                gj[i * 3 + l] = acc;
            }
        /* g_cov_world = Rc^T g_cov_cam Rc  (einsum "ji,njk,kl->nil") */
        double gw[9];
        for (int i = 0; i < 3; ++i)
            for (int l = 0; l < 3; ++l) {
                double acc = 0.0;
                for (int j = 0; j < 3; ++j)
                    for (int k = 0; k < 3; ++k) acc += rc[j * 3 + i] * gcc[j * 3 + k] * rc[k * 3 + l];
                gw[i * 3 + l] = acc;
            }
        const double *q = world_rot + 4 * n;
        const double *sc = world_scale + 3 * n;
        double R[9];
        quat_to_mat(q, R);
        double ss[3] = {sc[0] * sc[0], sc[1] * sc[1], sc[2] * sc[2]};
        /* g_rot = (g + g^T) (R diag(s^2)) */
        double grot[9];
        for (int i = 0; i < 3; ++i)
            for (int k = 0; k < 3; ++k) {
                double acc = 0.0;
                for (int j = 0; j < 3; ++j) acc += (gw[i * 3 + j] + gw[j * 3 + i]) * (R[j * 3 + k] * ss[k]);
                grot[i * 3 + k] = acc;
            }
        /* g_scale = 2 s diag(R^T g R) */
        for (int i = 0; i < 3; ++i) {
            double acc = 0.0;
            for (int j = 0; j < 3; ++j)
                for (int k = 0; k < 3; ++k) acc += R[j * 3 + i] * gw[j * 3 + k] * R[k * 3 + i];
            o_scale[3 * n + i] = 2.0 * sc[i] * acc;
        }
        quat_to_mat_bwd(q, grot, o_rot + 4 * n);
        const double *gm = g_mean + 2 * s;
        double gx = gm[0] * fx * inv_z + gj[2] * (-fx * inv_z * inv_z);
        double gy = gm[1] * fy * inv_z + gj[5] * (-fy * inv_z * inv_z);
        double gz = -gm[0] * fx * xc[0] * inv_z * inv_z
                    - gm[1] * fy * xc[1] * inv_z * inv_z
                    + gj[0] * (-fx * inv_z * inv_z)
                    + gj[2] * (2.0 * fx * xc[0] * (inv_z * inv_z * inv_z))
                    + gj[4] * (-fy * inv_z * inv_z)
                    + gj[5] * (2.0 * fy * xc[1] * (inv_z * inv_z * inv_z));
        /* g_pos = g_x_cam @ rc */
        for (int j = 0; j < 3; ++j) o_pos[3 * n + j] = gx * rc[0 * 3 + j] + gy * rc[1 * 3 + j] + gz * rc[2 * 3 + j];
        o_opac[n] = g_opacity[s];
        for (int c = 0; c < 3; ++c) o_col[3 * n + c] = g_color[3 * s + c];
    }
}

/* -------------------------------------------------------------- Adam */

/* S/optim.py:28-40  in-place bias-corrected Adam over one group. */
void or_adam(int64_t n, double *param, const double *grad, double *m, double *v,
             int step, double lr, double beta1, double beta2, double eps) {
    double bc1 = 1.0 - pow(beta1, step);
    double bc2 = 1.0 - pow(beta2, step);
    for (int64_t i = 0; i < n; ++i) {
        m[i] = m[i] * beta1;
        m[i] = m[i] + (1.0 - beta1) * grad[i];
        v[i] = v[i] * beta2;
        v[i] = v[i] + (1.0 - beta2) * (grad[i] * grad[i]);
        double mh = m[i] / bc1;
        double vh = v[i] / bc2;
        param[i] = param[i] - lr * mh / (sqrt(vh) + eps);
    }
}
