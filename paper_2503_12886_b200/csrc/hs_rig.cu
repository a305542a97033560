// hs_rig.cu -- device head rig and per-triangle tangent frames.
//
// Turns rig parameters theta (B x (E + 3): E expression coefficients, then an
// axis-angle pose) into the MeshFrames the projection consumes (B x F x 22 fp32:
// TBN rotation 9 | polar-factor quaternion 4 | deformed triangle vertices 9), so
// a render or a training step with unseen theta needs no host mesh work.
//
//   rig_evaluate          S/rig.py:57-66      verts = (base + sum_e theta_e X_e) R(pose)^T
//   axis_angle_to_matrix  S/quatmath.py:152-161  (Rodrigues, identity below 1e-12 rad)
//   mesh_frames/_tbn_batch S/binding.py:67-78, :93-115  (exact tangent solve, unit normal,
//                         DegenerateTriangleError for |det_uv| or |e1 x e2| < 1e-12)
//   polar_rotation        S/binding.py:80-90  (rotation factor of the SVD, det fixed to +1)
//   matrix_to_quat        S/quatmath.py:105-149  (four-branch, first max wins, unnormalised)
//
// Grid (face blocks, frames): each CTA builds the frame's deformed vertices in shared
// memory (fp64, like the reference; V = 561 is cheap to redo) and then handles 128
// faces, one thread per face.  The polar factor is computed from
// the eigen-decomposition of M^T M (cyclic Jacobi, fp64):
//   R = u1 v1^T + u2 v2^T + (u1 x u2)(v1 x v2)^T,   u_i = M v_i / sigma_i
// for the two largest singular pairs -- the reference's U V^T with the third column
// of U flipped when det < 0, independent of the eigenvector signs.
#include "hs_common.cuh"

namespace hs {

__device__ __forceinline__ void cross3(const double *a, const double *b, double *c) {
    c[0] = a[1] * b[2] - a[2] * b[1];
    c[1] = a[2] * b[0] - a[0] * b[2];
    c[2] = a[0] * b[1] - a[1] * b[0];
}

// Eigen-decomposition of a symmetric 3x3 (cyclic Jacobi); columns of V are the
// eigenvectors, eigenvalues sorted descending.
__device__ void sym_eig3(double S[3][3], double V[3][3], double lam[3]) {
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) V[i][j] = i == j ? 1.0 : 0.0;
    for (int sweep = 0; sweep < 12; ++sweep) {
        const double off = S[0][1] * S[0][1] + S[0][2] * S[0][2] + S[1][2] * S[1][2];
        const double diag = S[0][0] * S[0][0] + S[1][1] * S[1][1] + S[2][2] * S[2][2];
        if (off <= 1e-34 * diag) break;
        for (int p = 0; p < 2; ++p) {
            for (int q = p + 1; q < 3; ++q) {
                const double apq = S[p][q];
                if (apq == 0.0) continue;
                const double theta = (S[q][q] - S[p][p]) / (2.0 * apq);
                const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
                for (int k = 0; k < 3; ++k) {          // S <- J^T S J
                    const double skp = S[k][p], skq = S[k][q];
                    S[k][p] = c * skp - s * skq;
                    S[k][q] = s * skp + c * skq;
                }
                for (int k = 0; k < 3; ++k) {
                    const double spk = S[p][k], sqk = S[q][k];
                    S[p][k] = c * spk - s * sqk;
                    S[q][k] = s * spk + c * sqk;
                }
                for (int k = 0; k < 3; ++k) {          // V <- V J
                    const double vkp = V[k][p], vkq = V[k][q];
                    V[k][p] = c * vkp - s * vkq;
                    V[k][q] = s * vkp + c * vkq;
                }
            }
        }
    }
    int order[3] = {0, 1, 2};
    for (int i = 0; i < 3; ++i) lam[i] = S[i][i];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2 - i; ++j)
            if (lam[order[j]] < lam[order[j + 1]]) {
                const int t = order[j];
                order[j] = order[j + 1];
                order[j + 1] = t;
            }
    double W[3][3], l2[3];
    for (int c = 0; c < 3; ++c) {
        l2[c] = lam[order[c]];
        for (int r = 0; r < 3; ++r) W[r][c] = V[r][order[c]];
    }
    for (int c = 0; c < 3; ++c) {
        lam[c] = l2[c];
        for (int r = 0; r < 3; ++r) V[r][c] = W[r][c];
    }
}

__device__ void polar_rotation(const double M[3][3], double R[3][3]) {
    double S[3][3], V[3][3], lam[3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) S[i][j] = M[0][i] * M[0][j] + M[1][i] * M[1][j] + M[2][i] * M[2][j];
    sym_eig3(S, V, lam);
    double u[2][3], v[2][3];
    for (int c = 0; c < 2; ++c) {
        for (int r = 0; r < 3; ++r) v[c][r] = V[r][c];
        double mv[3];
        for (int r = 0; r < 3; ++r) mv[r] = M[r][0] * v[c][0] + M[r][1] * v[c][1] + M[r][2] * v[c][2];
        const double nrm = sqrt(mv[0] * mv[0] + mv[1] * mv[1] + mv[2] * mv[2]);
        for (int r = 0; r < 3; ++r) u[c][r] = mv[r] / nrm;
    }
    double u3[3], v3[3];
    cross3(u[0], u[1], u3);
    cross3(v[0], v[1], v3);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) R[i][j] = u[0][i] * v[0][j] + u[1][i] * v[1][j] + u3[i] * v3[j];
}

// S/quatmath.py:105-149 (wxyz, not normalised; np.argmax: first max wins)
__device__ void matrix_to_quat(const double m[3][3], double q[4]) {
    const double t[4] = {1.0 + m[0][0] + m[1][1] + m[2][2], 1.0 + m[0][0] - m[1][1] - m[2][2],
                         1.0 - m[0][0] + m[1][1] - m[2][2], 1.0 - m[0][0] - m[1][1] + m[2][2]};
    int br = 0;
    for (int i = 1; i < 4; ++i)
        if (t[i] > t[br]) br = i;
    const double s = 2.0 * sqrt(fmax(t[br], 1e-30));
    switch (br) {
        case 0:
            q[0] = 0.25 * s;
            q[1] = (m[2][1] - m[1][2]) / s;
            q[2] = (m[0][2] - m[2][0]) / s;
            q[3] = (m[1][0] - m[0][1]) / s;
            break;
        case 1:
            q[0] = (m[2][1] - m[1][2]) / s;
            q[1] = 0.25 * s;
            q[2] = (m[0][1] + m[1][0]) / s;
            q[3] = (m[0][2] + m[2][0]) / s;
            break;
        case 2:
            q[0] = (m[0][2] - m[2][0]) / s;
            q[1] = (m[0][1] + m[1][0]) / s;
            q[2] = 0.25 * s;
            q[3] = (m[1][2] + m[2][1]) / s;
            break;
        default:
            q[0] = (m[1][0] - m[0][1]) / s;
            q[1] = (m[0][2] + m[2][0]) / s;
            q[2] = (m[1][2] + m[2][1]) / s;
            q[3] = 0.25 * s;
            break;
    }
}

// rig_evaluate (S/rig.py:57-66) of one frame into verts[V][3]:
// (base + sum_e theta_e X_e) R^T with R = axis_angle_to_matrix(pose) (S/quatmath.py:152-161)
__device__ void rig_vertices(int V, int E, const double *__restrict__ base, const double *__restrict__ bases,
                             const float *__restrict__ th, double *verts) {
    const double px = th[E], py = th[E + 1], pz = th[E + 2];
    const double ang = sqrt(px * px + py * py + pz * pz);
    double R[3][3] = {{1.0, 0.0, 0.0}, {0.0, 1.0, 0.0}, {0.0, 0.0, 1.0}};
    if (!(ang < 1e-12)) {
        const double kx = px / ang, ky = py / ang, kz = pz / ang;
        const double K[3][3] = {{0.0, -kz, ky}, {kz, 0.0, -kx}, {-ky, kx, 0.0}};
        const double sn = sin(ang), cs1 = 1.0 - cos(ang);
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) {
                const double kk = K[i][0] * K[0][j] + K[i][1] * K[1][j] + K[i][2] * K[2][j];
                R[i][j] += sn * K[i][j] + cs1 * kk;
            }
    }
    for (int v = threadIdx.x; v < V; v += blockDim.x) {
        double p[3] = {base[3 * v], base[3 * v + 1], base[3 * v + 2]};
        for (int e = 0; e < E; ++e) {
            const double t = th[e];
            const double *x = bases + ((int64_t)e * V + v) * 3;
            p[0] += t * x[0];
            p[1] += t * x[1];
            p[2] += t * x[2];
        }
        for (int i = 0; i < 3; ++i) verts[3 * v + i] = p[0] * R[i][0] + p[1] * R[i][1] + p[2] * R[i][2];
    }
}

constexpr int kRigThreads = 128;   // faces per CTA (each CTA rebuilds the small vertex set)

__global__ void __launch_bounds__(kRigThreads) rig_frames_kernel(int V, int F, int E, const double *__restrict__ base,
                                                                 const double *__restrict__ bases,
                                                                 const int32_t *__restrict__ faces,
                                                                 const double *__restrict__ uv,
                                                                 const float *__restrict__ theta,
                                                                 const double *__restrict__ vertices,
                                                                 float *__restrict__ frames,
                                                                 unsigned long long *err) {
    pdl_prologue();
    extern __shared__ double s_verts[];           // [V][3]
    const int b = blockIdx.y;
    if (vertices) {                               // mesh_frames of given vertices (no rig)
        for (int i = threadIdx.x; i < 3 * V; i += blockDim.x) s_verts[i] = vertices[(int64_t)b * 3 * V + i];
    } else {
        rig_vertices(V, E, base, bases, theta + (int64_t)b * (E + 3), s_verts);
    }
    __syncthreads();
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < F; f += gridDim.x * blockDim.x) {
        double tri[3][3];
        double tuv[3][2];
        for (int c = 0; c < 3; ++c) {
            const int vi = faces[3 * f + c];
            for (int i = 0; i < 3; ++i) tri[c][i] = s_verts[3 * vi + i];
            tuv[c][0] = uv[2 * vi];
            tuv[c][1] = uv[2 * vi + 1];
        }
        double e1[3], e2[3], cr[3];
        for (int i = 0; i < 3; ++i) {
            e1[i] = tri[1][i] - tri[0][i];
            e2[i] = tri[2][i] - tri[0][i];
        }
        cross3(e1, e2, cr);
        const double cn = sqrt(cr[0] * cr[0] + cr[1] * cr[1] + cr[2] * cr[2]);
        const double du1 = tuv[1][0] - tuv[0][0], du2 = tuv[2][0] - tuv[0][0];
        const double dv1 = tuv[1][1] - tuv[0][1], dv2 = tuv[2][1] - tuv[0][1];
        const double det = du1 * dv2 - du2 * dv1;
        if (fabs(det) < 1e-12) {
            atomicMin(err, err_code(3, b, 0, f));
            continue;
        }
        if (cn < 1e-12) {
            atomicMin(err, err_code(3, b, 1, f));
            continue;
        }
        const double inv = 1.0 / det;
        double M[3][3];                            // columns T, B, N
        for (int i = 0; i < 3; ++i) {
            M[i][0] = (dv2 * e1[i] - dv1 * e2[i]) * inv;
            M[i][1] = (-du2 * e1[i] + du1 * e2[i]) * inv;
            M[i][2] = cr[i] / cn;
        }
        double Rp[3][3], q[4];
        polar_rotation(M, Rp);
        matrix_to_quat(Rp, q);
        float *o = frames + ((int64_t)b * F + f) * 22;
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) o[3 * i + j] = (float)M[i][j];
        for (int i = 0; i < 4; ++i) o[9 + i] = (float)q[i];
        for (int c = 0; c < 3; ++c)
            for (int i = 0; i < 3; ++i) o[13 + 3 * c + i] = (float)tri[c][i];
    }
}

}  // namespace hs

using namespace hs;

extern "C" {

int hs_rig_frames(int B, int V, int F, int E, const double *base_vertices, const double *expr_bases,
                  const int32_t *faces, const double *uv_coords, const float *theta, const double *vertices,
                  float *frames, unsigned long long *err, void *stream) {
    const size_t smem = sizeof(double) * 3 * (size_t)V;
    if (B < 1 || V < 3 || F < 1 || E < 0 || smem > 200 * 1024 || (!theta && !vertices)) {
        set_error("hs_rig_frames: unsupported sizes B=%d V=%d F=%d E=%d", B, V, F, E);
        return HS_ERR_SHAPE;
    }
    if (smem > 48 * 1024) cudaFuncSetAttribute(rig_frames_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const dim3 grid((F + kRigThreads - 1) / kRigThreads, B);
    launch_k(rig_frames_kernel, grid, kRigThreads, smem, HS_CHECK_STREAM(stream), V, F, E, base_vertices, expr_bases, faces,
                                                                        uv_coords, theta, vertices, frames, err);
    return check_launch("hs_rig_frames");
}

}  // extern "C"
