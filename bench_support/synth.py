"""BENCH / TEST SUPPORT (not the product): host-side synthetic workload -- the head rig,
UV binding, mesh frames and avatar init.

These are the data producers on either side of the hot path (SURVEY §8f #2 marks
the device rig as "next"; today they run once per frame on the host, cached,
exactly as in the reference).  Restated from the reference so the bench and the
GPU tests can build the BASELINE.json shapes on the GPU box, where the reference
package does not exist.  Parity with the reference is checked by
tests/test_synth.py against tests/golden/binding.npz and counts.json (UV-binding
checksums at uv 141/224/317).

  build_head_rig   S/rig.py:69-114      rig_evaluate   S/rig.py:57-66
  mesh_frames      S/binding.py:67-115  (TBN, polar rotation, S/quatmath.py:105-149)
  bind_gaussians   S/binding.py:118-171 init_avatar    S/train.py:96-120
  frontal camera   S/render.py:75-84
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from paper_2503_12886_b200.io import Rig

# ------------------------------------------------------------------------ rig


HeadRig = Rig     # the rig container of the product's io module


def build_head_rig(rows=16, cols=32, num_expressions=10, seed=7) -> HeadRig:
    """Egg-shaped spherical band with a duplicated UV seam column (S/rig.py:69-114)."""
    lat = np.linspace(np.radians(-75.0), np.radians(75.0), rows + 1)
    lon = np.linspace(0.0, 2.0 * np.pi, cols + 1)
    la, lo = np.meshgrid(lat, lon, indexing="ij")
    verts = np.stack([(np.cos(la) * np.cos(lo)).ravel(), (np.sin(la) * 1.15).ravel(),
                      (np.cos(la) * np.sin(lo) * 0.9).ravel()], axis=-1)
    u = (lo / (2.0 * np.pi)).ravel()
    v = ((la - lat[0]) / (lat[-1] - lat[0])).ravel()
    stride = cols + 1
    ii, jj = np.meshgrid(np.arange(rows), np.arange(cols), indexing="ij")
    a = (ii * stride + jj).ravel()
    quads = np.stack([a, a + 1, a + stride + 1, a + stride], axis=-1)    # a, b, d, c
    faces = np.empty((rows * cols * 2, 3), dtype=np.int64)
    faces[0::2] = quads[:, [0, 1, 2]]
    faces[1::2] = quads[:, [0, 2, 3]]
    rng = np.random.default_rng(seed)
    radial = verts / np.linalg.norm(verts, axis=-1, keepdims=True)
    bases = np.empty((num_expressions, verts.shape[0], 3))
    for e in range(num_expressions):
        fu = rng.integers(1, 4)
        fv = rng.integers(1, 4)
        pu = rng.uniform(0.0, 2.0 * np.pi)
        pv = rng.uniform(0.0, np.pi)
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        amp = 0.05 * np.sin(2.0 * np.pi * fu * u + pu) * np.sin(np.pi * fv * v + pv)
        bases[e] = amp[:, None] * (0.6 * radial + 0.4 * d)
    return HeadRig(verts, faces, np.stack([u, v], axis=-1), bases)


def _rodrigues(vec):
    vec = np.asarray(vec, np.float64)
    ang = np.linalg.norm(vec)
    if ang < 1e-12:
        return np.eye(3)
    k = vec / ang
    K = np.array([[0.0, -k[2], k[1]], [k[2], 0.0, -k[0]], [-k[1], k[0], 0.0]])
    return np.eye(3) + np.sin(ang) * K + (1.0 - np.cos(ang)) * (K @ K)


def rig_evaluate(rig: HeadRig, theta) -> np.ndarray:
    """Deformed vertices for theta = (expressions..., axis-angle pose) (S/rig.py:57-66)."""
    theta = np.asarray(theta, np.float64)
    if theta.shape != (rig.param_dim,):
        raise ValueError(f"theta has shape {theta.shape}, rig expects ({rig.param_dim},)")
    e = rig.num_expressions
    verts = rig.base_vertices + np.tensordot(theta[:e], rig.expr_bases, axes=(0, 0))
    return verts @ _rodrigues(theta[e:]).T


# -------------------------------------------------------------- mesh frames


@dataclass
class MeshFrames:
    rotation: np.ndarray       # (F, 3, 3) columns T, B, N
    quat: np.ndarray           # (F, 4) quaternion of the polar rotation (not normalized)
    tri_vertices: np.ndarray   # (F, 3, 3)

    def packed(self) -> np.ndarray:
        """(F, 22) float32 device layout (include/hs_api.h)."""
        f = self.rotation.shape[0]
        return np.concatenate([self.rotation.reshape(f, 9), self.quat.reshape(f, 4),
                               self.tri_vertices.reshape(f, 9)], axis=1).astype(np.float32)


def _tbn(tri, tri_uv):
    e1 = tri[:, 1] - tri[:, 0]
    e2 = tri[:, 2] - tri[:, 0]
    cr = np.cross(e1, e2)
    crn = np.linalg.norm(cr, axis=-1)
    du1 = tri_uv[:, 1, 0] - tri_uv[:, 0, 0]
    du2 = tri_uv[:, 2, 0] - tri_uv[:, 0, 0]
    dv1 = tri_uv[:, 1, 1] - tri_uv[:, 0, 1]
    dv2 = tri_uv[:, 2, 1] - tri_uv[:, 0, 1]
    det = du1 * dv2 - du2 * dv1
    if np.any(np.abs(det) < 1e-12) or np.any(crn < 1e-12):
        raise ValueError("degenerate triangle")
    inv = 1.0 / det
    t = (dv2[:, None] * e1 - dv1[:, None] * e2) * inv[:, None]
    b = (-du2[:, None] * e1 + du1[:, None] * e2) * inv[:, None]
    return np.stack([t, b, cr / crn[:, None]], axis=-1)


def _polar(m):
    u, _, vt = np.linalg.svd(m)
    r = u @ vt
    flip = np.linalg.det(r) < 0
    if np.any(flip):
        u = u.copy()
        u[flip, :, 2] *= -1.0
        r = u @ vt
    return r


def _mat_to_quat(m):
    """Four-branch extraction, unnormalized (S/quatmath.py:105-149)."""
    tr = np.stack([1.0 + m[:, 0, 0] + m[:, 1, 1] + m[:, 2, 2], 1.0 + m[:, 0, 0] - m[:, 1, 1] - m[:, 2, 2],
                   1.0 - m[:, 0, 0] + m[:, 1, 1] - m[:, 2, 2], 1.0 - m[:, 0, 0] - m[:, 1, 1] + m[:, 2, 2]], -1)
    br = np.argmax(tr, axis=-1)
    q = np.empty((m.shape[0], 4))
    # (component order of the 3 off-diagonal terms per branch, with sign pattern)
    for k in range(4):
        sel = br == k
        if not np.any(sel):
            continue
        mm = m[sel]
        s = 2.0 * np.sqrt(np.maximum(tr[sel, k], 1e-30))
        d21, d02, d10 = mm[:, 2, 1] - mm[:, 1, 2], mm[:, 0, 2] - mm[:, 2, 0], mm[:, 1, 0] - mm[:, 0, 1]
        s01, s02, s12 = mm[:, 0, 1] + mm[:, 1, 0], mm[:, 0, 2] + mm[:, 2, 0], mm[:, 1, 2] + mm[:, 2, 1]
        if k == 0:
            cols = (0.25 * s, d21 / s, d02 / s, d10 / s)
        elif k == 1:
            cols = (d21 / s, 0.25 * s, s01 / s, s02 / s)
        elif k == 2:
            cols = (d02 / s, s01 / s, 0.25 * s, s12 / s)
        else:
            cols = (d10 / s, s02 / s, s12 / s, 0.25 * s)
        q[sel] = np.stack(cols, axis=-1)
    return q


def mesh_frames(rig: HeadRig, vertices) -> MeshFrames:
    """Per-face tangent frames of a deformed mesh (S/binding.py:67-77)."""
    tri = vertices[rig.faces]
    rot = _tbn(tri, rig.uv_coords[rig.faces])
    return MeshFrames(rot, _mat_to_quat(_polar(rot)), tri)


# -------------------------------------------------------------- UV binding


def _bary(tri_uv, pts):
    a, b, c = tri_uv
    v0 = b - a
    v1 = c - a
    den = v0[0] * v1[1] - v1[0] * v0[1]
    d = pts - a
    b1 = (d[:, 0] * v1[1] - v1[0] * d[:, 1]) / den
    b2 = (v0[0] * d[:, 1] - d[:, 0] * v0[1]) / den
    return np.stack([1.0 - b1 - b2, b1, b2], axis=-1)


def bind_gaussians(rig: HeadRig, uv_resolution: int):
    """One Gaussian per covered UV texel centre; first covering face wins; output in
    (u index, v index) order (S/binding.py:118-156).  Returns (tri_index, barycentric)."""
    if uv_resolution < 1:
        raise ValueError(f"uv_resolution must be >= 1, got {uv_resolution}")
    res = int(uv_resolution)
    centers = (np.arange(res) + 0.5) / res
    tri_uv = rig.uv_coords[rig.faces]
    owner = np.full((res, res), -1, dtype=np.int64)
    bary = np.zeros((res, res, 3))
    half = 0.5 / res
    for f in range(rig.num_faces):
        uv = tri_uv[f]
        lo, hi = uv.min(axis=0), uv.max(axis=0)
        ui = np.flatnonzero((centers >= lo[0] - half) & (centers <= hi[0] + half))
        vi = np.flatnonzero((centers >= lo[1] - half) & (centers <= hi[1] + half))
        if ui.size == 0 or vi.size == 0:
            continue
        gu, gv = np.meshgrid(ui, vi, indexing="ij")
        pts = np.stack([centers[gu].ravel(), centers[gv].ravel()], axis=-1)
        b = _bary(uv, pts).reshape(gu.shape + (3,))
        take = np.all(b >= -1e-12, axis=-1) & (owner[gu, gv] < 0)
        owner[gu[take], gv[take]] = f
        bary[gu[take], gv[take]] = b[take]
    si, sj = np.nonzero(owner >= 0)          # row-major == lexsort((j, i))
    if si.size == 0:
        raise ValueError("rig UV layout covers no texel at this resolution")
    return owner[si, sj].astype(np.int64), bary[si, sj]


def bindings_checksum(tri_index, barycentric) -> str:
    """S/binding.py:40-44."""
    import hashlib
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(tri_index, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(barycentric, dtype=np.float64).tobytes())
    return h.hexdigest()


# ------------------------------------------------------------------- camera


@dataclass
class Camera:
    fx: float
    fy: float
    cx: float
    cy: float
    rotation: np.ndarray
    translation: np.ndarray
    width: int
    height: int

    @classmethod
    def frontal(cls, image_size, distance=3.2, focal_factor=1.2, yaw=0.0):
        """S/render.py:75-84."""
        c, s = np.cos(yaw), np.sin(yaw)
        orbit = np.array([[c, 0.0, s], [0.0, 1.0, 0.0], [-s, 0.0, c]])
        f = focal_factor * image_size
        return cls(f, f, image_size / 2.0, image_size / 2.0, orbit.T, np.array([0.0, 0.0, distance]),
                   image_size, image_size)

    def packed(self) -> np.ndarray:
        return np.concatenate([np.asarray(self.rotation, np.float64).ravel(), np.asarray(self.translation).ravel(),
                               [self.fx, self.fy, self.cx, self.cy]]).astype(np.float32)


# ------------------------------------------------------------------- avatar


@dataclass
class HostAvatar:
    """Float64 host copy of an avatar in the reference's structure."""
    base: dict                      # position rotation scale opacity color
    deltas: np.ndarray              # (K, 10N) [pos 3N | rot 4N | color 3N]
    mlp: dict                       # w1 b1 w2 b2 w3 b3
    tri_index: np.ndarray
    barycentric: np.ndarray

    @property
    def count(self):
        return self.base["position"].shape[0]

    @property
    def K(self):
        return self.deltas.shape[0]


class _Obj:
    def __init__(self, **kw):
        self.__dict__.update(kw)


def init_avatar(rig: HeadRig, uv_resolution=256, num_blendshapes=20, hidden_dim=128, init_opacity=0.1,
                seed=0) -> HostAvatar:
    """S/train.py:96-120 (MlpWeights.create S/model.py:60-76, then w3 ~ N(0, 0.01))."""
    rng = np.random.default_rng(seed)
    tri_index, bary = bind_gaussians(rig, uv_resolution)
    n = tri_index.shape[0]
    tri = rig.base_vertices[rig.faces]
    area = 0.5 * np.linalg.norm(np.cross(tri[:, 1] - tri[:, 0], tri[:, 2] - tri[:, 0]), axis=-1).sum()
    spacing = np.sqrt(area / n)
    p = np.clip(init_opacity, 1e-4, 1 - 1e-4)
    base = {"position": np.zeros((n, 3)), "rotation": np.tile([1.0, 0.0, 0.0, 0.0], (n, 1)),
            "scale": np.full((n, 3), np.log(0.55 * spacing)), "opacity": np.full(n, np.log(p) - np.log1p(-p)),
            "color": np.zeros((n, 3))}
    h = rig.param_dim
    mlp = {"w1": rng.normal(0.0, np.sqrt(2.0 / h), (hidden_dim, h)), "b1": np.zeros(hidden_dim),
           "w2": rng.normal(0.0, np.sqrt(2.0 / hidden_dim), (hidden_dim, hidden_dim)), "b2": np.zeros(hidden_dim),
           "w3": np.zeros((num_blendshapes, hidden_dim)), "b3": np.zeros(num_blendshapes)}
    mlp["w3"] = rng.normal(0.0, 0.01, size=mlp["w3"].shape)
    return HostAvatar(base, np.zeros((num_blendshapes, 10 * n)), mlp, tri_index, bary)


def perturb(av: HostAvatar, seed=0):
    """deltas pos N(0,0.002), rot N(0,0.02), colour N(0,0.1);
    opacity logit U(-2,2); colour logit N(0,1)."""
    rng = np.random.default_rng(seed)
    n = av.count
    for k in range(av.K):
        av.deltas[k, :3 * n] = rng.normal(0, 0.002, 3 * n)
        av.deltas[k, 3 * n:7 * n] = rng.normal(0, 0.02, 4 * n)
        av.deltas[k, 7 * n:] = rng.normal(0, 0.1, 3 * n)
    av.base["opacity"][:] = rng.uniform(-2, 2, n)
    av.base["color"][:] = rng.normal(0, 1, (n, 3))
    return av


# Config shapes (BASELINE.json configs; SURVEY §2.2 legend).
CONFIGS = {
    "C1": dict(uv=141, batch=4, size=256),
    "C2": dict(uv=224, batch=16, size=512),
    "C3": dict(uv=317, batch=64, size=512),
    "C4": dict(uv=317, batch=128, size=512),
}


@dataclass
class Workload:
    rig: HeadRig
    avatar: HostAvatar
    camera: Camera
    thetas: np.ndarray             # (B, H)
    frames: np.ndarray             # (B, F, 22) float32
    targets: np.ndarray            # (B, S, S, 4) uint8
    backgrounds: np.ndarray        # (B, 3)
    mesh: list = field(default_factory=list)


def make_workload(uv, batch, size, K=20, hidden=128, seed=0, frames_seed=1, distinct_frames=None) -> Workload:
    """Synthetic head-avatar workload of the named shapes."""
    rig = build_head_rig()
    av = perturb(init_avatar(rig, uv, K, hidden, seed=seed), seed=seed + 1)
    rng = np.random.default_rng(frames_seed)
    nd = distinct_frames or batch
    th = rng.normal(0, 0.3, (nd, rig.param_dim))
    mesh = [mesh_frames(rig, rig_evaluate(rig, t)) for t in th]
    idx = np.arange(batch) % nd
    thetas = th[idx]
    frames = np.stack([mesh[i].packed() for i in idx])
    targets = rng.integers(0, 256, size=(batch, size, size, 4), dtype=np.uint8)
    bgs = rng.uniform(0.0, 1.0, size=(batch, 3))
    return Workload(rig, av, Camera.frontal(size), thetas, frames, targets, bgs, [mesh[i] for i in idx])
