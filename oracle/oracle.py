"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the RGBAvatar training hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its cpu_baseline
and ``--impl reference`` legs) may import this module, and only as the checker or
the timed CPU baseline.  The product package ``paper_2503_12886_b200`` never
imports it and has no CPU fallback.

This is a float64 restatement of the reference package ``headsplat``
(``/root/reference/pkg/src/headsplat``, abbreviated ``S/``).  The numeric kernels
live in ``hs_oracle.c`` (built by ``oracle/Makefile``); this module is the numpy
glue with the reference's call signatures and data flow.  Parity of every
function is pinned against vectors produced by running the reference itself
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``, checked by
``tests/test_oracle_golden.py``).

Extensions over the reference (used only to replay another implementation's
decisions, never changing the math):
  * ``rasterize``/``render_backward``/``splat_weight_sums`` accept ``order``
    (the compositing order) and ``bbox`` (the per-splat integer pixel bbox) so a
    checker can feed the device path's fp32 depth order and bbox.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "libhs_oracle.so")
_lib = None
_lock = threading.Lock()

# S/render.py:34-37
NEAR_PLANE = 0.01
MIN_RADIUS = 0.3
ALPHA_CUTOFF = 1.0 / 255.0
TERMINATION_EPS = 1e-14

_D = ctypes.POINTER(ctypes.c_double)
_I64 = ctypes.POINTER(ctypes.c_int64)
_I32 = ctypes.POINTER(ctypes.c_int32)
_U8 = ctypes.POINTER(ctypes.c_uint8)


def build():
    """Compile hs_oracle.c (idempotent)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(_SO):
                build()
            _lib = ctypes.CDLL(_SO)
            _lib.or_activate.restype = ctypes.c_int64
    return _lib


def _p(a, ptr=_D):
    return a.ctypes.data_as(ptr) if a is not None else None


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None and a.shape != shape:
        raise ValueError(f"expected shape {shape}, got {a.shape}")
    return a


# ------------------------------------------------------------------ containers

@dataclass
class GSet:
    """S/gaussians.py:24-69 GaussianSet (also used for GaussianGrad)."""
    position: np.ndarray
    rotation: np.ndarray
    scale: np.ndarray
    opacity: np.ndarray
    color: np.ndarray

    @property
    def count(self):
        return self.position.shape[0]

    def copy(self):
        return GSet(*(getattr(self, n).copy() for n in _ATTRS))

    @classmethod
    def zeros(cls, n):
        return cls(np.zeros((n, 3)), np.zeros((n, 4)), np.zeros((n, 3)), np.zeros(n), np.zeros((n, 3)))


_ATTRS = ("position", "rotation", "scale", "opacity", "color")


@dataclass
class Model:
    """S/model.py:98-127 AvatarModel (deltas as a (K, 10N) array in the
    [pos 3N | rot 4N | color 3N] layout) + S/binding.py:25-44 bindings."""
    base: GSet
    deltas: np.ndarray          # (K, 10N)
    mlp: dict                   # w1 b1 w2 b2 w3 b3
    tri_index: np.ndarray       # (N,) int64
    barycentric: np.ndarray     # (N, 3)

    @property
    def count(self):
        return self.base.count

    @property
    def K(self):
        return self.deltas.shape[0]

    def copy(self):
        return Model(self.base.copy(), self.deltas.copy(), {k: v.copy() for k, v in self.mlp.items()},
                     self.tri_index, self.barycentric)


@dataclass
class Cam:
    """S/render.py:40-84 Camera."""
    fx: float
    fy: float
    cx: float
    cy: float
    rotation: np.ndarray
    translation: np.ndarray
    width: int
    height: int

    def flat(self):
        return np.concatenate([np.asarray(self.rotation, np.float64).ravel(),
                               np.asarray(self.translation, np.float64).ravel(),
                               [self.fx, self.fy, self.cx, self.cy]]).astype(np.float64)

    @classmethod
    def frontal(cls, image_size, distance=3.2, focal_factor=1.2, yaw=0.0):
        c, s = np.cos(yaw), np.sin(yaw)
        orbit = np.array([[c, 0.0, s], [0.0, 1.0, 0.0], [-s, 0.0, c]])
        f = focal_factor * image_size
        return cls(f, f, image_size / 2.0, image_size / 2.0, orbit.T,
                   np.array([0.0, 0.0, distance]), image_size, image_size)


@dataclass
class Frames:
    """S/binding.py:47-53 MeshFrames."""
    rotation: np.ndarray     # (F, 3, 3)
    quat: np.ndarray         # (F, 4)
    tri_vertices: np.ndarray  # (F, 3, 3)


@dataclass
class Splats:
    """S/render.py:87-111 ProjectedSplats."""
    index: np.ndarray
    mean2d: np.ndarray
    conic: np.ndarray
    depth: np.ndarray
    color: np.ndarray
    opacity: np.ndarray
    radius: np.ndarray
    source_count: int
    x_cam: np.ndarray = None
    cov_cam: np.ndarray = None
    world: GSet = None
    camera: Cam = None
    sort_order: np.ndarray = None

    def __len__(self):
        return self.index.shape[0]


@dataclass
class Aux:
    """S/render.py:114-129 RenderAux (+ the bbox used, for replay)."""
    transmittance: np.ndarray
    max_weight: np.ndarray
    splats: Splats
    background: np.ndarray
    stop: np.ndarray
    bbox: np.ndarray = None


# ------------------------------------------------------------------------ MLP

def map_params(mlp, theta):
    """S/model.py:130-142."""
    theta = _f64(theta)
    H = mlp["w1"].shape[1]
    D = mlp["w1"].shape[0]
    K = mlp["w3"].shape[0]
    if theta.shape != (H,):
        raise ValueError(f"theta has shape {theta.shape}, MLP expects ({H},)")
    if not np.all(np.isfinite(theta)):
        raise ValueError("theta contains non-finite values")
    w = {k: _f64(v) for k, v in mlp.items()}
    z1, h1, z2, h2 = (np.empty(D) for _ in range(4))
    psi = np.empty(K)
    lib().or_mlp_fwd(H, D, K, _p(w["w1"]), _p(w["b1"]), _p(w["w2"]), _p(w["b2"]),
                     _p(w["w3"]), _p(w["b3"]), _p(theta), _p(z1), _p(h1), _p(z2), _p(h2), _p(psi))
    return psi, (theta, z1, h1, z2, h2)


def mlp_backward(mlp, cache, grad_psi, into=None):
    """S/model.py:145-162.  Returns dict of weight grads (accumulated into `into`)."""
    theta, z1, h1, z2, h2 = cache
    H = mlp["w1"].shape[1]
    D = mlp["w1"].shape[0]
    K = mlp["w3"].shape[0]
    g = into if into is not None else {k: np.zeros_like(v, dtype=np.float64) for k, v in mlp.items()}
    gpsi = _f64(grad_psi)
    w2 = _f64(mlp["w2"])
    w3 = _f64(mlp["w3"])
    lib().or_mlp_bwd(H, D, K, _p(w2), _p(w3), _p(theta), _p(z1), _p(h1), _p(z2), _p(h2), _p(gpsi),
                     _p(g["w1"]), _p(g["b1"]), _p(g["w2"]), _p(g["b2"]), _p(g["w3"]), _p(g["b3"]))
    return g


# ---------------------------------------------------------------------- blend

def _ten(gs):
    return np.concatenate([gs.position.ravel(), gs.rotation.ravel(), gs.color.ravel()])


def blend(model: Model, psi) -> GSet:
    """S/model.py:165-185."""
    psi = _f64(psi)
    if psi.shape != (model.K,):
        raise ValueError(f"psi has shape {psi.shape}, model has K={model.K}")
    n = model.count
    out = np.empty(10 * n)
    base10 = np.ascontiguousarray(_ten(model.base))
    deltas = _f64(model.deltas)
    lib().or_blend(n, model.K, _p(base10), _p(deltas), _p(psi), _p(out))
    return GSet(out[:3 * n].reshape(n, 3).copy(), out[3 * n:7 * n].reshape(n, 4).copy(),
                model.base.scale.copy(), model.base.opacity.copy(), out[7 * n:].reshape(n, 3).copy())


def blend_backward(model: Model, psi, g_raw: GSet, g_base14=None, g_deltas=None):
    """S/model.py:188-216 with the cross-item sum of S/train.py:253-255 folded in:
    g_base14 (14N, [pos|rot|color|scale|opacity]) and g_deltas (K, 10N) accumulate."""
    n = model.count
    K = model.K
    if g_base14 is None:
        g_base14 = np.zeros(14 * n)
    if g_deltas is None:
        g_deltas = np.zeros((K, 10 * n))
    g14 = np.concatenate([_ten(g_raw), g_raw.scale.ravel(), g_raw.opacity.ravel()])
    g_psi = np.empty(K)
    lib().or_blend_backward(n, K, _p(_f64(model.deltas)), _p(_f64(psi)), _p(g14),
                            _p(g_base14), _p(g_deltas), _p(g_psi))
    return g_base14, g_deltas, g_psi


# ------------------------------------------------------------------- activate

def activate(raw: GSet) -> GSet:
    """S/model.py:219-234."""
    n = raw.count
    out = GSet.zeros(n)
    bad = lib().or_activate(n, _p(_f64(raw.rotation)), _p(_f64(raw.scale)), _p(_f64(raw.opacity)),
                            _p(_f64(raw.color)), _p(out.rotation), _p(out.scale), _p(out.opacity),
                            _p(out.color))
    if bad >= 0:
        raise FloatingPointError(f"zero-norm quaternion at Gaussian index {bad}")
    out.position = raw.position.copy()
    return out


def activate_backward(raw: GSet, act: GSet, g: GSet) -> GSet:
    """S/model.py:237-248."""
    n = raw.count
    out = GSet.zeros(n)
    lib().or_activate_backward(n, _p(_f64(raw.rotation)), _p(_f64(act.rotation)), _p(_f64(act.scale)),
                               _p(_f64(act.opacity)), _p(_f64(act.color)), _p(_f64(g.position)),
                               _p(_f64(g.rotation)), _p(_f64(g.scale)), _p(_f64(g.opacity)),
                               _p(_f64(g.color)), _p(out.position), _p(out.rotation), _p(out.scale),
                               _p(out.opacity), _p(out.color))
    return out


# ------------------------------------------------------------------ transform

def _frames_arrays(frames: Frames):
    return (_f64(frames.rotation).reshape(-1), _f64(frames.quat).reshape(-1),
            _f64(frames.tri_vertices).reshape(-1))


def transform_to_deformed(tangent: GSet, frames: Frames, tri_index, barycentric) -> GSet:
    """S/binding.py:174-188."""
    n = tangent.count
    frot, fq, ftri = _frames_arrays(frames)
    tri = np.ascontiguousarray(tri_index, dtype=np.int64)
    pos = np.empty((n, 3))
    rot = np.empty((n, 4))
    lib().or_transform(n, _p(_f64(tangent.position)), _p(_f64(tangent.rotation)), _p(frot), _p(fq),
                       _p(ftri), _p(tri, _I64), _p(_f64(barycentric)), _p(pos), _p(rot))
    return GSet(pos, rot, tangent.scale.copy(), tangent.opacity.copy(), tangent.color.copy())


def transform_backward(tangent: GSet, frames: Frames, tri_index, g_world: GSet) -> GSet:
    """S/binding.py:191-204."""
    n = tangent.count
    frot, fq, _ = _frames_arrays(frames)
    tri = np.ascontiguousarray(tri_index, dtype=np.int64)
    gp = np.empty((n, 3))
    gr = np.empty((n, 4))
    lib().or_transform_backward(n, _p(_f64(tangent.rotation)), _p(frot), _p(fq), _p(tri, _I64),
                                _p(_f64(g_world.position)), _p(_f64(g_world.rotation)), _p(gp), _p(gr))
    return GSet(gp, gr, g_world.scale.copy(), g_world.opacity.copy(), g_world.color.copy())


# --------------------------------------------------------------------- render

def preprocess(world: GSet, camera: Cam) -> Splats:
    """S/render.py:201-230."""
    for name in _ATTRS:
        arr = getattr(world, name)
        if not np.all(np.isfinite(arr)):
            bad = int(np.flatnonzero(~np.all(np.isfinite(arr.reshape(arr.shape[0], -1)), axis=1))[0])
            raise FloatingPointError(f"non-finite {name} at Gaussian index {bad}")
    n = world.count
    x_cam = np.empty((n, 3))
    cov_cam = np.empty((n, 3, 3))
    mean2d = np.empty((n, 2))
    conic = np.empty((n, 3))
    radius = np.empty(n)
    valid = np.ones(n, dtype=np.uint8)
    cam = camera.flat()
    lib().or_project(n, _p(_f64(world.position)), _p(_f64(world.rotation)), _p(_f64(world.scale)),
                     _p(cam), _p(x_cam), _p(cov_cam), _p(mean2d), _p(conic), _p(radius),
                     _p(valid, _U8))
    idx = np.flatnonzero(valid)
    z = np.ascontiguousarray(x_cam[idx, 2])
    order = stable_argsort(z)
    return Splats(idx, mean2d[idx], conic[idx], z, world.color[idx], world.opacity[idx], radius[idx],
                  n, x_cam[idx], cov_cam[idx], world, camera, order)


def stable_argsort(z):
    z = _f64(z)
    order = np.empty(z.shape[0], dtype=np.int64)
    lib().or_stable_argsort(z.shape[0], _p(z), _p(order, _I64))
    return order


def _sorted(splats: Splats, order, bbox):
    o = order
    sb = None if bbox is None else np.ascontiguousarray(np.asarray(bbox, dtype=np.int32)[o])
    return (_f64(splats.mean2d[o]), _f64(splats.conic[o]), _f64(splats.opacity[o]),
            _f64(splats.color[o]), _f64(splats.radius[o]), sb)


def rasterize(splats: Splats, camera: Cam, background, order=None, bbox=None):
    """S/render.py:389-407.  `order`/`bbox` replay another implementation's
    compositing order / integer pixel bbox (defaults: the reference's own)."""
    background = _f64(background)
    h, w = camera.height, camera.width
    m = len(splats)
    order = splats.sort_order if order is None else np.asarray(order, dtype=np.int64)
    image = np.zeros((h, w, 3))
    trans = np.ones((h, w))
    stop = np.full((h, w), m, dtype=np.int64)
    maxw_sorted = np.zeros(m)
    if m:
        mean, con, op, col, rad, sb = _sorted(splats, order, bbox)
        lib().or_composite(m, _p(mean), _p(con), _p(op), _p(col), _p(rad), _p(sb, _I32), h, w,
                           _p(image), _p(trans), _p(stop, _I64), _p(maxw_sorted))
    image += trans[:, :, None] * background[None, None, :]
    max_weight = np.zeros(splats.source_count)
    if m:
        max_weight[splats.index[order]] = maxw_sorted
    aux = Aux(trans, max_weight, splats, background, stop, bbox)
    aux.order = order
    return image, aux


def flip_mask(splats: Splats, camera: Cam, order=None, bbox=None, out=None):
    """Checker extension (hs_oracle.c:or_flip_mask): (h, w) bool, the pixels where an
    alpha-cutoff / ellipse-cutoff / alpha->1 / termination decision of the reference's
    compositing (S/render.py:233-273) is within fp32 noise of its threshold.  ``out``
    (h, w) uint8 accumulates across calls."""
    h, w = camera.height, camera.width
    mask = np.zeros((h, w), np.uint8) if out is None else out
    m = len(splats)
    if m:
        order = splats.sort_order if order is None else np.asarray(order, dtype=np.int64)
        mean, con, op, _, rad, sb = _sorted(splats, order, bbox)
        lib().or_flip_mask(m, _p(mean), _p(con), _p(op), _p(rad), _p(sb, _I32), h, w, _p(mask, _U8))
    return mask.astype(bool) if out is None else mask


def render_backward(splats: Splats, aux: Aux, grad_image) -> GSet:
    """S/render.py:410-429 (+ _preprocess_backward :432-497)."""
    grad_image = _f64(grad_image)
    camera = splats.camera
    h, w = camera.height, camera.width
    m = len(splats)
    order = getattr(aux, "order", splats.sort_order)
    gs_mean = np.zeros((m, 2))
    gs_conic = np.zeros((m, 3))
    gs_op = np.zeros(m)
    gs_col = np.zeros((m, 3))
    if m:
        mean, con, op, col, rad, sb = _sorted(splats, order, aux.bbox)
        lib().or_composite_backward(m, _p(mean), _p(con), _p(op), _p(col), _p(rad), _p(sb, _I32), h, w,
                                    _p(_f64(aux.transmittance)), _p(np.ascontiguousarray(aux.stop, np.int64), _I64),
                                    _p(grad_image), _p(_f64(aux.background)), _p(gs_mean), _p(gs_conic),
                                    _p(gs_op), _p(gs_col))
    g_mean = np.zeros((m, 2)); g_mean[order] = gs_mean
    g_conic = np.zeros((m, 3)); g_conic[order] = gs_conic
    g_op = np.zeros(m); g_op[order] = gs_op
    g_col = np.zeros((m, 3)); g_col[order] = gs_col
    return preprocess_backward(splats, g_mean, g_conic, g_op, g_col)


def splat_space_grads(splats: Splats, aux: Aux, grad_image):
    """The raster adjoint alone (S/render.py:276-336), in kept-splat order:
    returns (g_mean (M,2), g_conic (M,3), g_opacity (M,), g_color (M,3))."""
    grad_image = _f64(grad_image)
    camera = splats.camera
    m = len(splats)
    order = getattr(aux, "order", splats.sort_order)
    gs = [np.zeros((m, 2)), np.zeros((m, 3)), np.zeros(m), np.zeros((m, 3))]
    if m:
        mean, con, op, col, rad, sb = _sorted(splats, order, aux.bbox)
        lib().or_composite_backward(m, _p(mean), _p(con), _p(op), _p(col), _p(rad), _p(sb, _I32),
                                    camera.height, camera.width, _p(_f64(aux.transmittance)),
                                    _p(np.ascontiguousarray(aux.stop, np.int64), _I64), _p(grad_image),
                                    _p(_f64(aux.background)), *(_p(g) for g in gs))
    out = []
    for g in gs:
        o = np.zeros_like(g)
        o[order] = g
        out.append(o)
    return tuple(out)


def preprocess_backward(splats: Splats, g_mean, g_conic, g_opacity, g_color) -> GSet:
    """S/render.py:432-497."""
    world = splats.world
    grad = GSet.zeros(world.count)
    m = len(splats)
    if m == 0:
        return grad
    lib().or_preprocess_backward(m, _p(np.ascontiguousarray(splats.index, np.int64), _I64),
                                 _p(_f64(splats.x_cam)), _p(_f64(splats.cov_cam)), _p(_f64(splats.conic)),
                                 _p(_f64(world.rotation)), _p(_f64(world.scale)), _p(splats.camera.flat()),
                                 _p(_f64(g_mean)), _p(_f64(g_conic)), _p(_f64(g_opacity)), _p(_f64(g_color)),
                                 _p(grad.position), _p(grad.rotation), _p(grad.scale), _p(grad.opacity),
                                 _p(grad.color))
    return grad


def splat_weight_sums(aux: Aux, image):
    """S/render.py:500-521."""
    image = _f64(image)
    splats = aux.splats
    camera = splats.camera
    m = len(splats)
    order = getattr(aux, "order", splats.sort_order)
    num_s = np.zeros((m, 3))
    den_s = np.zeros(m)
    if m:
        mean, con, op, _, rad, sb = _sorted(splats, order, aux.bbox)
        lib().or_weight_sums(m, _p(mean), _p(con), _p(op), _p(rad), _p(sb, _I32), camera.height,
                             camera.width, _p(image), _p(num_s), _p(den_s))
    num = np.zeros((splats.source_count, 3))
    den = np.zeros(splats.source_count)
    if m:
        src = splats.index[order]
        num[src] = num_s
        den[src] = den_s
    return num, den


# ---------------------------------------------------------------- metrics/colour

def composite_over(rgba, background):
    """S/metrics.py:80-85."""
    rgba = _f64(rgba)
    bg = _f64(background)
    alpha = rgba[:, :, 3:4]
    return rgba[:, :, :3] * alpha + (1.0 - alpha) * bg[None, None, :]


def l1_loss(pred, target):
    """S/metrics.py:10-22."""
    diff = _f64(pred) - _f64(target)
    return float(np.mean(np.abs(diff))), np.sign(diff) / diff.size


def logit(p, eps=1e-4):
    """S/model.py:260-263."""
    p = np.clip(_f64(p), eps, 1.0 - eps)
    return np.log(p) - np.log1p(-p)


def estimate_colors(aux: Aux, target, threshold=0.1):
    """S/color_init.py:45-65."""
    target = _f64(target)
    cam = aux.splats.camera
    if target.shape != (cam.height, cam.width, 3):
        raise ValueError(f"target shape {target.shape} does not match the render "
                         f"({cam.height}, {cam.width}, 3)")
    num, den = splat_weight_sums(aux, target)
    eligible = aux.max_weight > threshold
    bad = eligible & (den <= 0.0)
    if np.any(bad):
        raise RuntimeError(f"Gaussian {int(np.flatnonzero(bad)[0])} exceeds the weight threshold "
                           "but accumulated zero total weight")
    safe = np.where(den > 0.0, den, 1.0)
    return num / safe[:, None], eligible


def apply_color_init(model: Model, estimates, eligible, visited):
    """S/color_init.py:68-80 (visited is the ColorInitState.visited array)."""
    fresh = eligible & ~visited
    if not np.any(fresh):
        return 0
    model.base.color[fresh] = logit(estimates[fresh])
    visited[fresh] = True
    return int(fresh.sum())


# ----------------------------------------------------------------------- Adam

ADAM_BETA1, ADAM_BETA2, ADAM_EPS = 0.9, 0.999, 1e-8   # S/optim.py:19-21


class Adam:
    """S/optim.py:14-40 + the per-attribute groups of S/train.py:164-199.
    All groups step together, so one step counter serves them all."""

    def __init__(self, model: Model, lrs: dict):
        self.lrs = lrs
        self.step_count = 0
        self.m = {}
        self.v = {}
        for name in _ATTRS:
            a = getattr(model.base, name)
            self.m["base." + name] = np.zeros(a.size)
            self.v["base." + name] = np.zeros(a.size)
        self.m["deltas"] = np.zeros(model.deltas.size)
        self.v["deltas"] = np.zeros(model.deltas.size)
        for k, w in model.mlp.items():
            self.m["mlp." + k] = np.zeros(w.size)
            self.v["mlp." + k] = np.zeros(w.size)

    def _one(self, key, param, grad, lr):
        flat = param.reshape(-1)   # a view: params are contiguous float64
        lib().or_adam(flat.size, _p(flat), _p(_f64(grad).reshape(-1)), _p(self.m[key]), _p(self.v[key]),
                      self.step_count, ctypes.c_double(lr), ctypes.c_double(ADAM_BETA1),
                      ctypes.c_double(ADAM_BETA2), ctypes.c_double(ADAM_EPS))

    def step(self, model: Model, g_base: GSet, g_deltas, g_mlp):
        self.step_count += 1
        lr = self.lrs
        for name in _ATTRS:
            self._one("base." + name, getattr(model.base, name), getattr(g_base, name), lr["base." + name])
        n = model.count
        K = model.K
        # delta groups: per k, per attribute (lr scaled, S/train.py:63-68, :193-196)
        gd = _f64(g_deltas).reshape(K, 10 * n)
        md = self.m["deltas"].reshape(K, 10 * n)
        vd = self.v["deltas"].reshape(K, 10 * n)
        for k in range(K):
            for lo, hi, key in ((0, 3 * n, "delta.position"), (3 * n, 7 * n, "delta.rotation"),
                                (7 * n, 10 * n, "delta.color")):
                p = model.deltas[k, lo:hi]
                mm = np.ascontiguousarray(md[k, lo:hi])
                vv = np.ascontiguousarray(vd[k, lo:hi])
                pp = np.ascontiguousarray(p)
                lib().or_adam(pp.size, _p(pp), _p(np.ascontiguousarray(gd[k, lo:hi])), _p(mm), _p(vv),
                              self.step_count, ctypes.c_double(lr[key]), ctypes.c_double(ADAM_BETA1),
                              ctypes.c_double(ADAM_BETA2), ctypes.c_double(ADAM_EPS))
                model.deltas[k, lo:hi] = pp
                md[k, lo:hi] = mm
                vd[k, lo:hi] = vv
        for name, w in model.mlp.items():
            self._one("mlp." + name, w, g_mlp[name], lr["mlp"])


def default_lrs(lr_position=0.0008, lr_opacity=0.25, lr_scale=0.025, lr_rotation=0.005,
                lr_color=0.0125, delta_position_scale=0.05, delta_rotation_scale=0.5,
                delta_color_scale=0.5, lr_mlp=0.001):
    """S/train.py:43-51, :63-68."""
    return {
        "base.position": lr_position, "base.rotation": lr_rotation, "base.scale": lr_scale,
        "base.opacity": lr_opacity, "base.color": lr_color,
        "delta.position": lr_position * delta_position_scale,
        "delta.rotation": lr_rotation * delta_rotation_scale,
        "delta.color": lr_color * delta_color_scale,
        "mlp": lr_mlp,
    }


# ----------------------------------------------------------------- train step

@dataclass
class FrameCtx:
    psi: np.ndarray
    cache: tuple
    raw: GSet
    act: GSet
    frames: Frames
    splats: Splats = None
    aux: Aux = None


def frame_forward(model: Model, theta, frames: Frames):
    """S/train.py:135-149 (use_mlp=True)."""
    psi, cache = map_params(model.mlp, theta)
    raw = blend(model, psi)
    act = activate(raw)
    world = transform_to_deformed(act, frames, model.tri_index, model.barycentric)
    return world, FrameCtx(psi, cache, raw, act, frames)


def frame_backward(model: Model, ctx: FrameCtx, grad_image):
    """S/train.py:152-161: the full per-item adjoint chain (runs on a worker thread,
    like the reference's map_items).  Returns (g_base14, g_deltas, g_mlp) of this item."""
    g_world = render_backward(ctx.splats, ctx.aux, grad_image)
    g_act = transform_backward(ctx.act, ctx.frames, model.tri_index, g_world)
    g_raw = activate_backward(ctx.raw, ctx.act, g_act)
    g_base14, g_deltas, g_psi = blend_backward(model, ctx.psi, g_raw)
    g_mlp = mlp_backward(model.mlp, ctx.cache, g_psi)
    return g_base14, g_deltas, g_mlp


class State:
    """S/train.py:202-211 TrainState (+ S/color_init.py:19-30 ColorInitState)."""

    def __init__(self, model: Model, camera: Cam, lrs=None, color_init=True, threshold=0.1, workers=1):
        self.model = model
        self.camera = camera
        self.adam = Adam(model, lrs or default_lrs())
        self.visited = np.zeros(model.count, dtype=bool)
        self.threshold = threshold
        self.color_init = color_init
        self.workers = max(1, int(workers))
        self.pool = ThreadPoolExecutor(self.workers) if self.workers > 1 else None
        self.last_grads = None

    def map(self, fn, items):
        if self.pool is None:
            return [fn(*a) for a in items]
        return [f.result() for f in [self.pool.submit(fn, *a) for a in items]]

    def close(self):
        if self.pool is not None:
            self.pool.shutdown()


def train_step(state: State, thetas, images, frames_list, backgrounds, replay=None, global_batch=None,
               reduce_fn=None):
    """S/train.py:214-260.  images: (B, H, W, 4) straight RGBA in [0, 1].
    Returns (mean loss, black-bg L1 per item).  The summed gradients passed to
    Adam are kept on state.last_grads (g_base14, g_deltas, g_mlp).

    ``global_batch`` / ``reduce_fn`` (checker extensions for the data-parallel
    split): image gradients are scaled by 1/global_batch and the summed
    gradients pass through ``reduce_fn`` (e.g. a gloo allreduce) before Adam.

    ``replay`` (checker extension): per frame a dict with ``order``
    (compositing order over the kept splats) and ``bbox`` (int pixel bbox per kept
    splat) taken from the implementation under test, so the fp32-vs-fp64 decision
    boundaries (depth ties, the 3-sigma bbox edge) are identical on both sides.
    Optional per-frame ``signs`` ((H, W, 3) in {-1, 0, 1}: the implementation's L1
    sign per pixel channel, replacing the oracle's) and ``gmask`` ((H, W) bool:
    pixels whose image gradient is zeroed on both sides, see ``flip_mask``)."""
    model = state.model
    cam = state.camera
    B = len(thetas)
    ctxs = []
    worlds = []
    for b in range(B):
        world, ctx = frame_forward(model, thetas[b], frames_list[b])
        ctxs.append(ctx)
        worlds.append(world)
    # two-stage schedule (S/scheduler.py:64-72): all preprocess, one barrier, all raster
    splats = state.map(lambda w: preprocess(w, cam), [(w,) for w in worlds])
    if replay is None:
        rendered = state.map(lambda s, bg: rasterize(s, cam, bg), list(zip(splats, backgrounds)))
    else:
        for s, r in zip(splats, replay):
            if not np.array_equal(s.index, r["index"]):
                raise ValueError("replay: kept-splat sets differ (a near-plane / min-radius cull flipped)")
        rendered = state.map(lambda s, bg, r: rasterize(s, cam, bg, order=r["order"], bbox=r["bbox"]),
                             list(zip(splats, backgrounds, replay)))
    losses = np.empty(B)
    black = np.empty(B)
    grads_img = []
    for b, (image, aux) in enumerate(rendered):
        ctxs[b].splats = aux.splats
        ctxs[b].aux = aux
        target = composite_over(images[b], backgrounds[b])
        loss, gimg = l1_loss(image, target)
        if replay is not None and replay[b].get("signs") is not None:
            # the implementation's own L1 sign per pixel channel (a decision like the
            # depth order: fp32 and fp64 differ where |pred - target| ~ 1e-7)
            gimg = np.asarray(replay[b]["signs"], np.float64) / image.size
        if replay is not None and replay[b].get("gmask") is not None:
            gimg = gimg * ~np.asarray(replay[b]["gmask"], bool)[:, :, None]
        losses[b] = loss
        grads_img.append(gimg / (global_batch or B))
        bp = image - aux.transmittance[:, :, None] * _f64(backgrounds[b])[None, None, :]
        bt = _f64(images[b])[:, :, :3] * _f64(images[b])[:, :, 3:4]
        black[b] = float(np.mean(np.abs(bp - bt)))
    per_item = state.map(lambda c, g: frame_backward(model, c, g), list(zip(ctxs, grads_img)))
    state.last_items = (ctxs, grads_img, per_item)      # checker: per-frame stages
    # ParamGradients reduction in item order (S/train.py:253-255)
    n = model.count
    g_base14 = np.zeros(14 * n)
    g_deltas = np.zeros((model.K, 10 * n))
    g_mlp = {k: np.zeros_like(v, dtype=np.float64) for k, v in model.mlp.items()}
    for gb, gd, gm in per_item:
        g_base14 += gb
        g_deltas += gd
        for k in g_mlp:
            g_mlp[k] += gm[k]
    if reduce_fn is not None:          # cross-rank sum (multi-process checker)
        g_base14, g_deltas, g_mlp = reduce_fn(g_base14, g_deltas, g_mlp)
    g_base = GSet(g_base14[:3 * n].reshape(n, 3), g_base14[3 * n:7 * n].reshape(n, 4),
                  g_base14[10 * n:13 * n].reshape(n, 3), g_base14[13 * n:], g_base14[7 * n:10 * n].reshape(n, 3))
    state.last_grads = (g_base.copy(), g_deltas.copy(), {k: v.copy() for k, v in g_mlp.items()})
    state.adam.step(model, g_base, g_deltas, g_mlp)
    if state.color_init and not state.visited.all():
        _attempt_color_init(state, images, rendered, backgrounds)
    return float(losses.mean()), black


def _attempt_color_init(state: State, images, rendered, backgrounds):
    """S/train.py:263-278."""
    stack = np.stack([aux.max_weight for (_, aux) in rendered], axis=0)
    best_item = np.argmax(stack, axis=0)
    best_weight = stack[best_item, np.arange(stack.shape[1])]
    need = (~state.visited) & (best_weight > state.threshold)
    if not np.any(need):
        return
    for i, ((image, aux), bg) in enumerate(zip(rendered, backgrounds)):
        mask = need & (best_item == i)
        if not np.any(mask):
            continue
        target = composite_over(images[i], bg)
        est, eligible = estimate_colors(aux, target, state.threshold)
        apply_color_init(state.model, est, eligible & mask, state.visited)
