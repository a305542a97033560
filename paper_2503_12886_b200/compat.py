"""Drop-in replacements for the reference's hot-path Python API (numpy in / numpy out).

Same names, argument meaning and exceptions as ``headsplat``; the
work runs in the sm_100a kernels of libhs_b200.so (fp32).  Inputs are duck typed,
so the reference's own GaussianSet / Camera / MeshFrames / AvatarModel objects
can be passed directly; outputs are small dataclasses with the reference's field
names.

  map_params / mlp_backward         S/model.py:130, :145
  blend / blend_backward            S/model.py:165, :188
  activate / activate_backward      S/model.py:219, :237
  transform_to_deformed / _backward S/binding.py:174, :191
  preprocess                        S/render.py:201
  rasterize                         S/render.py:389
  render_backward                   S/render.py:410
  splat_weight_sums                 S/render.py:500
  estimate_colors / apply_color_init S/color_init.py:45, :68
  BatchRenderer / render_batch      S/scheduler.py:26-88
  train_step                        S/train.py:214
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from .device import (AvatarParams, Binner, Trainer, _p, _stream, camera_array, frames_array, key_layout,
                     lrs_from_config, require_cuda, split_flat)

ATTRS = ("position", "rotation", "scale", "opacity", "color")
ALPHA_CUTOFF = 1.0 / 255.0


# ------------------------------------------------------------------ containers

@dataclass
class GaussianSet:
    position: np.ndarray
    rotation: np.ndarray
    scale: np.ndarray
    opacity: np.ndarray
    color: np.ndarray

    @property
    def count(self):
        return self.position.shape[0]


GaussianGrad = GaussianSet


@dataclass
class DeltaSet:
    position: np.ndarray
    rotation: np.ndarray
    color: np.ndarray


@dataclass
class MlpGrad:
    w1: np.ndarray
    b1: np.ndarray
    w2: np.ndarray
    b2: np.ndarray
    w3: np.ndarray
    b3: np.ndarray


@dataclass
class ProjectedSplats:
    """S/render.py:87-111 (device handles of the fp32 projection kept in ``_dev``)."""
    index: np.ndarray
    mean2d: np.ndarray
    conic: np.ndarray
    depth: np.ndarray
    color: np.ndarray
    opacity: np.ndarray
    radius: np.ndarray
    source_count: int
    x_cam: np.ndarray = field(repr=False, default=None)
    cov_cam: np.ndarray = field(repr=False, default=None)
    world: object = field(repr=False, default=None)
    camera: object = field(repr=False, default=None)
    sort_order: np.ndarray = field(repr=False, default=None)
    _dev: dict = field(repr=False, default=None)

    def __len__(self):
        return self.index.shape[0]


@dataclass
class RenderAux:
    """S/render.py:114-129."""
    transmittance: np.ndarray
    max_weight: np.ndarray
    splats: ProjectedSplats
    background: np.ndarray
    stop: np.ndarray = None
    _dev: dict = field(repr=False, default=None)


def _dev():
    require_cuda()
    return torch.device("cuda")


def _t(a, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(a)).to(device=_dev(), dtype=dtype)


_KEPT = []


def _keep(t):
    """Pointer to a temporary device tensor that stays referenced past the launch
    (otherwise the caching allocator could hand its block to the next temporary of
    the same argument list and the two pointers would alias)."""
    _KEPT.append(t)
    if len(_KEPT) > 64:
        del _KEPT[:-32]
    return _p(t)


def _pack14(g) -> np.ndarray:
    return np.concatenate([np.asarray(g.position, np.float64).ravel(), np.asarray(g.rotation, np.float64).ravel(),
                           np.asarray(g.color, np.float64).ravel(), np.asarray(g.scale, np.float64).ravel(),
                           np.asarray(g.opacity, np.float64).ravel()])


def _unpack14(flat, n) -> GaussianSet:
    f = np.asarray(flat, np.float64)
    return GaussianSet(f[:3 * n].reshape(n, 3).copy(), f[3 * n:7 * n].reshape(n, 4).copy(),
                       f[10 * n:13 * n].reshape(n, 3).copy(), f[13 * n:14 * n].copy(), f[7 * n:10 * n].reshape(n, 3).copy())


def _err():
    return torch.full((1,), -1, dtype=torch.int64, device=_dev())


def _raise(err):
    L.raise_device_error(int(err.item()) & 0xFFFFFFFFFFFFFFFF)


# ------------------------------------------------------------------------ MLP

def _mlp_flat(mlp):
    return np.concatenate([np.asarray(getattr(mlp, k), np.float64).ravel() for k in ("w1", "b1", "w2", "b2", "w3", "b3")])


def map_params(mlp, theta):
    """S/model.py:130-142.  Returns (psi, cache)."""
    theta = np.asarray(theta, np.float64)
    H, D, K = mlp.w1.shape[1], mlp.w1.shape[0], mlp.w3.shape[0]
    if theta.shape != (H,):
        raise ValueError(f"theta has shape {theta.shape}, MLP expects ({H},)")
    w = _t(_mlp_flat(mlp))
    th = _t(theta)
    cache = torch.empty(4 * D, dtype=torch.float32, device=_dev())
    psi = torch.empty(K, dtype=torch.float32, device=_dev())
    err = _err()
    L.call("hs_mlp_fwd", 1, H, D, K, _p(w), _p(th), _p(cache), _p(psi), _p(err), _stream())
    _raise(err)
    c = cache.cpu().numpy().astype(np.float64)
    return psi.cpu().numpy().astype(np.float64), (theta, c[:D], c[D:2 * D], c[2 * D:3 * D], c[3 * D:])


def mlp_backward(mlp, cache, grad_psi):
    """S/model.py:145-162.  Returns (MlpGrad, grad_theta)."""
    theta, z1, h1, z2, h2 = cache
    H, D, K = mlp.w1.shape[1], mlp.w1.shape[0], mlp.w3.shape[0]
    grad_psi = np.asarray(grad_psi, np.float64)
    if grad_psi.shape != (K,):
        raise ValueError("grad_psi shape mismatch")
    w = _t(_mlp_flat(mlp))
    c = _t(np.concatenate([z1, h1, z2, h2]))
    parts = _t(grad_psi.reshape(K, 1))          # one partial per basis
    gpsi = torch.empty(K, dtype=torch.float32, device=_dev())
    scratch = torch.empty(K + 2 * D + 16, dtype=torch.float32, device=_dev())
    g = torch.empty(int(L.load().hs_mlp_size(H, D, K)), dtype=torch.float32, device=_dev())
    L.call("hs_mlp_bwd", 1, H, D, K, _p(w), _keep(_t(theta)), _p(c), _p(parts), 1, _p(gpsi), _p(scratch), _p(g), _stream())
    gz1 = scratch[D:2 * D].cpu().numpy().astype(np.float64)
    flat = g.cpu().numpy().astype(np.float64)
    o = 0
    out = {}
    for k, shape in (("w1", (D, H)), ("b1", (D,)), ("w2", (D, D)), ("b2", (D,)), ("w3", (K, D)), ("b3", (K,))):
        sz = int(np.prod(shape))
        out[k] = flat[o:o + sz].reshape(shape)
        o += sz
    grad_theta = np.asarray(mlp.w1, np.float64).T @ gz1
    return MlpGrad(**out), grad_theta


# ---------------------------------------------------------------------- blend

def _deltas10(model):
    return np.stack([np.concatenate([np.asarray(d.position, np.float64).ravel(), np.asarray(d.rotation, np.float64).ravel(),
                                     np.asarray(d.color, np.float64).ravel()]) for d in model.deltas])


def blend(model, psi) -> GaussianSet:
    """S/model.py:165-185."""
    psi = np.asarray(psi, np.float64)
    K = len(model.deltas)
    if psi.shape != (K,):
        raise ValueError(f"psi has shape {psi.shape}, model has K={K}")
    n = model.base.position.shape[0]
    base14 = _t(_pack14(model.base))
    raw = torch.empty(10 * n, dtype=torch.float32, device=_dev())
    L.call("hs_blend_fwd", n, K, 1, _p(base14), _keep(_t(_deltas10(model))), _keep(_t(psi)), _p(raw), _stream())
    r = raw.cpu().numpy().astype(np.float64)
    return GaussianSet(r[:3 * n].reshape(n, 3), r[3 * n:7 * n].reshape(n, 4),
                       np.asarray(model.base.scale, np.float64).copy(), np.asarray(model.base.opacity, np.float64).copy(),
                       r[7 * n:].reshape(n, 3))


def blend_backward(model, psi, grad_out):
    """S/model.py:188-216.  Returns (grad_base, list[DeltaSet], grad_psi)."""
    psi = np.asarray(psi, np.float64)
    K = len(model.deltas)
    if psi.shape != (K,):
        raise ValueError("psi shape mismatch")
    n = model.base.position.shape[0]
    g14 = _t(_pack14(grad_out))
    gb = torch.empty(14 * n, dtype=torch.float32, device=_dev())
    gd = torch.empty(K * 10 * n, dtype=torch.float32, device=_dev())
    parts = torch.empty(K * int(L.load().hs_blend_bwd_partials(n)), dtype=torch.float32, device=_dev())
    np_ = ctypes.c_int(0)
    L.call("hs_blend_bwd", n, K, 1, _keep(_t(_deltas10(model))), _keep(_t(psi)), _p(g14), _p(gb), _p(gd), _p(parts),
           ctypes.byref(np_), _stream())
    g_psi = parts.view(K, np_.value).sum(dim=1).double().cpu().numpy()
    gdn = gd.cpu().numpy().astype(np.float64).reshape(K, 10 * n)
    deltas = [DeltaSet(x[:3 * n].reshape(n, 3), x[3 * n:7 * n].reshape(n, 4), x[7 * n:].reshape(n, 3)) for x in gdn]
    return _unpack14(gb.cpu().numpy(), n), deltas, g_psi


# ------------------------------------------------------------------- activate

def activate(raw) -> GaussianSet:
    """S/model.py:219-234."""
    n = raw.position.shape[0]
    out = torch.empty(14 * n, dtype=torch.float32, device=_dev())
    err = _err()
    L.call("hs_activate_fwd", n, _keep(_t(_pack14(raw))), _p(out), _p(err), _stream())
    _raise(err)
    return _unpack14(out.cpu().numpy(), n)


def activate_backward(raw, activated, grad_out) -> GaussianSet:
    """S/model.py:237-248."""
    n = raw.position.shape[0]
    out = torch.empty(14 * n, dtype=torch.float32, device=_dev())
    L.call("hs_activate_bwd", n, _keep(_t(_pack14(raw))), _keep(_t(_pack14(activated))), _keep(_t(_pack14(grad_out))),
           _p(out), _stream())
    return _unpack14(out.cpu().numpy(), n)


def transform_to_deformed(tangent, frames, bindings) -> GaussianSet:
    """S/binding.py:174-188."""
    n = tangent.position.shape[0]
    out = torch.empty(14 * n, dtype=torch.float32, device=_dev())
    L.call("hs_transform_fwd", n, _keep(_t(_pack14(tangent))), _keep(_t(frames_array(frames))),
           _keep(_t(bindings.triangle_index, torch.int32)), _keep(_t(bindings.barycentric)), _p(out), _stream())
    return _unpack14(out.cpu().numpy(), n)


def transform_backward(tangent, frames, bindings, grad_world) -> GaussianSet:
    """S/binding.py:191-204."""
    n = tangent.position.shape[0]
    out = torch.empty(14 * n, dtype=torch.float32, device=_dev())
    L.call("hs_transform_bwd", n, _keep(_t(_pack14(tangent))), _keep(_t(frames_array(frames))),
           _keep(_t(bindings.triangle_index, torch.int32)), _keep(_t(_pack14(grad_world))), _p(out), _stream())
    return _unpack14(out.cpu().numpy(), n)


# --------------------------------------------------------------------- render

@dataclass
class MeshFrames:
    """S/binding.py:47-53."""
    rotation: np.ndarray       # (F, 3, 3), columns T, B, N
    quat: np.ndarray           # (F, 4)
    tri_vertices: np.ndarray   # (F, 3, 3)


_RIGS = {}


def _device_rig(rig):
    from .device import DeviceRig
    key = id(rig)
    hit = _RIGS.get(key)
    if hit is None or hit[0] is not rig:
        hit = _RIGS[key] = (rig, DeviceRig(rig, _dev()))
    return hit[1]


def mesh_frames(rig, vertices) -> MeshFrames:
    """S/binding.py:67-78 on the device (hs_rig_frames; fp64 TBN / polar / quaternion,
    returned through fp32).  Raises the reference's DegenerateTriangleError
    (a ValueError) naming the first bad face."""
    v = torch.from_numpy(np.ascontiguousarray(vertices, np.float64)[None]).to(_dev())
    out = _device_rig(rig).frames(vertices=v)[0].cpu().numpy().astype(np.float64)
    F = out.shape[0]
    return MeshFrames(out[:, :9].reshape(F, 3, 3), out[:, 9:13].copy(), out[:, 13:].reshape(F, 3, 3))


def rig_mesh_frames(rig, theta) -> MeshFrames:
    """mesh_frames(rig, rig_evaluate(rig, theta)) in one device call (S/rig.py:57-66 +
    S/binding.py:67-78); theta is taken in fp32."""
    theta = np.asarray(theta, np.float64)
    if theta.shape != (rig.num_expressions + 3,) and theta.shape != (getattr(rig, "param_dim", -1),):
        raise ValueError(f"theta has shape {theta.shape}, rig expects ({rig.num_expressions + 3},)")
    t = torch.from_numpy(theta.astype(np.float32)[None]).to(_dev())
    out = _device_rig(rig).frames(t)[0].cpu().numpy().astype(np.float64)
    F = out.shape[0]
    return MeshFrames(out[:, :9].reshape(F, 3, 3), out[:, 9:13].copy(), out[:, 13:].reshape(F, 3, 3))


def _check_camera(camera):
    if camera.fx <= 0 or camera.fy <= 0:
        raise ValueError("focal lengths must be positive")
    r = np.asarray(camera.rotation, np.float64)
    if np.max(np.abs(r @ r.T - np.eye(3))) > 1e-9:
        raise ValueError("camera rotation is not orthonormal")


def _project_batch(worlds, cameras):
    """One launch over all items (same N and image size)."""
    B = len(worlds)
    n = worlds[0].position.shape[0]
    W, H = int(cameras[0].width), int(cameras[0].height)
    d = _dev()
    w14 = _t(np.concatenate([_pack14(w) for w in worlds]))
    cams = _t(np.stack([camera_array(c) for c in cameras]))
    f32 = dict(dtype=torch.float32, device=d)
    dev = {"B": B, "N": n, "W": W, "H": H, "world14": w14, "cams": cams,
           "records": torch.empty(B * n * 12, **f32), "depth": torch.empty(B * n, **f32),
           "counts": torch.empty(B * n, dtype=torch.int32, device=d), "radius": torch.empty(B * n, **f32),
           "x_cam": torch.empty(B * n * 3, **f32), "cov_cam": torch.empty(B * n * 9, **f32)}
    nb = int(L.load().hs_scan_blocks(B * n))
    dev["block_sums"] = torch.empty(nb, dtype=torch.int32, device=d)
    err = _err()
    binner = Binner(d)
    L.call("hs_project_world_fwd", B, n, W, H, _p(w14), _p(cams), _p(dev["records"]), _p(dev["depth"]),
           _p(dev["counts"]), _p(dev["block_sums"]), _p(binner.reset_depth_range()), _p(dev["radius"]),
           _p(dev["x_cam"]), _p(dev["cov_cam"]), _p(err), _stream())
    total, code = binner.scan(dev["block_sums"], nb, err)
    L.raise_device_error(code)
    dev["binned"] = binner.bin(B, n, W, H, dev["records"], dev["depth"], dev["counts"], total)
    dev["binner"] = binner
    dev["total"] = total
    # the persistent raster's workspace for this batch (counters zeroed once)
    dev["raster_ws"] = torch.zeros(int(L.load().hs_raster_workspace_size(B, W, H)), dtype=torch.uint8, device=d)
    return dev


def _splats_from(dev, b, world, camera):
    n = dev["N"]
    sl = slice(b * n, (b + 1) * n)
    rec = dev["records"].view(-1, 12)[sl].cpu().numpy().astype(np.float64)
    rad = dev["radius"][sl].cpu().numpy().astype(np.float64)
    dep = dev["depth"][sl].cpu().numpy()
    idx = np.flatnonzero(rad > 0)
    z = dep[idx]
    order = np.argsort(z, kind="stable")
    xc = dev["x_cam"].view(-1, 3)[sl].cpu().numpy().astype(np.float64)[idx]
    cov = dev["cov_cam"].view(-1, 3, 3)[sl].cpu().numpy().astype(np.float64)[idx]
    sp = ProjectedSplats(idx, rec[idx, 0:2], rec[idx, 2:5], z.astype(np.float64), rec[idx, 9:12], rec[idx, 5],
                         rad[idx], n, xc, cov, world, camera, order)
    sp._dev = {"batch": dev, "b": b}
    return sp


def preprocess(world, camera) -> ProjectedSplats:
    """S/render.py:201-230 (non-finite inputs raise FloatingPointError naming the index)."""
    _check_camera(camera)
    dev = _project_batch([world], [camera])
    return _splats_from(dev, 0, world, camera)


def _stop_global(dev, b, splats, state, m):
    """Translate the per-tile local stop index into the reference's global sorted
    index (S/render.py:255-259): the first covering splat after termination, else M."""
    W, H = dev["W"], dev["H"]
    stop_local = (state & ((1 << 26) - 1)).reshape(H, W)
    out = np.full((H, W), m, dtype=np.int64)
    keys, vals, ranges, tile_bits, tiles = dev["binned"]
    rg = ranges.view(-1, 2).cpu().numpy().astype(np.int64)
    tiles_x = (W + 15) // 16
    rank = np.empty(splats.source_count, dtype=np.int64)
    rank[splats.index[splats.sort_order]] = np.arange(m)
    recs = dev["records"].view(-1, 12)[b * dev["N"]:(b + 1) * dev["N"]].cpu().numpy()
    rows = recs[:, 7].view(np.uint32)
    cols = recs[:, 8].view(np.uint32)
    lo16 = lambda v: (v & 0xFFFF).astype(np.int16).astype(np.int64)
    hi16 = lambda v: (v >> 16).astype(np.int16).astype(np.int64)
    vals_h = None
    yy, xx = np.mgrid[0:H, 0:W]
    tile_of = (b << tile_bits) + (yy // 16) * tiles_x + xx // 16
    counts = rg[tile_of, 1] - rg[tile_of, 0]
    for py, px in zip(*np.nonzero(stop_local < counts)):      # terminated pixels only
        s0, e0 = rg[tile_of[py, px]]
        sl = int(stop_local[py, px])
        if vals_h is None:
            vals_h = vals.cpu().numpy().astype(np.int64)
        for j in range(s0 + sl, e0):
            g = vals_h[j]
            if lo16(rows[g]) <= py <= hi16(rows[g]) and lo16(cols[g]) <= px <= hi16(cols[g]):
                out[py, px] = rank[g]
                break
    return out


def _raster_batch(dev, backgrounds, flags=L.RASTER_IMAGE | L.RASTER_MAXW_ALL, wsum_images=None):
    B, n, W, H = dev["B"], dev["N"], dev["W"], dev["H"]
    d = _dev()
    keys, vals, ranges, tile_bits, tiles = dev["binned"]
    bgs = _t(np.stack([np.asarray(bg, np.float64) for bg in backgrounds]))
    f32 = dict(dtype=torch.float32, device=d)
    out = {"bgs": bgs, "pix_T": torch.empty(B * H * W, **f32),
           "pix_state": torch.empty(B * H * W, dtype=torch.int32, device=d),
           "image": torch.empty(B * H * W * 3, **f32), "maxw": torch.zeros(B * n, **f32),
           "wsums": torch.zeros(B * n * 4, **f32)}
    wimg = None
    if wsum_images is not None:
        wimg = _t(np.stack([np.asarray(x, np.float64) for x in wsum_images]))
        flags |= L.RASTER_WSUMS | L.RASTER_WSUMS_IMAGE | L.RASTER_MAXW_ALL
    L.call("hs_raster_fwd", B, n, W, H, flags, _p(dev["records"]), _p(vals), _p(ranges), tile_bits, _p(bgs), None,
           _p(wimg), None, _p(out["pix_T"]), _p(out["pix_state"]), _p(out["image"]), _p(out["maxw"]),
           _p(out["wsums"]), None, None, _p(dev["raster_ws"]), _stream())
    return out


def _rasterize_items(dev, splats_list, backgrounds):
    out = _raster_batch(dev, backgrounds)
    B, n, W, H = dev["B"], dev["N"], dev["W"], dev["H"]
    img = out["image"].view(B, H, W, 3).cpu().numpy().astype(np.float64)
    T = out["pix_T"].view(B, H, W).cpu().numpy().astype(np.float64)
    st = out["pix_state"].view(B, H * W).cpu().numpy().view(np.uint32)
    mw = out["maxw"].view(B, n).cpu().numpy().astype(np.float64)
    res = []
    for b, sp in enumerate(splats_list):
        m = len(sp)
        stop = _stop_global(dev, b, sp, st[b], m)
        maxw = np.zeros(n)
        maxw[sp.index] = mw[b, sp.index]
        aux = RenderAux(T[b], maxw, sp, np.asarray(backgrounds[b], np.float64), stop)
        aux._dev = {"batch": dev, "b": b, "raster": out}
        res.append((img[b], aux))
    return res


def rasterize(splats: ProjectedSplats, camera, background):
    """S/render.py:389-407.  Returns (image (H, W, 3), RenderAux)."""
    dev = splats._dev["batch"]
    if dev["B"] != 1:
        dev = _project_batch([splats.world], [camera])
    return _rasterize_items(dev, [splats], [background])[0]


def render_backward(splats: ProjectedSplats, aux: RenderAux, grad_image) -> GaussianSet:
    """S/render.py:410-429: adjoint of preprocess + rasterize w.r.t. the world set."""
    dev, b, out = aux._dev["batch"], aux._dev["b"], aux._dev["raster"]
    B, n, W, H = dev["B"], dev["N"], dev["W"], dev["H"]
    keys, vals, ranges, tile_bits, tiles = dev["binned"]
    g = np.zeros((B, H, W, 3))
    g[b] = np.asarray(grad_image, np.float64)
    g_splat = torch.zeros(B * n * 9, dtype=torch.float32, device=_dev())
    L.call("hs_raster_bwd", B, n, W, H, _p(dev["records"]), _p(vals), _p(ranges), tile_bits, _p(out["bgs"]),
           _p(out["pix_T"]), _p(out["pix_state"]), _keep(_t(g)), ctypes.c_float(0.0), _p(g_splat), 0,
           _p(dev["raster_ws"]), _stream())
    g14 = torch.empty(B * 14 * n, dtype=torch.float32, device=_dev())
    L.call("hs_project_world_bwd", B, n, _p(dev["world14"]), _p(dev["cams"]), _p(g_splat), _p(g14), _stream())
    return _unpack14(g14[b * 14 * n:(b + 1) * 14 * n].cpu().numpy(), n)


def splat_space_grads(aux: RenderAux, grad_image):
    """The raster adjoint alone (per source Gaussian: g_mean 2, g_conic 3, g_opacity, g_color 3)."""
    dev, b, out = aux._dev["batch"], aux._dev["b"], aux._dev["raster"]
    B, n, W, H = dev["B"], dev["N"], dev["W"], dev["H"]
    keys, vals, ranges, tile_bits, tiles = dev["binned"]
    g = np.zeros((B, H, W, 3))
    g[b] = np.asarray(grad_image, np.float64)
    g_splat = torch.zeros(B * n * 9, dtype=torch.float32, device=_dev())
    L.call("hs_raster_bwd", B, n, W, H, _p(dev["records"]), _p(vals), _p(ranges), tile_bits, _p(out["bgs"]),
           _p(out["pix_T"]), _p(out["pix_state"]), _keep(_t(g)), ctypes.c_float(0.0), _p(g_splat), 0,
           _p(dev["raster_ws"]), _stream())
    return g_splat.view(B, n, 9)[b].cpu().numpy().astype(np.float64)


def splat_weight_sums(aux: RenderAux, image):
    """S/render.py:500-521: (sum w I, sum w) per source Gaussian, replaying the forward."""
    dev, b = aux._dev["batch"], aux._dev["b"]
    B, n, W, H = dev["B"], dev["N"], dev["W"], dev["H"]
    imgs = [np.zeros((H, W, 3))] * B
    imgs = list(imgs)
    imgs[b] = np.asarray(image, np.float64)
    bgs = [np.zeros(3)] * B
    bgs[b] = aux.background
    out = _raster_batch(dev, bgs, flags=L.RASTER_MAXW_ALL, wsum_images=imgs)
    ws = out["wsums"].view(B, n, 4)[b].cpu().numpy().astype(np.float64)
    sp = aux.splats
    num = np.zeros((n, 3))
    den = np.zeros(n)
    num[sp.index] = ws[sp.index, :3]
    den[sp.index] = ws[sp.index, 3]
    return num, den


def estimate_colors(aux: RenderAux, target, threshold=0.1):
    """S/color_init.py:45-65."""
    target = np.asarray(target, np.float64)
    cam = aux.splats.camera
    if target.shape != (cam.height, cam.width, 3):
        raise ValueError(f"target shape {target.shape} does not match the render ({cam.height}, {cam.width}, 3)")
    num, den = splat_weight_sums(aux, target)
    eligible = aux.max_weight > threshold
    bad = eligible & (den <= 0.0)
    if np.any(bad):
        raise RuntimeError(f"Gaussian {int(np.flatnonzero(bad)[0])} exceeds the weight threshold "
                           "but accumulated zero total weight")
    safe = np.where(den > 0.0, den, 1.0)
    return num / safe[:, None], eligible


def _logit(p, eps=1e-4):
    p = np.clip(np.asarray(p, np.float64), eps, 1.0 - eps)
    return np.log(p) - np.log1p(-p)


def apply_color_init(model, estimates, eligible, state):
    """S/color_init.py:68-80 (host bookkeeping on the caller's model/state)."""
    fresh = eligible & ~state.visited
    if not np.any(fresh):
        return 0
    model.base.color[fresh] = _logit(estimates[fresh])
    state.visited[fresh] = True
    return int(fresh.sum())


# ------------------------------------------------------------------ scheduler

SCHEMES = ("sequential", "naive", "two_stage")


class BatchRenderer:
    """S/scheduler.py:26-82.  On the device every scheme renders the whole batch
    with one launch per stage and ONE host sync (the key total); ``barrier_count``
    keeps the reference's accounting (two_stage: +1 per batch, naive: +B,
    sequential: 0) so callers and tests that read it behave the same."""

    def __init__(self, workers: int = 1, scheme: str = "two_stage"):
        if scheme not in SCHEMES:
            raise ValueError(f"unknown scheme {scheme!r}, expected one of {SCHEMES}")
        self.workers = max(1, int(workers))
        self.scheme = scheme
        self.barrier_count = 0
        self.batches_rendered = 0

    def close(self):
        pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def render_batch(self, items):
        if len(items) < 1:
            raise ValueError("batch must contain at least one item")
        for _, cam, _ in items:
            _check_camera(cam)
        groups = {}
        for i, (g, cam, bg) in enumerate(items):
            key = (g.position.shape[0], int(cam.width), int(cam.height))
            groups.setdefault(key, []).append(i)
        out = [None] * len(items)
        for key, idx in groups.items():
            dev = _project_batch([items[i][0] for i in idx], [items[i][1] for i in idx])
            splats = [_splats_from(dev, j, items[i][0], items[i][1]) for j, i in enumerate(idx)]
            res = _rasterize_items(dev, splats, [items[i][2] for i in idx])
            for j, i in enumerate(idx):
                out[i] = res[j]
        if self.scheme == "two_stage":
            self.barrier_count += 1
        elif self.scheme == "naive":
            self.barrier_count += len(items)
        self.batches_rendered += 1
        return out

    def map_items(self, fn, items):
        return [fn(*args) for args in items]


def render_batch(items, workers: int = 1, scheme: str = "two_stage"):
    with BatchRenderer(workers=workers, scheme=scheme) as r:
        return r.render_batch(items)


# ---------------------------------------------------------------- train step

def _trainer_for(state, batch, camera):
    """Device mirror of a reference TrainState, created on first use."""
    tr = getattr(state, "_b200_trainer", None)
    model = state.model
    if tr is None or tr.B != batch:
        av = AvatarParams.from_host(model.base, model.deltas, model.mlp, model.bindings.triangle_index,
                                    model.bindings.barycentric)
        cfg = state.config
        tr = Trainer(av, int(camera.width), int(camera.height), batch, lrs=lrs_from_config(cfg),
                     color_init=cfg.color_init, threshold=state.color_state.threshold)
        tr.visited.copy_(torch.from_numpy(state.color_state.visited.astype(np.uint8)))
        prev = getattr(state, "_b200_trainer", None)
        if prev is not None:                    # keep Adam moments across batch-size changes
            tr.m.copy_(prev.m)
            tr.v.copy_(prev.v)
            tr.step_count = prev.step_count
        state._b200_trainer = tr
    return tr


def train_step(state, samples, backgrounds, mesh_of):
    """S/train.py:214-260 on the device.  ``state`` is a reference-style TrainState
    (model, config, camera, color_state); the updated parameters and visited flags
    are written back into it.  Returns (mean loss, black-background L1 per item)."""
    cam = state.camera
    B = len(samples)
    tr = _trainer_for(state, B, cam)
    if not state.config.use_mlp:
        raise ValueError("use_mlp=False is not supported on the device path")
    d = tr.av.device
    # the samples' u8 targets and mesh frames are uploaded once and cached on the sample /
    # mesh objects (the reference caches mesh frames on its samples the same way,
    # S/dataset.py:54-57): a step moves only theta, the cameras and the backgrounds H2D
    thetas = torch.from_numpy(np.stack([np.asarray(s.theta, np.float32) for s in samples])).to(d, non_blocking=True)
    targets = torch.stack([_sample_dev(s, d) for s in samples])
    frames = torch.stack([_mesh_dev(mesh_of(s), d) for s in samples])
    cams = torch.from_numpy(np.tile(camera_array(cam), (B, 1))).to(d, non_blocking=True)
    bgs = torch.from_numpy(np.asarray(backgrounds, np.float32)).to(d, non_blocking=True)
    tr.step(thetas, targets, frames, cams, bgs)
    res = tr.result()
    # write back (the reference mutates model / colour state in place): one DMA of the
    # flat fp32 parameters into a pinned buffer, then the float64 host writes
    host = getattr(tr, "_host_params", None)
    if host is None:
        host = tr._host_params = torch.empty(tr.av.size, dtype=torch.float32, pin_memory=True)
    host.copy_(tr.av.params, non_blocking=True)
    vis = tr.visited.to("cpu", non_blocking=True)
    torch.cuda.current_stream().synchronize()
    base, deltas, mlp = tr.av.split_host(host.numpy(), dtype=None)
    m = state.model
    for k in ATTRS:
        getattr(m.base, k)[...] = base[k]
    n = tr.av.N
    for k, d in enumerate(m.deltas):
        d.position[...] = deltas[k, :3 * n].reshape(n, 3)
        d.rotation[...] = deltas[k, 3 * n:7 * n].reshape(n, 4)
        d.color[...] = deltas[k, 7 * n:].reshape(n, 3)
    for k in ("w1", "b1", "w2", "b2", "w3", "b3"):
        getattr(m.mlp, k)[...] = mlp[k]
    state.color_state.visited[...] = vis.numpy().astype(bool)
    return res.loss, res.black_l1.astype(np.float64)


def _sample_u8(sample):
    """The sample's straight-RGBA image as u8 (PNG-backed [0, 1] floats round exactly),
    cached on the sample like the reference caches its mesh frames on it
    (S/dataset.py:54-57); recomputed when sample.image is replaced."""
    img = sample.image
    hit = getattr(sample, "_b200_u8", None)
    if hit is not None and hit[0] is img:
        return hit[1]
    a = np.asarray(img)
    u8 = a if a.dtype == np.uint8 else np.clip(np.round(np.asarray(a, np.float64) * 255.0), 0, 255).astype(np.uint8)
    try:
        sample._b200_u8 = (img, u8)
    except AttributeError:
        pass
    return u8


def _sample_dev(sample, device):
    """The sample's u8 target as a device tensor, cached on the sample (re-uploaded when
    sample.image is replaced)."""
    img = sample.image
    hit = getattr(sample, "_b200_dev", None)
    if hit is not None and hit[0] is img:
        return hit[1]
    t = torch.from_numpy(np.ascontiguousarray(_sample_u8(sample))).to(device)
    try:
        sample._b200_dev = (img, t)
    except AttributeError:
        pass
    return t


def _mesh_dev(mesh, device):
    """A MeshFrames' (F, 22) device layout, cached on the object."""
    hit = getattr(mesh, "_b200_dev", None)
    if hit is not None and hit[0] is mesh.rotation:
        return hit[1]
    t = torch.from_numpy(_mesh_array(mesh)).to(device)
    try:
        mesh._b200_dev = (mesh.rotation, t)
    except AttributeError:
        pass
    return t


def _mesh_array(mesh):
    """(F, 22) fp32 device layout of a MeshFrames, cached on the object."""
    hit = getattr(mesh, "_b200_frames", None)
    if hit is not None and hit[0] is mesh.rotation:
        return hit[1]
    arr = frames_array(mesh)
    try:
        mesh._b200_frames = (mesh.rotation, arr)
    except AttributeError:
        pass
    return arr
