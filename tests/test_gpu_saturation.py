"""Saturated opacities: fp32 alpha == 1 must not poison the adjoint (S/render.py:264,
:318-319).

The reference evaluates alpha in float64, where sigmoid(logit) < 1 until logit ~36.7;
fp32 rounds the opacity to 1.0 above logit ~16.6, and the Gaussian factor to 1.0 at a
pixel centre within ~1e-3 px of the mean, so alpha == 1.0f exactly.  The raster clamps the
opacity at 1 - 2^-24 when it stages a splat, so 1 - alpha >= 2^-24 in the transmittance
update and in the adjoint's T recovery (hs_raster.cu: kOpacityMax), instead of producing
T = 0 and 0 * inf = NaN.

Scenes: 32x32, stacks of three Gaussians (depths 2, 2.5, 3) whose means project 1.6e-5
px from a pixel centre, opacity logit 15 / 17 / 20 / 30 / 40, over a layer of random
background Gaussians.  Checked: everything finite; pixels max-abs 1e-4 and splat-space
and world-space gradients rel 1e-3 against the oracle (float64, replaying the device's
order and bbox) outside the flip-masked pixels, whose image gradient is zeroed on both
sides (the alpha -> 1 pixels are among them: there fp32 and float64 composite
differently by construction).  Plus a C1-size training step with saturated logits.
"""
import numpy as np
import pytest
import torch

import oracle as O
from gpu_helpers import MaskedReplay, rel_fail

pytestmark = pytest.mark.gpu
ATTRS = ("position", "rotation", "scale", "opacity", "color")
LOGITS = [15.0, 17.0, 20.0, 30.0, 40.0]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2503_12886_b200 import build
    build.build()


def f32(a):
    return np.asarray(a, np.float32).astype(np.float64)


def sigmoid(x):
    return 1.0 / (1.0 + np.exp(-np.asarray(x, np.float64)))


def scene(logit, seed=0):
    rng = np.random.default_rng(seed)
    W = H = 32
    fx = 32.0
    cam = O.Cam(fx, fx, 16.0, 16.0, np.eye(3), np.array([0.0, 0.0, 2.0]), W, H)
    pos, op = [], []
    for (kx, ky) in [(-6, -5), (-1, 0), (0, 4), (5, -3), (7, 7)]:
        for zc in (2.0, 2.5, 3.0):
            # camera z = zc; pixel centre k + 0.5 + 16 -> x = (k + 0.5) zc / fx, + 1e-6
            pos.append([(kx + 0.5) * zc / fx + 1e-6, (ky + 0.5) * zc / fx, zc - 2.0])
            op.append(sigmoid(logit))
    ns = len(pos)
    nb = 40
    pos += list(np.c_[rng.uniform(-0.8, 0.8, (nb, 2)), rng.uniform(1.5, 2.0, nb)])
    op += list(rng.uniform(0.3, 0.95, nb))
    n = ns + nb
    q = np.tile([1.0, 0.0, 0.0, 0.0], (n, 1))
    q[ns:] = rng.normal(size=(nb, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    scale = np.full((n, 3), 0.05)
    scale[ns:] = rng.uniform(0.03, 0.12, (nb, 3))
    world = O.GSet(np.array(pos), q, scale, np.array(op), rng.uniform(0, 1, (n, 3)))
    world = O.GSet(*(f32(getattr(world, a)) for a in ATTRS))
    return world, cam, f32(rng.uniform(0, 1, 3)), rng


def oracle_from_device(sp, world, cam):
    dev = sp._dev["batch"]
    n = dev["N"]
    rec = dev["records"].view(-1, 12)[:n].cpu().numpy()
    from gpu_helpers import unpack_bbox
    bbox = unpack_bbox(rec)
    idx = sp.index
    osp = O.preprocess(world, cam)
    assert np.array_equal(osp.index, idx)
    osp.mean2d = f32(rec[idx, 0:2])
    osp.conic = f32(rec[idx, 2:5])
    osp.opacity = f32(rec[idx, 5])
    osp.color = f32(rec[idx, 9:12])
    osp.radius = f32(sp.radius)
    order = np.argsort(np.asarray(sp.depth, np.float32), kind="stable")
    return osp, order, bbox[idx]


@pytest.mark.parametrize("logit", LOGITS)
def test_saturated_stack_raster_and_adjoint(logit):
    from paper_2503_12886_b200 import compat as C
    world, cam, bg, rng = scene(logit)
    sp = C.preprocess(world, cam)
    image, aux = C.rasterize(sp, cam, bg)
    assert np.isfinite(image).all() and np.isfinite(aux.transmittance).all()
    osp, order, bbox = oracle_from_device(sp, world, cam)
    # the compat route takes activated opacities: fp32(sigmoid(logit)) is 1.0 from
    # logit ~17.3 (the Trainer's own fp32 sigmoid saturates from ~16.6)
    saturated = int((np.float32(osp.opacity) == np.float32(1.0)).sum())
    assert saturated == (15 if np.float32(sigmoid(logit)) == np.float32(1.0) else 0), saturated
    oimg, oaux = O.rasterize(osp, cam, bg, order=order, bbox=bbox)
    mask = O.flip_mask(osp, cam, order=order, bbox=bbox)
    if saturated:
        assert mask.sum() >= 5          # the alpha -> 1 pixels (one per stack at least)
    ok = ~mask
    assert np.max(np.abs(image - oimg)[ok]) <= 1e-4
    assert np.max(np.abs(aux.transmittance - oaux.transmittance)[ok]) <= 1e-4
    gimg = f32(rng.normal(size=image.shape)) * ok[:, :, None]
    gs = C.splat_space_grads(aux, gimg)[sp.index]
    assert np.isfinite(gs).all()
    om, oc, oo, ocol = O.splat_space_grads(osp, oaux, gimg)
    for name, a, b in (("mean", gs[:, 0:2], om), ("conic", gs[:, 2:5], oc), ("opacity", gs[:, 5], oo),
                       ("color", gs[:, 6:9], ocol)):
        nbad, worst, _ = rel_fail(a, b)
        assert nbad == 0, (logit, name, worst)
    g = C.render_backward(sp, aux, gimg)
    og = O.render_backward(osp, oaux, gimg)
    for a in ATTRS:
        assert np.isfinite(getattr(g, a)).all(), a
        nbad, worst, _ = rel_fail(getattr(g, a), getattr(og, a))
        assert nbad == 0, (logit, a, worst)
    # the same pixels with their full (unmasked) gradient: still finite on the device
    g_all = C.splat_space_grads(aux, f32(rng.normal(size=image.shape)))
    assert np.isfinite(g_all).all()


def test_saturated_training_step():
    """C1 shape (19,881 Gaussians, 4 x 256^2) with every opacity logit in {15, 17, 20,
    30, 40}: two fused steps stay finite; the unfused step with the masked replay
    matches the oracle entrywise."""
    from bench_support import synth
    from paper_2503_12886_b200.device import AvatarParams, Trainer, split_flat
    wl = synth.make_workload(141, 4, 256)
    av = wl.avatar
    base = {a: np.array(av.base[a], copy=True) for a in ATTRS}
    base["opacity"] = np.resize(np.array(LOGITS), base["opacity"].shape)
    base["scale"] = base["scale"] + 0.7          # larger splats: more near-centre pixels
    mk = lambda: AvatarParams.from_host(O.GSet(*(base[a] for a in ATTRS)), av.deltas, av.mlp, av.tri_index,
                                        av.barycentric)
    B = 4
    cams = np.tile(wl.camera.packed(), (B, 1))
    bgs = np.asarray(wl.backgrounds, np.float32).astype(np.float64)
    fused = Trainer(mk(), 256, 256, B)
    for _ in range(2):
        r = fused.step_from_host(wl.thetas, wl.targets, wl.frames, cams, bgs)
        torch.cuda.synchronize()
        assert np.isfinite(r.loss)
        assert torch.isfinite(fused.g_splat).all() and torch.isfinite(fused.grads).all()
        assert torch.isfinite(fused.av.params).all()
    # parity of the first step
    tr = Trainer(mk(), 256, 256, B)
    tr.fused_raster = False
    tr.radius = torch.empty(B * tr.av.N, device="cuda")
    model = O.Model(O.GSet(*(f32(base[a]) for a in ATTRS)), f32(av.deltas), {k: f32(v) for k, v in av.mlp.items()},
                    av.tri_index, f32(av.barycentric))
    p = wl.camera.packed().astype(np.float64)
    cam = O.Cam(p[12], p[13], p[14], p[15], p[:9].reshape(3, 3), p[9:12], 256, 256)
    frames = [O.Frames(f[:, :9].reshape(-1, 3, 3).astype(np.float64), f[:, 9:13].astype(np.float64),
                       f[:, 13:].reshape(-1, 3, 3).astype(np.float64)) for f in wl.frames]
    th = f32(wl.thetas)
    hook = MaskedReplay(O, model, cam, th, frames, wl.targets, bgs)
    tr.debug_before_backward = hook
    tr.step_from_host(wl.thetas, wl.targets, wl.frames, cams, bgs)
    torch.cuda.synchronize()
    state = O.State(model, cam, workers=8)
    O.train_step(state, th, wl.targets.astype(np.float64) / 255.0, frames, bgs, replay=hook.replay)
    state.close()
    print("saturated step:", hook.report)
    assert hook.report["t_maxabs"] <= 1e-4
    g_base, g_deltas, g_mlp = state.last_grads
    gb, gd, gm = split_flat(tr.grads.cpu().numpy(), tr.av.N, tr.av.K, tr.av.H, tr.av.D)
    assert np.isfinite(tr.grads.cpu().numpy()).all()
    for a in ATTRS:
        nbad, worst, _ = rel_fail(gb[a], getattr(g_base, a), scale=np.abs(g_base.position).max())
        assert nbad == 0, (a, worst)
    nbad, worst, _ = rel_fail(gd, g_deltas)
    assert nbad == 0, ("deltas", worst)
