"""Generate the golden vectors that pin the oracle to the reference.

Run HERE (the build container), where the reference package is importable:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports ``headsplat`` from ``/root/reference/pkg/src`` (read-only), runs the
reference's own functions on small seeded inputs and writes compressed ``.npz``
fixtures next to this script.  The GPU box never runs this script (the reference
does not exist there); the committed fixtures travel instead.

Fixtures (all float64 unless stated):
  model.npz    map_params / mlp_backward / blend / blend_backward / activate /
               activate_backward                          (S/model.py:130-248)
  binding.npz  build_head_rig, bind_gaussians(uv 24), rig_evaluate, mesh_frames,
               transform_to_deformed / transform_backward  (S/rig.py, S/binding.py)
  render.npz   preprocess / rasterize / render_backward / splat_weight_sums on
               random activated scenes incl. culled, opaque and empty cases
                                                           (S/render.py:201-521)
  color.npz    estimate_colors / apply_color_init          (S/color_init.py:45-80)
  train.npz    two reference train_step calls on a tiny synthetic avatar with the
               summed ParamGradients captured at Optimizer.step (S/train.py:214-278)
  counts.json  bind_gaussians counts at uv 141/224/317
  io.npz       save_model bytes, a synth_generate sequence + load_sequence/evaluate,
               psnr/ssim/l1 values                 (S/model_io.py, S/dataset.py:175-275,
                                                    S/metrics.py:25-85, S/train.py:342-360)
  pools.npz    SamplePools / sample_batch bookkeeping        (S/stream.py:27-86)
  rig.npz      rig_evaluate + mesh_frames on a theta batch, DegenerateTriangleError
               messages                                    (S/rig.py:57-66, S/binding.py:67-115)
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _ref():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.dont_write_bytecode = True
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import headsplat  # noqa: F401
    return headsplat


def gset_arrays(prefix, g):
    return {f"{prefix}.{n}": np.asarray(getattr(g, n)) for n in ("position", "rotation", "scale", "opacity", "color")}


def make_model(out):
    from headsplat.binding import GaussianBindings
    from headsplat.gaussians import DeltaSet, GaussianGrad, GaussianSet
    from headsplat.model import (AvatarModel, MlpWeights, activate, activate_backward, blend,
                                 blend_backward, map_params, mlp_backward)
    rng = np.random.default_rng(11)
    n, k, h, hidden = 37, 5, 13, 32
    base = GaussianSet(rng.normal(size=(n, 3)), rng.normal(size=(n, 4)) + np.array([2.0, 0, 0, 0]),
                       rng.normal(scale=0.5, size=(n, 3)), rng.normal(size=n), rng.normal(size=(n, 3)))
    deltas = [DeltaSet(rng.normal(scale=0.1, size=(n, 3)), rng.normal(scale=0.1, size=(n, 4)),
                       rng.normal(scale=0.1, size=(n, 3))) for _ in range(k)]
    mlp = MlpWeights(rng.normal(size=(hidden, h)), rng.normal(size=hidden),
                     rng.normal(size=(hidden, hidden)) / 4, rng.normal(size=hidden),
                     rng.normal(size=(k, hidden)), rng.normal(size=k))
    model = AvatarModel(base, deltas, mlp, GaussianBindings(np.zeros(n, np.int64), np.tile([1.0, 0, 0], (n, 1))))
    theta = rng.normal(size=h)
    psi, cache = map_params(mlp, theta)
    psi = psi.copy()
    psi[1] = 0.0                      # exercise the psi_k == 0 skip (S/model.py:179)
    raw = blend(model, psi)
    act = activate(raw)
    g_act = GaussianGrad(rng.normal(size=(n, 3)), rng.normal(size=(n, 4)), rng.normal(size=(n, 3)),
                         rng.normal(size=n), rng.normal(size=(n, 3)))
    g_raw = activate_backward(raw, act, g_act)
    g_base, g_deltas, g_psi = blend_backward(model, psi, g_raw)
    g_mlp, g_theta = mlp_backward(mlp, cache, g_psi)
    d = {"theta": theta, "psi": psi, "psi_mlp": map_params(mlp, theta)[0]}
    for nm in ("w1", "b1", "w2", "b2", "w3", "b3"):
        d["mlp." + nm] = getattr(mlp, nm)
        d["gmlp." + nm] = getattr(g_mlp, nm)
    d.update(gset_arrays("base", base))
    d["deltas"] = np.stack([np.concatenate([x.position.ravel(), x.rotation.ravel(), x.color.ravel()]) for x in deltas])
    d.update(gset_arrays("raw", raw))
    d.update(gset_arrays("act", act))
    d.update(gset_arrays("g_act", g_act))
    d.update(gset_arrays("g_raw", g_raw))
    d.update(gset_arrays("g_base", g_base))
    d["g_deltas"] = np.stack([np.concatenate([x.position.ravel(), x.rotation.ravel(), x.color.ravel()]) for x in g_deltas])
    d["g_psi"] = g_psi
    # basis recovery with unit weights (T/test_model.py:103-113)
    unit = np.zeros(k); unit[2] = 1.0
    d["unit_blend.position"] = blend(model, unit).position
    out["model"] = d


def make_binding(out, counts):
    from headsplat.binding import bind_gaussians, mesh_frames, transform_backward, transform_to_deformed
    from headsplat.gaussians import GaussianGrad, GaussianSet
    from headsplat.rig import build_head_rig, rig_evaluate
    rig = build_head_rig()
    rng = np.random.default_rng(5)
    bindings, _ = bind_gaussians(rig, 24)
    n = bindings.count
    theta = rng.normal(0.0, 0.3, rig.param_dim)
    verts = rig_evaluate(rig, theta)
    frames = mesh_frames(rig, verts)
    q = rng.normal(size=(n, 4)); q /= np.linalg.norm(q, axis=-1, keepdims=True)
    tangent = GaussianSet(rng.normal(0, 0.01, (n, 3)), q, rng.uniform(0.01, 0.03, (n, 3)),
                          rng.uniform(0.1, 0.9, n), rng.uniform(0, 1, (n, 3)))
    world = transform_to_deformed(tangent, frames, bindings)
    g_world = GaussianGrad(rng.normal(size=(n, 3)), rng.normal(size=(n, 4)), rng.normal(size=(n, 3)),
                           rng.normal(size=n), rng.normal(size=(n, 3)))
    g_t = transform_backward(tangent, frames, bindings, g_world)
    d = {
        "rig.base_vertices": rig.base_vertices, "rig.faces": rig.faces, "rig.uv_coords": rig.uv_coords,
        "rig.expr_bases": rig.expr_bases,
        "tri_index": bindings.triangle_index, "barycentric": bindings.barycentric,
        "theta": theta, "verts": verts,
        "frames.rotation": frames.rotation, "frames.quat": frames.quat, "frames.tri_vertices": frames.tri_vertices,
    }
    d.update(gset_arrays("tangent", tangent))
    d.update(gset_arrays("world", world))
    d.update(gset_arrays("g_world", g_world))
    d.update(gset_arrays("g_tangent", g_t))
    out["binding"] = d
    for r in (141, 224, 317):
        b, _ = bind_gaussians(rig, r)
        counts[f"uv{r}"] = int(b.count)
        counts[f"uv{r}_checksum"] = b.checksum()


def _small_camera(size=8, f=12.0):
    from headsplat.render import Camera
    return Camera(f, f, size / 2.0, size / 2.0, np.eye(3), np.array([0.0, 0.0, 2.0]), size, size)


def _activated_world(rng, n, spread=0.5, scale_range=(0.05, 0.25), opacity_range=(0.3, 0.9)):
    from headsplat.gaussians import GaussianSet
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=-1, keepdims=True)
    return GaussianSet(rng.uniform(-spread, spread, size=(n, 3)), q, rng.uniform(*scale_range, size=(n, 3)),
                       rng.uniform(*opacity_range, size=n), rng.uniform(0.1, 0.9, size=(n, 3)))


def make_render(out):
    from headsplat.gaussians import GaussianSet
    from headsplat.render import Camera, preprocess, rasterize, render_backward, splat_weight_sums
    rng = np.random.default_rng(21)
    scenes = []
    # (a) random scenes with some culled Gaussians, 16x16 and a 24x20 non-square
    for i, (n, w, h, spread) in enumerate([(12, 16, 16, 1.0), (40, 24, 20, 0.7), (60, 32, 32, 0.6)]):
        world = _activated_world(rng, n, spread=spread)
        world.position[:, 2] = rng.uniform(-1.0, 3.0, size=n) if i == 0 else world.position[:, 2]
        cam = Camera(1.5 * w, 1.5 * w, w / 2.0, h / 2.0, np.eye(3), np.array([0.0, 0.0, 2.0]), w, h)
        scenes.append((world, cam))
    # (b) saturating / terminating scene: many near-opaque splats stacked (stop < M)
    n = 48
    world = _activated_world(rng, n, spread=0.05, scale_range=(0.3, 0.5), opacity_range=(0.95, 0.999))
    scenes.append((world, _small_camera(12)))
    # (c) frontal camera with yaw (non-identity rotation)
    world = _activated_world(rng, 80, spread=0.6, scale_range=(0.02, 0.1))
    scenes.append((world, Camera.frontal(32, yaw=0.3)))
    # (d) empty: everything behind the camera
    world = _activated_world(rng, 3)
    world.position[:, 2] = -5.0
    scenes.append((world, _small_camera(8)))
    d = {"num_scenes": np.array(len(scenes))}
    for s, (world, cam) in enumerate(scenes):
        splats = preprocess(world, cam)
        bg = rng.uniform(0, 1, 3)
        image, aux = rasterize(splats, cam, bg)
        gimg = rng.normal(size=(cam.height, cam.width, 3))
        grad = render_backward(splats, aux, gimg)
        target = rng.uniform(0, 1, size=(cam.height, cam.width, 3))
        num, den = splat_weight_sums(aux, target)
        p = f"s{s}."
        d.update({p + k: v for k, v in gset_arrays("world", world).items()})
        d[p + "cam"] = np.concatenate([cam.rotation.ravel(), cam.translation, [cam.fx, cam.fy, cam.cx, cam.cy]])
        d[p + "wh"] = np.array([cam.width, cam.height])
        d[p + "bg"] = bg
        for k in ("index", "mean2d", "conic", "depth", "radius", "x_cam", "cov_cam", "sort_order"):
            d[p + "splats." + k] = np.asarray(getattr(splats, k))
        d[p + "image"] = image
        d[p + "trans"] = aux.transmittance
        d[p + "stop"] = aux.stop
        d[p + "max_weight"] = aux.max_weight
        d[p + "grad_image"] = gimg
        d.update({p + k: v for k, v in gset_arrays("grad", grad).items()})
        d[p + "target"] = target
        d[p + "num"] = num
        d[p + "den"] = den
    out["render"] = d


def make_color(out):
    from headsplat.binding import GaussianBindings
    from headsplat.color_init import ColorInitState, apply_color_init, estimate_colors
    from headsplat.gaussians import DeltaSet, GaussianSet
    from headsplat.model import AvatarModel, MlpWeights
    from headsplat.render import preprocess, rasterize
    rng = np.random.default_rng(31)
    n = 30
    world = _activated_world(rng, n, spread=0.4)
    cam = _small_camera(16)
    splats = preprocess(world, cam)
    _, aux = rasterize(splats, cam, np.zeros(3))
    target = rng.uniform(0, 1, (16, 16, 3))
    est, eligible = estimate_colors(aux, target, 0.1)
    base = GaussianSet(np.zeros((n, 3)), np.tile([1.0, 0, 0, 0], (n, 1)), np.zeros((n, 3)), np.zeros(n),
                       rng.normal(size=(n, 3)))
    model = AvatarModel(base, [DeltaSet.zeros(n)], MlpWeights.create(3, 1, 4),
                        GaussianBindings(np.zeros(n, np.int64), np.tile([1.0, 0, 0], (n, 1))))
    state = ColorInitState.create(n, 0.1)
    state.visited[:3] = True
    color_before = model.base.color.copy()
    count = apply_color_init(model, est, eligible, state)
    d = {f"world.{k}": np.asarray(getattr(world, k)) for k in ("position", "rotation", "scale", "opacity", "color")}
    d.update({"target": target, "est": est, "eligible": eligible, "color_before": color_before,
              "color_after": model.base.color, "visited": state.visited, "count": np.array(count),
              "cam": np.concatenate([cam.rotation.ravel(), cam.translation, [cam.fx, cam.fy, cam.cx, cam.cy]]),
              "max_weight": aux.max_weight})
    out["color"] = d


def make_train(out):
    from headsplat.color_init import ColorInitState
    from headsplat.dataset import FrameSample, SequenceDataset
    from headsplat.render import Camera
    from headsplat.rig import build_head_rig
    from headsplat.scheduler import BatchRenderer
    from headsplat.train import Optimizer, TrainConfig, TrainState, init_avatar, train_step
    rng = np.random.default_rng(0)
    rig = build_head_rig()
    size, B = 32, 3
    cfg = TrainConfig(uv_resolution=20, num_blendshapes=4, hidden_dim=16, batch_size=B, workers=1)
    model = init_avatar(rig, cfg)
    n = model.count
    for d in model.deltas:          # SURVEY §8d perturbation
        d.position[:] = rng.normal(0, 0.002, (n, 3))
        d.rotation[:] = rng.normal(0, 0.02, (n, 4))
        d.color[:] = rng.normal(0, 0.1, (n, 3))
    model.base.opacity[:] = rng.uniform(-2, 2, n)
    model.base.color[:] = rng.normal(0, 1, (n, 3))
    cam = Camera.frontal(size)
    thetas = rng.normal(0, 0.3, (B, rig.param_dim))
    images = [np.round(rng.uniform(0, 1, (size, size, 4)) * 255) / 255 for _ in range(B)]
    ds = SequenceDataset(None, cam, rig, thetas, images)
    samples = [ds.frame(i) for i in range(B)]
    d = {"tri_index": model.bindings.triangle_index, "barycentric": model.bindings.barycentric,
         "thetas": thetas, "images": np.stack(images), "cam": np.concatenate(
             [cam.rotation.ravel(), cam.translation, [cam.fx, cam.fy, cam.cx, cam.cy]]), "size": np.array(size)}
    d.update({k: v.copy() for k, v in gset_arrays("base0", model.base).items()})
    d["deltas0"] = np.stack([np.concatenate([x.position.ravel(), x.rotation.ravel(), x.color.ravel()]) for x in model.deltas])
    for nm in ("w1", "b1", "w2", "b2", "w3", "b3"):
        d["mlp0." + nm] = getattr(model.mlp, nm).copy()
    for i, s in enumerate(samples):
        m = ds.mesh_for(s)
        d[f"frames{i}.rotation"] = m.rotation
        d[f"frames{i}.quat"] = m.quat
        d[f"frames{i}.tri_vertices"] = m.tri_vertices
    state = TrainState(model, Optimizer(model, cfg), BatchRenderer(1), ColorInitState.create(n, 0.1), cfg, cam)
    captured = []
    orig = state.optimizer.step

    def capture(mdl, grads):
        captured.append((gset_arrays("g", grads.base),
                         np.stack([np.concatenate([x.position.ravel(), x.rotation.ravel(), x.color.ravel()]) for x in grads.deltas]),
                         {nm: getattr(grads.mlp, nm).copy() for nm in ("w1", "b1", "w2", "b2", "w3", "b3")}))
        return orig(mdl, grads)
    state.optimizer.step = capture
    for step in range(2):
        bgs = rng.uniform(0, 1, (B, 3))
        loss, black = train_step(state, samples, bgs, ds.mesh_for)
        d[f"step{step}.bgs"] = bgs
        d[f"step{step}.loss"] = np.array(loss)
        d[f"step{step}.black"] = black
        gb, gdel, gm = captured[-1]
        d.update({f"step{step}.{k}": v for k, v in gb.items()})
        d[f"step{step}.g_deltas"] = gdel
        d.update({f"step{step}.gmlp.{k}": v for k, v in gm.items()})
        d.update({f"step{step}.{k}": v.copy() for k, v in gset_arrays("base", model.base).items()})
        d[f"step{step}.deltas"] = np.stack([np.concatenate([x.position.ravel(), x.rotation.ravel(), x.color.ravel()]) for x in model.deltas])
        for nm in ("w1", "b1", "w2", "b2", "w3", "b3"):
            d[f"step{step}.mlp.{nm}"] = getattr(model.mlp, nm).copy()
        d[f"step{step}.visited"] = state.color_state.visited.copy()
    out["train"] = d


def make_rig(out):
    """rig.npz: rig_evaluate + mesh_frames for a batch of theta (incl. a zero pose,
    which takes the identity branch of axis_angle_to_matrix, and a large pose), and
    the DegenerateTriangleError messages of a collapsed UV and a collapsed 3D face."""
    from headsplat.binding import DegenerateTriangleError, mesh_frames
    from headsplat.rig import ParametricHeadRig, build_head_rig, rig_evaluate
    rig = build_head_rig()
    rng = np.random.default_rng(9)
    th = rng.normal(0.0, 0.3, (5, rig.param_dim))
    th[1, -3:] = 0.0                                     # identity pose
    th[2, -3:] = [2.5, -1.0, 0.7]                        # large rotation
    th[3, :-3] *= 4.0                                    # strong expressions
    verts = np.stack([rig_evaluate(rig, t) for t in th])
    frames = [mesh_frames(rig, v) for v in verts]
    d = {"theta": th, "verts": verts,
         "frames.rotation": np.stack([f.rotation for f in frames]),
         "frames.quat": np.stack([f.quat for f in frames]),
         "frames.tri_vertices": np.stack([f.tri_vertices for f in frames])}
    # degenerate UV: give vertex faces[37][1] the UV of faces[37][0]
    uv = rig.uv_coords.copy()
    f37 = rig.faces[37]
    uv[f37[1]] = uv[f37[0]]
    bad = ParametricHeadRig(rig.base_vertices, rig.faces, uv, rig.expr_bases)
    try:
        mesh_frames(bad, rig_evaluate(bad, th[0]))
        msg = ""
    except DegenerateTriangleError as e:
        msg = str(e)
    d["bad_uv.uv_coords"], d["bad_uv.message"] = uv, np.array(msg)
    # degenerate 3D: collapse the vertices of face 300 onto one point
    v3 = rig.base_vertices.copy()
    eb = rig.expr_bases.copy()
    f300 = rig.faces[300]
    v3[f300[1]] = v3[f300[2]] = v3[f300[0]]
    eb[:, f300[1]] = eb[:, f300[2]] = eb[:, f300[0]]
    bad3 = ParametricHeadRig(v3, rig.faces, rig.uv_coords, eb)
    try:
        mesh_frames(bad3, rig_evaluate(bad3, th[0]))
        msg = ""
    except DegenerateTriangleError as e:
        msg = str(e)
    d["bad_3d.base_vertices"], d["bad_3d.expr_bases"], d["bad_3d.message"] = v3, eb, np.array(msg)
    out["rig"] = d


def make_pools(out):
    """pools.npz: S/stream.py SamplePools / sample_batch driven by a seeded rng --
    pool contents (frame indices) after every ingest and the batch picks, for the
    three sampling modes of run_online (full, no_global, no_local)."""
    from headsplat.stream import SamplePools, sample_batch

    class _S:                     # process_frame / sample_batch only read .index
        def __init__(self, i):
            self.index = i

    d = {}
    for mode, (lc, gc, keep) in {"full": (5, 12, True), "no_global": (5, 12, False),
                                 "no_local": (1, 12, True)}.items():
        rng = np.random.default_rng(3)
        pools = SamplePools(lc, gc, keep_evicted=keep)
        local, glob, picks, counters = [], [], [], []
        for i in range(1, 81):
            pools.process_frame(_S(i), rng)
            local.append([s.index for s in pools.local] + [0] * (lc - len(pools.local)))
            glob.append([s.index for s in pools.global_pool] + [0] * (gc - len(pools.global_pool)))
            counters.append([pools.evictions, pools.discarded, pools.reservoir_inserts])
            if i % 3 == 0:
                picks.append([s.index for s in sample_batch(pools, 8, 0.7 if mode == "full" else 1.0, rng)])
                rng.uniform(0.0, 1.0, size=(8, 3))       # the step's backgrounds (S/stream.py:140)
        d[f"{mode}.local"] = np.array(local)
        d[f"{mode}.global"] = np.array(glob)
        d[f"{mode}.picks"] = np.array(picks)
        d[f"{mode}.counters"] = np.array(counters)
    out["pools"] = d


def make_io(out):
    """io.npz: (1) a reference save_model file of a small perturbed avatar with random
    visited flags (bytes + arrays); (2) a reference synth_generate sequence (3 frames,
    48^2) as the raw files (params.json, rig.json, PNG bytes, gt_model.bin) with the
    reference load_sequence / evaluate(gt model) results; (3) psnr / ssim / l1 of
    random image pairs (S/metrics.py:25-85)."""
    import tempfile
    from pathlib import Path
    from headsplat.color_init import ColorInitState
    from headsplat.dataset import SynthConfig, load_sequence, synth_generate
    from headsplat.metrics import composite_over, psnr, ssim
    from headsplat.model_io import load_model, save_model
    from headsplat.rig import build_head_rig
    from headsplat.train import TrainConfig, evaluate, init_avatar
    rng = np.random.default_rng(21)
    d = {}
    rig = build_head_rig()
    model = init_avatar(rig, TrainConfig(uv_resolution=18, num_blendshapes=3, hidden_dim=8))
    n = model.count
    for x in model.deltas:
        x.position[:] = rng.normal(0, 0.002, (n, 3))
        x.rotation[:] = rng.normal(0, 0.02, (n, 4))
        x.color[:] = rng.normal(0, 0.1, (n, 3))
    model.base.opacity[:] = rng.uniform(-2, 2, n)
    for nm in ("w1", "b1", "w2", "b2", "w3", "b3"):
        getattr(model.mlp, nm)[...] = rng.normal(0, 0.3, getattr(model.mlp, nm).shape)
    vis = rng.uniform(size=n) < 0.4
    with tempfile.TemporaryDirectory() as td:
        save_model(model, ColorInitState(vis.copy()), Path(td) / "m.bin")
        d["model.bytes"] = np.frombuffer((Path(td) / "m.bin").read_bytes(), np.uint8).copy()
        seq_dir = Path(td) / "seq"
        synth_generate(seq_dir, SynthConfig(frames=3, image_size=48, uv_resolution=16, hidden_dim=16), seed=4)
        d["seq.params"] = np.array((seq_dir / "params.json").read_text())
        d["seq.rig"] = np.array((seq_dir / "rig.json").read_text())
        for i in range(3):
            d[f"seq.png{i}"] = np.frombuffer((seq_dir / "frames" / f"{i:06d}.png").read_bytes(), np.uint8).copy()
        d["seq.gt_model"] = np.frombuffer((seq_dir / "gt_model.bin").read_bytes(), np.uint8).copy()
        ds = load_sequence(seq_dir)
        d["seq.thetas"] = ds.thetas
        d["seq.images"] = np.stack(ds.images)
        gt, _ = load_model(seq_dir / "gt_model.bin")
        ev = evaluate(gt, ds)
        d["seq.eval"] = np.array([[f["psnr"], f["ssim"], f["l1"]] for f in ev["frames"]])
    d.update({f"model.{k}": v for k, v in gset_arrays("base", model.base).items()})
    d["model.deltas"] = np.stack([np.concatenate([x.position.ravel(), x.rotation.ravel(), x.color.ravel()])
                                  for x in model.deltas])
    for nm in ("w1", "b1", "w2", "b2", "w3", "b3"):
        d[f"model.mlp.{nm}"] = getattr(model.mlp, nm).copy()
    d["model.tri_index"] = model.bindings.triangle_index
    d["model.barycentric"] = model.bindings.barycentric
    d["model.visited"] = vis
    preds, tgts, vals = [], [], []
    for i in range(3):
        h, w = (24, 40) if i < 2 else (11, 11)
        t = rng.integers(0, 256, (h, w, 4)).astype(np.uint8)
        if i == 0:
            pred = composite_over(t / 255.0, np.zeros(3)).astype(np.float32)
            pred[3, 4, 1] += np.float32(0.25)
        else:
            pred = rng.uniform(0, 1, (h, w, 3)).astype(np.float32)
        tb = composite_over(t / 255.0, np.zeros(3))
        p64 = pred.astype(np.float64)
        d[f"metrics{i}.pred"], d[f"metrics{i}.target"] = pred, t
        d[f"metrics{i}.values"] = np.array([psnr(p64, tb), ssim(p64, tb), float(np.mean(np.abs(p64 - tb)))])
    out["io"] = d


def main():
    hs = _ref()
    import numba
    out = {}
    only = set(sys.argv[1:])            # e.g. `make_golden.py rig` regenerates rig.npz only
    if only:
        for name in only:
            globals()[f"make_{name}"](out)
        for name, d in out.items():
            np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)
            print(name, os.path.getsize(os.path.join(HERE, f"{name}.npz")))
        return
    counts = {"numpy": np.__version__, "numba": numba.__version__, "headsplat": getattr(hs, "__version__", "0.1.0")}
    make_model(out)
    make_binding(out, counts)
    make_render(out)
    make_color(out)
    make_train(out)
    make_rig(out)
    make_pools(out)
    make_io(out)
    for name, d in out.items():
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)
    with open(os.path.join(HERE, "counts.json"), "w") as f:
        json.dump(counts, f, indent=1, sort_keys=True)
    for name in out:
        print(name, os.path.getsize(os.path.join(HERE, f"{name}.npz")))


if __name__ == "__main__":
    main()
