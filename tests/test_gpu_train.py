"""The device training step (Trainer.step, through the C ABI) against the reference.

* test_reference_fixture_steps: two steps on the golden tiny avatar produced by the
  reference's own train_step (tests/golden/train.npz, captured gradients at
  Optimizer.step) -- loss, black L1, summed ParamGradients, updated parameters and
  colour-init visited flags.
* test_c1_step_vs_oracle: BASELINE configs[0] (20 bases, 19,881 Gaussians, B 4, 256^2)
  one step against the float64 oracle.
* test_c2_full_size_properties: configs[1] size (50,176 Gaussians, B 16, 512^2):
  bit-exact binning vs the oracle on the device's fp32 projection, sorted keys,
  consistent ranges, deterministic forward, finite loss.
"""
import numpy as np
import pytest
import torch

import binning as BO
import oracle as O
from conftest import golden
from gpu_helpers import normwise, replay_from_trainer

pytestmark = pytest.mark.gpu
ATTRS = ("position", "rotation", "scale", "opacity", "color")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2503_12886_b200 import build
    build.build()


def rel_fail_frac(a, b, rtol=1e-3, floor_frac=1e-6, scale=None):
    """Fraction of entries failing |a-b| <= max(floor, rtol*max(|a|,|b|)); the floor is
    floor_frac * max|b| of the tensor, or of `scale` (the whole gradient) when given --
    needed where the exact gradient is 0 and both sides hold only roundoff (e.g. the
    quaternion gradient of isotropic Gaussians at init, where R(q) cancels from Sigma)."""
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    ref = np.abs(b).max(initial=0.0) if scale is None else scale
    floor = floor_frac * max(ref, 1e-30)
    diff = np.abs(a - b)
    bad = (diff > floor) & (diff > rtol * np.maximum(np.abs(a), np.abs(b)))
    return float(bad.mean()) if bad.size else 0.0, int(bad.sum())


def split_grads(flat, N, K, H, D):
    from paper_2503_12886_b200.device import split_flat
    return split_flat(flat, N, K, H, D)


def test_reference_fixture_steps():
    from paper_2503_12886_b200.device import AvatarParams, Trainer
    d = golden("train")
    size = int(d["size"])
    base = O.GSet(*(d[f"base0.{a}"] for a in ATTRS))
    mlp = {k: d["mlp0." + k] for k in ("w1", "b1", "w2", "b2", "w3", "b3")}
    av = AvatarParams.from_host(base, d["deltas0"], mlp, d["tri_index"], d["barycentric"])
    B = d["thetas"].shape[0]
    tr = Trainer(av, size, size, B)
    frames = np.stack([np.concatenate([d[f"frames{i}.rotation"].reshape(-1, 9), d[f"frames{i}.quat"],
                                       d[f"frames{i}.tri_vertices"].reshape(-1, 9)], axis=1) for i in range(B)])
    cam = np.tile(d["cam"], (B, 1))
    targets = np.round(d["images"] * 255).astype(np.uint8)
    N, K = av.N, av.K
    for step in range(2):
        p = f"step{step}."
        res = tr.step_from_host(d["thetas"], targets, frames, cam, d[p + "bgs"])
        assert abs(res.loss - float(d[p + "loss"])) < 2e-5
        np.testing.assert_allclose(res.black_l1, d[p + "black"], atol=2e-5)
        gb, gd, gm = split_grads(tr.grads.cpu().numpy(), N, K, av.H, av.D)
        gscale = max(np.abs(d[p + "g." + a]).max() for a in ATTRS)
        for a in ATTRS:
            frac, nbad = rel_fail_frac(gb[a], d[p + "g." + a], scale=gscale)
            assert frac < 2e-3, (step, a, nbad)
        frac, nbad = rel_fail_frac(gd, d[p + "g_deltas"])
        assert frac < 2e-3, (step, "deltas", nbad)
        for k in gm:
            frac, nbad = rel_fail_frac(gm[k], d[p + "gmlp." + k], rtol=2e-3)
            assert frac < 5e-3, (step, k, nbad)
        # Parameters after Adam: Adam's first steps map gradients at or below eps=1e-8
        # (here the exactly-zero quaternion gradient of isotropic Gaussians, where fp32
        # roundoff is ~1e-9 and fp64 roundoff ~1e-17) to updates up to lr*|g|/(|g|+eps),
        # so the tolerance is a fraction of each group's learning rate.
        pb, pd, pm = av.split_host()
        lrs = {"position": 8e-4, "rotation": 5e-3, "scale": 2.5e-2, "opacity": 0.25, "color": 1.25e-2}
        for a in ATTRS:
            bad = np.abs(pb[a] - d[p + "base." + a]) > 0.05 * lrs[a] + 1e-4 * np.abs(d[p + "base." + a])
            assert bad.mean() < 5e-3, (step, a, int(bad.sum()))
        np.testing.assert_allclose(pd, d[p + "deltas"], rtol=1e-4, atol=0.05 * 2.5e-3)
        vis = tr.visited.cpu().numpy().astype(bool)
        assert (vis != d[p + "visited"]).sum() <= 2
    assert tr.visited.cpu().numpy().any()


def _oracle_model(wl):
    av = wl.avatar
    base = O.GSet(*(np.asarray(av.base[a], np.float32).astype(np.float64) for a in ATTRS))
    mlp = {k: np.asarray(v, np.float32).astype(np.float64) for k, v in av.mlp.items()}
    return O.Model(base, np.asarray(av.deltas, np.float32).astype(np.float64), mlp, av.tri_index,
                   np.asarray(av.barycentric, np.float32).astype(np.float64))


def test_c1_step_vs_oracle():
    from paper_2503_12886_b200 import synth
    from paper_2503_12886_b200.device import AvatarParams, Trainer
    wl = synth.make_workload(141, 4, 256)
    av = wl.avatar
    dev = AvatarParams.from_host(O.GSet(*(av.base[a] for a in ATTRS)), av.deltas, av.mlp, av.tri_index,
                                 av.barycentric)
    B = 4
    tr = Trainer(dev, 256, 256, B)
    tr.radius = torch.empty(B * dev.N, device="cuda")
    cams = np.tile(wl.camera.packed(), (B, 1))
    bgs = np.asarray(wl.backgrounds, np.float32).astype(np.float64)
    res = tr.step_from_host(wl.thetas, wl.targets, wl.frames, cams, bgs)
    replay = replay_from_trainer(tr)
    # oracle on the same fp32-quantized inputs
    model = _oracle_model(wl)
    cam = O.Cam(*[float(x) for x in wl.camera.packed()[12:16]], wl.camera.packed()[:9].reshape(3, 3).astype(np.float64),
                wl.camera.packed()[9:12].astype(np.float64), 256, 256)
    frames = [O.Frames(f[:, :9].reshape(-1, 3, 3).astype(np.float64), f[:, 9:13].astype(np.float64),
                       f[:, 13:].reshape(-1, 3, 3).astype(np.float64)) for f in wl.frames]
    state = O.State(model, cam, workers=4)
    images = wl.targets.astype(np.float64) / 255.0
    loss, black = O.train_step(state, np.asarray(wl.thetas, np.float32).astype(np.float64), images, frames, bgs,
                               replay=replay)
    state.close()
    assert abs(res.loss - loss) < 1e-4 * max(loss, 1e-3)
    np.testing.assert_allclose(res.black_l1, black, rtol=1e-3, atol=1e-5)
    g_base, g_deltas, g_mlp = state.last_grads
    gb, gd, gm = split_grads(tr.grads.cpu().numpy(), dev.N, dev.K, dev.H, dev.D)
    # Normwise relative errors.  The remaining fp32-vs-fp64 decision flips (alpha
    # cutoff, the L1 sign at |pred - target| ~ 1e-6) change whole per-pixel
    # gradients, so entrywise checks on the cancellation-heavy reductions (g_psi,
    # MLP) are not meaningful at this scale; the stage-wise blend/MLP adjoint fed
    # the device's own g_raw is checked tightly in test_c1_blend_mlp_stagewise.
    gscale = np.linalg.norm(g_base.position)
    report = {a: normwise(gb[a], getattr(g_base, a), scale=gscale if a == "rotation" else None) for a in ATTRS}
    report["deltas"] = normwise(gd, g_deltas)
    report.update({"mlp." + k: normwise(gm[k], g_mlp[k]) for k in gm})
    print("C1 normwise gradient errors:", report)
    for k, e in report.items():
        assert e < 2e-3, (k, e)
    # entrywise on the base/delta gradients: rel 1e-3 with a 1e-6 * max floor
    for a in ATTRS:
        frac, nbad = rel_fail_frac(gb[a], getattr(g_base, a), scale=np.abs(g_base.position).max())
        assert frac < 1e-3, (a, frac, nbad)
    frac, nbad = rel_fail_frac(gd, g_deltas)
    assert frac < 1e-3, ("deltas", frac, nbad)


def test_c1_blend_mlp_stagewise():
    """blend_bwd + mlp_bwd fed the device's own per-frame g_raw (C1 sizes)."""
    from paper_2503_12886_b200 import synth
    from paper_2503_12886_b200.device import AvatarParams, Trainer
    wl = synth.make_workload(141, 4, 256)
    av = wl.avatar
    dev = AvatarParams.from_host(O.GSet(*(av.base[a] for a in ATTRS)), av.deltas, av.mlp, av.tri_index,
                                 av.barycentric)
    B, n = 4, dev.N
    tr = Trainer(dev, 256, 256, B, color_init=False)
    tr.step_from_host(wl.thetas, wl.targets, wl.frames, np.tile(wl.camera.packed(), (B, 1)), wl.backgrounds)
    model = _oracle_model(wl)
    thetas = np.asarray(wl.thetas, np.float32).astype(np.float64)
    graw = tr.g_raw14.view(B, 14 * n).cpu().numpy().astype(np.float64)
    gpsi_dev = tr.gpsi.cpu().numpy().astype(np.float64)
    g_base14 = np.zeros(14 * n)
    g_deltas = np.zeros((dev.K, 10 * n))
    acc = {k: np.zeros_like(v) for k, v in model.mlp.items()}
    for b in range(B):
        g = graw[b]
        gr = O.GSet(g[:3 * n].reshape(n, 3), g[3 * n:7 * n].reshape(n, 4), g[10 * n:13 * n].reshape(n, 3),
                    g[13 * n:], g[7 * n:10 * n].reshape(n, 3))
        psi, cache = O.map_params(model.mlp, thetas[b])
        _, _, gpsi = O.blend_backward(model, psi, gr, g_base14, g_deltas)
        absum = np.abs(model.deltas * g[None, :10 * n]).sum(axis=1)
        assert np.max(np.abs(gpsi - gpsi_dev[b]) / absum) < 1e-6
        O.mlp_backward(model.mlp, cache, gpsi_dev[b], into=acc)
    gb, gd, gm = split_grads(tr.grads.cpu().numpy(), n, dev.K, dev.H, dev.D)
    assert normwise(gd, g_deltas) < 1e-6
    for k in gm:
        assert normwise(gm[k], acc[k]) < 1e-5, k


def test_c2_full_size_properties():
    from paper_2503_12886_b200 import synth
    from paper_2503_12886_b200.device import AvatarParams, Trainer
    wl = synth.make_workload(224, 16, 512, distinct_frames=4)
    av = wl.avatar
    dev = AvatarParams.from_host(O.GSet(*(av.base[a] for a in ATTRS)), av.deltas, av.mlp, av.tri_index,
                                 av.barycentric)
    assert dev.N == 50176
    B = 16
    tr = Trainer(dev, 512, 512, B)
    tr.radius = torch.empty(B * dev.N, device="cuda")
    cams = torch.from_numpy(np.tile(wl.camera.packed(), (B, 1))).cuda()
    th = torch.from_numpy(np.asarray(wl.thetas, np.float32)).cuda()
    fr = torch.from_numpy(wl.frames).cuda()
    bg = torch.from_numpy(np.asarray(wl.backgrounds, np.float32)).cuda()
    img1 = tr.render(th, fr, cams, bg).clone()
    keys, vals, ranges, tile_bits, tiles = tr.binner.result
    # two-level binning: 32-bit (frame, tile) keys, lists in depth order within a tile
    k = keys.cpu().numpy().view(np.uint32)
    assert k.size == tr.last_total and k.size > 1_000_000
    assert np.all(k[1:] >= k[:-1])
    # bit-exact against the oracle on the device's own fp32 projection
    rec = tr.records.view(B, dev.N, 12).cpu().numpy()
    rad = tr.radius.view(B, dev.N).cpu().numpy()
    res = BO.bin_batch(rec[..., 0:2], rad, tr.depth.view(B, dev.N).cpu().numpy(), rec[..., 5], rad > 0, 512, 512)
    assert np.array_equal(k.astype(np.uint64), res["keys"] >> np.uint64(32))
    assert np.array_equal(vals.cpu().numpy().view(np.uint32), res["values"])
    assert np.array_equal(ranges.view(B, -1, 2).cpu().numpy().view(np.uint32)[:, :tiles], res["ranges"])
    img2 = tr.render(th, fr, cams, bg)
    assert torch.equal(img1, img2)                      # forward is deterministic
    assert float(img1.min()) >= -1e-6 and float(img1.max()) <= 1.0 + 1e-5
    tg = torch.from_numpy(wl.targets).cuda()
    for _ in range(2):
        tr.step(th, tg, fr, cams, bg)
    r = tr.result()
    assert np.isfinite(r.loss) and 0.0 < r.loss < 1.0
    assert torch.isfinite(tr.grads).all()


def test_fused_raster_matches_separate_kernels():
    """hs_raster_train (forward + adjoint per pixel block) against hs_raster_fwd +
    hs_raster_bwd: identical losses and visited flags; gradients equal up to the
    order of the float atomics."""
    from paper_2503_12886_b200 import synth
    from paper_2503_12886_b200.device import AvatarParams, Trainer
    wl = synth.make_workload(64, 4, 192, distinct_frames=4)
    av = wl.avatar
    mk = lambda: AvatarParams.from_host(O.GSet(*(av.base[a] for a in ATTRS)), av.deltas, av.mlp, av.tri_index,
                                        av.barycentric)
    th = torch.from_numpy(np.asarray(wl.thetas, np.float32)).cuda()
    tg = torch.from_numpy(wl.targets).cuda()
    fr = torch.from_numpy(wl.frames).cuda()
    cams = torch.from_numpy(np.tile(wl.camera.packed(), (4, 1))).cuda()
    bg = torch.from_numpy(np.asarray(wl.backgrounds, np.float32)).cuda()
    a, b = Trainer(mk(), 192, 192, 4), Trainer(mk(), 192, 192, 4)
    b.fused_raster = False
    for step in range(3):
        la = a.step(th, tg, fr, cams, bg).clone()
        lb = b.step(th, tg, fr, cams, bg).clone()
        if step == 0:
            assert torch.equal(la, lb)
        else:
            assert torch.allclose(la, lb, rtol=1e-5, atol=1e-7)
        ga, gb = a.g_splat.cpu().numpy(), b.g_splat.cpu().numpy()
        assert np.linalg.norm(ga - gb) <= 1e-5 * np.linalg.norm(gb)
    assert torch.equal(a.visited, b.visited)


@pytest.mark.parametrize("crowded", [False, True])
def test_tile_binning_matches_two_level(crowded):
    """The training step with tile-major binning against the two-level global sort: the
    same lists, so the first step's losses are identical and the gradients equal up to
    the order of the float atomics.  crowded: Gaussians inflated until some (frame,
    tile) list exceeds hs_tile_sort_cap(), so the tile-major binner takes its
    two-level fallback inside the step."""
    from paper_2503_12886_b200 import synth
    from paper_2503_12886_b200.device import AvatarParams, Trainer, tile_sort_cap
    uv, size = (140, 64) if crowded else (64, 192)
    wl = synth.make_workload(uv, 4, size, distinct_frames=4)
    av = wl.avatar
    base = {a: np.array(av.base[a], copy=True) for a in ATTRS}
    if crowded:
        base["scale"] = base["scale"] + 3.0
    mk = lambda: AvatarParams.from_host(O.GSet(*(base[a] for a in ATTRS)), av.deltas, av.mlp, av.tri_index,
                                        av.barycentric)
    th = torch.from_numpy(np.asarray(wl.thetas, np.float32)).cuda()
    tg = torch.from_numpy(wl.targets).cuda()
    fr = torch.from_numpy(wl.frames).cuda()
    cams = torch.from_numpy(np.tile(wl.camera.packed(), (4, 1))).cuda()
    bg = torch.from_numpy(np.asarray(wl.backgrounds, np.float32)).cuda()
    a, b = Trainer(mk(), size, size, 4), Trainer(mk(), size, size, 4)
    b.tile_binning = False
    for step in range(2):
        la = a.step(th, tg, fr, cams, bg).clone()
        lb = b.step(th, tg, fr, cams, bg).clone()
        assert a.binner.mode == ("two_level" if crowded else "tiles"), a.binner.longest
        if crowded:
            assert a.binner.longest > tile_sort_cap()
        if step == 0:
            assert torch.equal(la, lb)
            ga, gb = a.g_splat.cpu().numpy(), b.g_splat.cpu().numpy()
            assert np.linalg.norm(ga - gb) <= 1e-5 * np.linalg.norm(gb)
        else:
            assert torch.allclose(la, lb, rtol=1e-4, atol=1e-7)
