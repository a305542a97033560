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
from gpu_helpers import normwise, rel_fail, replay_from_trainer

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


def masked_step_parity(wl, B, W, H, cam_packed=None, targets=None, workers=8):
    """One unfused device step with the MaskedReplay hook against the oracle's
    train_step replaying the device's order, bbox, L1 signs and flip mask.
    Returns (hook report, {tensor: (failing entries, worst rel err)}, device trainer)."""
    from paper_2503_12886_b200.device import AvatarParams, Trainer
    from gpu_helpers import MaskedReplay, rel_fail
    av = wl.avatar
    dev = AvatarParams.from_host(O.GSet(*(av.base[a] for a in ATTRS)), av.deltas, av.mlp, av.tri_index,
                                 av.barycentric)
    tr = Trainer(dev, W, H, B)
    tr.fused_raster = False
    tr.radius = torch.empty(B * dev.N, device="cuda")
    cp = wl.camera.packed() if cam_packed is None else cam_packed
    targets = wl.targets if targets is None else targets
    cams = np.tile(cp, (B, 1))
    bgs = np.asarray(wl.backgrounds, np.float32).astype(np.float64)
    model = _oracle_model(wl)
    p = np.asarray(cp, np.float64)
    cam = O.Cam(p[12], p[13], p[14], p[15], p[:9].reshape(3, 3), p[9:12], W, H)
    frames = [O.Frames(f[:, :9].reshape(-1, 3, 3).astype(np.float64), f[:, 9:13].astype(np.float64),
                       f[:, 13:].reshape(-1, 3, 3).astype(np.float64)) for f in wl.frames]
    th = np.asarray(wl.thetas, np.float32).astype(np.float64)
    hook = MaskedReplay(O, model, cam, th, frames, targets, bgs)
    tr.debug_before_backward = hook
    res = tr.step_from_host(wl.thetas, targets, wl.frames, cams, bgs)
    torch.cuda.synchronize()
    state = O.State(model, cam, workers=workers)
    loss, black = O.train_step(state, th, targets.astype(np.float64) / 255.0, frames, bgs, replay=hook.replay)
    state.close()
    tr._oracle_state = state
    rep = dict(hook.report)
    rep["loss_dev"], rep["loss_oracle"] = res.loss, loss
    rep["black_maxabs"] = float(np.abs(res.black_l1 - black).max())
    g_base, g_deltas, g_mlp = state.last_grads
    gb, gd, gm = split_grads(tr.grads.cpu().numpy(), dev.N, dev.K, dev.H, dev.D)
    errs = {}
    for a in ATTRS:
        # rotation: the exact gradient of isotropic Gaussians is 0 and both sides hold
        # only roundoff, so its floor is taken from the position gradient
        errs[a] = rel_fail(gb[a], getattr(g_base, a), scale=np.abs(g_base.position).max() if a == "rotation" else None)
    errs["deltas"] = rel_fail(gd, g_deltas)
    for k in gm:
        errs["mlp." + k] = rel_fail(gm[k], g_mlp[k])
    return rep, errs, tr


def check_masked_parity(rep, errs, tag):
    print(tag, "masked replay:", rep)
    print(tag, "gradient (failing entries, worst rel):", errs)
    # the device's L1 signs differ from float64 only where |pred - target| is fp32 noise
    assert rep["sign_flip_max_absdiff"] <= 2e-6, rep
    assert rep["t_maxabs"] <= 1e-4, rep
    assert rep["masked"] <= 1e-2 * rep["pixels"], rep
    assert abs(rep["loss_dev"] - rep["loss_oracle"]) < 1e-4 * max(rep["loss_oracle"], 1e-3), rep
    assert rep["black_maxabs"] < 1e-5, rep
    bad = {k: v for k, v in errs.items() if v[0] != 0}
    assert not bad, bad


def test_c1_step_vs_oracle():
    """BASELINE configs[0]: every gradient entry within rel 1e-3 (floor 1e-6 max|g|)."""
    from bench_support import synth
    wl = synth.make_workload(141, 4, 256)
    rep, errs, _ = masked_step_parity(wl, 4, 256, 256)
    check_masked_parity(rep, errs, "C1")


def test_c2_step_vs_oracle():
    """BASELINE configs[1] (the bench workload: 50,176 Gaussians, 16 x 512^2), one step,
    stage-exact replay, every gradient entry within rel 1e-3."""
    import os
    from bench_support import synth
    wl = synth.make_workload(224, 16, 512)
    rep, errs, _ = masked_step_parity(wl, 16, 512, 512, workers=min(16, os.cpu_count() or 1))
    check_masked_parity(rep, errs, "C2")


def test_c1_blend_mlp_stagewise():
    """blend_bwd + mlp_bwd fed the device's own per-frame g_raw (C1 sizes)."""
    from bench_support import synth
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
    from bench_support import synth
    from paper_2503_12886_b200.device import AvatarParams, Trainer
    wl = synth.make_workload(224, 16, 512, distinct_frames=4)
    av = wl.avatar
    dev = AvatarParams.from_host(O.GSet(*(av.base[a] for a in ATTRS)), av.deltas, av.mlp, av.tri_index,
                                 av.barycentric)
    assert dev.N == 50176
    B = 16
    tr = Trainer(dev, 512, 512, B)
    tr.radius = torch.empty(B * dev.N, device="cuda")
    tr.binner.write_keys = True                  # (the step itself does not need the keys)
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
    # (the projection had tile_rects: the binner's exact tile cull is on, so is the oracle's)
    res = BO.bin_batch(rec[..., 0:2], rad, tr.depth.view(B, dev.N).cpu().numpy(), rec[..., 5], rad > 0, 512, 512,
                       conic=rec[..., 2:5], qmax=rec[..., 6])
    full = BO.bin_batch(rec[..., 0:2], rad, tr.depth.view(B, dev.N).cpu().numpy(), rec[..., 5], rad > 0, 512, 512)
    assert 0.6 * full["keys"].size < k.size < 0.95 * full["keys"].size
    assert np.array_equal(k.astype(np.uint64), res["keys"] >> np.uint64(32))
    assert np.array_equal(vals.cpu().numpy().view(np.uint32), res["values"])
    assert np.array_equal(ranges.view(B, -1, 2).cpu().numpy().view(np.uint32)[:, :tiles], res["ranges"])
    # the render raster (no per-pixel state: no stop index, no pix_T / pix_state writes)
    # against the stateful forward on the same lists: the same image bitwise
    import ctypes
    from paper_2503_12886_b200 import _lib as L
    from paper_2503_12886_b200.device import _p
    img_s = torch.empty_like(img1)
    pix_T = torch.empty(B * 512 * 512, device="cuda")
    pix_state = torch.empty(B * 512 * 512, dtype=torch.int32, device="cuda")
    L.call("hs_raster_fwd", B, dev.N, 512, 512, L.RASTER_IMAGE, _p(tr.records), _p(vals), _p(ranges), tile_bits,
           _p(bg), None, None, None, _p(pix_T), _p(pix_state), _p(img_s), None, None, None, None, _p(tr.raster_ws),
           ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    assert torch.equal(img1, img_s)
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
    from bench_support import synth
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
        # (from the second step on the parameters already differ by the first step's
        # summation-order noise, which Adam's normalisation amplifies)
        assert np.linalg.norm(ga - gb) <= (1e-5 if step == 0 else 5e-5) * np.linalg.norm(gb)
    assert torch.equal(a.visited, b.visited)


@pytest.mark.parametrize("crowded", [False, True])
def test_tile_binning_matches_two_level(crowded):
    """The training step with tile-major binning against the two-level global sort: the
    same lists, so the first step's losses are identical and the gradients equal up to
    the order of the float atomics.  crowded: Gaussians inflated until some (frame,
    tile) list exceeds hs_tile_sort_cap(), so the tile-major binner takes its
    two-level fallback inside the step."""
    from bench_support import synth
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


def test_fused_raster_pixels_and_grads_c2():
    """The hot-path kernel (hs_raster_train, forward + adjoint per pixel block) at C2:
    its per-pixel transmittance and state words (stop index + L1 signs) are bitwise
    those of the separate forward kernel, and its splat gradients agree with the
    separate adjoint entrywise (rel 1e-4, floor 1e-6 max|g|: float-atomic order only).
    With test_c2_step_vs_oracle (separate kernels vs the oracle) this pins the fused
    kernel to the oracle."""
    from bench_support import synth
    from paper_2503_12886_b200.device import AvatarParams, Trainer
    wl = synth.make_workload(224, 16, 512)
    av = wl.avatar
    mk = lambda: AvatarParams.from_host(O.GSet(*(av.base[a] for a in ATTRS)), av.deltas, av.mlp, av.tri_index,
                                        av.barycentric)
    B = 16
    th = torch.from_numpy(np.asarray(wl.thetas, np.float32)).cuda()
    tg = torch.from_numpy(wl.targets).cuda()
    fr = torch.from_numpy(wl.frames).cuda()
    cams = torch.from_numpy(np.tile(wl.camera.packed(), (B, 1))).cuda()
    bg = torch.from_numpy(np.asarray(wl.backgrounds, np.float32)).cuda()
    a, b = Trainer(mk(), 512, 512, B), Trainer(mk(), 512, 512, B)
    a.capture_pixels = True
    b.fused_raster = False
    la = a.step(th, tg, fr, cams, bg).clone()
    lb = b.step(th, tg, fr, cams, bg).clone()
    torch.cuda.synchronize()
    assert torch.equal(la, lb)
    assert torch.equal(a.pix_T, b.pix_T)
    assert torch.equal(a.pix_state, b.pix_state)
    nbad, worst, _ = rel_fail(a.g_splat.cpu().numpy(), b.g_splat.cpu().numpy(), rtol=1e-4)
    assert nbad == 0, worst
    nbad, worst, _ = rel_fail(a.grads.cpu().numpy()[:14 * a.av.N], b.grads.cpu().numpy()[:14 * a.av.N], rtol=1e-4)
    assert nbad == 0, worst


def test_c3_binning_bit_exact():
    """The render's tile-major binning at the C3 Gaussian count (100,489, 16 frames at 512^2:
    lists of ~300 entries, thousands of 257..1,024 (the long-list sort), a few past 1,024
    (the CTA sort, enqueued inside the fill on the second batch)): keys, values and ranges
    bit-exact against the oracle, on both batches."""
    from bench_support import synth
    from paper_2503_12886_b200.device import AvatarParams, Trainer
    B = 16
    wl = synth.make_workload(317, B, 512, distinct_frames=B)
    av = wl.avatar
    dev = AvatarParams.from_host(O.GSet(*(av.base[a] for a in ATTRS)), av.deltas, av.mlp, av.tri_index,
                                 av.barycentric)
    tr = Trainer(dev, 512, 512, B)
    tr.radius = torch.empty(B * dev.N, device="cuda")
    tr.binner.write_keys = True
    th = torch.from_numpy(np.asarray(wl.thetas, np.float32)).cuda()
    fr = torch.from_numpy(wl.frames).cuda()
    cams = torch.from_numpy(np.tile(wl.camera.packed(), (B, 1))).cuda()
    bg = torch.zeros(B, 3, device="cuda")
    for rep in range(2):
        tr.render(th, fr, cams, bg)
        torch.cuda.synchronize()
        assert tr.binner.mode == "tiles"
        keys, vals, ranges, tile_bits, tiles = tr.binner.result
        rec = tr.records.view(B, dev.N, 12).cpu().numpy()
        rad = tr.radius.view(B, dev.N).cpu().numpy()
        res = BO.bin_batch(rec[..., 0:2], rad, tr.depth.view(B, dev.N).cpu().numpy(), rec[..., 5], rad > 0, 512,
                           512, conic=rec[..., 2:5], qmax=rec[..., 6])
        r = ranges.view(B, -1, 2).cpu().numpy().view(np.uint32)[:, :tiles]
        ln = (r[..., 1] - r[..., 0]).ravel()
        if rep == 0:
            assert ((ln > 256) & (ln <= 512)).sum() > 1000 and (ln > 512).sum() > 100, np.bincount(ln // 256)
        assert np.array_equal(keys.cpu().numpy().view(np.uint32).astype(np.uint64), res["keys"] >> np.uint64(32))
        assert np.array_equal(vals.cpu().numpy().view(np.uint32), res["values"])
        assert np.array_equal(r, res["ranges"])


def test_c3_render_vs_oracle():
    """BASELINE configs[2] (100,489 Gaussians, 64 frames at 512^2): the render kernel's
    images against the oracle's own float64 forward (map_params -> blend -> activate
    -> transform -> project -> composite) in the device's order and bbox, on 4 of the
    64 frames: max-abs 1e-4 outside the flip-masked pixels."""
    from bench_support import synth
    from paper_2503_12886_b200.device import AvatarParams, Trainer
    B = 64
    wl = synth.make_workload(317, B, 512, distinct_frames=B)
    av = wl.avatar
    dev = AvatarParams.from_host(O.GSet(*(av.base[a] for a in ATTRS)), av.deltas, av.mlp, av.tri_index,
                                 av.barycentric)
    assert dev.N == 100489
    tr = Trainer(dev, 512, 512, B)
    tr.radius = torch.empty(B * dev.N, device="cuda")
    th = torch.from_numpy(np.asarray(wl.thetas, np.float32)).cuda()
    fr = torch.from_numpy(wl.frames).cuda()
    cams = torch.from_numpy(np.tile(wl.camera.packed(), (B, 1))).cuda()
    bgs = np.asarray(wl.backgrounds, np.float32)
    img = tr.render(th, fr, cams, torch.from_numpy(bgs).cuda()).cpu().numpy()
    assert np.isfinite(img).all()
    replay = replay_from_trainer(tr)
    rec = tr.records.view(B, dev.N, 12).cpu().numpy().astype(np.float64)
    rad = tr.radius.view(B, dev.N).cpu().numpy().astype(np.float64)
    model = _oracle_model(wl)
    p = wl.camera.packed().astype(np.float64)
    cam = O.Cam(p[12], p[13], p[14], p[15], p[:9].reshape(3, 3), p[9:12], 512, 512)
    masked = 0
    for b in (0, 21, 42, 63):
        f = wl.frames[b]
        frames = O.Frames(f[:, :9].reshape(-1, 3, 3).astype(np.float64), f[:, 9:13].astype(np.float64),
                          f[:, 13:].reshape(-1, 3, 3).astype(np.float64))
        world, _ = O.frame_forward(model, np.asarray(wl.thetas[b], np.float32).astype(np.float64), frames)
        sp = O.preprocess(world, cam)
        r = replay[b]
        assert np.array_equal(sp.index, r["index"])
        oimg, _ = O.rasterize(sp, cam, bgs[b].astype(np.float64), order=r["order"], bbox=r["bbox"])
        mask = O.flip_mask(sp, cam, order=r["order"], bbox=r["bbox"]).astype(np.uint8)
        i = r["index"]
        sp.mean2d, sp.conic = rec[b, i, 0:2].copy(), rec[b, i, 2:5].copy()
        sp.opacity, sp.radius = rec[b, i, 5].copy(), rad[b, i].copy()
        O.flip_mask(sp, cam, order=r["order"], bbox=r["bbox"], out=mask)
        ok = mask == 0
        masked += int(mask.sum())
        err = np.abs(img[b] - oimg)[ok].max()
        print(f"C3 frame {b}: max-abs {err:.2e}, masked {int(mask.sum())} of {mask.size}")
        assert err <= 1e-4, (b, err)
    assert masked <= 1e-2 * 4 * 512 * 512


@pytest.mark.parametrize("case", ["valid", "regrow", "crowded"])
def test_speculative_raster(case):
    """The fused raster enqueued before the step's host sync (hs_raster_guard_t): when the
    lists are complete it is the step's raster (spec_valid); when the fill was skipped
    (buffers too small: regrow) or a list needs the CTA / two-level sorts (crowded), it
    exits on the device and the re-launch gives the same result as a non-speculative
    step (deterministic mode: bitwise)."""
    from bench_support import synth
    from paper_2503_12886_b200.device import AvatarParams, Trainer
    uv, size = (140, 64) if case == "crowded" else (64, 192)
    wl = synth.make_workload(uv, 4, size)
    av = wl.avatar
    base = {a: np.array(av.base[a], copy=True) for a in ATTRS}
    if case == "crowded":
        base["scale"] = base["scale"] + 2.0
    mk = lambda: Trainer(AvatarParams.from_host(O.GSet(*(base[a] for a in ATTRS)), av.deltas, av.mlp,
                                                av.tri_index, av.barycentric), size, size, 4, deterministic=True)
    th = torch.from_numpy(np.asarray(wl.thetas, np.float32)).cuda()
    tg = torch.from_numpy(wl.targets).cuda()
    fr = torch.from_numpy(wl.frames).cuda()
    cams = torch.from_numpy(np.tile(wl.camera.packed(), (4, 1))).cuda()
    bg = torch.from_numpy(np.asarray(wl.backgrounds, np.float32)).cuda()
    a, b = mk(), mk()
    b.speculative = False
    for step in range(2):
        if case == "regrow" and step == 0:
            a.binner._ensure(1)
            a.binner.cap = 1
        la = a.step(th, tg, fr, cams, bg).clone()
        lb = b.step(th, tg, fr, cams, bg).clone()
        torch.cuda.synchronize()
        if case == "valid" or step == 1 and case == "regrow":
            assert a.binner.spec_valid
        elif step == 0:
            assert not a.binner.spec_valid, (case, a.binner.longest)
        assert torch.equal(la, lb)
        assert torch.equal(a.grads, b.grads)
    assert torch.equal(a.av.params, b.av.params)
