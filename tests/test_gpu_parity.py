"""Parity of the sm_100a path (through the C ABI) against the float64 CPU oracle.

Protocol: inputs are quantized to fp32 and the oracle receives the
float64 upcast; each device stage is checked against the oracle fed the previous
device stage's fp32 outputs (compositing order from the device's fp32 depths,
integer pixel bbox from the device record).  Tolerances:
  * binning keys / values / ranges: bit-exact;
  * pixels, transmittance, max weight: max-abs <= 1e-4 outside pixels whose oracle
    decision margin is below fp32 resolution (|alpha - 1/255| < 2e-6 or
    |q - qmax| < 1e-4), which are counted and must be rare;
  * gradients: relative <= 1e-3 with an absolute floor of 1e-6 * max|g| per tensor.
"""
import numpy as np
import pytest
import torch

import binning as BO
import oracle as O
from conftest import golden

pytestmark = pytest.mark.gpu

ATTRS = ("position", "rotation", "scale", "opacity", "color")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2503_12886_b200 import build
    build.build()


def f32(a):
    return np.asarray(a, np.float32).astype(np.float64)


def gq(g):
    return O.GSet(*(f32(getattr(g, a)) for a in ATTRS))


def gset(d, prefix):
    return O.GSet(*(np.asarray(d[f"{prefix}.{a}"], dtype=np.float64) for a in ATTRS))


def cam_from(flat, w, h):
    flat = np.asarray(flat)
    return O.Cam(flat[12], flat[13], flat[14], flat[15], flat[:9].reshape(3, 3), flat[9:12], int(w), int(h))


def rel_err(a, b, floor_frac=1e-6):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    floor = floor_frac * max(np.abs(b).max(initial=0.0), 1e-30)
    diff = np.abs(a - b)
    scale = np.maximum(np.abs(a), np.abs(b))
    r = np.where(diff <= floor, 0.0, diff / np.maximum(scale, 1e-300))
    return float(r.max(initial=0.0))


def scenes():
    d = golden("render")
    for s in range(int(d["num_scenes"])):
        p = f"s{s}."
        w, h = d[p + "wh"]
        yield s, p, d, gq(gset(d, p + "world")), cam_from(d[p + "cam"], w, h)


def record_fields(dev, b=0):
    n = dev["N"]
    rec = dev["records"].view(-1, 12)[b * n:(b + 1) * n].cpu().numpy()
    bits = rec.view(np.uint32)
    lo = lambda v: (v & 0xFFFF).astype(np.int16).astype(np.int32)
    hi = lambda v: (v >> 16).astype(np.int16).astype(np.int32)
    bbox = np.stack([lo(bits[:, 7]), hi(bits[:, 7]), lo(bits[:, 8]), hi(bits[:, 8])], axis=-1)
    return rec, bbox


def flip_mask(splats, order, bbox, h, w):
    """Pixels where an oracle decision (alpha cutoff / qmax / alpha -> 1 / termination)
    is within fp32 noise (oracle.flip_mask)."""
    cam = type("Hw", (), {"height": h, "width": w})()
    return O.flip_mask(splats, cam, order=order, bbox=bbox)


def oracle_from_device(sp_dev, dev, world, cam):
    """Oracle ProjectedSplats built from the device's fp32 projection (stage-wise check)."""
    rec, bbox = record_fields(dev)
    idx = sp_dev.index
    osp = O.preprocess(world, cam)            # x_cam / cov_cam / world for the adjoint
    assert np.array_equal(osp.index, idx)
    osp.mean2d = f32(rec[idx, 0:2])
    osp.conic = f32(rec[idx, 2:5])
    osp.opacity = f32(rec[idx, 5])
    osp.color = f32(rec[idx, 9:12])
    osp.radius = f32(sp_dev.radius)
    order = np.argsort(np.asarray(sp_dev.depth, np.float32), kind="stable")
    return osp, order, bbox[idx]


# ------------------------------------------------------------------ projection

def test_project_matches_oracle():
    from paper_2503_12886_b200 import compat as C
    for s, p, d, world, cam in scenes():
        sp = C.preprocess(world, cam)
        ref = O.preprocess(world, cam)
        assert np.array_equal(sp.index, ref.index), s
        if len(ref) == 0:
            continue
        np.testing.assert_allclose(sp.mean2d, ref.mean2d, rtol=0, atol=2e-4 * max(cam.width, 1) / 16)
        np.testing.assert_allclose(sp.depth, ref.depth, rtol=2e-6)
        np.testing.assert_allclose(sp.radius, ref.radius, rtol=1e-4)
        cscale = np.abs(ref.conic).max(axis=1, keepdims=True)
        assert np.max(np.abs(sp.conic - ref.conic) / cscale) < 2e-4, s
        np.testing.assert_allclose(sp.x_cam, ref.x_cam, rtol=0, atol=2e-6)
        np.testing.assert_allclose(sp.cov_cam, ref.cov_cam, rtol=1e-4, atol=1e-7)


def test_preprocess_nonfinite_raises_with_index():
    from paper_2503_12886_b200 import compat as C
    _, _, d, world, cam = next(scenes())
    world.position[3, 1] = np.nan
    with pytest.raises(FloatingPointError, match="non-finite position at Gaussian index 3"):
        C.preprocess(world, cam)
    world.position[3, 1] = 0.0
    world.color[5, 0] = np.inf
    with pytest.raises(FloatingPointError, match="non-finite color at Gaussian index 5"):
        C.preprocess(world, cam)


# --------------------------------------------------------------------- binning

def check_two_level(dev, res, tag=""):
    """Two-level binning (depth order, then 32-bit (frame, tile) keys; the training
    path) on the same projection: the same lists and ranges as the oracle."""
    bn = dev["binner"]          # its depth range is the projection's
    bn.depth_order(dev["B"], dev["N"], dev["depth"])
    keys, vals, ranges, tile_bits, tiles = bn.bin(dev["B"], dev["N"], dev["W"], dev["H"], dev["records"],
                                                  dev["depth"], dev["counts"], dev["total"])
    k = keys.cpu().numpy().view(np.uint32).astype(np.uint64)
    assert np.array_equal(k, res["keys"] >> np.uint64(32)), tag
    assert np.array_equal(vals.cpu().numpy().view(np.uint32), res["values"]), tag
    r = ranges.view(-1, 2).cpu().numpy().view(np.uint32)[:res["ranges"].shape[1]]
    assert np.array_equal(r, res["ranges"][0]), tag

def check_tiles(dev, res, tag="", regrow=False):
    """Tile-major binning (count, scan, scatter, per-list sort; the training path) on
    the same projection: the same lists and ranges as the oracle.  regrow: start from
    a capacity of one key, so the device skips the fill and the host re-runs it."""
    import torch
    bn = dev["binner"]
    if regrow:
        bn._ensure(1)
        bn.cap = 1
    err = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    total, code = bn.bin_tiles(dev["B"], dev["N"], dev["W"], dev["H"], dev["records"], dev["depth"],
                               dev["counts"], err)
    assert total == res["keys"].size, tag
    keys, vals, ranges, tile_bits, tiles = bn.result
    k = keys.cpu().numpy().view(np.uint32).astype(np.uint64)
    assert np.array_equal(k, res["keys"] >> np.uint64(32)), tag
    assert np.array_equal(vals.cpu().numpy().view(np.uint32), res["values"]), tag
    r = ranges.view(-1, 2).cpu().numpy().view(np.uint32)[:res["ranges"].shape[1]]
    assert np.array_equal(r, res["ranges"][0]), tag
    return bn.mode


def test_binning_bit_exact():
    from paper_2503_12886_b200 import compat as C
    for s, p, d, world, cam in scenes():
        sp = C.preprocess(world, cam)
        dev = sp._dev["batch"]
        n = dev["N"]
        rec, bbox = record_fields(dev)
        rad = dev["radius"].cpu().numpy()[None]
        res = BO.bin_batch(rec[None, :, 0:2], rad, dev["depth"].cpu().numpy()[None], rec[None, :, 5],
                           rad > 0, cam.width, cam.height)
        keys, vals, ranges, tile_bits, tiles = dev["binned"]
        assert np.array_equal(keys.cpu().numpy().view(np.uint64), res["keys"]), s
        assert np.array_equal(vals.cpu().numpy().view(np.uint32), res["values"]), s
        r = ranges.view(-1, 2).cpu().numpy().view(np.uint32)[:res["ranges"].shape[1]]
        assert np.array_equal(r, res["ranges"][0]), s
        live = (rad[0] > 0) & (rec[:, 5] >= np.float32(1 / 255))
        np.testing.assert_array_equal(bbox[live], res["bbox"][0][live])
        check_two_level(dev, res, s)
        check_tiles(dev, res, s)
        check_tiles(dev, res, s, regrow=True)


@pytest.mark.parametrize("n", [200, 1000, 3000, 9000])
def test_binning_bit_exact_crowded_tiles(n):
    """One 16x16 tile holding 200 / 1000 / 3000 / 9000 splats with many exact depth ties
    (quantized positions): the stable sort must break ties by Gaussian index."""
    from paper_2503_12886_b200 import compat as C
    rng = np.random.default_rng(n)
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=-1, keepdims=True)
    pos = np.round(rng.uniform(-0.3, 0.3, (n, 3)) * 8) / 8          # few distinct depths -> ties
    world = O.GSet(pos, q, rng.uniform(0.02, 0.06, (n, 3)), rng.uniform(0.3, 0.9, n), rng.uniform(0, 1, (n, 3)))
    world = gq(world)
    cam = O.Cam(24.0, 24.0, 8.0, 8.0, np.eye(3), np.array([0.0, 0.0, 2.0]), 16, 16)
    sp = C.preprocess(world, cam)
    dev = sp._dev["batch"]
    rec, bbox = record_fields(dev)
    rad = dev["radius"].cpu().numpy()[None]
    res = BO.bin_batch(rec[None, :, 0:2], rad, dev["depth"].cpu().numpy()[None], rec[None, :, 5], rad > 0, 16, 16)
    keys, vals, ranges, tile_bits, tiles = dev["binned"]
    assert np.array_equal(keys.cpu().numpy().view(np.uint64), res["keys"])
    assert np.array_equal(vals.cpu().numpy().view(np.uint32), res["values"])
    r = ranges.view(-1, 2).cpu().numpy().view(np.uint32)[:res["ranges"].shape[1]]
    assert np.array_equal(r, res["ranges"][0])
    check_two_level(dev, res, n)
    # lists past the shared-memory sort's cap take the two-level fallback
    assert check_tiles(dev, res, n) == ("two_level" if n > 8192 else "tiles")
    # again with the same Binner: the previous batch had lists past the warp runs, so the
    # fill sorts them itself (HS_FILL_CTA_SORT, before the summary read), with and without
    # a capacity regrow
    assert check_tiles(dev, res, n) == ("two_level" if n > 8192 else "tiles")
    if 1024 < n <= 8192:
        assert dev["binner"].launches_extra == 1
    assert check_tiles(dev, res, n, regrow=True) == ("two_level" if n > 8192 else "tiles")


# --------------------------------------------------------------------- raster

def test_rasterize_matches_oracle():
    from paper_2503_12886_b200 import compat as C
    flips = 0
    for s, p, d, world, cam in scenes():
        bg = f32(d[p + "bg"])
        sp = C.preprocess(world, cam)
        image, aux = C.rasterize(sp, cam, bg)
        dev = sp._dev["batch"]
        if len(sp) == 0:
            assert np.array_equal(image, np.broadcast_to(np.float32(bg).astype(np.float64), image.shape))
            continue
        osp, order, bbox = oracle_from_device(sp, dev, world, cam)
        oimg, oaux = O.rasterize(osp, cam, bg, order=order, bbox=bbox)
        mask = flip_mask(osp, order, bbox, cam.height, cam.width)
        flips += int(mask.sum())
        ok = ~mask
        assert np.max(np.abs(image - oimg)[ok]) <= 1e-4, s
        assert np.max(np.abs(aux.transmittance - oaux.transmittance)[ok]) <= 1e-4, s
        assert np.array_equal(aux.stop[ok], oaux.stop[ok]), s
        mw_ok = np.ones(world.count, bool)
        if mask.any():
            mw_ok[:] = False                      # only compare max weights when no pixel is ambiguous
        np.testing.assert_allclose(aux.max_weight[mw_ok], oaux.max_weight[mw_ok], rtol=1e-4, atol=1e-6)
    assert flips <= 3


def _touching(splats, bbox, mask):
    """Per kept splat: does a masked pixel lie inside its integer bbox and its
    alpha >= 1/255 ellipse (q <= qmax, plus a margin)?"""
    out = np.zeros(len(bbox), bool)
    if not mask.any():
        return out
    ys, xs = np.nonzero(mask)
    for s, (r0, r1, c0, c1) in enumerate(bbox):
        inb = (ys >= r0) & (ys <= r1) & (xs >= c0) & (xs <= c1)
        if not inb.any():
            continue
        dx = xs[inb] + 0.5 - splats.mean2d[s, 0]
        dy = ys[inb] + 0.5 - splats.mean2d[s, 1]
        a, b, c = splats.conic[s]
        q = a * dx * dx + 2 * b * dx * dy + c * dy * dy
        out[s] = np.any(q <= 2.0 * np.log(splats.opacity[s] * 255.0) + 1e-3)
    return out


def test_weight_sums_and_estimate_colors():
    """Every non-empty scene is compared; splats whose bbox holds a flip-masked pixel
    are excluded (their weight sums legitimately differ by one alpha ~ 1/255 term) and
    counted."""
    from paper_2503_12886_b200 import compat as C
    compared = excluded = scenes_done = 0
    for s, p, d, world, cam in scenes():
        sp = C.preprocess(world, cam)
        if len(sp) == 0:
            continue
        bg = f32(d[p + "bg"])
        _, aux = C.rasterize(sp, cam, bg)
        target = f32(d[p + "target"])
        num, den = C.splat_weight_sums(aux, target)
        osp, order, bbox = oracle_from_device(sp, sp._dev["batch"], world, cam)
        _, oaux = O.rasterize(osp, cam, bg, order=order, bbox=bbox)
        onum, oden = O.splat_weight_sums(oaux, target)
        mask = flip_mask(osp, order, bbox, cam.height, cam.width)
        keep = np.ones(world.count, bool)
        keep[osp.index[_touching(osp, bbox, mask)]] = False
        compared += int(keep[osp.index].sum())
        excluded += int((~keep[osp.index]).sum())
        scenes_done += 1
        np.testing.assert_allclose(den[keep], oden[keep], rtol=1e-4, atol=1e-5)
        np.testing.assert_allclose(num[keep], onum[keep], rtol=1e-4, atol=1e-5)
        est, eligible = C.estimate_colors(aux, target, 0.1)
        oest, oelig = O.estimate_colors(oaux, target, 0.1)
        assert np.array_equal(eligible[keep], oelig[keep])
        e = eligible & keep
        np.testing.assert_allclose(est[e], oest[e], rtol=1e-4, atol=1e-5)
    print(f"weight sums: {scenes_done} scenes, {compared} splats compared, {excluded} excluded")
    assert scenes_done >= 5
    assert excluded <= 0.25 * compared


def test_render_backward_matches_oracle():
    """Every non-empty scene: the image gradient is zeroed on the flip-masked pixels on
    both sides, so every gradient entry is compared (rel 1e-3, floor 1e-6 max|g|)."""
    from paper_2503_12886_b200 import compat as C
    scenes_done = masked = 0
    for s, p, d, world, cam in scenes():
        sp = C.preprocess(world, cam)
        if len(sp) == 0:
            continue
        bg = f32(d[p + "bg"])
        _, aux = C.rasterize(sp, cam, bg)
        osp, order, bbox = oracle_from_device(sp, sp._dev["batch"], world, cam)
        mask = flip_mask(osp, order, bbox, cam.height, cam.width)
        masked += int(mask.sum())
        gimg = f32(d[p + "grad_image"]) * ~mask[:, :, None]
        _, oaux = O.rasterize(osp, cam, bg, order=order, bbox=bbox)
        # splat-space adjoint (S/render.py:276-336)
        gs = C.splat_space_grads(aux, gimg)[sp.index]
        om, oc, oo, ocol = O.splat_space_grads(osp, oaux, gimg)
        assert rel_err(gs[:, 0:2], om) < 1e-3, s
        assert rel_err(gs[:, 2:5], oc) < 1e-3, s
        assert rel_err(gs[:, 5], oo) < 1e-3, s
        assert rel_err(gs[:, 6:9], ocol) < 1e-3, s
        # full world-space adjoint (+ S/render.py:432-497)
        g = C.render_backward(sp, aux, gimg)
        og = O.render_backward(osp, oaux, gimg)
        for a in ATTRS:
            assert rel_err(getattr(g, a), getattr(og, a)) < 1e-3, (s, a, rel_err(getattr(g, a), getattr(og, a)))
        scenes_done += 1
    print(f"render backward: {scenes_done} scenes, {masked} masked pixels")
    assert scenes_done >= 5


# ---------------------------------------------------------------- model ops

def test_blend_activate_transform_match_oracle():
    from paper_2503_12886_b200 import compat as C
    d = golden("model")

    class M:
        pass
    m = M()
    m.base = gq(gset(d, "base"))
    n = m.base.count
    dl = f32(d["deltas"])
    m.deltas = [type("D", (), {"position": x[:3 * n].reshape(n, 3), "rotation": x[3 * n:7 * n].reshape(n, 4),
                               "color": x[7 * n:].reshape(n, 3)})() for x in dl]
    om = O.Model(m.base, dl, {}, None, None)
    psi = f32(d["psi"])
    raw = C.blend(m, psi)
    oraw = O.blend(om, psi)
    for a in ("position", "rotation", "color"):
        np.testing.assert_allclose(getattr(raw, a), getattr(oraw, a), rtol=1e-6, atol=1e-6)
    # basis recovery is bitwise against an fp32 restatement (T/test_model.py:103-113)
    unit = np.zeros(len(m.deltas))
    unit[2] = 1.0
    rb = C.blend(m, unit)
    exp = np.float32(m.base.position) + np.float32(m.deltas[2].position)
    assert np.array_equal(np.float32(rb.position), exp)
    act = C.activate(raw)
    oact = O.activate(gq(raw))
    for a in ATTRS:
        np.testing.assert_allclose(getattr(act, a), getattr(oact, a), rtol=2e-6, atol=1e-6)
    g_act = gq(gset(d, "g_act"))
    g_raw = C.activate_backward(raw, act, g_act)
    og_raw = O.activate_backward(gq(raw), gq(act), g_act)
    for a in ATTRS:
        assert rel_err(getattr(g_raw, a), getattr(og_raw, a)) < 1e-4, a
    gb, gdel, gpsi = C.blend_backward(m, psi, g_raw)
    ogb, ogd, ogpsi = O.blend_backward(om, psi, gq(g_raw))
    assert rel_err(gpsi, ogpsi) < 1e-4
    assert rel_err(np.stack([np.concatenate([x.position.ravel(), x.rotation.ravel(), x.color.ravel()]) for x in gdel]),
                   ogd) < 1e-5


def test_zero_quaternion_raises():
    from paper_2503_12886_b200 import compat as C
    n = 6
    raw = O.GSet(np.zeros((n, 3)), np.tile([1.0, 0, 0, 0], (n, 1)), np.zeros((n, 3)), np.zeros(n), np.zeros((n, 3)))
    raw.rotation[4] = 0.0
    with pytest.raises(FloatingPointError, match="zero-norm quaternion at Gaussian index 4"):
        C.activate(raw)


def test_transform_matches_oracle():
    from paper_2503_12886_b200 import compat as C
    d = golden("binding")
    frames = O.Frames(f32(d["frames.rotation"]), f32(d["frames.quat"]), f32(d["frames.tri_vertices"]))
    tangent = gq(gset(d, "tangent"))

    class Bd:
        triangle_index = d["tri_index"]
        barycentric = f32(d["barycentric"])
    w = C.transform_to_deformed(tangent, frames, Bd)
    ow = O.transform_to_deformed(tangent, frames, d["tri_index"], Bd.barycentric)
    for a in ATTRS:
        np.testing.assert_allclose(getattr(w, a), getattr(ow, a), rtol=1e-5, atol=2e-6)
    gw = gq(gset(d, "g_world"))
    g = C.transform_backward(tangent, frames, Bd, gw)
    og = O.transform_backward(tangent, frames, d["tri_index"], gw)
    for a in ATTRS:
        assert rel_err(getattr(g, a), getattr(og, a)) < 1e-4, a
