"""The bit-exact binning oracle (oracle/binning.py) against the reference's compositing
order: for every pixel, the splats listed in its tile range that cover it (bbox test),
in list order, are exactly the reference's depth-ordered covering splats
(S/render.py:221-223 stable depth argsort + :248-251 pixel bbox)."""
import numpy as np
import pytest

import binning as BO
from conftest import golden


def _scene(d, s):
    p = f"s{s}."
    w, h = (int(x) for x in d[p + "wh"])
    idx = d[p + "splats.index"]
    n = d[p + "world.position"].shape[0]
    mean = np.zeros((1, n, 2), np.float32)
    rad = np.zeros((1, n), np.float32)
    dep = np.ones((1, n), np.float32)
    op = np.zeros((1, n), np.float32)
    valid = np.zeros((1, n), bool)
    mean[0, idx] = d[p + "splats.mean2d"]
    rad[0, idx] = d[p + "splats.radius"]
    dep[0, idx] = d[p + "splats.depth"]
    op[0] = d[p + "world.opacity"]
    valid[0, idx] = True
    return w, h, mean, rad, dep, op, valid


@pytest.mark.parametrize("s", range(6))
def test_tile_lists_reproduce_reference_order(s):
    d = golden("render")
    w, h, mean, rad, dep, op, valid = _scene(d, s)
    res = BO.bin_batch(mean, rad, dep, op, valid, w, h)
    assert BO.lexsort_check(res, dep)
    bbox = res["bbox"][0]
    live = valid[0] & (op[0] >= BO.ALPHA_CUTOFF_F32)
    # reference order from float32 depths (stable, ties to lower index)
    order = np.argsort(dep[0], kind="stable")
    tiles_x = res["tiles_x"]
    for py in range(h):
        for px in range(w):
            cover = lambda n: (bbox[n, 0] <= py <= bbox[n, 1]) and (bbox[n, 2] <= px <= bbox[n, 3])
            expect = [n for n in order if live[n] and cover(n)]
            t = (py // 16) * tiles_x + px // 16
            lo, hi = res["ranges"][0, t]
            got = [int(n) for n in res["values"][lo:hi] if cover(n)]
            assert got == expect, (py, px)


def test_float32_bbox_matches_reference_rule_when_exact():
    # values exactly representable in fp32: fp32 and fp64 bbox agree (S/render.py:248-251)
    mean = np.array([[[10.25, 7.5], [0.0, 3.0], [31.75, 31.75]]], np.float32)
    rad = np.array([[2.5, 4.0, 1.25]], np.float32)
    bb = BO.pixel_bbox(mean, rad, 32, 32)[0]
    import math
    for n in range(3):
        mx, my, r = (float(mean[0, n, 0]), float(mean[0, n, 1]), float(rad[0, n]))
        exp = [max(0, math.ceil(my - r - 0.5)), min(31, math.floor(my + r - 0.5)),
               max(0, math.ceil(mx - r - 0.5)), min(31, math.floor(mx + r - 0.5))]
        assert list(bb[n]) == exp


def test_batch_keys_sorted_by_frame_then_tile():
    rng = np.random.default_rng(0)
    B, N, W, H = 3, 200, 48, 40
    mean = rng.uniform(-5, 53, (B, N, 2)).astype(np.float32)
    rad = rng.uniform(0.3, 9, (B, N)).astype(np.float32)
    dep = rng.choice(np.float32([0.5, 1.0, 1.5, 2.0]), (B, N))      # many exact depth ties
    op = rng.uniform(0, 1, (B, N)).astype(np.float32)
    valid = rng.uniform(size=(B, N)) > 0.1
    res = BO.bin_batch(mean, rad, dep, op, valid, W, H)
    assert BO.lexsort_check(res, dep)
    assert np.all(np.diff(res["keys"].astype(np.float64)) >= 0)
    # empty tiles have [0, 0)
    r = res["ranges"].reshape(-1, 2)
    assert np.all((r[:, 1] > r[:, 0]) | ((r[:, 0] == 0) & (r[:, 1] == 0)))


@pytest.mark.parametrize("seed", range(4))
def test_tile_cull_keeps_every_pixel_that_can_composite(seed):
    """The tile cull (conic + qmax given) only drops (splat, tile) keys where no pixel of
    the tile passes the reference's bbox and q <= qmax tests (S/render.py:248-262, q at
    the pixel centre in float64): for every pixel, the splats of its tile list that pass
    both tests are exactly those of the unculled list, in the same order -- and the cull
    does drop keys (elongated, rotated ellipses in large bboxes)."""
    rng = np.random.default_rng(seed)
    W = H = 96
    n = 300
    mean = rng.uniform(-8, W + 8, (1, n, 2)).astype(np.float32)
    s1, s2 = rng.uniform(0.5, 9, n), rng.uniform(0.5, 3, n)
    th = rng.uniform(0, np.pi, n)
    c, s_ = np.cos(th), np.sin(th)
    cov = np.stack([c * c * s1 ** 2 + s_ * s_ * s2 ** 2, c * s_ * (s1 ** 2 - s2 ** 2), s_ * s_ * s1 ** 2 + c * c * s2 ** 2])
    det = cov[0] * cov[2] - cov[1] ** 2
    conic = np.stack([cov[2] / det, -cov[1] / det, cov[0] / det], -1)[None].astype(np.float32)
    rad = (3 * np.sqrt(np.maximum(cov[0], cov[2]) + np.abs(cov[1])))[None].astype(np.float32)
    op = rng.uniform(0.02, 1.0, (1, n)).astype(np.float32)
    qmax = (2 * np.log(op * 255.0) + 1e-9).astype(np.float32)
    dep = rng.uniform(1, 4, (1, n)).astype(np.float32)
    valid = np.ones((1, n), bool)
    full = BO.bin_batch(mean, rad, dep, op, valid, W, H)
    cull = BO.bin_batch(mean, rad, dep, op, valid, W, H, conic=conic, qmax=qmax)
    assert BO.lexsort_check(cull, dep)
    assert 0 < cull["keys"].size < 0.9 * full["keys"].size
    bbox = full["bbox"][0]
    tiles_x = full["tiles_x"]
    m64, k64, q64 = mean[0].astype(np.float64), conic[0].astype(np.float64), qmax[0].astype(np.float64)
    for py in range(H):
        for px in range(W):
            t = (py // 16) * tiles_x + px // 16

            def passing(res):
                lo, hi = res["ranges"][0, t]
                out = []
                for v in res["values"][lo:hi]:
                    if not (bbox[v, 0] <= py <= bbox[v, 1] and bbox[v, 2] <= px <= bbox[v, 3]):
                        continue
                    dx, dy = px + 0.5 - m64[v, 0], py + 0.5 - m64[v, 1]
                    q = k64[v, 0] * dx * dx + 2 * k64[v, 1] * dx * dy + k64[v, 2] * dy * dy
                    if q <= q64[v]:
                        out.append(int(v))
                return out
            assert passing(cull) == passing(full), (py, px)
