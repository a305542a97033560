"""Pin the float64 CPU oracle to the reference package.

Every fixture under tests/golden/ was produced by running the reference itself
(tests/golden/make_golden.py).  These tests run on CPU (no GPU marker) and are
the reason the oracle may be used as the parity checker for the device path.
"""
import numpy as np
import pytest

import oracle as O
from conftest import golden

ATTRS = ("position", "rotation", "scale", "opacity", "color")


def gset(d, prefix):
    return O.GSet(*(np.asarray(d[f"{prefix}.{a}"], dtype=np.float64) for a in ATTRS))


def close(a, b, rtol=1e-12, atol=1e-12):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    assert a.shape == b.shape, (a.shape, b.shape)
    np.testing.assert_allclose(a, b, rtol=rtol, atol=atol)


def cam_from(flat, w, h):
    flat = np.asarray(flat)
    return O.Cam(flat[12], flat[13], flat[14], flat[15], flat[:9].reshape(3, 3), flat[9:12], int(w), int(h))


# ----------------------------------------------------------------- model ops

def _model(d):
    mlp = {k: d["mlp." + k] for k in ("w1", "b1", "w2", "b2", "w3", "b3")}
    n = d["base.position"].shape[0]
    return O.Model(gset(d, "base"), d["deltas"], mlp, np.zeros(n, np.int64), np.tile([1.0, 0, 0], (n, 1)))


def test_map_params_and_mlp_backward():
    d = golden("model")
    model = _model(d)
    psi, cache = O.map_params(model.mlp, d["theta"])
    close(psi, d["psi_mlp"], rtol=1e-12, atol=1e-12)
    g = O.mlp_backward(model.mlp, cache, d["g_psi"])
    for k in g:
        close(g[k], d["gmlp." + k], rtol=1e-10, atol=1e-12)


def test_map_params_rejects_nonfinite():
    d = golden("model")
    theta = d["theta"].copy()
    theta[3] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        O.map_params(_model(d).mlp, theta)


def test_blend_bitwise_and_basis_recovery():
    d = golden("model")
    model = _model(d)
    raw = O.blend(model, d["psi"])
    for a in ("position", "rotation", "color"):
        assert np.array_equal(getattr(raw, a), d["raw." + a]), a      # same op order -> bitwise
    unit = np.zeros(model.K)
    unit[2] = 1.0
    assert np.array_equal(O.blend(model, unit).position, d["unit_blend.position"])


def test_activate_and_backward():
    d = golden("model")
    raw = gset(d, "raw")
    act = O.activate(raw)
    for a in ATTRS:
        close(getattr(act, a), d["act." + a], rtol=1e-14, atol=1e-15)
    g_raw = O.activate_backward(raw, act, gset(d, "g_act"))
    for a in ATTRS:
        close(getattr(g_raw, a), d["g_raw." + a], rtol=1e-13, atol=1e-15)


def test_activate_zero_quaternion_raises():
    raw = O.GSet(np.zeros((3, 3)), np.array([[1.0, 0, 0, 0], [0, 0, 0, 0], [1, 0, 0, 0]]),
                 np.zeros((3, 3)), np.zeros(3), np.zeros((3, 3)))
    with pytest.raises(FloatingPointError, match="index 1"):
        O.activate(raw)


def test_blend_backward():
    d = golden("model")
    model = _model(d)
    g_base14, g_deltas, g_psi = O.blend_backward(model, d["psi"], gset(d, "g_raw"))
    n = model.count
    close(g_base14[:3 * n], d["g_base.position"].ravel(), 0, 0)
    close(g_base14[10 * n:13 * n], d["g_base.scale"].ravel(), 0, 0)
    close(g_deltas, d["g_deltas"], 0, 0)
    close(g_psi, d["g_psi"], rtol=1e-12, atol=1e-12)


# --------------------------------------------------------------- binding

def test_transform_and_backward():
    d = golden("binding")
    frames = O.Frames(d["frames.rotation"], d["frames.quat"], d["frames.tri_vertices"])
    tangent = gset(d, "tangent")
    world = O.transform_to_deformed(tangent, frames, d["tri_index"], d["barycentric"])
    for a in ATTRS:
        close(getattr(world, a), d["world." + a], rtol=1e-13, atol=1e-15)
    g = O.transform_backward(tangent, frames, d["tri_index"], gset(d, "g_world"))
    for a in ATTRS:
        close(getattr(g, a), d["g_tangent." + a], rtol=1e-12, atol=1e-14)


# ---------------------------------------------------------------- render

def _scenes():
    d = golden("render")
    for s in range(int(d["num_scenes"])):
        p = f"s{s}."
        w, h = d[p + "wh"]
        yield s, p, d, gset(d, p + "world"), cam_from(d[p + "cam"], w, h)


@pytest.mark.parametrize("which", range(6))
def test_render_scene(which):
    for s, p, d, world, cam in _scenes():
        if s != which:
            continue
        splats = O.preprocess(world, cam)
        assert np.array_equal(splats.index, d[p + "splats.index"])
        assert np.array_equal(splats.sort_order, d[p + "splats.sort_order"])
        for k in ("mean2d", "conic", "depth", "radius", "x_cam", "cov_cam"):
            close(getattr(splats, k), d[p + "splats." + k], rtol=1e-13, atol=1e-13)
        image, aux = O.rasterize(splats, cam, d[p + "bg"])
        close(image, d[p + "image"], rtol=0, atol=1e-12)
        close(aux.transmittance, d[p + "trans"], rtol=0, atol=1e-12)
        assert np.array_equal(aux.stop, d[p + "stop"])
        close(aux.max_weight, d[p + "max_weight"], rtol=1e-12, atol=1e-14)
        grad = O.render_backward(splats, aux, d[p + "grad_image"])
        for a in ATTRS:
            ref = d[p + "grad." + a]
            scale = max(1.0, float(np.abs(ref).max()))
            close(getattr(grad, a), ref, rtol=1e-9, atol=1e-11 * scale)
        num, den = O.splat_weight_sums(aux, d[p + "target"])
        close(num, d[p + "num"], rtol=0, atol=1e-12)
        close(den, d[p + "den"], rtol=0, atol=1e-12)


def test_render_fixture_covers_termination_and_empty():
    d = golden("render")
    # scene 3 stacks near-opaque splats: some pixel must terminate (stop < M)
    m3 = d["s3.splats.index"].shape[0]
    assert (d["s3.stop"] < m3).any()
    # scene 5 is empty: the image is the background
    assert d["s5.splats.index"].shape[0] == 0
    assert np.array_equal(d["s5.image"], np.broadcast_to(d["s5.bg"], d["s5.image"].shape))


def test_preprocess_nonfinite_raises():
    d = golden("render")
    world = gset(d, "s0.world")
    world.scale[4, 1] = np.inf
    with pytest.raises(FloatingPointError, match="non-finite scale at Gaussian index 4"):
        O.preprocess(world, cam_from(d["s0.cam"], 16, 16))


# ------------------------------------------------------------ colour init

def test_estimate_and_apply_color_init():
    d = golden("color")
    world = gset(d, "world")
    cam = cam_from(d["cam"], 16, 16)
    splats = O.preprocess(world, cam)
    _, aux = O.rasterize(splats, cam, np.zeros(3))
    close(aux.max_weight, d["max_weight"], rtol=1e-12, atol=1e-14)
    est, eligible = O.estimate_colors(aux, d["target"], 0.1)
    assert np.array_equal(eligible, d["eligible"])
    close(est, d["est"], rtol=1e-12, atol=1e-13)
    n = world.count
    model = O.Model(O.GSet(np.zeros((n, 3)), np.tile([1.0, 0, 0, 0], (n, 1)), np.zeros((n, 3)), np.zeros(n),
                           d["color_before"].copy()), np.zeros((1, 10 * n)), {}, None, None)
    visited = np.zeros(n, bool)
    visited[:3] = True
    count = O.apply_color_init(model, est, eligible, visited)
    assert count == int(d["count"])
    assert np.array_equal(visited, d["visited"])
    close(model.base.color, d["color_after"], rtol=1e-12, atol=1e-12)


# -------------------------------------------------------------- train step

def test_train_steps_match_reference():
    d = golden("train")
    size = int(d["size"])
    cam = cam_from(d["cam"], size, size)
    mlp = {k: d["mlp0." + k].copy() for k in ("w1", "b1", "w2", "b2", "w3", "b3")}
    model = O.Model(gset(d, "base0"), d["deltas0"].copy(), mlp, d["tri_index"], d["barycentric"])
    B = d["thetas"].shape[0]
    frames = [O.Frames(d[f"frames{i}.rotation"], d[f"frames{i}.quat"], d[f"frames{i}.tri_vertices"])
              for i in range(B)]
    state = O.State(model, cam, workers=2)
    for step in range(2):
        p = f"step{step}."
        loss, black = O.train_step(state, d["thetas"], d["images"], frames, d[p + "bgs"])
        assert abs(loss - float(d[p + "loss"])) < 1e-12
        close(black, d[p + "black"], rtol=0, atol=1e-12)
        g_base, g_deltas, g_mlp = state.last_grads
        for a in ATTRS:
            ref = d[p + "g." + a]
            close(getattr(g_base, a), ref, rtol=1e-8, atol=1e-12 * max(1.0, np.abs(ref).max()))
        close(g_deltas, d[p + "g_deltas"], rtol=1e-8, atol=1e-14)
        for k in g_mlp:
            close(g_mlp[k], d[p + "gmlp." + k], rtol=1e-8, atol=1e-14)
        for a in ATTRS:
            close(getattr(model.base, a), d[p + "base." + a], rtol=1e-9, atol=1e-10)
        close(model.deltas, d[p + "deltas"], rtol=1e-9, atol=1e-10)
        for k in model.mlp:
            close(model.mlp[k], d[p + "mlp." + k], rtol=1e-9, atol=1e-10)
        assert np.array_equal(state.visited, d[p + "visited"])
    assert state.visited.any()          # colour init actually fired in the fixture
    state.close()
