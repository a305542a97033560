"""The reference-facing drop-in (compat.train_step / BatchRenderer) against the
reference's own outputs.  Reference-shaped objects are built here (the reference package
is not available on the GPU box); their fields are exactly the ones headsplat's
TrainState / FrameSample / MeshFrames / AvatarModel carry (S/train.py:202-211,
S/dataset.py:27-34, S/binding.py:47-53, S/model.py:98-127)."""
from types import SimpleNamespace as NS

import numpy as np
import pytest
import torch

from conftest import golden

pytestmark = pytest.mark.gpu
ATTRS = ("position", "rotation", "scale", "opacity", "color")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2503_12886_b200 import build
    build.build()


def _ref_state(d):
    from bench_support import synth
    n = d["base0.position"].shape[0]
    base = NS(**{a: d[f"base0.{a}"].copy() for a in ATTRS})
    deltas = [NS(position=x[:3 * n].reshape(n, 3).copy(), rotation=x[3 * n:7 * n].reshape(n, 4).copy(),
                 color=x[7 * n:].reshape(n, 3).copy()) for x in d["deltas0"]]
    mlp = NS(**{k: d["mlp0." + k].copy() for k in ("w1", "b1", "w2", "b2", "w3", "b3")})
    model = NS(base=base, deltas=deltas, mlp=mlp,
               bindings=NS(triangle_index=d["tri_index"], barycentric=d["barycentric"]))
    cfg = NS(lr_position=0.0008, lr_opacity=0.25, lr_scale=0.025, lr_rotation=0.005, lr_color=0.0125,
             delta_position_scale=0.05, delta_rotation_scale=0.5, delta_color_scale=0.5, lr_mlp=0.001,
             color_init=True, use_mlp=True)
    size = int(d["size"])
    c = d["cam"]
    cam = synth.Camera(c[12], c[13], c[14], c[15], c[:9].reshape(3, 3), c[9:12], size, size)
    state = NS(model=model, config=cfg, camera=cam, color_state=NS(visited=np.zeros(n, bool), threshold=0.1))
    B = d["thetas"].shape[0]
    samples = [NS(index=i + 1, image=d["images"][i], theta=d["thetas"][i]) for i in range(B)]
    meshes = [NS(rotation=d[f"frames{i}.rotation"], quat=d[f"frames{i}.quat"],
                 tri_vertices=d[f"frames{i}.tri_vertices"]) for i in range(B)]
    return state, samples, (lambda s: meshes[s.index - 1])


def test_compat_train_step_matches_reference_fixture():
    from paper_2503_12886_b200 import compat
    d = golden("train")
    state, samples, mesh_of = _ref_state(d)
    lrs = {"position": 8e-4, "rotation": 5e-3, "scale": 2.5e-2, "opacity": 0.25, "color": 1.25e-2}
    for step in range(2):
        p = f"step{step}."
        loss, black = compat.train_step(state, samples, d[p + "bgs"], mesh_of)
        assert abs(loss - float(d[p + "loss"])) < 2e-5
        np.testing.assert_allclose(black, d[p + "black"], atol=2e-5)
        for a in ATTRS:       # written back into the caller's (reference-shaped) model
            ref = d[p + "base." + a]
            bad = np.abs(getattr(state.model.base, a) - ref) > 0.05 * lrs[a] + 1e-4 * np.abs(ref)
            assert bad.mean() < 5e-3, (step, a)
        assert (state.color_state.visited != d[p + "visited"]).sum() <= 2


def test_batch_renderer_matches_single_calls():
    from paper_2503_12886_b200 import compat
    d = golden("render")
    items = []
    for s in range(3):
        p = f"s{s}."
        w, h = (int(x) for x in d[p + "wh"])
        if (w, h) != (16, 16) and s:
            continue
        world = NS(**{a: d[f"{p}world.{a}"] for a in ATTRS})
        c = d[p + "cam"]
        cam = NS(fx=c[12], fy=c[13], cx=c[14], cy=c[15], rotation=c[:9].reshape(3, 3), translation=c[9:12],
                 width=w, height=h)
        items.append((world, cam, d[p + "bg"]))
    items = items * 3                       # same-size items batch into one launch
    r = compat.BatchRenderer(workers=4, scheme="two_stage")
    out = r.render_batch(items)
    assert r.barrier_count == 1
    for (world, cam, bg), (img, aux) in zip(items, out):
        img1, aux1 = compat.rasterize(compat.preprocess(world, cam), cam, bg)
        assert np.array_equal(img, img1)             # batched == per-item, bitwise
        assert np.array_equal(aux.max_weight, aux1.max_weight)


def test_step_from_host_prefetch_then_other_batch():
    """step_from_host(X, prefetch=B), then a different batch C, then B: every step must
    train on its own inputs (a pending prefetch of B may not leak into C's buffers, and
    B must be re-uploaded after C reused them) -- same losses and parameters as the
    same steps without prefetch."""
    from bench_support import synth
    from paper_2503_12886_b200.device import AvatarParams, Trainer
    wl = synth.make_workload(48, 4, 96, K=6, hidden=32, seed=5)
    av = wl.avatar
    mk = lambda: Trainer(AvatarParams.from_host(NS(**{a: av.base[a] for a in ATTRS}), av.deltas, av.mlp,
                                                av.tri_index, av.barycentric), 96, 96, 4)
    rng = np.random.default_rng(9)
    cams = np.tile(wl.camera.packed(), (4, 1))

    def batch(k):
        return (np.asarray(wl.thetas, np.float32) + np.float32(0.01 * k),
                rng.integers(0, 256, wl.targets.shape, dtype=np.uint8), wl.frames, cams,
                rng.uniform(0, 1, (4, 3)).astype(np.float32))
    X, Bb, C = batch(0), batch(1), batch(2)
    a, b = mk(), mk()
    la = [a.step_from_host(*X, prefetch=Bb).loss, a.step_from_host(*C).loss, a.step_from_host(*Bb).loss]
    lb = [b.step_from_host(*X).loss, b.step_from_host(*C).loss, b.step_from_host(*Bb).loss]
    torch.cuda.synchronize()
    np.testing.assert_allclose(la, lb, rtol=1e-5)
    pa, pb = a.av.params.cpu().numpy(), b.av.params.cpu().numpy()
    assert np.mean(np.abs(pa - pb) > 1e-5) < 1e-3
