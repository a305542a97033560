"""Deterministic mode and re-entrancy of the device step (SURVEY §7 hard part 6, §8b).

* Trainer(deterministic=True) accumulates the raster's splat gradients and colour-init
  sums in int64 fixed point (HS_RASTER_DETERMINISTIC): two runs of the same steps give
  bitwise identical gradients and parameters (the reference is bitwise identical across
  worker counts, T/test_train.py:58-71), and the result agrees with the float-atomic mode
  entrywise.
* Re-entrancy of the C ABI: two Trainers stepping concurrently on two CUDA streams (each
  with its own raster workspace and fork context) produce bitwise the results of the same
  Trainers run one after the other; a second device is used when present.
"""
import numpy as np
import pytest
import torch

import oracle as O
from gpu_helpers import rel_fail

pytestmark = pytest.mark.gpu
ATTRS = ("position", "rotation", "scale", "opacity", "color")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2503_12886_b200 import build
    build.build()


def _setup(seed=0, uv=64, B=4, size=192):
    from bench_support import synth
    wl = synth.make_workload(uv, B, size, seed=seed, frames_seed=seed + 1)
    return wl


def _trainer(wl, size=192, device="cuda", **kw):
    from paper_2503_12886_b200.device import AvatarParams, Trainer
    av = wl.avatar
    dev = AvatarParams.from_host(O.GSet(*(av.base[a] for a in ATTRS)), av.deltas, av.mlp, av.tri_index,
                                 av.barycentric, device=device)
    return Trainer(dev, size, size, wl.thetas.shape[0], **kw)


def _inputs(wl, device="cuda"):
    B = wl.thetas.shape[0]
    t = lambda a, dt=torch.float32: torch.as_tensor(np.asarray(a), dtype=dt).to(device)
    return (t(wl.thetas), t(wl.targets, torch.uint8), t(wl.frames), t(np.tile(wl.camera.packed(), (B, 1))),
            t(wl.backgrounds))


def _run(tr, inp, steps=3):
    g = []
    for _ in range(steps):
        tr.step(*inp)
        g.append(tr.grads.clone())
    torch.cuda.synchronize()
    return g, tr.av.params.clone(), tr.loss_out.clone()


def test_deterministic_mode_is_bitwise_reproducible():
    wl = _setup()
    inp = _inputs(wl)
    ga, pa, la = _run(_trainer(wl, deterministic=True), inp)
    gb, pb, lb = _run(_trainer(wl, deterministic=True), inp)
    for x, y in zip(ga, gb):
        assert torch.equal(x, y)
    assert torch.equal(pa, pb) and torch.equal(la, lb)
    # the float-atomic mode: same loss, gradients equal up to the summation order
    gf, pf, lf = _run(_trainer(wl), inp, steps=1)
    assert torch.equal(lf, _run(_trainer(wl, deterministic=True), inp, steps=1)[2])
    nbad, worst, need = rel_fail(gf[0].cpu().numpy(), ga[0].cpu().numpy(), rtol=1e-4)
    assert nbad == 0, (worst, need)


def test_float_mode_differs_only_by_summation_order():
    """(Documents why the mode exists: float atomics make two identical runs differ in
    the last bits of some gradient entries, never by more than reduction-order noise.)"""
    wl = _setup(seed=2)
    inp = _inputs(wl)
    ga, _, _ = _run(_trainer(wl), inp, steps=1)
    gb, _, _ = _run(_trainer(wl), inp, steps=1)
    nbad, worst, _ = rel_fail(ga[0].cpu().numpy(), gb[0].cpu().numpy(), rtol=1e-5)
    assert nbad == 0, worst


def _concurrent(streams, trainers, inputs, steps=3):
    """Interleave the steps of several Trainers, each on its own stream."""
    out = [[] for _ in trainers]
    for _ in range(steps):
        for i, (s, tr, inp) in enumerate(zip(streams, trainers, inputs)):
            with torch.cuda.device(s.device), torch.cuda.stream(s):
                tr.step(*inp)
                out[i].append(tr.grads.clone())
    for s in streams:
        s.synchronize()
    return out


def test_two_trainers_on_two_streams_match_serial():
    wa, wb = _setup(seed=0), _setup(seed=5)
    ia, ib = _inputs(wa), _inputs(wb)
    serial_a = _run(_trainer(wa, deterministic=True), ia)
    serial_b = _run(_trainer(wb, deterministic=True), ib)
    ta, tb = _trainer(wa, deterministic=True), _trainer(wb, deterministic=True)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    ga, gb = _concurrent([s1, s2], [ta, tb], [ia, ib])
    for x, y in zip(ga, serial_a[0]):
        assert torch.equal(x, y)
    for x, y in zip(gb, serial_b[0]):
        assert torch.equal(x, y)
    assert torch.equal(ta.av.params, serial_a[1]) and torch.equal(tb.av.params, serial_b[1])


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two devices")
def test_two_devices_match_single_device():
    wl = _setup(seed=3)
    ref = _run(_trainer(wl, deterministic=True), _inputs(wl))
    t1 = _trainer(wl, device="cuda:1", deterministic=True)
    s0, s1 = torch.cuda.Stream(device=0), torch.cuda.Stream(device=1)
    t0 = _trainer(wl, deterministic=True)
    g0, g1 = _concurrent([s0, s1], [t0, t1], [_inputs(wl), _inputs(wl, "cuda:1")])
    for x, y, z in zip(g0, g1, ref[0]):
        assert torch.equal(x, z) and torch.equal(y.cpu(), z.cpu())
