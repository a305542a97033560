"""Shape coverage of the device training step against the float64 oracle (replaying the
device's compositing order and bbox, like test_c1_step_vs_oracle):

* non-square image whose sides are not multiples of the 16-px tile, one frame, K = 1;
* 17 frames (two frame chunks in blend_bwd, 5 frame bits), K = 25;
* an image with more than 1024 tiles (12 tile bits in the sort keys);
* Gaussian counts whose CTAs straddle frames, and 16,384 tiles per frame (past the
  shared-memory tile histograms);
and, at each shape, the fused training raster against the separate forward/adjoint
kernels."""
import numpy as np
import pytest
import torch

import oracle as O
from gpu_helpers import normwise, replay_from_trainer

pytestmark = pytest.mark.gpu
ATTRS = ("position", "rotation", "scale", "opacity", "color")

CASES = {
    "nonsquare_b1_k1": dict(uv=40, B=1, W=200, H=136, K=1, hidden=8),
    "b17_k25": dict(uv=32, B=17, W=64, H=64, K=25, hidden=16),
    "tiles3185": dict(uv=48, B=2, W=1040, H=784, K=4, hidden=16),
    # 1,296 Gaussians: projection / scatter CTAs straddle frame boundaries
    "b3_unaligned": dict(uv=36, B=3, W=96, H=80, K=3, hidden=8),
    # 16,384 tiles per frame: the tile counts and the scatter take the global-atomic path
    "tiles16384": dict(uv=24, B=1, W=2048, H=2048, K=2, hidden=8),
}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2503_12886_b200 import build
    build.build()


def _setup(c, seed=0):
    from paper_2503_12886_b200 import synth
    wl = synth.make_workload(c["uv"], c["B"], 16, K=c["K"], hidden=c["hidden"], seed=seed,
                             distinct_frames=c["B"])
    W, H = c["W"], c["H"]
    f = 1.2 * min(W, H)
    cam = synth.Camera(f, f, W / 2.0, H / 2.0, wl.camera.rotation, wl.camera.translation, W, H)
    rng = np.random.default_rng(seed + 7)
    targets = rng.integers(0, 256, (c["B"], H, W, 4), dtype=np.uint8)
    return wl, cam, targets


def _device(wl):
    from paper_2503_12886_b200.device import AvatarParams
    av = wl.avatar
    return AvatarParams.from_host(O.GSet(*(av.base[a] for a in ATTRS)), av.deltas, av.mlp, av.tri_index,
                                  av.barycentric)


@pytest.mark.parametrize("case", sorted(CASES))
def test_step_vs_oracle(case):
    from paper_2503_12886_b200.device import Trainer, split_flat
    c = CASES[case]
    wl, cam, targets = _setup(c)
    B, W, H = c["B"], c["W"], c["H"]
    dev = _device(wl)
    tr = Trainer(dev, W, H, B)
    tr.radius = torch.empty(B * dev.N, device="cuda")
    cams = np.tile(cam.packed(), (B, 1))
    bgs = np.asarray(wl.backgrounds, np.float32).astype(np.float64)
    res = tr.step_from_host(wl.thetas, targets, wl.frames, cams, bgs)
    assert tr.tile_bits == int(((W + 15) // 16) * ((H + 15) // 16) - 1).bit_length()
    replay = replay_from_trainer(tr)
    av = wl.avatar
    model = O.Model(O.GSet(*(np.asarray(av.base[a], np.float32).astype(np.float64) for a in ATTRS)),
                    np.asarray(av.deltas, np.float32).astype(np.float64),
                    {k: np.asarray(v, np.float32).astype(np.float64) for k, v in av.mlp.items()}, av.tri_index,
                    np.asarray(av.barycentric, np.float32).astype(np.float64))
    p = cam.packed().astype(np.float64)
    ocam = O.Cam(p[12], p[13], p[14], p[15], p[:9].reshape(3, 3), p[9:12], W, H)
    frames = [O.Frames(f[:, :9].reshape(-1, 3, 3).astype(np.float64), f[:, 9:13].astype(np.float64),
                       f[:, 13:].reshape(-1, 3, 3).astype(np.float64)) for f in wl.frames]
    state = O.State(model, ocam, workers=4)
    loss, black = O.train_step(state, np.asarray(wl.thetas, np.float32).astype(np.float64),
                               targets.astype(np.float64) / 255.0, frames, bgs, replay=replay)
    state.close()
    assert abs(res.loss - loss) < 1e-4 * max(loss, 1e-3), (res.loss, loss)
    np.testing.assert_allclose(res.black_l1, black, rtol=1e-3, atol=1e-5)
    g_base, g_deltas, g_mlp = state.last_grads
    gb, gd, gm = split_flat(tr.grads.cpu().numpy(), dev.N, dev.K, dev.H, dev.D)
    gscale = np.linalg.norm(g_base.position)
    errs = {a: normwise(gb[a], getattr(g_base, a), scale=gscale if a == "rotation" else None) for a in ATTRS}
    errs["deltas"] = normwise(gd, g_deltas)
    print(case, errs)
    for k, e in errs.items():
        assert e < 5e-3, (k, e)


@pytest.mark.parametrize("case", sorted(CASES))
def test_fused_equals_separate(case):
    from paper_2503_12886_b200.device import Trainer
    c = CASES[case]
    wl, cam, targets = _setup(c, seed=3)
    B, W, H = c["B"], c["W"], c["H"]
    th = torch.from_numpy(np.asarray(wl.thetas, np.float32)).cuda()
    tg = torch.from_numpy(targets).cuda()
    fr = torch.from_numpy(wl.frames).cuda()
    cams = torch.from_numpy(np.tile(cam.packed(), (B, 1))).cuda()
    bg = torch.from_numpy(np.asarray(wl.backgrounds, np.float32)).cuda()
    a, b = Trainer(_device(wl), W, H, B), Trainer(_device(wl), W, H, B)
    b.fused_raster = False
    la = a.step(th, tg, fr, cams, bg).clone()
    lb = b.step(th, tg, fr, cams, bg).clone()
    assert torch.equal(la, lb)
    ga, gb = a.g_splat.cpu().numpy(), b.g_splat.cpu().numpy()
    assert np.linalg.norm(ga - gb) <= 1e-5 * max(np.linalg.norm(gb), 1e-30)
