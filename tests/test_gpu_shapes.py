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
    from bench_support import synth
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
    """Stage-exact replay (device order, bbox, L1 signs; flip-masked pixels zeroed on
    both sides): every gradient entry within rel 1e-3 (floor 1e-5 max|g|)."""
    from test_gpu_train import check_masked_parity, masked_step_parity
    c = CASES[case]
    wl, cam, targets = _setup(c)
    B, W, H = c["B"], c["W"], c["H"]
    rep, errs, tr = masked_step_parity(wl, B, W, H, cam_packed=cam.packed(), targets=targets)
    assert tr.tile_bits == int(((W + 15) // 16) * ((H + 15) // 16) - 1).bit_length()
    check_masked_parity(rep, errs, case)


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
    from gpu_helpers import rel_fail
    nbad, worst, _ = rel_fail(a.g_splat.cpu().numpy(), b.g_splat.cpu().numpy(), rtol=1e-4)
    assert nbad == 0, worst
