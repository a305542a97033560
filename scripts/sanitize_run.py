"""Workloads for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
    compute-sanitizer --tool <tool> python scripts/sanitize_run.py <case>
case: c1_step (two C1 training steps: 19,881 Gaussians, 4 x 256^2, fused raster, the
tile-major binner, Adam + colour init; then one unfused step), c3_render (BASELINE
configs[2] shape: 100,489 Gaussians at 512^2, 16 of the 64 frames, device rig), crowded
(one 16x16 tile with 3,000 / 9,000 splats: warp, CTA-merge, shared-memory CTA and
two-level fallback sorts), det (deterministic mode step)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import numpy as np
import torch

ATTRS = ("position", "rotation", "scale", "opacity", "color")


def trainer(uv, B, size, **kw):
    from bench_support import synth
    from paper_2503_12886_b200.device import AvatarParams, DeviceRig, Trainer
    wl = synth.make_workload(uv, B, size)
    av = wl.avatar
    dev = AvatarParams.from_host(type("G", (), {a: av.base[a] for a in ATTRS})(), av.deltas, av.mlp, av.tri_index,
                                 av.barycentric)
    tr = Trainer(dev, size, size, B, rig=DeviceRig(wl.rig), **kw)
    t = lambda a, dt=torch.float32: torch.as_tensor(np.asarray(a), dtype=dt).cuda()
    inp = (t(wl.thetas), t(wl.targets, torch.uint8), None, t(np.tile(wl.camera.packed(), (B, 1))),
           t(wl.backgrounds))
    return tr, inp


case = sys.argv[1]
if case in ("c1_step", "det"):
    tr, inp = trainer(141, 4, 256, deterministic=case == "det")
    for _ in range(2):
        tr.step(*inp)
    if case == "c1_step":
        tr.fused_raster = False
        tr.step(*inp)
    torch.cuda.synchronize()
    print(case, "ok", tr.result().loss)
elif case == "c3_render":
    tr, inp = trainer(317, 16, 512, color_init=False)
    img = tr.render(inp[0], None, inp[3], inp[4])
    torch.cuda.synchronize()
    print(case, "ok", float(img.mean()))
elif case == "crowded":
    import oracle as O
    from paper_2503_12886_b200 import compat as C
    for n in (3000, 9000):
        rng = np.random.default_rng(n)
        q = rng.normal(size=(n, 4))
        q /= np.linalg.norm(q, axis=-1, keepdims=True)
        pos = np.round(rng.uniform(-0.3, 0.3, (n, 3)) * 8) / 8
        world = O.GSet(pos, q, rng.uniform(0.02, 0.06, (n, 3)), rng.uniform(0.3, 0.9, n), rng.uniform(0, 1, (n, 3)))
        cam = O.Cam(24.0, 24.0, 8.0, 8.0, np.eye(3), np.array([0.0, 0.0, 2.0]), 16, 16)
        sp = C.preprocess(world, cam)
        dev = sp._dev["batch"]
        err = torch.full((1,), -1, dtype=torch.int64, device="cuda")
        total, code = dev["binner"].bin_tiles(dev["B"], dev["N"], dev["W"], dev["H"], dev["records"], dev["depth"],
                                             dev["counts"], err)
        img, aux = C.rasterize(sp, cam, np.zeros(3))
        g = C.render_backward(sp, aux, rng.normal(size=img.shape))
        torch.cuda.synchronize()
        print(case, n, "ok", total, dev["binner"].mode)
else:
    raise SystemExit(f"unknown case {case}")
