"""Diagnostics: C1 device step vs oracle, normwise errors per gradient tensor and the
stage-wise blend/MLP adjoint check fed the device's own g_raw."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import oracle as O  # noqa: E402
from bench_support import synth  # noqa: E402
from paper_2503_12886_b200.device import AvatarParams, Trainer, split_flat  # noqa: E402

ATTRS = ("position", "rotation", "scale", "opacity", "color")


def nerr(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def main(uv=141, B=4, size=256):
    wl = synth.make_workload(uv, B, size)
    av = wl.avatar
    dev = AvatarParams.from_host(O.GSet(*(av.base[a] for a in ATTRS)), av.deltas, av.mlp, av.tri_index, av.barycentric)
    tr = Trainer(dev, size, size, B)
    cams = np.tile(wl.camera.packed(), (B, 1))
    bgs = np.asarray(wl.backgrounds, np.float32).astype(np.float64)
    res = tr.step_from_host(wl.thetas, wl.targets, wl.frames, cams, bgs)
    f = lambda a: np.asarray(a, np.float32).astype(np.float64)
    model = O.Model(O.GSet(*(f(av.base[a]) for a in ATTRS)), f(av.deltas), {k: f(v) for k, v in av.mlp.items()},
                    av.tri_index, f(av.barycentric))
    c = wl.camera.packed().astype(np.float64)
    cam = O.Cam(c[12], c[13], c[14], c[15], c[:9].reshape(3, 3), c[9:12], size, size)
    frames = [O.Frames(x[:, :9].reshape(-1, 3, 3).astype(np.float64), x[:, 9:13].astype(np.float64),
                       x[:, 13:].reshape(-1, 3, 3).astype(np.float64)) for x in wl.frames]
    model0 = model.copy()
    state = O.State(model, cam, workers=8)
    thetas = f(wl.thetas)
    loss, black = O.train_step(state, thetas, wl.targets.astype(np.float64) / 255.0, frames, bgs)
    print("loss", res.loss, loss)
    g_base, g_deltas, g_mlp = state.last_grads
    gb, gd, gm = split_flat(tr.grads.cpu().numpy(), dev.N, dev.K, dev.H, dev.D)
    for a in ATTRS:
        print("base", a, "normwise", nerr(gb[a], getattr(g_base, a)))
    print("deltas normwise", nerr(gd, g_deltas))
    for k in gm:
        print("mlp", k, "normwise", nerr(gm[k], g_mlp[k]))
    # stage-wise: oracle blend/MLP adjoint fed the device's g_raw
    n = dev.N
    graw = tr.g_raw14.view(B, 14 * n).cpu().numpy().astype(np.float64)
    gpsi_dev = tr.gpsi.cpu().numpy().astype(np.float64)
    acc = {k: np.zeros_like(v, dtype=np.float64) for k, v in model0.mlp.items()}
    for b in range(B):
        g = graw[b]
        gr = O.GSet(g[:3 * n].reshape(n, 3), g[3 * n:7 * n].reshape(n, 4), g[10 * n:13 * n].reshape(n, 3),
                    g[13 * n:], g[7 * n:10 * n].reshape(n, 3))
        psi, cache = O.map_params(model0.mlp, thetas[b])
        _, _, gpsi = O.blend_backward(model0, psi, gr)
        absum = np.abs(model0.deltas * g[None, :10 * n]).sum(axis=1)
        print("frame", b, "gpsi max err / abs-sum", float(np.max(np.abs(gpsi - gpsi_dev[b]) / absum)),
              "normwise", nerr(gpsi_dev[b], gpsi))
        O.mlp_backward(model0.mlp, cache, gpsi_dev[b], into=acc)
    for k in gm:
        print("stage mlp", k, "normwise (oracle fed device gpsi)", nerr(gm[k], acc[k]))


if __name__ == "__main__":
    main()
