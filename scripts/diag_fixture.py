"""Diagnostics: device Trainer vs the reference's golden train fixture (colour init)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import oracle as O  # noqa: E402
from conftest import golden  # noqa: E402
from paper_2503_12886_b200.device import AvatarParams, Trainer, split_flat  # noqa: E402

ATTRS = ("position", "rotation", "scale", "opacity", "color")
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
res = tr.step_from_host(d["thetas"], targets, frames, cam, d["step0.bgs"])
vis = tr.visited.cpu().numpy().astype(bool)
ref_vis = d["step0.visited"]
print("visited gpu", vis.sum(), "ref", ref_vis.sum(), "xor", (vis ^ ref_vis).sum())
pb, _, _ = av.split_host()
col = pb["color"]
rc = d["step0.base.color"]
diff = np.abs(col - rc).max(axis=1)
print("color diff > 6e-4:", (diff > 6e-4).sum(), "of which visited in ref:", ((diff > 6e-4) & ref_vis).sum())
idx = np.flatnonzero((diff > 6e-4) & ref_vis)[:10]
maxw = tr.maxw.view(B, -1).cpu().numpy()
ws = tr.wsums.view(B, -1, 4).cpu().numpy()
for i in idx:
    b = int(np.argmax(maxw[:, i]))
    print(i, "gpu", col[i], "ref", rc[i], "maxw", maxw[:, i], "ws", ws[b, i])
g0 = d["base0.color"]
print("ref delta (first 5 mismatching, not visited):")
for i in np.flatnonzero((diff > 6e-4) & ~ref_vis)[:5]:
    print(i, "gpu", col[i] - g0[i], "ref", rc[i] - g0[i], "g_ref", d["step0.g.color"][i])
