"""How many (splat, 16x16 tile) keys of the C2 step an exact tile cull would drop: the
alpha >= 1/255 ellipse (q <= qmax) cannot reach the tile's rectangle of pixel centres
inside the splat's integer bbox (the raster's per-block cull, at tile granularity)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS, make_trainer  # noqa: E402

tr, d, wl = make_trainer(CONFIGS["C2"])
for _ in range(20):
    tr.step(d["thetas"], d["targets"], None, d["cameras"], d["backgrounds"])
torch.cuda.synchronize()
rec = tr.records.view(-1, 12)
u = rec.view(torch.int32)
mx, my, a, b, c, op, qmax = rec[:, 0], rec[:, 1], rec[:, 2], rec[:, 3], rec[:, 4], rec[:, 5], rec[:, 6]
rows, cols = u[:, 7], u[:, 8]
rl = (rows << 16) >> 16
rh = rows >> 16
cl = (cols << 16) >> 16
ch = cols >> 16
live = (rl <= rh) & (cl <= ch) & (qmax >= 0)
T = 16
keys = kept = 0
ty0, ty1, tx0, tx1 = rl // T, rh // T, cl // T, ch // T
maxr = int((ty1 - ty0 + 1)[live].max()), int((tx1 - tx0 + 1)[live].max())
for dy in range(maxr[0]):
    for dx in range(maxr[1]):
        ty, tx = ty0 + dy, tx0 + dx
        m = live & (ty <= ty1) & (tx <= tx1)
        # the tile's pixels inside the bbox
        ys, ye = torch.maximum(ty * T, rl), torch.minimum(ty * T + T - 1, rh)
        xs, xe = torch.maximum(tx * T, cl), torch.minimum(tx * T + T - 1, ch)
        dxlo, dxhi = xs.float() + 0.5 - mx, xe.float() + 0.5 - mx
        dylo, dyhi = ys.float() + 0.5 - my, ye.float() + 0.5 - my
        # exact min of q over the rectangle (positive definite q): candidates on the edges facing the mean
        dxv = torch.clamp(torch.zeros_like(dxlo), dxlo, dxhi) if False else torch.minimum(torch.maximum(torch.zeros_like(dxlo), dxlo), dxhi)
        dyv = torch.minimum(torch.maximum(-b * dxv / c, dylo), dyhi)
        dyh = torch.minimum(torch.maximum(torch.zeros_like(dylo), dylo), dyhi)
        dxh = torch.minimum(torch.maximum(-b * dyh / a, dxlo), dxhi)
        qv = a * dxv * dxv + 2 * b * dxv * dyv + c * dyv * dyv
        qh = a * dxh * dxh + 2 * b * dxh * dyh + c * dyh * dyh
        q = torch.minimum(qv, qh)
        keep = m & ~(q * 0.999 - 1e-3 > qmax)
        keys += int(m.sum())
        kept += int(keep.sum())
print(f"keys {keys} (binner {tr.last_total}), kept by an exact tile cull {kept} ({kept / keys * 100:.1f}%)")
