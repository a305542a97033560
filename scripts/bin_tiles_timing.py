"""CUDA-event timing of the tile-major binner's stages inside the C2 step's stream
(scan, fill) and of the whole bin_tiles call, against the projection before it."""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS, make_trainer  # noqa: E402
from paper_2503_12886_b200 import _lib as L  # noqa: E402
from paper_2503_12886_b200.device import _p, _stream, key_layout  # noqa: E402

tr, d, wl = make_trainer(CONFIGS["C2"])
args = (d["thetas"], d["targets"], None, d["cameras"], d["backgrounds"])
for _ in range(5):
    tr.step(*args)
torch.cuda.synchronize()
bn, B, N = tr.binner, tr.B, tr.av.N
tiles_x, tiles_y, tiles, tile_bits, frame_bits = key_layout(B, tr.W, tr.H)
nseg = B << tile_bits
ranges = bn.ranges[:2 * nseg]
s = _stream()
reps = 30
ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(reps)]
# re-run count (via the projection's output: recount with hs_tile_count), scan and fill
for r in range(reps):
    e = ev[r]
    e[0].record()
    L.call("hs_tile_count", B, N, tr.W, tr.H, _p(tr.records), _p(tr.counts), _p(bn.tile_counts), s)
    e[1].record()
    L.call("hs_tile_scan", B, tr.W, tr.H, _p(bn.tile_counts), _p(ranges), _p(bn.cursor), _p(bn.lists),
           _p(bn.list_counts), bn.list_half, _p(tr.err), _p(bn.depth_range), _p(bn.summary), s)
    e[2].record()
    L.call("hs_tile_fill", B, N, tr.W, tr.H, _p(tr.records), _p(tr.counts), _p(bn.rects), _p(tr.depth), _p(ranges),
           _p(bn.cursor), _p(bn.lists), _p(bn.list_counts), bn.list_half, _p(bn.summary), bn.cap, _p(bn.keys),
           _p(bn.vals), 0, bn.fork, s)
    e[3].record()
torch.cuda.synchronize()
acc = [0.0, 0.0, 0.0]
for e in ev[3:]:
    for k in range(3):
        acc[k] += e[k].elapsed_time(e[k + 1])
n = reps - 3
print(f"count {acc[0] / n * 1000:.1f} us, scan {acc[1] / n * 1000:.1f} us, fill {acc[2] / n * 1000:.1f} us "
      f"(back to back, GPU never waits for the host)")
