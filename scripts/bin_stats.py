"""Fraction of (splat, tile) keys the exact ellipse-rectangle test would cull at
emission (needs a -DHS_BIN_STATS build: HS_B200_LIB=... python scripts/bin_stats.py)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import CONFIGS, make_trainer  # noqa: E402
from paper_2503_12886_b200 import _lib as L  # noqa: E402

tr, d, wl = make_trainer(CONFIGS["C2"])
tr.tile_binning = tr.two_level_binning = False     # the counters live in the one-level emission
buf = (ctypes.c_uint64 * 2)()
for _ in range(3):
    tr.step(d["thetas"], d["targets"], None, d["cameras"], d["backgrounds"])
torch.cuda.synchronize()
L.load().hs_bin_stats(buf, 1)
tr.step(d["thetas"], d["targets"], None, d["cameras"], d["backgrounds"])
torch.cuda.synchronize()
L.load().hs_bin_stats(buf, 1)
print(f"keys {buf[0]}  cullable {buf[1]} ({buf[1] / max(buf[0], 1) * 100:.1f}%)")
