"""Load balance of the persistent raster: per-warp start / end times of one fused raster
launch (a -DHS_RASTER_TIMING build, HS_B200_LIB=...), as the number of warps still working
over the launch and the idle fraction of warp-time."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import bench
from paper_2503_12886_b200 import _lib as L

tr, d, wl = bench.make_trainer(bench.CONFIGS["C2"])
for _ in range(100):
    tr.step(d["thetas"], d["targets"], None, d["cameras"], d["backgrounds"])
torch.cuda.synchronize()
n = 148 * 28
buf = (ctypes.c_uint64 * (3 * n))()
L.load().hs_raster_warp_times(buf, n)
a = np.frombuffer(buf, dtype=np.uint64).reshape(n, 3).astype(np.float64)
t0 = a[:, 0].min()
st, en, it = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3, a[:, 2]
span = en.max()
print(f"launch span {span:.1f} us; warp end times: p10 {np.percentile(en, 10):.1f} p50 {np.median(en):.1f} "
      f"p90 {np.percentile(en, 90):.1f} max {en.max():.1f}; start max {st.max():.1f}")
busy = (en - st).sum()
print(f"idle fraction of warp-time: {1 - busy / (n * span):.3f}; items per warp p10 {np.percentile(it, 10):.0f} "
      f"p50 {np.median(it):.0f} p90 {np.percentile(it, 90):.0f}")
for f in (0.5, 0.8, 0.9, 0.95, 1.0):
    print(f"  at {f:.0%} of the span: {(en > f * span).sum()} warps still working" if f < 1 else "")
