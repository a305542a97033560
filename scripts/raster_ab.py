"""Kernel-level A/B of the fused training raster: after one C2 step, time hs_raster_train
alone (g_splat zeroed before each launch, L2 flushed) -- median of R launches per lib.
    HS_B200_LIB=... python scripts/raster_ab.py [reps]"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import bench
from paper_2503_12886_b200 import _lib as L
from paper_2503_12886_b200.device import _p

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 40
tr, d, wl = bench.make_trainer(bench.CONFIGS["C2"])
for _ in range(int(os.environ.get('RAB_STEPS', '100'))):
    tr.step(d["thetas"], d["targets"], None, d["cameras"], d["backgrounds"])
torch.cuda.synchronize()
keys, vals, ranges, tile_bits, tiles = tr.binner.result
B, N = tr.B, tr.av.N
flags = L.RASTER_LOSS | (L.RASTER_MAXW_UNVISITED | L.RASTER_WSUMS if os.environ.get("RAB_CI", "3") == "3" else 0)
flush = torch.empty(256 << 18, dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream()
times = []
for r in range(reps + 3):
    if os.environ.get('RAB_FLUSH'):
        flush.fill_(1.0)
    tr.g_splat.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    L.call("hs_raster_train", B, N, tr.W, tr.H, flags, _p(tr.records), _p(vals), _p(ranges), tile_bits,
           _p(d["backgrounds"]), _p(d["targets"]), _p(tr.visited), _p(tr.maxw), _p(tr.wsums), _p(tr.loss_partials),
           ctypes.c_float(1.0 / (tr.H * tr.W * 3.0) / B), _p(tr.g_splat), None, None, None, _p(tr.raster_ws),
           ctypes.c_void_p(s.cuda_stream))
    b.record()
    b.synchronize()
    if r >= 3:
        times.append(a.elapsed_time(b))
t = np.array(times)
print(f"{os.path.basename(os.environ.get('HS_B200_LIB', 'default'))}: raster median {np.median(t) * 1000:.1f} us "
      f"(p10 {np.percentile(t, 10) * 1000:.1f}, p90 {np.percentile(t, 90) * 1000:.1f}), keys {tr.last_total}")
