"""Forward-raster work counters on the C2 step (needs a -DHS_RASTER_STATS build)."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS, make_trainer
from paper_2503_12886_b200 import _lib as L
import torch
tr, d, wl = make_trainer(CONFIGS["C2"])
for _ in range(3):
    tr.step(d["thetas"], d["targets"], d["frames"], d["cameras"], d["backgrounds"])
torch.cuda.synchronize()
buf = (ctypes.c_uint64 * 16)()
L.load().hs_raster_stats(buf, 1)
tr.step(d["thetas"], d["targets"], d["frames"], d["cameras"], d["backgrounds"])
torch.cuda.synchronize()
L.load().hs_raster_stats(buf, 1)
it, test, q, c, empty, full, batches, _ = list(buf)[:8]
hist = list(buf)[8:15]
print(f"forward: iterations {it}, live pixel slots per iteration {test / max(it, 1):.1f} of 64, "
      f"iterations with no composited pixel {empty} ({empty / max(it, 1) * 100:.1f}%), composited pixels per iteration "
      f"{c / max(it, 1):.1f}")
print(f"keys {tr.last_total}  warp-iters {it}  per key {it / tr.last_total:.2f}  pixel-tests {test} "
      f"({test / max(it, 1):.1f} per iter of 64 slots)  q-pass {q} ({q / max(test, 1) * 100:.1f}%)  contrib {c} "
      f"({c / max(test, 1) * 100:.1f}%)  no-q iters {empty} ({empty / max(it, 1) * 100:.1f}%)  full-cover iters {full} "
      f"({full / max(it, 1) * 100:.1f}%)  batches {batches}")
tot = max(sum(hist), 1)
print("adjoint iterations by contributing lanes [0,1,2,3-4,5-8,9-16,17-32]:", hist,
      [f"{h / tot * 100:.1f}%" for h in hist])
