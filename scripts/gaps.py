"""Idle gaps on the compute stream of the C2 step: the Trainer's per-stage CUDA events
(enable_profiling; no CUPTI) give each stage's start / end on the GPU clock; printed per
stage in stream order as start offset, duration and the gap since the previous stage's
end.  The speculative raster launch is left on (its stage events then nest inside
bin_tiles: the raster line shows the real kernel)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import bench

tr, d, wl = bench.make_trainer(bench.CONFIGS["C2"])
step = lambda: tr.step(d["thetas"], d["targets"], None, d["cameras"], d["backgrounds"])
for _ in range(200):
    step()
torch.cuda.synchronize()
spec = os.environ.get("SPEC", "1") == "1"
tr.enable_profiling(True)
tr.profile_speculative = spec
t0 = torch.cuda.Event(enable_timing=True)
t0.record()
steps = 5
a = torch.cuda.Event(enable_timing=True)
b = torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(steps):
    step()
b.record()
torch.cuda.synchronize()
print(f"{a.elapsed_time(b) / steps * 1000:.1f} us/step with stage events")
ev = []
for name, lst in tr.events.items():
    for s, e in lst:
        if e is None:
            continue
        ev.append((t0.elapsed_time(s) * 1000, t0.elapsed_time(e) * 1000, name))
ev.sort()
prev_end = None
for s, e, name in ev[-40:]:
    gap = s - prev_end if prev_end is not None else 0.0
    print(f"{s:10.1f} {e - s:8.1f} gap {gap:7.1f}  {name}")
    prev_end = max(prev_end or 0.0, e)
