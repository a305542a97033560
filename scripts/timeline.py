"""GPU timeline of a few C2 steps (torch.profiler / CUPTI: every kernel of the process,
ours included), printed per step as start offset, duration and stream -- finds the gaps
between kernels that the per-stage events cannot separate from host latency.
    python scripts/timeline.py [steps] [config]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from torch.profiler import ProfilerActivity, profile

import bench

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = bench.CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "C2"]
tr, d, wl = bench.make_trainer(cfg)
step = lambda: tr.step(d["thetas"], d["targets"], None, d["cameras"], d["backgrounds"])
for _ in range(300):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(steps):
        step()
    torch.cuda.synchronize()
path = os.path.join(ROOT, "gpurun_out", "timeline.json")
os.makedirs(os.path.dirname(path), exist_ok=True)
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]
busy_end = t0
gaps = 0.0
for e in ev:
    s, dur = e["ts"], e["dur"]
    gap = s - busy_end
    if gap > 0:
        gaps += gap
    name = e["name"].split("(")[0][-40:]
    print(f"{s - t0:9.1f} {dur:8.1f} gap {max(gap, 0):7.1f} stream {e['args'].get('stream', '?'):>4} {name}")
    busy_end = max(busy_end, s + dur)
span = busy_end - t0
print(f"span {span:.1f} us over {steps} steps = {span / steps:.1f} us/step; idle gaps {gaps:.1f} us "
      f"({gaps / steps:.1f} us/step)")
