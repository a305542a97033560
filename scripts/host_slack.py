"""Host slack of the C2 step: how long the host waits at the step's one sync (the binning
summary read) -- time the host is ahead of the GPU.  A step whose host work exceeded the GPU's
would show ~0 wait and idle GPU gaps."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import bench

tr, d, wl = bench.make_trainer(bench.CONFIGS["C2"])
step = lambda: tr.step(d["thetas"], d["targets"], None, d["cameras"], d["backgrounds"])
for _ in range(100):
    step()
torch.cuda.synchronize()
waits = []
orig = torch.cuda.Event.synchronize


def timed_sync(self):
    t0 = time.perf_counter()
    orig(self)
    waits.append(time.perf_counter() - t0)


torch.cuda.Event.synchronize = timed_sync
n = 50
t0 = time.perf_counter()
for _ in range(n):
    step()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / n
torch.cuda.Event.synchronize = orig
w = sorted(waits)
print(f"{wall * 1e6:.0f} us/step wall; host waits at the sync: median {w[len(w) // 2] * 1e6:.0f} us, "
      f"min {w[0] * 1e6:.0f} us over {len(w)} syncs -> host busy ~{(wall - w[len(w) // 2]) * 1e6:.0f} us/step")
