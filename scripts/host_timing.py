"""Host-side timing of the C2 training step: wall time per step, time the host spends
waiting at the step's one sync (Binner.bin_tiles), and the host time to enqueue the
work before / after it -- shows whether the GPU ever waits for the host."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS, make_trainer  # noqa: E402

tr, d, wl = make_trainer(CONFIGS["C2"])
args = (d["thetas"], d["targets"], None, d["cameras"], d["backgrounds"])
for _ in range(10):
    tr.step(*args)
torch.cuda.synchronize()
orig = torch.cuda.Event.synchronize
wait = [0.0]


def timed_sync(self):
    t = time.perf_counter()
    orig(self)
    wait[0] += time.perf_counter() - t


torch.cuda.Event.synchronize = timed_sync
steps = 100
t0 = time.perf_counter()
for _ in range(steps):
    tr.step(*args)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"wall per step {(t2 - t0) / steps * 1e6:.0f} us (host loop {(t1 - t0) / steps * 1e6:.0f} us), "
      f"host waiting at the sync {wait[0] / steps * 1e6:.0f} us -> host busy {((t1 - t0) - wait[0]) / steps * 1e6:.0f} us")
