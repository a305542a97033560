"""A few C2 training steps (for ncu captures): python scripts/prof_step.py [steps] [config]."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import bench

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
cfg = bench.CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "C2"]
tr, d, wl = bench.make_trainer(cfg)
for _ in range(steps):
    tr.step(d["thetas"], d["targets"], None, d["cameras"], d["backgrounds"])
torch.cuda.synchronize()
print("ok", tr.last_total)
