"""Device-resident step loop vs step_from_host loop, alternating, to find where the
device-timed value loses time (host bubbles after the step's sync)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import bench

cfg = bench.CONFIGS["C2"]
tr, d, wl = bench.make_trainer(cfg)
h = {k: v.cpu().numpy() for k, v in d.items()}
hb = (h["thetas"], h["targets"], None, h["cameras"], h["backgrounds"])
K = int(sys.argv[1]) if len(sys.argv) > 1 else 50


def dev_loop():
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(K):
        tr.step(d["thetas"], d["targets"], None, d["cameras"], d["backgrounds"])
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / K


def dev_loop_wall():
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(K):
        tr.step(d["thetas"], d["targets"], None, d["cameras"], d["backgrounds"])
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1000 / K


def e2e_loop():
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(K):
        tr.step_from_host(*hb, prefetch=hb)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1000 / K


for _ in range(5):
    tr.step(d["thetas"], d["targets"], None, d["cameras"], d["backgrounds"])
for r in range(3):
    print(f"rep {r}: device {dev_loop():.4f} ms  device-wall {dev_loop_wall():.4f} ms  e2e {e2e_loop():.4f} ms",
          flush=True)
# host time per step phase
import cProfile
import pstats
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    tr.step(d["thetas"], d["targets"], None, d["cameras"], d["backgrounds"])
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
