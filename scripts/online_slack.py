"""Online step (bench.online_rate's setup): wall clock per optimize_once vs the GPU's own
time for the same steps (CUDA events), and the step's device-resident time at B=10."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench_support import synth
from paper_2503_12886_b200.device import AvatarParams, DeviceRig, Trainer
from paper_2503_12886_b200.online import OnlineConfig, OnlineTrainer
B = 10
wl = synth.make_workload(224, 120, 512)
av = wl.avatar
dev = AvatarParams.from_host(type("G", (), {a: av.base[a] for a in av.base})(), av.deltas, av.mlp, av.tri_index, av.barycentric)
tr = Trainer(dev, 512, 512, B, rig=DeviceRig(wl.rig))
on = OnlineTrainer(tr, wl.camera.packed(), OnlineConfig(batch_size=B, steps_per_frame=0, check_every=10_000))
for i in range(120):
    on.ingest(i + 1, wl.targets[i], wl.thetas[i])
for _ in range(10):
    on.optimize_once()
torch.cuda.synchronize()
n = 200
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter(); s.record()
for _ in range(n):
    on.optimize_once()
e.record(); torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"online: wall {1e3 * (t1 - t0) / n:.3f} ms/step, GPU events {s.elapsed_time(e) / n:.3f} ms/step")
# host time of the draw + gather part alone
t0 = time.perf_counter()
for _ in range(n):
    on._draw()
t1 = time.perf_counter()
print(f"draw alone: {1e6 * (t1 - t0) / n:.1f} us")
# device-resident steps on the gathered batch
th, tg = on.thetas.clone(), on.targets.clone()
torch.cuda.synchronize()
s.record()
for _ in range(n):
    tr.step(th, tg, None, on.cameras, on.bgs)
e.record(); torch.cuda.synchronize()
print(f"device-resident B=10 step: {s.elapsed_time(e) / n:.3f} ms")
