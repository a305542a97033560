"""Kernel timeline of the render bench (BASELINE configs[2]: 100,489 Gaussians, 512^2, batch 64)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

from bench_support import synth
from paper_2503_12886_b200.device import AvatarParams, DeviceRig, Trainer

wl = synth.make_workload(317, 64, 512, distinct_frames=8)
av = wl.avatar
dev = AvatarParams.from_host(type("G", (), {a: av.base[a] for a in av.base})(), av.deltas, av.mlp, av.tri_index,
                             av.barycentric)
tr = Trainer(dev, 512, 512, 64, color_init=False, rig=DeviceRig(wl.rig))
th = torch.from_numpy(np.asarray(wl.thetas, np.float32)).cuda()
cams = torch.from_numpy(np.tile(wl.camera.packed(), (64, 1))).cuda()
bg = torch.zeros(64, 3, device="cuda")
out = torch.empty(64, 512, 512, 3, device="cuda")
for _ in range(5):
    tr.render(th, None, cams, bg, out)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    tr.render(th, None, cams, bg, out)
    torch.cuda.synchronize()
path = os.path.join(ROOT, "gpurun_out", "render_tl.json")
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]
for e in ev:
    print(f"{e['ts'] - t0:9.1f} {e['dur']:8.1f}  {e['name'][:80]}")
print("keys", tr.last_total)
