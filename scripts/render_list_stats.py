import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from bench_support import synth
from paper_2503_12886_b200.device import AvatarParams, DeviceRig, Trainer
wl = synth.make_workload(317, 64, 512, distinct_frames=8)
av = wl.avatar
dev = AvatarParams.from_host(type("G", (), {a: av.base[a] for a in av.base})(), av.deltas, av.mlp, av.tri_index, av.barycentric)
tr = Trainer(dev, 512, 512, 64, color_init=False, rig=DeviceRig(wl.rig))
th = torch.from_numpy(np.asarray(wl.thetas, np.float32)).cuda()
cams = torch.from_numpy(np.tile(wl.camera.packed(), (64, 1))).cuda()
bg = torch.zeros(64, 3, device="cuda"); out = torch.empty(64, 512, 512, 3, device="cuda")
tr.render(th, None, cams, bg, out); torch.cuda.synchronize()
keys, vals, ranges, tile_bits, tiles = tr.binner.result
r = ranges.view(-1, 2).cpu().numpy().astype(np.int64)
ln = r[:, 1] - r[:, 0]; ln = ln[ln > 0]; tot = ln.sum()
print("keys", tot, "lists", ln.size, "mean", ln.mean(), "max", ln.max())
for lo, hi in [(1, 32), (33, 64), (65, 128), (129, 256), (257, 512), (513, 1024), (1025, 8192), (8193, 1 << 40)]:
    m = (ln >= lo) & (ln <= hi)
    print(f"  {lo:5d}..{hi:<8d} lists {m.sum():6d}  entries {ln[m].sum() / tot * 100:5.1f}%")
