# raster time with the colour-init variant (CI 3) vs none (CI 0) at the C2 steady state, and
# the fraction of Gaussians visited then
python - <<'PY'
import sys; sys.path.insert(0,'.')
import torch, bench
tr, d, wl = bench.make_trainer(bench.CONFIGS["C2"])
for _ in range(100):
    tr.step(d["thetas"], d["targets"], None, d["cameras"], d["backgrounds"])
torch.cuda.synchronize()
v = tr.visited.float().mean().item()
print("visited fraction after 100 steps:", v)
PY
for ci in 3 0 3 0; do echo -n "CI=$ci "; RAB_CI=$ci python scripts/raster_ab.py 30 | tail -1; done
