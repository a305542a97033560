import sys, os
sys.path.insert(0, os.getcwd())
import torch
from bench import CONFIGS, make_trainer
for ci in (True, False):
    tr, d, wl = make_trainer(CONFIGS["C2"])
    tr.color_init = ci
    for _ in range(5):
        tr.step(d["thetas"], d["targets"], None, d["cameras"], d["backgrounds"])
    torch.cuda.synchronize()
    tr.enable_profiling(True)
    for _ in range(10):
        tr.step(d["thetas"], d["targets"], None, d["cameras"], d["backgrounds"])
    st = tr.stage_ms()
    print("color_init", ci, "visited", int(tr.visited.sum()), "of", tr.av.N, {k: round(v / 10, 4) for k, v in st.items() if v / 10 > 0.03})
