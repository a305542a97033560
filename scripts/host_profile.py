"""cProfile of the host side of the C2 training step (where the ~1 ms of Python goes)."""
import cProfile
import os
import pstats
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS, make_trainer  # noqa: E402

tr, d, wl = make_trainer(CONFIGS["C2"])
args = (d["thetas"], d["targets"], None, d["cameras"], d["backgrounds"])
for _ in range(10):
    tr.step(*args)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    tr.step(*args)
pr.disable()
torch.cuda.synchronize()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(30)
