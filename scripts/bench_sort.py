"""Micro-benchmark of the binning sort on the C2 key list (CUDA events)."""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS, make_trainer  # noqa: E402
from paper_2503_12886_b200 import _lib as L  # noqa: E402
from paper_2503_12886_b200.device import _p, _stream  # noqa: E402


def main(reps=20):
    tr, d, wl = make_trainer(CONFIGS["C2"])
    tr.step(d["thetas"], d["targets"], d["frames"], d["cameras"], d["backgrounds"])
    bn = tr.binner
    total = tr.last_total
    mask = bn.sort_mask(tr.tile_bits, tr.frame_bits)
    s = _stream()

    def emit():
        L.call("hs_bin_emit", tr.B, tr.av.N, tr.W, tr.H, _p(tr.records), _p(tr.depth), _p(tr.counts),
               _p(bn.offsets), None, _p(bn.keys), _p(bn.vals), s)

    def sort():
        alt = ctypes.c_int(0)
        L.call("hs_sort_pairs", total, ctypes.c_uint64(mask), _p(bn.keys), _p(bn.vals), _p(bn.keys_alt),
               _p(bn.vals_alt), _p(bn.ws), bn.ws.numel(), ctypes.byref(alt), s)

    for _ in range(3):
        emit()
        sort()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    te = ts = 0.0
    for _ in range(reps):
        ev[0].record()
        emit()
        ev[1].record()
        sort()
        ev[2].record()
        ev[2].synchronize()
        te += ev[0].elapsed_time(ev[1])
        ts += ev[1].elapsed_time(ev[2])
    print(f"keys {total} mask {mask:#x} passes {sum(1 for sh in range(0, 64, 8) if (mask >> sh) & 0xFF)} "
          f"emit {te / reps * 1000:.1f} us sort {ts / reps * 1000:.1f} us")


if __name__ == "__main__":
    main()
