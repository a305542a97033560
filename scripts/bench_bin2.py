"""Micro-benchmark of the two-level binning stages on the C2 workload (CUDA events)."""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS, make_trainer  # noqa: E402
from paper_2503_12886_b200 import _lib as L  # noqa: E402
from paper_2503_12886_b200.device import _p, _stream, key_layout  # noqa: E402


def main(reps=30):
    tr, d, wl = make_trainer(CONFIGS["C2"])
    for _ in range(3):
        tr.step(d["thetas"], d["targets"], None, d["cameras"], d["backgrounds"])
    torch.cuda.synchronize()
    bn, B, N = tr.binner, tr.B, tr.av.N
    total = tr.last_total
    tiles_x, tiles_y, tiles, tile_bits, frame_bits = key_layout(B, tr.W, tr.H)
    s = _stream()
    k32, k32a = bn.keys.view(torch.int32), bn.keys_alt.view(torch.int32)
    nr = B << tile_bits
    mask = (1 << (tile_bits + frame_bits)) - 1
    stages = {
        "depth_order": lambda: L.call("hs_depth_order", B * N, _p(tr.depth), _p(bn.depth_range), _p(bn.order),
                                      _p(bn.order_alt), _p(bn.dkeys_a), _p(bn.dkeys_b), _p(bn.dws),
                                      bn.dws.numel(), s),
        "emit_sorted": lambda: L.call("hs_bin_emit_sorted", B, N, tr.W, tr.H, _p(tr.records), _p(tr.counts), None,
                                      _p(bn.order), _p(bn.sblock_sums), _p(bn.sblock_offs), _p(k32),
                                      _p(bn.vals), s),
        "sort32": lambda: L.call("hs_sort_pairs32", total, ctypes.c_uint32(mask),
                                 _p(k32), _p(bn.vals), _p(k32a), _p(bn.vals_alt), _p(bn.ws), bn.ws.numel(),
                                 ctypes.byref(ctypes.c_int(0)), s),
        "ranges32": lambda: (bn.ranges[:2 * nr].zero_(),
                             L.call("hs_tile_ranges32", total, _p(k32a), _p(bn.ranges), s)),
    }
    ev = {k: [torch.cuda.Event(enable_timing=True) for _ in range(2)] for k in stages}
    acc = {k: 0.0 for k in stages}
    for r in range(reps + 3):
        for k, f in stages.items():
            ev[k][0].record()
            f()
            ev[k][1].record()
        torch.cuda.synchronize()
        if r >= 3:
            for k in stages:
                acc[k] += ev[k][0].elapsed_time(ev[k][1])
    print(f"items {B * N} keys {total}: " + ", ".join(f"{k} {v / reps * 1000:.1f} us" for k, v in acc.items()))


if __name__ == "__main__":
    main()
