"""Per-(frame, tile) list lengths of the C2 training workload: how the tile-major
binner's entries split over its sort classes (1 / <=32 / <=256 / <=8192 / longer)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS, make_trainer  # noqa: E402


def main():
    tr, d, wl = make_trainer(CONFIGS["C2"])
    for _ in range(3):
        tr.step(d["thetas"], d["targets"], None, d["cameras"], d["backgrounds"])
    torch.cuda.synchronize()
    keys, vals, ranges, tile_bits, tiles = tr.binner.result
    r = ranges.view(-1, 2).cpu().numpy().astype(np.int64)
    ln = r[:, 1] - r[:, 0]
    ln = ln[ln > 0]
    tot = ln.sum()
    print(f"keys {tot} lists {ln.size} mean {ln.mean():.1f} max {ln.max()}")
    for lo, hi in [(1, 1), (2, 32), (33, 256), (257, 1024), (1025, 4096), (4097, 8192), (8193, 1 << 40)]:
        m = (ln >= lo) & (ln <= hi)
        print(f"  {lo:5d}..{hi:<8d} lists {m.sum():6d}  entries {ln[m].sum() / tot * 100:5.1f}%")
    # depth-bit span and exact depth ties per list (the 32-bit list sort's conditions)
    N = tr.av.N
    v = vals.cpu().numpy().view(np.uint32).astype(np.int64)
    dep = tr.depth.cpu().numpy().view(np.uint32).astype(np.int64)
    span_hist, ties = {}, 0
    wide = 0
    for seg in np.nonzero(r[:, 1] > r[:, 0])[0]:
        a0, a1 = r[seg]
        b = seg >> tile_bits
        d = dep[b * N + v[a0:a1]]
        span = int(d.max() - d.min()).bit_length()
        span_hist[span] = span_hist.get(span, 0) + 1
        L = int(a1 - a0)
        ib = max(5, (max(L, 32) - 1).bit_length())
        t = np.unique(d).size < d.size
        ties += t
        wide += (span > 31 - ib) or t
    print("depth-bit span per list:", dict(sorted(span_hist.items())))
    print(f"lists with exact depth ties {ties}, lists the 32-bit sort declines {wide}")
    print("wide count on device:", int(tr.binner.list_counts[4]))


if __name__ == "__main__":
    main()
