"""Kernel-level timing of one stage of the C2 step in isolation (after 100 steps):
    HS_B200_LIB=... python scripts/stage_ab.py <stage> [reps] [flush]
stage: blend_fwd | blend_bwd | project_fwd | project_bwd | adam | fill | copy.  flush=1 writes
256 MB between launches (cold L2, but the evicted lines are dirty: their write-back lands in
the timed kernel), flush=2 reads 256 MB (cold and clean), else the inputs may be L2-resident."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import bench
from paper_2503_12886_b200 import _lib as L
from paper_2503_12886_b200.device import _p

stage = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
flush_on = len(sys.argv) > 3 and sys.argv[3] in ("1", "2")
flush_read = len(sys.argv) > 3 and sys.argv[3] == "2"     # 2: evict L2 by reading (no dirty lines left)
tr, d, wl = bench.make_trainer(bench.CONFIGS["C2"])
nsteps = int(os.environ.get("RAB_STEPS", "100"))
for _ in range(nsteps):
    tr.step(d["thetas"], d["targets"], None, d["cameras"], d["backgrounds"])
if nsteps == 0:               # (diagnostic builds that cannot train: blend inputs only)
    tr.psi.normal_()
torch.cuda.synchronize()
av = tr.av
N, K, B = av.N, av.K, tr.B
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
flush = torch.empty(256 << 18, dtype=torch.float32, device="cuda")
frames = tr._last_frames
F = frames.shape[-2] if frames is not None else 0


bn = tr.binner
bn.depth_range_scratch = torch.tensor([0xFFFFFFFF, 0], dtype=torch.int64, device="cuda").to(torch.int32)
if bn.result is not None:
    keys_, vals_, ranges_, tile_bits_, tiles_ = bn.result
    nseg = B << tile_bits_


copy_src = torch.empty(37 << 18, dtype=torch.float32, device="cuda").fill_(1.0)
copy_dst = torch.empty_like(copy_src)
read_src = torch.empty(42 << 18, dtype=torch.float32, device="cuda").fill_(1.0)
read_out = torch.empty((), dtype=torch.float32, device="cuda")


def prep():
    if stage == "project_fwd":   # the fused tile count adds into zeroed counters (untimed)
        bn.tile_counts.zero_()
    if stage == "fill":        # the fill consumes the scan's cursors: reset them (untimed)
        bn.cursor[:nseg].copy_(ranges_.view(-1, 2)[:, 0])


def call():
    if stage == "fill":
        rects = bn.tile_rects_buffer(B, N, tr.W, tr.H)
        L.call("hs_tile_fill", B, N, tr.W, tr.H, _p(tr.records), _p(tr.counts), _p(rects), _p(tr.depth),
               _p(ranges_), _p(bn.cursor), _p(bn.lists), _p(bn.list_counts), bn.list_half, _p(bn.summary), bn.cap,
               None, _p(bn.vals), 0, bn.fork, s)
    elif stage == "project_fwd":
        rects = bn.tile_rects_buffer(B, N, tr.W, tr.H)
        L.call("hs_project_avatar_fwd", B, N, F, tr.W, tr.H, _p(tr.raw10), _p(av.base14), _p(av.tri_index),
               _p(av.barycentric), _p(frames), _p(d["cameras"]), _p(tr.records), _p(tr.depth), _p(tr.counts),
               _p(tr.block_sums), _p(bn.depth_range_scratch), _p(tr.radius), _p(tr.g_splat), None, None,
               _p(bn.tile_counts), _p(rects), _p(tr.err), s)
    elif stage == "copy":        # calibration: a 37 MB device copy (74 MB of traffic, blend_fwd's size)
        copy_dst.copy_(copy_src)
    elif stage == "read":        # calibration: a 42 MB read (blend_fwd's loads)
        read_out.copy_(read_src.sum())
    elif stage == "blend_fwd":
        L.call("hs_blend_fwd", N, K, B, _p(av.base14), _p(av.deltas), _p(tr.psi), _p(tr.raw10), s)
    elif stage == "blend_bwd":
        n = ctypes.c_int(0)
        L.call("hs_blend_bwd", N, K, B, _p(av.deltas), _p(tr.psi), _p(tr.g_raw14), _p(tr.grads),
               _p(tr.grads[14 * N:]), _p(tr.gpsi_partials), ctypes.byref(n), s)
    elif stage == "project_bwd":
        L.call("hs_project_avatar_bwd", B, N, F, _p(tr.raw10), _p(av.base14), _p(av.tri_index), _p(av.barycentric),
               _p(frames), _p(d["cameras"]), _p(tr.g_splat), 1, _p(tr.g_raw14), s)
    elif stage == "adam":
        tr._adam(0, 14 * N + 10 * K * N, 0, s)
    else:
        raise SystemExit("unknown stage")


times = []
for r in range(reps + 3):
    if flush_read:
        flush_sum = flush.sum()
    elif flush_on:
        flush.fill_(1.0)
    prep()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    call()
    b.record()
    b.synchronize()
    if r >= 3:
        times.append(a.elapsed_time(b))
t = np.array(times) * 1000
print(f"{os.path.basename(os.environ.get('HS_B200_LIB', 'default'))} {stage} flush={int(flush_on)}: "
      f"median {np.median(t):.1f} us (p10 {np.percentile(t, 10):.1f}, p90 {np.percentile(t, 90):.1f})")
