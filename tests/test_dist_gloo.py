"""Multi-process (world_size 2, gloo, CPU) checks of the data-parallel design.

The device kernels need a GPU; what is tested here is the decomposition the
multi-GPU path relies on, with the float64 oracle standing in for each rank's
local work:
  * each rank renders its own frames with image gradients scaled by 1/B_global,
    and ONE allreduce-sum of the [g_base | g_deltas | g_mlp] buffer reproduces the
    single-process full-batch gradient, Adam update and parameters bitwise-close;
  * the colour-init winner across ranks is an allreduce-MAX over the packed int64
    (float_bits(max_weight) << 32 | 0xFFFFFFFF - global_frame), which equals the
    reference's first-max argmax over the concatenated frame batch
    (S/train.py:266-268), ties included -- the same encoding as hs_color_pack.
"""
import os
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def pack(maxw_local, frame_offset, visited):
    """Python mirror of hs_color_pack (hs_model.cu)."""
    B, N = maxw_local.shape
    best = np.zeros(N, np.uint64)
    for b in range(B):
        w = np.maximum(maxw_local[b].astype(np.float32), 0).view(np.uint32).astype(np.uint64)
        v = (w << np.uint64(32)) | np.uint64(0xFFFFFFFF - (frame_offset + b))
        best = np.maximum(best, v)
    best[visited] = 0
    return best.astype(np.int64)


def unpack(packed):
    v = packed.astype(np.uint64)
    w = (v >> np.uint64(32)).astype(np.uint32).view(np.float32)
    f = (np.uint64(0xFFFFFFFF) - (v & np.uint64(0xFFFFFFFF))).astype(np.int64)
    return w, f


def _workload():
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
    import oracle as O
    from bench_support import synth
    wl = synth.make_workload(16, 4, 32, K=3, hidden=16, seed=3)
    av = wl.avatar
    f = lambda a: np.asarray(a, np.float32).astype(np.float64)
    attrs = ("position", "rotation", "scale", "opacity", "color")
    model = O.Model(O.GSet(*(f(av.base[a]) for a in attrs)), f(av.deltas), {k: f(v) for k, v in av.mlp.items()},
                    av.tri_index, f(av.barycentric))
    c = wl.camera
    cam = O.Cam(c.fx, c.fy, c.cx, c.cy, np.asarray(c.rotation, np.float64), np.asarray(c.translation, np.float64),
                c.width, c.height)
    frames = [O.Frames(m.rotation, m.quat, m.tri_vertices) for m in wl.mesh]
    images = wl.targets.astype(np.float64) / 255.0
    return O, model, cam, frames, images, wl


def _flat(g_base14, g_deltas, g_mlp):
    return np.concatenate([g_base14.ravel(), g_deltas.ravel()] + [g_mlp[k].ravel() for k in sorted(g_mlp)])


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        O, model, cam, frames, images, wl = _workload()
        B = len(frames)
        per = B // world
        sl = slice(rank * per, (rank + 1) * per)

        def allreduce(g_base14, g_deltas, g_mlp):
            keys = sorted(g_mlp)
            flat = torch.from_numpy(_flat(g_base14, g_deltas, g_mlp).copy())
            dist.all_reduce(flat, op=dist.ReduceOp.SUM)
            v = flat.numpy()
            o = 0
            gb = v[o:o + g_base14.size].reshape(g_base14.shape); o += g_base14.size
            gd = v[o:o + g_deltas.size].reshape(g_deltas.shape); o += g_deltas.size
            gm = {}
            for k in keys:
                gm[k] = v[o:o + g_mlp[k].size].reshape(g_mlp[k].shape); o += g_mlp[k].size
            return gb, gd, gm

        state = O.State(model, cam, color_init=False)
        O.train_step(state, wl.thetas[sl], images[sl], frames[sl], wl.backgrounds[sl], global_batch=B,
                     reduce_fn=allreduce)
        g = state.last_grads
        np.save(os.path.join(out_dir, f"grads{rank}.npy"),
                np.concatenate([np.concatenate([getattr(g[0], a).ravel() for a in
                                                ("position", "rotation", "scale", "opacity", "color")]),
                                g[1].ravel()] + [g[2][k].ravel() for k in sorted(g[2])]))
        np.save(os.path.join(out_dir, f"params{rank}.npy"), model.base.position)
        # colour-init winner: packed allreduce-MAX
        rng = np.random.default_rng(7)
        maxw = rng.uniform(0, 1, (B, 64)).astype(np.float32)
        maxw[:, :8] = 0.5                        # exact ties across frames and ranks
        visited = np.zeros(64, bool)
        visited[60:] = True
        packed = torch.from_numpy(pack(maxw[sl], rank * per, visited))
        dist.all_reduce(packed, op=dist.ReduceOp.MAX)
        np.save(os.path.join(out_dir, f"packed{rank}.npy"), packed.numpy())
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def dist_run(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("dist"))
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    return out


def test_sharded_gradients_match_full_batch(dist_run):
    O, model, cam, frames, images, wl = _workload()
    state = O.State(model, cam, color_init=False)
    O.train_step(state, wl.thetas, images, frames, wl.backgrounds)
    g = state.last_grads
    full = np.concatenate([np.concatenate([getattr(g[0], a).ravel() for a in
                                           ("position", "rotation", "scale", "opacity", "color")]),
                           g[1].ravel()] + [g[2][k].ravel() for k in sorted(g[2])])
    g0 = np.load(os.path.join(dist_run, "grads0.npy"))
    g1 = np.load(os.path.join(dist_run, "grads1.npy"))
    assert np.array_equal(g0, g1)                       # replicas identical after the allreduce
    np.testing.assert_allclose(g0, full, rtol=1e-12, atol=1e-15)
    p0 = np.load(os.path.join(dist_run, "params0.npy"))
    p1 = np.load(os.path.join(dist_run, "params1.npy"))
    assert np.array_equal(p0, p1)                       # no broadcast needed: Adam is elementwise
    np.testing.assert_allclose(p0, model.base.position, rtol=1e-12, atol=1e-15)


def test_colour_init_packed_argmax_equals_first_max(dist_run):
    rng = np.random.default_rng(7)
    B = 4
    maxw = rng.uniform(0, 1, (B, 64)).astype(np.float32)
    maxw[:, :8] = 0.5
    visited = np.zeros(64, bool)
    visited[60:] = True
    p0 = np.load(os.path.join(dist_run, "packed0.npy"))
    p1 = np.load(os.path.join(dist_run, "packed1.npy"))
    assert np.array_equal(p0, p1)
    w, f = unpack(p0)
    best = np.argmax(maxw, axis=0)                      # first max wins (np.argmax)
    live = ~visited
    assert np.array_equal(f[live], best[live])
    assert np.array_equal(w[live], maxw[best, np.arange(64)][live])
    assert np.all(f[:8] == 0)                           # ties resolve to the lowest global frame
    assert np.all(p0[visited] == 0)


def test_pack_order_is_monotone_in_int64():
    # the signed int64 MAX must order (weight, -frame) lexicographically
    ws = np.float32([0.0, 1e-30, 0.1, 0.1, 0.5, 1.0])
    fr = [3, 2, 7, 1, 0, 9]
    vals = [int(pack(np.array([[w]]), f, np.zeros(1, bool))[0]) for w, f in zip(ws, fr)]
    assert all(v >= 0 for v in vals)
    order = sorted(range(len(vals)), key=lambda i: vals[i])
    assert order == [0, 1, 2, 3, 4, 5]                  # 0.1@frame7 < 0.1@frame1
