"""The data-parallel Trainer path on the device, on ONE GPU.

Two processes share cuda:0 and a gloo process group (host-mediated allreduce, so no
kernel ever waits on another rank).  Each rank steps on half the frame batch with
gradients scaled by 1/B_global and the flat gradient allreduced; the colour init
uses the packed allreduce-MAX path (hs_color_pack / hs_color_select /
hs_color_apply).  The result must match one process stepping on the whole batch
(fused hs_color_init) within fp32 reduction-order tolerance, and the two replicas
must stay bitwise identical.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ATTRS = ("position", "rotation", "scale", "opacity", "color")


def _setup(B):
    sys.path[:0] = [ROOT]
    from bench_support import synth
    wl = synth.make_workload(48, B, 96, K=6, hidden=32, seed=5)
    return wl


def _trainer(wl, B, pg=None, global_batch=None, frame_offset=0):
    from paper_2503_12886_b200.device import AvatarParams, Trainer
    av = wl.avatar
    dev = AvatarParams.from_host(type("G", (), {a: av.base[a] for a in ATTRS})(), av.deltas, av.mlp, av.tri_index,
                                 av.barycentric)
    return Trainer(dev, 96, 96, B, process_group=pg, global_batch=global_batch, frame_offset=frame_offset)


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B = 4
        wl = _setup(B)
        per = B // world
        sl = slice(rank * per, (rank + 1) * per)
        tr = _trainer(wl, per, dist.group.WORLD, global_batch=B, frame_offset=rank * per)
        cams = np.tile(wl.camera.packed(), (per, 1))
        for step in range(2):
            tr.step_from_host(wl.thetas[sl], wl.targets[sl], wl.frames[sl], cams, wl.backgrounds[sl])
            torch.cuda.synchronize()
            if step == 0:       # the allreduced gradient Adam consumed
                np.save(os.path.join(out, f"grads{rank}.npy"), tr.grads.cpu().numpy())
        np.save(os.path.join(out, f"params{rank}.npy"), tr.av.params.cpu().numpy())
        np.save(os.path.join(out, f"visited{rank}.npy"), tr.visited.cpu().numpy())
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def run_dist(tmp_path_factory):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    from paper_2503_12886_b200 import build
    build.build()
    out = str(tmp_path_factory.mktemp("gdist"))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    return out


def test_two_rank_step_matches_single_rank(run_dist):
    """Rank grads after the first step's allreduce equal the single-rank batch gradient
    entrywise (rel 1e-4, floor 1e-5 max|g|: only the summation order differs); the
    replicas are bitwise identical; parameters after two Adam steps match the
    single-rank run to a small fraction of the learning rate."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from gpu_helpers import rel_fail
    B = 4
    wl = _setup(B)
    tr = _trainer(wl, B)
    cams = np.tile(wl.camera.packed(), (B, 1))
    for step in range(2):
        tr.step_from_host(wl.thetas, wl.targets, wl.frames, cams, wl.backgrounds)
        torch.cuda.synchronize()
        if step == 0:
            g_ref = tr.grads.cpu().numpy()
    ref = tr.av.params.cpu().numpy()
    g0 = np.load(os.path.join(run_dist, "grads0.npy"))
    assert np.array_equal(g0, np.load(os.path.join(run_dist, "grads1.npy")))
    n, K = tr.av.N, tr.av.K
    for name, sl in (("base", slice(0, 14 * n)), ("deltas", slice(14 * n, 14 * n + 10 * K * n)),
                     ("mlp", slice(14 * n + 10 * K * n, None))):
        nbad, worst, need = rel_fail(g0[sl], g_ref[sl], rtol=1e-4)
        assert nbad == 0, (name, worst, need)
    p0 = np.load(os.path.join(run_dist, "params0.npy"))
    p1 = np.load(os.path.join(run_dist, "params1.npy"))
    assert np.array_equal(p0, p1)
    v0 = np.load(os.path.join(run_dist, "visited0.npy"))
    assert np.array_equal(v0, np.load(os.path.join(run_dist, "visited1.npy")))
    assert (v0 != tr.visited.cpu().numpy()).sum() <= 2
    assert v0.any()
    # Adam's update is lr * m / (sqrt(v) + eps): entries whose gradient is at the
    # roundoff level (|g| ~ eps) can move by up to ~lr; everything else agrees closely
    d = np.abs(p0 - ref)
    assert np.mean(d > 1e-5) < 1e-3, np.sort(d)[-10:]
    assert d.max() < 2.6e-2 * 2, d.max()
