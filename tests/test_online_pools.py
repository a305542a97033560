"""Host bookkeeping of the online pools (paper_2503_12886_b200/online.py) against the
reference's SamplePools / sample_batch (S/stream.py:27-90; golden pools.npz made by
tests/golden/make_golden.py from the reference with the same seeded rng), plus the
device-slot invariants: a frame's slot is released exactly when it leaves both pools."""
import numpy as np
import pytest

from conftest import golden
from paper_2503_12886_b200.online import FrameRef, SamplePools, sample_batch

MODES = {"full": (5, 12, True, 0.7), "no_global": (5, 12, False, 1.0), "no_local": (1, 12, True, 1.0)}


@pytest.mark.parametrize("mode", sorted(MODES))
def test_pools_match_reference(mode):
    d = golden("pools")
    lc, gc, keep, eta = MODES[mode]
    rng = np.random.default_rng(3)
    free = list(range(lc + gc + 1))
    live = set()

    def release(ref):
        assert ref.slot in live
        live.remove(ref.slot)
        free.append(ref.slot)

    pools = SamplePools(lc, gc, keep_evicted=keep, release=release)
    k = 0
    for i in range(1, 81):
        slot = free.pop(0)
        assert slot not in live
        live.add(slot)
        pools.process_frame(FrameRef(i, slot), rng)
        loc = [r.index for r in pools.local]
        glo = [r.index for r in pools.global_pool]
        assert loc == [x for x in d[f"{mode}.local"][i - 1] if x] or (loc == [] and not d[f"{mode}.local"][i - 1].any())
        assert glo == [x for x in d[f"{mode}.global"][i - 1] if x]
        assert [pools.evictions, pools.discarded, pools.reservoir_inserts] == list(d[f"{mode}.counters"][i - 1])
        # every live slot belongs to exactly one pooled frame
        assert sorted(r.slot for r in list(pools.local) + pools.global_pool) == sorted(live)
        if i % 3 == 0:
            picks = sample_batch(pools, 8, eta, rng)
            assert [r.index for r in picks] == list(d[f"{mode}.picks"][k])
            rng.uniform(0.0, 1.0, size=(8, 3))
            k += 1


def test_sample_batch_errors_and_order():
    rng = np.random.default_rng(0)
    pools = SamplePools(2, 3)
    with pytest.raises(ValueError, match="both pools are empty"):
        sample_batch(pools, 4, 0.7, rng)
    with pytest.raises(ValueError, match="does not follow"):
        pools.process_frame(FrameRef(2, 0), rng)


def _shard_worker(rank, world, port, out):
    """One rank of the data-parallel online loop's host side (OnlineTrainer._draw):
    identical pools and rng on every rank, the global draw, this rank's slice."""
    import os
    import torch
    import torch.distributed as dist
    from paper_2503_12886_b200.online import OnlineConfig, draw_step
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = OnlineConfig(batch_size=8, local_capacity=5, global_capacity=12)
        B = cfg.batch_size // world
        rng = np.random.default_rng(cfg.seed)
        pools = SamplePools(cfg.local_capacity, cfg.global_capacity)
        rows = []
        for i in range(1, 61):
            pools.process_frame(FrameRef(i, i), rng)
            for _ in range(2):
                batch, bgs = draw_step(pools, cfg, rng, cfg.batch_size)
                mine = batch[rank * B:(rank + 1) * B]
                rows.append(np.concatenate([[r.index for r in mine], bgs[rank * B:(rank + 1) * B].ravel()]))
        t = torch.from_numpy(np.stack(rows))
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        if rank == 0:
            np.save(os.path.join(out, "gathered.npy"), np.stack([p.numpy() for p in parts]))
    finally:
        dist.destroy_process_group()


def test_sharded_online_draws_match_single_process(tmp_path):
    """BASELINE configs[4] on N ranks: the ranks' slices, concatenated in rank order,
    are exactly the single-process draws of S/stream.py:124-140 (frames, then the
    backgrounds) for the whole batch."""
    import socket
    import torch.multiprocessing as mp
    from paper_2503_12886_b200.online import OnlineConfig, draw_step
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    world = 2
    mp.spawn(_shard_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    got = np.load(tmp_path / "gathered.npy")               # (world, steps, B + 3B)
    cfg = OnlineConfig(batch_size=8, local_capacity=5, global_capacity=12)
    B = cfg.batch_size // world
    rng = np.random.default_rng(cfg.seed)
    pools = SamplePools(cfg.local_capacity, cfg.global_capacity)
    k = 0
    for i in range(1, 61):
        pools.process_frame(FrameRef(i, i), rng)
        for _ in range(2):
            batch, bgs = draw_step(pools, cfg, rng, cfg.batch_size)
            idx = np.concatenate([got[r, k, :B] for r in range(world)])
            bg = np.concatenate([got[r, k, B:].reshape(B, 3) for r in range(world)])
            assert np.array_equal(idx, [r.index for r in batch])
            assert np.array_equal(bg, bgs)
            k += 1
