"""Online training on device-resident frame pools (online.py).

* every step's gathered device batch (targets, thetas) equals the host frames of the
  batch the reference rule drew, and the step equals a plain Trainer.step on those
  host frames with the same backgrounds (first-step loss bit for bit);
* a short stream with small pools (eviction, reservoir replacement, slot reuse)
  trains with finite losses, logs one entry per step and tracks min L1 per frame;
* the three sampling modes run; the forgetting report covers every processed frame.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2503_12886_b200 import build
    build.build()


def _setup(B=4, frames=14, size=96, seed=0):
    from bench_support import synth
    from paper_2503_12886_b200.device import AvatarParams, DeviceRig, Trainer
    import oracle as O
    wl = synth.make_workload(40, frames, size, distinct_frames=frames, frames_seed=seed + 1)
    av = wl.avatar

    def trainer():
        dev = AvatarParams.from_host(O.GSet(*(av.base[a] for a in ("position", "rotation", "scale", "opacity",
                                                                       "color"))),
                                     av.deltas, av.mlp, av.tri_index, av.barycentric)
        return Trainer(dev, size, size, B, rig=DeviceRig(wl.rig))
    return wl, trainer


def test_gathered_batch_and_step_match_host_frames():
    from paper_2503_12886_b200.online import OnlineConfig, OnlineTrainer
    wl, make = _setup()
    cfg = OnlineConfig(batch_size=4, local_capacity=3, global_capacity=4, steps_per_frame=1, seed=5)
    on = OnlineTrainer(make(), wl.camera.packed(), cfg)
    for i in range(6):
        on.ingest(i + 1, wl.targets[i], wl.thetas[i])
    rng_state = on.rng.bit_generator.state
    on.optimize_once()
    torch.cuda.synchronize()
    # replay the draw on the host: which frames, which backgrounds
    from paper_2503_12886_b200.online import sample_batch
    rng = np.random.default_rng()
    rng.bit_generator.state = rng_state
    batch = sample_batch(on.pools, 4, cfg.eta, rng)
    bgs = rng.uniform(0.0, 1.0, size=(4, 3))
    idx = [r.index - 1 for r in batch]
    assert np.array_equal(on.targets.cpu().numpy(), wl.targets[idx])
    np.testing.assert_array_equal(on.thetas.cpu().numpy(), np.asarray(wl.thetas, np.float32)[idx])
    # the same step through a plain Trainer on host-provided frames
    tr = make()
    cams = torch.from_numpy(np.tile(wl.camera.packed(), (4, 1))).cuda()
    loss = tr.step(torch.from_numpy(np.asarray(wl.thetas, np.float32)[idx]).cuda(),
                   torch.from_numpy(wl.targets[idx]).cuda(), None, cams,
                   torch.from_numpy(bgs.astype(np.float32)).cuda())
    on.flush()
    assert on.log[0]["loss"] == float(loss[2 * 4].item())


@pytest.mark.parametrize("mode", ["full", "no_global", "no_local"])
def test_stream_trains(mode):
    from paper_2503_12886_b200.online import OnlineConfig, OnlineTrainer, forgetting_gap
    wl, make = _setup()
    cfg = OnlineConfig(batch_size=4, local_capacity=3, global_capacity=4, steps_per_frame=2, sampling=mode,
                       seed=1, check_every=5)
    on = OnlineTrainer(make(), wl.camera.packed(), cfg)
    stream = [(i + 1, wl.targets[i], wl.thetas[i]) for i in range(len(wl.targets))]
    log = on.run(stream)
    assert len(log) == 2 * len(stream)
    assert [e["step"] for e in log] == list(range(len(log)))
    assert all(np.isfinite(e["loss"]) for e in log)
    # slots: live frames + free slots partition the pool
    live = [r.slot for r in list(on.pools.local) + on.pools.global_pool]
    assert len(set(live)) == len(live)
    assert sorted(live + on.pool.free) == list(range(on.pool.capacity))
    rep = on.forgetting_report(wl.targets, wl.thetas)
    assert [r["frame"] for r in rep] == list(range(1, len(stream) + 1))
    assert all(np.isfinite(r["final_l1"]) for r in rep)
    seen = [r for r in rep if np.isfinite(r["min_l1"])]
    assert len(seen) >= 4
    assert np.isfinite(forgetting_gap(rep))
