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
