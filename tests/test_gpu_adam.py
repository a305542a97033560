"""Multi-tensor Adam through the C ABI.

* bucketed hs_adam_fused calls reproduce one full-range hs_adam bit for bit (the
  per-bucket update the multi-GPU step overlaps with the bucket allreduces), for
  float4 and scalar ranges;
* the update matches a numpy restatement of S/optim.py:28-40 with the per-group
  learning rates of S/train.py:184-199;
* colour init fused into the base bucket (ci_mode 1 / 2) equals hs_adam followed by
  hs_color_init / hs_color_apply -- parameters, visited flags and the init count;
* a colour-init bucket that splits the colour segment is rejected (ValueError).
"""
import ctypes

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


N, K, H, D = 1000, 5, 13, 16
BETAS, EPS = (0.9, 0.999), 1e-15


def _state(seed=0):
    from paper_2503_12886_b200 import _lib as L
    mlp = int(L.load().hs_mlp_size(H, D, K))
    total = 14 * N + 10 * K * N + mlp
    g = np.random.default_rng(seed)
    arr = lambda s=1.0: torch.from_numpy((g.standard_normal(total) * s).astype(np.float32)).cuda()
    return dict(p=arr(), g=arr(1e-2), m=arr(1e-3), v=torch.abs(arr(1e-4)), mlp=mlp, total=total)


def _lrs():
    return (ctypes.c_float * 9)(0.0008, 0.005, 0.0125, 0.025, 0.25, 4e-5, 2.5e-3, 6.25e-3, 1e-3)


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _adam_full(st, step):
    from paper_2503_12886_b200 import _lib as L
    L.call("hs_adam", N, K, st["mlp"], _p(st["p"]), _p(st["g"]), _p(st["m"]), _p(st["v"]), _lrs(), step,
           BETAS[0], BETAS[1], EPS, _stream())


def _adam_range(st, step, lo, hi, mode=0, B=0, maxw=None, wsums=None, packed=None, est4=None, visited=None,
                n_init=None, err=None, thr=0.1):
    from paper_2503_12886_b200 import _lib as L
    L.call("hs_adam_fused", N, K, st["mlp"], _p(st["p"]), _p(st["g"]), _p(st["m"]), _p(st["v"]), _lrs(), step,
           BETAS[0], BETAS[1], EPS, lo, hi, mode, B, _p(maxw), _p(wsums), _p(packed), _p(est4), ctypes.c_float(thr),
           _p(visited), _p(n_init), _p(err), _stream())


def _clone(st):
    return {k: (v.clone() if torch.is_tensor(v) else v) for k, v in st.items()}


def _buckets(total, aligned=True):
    b = [0, 14 * N]
    for k in range(0, K, 2):
        b.append(14 * N + 10 * N * min(K, k + 2))
    if not aligned:                     # odd boundaries inside the deltas: scalar path
        b.insert(2, 14 * N + 10 * N + 3)
    b.append(total)
    return list(zip(b[:-1], b[1:]))


@pytest.mark.parametrize("aligned", [True, False])
def test_bucketed_equals_full(aligned):
    a = _state()
    b = _clone(a)
    for step in (1, 2, 3):
        _adam_full(a, step)
        for lo, hi in _buckets(a["total"], aligned):
            _adam_range(b, step, lo, hi)
    torch.cuda.synchronize()
    for k in ("p", "m", "v"):
        assert torch.equal(a[k], b[k]), k


def test_matches_numpy_restatement():
    st = _state(1)
    p0, g, m0, v0 = (st[k].cpu().numpy().copy() for k in ("p", "g", "m", "v"))
    _adam_full(st, 3)
    lr = np.empty(st["total"], np.float32)
    l = np.frombuffer(_lrs(), np.float32)
    seg = np.cumsum([0, 3 * N, 4 * N, 3 * N, 3 * N, N])
    for i in range(5):
        lr[seg[i]:seg[i + 1]] = l[i]
    for k in range(K):
        o = 14 * N + 10 * N * k
        lr[o:o + 3 * N], lr[o + 3 * N:o + 7 * N], lr[o + 7 * N:o + 10 * N] = l[5], l[6], l[7]
    lr[14 * N + 10 * K * N:] = l[8]
    f = np.float32
    b1, b2 = f(BETAS[0]), f(BETAS[1])
    m = m0 * b1 + (f(1) - b1) * g
    v = v0 * b2 + (f(1) - b2) * (g * g)
    mh = m * f(1.0 / (1.0 - BETAS[0] ** 3))
    vh = v * f(1.0 / (1.0 - BETAS[1] ** 3))
    p = p0 - lr * mh / (np.sqrt(vh) + f(EPS))
    # the device contracts a*b + c into one FMA; allow that rounding, scaled per tensor
    for got, want in ((st["m"], m), (st["v"], v), (st["p"], p)):
        want = want.astype(np.float64)
        np.testing.assert_allclose(got.cpu().numpy(), want, rtol=1e-6, atol=1e-6 * np.abs(want).max())


def _ci_inputs(B=3, seed=2):
    g = np.random.default_rng(seed)
    maxw = g.uniform(0, 0.3, (B, N)).astype(np.float32)
    maxw[:, ::7] = 0.0                                   # never seen
    maxw[1, 5] = maxw[2, 5] = 0.29                       # tie: first frame wins
    wsums = g.uniform(0.05, 1.0, (B, N, 4)).astype(np.float32)
    visited = (g.uniform(size=N) < 0.3).astype(np.uint8)
    t = lambda x: torch.from_numpy(x).cuda()
    return B, t(maxw), t(wsums), t(visited)


def test_fused_color_init_local_equals_sequential():
    from paper_2503_12886_b200 import _lib as L
    B, maxw, wsums, visited = _ci_inputs()
    a, b = _state(3), None
    b = _clone(a)
    va, vb = visited.clone(), visited.clone()
    na, nb = torch.zeros(1, dtype=torch.int32, device="cuda"), torch.zeros(1, dtype=torch.int32, device="cuda")
    ea, eb = (torch.full((1,), -1, dtype=torch.int64, device="cuda") for _ in range(2))
    _adam_full(a, 1)
    L.call("hs_color_init", B, N, _p(maxw), _p(wsums), ctypes.c_float(0.1), _p(va), _p(a["p"]), _p(na), _p(ea),
           _stream())
    for lo, hi in _buckets(b["total"]):
        _adam_range(b, 1, lo, hi, 1, B, maxw, wsums, visited=vb, n_init=nb, err=eb)
    torch.cuda.synchronize()
    assert int(na.item()) > 0 and int(na.item()) == int(nb.item())
    assert torch.equal(va, vb)
    for k in ("p", "m", "v"):
        assert torch.equal(a[k], b[k]), k
    assert int(eb.item()) == -1


def test_fused_color_init_reduced_equals_sequential():
    from paper_2503_12886_b200 import _lib as L
    B, maxw, wsums, visited = _ci_inputs(seed=4)
    packed = torch.empty(N, dtype=torch.int64, device="cuda")
    est4 = torch.empty(N * 4, dtype=torch.float32, device="cuda")
    err = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    L.call("hs_color_pack", B, N, 0, _p(maxw), _p(visited), _p(packed), _stream())
    L.call("hs_color_select", B, N, 0, _p(packed), _p(wsums), _p(est4), _p(err), _stream())
    a = _state(5)
    b = _clone(a)
    va, vb = visited.clone(), visited.clone()
    na, nb = torch.zeros(1, dtype=torch.int32, device="cuda"), torch.zeros(1, dtype=torch.int32, device="cuda")
    _adam_full(a, 2)
    L.call("hs_color_apply", N, _p(packed), _p(est4), ctypes.c_float(0.1), _p(va), _p(a["p"]), _p(na), _stream())
    _adam_range(b, 2, 0, b["total"], 2, B, packed=packed, est4=est4, visited=vb, n_init=nb)
    torch.cuda.synchronize()
    assert int(na.item()) > 0 and int(na.item()) == int(nb.item())
    assert torch.equal(va, vb)
    for k in ("p", "m", "v"):
        assert torch.equal(a[k], b[k]), k


def test_split_colour_segment_rejected():
    B, maxw, wsums, visited = _ci_inputs()
    st = _state()
    err = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    with pytest.raises(ValueError, match="colour segment"):
        _adam_range(st, 1, 0, 8 * N, 1, B, maxw, wsums, visited=visited, err=err)
    _adam_range(st, 1, 0, 7 * N, 1, B, maxw, wsums, visited=visited, err=err)   # disjoint: fine
