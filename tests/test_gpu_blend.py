"""Blend forward / adjoint kernels against float64 (S/model.py:165-216, the item-order
reduce of S/train.py:253-255), over the shapes that select each kernel variant:

* N % 128 == 0 with 9..16-frame passes: the TMA-tiled adjoint (1 KB rows), incl. a
  32-frame batch (two passes, the second accumulating);
* other N / frame counts up to 16: the register-streaming adjoint;
* more than 16 frames: the split adjoint (g_base / g_delta over all frames in one pass,
  then g_psi per <= 128 frames from cp.async-staged tiles), incl. odd N, K > 20 (the
  32-basis instantiation), 130 frames (two g_psi launches) and N < 17 (the fused kernels);
* the forward's TMA tiles (frames in two groups) for 4 / 8 / 16 / 24 frames, with and
  without zero weights (the reference skips psi == 0 terms).

Tolerances: outputs relative to their largest magnitude, 2e-6 (fp32 sums of <= 20
products; g_psi sums 10 N products per entry: 1e-5).
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


def _p(t):
    return ctypes.c_void_p(t.data_ptr())


def _rel(a, b):
    return float((a - b).abs().max() / max(float(b.abs().max()), 1e-30))


@pytest.mark.parametrize("N,K,B", [(50176, 20, 16), (4096, 20, 16), (256, 20, 32), (19881, 20, 4), (1000, 7, 12),
                                   (1280, 20, 9), (30011, 20, 48), (4097, 20, 40), (2048, 20, 32), (1000, 7, 130),
                                   (1001, 25, 20), (16, 20, 20)])
def test_blend_bwd_matches_float64(N, K, B):
    from paper_2503_12886_b200 import _lib as L
    g = torch.Generator().manual_seed(N + K + B)
    deltas = torch.randn(K * 10 * N, generator=g).cuda()
    psi = torch.randn(B * K, generator=g).cuda()
    g_raw = torch.randn(B * 14 * N, generator=g).cuda()
    grads = torch.full((14 * N + K * 10 * N,), float("nan"), device="cuda")
    P = int(L.load().hs_blend_bwd_partials(N))
    parts = torch.zeros(B * K * P, device="cuda")
    n = ctypes.c_int(0)
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    L.call("hs_blend_bwd", N, K, B, _p(deltas), _p(psi), _p(g_raw), _p(grads), _p(grads[14 * N:]), _p(parts),
           ctypes.byref(n), s)
    torch.cuda.synchronize()
    assert 1 <= n.value <= P
    gr = g_raw.view(B, 14 * N).double()
    out = grads.double()
    assert torch.isfinite(out).all()
    assert _rel(out[:14 * N], gr.sum(0)) <= 2e-6
    ref_d = psi.view(B, K).double().t() @ gr[:, :10 * N]
    assert _rel(out[14 * N:].view(K, 10 * N), ref_d) <= 2e-6
    gpsi = parts.view(B * K, P)[:, :n.value].double().sum(1).view(B, K)
    ref_psi = gr[:, :10 * N] @ deltas.view(K, 10 * N).double().t()
    assert _rel(gpsi, ref_psi) <= 1e-5


@pytest.mark.parametrize("N,B,zero", [(2048, 4, False), (2048, 8, True), (2048, 16, False), (2048, 16, True), (2048, 24, False), (2049, 16, False), (2049, 64, True), (1023, 5, False),
                                      (1023, 24, False), (2049, 130, True)])
def test_blend_fwd_matches_float64(N, B, zero):
    from paper_2503_12886_b200 import _lib as L
    K = 20
    g = torch.Generator().manual_seed(B)
    base14 = torch.randn(14 * N, generator=g).cuda()
    deltas = torch.randn(K * 10 * N, generator=g).cuda()
    psi = torch.randn(B, K, generator=g)
    if zero:
        psi[::2, ::3] = 0.0
    psi = psi.cuda()
    raw = torch.full((B * 10 * N,), float("nan"), device="cuda")
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    L.call("hs_blend_fwd", N, K, B, _p(base14), _p(deltas), _p(psi), _p(raw), s)
    torch.cuda.synchronize()
    ref = base14[:10 * N].double()[None] + psi.double() @ deltas.view(K, 10 * N).double()
    assert torch.isfinite(raw).all()
    assert _rel(raw.view(B, 10 * N).double(), ref) <= 2e-6

