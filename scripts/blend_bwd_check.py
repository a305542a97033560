"""blend_bwd output check and kernel name: HS_B200_LIB=... python scripts/blend_bwd_check.py out.npz"""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile
from paper_2503_12886_b200 import _lib as L
from paper_2503_12886_b200.device import _p

N, K, B = 50176, 20, 16
g = torch.Generator(device="cpu").manual_seed(0)
deltas = torch.randn(K * 10 * N, generator=g).cuda()
psi = torch.randn(B * K, generator=g).cuda()
g_raw = torch.randn(B * 14 * N, generator=g).cuda()
grads = torch.zeros(14 * N + K * 10 * N, device="cuda")
P = int(L.load().hs_blend_bwd_partials(N))
parts = torch.zeros(B * K * P, device="cuda")
n = ctypes.c_int(0)
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    L.call("hs_blend_bwd", N, K, B, _p(deltas), _p(psi), _p(g_raw), _p(grads), _p(grads[14 * N:]), _p(parts),
           ctypes.byref(n), s)
    torch.cuda.synchronize()
print([e.name for e in prof.events() if "blend" in e.name][:3])
gpsi = parts.view(B * K, P)[:, :n.value].double().sum(1).cpu().numpy()
print("checksum", float(grads.double().abs().sum()), float(np.abs(gpsi).sum()))
# float64 reference
gr = g_raw.view(B, 14 * N).double()
ref_base = gr.sum(0)
ref_d = (psi.view(B, K).double().t() @ gr[:, :10 * N])
ref_psi = (gr[:, :10 * N] @ deltas.view(K, 10 * N).double().t())
out = grads.double()
print("g_base max rel", float(((out[:14 * N] - ref_base).abs().max() / ref_base.abs().max())),
      "g_delta max rel", float(((out[14 * N:].view(K, 10 * N) - ref_d).abs().max() / ref_d.abs().max())),
      "g_psi max rel", float((torch.tensor(gpsi).view(B, K).cuda() - ref_psi).abs().max() / ref_psi.abs().max()))
