"""hs_blend_bwd alone on random inputs, L2 evicted (256 MB read) before each launch:
    HS_B200_LIB=... python scripts/blend_bwd_time.py N K B [reps]  -> median us, GB/s of g + deltas + outputs"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2503_12886_b200 import _lib as L

N, K, B = (int(x) for x in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 30
dev = "cuda"
params = torch.randn(14 * N + K * 10 * N, device=dev)
deltas = params[14 * N:]
psi = torch.randn(B * K, device=dev)
g_raw = torch.randn(B * 14 * N, device=dev)
grads = torch.empty(14 * N + K * 10 * N, device=dev)
P = int(L.load().hs_blend_bwd_partials(N))
parts = torch.empty(B * K * P, device=dev)
flush = torch.empty(256 << 18, device=dev)
n = ctypes.c_int(0)
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
p = lambda t: ctypes.c_void_p(t.data_ptr())
ts = []
for i in range(reps + 3):
    flush.sum()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    L.call("hs_blend_bwd", N, K, B, p(deltas), p(psi), p(g_raw), p(grads), p(grads[14 * N:]), p(parts), ctypes.byref(n), s)
    b.record()
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(a.elapsed_time(b) * 1000)
ts.sort()
us = ts[len(ts) // 2]
byts = 4 * (B * 14 * N + K * 10 * N + 14 * N + K * 10 * N)
print(f"N={N} K={K} B={B} kernels={L.load().hs_blend_bwd_kernels(N, K, B)} {us:.1f} us  {byts / us / 1e3:.0f} GB/s")
