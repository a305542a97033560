for l in "$@"; do echo -n "$l render-shape blend_fwd: "; HS_B200_LIB=paper_2503_12886_b200/lib/exp/$l.so python - <<'PY'
import sys, ctypes, torch
sys.path.insert(0, '.')
from paper_2503_12886_b200 import _lib as L
N, K, B = 100489, 20, 64
base = torch.randn(14 * N, device="cuda"); params = torch.randn(14 * N + K * 10 * N, device="cuda")
deltas = params[14 * N:]; psi = torch.randn(B * K, device="cuda"); raw = torch.empty(B * 10 * N, device="cuda")
flush = torch.empty(256 << 18, device="cuda"); s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
p = lambda t: ctypes.c_void_p(t.data_ptr()); ts = []
for i in range(23):
    flush.sum(); a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); L.call("hs_blend_fwd", N, K, B, p(params), p(deltas), p(psi), p(raw), s); b.record(); torch.cuda.synchronize()
    if i >= 3: ts.append(a.elapsed_time(b) * 1000)
ts.sort(); print(f"{ts[len(ts)//2]:.1f} us")
PY
done
bash scripts/ab_render_dev.sh "$@"
