"""Diagnostics for the masked-replay step parity: dump device and oracle gradients
(summed and per frame) plus the splat-space adjoint of frame 0 to gpurun_out/."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import numpy as np
import torch

import oracle as O
from test_gpu_train import masked_step_parity
from bench_support import synth

uv, B, size = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (141, 4, 256)))
wl = synth.make_workload(uv, B, size)
rep, errs, tr = masked_step_parity(wl, B, size, size)
print(rep)
print(errs)
st = tr._diag_state if hasattr(tr, "_diag_state") else None
state = tr._oracle_state
ctxs, gimgs, items = state.last_items
N = tr.av.N
out = dict(dev_grads=tr.grads.cpu().numpy(), dev_gsplat=tr.g_splat.view(B, N, 9).cpu().numpy(),
           dev_graw=tr.g_raw14.view(B, 14 * N).cpu().numpy(),
           or_base14=np.stack([it[0] for it in items]), or_deltas_sum=state.last_grads[1])
for b in range(min(B, 2)):
    c = ctxs[b]
    gm, gc, go, gcol = O.splat_space_grads(c.splats, c.aux, gimgs[b])
    full = np.zeros((N, 9))
    full[c.splats.index] = np.concatenate([gm, gc, go[:, None], gcol], axis=1)
    out[f"or_gsplat{b}"] = full
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
np.savez_compressed(os.path.join(ROOT, "gpurun_out", f"diag_{uv}_{B}_{size}.npz"), **out)
