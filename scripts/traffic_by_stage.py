"""Per-stage DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of one
training step from an ncu --set full capture covering >= one whole step; writes the
JSON bench.py reads (profiles/ncu_traffic.json).
Usage: python scripts/traffic_by_stage.py report.ncu-rep out.json"""
import csv
import io
import json
import subprocess
import sys

STAGE = [("raster", "raster_train_kernel"), ("raster_bwd", "raster_bwd_kernel"), ("raster_fwd", "raster_fwd_kernel"), ("blend_bwd", "blend_bwd_kernel"),
         ("blend_fwd", "blend_fwd_kernel"), ("project_fwd", "project_avatar_fwd"),
         ("project_bwd", "project_avatar_bwd"), ("adam", "adam_kernel"), ("mlp_fwd", "mlp_fwd_kernel"),
         ("rig_frames", "rig_frames_kernel"),
         ("bin_sort", ("emit_kernel", "radix_hist_all", "radix_digit_scan", "radix_onesweep", "tile_ranges"))]

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
ir, iw, ik = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum"), h.index("Kernel Name")
seq = []
for r in rows[2:]:
    b = float(r[ir]) * scale.get(units[ir], 1) + float(r[iw]) * scale.get(units[iw], 1)
    seq.append((r[ik], b))
# one step: from the first raster_bwd back to the previous raster_bwd-free window -- take
# the LAST complete step: stages are summed over the launches between two rig_frames
starts = [i for i, (k, _) in enumerate(seq) if "rig_frames_kernel" in k]
lo = starts[0] if starts else 0
hi = starts[1] if len(starts) > 1 else len(seq)
step = seq[lo:hi]
if not any("raster_bwd" in k for k, _ in step):
    # capture starts mid-step: the forward half from the last rig_frames onwards, the
    # backward half (after the previous step's forward raster) from before it
    head = seq[:lo]
    rf = max((i for i, (k, _) in enumerate(head) if "raster_fwd" in k or "raster_train" in k), default=-1)
    step = seq[lo:] + head[rf + 1:]
res = {}
for name, pat in STAGE:
    pats = (pat,) if isinstance(pat, str) else pat
    tot = sum(b for k, b in step if any(p in k for p in pats))
    if tot:
        res[name] = tot
res["_source"] = ("ncu --set full --clock-control none (dram__bytes_read.sum + dram__bytes_write.sum), one C2 "
                  "bench step; per-stage sum over the step's launches; profiles/r1_ncu_c2_step.md")
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
