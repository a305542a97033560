"""Per-stage DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of one
training step from an ncu --set full capture covering >= one whole step; writes the
JSON bench.py reads (profiles/ncu_traffic.json).
Usage: python scripts/traffic_by_stage.py report.ncu-rep out.json"""
import csv
import io
import json
import subprocess
import sys

STAGE = [("raster", "raster_train_kernel"), ("raster_bwd", "raster_bwd_kernel"), ("raster_fwd", "raster_fwd_kernel"), ("blend_bwd", ("blend_bwd_kernel", "blend_bwd_tma_kernel")),
         ("blend_fwd", ("blend_fwd_kernel", "blend_fwd_tma_kernel")), ("project_fwd", "project_avatar_fwd"),
         ("project_bwd", "project_avatar_bwd"), ("adam", "adam_kernel"), ("mlp_fwd", "mlp_fwd_kernel"),
         ("rig_frames", "rig_frames_kernel"),
         ("bin_sort", ("emit_kernel", "radix_hist_all", "radix_digit_scan", "radix_onesweep", "tile_ranges")),
         ("bin_tiles", ("tile_count", "tile_scan", "tile_scatter", "tile_sort", "tile_order"))]

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
# per kernel (full name, i.e. per template instance): the average over the captured
# launches; a stage = the sum over its distinct kernels (each runs once per step)
per = {}
for k, b in seq:
    per.setdefault(k, []).append(b)
avg = {k: sum(v) / len(v) for k, v in per.items()}
res = {}
for name, pat in STAGE:
    pats = (pat,) if isinstance(pat, str) else pat
    tot = sum(b for k, b in avg.items() if any(p in k for p in pats))
    if tot:
        res[name] = tot
res["_source"] = ("ncu --set full --clock-control none (dram__bytes_read.sum + dram__bytes_write.sum), one C2 "
                  "bench step; per stage: the sum over its kernels of each kernel's average per launch; "
                  "profiles/r2_ncu_c2_step.md")
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
