#!/bin/bash
# ncu --set full with source of every non-raster kernel of one steady-state C2 step
# (outputs in gpurun_out/pk/): step.ncu-rep + per-kernel SASS source CSVs.
mkdir -p gpurun_out/pk
ncu --set full --import-source on --clock-control none -k regex:'^(?!.*raster_train)' --launch-skip 2000 -c 21 \
    -o gpurun_out/pk/step python scripts/prof_step.py 145 > gpurun_out/pk/ncu.log 2>&1
ncu -i gpurun_out/pk/step.ncu-rep --page raw --csv > gpurun_out/pk/raw.csv
for k in project_avatar_fwd project_avatar_bwd blend_bwd blend_fwd tile_scatter tile_sort_warp tile_sort_long adam_kernel; do
  ncu -i gpurun_out/pk/step.ncu-rep -k regex:$k -c 1 --page source --csv --print-source sass > gpurun_out/pk/src_$k.csv 2>/dev/null
done
