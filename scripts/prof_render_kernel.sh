#!/bin/bash
# ncu --set full with source of one kernel (regex $1) in the render bench shape:
#   bash scripts/prof_render_kernel.sh REGEX NAME   -> gpurun_out/pk/NAME.ncu-rep, NAME_src.csv, NAME_details.txt
mkdir -p gpurun_out/pk
ncu --set full --import-source on --clock-control none -k regex:"$1" --launch-skip 5 -c 1 \
    -o gpurun_out/pk/$2 python scripts/render_timeline.py > gpurun_out/pk/$2.log 2>&1
ncu -i gpurun_out/pk/$2.ncu-rep --page source --csv --print-source sass > gpurun_out/pk/$2_src.csv
ncu -i gpurun_out/pk/$2.ncu-rep --page details > gpurun_out/pk/$2_details.txt
