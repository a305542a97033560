#!/bin/bash
# ncu --set full with source of one kernel (regex $1) in a steady-state C2 step:
#   bash scripts/prof_kernel.sh REGEX NAME   -> gpurun_out/pk/NAME.ncu-rep, NAME_src.csv
mkdir -p gpurun_out/pk
ncu --set full --import-source on --clock-control none -k regex:"$1" --launch-skip 100 -c 1 \
    -o gpurun_out/pk/$2 python scripts/prof_step.py 105 > gpurun_out/pk/$2.log 2>&1
ncu -i gpurun_out/pk/$2.ncu-rep --page source --csv --print-source sass > gpurun_out/pk/$2_src.csv
