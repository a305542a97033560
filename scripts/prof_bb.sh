#!/bin/bash
# ncu --set full of the split blend adjoint's kernels at N K B ($1 $2 $3)
mkdir -p gpurun_out/pk
for k in blend_bwd_gd blend_bwd_psi; do
ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip 2 -c 1 -o gpurun_out/pk/$k \
    python scripts/blend_bwd_time.py $1 $2 $3 4 > gpurun_out/pk/$k.log 2>&1
ncu -i gpurun_out/pk/$k.ncu-rep --page details > gpurun_out/pk/${k}_details.txt
ncu -i gpurun_out/pk/$k.ncu-rep --page source --csv --print-source sass > gpurun_out/pk/${k}_src.csv
done
