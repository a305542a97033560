#!/bin/bash
# Round-2 profile set (run on the GPU box; outputs in gpurun_out/prof/):
#   bench.json      the default bench line
#   launches.csv    ncu launch list (gpu__time_duration.sum) of two steady-state C2 steps
#   step.ncu-rep    ncu --set full of one whole steady-state step (traffic per stage)
#   raster.ncu-rep  ncu --set full --import-source of the fused training raster
set -x
mkdir -p gpurun_out/prof
[ -n "$SKIP_BENCH" ] || python bench.py > gpurun_out/prof/bench.json 2> gpurun_out/prof/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 2000 -c 44 --csv \
    --log-file gpurun_out/prof/launches.csv python scripts/prof_step.py 150 > gpurun_out/prof/ncu1.log 2>&1
ncu --set full --clock-control none --launch-skip 2000 -c 22 -o gpurun_out/prof/step \
    python scripts/prof_step.py 145 > gpurun_out/prof/ncu2.log 2>&1
[ -n "$SKIP_RASTER" ] || ncu --set full --import-source on --clock-control none -k regex:raster_train --launch-skip 140 -c 1 \
    -o gpurun_out/prof/raster python scripts/prof_step.py 145 > gpurun_out/prof/ncu3.log 2>&1
ncu -i gpurun_out/prof/raster.ncu-rep --page raw --csv > gpurun_out/prof/raster_raw.csv
ncu -i gpurun_out/prof/raster.ncu-rep --page source --csv --print-source sass > gpurun_out/prof/raster_src.csv
ncu -i gpurun_out/prof/raster.ncu-rep --page details > gpurun_out/prof/raster_details.txt
python scripts/profile_summary.py gpurun_out/prof/launches.csv gpurun_out/prof/step.ncu-rep gpurun_out/prof/step_summary.md
python scripts/traffic_by_stage.py gpurun_out/prof/step.ncu-rep gpurun_out/prof/ncu_traffic.json
