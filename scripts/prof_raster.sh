mkdir -p gpurun_out/pr
ncu --set full --import-source on --clock-control none -k regex:raster_train --launch-skip 140 -c 1 \
    -o gpurun_out/pr/raster python scripts/prof_step.py 145 > gpurun_out/pr/ncu.log 2>&1
ncu -i gpurun_out/pr/raster.ncu-rep --page source --csv --print-source sass > gpurun_out/pr/raster_src.csv
ncu -i gpurun_out/pr/raster.ncu-rep --page raw --csv > gpurun_out/pr/raster_raw.csv
