#!/bin/bash
# Kernel-level raster A/B over experimental libraries, two interleaved rounds:
#   bash scripts/ab_raster_libs.sh base s64 ...   (paper_2503_12886_b200/lib/exp/NAME.so)
for rep in 1 2; do
  for n in "$@"; do
    HS_B200_LIB=paper_2503_12886_b200/lib/exp/$n.so python scripts/raster_ab.py 60 2>&1 | tail -1
  done
done
