#!/bin/bash
# raster A/B with colour init finished (raster_train_kernel<0>)
for rep in 1 2; do for n in "$@"; do RAB_CI=0 HS_B200_LIB=paper_2503_12886_b200/lib/exp/$n.so python scripts/raster_ab.py 60 2>&1 | tail -1; done; done
