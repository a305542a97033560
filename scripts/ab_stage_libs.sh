#!/bin/bash
# Stage-level A/B over experimental libraries, two interleaved rounds:
#   bash scripts/ab_stage_libs.sh STAGE FLUSH base new ...   (paper_2503_12886_b200/lib/exp/NAME.so)
stage=$1; fl=$2; shift 2
for rep in 1 2; do
  for n in "$@"; do
    HS_B200_LIB=paper_2503_12886_b200/lib/exp/$n.so python scripts/stage_ab.py $stage 60 $fl 2>&1 | tail -1
  done
done
