# usage: bash scripts/ab_blend_bwd.sh lib1 lib2 ...  (libs in lib/exp)
for shape in "50176 20 16" "100489 20 128" "100489 20 16" "19881 20 4" "100489 20 64"; do
  for l in "$@"; do echo -n "$l "; HS_B200_LIB=paper_2503_12886_b200/lib/exp/$l.so python scripts/blend_bwd_time.py $shape; done
done
