for shape in "100489 20 128" "100489 20 64" "100489 20 32"; do
  for l in "$@"; do echo -n "$l "; HS_B200_LIB=paper_2503_12886_b200/lib/exp/$l.so python scripts/blend_bwd_time.py $shape; done
done
