for l in "$@"; do echo -n "$l raster: "; HS_B200_LIB=paper_2503_12886_b200/lib/exp/$l.so python scripts/raster_ab.py 30 | tail -1; done
