#!/bin/bash
# A/B the experimental libraries in paper_2503_12886_b200/lib/exp/ with the bench step.
for lib in "$@"; do
  HS_B200_LIB=$lib python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-render 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['stages_ms']; print('$lib', round(d['value'],1), round(d['ms_per_step'],3), 'fwd', s['raster_fwd'], 'bwd', s['raster_bwd'])"
done
