#!/bin/bash
# bench value + raster stage per library (2 runs each)
for lib in "$@"; do
  for i in 1 2; do
    HS_B200_LIB=$lib python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-render 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib'.split('/')[-1], round(d['value']), round(d['ms_per_step'],4), d['stages_ms'].get('raster'))"
  done
done
