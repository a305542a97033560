#!/bin/bash
# A/B experimental libraries (paper_2503_12886_b200/lib/exp/*.so) on the bench step.
for lib in "$@"; do
  HS_B200_LIB=$lib python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-render 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['stages_ms']; print('$lib'.split('/')[-1], round(d['value'],1), round(d['ms_per_step'],3), {k: round(v,3) for k,v in s.items() if v > 0.012})"
done
