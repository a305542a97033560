for l in "$@"; do echo -n "$l fill: "; HS_B200_LIB=paper_2503_12886_b200/lib/exp/$l.so python scripts/stage_ab.py fill 40 2 | tail -1; done
bash scripts/ab_render_dev.sh "$@"
for l in "$@"; do echo -n "$l bench: "; HS_B200_LIB=paper_2503_12886_b200/lib/exp/$l.so python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-render 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4), d['stages_ms'].get('bin_tiles'))"; done
