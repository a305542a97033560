ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tl.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-render > /dev/null 2>&1; python - <<PY
import csv,collections
rows=list(csv.reader(open("gpurun_out/tl.csv")))
hdr=None; agg=collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r: hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r))
        if d.get("Metric Name")=="gpu__time_duration.sum":
            agg.setdefault(d["Kernel Name"][:50],[]).append(float(d["Metric Value"]))
for k,v in sorted(agg.items(), key=lambda kv:-sum(kv[1]))[:16]: print(f"{len(v):4d} {sum(v)/len(v)/1000:8.1f}us {max(v)/1000:8.1f}max {k}")
PY
python bench.py --steps 100 --warmup 10 --no-cpu-baseline 2>gpurun_out/berr.log | tail -1 > gpurun_out/b.json; python -c "import json; d=json.load(open('gpurun_out/b.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['gpu_launches'], {k: round(v,3) for k,v in d['stages_ms'].items() if v>0.01})"
