#!/bin/bash
# per-kernel launch times (ncu, 3 steps) of the bench step for each library given
for lib in "$@"; do
  echo "== $lib"
  HS_B200_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/ab.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-render > /dev/null 2>&1
  python - <<PY
import csv,collections
rows=list(csv.reader(open("/tmp/ab.csv")))
hdr=None; agg=collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r: hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r))
        if d.get("Metric Name")=="gpu__time_duration.sum":
            agg.setdefault(d["Kernel Name"][:45],[]).append(float(d["Metric Value"]))
for k,v in sorted(agg.items(), key=lambda kv:-sum(kv[1])):
    if "tile_" in k: print(f"{sum(v)/len(v)/1000:8.1f}us {k}")
PY
done
