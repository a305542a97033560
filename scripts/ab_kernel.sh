#!/bin/bash
# mean ncu launch time of kernels matching $1 over a 3-step bench, per library
pat=$1; shift
for lib in "$@"; do
  HS_B200_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/abk.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-render > /dev/null 2>&1
  python - "$lib" "$pat" <<'PY'
import csv, collections, sys
rows = list(csv.reader(open("/tmp/abk.csv")))
hdr = None; agg = collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r: hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum" and sys.argv[2] in d["Kernel Name"]:
            agg.setdefault(d["Kernel Name"][:40], []).append(float(d["Metric Value"]))
print(sys.argv[1].split("/")[-1], {k: round(sum(v) / len(v) / 1000, 1) for k, v in agg.items()})
PY
done
