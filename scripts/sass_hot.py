"""Summarize an ncu source page (SASS) CSV: instructions executed per SASS line,
stall samples, and totals; prints the hottest region."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ie = hdr.index("Instructions Executed")
st = hdr.index("Warp Stall Sampling (All Samples)")
th = hdr.index("Avg. Threads Executed")
data = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        data.append((r[0], r[1].strip(), int(r[ie]), int(r[st]), float(r[th])))
    except ValueError:
        pass
tot = sum(d[2] for d in data)
tst = sum(d[3] for d in data)
print("total warp instructions", tot, "stall samples", tst, "sass lines", len(data))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 60
# print lines in address order with their counts, only those above 0.2% of total
for a, s, n, ss, t in data:
    if n > tot * float(sys.argv[3] if len(sys.argv) > 3 else 0.004):
        print(f"{n/tot*100:5.1f}% st{ss/tst*100:5.1f}% thr{t:5.1f} {s[:90]}")
