"""Per-iteration instruction profile of a kernel's hot loop from an ncu SASS source
page CSV: counts are normalised by the execution count of the loop-head marker
instruction (first SASS line containing the given opcode substring)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ie = hdr.index("Instructions Executed")
th = hdr.index("Avg. Threads Executed")
st = hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        data.append((r[1].strip(), int(r[ie]), float(r[th]), int(r[st])))
    except ValueError:
        pass
marker = sys.argv[2] if len(sys.argv) > 2 else "UFLO"
head = next(i for i, d in enumerate(data) if marker in d[0] and d[1] > 0)
n_it = data[head][1]
tot = sum(d[1] for d in data)
tst = sum(d[3] for d in data)
print(f"loop-head count {n_it}, total {tot} -> {tot / n_it:.1f} warp instr per iteration")
cats = {}
inloop = 0.0
for s, n, t, stl in data:
    f = n / n_it
    if f > 0.05:
        op = s.split()[0] if not s.startswith("@") else s.split()[1]
        op = op.split(".")[0]
        cats[op] = cats.get(op, 0.0) + f
        inloop += f
for op, f in sorted(cats.items(), key=lambda kv: -kv[1]):
    print(f"  {op:12s} {f:6.2f}")
print(f"sum over lines executed > 0.05x per iteration: {inloop:.1f}")
if len(sys.argv) > 3:
    for s, n, t, stl in data:
        if n / n_it > 0.05:
            print(f"{n / n_it:5.2f} thr{t:5.1f} st{stl / tst * 100:5.1f}% {s[:80]}")
