"""Attribute an ncu SASS source page (CSV) to CUDA source lines using the line table of
the same build (nvdisasm -g of the kernel's cubin): warp instructions executed and stall
samples per (file, line), plus totals per line range given as name=file:lo-hi.

usage: sass_by_line.py SRC.csv DISASM.sass KERNEL_MANGLED [name=file:lo-hi ...]"""
import csv
import re
import sys

src_csv, sass, kern = sys.argv[1:4]
ranges = []
for spec in sys.argv[4:]:
    name, rest = spec.split("=")
    f, lh = rest.split(":")
    lo, hi = map(int, lh.split("-"))
    ranges.append((name, f, lo, hi))

lines = open(sass).read().split("\n")
i0 = next(i for i, l in enumerate(lines) if l.startswith(kern + ":"))
# (nvdisasm -gi: each group of "//## File" comments is the inlining chain of the
# instructions that follow; the first is the innermost location)
table, cur, chain, fresh = {}, None, [], True
for l in lines[i0 + 1:]:
    if l.startswith("//----"):
        break
    if "//## File" in l:
        if fresh:
            chain, fresh = [], False
        for f, ln in re.findall(r'File "([^"]+)", line (\d+)', l):
            chain.append((f.split("/")[-1], int(ln)))
        cur = chain[0]
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);?\s*$", l)
    if m:
        fresh = True
        table[int(m.group(1), 16)] = (cur, m.group(2), tuple(chain))

rows = list(csv.reader(open(src_csv)))
h0 = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[h0]
ie, st = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows[h0 + 1:] if len(r) >= len(hdr) and r[0].startswith("0x")]
base = int(data[0][0], 16)
per, mism, tot, tst = {}, 0, 0, 0
reg = {name: [0, 0] for name, *_ in ranges}
reg["(other)"] = [0, 0]
for r in data:
    off = int(r[0], 16) - base
    n, s = int(r[ie]), int(r[st])
    tot += n
    tst += s
    loc, ins, ch = table.get(off, (("?", 0), "", ()))
    if ins.split()[:1] != r[1].split()[:1]:
        mism += 1
    a = per.setdefault(loc, [0, 0])
    a[0] += n
    a[1] += s
    for name, f, lo, hi in ranges:          # first matching range (most specific first)
        if any(ff == f and lo <= ln <= hi for ff, ln in ch):
            reg[name][0] += n
            reg[name][1] += s
            break
    else:
        reg["(other)"][0] += n
        reg["(other)"][1] += s
print(f"total {tot} warp instr, {tst} samples; opcode mismatches vs disasm: {mism} of {len(data)}")
for name, (n, s) in reg.items():
    print(f"{name:24s} {n / tot * 100:5.1f}% instr  {s / tst * 100:5.1f}% stalls")
print("top lines:")
for (f, ln), (n, s) in sorted(per.items(), key=lambda kv: -kv[1][0])[:40]:
    print(f"  {f}:{ln:<5d} {n / tot * 100:5.1f}% instr {s / tst * 100:5.1f}% stalls")
import os
focus = os.environ.get("FOCUS")          # name of a range: its top innermost lines
if focus:
    name, f, lo, hi = next(r for r in ranges if r[0] == focus)
    acc = {}
    for r in data:
        off = int(r[0], 16) - base
        loc, ins, ch = table.get(off, (("?", 0), "", ()))
        if any(ff == f and lo <= ln <= hi for ff, ln in ch):
            a = acc.setdefault(loc, [0, 0, []])
            a[0] += int(r[ie])
            a[1] += int(r[st])
            a[2].append(ins.split()[0] if ins else "?")
    print(f"{focus}: innermost lines")
    for loc, (n, s, ops) in sorted(acc.items(), key=lambda kv: -kv[1][0])[:25]:
        print(f"  {loc[0]}:{loc[1]:<5d} {n / tot * 100:5.2f}% {s / tst * 100:5.2f}%st  {' '.join(ops[:12])}")
