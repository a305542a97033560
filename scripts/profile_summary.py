"""Summarize ncu outputs into profiles/:
  * a launch list CSV (--metrics gpu__time_duration.sum) -> per-kernel totals and shares;
  * a --set full report -> per-kernel duration, DRAM/L2/L1 throughput, IPC, occupancy,
    dram bytes per launch.
Usage: python scripts/profile_summary.py launches.csv report.ncu-rep out.md [traffic.json]
"""
import collections
import csv
import io
import json
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            name = d["Kernel Name"].split("(")[0]
            agg.setdefault(name, []).append(float(d["Metric Value"]))
    tot = sum(sum(v) for v in agg.values())
    lines = ["| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| `{k}` | {len(v)} | {sum(v)/1e3:.1f} | {sum(v)/len(v)/1e3:.2f} | {sum(v)/tot*100:.1f}% |")
    return "\n".join(lines)


WANT = ["Duration", "DRAM Throughput", "L2 Cache Throughput", "L1/TEX Cache Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Achieved Occupancy", "Registers Per Thread"]


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    ki, mi, vi, ui, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    per = collections.OrderedDict()
    for r in rows[1:]:
        if r[mi] in WANT:
            per.setdefault((r[ii], r[ki].split("(")[0]), {})[r[mi]] = f"{r[vi]} {r[ui]}"
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    h = rr[0]
    traffic = {}
    for r in rr[2:]:
        try:
            idx = r[h.index("ID")]
            rd = float(r[h.index("dram__bytes_read.sum")])
            wr = float(r[h.index("dram__bytes_write.sum")])
            unit_r, unit_w = rr[1][h.index("dram__bytes_read.sum")], rr[1][h.index("dram__bytes_write.sum")]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            traffic[idx] = rd * scale.get(unit_r, 1) + wr * scale.get(unit_w, 1)
        except (ValueError, IndexError):
            pass
    lines = ["| id | kernel | " + " | ".join(WANT) + " | DRAM bytes |", "|" + "---|" * (len(WANT) + 3)]
    by_kernel = {}
    for (i, k), m in per.items():
        t = traffic.get(i)
        lines.append(f"| {i} | `{k}` | " + " | ".join(m.get(w, "") for w in WANT) +
                     f" | {t/1e6:.1f} MB |" if t is not None else " | |")
        if t is not None:
            by_kernel.setdefault(k, []).append(t)
    return "\n".join(lines), {k: sum(v) / len(v) for k, v in by_kernel.items()}


if __name__ == "__main__":
    lc, rep, out = sys.argv[1:4]
    body = ["# ncu summary", "", "## Launch list (gpu__time_duration.sum, cold-cache, serialised)", "", launches(lc),
            "", "## --set full", ""]
    table, traffic = full(rep)
    body.append(table)
    open(out, "w").write("\n".join(body) + "\n")
    if len(sys.argv) > 4:
        json.dump(traffic, open(sys.argv[4], "w"), indent=1)
    print("\n".join(body))
