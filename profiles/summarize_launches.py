"""Summarise an ncu launch list (--csv --metrics gpu__time_duration.sum,...)
per kernel and grid size: launches, mean duration, DRAM bytes per launch.

    python profiles/summarize_launches.py gpurun_out/launches.csv
"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, gi, mi, vi, ii = (h.index(x) for x in ("Kernel Name", "Grid Size", "Metric Name", "Metric Value", "ID"))
per = collections.defaultdict(dict)
for r in rows[1:]:
    per[(int(r[ii]), r[ki].split("(")[0], r[gi])][r[mi]] = float(r[vi].replace(",", ""))
agg = collections.defaultdict(list)
for (i, k, g), m in per.items():
    # launches of one kernel differ by batch size (device-resident steps vs
    # host-pipeline chunks): group by grid and DRAM-read magnitude
    mag = int(m.get("dram__bytes_read.sum", 0)).bit_length()
    agg[(k, f"{g} ~2^{mag}B")].append(m)
tot = sum(m.get("gpu__time_duration.sum", 0) for ms in agg.values() for m in ms)
print(f"{'kernel':40s} {'grid / read size':>22s} {'n':>4s} {'mean ms':>9s} {'share':>6s} {'rd MB':>9s} {'wr MB':>9s}")
for (k, g), ms in sorted(agg.items(), key=lambda kv: -sum(m.get("gpu__time_duration.sum", 0) for m in kv[1])):
    t = [m.get("gpu__time_duration.sum", 0) for m in ms]
    rd = sum(m.get("dram__bytes_read.sum", 0) for m in ms) / len(ms) / 1e6
    wr = sum(m.get("dram__bytes_write.sum", 0) for m in ms) / len(ms) / 1e6
    print(f"{k[:40]:40s} {g:>22s} {len(ms):4d} {sum(t) / len(t) / 1e6:9.3f} {sum(t) / tot * 100:5.1f}% {rd:9.1f} {wr:9.1f}")
