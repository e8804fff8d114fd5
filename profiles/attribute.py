"""Attribute ncu per-SASS 'Instructions Executed' to source lines (no
double counting of inlined code) and print the hottest lines.

    ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > mix.csv
    python profiles/attribute.py mix.csv [n]
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = next(r for r in rows if r and r[0] == "Line No")
ie = hdr.index("Instructions Executed")
ws = hdr.index("Warp Stall Sampling (All Samples)")
cur_file, cur_line, cur_src = "?", 0, ""
inst = defaultdict(int)
stall = defaultdict(int)
src = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0].isdigit():
        cur_line, cur_src = int(r[0]), r[1]
        src[(cur_file, cur_line)] = cur_src.strip()[:80]
        continue
    if len(r) > ie and r[2].startswith("0x") and r[ie].isdigit():
        inst[(cur_file, cur_line)] += int(r[ie])
        stall[(cur_file, cur_line)] += int(r[ws]) if r[ws].isdigit() else 0
tot = sum(inst.values())
st = sum(stall.values()) or 1
print(f"total instructions {tot}")
for k in sorted(inst, key=lambda k: -inst[k])[:top]:
    print(f"{inst[k] / tot * 100:5.1f}% inst {stall[k] / st * 100:5.1f}% stall  {k[0]}:{k[1]:<4d} {src.get(k, '')}")
