"""Attribute ncu per-SASS 'Instructions Executed' (warp instructions) and
'Thread Instructions Executed' to source lines (no double counting of
inlined code) and print the hottest lines with their average active lanes.

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
te = hdr.index("Thread Instructions Executed") if "Thread Instructions Executed" in hdr else None
ws = hdr.index("Warp Stall Sampling (All Samples)")
cur_file, cur_line, cur_src = "?", 0, ""
inst = defaultdict(int)
thr = defaultdict(int)
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
        src[(cur_file, cur_line)] = cur_src.strip()[:72]
        continue
    if len(r) > ie and r[2].startswith("0x") and r[ie].isdigit():
        inst[(cur_file, cur_line)] += int(r[ie])
        if te is not None and r[te].isdigit():
            thr[(cur_file, cur_line)] += int(r[te])
        stall[(cur_file, cur_line)] += int(r[ws]) if r[ws].isdigit() else 0
tot = sum(inst.values())
st = sum(stall.values()) or 1
print(f"total warp instructions {tot}, thread instructions {sum(thr.values())} "
      f"({sum(thr.values()) / max(tot, 1):.2f} lanes/inst)")
for k in sorted(inst, key=lambda k: -inst[k])[:top]:
    lanes = thr[k] / inst[k] if inst[k] else 0
    print(f"{inst[k] / tot * 100:5.1f}% inst {stall[k] / st * 100:5.1f}% stall {lanes:5.1f} lanes  "
          f"{k[0]}:{k[1]:<4d} {src.get(k, '')}")
