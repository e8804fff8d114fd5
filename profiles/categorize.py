"""Group per-source-line instruction counts (attribute.py input) of the K1
lane kernel into code regions by line range of sgpu_lanesim.cuh / sgpu_lane.cu.

    python profiles/categorize.py mix.csv
"""
import csv
import re
import sys
from collections import defaultdict

CSRC = "paper_1712_04495_b200/csrc/"
# region starts per source file: (regex on the source line, name)
MARKS = {
    "sgpu_lanesim.cuh": [
        (r"struct LaneKey", "keys/helpers"), (r"SG_HD void push\(", "heap push"), (r"SG_HD Key min_child\(", "heap pop"),
        (r"SG_HD void pop\(", "heap pop"), (r"SG_HD uint32_t fifo_get\(", "wake fifo"), (r"SG_HD void enqueue\(", "queue mask"),
        (r"SG_HD uint32_t fit_rank\(", "fit_rank/fit_set"), (r"SG_HD void grant_one\(", "grant (scan path)"),
        (r"SG_HD void init_round\(", "grant round init"), (r"SG_HD void grant_step\(", "grant step"),
        (r"SG_HD void end_round\(", "grant round end"), (r"SG_HD void grant_waiters_tbl\(", "grant round init"),
        (r"SG_HD void grant_waiters_scan\(", "grant (scan path)"), (r"SG_HD void end_app\(", "end_app/outputs"),
        (r"SG_HD void run_from_busy\(", "advance (phase 0)"), (r"SG_HD bool run\(", "event loop"),
        (r"SG_HD void finish\(", "finish/stats")],
    "sgpu_lane.cu": [
        (r"void lane_trace_range\(", "staging"), (r"bool lane_run\(", "lane setup"),
        (r"__global__", "kernel body"), (r"exact fallback", "fallback"),
        (r"static inline uint32_t align16", "host")],
}
STARTS = {}
for fname, marks in MARKS.items():
    lines = open(CSRC + fname).read().split("\n")
    st = []
    for i, l in enumerate(lines, 1):
        for rx, name in marks:
            if re.search(rx, l):
                st.append((i, name))
    STARTS[fname] = sorted(st)


def region(fname, n):
    r = "header/helpers"
    for s, name in STARTS[fname]:
        if n >= s:
            r = name
    return r


rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if r and r[0] == "Line No")
ie, te = hdr.index("Instructions Executed"), hdr.index("Thread Instructions Executed")
cur_file, cur_line = "?", 0
inst, thr = defaultdict(int), defaultdict(int)
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0].isdigit():
        cur_line = int(r[0])
        continue
    if len(r) > ie and r[2].startswith("0x") and r[ie].isdigit():
        k = region(cur_file, cur_line) if cur_file in STARTS else f"[{cur_file}]"
        inst[k] += int(r[ie])
        thr[k] += int(r[te]) if r[te].isdigit() else 0
tot = sum(inst.values())
for k in sorted(inst, key=lambda k: -inst[k]):
    print(f"{inst[k] / tot * 100:5.1f}%  {thr[k] / max(inst[k], 1):5.1f} lanes  {k}")
