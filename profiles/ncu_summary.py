"""Key counters of ncu --set full captures as one markdown table (one row
per .ncu-rep; the first profiled kernel of each).

    python profiles/ncu_summary.py gpurun_out/r02_c2.ncu-rep ...

Columns: kernel time, warp instructions, active lanes per warp instruction,
issue-slot utilisation, achieved resident warps per SM, registers, dynamic
shared memory per block, DRAM bytes read + written, and the three largest
stall reasons (cycles per issued instruction).
"""
import csv
import io
import os
import subprocess
import sys


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units, first = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(head, units, first)}


def num(d, k, default=None):
    if k not in d:
        return default
    v = d[k][0].replace(",", "")
    try:
        return float(v)
    except ValueError:
        return default


def scale(d, k):
    """value in base units (ms for time, bytes for bytes)."""
    v = num(d, k)
    if v is None:
        return None
    u = d[k][1]
    mult = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3,
            "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1.0)
    return v * mult


def main():
    print("| capture | kernel | time ms | warp inst | lanes/inst | issue active % | warps/SM | regs | smem/block KB | DRAM rd+wr GB | top stalls (cycles/issue) |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for p in sys.argv[1:]:
        d = raw(p)
        name = d.get("Kernel Name", ("?", ""))[0].split("(")[0]
        t = scale(d, "gpu__time_duration.sum")
        inst = num(d, "smsp__inst_executed.sum")
        lanes = num(d, "smsp__thread_inst_executed_per_inst_executed.ratio")
        issue = num(d, "smsp__issue_active.avg.pct_of_peak_sustained_active")
        warps = num(d, "sm__warps_active.avg.per_cycle_active")
        regs = num(d, "launch__registers_per_thread")
        smem = scale(d, "launch__shared_mem_per_block_dynamic")
        rd = scale(d, "dram__bytes_read.sum")
        wr = scale(d, "dram__bytes_write.sum")
        stalls = []
        pre = "smsp__average_warps_issue_stalled_"
        for k in d:
            if k.startswith(pre) and k.endswith("_per_issue_active.ratio"):
                v = num(d, k)
                if v:
                    stalls.append((v, k[len(pre):-len("_per_issue_active.ratio")]))
        stalls.sort(reverse=True)
        st = ", ".join(f"{n} {v:.2f}" for v, n in stalls[:3])
        f = lambda x, fmt: (fmt % x) if x is not None else "n/a"
        print(f"| {os.path.basename(p)} | `{name[:48]}` | {f(t, '%.2f')} | {f(inst, '%.3g')} | {f(lanes, '%.1f')} | "
              f"{f(issue, '%.1f')} | {f(warps, '%.1f')} | {f(regs, '%.0f')} | {f(smem / 1e3 if smem else None, '%.1f')} | "
              f"{f((rd + wr) / 1e9 if rd is not None and wr is not None else None, '%.2f')} | {st} |")


if __name__ == "__main__":
    main()
