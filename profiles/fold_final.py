"""Fold the outputs of profiles/run_r02_final.sh (gpurun_out/) into the
committed round-2 evidence under profiles/r02_final_*:

    python profiles/fold_final.py

bench / reference-arm / 2-rank lines, the launch list, the ncu summary, the
C3-C5 bench lines with the counters of their own ncu capture, the GPU test
tail, the drop-in latencies, and per-source-line attribution of the C2 and
C3 captures (profiles/attribute.py).  Run profiles/update_traffic.py on
fin_c2 first (the bench line reads profiles/k1_traffic.json).
"""
import json
import os
import shutil
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_summary as NS  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")


def last_json(path):
    return json.loads([ln for ln in open(path).read().splitlines() if ln.startswith("{")][-1])


def write_line(src, dst):
    with open(os.path.join(P, dst), "w") as f:
        f.write(json.dumps(last_json(os.path.join(G, src))) + "\n")


def counters(rep):
    d = NS.raw(rep)
    lanes = NS.num(d, "smsp__thread_inst_executed_per_inst_executed.ratio")
    rd = NS.scale(d, "dram__bytes_read.sum") or 0.0
    wr = NS.scale(d, "dram__bytes_write.sum") or 0.0
    return {
        "traffic": int(rd + wr),
        "issue_active_frac": round(NS.num(d, "smsp__issue_active.avg.pct_of_peak_sustained_active") / 100.0, 4),
        "active_lanes_per_inst": round(lanes, 1) if lanes else None,
        "warps_per_sm": round(NS.num(d, "sm__warps_active.avg.per_cycle_active"), 1),
        "registers": int(NS.num(d, "launch__registers_per_thread")),
    }


def main():
    write_line("bench.json", "r02_final_bench.json")
    write_line("bench_ref.json", "r02_final_reference_arm.json")
    write_line("bench_2rank.json", "r02_final_bench_2rank_gloo_1gpu.json")
    shutil.copy(os.path.join(G, "launches.csv"), os.path.join(P, "r02_final_launches.csv"))
    shutil.copy(os.path.join(G, "launches_summary.txt"), os.path.join(P, "r02_final_launches_summary.txt"))
    shutil.copy(os.path.join(G, "ncu_summary.md"), os.path.join(P, "r02_final_ncu_summary.md"))
    shutil.copy(os.path.join(G, "dropin_latency.txt"), os.path.join(P, "r02_dropin_latency.txt"))
    shutil.copy(os.path.join(G, "program_mode.txt"), os.path.join(P, "r02_program_mode.txt"))
    tail = open(os.path.join(G, "pytest_gpu.log")).read().splitlines()[-2:]
    smoke = open(os.path.join(G, "smoke.log")).read().splitlines()[-1:]
    with open(os.path.join(P, "r02_final_pytest_gpu_tail.txt"), "w") as f:
        f.write("\n".join(tail + smoke) + "\n")
    out = {"note": ("bench lines (python bench.py --config Cx --steps 3 --warmup 3, profiles/run_r02_final.sh) "
                    "with the counters of one ncu --set full capture of the same configuration's K1 launch "
                    "(profiles/r02_final_ncu_summary.md); parity cases of BASELINE.json, not the headline metric")}
    for c in ("C3", "C4", "C5"):
        d = last_json(os.path.join(G, f"other_{c}.json"))
        line = {k: d[k] for k in ("value", "unit", "ms_per_step", "config", "aggregate", "roofline", "e2e",
                                  "cpu_baseline", "clocks", "gpu_launches") if k in d}
        rep = os.path.join(G, f"fin_{c.lower()}.ncu-rep")
        if os.path.exists(rep):
            cn = counters(rep)
            line["roofline"].update(cn)
            line["roofline"]["traffic_source"] = ("dram__bytes_read.sum + dram__bytes_write.sum, "
                                                  "profiles/r02_final_ncu_summary.md")
        out[c] = line
    with open(os.path.join(P, "r02_final_other_configs.json"), "w") as f:
        json.dump(out, f, indent=1)
        f.write("\n")
    for c in ("c2", "c3"):
        rep = os.path.join(G, f"fin_{c}.ncu-rep")
        if not os.path.exists(rep):
            continue
        mix = os.path.join(G, f"mix_{c}.csv")
        with open(mix, "w") as f:
            subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                           stdout=f, check=True)
        with open(os.path.join(P, f"r02_final_{c}_source_hotspots.txt"), "w") as f:
            subprocess.run([sys.executable, os.path.join(P, "attribute.py"), mix, "40"], stdout=f, check=True)


if __name__ == "__main__":
    main()
