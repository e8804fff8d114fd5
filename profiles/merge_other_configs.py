"""Fold gpurun_out/other_C{3,4,5}.json (profiles/run_other_configs.sh) into
profiles/r01_other_configs.json (the kept fields of each bench line)."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEEP = ("value", "unit", "ms_per_step", "config", "aggregate", "roofline", "cpu_baseline", "clocks",
        "gpu_launches")


def main():
    path = os.path.join(ROOT, "profiles", "r01_other_configs.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    out["note"] = ("kernel-only bench lines (python bench.py --config Cx --steps 3 --warmup 3 --no-e2e, "
                   "profiles/run_other_configs.sh) with the reference's own simulate() timed on the box's "
                   "host cores beside them; parity cases of BASELINE.json, not the headline metric")
    for c in ("C3", "C4", "C5"):
        f = os.path.join(ROOT, "gpurun_out", f"other_{c}.json")
        line = [ln for ln in open(f).read().splitlines() if ln.startswith("{")][-1]
        d = json.loads(line)
        out[c] = {k: d[k] for k in KEEP if k in d}
        print(c, d["value"], d["ms_per_step"], (d.get("cpu_baseline") or {}).get("value"))
    json.dump(out, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
