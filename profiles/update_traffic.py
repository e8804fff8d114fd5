"""Write profiles/k1_traffic.json (the DRAM bytes and issue-active share of
one K1 launch that bench.py's roofline quotes) from an ncu --set full
capture of the C2 main pass.

    python profiles/update_traffic.py gpurun_out/<capture>.ncu-rep
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    rep = sys.argv[1]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]

    def get(name):
        i = hdr.index(name)
        v = float(vals[i].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(units[i], 1)
        return v * scale

    out = {
        "kernel": vals[hdr.index("Kernel Name")],
        "config": "C2",
        "dram_bytes_read": int(get("dram__bytes_read.sum")),
        "dram_bytes_write": int(get("dram__bytes_write.sum")),
        "source": f"ncu --set full capture {os.path.basename(rep)} (one launch, 1M traces x 4 policies); "
                  "issue_active_pct = smsp__issue_active.avg.pct_of_peak_sustained_active",
        "issue_active_pct": round(get("smsp__issue_active.avg.pct_of_peak_sustained_active"), 2),
    }
    json.dump(out, open(os.path.join(ROOT, "profiles", "k1_traffic.json"), "w"), indent=1)
    print(out)


if __name__ == "__main__":
    main()
