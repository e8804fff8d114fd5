set -x
mkdir -p gpurun_out
timeout 300 python profiles/pcie_probe.py
timeout 600 python profiles/e2e_probe.py 32768 65536 131072 262144
