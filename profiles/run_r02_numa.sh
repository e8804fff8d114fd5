# Host pipeline threads bound to the GPU's NUMA node: parity, the sysfs
# CPU list, and the C2 e2e leg with and without binding -> gpurun_out/numa.txt
mkdir -p gpurun_out
exec > gpurun_out/numa.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "host_pipeline" 2>&1 | tail -1
bus=$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | head -1 | tr 'A-F' 'a-f' | sed 's/^0000//;s/^/0000/' | cut -c1-12); echo "bus $bus: $(cat /sys/bus/pci/devices/$bus/local_cpulist 2>/dev/null) numa $(cat /sys/bus/pci/devices/$bus/numa_node 2>/dev/null)"
SGPU_PIPE_TRACE=1 timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu 2>&1 >/dev/null | grep "numa bind" | head -1
for i in 1 2; do for b in 1 0; do
  SGPU_NUMA_BIND=$b timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/e.json 2> gpurun_out/e.err
  python -c "import json;d=json.load(open('gpurun_out/e.json'));print('bind=$b', 'e2e', round(d['e2e']['value']/1e6,1), 'M')"
done; done
