set -x
mkdir -p gpurun_out
lscpu > gpurun_out/lscpu.txt; numactl -H > gpurun_out/numa.txt 2>&1; nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
for c in C2 C4 C5; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/bench_$c.json'));print('$c', d['value'], d['ms_per_step'], d['e2e']['value'])"
done
nvcc -O3 -std=c++17 -Xcompiler -mavx2 -Xcompiler -pthread -o /tmp/ring profiles/ring_probe.cu && timeout 600 /tmp/ring 15 > gpurun_out/ring_probe.txt 2>&1; echo "ring rc=$?"; cat gpurun_out/ring_probe.txt
TOOLS="racecheck initcheck" SAN_TIMEOUT=700 bash profiles/run_sanitize.sh
