set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_parity.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_parity.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_lane.json 2> gpurun_out/bench_lane.err; echo "bench rc=$?"
cat gpurun_out/bench_lane.json; tail -3 gpurun_out/bench_lane.err
SGPU_K1=warp timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_warp.json 2>&1; echo "bench warp rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_warp.json'));print('warp',d['value'],d['ms_per_step'])"
