# Refresh after the pipeline's u32 fallback: GPU tests, smoke, C2-C5 bench
# lines (kernel + e2e) -> gpurun_out/
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
for c in C3 C4 C5; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/other_$c.json 2> gpurun_out/other_$c.err; echo "$c rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/other_$c.json'));print('$c', d['value'], d['e2e']['value'])"
done
