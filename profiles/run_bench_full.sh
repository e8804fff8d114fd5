set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
cat gpurun_out/bench_full.json; tail -3 gpurun_out/bench_full.err
for c in C3 C4 C5; do
  timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_$c.json 2>&1; echo "$c lane rc=$?"
  SGPU_K1=warp timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_${c}_warp.json 2>&1; echo "$c warp rc=$?"
  python -c "import json;a=json.load(open('gpurun_out/bench_$c.json'));b=json.load(open('gpurun_out/bench_${c}_warp.json'));print('$c lane',a['value'],a['ms_per_step'],'warp',b['value'],b['ms_per_step'])"
done
