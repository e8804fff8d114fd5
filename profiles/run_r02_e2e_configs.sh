mkdir -p gpurun_out
exec > gpurun_out/e2efix.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "host_pipeline or integration or dist" 2>&1 | tail -2
for c in C2 C4 C5 C3; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu > gpurun_out/e.json 2> gpurun_out/e.err
  python -c "import json;d=json.load(open('gpurun_out/e.json'));print('$c', 'kernel', d['value'], 'e2e', d['e2e']['value'], d['e2e']['d2h_bytes_per_step'])" || tail -3 gpurun_out/e.err
done
