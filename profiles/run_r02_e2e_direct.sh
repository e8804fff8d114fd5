# Host pipeline: parity with SGPU_DIRECT_POLS=1..3, then the C2 e2e leg at
# k = 0, 1, 2 interleaved on one box -> gpurun_out/e2e_direct.txt
mkdir -p gpurun_out
exec > gpurun_out/e2e_direct.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "host_pipeline" 2>&1 | tail -2
for i in 1 2 3; do for k in 0 1 2; do
  SGPU_DIRECT_POLS=$k timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/e.json 2> gpurun_out/e.err
  python -c "import json;d=json.load(open('gpurun_out/e.json'));print('k=$k', 'e2e', round(d['e2e']['value']/1e6,1), 'M', d['e2e']['d2h_bytes_per_step'])" || tail -3 gpurun_out/e.err
done; done
