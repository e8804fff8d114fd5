# Host pipeline: parity tests, then the C2 e2e leg with the pack16 transfer
# and without it (end ticks as u32, grants derived from the records),
# interleaved on one box (all output -> gpurun_out/e2e_ab.txt).
mkdir -p gpurun_out
exec > gpurun_out/e2e_ab.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "host_pipeline or integration or dropin or abi" > gpurun_out/pytest_e2e.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_e2e.log
for i in 1 2; do
for cfg in "SGPU_PACK16=1" "SGPU_PACK16=0" "SGPU_PACK16=1 SGPU_PIPE_BUFS=3" "SGPU_PACK16=1 SGPU_PIPE_BUFS=6" "SGPU_PACK16=1 SGPU_HOST_THREADS=8"; do
  env $cfg timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/e2e.json 2> gpurun_out/e2e.err
  python -c "import json;d=json.load(open('gpurun_out/e2e.json'));print('[$cfg]', 'kernel', d['value'], 'e2e', d['e2e']['value'], d['e2e']['d2h_bytes_per_step'])"
done
done
for ch in 32768 131072; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --chunk $ch > gpurun_out/e2e.json 2> gpurun_out/e2e.err
  python -c "import json;d=json.load(open('gpurun_out/e2e.json'));print('[chunk $ch]', 'e2e', d['e2e']['value'])"
done
SGPU_PIPE_TRACE=1 timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu > /dev/null 2> gpurun_out/pipe_trace.txt; tail -20 gpurun_out/pipe_trace.txt
