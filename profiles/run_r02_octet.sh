mkdir -p gpurun_out
exec > gpurun_out/oct.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "octet or C3 or shapes or ragged or golden" 2>&1 | tail -25
timeout 600 python bench.py --config C3 --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/c3n.json 2> gpurun_out/c3n.err; python -c "import json;d=json.load(open('gpurun_out/c3n.json'));print('new C3', d['value'], d['ms_per_step'])"; tail -3 gpurun_out/c3n.err
