# K1 v9 (lane256) vs v8 (octet) on 256-app traces: parity, then C3 timing
mkdir -p gpurun_out
exec > gpurun_out/l256.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "octet" 2>&1 | tail -3
for i in 1 2; do for k in octet lane256; do
  SGPU_K1=$k timeout 600 python bench.py --config C3 --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/c3.json 2> gpurun_out/c3.err
  python -c "import json;d=json.load(open('gpurun_out/c3.json'));print('$k', round(d['value']/1e6,3), 'M', round(d['ms_per_step'],2), 'ms')" || tail -5 gpurun_out/c3.err
done; done
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "C3" 2>&1 | tail -2
for i in 1 2; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/c2.json 2> gpurun_out/c2.err; python -c "import json;d=json.load(open('gpurun_out/c2.json'));print('tree C2', round(d['ms_per_step'],3))"
  SGPU_LIB=$PWD/build_ab/libsgpu_old.so timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/c2.json 2> gpurun_out/c2.err; python -c "import json;d=json.load(open('gpurun_out/c2.json'));print('old C2', round(d['ms_per_step'],3))"
done
